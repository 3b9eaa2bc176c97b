// transfer.cuh — p-transfers between order fields as batched separable
// tensor-product contractions (multigrid.py:101-143; fields.py:165-181).
//
// A work item is a run of elements sharing (source orders, target orders).
// The source block is staged in shared memory and contracted one direction at
// a time (x, then y, then z) with the 1D transfer matrices; the restriction is
// the L2 projection, prolongation the interpolation (spectral tables).
#pragma once
#include "common.cuh"

namespace tdg {

enum { TR_RESTRICT = 0, TR_PROLONG = 1, TR_PROLONG_ADD = 2 };

struct DevTransfer {
  const double* tables;
  int nv;
  const int* f_orders;
  const long long* f_node_off;
  const int* c_orders;
  const long long* c_node_off;
  const int* c_slot_of_f;   // coarse slot of each fine slot
  const int2* work;         // (first fine slot, count)
};

// NVC > 0, NSC > 0, NDC > 0: compile-time component count and isotropic
// source / target point counts (the uniform p-multigrid level pairs), so the
// index arithmetic of every pass folds to constant divisors; otherwise all
// runtime.
template <int MODE, int NVC = -1, int NSC = -1, int NDC = -1>
__global__ void __launch_bounds__(ELEM_THREADS) k_transfer(DevTransfer T, const double* __restrict__ in,
                                                           const double* __restrict__ in2,
                                                           double* __restrict__ out) {
  extern __shared__ double sm[];
  __shared__ double mat[3][64];
  const int2 wi = T.work[blockIdx.x];
  const int fs0 = wi.x;
  const int cs0 = T.c_slot_of_f[fs0];
  const int* fo = T.f_orders + 3 * fs0;
  const int* co = T.c_orders + 3 * cs0;
  const bool down = (MODE == TR_RESTRICT);
  int sn[3], dn[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    sn[d] = NSC > 0 ? NSC : (down ? fo[d] : co[d]) + 1;
    dn[d] = NDC > 0 ? NDC : (down ? co[d] : fo[d]) + 1;
  }
  for (int u = threadIdx.x; u < 3 * 64; u += blockDim.x) {
    const int d = u / 64;
    mat[d][u % 64] = T.tables[OFF_T + ((sn[d] - 1) * 8 + (dn[d] - 1)) * 64 + (u % 64)];
  }
  const int nv = NVC > 0 ? NVC : T.nv;
  const int ns = sn[0] * sn[1] * sn[2], nd = dn[0] * dn[1] * dn[2];
  const int s1 = dn[0] * sn[1] * sn[2], s2 = dn[0] * dn[1] * sn[2];
  int mx = ns > nd ? ns : nd;
  mx = mx > s1 ? mx : s1;
  mx = mx > s2 ? mx : s2;
  const int E = wi.y;
  double* b0 = sm;                    // [E][nv][mx]
  double* b1 = sm + E * nv * mx;
  // stage source
  for (int u = threadIdx.x; u < E * nv * ns; u += blockDim.x) {
    const int e = u / (nv * ns), r = u % (nv * ns);
    const int fs = fs0 + e;
    const int cs = T.c_slot_of_f[fs];
    double x;
    if (down) {
      x = in[T.f_node_off[fs] * nv + r];
    } else {
      const long long ix = T.c_node_off[cs] * nv + r;
      x = in[ix];
      if (MODE == TR_PROLONG_ADD && in2) x -= in2[ix];
    }
    b0[(e * nv + r / ns) * mx + (r % ns)] = x;
  }
  __syncthreads();
  // x pass: b1[a + d0*(j + s1y*k)] = sum_i M0[a][i] b0[i + s0*(j + s1y*k)]
  for (int u = threadIdx.x; u < E * nv * s1; u += blockDim.x) {
    const int ev = u / s1, r = u % s1;
    const int a = r % dn[0], jk = r / dn[0];
    const double* src = b0 + ev * mx + jk * sn[0];
    double acc = 0.0;
    for (int i = 0; i < sn[0]; ++i) acc += mat[0][a * 8 + i] * src[i];
    b1[ev * mx + r] = acc;
  }
  __syncthreads();
  // y pass
  for (int u = threadIdx.x; u < E * nv * s2; u += blockDim.x) {
    const int ev = u / s2, r = u % s2;
    const int a = r % dn[0], b = (r / dn[0]) % dn[1], k = r / (dn[0] * dn[1]);
    const double* src = b1 + ev * mx + a + dn[0] * sn[1] * k;
    double acc = 0.0;
    for (int j = 0; j < sn[1]; ++j) acc += mat[1][b * 8 + j] * src[dn[0] * j];
    b0[ev * mx + r] = acc;
  }
  __syncthreads();
  // z pass + store
  for (int u = threadIdx.x; u < E * nv * nd; u += blockDim.x) {
    const int ev = u / nd, r = u % nd;
    const int e = ev / nv, v = ev % nv;
    const int ab = r % (dn[0] * dn[1]), c = r / (dn[0] * dn[1]);
    const double* src = b0 + ev * mx + ab;
    double acc = 0.0;
    for (int k = 0; k < sn[2]; ++k) acc += mat[2][c * 8 + k] * src[dn[0] * dn[1] * k];
    const int fs = fs0 + e;
    if (down) {
      const int cs = T.c_slot_of_f[fs];
      out[T.c_node_off[cs] * nv + (long long)v * nd + r] = acc;
    } else if (MODE == TR_PROLONG_ADD) {
      out[T.f_node_off[fs] * nv + (long long)v * nd + r] += acc;
    } else {
      out[T.f_node_off[fs] * nv + (long long)v * nd + r] = acc;
    }
  }
}

}  // namespace tdg
