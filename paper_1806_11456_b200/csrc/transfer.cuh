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

#ifndef TDG_TRANSFER_BLOCKS
#define TDG_TRANSFER_BLOCKS 5   // <= 51 registers (measured best with 2 outputs per line at a time)
#endif
#ifndef TDG_TRANSFER_UNROLL
#define TDG_TRANSFER_UNROLL 2   // outputs per line computed together (ILP vs registers)
#endif
constexpr int kTransferUnroll = TDG_TRANSFER_UNROLL;

// Uniform isotropic level pairs (every fine element NS^3 -> NS^3 points, every
// coarse element ND^3 <-> ...) whose work items are runs of consecutive slots
// on both levels (checked at transfer creation): the item's source span is
// one contiguous range, loaded with independent unrolled loads (PROLONG_ADD:
// Q_c - Q_c0 formed on the fly); each pass is one 1D line per thread, held in
// registers (NS loads -> ND outputs), instead of one output per thread
// re-reading the line.  Same per-output summation order as k_transfer.
// Block size: the N=7 <-> 6 pairs (one element per item) have 320, 280 and
// 245 lines in their three passes, so 320 threads run each pass in one round
// (256 need two rounds for two of them); other pairs use 256.
template <int NS, int ND>
__host__ __device__ constexpr int transfer_lines_threads() { return (NS == 8 || ND == 8) ? 320 : ELEM_THREADS; }

template <int MODE, int NVC, int NS, int ND>
__global__ void __launch_bounds__(transfer_lines_threads<NS, ND>(),
                                  TDG_TRANSFER_BLOCKS * ELEM_THREADS / transfer_lines_threads<NS, ND>())
    k_transfer_lines(DevTransfer T, const double* __restrict__ in,
                                                                 const double* __restrict__ in2,
                                                                 double* __restrict__ out) {
  extern __shared__ double sm[];
  __shared__ double mat[64];
  constexpr bool down = MODE == TR_RESTRICT;
  constexpr int ns = NS * NS * NS, nd = ND * ND * ND;
  constexpr int S1 = ND * NS * NS, S2 = ND * ND * NS;
  constexpr int MA = ns > S2 ? ns : S2, MB = S1;
  constexpr int NT = transfer_lines_threads<NS, ND>();
  constexpr int R = (MAXN * NVC + NT - 1) / NT;
  const int2 wi = T.work[blockIdx.x];
  const int fs0 = wi.x, E = wi.y;
  const int cs0 = T.c_slot_of_f[fs0];
  const long long fb = T.f_node_off[fs0] * NVC, cb = T.c_node_off[cs0] * NVC;
  // stage the source: E * NVC * ns contiguous values
  const long long ib = down ? fb : cb;
  const int tot = E * NVC * ns;
  double x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int u = threadIdx.x + r * NT;
    if (u < tot) {
      x[r] = in[ib + u];
      if (MODE == TR_PROLONG_ADD && in2) x[r] -= in2[ib + u];
    }
  }
  for (int u = threadIdx.x; u < 64; u += blockDim.x)
    mat[u] = T.tables[OFF_T + ((NS - 1) * 8 + (ND - 1)) * 64 + u];
  double* A = sm;                      // [E*NVC][MA]
  double* B = sm + E * NVC * MA;       // [E*NVC][MB]
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int u = threadIdx.x + r * NT;
    if (u < tot) A[(u / ns) * MA + u % ns] = x[r];
  }
  __syncthreads();
  // x pass: lines (ev, jk) -> B[ev][a + ND * jk]
  for (int L = threadIdx.x; L < E * NVC * NS * NS; L += blockDim.x) {
    const int ev = L / (NS * NS), jk = L % (NS * NS);
    const double* src = A + ev * MA + jk * NS;
    double v[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) v[i] = src[i];
    double* dst = B + ev * MB + jk * ND;
#pragma unroll kTransferUnroll
    for (int a = 0; a < ND; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < NS; ++i) acc += mat[a * 8 + i] * v[i];
      dst[a] = acc;
    }
  }
  __syncthreads();
  // y pass: lines (ev, a, k) -> A[ev][a + ND * (b + ND * k)]
  for (int L = threadIdx.x; L < E * NVC * ND * NS; L += blockDim.x) {
    const int ev = L / (ND * NS), r = L % (ND * NS);
    const int a = r % ND, k = r / ND;
    const double* src = B + ev * MB + a + ND * NS * k;
    double v[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) v[j] = src[ND * j];
    double* dst = A + ev * MA + a + ND * ND * k;
#pragma unroll kTransferUnroll
    for (int b = 0; b < ND; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NS; ++j) acc += mat[b * 8 + j] * v[j];
      dst[ND * b] = acc;
    }
  }
  __syncthreads();
  // z pass + store: lines (ev, ab) -> out[e][v][ab + ND^2 c]
  const long long ob = down ? cb : fb;
  for (int L = threadIdx.x; L < E * NVC * ND * ND; L += blockDim.x) {
    const int ev = L / (ND * ND), ab = L % (ND * ND);
    const double* src = A + ev * MA + ab;
    double v[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) v[k] = src[ND * ND * k];
    double* dst = out + ob + (long long)ev * nd + ab;
#pragma unroll kTransferUnroll
    for (int c = 0; c < ND; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < NS; ++k) acc += mat[c * 8 + k] * v[k];
      if (MODE == TR_PROLONG_ADD)
        dst[ND * ND * c] += acc;
      else
        dst[ND * ND * c] = acc;
    }
  }
}

}  // namespace tdg
