// faces.cuh — interior-face (mortar) and element-side kernels.
//
// Interior faces (operators.py:146-171, 211-217, 251-261, 312-334): both
// traces are interpolated onto a mortar of order max(own, neighbour) per
// tangential direction, the numerical flux is evaluated there with the left
// element's sigma and normal, and flux*sigma is L2-projected back to each
// side (negated for the right side).  The right trace is re-indexed into the
// left's face axes by the face orientation code (3D generalisation of the
// reference's `flip`).  One 64-thread block per face; the separable 2D
// projections run through shared memory.
//
// Side kernels handle physical boundaries (coupled evaluation) and every
// element side in the isolated evaluation (operators.py:235-249, 294-310).
#pragma once
#include "common.cuh"
#include "laws.cuh"

namespace tdg {

// right own face index of the left-aligned position (a, b)
__device__ __forceinline__ int right_index(int a, int b, int R1, int R2, int orient) {
  const int ap = (orient & 1) ? (R1 - a) : a;
  const int bp = (orient & 2) ? (R2 - b) : b;
  // own right dims: non-swapped (R1+1, R2+1); swapped (R2+1, R1+1)
  return (orient & 4) ? (bp + (R2 + 1) * ap) : (ap + (R1 + 1) * bp);
}

// dst[c][A + ma*B] = sum_{a,b} T1[A][a] T2[B][b] src[c][a + na*b]   (stride 64 per c)
__device__ __forceinline__ void proj2(const double* src, int na, int nb, const double* T1,
                                      int ma, const double* T2, int mb, double* tmp, double* dst,
                                      int C) {
  for (int u = threadIdx.x; u < C * ma * nb; u += blockDim.x) {
    const int c = u / (ma * nb), r = u % (ma * nb), A = r % ma, b = r / ma;
    double acc = 0.0;
    for (int a = 0; a < na; ++a) acc += T1[A * 8 + a] * src[c * 64 + a + na * b];
    tmp[c * 64 + A + ma * b] = acc;
  }
  __syncthreads();
  for (int u = threadIdx.x; u < C * ma * mb; u += blockDim.x) {
    const int c = u / (ma * mb), r = u % (ma * mb), A = r % ma, B = r / ma;
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += T2[B * 8 + b] * tmp[c * 64 + A + ma * b];
    dst[c * 64 + A + ma * B] = acc;
  }
  __syncthreads();
}

template <int LAW, bool FLUX>
constexpr int face_smem_doubles() {
  constexpr int NV = Law<LAW>::NV, NG = 3 * Law<LAW>::NGV;
  constexpr int CIN = FLUX ? NV + NG : NV, COUT = FLUX ? NV : NG;
  constexpr int CM = CIN > COUT ? CIN : COUT;
  return 2 * CIN * 64 + 3 * CM * 64 + COUT * 64 + 8 * 64;
}

template <int LAW, bool FLUX>
__global__ void __launch_bounds__(FACE_THREADS) k_face(DevPlan P) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  constexpr int CIN = FLUX ? NV + NG : NV;      // trace components read per side
  constexpr int COUT = FLUX ? NV : NG;          // surface components written per side
  constexpr int CM = CIN > COUT ? CIN : COUT;   // mortar / projection buffers hold either
  extern __shared__ double fsm[];
  double* inL = fsm;
  double* inR = inL + CIN * 64;
  double* mL = inR + CIN * 64;
  double* mR = mL + CM * 64;
  double* tmp = mR + CM * 64;
  double* res = tmp + CM * 64;
  double(*Tm)[64] = reinterpret_cast<double(*)[64]>(res + COUT * 64);
  const int f = blockIdx.x;
  const int* fi = P.face_info + 12 * f;
  const int slotL = fi[0], sideL = fi[1], slotR = fi[2], sideR = fi[3], orient = fi[4];
  const int L1 = fi[5], L2 = fi[6], R1 = fi[7], R2 = fi[8], M1 = fi[9], M2 = fi[10];
  const int nL = (L1 + 1) * (L2 + 1), nR = (R1 + 1) * (R2 + 1), nm = (M1 + 1) * (M2 + 1);
  const bool visc = L::viscous(P.prm);
  const int cin = (FLUX && visc) ? CIN : NV;
  const bool conf = (L1 == M1) && (L2 == M2) && (R1 == M1) && (R2 == M2);
  const long long offL = P.side_off[slotL * 6 + sideL];
  const long long offR = P.side_off[slotR * 6 + sideR];

  if (!conf) {
    // up: L->M (dirs 1,2), R->M ; down: M->L, M->R
    const int fr[8] = {L1, L2, R1, R2, M1, M2, M1, M2};
    const int to[8] = {M1, M2, M1, M2, L1, L2, R1, R2};
    for (int u = threadIdx.x; u < 8 * 64; u += blockDim.x) {
      const int k = u / 64;
      Tm[k][u % 64] = P.tables[OFF_T + (fr[k] * 8 + to[k]) * 64 + (u % 64)];
    }
  }
  // load traces (left own, right re-indexed into left axes)
  for (int u = threadIdx.x; u < cin * 64; u += blockDim.x) {
    const int c = u / 64, k = u % 64;
    if (k < nL) {
      inL[u] = (c < NV) ? P.qtr[offL * NV + (long long)c * nL + k]
                        : P.gtr[offL * NG + (long long)(c - NV) * nL + k];
    }
    if (k < nR) {
      const int a = k % (R1 + 1), b = k / (R1 + 1);
      const int kr = right_index(a, b, R1, R2, orient);
      inR[u] = (c < NV) ? P.qtr[offR * NV + (long long)c * nR + kr]
                        : P.gtr[offR * NG + (long long)(c - NV) * nR + kr];
    }
  }
  __syncthreads();
  const double* qL = inL;
  const double* qR = inR;
  if (!conf) {
    proj2(inL, L1 + 1, L2 + 1, Tm[0], M1 + 1, Tm[1], M2 + 1, tmp, mL, cin);
    proj2(inR, R1 + 1, R2 + 1, Tm[2], M1 + 1, Tm[3], M2 + 1, tmp, mR, cin);
    qL = mL;
    qR = mR;
  }
  // pointwise mortar flux
  const int t = threadIdx.x;
  if (t < nm) {
    const double* geo = P.face_geo + P.face_geo_off[f];
    const double sigma = geo[t];
    const double nrm[3] = {geo[nm + t], geo[2 * nm + t], geo[3 * nm + t]};
    double ql[NV], qr[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      ql[v] = qL[v * 64 + t];
      qr[v] = qR[v * 64 + t];
    }
    if (!FLUX) {
      double gl[NGV], gr[NGV];
      L::grad_vars(P.prm, ql, gl);
      L::grad_vars(P.prm, qr, gr);
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < NGV; ++k)
          res[(d * NGV + k) * 64 + t] = 0.5 * (gl[k] + gr[k]) * nrm[d] * sigma;
    } else {
      double F[NV];
      L::riemann(P.prm, ql, qr, nrm, F);
      if (visc) {
        double GL[3][NGV], GR[3][NGV], fl[NV], fr2[NV];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int k = 0; k < NGV; ++k) {
            GL[d][k] = qL[(NV + d * NGV + k) * 64 + t];
            GR[d][k] = qR[(NV + d * NGV + k) * 64 + t];
          }
        L::visc_normal(P.prm, ql, GL, nrm, fl);
        L::visc_normal(P.prm, qr, GR, nrm, fr2);
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] -= 0.5 * (fl[v] + fr2[v]);
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) res[v * 64 + t] = F[v] * sigma;
    }
  }
  __syncthreads();
  const double* oL = res;
  const double* oR = res;
  if (!conf) {
    proj2(res, M1 + 1, M2 + 1, Tm[4], L1 + 1, Tm[5], L2 + 1, tmp, mL, COUT);
    proj2(res, M1 + 1, M2 + 1, Tm[6], R1 + 1, Tm[7], R2 + 1, tmp, mR, COUT);
    oL = mL;
    oR = mR;
  }
  double* dst = FLUX ? P.fsurf : P.lsurf;
  for (int u = threadIdx.x; u < COUT * 64; u += blockDim.x) {
    const int c = u / 64, k = u % 64;
    if (k < nL) dst[offL * COUT + (long long)c * nL + k] = oL[u];
    if (k < nR) {
      const int a = k % (R1 + 1), b = k / (R1 + 1);
      const int kr = right_index(a, b, R1, R2, orient);
      dst[offR * COUT + (long long)c * nR + kr] = -oR[u];
    }
  }
}

// Side kernel: item = (slot, side, kind [-1 = isolated], ghost offset).
template <int LAW, bool FLUX>
__global__ void __launch_bounds__(SIDE_THREADS) k_side(DevPlan P, const int4* __restrict__ items,
                                                      int nitems) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  const int it = blockIdx.x * SIDES_PER_BLOCK + threadIdx.x / 64;
  const int kf = threadIdx.x % 64;
  if (it >= nitems) return;
  const int4 w = items[it];
  const int slot = w.x, side = w.y, kind = w.z;
  const int* od = P.orders + 3 * slot;
  int d, a, b;
  side_dirs(side, d, a, b);
  const int nf = (od[a] + 1) * (od[b] + 1);
  if (kf >= nf) return;
  const long long so = P.side_off[slot * 6 + side];
  const double* geo = P.side_geo + so * 4;
  const double sigma = geo[kf];
  const double nrm[3] = {geo[nf + kf], geo[2 * nf + kf], geo[3 * nf + kf]};
  double q[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) q[v] = P.qtr[so * NV + (long long)v * nf + kf];
  double gh[NV];
  if (kind >= 0) {
    // ghost offset (doubles); negative: the BC needs no ghost array
    if (w.w >= 0) {
      const double* gp = P.ghost + w.w;
#pragma unroll
      for (int v = 0; v < NV; ++v) gh[v] = gp[(long long)v * nf + kf];
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) gh[v] = q[v];
    }
  }
  if (!FLUX) {
    double g[NGV];
    if (kind < 0)
      L::grad_vars(P.prm, q, g);
    else
      L::bc_lift(P.prm, q, nrm, kind, gh, g);
    double* dst = P.lsurf + so * NG + kf;
#pragma unroll
    for (int dd = 0; dd < 3; ++dd)
#pragma unroll
      for (int k = 0; k < NGV; ++k) dst[(long long)(dd * NGV + k) * nf] = g[k] * nrm[dd] * sigma;
  } else {
    const bool visc = L::viscous(P.prm);
    double F[NV];
    double G[3][NGV];
    if (visc) {
#pragma unroll
      for (int dd = 0; dd < 3; ++dd)
#pragma unroll
        for (int k = 0; k < NGV; ++k) G[dd][k] = P.gtr[so * NG + (long long)(dd * NGV + k) * nf + kf];
    }
    if (kind < 0) {
      double f[3][NV];
      L::adv_flux(P.prm, q, f);
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] = f[0][v] * nrm[0] + f[1][v] * nrm[1] + f[2][v] * nrm[2];
      if (visc) {
        double fv[NV];
        L::visc_normal(P.prm, q, G, nrm, fv);
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] -= fv[v];
      }
    } else {
      double qg[NV];
      L::bc_ghost(P.prm, q, nrm, kind, gh, qg);
      L::riemann(P.prm, q, qg, nrm, F);
      if (visc) {
        double fv[NV];
        L::bc_visc_normal(P.prm, q, G, nrm, kind, fv);
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] -= fv[v];
      }
    }
    double* dst = P.fsurf + so * NV + kf;
#pragma unroll
    for (int v = 0; v < NV; ++v) dst[(long long)v * nf] = F[v] * sigma;
  }
}

}  // namespace tdg
