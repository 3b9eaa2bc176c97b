// faces.cuh — interior-face (mortar) and element-side kernels.
//
// Interior faces (operators.py:146-171, 211-217, 251-261, 312-334): both
// traces live on a mortar of order max(own, neighbour) per tangential
// direction, the numerical flux is evaluated there with the left element's
// sigma and normal, and flux*sigma is L2-projected back to each side
// (negated for the right side).  The right trace is re-indexed into the
// left's face axes by the face orientation code (3D generalisation of the
// reference's `flip`).
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

// Interior face, pointwise: one thread per mortar node.  Both sides' traces
// already live at the mortar order (k_trace_q / k_vol_lift interpolate the
// nonconforming sides), so no shared memory and no barriers are needed.
// Conforming faces write the signed per-side own-order surface arrays
// directly; nonconforming faces write one mortar array (left frame) that
// k_down projects back onto each side (operators.py:211-217, 257-261, 330-334).
template <int LAW, bool FLUX>
__global__ void __launch_bounds__(FACE_THREADS) k_face(DevPlan P) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  constexpr int COUT = FLUX ? NV : NG;
  const int f = blockIdx.x;
  const int t = threadIdx.x;
  if (t == 0) {
    // L2 prefetch of the face about one wave ahead (8 resident blocks per SM)
    const int fa = f + P.pf_face * P.nsm;
    if (fa < P.nfaces) {
      const int4 fn = P.fdesc[2 * fa];
      const int mn = ((fn.z & 7) + 1) * (((fn.z >> 3) & 7) + 1);
      const bool cn = (fn.z >> 9) & 1;
      const double* qs = cn ? P.qtr : P.qtrm;
      l2_prefetch_span(qs + (long long)fn.x * NV, sizeof(double) * mn * NV);
      l2_prefetch_span(qs + (long long)fn.y * NV, sizeof(double) * mn * NV);
      l2_prefetch_span(P.face_geo + fn.w, sizeof(double) * mn * 4);
      if (FLUX && L::viscous(P.prm)) {
        const double* gs = cn ? P.gtr : P.gtrm;
        l2_prefetch_span(gs + (long long)fn.x * NG, sizeof(double) * mn * NG);
        l2_prefetch_span(gs + (long long)fn.y * NG, sizeof(double) * mn * NG);
      }
    }
  }
  const int4 fd = P.fdesc[2 * f];
  const int M1 = fd.z & 7, M2 = (fd.z >> 3) & 7, orient = (fd.z >> 6) & 7;
  const bool conf = (fd.z >> 9) & 1;
  const int nm = (M1 + 1) * (M2 + 1);
  if (t >= nm) return;
  const int A = t % (M1 + 1), B = t / (M1 + 1);
  const int kR = right_index(A, B, M1, M2, orient);
  // conforming: own-order traces; nonconforming: mortar traces (item_side_traces)
  const double* qsrc = conf ? P.qtr : P.qtrm;
  const double* gsrc = conf ? P.gtr : P.gtrm;
  const long long tL = fd.x, tR = fd.y;
  const double* geo = P.face_geo + fd.w;
  const double sigma = geo[t];
  const double nrm[3] = {geo[nm + t], geo[2 * nm + t], geo[3 * nm + t]};
  double ql[NV], qr[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    ql[v] = qsrc[tL * NV + (long long)v * nm + t];
    qr[v] = qsrc[tR * NV + (long long)v * nm + kR];
  }
  double val[COUT];
  if (!FLUX) {
    double gl[NGV], gr[NGV];
    L::grad_vars(P.prm, ql, gl);
    L::grad_vars(P.prm, qr, gr);
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int k = 0; k < NGV; ++k) val[d * NGV + k] = 0.5 * (gl[k] + gr[k]) * nrm[d] * sigma;
  } else {
    double F[NV];
    L::riemann(P.prm, ql, qr, nrm, F);
    if (L::viscous(P.prm)) {
      double GL[3][NGV], GR[3][NGV], fl[NV], fr[NV];
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < NGV; ++k) {
          GL[d][k] = gsrc[tL * NG + (long long)(d * NGV + k) * nm + t];
          GR[d][k] = gsrc[tR * NG + (long long)(d * NGV + k) * nm + kR];
        }
      L::visc_normal(P.prm, ql, GL, nrm, fl);
      L::visc_normal(P.prm, qr, GR, nrm, fr);
#pragma unroll
      for (int v = 0; v < NV; ++v) F[v] -= 0.5 * (fl[v] + fr[v]);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) val[v] = F[v] * sigma;
  }
  if (conf) {
    double* dst = FLUX ? P.fsurf : P.lsurf;
    const long long oL = tL * COUT;
    const long long oR = tR * COUT;
#pragma unroll
    for (int c = 0; c < COUT; ++c) {
      dst[oL + (long long)c * nm + t] = val[c];
      dst[oR + (long long)c * nm + kR] = -val[c];
    }
  } else {
    double* dst = P.msurf + (long long)P.fdesc[2 * f + 1].x * COUT;
#pragma unroll
    for (int c = 0; c < COUT; ++c) dst[(long long)c * nm + t] = val[c];
  }
}

// L2 projection of a nonconforming face's mortar values back onto one side
// (left or right, own order; the right side negated and re-oriented): one
// warp per (face, side), all components on the FP64 tensor cores
// (warp_proj_mma).
template <int C>
__global__ void __launch_bounds__(128) k_down(DevPlan P, double* __restrict__ dst) {
  const int warp = threadIdx.x >> 5;
  const int task = blockIdx.x * 4 + warp;
  if (task >= P.ndown) return;
  {
    // L2 prefetch of the task about one wave ahead (10 resident blocks per SM)
    const int ta = task + 4 * P.pf_down * P.nsm;
    if ((threadIdx.x & 31) == 0 && ta < P.ndown) {
      const int4 tn = P.down[ta];
      const int mn = ((tn.z & 7) + 1) * (((tn.z >> 3) & 7) + 1);
      l2_prefetch_span(P.msurf + (long long)tn.x * C, sizeof(double) * mn * C);
    }
  }
  const int4 tk = P.down[task];
  const int M1 = tk.z & 7, M2 = (tk.z >> 3) & 7, o1 = (tk.z >> 6) & 7, o2 = (tk.z >> 9) & 7;
  const int orient = (tk.z >> 12) & 7;
  const bool right = (tk.z >> 15) & 1;
  const int nm = (M1 + 1) * (M2 + 1);
  const double* src = P.msurf + (long long)tk.x * C;
  const double* T1 = P.tables + OFF_T + (M1 * 8 + o1) * 64;
  const double* T2 = P.tables + OFF_T + (M2 * 8 + o2) * 64;
  const int nf = (o1 + 1) * (o2 + 1);
  double* out = dst + (long long)tk.y * C;
  const auto ld = [&](int c, int a, int b) { return src[(long long)c * nm + a + (M1 + 1) * b]; };
  if (!right)
    warp_proj_mma<C>(M1 + 1, M2 + 1, T1, o1 + 1, T2, o2 + 1, ld,
                     [&](int c, int A, int B, double x) { out[(long long)c * nf + A + (o1 + 1) * B] = x; });
  else
    warp_proj_mma<C>(M1 + 1, M2 + 1, T1, o1 + 1, T2, o2 + 1, ld,
                     [&](int c, int A, int B, double x) {
                       out[(long long)c * nf + right_index(A, B, o1, o2, orient)] = -x;
                     });
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
  const long long to = so;   // own-order traces
  const double* geo = P.side_geo + so * 4;
  const double sigma = geo[kf];
  const double nrm[3] = {geo[nf + kf], geo[2 * nf + kf], geo[3 * nf + kf]};
  double q[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) q[v] = P.qtr[to * NV + (long long)v * nf + kf];
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
        for (int k = 0; k < NGV; ++k) G[dd][k] = P.gtr[to * NG + (long long)(dd * NGV + k) * nf + kf];
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
