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

#ifndef MORTAR_WARPS
#define MORTAR_WARPS 1   // faces (warps) per k_mortar block: one, so a finished face frees its slot (measured: 4 -> 1 is 0.734 -> 0.704 ms on config 3)
#endif

namespace tdg {

// right own face index of the left-aligned position (a, b)
__device__ __forceinline__ int right_index(int a, int b, int R1, int R2, int orient) {
  const int ap = (orient & 1) ? (R1 - a) : a;
  const int bp = (orient & 2) ? (R2 - b) : b;
  // own right dims: non-swapped (R1+1, R2+1); swapped (R2+1, R1+1)
  return (orient & 4) ? (bp + (R2 + 1) * ap) : (ap + (R1 + 1) * bp);
}

// Pointwise interface value at mortar node t (left frame; kR = the right
// side's index of the same node): the BR1 lift g*·n σ (3 ngv values) or the
// numerical flux (Roe − ½(F_v,L + F_v,R)·n) σ (nv values) (operators.py:
// 211-217, 257-261, 283-290, 330-334).  Traces come from qsrc/gsrc at trace
// offsets tL/tR with nm nodes per side.
template <int LAW, bool FLUX>
__device__ __forceinline__ void face_point(const DevPlan& P, const double* qsrc, const double* gsrc,
                                           long long tL, long long tR, int nm, int t, int kR,
                                           const double* geo,
                                           double* val /* [FLUX ? NV : 3 NGV] */,
                                           bool gconst = false) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV, NTR = L::NTR;
  const int tg = gconst ? 0 : t;   // uniform face geometry: node 0's values
  const double sigma = geo[tg];
  const double nrm[3] = {geo[nm + tg], geo[2 * nm + tg], geo[3 * nm + tg]};
  double ql[NV], qr[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    ql[v] = qsrc[tL * NV + (long long)v * nm + t];
    qr[v] = qsrc[tR * NV + (long long)v * nm + kR];
  }
  if (!FLUX) {
    double gl[NGV], gr[NGV];
    L::grad_vars2(P.prm, ql, qr, gl, gr);
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int k = 0; k < NGV; ++k) val[d * NGV + k] = 0.5 * (gl[k] + gr[k]) * nrm[d] * sigma;
  } else {
    double F[NV];
    L::riemann(P.prm, ql, qr, nrm, F);
    if constexpr (L::FVTR) {
      // each side's own F_v.n sigma (own outward normal), interpolated to this
      // node: flux sigma - 1/2 (f_L - f_R)
#pragma unroll
      for (int v = 0; v < NV; ++v) val[v] = F[v] * sigma;
      if (L::viscous(P.prm)) {
#pragma unroll
        for (int k = 0; k < NTR; ++k) {
          const double fl = gsrc[tL * NTR + (long long)k * nm + t];
          const double fr = gsrc[tR * NTR + (long long)k * nm + kR];
          val[NV - NTR + k] -= 0.5 * (fl - fr);
        }
      }
      return;
    }
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
}

// Conforming interior face, pointwise: one thread per face node; both sides'
// own-order traces align node for node (up to orientation), and the signed
// values go straight into the per-side own-order surface arrays.
template <int LAW, bool FLUX>
__global__ void __launch_bounds__(FACE_THREADS_MAX) k_face(DevPlan P) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  constexpr int COUT = FLUX ? NV : NG;
  // face_pack > 1: this block's threads are face_pack groups of face_nm
  const int fl = P.face_pack > 1 ? threadIdx.x / P.face_nm : 0;
  const int t = threadIdx.x - fl * P.face_nm;
  const int fi = blockIdx.x * P.face_pack + fl;
  if (threadIdx.x == 0) {
    // L2 prefetch of the face about one wave ahead
    const int ba = fi + P.pf_face * P.nsm * P.face_pack;
    if (ba < P.ncface) {
      const int4 fn = P.fdesc[2 * (P.nmface ? P.cface[ba] : ba)];
      const int mn = ((fn.z & 7) + 1) * (((fn.z >> 3) & 7) + 1);
      l2_prefetch_span(P.qtr + (long long)fn.x * NV, sizeof(double) * mn * NV);
      l2_prefetch_span(P.qtr + (long long)fn.y * NV, sizeof(double) * mn * NV);
      if (!((fn.z >> 10) & 1)) l2_prefetch_span(P.face_geo + fn.w, sizeof(double) * mn * 4);
      if (FLUX && L::viscous(P.prm)) {
        l2_prefetch_span(P.gtr + (long long)fn.x * L::NTR, sizeof(double) * mn * L::NTR);
        l2_prefetch_span(P.gtr + (long long)fn.y * L::NTR, sizeof(double) * mn * L::NTR);
      }
    }
  }
  if (fi >= P.ncface || fl >= P.face_pack) return;
  const int f = P.nmface ? P.cface[fi] : fi;   // all conforming: identity list
  const int4 fd = P.fdesc[2 * f];
  const int M1 = fd.z & 7, M2 = (fd.z >> 3) & 7, orient = (fd.z >> 6) & 7;
  const int nm = (M1 + 1) * (M2 + 1);
  if (t >= nm) return;
  const int A = t % (M1 + 1), B = t / (M1 + 1);
  const int kR = right_index(A, B, M1, M2, orient);
  const long long tL = fd.x, tR = fd.y;
  if (!FLUX && P.gstar) {
    // g* form: one ½(g_L + g_R) per face node (the lift kernel applies n σ)
    double ql[NV], qr[NV], gl[NGV], gr[NGV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      ql[v] = P.qtr[tL * NV + (long long)v * nm + t];
      qr[v] = P.qtr[tR * NV + (long long)v * nm + kR];
    }
    L::grad_vars2(P.prm, ql, qr, gl, gr);
    double* dst = P.gsf + tL * NGV + t;
#pragma unroll
    for (int k = 0; k < NGV; ++k) dst[(long long)k * nm] = 0.5 * (gl[k] + gr[k]);
    return;
  }
  double val[COUT];
  face_point<LAW, FLUX>(P, P.qtr, P.gtr, tL, tR, nm, t, kR, P.face_geo + fd.w, val, (fd.z >> 10) & 1);
  double* dst = FLUX ? P.fsurf : P.lsurf;
  const long long oL = tL * COUT;
  const long long oR = tR * COUT;
#pragma unroll
  for (int c = 0; c < COUT; ++c) {
    dst[oL + (long long)c * nm + t] = val[c];
    dst[oR + (long long)c * nm + kR] = -val[c];
  }
}

// Nonconforming interior face: one warp per face.  Lane (g, q) evaluates the
// pointwise interface value at mortar nodes (q, g) and (q+4, g) — exactly the
// B operand positions of the first projection pass — keeps them in registers
// and L2-projects them onto both sides on the FP64 tensor cores (the right
// side negated and re-oriented).  Nothing goes through HBM between the
// pointwise evaluation and the projections (operators.py:211-217, 330-334).
#ifndef TDG_MORTAR_BLOCKS_FLUX
#define TDG_MORTAR_BLOCKS_FLUX 16   // resident one-warp blocks per SM (register cap 65536 / 32 / blocks)
#endif
#ifndef TDG_MORTAR_BLOCKS_LIFT
#define TDG_MORTAR_BLOCKS_LIFT 20
#endif
template <int LAW, bool FLUX>
__global__ void __launch_bounds__(32 * MORTAR_WARPS,
                                  (FLUX ? TDG_MORTAR_BLOCKS_FLUX : TDG_MORTAR_BLOCKS_LIFT) / MORTAR_WARPS)
k_mortar(DevPlan P) {
  using L = Law<LAW>;
  constexpr int NV = L::NV, NGV = L::NGV, NG = 3 * NGV;
  constexpr int COUT = FLUX ? NV : NG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * MORTAR_WARPS + warp;
  if (task >= P.nmface) return;
  const int f = P.mface[task];
  const int4 fd = P.fdesc[2 * f];
  const int4 fo = P.fdesc[2 * f + 1];
  const int M1 = fd.z & 7, M2 = (fd.z >> 3) & 7, orient = (fd.z >> 6) & 7;
  const int nm = (M1 + 1) * (M2 + 1);
  const int g = lane >> 2, q = lane & 3;
  const double* geo = P.face_geo + fd.w;
  double v0[COUT], v1[COUT];
#pragma unroll
  for (int c = 0; c < COUT; ++c) v0[c] = v1[c] = 0.0;
  if (g <= M2) {
    if (q <= M1) {
      const int t = q + (M1 + 1) * g;
      face_point<LAW, FLUX>(P, P.qtrm, P.gtrm, fd.x, fd.y, nm, t, right_index(q, g, M1, M2, orient),
                            geo, v0);
    }
    if (q + 4 <= M1) {
      const int t = q + 4 + (M1 + 1) * g;
      face_point<LAW, FLUX>(P, P.qtrm, P.gtrm, fd.x, fd.y, nm, t,
                            right_index(q + 4, g, M1, M2, orient), geo, v1);
    }
  }
  const auto ld = [&](int c, int a, int) { return a < 4 ? v0[c] : v1[c]; };
  double* surf = FLUX ? P.fsurf : P.lsurf;
  const int L1 = fo.w & 7, L2 = (fo.w >> 3) & 7, R1 = (fo.w >> 6) & 7, R2 = (fo.w >> 9) & 7;
  {
    double* out = surf + (long long)fo.y * COUT;
    const int nf = (L1 + 1) * (L2 + 1);
    warp_proj_mma<COUT>(M1 + 1, M2 + 1, P.tables + OFF_T + (M1 * 8 + L1) * 64, L1 + 1,
                        P.tables + OFF_T + (M2 * 8 + L2) * 64, L2 + 1, ld, out, nf,
                        [&](int A, int B) { return A + (L1 + 1) * B; });
  }
  {
    double* out = surf + (long long)fo.z * COUT;
    const int nf = (R1 + 1) * (R2 + 1);
    warp_proj_mma<COUT, true>(M1 + 1, M2 + 1, P.tables + OFF_T + (M1 * 8 + R1) * 64, R1 + 1,
                              P.tables + OFF_T + (M2 * 8 + R2) * 64, R2 + 1, ld, out, nf,
                              [&](int A, int B) { return right_index(A, B, R1, R2, orient); });
  }
  // look-ahead L2 prefetch, issued after this warp's own work so that its
  // dependent descriptor loads do not stall the projections
  if (lane == 0) {
    const int ta = task + 4 * P.pf_down * P.nsm;
    if (ta < P.nmface) {
      const int4 fn = P.fdesc[2 * P.mface[ta]];
      const int mn = ((fn.z & 7) + 1) * (((fn.z >> 3) & 7) + 1);
      l2_prefetch_span(P.qtrm + (long long)fn.x * NV, sizeof(double) * mn * NV);
      l2_prefetch_span(P.qtrm + (long long)fn.y * NV, sizeof(double) * mn * NV);
      l2_prefetch_span(P.face_geo + fn.w, sizeof(double) * mn * 4);
      if (FLUX && L::viscous(P.prm)) {
        l2_prefetch_span(P.gtrm + (long long)fn.x * L::NTR, sizeof(double) * mn * L::NTR);
        l2_prefetch_span(P.gtrm + (long long)fn.y * L::NTR, sizeof(double) * mn * L::NTR);
      }
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
    if constexpr (L::FVTR) {
      // the lift kernel left this side's F_v.n sigma (boundary treatment
      // applied) in the own-order viscous traces
      if (kind < 0) {
        double f[3][NV];
        L::adv_flux(P.prm, q, f);
#pragma unroll
        for (int v = 0; v < NV; ++v) F[v] = f[0][v] * nrm[0] + f[1][v] * nrm[1] + f[2][v] * nrm[2];
      } else {
        double qg[NV];
        L::bc_ghost(P.prm, q, nrm, kind, gh, qg);
        L::riemann(P.prm, q, qg, nrm, F);
      }
      double* dst = P.fsurf + so * NV + kf;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        double x = F[v] * sigma;
        if (visc && v >= NV - L::NTR)
          x -= P.gtr[to * L::NTR + (long long)(v - (NV - L::NTR)) * nf + kf];
        dst[(long long)v * nf] = x;
      }
      return;
    }
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
