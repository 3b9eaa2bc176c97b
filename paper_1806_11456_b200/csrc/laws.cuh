// laws.cuh — pointwise physics in registers (FP64).
//
// Scalar laws restate /root/reference/pkg/src/taudg/physics.py:49-88 in 3D;
// Navier-Stokes follows PAPER.md:744-816 with the choices of DESIGN.md
// (mu = 1 non-dimensional, BR1 on (u, v, w, T), Roe flux without entropy fix,
// mean-of-sides interface viscous flux).  Parameters (plan prm[8]):
//   advdiff: a, b, c, mu        burgers: bx, by, bz, mu
//   NS:      gamma, Pr, M, Re (Re = 0: inviscid), [4] = 1/Re, [5] = 1/((gamma-1) Pr M^2)   prm[7] = mu_cfl
#pragma once
#include "common.cuh"

namespace tdg {

enum { LAW_ADVDIFF = 0, LAW_BURGERS = 1, LAW_NS = 2 };
enum { BC_DIRICHLET = 0, BC_FREESTREAM = 1, BC_WALL = 2, BC_SYMMETRY = 3 };

template <int LAW>
struct Law;

// ---------------------------------------------------------------------------
template <>
struct Law<LAW_ADVDIFF> {
  static constexpr int NV = 1, NGV = 1;
  // side traces of the viscous term: the gradient itself, taken to the mortar
  // as the reference does (operators.py:318-329)
  static constexpr bool FVTR = false;
  static constexpr int NTR = 3 * NGV;
  __device__ static bool viscous(const double* P) { return P[3] > 0.0; }
  __device__ static void grad_vars(const double*, const double* q, double* g) { g[0] = q[0]; }
  __device__ static void grad_vars2(const double*, const double* ql, const double* qr, double* gl,
                                    double* gr) {
    gl[0] = ql[0];
    gr[0] = qr[0];
  }
  __device__ static void adv_flux(const double* P, const double* q, double f[3][NV]) {
    f[0][0] = P[0] * q[0];
    f[1][0] = P[1] * q[0];
    f[2][0] = P[2] * q[0];
  }
  // f -= mu grad q   (operators.py:284-287)
  __device__ static void sub_visc(const double* P, const double*, const double G[3][NGV],
                                  double f[3][NV]) {
    f[0][0] -= P[3] * G[0][0];
    f[1][0] -= P[3] * G[1][0];
    f[2][0] -= P[3] * G[2][0];
  }
  __device__ static void visc_normal(const double* P, const double*, const double G[3][NGV],
                                     const double* n, double* out) {
    out[0] = P[3] * (G[0][0] * n[0] + G[1][0] * n[1] + G[2][0] * n[2]);
  }
  __device__ static void side_visc(const double*, const double*, const double[3][NGV], const double*,
                                   double, int, double*) {}
  __device__ static double wave_speed(const double* P, const double*) {
    return sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]);
  }
  __device__ static void riemann(const double* P, const double* ql, const double* qr,
                                 const double* n, double* F) {
    const double an = P[0] * n[0] + P[1] * n[1] + P[2] * n[2];
    F[0] = 0.5 * an * (ql[0] + qr[0]) + 0.5 * fabs(an) * (ql[0] - qr[0]);
  }
  __device__ static void bc_ghost(const double*, const double*, const double*, int,
                                  const double* ghost, double* qg) { qg[0] = ghost[0]; }
  __device__ static void bc_lift(const double*, const double*, const double*, int,
                                 const double* ghost, double* g) { g[0] = ghost[0]; }
  __device__ static void bc_visc_normal(const double* P, const double* q, const double G[3][NGV],
                                        const double* n, int, double* out) {
    visc_normal(P, q, G, n, out);
  }
};

// ---------------------------------------------------------------------------
template <>
struct Law<LAW_BURGERS> {
  static constexpr int NV = 1, NGV = 1;
  // side traces of the viscous term: the gradient itself, taken to the mortar
  // as the reference does (operators.py:318-329)
  static constexpr bool FVTR = false;
  static constexpr int NTR = 3 * NGV;
  __device__ static bool viscous(const double* P) { return P[3] > 0.0; }
  __device__ static void grad_vars(const double*, const double* q, double* g) { g[0] = q[0]; }
  __device__ static void grad_vars2(const double*, const double* ql, const double* qr, double* gl,
                                    double* gr) {
    gl[0] = ql[0];
    gr[0] = qr[0];
  }
  __device__ static void adv_flux(const double* P, const double* q, double f[3][NV]) {
    const double h = 0.5 * q[0] * q[0];
    f[0][0] = P[0] * h;
    f[1][0] = P[1] * h;
    f[2][0] = P[2] * h;
  }
  __device__ static void sub_visc(const double* P, const double*, const double G[3][NGV],
                                  double f[3][NV]) {
    f[0][0] -= P[3] * G[0][0];
    f[1][0] -= P[3] * G[1][0];
    f[2][0] -= P[3] * G[2][0];
  }
  __device__ static void visc_normal(const double* P, const double*, const double G[3][NGV],
                                     const double* n, double* out) {
    out[0] = P[3] * (G[0][0] * n[0] + G[1][0] * n[1] + G[2][0] * n[2]);
  }
  __device__ static void side_visc(const double*, const double*, const double[3][NGV], const double*,
                                   double, int, double*) {}
  __device__ static double wave_speed(const double* P, const double* q) {
    return sqrt(P[0] * P[0] + P[1] * P[1] + P[2] * P[2]) * fabs(q[0]);
  }
  // Rusanov with lambda = max(|ql|, |qr|)  (physics.py:83-88)
  __device__ static void riemann(const double* P, const double* ql, const double* qr,
                                 const double* n, double* F) {
    const double bn = P[0] * n[0] + P[1] * n[1] + P[2] * n[2];
    const double lam = fmax(fabs(ql[0]), fabs(qr[0]));
    F[0] = 0.25 * (ql[0] * ql[0] + qr[0] * qr[0]) * bn - 0.5 * lam * (qr[0] - ql[0]);
  }
  __device__ static void bc_ghost(const double*, const double*, const double*, int,
                                  const double* ghost, double* qg) { qg[0] = ghost[0]; }
  __device__ static void bc_lift(const double*, const double*, const double*, int,
                                 const double* ghost, double* g) { g[0] = ghost[0]; }
  __device__ static void bc_visc_normal(const double* P, const double* q, const double G[3][NGV],
                                        const double* n, int, double* out) {
    visc_normal(P, q, G, n, out);
  }
};

// ---------------------------------------------------------------------------
template <>
struct Law<LAW_NS> {
  static constexpr int NV = 5, NGV = 4;
  // side traces of the viscous term: each side's own normal viscous flux
  // F_v.n sigma (components 1..4; the mass equation has none), evaluated at the
  // side's own face nodes and averaged on the mortar (oracle/physics.py
  // NavierStokes.side_flux_traces; DESIGN.md §3 decision 3)
  static constexpr bool FVTR = true;
  static constexpr int NTR = 4;
  __device__ static bool viscous(const double* P) { return P[3] > 0.0; }

  // ir = 1 / rho is formed once per state and reused wherever the oracle
  // divides by rho (one FP64 division is ~20 instructions)
  __device__ static void prim(const double* P, const double* q, double& rho, double& u,
                              double& v, double& w, double& p, double& ir) {
    rho = q[0];
    ir = 1.0 / rho;
    u = q[1] * ir;
    v = q[2] * ir;
    w = q[3] * ir;
    p = (P[0] - 1.0) * (q[4] - 0.5 * rho * (u * u + v * v + w * w));
  }
  __device__ static void prim(const double* P, const double* q, double& rho, double& u,
                              double& v, double& w, double& p) {
    double ir;
    prim(P, q, rho, u, v, w, p, ir);
  }
  __device__ static void grad_vars(const double* P, const double* q, double* g) {
    double rho, u, v, w, p, ir;
    prim(P, q, rho, u, v, w, p, ir);
    g[0] = u;
    g[1] = v;
    g[2] = w;
    g[3] = P[0] * P[2] * P[2] * p * ir;
  }
  // lifted variables of the two states of a face node, one division for both
  __device__ static void grad_vars2(const double* P, const double* ql, const double* qr, double* gl,
                                    double* gr) {
    const double rl = ql[0], rr = qr[0];
    const double tinv = 1.0 / (rl * rr);
    const double irl = tinv * rr, irr = tinv * rl;
    const double c = P[0] * P[2] * P[2], gm1 = P[0] - 1.0;
    gl[0] = ql[1] * irl;
    gl[1] = ql[2] * irl;
    gl[2] = ql[3] * irl;
    gl[3] = c * (gm1 * (ql[4] - 0.5 * rl * (gl[0] * gl[0] + gl[1] * gl[1] + gl[2] * gl[2]))) * irl;
    gr[0] = qr[1] * irr;
    gr[1] = qr[2] * irr;
    gr[2] = qr[3] * irr;
    gr[3] = c * (gm1 * (qr[4] - 0.5 * rr * (gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2]))) * irr;
  }
  __device__ static void adv_flux(const double* P, const double* q, double f[3][NV]) {
    double rho, u, v, w, p;
    prim(P, q, rho, u, v, w, p);
    const double H = q[4] + p;
    const double vel[3] = {u, v, w};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double vd = vel[d];
      f[d][0] = q[0] * vd;
      f[d][1] = q[1] * vd;
      f[d][2] = q[2] * vd;
      f[d][3] = q[3] * vd;
      f[d][1 + d] += p;
      f[d][4] = vd * H;
    }
  }
  // viscous flux (1/Re)[0, tau_d., u.tau_d + kappa T_d] in direction d
  __device__ static void visc_dir(const double* P, double u, double v, double w,
                                  const double G[3][NGV], int d, double* fv) {
    const double inv_re = P[4];   // 1 / Re and 1 / ((gamma - 1) Pr M^2), set by tdg_plan_create
    const double kappa = P[5];
    const double div = G[0][0] + G[1][1] + G[2][2];
    double tau[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double t = G[d][i] + G[i][d];
      if (i == d) t -= (2.0 / 3.0) * div;
      tau[i] = t;
    }
    fv[0] = 0.0;
    fv[1] = inv_re * tau[0];
    fv[2] = inv_re * tau[1];
    fv[3] = inv_re * tau[2];
    fv[4] = inv_re * (u * tau[0] + v * tau[1] + w * tau[2] + kappa * G[d][3]);
  }
  __device__ static void sub_visc(const double* P, const double* q, const double G[3][NGV],
                                  double f[3][NV]) {
    double rho, u, v, w, p;
    prim(P, q, rho, u, v, w, p);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double fv[5];
      visc_dir(P, u, v, w, G, d, fv);
#pragma unroll
      for (int k = 0; k < 5; ++k) f[d][k] -= fv[k];
    }
  }
  __device__ static void visc_normal(const double* P, const double* q, const double G[3][NGV],
                                     const double* n, double* out) {
    double rho, u, v, w, p;
    prim(P, q, rho, u, v, w, p);
#pragma unroll
    for (int k = 0; k < 5; ++k) out[k] = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double fv[5];
      visc_dir(P, u, v, w, G, d, fv);
#pragma unroll
      for (int k = 0; k < 5; ++k) out[k] += n[d] * fv[k];
    }
  }
  // F_v.n sigma at a side's own face node (oracle NavierStokes.side_visc_normal
  // times sigma) from the traces gv of (u, v, w, T) and G of their gradient;
  // kind < 0: interior or isolated side, else the boundary treatment of
  // bc_visc_normal.  out[k] = component 1 + k.
  __device__ static void side_visc(const double* P, const double* gv, const double G[3][NGV],
                                   const double* n, double sigma, int kind, double* out) {
    if (kind == BC_SYMMETRY) {
#pragma unroll
      for (int k = 0; k < NTR; ++k) out[k] = 0.0;
      return;
    }
    const bool wall = kind == BC_WALL;
    const double u = wall ? 0.0 : gv[0], v = wall ? 0.0 : gv[1], w = wall ? 0.0 : gv[2];
    double Gw[3][NGV];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      Gw[d][0] = G[d][0];
      Gw[d][1] = G[d][1];
      Gw[d][2] = G[d][2];
      Gw[d][3] = wall ? 0.0 : G[d][3];
    }
    double acc[NTR];
#pragma unroll
    for (int k = 0; k < NTR; ++k) acc[k] = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double fv[5];
      visc_dir(P, u, v, w, Gw, d, fv);
#pragma unroll
      for (int k = 0; k < NTR; ++k) acc[k] += n[d] * fv[1 + k];
    }
#pragma unroll
    for (int k = 0; k < NTR; ++k) out[k] = acc[k] * sigma;
  }
  __device__ static double wave_speed(const double* P, const double* q) {
    double rho, u, v, w, p;
    prim(P, q, rho, u, v, w, p);
    return sqrt(u * u + v * v + w * w) + sqrt(P[0] * p / rho);
  }
  // Roe flux, no entropy fix (oracle/physics.py NavierStokes.riemann)
  __device__ static void riemann(const double* P, const double* ql, const double* qr,
                                 const double* n, double* F) {
    const double g = P[0];
    // One division, one square root and one rsqrt serve the whole flux: with
    // rt = sqrt(rho_l rho_r) the Roe weights are rho_l : rt (sqrt(rho_l) taken
    // out of numerator and denominator), 1/rho_l, 1/rho_r and 1/(rho_l + rt)
    // come from the reciprocal of their product, and c, 1/c^2 from rsqrt(c^2)
    // (an FP64 division or square root is 20-25 instructions).
    const double rl = ql[0], rr = qr[0];
    const double rt = sqrt(rl * rr);
    const double den = rl + rt;
    const double lr = rl * rr;
    const double tinv = 1.0 / (lr * den);
    const double irl = tinv * (rr * den), irr = tinv * (rl * den), inv = tinv * lr;
    const double ul = ql[1] * irl, vl = ql[2] * irl, wl = ql[3] * irl;
    const double ur = qr[1] * irr, vr = qr[2] * irr, wr = qr[3] * irr;
    const double pl = (g - 1.0) * (ql[4] - 0.5 * rl * (ul * ul + vl * vl + wl * wl));
    const double pr = (g - 1.0) * (qr[4] - 0.5 * rr * (ur * ur + vr * vr + wr * wr));
    const double nx = n[0], ny = n[1], nz = n[2];
    const double vnl = ul * nx + vl * ny + wl * nz;
    const double vnr = ur * nx + vr * ny + wr * nz;
    const double Hr = (qr[4] + pr) * irr;
    const double ut = (ql[1] + rt * ur) * inv;
    const double vt = (ql[2] + rt * vr) * inv;
    const double wt = (ql[3] + rt * wr) * inv;
    const double Ht = ((ql[4] + pl) + rt * Hr) * inv;
    const double q2 = ut * ut + vt * vt + wt * wt;
    const double c2 = (g - 1.0) * (Ht - 0.5 * q2);
    const double ic = rsqrt(c2);
    const double ct = c2 * ic;
    const double vnt = ut * nx + vt * ny + wt * nz;
    const double drho = rr - rl, dp = pr - pl;
    const double du = ur - ul, dv = vr - vl, dw = wr - wl;
    const double dvn = vnr - vnl;
    const double ic2 = ic * ic, hic2 = 0.5 * ic2;
    const double a1 = (dp - rt * ct * dvn) * hic2;
    const double a2 = drho - dp * ic2;
    const double a5 = (dp + rt * ct * dvn) * hic2;
    const double l1 = fabs(vnt - ct), l2 = fabs(vnt), l5 = fabs(vnt + ct);
    const double sx = du - dvn * nx, sy = dv - dvn * ny, sz = dw - dvn * nz;
    double D[5];
    D[0] = l1 * a1 + l2 * a2 + l5 * a5;
    D[1] = l1 * a1 * (ut - ct * nx) + l2 * (a2 * ut + rt * sx) + l5 * a5 * (ut + ct * nx);
    D[2] = l1 * a1 * (vt - ct * ny) + l2 * (a2 * vt + rt * sy) + l5 * a5 * (vt + ct * ny);
    D[3] = l1 * a1 * (wt - ct * nz) + l2 * (a2 * wt + rt * sz) + l5 * a5 * (wt + ct * nz);
    D[4] = l1 * a1 * (Ht - ct * vnt) +
           l2 * (a2 * 0.5 * q2 + rt * (ut * du + vt * dv + wt * dw - vnt * dvn)) +
           l5 * a5 * (Ht + ct * vnt);
    // 0.5 (Fn(ql) + Fn(qr))
    const double Hql = ql[4] + pl, Hqr = qr[4] + pr;
    F[0] = 0.5 * (ql[0] * vnl + qr[0] * vnr) - 0.5 * D[0];
    F[1] = 0.5 * (ql[1] * vnl + pl * nx + qr[1] * vnr + pr * nx) - 0.5 * D[1];
    F[2] = 0.5 * (ql[2] * vnl + pl * ny + qr[2] * vnr + pr * ny) - 0.5 * D[2];
    F[3] = 0.5 * (ql[3] * vnl + pl * nz + qr[3] * vnr + pr * nz) - 0.5 * D[3];
    F[4] = 0.5 * (vnl * Hql + vnr * Hqr) - 0.5 * D[4];
  }
  // boundary states (oracle/physics.py NavierStokes.bc_*)
  __device__ static void bc_ghost(const double*, const double* q, const double* n, int kind,
                                  const double* ghost, double* qg) {
    if (kind == BC_WALL) {
      qg[0] = q[0];
      qg[1] = -q[1];
      qg[2] = -q[2];
      qg[3] = -q[3];
      qg[4] = q[4];
    } else if (kind == BC_SYMMETRY) {
      const double mn = q[1] * n[0] + q[2] * n[1] + q[3] * n[2];
      qg[0] = q[0];
      qg[1] = q[1] - 2.0 * mn * n[0];
      qg[2] = q[2] - 2.0 * mn * n[1];
      qg[3] = q[3] - 2.0 * mn * n[2];
      qg[4] = q[4];
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) qg[k] = ghost[k];
    }
  }
  __device__ static void bc_lift(const double* P, const double* q, const double* n, int kind,
                                 const double* ghost, double* g) {
    if (kind == BC_WALL) {
      grad_vars(P, q, g);
      g[0] = g[1] = g[2] = 0.0;
    } else if (kind == BC_SYMMETRY) {
      grad_vars(P, q, g);
      const double vn = g[0] * n[0] + g[1] * n[1] + g[2] * n[2];
      g[0] -= vn * n[0];
      g[1] -= vn * n[1];
      g[2] -= vn * n[2];
    } else {
      grad_vars(P, ghost, g);
    }
  }
  __device__ static void bc_visc_normal(const double* P, const double* q, const double G[3][NGV],
                                        const double* n, int kind, double* out) {
    if (kind == BC_SYMMETRY) {
#pragma unroll
      for (int k = 0; k < 5; ++k) out[k] = 0.0;
    } else if (kind == BC_WALL) {
      double Gw[3][NGV];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        Gw[d][0] = G[d][0];
        Gw[d][1] = G[d][1];
        Gw[d][2] = G[d][2];
        Gw[d][3] = 0.0;
      }
#pragma unroll
      for (int k = 0; k < 5; ++k) out[k] = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double fv[5];
        visc_dir(P, 0.0, 0.0, 0.0, Gw, d, fv);
#pragma unroll
        for (int k = 0; k < 5; ++k) out[k] += n[d] * fv[k];
      }
    } else {
      visc_normal(P, q, G, n, out);
    }
  }
};

}  // namespace tdg
