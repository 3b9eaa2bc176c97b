"""Conservation laws (oracle): flux functors for the operator.

Scalar laws restate /root/reference/pkg/src/taudg/physics.py:49-88 in 3D
(a third flux component, zero for the reference's 2D cases).  The
compressible Navier-Stokes law follows PAPER.md:744-816 (non-dimensional,
Stokes hypothesis, gamma, Pr, M, Re) with the choices recorded in DESIGN.md
(Appendix A of SURVEY.md): constant viscosity mu=1 (non-dimensional), BR1
lifting of the primitive variables (u, v, w, T), Roe's approximate Riemann
solver without entropy fix, and a BR1 interface viscous flux equal to the
mean of the two sides' viscous fluxes.

Array conventions: component axes sit at axis 1 — states (B, nv, ...),
gradients (B, 3, ngv, ...) with G[:, d, k] = d g_k / d x_d, fluxes
(B, 3, nv, ...), normals (B, 3, ...).
"""

from __future__ import annotations

import numpy as np


class ScalarLaw:
    nv = 1
    ngv = 1
    # interior faces carry the gradient traces to the mortar and evaluate the
    # viscous flux there, as the reference does (operators.py:318-329)
    side_flux_traces = False

    def __init__(self, mu=0.0):
        if mu < 0.0:
            raise ValueError("viscosity must be >= 0")
        self.mu = float(mu)
        self.exact = None
        self.source = None

    @property
    def viscous(self):
        return self.mu > 0.0

    @property
    def mu_cfl(self):
        return self.mu

    def with_manufactured(self, exact, source):
        self.exact = exact
        self.source = source
        return self

    def grad_vars(self, q):
        return q

    def visc_flux(self, q, G):
        # mu * grad q   (reference operators.py:284-287)
        return self.mu * G

    # boundary treatment (reference operators.py:238-243, 304-309)
    def bc_riemann_ghost(self, q, n, kind, ghost):
        return ghost

    def bc_lift_value(self, q, n, kind, ghost):
        return self.grad_vars(ghost)

    def bc_visc_normal(self, q, G, n, kind):
        fv = self.visc_flux(q, G)
        return np.einsum("bd...,bdv...->bv...", n, fv)


class AdvectionDiffusion(ScalarLaw):
    """flux = (a q, b q, c q) - mu grad q; full upwind (physics.py:49-69)."""

    def __init__(self, velocity=(1.0, 1.0, 0.0), mu=0.0):
        super().__init__(mu)
        v = tuple(float(x) for x in velocity) + (0.0,) * (3 - len(velocity))
        self.velocity = v[:3]

    def adv_flux(self, q):
        a = np.array(self.velocity).reshape((1, 3, 1) + (1,) * (q.ndim - 2))
        return a * q[:, None]

    def wave_speed(self, q):
        return np.full_like(q[:, 0], float(np.sqrt(sum(c * c for c in self.velocity))))

    def riemann(self, ql, qr, n):
        an = sum(self.velocity[d] * n[:, d] for d in range(3))[:, None]
        return 0.5 * an * (ql + qr) + 0.5 * np.abs(an) * (ql - qr)


class ViscousBurgers(ScalarLaw):
    """flux = q^2/2 * beta - mu grad q, Rusanov with lambda = max|q|
    (physics.py:72-88; beta = (1, 1, 0) reproduces the reference)."""

    def __init__(self, mu=0.0, beta=(1.0, 1.0, 0.0)):
        super().__init__(mu)
        self.beta = tuple(float(x) for x in beta)

    def adv_flux(self, q):
        b = np.array(self.beta).reshape((1, 3, 1) + (1,) * (q.ndim - 2))
        return b * (0.5 * q * q)[:, None]

    def wave_speed(self, q):
        return float(np.sqrt(sum(c * c for c in self.beta))) * np.abs(q[:, 0])

    def riemann(self, ql, qr, n):
        bn = sum(self.beta[d] * n[:, d] for d in range(3))[:, None]
        lam = np.maximum(np.abs(ql), np.abs(qr))
        return 0.25 * (ql * ql + qr * qr) * bn - 0.5 * lam * (qr - ql)


class NavierStokes:
    """Compressible NS, q = (rho, rho u, rho v, rho w, rho E)."""

    # Every element side evaluates its own normal viscous flux F_v.n sigma at
    # its own face nodes — from the traces of the lifted variables (u, v, w, T)
    # and of their gradient, with the side's own outward normal (boundary
    # treatment included) — and interior faces average the two sides'
    # interpolants on the mortar (decision 3).  The reference has
    # no Navier-Stokes law; this choice is this repo's.
    side_flux_traces = True

    nv = 5
    ngv = 4

    def __init__(self, gamma=1.4, prandtl=0.72, mach=0.3, reynolds=100.0,
                 aoa=(0.0, 0.0)):
        self.gamma = float(gamma)
        self.prandtl = float(prandtl)
        self.mach = float(mach)
        self.reynolds = float(reynolds)
        self.aoa = aoa
        self.exact = None
        self.source = None

    @property
    def viscous(self):
        return self.reynolds > 0.0 and np.isfinite(self.reynolds)

    @property
    def mu(self):
        return 1.0 / self.reynolds if self.viscous else 0.0

    @property
    def mu_cfl(self):
        return max(4.0 / 3.0, self.gamma / self.prandtl) / self.reynolds if self.viscous else 0.0

    def freestream(self):
        a, b = self.aoa
        v = np.array([np.cos(a) * np.cos(b), np.sin(a) * np.cos(b), np.sin(b)])
        p = 1.0 / (self.gamma * self.mach ** 2)
        rhoE = p / (self.gamma - 1.0) + 0.5
        return np.array([1.0, v[0], v[1], v[2], rhoE])

    def _prim(self, q):
        rho = q[:, 0]
        u, v, w = q[:, 1] / rho, q[:, 2] / rho, q[:, 3] / rho
        p = (self.gamma - 1.0) * (q[:, 4] - 0.5 * rho * (u * u + v * v + w * w))
        return rho, u, v, w, p

    def pressure(self, q):
        return self._prim(q)[4]

    def grad_vars(self, q):
        rho, u, v, w, p = self._prim(q)
        T = self.gamma * self.mach ** 2 * p / rho
        return np.stack([u, v, w, T], axis=1)

    def adv_flux(self, q):
        rho, u, v, w, p = self._prim(q)
        vel = (u, v, w)
        H = q[:, 4] + p
        out = np.empty((q.shape[0], 3, 5) + q.shape[2:])
        for d in range(3):
            vd = vel[d]
            out[:, d, 0] = q[:, 0] * vd
            out[:, d, 1] = q[:, 1] * vd
            out[:, d, 2] = q[:, 2] * vd
            out[:, d, 3] = q[:, 3] * vd
            out[:, d, 1 + d] += p
            out[:, d, 4] = vd * H
        return out

    def visc_flux(self, q, G):
        """(1/Re) [0, tau_dx, tau_dy, tau_dz, u.tau_d + T_d/((g-1) Pr M^2)]."""
        rho, u, v, w, p = self._prim(q)
        return self.visc_flux_vel((u, v, w), G)

    def visc_flux_vel(self, vel, G):
        """The viscous flux from the velocity (u, v, w) and the gradient G."""
        inv_re = 1.0 / self.reynolds
        kappa = 1.0 / ((self.gamma - 1.0) * self.prandtl * self.mach ** 2)
        # G[:, d, k]: d/dx_d of (u, v, w, T)[k]
        div = G[:, 0, 0] + G[:, 1, 1] + G[:, 2, 2]
        out = np.zeros((G.shape[0], 3, 5) + G.shape[3:])
        for d in range(3):
            tau = []
            for i in range(3):
                t = G[:, d, i] + G[:, i, d]
                if i == d:
                    t = t - (2.0 / 3.0) * div
                tau.append(t)
            out[:, d, 1] = inv_re * tau[0]
            out[:, d, 2] = inv_re * tau[1]
            out[:, d, 3] = inv_re * tau[2]
            out[:, d, 4] = inv_re * (vel[0] * tau[0] + vel[1] * tau[1] + vel[2] * tau[2]
                                     + kappa * G[:, d, 3])
        return out

    def side_visc_normal(self, gv, G, n, kind=None):
        """F_v.n at a side's own face nodes from the traces gv (B, ngv, ...) of
        (u, v, w, T) and G of their gradient; ``kind`` applies the boundary
        treatment of bc_visc_normal (wall: no slip, adiabatic; symmetry: 0)."""
        if kind == "symmetry":
            return np.zeros((gv.shape[0], 5) + gv.shape[2:])
        if kind == "wall":
            zero = np.zeros_like(gv[:, 0])
            Gw = G.copy()
            Gw[:, :, 3] = 0.0
            fv = self.visc_flux_vel((zero, zero, zero), Gw)
        else:
            fv = self.visc_flux_vel((gv[:, 0], gv[:, 1], gv[:, 2]), G)
        return np.einsum("bd...,bdv...->bv...", n, fv)

    def wave_speed(self, q):
        rho, u, v, w, p = self._prim(q)
        return np.sqrt(u * u + v * v + w * w) + np.sqrt(self.gamma * p / rho)

    def riemann(self, ql, qr, n):
        """Roe flux through unit normal n (no entropy fix)."""
        g = self.gamma
        rl, ul, vl, wl, pl = self._prim(ql)
        rr, ur, vr, wr, pr = self._prim(qr)
        nx, ny, nz = n[:, 0], n[:, 1], n[:, 2]
        vnl = ul * nx + vl * ny + wl * nz
        vnr = ur * nx + vr * ny + wr * nz
        Hl = (ql[:, 4] + pl) / rl
        Hr = (qr[:, 4] + pr) / rr
        sl, sr = np.sqrt(rl), np.sqrt(rr)
        inv = 1.0 / (sl + sr)
        ut = (sl * ul + sr * ur) * inv
        vt = (sl * vl + sr * vr) * inv
        wt = (sl * wl + sr * wr) * inv
        Ht = (sl * Hl + sr * Hr) * inv
        rt = sl * sr
        q2 = ut * ut + vt * vt + wt * wt
        c2 = (g - 1.0) * (Ht - 0.5 * q2)
        ct = np.sqrt(c2)
        vnt = ut * nx + vt * ny + wt * nz
        drho = rr - rl
        dp = pr - pl
        du, dv, dw = ur - ul, vr - vl, wr - wl
        dvn = vnr - vnl
        a1 = (dp - rt * ct * dvn) / (2.0 * c2)
        a2 = drho - dp / c2
        a5 = (dp + rt * ct * dvn) / (2.0 * c2)
        l1 = np.abs(vnt - ct)
        l2 = np.abs(vnt)
        l5 = np.abs(vnt + ct)
        # shear jump
        sx, sy, sz = du - dvn * nx, dv - dvn * ny, dw - dvn * nz
        D = np.empty_like(ql)
        D[:, 0] = l1 * a1 + l2 * a2 + l5 * a5
        D[:, 1] = l1 * a1 * (ut - ct * nx) + l2 * (a2 * ut + rt * sx) + l5 * a5 * (ut + ct * nx)
        D[:, 2] = l1 * a1 * (vt - ct * ny) + l2 * (a2 * vt + rt * sy) + l5 * a5 * (vt + ct * ny)
        D[:, 3] = l1 * a1 * (wt - ct * nz) + l2 * (a2 * wt + rt * sz) + l5 * a5 * (wt + ct * nz)
        D[:, 4] = (l1 * a1 * (Ht - ct * vnt)
                   + l2 * (a2 * 0.5 * q2 + rt * (ut * du + vt * dv + wt * dw - vnt * dvn))
                   + l5 * a5 * (Ht + ct * vnt))
        fl = self.adv_flux(ql)
        fr = self.adv_flux(qr)
        fnl = fl[:, 0] * nx[:, None] + fl[:, 1] * ny[:, None] + fl[:, 2] * nz[:, None]
        fnr = fr[:, 0] * nx[:, None] + fr[:, 1] * ny[:, None] + fr[:, 2] * nz[:, None]
        return 0.5 * (fnl + fnr) - 0.5 * D

    # boundary conditions ---------------------------------------------------------
    def _reflect(self, q, n, full):
        rho = q[:, 0]
        mn = q[:, 1] * n[:, 0] + q[:, 2] * n[:, 1] + q[:, 3] * n[:, 2]
        out = q.copy()
        if full:                      # no-slip: reverse the whole momentum
            out[:, 1:4] = -q[:, 1:4]
        else:                         # slip: mirror the normal momentum
            for d in range(3):
                out[:, 1 + d] = q[:, 1 + d] - 2.0 * mn * n[:, d]
        return out

    def bc_riemann_ghost(self, q, n, kind, ghost):
        if kind == "wall":
            return self._reflect(q, n, True)
        if kind == "symmetry":
            return self._reflect(q, n, False)
        return ghost      # freestream / dirichlet: fixed state

    def bc_lift_value(self, q, n, kind, ghost):
        if kind == "wall":
            g = self.grad_vars(q)
            g[:, 0:3] = 0.0
            return g
        if kind == "symmetry":
            g = self.grad_vars(q)
            vn = g[:, 0] * n[:, 0] + g[:, 1] * n[:, 1] + g[:, 2] * n[:, 2]
            for d in range(3):
                g[:, d] = g[:, d] - vn * n[:, d]
            return g
        return self.grad_vars(ghost)

    def bc_visc_normal(self, q, G, n, kind):
        if kind == "symmetry":
            return np.zeros_like(q)
        if kind == "wall":
            qw = q.copy()
            rho, u, v, w, p = self._prim(q)
            qw[:, 1:4] = 0.0
            qw[:, 4] = p / (self.gamma - 1.0)
            Gw = G.copy()
            Gw[:, :, 3] = 0.0         # adiabatic: no heat flux
            fv = self.visc_flux(qw, Gw)
        else:
            fv = self.visc_flux(q, G)
        return np.einsum("bd...,bdv...->bv...", n, fv)
