"""DGSEM spatial operator on 3D hex meshes with per-element anisotropic orders
(oracle).  Restates /root/reference/pkg/src/taudg/operators.py:1-389:

    M dQ/dt + F(Q) = M S,     M = (w1 x w2 x w3) J            (operators.py:119)

* weak volume divergence of the contravariant fluxes          (:196-200, :283-290)
* traces via boundary rows                                     (:73-80, :185-194)
* interfaces on a mortar at max(own, neighbour) order per tangential
  direction, interpolated up and L2-projected back             (:146-171, :211-217)
* BR1 lifted gradient, q* = mortar mean / boundary ghost / own trace
                                                               (:224-265)
* face fluxes: Riemann + mean viscous flux on interior mortars, Riemann with
  the ghost + interior viscous flux on boundaries, and the analytic own-trace
  flux for every side in the isolated variant                  (:292-334).
  Scalar laws take the gradient traces to the mortar as the reference does;
  Navier-Stokes (no reference counterpart) takes each side's own normal
  viscous flux F_v(q, G).n sigma there (``law.side_flux_traces``)
* A = F / M, r = S - A, tau_e = max |M (S_pde - A)|            (:337-364)

Differences from the reference, all recorded in DESIGN.md: 3D, nv unknowns,
node family LG | LGL, face orientation codes instead of the 2D ``flip``,
state-dependent boundary ghosts for Navier-Stokes walls, and faces evaluated
in vectorised groups (same faces, same arithmetic; summation order differs).
"""

from __future__ import annotations

import numpy as np

from . import geometry, spectral
from .fields import NodalField, OrderField


def _aligned_from_right(arr, o):
    out = np.swapaxes(arr, -1, -2) if o & 4 else arr
    if o & 1:
        out = out[..., ::-1, :]
    if o & 2:
        out = out[..., :, ::-1]
    return out


def _right_from_aligned(arr, o):
    out = arr
    if o & 1:
        out = out[..., ::-1, :]
    if o & 2:
        out = out[..., :, ::-1]
    return np.swapaxes(out, -1, -2) if o & 4 else out


def _face_dirs(side):
    d = side // 2
    t = [x for x in range(3) if x != d]
    return d, t[0], t[1]


class _Group:
    pass


class DGOperator:
    def __init__(self, msh, law, orders: OrderField, family="LG", form="cross"):
        if orders.num_elements != msh.num_elements:
            raise ValueError("order field does not match the mesh element count")
        self.mesh = msh
        self.law = law
        self.orders = orders
        self.family = family
        self.form = form
        self.nv = law.nv
        self.calls = {"apply": 0, "apply_isolated": 0}
        self._build_groups()
        self._build_faces()
        self.source = (
            self.project_function(law.source) if law.source is not None
            else NodalField.zeros(orders, self.nv)
        )

    # construction --------------------------------------------------------------
    def _build_groups(self):
        of = self.orders
        fam = self.family
        self.group_ops = []
        for sig, ids in zip(of.group_orders, of.group_elements):
            go = _Group()
            go.orders = sig
            rules = [spectral.rule(n, fam) for n in sig]
            go.w = [r[1] for r in rules]
            go.x = [r[0] for r in rules]
            go.dhat = [go.w[d][:, None] * spectral.differentiation_matrix(sig[d], fam) for d in range(3)]
            go.bounds = [spectral.boundary_rows(sig[d], fam) for d in range(3)]
            jac, ja, sizes, coords = [], [], [], []
            for e in ids:
                j, a, s = geometry.volume_metrics(self.mesh.nodes[e], sig, fam, self.form, int(e))
                jac.append(j)
                ja.append(a)
                sizes.append(s)
                coords.append(geometry.map_points_ordered(self.mesh.nodes[e], *go.x) if self.form == "curl"
                              else geometry.map_points(self.mesh.nodes[e], *go.x))
            go.jac = np.stack(jac)
            go.ja = np.stack(ja)                       # (B, 3, 3, n1, n2, n3)
            go.sizes = np.array(sizes)
            go.coords = np.stack(coords)               # (B, n1, n2, n3, 3)
            www = go.w[0][:, None, None] * go.w[1][None, :, None] * go.w[2][None, None, :]
            go.mass = www[None] * go.jac
            go.inv_mass = 1.0 / go.mass
            # own-order side geometry for every side (isolated + boundary use)
            go.side_sigma, go.side_normal = [], []
            for s in range(6):
                sig_l, nrm_l = [], []
                d, a, b = _face_dirs(s)
                for k, e in enumerate(ids):
                    if self.form == "cross":
                        jf = geometry.face_ja_analytic(self.mesh.nodes[e], s, go.x[a], go.x[b])
                    else:
                        jf = geometry.face_ja_from_volume(go.ja[k], s, sig, fam)
                    sg, nm = geometry.sigma_normal(jf, s)
                    sig_l.append(sg)
                    nrm_l.append(np.moveaxis(nm, -1, 0))
                go.side_sigma.append(np.stack(sig_l))         # (B, nt1, nt2)
                go.side_normal.append(np.stack(nrm_l))        # (B, 3, nt1, nt2)
            self.group_ops.append(go)

    def _tan_orders(self, e, side):
        _, a, b = _face_dirs(side)
        o = self.orders.orders[e]
        return int(o[a]), int(o[b])

    def _build_faces(self):
        fam = self.family
        slot = self.orders.element_slot
        inter, bnd = {}, {}
        for fi, f in enumerate(self.mesh.faces):
            gl, rl = (int(v) for v in slot[f.left])
            if f.is_boundary:
                kind = self.mesh.bc_kind(f.tag)
                bnd.setdefault((gl, f.side_left, kind), []).append((rl, fi))
            else:
                gr, rr = (int(v) for v in slot[f.right])
                inter.setdefault((gl, f.side_left, gr, f.side_right, f.orient), []).append((rl, rr, fi))
        self.interior_groups = []
        for (gl, sl, gr, sr, o), items in inter.items():
            fg = _Group()
            fg.gl, fg.sl, fg.gr, fg.sr, fg.orient = gl, sl, gr, sr, o
            fg.rows_l = np.array([i[0] for i in items])
            fg.rows_r = np.array([i[1] for i in items])
            fg.faces = [i[2] for i in items]
            el0 = self.mesh.faces[fg.faces[0]].left
            er0 = self.mesh.faces[fg.faces[0]].right
            L = self._tan_orders(el0, sl)
            Rown = self._tan_orders(er0, sr)
            R = (Rown[1], Rown[0]) if o & 4 else Rown
            M = (max(L[0], R[0]), max(L[1], R[1]))
            fg.L, fg.R, fg.M = L, R, M
            fg.upL = [spectral.transfer(L[k], M[k], fam) for k in range(2)]
            fg.dnL = [spectral.transfer(M[k], L[k], fam) for k in range(2)]
            fg.upR = [spectral.transfer(R[k], M[k], fam) for k in range(2)]
            fg.dnR = [spectral.transfer(M[k], R[k], fam) for k in range(2)]
            # mortar geometry from the left element (operators.py:168-170)
            xm = [spectral.rule(M[k], fam)[0] for k in range(2)]
            sig_l, nrm_l = [], []
            gop = self.group_ops[gl]
            for fi, rl in zip(fg.faces, fg.rows_l):
                e = self.mesh.faces[fi].left
                if self.form == "cross":
                    jf = geometry.face_ja_analytic(self.mesh.nodes[e], sl, xm[0], xm[1])
                else:
                    own = geometry.face_ja_from_volume(gop.ja[rl], sl, gop.orders, fam)
                    jf = np.einsum("Aa,Bb,abx->ABx", fg.upL[0], fg.upL[1], own)
                sg, nm = geometry.sigma_normal(jf, sl)
                sig_l.append(sg)
                nrm_l.append(np.moveaxis(nm, -1, 0))
            fg.sigma = np.stack(sig_l)
            fg.normal = np.stack(nrm_l)
            self.interior_groups.append(fg)
        self.boundary_groups = []
        for (g, s, kind), items in bnd.items():
            fg = _Group()
            fg.g, fg.s, fg.kind = g, s, kind
            fg.rows = np.array([i[0] for i in items])
            fg.faces = [i[1] for i in items]
            gop = self.group_ops[g]
            fg.sigma = gop.side_sigma[s][fg.rows]
            fg.normal = gop.side_normal[s][fg.rows]
            d, a, b = _face_dirs(s)
            fg.ghost = None
            if kind == "dirichlet":
                if self.law.exact is None:
                    raise ValueError("law provides no boundary data (exact field missing)")
                pts = np.stack([
                    geometry.face_points(self.mesh.nodes[self.mesh.faces[fi].left], s, gop.x[a], gop.x[b])
                    for fi in fg.faces
                ])
                fg.ghost = self._eval(self.law.exact, pts)
            elif kind == "freestream":
                fs = self.law.freestream()
                nt = (len(gop.x[a]), len(gop.x[b]))
                fg.ghost = np.broadcast_to(fs[None, :, None, None], (len(fg.rows), self.nv) + nt).copy()
            self.boundary_groups.append(fg)

    def _eval(self, fn, pts):
        """fn(x, y, z) at points (..., 3) -> (F, nv, ...) array."""
        vals = np.asarray(fn(pts[..., 0], pts[..., 1], pts[..., 2]), dtype=float)
        if self.nv == 1:
            return vals[:, None]
        return np.moveaxis(vals, 0, 1)

    # helpers ------------------------------------------------------------------
    def project_function(self, fn):
        out = NodalField.zeros(self.orders, self.nv)
        for g, gop in enumerate(self.group_ops):
            out.blocks[g][:] = self._eval(fn, gop.coords)
        return out

    def mass_blocks(self):
        return [gop.mass for gop in self.group_ops]

    @staticmethod
    def _trace_block(block, side, bounds, lead):
        d = side // 2
        row = bounds[d][side % 2]
        return np.tensordot(block, row, axes=([lead + d], [0]))

    def _traces(self, blocks, lead=2):
        return [
            [self._trace_block(blocks[g], s, gop.bounds, lead) for s in range(6)]
            for g, gop in enumerate(self.group_ops)
        ]

    def _weak_div(self, g, ft):
        """ft (B, 3, c, n1, n2, n3) -> (B, c, n1, n2, n3)."""
        go = self.group_ops[g]
        w1, w2, w3 = go.w
        t1 = np.einsum("mi,bcmjk->bcijk", go.dhat[0], ft[:, 0]) * (w2[:, None] * w3[None, :])
        t2 = np.einsum("mj,bcimk->bcijk", go.dhat[1], ft[:, 1]) * (w1[:, None, None] * w3[None, None, :])
        t3 = np.einsum("mk,bcijm->bcijk", go.dhat[2], ft[:, 2]) * (w1[:, None, None] * w2[None, :, None])
        return t1 + t2 + t3

    def _scatter(self, blocks, g, rows, side, vec):
        """blocks[g][rows] += l_side (x) (w_t1 w_t2 vec); vec (F, c, nt1, nt2)."""
        go = self.group_ops[g]
        d, a, b = _face_dirs(side)
        contrib = vec * (go.w[a][:, None] * go.w[b][None, :])
        row = go.bounds[d][side % 2]
        shape = [1] * 3
        shape[d] = len(row)
        full = np.expand_dims(contrib, 2 + d) * row.reshape([1, 1] + shape)
        blocks[g][rows] += full

    @staticmethod
    def _up(T, arr):
        return np.einsum("Aa,Bb,...ab->...AB", T[0], T[1], arr)

    # gradient lift -----------------------------------------------------------------
    def _lift_gradient(self, Q, trq, isolated):
        law = self.law
        ngv = law.ngv
        comps = []
        for g, go in enumerate(self.group_ops):
            gv = law.grad_vars(Q.blocks[g])                 # (B, ngv, ...)
            acc = np.empty((gv.shape[0], 3, ngv) + gv.shape[2:])
            for d in range(3):
                ft = go.ja[:, :, d][:, :, None] * gv[:, None]   # (B, 3, ngv, ...)
                acc[:, d] = -self._weak_div(g, ft)
            comps.append(acc)
        # scatter target: view comps[g] as (B, 3*ngv, ...)
        flat = [c.reshape((c.shape[0], 3 * ngv) + c.shape[3:]) for c in comps]

        def scat(g, rows, side, gstar, sigma, normal):
            val = (gstar[:, None] * (normal * sigma[:, None])[:, :, None])   # (F, 3, ngv, a, b)
            self._scatter(flat, g, rows, side, val.reshape((val.shape[0], 3 * ngv) + val.shape[3:]))

        if isolated:
            for g, go in enumerate(self.group_ops):
                rows = np.arange(Q.blocks[g].shape[0])
                for s in range(6):
                    scat(g, rows, s, law.grad_vars(trq[g][s]), go.side_sigma[s], go.side_normal[s])
        else:
            for fg in self.boundary_groups:
                q_in = trq[fg.g][fg.s][fg.rows]
                gstar = law.bc_lift_value(q_in, fg.normal, fg.kind, fg.ghost)
                scat(fg.g, fg.rows, fg.s, gstar, fg.sigma, fg.normal)
            for fg in self.interior_groups:
                ql = trq[fg.gl][fg.sl][fg.rows_l]
                qr = _aligned_from_right(trq[fg.gr][fg.sr][fg.rows_r], fg.orient)
                qlm = self._up(fg.upL, ql)
                qrm = self._up(fg.upR, qr)
                gstar = 0.5 * (law.grad_vars(qlm) + law.grad_vars(qrm))
                val = gstar[:, None] * (fg.normal * fg.sigma[:, None])[:, :, None]
                val = val.reshape((val.shape[0], 3 * ngv) + val.shape[3:])
                self._scatter(flat, fg.gl, fg.rows_l, fg.sl, self._up(fg.dnL, val))
                back = _right_from_aligned(self._up(fg.dnR, val), fg.orient)
                self._scatter(flat, fg.gr, fg.rows_r, fg.sr, -back)
        for g, go in enumerate(self.group_ops):
            comps[g] *= go.inv_mass[:, None, None]
        return comps

    # main evaluation ------------------------------------------------------------
    def apply(self, Q: NodalField, isolated=False) -> NodalField:
        if Q.field is not self.orders:
            raise ValueError("field/operator order mismatch")
        self.calls["apply_isolated" if isolated else "apply"] += 1
        law = self.law
        visc = law.viscous
        trq = self._traces(Q.blocks)
        if visc:
            G = self._lift_gradient(Q, trq, isolated)
            trg = self._traces(G, lead=3)                     # (B, 3, ngv, a, b)
        out = NodalField.zeros(self.orders, self.nv)
        for g, go in enumerate(self.group_ops):
            q = Q.blocks[g]
            f = law.adv_flux(q)
            if visc:
                f = f - law.visc_flux(q, G[g])
            ft = np.einsum("bidxyz,bdvxyz->bivxyz", go.ja, f)
            out.blocks[g] -= self._weak_div(g, ft)

        def normal_flux(fl, n):
            return np.einsum("bd...,bdv...->bv...", n, fl)

        side_fv = visc and getattr(law, "side_flux_traces", False)
        if side_fv:
            # traces of the lifted variables: every side's own F_v.n sigma at
            # its own face nodes comes from them and the gradient traces
            trv = self._traces([law.grad_vars(b) for b in Q.blocks])

            def side_fv_sigma(g, s, rows, kind=None):
                go = self.group_ops[g]
                return (law.side_visc_normal(trv[g][s][rows], trg[g][s][rows], go.side_normal[s][rows], kind)
                        * go.side_sigma[s][rows][:, None])

        if isolated:
            for g, go in enumerate(self.group_ops):
                rows = np.arange(Q.blocks[g].shape[0])
                for s in range(6):
                    q_in = trq[g][s]
                    n = go.side_normal[s]
                    flux = normal_flux(law.adv_flux(q_in), n)
                    if side_fv:
                        self._scatter(out.blocks, g, rows, s,
                                      flux * go.side_sigma[s][:, None] - side_fv_sigma(g, s, rows))
                        continue
                    if visc:
                        flux = flux - normal_flux(law.visc_flux(q_in, trg[g][s]), n)
                    self._scatter(out.blocks, g, rows, s, flux * go.side_sigma[s][:, None])
            return out
        for fg in self.boundary_groups:
            q_in = trq[fg.g][fg.s][fg.rows]
            qg = law.bc_riemann_ghost(q_in, fg.normal, fg.kind, fg.ghost)
            flux = law.riemann(q_in, qg, fg.normal)
            if side_fv:
                self._scatter(out.blocks, fg.g, fg.rows, fg.s,
                              flux * fg.sigma[:, None] - side_fv_sigma(fg.g, fg.s, fg.rows, fg.kind))
                continue
            if visc:
                flux = flux - law.bc_visc_normal(q_in, trg[fg.g][fg.s][fg.rows], fg.normal, fg.kind)
            self._scatter(out.blocks, fg.g, fg.rows, fg.s, flux * fg.sigma[:, None])
        for fg in self.interior_groups:
            ql = trq[fg.gl][fg.sl][fg.rows_l]
            qr = _aligned_from_right(trq[fg.gr][fg.sr][fg.rows_r], fg.orient)
            qlm = self._up(fg.upL, ql)
            qrm = self._up(fg.upR, qr)
            flux = law.riemann(qlm, qrm, fg.normal)
            if side_fv:
                # mortar mean of the two sides' interpolated normal viscous
                # fluxes; the right side's carries its own (opposite) normal
                fl = self._up(fg.upL, side_fv_sigma(fg.gl, fg.sl, fg.rows_l))
                fr = self._up(fg.upR, _aligned_from_right(side_fv_sigma(fg.gr, fg.sr, fg.rows_r), fg.orient))
                val = flux * fg.sigma[:, None] - 0.5 * (fl - fr)
            else:
                if visc:
                    gl = self._up(fg.upL, trg[fg.gl][fg.sl][fg.rows_l])
                    gr = self._up(fg.upR, _aligned_from_right(trg[fg.gr][fg.sr][fg.rows_r], fg.orient))
                    fv = 0.5 * (normal_flux(law.visc_flux(qlm, gl), fg.normal)
                                + normal_flux(law.visc_flux(qrm, gr), fg.normal))
                    flux = flux - fv
                val = flux * fg.sigma[:, None]
            self._scatter(out.blocks, fg.gl, fg.rows_l, fg.sl, self._up(fg.dnL, val))
            back = _right_from_aligned(self._up(fg.dnR, val), fg.orient)
            self._scatter(out.blocks, fg.gr, fg.rows_r, fg.sr, -back)
        return out

    def m_inv_apply(self, Q, isolated=False):
        out = self.apply(Q, isolated=isolated)
        for g, go in enumerate(self.group_ops):
            out.blocks[g] *= go.inv_mass[:, None]
        return out

    def residual(self, Q, source=None):
        src = self.source if source is None else source
        r = self.m_inv_apply(Q)
        for g in range(len(r.blocks)):
            r.blocks[g] = src.blocks[g] - r.blocks[g]
        return r

    def residual_norm(self, Q, source=None):
        return self.residual(Q, source).norm_inf()

    def truncation_from_avalue(self, a_value):
        tau = NodalField.zeros(self.orders, self.nv)
        for g, go in enumerate(self.group_ops):
            tau.blocks[g] = go.mass[:, None] * (self.source.blocks[g] - a_value.blocks[g])
        return tau.element_norms_inf()

    def truncation(self, Q, isolated=False):
        return self.truncation_from_avalue(self.m_inv_apply(Q, isolated=isolated))

    def term_scale(self, Q, isolated=False):
        """max |WD(f~)| over nodes: the magnitude of the terms that cancel in
        F for near-freestream states — the normaliser for round-off-level
        parity of F, r and tau."""
        law = self.law
        G = self._lift_gradient(Q, self._traces(Q.blocks), isolated) if law.viscous else None
        out = 0.0
        for g, go in enumerate(self.group_ops):
            q = Q.blocks[g]
            f = law.adv_flux(q)
            if G is not None:
                f = f - law.visc_flux(q, G[g])
            ft = np.einsum("bidxyz,bdvxyz->bivxyz", go.ja, f)
            out = max(out, float(np.abs(self._weak_div(g, ft)).max()))
        return out

    def gradient(self, Q, isolated=False):
        """Lifted gradient blocks (B, 3, ngv, ...) — exposed for kernel parity."""
        return self._lift_gradient(Q, self._traces(Q.blocks), isolated)
