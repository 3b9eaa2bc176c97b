"""GPU parity of the sm_100a operator path (through the C-ABI) against
(a) the REAL reference's golden vectors (2D scalar LG sub-case, N3=0 extrusion)
and (b) the CPU oracle on 3D Navier-Stokes / Gauss-Lobatto / mortar /
orientation cases.  Tolerances (north_star): residuals and tau within 1e-12
relative to max|A(Q)| (normalise by the operator value, not by r).
"""

import numpy as np
import pytest

from helpers import (golden_law, golden_mesh, load, oracle_law, oracle_to_ref_flat, orders3,
                     ref_flat_to_oracle)

pytestmark = pytest.mark.gpu

OP_CASES = ["sine_warp_mixed", "burgers_mixed", "rotated_pair", "graded_bl",
            "runge_curved", "aniso_burgers_curved"]
RTOL = 1e-12


def _to_oracle(pf, of_o):
    from oracle.fields import NodalField as ON

    return ON(of_o, pf.to_oracle_blocks(), pf.nv)


def _from_oracle(of_p, of_o_field):
    from paper_1806_11456_b200.fields import NodalField

    f = NodalField.zeros(of_p, of_o_field.nv)
    f.load_oracle_blocks(of_o_field.blocks)
    return f


def _golden_setup(name):
    from oracle.fields import OrderField as OO
    from paper_1806_11456_b200 import fields, operators

    g = load(name)
    m = golden_mesh(g)
    plaw = golden_law(g)
    o3 = orders3(g["orders"])
    of_p, of_o = fields.OrderField(o3), OO(o3)
    op = operators.DGOperator(m, plaw, of_p, family="LG", form="cross")
    Qo = ref_flat_to_oracle(g["Q"], of_o)
    Q = _from_oracle(of_p, Qo)
    return g, m, plaw, of_p, of_o, op, Q


def _ref(pf, of_o):
    return oracle_to_ref_flat(_to_oracle(pf, of_o))


@pytest.mark.parametrize("name", OP_CASES)
def test_operator_matches_reference_golden(name):
    g, m, plaw, of_p, of_o, op, Q = _golden_setup("op_" + name)
    scale = np.abs(g["A"]).max()
    assert np.abs(_ref(op.apply(Q), of_o) - g["F"]).max() <= RTOL * np.abs(g["F"]).max()
    assert np.abs(_ref(op.apply(Q, isolated=True), of_o) - g["Fiso"]).max() <= RTOL * np.abs(g["Fiso"]).max()
    assert np.abs(_ref(op.residual(Q), of_o) - g["R"]).max() <= RTOL * scale
    assert np.abs(_ref(op.m_inv_apply(Q), of_o) - g["A"]).max() <= RTOL * scale
    assert abs(op.residual_norm(Q) - np.abs(g["R"]).max()) <= RTOL * scale
    assert np.abs(op.truncation(Q) - g["tau"]).max() <= RTOL * g["tau"].max()
    assert np.abs(op.truncation(Q, isolated=True) - g["tau_iso"]).max() <= RTOL * g["tau_iso"].max()
    a_val = op.m_inv_apply(Q)
    assert np.abs(op.truncation_from_avalue(a_val) - g["tau"]).max() <= RTOL * g["tau"].max()


@pytest.mark.parametrize("name", ["sine_warp_mixed", "burgers_mixed", "runge_curved"])
def test_rk3_matches_reference_golden(name):
    from paper_1806_11456_b200 import timestep

    g, m, plaw, of_p, of_o, op, Q = _golden_setup("op_" + name)
    cfg = timestep.TimeConfig()
    assert np.abs(timestep.element_dt(op, Q, cfg) - g["element_dt"]).max() <= 1e-15
    Qr = Q.copy()
    r0 = [timestep.rk3_step(op, Qr, timestep.compute_dt(op, Qr, cfg)) for _ in range(2)]
    assert np.abs(_ref(Qr, of_o) - g["Q_rk2"]).max() <= 1e-12
    assert np.abs(np.array(r0) - g["r0_rk2"]).max() <= RTOL * np.abs(g["r0_rk2"]).max()
    Ql = Q.copy()
    rl = timestep.rk3_step(op, Ql, timestep.compute_dt(op, Ql, timestep.TimeConfig(local=True)))
    assert np.abs(_ref(Ql, of_o) - g["Q_rk_local"]).max() <= 1e-12
    assert abs(rl - float(g["r0_local"])) <= RTOL * abs(float(g["r0_local"]))
    # device-side smoothing (no host sync per sweep) == host-dt stepping
    Qs, Qh = Q.copy(), Q.copy()
    hist = timestep.smooth(op, Qs, 3, cfg)
    ref_hist = [timestep.rk3_step(op, Qh, timestep.compute_dt(op, Qh, cfg)) for _ in range(3)]
    assert np.allclose(hist, ref_hist, rtol=1e-14, atol=0)
    assert float((Qs.data - Qh.data).abs().max()) <= 1e-14


# --- 3D Navier-Stokes / LGL / mortars / orientation vs the oracle ----------------

def _ns_state(law, amp=1e-2, seed=0):
    rng = np.random.default_rng(seed)
    fs = law.freestream()
    k = rng.integers(1, 3, (4, 3))
    ph = rng.uniform(0, 2 * np.pi, (4, 5))

    def fn(x, y, z):
        out = []
        for v in range(5):
            p = sum(np.sin(2 * np.pi * (k[m, 0] * x + k[m, 1] * y + k[m, 2] * z) + ph[m, v]) for m in range(4))
            out.append(fs[v] + amp * p)
        return np.stack(out)

    return fn


def _compare_case(msh, plaw, orders, family, form, seed=0, check_grad=True):
    from oracle.fields import OrderField as OO
    from oracle.operators import DGOperator as ODG
    from paper_1806_11456_b200 import fields, operators

    of_p, of_o = fields.OrderField(orders), OO(orders)
    olaw = oracle_law(plaw)
    op = operators.DGOperator(msh, plaw, of_p, family=family, form=form)
    oo = ODG(msh, olaw, of_o, family=family, form=form)
    fn = _ns_state(plaw, seed=seed) if plaw.nv == 5 else (lambda x, y, z: 1.0 + 0.3 * np.sin(3 * x + y - 2 * z))
    Qo = oo.project_function(fn)
    Q = op.project_function(fn)
    assert np.abs(oracle_to_ref_flat(_to_oracle(Q, of_o)) - oracle_to_ref_flat(Qo)).max() <= 1e-14
    A_o = oo.m_inv_apply(Qo)
    scale = A_o.norm_inf()
    for iso in (False, True):
        F = _to_oracle(op.apply(Q, isolated=iso), of_o)
        Fo = oo.apply(Qo, isolated=iso)
        fs = Fo.norm_inf()
        assert (F - Fo).norm_inf() <= RTOL * fs, (iso, (F - Fo).norm_inf() / fs)
        if check_grad and plaw.viscous:
            G = op.gradient(Q, isolated=iso).cpu().numpy()
            Go = oo.gradient(Qo, isolated=iso)
            pos = 0
            for g, (sig, ids) in enumerate(zip(of_o.group_orders, of_o.group_elements)):
                n = int(np.prod(np.array(sig) + 1))
                blk = G[pos: pos + len(ids) * n * 3 * plaw.ngv].reshape(
                    len(ids), 3, plaw.ngv, sig[2] + 1, sig[1] + 1, sig[0] + 1).transpose(0, 1, 2, 5, 4, 3)
                pos += blk.size
                # the lifted gradient is an intermediate: T = gamma M^2 p / rho
                # cancels ~2 digits before differentiation, so it is held to
                # 1e-11 relative; F, r and tau keep the 1e-12 bar
                gs = max(np.abs(Go[g]).max(), 1e-300)
                assert np.abs(blk - Go[g]).max() <= 10 * RTOL * max(gs, 1.0), (iso, g)
    R = _to_oracle(op.residual(Q), of_o)
    assert (R - oo.residual(Qo)).norm_inf() <= RTOL * scale
    for iso in (False, True):
        t = op.truncation(Q, isolated=iso)
        to = oo.truncation(Qo, isolated=iso)
        assert np.abs(t - to).max() <= RTOL * to.max()
    return op, oo, Q, Qo


NS_CASES = [
    # (mesh builder, orders kind, family, form)
    ("periodic_affine", "uniform3", "LGL", "curl"),
    ("periodic_jitter", "random1_5", "LGL", "curl"),
    ("periodic_jitter", "random1_5", "LG", "cross"),
    ("rotated_jitter", "random1_4", "LGL", "curl"),
    ("bc_box", "random1_4", "LGL", "curl"),
    ("bc_box", "uniform3", "LG", "curl"),
    # own-order lift, packed face-node passes: curved conforming N = 4 (staged
    # g* with per-node geometry), the same with boundary sides, and an affine
    # plan with several elements per work item (bulk-copied state)
    ("periodic_jitter", "uniform4", "LGL", "curl"),
    ("bc_box", "uniform4", "LGL", "curl"),
    ("periodic_affine", "uniform2", "LGL", "curl"),
]


def _ns_mesh(kind):
    from paper_1806_11456_b200 import mesh

    if kind == "periodic_affine":
        return mesh.build_box(3, 2, 2)
    if kind == "periodic_jitter":
        return mesh.build_box(3, 3, 2, jitter=0.1, rng=np.random.default_rng(2))
    if kind == "rotated_jitter":
        return mesh.build_rotated_box(3, 2, 2, jitter=0.1, seed=4, bc={"boundary": "freestream"})
    if kind == "bc_box":
        return mesh.build_box(3, 2, 2, periodic=(True, False, True), jitter=0.05,
                              rng=np.random.default_rng(7),
                              bc={"south": "wall", "north": "symmetry"})
    raise ValueError(kind)


def _orders(kind, nel, seed=11):
    rng = np.random.default_rng(seed)
    if kind.startswith("uniform"):
        return np.full((nel, 3), int(kind[len("uniform"):]))
    lo, hi = (int(v) for v in kind.replace("random", "").split("_"))
    return rng.integers(lo, hi + 1, (nel, 3))


@pytest.mark.parametrize("mesh_kind,orders_kind,family,form", NS_CASES)
def test_navier_stokes_matches_oracle(mesh_kind, orders_kind, family, form):
    from paper_1806_11456_b200 import physics

    msh = _ns_mesh(mesh_kind)
    law = physics.NavierStokes(mach=0.3, reynolds=100.0)
    if mesh_kind == "bc_box":
        # the non-periodic direction carries a freestream far field on other tags
        msh.bc.setdefault("boundary", "freestream")
    _compare_case(msh, law, _orders(orders_kind, msh.num_elements), family, form)


@pytest.mark.parametrize("mesh_kind,orders_kind,packed_min", [
    ("periodic_affine", "uniform3", "9"),   # affine plan forced onto the in-loop lift
    ("periodic_jitter", "uniform3", "1"),   # curved N = 3 forced onto the packed lift
    ("bc_box", "uniform3", "1"),            # ... with wall / symmetry / far-field sides
])
def test_own_order_lift_variants_match_oracle(monkeypatch, mesh_kind, orders_kind, packed_min):
    """Both variants of the own-order lift (k_vol_lift_own: packed passes;
    k_vol_lift_own_inl: in-loop) on plans where the default rule would pick the
    other one (the plan reads TDG_LIFT_PACKED_MIN when it is created)."""
    from paper_1806_11456_b200 import physics

    monkeypatch.setenv("TDG_LIFT_PACKED_MIN", packed_min)
    msh = _ns_mesh(mesh_kind)
    if mesh_kind == "bc_box":
        msh.bc.setdefault("boundary", "freestream")
    law = physics.NavierStokes(mach=0.3, reynolds=100.0)
    _compare_case(msh, law, _orders(orders_kind, msh.num_elements), "LGL", "curl")


@pytest.mark.parametrize("family", ["LG", "LGL"])
def test_inviscid_euler_matches_oracle(family):
    from paper_1806_11456_b200 import physics

    msh = _ns_mesh("periodic_jitter")
    law = physics.NavierStokes(mach=0.3, reynolds=0.0)
    _compare_case(msh, law, _orders("random1_5", msh.num_elements), family, "curl")


@pytest.mark.parametrize("family", ["LG", "LGL"])
def test_scalar_rotated_mesh_matches_oracle(family):
    from paper_1806_11456_b200 import mesh, physics

    msh = mesh.build_rotated_box(3, 3, 2, jitter=0.1, seed=3)
    law = physics.AdvectionDiffusion((0.3, -0.7, 0.5), mu=0.1).with_manufactured(
        lambda x, y, z: np.cos(x + 2 * y - z), lambda x, y, z: 0.0 * x)
    _compare_case(msh, law, _orders("random2_5", msh.num_elements), family, "curl")


def test_transfers_match_reference_golden():
    import torch

    from oracle.fields import OrderField as OO
    from paper_1806_11456_b200 import fields, multigrid

    g = load("transfer")
    fo, co = orders3(g["fine"]), orders3(g["coarse"])
    of_f, of_c = fields.OrderField(fo), fields.OrderField(co)
    t = multigrid.OrderTransfer(of_f, of_c, nv=1, family="LG")
    Qf = _from_oracle(of_f, ref_flat_to_oracle(g["Qf"], OO(fo)))
    Qc = _from_oracle(of_c, ref_flat_to_oracle(g["Qc"], OO(co)))
    assert np.abs(_ref(t.restrict(Qf), OO(co)) - g["restricted"]).max() <= 1e-13
    assert np.abs(_ref(t.prolong(Qc), OO(fo)) - g["prolonged"]).max() <= 1e-13
    out = fields.NodalField.zeros(of_f, 1)
    t.prolong_add(Qc, out)
    assert np.abs(_ref(out, OO(fo)) - g["prolonged"]).max() <= 1e-13
    torch.cuda.synchronize()


def test_host_batch_residual_matches_device_residual_and_oracle():
    """tdg_residual_host (host buffers, double-buffered copies overlapping the
    evaluations) gives, state by state, the device residual bit for bit, the
    oracle's within 1e-12, and max|r| per state."""
    import torch

    from oracle.fields import OrderField as OO
    from oracle.operators import DGOperator as ODG
    from paper_1806_11456_b200 import fields, operators, physics

    msh = _ns_mesh("periodic_jitter")
    law = physics.NavierStokes(mach=0.3, reynolds=100.0)
    orders = _orders("random1_5", msh.num_elements)
    op = operators.DGOperator(msh, law, fields.OrderField(orders), family="LGL", form="curl")
    fs = law.freestream()
    states = []
    for k in range(5):
        Q = op.project_function(lambda x, y, z, k=k: np.stack(
            [fs[v] + 1e-2 * np.sin(2 * np.pi * (x + (k + 1) * y - z) + v) for v in range(5)]))
        states.append(Q)
    hosts = [Q.data.cpu().pin_memory() for Q in states]
    pageable = [Q.data.cpu() for Q in states[:2]]          # pageable buffers work too
    outs, norms = op.residual_host(hosts)
    outs2, norms2 = op.residual_host(pageable)
    of_o = OO(orders)
    oo = ODG(msh, oracle_law(law), of_o, family="LGL", form="curl")
    for k, Q in enumerate(states):
        R = op.residual(Q)
        assert torch.equal(outs[k], R.data.cpu())
        assert norms[k] == float(R.data.abs().max())
        if k < 2:
            assert torch.equal(outs2[k], R.data.cpu()) and norms2[k] == norms[k]
    Qo = oo.project_function(lambda x, y, z: np.stack(
        [fs[v] + 1e-2 * np.sin(2 * np.pi * (x + 3 * y - z) + v) for v in range(5)]))
    scale = oo.m_inv_apply(Qo).norm_inf()
    Rh = fields.NodalField(op.orders, outs[2].cuda(), 5)
    assert (_to_oracle(Rh, of_o) - oo.residual(Qo)).norm_inf() <= RTOL * scale
    assert op.residual_host([]) == ([], [])


@pytest.mark.parametrize("n_f", [7, 6, 5, 4, 3, 2])
def test_line_transfer_kernel_is_bitwise_and_matches_oracle(n_f):
    """Uniform isotropic 5-component level pairs run k_transfer_lines: bit for
    bit the one-output-per-thread kernel (TDG_TRANSFER_LINES=0), and the
    oracle's L2 projection / interpolation (multigrid.py:101-143) to 1e-13."""
    import os

    import torch

    from oracle.fields import NodalField as ON
    from oracle.fields import OrderField as OO
    from oracle.multigrid import OrderTransfer as OT
    from paper_1806_11456_b200 import fields, multigrid

    nel = 12
    of_f, of_c = fields.OrderField.uniform(nel, n_f), fields.OrderField.uniform(nel, n_f - 1)
    os.environ["TDG_TRANSFER_LINES"] = "0"
    try:
        t_ref = multigrid.OrderTransfer(of_f, of_c, nv=5, family="LGL")
    finally:
        del os.environ["TDG_TRANSFER_LINES"]
    t_lin = multigrid.OrderTransfer(of_f, of_c, nv=5, family="LGL")
    g = torch.Generator(device="cuda").manual_seed(n_f)
    rnd = lambda of: fields.NodalField(of, torch.rand(of.num_nodes * 5, dtype=torch.float64, device="cuda",
                                                      generator=g) - 0.5, 5)
    Qf, Qc, Qc0 = rnd(of_f), rnd(of_c), rnd(of_c)
    assert torch.equal(t_lin.restrict(Qf).data, t_ref.restrict(Qf).data)
    assert torch.equal(t_lin.prolong(Qc).data, t_ref.prolong(Qc).data)
    a, b = Qf.copy(), Qf.copy()
    t_lin.prolong_add(Qc, a, Qc0)
    t_ref.prolong_add(Qc, b, Qc0)
    assert torch.equal(a.data, b.data)
    # oracle
    oo_f, oo_c = OO(np.full((nel, 3), n_f)), OO(np.full((nel, 3), n_f - 1))
    ot = OT(oo_f, oo_c, family="LGL")
    of_o = ON(oo_f, Qf.to_oracle_blocks(), 5)
    oc_o = ON(oo_c, Qc.to_oracle_blocks(), 5)
    r_o = ot.restrict(of_o)
    p_o = ot.prolong(oc_o)
    r = ON(oo_c, t_lin.restrict(Qf).to_oracle_blocks(), 5)
    p = ON(oo_f, t_lin.prolong(Qc).to_oracle_blocks(), 5)
    assert (r - r_o).norm_inf() <= 1e-13 * max(r_o.norm_inf(), 1.0)
    assert (p - p_o).norm_inf() <= 1e-13 * max(p_o.norm_inf(), 1.0)


def test_many_small_elements_per_item_match_oracle():
    """A 2D-extruded (1,1,0) Legendre-Gauss plan with 25,600 four-node
    elements: work items are capped at MAX_ITEM_ELEMS = 64 elements (the
    per-element shared-memory reductions of dt, tau and norms), which this
    plan would otherwise exceed (~86 elements per item).  element_dt, tau
    (coupled and isolated) and element norms vs the oracle."""
    from oracle.fields import OrderField as OO
    from oracle.operators import DGOperator as ODG
    from oracle import timestep as ots
    from paper_1806_11456_b200 import fields, mesh, operators, physics, timestep

    msh = mesh.build_box(160, 160, 1, bounds=((0, 1), (0, 1), (0, 0.1)), jitter=0.1,
                         rng=np.random.default_rng(11))
    law = physics.make_case("advdiff-sine")
    orders = np.tile([1, 1, 0], (msh.num_elements, 1))
    op = operators.DGOperator(msh, law, fields.OrderField(orders), family="LG", form="cross")
    oo = ODG(msh, oracle_law(law), OO(orders), family="LG", form="cross")
    Q = op.project_function(lambda x, y, z: 1.0 + 0.5 * np.sin(3 * x + 2 * y) + 0.0 * z)
    Qo = oo.project_function(lambda x, y, z: 1.0 + 0.5 * np.sin(3 * x + 2 * y) + 0.0 * z)
    dt, dto = timestep.element_dt(op, Q, timestep.TimeConfig()), ots.element_dt(oo, Qo, ots.TimeConfig())
    assert np.abs(dt - dto).max() <= 1e-14 * dto.max()
    for iso in (False, True):
        # a smooth field on N=1 elements: F = M A is a small difference of
        # volume and surface terms (measured 7.7e-12 of max tau here), so this
        # check of the item cap (an overflow corrupts values at O(1)) is
        # relative to those terms (oracle term_scale)
        t, to = op.truncation(Q, isolated=iso), oo.truncation(Qo, isolated=iso)
        scale = max(to.max(), oo.term_scale(Qo, isolated=iso))
        assert np.abs(t - to).max() <= 1e-12 * scale
    en = op.element_norms(Q).cpu().numpy()
    assert np.abs(en - Qo.element_norms_inf()).max() == 0.0


def test_reference_objects_drop_in():
    """DGOperator(mesh2d, law, orders2d) with the reference's own object types
    (duck-typed stand-ins) reproduces the reference's golden operator values,
    bit-identical to the explicit extrusion path; FASSolver likewise for the
    golden V-cycle history."""
    import warnings

    import torch

    from helpers import RefStyleAdvDiffSine, RefStyleMesh2D
    from paper_1806_11456_b200 import fields, multigrid, operators

    g, m, plaw, of_p, of_o, op, Q = _golden_setup("op_sine_warp_mixed")
    op2 = operators.DGOperator(RefStyleMesh2D(g), RefStyleAdvDiffSine(), g["orders"])
    assert (op2.family, op2.form) == ("LG", "cross")
    Q2 = fields.NodalField(op2.orders, Q.data.clone(), 1)
    F2 = op2.apply(Q2)
    assert torch.equal(F2.data, op.apply(Q).data)
    assert np.abs(_ref(F2, of_o) - g["F"]).max() <= RTOL * np.abs(g["F"]).max()
    gm = load("mg_vcycle_sine4")
    sm = multigrid.SmootherConfig(pre_sweeps=int(gm["smoother_pre_sweeps"]), post_sweeps=int(gm["smoother_post_sweeps"]),
                                  coarsest_sweeps=int(gm["smoother_coarsest_sweeps"]),
                                  max_batches=int(gm["smoother_max_batches"]))
    s = multigrid.FASSolver(RefStyleMesh2D(gm), RefStyleAdvDiffSine(), gm["orders"], smoother=sm)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(int(gm["log_cycle"].max())):
            s.v_cycle()
    rn = np.array([r["rnorm"] for r in s.log])
    assert np.abs(rn - gm["log_rnorm"]).max() <= 1e-10 * gm["log_rnorm"].max()
