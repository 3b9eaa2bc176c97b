"""Invariants that pin the oracle's arithmetic where the reference has no
counterpart (3D, Gauss-Lobatto, orientation codes, Navier-Stokes): free-stream
preservation, polynomial exactness across mortars and every face
orientation, telescoping/conservation, isolated locality, transfer round
trips, RK3 fixed point."""

import numpy as np
import pytest

from helpers import oracle_law
from oracle import multigrid, timestep
from oracle import physics as ophys
from oracle.fields import OrderField
from oracle.operators import DGOperator
from paper_1806_11456_b200 import mesh


def _ns_uniform(law):
    fs = law.freestream()
    return lambda x, y, z: np.stack([fs[i] + 0.0 * x for i in range(5)])


@pytest.mark.parametrize("family", ["LG", "LGL"])
@pytest.mark.parametrize("jitter", [0.0, 0.15])
def test_ns_free_stream_rotated_curved_conforming(family, jitter):
    m = mesh.build_rotated_box(3, 3, 2, seed=3, jitter=jitter, bc={"boundary": "freestream"})
    law = ophys.NavierStokes(mach=0.3, reynolds=100.0)
    op = DGOperator(m, law, OrderField.uniform(m.num_elements, 3), family=family, form="curl")
    q = op.project_function(_ns_uniform(law))
    scale = 1.0 / (law.gamma * law.mach ** 2)        # freestream pressure flux
    assert op.apply(q).norm_inf() < 1e-12 * scale
    assert op.apply(q, isolated=True).norm_inf() < 1e-12 * scale


@pytest.mark.parametrize("family", ["LG", "LGL"])
def test_ns_free_stream_affine_nonconforming(family):
    m = mesh.build_rotated_box(3, 3, 2, seed=5, bc={"boundary": "freestream"})
    law = ophys.NavierStokes(mach=0.3, reynolds=100.0)
    of = OrderField(np.random.default_rng(2).integers(1, 6, (m.num_elements, 3)))
    op = DGOperator(m, law, of, family=family, form="curl")
    q = op.project_function(_ns_uniform(law))
    assert op.apply(q).norm_inf() < 1e-11


@pytest.mark.parametrize("family", ["LG", "LGL"])
def test_polynomial_exactness_mixed_orders_all_orientations(family):
    a, mu = (0.3, -0.7, 0.5), 0.1
    ex = lambda x, y, z: x * x * y + y * y + 2 * x + z * z + x * z
    src = lambda x, y, z: (a[0] * (2 * x * y + 2 + z) + a[1] * (x * x + 2 * y) + a[2] * (2 * z + x)
                           - mu * (2 * y + 2 + 2))
    m = mesh.build_rotated_box(3, 3, 2, seed=3)
    L, SL, R, SR, O = m.face_arrays()
    assert len(set(O[R >= 0].tolist())) == 8          # every orientation code present
    of = OrderField(np.random.default_rng(5).integers(2, 5, (m.num_elements, 3)))
    law = ophys.AdvectionDiffusion(a, mu).with_manufactured(ex, src)
    for form in ("cross", "curl"):
        op = DGOperator(m, law, of, family=family, form=form)
        r = op.residual(op.project_function(ex))
        assert r.norm_inf() < 1e-10


def test_periodic_telescoping_conserves_mass():
    m = mesh.build_box(3, 3, 2, jitter=0.1, rng=np.random.default_rng(1))
    law = ophys.NavierStokes(mach=0.3, reynolds=100.0)
    of = OrderField(np.random.default_rng(3).integers(1, 5, (m.num_elements, 3)))
    op = DGOperator(m, law, of, family="LGL", form="curl")
    rng = np.random.default_rng(9)
    q = op.project_function(_ns_uniform(law))
    for b in q.blocks:
        b *= 1.0 + 0.02 * rng.standard_normal(b.shape)
    F = op.apply(q)
    total = sum(float(b[:, 0].sum()) for b in F.blocks)        # sum of continuity rows
    scale = max(float(np.abs(b[:, 0]).max()) for b in F.blocks)
    assert abs(total) < 1e-12 * scale * of.dofs()


def test_isolated_operator_is_element_local():
    m = mesh.build_box(3, 2, 2, jitter=0.1, rng=np.random.default_rng(4))
    law = ophys.NavierStokes(mach=0.3, reynolds=100.0)
    of = OrderField(np.random.default_rng(6).integers(1, 5, (m.num_elements, 3)))
    op = DGOperator(m, law, of, family="LGL", form="curl")
    q = op.project_function(_ns_uniform(law))
    base = op.apply(q, isolated=True).element(4).copy()
    for e in (0, 3, 5, 7):
        q.element(e)[...] *= 1.01
    after = op.apply(q, isolated=True).element(4)
    assert np.abs(after - base).max() < 1e-13 * np.abs(base).max()


@pytest.mark.parametrize("family", ["LG", "LGL"])
def test_transfer_round_trip_3d(family):
    fine = OrderField(np.random.default_rng(1).integers(2, 7, (5, 3)))
    coarse = OrderField(np.maximum(fine.orders - 1, 1))
    t = multigrid.OrderTransfer(fine, coarse, family)
    from oracle.fields import NodalField

    qc = NodalField.zeros(coarse, 5)
    for b in qc.blocks:
        b[:] = np.random.default_rng(2).standard_normal(b.shape)
    back = t.restrict(t.prolong(qc))
    assert (back - qc).norm_inf() < 1e-12


def test_rk3_exact_discrete_solution_is_fixed_point():
    m = mesh.build_box(2, 2, 2, jitter=0.05, rng=np.random.default_rng(0))
    law = ophys.NavierStokes(mach=0.3, reynolds=100.0)
    of = OrderField.uniform(m.num_elements, 2)
    op = DGOperator(m, law, of, family="LGL", form="curl")
    q = op.project_function(_ns_uniform(law))
    for b in q.blocks:
        b *= 1.0 + 0.01 * np.random.default_rng(1).standard_normal(b.shape)
    S = op.m_inv_apply(q)                       # q is the exact discrete solution for S
    q2 = q.copy()
    dt = timestep.compute_dt(op, q2, timestep.TimeConfig())
    timestep.rk3_step(op, q2, dt, source=S)
    assert (q2 - q).norm_inf() < 1e-12


def test_rk3_is_third_order_for_linear_ode():
    """RK3 on dQ/dt = S - A(Q) with a linear operator reproduces the Taylor
    polynomial 1 + z + z^2/2 + z^3/6 (timestep.py:18-20 coefficients)."""
    a = np.array(timestep.RK_A)
    b = np.array(timestep.RK_B)
    lam = -0.37
    q, g = 1.0, 0.0
    for k in range(3):
        r = lam * q
        g = r if k == 0 else a[k] * g + r
        q += b[k] * 1.0 * g
    assert abs(q - (1 + lam + lam ** 2 / 2 + lam ** 3 / 6)) < 1e-15


def test_level_order_fields_3d_rules():
    of = OrderField(np.array([[3, 5, 2], [4, 4, 4], [1, 2, 7]]))
    lv = multigrid.level_order_fields(of, "high-order")
    assert len(lv) == 7 and lv[-1].same_orders(of)
    assert (lv[0].orders == 1).all()
    lz = multigrid.level_order_fields(of, "high-order", direction=3)
    assert [int(f.orders[2, 2]) for f in lz] == [1, 2, 3, 4, 5, 6, 7]
    assert all((f.orders[:, :2] == of.orders[:, :2]).all() for f in lz)
    lu = multigrid.level_order_fields(of, "uniform")
    assert (lu[-2].orders == np.maximum(of.orders - 1, 1)).all()
    # collapsed direction (N3 = 0 extrusion) is never coarsened
    flat = OrderField(np.array([[3, 2, 0], [2, 3, 0]]))
    assert all((f.orders[:, 2] == 0).all() for f in multigrid.level_order_fields(flat, "high-order"))


def test_wall_and_symmetry_states():
    law = ophys.NavierStokes(mach=0.3, reynolds=100.0)
    q = np.array([[1.1, 0.3, -0.2, 0.1, 20.0]])[..., None]
    n = np.array([[0.0, 1.0, 0.0]])[..., None]
    g = law.bc_riemann_ghost(q, n, "symmetry", None)
    assert np.allclose(g[:, 2], -q[:, 2]) and np.allclose(g[:, [1, 3]], q[:, [1, 3]])
    w = law.bc_riemann_ghost(q, n, "wall", None)
    assert np.allclose(w[:, 1:4], -q[:, 1:4])
    # Roe with the mirrored state has zero mass flux through the wall
    F = law.riemann(q, g, n)
    assert abs(F[0, 0, 0]) < 1e-14
    # consistency: Roe(q, q) = physical normal flux
    fl = law.adv_flux(q)
    Fn = np.einsum("bd...,bdv...->bv...", n, fl)
    assert np.allclose(law.riemann(q, q, n), Fn, atol=1e-13)
