"""Operator contract on the GPU path (through the C-ABI), mirroring the
reference's own operator tests and error behaviour:

- a field of another OrderField instance is rejected with ValueError
  (operators.py:271-272), an inverted element with MeshError (mesh.py:148-158),
  a non-finite state during smoothing with DivergedError (timestep.py:135-139);
- isolated evaluation is element-local and coupled evaluation reaches the
  face neighbours and, through BR1's lifted gradient, no further than their
  face neighbours (tests/test_operators.py:196-225);
- repeated evaluations and tau estimates are bit-identical (tests/test_tau.py:
  144-148), and the ``calls`` counters follow the reference's contract
  (operators.py:94, tests/test_tau.py:227-272).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ns_setup(nx=3, ny=3, nz=2, seed=5, lo=1, hi=4):
    from paper_1806_11456_b200 import fields, mesh, operators, physics

    msh = mesh.build_box(nx, ny, nz, jitter=0.1, rng=np.random.default_rng(seed))
    law = physics.NavierStokes(mach=0.3, reynolds=100.0)
    orders = np.random.default_rng(seed + 1).integers(lo, hi + 1, (msh.num_elements, 3))
    of = fields.OrderField(orders)
    op = operators.DGOperator(msh, law, of, family="LGL", form="curl")
    fs = law.freestream()

    def init(x, y, z):
        return np.stack([fs[v] + 1e-2 * np.sin(2 * np.pi * (x + 2 * y - z) + v) for v in range(5)])

    return msh, law, orders, op, op.project_function(init)


def _element_blocks(op, X):
    """Per-element max |X| (host), by element id."""
    return op.element_norms(X).cpu().numpy()


def test_foreign_field_and_wrong_unknowns_are_rejected():
    from paper_1806_11456_b200 import fields

    msh, law, orders, op, Q = _ns_setup()
    other = fields.NodalField.zeros(fields.OrderField(orders), 5)   # same orders, other instance
    with pytest.raises(ValueError):
        op.apply(other)
    with pytest.raises(ValueError):
        op.residual(other)
    scalar = fields.NodalField.zeros(op.orders, 1)
    with pytest.raises(ValueError):
        op.apply(scalar)


def test_inverted_element_raises_mesh_error():
    from paper_1806_11456_b200 import errors, fields, mesh, operators, physics

    msh = mesh.build_box(2, 2, 2)
    msh.nodes[3] = msh.nodes[3][::-1].copy()     # mirror element 3 in xi: J < 0
    law = physics.NavierStokes(mach=0.3, reynolds=100.0)
    with pytest.raises(errors.MeshError):
        operators.DGOperator(msh, law, fields.OrderField(np.full((8, 3), 2)), family="LGL", form="curl")


def test_non_finite_state_raises_diverged_error():
    import torch

    from paper_1806_11456_b200 import errors, timestep

    msh, law, orders, op, Q = _ns_setup()
    Q.data[17] = float("nan")
    with pytest.raises(errors.DivergedError):
        timestep.smooth(op, Q, 2, timestep.TimeConfig())
    torch.cuda.synchronize()


def test_isolated_is_element_local_and_coupled_stencil_is_the_br1_two_ring():
    msh, law, orders, op, Q = _ns_setup(5, 5, 3)
    e0 = 12                                         # 5x5x3 periodic box: the two-ring is a strict subset
    base_iso, base_cpl = op.apply(Q, isolated=True), op.apply(Q)
    P = Q.copy()
    blk = P.element(e0)
    blk += 1e-3 * (1.0 + torch_arange_like(blk))
    d_iso = _element_blocks(op, op.apply(P, isolated=True) - base_iso)
    d_cpl = _element_blocks(op, op.apply(P) - base_cpl)
    changed_iso = set(np.nonzero(d_iso > 0)[0].tolist())
    changed_cpl = set(np.nonzero(d_cpl > 0)[0].tolist())
    assert changed_iso == {e0}
    def ring(es):
        return set(es) | {f.right if f.left == e else f.left for e in es for _, f in msh.faces_of_element(e)}

    # BR1: the neighbours' lifted gradients see e0's trace, and their viscous
    # face fluxes reach the next layer: the stencil is the two-ring, and
    # every face neighbour is reached
    one, two = ring({e0}), ring(ring({e0}))
    assert one <= changed_cpl <= two
    assert len(one) == 7 and len(two) < msh.num_elements


def torch_arange_like(x):
    import torch

    return torch.arange(x.numel(), dtype=x.dtype, device=x.device).reshape(x.shape) / x.numel()


def test_repeated_evaluations_and_tau_are_bit_identical():
    import torch

    msh, law, orders, op, Q = _ns_setup()
    r1, r2 = op.residual(Q), op.residual(Q)
    assert torch.equal(r1.data, r2.data)
    for iso in (False, True):
        t1, t2 = op.truncation(Q, isolated=iso), op.truncation(Q, isolated=iso)
        assert np.array_equal(t1, t2)


def test_call_counters_follow_the_reference_contract():
    msh, law, orders, op, Q = _ns_setup()
    op.calls.update(apply=0, apply_isolated=0)
    op.apply(Q)
    op.residual(Q)
    op.m_inv_apply(Q, isolated=True)
    op.truncation(Q, isolated=True)
    assert op.calls == {"apply": 2, "apply_isolated": 2}
