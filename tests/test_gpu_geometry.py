"""Device construction of the invariant-curl metrics (SURVEY §8f.2,
tdg_volume_metrics) against the host build (geometry.volume_metrics, the
arithmetic the oracle shares), on trilinear jittered, cubed-sphere (mapping
order 3) and affine meshes, LGL and LG, isotropic and anisotropic orders."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cases():
    from paper_1806_11456_b200 import mesh

    rng = np.random.default_rng(4)
    yield "jittered", mesh.build_box(3, 3, 2, jitter=0.1, rng=rng), [(1, 1, 1), (3, 5, 2), (7, 7, 7), (4, 2, 6)]
    yield "sphere", mesh.build_cubed_sphere(2, 2, 0.5, 2.0, 1.15, mapping_order=3), [(3, 3, 3), (5, 4, 6)]
    yield "affine", mesh.build_box(2, 2, 2, bounds=((0, 2.0), (0, 1.0), (0, 0.5))), [(7, 7, 7), (2, 3, 4)]


@pytest.mark.parametrize("family", ["LGL", "LG"])
def test_device_metrics_bit_identical_to_host_and_oracle(family):
    """J, Ja, sizes and node coordinates from the kernel equal the host build
    bit for bit, and the oracle's per-element build (oracle/geometry.py) too —
    sizes there to a few ulp: the oracle's LGL weight tables differ from the
    product's by 1 ulp at N = 4, 6, 7."""
    from oracle import geometry as og
    from paper_1806_11456_b200 import geometry

    for name, msh, orders_list in _cases():
        for orders in orders_list:
            nodes = msh.nodes
            h = geometry.volume_metrics(nodes, orders, family, "curl")
            d = geometry.volume_metrics(nodes, orders, family, "curl", device="cuda")
            for a, b, what in zip(h, d, ("jac", "ja", "sizes", "coords")):
                assert np.array_equal(a, b), f"{name} {orders} {family} {what}: device != host"
            for e in range(msh.num_elements):
                jo, ao, so = og.volume_metrics(nodes[e], orders, family, "curl", e)
                assert np.array_equal(d[0][e], jo) and np.array_equal(d[1][e], ao)
                assert np.abs(d[2][e] - so).max() <= 1e-15 * np.abs(so).max()


def test_operator_with_device_metrics_matches_oracle():
    """The DGOperator plan built from device metrics reproduces the oracle's
    residual (host metrics) on a curved mixed-order mesh at 1e-12."""
    from oracle.fields import OrderField as OO
    from oracle.operators import DGOperator as ODG
    from paper_1806_11456_b200 import configs, operators
    from helpers import oracle_law

    w = configs.config3(n=4)
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    oo = ODG(w.mesh, oracle_law(w.law), OO(np.asarray(w.orders.orders)), family=w.family, form=w.form)
    Q, Qo = op.project_function(w.init), oo.project_function(w.init)
    from oracle.fields import NodalField as ON

    R = ON(oo.orders, op.residual(Q).to_oracle_blocks(), 5)
    R.field = oo.orders
    assert (R - oo.residual(Qo)).norm_inf() <= 1e-12 * oo.m_inv_apply(Qo).norm_inf()
