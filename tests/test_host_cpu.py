"""Host-side logic of the product (no GPU): selection / jump limiting against
the reference goldens, multigrid level rules, config builders, mesh
connectivity, and the multi-process (replica) timing reduction over gloo."""

import os

import numpy as np
import pytest

from helpers import golden_mesh, load, orders3
from paper_1806_11456_b200 import adaptation, configs, mesh, multigrid, tau
from paper_1806_11456_b200.fields import OrderField


@pytest.mark.parametrize("name", ["sine4", "aniso5"])
def test_selection_and_limiting_match_reference(name):
    g = load("tau_" + name)
    m = golden_mesh(g)
    of = OrderField(orders3(g["orders"]))
    tm = tau.TauMap(of, tau.EstimationContext(1e5, 0.0, True))
    ref = g["tau_iso"]
    for e in range(of.num_elements):
        for d in range(2):
            for n in range(ref.shape[2]):
                if np.isfinite(ref[e, d, n]):
                    tm.record(e, d + 1, n, ref[e, d, n])
    nmax = int(of.orders.max()) + 2
    tau.extrapolate_map(tm, nmax)
    for k, tmax in enumerate(g["tau_max_list"]):
        sel, rep = adaptation.select_orders(tm, adaptation.AdaptConfig(tau_max=float(tmax), n_max=nmax))
        assert (sel.orders[:, :2] == g[f"select_{k}"]).all()
        assert (sel.orders[:, 2] == 0).all()
        assert [d.path for d in rep.decisions] == list(g[f"select_paths_{k}"])
        assert (adaptation.limit_jumps(m, sel).orders[:, :2] == g[f"limited_{k}"]).all()
        assert (adaptation.limit_jumps(m, sel, "softened").orders[:, :2] == g[f"softened_{k}"]).all()


def test_level_rules_match_oracle():
    from oracle import multigrid as omg
    from oracle.fields import OrderField as OO

    arr = np.random.default_rng(3).integers(1, 8, (40, 3))
    for rule in ("uniform", "high-order"):
        for direction in (None, 1, 2, 3):
            a = multigrid.level_order_fields(OrderField(arr), rule, direction)
            b = omg.level_order_fields(OO(arr), rule, direction)
            assert len(a) == len(b)
            assert all((x.orders == y.orders).all() for x, y in zip(a, b))


def test_limit_jumps_3d_fixed_point_properties():
    m = mesh.build_rotated_box(3, 3, 3, seed=2)
    of = OrderField(np.random.default_rng(0).integers(1, 8, (m.num_elements, 3)))
    for rule in ("strict-one", "softened"):
        lim = adaptation.limit_jumps(m, of, rule)
        assert (lim.orders >= of.orders).all()
        for ea, da, eb, db in adaptation._face_slot_pairs(m):
            a, b = lim.orders[ea, da], lim.orders[eb, db]
            if rule == "strict-one":
                assert abs(a - b) <= 1
            else:
                assert a >= (2 * b) // 3 and b >= (2 * a) // 3


def test_order_field_layout():
    of = OrderField(np.array([[3, 2, 1], [1, 1, 1], [3, 2, 1], [2, 2, 2]]))
    assert of.group_orders == [(1, 1, 1), (2, 2, 2), (3, 2, 1)]
    assert list(of.slot_elem) == [1, 3, 0, 2]
    assert list(of.node_off) == [0, 8, 35, 59, 83]
    assert of.dofs() == 83


def test_config_builders():
    w1 = configs.config1()
    assert w1.orders.num_nodes == 4096 and w1.mesh.num_elements == 64
    w3 = configs.config3(n=8)
    assert w3.mesh.num_elements == 512
    assert w3.orders.orders.min() >= 1 and w3.orders.orders.max() <= 7
    w3b = configs.config3(n=8)
    assert (w3.orders.orders == w3b.orders.orders).all() and np.array_equal(w3.mesh.nodes, w3b.mesh.nodes)
    w4 = configs.config4(n=4, order=3)
    assert w4.orders.num_nodes == 64 * 64
    x = np.linspace(0, 1, 5)
    q = w1.init(x, x, 0 * x)
    assert q.shape == (5, 5) and np.all(q[0] > 0.9)


def test_periodic_box_connectivity():
    m = mesh.build_box(3, 2, 1)
    interior = [f for f in m.faces if not f.is_boundary]
    assert len(interior) == 3 * 6 and not m.boundary_tags
    # self-periodic z: each element meets itself
    assert sum(1 for f in interior if f.left == f.right) == 6
    mb = mesh.build_box(2, 2, 2, periodic=(True, False, True))
    assert set(mb.boundary_tags) == {"south", "north"}


def _replica_worker(rank, world, port, out):
    import torch.distributed as dist

    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v = bench.max_over_ranks(float(rank + 1) * 1.5, dist, "cpu")
    out[rank] = v
    dist.destroy_process_group()


def test_replica_timing_reduction_gloo():
    import torch.multiprocessing as mp

    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + (os.getpid() % 1000)
    mp.spawn(_replica_worker, args=(2, port, out), nprocs=2, join=True)
    assert dict(out) == {0: 3.0, 1: 3.0}


def test_affine_metrics_are_exact_and_shared_with_the_oracle():
    """Affine elements take exact constant curl-form metrics, by the same
    element-wise rule in product and oracle (bit-identical); a jittered
    (trilinear, non-parallelepiped) element keeps its collocated metrics."""
    from oracle import geometry as og
    from paper_1806_11456_b200 import geometry as pg

    box = mesh.build_box(3, 2, 2, bounds=((0.0, 2 * np.pi), (0.0, 1.0), (-1.0, 3.0)))
    jit = mesh.build_box(3, 2, 2, jitter=0.1, rng=np.random.default_rng(2))
    assert pg.affine_map(box.nodes)[0].all() and not pg.affine_map(jit.nodes)[0].any()
    for msh, affine in ((box, True), (jit, False)):
        for fam in ("LGL", "LG"):
            orders = (5, 3, 7)
            jac, ja, _, _ = pg.volume_metrics(msh.nodes, orders, fam, "curl")
            for e in range(msh.num_elements):
                j2, a2, _ = og.volume_metrics(msh.nodes[e], orders, fam, "curl", e)
                assert np.array_equal(j2, jac[e]) and np.array_equal(a2, ja[e])
            flat = ja.reshape(len(ja), 9, -1)
            spread = np.abs(flat - flat[:, :, :1]).max()
            assert (spread == 0.0) == affine
    # exact values: a box element of sides (hx, hy, hz) has J = hx hy hz / 8,
    # Ja^i = (h_j h_k / 4) e_i
    jac, ja, _, _ = pg.volume_metrics(box.nodes, (2, 2, 2), "LGL", "curl")
    h = np.array([2 * np.pi / 3, 0.5, 2.0])
    assert np.allclose(jac, np.prod(h) / 8, rtol=1e-15, atol=0)
    for i in range(3):
        j, k = (i + 1) % 3, (i + 2) % 3
        assert np.allclose(ja[:, i, i], h[j] * h[k] / 4, rtol=1e-15, atol=0)
        assert (ja[:, i, j] == 0).all() and (ja[:, i, k] == 0).all()


@pytest.mark.parametrize("k", [0, 1, 2])
@pytest.mark.parametrize("rule", [None, "strict-one", "softened"])
def test_conforming_pass_matches_reference(k, rule):
    """conforming_pass (adaptation.py:212-250) on the reference's own golden
    case (graded 5x4 mesh, three tag sets), product and oracle."""
    from oracle import adaptation as oad
    from oracle.fields import OrderField as OO

    g = load("conforming")
    m = golden_mesh(g)
    orders = orders3(g["orders_in"])
    tags = tuple(str(t) for t in g[f"tags_{k}"])
    want = g[{None: "share", "strict-one": "strict", "softened": "soft"}[rule] + f"_{k}"]
    got = adaptation.conforming_pass(m, OrderField(orders), tags, rule)
    assert (got.orders[:, :2] == want).all()
    assert (got.orders[:, 2] == 0).all()
    assert (oad.conforming_pass(m, OO(orders), tags, rule).orders[:, :2] == want).all()


@pytest.mark.parametrize("builder", ["rotated_box", "cubed_sphere"])
def test_conforming_pass_3d_matches_oracle(builder):
    """3D meshes whose boundary elements are rotated against each other
    (every orientation code; the six cubed-sphere panels): the product's
    frame-transported sharing equals the oracle's, is idempotent, and with a
    jump rule leaves every interior face within the rule."""
    from oracle import adaptation as oad
    from oracle.fields import OrderField as OO

    if builder == "rotated_box":
        m = mesh.build_rotated_box(3, 3, 2, seed=5)
        tags = ("boundary",)
    else:
        m = mesh.build_cubed_sphere(2, 2, 0.5, 2.0, 1.15)
        tags = tuple(sorted(m.boundary_tags))[:1]
    arr = np.random.default_rng(7).integers(1, 7, (m.num_elements, 3))
    for rule in (None, "strict-one"):
        got = adaptation.conforming_pass(m, OrderField(arr), tags, rule)
        ref = oad.conforming_pass(m, OO(arr), tags, rule)
        assert (got.orders == ref.orders).all()
        assert (got.orders >= arr).all()
        again = adaptation.conforming_pass(m, got, tags, rule)
        assert (again.orders == got.orders).all()
        if rule:
            for ea, da, eb, db in adaptation._face_slot_pairs(m):
                assert abs(int(got.orders[ea, da]) - int(got.orders[eb, db])) <= 1


def test_reference_objects_are_lifted_literally():
    """compat.resolve: the reference's 2D mesh, (N1, N2) orders and 2D law
    become the N3 = 0 extrusion with LG nodes and cross metrics; 3D inputs keep
    LGL / curl."""
    from helpers import RefStyleAdvDiffSine, RefStyleMesh2D
    from paper_1806_11456_b200 import compat, physics

    g = load("op_sine_warp_mixed")
    ref_mesh = RefStyleMesh2D(g)
    hexm, law, of, fam, form = compat.resolve(ref_mesh, RefStyleAdvDiffSine(), g["orders"])
    assert (fam, form) == ("LG", "cross")
    assert (of.orders[:, 2] == 0).all() and (of.orders[:, :2] == g["orders"]).all()
    ext = golden_mesh(g)
    assert np.array_equal(hexm.nodes, ext.nodes)
    assert [tuple(a) for a in zip(*hexm.face_arrays())] == [tuple(a) for a in zip(*ext.face_arrays())]
    assert compat.as_hex_mesh(ref_mesh) is hexm                       # cached
    assert isinstance(law, physics.AdvectionDiffusion) and law.velocity == (1.0, 1.0, 0.0)
    assert law.exact(np.array([0.25]), np.array([0.5]), np.array([7.0]))[0] == np.sin(np.pi / 4)
    assert compat.resolve(ext, law, of)[3:] == ("LGL", "curl")
