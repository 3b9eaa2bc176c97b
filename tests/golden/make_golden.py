"""Generate golden vectors by running the REAL reference package.

Run in the build container only (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/ref_*.npz.  Every case records the reference's 2D mesh
(control nodes, faces with flip flags, boundary tags), the per-element orders,
the manufactured-case name/parameters, the seeded inputs and the reference's
outputs.  Nodal fields are stored element by element in the reference's
(n1+1, n2+1) xi-slowest layout, concatenated in element order.

The oracle (and, through it, the CUDA path) reproduces these through the
one-element-deep N3=0 Legendre-Gauss extrusion.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

from taudg import mesh, multigrid, physics, spectral, tau, timestep  # noqa: E402
from taudg import adaptation as ad
from taudg.fields import NodalField, OrderField
from taudg.operators import DGOperator

OUT = os.path.dirname(os.path.abspath(__file__))


def _warp(x, y):
    s = np.sin(np.pi * x) * np.sin(np.pi * y)
    return x + 0.06 * s, y + 0.07 * s


def mesh_arrays(m):
    nodes = np.stack([el.nodes for el in m.elements])
    faces = np.array([(f.left, f.side_left, f.right, f.side_right, int(f.flip)) for f in m.faces])
    tag_names = sorted(m.boundary_tags)
    tag_faces = [np.array(m.boundary_tags[t]) for t in tag_names]
    out = {"nodes2d": nodes, "faces2d": faces, "tag_names": np.array(tag_names)}
    for i, t in enumerate(tag_faces):
        out[f"tag_{i}"] = t
    return out


def flat(field: NodalField):
    return np.concatenate([field.element(e).ravel() for e in range(field.field.num_elements)])


def random_field(of, seed, lo=0.5, hi=2.0):
    rng = np.random.default_rng(seed)
    q = NodalField.zeros(of)
    for b in q.blocks:
        b[:] = rng.uniform(lo, hi, b.shape)
    return q


def save(name, **arrays):
    path = os.path.join(OUT, f"ref_{name}.npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path)


def spectral_case():
    out = {}
    for n in range(0, 9):
        q = spectral.gauss_nodes(n)
        out[f"x_{n}"] = q.nodes
        out[f"w_{n}"] = q.weights
        out[f"D_{n}"] = spectral.differentiation_matrix(n)
        out[f"B_{n}"] = spectral.boundary_rows(n)
    for a in range(0, 8):
        for b in range(0, 8):
            out[f"T_{a}_{b}"] = spectral.l2_projection(a, b)
    save("spectral", **out)


OP_CASES = {
    "sine_warp_mixed": dict(
        mesh=lambda: mesh.build_cartesian(2, 2, mapping_order=(2, 2), warp=_warp),
        case="advdiff-sine", params={}, orders=[[3, 3], [4, 3], [3, 5], [4, 4]], seed=4),
    "burgers_mixed": dict(
        mesh=lambda: mesh.build_cartesian(2, 2),
        case="burgers-tanh", params={}, orders=[[3, 2], [4, 4], [2, 5], [3, 3]], seed=3),
    "rotated_pair": dict(
        mesh=lambda: mesh.build_from_arrays(
            [[0, 0], [1, 0], [1, 1], [0, 1], [2, 0], [2, 1]], [[0, 1, 2, 3], [2, 1, 4, 5]]),
        case="advdiff-sine", params={}, orders=[[3, 4], [5, 2]], seed=6),
    "graded_bl": dict(
        mesh=lambda: mesh.build_cartesian(3, 4, grading=("south", 1.3)),
        case="advdiff-boundary-layer", params={}, orders=[[4, 4]] * 12, seed=7),
    "runge_curved": dict(
        mesh=lambda: mesh.build_cartesian(3, 2, mapping_order=(3, 3), warp=_warp),
        case="advdiff-runge", params={},
        orders=np.random.default_rng(8).integers(3, 7, (6, 2)).tolist(), seed=8),
    "aniso_burgers_curved": dict(
        mesh=lambda: mesh.build_cartesian(2, 3, mapping_order=(2, 2), warp=_warp),
        case="burgers-tanh", params={"mu": 0.05},
        orders=np.random.default_rng(9).integers(2, 7, (6, 2)).tolist(), seed=9),
}


def op_case(name, spec):
    m = spec["mesh"]()
    law = physics.make_case(spec["case"], **spec["params"])
    of = OrderField(np.array(spec["orders"]))
    op = DGOperator(m, law, of)
    q = random_field(of, spec["seed"])
    F = op.apply(q)
    Fi = op.apply(q, isolated=True)
    R = op.residual(q)
    A = op.m_inv_apply(q)
    tau_c = op.truncation(q)
    tau_i = op.truncation(q, isolated=True)
    mass = np.concatenate([op.group_ops[of.element_slot[e][0]].mass[of.element_slot[e][1]].ravel()
                           for e in range(of.num_elements)])
    # RK3: two global-dt steps and one local-dt step from the same state
    tcfg = timestep.TimeConfig()
    dts = timestep.element_dt(op, q, tcfg)
    Qrk = q.copy()
    r0 = []
    for _ in range(2):
        dt = timestep.compute_dt(op, Qrk, tcfg)
        r0.append(timestep.rk3_step(op, Qrk, dt))
    Qloc = q.copy()
    dtl = timestep.compute_dt(op, Qloc, timestep.TimeConfig(local=True))
    r0l = timestep.rk3_step(op, Qloc, dtl)
    save(f"op_{name}", case=spec["case"], params=str(spec["params"]), orders=of.orders,
         Q=flat(q), F=flat(F), Fiso=flat(Fi), R=flat(R), A=flat(A), S=flat(op.source),
         tau=tau_c, tau_iso=tau_i, mass=mass, element_dt=dts,
         Q_rk2=flat(Qrk), r0_rk2=np.array(r0), Q_rk_local=flat(Qloc), r0_local=r0l,
         **mesh_arrays(m))


def transfer_case():
    rng = np.random.default_rng(12)
    fine = OrderField(rng.integers(2, 7, (6, 2)))
    coarse = OrderField(np.maximum(fine.orders - 1, 1))
    t = multigrid.OrderTransfer(fine, coarse)
    q = random_field(fine, 13)
    qc = random_field(coarse, 14)
    out = NodalField.zeros(fine)
    t.prolong_add(qc, out)
    save("transfer", fine=fine.orders, coarse=coarse.orders, Qf=flat(q), Qc=flat(qc),
         restricted=flat(t.restrict(q)), prolonged=flat(t.prolong(qc)))


MG_CASES = {
    "vcycle_sine4": dict(nx=2, ny=2, case="advdiff-sine", order=4, cycles=3,
                         smoother=dict(pre_sweeps=4, post_sweeps=4, coarsest_sweeps=10, max_batches=1)),
    "vcycle_burgers3": dict(nx=2, ny=2, case="burgers-tanh", order=3, cycles=3,
                            smoother=dict(pre_sweeps=3, post_sweeps=3, coarsest_sweeps=6, max_batches=1)),
    "vcycle_sine3_tuned": dict(nx=2, ny=2, case="advdiff-sine", order=3, cycles=2,
                               smoother=dict(pre_sweeps=5, post_sweeps=5, coarsest_sweeps=20, max_batches=3)),
}


def mg_case(name, spec):
    m = mesh.build_cartesian(spec["nx"], spec["ny"])
    law = physics.make_case(spec["case"])
    of = OrderField.uniform(m.num_elements, spec["order"])
    solver = multigrid.FASSolver(m, law, of, smoother=multigrid.SmootherConfig(**spec["smoother"]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        for _ in range(spec["cycles"]):
            solver.v_cycle()
    log = solver.log
    save(f"mg_{name}", case=spec["case"], orders=of.orders,
         log_level=np.array([r["level"] for r in log]),
         log_phase=np.array([r["phase"] for r in log]),
         log_sweeps=np.array([r["sweeps"] for r in log]),
         log_rnorm=np.array([r["rnorm"] for r in log]),
         log_cycle=np.array([r["cycle"] for r in log]),
         work_units=solver.work_units, Q=flat(solver.Q), **mesh_arrays(m),
         **{f"smoother_{k}": v for k, v in spec["smoother"].items()})


def tau_case():
    for name, case, nx, ny, order in (("sine4", "advdiff-sine", 2, 2, 4),
                                      ("aniso5", "advdiff-aniso", 3, 2, 5)):
        m = mesh.build_cartesian(nx, ny)
        law = physics.make_case(case)
        of = OrderField.uniform(m.num_elements, order)
        op = DGOperator(m, law, of)
        Q = op.project_function(law.exact)
        out = {}
        for iso in (True, False):
            tm = tau.estimate(m, law, Q, 1e6, isolated=iso, fine_op=op)
            arr = np.full((of.num_elements, 2, order + 1), np.nan)
            for e in range(of.num_elements):
                for d in range(2):
                    for n, v in tm.tau[e][d].items():
                        arr[e, d, n] = v
            out[f"tau_{'iso' if iso else 'coupled'}"] = arr
            if iso:
                nmax = order + 2
                tau.extrapolate_map(tm, nmax)
                ext = np.full((of.num_elements, 2, nmax + 1), np.nan)
                for e in range(of.num_elements):
                    for d in range(2):
                        for n, v in tm.tau[e][d].items():
                            ext[e, d, n] = v
                out["tau_extrap"] = ext
                for k, tmax in enumerate((1e-2, 1e-4, 1e-6)):
                    cfg = ad.AdaptConfig(tau_max=tmax, n_max=nmax)
                    sel, rep = ad.select_orders(tm, cfg)
                    out[f"select_{k}"] = sel.orders
                    out[f"select_paths_{k}"] = np.array([d.path for d in rep.decisions])
                    out[f"limited_{k}"] = ad.limit_jumps(m, sel).orders
                    out[f"softened_{k}"] = ad.limit_jumps(m, sel, "softened").orders
                out["tau_max_list"] = np.array([1e-2, 1e-4, 1e-6])
        save(f"tau_{name}", case=case, orders=of.orders, Q=flat(Q), **out, **mesh_arrays(m))


ADAPT_CASES = {
    "single_sine_p4": dict(stages=(4,), tau_max=1e-2, n_max=6, final_tol=1e-9),
    "multi_sine_2_4": dict(stages=(2, 4), tau_max=1e-5, n_max=6, final_tol=1e-8),
}


def adapt_case(name, spec):
    m = mesh.build_cartesian(2, 2)
    law = physics.make_case("advdiff-sine")
    cfg = ad.AdaptConfig(tau_max=spec["tau_max"], n_max=spec["n_max"], stages=spec["stages"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        run = ad.run_multi_stage(m, law, cfg, final_tol=spec["final_tol"])
    out = {"final_orders": run.orders.orders, "Q": flat(run.Q), "work_units": run.work_units,
           "nreports": len(run.reports), "stages": np.array(spec["stages"]), "tau_max": spec["tau_max"],
           "n_max": spec["n_max"], "final_tol": spec["final_tol"]}
    for i, rep in enumerate(run.reports):
        out[f"rep{i}_new"] = np.array([d.new_orders for d in rep.decisions])
        out[f"rep{i}_paths"] = np.array([d.path for d in rep.decisions])
        out[f"rep{i}_pred"] = np.array([d.predicted_tau for d in rep.decisions])
        out[f"rep{i}_dofs"] = np.array([rep.dofs_before, rep.dofs_after])
    save(f"adapt_{name}", case="advdiff-sine", **out, **mesh_arrays(m))


def conforming_case():
    """conforming_pass (adaptation.py:212-250): tag-max sharing alone and
    alternated with both jump rules, on a graded mesh with random orders."""
    m = mesh.build_cartesian(5, 4, grading=("south", 1.2))
    rng = np.random.default_rng(21)
    of = OrderField(rng.integers(1, 7, (m.num_elements, 2)))
    out = {"orders_in": of.orders}
    for k, tags in enumerate((("south",), ("south", "north"), ("west", "east", "north"))):
        out[f"tags_{k}"] = np.array(tags)
        out[f"share_{k}"] = ad.conforming_pass(m, of, tags).orders
        out[f"strict_{k}"] = ad.conforming_pass(m, of, tags, "strict-one").orders
        out[f"soft_{k}"] = ad.conforming_pass(m, of, tags, "softened").orders
    save("conforming", **out, **mesh_arrays(m))


def main():
    np.set_printoptions(precision=3)
    if len(sys.argv) > 1:        # named cases only, e.g. `make_golden.py conforming`
        for name in sys.argv[1:]:
            globals()[f"{name}_case"]()
        return
    spectral_case()
    for name, spec in OP_CASES.items():
        op_case(name, spec)
    transfer_case()
    for name, spec in MG_CASES.items():
        mg_case(name, spec)
    tau_case()
    for name, spec in ADAPT_CASES.items():
        adapt_case(name, spec)
    conforming_case()


if __name__ == "__main__":
    if "taudg" not in sys.modules:
        pass
    main()
