"""Time the UNMODIFIED reference (pure-Python taudg, /root/reference) on its
own 2D scalar analogues of configs 1 and 2, one core.

Build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src OMP_NUM_THREADS=1 python tools/ref_cpu_2d.py

Writes profiles/reference_cpu_2d.json, which bench.py reports verbatim as
``reference_cpu_2d`` (labelled with this container's CPU).
"""
import json
import os
import platform
import time
import warnings

import numpy as np
from taudg import mesh, multigrid, physics
from taudg.fields import NodalField, OrderField
from taudg.operators import DGOperator

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cpu_model():
    with open("/proc/cpuinfo") as fh:
        for line in fh:
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()


def case(nx, ny, n, levels_sweeps, cycles, budget=20.0, seed=0):
    m = mesh.build_cartesian(nx, ny)
    law = physics.make_case("advdiff-sine")
    of = OrderField(np.full((nx * ny, 2), n))
    t = time.perf_counter()
    op = DGOperator(m, law, of)
    build = time.perf_counter() - t
    q = NodalField.zeros(of)
    rng = np.random.default_rng(seed)
    for b in q.blocks:
        b[:] = rng.uniform(0.5, 2.0, b.shape)
    op.residual(q)
    k, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget / 2:
        op.residual(q)
        k += 1
    res_s = (time.perf_counter() - t0) / k
    pre, post, coarse = levels_sweeps
    s = multigrid.FASSolver(m, law, of, smoother=multigrid.SmootherConfig(pre_sweeps=pre, post_sweeps=post,
                                                                          coarsest_sweeps=coarse, max_batches=1))
    s.set_state(q)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s.v_cycle()
        ts = []
        for _ in range(cycles):
            t0 = time.perf_counter()
            s.v_cycle()
            ts.append(time.perf_counter() - t0)
    return {"mesh": f"{nx}x{ny} Cartesian quads", "law": "advdiff-sine (reference manufactured case)",
            "order": n, "dofs": of.dofs(), "operator_build_s": round(build, 3),
            "residual_ms": 1e3 * res_s, "dof_evals_per_s": of.dofs() / res_s, "residual_evals": k,
            "vcycle_ms": 1e3 * float(np.median(ts)), "vcycles": cycles,
            "smoother": {"pre": pre, "post": post, "coarsest": coarse, "max_batches": 1},
            "levels": len(s.levels)}


if __name__ == "__main__":
    out = {"kind": "reference (unmodified taudg from /root/reference, pure Python + NumPy)",
           "where": "build container (no GPU); the reference does not travel to the GPU box",
           "cpu_model": cpu_model(), "python": platform.python_version(), "numpy": np.__version__,
           "cores": 1, "threads_env": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")},
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "cfg1_2d": case(8, 8, 3, (3, 3, 3), 5),
           "cfg2_2d": case(40, 20, 5, (3, 3, 10), 2)}
    path = os.path.join(ROOT, "profiles", "reference_cpu_2d.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))
