"""Generate BASELINE-size parity fixtures by running the CPU ORACLE (oracle/)
on the full BASELINE.json configurations.

Run in the build container (it needs no GPU and no reference tree; the oracle
itself is pinned against the real reference by make_golden.py's vectors):

    python tests/golden/make_config_fixtures.py cfg3 cfg3_tau cfg4 cfg4_vcycle cfg2 cfg5

Each part writes tests/golden/oracle_<part>.npz.  Inputs are the seeded
configurations of paper_1806_11456_b200.configs (bit-identical on both
sides: test_gpu_operator checks project_function bitwise).  Full-size
fields are stored as per-element summaries plus a seeded element sample
(tests/fullsize.py).  Oracle wall times on this container (8 cores, one
used): cfg3 operator build 101 s, one residual 88 s.
"""

from __future__ import annotations

import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from fullsize import field_summary, sample_elements, tau_dense  # noqa: E402
from helpers import oracle_law  # noqa: E402
from oracle import adaptation as oad  # noqa: E402
from oracle import multigrid as omg  # noqa: E402
from oracle import tau as otau  # noqa: E402
from oracle import timestep as ots  # noqa: E402
from oracle.fields import OrderField as OO  # noqa: E402
from oracle.operators import DGOperator as ODG  # noqa: E402
from paper_1806_11456_b200 import configs  # noqa: E402


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


SMOKE = os.environ.get("FIXTURE_SMOKE") == "1"   # tiny meshes, output to /tmp (script check)


def save(part, **kw):
    path = os.path.join("/tmp" if SMOKE else HERE, f"oracle_{part}.npz")
    np.savez_compressed(path, **kw)
    log(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


def _setup(w):
    law = oracle_law(w.law)
    of = OO(np.asarray(w.orders.orders))
    t = time.time()
    op = ODG(w.mesh, law, of, family=w.family, form=w.form)
    log(f"  operator build {time.time() - t:.1f} s ({of.dofs()} nodes)")
    return law, of, op, op.project_function(w.init)


def _log_arrays(slog):
    return {"log_level": np.array([r["level"] for r in slog]),
            "log_phase": np.array([r["phase"] for r in slog]),
            "log_sweeps": np.array([r["sweeps"] for r in slog]),
            "log_rnorm": np.array([r["rnorm"] for r in slog])}


def part_cfg3():
    """32^3 jittered box, orders U{1..7}^3: residual, one RK3 step, element tau."""
    w = configs.config3(n=3 if SMOKE else 32)
    law, of, oo, Q0 = _setup(w)
    samp = sample_elements(of.num_elements, seed=3)
    out = {"sample": samp}
    out.update(field_summary("Q0", of, Q0.blocks, samp))
    t = time.time()
    A = oo.m_inv_apply(Q0)
    log(f"  m_inv_apply {time.time() - t:.1f} s")
    out["A_norm"] = A.norm_inf()
    out["F_norm"] = oo.apply(Q0).norm_inf()
    r = oo.residual(Q0)
    out["r_norm"] = r.norm_inf()
    out.update(field_summary("r", of, r.blocks, samp))
    for iso in (False, True):
        out[f"tau_elem_{int(iso)}"] = oo.truncation(Q0, isolated=iso)
    cfg = ots.TimeConfig()
    dt = ots.compute_dt(oo, Q0, cfg)
    Q1 = Q0.copy()
    out["rk_r0"] = ots.rk3_step(oo, Q1, dt)
    out["rk_dt"] = dt
    out.update(field_summary("dQ", of, (Q1 - Q0).blocks, samp))
    log("  cfg3 done")
    save("cfg3", **out)


def part_cfg3_tau():
    """Config 3's one tau estimation (isolated, gate bypassed as config 1)."""
    w = configs.config3(n=3 if SMOKE else 32)
    law, of, oo, Q0 = _setup(w)
    t = time.time()
    tm = otau.estimate(w.mesh, law, Q0, 1e6, isolated=True, fine_op=oo, family=w.family, form=w.form)
    log(f"  tau.estimate {time.time() - t:.1f} s")
    save("cfg3_tau", tau=tau_dense(tm, of.num_elements), work_units=tm.work_units,
         rnorm=tm.context.residual_norm, F_norm=oo.apply(Q0, isolated=True).norm_inf())


def part_cfg4():
    """24^3 N=7: fine residual and every restriction / prolongation pair."""
    w = configs.config4(n=2 if SMOKE else 24)
    law, of, oo, Q0 = _setup(w)
    samp = sample_elements(of.num_elements, seed=4, k=8)
    out = {"sample": samp}
    out.update(field_summary("Q0", of, Q0.blocks, samp))
    A = oo.m_inv_apply(Q0)
    out["A_norm"] = A.norm_inf()
    r = oo.residual(Q0)
    out["r_norm"] = r.norm_inf()
    out.update(field_summary("r", of, r.blocks, samp))
    fields = omg.level_order_fields(of, "high-order")
    X = Q0
    for k in range(len(fields) - 1, 0, -1):
        t = omg.OrderTransfer(fields[k], fields[k - 1], w.family)
        Xc = t.restrict(X)
        n = int(fields[k].orders[0, 0])
        out.update(field_summary(f"R{n}", fields[k - 1], Xc.blocks, samp))
        out.update(field_summary(f"P{n}", fields[k], t.prolong(Xc).blocks, samp))
        out[f"R{n}_norm"] = Xc.norm_inf()
        X = Xc
    log("  cfg4 done")
    save("cfg4", **out)


def part_cfg4_vcycle():
    """Config 4's protocol (7 levels, 2/2/2 pinned sweeps) on an 8^3 box: 3 cycles."""
    w = configs.config4(n=2 if SMOKE else 8)
    law = oracle_law(w.law)
    so = omg.FASSolver(w.mesh, law, OO(np.asarray(w.orders.orders)), smoother=omg.SmootherConfig(**w.smoother),
                       family=w.family, form=w.form)
    so.set_state(so.finest.op.project_function(w.init))
    samp = sample_elements(w.mesh.num_elements, seed=8)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for c in range(3):
            t = time.time()
            so.v_cycle()
            log(f"  cycle {c}: {time.time() - t:.1f} s")
    out = {"sample": samp, "work_units": so.work_units, "Q_norm": so.Q.norm_inf()}
    out.update(_log_arrays(so.log))
    out.update(field_summary("Q", so.Q.field, so.Q.blocks, samp))
    save("cfg4_vcycle", **out)


def _select(w, law, tm, tau_max, n_max, of):
    otau.extrapolate_map(tm, n_max)
    sel, _, _ = oad.select_orders(tm, oad.AdaptConfig(tau_max=tau_max, n_max=n_max))
    lim = oad.limit_jumps(w.mesh, sel)
    return {"tau_ext": tau_dense(tm, of.num_elements), "sel_orders": np.asarray(sel.orders),
            "lim_orders": np.asarray(lim.orders), "tau_max": tau_max, "n_max": n_max}


def part_cfg2():
    """40x20 N=5 flat plate: 2 five-level V-cycles, then tau (Nz frozen) and the
    p-map (tau_max 1e-4, orders 1..5) from the oracle's state."""
    from paper_1806_11456_b200 import configs as _c  # noqa: F401

    w = configs.config2(nx=6, ny=4) if SMOKE else configs.config2()
    law = oracle_law(w.law)
    of = OO(np.asarray(w.orders.orders))
    so = omg.FASSolver(w.mesh, law, of, smoother=omg.SmootherConfig(**w.smoother),
                       time_config=ots.TimeConfig(**w.time), family=w.family, form=w.form)
    so.set_state(so.finest.op.project_function(w.init))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for c in range(2):
            t = time.time()
            so.v_cycle()
            log(f"  cycle {c}: {time.time() - t:.1f} s")
    out = {"work_units": so.work_units, "Q_state": np.concatenate([b.ravel() for b in so.Q.blocks])}
    out.update(_log_arrays(so.log))
    oo = so.finest.op
    out["F_norm"] = oo.apply(so.Q, isolated=True).norm_inf()
    tm = otau.estimate(w.mesh, law, so.Q, 1e6, isolated=True, fine_op=oo, family=w.family, form=w.form,
                       frozen=(2,))
    out["tau"] = tau_dense(tm, of.num_elements)
    out.update(_select(w, law, tm, 1e-4, 5, of))
    save("cfg2", **out)


def part_cfg5():
    """Cubed-sphere shell at N=3 (full size): residual, tau (isolated) and the
    stage-1 p-map (tau_max 1e-2, orders 1..6) of the seeded state."""
    w = configs.config5(na=2, nr=3, r1=2.0) if SMOKE else configs.config5()
    law, of, oo, Q0 = _setup(w)
    samp = sample_elements(of.num_elements, seed=5)
    out = {"sample": samp}
    out.update(field_summary("Q0", of, Q0.blocks, samp))
    out["A_norm"] = oo.m_inv_apply(Q0).norm_inf()
    r = oo.residual(Q0)
    out["r_norm"] = r.norm_inf()
    out.update(field_summary("r", of, r.blocks, samp))
    out["F_norm"] = oo.apply(Q0, isolated=True).norm_inf()
    t = time.time()
    tm = otau.estimate(w.mesh, law, Q0, 1e6, isolated=True, fine_op=oo, family=w.family, form=w.form)
    log(f"  tau.estimate {time.time() - t:.1f} s")
    out["tau"] = tau_dense(tm, of.num_elements)
    out.update(_select(w, law, tm, 1e-2, 6, of))
    save("cfg5", **out)


PARTS = {"cfg3": part_cfg3, "cfg3_tau": part_cfg3_tau, "cfg4": part_cfg4, "cfg4_vcycle": part_cfg4_vcycle,
         "cfg2": part_cfg2, "cfg5": part_cfg5}

if __name__ == "__main__":
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    for name in sys.argv[1:] or list(PARTS):
        log(f"part {name}")
        t0 = time.time()
        PARTS[name]()
        log(f"part {name}: {time.time() - t0:.1f} s")
