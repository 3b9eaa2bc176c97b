"""BASELINE.json adaptation protocols of configs 2 and 5, on the device path.

The reference's drivers (adaptation.py:276-375, run_single_stage /
run_multi_stage) converge, estimate tau, select, limit, transfer and repeat
with ONE tau_max and stage caps.  Config 5 instead tightens the threshold
per stage (1e-2, then 1e-4) and config 2 adapts once at 1e-4 with Nz
frozen, so this module composes the same building blocks — FASSolver
V-cycles, tau.estimate, select_orders, limit_jumps and the device transfer —
into the two BASELINE protocols and records per-stage facts: V-cycles and
their device time, tau-estimation time, DOFs before and after, decision paths
and the per-direction order histogram of the new p-map.

Every stage's V-cycles are bounded by ``max_cycles``; a stage that does not
reach its tolerance in that budget is reported as such (``converged``:
False) and the protocol continues from the state it reached, with the tau
gate (|r| <= tau_max/10, tau.py:204-210) bypassed for that estimate and the
bypass recorded.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import asdict, dataclass, field

import numpy as np

from . import adaptation, multigrid, tau, timestep
from .errors import DivergedError, StallError, TimeScaleError
from .fields import OrderField


@dataclass
class StageReport:
    stage: int
    tau_max: float
    orders_in: dict                  # per-direction histogram of the stage's orders
    dofs_before: int
    dofs_after: int
    cycles: int
    rnorm_start: float
    rnorm_end: float
    tol: float
    converged: bool
    stalled: bool
    cycle_ms_total: float
    cycle_ms_median: float
    tau_ms: float
    tau_gate_bypassed: bool
    setup_s: float
    paths: dict = field(default_factory=dict)
    orders_out: dict = field(default_factory=dict)


@dataclass
class ProtocolRun:
    name: str
    stages: list
    final: dict
    Q: object = None
    orders: OrderField | None = None

    def to_dict(self):
        return {"name": self.name, "stages": [asdict(s) for s in self.stages], "final": self.final}


def order_histogram(orders: OrderField):
    arr = np.asarray(orders.orders)
    return {f"N{d + 1}": {str(int(k)): int(v) for k, v in zip(*np.unique(arr[:, d], return_counts=True))}
            for d in range(3)}


def _converge(solver, tol, max_cycles, stall_window=10, stall_factor=0.99):
    """V-cycles until |r| <= tol, at most max_cycles, stopping early on a
    stall (multigrid.py:372-376 rule: no 1% decrease over 10 cycles);
    device-event timed per cycle."""
    import torch

    r0 = solver.residual_norm()
    norms, times, stalled = [r0], [], False
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        while norms[-1] > tol and len(times) < max_cycles:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            solver.cycle += 1
            rn = solver._descend(len(solver.levels) - 1, None, tol)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
            norms.append(rn)
            if not np.isfinite(rn):
                raise StallError(f"non-finite residual after {len(times)} cycles")
            if len(norms) > stall_window and rn > stall_factor * norms[-1 - stall_window]:
                stalled = True
                break
    return r0, norms[-1], times, stalled


def _estimate(msh, law, Q, tau_max, fine_op, frozen, solvers):
    import torch

    torch.cuda.synchronize()
    t = time.perf_counter()
    rn = fine_op.residual_norm(Q)
    bypass = rn > tau_max / 10.0
    tm = tau.estimate(msh, law, Q, tau_max if not bypass else 10.0 * rn * (1 + 1e-12), isolated=True,
                      fine_op=fine_op, solvers=solvers, frozen=frozen)
    torch.cuda.synchronize()
    return tm, 1e3 * (time.perf_counter() - t), bypass


def run_stages(name, msh, law, orders, init, thresholds, n_max, smoother, time_config=None, frozen=(),
               n_min=1, max_cycles=100, final_tol=None, family="LGL", form="curl"):
    """Converge -> tau -> select/limit -> transfer, once per threshold, then a
    final convergence on the last p-map."""
    import torch

    stages = []
    t0 = time.perf_counter()
    solver = multigrid.FASSolver(msh, law, orders, smoother=smoother, time_config=time_config,
                                 family=family, form=form)
    solver.set_state(init(solver.finest.op))
    setup = time.perf_counter() - t0
    for k, tmax in enumerate(thresholds):
        tol = tmax / 10.0
        try:
            r0, rn, times, stalled = _converge(solver, tol, max_cycles)
        except (DivergedError, TimeScaleError, StallError) as exc:
            return ProtocolRun(name, stages, {"failed": f"stage {k + 1} V-cycles: {exc}"}, solver.Q,
                               solver.finest.orders)
        t1 = time.perf_counter()
        solvers = {}
        tm, tau_ms, bypass = _estimate(msh, law, solver.Q, tmax, solver.finest.op, frozen, solvers)
        tau.extrapolate_map(tm, n_max)
        cfg = adaptation.AdaptConfig(tau_max=tmax, n_max=n_max, n_min=n_min)
        sel, rep = adaptation.select_orders(tm, cfg)
        new = adaptation.limit_jumps(msh, sel)
        setup_tau = time.perf_counter() - t1 - tau_ms / 1e3
        stages.append(StageReport(
            stage=k + 1, tau_max=tmax, orders_in=order_histogram(solver.finest.orders),
            dofs_before=int(solver.finest.orders.dofs()), dofs_after=int(new.dofs()), cycles=len(times),
            rnorm_start=float(r0), rnorm_end=float(rn), tol=tol, converged=bool(rn <= tol), stalled=stalled,
            cycle_ms_total=float(sum(times)), cycle_ms_median=float(np.median(times)) if times else 0.0,
            tau_ms=tau_ms, tau_gate_bypassed=bool(bypass), setup_s=round(setup + max(setup_tau, 0.0), 2),
            paths=rep.histogram(), orders_out=order_histogram(new)))
        state = adaptation.transfer(solver.Q, new, family)
        del solver, solvers, tm
        t0 = time.perf_counter()
        solver = multigrid.FASSolver(msh, law, new, smoother=smoother, time_config=time_config,
                                     family=family, form=form)
        solver.set_state(state)
        setup = time.perf_counter() - t0
    tol = final_tol if final_tol is not None else thresholds[-1] / 10.0
    try:
        r0, rn, times, stalled = _converge(solver, tol, max_cycles)
    except (DivergedError, TimeScaleError, StallError) as exc:
        return ProtocolRun(name, stages, {"failed": f"final V-cycles: {exc}",
                                          "orders": order_histogram(solver.finest.orders),
                                          "dofs": int(solver.finest.orders.dofs())}, solver.Q,
                           solver.finest.orders)
    torch.cuda.synchronize()
    final = {"orders": order_histogram(solver.finest.orders), "dofs": int(solver.finest.orders.dofs()),
             "cycles": len(times), "rnorm_start": float(r0), "rnorm_end": float(rn), "tol": tol,
             "converged": bool(rn <= tol), "cycle_ms_total": float(sum(times)),
             "cycle_ms_median": float(np.median(times)) if times else 0.0, "setup_s": round(setup, 2),
             "levels": len(solver.levels)}
    return ProtocolRun(name, stages, final, solver.Q, solver.finest.orders)


def run_config2(max_cycles=100, **kw):
    """Config 2: converge at N=5 (5-level V-cycles), tau with Nz frozen,
    adapt (Nx, Ny) in 1..5 at tau_max 1e-4, converge the adapted mesh."""
    from . import configs

    w = configs.config2(**kw)
    return run_stages("cfg2", w.mesh, w.law, w.orders, lambda op: op.project_function(w.init), (1e-4,), 5,
                      multigrid.SmootherConfig(**w.smoother), timestep.TimeConfig(**w.time), frozen=(2,),
                      max_cycles=max_cycles, family=w.family, form=w.form)


def run_config5(max_cycles=100, stages=2, **kw):
    """Config 5: converge at N=3, tau, adapt per direction in 1..6 at tau_max
    1e-2; converge at the new orders, tau, adapt at 1e-4; converge.
    ``stages`` = 1 stops after the first threshold (and its convergence)."""
    from . import configs

    w = configs.config5(**kw)
    return run_stages("cfg5", w.mesh, w.law, w.orders, lambda op: op.project_function(w.init),
                      (1e-2, 1e-4)[:stages], 6,
                      multigrid.SmootherConfig(**w.smoother), timestep.TimeConfig(**w.time),
                      max_cycles=max_cycles, family=w.family, form=w.form)
