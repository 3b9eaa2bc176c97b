"""Benchmark: NS residual DOF-evals/s (config 3), p-multigrid V-cycle ms
(config 4) and % of the HBM roofline, on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one full Navier-Stokes residual evaluation r = S - M^-1 F(Q) of
config 3 (32^3 jittered periodic box, orders U{1..7}^3, 4.11 M nodes), with
Q resident in HBM (163 MB > L2, so every step streams from HBM).  ``e2e``
repeats it through the public API with the state copied from pinned host
memory and the residual copied back every step.  Multi-GPU runs are
independent replicas (the north_star path runs on one GPU), one
process per GPU, value = all ranks' node-evaluations / max-over-ranks time.

--impl reference times the reference algorithm's CPU implementation (the
NumPy oracle port — the reference package is pure Python and cannot travel
to the GPU box) on the host cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02", "ncu_summary.json")
# the unmodified reference (pure Python, not present on the GPU box) timed in the
# build container on its own 2D-scalar analogues of configs 1-2
REF2D = os.path.join(ROOT, "profiles", "reference_cpu_2d.json")
METRIC = "NS residual DOF-evals/s; p-multigrid V-cycle ms; % of HBM roofline (1 B200)"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x, dist=None, device="cpu"):
    """Max of a per-rank float over all ranks (timing rule: max over ranks)."""
    if dist is None or not dist.is_initialized():
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _peak_hbm():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------
def cpu_sample_rate(n=6, evals=None, budget_s=12.0):
    """Oracle (NumPy restatement of the reference path) residual throughput on a
    bounded sample of config 3: an n^3 jittered periodic box with the same
    order distribution and state.  Single process, single thread."""
    import numpy as np

    from oracle.fields import OrderField as OO
    from oracle.operators import DGOperator as ODG
    from oracle.physics import NavierStokes as ONS
    from paper_1806_11456_b200 import configs

    w = configs.config3(n=n)
    law = ONS(w.law.gamma, w.law.prandtl, w.law.mach, w.law.reynolds)
    of = OO(np.asarray(w.orders.orders))
    op = ODG(w.mesh, law, of, family=w.family, form=w.form)
    Q = op.project_function(w.init)
    op.residual(Q)
    t0 = time.perf_counter()
    k = 0
    while True:
        op.residual(Q)
        k += 1
        if (evals is not None and k >= evals) or (evals is None and time.perf_counter() - t0 > budget_s):
            break
    dt = time.perf_counter() - t0
    return of.dofs() * k / dt, {"nodes": of.dofs(), "evals": k, "seconds": round(dt, 3),
                                "sample": f"config-3 distribution on a {n}^3 jittered periodic box "
                                          f"({of.dofs()} nodes), oracle residual evaluations"}


def _worker(args):
    n, budget = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    rate, info = cpu_sample_rate(n=n, budget_s=budget)
    return rate, info


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    procs = max(1, cores)
    steps = max(1, args.steps)
    per_step = max(2.0, min(20.0, 120.0 / (steps + args.warmup)))
    # warmup: one short single-process pass
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample_rate(n=4, evals=1)
    rates = []
    t_all = time.perf_counter()
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for _ in range(steps):
            res = pool.map(_worker, [(6, per_step)] * procs)
            rates.append(sum(r for r, _ in res))
    info = res[0][1]
    value = statistics.median(rates)
    nodes = info["nodes"]
    out = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "DOF-evals/s",
        "n_gpus": ws, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * nodes / (value / procs) if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "cfg3 sample: config-3 order/jitter/state distribution on a 6^3 box",
                   "global_batch": nodes, "parallelism": f"{procs} host processes (replicas)"},
        "cpu_baseline": {"value": value, "unit": "DOF-evals/s", "cores": procs, "kind": "port",
                         "sample": info["sample"] + f"; {procs} concurrent processes"},
        "e2e": {"value": value, "unit": "DOF-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_all, 1),
    }
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------
def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "threads_env": {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                                           "MKL_NUM_THREADS")}}


def curved_fraction(op):
    of = op.orders
    cn = sum(int(of.slot_nodes[s]) for s in range(of.num_elements) if not op._affine_slots[s])
    return cn / max(1, of.num_nodes)


def vcycle_bytes(solver, m_of):
    """Algorithmic HBM bytes of one pinned-sweep V-cycle: per
    level 6s fused RK stages (8(60+2m) B/node, + 40 for the FAS source on
    coarse levels), the other evaluations (finest 2, intermediate 3,
    coarsest 3c+2 in all; 8(45+2m) B/node), one element_dt read (40 B/node)
    per sweep and 160 (n_f + n_c) per level pair for the two restrictions and
    the prolong-add.  m_of(level) = metric doubles per node."""
    sm = solver.smoother
    nl = len(solver.levels)
    vbytes = 0.0
    for li, lev in enumerate(solver.levels):
        n = lev.orders.num_nodes
        m = m_of(lev)
        src = 0 if li == nl - 1 else 40
        if li == 0:
            stages, evals, sweeps = 3 * sm.coarsest_sweeps, 2, sm.coarsest_sweeps
        else:
            sweeps = sm.pre_sweeps + sm.post_sweeps
            stages, evals = 3 * sweeps, (2 if li == nl - 1 else 3)
        vbytes += n * (stages * (8 * (60 + 2 * m) + src) + evals * (8 * (45 + 2 * m) + src) + sweeps * 40)
        if li > 0:
            vbytes += 160 * (n + solver.levels[li - 1].orders.num_nodes)
    return vbytes


def run_b200(args):
    import numpy as np
    import torch

    from paper_1806_11456_b200 import _lib, configs, multigrid, operators, tau, timestep

    ws, rank, local = _dist()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product path has no CPU fallback)")
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        return globals()["max_over_ranks"](x, dist, "cuda")

    stream = torch.cuda.current_stream()
    peak, peak_kind = _peak_hbm()

    def timed(fn, reps):
        """Device time (ms) of ``reps`` calls of fn on the current stream, max over ranks."""
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(a.elapsed_time(b))

    # ---- residual throughput, config 3 (headline) -------------------------------
    t_setup = time.perf_counter()
    w = configs.config3()
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q = op.project_function(w.init)
    R = op.new_field()
    norm = torch.zeros(1, dtype=torch.float64, device="cuda")
    nodes = w.orders.num_nodes
    setup_s = time.perf_counter() - t_setup
    m3 = 10.0 * curved_fraction(op)

    def resid():
        op.residual_device(Q, None, out=R, norm=norm)

    for _ in range(args.warmup):
        resid()
    torch.cuda.synchronize()
    # timed region: no per-launch instrumentation; clocks sampled meanwhile
    clocks = Clocks(local)
    clocks.start()
    ms = timed(resid, args.steps)
    clk = clocks.stop()
    ms_step = ms / args.steps
    value = nodes * args.steps * ws / (ms / 1000.0)

    # kernel split: the same K evaluations again with the library's per-launch
    # CUDA events (on the launch stream), for the roofline of the dominant kernel
    _lib.timing_read()
    _lib.timing_enable(True)
    ms_instr = timed(resid, args.steps)
    _lib.timing_enable(False)
    kt = _lib.timing_read()
    launches = int(sum(c for _, c in kt.values()))
    per_node = {
        "vol_flux": 8.0 * (5 + 12 + 5 + m3),      # Q, grad, metrics -> R
        "vol_lift": 8.0 * (5 + 12 + m3),          # Q, metrics -> grad
    }
    shares = {k: v[0] for k, v in kt.items() if v[1]}
    dom = max(("vol_flux", "vol_lift"), key=lambda k: shares.get(k, 0.0))
    dom_ms = kt[dom][0] / max(kt[dom][1], 1)
    achieved = per_node[dom] * nodes / (dom_ms / 1000.0) / 1e9
    traffic = None
    try:
        with open(NCU_SUMMARY) as fh:
            traffic = json.load(fh).get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    resid_bytes = 8.0 * (45 + 2 * m3) * nodes                    # SURVEY §8d, per evaluation
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                "bytes_per_node": per_node[dom], "kernel_ms": dom_ms,
                "residual_eval_frac": resid_bytes / (ms_step / 1000.0) / 1e9 / peak,
                "residual_bytes_per_node": 8.0 * (45 + 2 * m3),
                "instrumented_ms_per_step": ms_instr / args.steps,
                "kernel_ms_per_step": {k: round(v / args.steps, 4) for k, v in shares.items()}}

    # ---- config 3: fused RK3 stages (100 in the protocol) ------------------------
    rk = None
    if not args.quick:
        s = timestep._scratch(op)
        cfg = timestep.TimeConfig()
        dt_dev = timestep._device_dt(op, Q, cfg, s)
        Qw = Q.copy()
        work = op.new_field()
        rn = torch.zeros(1, dtype=torch.float64, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        state = {"k": 0}

        def stage():
            k = state["k"] % 3
            op.rk3_stage(Qw, work, op.source, k, dt_dev, False, rnorm=rn, nonfinite=flag, fresh=k > 0)
            state["k"] += 1

        for _ in range(3):
            stage()
        nst = 3 * max(1, args.steps)
        ms_rk = timed(stage, nst) / nst
        rk_bpn = 8.0 * (60 + 2 * m3)
        rk = {"stages": nst, "ms_per_stage": ms_rk, "dof_evals_per_s": nodes / (ms_rk / 1000.0),
              "ms_per_100_stages": 100 * ms_rk,
              "roofline": {"bound": "hbm", "bytes_per_node": rk_bpn, "peak": peak, "unit": "GB/s",
                           "achieved": rk_bpn * nodes / (ms_rk / 1000.0) / 1e9,
                           "frac": rk_bpn * nodes / (ms_rk / 1000.0) / 1e9 / peak}}
        del Qw, work

    # ---- end to end through the public API with host buffers -------------------
    # Page-locked host states (4 distinct buffers, cycled) evaluated by the
    # host-buffer batch call: every one of the K steps copies its state in and
    # its residual and max|r| out, the copies of neighbouring steps overlapping
    # the evaluation (tdg_residual_host)
    q0 = Q.data.cpu()
    nbuf = min(4, args.steps)
    bufs = [q0.clone().pin_memory() for _ in range(nbuf)]
    for k, q in enumerate(bufs):
        q[k] += 1e-12 * k        # distinct states
    outs = [torch.empty_like(q0).pin_memory() for _ in range(nbuf)]
    Qh = [bufs[k % nbuf] for k in range(args.steps)]
    Rh = [outs[k % nbuf] for k in range(args.steps)]
    op.residual_host(Qh[:nbuf], out=Rh[:nbuf])     # untimed: every staging buffer once
    torch.cuda.synchronize()
    # the copies run at the mercy of the host (PCIe, NUMA, other tenants): the K-step
    # batch is timed three times and the fastest is reported, all three listed
    e_all = [timed(lambda: op.residual_host(Qh, out=Rh), 1) for _ in range(3)]
    e_ms = min(e_all)
    e2e = {"value": nodes * args.steps * ws / (e_ms / 1000.0), "unit": "DOF-evals/s",
           "h2d_bytes_per_step": q0.numel() * 8, "d2h_bytes_per_step": q0.numel() * 8 + 8,
           "ms_per_step": e_ms / args.steps, "api": "DGOperator.residual_host (tdg_residual_host)",
           "overlap": "double-buffered: H2D of step k+1 and D2H of step k-1 overlap step k",
           "repeats": {"stat": "min of 3 batches of K steps", "ms_per_step_all": [t / args.steps for t in e_all]}}
    del Qh, Rh, bufs, outs

    # ---- config 3: the tau estimation (isolated, all directions) -----------------
    tau_est = None
    if not args.quick:
        solvers = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tm = tau.estimate(w.mesh, w.law, Q, 1e6, isolated=True, fine_op=op, solvers=solvers)
        torch.cuda.synchronize()
        first = time.perf_counter() - t0
        reps = 3
        t0 = time.perf_counter()
        ms_tau = timed(lambda: tau.estimate(w.mesh, w.law, Q, 1e6, isolated=True, fine_op=op, solvers=solvers),
                       reps) / reps
        wall_tau = (time.perf_counter() - t0) / reps
        tau_est = {"ms": ms_tau, "wall_ms": 1e3 * wall_tau, "first_call_with_setup_s": round(first, 1),
                   "levels_per_direction": {d: len(sv.levels) for d, sv in solvers.items()},
                   "entries": int(sum(len(tm.tau[e][d]) for e in range(w.mesh.num_elements) for d in range(3))),
                   "note": "device-event time of a cached-solver estimate (residual + per-direction descent "
                           "+ isolated evaluations + per-element reductions); first call includes the host "
                           "construction of the 18 per-direction level operators"}
        del solvers, tm
    del op, Q, R

    # ---- V-cycle, config 4 --------------------------------------------------------
    vcycle = None
    if not args.no_vcycle:
        import warnings

        w4 = configs.config4()
        t4 = time.perf_counter()
        solver = multigrid.FASSolver(w4.mesh, w4.law, w4.orders,
                                     smoother=multigrid.SmootherConfig(**w4.smoother),
                                     family=w4.family, form=w4.form)
        solver.set_state(solver.finest.op.project_function(w4.init))
        setup4 = time.perf_counter() - t4
        times = []
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            solver.v_cycle()
            torch.cuda.synchronize()
            for _ in range(args.vcycles):
                times.append(timed(solver.v_cycle, 1))
        hist = [r["rnorm"] for r in solver.log if r["phase"] in ("post", "coarse") and r["level"] == len(solver.levels)]
        vbytes = vcycle_bytes(solver, lambda lev: 0.0)
        v_roof_ms = vbytes / (peak * 1e6)
        vcycle = {"config": w4.name, "levels": len(solver.levels), "ms_median": statistics.median(times),
                  "ms_all": [round(t, 3) for t in times], "fine_nodes": w4.orders.num_nodes,
                  "smoother": w4.smoother, "setup_s": round(setup4, 1),
                  "rnorm_post": [float(x) for x in hist[-len(times):]],
                  "roofline": {"bound": "hbm", "algorithmic_gb": vbytes / 1e9, "peak": peak, "unit": "GB/s",
                               "roofline_ms": v_roof_ms, "frac": v_roof_ms / statistics.median(times)}}
        del solver

    # ---- config 5: curved shell residual and V-cycle -------------------------------
    cfg5 = None
    if not args.no_vcycle and not args.quick:
        import warnings

        w5 = configs.config5()
        t5 = time.perf_counter()
        sv = multigrid.FASSolver(w5.mesh, w5.law, w5.orders, smoother=multigrid.SmootherConfig(**w5.smoother),
                                 time_config=timestep.TimeConfig(**w5.time), family=w5.family, form=w5.form)
        sv.set_state(sv.finest.op.project_function(w5.init))
        setup5 = time.perf_counter() - t5
        op5 = sv.finest.op
        m5 = 10.0 * curved_fraction(op5)
        R5 = op5.new_field()
        n5 = w5.orders.num_nodes
        for _ in range(3):
            op5.residual_device(sv.Q, None, out=R5, norm=norm)
        ms5 = timed(lambda: op5.residual_device(sv.Q, None, out=R5, norm=norm), args.steps) / args.steps
        bpn5 = 8.0 * (45 + 2 * m5)
        times = []
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            sv.v_cycle()
            torch.cuda.synchronize()
            for _ in range(args.vcycles):
                times.append(timed(sv.v_cycle, 1))
        vb5 = vcycle_bytes(sv, lambda lev: 10.0 * curved_fraction(lev.op))
        cfg5 = {"config": w5.name, "nodes": n5, "setup_s": round(setup5, 1),
                "residual": {"ms": ms5, "dof_evals_per_s": n5 / (ms5 / 1000.0),
                             "roofline": {"bound": "hbm", "bytes_per_node": bpn5, "peak": peak, "unit": "GB/s",
                                          "frac": bpn5 * n5 / (ms5 / 1000.0) / 1e9 / peak}},
                "vcycle": {"levels": len(sv.levels), "ms_median": statistics.median(times),
                           "ms_all": [round(t, 3) for t in times], "smoother": w5.smoother, "time": w5.time,
                           "roofline": {"bound": "hbm", "algorithmic_gb": vb5 / 1e9, "peak": peak,
                                        "roofline_ms": vb5 / (peak * 1e6),
                                        "frac": vb5 / (peak * 1e6) / statistics.median(times)}}}
        del sv, op5, R5

    # small configs: V-cycle latency (CUDA-graph replay of pinned-sweep cycles)
    if not args.no_vcycle and vcycle is not None:
        import warnings

        for cid in (1, 2):
            wk = configs.CONFIGS[cid]()
            sv = multigrid.FASSolver(wk.mesh, wk.law, wk.orders, smoother=multigrid.SmootherConfig(**wk.smoother),
                                     time_config=timestep.TimeConfig(**wk.time), family=wk.family, form=wk.form)
            sv.set_state(sv.finest.op.project_function(wk.init))
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                sv.v_cycle()
                torch.cuda.synchronize()
                vcycle[f"cfg{cid}_vcycle_ms"] = timed(sv.v_cycle, 5) / 5
            del sv

    # ---- adaptation protocols (configs 2 and 5), bounded V-cycle budgets -----------
    protos = None
    if rank == 0 and ws == 1 and not args.no_protocols and not args.quick:
        from paper_1806_11456_b200 import protocols

        protos = {}
        t0 = time.perf_counter()
        run2 = protocols.run_config2(max_cycles=args.protocol_cycles)
        protos["cfg2"] = dict(run2.to_dict(), wall_s=round(time.perf_counter() - t0, 1))
        del run2
        t0 = time.perf_counter()
        run5 = protocols.run_config5(max_cycles=args.protocol_cycles, stages=args.cfg5_stages)
        protos["cfg5"] = dict(run5.to_dict(), wall_s=round(time.perf_counter() - t0, 1))
        del run5
        protos["note"] = (f"at most {args.protocol_cycles} V-cycles per stage; a stage that misses |r| <= "
                          "tau_max/10 in that budget estimates tau with the gate bypassed (recorded); "
                          "cfg5 runs its first {} threshold stage(s) here".format(args.cfg5_stages))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, info = cpu_sample_rate(n=6, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": "DOF-evals/s", "cores": 1, "kind": "port", "sample": info["sample"],
               "evals": info["evals"], "seconds": info["seconds"], **cpu_info()}
    ref2d = None
    try:
        with open(REF2D) as fh:
            ref2d = json.load(fh)
    except Exception:
        pass

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "DOF-evals/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "nodes": nodes, "unknowns": 5 * nodes,
                       "global_batch": nodes * ws, "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                       "family": w.family, "metrics": w.form, "l2": "inputs > L2 (Q is 163 MB)",
                       "note": "98 % of the faces are p-nonconforming and curved: free-stream "
                               "preservation there is not exact (0.1; oracle and GPU agree, DESIGN §3), "
                               "so the evaluated state's residual is dominated by mortar metric terms"},
            "roofline": roofline, "e2e": e2e, "gpu_launches": launches * 1, "clocks": clk,
            "rk3_stage": rk, "tau_estimate": tau_est, "vcycle": vcycle, "cfg5": cfg5, "protocols": protos,
            "cpu_baseline": cpu, "reference_cpu_2d": ref2d, "setup_s": round(setup_s, 1),
        }
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--vcycles", type=int, default=3)
    ap.add_argument("--no-vcycle", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--quick", action="store_true", help="headline residual, e2e and V-cycles only")
    ap.add_argument("--no-protocols", action="store_true")
    ap.add_argument("--protocol-cycles", type=int, default=30)
    ap.add_argument("--cfg5-stages", type=int, default=1)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
