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
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary.json")
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
def run_b200(args):
    import numpy as np
    import torch

    from paper_1806_11456_b200 import _lib, configs, multigrid, operators

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

    # ---- residual throughput, config 3 -------------------------------------
    t_setup = time.perf_counter()
    w = configs.config3()
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q = op.project_function(w.init)
    R = op.new_field()
    norm = torch.zeros(1, dtype=torch.float64, device="cuda")
    nodes = w.orders.num_nodes
    setup_s = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        op.residual_device(Q, None, out=R, norm=norm)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    _lib.timing_read()
    _lib.timing_enable(True)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        op.residual_device(Q, None, out=R, norm=norm)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    _lib.timing_enable(False)
    kt = _lib.timing_read()
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local)
    ms_step = ms / args.steps
    value = nodes * args.steps * ws / (ms / 1000.0)
    launches = int(sum(c for _, c in kt.values()))

    # roofline of the dominant kernel (algorithmic bytes)
    peak, peak_kind = _peak_hbm()
    curved_nodes = int(sum(int(op.orders.slot_nodes[s]) for s in range(op.orders.num_elements)
                           if not op._affine_slots[s]))
    m_per_node = 10.0 * curved_nodes / nodes
    per_node = {
        "vol_flux": 8.0 * (5 + 12 + 5 + m_per_node),      # Q, grad, metrics -> R
        "vol_lift": 8.0 * (5 + 12 + m_per_node),          # Q, metrics -> grad
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
    resid_bytes = 8.0 * (45 + 2 * m_per_node) * nodes                    # SURVEY §8d, per evaluation
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                "bytes_per_node": per_node[dom],
                "residual_eval_frac": resid_bytes / (ms_step / 1000.0) / 1e9 / peak,
                "kernel_ms_per_step": {k: round(v / args.steps, 4) for k, v in shares.items()}}

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
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _, host_norms = op.residual_host(Qh, out=Rh)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e = {"value": nodes * args.steps * ws / (e_ms / 1000.0), "unit": "DOF-evals/s",
           "h2d_bytes_per_step": q0.numel() * 8, "d2h_bytes_per_step": q0.numel() * 8 + 8,
           "ms_per_step": e_ms / args.steps, "api": "DGOperator.residual_host (tdg_residual_host)",
           "overlap": "double-buffered: H2D of step k+1 and D2H of step k-1 overlap step k"}
    del op, Q, R, Qh, Rh, bufs, outs

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
                barrier()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                solver.v_cycle()
                b.record(stream)
                torch.cuda.synchronize()
                times.append(max_over_ranks(a.elapsed_time(b)))
        hist = [r["rnorm"] for r in solver.log if r["phase"] in ("post", "coarse") and r["level"] == len(solver.levels)]
        # algorithmic HBM bytes of one pinned-sweep V-cycle (affine:
        # m = 0): per level 6s fused RK stages (finest 480 B/node, coarse levels
        # + 40 for the FAS source) and the other operator evaluations (finest 2,
        # intermediate 3, coarsest 3c + 2 in all), one element_dt read (40
        # B/node) per sweep, 160 (n_f + n_c) per level pair for the two
        # restrictions and the prolong-add
        sm = w4.smoother
        nl = len(solver.levels)
        vbytes = 0.0
        for li, lev in enumerate(solver.levels):
            n = lev.orders.num_nodes
            src = 0 if li == nl - 1 else 40
            if li == 0:
                stages, evals, sweeps = 3 * sm["coarsest_sweeps"], 2, sm["coarsest_sweeps"]
            else:
                sweeps = sm["pre_sweeps"] + sm["post_sweeps"]
                stages, evals = 3 * sweeps, (2 if li == nl - 1 else 3)
            vbytes += n * (stages * (480 + src) + evals * (360 + src) + sweeps * 40)
            if li > 0:
                vbytes += 160 * (n + solver.levels[li - 1].orders.num_nodes)
        vpeak, _ = _peak_hbm()
        v_roof_ms = vbytes / (vpeak * 1e6)
        vcycle = {"config": w4.name, "levels": len(solver.levels), "ms_median": statistics.median(times),
                  "ms_all": [round(t, 3) for t in times], "fine_nodes": w4.orders.num_nodes,
                  "smoother": w4.smoother, "setup_s": round(setup4, 1),
                  "rnorm_post": [float(x) for x in hist[-len(times):]],
                  "roofline": {"bound": "hbm", "algorithmic_gb": vbytes / 1e9, "peak": vpeak, "unit": "GB/s",
                               "roofline_ms": v_roof_ms, "frac": v_roof_ms / statistics.median(times)}}
        del solver

    # small configs: V-cycle latency (CUDA-graph replay of pinned-sweep cycles)
    small = {}
    if not args.no_vcycle:
        import warnings

        from paper_1806_11456_b200 import timestep

        for cid in (1, 2):
            wk = configs.CONFIGS[cid]()
            sv = multigrid.FASSolver(wk.mesh, wk.law, wk.orders, smoother=multigrid.SmootherConfig(**wk.smoother),
                                     time_config=timestep.TimeConfig(**wk.time), family=wk.family, form=wk.form)
            sv.set_state(sv.finest.op.project_function(wk.init))
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                sv.v_cycle()
                torch.cuda.synchronize()
                a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(5):
                    sv.v_cycle()
                b2.record(stream)
                torch.cuda.synchronize()
            small[f"cfg{cid}_vcycle_ms"] = max_over_ranks(a.elapsed_time(b2) / 5)
            del sv
        if vcycle is not None:
            vcycle.update(small)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, info = cpu_sample_rate(n=6, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": "DOF-evals/s", "cores": 1, "kind": "port", "sample": info["sample"],
               "evals": info["evals"], "seconds": info["seconds"]}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "DOF-evals/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "nodes": nodes, "unknowns": 5 * nodes,
                       "global_batch": nodes * ws, "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                       "family": w.family, "metrics": w.form, "l2": "inputs > L2 (Q is 163 MB)"},
            "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "vcycle": vcycle, "cpu_baseline": cpu, "setup_s": round(setup_s, 1),
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
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
