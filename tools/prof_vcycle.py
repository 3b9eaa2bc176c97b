"""V-cycle breakdown: kernel classes vs wall (development tool)."""
import sys, os, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
from paper_1806_11456_b200 import configs, multigrid, _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--order", type=int, default=7)
ap.add_argument("--cycles", type=int, default=2)
a = ap.parse_args()
w = configs.config4(n=a.n, order=a.order)
t0 = time.time()
s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                        family=w.family, form=w.form)
s.set_state(s.finest.op.project_function(w.init))
print("setup %.1fs" % (time.time() - t0))
warnings.simplefilter("ignore")
s.v_cycle(); torch.cuda.synchronize()
_lib.timing_read(); _lib.timing_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(a.cycles):
    s.v_cycle()
e1.record(); torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / a.cycles
_lib.timing_enable(False)
kt = _lib.timing_read()
tot = sum(v[0] for v in kt.values()) / a.cycles
print("v-cycle ms (events) %.2f wall %.2f kernels %.2f" % (e0.elapsed_time(e1) / a.cycles, wall * 1e3, tot))
print({k: (round(v[0] / a.cycles, 2), v[1] // a.cycles) for k, v in kt.items() if v[1]})
print([round(r["rnorm"], 4) for r in s.log[-8:]])
