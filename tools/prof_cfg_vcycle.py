"""V-cycle timing for any config (development tool)."""
import sys, os, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1806_11456_b200 import configs, multigrid, timestep, _lib
cfg = int(sys.argv[1]); cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kw = {}
w = configs.CONFIGS[cfg](**kw)
s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                        time_config=timestep.TimeConfig(**w.time), family=w.family, form=w.form)
s.set_state(s.finest.op.project_function(w.init))
warnings.simplefilter("ignore")
s.v_cycle(); torch.cuda.synchronize()
_lib.timing_read(); _lib.timing_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for _ in range(cycles):
    s.v_cycle()
e1.record(); torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / cycles
_lib.timing_enable(False)
kt = _lib.timing_read()
print(w.name, "levels", len(s.levels), "v-cycle ms events %.2f wall %.2f kernels %.2f launches/cycle %d" % (
    e0.elapsed_time(e1) / cycles, wall * 1e3, sum(v[0] for v in kt.values()) / cycles,
    sum(v[1] for v in kt.values()) // cycles))
print({k: (round(v[0] / cycles, 3), v[1] // cycles) for k, v in kt.items() if v[1]})
