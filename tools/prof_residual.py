"""Profiling driver: a few NS residual evaluations of a config-3-type box."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
from paper_1806_11456_b200 import configs, operators

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--evals", type=int, default=3)
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--timing", action="store_true")
a = ap.parse_args()
w = configs.config3(n=a.n) if a.config == 3 else configs.config4(n=a.n)
op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
Q = op.project_function(w.init)
R = op.new_field()
norm = torch.zeros(1, dtype=torch.float64, device="cuda")
for _ in range(a.evals):
    op.residual_device(Q, None, out=R, norm=norm)
torch.cuda.synchronize()
print("ok", w.orders.num_nodes, float(norm.item()))
if "--timing" in sys.argv or True:
    from paper_1806_11456_b200 import _lib
    _lib.timing_read(); _lib.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.evals):
        op.residual_device(Q, None, out=R, norm=norm)
    e1.record(); torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_read()
    print("ms/eval %.3f" % (e0.elapsed_time(e1) / a.evals),
          {k: round(v[0] / a.evals, 4) for k, v in kt.items() if v[1]})
