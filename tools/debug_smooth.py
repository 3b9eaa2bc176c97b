"""Debug: plain RK3 smoothing stability of config 2 (no multigrid)."""
import os, sys, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1806_11456_b200 import configs, operators, timestep
from paper_1806_11456_b200.fields import OrderField

cfla, cflv, order, nsw = float(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
bc = sys.argv[5] if len(sys.argv) > 5 else "default"
w = configs.config2(nx=8, ny=6, order=order)
if bc == "allfree":
    w.mesh.bc = {k: "freestream" for k in w.mesh.bc}
elif bc == "nowall":
    w.mesh.bc["wall"] = "symmetry"
op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
Q = op.project_function(w.init)
tc = timestep.TimeConfig(cfl_advective=cfla, cfl_viscous=cflv)
print("cfl", cfla, cflv, "order", order, "bc", bc, "r0 %.3e" % op.residual_norm(Q), "dt %.3e" % timestep.compute_dt(op, Q, tc))
warnings.simplefilter("ignore")
for k in range(nsw // 50):
    try:
        h = timestep.smooth(op, Q, 50, tc)
    except Exception as e:
        print("EXC", k * 50, e); break
    print(k * 50 + 50, "%.3e" % h[-1], flush=True)
