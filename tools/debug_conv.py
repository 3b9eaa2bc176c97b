"""Debug: V-cycle convergence of configs 2 / 5 under smoother settings."""
import os, sys, warnings, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1806_11456_b200 import configs, multigrid, timestep

which, local, cfla, cflv, ncyc = sys.argv[1], sys.argv[2] == "1", float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
full = len(sys.argv) > 6 and sys.argv[6] == "full"
if which == "cfg2":
    w = configs.config2() if full else configs.config2(nx=8, ny=6, order=4)
else:
    w = configs.config5() if full else configs.config5(na=4, nr=6, order=3)
warnings.simplefilter("ignore")
sm = multigrid.SmootherConfig(**w.smoother)
tc = timestep.TimeConfig(cfl_advective=cfla, cfl_viscous=cflv, local=local)
s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=sm, time_config=tc, family=w.family, form=w.form)
s.set_state(s.finest.op.project_function(w.init))
print(which, "local", local, cfla, cflv, "nodes", w.orders.num_nodes, "r0", s.residual_norm(), flush=True)
t = time.time()
hist = []
for c in range(ncyc):
    try:
        rn = s.v_cycle()
    except Exception as e:
        print("EXC at cycle", c, type(e).__name__, e); break
    hist.append(rn)
    if c % max(1, ncyc // 25) == 0 or c == ncyc - 1:
        print(c, "%.4e" % rn, flush=True)
print("wall", time.time() - t)
