"""Debug: V-cycles on an adapted (mixed-order) config-2/5 p-map, GPU vs oracle."""
import os, sys, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from helpers import oracle_law
from paper_1806_11456_b200 import adaptation, configs, multigrid, tau, timestep
from paper_1806_11456_b200.fields import OrderField

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "cfg2":
    w = configs.config2(nx=8, ny=6, order=4)
    frozen, tmax, nmax = (2,), 1e-4, 5
else:
    w = configs.config5(na=2, nr=3, order=3, r1=2.0)
    w.time = dict(cfl_advective=0.025, cfl_viscous=0.0125)
    frozen, tmax, nmax = (), 1e-2, 6
warnings.simplefilter("ignore")
sm = multigrid.SmootherConfig(**w.smoother)
tc = timestep.TimeConfig(**w.time)
s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=sm, time_config=tc, family=w.family, form=w.form)
s.set_state(s.finest.op.project_function(w.init))
for c in range(20):
    rn = s.v_cycle()
print("stage-1 |r| after 20 cycles", rn)
tm = tau.estimate(w.mesh, w.law, s.Q, 1e6, isolated=True, fine_op=s.finest.op, frozen=frozen)
tau.extrapolate_map(tm, nmax)
sel, rep = adaptation.select_orders(tm, adaptation.AdaptConfig(tau_max=tmax, n_max=nmax))
new = adaptation.limit_jumps(w.mesh, sel)
print("orders", {d: np.unique(new.orders[:, d], return_counts=True) for d in range(3)})
state = adaptation.transfer(s.Q, new, w.family)
s2 = multigrid.FASSolver(w.mesh, w.law, new, smoother=sm, time_config=tc, family=w.family, form=w.form)
s2.use_graphs = False
s2.set_state(state)
print("levels", [l.orders.orders.max(axis=0) for l in s2.levels])
r0 = s2.residual_norm(); print("adapted start |r|", r0)
# oracle comparison of one cycle
from oracle import multigrid as omg, timestep as ots
from oracle.fields import OrderField as OO
law = oracle_law(w.law)
so = omg.FASSolver(w.mesh, law, OO(np.asarray(new.orders)), smoother=omg.SmootherConfig(**w.smoother),
                   time_config=ots.TimeConfig(**w.time), family=w.family, form=w.form)
so.set_state(so.finest.op.project_function(lambda x, y, z: 0 * x))
so.finest.Q.blocks = [b.copy() for b in state.to_oracle_blocks()]
so.finest.Q.field = so.finest.orders
for c in range(3):
    a = s2.v_cycle(); b = so.v_cycle()
    rn = np.array([r["rnorm"] for r in s2.log]); rno = np.array([r["rnorm"] for r in so.log])
    print("cycle", c, a, b, "hist err", np.abs(rn - rno).max() / rno.max())
for c in range(30):
    try:
        a = s2.v_cycle()
    except Exception as e:
        print("EXC", c, e); break
    print("cycle", c + 3, a, [ (r["level"], r["phase"], "%.3e" % r["rnorm"]) for r in s2.log[-3:]])
