"""Debug: RK3 smoothing / V-cycle stability on mixed-order (mortar) meshes."""
import os, sys, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1806_11456_b200 import configs, multigrid, operators, timestep
from paper_1806_11456_b200.fields import OrderField

case, mode, cfla, nsw = sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4])
warnings.simplefilter("ignore")
if case == "cfg3":
    w = configs.config3(n=6)
elif case == "cfg3affine":
    w = configs.config3(n=6)
    from paper_1806_11456_b200 import mesh
    w.mesh = mesh.build_box(6, 6, 6)
elif case == "cfg5mixed":
    w = configs.config5(na=4, nr=6, order=3)
    rng = np.random.default_rng(0)
    w.orders = OrderField(rng.integers(2, 5, (w.mesh.num_elements, 3)))
elif case == "cfg2mixed":
    w = configs.config2(nx=8, ny=6, order=4)
    rng = np.random.default_rng(0)
    o = rng.integers(2, 6, (w.mesh.num_elements, 3)); o[:, 2] = 1
    w.orders = OrderField(o)
tc = timestep.TimeConfig(cfl_advective=cfla, cfl_viscous=cfla / 2)
if mode == "smooth":
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q = op.project_function(w.init)
    print(case, mode, cfla, "r0 %.3e" % op.residual_norm(Q))
    for k in range(nsw // 50):
        try:
            h = timestep.smooth(op, Q, 50, tc)
        except Exception as e:
            print("EXC", k * 50, e); break
        print(k * 50 + 50, "%.3e" % h[-1], flush=True)
else:
    sm = multigrid.SmootherConfig(pre_sweeps=3, post_sweeps=3, coarsest_sweeps=5, max_batches=1)
    s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=sm, time_config=tc, family=w.family, form=w.form)
    s.set_state(s.finest.op.project_function(w.init))
    print(case, mode, cfla, "levels", len(s.levels), "r0 %.3e" % s.residual_norm())
    for c in range(nsw):
        try:
            rn = s.v_cycle()
        except Exception as e:
            print("EXC", c, e); break
        if c % 10 == 0: print(c, "%.3e" % rn, flush=True)
