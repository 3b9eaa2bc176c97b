"""Profile the host side of DGOperator construction (development tool)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_11456_b200 import configs, operators, multigrid

which = sys.argv[1] if len(sys.argv) > 1 else "3"
w = configs.config3() if which == "3" else configs.config4() if which == "4" else configs.config5()
pr = cProfile.Profile()
t = time.time()
pr.enable()
op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
pr.disable()
print("build", round(time.time() - t, 2))
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
