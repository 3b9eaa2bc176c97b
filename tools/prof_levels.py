"""Per-level residual and RK-stage timing of a config's p-multigrid hierarchy
(development tool): ms per evaluation, ns per node, kernel split."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1806_11456_b200 import configs, multigrid, timestep, _lib

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = configs.CONFIGS[cfg]()
s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                        time_config=timestep.TimeConfig(**w.time), family=w.family, form=w.form)
s.set_state(s.finest.op.project_function(w.init))
Qf = s.finest.Q
for li in range(len(s.levels) - 1, 0, -1):
    s.levels[li - 1].Q = s.levels[li].down.restrict(s.levels[li].Q)
for lev in s.levels:
    op, Q = lev.op, lev.Q
    R = op.new_field()
    norm = torch.zeros(1, dtype=torch.float64, device="cuda")
    S = op.m_inv_apply(Q)          # nonzero source like a coarse FAS level
    for _ in range(3):
        op.residual_device(Q, S, out=R, norm=norm)
    torch.cuda.synchronize()
    _lib.timing_read(); _lib.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 10
    e0.record()
    for _ in range(k):
        op.residual_device(Q, S, out=R, norm=norm)
    e1.record(); torch.cuda.synchronize()
    _lib.timing_enable(False)
    kt = _lib.timing_read()
    ms = e0.elapsed_time(e1) / k
    n = op.orders.num_nodes
    print(f"N={op.orders.orders[0].tolist()} nodes {n} ms/eval {ms:.4f} ns/node {1e6 * ms / n:.3f}",
          {a: round(v[0] / k, 4) for a, v in kt.items() if v[1]})
