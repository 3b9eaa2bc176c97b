"""element_dt / norm kernels on the config-4 levels: CUDA-event times and
achieved HBM bandwidth (development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1806_11456_b200 import configs, fields, operators

peak = 6550.1
w = configs.config4(n=24)
for N in (7, 5, 3, 1):
    of = fields.OrderField.uniform(24 ** 3, N)
    op = operators.DGOperator(w.mesh, w.law, of, family=w.family, form=w.form)
    Q = op.project_function(w.init)
    dt_slot = torch.zeros(24 ** 3, dtype=torch.float64, device="cuda")
    dt_min = torch.full((1,), float("inf"), dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")

    def timed(fn, reps=20):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    b = 40 * of.num_nodes
    t_dt = timed(lambda: op.element_dt_device(Q, 0.2, 0.1, dt_slot=dt_slot, dt_min=dt_min))
    t_n = timed(lambda: op.norm_inf_device(Q, out=out))
    print("N=%d nodes %d  element_dt %.4f ms (%.0f%%)  norm %.4f ms (%.0f%%)" % (
        N, of.num_nodes, t_dt, 100 * b / t_dt / 1e6 / peak, t_n, 100 * b / t_n / 1e6 / peak), flush=True)
