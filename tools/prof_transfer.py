"""Transfer kernels of the config-4 level pairs: the line kernel vs the
one-output-per-thread kernel (TDG_TRANSFER_LINES=0), bitwise comparison and
CUDA-event times with achieved HBM bandwidth (development tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import torch
from paper_1806_11456_b200 import fields, multigrid

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=24)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
nel = a.n ** 3
peak = 6550.1


def timed(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


tot = {0: 0.0, 1: 0.0}
for N in range(7, 1, -1):
    of_f, of_c = fields.OrderField.uniform(nel, N), fields.OrderField.uniform(nel, N - 1)
    os.environ["TDG_TRANSFER_LINES"] = "0"
    t0 = multigrid.OrderTransfer(of_f, of_c, nv=5)
    del os.environ["TDG_TRANSFER_LINES"]
    t1 = multigrid.OrderTransfer(of_f, of_c, nv=5)
    g = torch.Generator(device="cuda").manual_seed(N)
    Qf = fields.NodalField(of_f, torch.rand(of_f.num_nodes * 5, dtype=torch.float64, device="cuda", generator=g), 5)
    Qc = fields.NodalField(of_c, torch.rand(of_c.num_nodes * 5, dtype=torch.float64, device="cuda", generator=g), 5)
    Qc0 = fields.NodalField(of_c, torch.rand(of_c.num_nodes * 5, dtype=torch.float64, device="cuda", generator=g), 5)
    nf, nc = of_f.num_nodes, of_c.num_nodes
    r = [t.restrict(Qf) for t in (t0, t1)]
    p = [t.prolong(Qc) for t in (t0, t1)]
    outs = [Qf.copy(), Qf.copy()]
    for t, o in zip((t0, t1), outs):
        t.prolong_add(Qc, o, Qc0)
    same = (torch.equal(r[0].data, r[1].data), torch.equal(p[0].data, p[1].data), torch.equal(outs[0].data, outs[1].data))
    row = []
    for k, t in enumerate((t0, t1)):
        oc, of = fields.NodalField.zeros(of_c, 5), fields.NodalField.zeros(of_f, 5)
        ms_r = timed(lambda: t.restrict(Qf, oc))
        ms_p = timed(lambda: t.prolong(Qc, of))
        ms_pa = timed(lambda: t.prolong_add(Qc, of, Qc0))
        b_r, b_p, b_pa = 40 * (nf + nc), 40 * (nf + nc), 40 * (2 * nf + 2 * nc)
        tot[k] += ms_r + ms_pa
        row.append("restrict %.3f ms (%.0f%%) prolong %.3f (%.0f%%) prolong_add %.3f (%.0f%%)" % (
            ms_r, 100 * b_r / ms_r / 1e6 / peak, ms_p, 100 * b_p / ms_p / 1e6 / peak,
            ms_pa, 100 * b_pa / ms_pa / 1e6 / peak))
    print("N=%d->%d bitwise %s\n  old  %s\n  line %s" % (N, N - 1, same, row[0], row[1]), flush=True)
print("sum restrict+prolong_add ms: old %.3f line %.3f" % (tot[0], tot[1]))
