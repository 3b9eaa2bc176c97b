import sys, os, ctypes as C
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_1806_11456_b200 import configs, operators, _lib
cfg = int(sys.argv[1])
nn = int(sys.argv[2]) if len(sys.argv) > 2 else (32 if cfg == 3 else 24)
w = configs.config3(n=nn) if cfg == 3 else configs.config4(n=nn)
op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
Q = op.project_function(w.init); R = op.new_field()
norm = torch.zeros(1, dtype=torch.float64, device="cuda")
lib = C.CDLL(os.path.join(os.getcwd(), "paper_1806_11456_b200", "_taudg.so"))
buf = (C.c_ulonglong * 32)()
for _ in range(3): op.residual_device(Q, None, out=R, norm=norm)
torch.cuda.synchronize()
lib.tdg_debug_phases(None, 1)
for _ in range(5): op.residual_device(Q, None, out=R, norm=norm)
torch.cuda.synchronize()
lib.tdg_debug_phases(buf, 0)
a = np.array(list(buf), dtype=np.float64)
for base, n, name in ((0, 8, "lift"), (8, 5, "flux")):
    cnt = a[base]
    if cnt == 0: continue
    print(name, "blocks", int(cnt), "cycles/block per phase:", [round(a[base + z] / cnt) for z in range(1, n)], "sum", round(sum(a[base+1:base+n]) / cnt))
