"""Stage-by-stage GPU-vs-oracle diagnostic (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from helpers import oracle_law
from oracle.fields import OrderField as OO, NodalField as ON
from oracle.operators import DGOperator as ODG
from paper_1806_11456_b200 import fields, operators, physics, mesh

def to_o(pf, of_o):
    return ON(of_o, pf.to_oracle_blocks(), pf.nv)

def run(label, msh, law, orders, fam, form):
    of_p, of_o = fields.OrderField(orders), OO(orders)
    op = operators.DGOperator(msh, law, of_p, family=fam, form=form)
    oo = ODG(msh, oracle_law(law), of_o, family=fam, form=form)
    if law.nv == 1:
        fn = lambda x, y, z: 1.0 + 0.3 * np.sin(3 * x + y - 2 * z)
    else:
        fs = law.freestream()
        fn = lambda x, y, z: np.stack([fs[v] + 1e-2 * np.sin(2*np.pi*(x + 2*y) + v) for v in range(5)])
    Q, Qo = op.project_function(fn), oo.project_function(fn)
    out = []
    for iso in (False, True):
        F = to_o(op.apply(Q, iso), of_o); Fo = oo.apply(Qo, iso)
        out.append((F - Fo).norm_inf() / max(Fo.norm_inf(), 1e-300))
        if law.viscous:
            G = op.gradient(Q, iso).cpu().numpy(); Go = oo.gradient(Qo, iso)
            pos = 0; err = 0
            for g, (sig, ids) in enumerate(zip(of_o.group_orders, of_o.group_elements)):
                n = int(np.prod(np.array(sig) + 1))
                blk = G[pos: pos + len(ids)*n*3*law.ngv].reshape(len(ids), 3, law.ngv, sig[2]+1, sig[1]+1, sig[0]+1).transpose(0,1,2,5,4,3)
                pos += blk.size
                err = max(err, np.abs(blk - Go[g]).max() / max(np.abs(Go[g]).max(), 1e-300))
            out.append(err)
    print(f"{label:40s}", " ".join(f"{v:.2e}" for v in out), flush=True)

box = mesh.build_box(2, 2, 1, bounds=((0,1),(0,1),(0,1)))
o_uni = lambda nel, n: np.full((nel, 3), n)
for mu in (0.0, 0.1):
    law = physics.AdvectionDiffusion((0.8, 1.7, 0.4), mu)
    run(f"advdiff mu={mu} LG uniform3 box", box, law, o_uni(4, 3), "LG", "cross")
    run(f"advdiff mu={mu} LGL uniform3 box", box, law, o_uni(4, 3), "LGL", "cross")
    run(f"advdiff mu={mu} LG aniso(2,3,4)", box, law, np.tile([2,3,4], (4,1)), "LG", "cross")
    run(f"advdiff mu={mu} LG mixed", box, law, np.random.default_rng(1).integers(1,5,(4,3)), "LG", "cross")
law = physics.NavierStokes(mach=0.3, reynolds=0.0)
run("euler LGL uniform3", box, law, o_uni(4,3), "LGL", "curl")
law = physics.NavierStokes(mach=0.3, reynolds=100.0)
run("NS LGL uniform3", box, law, o_uni(4,3), "LGL", "curl")

# per-side trace comparison, mixed orders viscous
law = physics.AdvectionDiffusion((0.8, 1.7, 0.4), 0.1)
orders = np.random.default_rng(1).integers(1,5,(4,3))
print("orders", orders.tolist())
of_p, of_o = fields.OrderField(orders), OO(orders)
op = operators.DGOperator(box, law, of_p, family="LG", form="cross")
oo = ODG(box, oracle_law(law), of_o, family="LG", form="cross")
fn = lambda x, y, z: 1.0 + 0.3 * np.sin(3 * x + y - 2 * z)
Q, Qo = op.project_function(fn), oo.project_function(fn)
op.apply(Q, True)
trq_o = oo._traces(Qo.blocks)
G = oo.gradient(Qo, True)
trg_o = oo._traces(G, lead=3)
for which, ref in ((0, trq_o), (2, trg_o)):
    buf = op.debug_buffer(which)
    for e in range(4):
        g, r = of_o.element_slot[e]
        errs = []
        for s in range(6):
            want = ref[g][s][r].reshape(-1, *ref[g][s][r].shape[-2:])
            got = buf[(e, s)]
            errs.append(np.abs(got - want).max() if got.shape == want.shape else -1)
        print("buf", which, "elem", e, orders[e].tolist(), " ".join(f"{x:.1e}" for x in errs))

# isolated flux surface buffer vs oracle per-side analytic flux * sigma
op.apply(Q, True)
fs_buf = op.debug_buffer(3)
for e in range(4):
    g, r = of_o.element_slot[e]
    go = oo.group_ops[g]
    errs = []
    for s in range(6):
        q_in = trq_o[g][s][r:r+1]; Gs = trg_o[g][s][r:r+1]
        n = go.side_normal[s][r:r+1]; sg = go.side_sigma[s][r:r+1]
        fl = oo.law.adv_flux(q_in); fv = oo.law.visc_flux(q_in, Gs)
        F = np.einsum("bd...,bdv...->bv...", n, fl) - np.einsum("bd...,bdv...->bv...", n, fv)
        want = (F * sg[:, None])[0]
        errs.append(np.abs(fs_buf[(e, s)] - want).max())
    print("fsurf iso elem", e, " ".join(f"{x:.1e}" for x in errs))

# rebuild isolated F from the GPU's own gradient + fsurf with oracle arithmetic
F_gpu = to_o(op.apply(Q, True), of_o)
Gg = op.gradient(Q, True).cpu().numpy()
fs_buf = op.debug_buffer(3)
pos = 0
for g, (sig, ids) in enumerate(zip(of_o.group_orders, of_o.group_elements)):
    n = int(np.prod(np.array(sig) + 1))
    blk = Gg[pos: pos + len(ids)*n*3].reshape(len(ids), 3, 1, sig[2]+1, sig[1]+1, sig[0]+1).transpose(0,1,2,5,4,3)
    pos += blk.size
    go = oo.group_ops[g]
    q = Qo.blocks[g]
    f = oo.law.adv_flux(q) - oo.law.visc_flux(q, blk)
    ft = np.einsum("bidxyz,bdvxyz->bivxyz", go.ja, f)
    Fv = -oo._weak_div(g, ft)
    tmp = [Fv.copy()]
    for s in range(6):
        vec = np.stack([fs_buf[(int(e), s)] for e in ids])
        oo._scatter(tmp, 0, np.arange(len(ids)), s, vec) if False else None
    # manual scatter into tmp[0]
    out = Fv.copy()
    for k, e in enumerate(ids):
        for s in range(6):
            d = s // 2; a, b = [x for x in range(3) if x != d]
            vec = fs_buf[(int(e), s)]
            contrib = vec * (go.w[a][:, None] * go.w[b][None, :])
            row = go.bounds[d][s % 2]
            shape = [1, 1, 1]; shape[d] = len(row)
            out[k] += np.expand_dims(contrib, 1 + d) * row.reshape([1] + shape)
    print("bucket", sig, "GPU F vs numpy(GPU G, fsurf):", np.abs(F_gpu.blocks[g] - out).max(),
          " oracle G vs GPU G:", np.abs(blk - G[g]).max())
