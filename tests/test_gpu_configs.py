"""BASELINE.json configurations on the GPU.

* config 1 (the PR1 oracle run): 10 three-level V-cycles 3->2->1 with 3/3/3
  pinned sweeps from the seeded state, then one isolated tau estimate at N=3 —
  residual histories vs the oracle to 1e-10, tau to 1e-12 (identical inputs).
* config 3 distribution on a 6^3 sample: residual, RK3 stages and tau vs the
  oracle at 1e-12.
* full-size configs 3 and 4: size-independent properties (periodic mass
  conservation, RK3 fixed point of S = A(Q), bitwise run-to-run determinism).
"""

import warnings

import numpy as np
import pytest

from helpers import oracle_law

pytestmark = pytest.mark.gpu


def _report(name, **vals):
    import json
    import os

    path = os.environ.get("PARITY_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"case": name, **vals}) + "\n")


def _to_oracle(pf, of_o):
    from oracle.fields import NodalField as ON

    return ON(of_o, pf.to_oracle_blocks(), pf.nv)


def test_config1_protocol_matches_oracle():
    from oracle import multigrid as omg
    from oracle import tau as otau
    from oracle.fields import OrderField as OO
    from paper_1806_11456_b200 import configs, fields, multigrid, tau

    w = configs.config1()
    law = oracle_law(w.law)
    s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                            family=w.family, form=w.form)
    s.set_state(s.finest.op.project_function(w.init))
    so = omg.FASSolver(w.mesh, law, OO(np.asarray(w.orders.orders)), smoother=omg.SmootherConfig(**w.smoother),
                       family=w.family, form=w.form)
    so.set_state(so.finest.op.project_function(w.init))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(10):
            s.v_cycle()
            so.v_cycle()
    rn = np.array([r["rnorm"] for r in s.log])
    rno = np.array([r["rnorm"] for r in so.log])
    assert [(r["level"], r["phase"], r["sweeps"]) for r in s.log] == \
           [(r["level"], r["phase"], r["sweeps"]) for r in so.log]
    assert np.abs(rn - rno).max() <= 1e-10 * rno.max()
    assert s.work_units == pytest.approx(so.work_units, rel=1e-14)
    # tau at N=3 on identical inputs
    Qin = fields.NodalField.zeros(s.finest.orders, 5)
    Qin.load_oracle_blocks(so.Q.blocks)
    tm = tau.estimate(w.mesh, w.law, Qin, 1e6, isolated=True, fine_op=s.finest.op)
    tmo = otau.estimate(w.mesh, law, so.Q, 1e6, isolated=True, fine_op=so.finest.op,
                        family=w.family, form=w.form)
    # tau = |M (S - A)|: relative to max(max tau, |M A|_inf);
    # the error relative to max tau alone is reported
    top = max(v for e in range(64) for d in range(3) for v in tmo.tau[e][d].values())
    scale = max(top, so.finest.op.apply(so.Q, isolated=True).norm_inf())
    err = 0.0
    for e in range(64):
        for d in range(3):
            assert set(tm.tau[e][d]) == set(tmo.tau[e][d])
            for n, v in tmo.tau[e][d].items():
                err = max(err, abs(tm.tau[e][d][n] - v))
    assert err <= 1e-12 * scale
    _report("cfg1_protocol", history=float(np.abs(rn - rno).max() / rno.max()), tau_rel_max_tau=err / top,
            tau_rel_scale=err / scale, max_tau=top)


def test_config4_reduced_protocol_matches_oracle():
    """Config 4's protocol (N=7 Taylor-Green state, 7-level V-cycles 7..1 with
    2/2/2 pinned sweeps) on a 3^3 box: residual histories vs the oracle to
    1e-10, identical phase/sweep logs, final states to 1e-10."""
    from oracle import multigrid as omg
    from oracle.fields import OrderField as OO
    from paper_1806_11456_b200 import configs, multigrid

    w = configs.config4(n=3)
    law = oracle_law(w.law)
    s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                            family=w.family, form=w.form)
    s.set_state(s.finest.op.project_function(w.init))
    so = omg.FASSolver(w.mesh, law, OO(np.asarray(w.orders.orders)), smoother=omg.SmootherConfig(**w.smoother),
                       family=w.family, form=w.form)
    so.set_state(so.finest.op.project_function(w.init))
    assert len(s.levels) == len(so.levels) == 7
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(2):
            s.v_cycle()
            so.v_cycle()
    rn = np.array([r["rnorm"] for r in s.log])
    rno = np.array([r["rnorm"] for r in so.log])
    assert [(r["level"], r["phase"], r["sweeps"]) for r in s.log] == \
           [(r["level"], r["phase"], r["sweeps"]) for r in so.log]
    assert np.abs(rn - rno).max() <= 1e-10 * rno.max()
    Qf = _to_oracle(s.finest.Q, so.Q.field)
    assert (Qf - so.Q).norm_inf() <= 1e-10 * so.Q.norm_inf()


def test_config3_sample_matches_oracle():
    from oracle import timestep as ots
    from oracle.fields import OrderField as OO
    from oracle.operators import DGOperator as ODG
    from paper_1806_11456_b200 import configs, operators, timestep

    w = configs.config3(n=6)
    law = oracle_law(w.law)
    of_o = OO(np.asarray(w.orders.orders))
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    oo = ODG(w.mesh, law, of_o, family=w.family, form=w.form)
    Q, Qo = op.project_function(w.init), oo.project_function(w.init)
    scale = oo.m_inv_apply(Qo).norm_inf()
    assert (_to_oracle(op.residual(Q), of_o) - oo.residual(Qo)).norm_inf() <= 1e-12 * scale
    for iso in (False, True):
        t, to = op.truncation(Q, isolated=iso), oo.truncation(Qo, isolated=iso)
        assert np.abs(t - to).max() <= 1e-12 * to.max()
    cfg, ocfg = timestep.TimeConfig(), ots.TimeConfig()
    for _ in range(2):
        r = timestep.rk3_step(op, Q, timestep.compute_dt(op, Q, cfg))
        ro = ots.rk3_step(oo, Qo, ots.compute_dt(oo, Qo, ocfg))
        assert abs(r - ro) <= 1e-12 * scale
    assert (_to_oracle(Q, of_o) - Qo).norm_inf() <= 1e-12 * Qo.norm_inf()


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_properties(cfg):
    import torch

    from paper_1806_11456_b200 import configs, operators, timestep

    w = configs.config3() if cfg == 3 else configs.config4()
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q = op.project_function(w.init)
    # periodic telescoping: the continuity rows of F sum to zero
    F = op.apply(Q)
    nv, of = 5, op.orders
    cont = 0.0
    mx = 0.0
    for b in F.blocks:
        cont += float(b[:, 0].sum())
        mx = max(mx, float(b[:, 0].abs().max()))
    assert abs(cont) <= 1e-13 * mx * of.num_nodes
    # determinism: no atomics in accumulation -> bitwise identical re-evaluation
    F2 = op.apply(Q)
    assert torch.equal(F.data, F2.data)
    # RK3 fixed point: with S = A(Q), Q is the exact discrete steady state
    S = op.m_inv_apply(Q)
    Q1 = Q.copy()
    timestep.rk3_step(op, Q1, timestep.compute_dt(op, Q1, timestep.TimeConfig()), source=S)
    assert float((Q1.data - Q.data).abs().max()) <= 1e-12 * float(Q.data.abs().max())
