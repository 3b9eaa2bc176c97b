"""Parity at the BASELINE.json sizes, against committed CPU-oracle fixtures
(tests/golden/oracle_*.npz, made by tests/golden/make_config_fixtures.py;
summaries and tolerances in tests/fullsize.py).

* config 3 (32^3, orders U{1..7}^3, 4.11 M nodes): residual, one RK3 step,
  coupled and isolated element tau, and the config's tau estimation;
* config 4 (24^3, N=7, 7.08 M nodes): fine residual and every restriction /
  prolongation pair 7->6 ... 2->1; the 7-level V-cycle protocol on 8^3
  (3 cycles: residual history, sweeps, final state);
* config 2 (40x20 flat plate, N=5): two 5-level V-cycles (history), then tau
  (Nz frozen) and the p-map (tau_max 1e-4, orders 1..5) from the oracle's state;
* config 5 (cubed-sphere shell, N=3, 2.36 M nodes): residual, tau and the
  stage-1 p-map (tau_max 1e-2, orders 1..6).

Tolerances (north_star): residuals 1e-12 relative to |A(Q)|_inf, tau 1e-12
relative to max tau, histories 1e-10 relative to max |r|, p-maps identical
except for elements whose tau sum lies within 1e-10 of the threshold.
Measured worst errors are appended to $PARITY_REPORT (JSON lines) when set.
"""

from __future__ import annotations

import itertools
import json
import os
import warnings

import numpy as np
import pytest

import fullsize as fz

pytestmark = pytest.mark.gpu


def _report(name, **vals):
    path = os.environ.get("PARITY_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps({"case": name, **vals}) + "\n")


def _oo(orders):
    from oracle.fields import OrderField as OO

    return OO(np.asarray(orders.orders))


def _need(name):
    if not fz.have(name):
        pytest.skip(f"fixture oracle_{name}.npz not generated")
    return fz.load(name)


def _tau_compare(dense_gpu, dense_ref, what):
    nan_g, nan_r = np.isnan(dense_gpu), np.isnan(dense_ref)
    assert (nan_g == nan_r).all(), f"{what}: recorded entries differ"
    fin = ~nan_r & np.isfinite(dense_ref)
    assert (np.isinf(dense_gpu[~nan_r]) == np.isinf(dense_ref[~nan_r])).all()
    top = float(np.max(dense_ref[fin]))
    err = float(np.max(np.abs(dense_gpu[fin] - dense_ref[fin]))) / top
    return err, top


def _near_threshold(tau_ext, e, orders_e, tau_max, n_min, n_max, frozen=()):
    """Some candidate order triple of element e sums to within 1e-10 of tau_max."""
    act = [d for d in range(3) if orders_e[d] > 0 and d not in frozen]
    choices = [[n for n in range(n_min, n_max + 1) if not np.isnan(tau_ext[e, d, n])] for d in act]
    for combo in itertools.product(*choices):
        v = sum(tau_ext[e, d, n] for d, n in zip(act, combo))
        if np.isfinite(v) and abs(v - tau_max) <= 1e-10 * tau_max:
            return True
    return False


def _pmap_compare(got, ref, tau_ext, fine_orders, tau_max, n_max, frozen=()):
    bad = np.flatnonzero((got != ref).any(axis=1))
    for e in bad:
        assert _near_threshold(tau_ext, e, fine_orders[e], tau_max, 1, n_max, frozen), \
            f"element {e}: orders {got[e]} vs oracle {ref[e]}"
    return len(bad)


# --------------------------------------------------------------------------- config 3
def test_config3_fullsize_residual_rk_and_tau():
    from paper_1806_11456_b200 import configs, operators, timestep

    fx = _need("cfg3")
    w = configs.config3()
    oo = _oo(w.orders)
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q0 = op.project_function(w.init)
    scale = float(fx["A_norm"])
    e_q = fz.compare_field(fx, "Q0", oo, Q0.to_oracle_blocks(), float(np.max(fx["Q0_emax"])), tol=1e-15)
    e_r = fz.compare_field(fx, "r", oo, op.residual(Q0).to_oracle_blocks(), scale)
    taus = {}
    for iso in (0, 1):
        t, to = op.truncation(Q0, isolated=bool(iso)), fx[f"tau_elem_{iso}"]
        taus[iso] = float(np.abs(t - to).max() / to.max())
        assert taus[iso] <= 1e-12, f"element tau (isolated={iso}) off by {taus[iso]:.3e} of max tau"
    dt = timestep.compute_dt(op, Q0, timestep.TimeConfig())
    assert abs(dt - float(fx["rk_dt"])) <= 1e-14 * float(fx["rk_dt"])
    Q1 = Q0.copy()
    r0 = timestep.rk3_step(op, Q1, dt)
    assert abs(r0 - float(fx["rk_r0"])) <= 1e-12 * scale
    e_dq = fz.compare_field(fx, "dQ", oo, (Q1 - Q0).to_oracle_blocks(), dt * scale)
    _report("cfg3_fullsize", Q0=e_q, r=e_r, tau_coupled=taus[0], tau_isolated=taus[1], dQ=e_dq,
            r0=abs(r0 - float(fx["rk_r0"])) / scale)


def test_config3_fullsize_tau_estimate():
    from paper_1806_11456_b200 import configs, operators, tau

    fx = _need("cfg3_tau")
    w = configs.config3()
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q0 = op.project_function(w.init)
    tm = tau.estimate(w.mesh, w.law, Q0, 1e6, isolated=True, fine_op=op)
    err, top = _tau_compare(fz.tau_dense(tm, w.mesh.num_elements), fx["tau"], "cfg3 tau map")
    assert err <= 1e-12, f"cfg3 tau map off by {err:.3e} of max tau"
    assert tm.work_units == pytest.approx(float(fx["work_units"]), rel=1e-14)
    _report("cfg3_tau_estimate", tau_rel_max_tau=err, max_tau=top,
            tau_rel_F=err * top / float(fx["F_norm"]))


# --------------------------------------------------------------------------- config 4
def test_config4_fullsize_residual_and_transfers():
    from paper_1806_11456_b200 import configs, multigrid, operators

    fx = _need("cfg4")
    w = configs.config4()
    oo = _oo(w.orders)
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q0 = op.project_function(w.init)
    qn = float(np.max(fx["Q0_emax"]))
    rep = {"Q0": fz.compare_field(fx, "Q0", oo, Q0.to_oracle_blocks(), qn, tol=1e-15),
           "r": fz.compare_field(fx, "r", oo, op.residual(Q0).to_oracle_blocks(), float(fx["A_norm"]))}
    del op
    fields = multigrid.level_order_fields(w.orders, "high-order")
    X = Q0
    for k in range(len(fields) - 1, 0, -1):
        t = multigrid.OrderTransfer(fields[k], fields[k - 1], nv=5, family=w.family)
        Xc = t.restrict(X)
        n = int(fields[k].orders[0, 0])
        rep[f"R{n}"] = fz.compare_field(fx, f"R{n}", _oo(fields[k - 1]), Xc.to_oracle_blocks(), qn)
        rep[f"P{n}"] = fz.compare_field(fx, f"P{n}", _oo(fields[k]), t.prolong(Xc).to_oracle_blocks(), qn)
        X = Xc
    _report("cfg4_fullsize", **rep)


def test_config4_vcycle_protocol_8cubed():
    from paper_1806_11456_b200 import configs, multigrid

    fx = _need("cfg4_vcycle")
    w = configs.config4(n=8)
    s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                            family=w.family, form=w.form)
    s.set_state(s.finest.op.project_function(w.init))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(3):
            s.v_cycle()
    assert [r["level"] for r in s.log] == list(fx["log_level"])
    assert [r["phase"] for r in s.log] == list(fx["log_phase"])
    assert [r["sweeps"] for r in s.log] == list(fx["log_sweeps"])
    rn = np.array([r["rnorm"] for r in s.log])
    ref = fx["log_rnorm"]
    e_h = float(np.abs(rn - ref).max() / ref.max())
    assert e_h <= 1e-10
    assert s.work_units == pytest.approx(float(fx["work_units"]), rel=1e-14)
    e_q = fz.compare_field(fx, "Q", _oo(s.finest.orders), s.Q.to_oracle_blocks(), float(fx["Q_norm"]),
                           tol=1e-10)
    _report("cfg4_vcycle_8cubed", history=e_h, Q=e_q)


# --------------------------------------------------------------------------- config 2
def _load_state(field, flat):
    from paper_1806_11456_b200.fields import NodalField

    blocks, pos = [], 0
    for sig, ids in zip(field.group_orders, field.group_elements):
        shape = (len(ids), 5) + tuple(int(x) + 1 for x in sig)
        k = int(np.prod(shape))
        blocks.append(flat[pos:pos + k].reshape(shape))
        pos += k
    assert pos == len(flat)
    return NodalField.zeros(field, 5).load_oracle_blocks(blocks)


def test_config2_fullsize_vcycles_tau_and_pmap():
    from paper_1806_11456_b200 import adaptation, configs, multigrid, tau, timestep

    fx = _need("cfg2")
    w = configs.config2()
    s = multigrid.FASSolver(w.mesh, w.law, w.orders, smoother=multigrid.SmootherConfig(**w.smoother),
                            time_config=timestep.TimeConfig(**w.time), family=w.family, form=w.form)
    s.set_state(s.finest.op.project_function(w.init))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(2):
            s.v_cycle()
    assert [(r["level"], r["phase"], r["sweeps"]) for r in s.log] == \
        list(zip(fx["log_level"], fx["log_phase"], fx["log_sweeps"]))
    rn = np.array([r["rnorm"] for r in s.log])
    e_h = float(np.abs(rn - fx["log_rnorm"]).max() / fx["log_rnorm"].max())
    assert e_h <= 1e-10
    # tau and the p-map from the oracle's state (identical inputs)
    Qin = _load_state(s.finest.orders, fx["Q_state"])
    tm = tau.estimate(w.mesh, w.law, Qin, 1e6, isolated=True, fine_op=s.finest.op, frozen=(2,))
    nel = w.mesh.num_elements
    err, top = _tau_compare(fz.tau_dense(tm, nel), fx["tau"], "cfg2 tau map")
    assert err <= 1e-12, f"cfg2 tau off by {err:.3e} of max tau"
    tmax, nmax = float(fx["tau_max"]), int(fx["n_max"])
    tau.extrapolate_map(tm, nmax)
    ext = fz.tau_dense(tm, nel)
    sel, _ = adaptation.select_orders(tm, adaptation.AdaptConfig(tau_max=tmax, n_max=nmax))
    nsel = _pmap_compare(np.asarray(sel.orders), fx["sel_orders"], fx["tau_ext"], w.orders.orders, tmax, nmax,
                         frozen=(2,))
    lim = adaptation.limit_jumps(w.mesh, sel)
    if nsel == 0:
        assert (np.asarray(lim.orders) == fx["lim_orders"]).all()
    assert (np.asarray(lim.orders)[:, 2] == 1).all()        # Nz held
    fin = np.isfinite(fx["tau_ext"])
    e_ext = float(np.max(np.abs(ext[fin] - fx["tau_ext"][fin]) / np.maximum(np.abs(fx["tau_ext"][fin]), 1e-300)))
    _report("cfg2_fullsize", history=e_h, tau_rel_max_tau=err, max_tau=top, pmap_mismatch=nsel,
            tau_ext_rel=e_ext, tau_rel_F=err * top / float(fx["F_norm"]),
            dofs_before=int(w.orders.dofs()), dofs_after=int(lim.dofs()))


# --------------------------------------------------------------------------- config 5
def test_config5_fullsize_residual_tau_and_pmap():
    from paper_1806_11456_b200 import adaptation, configs, operators, tau

    fx = _need("cfg5")
    w = configs.config5()
    oo = _oo(w.orders)
    op = operators.DGOperator(w.mesh, w.law, w.orders, family=w.family, form=w.form)
    Q0 = op.project_function(w.init)
    e_q = fz.compare_field(fx, "Q0", oo, Q0.to_oracle_blocks(), float(np.max(fx["Q0_emax"])), tol=1e-15)
    e_r = fz.compare_field(fx, "r", oo, op.residual(Q0).to_oracle_blocks(), float(fx["A_norm"]))
    tm = tau.estimate(w.mesh, w.law, Q0, 1e6, isolated=True, fine_op=op)
    nel = w.mesh.num_elements
    err, top = _tau_compare(fz.tau_dense(tm, nel), fx["tau"], "cfg5 tau map")
    assert err <= 1e-12, f"cfg5 tau off by {err:.3e} of max tau"
    tmax, nmax = float(fx["tau_max"]), int(fx["n_max"])
    tau.extrapolate_map(tm, nmax)
    sel, _ = adaptation.select_orders(tm, adaptation.AdaptConfig(tau_max=tmax, n_max=nmax))
    nsel = _pmap_compare(np.asarray(sel.orders), fx["sel_orders"], fx["tau_ext"], w.orders.orders, tmax, nmax)
    lim = adaptation.limit_jumps(w.mesh, sel)
    if nsel == 0:
        assert (np.asarray(lim.orders) == fx["lim_orders"]).all()
    _report("cfg5_fullsize", Q0=e_q, r=e_r, tau_rel_max_tau=err, max_tau=top, pmap_mismatch=nsel,
            tau_rel_F=err * top / float(fx["F_norm"]), dofs_before=int(w.orders.dofs()),
            dofs_after=int(lim.dofs()))
