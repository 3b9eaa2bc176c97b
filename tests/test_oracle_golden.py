"""Pin the CPU oracle against golden vectors produced by the REAL reference
(tests/golden/make_golden.py).  The reference's 2D scalar Legendre-Gauss path
is reproduced through the one-element-deep, z-self-periodic N3=0 extrusion."""

import warnings

import numpy as np
import numpy.polynomial.legendre as npleg
import pytest

from helpers import (golden_law, golden_mesh, load, oracle_law, oracle_to_ref_flat,
                     orders3, ref_flat_to_oracle)
from oracle import adaptation, multigrid, spectral, tau, timestep
from oracle.fields import OrderField
from oracle.operators import DGOperator

OP_CASES = ["sine_warp_mixed", "burgers_mixed", "rotated_pair", "graded_bl",
            "runge_curved", "aniso_burgers_curved"]


def _setup(name):
    g = load(name)
    m = golden_mesh(g)
    law = oracle_law(golden_law(g))
    of = OrderField(orders3(g["orders"]))
    return g, m, law, of


def test_spectral_matches_reference():
    g = load("spectral")
    for n in range(9):
        x, w = spectral.rule(n, "LG")
        assert np.max(np.abs(x - g[f"x_{n}"])) < 5e-15
        assert np.max(np.abs(w - g[f"w_{n}"])) < 5e-15
        assert np.max(np.abs(spectral.differentiation_matrix(n) - g[f"D_{n}"])) < 1e-12
        assert np.max(np.abs(spectral.boundary_rows(n) - g[f"B_{n}"])) < 1e-13
    for a in range(8):
        for b in range(8):
            # modal projection == reference closed form on LG nodes
            assert np.max(np.abs(spectral.transfer(a, b) - g[f"T_{a}_{b}"])) < 1e-13


def test_lobatto_rule_exactness_and_transfers():
    for n in range(1, 9):
        x, w = spectral.rule(n, "LGL")
        assert x[0] == -1.0 and x[-1] == 1.0
        for k in range(2 * n):            # LGL exact to degree 2N-1
            exact = 0.0 if k % 2 else 2.0 / (k + 1)
            assert abs(np.sum(w * x ** k) - exact) < 1e-13
        xl, _ = npleg.leggauss(n + 1)
        # restrict o prolong = identity on both families
        for fam in ("LG", "LGL"):
            if n >= 2:
                rp = spectral.transfer(n, n - 1, fam) @ spectral.transfer(n - 1, n, fam)
                assert np.max(np.abs(rp - np.eye(n))) < 1e-12


@pytest.mark.parametrize("name", OP_CASES)
def test_operator_matches_reference(name):
    g, m, law, of = _setup("op_" + name)
    op = DGOperator(m, law, of, family="LG", form="cross")
    Q = ref_flat_to_oracle(g["Q"], of)
    scale = np.abs(g["A"]).max()
    assert np.abs(oracle_to_ref_flat(op.apply(Q)) - g["F"]).max() < 1e-13 * np.abs(g["F"]).max()
    assert np.abs(oracle_to_ref_flat(op.apply(Q, isolated=True)) - g["Fiso"]).max() < 1e-13 * np.abs(g["Fiso"]).max()
    assert np.abs(oracle_to_ref_flat(op.residual(Q)) - g["R"]).max() < 1e-13 * scale
    assert np.abs(op.truncation(Q) - g["tau"]).max() < 1e-13 * g["tau"].max()
    assert np.abs(op.truncation(Q, isolated=True) - g["tau_iso"]).max() < 1e-13 * g["tau_iso"].max()
    mass = np.concatenate([op.group_ops[of.element_slot[e][0]].mass[of.element_slot[e][1]].ravel()
                           for e in range(of.num_elements)])
    assert np.abs(mass - g["mass"]).max() < 1e-14 * g["mass"].max()


@pytest.mark.parametrize("name", ["sine_warp_mixed", "burgers_mixed", "runge_curved"])
def test_rk3_matches_reference(name):
    g, m, law, of = _setup("op_" + name)
    op = DGOperator(m, law, of)
    Q = ref_flat_to_oracle(g["Q"], of)
    cfg = timestep.TimeConfig()
    assert np.abs(timestep.element_dt(op, Q, cfg) - g["element_dt"]).max() < 1e-15
    Qr, r0 = Q.copy(), []
    for _ in range(2):
        r0.append(timestep.rk3_step(op, Qr, timestep.compute_dt(op, Qr, cfg)))
    assert np.abs(oracle_to_ref_flat(Qr) - g["Q_rk2"]).max() < 1e-13
    assert np.abs(np.array(r0) - g["r0_rk2"]).max() < 1e-13 * np.abs(g["r0_rk2"]).max()
    Ql = Q.copy()
    rl = timestep.rk3_step(op, Ql, timestep.compute_dt(op, Ql, timestep.TimeConfig(local=True)))
    assert np.abs(oracle_to_ref_flat(Ql) - g["Q_rk_local"]).max() < 1e-13
    assert abs(rl - float(g["r0_local"])) < 1e-13 * abs(float(g["r0_local"]))


def test_transfers_match_reference():
    g = load("transfer")
    fo, co = OrderField(orders3(g["fine"])), OrderField(orders3(g["coarse"]))
    t = multigrid.OrderTransfer(fo, co)
    assert np.abs(oracle_to_ref_flat(t.restrict(ref_flat_to_oracle(g["Qf"], fo))) - g["restricted"]).max() < 1e-13
    assert np.abs(oracle_to_ref_flat(t.prolong(ref_flat_to_oracle(g["Qc"], co))) - g["prolonged"]).max() < 1e-13


@pytest.mark.parametrize("name", ["vcycle_sine4", "vcycle_burgers3", "vcycle_sine3_tuned"])
def test_vcycle_history_matches_reference(name):
    g, m, law, of = _setup("mg_" + name)
    sm = multigrid.SmootherConfig(
        pre_sweeps=int(g["smoother_pre_sweeps"]), post_sweeps=int(g["smoother_post_sweeps"]),
        coarsest_sweeps=int(g["smoother_coarsest_sweeps"]), max_batches=int(g["smoother_max_batches"]))
    s = multigrid.FASSolver(m, law, of, smoother=sm)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for _ in range(int(g["log_cycle"].max())):
            s.v_cycle()
    rn = np.array([r["rnorm"] for r in s.log])
    assert len(rn) == len(g["log_rnorm"])
    assert [r["phase"] for r in s.log] == list(g["log_phase"])
    assert (np.array([r["sweeps"] for r in s.log]) == g["log_sweeps"]).all()
    # history parity measured against max(|r0|, |A|)
    assert np.abs(rn - g["log_rnorm"]).max() < 1e-10 * g["log_rnorm"].max()
    assert np.abs(oracle_to_ref_flat(s.Q) - g["Q"]).max() < 1e-12
    assert s.work_units == pytest.approx(float(g["work_units"]), rel=1e-14)


@pytest.mark.parametrize("name", ["sine4", "aniso5"])
def test_tau_maps_and_selection_match_reference(name):
    g, m, law, of = _setup("tau_" + name)
    op = DGOperator(m, law, of)
    Q = ref_flat_to_oracle(g["Q"], of)
    for iso in (True, False):
        tm = tau.estimate(m, law, Q, 1e6, isolated=iso, fine_op=op)
        ref = g["tau_iso" if iso else "tau_coupled"]
        for e in range(of.num_elements):
            assert not tm.tau[e][2]
            for d in range(2):
                want = {n: ref[e, d, n] for n in range(ref.shape[2]) if np.isfinite(ref[e, d, n])}
                assert set(tm.tau[e][d]) == set(want)
                for n, v in want.items():
                    assert abs(tm.tau[e][d][n] - v) <= 1e-11 * max(v, 1e-300)
        if not iso:
            continue
        nmax = int(of.orders.max()) + 2
        tau.extrapolate_map(tm, nmax)
        for k, tmax in enumerate(g["tau_max_list"]):
            cfg = adaptation.AdaptConfig(tau_max=float(tmax), n_max=nmax)
            sel, paths, _ = adaptation.select_orders(tm, cfg)
            assert (sel.orders[:, :2] == g[f"select_{k}"]).all()
            assert list(paths) == list(g[f"select_paths_{k}"])
            assert (adaptation.limit_jumps(m, sel).orders[:, :2] == g[f"limited_{k}"]).all()
            assert (adaptation.limit_jumps(m, sel, "softened").orders[:, :2] == g[f"softened_{k}"]).all()
