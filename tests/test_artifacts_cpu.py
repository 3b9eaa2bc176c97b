"""Binary artifacts: solution and tau-map round trips, on CPU
tensors (the writer's device->host copy is the same call on the GPU)."""

import numpy as np
import pytest
import torch

from paper_1806_11456_b200 import artifacts, tau
from paper_1806_11456_b200.errors import ConfigError
from paper_1806_11456_b200.fields import NodalField, OrderField


def _field(seed=0, nel=37, nv=5):
    rng = np.random.default_rng(seed)
    of = OrderField(rng.integers(1, 8, (nel, 3)))
    vals = rng.standard_normal(of.num_nodes * nv)
    vals[::17] = np.array([np.pi, -0.0, 1e-300, 1.0 / 3.0, 2.0 ** -1074])[np.arange(len(vals[::17])) % 5]
    return NodalField.from_slot_array(of, vals, nv, "cpu")


def test_solution_round_trip_is_bit_exact(tmp_path):
    Q = _field()
    p = artifacts.write_solution(tmp_path / "sol.tdgsol", Q, digest="abc123", case="cfg-test")
    R, digest, case = artifacts.read_solution(p, device="cpu")
    assert (digest, case) == ("abc123", "cfg-test")
    assert (np.asarray(R.field.orders) == np.asarray(Q.field.orders)).all()
    assert torch.equal(R.data.view(torch.int64), Q.data.view(torch.int64))      # bitwise
    # 8 bytes per value plus a small header: the reference's text dump needs ~20
    assert p.stat().st_size < 8 * Q.data.numel() + 64 + 16 * Q.field.num_elements + 32


def test_solution_rejects_foreign_and_truncated_files(tmp_path):
    bad = tmp_path / "x.tdgsol"
    bad.write_bytes(b"taudg solution 1\n")
    with pytest.raises(ConfigError):
        artifacts.read_solution(bad, device="cpu")
    p = artifacts.write_solution(tmp_path / "s.tdgsol", _field(1), "d", "c")
    raw = p.read_bytes()
    (tmp_path / "t.tdgsol").write_bytes(raw[:-8])
    with pytest.raises((ConfigError, ValueError)):
        artifacts.read_solution(tmp_path / "t.tdgsol", device="cpu")


def test_atomic_write_leaves_no_temp_files(tmp_path):
    artifacts.write_solution(tmp_path / "a.tdgsol", _field(2), "d", "c")
    assert sorted(x.name for x in tmp_path.iterdir()) == ["a.tdgsol"]


def _tau_map(seed=3, nel=25):
    rng = np.random.default_rng(seed)
    of = OrderField(np.concatenate([rng.integers(2, 7, (nel, 2)), np.ones((nel, 1), int)], axis=1))
    tm = tau.TauMap(of, tau.EstimationContext(1e-5, 3.2e-6, True))
    tm.frozen |= {2}
    tm.work_units = 1.75
    for e in range(nel):
        for d in range(2):
            p = int(of.orders[e, d])
            for n in range(1, p):
                tm.record(e, d + 1, n, float(10.0 ** (-n) * rng.uniform(0.5, 2.0)))
    tau.extrapolate_map(tm, 7)
    return tm


def test_tau_map_round_trip(tmp_path):
    tm = _tau_map()
    p = artifacts.write_tau_map(tmp_path / "tau.npz", tm, digest="dd")
    rt, digest = artifacts.read_tau_map(p)
    assert digest == "dd"
    assert rt.frozen == tm.frozen and rt.n_max == tm.n_max and rt.work_units == tm.work_units
    assert rt.context == tm.context
    for e in range(tm.num_elements):
        for d in range(3):
            assert rt.tau[e][d] == tm.tau[e][d]                 # exact floats, inf included
            assert rt.extrapolated[e][d] == tm.extrapolated[e][d]
            assert rt.fits[e][d] == tm.fits[e][d]
            assert rt.non_spectral[e][d] == tm.non_spectral[e][d]
    assert rt.to_dict() == tm.to_dict()


def test_write_run_file_set(tmp_path):
    Q = _field(4, nel=8)
    hist = [{"cycle": 1, "level": 3, "phase": "post", "sweeps": 3, "rnorm": 1e-3, "work_units": 2.0, "wall": 0.1}]
    summary = artifacts.write_run(tmp_path / "run", Q=Q, history=hist, work_units=2.0, residual_norm=1e-3,
                                  digest="d0", name="t", case="c", maps=[_tau_map(5, 8)])
    names = sorted(x.name for x in (tmp_path / "run").iterdir())
    assert names == sorted(summary["files"])
    assert {"solution.tdgsol", "tau_map_stage1.npz", "residual_history.csv", "summary.json"} <= set(names)
