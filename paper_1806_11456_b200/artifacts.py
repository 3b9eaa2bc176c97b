"""Binary run artifacts: solutions and truncation-error maps.

The reference writes the solution as text, one ``repr(float)`` per node
(artifacts.py:58-105), and tau maps as JSON (tau.py:114-146); at 10^7 nodes
the string formatting dominates a run's I/O.  Here both are binary and
self-describing, keep the reference's atomic-write contract (temp file in
the target directory, then rename, artifacts.py:33-45) and round-trip
bit-exactly:

* solution ``.tdgsol``: a fixed 56-byte header (magic, format version,
  unknowns per node, element count, string and value lengths), the config digest and case
  name, the per-slot element ids and (N1, N2, N3) orders (int32), then the
  field's float64 values in the device layout (slot order, per element
  [nv][N3+1][N2+1][N1+1]) — one device->host copy and one write, no
  per-node formatting.  ``read_solution`` rebuilds the OrderField (same
  slots) and uploads the values.
* tau map ``.npz`` (NumPy's binary container): dense per-(element,
  direction, order) tau values with NaN for "no entry", the extrapolated
  mask, the log-linear fits, non-spectral flags, frozen directions and the
  estimation context — everything ``TauMap.to_dict`` carries.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile
from pathlib import Path

import numpy as np

from .errors import ConfigError
from .fields import NodalField, OrderField

SOLUTION_MAGIC = b"TAUDGSOL"
SOLUTION_FORMAT = 1
_HEADER = struct.Struct("<8sIIqqqqq")      # magic, version, nv, nel, digest len, case len, value count, pad


def _atomic_write_bytes(path, chunks) -> Path:
    """Write byte chunks to ``path`` via a temp file and an atomic rename."""
    path = Path(path)
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=path.name + ".")
    try:
        with os.fdopen(fd, "wb") as fh:
            for c in chunks:
                fh.write(c)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
    return path


def write_solution(path, Q: NodalField, digest: str = "", case: str = "") -> Path:
    """Binary counterpart of solution_text (artifacts.py:58-76)."""
    of = Q.field
    dig, cs = digest.encode(), case.encode()
    vals = Q.data.detach().to("cpu").numpy()
    if vals.dtype != np.float64:
        raise ConfigError("solution values must be float64")
    head = _HEADER.pack(SOLUTION_MAGIC, SOLUTION_FORMAT, Q.nv, of.num_elements, len(dig), len(cs), vals.size, 0)
    meta = np.concatenate([np.asarray(of.slot_elem, np.int32),
                           np.asarray(of.slot_orders, np.int32).ravel()]).astype("<i4")
    return _atomic_write_bytes(path, [head, dig, cs, meta.tobytes(), np.ascontiguousarray(vals, "<f8").tobytes()])


def read_solution(path, device="cuda") -> tuple[NodalField, str, str]:
    """Rebuild (field, digest, case) from write_solution output (artifacts.py:79-105)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER.size:
        raise ConfigError(f"not a solution file: {path}")
    magic, version, nv, nel, ld, lc, nval, _ = _HEADER.unpack_from(raw, 0)
    if magic != SOLUTION_MAGIC:
        raise ConfigError(f"not a solution file: {path}")
    if version != SOLUTION_FORMAT:
        raise ConfigError(f"unsupported solution format {version}")
    pos = _HEADER.size
    digest = raw[pos:pos + ld].decode()
    pos += ld
    case = raw[pos:pos + lc].decode()
    pos += lc
    meta = np.frombuffer(raw, "<i4", 4 * nel, pos)
    pos += 16 * nel
    slot_elem, slot_orders = meta[:nel], meta[nel:].reshape(nel, 3)
    orders = np.zeros((nel, 3), np.int64)
    orders[slot_elem] = slot_orders
    field = OrderField(orders)
    if not (np.asarray(field.slot_elem) == slot_elem).all():
        raise ConfigError("solution slot order does not match the order field's bucketing")
    vals = np.frombuffer(raw, "<f8", nval, pos)
    if vals.size != field.num_nodes * nv:
        raise ConfigError("solution value count does not match its orders")
    return NodalField.from_slot_array(field, vals.copy(), nv, device), digest, case


def write_tau_map(path, tmap, digest: str = "") -> Path:
    """Binary counterpart of TauMap.to_dict / to_json (tau.py:114-146)."""
    nel = tmap.num_elements
    nmax = max(int(tmap.n_max), int(np.max(tmap.fine_orders.orders))) + 1
    for e in range(nel):
        for d in range(3):
            if tmap.tau[e][d]:
                nmax = max(nmax, max(tmap.tau[e][d]) + 1)
    tau = np.full((nel, 3, nmax), np.nan)
    extrap = np.zeros((nel, 3, nmax), bool)
    fits = np.full((nel, 3, 3), np.nan)
    nonspec = np.zeros((nel, 3), bool)
    for e in range(nel):
        for d in range(3):
            for n, v in tmap.tau[e][d].items():
                tau[e, d, n] = v
            for n in tmap.extrapolated[e][d]:
                extrap[e, d, n] = True
            f = tmap.fits[e][d]
            if f is not None:
                fits[e, d] = (f.slope, f.intercept, f.residual)
            nonspec[e, d] = bool(tmap.non_spectral[e][d])
    ctx = tmap.context
    meta = json.dumps({"config": digest, "isolated": bool(ctx.isolated), "threshold": float(ctx.threshold),
                       "residual_norm": float(ctx.residual_norm), "norm": "elementwise-inf",
                       "n_max": int(tmap.n_max), "frozen": sorted(int(d) for d in tmap.frozen),
                       "work_units": float(getattr(tmap, "work_units", 0.0))})
    path = Path(path)
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=path.name + ".", suffix=".npz")
    os.close(fd)
    try:
        np.savez(tmp, tau=tau, extrapolated=extrap, fits=fits, non_spectral=nonspec,
                 orders=np.asarray(tmap.fine_orders.orders, np.int32), meta=np.array(meta))
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
    return path


def read_tau_map(path):
    """Rebuild a TauMap written by write_tau_map."""
    from .tau import DirectionalFit, EstimationContext, TauMap

    with np.load(path, allow_pickle=False) as z:
        meta = json.loads(str(z["meta"]))
        tau, extrap, fits, nonspec = z["tau"], z["extrapolated"], z["fits"], z["non_spectral"]
        orders = OrderField(z["orders"].astype(np.int64))
    tm = TauMap(orders, EstimationContext(meta["threshold"], meta["residual_norm"], meta["isolated"]))
    tm.n_max = meta["n_max"]
    tm.frozen = set(meta["frozen"])
    tm.work_units = meta["work_units"]
    for e, d, n in zip(*np.nonzero(~np.isnan(tau))):
        tm.tau[e][d][int(n)] = float(tau[e, d, n])
    for e, d, n in zip(*np.nonzero(extrap)):
        tm.extrapolated[e][d].add(int(n))
    for e, d in zip(*np.nonzero(~np.isnan(fits[:, :, 0]))):
        tm.fits[e][d] = DirectionalFit(*(float(x) for x in fits[e, d]))
    for e, d in zip(*np.nonzero(nonspec)):
        tm.non_spectral[e][d] = True
    return tm, meta.get("config", "")


def write_run(out_dir, *, Q: NodalField, history, work_units: float, residual_norm: float, digest: str = "",
              name: str = "", case: str = "", maps=(), reports=()) -> dict:
    """Persist one finished run (artifacts.py:118-165) with binary solution and
    tau maps; the history stays CSV and the summary JSON (both O(cycles))."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    files = []

    def emit_text(fname, text):
        _atomic_write_bytes(out_dir / fname, [text.encode()])
        files.append(fname)

    cols = ("iteration", "level", "phase", "sweeps", "rnorm", "work_units", "wall_time")
    lines = [f"# config {digest}", ",".join(cols)]
    for r in history:
        lines.append(f"{r['cycle']},{r['level']},{r['phase']},{r['sweeps']},{r['rnorm']:.6e},"
                     f"{r['work_units']:.6f},{r['wall']:.4f}")
    emit_text("residual_history.csv", "\n".join(lines) + "\n")
    write_solution(out_dir / "solution.tdgsol", Q, digest, case)
    files.append("solution.tdgsol")
    for k, tmap in enumerate(maps, start=1):
        write_tau_map(out_dir / f"tau_map_stage{k}.npz", tmap, digest)
        files.append(f"tau_map_stage{k}.npz")
    for rep in reports:
        emit_text(f"adaptation_stage{rep.stage}.json",
                  json.dumps({"config": digest, **rep.to_dict()}, indent=1, sort_keys=True) + "\n")
    summary = {"config": digest, "name": name, "case": case, "elements": Q.field.num_elements,
               "dofs": int(Q.field.dofs()), "work_units": float(work_units), "iterations": len(history),
               "residual_norm": float(residual_norm), "stages": len(reports),
               "histograms": [r.histogram() for r in reports], "files": files + ["summary.json"]}
    emit_text("summary.json", json.dumps(summary, indent=1, sort_keys=True) + "\n")
    return summary
