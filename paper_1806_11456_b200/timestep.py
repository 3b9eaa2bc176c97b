"""Williamson low-storage RK3 smoother on the device.

Mirrors /root/reference/pkg/src/taudg/timestep.py:18-140.  Each RK stage is
ONE fused kernel pass (residual + register update + state update + stage-0
residual norm + non-finite flag, include/taudg.h tdg_rk3_stage) after the
face kernels; dt is computed and consumed on the device (tdg_element_dt), so
a sweep issues no host synchronisation.  ``smooth`` checks the device
non-finite flag and the time scale once at the end of the call and raises the
reference's DivergedError / TimeScaleError, naming the first bad sweep.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DivergedError, TimeScaleError
from .fields import NodalField

RK_A = (0.0, -5.0 / 9.0, -153.0 / 128.0)     # timestep.py:18-20
RK_B = (1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0)


@dataclass(frozen=True)
class TimeConfig:
    """CFL constants and step mode (timestep.py:23-37)."""

    cfl_advective: float = 0.2
    cfl_viscous: float = 0.1
    local: bool = False

    def __post_init__(self):
        if self.cfl_advective <= 0.0 or self.cfl_viscous <= 0.0:
            raise ConfigError("CFL constants must be positive")


class _Scratch:
    """Per-operator device scratch reused across sweeps."""

    def __init__(self, op):
        import torch

        dev = op.device
        self.dt_slot = torch.empty(op.orders.num_elements, dtype=torch.float64, device=dev)
        self.dt_min = torch.empty(1, dtype=torch.float64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.work = NodalField.zeros(op.orders, op.nv, dev)


def _scratch(op):
    s = getattr(op, "_ts_scratch", None)
    if s is None:
        s = _Scratch(op)
        op._ts_scratch = s
    return s


def element_dt(op, Q: NodalField, config: TimeConfig) -> np.ndarray:
    """Per-element step sizes, indexed by element id (timestep.py:40-66)."""
    s = _scratch(op)
    op.element_dt_device(Q, config.cfl_advective, config.cfl_viscous, dt_slot=s.dt_slot)
    out = np.empty(op.orders.num_elements)
    out[op.orders.slot_elem] = s.dt_slot.cpu().numpy()
    return out


def compute_dt(op, Q: NodalField, config: TimeConfig):
    """Global minimum (float) or per-element array (timestep.py:69-80)."""
    dts = element_dt(op, Q, config)
    finite = np.isfinite(dts)
    if not finite.any():
        raise TimeScaleError("no time scale: zero wave speed and zero viscosity everywhere")
    if config.local:
        return np.where(finite, dts, dts[finite].min())
    return float(dts.min())


def _device_dt(op, Q, config, s):
    """dt on the device: the global min into s.dt_min, or per slot into s.dt_slot."""
    op.element_dt_device(Q, config.cfl_advective, config.cfl_viscous, dt_slot=s.dt_slot,
                         dt_min=s.dt_min)
    if config.local:
        # elements without a finite scale borrow the global minimum
        import torch

        torch.where(torch.isfinite(s.dt_slot), s.dt_slot, s.dt_min.expand_as(s.dt_slot), out=s.dt_slot)
        return s.dt_slot
    return s.dt_min


def rk3_step(op, Q: NodalField, dt, source: NodalField | None = None,
             work: NodalField | None = None, rnorm=None, nonfinite=None, fresh=False):
    """One RK3 step; ``dt`` is a float, a per-element numpy array (by element
    id) or a device tensor (scalar or per slot).  Returns the stage-0 residual
    inf-norm as a float when ``rnorm`` is None (reference semantics), else
    leaves it in the device scalar ``rnorm``.  ``fresh``: Q is unchanged since
    the previous RK stage on ``op`` (later stages always are)."""
    import torch

    s = _scratch(op)
    work = work if work is not None else s.work
    src = op.source if source is None else source
    if isinstance(dt, torch.Tensor):
        dt_dev = dt
        local = dt.numel() > 1
    elif np.isscalar(dt):
        dt_dev = torch.full((1,), float(dt), dtype=torch.float64, device=op.device)
        local = False
    else:
        dt_dev = torch.as_tensor(np.asarray(dt)[op.orders.slot_elem], device=op.device)
        local = True
    sync = rnorm is None
    if sync:
        rnorm = torch.zeros(1, dtype=torch.float64, device=op.device)
    for stage in range(3):
        op.calls["apply"] += 1
        op.rk3_stage(Q, work, src, stage, dt_dev, local, rnorm=rnorm, nonfinite=nonfinite,
                     fresh=fresh or stage > 0)
    return float(rnorm.item()) if sync else rnorm


def smooth(op, Q: NodalField, sweeps: int, config: TimeConfig, source: NodalField | None = None,
           history: list | None = None):
    """``sweeps`` RK3 steps with a fresh dt each sweep (timestep.py:116-140).

    The stage-0 norms stay on the device until the end of the call; the
    returned history matches the reference's list of first-stage norms.
    """
    import torch

    out = [] if history is None else history
    sweeps = int(sweeps)
    if sweeps <= 0:
        return out
    s = _scratch(op)
    norms = torch.zeros(sweeps, dtype=torch.float64, device=op.device)
    dts = torch.empty(sweeps, dtype=torch.float64, device=op.device)
    flags = torch.zeros(sweeps, dtype=torch.int32, device=op.device)
    for k in range(sweeps):
        dt = _device_dt(op, Q, config, s)
        dts[k: k + 1].copy_(s.dt_min)
        rk3_step(op, Q, dt, source=source, work=s.work, rnorm=norms[k: k + 1], nonfinite=flags[k: k + 1],
                 fresh=k > 0)
    h_norms = norms.cpu().numpy()
    h_dts = dts.cpu().numpy()
    h_flags = flags.cpu().numpy()
    for k in range(sweeps):
        if not np.isfinite(h_dts[k]) and h_dts[k] > 0:
            raise TimeScaleError("no time scale: zero wave speed and zero viscosity everywhere")
        out.append(float(h_norms[k]))
        if h_flags[k]:
            bad = first_bad_element(op, Q)
            raise DivergedError(f"non-finite state in element {bad} after sweep {len(out)}")
    return out


def first_bad_element(op, Q: NodalField):
    import torch

    norms = op.element_norms(Q)
    bad = ~torch.isfinite(norms)
    if not bool(bad.any()):
        return None
    return int(torch.nonzero(bad)[0].item())
