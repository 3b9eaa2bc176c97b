"""Truncation-error estimation (oracle).  Restates
/root/reference/pkg/src/taudg/tau.py:52-279 for three directions."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import multigrid


class EstimationError(Exception):
    pass


@dataclass(frozen=True)
class DirectionalFit:
    slope: float
    intercept: float
    residual: float

    def value(self, n):
        return 10.0 ** (self.intercept + self.slope * n)


@dataclass(frozen=True)
class EstimationContext:
    threshold: float
    residual_norm: float
    isolated: bool


class TauMap:
    def __init__(self, fine_orders, context):
        self.fine_orders = fine_orders
        self.context = context
        n = fine_orders.num_elements
        self.tau = [[{}, {}, {}] for _ in range(n)]
        self.extrapolated = [[set(), set(), set()] for _ in range(n)]
        self.fits = [[None, None, None] for _ in range(n)]
        self.non_spectral = [[False, False, False] for _ in range(n)]
        self.n_max = fine_orders.max_order()
        self.work_units = 0.0
        # directions held at their fine order (never estimated / adapted):
        # collapsed order-0 directions plus any the caller freezes
        self.frozen = {d for d in range(3) if int(np.max(fine_orders.orders[:, d])) == 0}

    @property
    def num_elements(self):
        return self.fine_orders.num_elements

    def record(self, e, direction, order, value):
        if value < 0.0:
            raise EstimationError("truncation-error norms cannot be negative")
        self.tau[e][direction - 1][int(order)] = float(value)

    def measured_orders(self, e, direction):
        d = direction - 1
        return sorted(n for n in self.tau[e][d] if n not in self.extrapolated[e][d])

    def combined(self, e, n):
        total = 0.0
        for d in range(3):
            if d in self.frozen:
                continue                      # collapsed / frozen direction: no contribution
            t = self.tau[e][d].get(int(n[d]))
            if t is None:
                return None
            total += t
        return total


def recorder_for(tmap, direction):
    fine_arr = tmap.fine_orders.orders

    def recorder(solver, li, a_val):
        lev = solver.levels[li]
        if tmap.context.isolated:
            a_val = lev.op.m_inv_apply(lev.Q, isolated=True)
            solver._account(li, 1)
        values = lev.op.truncation_from_avalue(a_val)
        lev_arr = lev.orders.orders
        d = direction - 1
        for e in range(len(values)):
            if lev_arr[e, d] < fine_arr[e, d]:
                tmap.record(e, direction, lev_arr[e, d], values[e])

    return recorder


def estimate(msh, law, Q, tau_max, isolated=True, fine_op=None, family="LG", form="cross", frozen=()):
    """tau.py:188-224: convergence gate, then one smoothing-free anisotropic
    high-order descent per direction."""
    from .operators import DGOperator

    orders = Q.field
    op = fine_op or DGOperator(msh, law, orders, family=family, form=form)
    rnorm = op.residual_norm(Q)
    threshold = tau_max / 10.0
    if rnorm > threshold:
        raise EstimationError(f"insufficient convergence for estimation: |r|={rnorm:.3e} "
                              f"exceeds tau_max/10={threshold:.3e}")
    tmap = TauMap(orders, EstimationContext(threshold, rnorm, isolated))
    tmap.frozen |= set(frozen)
    tmap.work_units = 1.0 / 3.0
    for direction in (1, 2, 3):
        if orders.max_order_dir(direction) <= multigrid.N_COARSE or direction - 1 in tmap.frozen:
            continue
        solver = multigrid.FASSolver(msh, law, orders, rule="high-order", direction=direction,
                                     fine_op=op, family=family, form=form)
        solver.set_state(Q)
        solver.estimation_descent(recorder_for(tmap, direction))
        tmap.work_units += solver.work_units
    return tmap


def _lsq_line(x, y):
    coeffs = np.polyfit(x, y, 1)
    fitted = np.polyval(coeffs, x)
    res = float(np.sqrt(np.mean((fitted - y) ** 2)))
    return (float(coeffs[0]), float(coeffs[1])), res


def extrapolate_map(tmap, n_max):
    """tau.py:227-268, per active direction."""
    tmap.n_max = max(tmap.n_max, n_max)
    for e in range(tmap.num_elements):
        for d in range(3):
            p = int(tmap.fine_orders.orders[e, d])
            if p == 0 or d in tmap.frozen:
                continue                      # collapsed direction
            points = [(n, v) for n, v in tmap.tau[e][d].items()
                      if n not in tmap.extrapolated[e][d] and v > 0.0]
            fit = None
            if len(points) >= 2:
                ns = np.array([n for n, _ in points], dtype=float)
                logs = np.log10([v for _, v in points])
                (slope, intercept), res = _lsq_line(ns, logs)
                fit = DirectionalFit(slope, intercept, res)
                tmap.fits[e][d] = fit
            if fit is None or fit.slope >= -1e-12:
                tmap.non_spectral[e][d] = True
                for n in range(p, n_max + 1):
                    tmap.tau[e][d][n] = float("inf")
                    tmap.extrapolated[e][d].add(n)
            else:
                for n in range(p, n_max + 1):
                    tmap.tau[e][d][n] = fit.value(n)
                    tmap.extrapolated[e][d].add(n)
    return tmap
