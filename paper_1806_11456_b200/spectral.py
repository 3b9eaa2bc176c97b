"""1D spectral tables for the device operator (host setup, cached).

Legendre-Gauss nodes follow /root/reference/pkg/src/taudg/spectral.py:45-65;
Gauss-Lobatto nodes are added for the north_star's LGL path.  Lowering
transfers are the exact modal L2 projection (the reference's closed form,
spectral.py:143-164, is exact on LG nodes only — SURVEY §0.7(i)).

``device_tables(family)`` packs everything the kernels read into one float64
array with a fixed 8-point padding (orders 0..7):

    [DHAT]  8 orders x 8 x 8    Dhat[m][i] = w_m D_mi            (operators.py:127)
    [W]     8 orders x 8        quadrature weights
    [BND]   8 orders x 2 x 8    l_i(-1), l_i(+1)                 (spectral.py:133-140)
    [T]     8 x 8 (from, to) x 8 x 8   transfer T[to_row][from_col]
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
import numpy.polynomial.legendre as npleg

MAX_ORDER = 7
PAD = 8
OFF_DHAT = 0
OFF_W = OFF_DHAT + PAD * PAD * PAD
OFF_BND = OFF_W + PAD * PAD
OFF_T = OFF_BND + PAD * 2 * PAD
TABLES_LEN = OFF_T + PAD * PAD * PAD * PAD

FAMILIES = {"LG": 0, "LGL": 1}


def _pn(n, x):
    p0, p1 = np.ones_like(x), x.copy()
    if n == 0:
        return p0, np.zeros_like(x)
    for k in range(2, n + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    return p1, p0


@lru_cache(maxsize=None)
def rule(order: int, family: str = "LGL"):
    """(nodes, weights) of the order-``order`` rule (order+1 points)."""
    if order < 0:
        raise ValueError("polynomial order must be >= 0")
    n = order + 1
    if family == "LG":
        if n == 1:
            return np.zeros(1), np.full(1, 2.0)
        x = -np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
        for _ in range(200):
            p, pm = _pn(n, x)
            dp = n * (x * p - pm) / (x * x - 1.0)
            dx = p / dp
            x = x - dx
            if np.max(np.abs(dx)) < 1e-15:
                break
        p, pm = _pn(n, x)
        dp = n * (x * p - pm) / (x * x - 1.0)
        w = 2.0 / ((1.0 - x * x) * dp * dp)
    elif family == "LGL":
        if order < 1:
            raise ValueError("Gauss-Lobatto rules need order >= 1")
        N = order
        x = -np.cos(np.pi * np.arange(N + 1) / N)
        if N > 1:
            xi = x[1:-1].copy()
            for _ in range(200):
                p, pm = _pn(N, xi)
                dp = N * (xi * p - pm) / (xi * xi - 1.0)
                d2 = (2.0 * xi * dp - N * (N + 1) * p) / (1.0 - xi * xi)
                dx = dp / d2
                xi = xi - dx
                if np.max(np.abs(dx)) < 1e-15:
                    break
            x[1:-1] = xi
        x[0], x[-1] = -1.0, 1.0
        pN, _ = _pn(N, x)
        w = 2.0 / (N * (N + 1) * pN * pN)
    else:
        raise ValueError(f"unknown node family {family!r}")
    x = 0.5 * (x - x[::-1])
    w = 0.5 * (w + w[::-1])
    return x, w


def lagrange_matrix(nodes, pts):
    """l_j(pts_i), barycentric form with exact node hits."""
    nodes = np.asarray(nodes, float)
    pts = np.atleast_1d(np.asarray(pts, float))
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    bary = 1.0 / diff.prod(axis=1)
    d = pts[:, None] - nodes[None, :]
    hit = np.abs(d) < 1e-14
    d = np.where(hit, 1.0, d)
    t = bary[None, :] / d
    out = t / t.sum(axis=1, keepdims=True)
    rows = hit.any(axis=1)
    out[rows] = hit[rows].astype(float)
    return out


def derivative_matrix(nodes):
    nodes = np.asarray(nodes, float)
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    bary = 1.0 / diff.prod(axis=1)
    D = (bary[None, :] / bary[:, None]) / diff
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, -D.sum(axis=1))
    return D


@lru_cache(maxsize=None)
def dmat(order, family="LGL"):
    return derivative_matrix(rule(order, family)[0])


@lru_cache(maxsize=None)
def bounds(order, family="LGL"):
    return lagrange_matrix(rule(order, family)[0], [-1.0, 1.0])


@lru_cache(maxsize=None)
def transfer(order_from, order_to, family="LGL"):
    xf, wf = rule(order_from, family)
    xt, _ = rule(order_to, family)
    if order_to >= order_from:
        return lagrange_matrix(xf, xt)
    k = np.arange(order_from + 1)
    analysis = (k[:, None] + 0.5) * wf[None, :] * npleg.legvander(xf, order_from).T
    return npleg.legvander(xt, order_to)[:, : order_to + 1] @ analysis[: order_to + 1]


@lru_cache(maxsize=None)
def device_tables(family: str) -> np.ndarray:
    t = np.zeros(TABLES_LEN)
    lo = 0 if family == "LG" else 1
    for n in range(lo, MAX_ORDER + 1):
        x, w = rule(n, family)
        dh = w[:, None] * dmat(n, family)
        blk = np.zeros((PAD, PAD))
        blk[: n + 1, : n + 1] = dh
        t[OFF_DHAT + n * 64: OFF_DHAT + (n + 1) * 64] = blk.ravel()
        t[OFF_W + n * PAD: OFF_W + n * PAD + n + 1] = w
        b = np.zeros((2, PAD))
        b[:, : n + 1] = bounds(n, family)
        t[OFF_BND + n * 16: OFF_BND + (n + 1) * 16] = b.ravel()
    for f in range(lo, MAX_ORDER + 1):
        for to in range(lo, MAX_ORDER + 1):
            blk = np.zeros((PAD, PAD))
            blk[: to + 1, : f + 1] = transfer(f, to, family)
            o = OFF_T + (f * PAD + to) * 64
            t[o: o + 64] = blk.ravel()
    t.setflags(write=False)
    return t
