"""1D collocation kernels (oracle).  Follows
/root/reference/pkg/src/taudg/spectral.py:1-164 for Legendre-Gauss nodes and
adds the Gauss-Lobatto rule and modal (Vandermonde-truncation) L2 transfers.

Node families: "LG" (Legendre-Gauss, orders >= 0) and "LGL" (Gauss-Lobatto,
orders >= 1).  Lowering transfers use the exact modal L2 projection for both
families (the reference's closed form spectral.py:143-164 is
exact only on LG nodes, where it agrees with the modal form to ~2e-15; the
modal analysis matches the reference test oracle tests/test_spectral.py:98-108).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
import numpy.polynomial.legendre as npleg

NEWTON_TOL = 1e-15
NEWTON_MAXIT = 200


def legendre_and_derivative(n: int, x):
    """P_n, P_n' by the three-term recurrence (reference spectral.py:29-42)."""
    x = np.asarray(x, dtype=float)
    p_prev = np.ones_like(x)
    if n == 0:
        return p_prev, np.zeros_like(x)
    p = x.copy()
    for k in range(2, n + 1):
        p_prev, p = p, ((2 * k - 1) * x * p - (k - 1) * p_prev) / k
    dp = n * (x * p - p_prev) / (x * x - 1.0)
    return p, dp


def _gauss(order: int):
    # reference spectral.py:45-65
    n = order + 1
    if n == 1:
        return np.zeros(1), np.full(1, 2.0)
    k = np.arange(n)
    x = -np.cos(np.pi * (k + 0.75) / (n + 0.5))
    for _ in range(NEWTON_MAXIT):
        p, dp = legendre_and_derivative(n, x)
        dx = p / dp
        x -= dx
        if np.max(np.abs(dx)) < NEWTON_TOL:
            break
    _, dp = legendre_and_derivative(n, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    x = 0.5 * (x - x[::-1])
    w = 0.5 * (w + w[::-1])
    return x, w


def _legendre_p(n, x):
    x = np.asarray(x, dtype=float)
    p_prev, p = np.ones_like(x), x.copy()
    if n == 0:
        return p_prev
    for k in range(2, n + 1):
        p_prev, p = p, ((2 * k - 1) * x * p - (k - 1) * p_prev) / k
    return p


def _lobatto(order: int):
    """Gauss-Lobatto: endpoints plus the roots of P_N'; w = 2/(N(N+1) P_N^2)."""
    if order < 1:
        raise ValueError("Gauss-Lobatto rules need order >= 1")
    N = order
    if N == 1:
        x = np.array([-1.0, 1.0])
    else:
        # Chebyshev-Gauss-Lobatto guesses, Newton on q = P_{N+1} - P_{N-1}
        # (proportional to (1-x^2) P_N').
        x = -np.cos(np.pi * np.arange(N + 1) / N)
        for _ in range(NEWTON_MAXIT):
            xi = x[1:-1]
            # (1-x^2) P_N'' - 2 x P_N' ... use q(x) = (1-x^2) P_N'(x)
            pN, dpN = legendre_and_derivative(N, xi)
            # P_N'' from the Legendre ODE: (1-x^2)P'' = 2xP' - N(N+1)P
            d2 = (2 * xi * dpN - N * (N + 1) * pN) / (1 - xi * xi)
            dx = dpN / d2
            x[1:-1] = xi - dx
            if np.max(np.abs(dx)) < NEWTON_TOL:
                break
        x[0], x[-1] = -1.0, 1.0
    w = 2.0 / (N * (N + 1) * _legendre_p(N, x) ** 2)
    x = 0.5 * (x - x[::-1])
    w = 0.5 * (w + w[::-1])
    return x, w


@lru_cache(maxsize=None)
def rule(order: int, family: str = "LG"):
    if order < 0:
        raise ValueError(f"polynomial order must be >= 0, got {order}")
    if family == "LG":
        return _gauss(order)
    if family == "LGL":
        return _lobatto(order)
    raise ValueError(f"unknown node family {family!r}")


def barycentric_weights(nodes):
    nodes = np.asarray(nodes, dtype=float)
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    return 1.0 / diff.prod(axis=1)


def lagrange_values(nodes, x):
    """l_j(x_i), shape (len(x), len(nodes)) (reference spectral.py:75-88)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    bary = barycentric_weights(nodes)
    diff = x[:, None] - nodes[None, :]
    hit = np.isclose(diff, 0.0, rtol=0.0, atol=1e-14)
    diff = np.where(hit, 1.0, diff)
    terms = bary[None, :] / diff
    vals = terms / terms.sum(axis=1, keepdims=True)
    rows_hit = hit.any(axis=1)
    if rows_hit.any():
        vals[rows_hit] = hit[rows_hit].astype(float)
    return vals


def diff_matrix(nodes):
    """D_ij = l_j'(x_i), negative-sum diagonal (reference spectral.py:91-100)."""
    nodes = np.asarray(nodes, dtype=float)
    bary = barycentric_weights(nodes)
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    d = (bary[None, :] / bary[:, None]) / diff
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, -d.sum(axis=1))
    return d


def lagrange_derivative_values(nodes, x):
    return lagrange_values(nodes, x) @ diff_matrix(nodes)


@lru_cache(maxsize=None)
def differentiation_matrix(order: int, family: str = "LG"):
    return diff_matrix(rule(order, family)[0])


@lru_cache(maxsize=None)
def boundary_rows(order: int, family: str = "LG"):
    """(2, order+1): cardinal values at xi=-1 (row 0), +1 (row 1)."""
    return lagrange_values(rule(order, family)[0], np.array([-1.0, 1.0]))


@lru_cache(maxsize=None)
def transfer(order_from: int, order_to: int, family: str = "LG"):
    """(to+1, from+1) nodal transfer.  Raising: interpolation (reference
    spectral.py:157-158).  Lowering: modal L2 projection."""
    xf, wf = rule(order_from, family)
    xt, _ = rule(order_to, family)
    if order_to >= order_from:
        return lagrange_values(xf, xt)
    k = np.arange(order_from + 1)
    analysis = (k[:, None] + 0.5) * wf[None, :] * npleg.legvander(xf, order_from).T
    keep = order_to + 1
    return npleg.legvander(xt, order_to)[:, :keep] @ analysis[:keep]
