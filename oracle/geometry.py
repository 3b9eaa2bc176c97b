"""Element metrics and face geometry (oracle).

3D restatement of /root/reference/pkg/src/taudg/mesh.py:103-192
(map_points, map_derivatives, volume_metrics, face_geometry).  Two metric
forms:

* "cross": Ja^i = a_j x a_k evaluated pointwise from the analytic mapping
  derivatives — the 3D analogue of the reference's 2D cross-product form
  (mesh.py:155-160); face sigma/normal are evaluated the same way at the face
  (or mortar) points, as mesh.py:167-187 does.
* "curl": Kopriva's invariant curl form,
  Ja^i_n = -1/2 x_i . curl_xi[ I^N(X_l grad X_m - X_m grad X_l) ], computed
  by collocation at the solution nodes; face values are the trace of that
  volume polynomial and mortar values its interpolation to the mortar nodes.

Sizes h_d are the weighted mean covariant lengths (mesh.py:161-163),
normalised so a cube of side L gives h = L.
"""

from __future__ import annotations

import numpy as np

from . import spectral


class MeshError(Exception):
    pass


def _ctrl_grid(m):
    return np.linspace(-1.0, 1.0, m + 1)


def map_points(ctrl, xi, eta, zeta):
    m = [s - 1 for s in ctrl.shape[:3]]
    l = [spectral.lagrange_values(_ctrl_grid(m[d]), p) for d, p in enumerate((xi, eta, zeta))]
    return np.einsum("ia,jb,kc,abcx->ijkx", l[0], l[1], l[2], ctrl)


def map_derivatives(ctrl, xi, eta, zeta):
    m = [s - 1 for s in ctrl.shape[:3]]
    pts = (xi, eta, zeta)
    l = [spectral.lagrange_values(_ctrl_grid(m[d]), pts[d]) for d in range(3)]
    dl = [spectral.lagrange_derivative_values(_ctrl_grid(m[d]), pts[d]) for d in range(3)]
    a1 = np.einsum("ia,jb,kc,abcx->ijkx", dl[0], l[1], l[2], ctrl)
    a2 = np.einsum("ia,jb,kc,abcx->ijkx", l[0], dl[1], l[2], ctrl)
    a3 = np.einsum("ia,jb,kc,abcx->ijkx", l[0], l[1], dl[2], ctrl)
    return a1, a2, a3


def _cross_ja(a1, a2, a3):
    return np.stack([np.cross(a2, a3), np.cross(a3, a1), np.cross(a1, a2)], axis=0)


def _d(arr, axis, D):
    """Collocation derivative of a nodal (n1,n2,n3) array along ``axis``."""
    return np.moveaxis(np.einsum("im,...m->...i", D, np.moveaxis(arr, axis, -1)), -1, axis)


def volume_metrics(ctrl, orders, family="LG", form="cross", index=-1):
    """Returns (jac (n1,n2,n3), ja (3, 3, n1,n2,n3) with ja[i, n] = Ja^i_n,
    sizes (3,))."""
    m = [s - 1 for s in ctrl.shape[:3]]
    # the cross-product form needs a sub/isoparametric map (reference
    # mesh.py:147-152); the curl form works with I^N of the map by design
    for d in range(3):
        if form == "cross" and orders[d] >= 1 and m[d] > orders[d]:
            raise MeshError(
                f"element {index}: mapping order {tuple(m)} exceeds solution order {tuple(orders)}"
            )
    q = [spectral.rule(int(n), family) for n in orders]
    a1, a2, a3 = map_derivatives(ctrl, q[0][0], q[1][0], q[2][0])
    if form == "cross":
        ja = np.moveaxis(_cross_ja(a1, a2, a3), -1, 1)          # (3, 3, ...)
        jac = np.einsum("ijkx,ijkx->ijk", a1, np.cross(a2, a3))
        av = (a1, a2, a3)
    elif form == "curl":
        X = map_points(ctrl, q[0][0], q[1][0], q[2][0])          # (n1,n2,n3,3)
        X = X - X.reshape(-1, 3).mean(axis=0)                      # element-local origin
        D = [spectral.differentiation_matrix(int(n), family) for n in orders]
        gX = [[_d(X[..., c], k, D[k]) for k in range(3)] for c in range(3)]  # gX[c][k]
        ja = np.empty((3, 3) + X.shape[:3])
        for n in range(3):
            mm, ll = (n + 1) % 3, (n + 2) % 3
            # V_k = X_l d_k X_m - X_m d_k X_l
            V = [X[..., ll] * gX[mm][k] - X[..., mm] * gX[ll][k] for k in range(3)]
            for i in range(3):
                j, k = (i + 1) % 3, (i + 2) % 3
                curl_i = _d(V[k], j, D[j]) - _d(V[j], k, D[k])
                ja[i, n] = -0.5 * curl_i
        av = tuple(np.stack([gX[c][k] for c in range(3)], axis=-1) for k in range(3))
        jac = np.einsum("ijkx,ijkx->ijk", av[0], np.cross(av[1], av[2]))
    else:
        raise ValueError(f"unknown metric form {form!r}")
    if np.min(jac) <= 0.0:
        raise MeshError(f"inverted element {index}: min Jacobian {np.min(jac):.3e}")
    www = q[0][1][:, None, None] * q[1][1][None, :, None] * q[2][1][None, None, :]
    sizes = np.array([float(np.sum(www * np.linalg.norm(av[d], axis=-1)) / 4.0) for d in range(3)])
    return jac, ja, sizes


def _face_axes(side):
    d = side // 2
    t = [x for x in range(3) if x != d]
    return d, t[0], t[1]


def _pts_for_side(side, t1pts, t2pts):
    d, a, b = _face_axes(side)
    pts = [None, None, None]
    pts[d] = np.array([-1.0 if side % 2 == 0 else 1.0])
    pts[a] = np.asarray(t1pts, dtype=float)
    pts[b] = np.asarray(t2pts, dtype=float)
    return pts


def _squeeze_face(arr, side):
    d = side // 2
    return np.take(arr, 0, axis=d)


def face_ja_analytic(ctrl, side, t1pts, t2pts):
    """Ja^d (normal-direction contravariant vector) at face points, (n1, n2, 3)."""
    pts = _pts_for_side(side, t1pts, t2pts)
    a = map_derivatives(ctrl, *pts)
    ja = _cross_ja(*a)[side // 2]
    return _squeeze_face(ja, side)


def face_ja_from_volume(ja_vol, side, orders, family):
    """Trace of the volume Ja^d polynomial on a side at own face nodes, (n1,n2,3)."""
    d = side // 2
    row = spectral.boundary_rows(int(orders[d]), family)[side % 2]
    vec = ja_vol[d]                                   # (3, n1, n2, n3)
    tr = np.tensordot(vec, row, axes=([1 + d], [0]))  # (3, nt1, nt2)
    return np.moveaxis(tr, 0, -1)


def sigma_normal(ja_face, side):
    sign = 1.0 if side % 2 == 1 else -1.0
    sigma = np.linalg.norm(ja_face, axis=-1)
    normal = sign * ja_face / sigma[..., None]
    return sigma, normal


def face_points(ctrl, side, t1pts, t2pts):
    pts = _pts_for_side(side, t1pts, t2pts)
    return _squeeze_face(map_points(ctrl, *pts), side)
