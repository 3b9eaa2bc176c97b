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


def map_points_ordered(ctrl, xi, eta, zeta):
    """map_points with a fixed summation order: x = sum over control nodes
    (a, b, c ascending) of ((l_a l_b) l_c) X_abc, each product and sum
    separately rounded — the arithmetic of the device metrics kernel
    (csrc/geometry.cuh), so the curl-form setup is bit-identical on both."""
    m = [s - 1 for s in ctrl.shape[:3]]
    l = [spectral.lagrange_values(_ctrl_grid(m[d]), p) for d, p in enumerate((xi, eta, zeta))]
    out = np.zeros((len(l[0]), len(l[1]), len(l[2]), 3))
    for a in range(m[0] + 1):
        for b in range(m[1] + 1):
            lab = l[0][:, a][:, None] * l[1][:, b][None, :]
            for c in range(m[2] + 1):
                lw = lab[:, :, None] * l[2][:, c][None, None, :]
                out += lw[..., None] * ctrl[a, b, c][None, None, None, :]
    return out


def _d_ordered(arr, axis, D):
    """Collocation derivative with the kernel's summation order (m ascending)."""
    a = np.moveaxis(arr, axis, -1)
    out = np.zeros_like(a)
    for m in range(a.shape[-1]):
        out += D[:, m] * a[..., m:m + 1]
    return np.moveaxis(out, -1, axis)


def _d(arr, axis, D):
    """Collocation derivative of a nodal (n1,n2,n3) array along ``axis``."""
    return np.moveaxis(np.einsum("im,...m->...i", D, np.moveaxis(arr, axis, -1)), -1, axis)


def affine_map(ctrl):
    """Affine elements of the invariant-curl form: ctrl (B, a1, a2, a3, 3)
    control nodes on the equispaced reference grid -> (mask (B,), A (B, 3, 3))
    with A[:, d] = dX/dxi_d, the element being affine (a parallelepiped map)
    when every control node lies within 1e-13 (relative to the edge vectors)
    of c + sum_d A_d xi_d.  Their curl-form metrics are replaced by the exact
    constants J = A_0 . (A_1 x A_2), Ja^i = A_j x A_k (collocated curl-form
    round-off is ~1e-12 at N = 7, enough to move an M = 0.1 residual by
    ~3e-11 relative); free-stream preservation is unaffected (constant
    metrics satisfy the metric identities exactly).  Same arithmetic in the
    product (paper_1806_11456_b200/geometry.py) and the oracle, element-wise
    only, so both produce identical bits."""
    x0 = ctrl[:, 0, 0, 0]
    A = np.stack([0.5 * (ctrl[:, -1, 0, 0] - x0), 0.5 * (ctrl[:, 0, -1, 0] - x0),
                  0.5 * (ctrl[:, 0, 0, -1] - x0)], axis=1)                 # (B, 3[d], 3[x])
    c = x0 + A[:, 0] + A[:, 1] + A[:, 2]
    xi = [np.linspace(-1.0, 1.0, s) for s in ctrl.shape[1:4]]
    pred = (c[:, None, None, None, :]
            + A[:, 0][:, None, None, None, :] * xi[0][None, :, None, None, None]
            + A[:, 1][:, None, None, None, :] * xi[1][None, None, :, None, None]
            + A[:, 2][:, None, None, None, :] * xi[2][None, None, None, :, None])
    scale = np.abs(A).max(axis=(1, 2))
    mask = (np.abs(pred - ctrl).max(axis=(1, 2, 3, 4)) <= 1e-13 * scale) & (scale > 0.0)
    return mask, A


def _cross3(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def affine_constants(A):
    """Exact metrics of affine maps A (B, 3[d], 3[x]): J (B,), Ja (B, 3[i], 3[n])."""
    ja = np.stack([_cross3(A[:, 1], A[:, 2]), _cross3(A[:, 2], A[:, 0]), _cross3(A[:, 0], A[:, 1])], axis=1)
    jac = A[:, 0, 0] * ja[:, 0, 0] + A[:, 0, 1] * ja[:, 0, 1] + A[:, 0, 2] * ja[:, 0, 2]
    return jac, ja


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
        # fixed summation orders, separately rounded products and sums, node 0
        # as the local origin: bit-identical to the device kernel
        X = map_points_ordered(ctrl, q[0][0], q[1][0], q[2][0])  # (n1,n2,n3,3)
        X = X - X[0, 0, 0]                                         # element-local origin
        D = [spectral.differentiation_matrix(int(n), family) for n in orders]
        gX = [[_d_ordered(X[..., c], k, D[k]) for k in range(3)] for c in range(3)]  # gX[c][k]
        ja = np.empty((3, 3) + X.shape[:3])
        for n in range(3):
            mm, ll = (n + 1) % 3, (n + 2) % 3
            # V_k = X_l d_k X_m - X_m d_k X_l
            V = [X[..., ll] * gX[mm][k] - X[..., mm] * gX[ll][k] for k in range(3)]
            for i in range(3):
                j, k = (i + 1) % 3, (i + 2) % 3
                curl_i = _d_ordered(V[k], j, D[j]) - _d_ordered(V[j], k, D[k])
                ja[i, n] = -0.5 * curl_i
        av = tuple(np.stack([gX[c][k] for c in range(3)], axis=-1) for k in range(3))
        c1 = av[1][..., 1] * av[2][..., 2] - av[1][..., 2] * av[2][..., 1]
        c2 = av[1][..., 2] * av[2][..., 0] - av[1][..., 0] * av[2][..., 2]
        c3 = av[1][..., 0] * av[2][..., 1] - av[1][..., 1] * av[2][..., 0]
        jac = av[0][..., 0] * c1 + av[0][..., 1] * c2 + av[0][..., 2] * c3
        aff, A = affine_map(ctrl[None])
        if aff[0]:
            jc, jac_c = affine_constants(A)
            ja = np.broadcast_to(jac_c[0][:, :, None, None, None], ja.shape).copy()
            jac = np.full(jac.shape, jc[0])
            av = tuple(np.broadcast_to(A[0, d], av[d].shape).copy() for d in range(3))
        if np.min(jac) <= 0.0:
            raise MeshError(f"inverted element {index}: min Jacobian {np.min(jac):.3e}")
        www = (q[0][1][:, None, None] * q[1][1][None, :, None] * q[2][1][None, None, :]).ravel()
        sizes = np.zeros(3)
        for d in range(3):
            nrm = np.sqrt(av[d][..., 0] * av[d][..., 0] + av[d][..., 1] * av[d][..., 1]
                          + av[d][..., 2] * av[d][..., 2]).ravel()
            acc = 0.0
            for t in range(len(www)):            # node order, as the kernel's sum
                acc += www[t] * nrm[t]
            sizes[d] = acc / 4.0
        return jac, ja, sizes
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
