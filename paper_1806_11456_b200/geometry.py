"""Element metrics and face geometry, vectorised over a bucket (host setup).

3D counterpart of /root/reference/pkg/src/taudg/mesh.py:103-192.  Two metric
forms:

* "cross": Ja^i = a_j x a_k from the analytic mapping derivatives, pointwise
  (the reference's cross-product form, mesh.py:155-160); face and mortar
  sigma/normal are evaluated analytically at their points (mesh.py:167-187).
* "curl":  the invariant curl form by collocation at the
  solution nodes; face values are the trace of that volume polynomial, mortar
  values its interpolation (free-stream preserving on conforming 3D meshes).

All arrays carry a leading bucket axis B.
"""

from __future__ import annotations

import numpy as np

from . import spectral
from .errors import MeshError


def _ctrl(m):
    return np.linspace(-1.0, 1.0, m + 1)


def _lag(m, pts):
    return spectral.lagrange_matrix(_ctrl(m), pts)


def _dlag(m, pts):
    return spectral.lagrange_matrix(_ctrl(m), pts) @ spectral.derivative_matrix(_ctrl(m))


def map_points(nodes, xs, ys, zs):
    """nodes (B, a1, a2, a3, 3) -> (B, len xs, len ys, len zs, 3)."""
    m = [s - 1 for s in nodes.shape[1:4]]
    return np.einsum("ia,jb,kc,Eabcx->Eijkx", _lag(m[0], xs), _lag(m[1], ys), _lag(m[2], zs), nodes)


def map_derivs(nodes, xs, ys, zs):
    m = [s - 1 for s in nodes.shape[1:4]]
    L = [_lag(m[0], xs), _lag(m[1], ys), _lag(m[2], zs)]
    dL = [_dlag(m[0], xs), _dlag(m[1], ys), _dlag(m[2], zs)]
    out = []
    for d in range(3):
        M = [dL[k] if k == d else L[k] for k in range(3)]
        out.append(np.einsum("ia,jb,kc,Eabcx->Eijkx", M[0], M[1], M[2], nodes))
    return out


def map_points_ordered(nodes, xs, ys, zs):
    """map_points with the device kernel's fixed summation order (control nodes
    a, b, c ascending, ((l_a l_b) l_c) X_abc, separately rounded): the
    curl-form setup is bit-identical on host, device and oracle."""
    m = [s - 1 for s in nodes.shape[1:4]]
    L = [_lag(m[0], xs), _lag(m[1], ys), _lag(m[2], zs)]
    out = np.zeros((nodes.shape[0], len(L[0]), len(L[1]), len(L[2]), 3))
    for a in range(m[0] + 1):
        for b in range(m[1] + 1):
            lab = L[0][:, a][:, None] * L[1][:, b][None, :]
            for c in range(m[2] + 1):
                lw = lab[:, :, None] * L[2][:, c][None, None, :]
                out += lw[None, ..., None] * nodes[:, a, b, c][:, None, None, None, :]
    return out


def _coll_ordered(arr, axis, D):
    """Collocation derivative along ``axis`` (1..3) with the kernel's order."""
    a = np.moveaxis(arr, axis, -1)
    out = np.zeros_like(a)
    for m in range(a.shape[-1]):
        out += D[:, m] * a[..., m:m + 1]
    return np.moveaxis(out, -1, axis)


def _coll(arr, axis, D):
    """Collocation derivative along spatial ``axis`` (1..3) of (B, n1, n2, n3)."""
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


def _device_curl_metrics(nodes, orders, family):
    """The curl-form J, Ja, sizes and coordinates from the sm_100a kernel
    (tdg_volume_metrics; same arithmetic as the host branch below up to
    summation order)."""
    import ctypes as C

    from . import _lib

    B = nodes.shape[0]
    a = [int(s) for s in nodes.shape[1:4]]
    npts = [int(o) + 1 for o in orders]
    tab = np.zeros(3 * 8 * 4 + 3 * 64 + 3 * 8)
    L = tab[:96].reshape(3, 8, 4)
    Dt = tab[96:288].reshape(3, 8, 8)
    W = tab[288:].reshape(3, 8)
    for d in range(3):
        x, w = spectral.rule(int(orders[d]), family)
        L[d, :npts[d], :a[d]] = _lag(a[d] - 1, x)
        Dt[d, :npts[d], :npts[d]] = spectral.derivative_matrix(x)
        W[d, :npts[d]] = w
    ctrl = np.ascontiguousarray(nodes, dtype=np.float64)
    n1, n2, n3 = npts
    jac = np.empty((B, n1, n2, n3))
    ja = np.empty((B, 3, 3, n1, n2, n3))
    coords = np.empty((B, n1, n2, n3, 3))
    sizes = np.empty((B, 3))
    p = lambda arr, t: arr.ctypes.data_as(C.POINTER(t))
    sh = np.array(a, np.int32)
    nn = np.array(npts, np.int32)
    _lib.call("tdg_volume_metrics", B, p(sh, C.c_int32), p(ctrl, C.c_double), p(nn, C.c_int32),
              p(tab, C.c_double), p(jac, C.c_double), p(ja, C.c_double), p(coords, C.c_double),
              p(sizes, C.c_double))
    return jac, ja, sizes, coords


def _jac_ordered(av):
    """J = a_1 . (a_2 x a_3), separately rounded in a fixed order."""
    c1 = av[1][..., 1] * av[2][..., 2] - av[1][..., 2] * av[2][..., 1]
    c2 = av[1][..., 2] * av[2][..., 0] - av[1][..., 0] * av[2][..., 2]
    c3 = av[1][..., 0] * av[2][..., 1] - av[1][..., 1] * av[2][..., 0]
    return av[0][..., 0] * c1 + av[0][..., 1] * c2 + av[0][..., 2] * c3


def _sizes_ordered(av, w):
    """h_d = sum_t w_t |a_d(t)| / 4, summed in node order (the kernel's loop)."""
    www = (w[0][:, None, None] * w[1][None, :, None] * w[2][None, None, :]).ravel()
    B = av[0].shape[0]
    out = np.zeros((B, 3))
    for d in range(3):
        a = av[d]
        nrm = np.sqrt(a[..., 0] * a[..., 0] + a[..., 1] * a[..., 1] + a[..., 2] * a[..., 2]).reshape(B, -1)
        acc = np.zeros(B)
        for t in range(len(www)):
            acc += www[t] * nrm[:, t]
        out[:, d] = acc / 4.0
    return out


def _check_jac(jac, ids):
    if jac.size and np.min(jac) <= 0.0:
        bad = int(np.argmin(jac.reshape(len(jac), -1).min(axis=1)))
        e = bad if ids is None else int(ids[bad])
        raise MeshError(f"inverted element {e}: min Jacobian {np.min(jac):.3e}")


def volume_metrics(nodes, orders, family, form, ids=None, device=None):
    """Returns J (B,n1,n2,n3), Ja (B,3,3,n1,n2,n3) [i, phys], sizes (B,3), coords.

    ``device="cuda"`` builds the curl form on the GPU (tdg_volume_metrics);
    the affine override and the Jacobian check stay here."""
    m = [s - 1 for s in nodes.shape[1:4]]
    # cross form: sub/isoparametric only (reference mesh.py:147-152); the
    # invariant curl form uses the interpolant I^N of the map
    for d in range(3):
        if form == "cross" and orders[d] >= 1 and m[d] > orders[d]:
            raise MeshError(f"mapping order {tuple(m)} exceeds solution order {tuple(orders)}")
    x = [spectral.rule(int(n), family)[0] for n in orders]
    w = [spectral.rule(int(n), family)[1] for n in orders]
    if form == "cross":
        coords = map_points(nodes, *x)
        a = map_derivs(nodes, *x)
        ja = np.stack([np.cross(a[1], a[2]), np.cross(a[2], a[0]), np.cross(a[0], a[1])], axis=1)
        ja = np.moveaxis(ja, -1, 2)                       # (B, 3[i], 3[n], ...)
        jac = np.einsum("Eijkx,Eijkx->Eijk", a[0], np.cross(a[1], a[2]))
        av = a
    elif form == "curl" and device == "cuda" and max(m) <= 3:
        jac, ja, sizes, coords = _device_curl_metrics(nodes, orders, family)
        aff, A = affine_map(nodes)
        if aff.any():
            jc, jac_c = affine_constants(A[aff])
            ja[aff] = jac_c[:, :, :, None, None, None]
            jac[aff] = jc[:, None, None, None]
            shape = (int(aff.sum()),) + jac.shape[1:] + (3,)
            sizes[aff] = _sizes_ordered([np.broadcast_to(A[aff][:, d][:, None, None, None, :], shape)
                                         for d in range(3)], w)
        _check_jac(jac, ids)
        return jac, ja, sizes, coords
    elif form == "curl":
        # same fixed-order arithmetic as the device kernel (tdg_volume_metrics)
        # and the oracle: bit-identical metrics on all three
        D = [spectral.derivative_matrix(xx) for xx in x]
        coords = map_points_ordered(nodes, *x)
        X = coords - coords[:, :1, :1, :1, :]                 # element-local origin: node 0
        g = [[_coll_ordered(X[..., c], k + 1, D[k]) for k in range(3)] for c in range(3)]
        ja = np.empty((X.shape[0], 3, 3) + X.shape[1:4])
        for n in range(3):
            mm, ll = (n + 1) % 3, (n + 2) % 3
            V = [X[..., ll] * g[mm][k] - X[..., mm] * g[ll][k] for k in range(3)]
            for i in range(3):
                j, k = (i + 1) % 3, (i + 2) % 3
                ja[:, i, n] = -0.5 * (_coll_ordered(V[k], j + 1, D[j]) - _coll_ordered(V[j], k + 1, D[k]))
        av = [np.stack([g[c][k] for c in range(3)], axis=-1) for k in range(3)]
        jac = _jac_ordered(av)
        aff, A = affine_map(nodes)
        if aff.any():
            jc, jac_c = affine_constants(A[aff])
            ja[aff] = jac_c[:, :, :, None, None, None]
            jac[aff] = jc[:, None, None, None]
            for d in range(3):
                av[d][aff] = A[aff][:, d][:, None, None, None, :]
        _check_jac(jac, ids)
        return jac, ja, _sizes_ordered(av, w), coords
    else:
        raise ValueError(f"unknown metric form {form!r}")
    if jac.size and np.min(jac) <= 0.0:
        bad = int(np.argmin(jac.reshape(len(jac), -1).min(axis=1)))
        e = bad if ids is None else int(ids[bad])
        raise MeshError(f"inverted element {e}: min Jacobian {np.min(jac):.3e}")
    www = w[0][:, None, None] * w[1][None, :, None] * w[2][None, None, :]
    sizes = np.stack([np.einsum("ijk,Eijk->E", www, np.linalg.norm(av[d], axis=-1)) / 4.0
                      for d in range(3)], axis=1)
    return jac, ja, sizes, coords


def face_dirs(side):
    d = side // 2
    t = [k for k in range(3) if k != d]
    return d, t[0], t[1]


def _side_pts(side, p1, p2):
    d, a, b = face_dirs(side)
    pts = [None] * 3
    pts[d] = np.array([-1.0 if side % 2 == 0 else 1.0])
    pts[a] = np.asarray(p1, float)
    pts[b] = np.asarray(p2, float)
    return pts


def face_ja_analytic(nodes, side, p1, p2):
    """Ja^d at face points (t1 x t2 grid): (B, n1, n2, 3)."""
    d = side // 2
    a = map_derivs(nodes, *_side_pts(side, p1, p2))
    j, k = (d + 1) % 3, (d + 2) % 3
    ja = np.cross(a[j], a[k])
    return np.take(ja, 0, axis=1 + d)


def face_ja_trace(ja_vol, side, orders, family):
    """Trace of the volume Ja^d polynomial at own face nodes: (B, nt1, nt2, 3)."""
    d = side // 2
    row = spectral.bounds(int(orders[d]), family)[side % 2]
    tr = np.tensordot(ja_vol[:, d], row, axes=([2 + d], [0]))   # (B, 3, nt1, nt2)
    return np.moveaxis(tr, 1, -1)


def face_points(nodes, side, p1, p2):
    d = side // 2
    return np.take(map_points(nodes, *_side_pts(side, p1, p2)), 0, axis=1 + d)


def sigma_normal(ja_face, side):
    sign = 1.0 if side % 2 == 1 else -1.0
    sigma = np.linalg.norm(ja_face, axis=-1)
    return sigma, sign * ja_face / sigma[..., None]
