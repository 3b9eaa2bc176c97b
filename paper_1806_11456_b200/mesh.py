"""3D hexahedral meshes with tensor-product Lagrange geometry mappings.

Host-side setup (SURVEY §2.1 "mesh": out of scope for the GPU).  Restates the
reference's 2D quad data model (/root/reference/pkg/src/taudg/mesh.py:34-68)
for hexahedra: every element carries its geometry as control nodes on an
equispaced (m1+1)x(m2+1)x(m3+1) reference grid, faces record which local side
of each neighbour they are, and how the neighbour's face coordinates are
oriented relative to the left element's (the 3D generalisation of the
reference's single ``flip`` flag, mesh.py:213).

Local side numbering extends the reference's (mesh.py:9-11, 23):
0 = xi-  (west), 1 = xi+  (east), 2 = eta- (south), 3 = eta+ (north),
4 = zeta- (bottom), 5 = zeta+ (top).  The normal direction of side s is s//2;
its two tangential directions are the remaining reference directions in
increasing order, giving face coordinates (t1, t2).

Face orientation code ``o`` (0..7) maps an array laid out along the LEFT
element's face axes (t1, t2) onto the right element's own face array:
bit0 reverses the axis aligned with t1, bit1 reverses the axis aligned with
t2, bit2 swaps (the right's first axis runs along the left's t2).  See
``aligned_from_right`` / ``right_from_aligned``.

The mesh object is plain data (numpy arrays); both the product operator and
the CPU oracle consume it, like seeded input states.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import MeshError

WEST, EAST, SOUTH, NORTH, BOTTOM, TOP = 0, 1, 2, 3, 4, 5
SIDE_NAMES = ("west", "east", "south", "north", "bottom", "top")
# 1-based reference directions, as in the reference (mesh.py:30-31)
SIDE_NORMAL_DIR = {s: s // 2 + 1 for s in range(6)}
_TANGENTS = {0: (1, 2), 1: (0, 2), 2: (0, 1)}
SIDE_TANGENT_DIRS = {s: tuple(t + 1 for t in _TANGENTS[s // 2]) for s in range(6)}
# first tangential direction, matching the reference's 2D SIDE_TANGENT_DIR
SIDE_TANGENT_DIR = {s: SIDE_TANGENT_DIRS[s][0] for s in range(6)}


def side_tangents(side: int) -> tuple[int, int]:
    """0-based tangential reference directions (t1, t2) of a side."""
    return _TANGENTS[side // 2]


@dataclass
class Face:
    left: int
    side_left: int
    right: int = -1
    side_right: int = -1
    orient: int = 0
    tag: str | None = None

    @property
    def is_boundary(self) -> bool:
        return self.right < 0

    @property
    def flip(self) -> bool:
        return bool(self.orient & 1)


@dataclass
class HexMesh:
    """Hexahedral mesh: control-node geometry plus face connectivity.

    ``nodes`` has shape (nel, m1+1, m2+1, m3+1, 3) (uniform mapping order).
    ``faces`` is ordered interior first by (left, side_left), then boundary
    faces, as in the reference (mesh.py:220-221).  ``bc`` maps a boundary tag
    to its boundary-condition kind ("dirichlet", "freestream", "wall",
    "symmetry"); unmapped tags default to "dirichlet" (the reference's
    exact-field ghost, operators.py:152-158).
    """

    nodes: np.ndarray
    faces: list[Face]
    boundary_tags: dict[str, list[int]] = field(default_factory=dict)
    bc: dict[str, str] = field(default_factory=dict)

    def __post_init__(self):
        self.nodes = np.ascontiguousarray(self.nodes, dtype=float)
        if self.nodes.ndim != 5 or self.nodes.shape[-1] != 3:
            raise MeshError("nodes must have shape (nel, m1+1, m2+1, m3+1, 3)")
        self._arrays = None

    @property
    def num_elements(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def mapping_order(self) -> tuple[int, int, int]:
        s = self.nodes.shape
        return (s[1] - 1, s[2] - 1, s[3] - 1)

    def face_arrays(self):
        """(left, side_left, right, side_right, orient) int arrays over faces."""
        if self._arrays is None:
            a = np.array(
                [(f.left, f.side_left, f.right, f.side_right, f.orient) for f in self.faces],
                dtype=np.int64,
            ).reshape(-1, 5)
            self._arrays = tuple(np.ascontiguousarray(a[:, i]) for i in range(5))
        return self._arrays

    def bc_kind(self, tag: str | None) -> str:
        return self.bc.get(tag, "dirichlet")

    def faces_of_element(self, e: int):
        return [(i, f) for i, f in enumerate(self.faces) if f.left == e or f.right == e]


# --- orientation helpers ------------------------------------------------------


def aligned_from_right(arr: np.ndarray, orient: int) -> np.ndarray:
    """Right element's own face array (..., r1, r2) -> left-aligned (..., a, b)."""
    out = np.swapaxes(arr, -1, -2) if orient & 4 else arr
    if orient & 1:
        out = out[..., ::-1, :]
    if orient & 2:
        out = out[..., :, ::-1]
    return out


def right_from_aligned(arr: np.ndarray, orient: int) -> np.ndarray:
    """Inverse of ``aligned_from_right``."""
    out = arr
    if orient & 1:
        out = out[..., ::-1, :]
    if orient & 2:
        out = out[..., :, ::-1]
    return np.swapaxes(out, -1, -2) if orient & 4 else out


def right_orders_aligned(orders_right_tangential: tuple[int, int], orient: int):
    """Right's tangential orders re-expressed along the left's (t1, t2)."""
    r1, r2 = orders_right_tangential
    return (r2, r1) if orient & 4 else (r1, r2)


# face corner positions (t1, t2) in {0,1}^2 -> element corner index (a,b,c)
def _face_corners(side: int):
    d = side // 2
    fixed = side % 2
    t1, t2 = side_tangents(side)
    out = {}
    for u in (0, 1):
        for v in (0, 1):
            idx = [0, 0, 0]
            idx[d] = fixed
            idx[t1] = u
            idx[t2] = v
            out[(u, v)] = tuple(idx)
    return out


def orientation_from_corners(left_ids: dict, right_ids: dict) -> int:
    """Orientation code from face-corner vertex ids.

    ``left_ids[(u, v)]`` / ``right_ids[(u, v)]`` give the vertex id at face
    corner (u, v) in each side's own (t1, t2) coordinates.
    """
    inv_right = {vid: uv for uv, vid in right_ids.items()}
    for o in range(8):
        ok = True
        for (u, v), vid in left_ids.items():
            a, b = (1 - u if o & 1 else u), (1 - v if o & 2 else v)
            ru, rv = (b, a) if o & 4 else (a, b)
            if inv_right.get(vid) != (ru, rv):
                ok = False
                break
        if ok:
            return o
    raise MeshError("inconsistent face vertex pairing")


# --- generic construction from vertex ids -----------------------------------


def faces_from_hexes(hexes: np.ndarray, boundary_of=None):
    """Derive faces by matching the corner-vertex sets of element sides
    (the 3D analogue of the reference's mesh.py:195-226).

    ``hexes`` has shape (nel, 2, 2, 2): vertex id at each element corner.
    ``boundary_of(e, side)`` returns a boundary tag for unmatched sides.
    """
    by_key: dict = {}
    corners = {s: _face_corners(s) for s in range(6)}
    for e in range(hexes.shape[0]):
        for s in range(6):
            ids = {uv: int(hexes[e][c]) for uv, c in corners[s].items()}
            key = tuple(sorted(ids.values()))
            by_key.setdefault(key, []).append((e, s, ids))
    faces: list[Face] = []
    for key in sorted(by_key):
        entries = by_key[key]
        if len(entries) > 2:
            raise MeshError(f"face with corner vertices {key} shared by >2 elements")
        if len(entries) == 2:
            (el, sl, il), (er, sr, ir) = entries
            faces.append(Face(el, sl, er, sr, orientation_from_corners(il, ir)))
        else:
            e, s, _ = entries[0]
            tag = boundary_of(e, s) if boundary_of else "boundary"
            faces.append(Face(e, s, tag=tag))
    return _finish_faces(faces)


def _finish_faces(faces: list[Face]):
    faces.sort(key=lambda f: (f.is_boundary, f.left, f.side_left))
    tags: dict[str, list[int]] = {}
    for i, f in enumerate(faces):
        if f.is_boundary:
            tags.setdefault(f.tag, []).append(i)
    return faces, tags


# --- generators -----------------------------------------------------------------


def grade_coordinates(n: int, lo: float, hi: float, ratio: float, at_start: bool) -> np.ndarray:
    """n+1 coordinates whose cell sizes grow geometrically by ``ratio`` away
    from the graded end (reference mesh.py:240-247)."""
    sizes = ratio ** np.arange(n, dtype=float)
    if not at_start:
        sizes = sizes[::-1]
    sizes *= (hi - lo) / sizes.sum()
    return lo + np.concatenate([[0.0], np.cumsum(sizes)])


def trilinear_nodes(corners: np.ndarray, m=(1, 1, 1)) -> np.ndarray:
    """Control nodes of the trilinear map of (..., 2, 2, 2, 3) corners on an
    equispaced (m1+1, m2+1, m3+1) grid."""
    s = [(np.linspace(-1.0, 1.0, mi + 1) + 1.0) / 2.0 for mi in m]
    out = 0.0
    for a in (0, 1):
        wa = s[0] if a else 1.0 - s[0]
        for b in (0, 1):
            wb = s[1] if b else 1.0 - s[1]
            for c in (0, 1):
                wc = s[2] if c else 1.0 - s[2]
                w = wa[:, None, None] * wb[None, :, None] * wc[None, None, :]
                out = out + w[..., None] * corners[..., a, b, c, None, None, None, :]
    return out


def build_box(
    nx: int, ny: int, nz: int,
    bounds=((0.0, 1.0), (0.0, 1.0), (0.0, 1.0)),
    periodic=(True, True, True),
    coords=None,
    jitter: float = 0.0,
    rng=None,
    mapping_order=(1, 1, 1),
    warp=None,
    bc=None,
) -> HexMesh:
    """Structured hex box, element id e = i + nx*(j + ny*k) (x fastest, as
    the reference's build_cartesian, mesh.py:276-281).

    ``coords`` optionally gives the (xs, ys, zs) vertex coordinates (for
    graded meshes).  ``jitter`` displaces every vertex by U(-j, j)*h per
    coordinate; the periodic vertex set is jittered once so images coincide
    (SURVEY §8d cfg 3).  Boundary vertices are not moved across their box face.
    ``warp(x, y, z) -> (x, y, z)`` curves the mesh through the control nodes.
    Boundary tags: west/east/south/north/bottom/top.
    """
    (x0, x1), (y0, y1), (z0, z1) = bounds
    if coords is None:
        xs = np.linspace(x0, x1, nx + 1)
        ys = np.linspace(y0, y1, ny + 1)
        zs = np.linspace(z0, z1, nz + 1)
    else:
        xs, ys, zs = (np.asarray(c, dtype=float) for c in coords)
    n = (nx, ny, nz)
    L = (xs[-1] - xs[0], ys[-1] - ys[0], zs[-1] - zs[0])
    # vertex lattice (nx+1, ny+1, nz+1, 3)
    V = np.stack(np.meshgrid(xs, ys, zs, indexing="ij"), axis=-1)
    if jitter > 0.0:
        rng = np.random.default_rng(0) if rng is None else rng
        h = np.array([L[0] / nx, L[1] / ny, L[2] / nz])
        # one displacement per distinct (periodically identified) vertex
        shape = tuple(n[d] if periodic[d] else n[d] + 1 for d in range(3))
        disp = rng.uniform(-jitter, jitter, shape + (3,)) * h
        ii = [np.arange(n[d] + 1) % n[d] if periodic[d] else np.arange(n[d] + 1) for d in range(3)]
        D = disp[np.ix_(ii[0], ii[1], ii[2])]
        for d in range(3):
            if not periodic[d]:
                sl = [slice(None)] * 3
                sl[d] = 0
                D[tuple(sl) + (d,)] = 0.0
                sl[d] = n[d]
                D[tuple(sl) + (d,)] = 0.0
        V = V + D
    nel = nx * ny * nz
    corners = np.empty((nel, 2, 2, 2, 3))
    ids = np.arange(nel)
    I = ids % nx
    J = (ids // nx) % ny
    K = ids // (nx * ny)
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                corners[:, a, b, c] = V[I + a, J + b, K + c]
    nodes = trilinear_nodes(corners, mapping_order)
    if warp is not None:
        wx, wy, wz = warp(nodes[..., 0], nodes[..., 1], nodes[..., 2])
        nodes = np.stack([wx, wy, wz], axis=-1)

    def eid(i, j, k):
        return i + nx * (j + ny * k)

    faces: list[Face] = []
    names = (("west", "east"), ("south", "north"), ("bottom", "top"))
    for e in range(nel):
        ijk = (int(I[e]), int(J[e]), int(K[e]))
        for d in range(3):
            # the face on the + side of e along d
            nb = list(ijk)
            nb[d] += 1
            if nb[d] == n[d]:
                if periodic[d]:
                    nb[d] = 0
                else:
                    faces.append(Face(e, 2 * d + 1, tag=names[d][1]))
                    continue
            faces.append(Face(e, 2 * d + 1, eid(*nb), 2 * d, 0))
            # non-periodic minus side
        for d in range(3):
            if ijk[d] == 0 and not periodic[d]:
                faces.append(Face(e, 2 * d, tag=names[d][0]))
    faces, tags = _finish_faces(faces)
    return HexMesh(nodes, faces, tags, dict(bc or {}))


def extrude_2d(nodes2d: np.ndarray, faces2d, tags2d: dict, dz: float = 1.0) -> HexMesh:
    """One-element-deep extrusion of a reference 2D quad mesh, self-periodic in z.

    ``nodes2d`` (nel, m1+1, m2+1, 2) are the reference control nodes
    (mesh.py:38-40); ``faces2d`` rows (left, side_left, right, side_right,
    flip) follow the reference's face list (mesh.py:44-54); z spans
    [-dz/2, dz/2] with mapping order 1.  With N3 = 0 Legendre-Gauss nodes the
    3D operator reduces to the 2D one times dz.
    """
    nel, a1, a2, _ = nodes2d.shape
    nodes = np.empty((nel, a1, a2, 2, 3))
    nodes[..., 0, :2] = nodes2d
    nodes[..., 1, :2] = nodes2d
    nodes[..., 0, 2] = -0.5 * dz
    nodes[..., 1, 2] = 0.5 * dz
    faces = []
    bmap = {}
    for tag, idx in tags2d.items():
        for i in idx:
            bmap[int(i)] = tag
    for i, row in enumerate(faces2d):
        l, sl, r, sr, flip = (int(v) for v in row)
        if r < 0:
            faces.append(Face(l, sl, tag=bmap.get(i, "boundary")))
        else:
            faces.append(Face(l, sl, r, sr, 1 if flip else 0))
    for e in range(nel):
        faces.append(Face(e, TOP, e, BOTTOM, 0))
    faces, tags = _finish_faces(faces)
    return HexMesh(nodes, faces, tags)


def extract_element(msh: HexMesh, e: int) -> HexMesh:
    """Single-element mesh with identical geometry; all six sides become
    boundary faces (reference mesh.py:291-297)."""
    faces = [Face(0, s, tag=SIDE_NAMES[s]) for s in range(6)]
    faces, tags = _finish_faces(faces)
    return HexMesh(msh.nodes[e : e + 1].copy(), faces, tags, dict(msh.bc))


def _proper_rotations():
    import itertools as it
    out = []
    for perm in it.permutations(range(3)):
        sgn = np.linalg.det(np.eye(3)[list(perm)])
        for flips in it.product((0, 1), repeat=3):
            if sgn * (-1) ** sum(flips) > 0:
                out.append((perm, flips))
    return out


def build_rotated_box(nx: int, ny: int, nz: int, bounds=((0.0, 1.0), (0.0, 1.0), (0.0, 1.0)),
                      jitter: float = 0.0, seed: int = 0, bc=None) -> HexMesh:
    """Non-periodic structured box whose elements carry randomly rotated local
    axes (one of the 24 proper cube rotations each), so that neighbouring
    faces meet with every orientation code.  Faces come from vertex matching
    (``faces_from_hexes``); boundary tags are 'boundary'."""
    rng = np.random.default_rng(seed)
    (x0, x1), (y0, y1), (z0, z1) = bounds
    V = np.stack(np.meshgrid(np.linspace(x0, x1, nx + 1), np.linspace(y0, y1, ny + 1),
                             np.linspace(z0, z1, nz + 1), indexing="ij"), axis=-1)
    if jitter > 0.0:
        h = np.array([(x1 - x0) / nx, (y1 - y0) / ny, (z1 - z0) / nz])
        D = rng.uniform(-jitter, jitter, V.shape) * h
        D[0, :, :, 0] = D[-1, :, :, 0] = 0.0
        D[:, 0, :, 1] = D[:, -1, :, 1] = 0.0
        D[:, :, 0, 2] = D[:, :, -1, 2] = 0.0
        V = V + D
    vid = np.arange(V[..., 0].size).reshape(V.shape[:3])
    flatV = V.reshape(-1, 3)
    rots = _proper_rotations()
    nel = nx * ny * nz
    hexes = np.empty((nel, 2, 2, 2), dtype=np.int64)
    e = 0
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                base = vid[i:i + 2, j:j + 2, k:k + 2]
                perm, flips = rots[rng.integers(len(rots))]
                loc = np.empty((2, 2, 2), dtype=np.int64)
                for a in (0, 1):
                    for b in (0, 1):
                        for c in (0, 1):
                            new = (a, b, c)
                            old = [0, 0, 0]
                            for kk in range(3):
                                v = new[kk]
                                old[perm[kk]] = 1 - v if flips[kk] else v
                            loc[a, b, c] = base[tuple(old)]
                hexes[e] = loc
                e += 1
    corners = flatV[hexes]                                   # (nel, 2, 2, 2, 3)
    nodes = trilinear_nodes(corners)
    faces, tags = faces_from_hexes(hexes, lambda e, s: "boundary")
    return HexMesh(nodes, faces, tags, dict(bc or {}))


def _cube_face_dirs():
    """Six cube faces as (normal axis, sign, tangent axes): equiangular blocks."""
    return [(0, +1), (0, -1), (1, +1), (1, -1), (2, +1), (2, -1)]


def build_cubed_sphere(na: int, nr: int, r0: float = 0.5, r1: float = 10.0, ratio: float = 1.15,
                       mapping_order: int = 3, bc=None) -> HexMesh:
    """Equiangular cubed-sphere shell: 6 blocks of na x na (angular) x nr
    (radial) elements between radii r0 and r1, radial sizes growing
    geometrically by ``ratio`` away from the inner sphere.  Geometry is the
    analytic map sampled on an equispaced control grid of ``mapping_order``
    per direction (curved elements).  Connectivity comes from vertex matching
    across block seams, so seam faces carry general orientation codes.
    Boundary tags: 'wall' (inner sphere), 'freestream' (outer)."""
    rs = grade_coordinates(nr, r0, r1, ratio, at_start=True)
    ang = np.linspace(-np.pi / 4, np.pi / 4, na + 1)
    m = mapping_order

    def direction(axis, sign, a, b):
        ta, tb = np.tan(a), np.tan(b)
        v = [None, None, None]
        others = [x for x in range(3) if x != axis]
        v[axis] = sign * np.ones_like(ta)
        v[others[0]] = ta
        v[others[1]] = tb
        v = np.stack(v, axis=-1)
        return v / np.linalg.norm(v, axis=-1, keepdims=True)

    def point(axis, sign, a, b, r):
        return direction(axis, sign, a, b) * np.asarray(r)[..., None]

    # vertex lattice per block, merged across seams by rounded coordinates
    all_pts, blocks = [], []
    for axis, sign in _cube_face_dirs():
        A, B, R = np.meshgrid(ang, ang, rs, indexing="ij")
        P = point(axis, sign, A, B, R)
        blocks.append((axis, sign))
        all_pts.append(P.reshape(-1, 3))
    pts = np.concatenate(all_pts)
    _, inverse = np.unique(np.round(pts, 10), axis=0, return_inverse=True)
    vid = inverse.reshape(6, na + 1, na + 1, nr + 1)
    nel = 6 * na * na * nr
    hexes = np.empty((nel, 2, 2, 2), dtype=np.int64)
    nodes = np.empty((nel, m + 1, m + 1, m + 1, 3))
    g = np.linspace(0.0, 1.0, m + 1)
    e = 0
    for bi, (axis, sign) in enumerate(blocks):
        for k in range(nr):
            for j in range(na):
                for i in range(na):
                    # local (a, b, r); flip a for negatively oriented blocks
                    a0, a1 = ang[i], ang[i + 1]
                    b0, b1 = ang[j], ang[j + 1]
                    rr0, rr1 = rs[k], rs[k + 1]
                    A = a0 + (a1 - a0) * g[:, None, None]
                    B = b0 + (b1 - b0) * g[None, :, None]
                    Rr = rr0 + (rr1 - rr0) * g[None, None, :]
                    A, B, Rr = np.broadcast_arrays(A, B, Rr)
                    X = point(axis, sign, A, B, Rr)
                    ids = vid[bi, i:i + 2, j:j + 2, k:k + 2]
                    # orientation: make the local frame right-handed
                    a1v = X[-1, 0, 0] - X[0, 0, 0]
                    b1v = X[0, -1, 0] - X[0, 0, 0]
                    r1v = X[0, 0, -1] - X[0, 0, 0]
                    if np.dot(np.cross(a1v, b1v), r1v) < 0:
                        X = X[::-1]
                        ids = ids[::-1]
                    nodes[e] = X
                    hexes[e] = ids
                    e += 1

    def tag(el, side):
        # radial direction is local zeta: bottom = inner sphere, top = outer
        return "wall" if side == BOTTOM else "freestream"

    faces, tags = faces_from_hexes(hexes, tag)
    bcs = {"wall": "wall", "freestream": "freestream"}
    bcs.update(bc or {})
    return HexMesh(nodes, faces, tags, bcs)
