"""Anisotropic order selection and jump limiting (oracle).  Restates
/root/reference/pkg/src/taudg/adaptation.py:115-375 for three directions;
collapsed (order-0) directions keep their order."""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from . import multigrid
from . import tau as tau_est
from .fields import OrderField, transfer


class AdaptationError(Exception):
    pass


@dataclass(frozen=True)
class AdaptConfig:
    tau_max: float
    n_max: int
    n_min: int = 1
    jump_rule: str = "strict-one"
    conforming_tags: tuple = ()
    stages: tuple = ()


def _key(n):
    # min DOF, ties to the smaller max order, then the smaller first orders
    return ((n[0] + 1) * (n[1] + 1) * (n[2] + 1), max(n), n[0], n[1])


def select_orders(tmap, cfg):
    nel = tmap.num_elements
    arr = np.empty((nel, 3), dtype=int)
    paths, preds = [], []
    lo, hi = cfg.n_min, cfg.n_max
    for e in range(nel):
        p = tmap.fine_orders.orders[e]
        frozen = getattr(tmap, "frozen", set())
        act = [d for d in range(3) if p[d] > 0 and d not in frozen]
        for d in act:
            if not tmap.tau[e][d]:
                raise AdaptationError(f"element {e} has an empty truncation-error map")

        def combos(choices):
            for vals in itertools.product(*choices):
                n = [int(x) for x in p]                 # frozen directions keep their order
                for d, v in zip(act, vals):
                    n[d] = v
                yield tuple(n)

        inner = [[n for n in tmap.measured_orders(e, d + 1) if n < p[d]] for d in act]
        feasible = []
        for n in combos(inner):
            v = sum(tmap.tau[e][d][n[d]] for d in act)
            if v <= cfg.tau_max and all(lo <= n[d] <= hi for d in act):
                feasible.append((n, v))
        path = "inner-map"
        if not feasible:
            rng = [[k for k in range(lo, hi + 1) if k in tmap.tau[e][d]] for d in act]
            for n in combos(rng):
                v = sum(tmap.tau[e][d][n[d]] for d in act)
                if v <= cfg.tau_max:
                    feasible.append((n, v))
            path = "extrapolated"
        if feasible:
            n, v = min(feasible, key=lambda it: _key(it[0]))
        else:
            n = tuple(hi if d in act else int(p[d]) for d in range(3))
            v = tmap.combined(e, n)
            v = float("inf") if v is None else v
            path = "fallback-N_max"
        arr[e] = n
        paths.append(path)
        preds.append(v)
    return OrderField(arr), paths, preds


def _face_slot_pairs(msh):
    pairs = []
    for f in msh.faces:
        if f.is_boundary:
            continue
        dl, dr = f.side_left // 2, f.side_right // 2
        tl = [x for x in range(3) if x != dl]
        tr = [x for x in range(3) if x != dr]
        if f.orient & 4:
            tr = tr[::-1]
        pairs.append((f.left, tl[0], f.right, tr[0]))
        pairs.append((f.left, tl[1], f.right, tr[1]))
        pairs.append((f.left, dl, f.right, dr))
    return pairs


def limit_jumps(msh, orders, rule="strict-one"):
    arr = orders.orders.copy()
    pairs = _face_slot_pairs(msh)
    for _ in range(arr.size * (int(arr.max()) + 1) + 1):
        changed = False
        for ea, da, eb, db in pairs:
            a, b = int(arr[ea, da]), int(arr[eb, db])
            fa = b - 1 if rule == "strict-one" else (2 * b) // 3
            if a < fa:
                a = fa
                arr[ea, da] = fa
                changed = True
            fb = a - 1 if rule == "strict-one" else (2 * a) // 3
            if b < fb:
                arr[eb, db] = fb
                changed = True
        if not changed:
            return OrderField(arr)
    raise AdaptationError("jump limiting failed to reach a fixed point")


def _boundary_face_frames(msh, face_ids):
    """Frame index (0 or 1) of each element-local tangential axis of the given
    boundary faces, transported across shared face edges: two faces sharing an
    edge give the axis running along it the same frame index, and likewise the
    axis crossing it.  Each connected piece starts from its first face's local
    order (t1 -> 0, t2 -> 1); on a closed surface whose frame cannot be
    transported consistently the first assignment wins."""
    M = np.array(msh.nodes.shape[1:4]) - 1
    edges = {}
    info = []
    for fi in face_ids:
        f = msh.faces[fi]
        e, s = f.left, f.side_left
        d = s // 2
        a, b = [x for x in range(3) if x != d]
        idx = [0, 0, 0]
        idx[d] = 0 if s % 2 == 0 else int(M[d])

        def corner(ia, ib):
            j = list(idx)
            j[a], j[b] = ia, ib
            return msh.nodes[e, j[0], j[1], j[2]]

        scale = float(np.abs(msh.nodes[e]).max()) + 1.0
        key = lambda p, q: tuple(sorted((tuple(np.round(p / scale, 9)), tuple(np.round(q / scale, 9)))))
        mine = []
        for ib in (0, int(M[b])):       # edges running along a
            mine.append((key(corner(0, ib), corner(int(M[a]), ib)), a, b))
        for ia in (0, int(M[a])):       # edges running along b
            mine.append((key(corner(ia, 0), corner(ia, int(M[b]))), b, a))
        info.append((e, a, b, mine))
        for k, along, across in mine:
            edges.setdefault(k, []).append((len(info) - 1, along, across))
    frame = [None] * len(info)
    for start in range(len(info)):
        if frame[start] is not None:
            continue
        e, a, b, _ = info[start]
        frame[start] = {a: 0, b: 1}
        queue = [start]
        while queue:
            u = queue.pop(0)
            for k, along, across in info[u][3]:
                for v, v_along, v_across in edges[k]:
                    if frame[v] is None:
                        frame[v] = {v_along: frame[u][along], v_across: frame[u][across]}
                        queue.append(v)
    return [(info[i][0], frame[i]) for i in range(len(info))]


def conforming_pass(msh, orders, tags, rule=None):
    """adaptation.py:212-250 in 3D: on each tagged boundary, every element's
    tangential order in frame direction k becomes the maximum over the tag
    (frames transported across shared edges, _boundary_face_frames); with a
    jump rule, alternate with limit_jumps until neither changes the field."""
    tags = tuple(tags)
    unknown = [t for t in tags if t not in msh.boundary_tags]
    if unknown:
        raise AdaptationError(f"unknown boundary tags: {unknown}")
    groups = []
    for tag in tags:
        slots = [[], []]
        for e, fr in _boundary_face_frames(msh, msh.boundary_tags[tag]):
            for axis, k in fr.items():
                slots[k].append((e, axis))
        groups += [g for g in slots if g]

    def share(arr):
        changed = False
        for slots in groups:
            top = max(int(arr[e, d]) for e, d in slots)
            for e, d in slots:
                if arr[e, d] != top:
                    arr[e, d] = top
                    changed = True
        return changed

    arr = orders.orders.copy()
    if rule is None:
        share(arr)
        return OrderField(arr)
    for _ in range(arr.size * (int(arr.max()) + 1) + 1):
        changed = share(arr)
        limited = limit_jumps(msh, OrderField(arr), rule)
        changed = changed or not np.array_equal(limited.orders, arr)
        arr = limited.orders.copy()
        if not changed:
            return limited
    raise AdaptationError("conforming pass failed to reach a fixed point")
