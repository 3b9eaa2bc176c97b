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
