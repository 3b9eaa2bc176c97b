"""Shared test helpers: golden-fixture loading and layout conversion.

Golden fields are stored element by element in the reference's (n1+1, n2+1)
xi-slowest layout.  The oracle's blocks are (B, nv, n1+1, n2+1, n3+1)
(xi slowest); the device layout is (nv, n3+1, n2+1, n1+1) per element (xi
fastest).
"""

from __future__ import annotations

import ast
import os

import numpy as np

from oracle import physics as ophys
from oracle.fields import NodalField as ONodal
from oracle.fields import OrderField as OOrders
from paper_1806_11456_b200 import mesh as pmesh
from paper_1806_11456_b200 import physics as pphys

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"ref_{name}.npz"), allow_pickle=False))


def golden_mesh(g, dz=1.0):
    tags = {}
    names = list(g["tag_names"])
    for i, t in enumerate(names):
        tags[str(t)] = [int(x) for x in g[f"tag_{i}"]]
    return pmesh.extrude_2d(g["nodes2d"], g["faces2d"], tags, dz=dz)


def orders3(orders2):
    o = np.asarray(orders2)
    return np.concatenate([o, np.zeros((len(o), 1), dtype=int)], axis=1)


def golden_law(g):
    params = ast.literal_eval(str(g["params"])) if "params" in g else {}
    return pphys.make_case(str(g["case"]), **params)


def oracle_law(plaw):
    """Oracle flux functors with the product law's parameters + manufactured data."""
    if isinstance(plaw, pphys.AdvectionDiffusion):
        law = ophys.AdvectionDiffusion(plaw.velocity, plaw.mu)
    elif isinstance(plaw, pphys.ViscousBurgers):
        law = ophys.ViscousBurgers(plaw.mu, plaw.beta)
    elif isinstance(plaw, pphys.NavierStokes):
        law = ophys.NavierStokes(plaw.gamma, plaw.prandtl, plaw.mach, plaw.reynolds, plaw.aoa)
        law.exact, law.source = plaw.exact, plaw.source
        return law
    else:
        raise TypeError(plaw)
    ex, src = plaw.exact, plaw.source
    return law.with_manufactured(
        None if ex is None else (lambda x, y, z: ex(x, y, z)),
        None if src is None else (lambda x, y, z: src(x, y, z)),
    )


def ref_flat_to_oracle(flatv, of: OOrders, nv=1):
    """Reference element-concatenated 2D field -> oracle NodalField (n3 = 0)."""
    f = ONodal.zeros(of, nv)
    pos = 0
    for e in range(of.num_elements):
        n1, n2, n3 = of.orders[e]
        k = (n1 + 1) * (n2 + 1) * (n3 + 1) * nv
        f.set_element(e, flatv[pos:pos + k].reshape(nv, n1 + 1, n2 + 1, n3 + 1))
        pos += k
    return f


def oracle_to_ref_flat(field: ONodal):
    return np.concatenate([field.element(e).ravel() for e in range(field.field.num_elements)])


class RefStyleMesh2D:
    """Stand-in with the reference Mesh2D's duck type (mesh.py:44-70):
    ``elements[e].nodes``, ``faces[f].left/side_left/right/side_right/flip``,
    ``boundary_tags`` — built from a golden case's arrays, so drop-in tests
    run where the reference package is absent (the GPU box)."""

    class _El:
        def __init__(self, nodes):
            self.nodes = nodes

    class _Face:
        def __init__(self, row):
            self.left, self.side_left, self.right, self.side_right = (int(v) for v in row[:4])
            self.flip = bool(row[4])

    def __init__(self, g):
        self.elements = [self._El(n) for n in g["nodes2d"]]
        self.faces = [self._Face(r) for r in g["faces2d"]]
        names = list(g["tag_names"])
        self.boundary_tags = {str(t): [int(x) for x in g[f"tag_{i}"]] for i, t in enumerate(names)}


class RefStyleAdvDiffSine:
    """The reference's advdiff-sine case (physics.py:94-106) as a 2D law object."""

    name = "advection-diffusion"

    def __init__(self, mu=0.1, velocity=(1.0, 1.0)):
        self.mu, self.velocity = mu, velocity
        a, b = velocity
        pi = np.pi
        self.exact = lambda x, y: np.sin(pi * x) * np.sin(pi * y)
        self.source = lambda x, y: (a * pi * np.cos(pi * x) * np.sin(pi * y) + b * pi * np.sin(pi * x) * np.cos(pi * y)
                                    + 2.0 * mu * pi * pi * np.sin(pi * x) * np.sin(pi * y))
