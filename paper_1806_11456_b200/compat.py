"""Literal drop-in for the reference's own 2D objects.

A user of the reference package holds a 2D ``Mesh2D`` (mesh.py:44-70: quad
elements with control nodes, faces with ``flip``, ``boundary_tags``), an
``OrderField`` of (N1, N2) pairs (fields.py:22-74) and a scalar law with
2D manufactured ``exact(x, y)`` / ``source(x, y)`` (physics.py:18-120).
The device operator works on 3D hexahedra, so these are lifted here —
duck-typed, without importing the reference — exactly as the parity tests
do: a one-element-deep, z-self-periodic extrusion with N3 = 0 Legendre-Gauss
nodes and the cross-product metrics, which reproduces the reference's 2D
operator.  ``DGOperator``, ``FASSolver``,
``tau.estimate`` and the adaptation drivers call ``resolve`` first, so
``DGOperator(mesh2d, law, orders2d)`` works unchanged and defaults to the
reference's LG nodes; 3D inputs default to LGL with curl-form metrics.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigError


def is_reference_mesh(msh) -> bool:
    return hasattr(msh, "elements") and hasattr(msh, "faces") and not hasattr(msh, "face_arrays")


def as_hex_mesh(msh):
    """HexMesh passthrough; a reference Mesh2D becomes its z-extrusion (cached)."""
    from . import mesh as pmesh

    if isinstance(msh, pmesh.HexMesh):
        return msh
    if not is_reference_mesh(msh):
        raise ConfigError(f"unsupported mesh type {type(msh).__name__}")
    cached = getattr(msh, "_b200_hex", None)
    if cached is not None:
        return cached
    nodes = np.stack([np.asarray(el.nodes, float) for el in msh.elements])
    faces = np.array([(f.left, f.side_left, f.right, f.side_right, int(bool(f.flip))) for f in msh.faces])
    tags = {str(k): [int(i) for i in v] for k, v in msh.boundary_tags.items()}
    hexm = pmesh.extrude_2d(nodes, faces, tags, dz=1.0)
    try:
        msh._b200_hex = hexm
    except AttributeError:      # frozen / slotted mesh: no cache
        pass
    return hexm


def as_order_field(orders):
    """Product OrderField passthrough; (nel, 2) orders (a reference OrderField
    or an array) get N3 = 0."""
    from .fields import OrderField

    if isinstance(orders, OrderField):
        return orders
    arr = np.asarray(getattr(orders, "orders", orders), dtype=np.int64)
    if arr.ndim == 2 and arr.shape[1] == 2:
        arr = np.concatenate([arr, np.zeros((len(arr), 1), np.int64)], axis=1)
    return OrderField(arr)


def as_law(law):
    """Product laws pass through; the reference's scalar laws map to their
    device counterparts with the 2D manufactured fields lifted to (x, y, z)."""
    from . import physics

    if hasattr(law, "law_id"):
        return law
    name = getattr(law, "name", None)
    mu = float(getattr(law, "mu", 0.0))
    if name == "advection-diffusion":
        out = physics.AdvectionDiffusion(tuple(law.velocity), mu)
    elif name == "viscous-burgers":
        out = physics.ViscousBurgers(mu)
    else:
        raise ConfigError(f"unsupported law {type(law).__name__}")
    ex, src = getattr(law, "exact", None), getattr(law, "source", None)
    return out.with_manufactured(None if ex is None else (lambda x, y, z, f=ex: f(x, y)),
                                 None if src is None else (lambda x, y, z, f=src: f(x, y)))


def resolve(msh, law, orders, family=None, form=None):
    """(hex mesh, device law, OrderField, family, form) with the reference's
    defaults (LG, cross-product metrics) for its 2D objects and LGL/curl for 3D."""
    two_d = is_reference_mesh(msh)
    fam = family if family is not None else ("LG" if two_d else "LGL")
    frm = form if form is not None else ("cross" if two_d else "curl")
    return as_hex_mesh(msh), as_law(law), (None if orders is None else as_order_field(orders)), fam, frm
