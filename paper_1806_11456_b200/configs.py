"""BASELINE.json workload configurations (seeded synthetic inputs).

Decisions the configs leave open are recorded here and in DESIGN.md
(SURVEY Appendix A): LGL nodes, invariant-curl metrics, constant mu = 1/Re,
BR1 on (u, v, w, T), Roe flux; perturbation amplitude is PER TERM; config 1
uses 3 coarsest sweeps; config 4 uses 2 coarsest sweeps; all sweeps pinned
with max_batches = 1.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import mesh, physics
from .fields import OrderField


@dataclass
class Workload:
    name: str
    mesh: mesh.HexMesh
    law: physics.NavierStokes
    orders: OrderField
    init: object                       # fn(x, y, z) -> (5, ...) conservative state
    family: str = "LGL"
    form: str = "curl"
    smoother: dict = field(default_factory=dict)
    time: dict = field(default_factory=dict)     # TimeConfig kwargs (CFL constants)
    notes: str = ""


def hashed_noise(seed, amp):
    """Deterministic per-point noise in [-amp, amp) from the node position
    (a seeded hash), so CPU oracle and GPU get bit-identical inputs whatever
    order they evaluate nodes in."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(10.0, 100.0, 3)
    ph = rng.uniform(0.0, 1.0, 5)

    def fn(x, y, z, comp):
        s = np.sin(a[0] * x + a[1] * y + a[2] * z + 7.0 * comp + ph[comp]) * 43758.5453123
        return amp * (2.0 * (s - np.floor(s)) - 1.0)

    return fn


def sinusoid_perturbation(law, rng, amp, kz=True, terms=4, kmax=3, box=(1.0, 1.0, 1.0)):
    """Freestream plus sum of ``terms`` sinusoids in rho, u, v, w with integer
    wavenumbers 1..kmax (per box length) and random phases; ``amp`` per term."""
    fs = law.freestream()
    k = rng.integers(1, kmax + 1, (terms, 3)).astype(float)
    if not kz:
        k[:, 2] = 0.0
    ph = rng.uniform(0.0, 2.0 * np.pi, (terms, 4))
    L = np.asarray(box, float)
    p_inf = 1.0 / (law.gamma * law.mach ** 2)

    def fn(x, y, z):
        arg = [2 * np.pi * (k[m, 0] * x / L[0] + k[m, 1] * y / L[1] + k[m, 2] * z / L[2]) for m in range(terms)]
        d = [amp * sum(np.sin(arg[m] + ph[m, c]) for m in range(terms)) for c in range(4)]
        rho = fs[0] + d[0]
        u, v, w = fs[1] + d[1], fs[2] + d[2], fs[3] + d[3]
        return law.conservative(rho, u, v, w, p_inf + 0.0 * x)

    return fn


def config1(seed=0) -> Workload:
    """Quasi-2D periodic box [0,1]^2 x [0,1/8], 8x8x1, N=3, M=0.3, Re=100."""
    msh = mesh.build_box(8, 8, 1, bounds=((0, 1), (0, 1), (0, 0.125)))
    law = physics.NavierStokes(gamma=1.4, prandtl=0.72, mach=0.3, reynolds=100.0)
    rng = np.random.default_rng(seed)
    init = sinusoid_perturbation(law, rng, 1e-2, kz=False, box=(1.0, 1.0, 0.125))
    return Workload("cfg1: 8x8x1 periodic quasi-2D, N=3 LGL, NS M=0.3 Re=100", msh, law,
                    OrderField.uniform(64, 3), init,
                    smoother=dict(pre_sweeps=3, post_sweeps=3, coarsest_sweeps=3, max_batches=1))


def config3(seed_mesh=2, seed_state=3, n=32) -> Workload:
    """32^3 periodic box, corners jittered 10%, orders iid U{1..7}^3, M=0.3, Re=1000."""
    rng = np.random.default_rng(seed_mesh)
    msh = mesh.build_box(n, n, n, jitter=0.1, rng=rng)
    orders = OrderField(rng.integers(1, 8, (n ** 3, 3)))
    law = physics.NavierStokes(gamma=1.4, prandtl=0.72, mach=0.3, reynolds=1000.0)
    init = sinusoid_perturbation(law, np.random.default_rng(seed_state), 1e-2)
    return Workload(f"cfg3: {n}^3 jittered periodic, orders U{{1..7}}^3, NS M=0.3 Re=1000", msh, law,
                    orders, init)


def config4(seed=4, n=24, order=7) -> Workload:
    """24^3 periodic affine box (2pi), N=7, Taylor-Green-like field, M=0.1, Re=1600."""
    L = 2.0 * np.pi
    msh = mesh.build_box(n, n, n, bounds=((0, L), (0, L), (0, L)))
    law = physics.NavierStokes(gamma=1.4, prandtl=0.72, mach=0.1, reynolds=1600.0)
    noise = hashed_noise(seed, 1e-3)
    p0 = 1.0 / (law.gamma * law.mach ** 2)

    def init(x, y, z):
        u = np.sin(x) * np.cos(y) * np.cos(z)
        v = -np.cos(x) * np.sin(y) * np.cos(z)
        w = 0.0 * x
        p = p0 + (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
        q = law.conservative(1.0 + 0.0 * x, u, v, w, p)
        return q + np.stack([noise(x, y, z, c) for c in range(5)])

    return Workload(f"cfg4: {n}^3 periodic affine (2pi), N={order} LGL, TGV M=0.1 Re=1600", msh, law,
                    OrderField.uniform(n ** 3, order), init,
                    smoother=dict(pre_sweeps=2, post_sweeps=2, coarsest_sweeps=2, max_batches=1))


def config2(seed=1, nx=40, ny=20, order=5, dz=0.05, nz_order=1) -> Workload:
    """Flat-plate-type steady case: x in [-0.5, 1], y in [0, 0.5], one element
    deep (dz, self-periodic, Nz held at 1), 40 x 20 elements graded (ratio 1.1)
    toward y = 0 and, two-sided, toward x = 0 (13 cells on the x < 0 side, 27
    on x >= 0).  No-slip adiabatic wall for x >= 0 and symmetry for x < 0 at
    y = 0, freestream elsewhere; M = 0.2, Re = 1e5 per unit length; freestream
    plus 1e-3 seeded nodal noise (relative to |q_inf| per variable)."""
    nl = int(round(nx * 0.5 / 1.5))
    xl = mesh.grade_coordinates(nl, -0.5, 0.0, 1.1, at_start=False)
    xr = mesh.grade_coordinates(nx - nl, 0.0, 1.0, 1.1, at_start=True)
    xs = np.concatenate([xl, xr[1:]])
    ys = mesh.grade_coordinates(ny, 0.0, 0.5, 1.1, at_start=True)
    zs = np.array([0.0, dz])
    msh = mesh.build_box(nx, ny, 1, coords=(xs, ys, zs), periodic=(False, False, True))
    # split the y = 0 boundary: wall for x >= 0, symmetry for x < 0
    faces = msh.faces
    tags = {}
    for fi, f in enumerate(faces):
        if f.is_boundary:
            if f.tag == "south":
                xc = msh.nodes[f.left][..., 0].mean()
                f.tag = "wall" if xc >= 0.0 else "symmetry"
            tags.setdefault(f.tag, []).append(fi)
    msh.boundary_tags = tags
    msh.bc = {"wall": "wall", "symmetry": "symmetry", "west": "freestream", "east": "freestream",
              "north": "freestream"}
    law = physics.NavierStokes(gamma=1.4, prandtl=0.72, mach=0.2, reynolds=1e5)
    fs = law.freestream()
    noise = hashed_noise(seed, 1e-3)

    def init(x, y, z):
        return np.stack([fs[c] + 0.0 * x + noise(x, y, z, c) * max(abs(fs[c]), 1.0) for c in range(5)])

    orders = np.tile([order, order, nz_order], (nx * ny, 1))
    return Workload(f"cfg2: {nx}x{ny}x1 graded flat plate, N={order} (Nz={nz_order}) LGL, NS M=0.2 Re=1e5",
                    msh, law, OrderField(orders), init,
                    smoother=dict(pre_sweeps=3, post_sweeps=3, coarsest_sweeps=10, max_batches=1),
                    time=dict(cfl_advective=0.05, cfl_viscous=0.025),
                    notes="Nz held at 1 (not adapted); two-sided x clustering 13/27 cells; CFL 0.05/0.025: "
                          "V-cycles at 0.2/0.1 diverge through the coarse-grid correction (measured)")


def config5(seed=5, na=16, nr=24, order=3, r1=10.0) -> Workload:
    """Cubed-sphere shell r in [0.5, 10] around a unit-diameter sphere, 6 blocks
    of na x na x nr elements, radial ratio 1.15, geometry at the solution
    order; no-slip adiabatic wall on the sphere, freestream outside; M = 0.2,
    Re = 200; freestream plus 1e-3 seeded noise."""
    msh = mesh.build_cubed_sphere(na, nr, 0.5, r1, 1.15, mapping_order=order)
    law = physics.NavierStokes(gamma=1.4, prandtl=0.72, mach=0.2, reynolds=200.0)
    fs = law.freestream()
    noise = hashed_noise(seed, 1e-3)

    def init(x, y, z):
        return np.stack([fs[c] + 0.0 * x + noise(x, y, z, c) * max(abs(fs[c]), 1.0) for c in range(5)])

    nel = msh.num_elements
    return Workload(f"cfg5: cubed-sphere shell 6x{na}x{na}x{nr}, N={order} LGL curved, NS M=0.2 Re=200",
                    msh, law, OrderField.uniform(nel, order), init,
                    smoother=dict(pre_sweeps=3, post_sweeps=3, coarsest_sweeps=5, max_batches=1),
                    time=dict(cfl_advective=0.05, cfl_viscous=0.025),
                    notes="CFL 0.05/0.025: the max(N,1)^2 bound under-estimates N=1 stiffness on "
                          "curved shell elements (SURVEY §0.7)")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
