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
    notes: str = ""


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
    rng = np.random.default_rng(seed)
    noise_cache = {}
    p0 = 1.0 / (law.gamma * law.mach ** 2)

    def init(x, y, z):
        u = np.sin(x) * np.cos(y) * np.cos(z)
        v = -np.cos(x) * np.sin(y) * np.cos(z)
        w = 0.0 * x
        p = p0 + (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
        q = law.conservative(1.0 + 0.0 * x, u, v, w, p)
        key = q.shape
        if key not in noise_cache:
            noise_cache[key] = rng.uniform(-1e-3, 1e-3, q.shape)
        return q + noise_cache[key]

    return Workload(f"cfg4: {n}^3 periodic affine (2pi), N={order} LGL, TGV M=0.1 Re=1600", msh, law,
                    OrderField.uniform(n ** 3, order), init,
                    smoother=dict(pre_sweeps=2, post_sweeps=2, coarsest_sweeps=2, max_batches=1))


CONFIGS = {1: config1, 3: config3, 4: config4}
