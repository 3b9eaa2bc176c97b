"""Conservation-law descriptors for the device operator.

The flux arithmetic lives in CUDA (csrc/laws.cuh); this module carries the
law's identity and parameters across the C-ABI, plus host-side manufactured
data (exact fields for boundary ghosts and sources).

Scalar laws mirror /root/reference/pkg/src/taudg/physics.py:18-88 in 3D (the
reference's 2D cases are the z-independent special case); the manufactured
cases restate physics.py:94-224.  NavierStokes follows PAPER.md:744-816 with
the choices recorded in DESIGN.md (constant non-dimensional viscosity, BR1 on
primitive variables (u, v, w, T), Roe flux).
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigError

LAW_ADVDIFF = 0
LAW_BURGERS = 1
LAW_NS = 2


class ScalarLaw:
    nv = 1
    ngv = 1
    law_id = -1
    name = "scalar"

    def __init__(self, mu: float = 0.0):
        if mu < 0.0:
            raise ConfigError(f"viscosity must be >= 0, got {mu}")
        self.mu = float(mu)
        self.exact = None
        self.source = None

    @property
    def viscous(self) -> bool:
        return self.mu > 0.0

    @property
    def mu_cfl(self) -> float:
        return self.mu

    def with_manufactured(self, exact, source):
        self.exact = exact
        self.source = source
        return self

    def params(self) -> list[float]:
        raise NotImplementedError


class AdvectionDiffusion(ScalarLaw):
    """flux = (a, b, c) q - mu grad q, full upwinding (physics.py:49-69)."""

    name = "advection-diffusion"
    law_id = LAW_ADVDIFF

    def __init__(self, velocity=(1.0, 1.0, 0.0), mu: float = 0.0):
        super().__init__(mu)
        v = tuple(float(x) for x in velocity) + (0.0,) * (3 - len(velocity))
        self.velocity = v[:3]

    def params(self):
        return [*self.velocity, self.mu]


class ViscousBurgers(ScalarLaw):
    """flux = beta q^2/2 - mu grad q, Rusanov lambda = max|q| (physics.py:72-88)."""

    name = "viscous-burgers"
    law_id = LAW_BURGERS

    def __init__(self, mu: float = 0.0, beta=(1.0, 1.0, 0.0)):
        super().__init__(mu)
        self.beta = tuple(float(x) for x in beta)

    def params(self):
        return [*self.beta, self.mu]


class NavierStokes:
    """Compressible Navier-Stokes, q = (rho, rho u, rho v, rho w, rho E).

    Non-dimensionalised by freestream density, speed and length: p_inf =
    1/(gamma M^2), T = gamma M^2 p / rho (T_inf = 1), viscosity 1/Re,
    heat flux coefficient 1/((gamma-1) Pr M^2 Re).
    """

    nv = 5
    ngv = 4
    law_id = LAW_NS
    name = "navier-stokes"

    def __init__(self, gamma=1.4, prandtl=0.72, mach=0.3, reynolds=100.0, aoa=(0.0, 0.0)):
        if mach <= 0.0:
            raise ConfigError("Mach number must be positive")
        self.gamma = float(gamma)
        self.prandtl = float(prandtl)
        self.mach = float(mach)
        self.reynolds = float(reynolds)
        self.aoa = tuple(aoa)
        self.exact = None
        self.source = None

    @property
    def viscous(self) -> bool:
        return np.isfinite(self.reynolds) and self.reynolds > 0.0

    @property
    def mu(self) -> float:
        return 1.0 / self.reynolds if self.viscous else 0.0

    @property
    def mu_cfl(self) -> float:
        if not self.viscous:
            return 0.0
        return max(4.0 / 3.0, self.gamma / self.prandtl) / self.reynolds

    def freestream(self) -> np.ndarray:
        a, b = self.aoa
        v = np.array([np.cos(a) * np.cos(b), np.sin(a) * np.cos(b), np.sin(b)])
        p = 1.0 / (self.gamma * self.mach ** 2)
        return np.array([1.0, v[0], v[1], v[2], p / (self.gamma - 1.0) + 0.5])

    def params(self):
        re = self.reynolds if self.viscous else 0.0
        return [self.gamma, self.prandtl, self.mach, re]

    def conservative(self, rho, u, v, w, p):
        return np.stack([rho, rho * u, rho * v, rho * w,
                         p / (self.gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)])


# --- manufactured scalar cases (reference physics.py:94-224) -------------------


def _case_advdiff_sine(mu=0.1, velocity=(1.0, 1.0)):
    a, b = velocity
    pi = np.pi

    def exact(x, y, z=None):
        return np.sin(pi * x) * np.sin(pi * y)

    def source(x, y, z=None):
        sx, cx, sy, cy = np.sin(pi * x), np.cos(pi * x), np.sin(pi * y), np.cos(pi * y)
        return a * pi * cx * sy + b * pi * sx * cy + 2.0 * mu * pi * pi * sx * sy

    return AdvectionDiffusion((a, b, 0.0), mu).with_manufactured(exact, source)


def _case_burgers_tanh(mu=0.1, delta=0.25):
    def exact(x, y, z=None):
        return np.tanh((x + y - 1.0) / delta)

    def source(x, y, z=None):
        t = np.tanh((x + y - 1.0) / delta)
        s2 = 1.0 - t * t
        return 2.0 * t * s2 / delta + 4.0 * mu * t * s2 / (delta * delta)

    return ViscousBurgers(mu).with_manufactured(exact, source)


def _case_advdiff_boundary_layer(mu=0.01, delta=0.05, slope=0.5, velocity=(1.0, 0.5)):
    a, b = velocity

    def exact(x, y, z=None):
        return (1.0 + slope * x) * (1.0 - np.exp(-y / delta))

    def source(x, y, z=None):
        e = np.exp(-y / delta)
        g = 1.0 + slope * x
        return a * slope * (1.0 - e) + b * g * e / delta + mu * g * e / (delta * delta)

    return AdvectionDiffusion((a, b, 0.0), mu).with_manufactured(exact, source)


def _rational(width, center):
    def f(t):
        zz = (t - center) / width
        return 1.0 / (1.0 + zz * zz)

    def fp(t):
        zz = (t - center) / width
        return -2.0 * zz / (width * (1.0 + zz * zz) ** 2)

    def fpp(t):
        zz = (t - center) / width
        return 2.0 * (3.0 * zz * zz - 1.0) / (width * width * (1.0 + zz * zz) ** 3)

    return f, fp, fpp


def _case_advdiff_runge(mu=0.1, width=0.35, center=0.5, velocity=(1.0, 1.0)):
    a, b = velocity
    f, fp, fpp = _rational(width, center)

    def exact(x, y, z=None):
        return f(x) * f(y)

    def source(x, y, z=None):
        return (a * fp(x) * f(y) + b * f(x) * fp(y)
                - mu * (fpp(x) * f(y) + f(x) * fpp(y)))

    return AdvectionDiffusion((a, b, 0.0), mu).with_manufactured(exact, source)


def _case_advdiff_aniso(mu=0.05, width=0.3, center=0.5, slope=0.5, velocity=(1.0, 0.5)):
    a, b = velocity
    f, fp, fpp = _rational(width, center)

    def exact(x, y, z=None):
        return f(x) * (1.0 + slope * y)

    def source(x, y, z=None):
        g = 1.0 + slope * y
        return a * fp(x) * g + b * f(x) * slope - mu * fpp(x) * g

    return AdvectionDiffusion((a, b, 0.0), mu).with_manufactured(exact, source)


def _case_advdiff_poly(mu=0.1, velocity=(1.0, 1.0)):
    a, b = velocity

    def exact(x, y, z=None):
        return x * x * y + y * y + 2.0 * x

    def source(x, y, z=None):
        return a * (2.0 * x * y + 2.0) + b * (x * x + 2.0 * y) - mu * (2.0 * y + 2.0)

    return AdvectionDiffusion((a, b, 0.0), mu).with_manufactured(exact, source)


CASES = {
    "advdiff-sine": _case_advdiff_sine,
    "burgers-tanh": _case_burgers_tanh,
    "advdiff-boundary-layer": _case_advdiff_boundary_layer,
    "advdiff-runge": _case_advdiff_runge,
    "advdiff-aniso": _case_advdiff_aniso,
    "advdiff-poly": _case_advdiff_poly,
}


def make_case(name: str, **params):
    try:
        factory = CASES[name]
    except KeyError:
        raise ConfigError(f"unknown case {name!r}; known cases: {', '.join(sorted(CASES))}") from None
    try:
        return factory(**params)
    except TypeError as exc:
        raise ConfigError(f"bad parameters for case {name!r}: {exc}") from None
