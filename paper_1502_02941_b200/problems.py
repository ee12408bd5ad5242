"""Coefficient descriptors: the device-evaluable stand-in for `dgfem::ProblemSpec`
(/root/reference/proj/include/dgfem/problems.hpp:52-68).

`ProblemSpec` wraps the C struct `dgb_problem` (include/dgfem_b200.h) plus the numpy arrays
that per-element fields point into.  Two families of constructors:

* `registry_get(name)` -- the reference's built-in problems (problems.cpp:78-232) that its own
  assembly tests use (smooth-sine, smooth-sine-mixed, poly-exact,
  paper-boundary-layer-linear, pure-advection-patch), restated as descriptors;
* `config_problem(i)` -- the five BASELINE.json configurations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import Problem, ScalarField, VectorField

PI = 3.14159265358979323846


def constant(value: float) -> ScalarField:
    f = ScalarField()
    f.kind = capi.FIELD_CONSTANT
    f.value = value
    return f


def function(fn: int, p=(0.0, 0.0, 0.0, 0.0), mode: int = capi.MODE_VALUE,
             q=(0.0, 0.0, 0.0, 0.0)) -> ScalarField:
    f = ScalarField()
    f.kind = capi.FIELD_FUNCTION
    f.fn = fn
    f.mode = mode
    for i, v in enumerate(p):
        f.p[i] = v
    for i, v in enumerate(q):
        f.q[i] = v
    return f


def source_of(fn: int, p, alpha: float, eps: float, bx: float, by: float) -> ScalarField:
    """Manufactured source f = alpha u - eps lap(u) + b.grad(u) for the family (fn, p)."""
    return function(fn, p, capi.MODE_SOURCE, (alpha, eps, bx, by))


def vec_constant(bx: float, by: float) -> VectorField:
    v = VectorField()
    v.kind = capi.VEC_CONSTANT
    v.p[0], v.p[1] = bx, by
    return v


def vec_affine(c0, c1, a00, a01, a10, a11) -> VectorField:
    """b = (c0 + a00 x + a01 y, c1 + a10 x + a11 y)."""
    v = VectorField()
    v.kind = capi.VEC_AFFINE
    for i, x in enumerate((c0, c1, a00, a01, a10, a11)):
        v.p[i] = x
    return v


def vec_trig(wy: float, wx: float) -> VectorField:
    """b = (cos(wy * y), sin(wx * x))."""
    v = VectorField()
    v.kind = capi.VEC_TRIG
    v.p[0], v.p[1] = wy, wx
    return v


@dataclass
class ProblemSpec:
    """A dgb_problem plus the host arrays its per-element fields point to."""
    name: str
    c: Problem
    per_element: dict = field(default_factory=dict)  # field name -> np.ndarray [n_elements]
    neumann_sides: int = 0  # unit-square sides tagged Neumann (mesh.hpp:74 neumann_on)
    exact: tuple | None = None  # (fn, p) of the exact solution, when known
    reaction: int | None = None  # nonlinear reaction r(u) (capi.REACTION_*), when the problem has one

    def set_per_element(self, name: str, values: np.ndarray) -> None:
        values = np.ascontiguousarray(values, dtype=np.float64)
        self.per_element[name] = values
        f = getattr(self.c, name)
        f.kind = capi.FIELD_PER_ELEMENT
        f.per_element = values.ctypes.data


def make_problem(name, eps, b, alpha, source, dirichlet, neumann=None, neumann_sides=0,
                 exact=None) -> ProblemSpec:
    p = Problem()
    p.diffusion = constant(eps) if isinstance(eps, (int, float)) else eps
    p.advection = b
    p.linear_reaction = constant(alpha) if isinstance(alpha, (int, float)) else alpha
    p.source = source
    p.dirichlet = dirichlet
    p.neumann = neumann if neumann is not None else constant(0.0)
    return ProblemSpec(name, p, neumann_sides=neumann_sides, exact=exact)


# ----------------------------------------------------------------------------- registry
def registry_get(name: str) -> ProblemSpec:
    """Descriptor twins of the reference registry (problems.cpp:197-221)."""
    if name in ("smooth-sine", "smooth-sine-mixed"):
        # problems.cpp:136-164: eps = 1, b = (1, 2), alpha = 1, u = sin(pi x) sin(pi y)
        u = (capi.FN_SIN_SIN, (1.0,))
        return make_problem(
            name, 1.0, vec_constant(1.0, 2.0), 1.0,
            source_of(*u, alpha=1.0, eps=1.0, bx=1.0, by=2.0),
            function(*u),
            neumann=function(capi.FN_SIN_SIN, (1.0,), capi.MODE_FLUX_X, (0.0, 1.0)),
            neumann_sides=2 if name == "smooth-sine-mixed" else 0, exact=u)
    if name == "poly-exact":
        # problems.cpp:166-180: u = 1 + 2x + 3y, f = 9 + 2x + 3y
        u = (capi.FN_AFFINE, (1.0, 2.0, 3.0))
        return make_problem(name, 1.0, vec_constant(1.0, 2.0), 1.0,
                            function(capi.FN_AFFINE, (9.0, 2.0, 3.0)), function(*u), exact=u)
    if name == "paper-boundary-layer-linear":
        # problems.cpp:78-134: eps = 1e-6, b = (1, 2)/sqrt(5), alpha = 1,
        # u = 0.5 (1 - tanh((2x - y - 0.25) / sqrt(5 eps)))
        eps = 1e-6
        b1, b2 = 1.0 / math.sqrt(5.0), 2.0 / math.sqrt(5.0)
        u = (capi.FN_TANH_LAYER, (2.0, -1.0, -0.25, math.sqrt(5.0 * eps)))
        return make_problem(name, eps, vec_constant(b1, b2), 1.0,
                            source_of(*u, alpha=1.0, eps=eps, bx=b1, by=b2), function(*u),
                            exact=u)
    if name == "paper-boundary-layer":
        # problems.cpp:78-134 (nonlinear = true): the layer above with r(u) = u^2 (r' = 2u) and
        # f += u^2; the reaction is applied by the Newton driver (ProblemSpec.reaction)
        eps = 1e-6
        b1, b2 = 1.0 / math.sqrt(5.0), 2.0 / math.sqrt(5.0)
        u = (capi.FN_TANH_LAYER, (2.0, -1.0, -0.25, math.sqrt(5.0 * eps)))
        spec = make_problem(name, eps, vec_constant(b1, b2), 1.0,
                            function(*u, mode=capi.MODE_SOURCE_SQUARE, q=(1.0, eps, b1, b2)),
                            function(*u), exact=u)
        spec.reaction = capi.REACTION_SQUARE
        return spec
    if name == "pure-advection-patch":
        # problems.cpp:182-193
        return make_problem(name, 1e-10, vec_constant(1.0, 0.0), 0.0, constant(0.0),
                            function(capi.FN_STEP_Y, (0.5, 1.0, 0.0)))
    raise KeyError(f"unknown problem {name!r}")


# ----------------------------------------------------------------------------- configs
# Seeds are not given by BASELINE.json; these are fixed here and recorded in DESIGN.md.
SEED_JITTER = 0x5EED0003
SEED_PERMUTE = 0x5EED0004
SEED_SPMV_X = 0x5EED0044
SEED_COEF = 0x5EED0005


@dataclass(frozen=True)
class Config:
    index: int
    n: int              # cells per side
    degree: int
    quad_order: int     # 2k+1: k+1 edge points, volume rule exact to >= 2k
    methods: tuple      # (dgb_method, ...)
    sigma: float        # sigma_interior override (sigma_boundary = 2 sigma)
    jitter: float = 0.0
    permute: bool = False
    neumann_sides: int = 0
    neumann_inflow: int = capi.INFLOW_ERROR

    @property
    def n_elements(self) -> int:
        return 2 * self.n * self.n

    @property
    def name(self) -> str:
        return f"C{self.index}"


CONFIGS = {
    1: Config(1, 32, 1, 3, (capi.SIPG,), 6.0),
    2: Config(2, 256, 2, 5, (capi.SIPG, capi.NIPG, capi.IIPG), 18.0),
    3: Config(3, 1024, 3, 7, (capi.SIPG,), 36.0, jitter=0.2, neumann_sides=2 | 8,
              neumann_inflow=capi.INFLOW_DROP),
    4: Config(4, 2048, 1, 3, (capi.SIPG,), 6.0, permute=True),
    5: Config(5, 512, 4, 9, (capi.IIPG,), 60.0),
}


def splitmix64(state: int):
    """The generator behind every seeded input (same as csrc/host/mesh.cpp)."""
    mask = (1 << 64) - 1
    while True:
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        yield z ^ (z >> 31)


def uniform01(seed: int, n: int) -> np.ndarray:
    """n doubles in [0,1): (splitmix64 >> 11) * 2^-53, vectorised in numpy."""
    mask = np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = (np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)) & mask
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def config_problem(index: int, n_elements: int | None = None) -> ProblemSpec:
    """Coefficients of BASELINE.json config `index` (1..5).  Config 5's per-element eps_K and
    alpha_K need the element count (it defaults to the config's own mesh)."""
    if index == 1:
        u = (capi.FN_SIN_SIN, (1.0,))
        return make_problem("C1", 1e-2, vec_constant(1.0, 1.0), 1.0,
                            source_of(*u, alpha=1.0, eps=1e-2, bx=1.0, by=1.0), function(*u),
                            exact=u)
    if index == 2:
        eps = 1e-4
        b = 1.0 / math.sqrt(2.0)
        u = (capi.FN_TANH_LAYER, (1.0, -1.0, -0.25, math.sqrt(eps)))
        return make_problem("C2", eps, vec_constant(b, b), 1.0,
                            source_of(*u, alpha=1.0, eps=eps, bx=b, by=b), function(*u),
                            exact=u)
    if index == 3:
        # b = (-(y - 1/2), x - 1/2); Neumann on x = 1 and y = 1 (outflow-only convention)
        return make_problem("C3", 1e-3, vec_affine(0.5, -0.5, 0.0, -1.0, 1.0, 0.0), 1.0,
                            constant(1.0), constant(0.0), constant(0.0), neumann_sides=2 | 8)
    if index == 4:
        u = (capi.FN_GAUSSIAN, (50.0, 0.5, 0.5))
        return make_problem("C4", 1e-2, vec_constant(1.0, 0.5), 1.0,
                            source_of(*u, alpha=1.0, eps=1e-2, bx=1.0, by=0.5), function(*u),
                            exact=u)
    if index == 5:
        ne = n_elements if n_elements is not None else CONFIGS[5].n_elements
        spec = make_problem("C5", 1.0, vec_trig(2.0 * PI, 2.0 * PI), 1.0, constant(1.0),
                            constant(0.0))
        r = uniform01(SEED_COEF, 2 * ne)
        spec.set_per_element("diffusion", 10.0 ** (-6.0 + 6.0 * r[:ne]))   # log-U[1e-6, 1]
        spec.set_per_element("linear_reaction", 2.0 * r[ne:])              # U[0, 2]
        return spec
    raise KeyError(index)
