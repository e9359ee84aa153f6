"""Benchmark problems, the device forcing registry, and GPU error norms.

* ``BenchmarkProblem`` mirrors reference analysis.py:52-77.
* Closed forms: the reference's own (analysis.py:83-167) plus the
  BASELINE configurations' manufactured solutions.
  Each numpy callable carries ``sgiga_id``, the device registry id of the
  same closed form (include/sgiga.h enum sgiga_forcing); reference callables
  are recognised by qualified name.  Unknown callables are evaluated on the
  host at device-computed physical quadrature points.
* ``error_norms`` replaces analysis.error_norms(combined_evaluator,
  analytic_evaluator, QuadGrid) (analysis.py:226-270) with one device pass.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib

__all__ = [
    "BenchmarkProblem",
    "forcing_id_of",
    "solution_id_of",
    "sin_product_solution", "sin_product_forcing", "sin_product_gradient",
    "annulus_polar_solution", "annulus_polar_forcing", "annulus_polar_gradient",
    "exp_bubble_solution", "exp_bubble_forcing", "exp_bubble_gradient",
    "cube_solution", "cube_forcing", "cube_gradient",
    "annulus_solution_2d", "annulus_forcing_2d", "annulus_gradient_2d",
    "constant_one", "lshape_solution", "lshape_gradient", "zero_forcing",
    "regular_annulus_problem", "polynomial_cube_problem",
]


@dataclass(frozen=True)
class BenchmarkProblem:
    """Poisson problem: patch, forcing, degree/regularity/grading (+ exact u)."""

    name: str
    patch: object
    forcing: Callable
    degree: int
    regularity: int
    grading: float = 1.0
    solution: Callable | None = None
    solution_gradient: Callable | None = None

    def __post_init__(self):
        if self.degree < 1:
            raise ValueError(f"degree must be >= 1, got {self.degree}")
        if not -1 <= self.regularity <= self.degree - 1:
            raise ValueError(f"regularity {self.regularity} invalid for degree {self.degree}")
        if self.grading < 1.0:
            raise ValueError(f"grading must be >= 1, got {self.grading}")


def _tag(fid):
    def deco(fn):
        fn.sgiga_id = fid
        return fn
    return deco


# ---- manufactured solutions of the BASELINE configs --------------------------
@_tag(_lib.FORCING_SIN_PRODUCT)
def sin_product_solution(x):
    return np.prod(np.sin(np.pi * x), axis=-1)


@_tag(_lib.FORCING_SIN_PRODUCT)
def sin_product_forcing(x):
    d = x.shape[-1]
    return (d * np.pi**2) * sin_product_solution(x)


@_tag(_lib.FORCING_SIN_PRODUCT)
def sin_product_gradient(x):
    s, c = np.sin(np.pi * x), np.cos(np.pi * x)
    out = np.empty_like(x)
    for m in range(x.shape[-1]):
        out[..., m] = np.pi * c[..., m] * np.prod(np.delete(s, m, axis=-1), axis=-1)
    return out


@_tag(_lib.FORCING_ANNULUS_POLAR)
def annulus_polar_solution(x):
    xx, yy = x[..., 0], x[..., 1]
    s = xx * xx + yy * yy
    return 2.0 * xx * yy * (s - 5.0 + 4.0 / s)


@_tag(_lib.FORCING_ANNULUS_POLAR)
def annulus_polar_forcing(x):
    xx, yy = x[..., 0], x[..., 1]
    s = xx * xx + yy * yy
    return 32.0 * xx * yy / (s * s) - 24.0 * xx * yy


@_tag(_lib.FORCING_ANNULUS_POLAR)
def annulus_polar_gradient(x):
    xx, yy = x[..., 0], x[..., 1]
    s = xx * xx + yy * yy
    h, hp = s - 5.0 + 4.0 / s, 1.0 - 4.0 / (s * s)
    return np.stack([2.0 * yy * h + 4.0 * xx * xx * yy * hp, 2.0 * xx * h + 4.0 * xx * yy * yy * hp], axis=-1)


@_tag(_lib.FORCING_EXP_BUBBLE)
def exp_bubble_solution(x):
    return np.exp(x.sum(axis=-1)) * np.prod(x * (1.0 - x), axis=-1)


@_tag(_lib.FORCING_EXP_BUBBLE)
def exp_bubble_forcing(x):
    b = x * (1.0 - x)
    tot = np.zeros(x.shape[:-1])
    for m in range(x.shape[-1]):
        tot = tot + x[..., m] * (x[..., m] + 3.0) * np.prod(np.delete(b, m, axis=-1), axis=-1)
    return np.exp(x.sum(axis=-1)) * tot


@_tag(_lib.FORCING_EXP_BUBBLE)
def exp_bubble_gradient(x):
    b = x * (1.0 - x)
    e = np.exp(x.sum(axis=-1))
    out = np.empty_like(x)
    for m in range(x.shape[-1]):
        out[..., m] = e * (b[..., m] + 1.0 - 2.0 * x[..., m]) * np.prod(np.delete(b, m, axis=-1), axis=-1)
    return out


# ---- the reference's own closed forms (analysis.py:83-167) -------------------
@_tag(_lib.FORCING_CUBE_POLY)
def cube_solution(x):
    return np.prod(x * (1.0 - x), axis=-1)


@_tag(_lib.FORCING_CUBE_POLY)
def cube_forcing(x):
    b = x * (1.0 - x)
    return sum(2.0 * np.prod(np.delete(b, m, axis=-1), axis=-1) for m in range(x.shape[-1]))


@_tag(_lib.FORCING_CUBE_POLY)
def cube_gradient(x):
    b = x * (1.0 - x)
    out = np.empty_like(x)
    for m in range(x.shape[-1]):
        out[..., m] = (1.0 - 2.0 * x[..., m]) * np.prod(np.delete(b, m, axis=-1), axis=-1)
    return out


@_tag(_lib.FORCING_ANNULUS_2D)
def annulus_solution_2d(x):
    xx, yy = x[..., 0], x[..., 1]
    r2 = xx**2 + yy**2
    return -(r2 - 1.0) * (r2 - 4.0) * xx * yy**2


@_tag(_lib.FORCING_ANNULUS_2D)
def annulus_forcing_2d(x):
    xx, yy = x[..., 0], x[..., 1]
    return 2.0 * xx * (xx**4 + 22.0 * xx**2 * yy**2 - 5.0 * xx**2 + 21.0 * yy**4 - 45.0 * yy**2 + 4.0)


@_tag(_lib.FORCING_ANNULUS_2D)
def annulus_gradient_2d(x):
    xx, yy = x[..., 0], x[..., 1]
    gx = -5 * xx**4 * yy**2 - 6 * xx**2 * yy**4 + 15 * xx**2 * yy**2 - yy**6 + 5 * yy**4 - 4 * yy**2
    gy = -2 * xx**5 * yy - 8 * xx**3 * yy**3 + 10 * xx**3 * yy - 6 * xx * yy**5 + 20 * xx * yy**3 - 8 * xx * yy
    return np.stack([gx, gy], axis=-1)


@_tag(_lib.FORCING_CONSTANT_ONE)
def constant_one(x):
    return np.ones(x.shape[0])


@_tag(_lib.FORCING_ZERO)
def zero_forcing(x):
    return np.zeros(x.shape[0])


@_tag(_lib.FORCING_LSHAPE)
def lshape_solution(x):
    r = np.hypot(x[..., 0], x[..., 1])
    th = np.mod(np.arctan2(x[..., 1], x[..., 0]), 2.0 * np.pi)
    return r ** (2.0 / 3.0) * np.sin(2.0 * th / 3.0)


@_tag(_lib.FORCING_LSHAPE)
def lshape_gradient(x):
    r = np.hypot(x[..., 0], x[..., 1])
    th = np.mod(np.arctan2(x[..., 1], x[..., 0]), 2.0 * np.pi)
    with np.errstate(divide="ignore", invalid="ignore"):
        rr = r ** (2.0 / 3.0)
        dr = (2.0 / 3.0) * rr / r * np.sin(2.0 * th / 3.0)
        dth = rr * (2.0 / 3.0) * np.cos(2.0 * th / 3.0)
        gx = dr * np.cos(th) - dth * np.sin(th) / r
        gy = dr * np.sin(th) + dth * np.cos(th) / r
    return np.stack([np.where(r > 0, gx, 0.0), np.where(r > 0, gy, 0.0)], axis=-1)


# reference callables recognised by qualified name (sparseiga/analysis.py)
_REFERENCE_NAMES = {
    "annulus_forcing_2d": _lib.FORCING_ANNULUS_2D,
    "annulus_solution_2d": _lib.FORCING_ANNULUS_2D,
    "annulus_forcing_3d": _lib.FORCING_ANNULUS_3D,
    "annulus_solution_3d": _lib.FORCING_ANNULUS_3D,
    "cube_forcing": _lib.FORCING_CUBE_POLY,
    "cube_solution": _lib.FORCING_CUBE_POLY,
    "constant_one": _lib.FORCING_CONSTANT_ONE,
}


def forcing_id_of(fn) -> int:
    """Device registry id of a forcing callable, or FORCING_HOST."""
    if fn is None:
        return _lib.FORCING_ZERO
    fid = getattr(fn, "sgiga_id", None)
    if fid is not None:
        return int(fid)
    if getattr(fn, "__module__", "") == "sparseiga.analysis":
        return _REFERENCE_NAMES.get(getattr(fn, "__qualname__", ""), _lib.FORCING_HOST)
    return _lib.FORCING_HOST


def solution_id_of(fn) -> int | None:
    fid = forcing_id_of(fn)
    return None if fid in (_lib.FORCING_HOST, _lib.FORCING_ZERO, _lib.FORCING_CONSTANT_ONE) else fid


def regular_annulus_problem(d=2, degree=2, regularity=None, grading=1.0) -> BenchmarkProblem:
    """Reference analysis.py:155-176 (2-D variant)."""
    from .geometry import quarter_annulus

    if d != 2:
        raise ValueError("only the 2-D annulus closed form is registered")
    return BenchmarkProblem(
        f"regular_annulus_{d}d", quarter_annulus(d), annulus_forcing_2d, degree,
        degree - 1 if regularity is None else regularity, grading,
        annulus_solution_2d, annulus_gradient_2d)


def polynomial_cube_problem(d, degree=2, regularity=None) -> BenchmarkProblem:
    """Reference analysis.py:199-212."""
    from .geometry import unit_hypercube

    return BenchmarkProblem(
        f"polynomial_cube_{d}d", unit_hypercube(d), cube_forcing, degree,
        degree - 1 if regularity is None else regularity, 1.0, cube_solution, cube_gradient)


def error_norms(plan, components, problem, grid):
    """(L2 error, H1-seminorm error) of the combined solution against the
    problem's closed-form solution on ``grid`` -- one device pass replacing
    error_norms(combined_evaluator(plan, comps), analytic_evaluator(u, grad u),
    QuadGrid) (reference analysis.py:226-270)."""
    from .combination import _combine_batch

    sid = solution_id_of(problem.solution)
    if sid is None:
        raise ValueError("error_norms on the device needs a registered closed-form solution")
    batch, owned = _combine_batch(plan, components, patch=problem.patch)
    try:
        return batch.error_norms(grid.points_per_dir, grid.weights_per_dir, sid)
    finally:
        if owned:
            batch.close()
