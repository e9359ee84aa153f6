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


@_tag(_lib.FORCING_ANNULUS_3D)
def annulus_solution_3d(x):
    """The 2-D annulus solution times sin(pi z) (prism over the annulus)."""
    return annulus_solution_2d(x) * np.sin(np.pi * x[..., 2])


@_tag(_lib.FORCING_ANNULUS_3D)
def annulus_gradient_3d(x):
    sz, cz = np.sin(np.pi * x[..., 2]), np.cos(np.pi * x[..., 2])
    g = annulus_gradient_2d(x)
    return np.stack([g[..., 0] * sz, g[..., 1] * sz, np.pi * cz * annulus_solution_2d(x)], axis=-1)


@_tag(_lib.FORCING_ANNULUS_3D)
def annulus_forcing_3d(x):
    # -Lap(u2 sin(pi z)) = (f2 + pi^2 u2) sin(pi z)
    return (annulus_forcing_2d(x) + np.pi**2 * annulus_solution_2d(x)) * np.sin(np.pi * x[..., 2])


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

    if d == 2:
        sol, grad, forc = annulus_solution_2d, annulus_gradient_2d, annulus_forcing_2d
    elif d == 3:
        sol, grad, forc = annulus_solution_3d, annulus_gradient_3d, annulus_forcing_3d
    else:
        raise ValueError(f"regular annulus problem needs d in (2, 3), got {d}")
    return BenchmarkProblem(
        f"regular_annulus_{d}d", quarter_annulus(d), forc, degree,
        degree - 1 if regularity is None else regularity, grading, sol, grad)


def constant_forcing_problem(d, grading=1.0, degree=3, regularity=None) -> BenchmarkProblem:
    """Quarter annulus with unit forcing, no closed form (reference
    analysis.py:192-205): errors need the overkill reference."""
    from .geometry import quarter_annulus

    if d not in (2, 3):
        raise ValueError(f"constant forcing problem needs d in (2, 3), got {d}")
    return BenchmarkProblem(
        f"constant_forcing_{d}d", quarter_annulus(d), constant_one, degree,
        degree - 1 if regularity is None else regularity, grading)


def polynomial_cube_problem(d, degree=2, regularity=None) -> BenchmarkProblem:
    """Reference analysis.py:199-212."""
    from .geometry import unit_hypercube

    return BenchmarkProblem(
        f"polynomial_cube_{d}d", unit_hypercube(d), cube_forcing, degree,
        degree - 1 if regularity is None else regularity, 1.0, cube_solution, cube_gradient)


class Evaluator:
    """A field the device error quadrature understands (reference
    analysis.py:226-259 returns closures; here they are descriptors):
    kind "analytic" (registered closed form), "spline" (one space +
    coefficients) or "combined" (plan + component solutions)."""

    def __init__(self, kind, **payload):
        self.kind = kind
        self.payload = payload

    def __call__(self, grid):
        raise TypeError("device evaluators are consumed by analysis.error_norms")

    def fields(self):
        """[(space, coefficients, weight), ...] in accumulation order."""
        if self.kind == "spline":
            return [(self.payload["space"], self.payload["coeffs"], 1.0)]
        if self.kind == "combined":
            from .combination import _lookup

            lookup = _lookup(self.payload["components"])
            out = []
            for beta, c in self.payload["plan"].terms:
                if beta not in lookup:
                    raise KeyError(f"no component solution supplied for index {beta}")
                s = lookup[beta]
                out.append((s.space, s.coefficients, float(c)))
            return out
        return []


def analytic_evaluator(solution, gradient):
    """Closed-form solution (must carry a device registry id)."""
    return Evaluator("analytic", solution=solution, gradient=gradient)


def spline_evaluator(space, coeffs):
    return Evaluator("spline", space=space, coeffs=coeffs)


def combined_evaluator(plan, components):
    return Evaluator("combined", plan=plan, components=components)


def _evaluator_error_norms(solution_eval, reference_eval, grid):
    """||a - b|| (L2, H1 seminorm) for two evaluators on a QuadGrid, one
    device pass: the spline / combined fields of both sides go into one
    handle as a signed term list, a closed-form side becomes the kernel's
    solution (reference analysis.py:262-270)."""
    from .assembly import space_batch

    sid = None
    terms = []   # (space, coeffs, weight)
    for ev, sign in ((solution_eval, 1.0), (reference_eval, -1.0)):
        if not isinstance(ev, Evaluator):
            raise TypeError("error_norms expects evaluators from analytic/spline/combined_evaluator")
        if ev.kind == "analytic":
            if sid is not None:
                raise ValueError("at most one closed-form side")
            sid = solution_id_of(ev.payload["solution"])
            if sid is None:
                raise ValueError("closed-form solution not registered on the device")
            sign_analytic = sign
            continue
        terms += [(s, c, sign * w) for s, c, w in ev.fields()]
    if not terms:
        raise ValueError("nothing to integrate")
    if sid is not None and sign_analytic > 0:   # ||u - f|| = ||f - u||
        terms = [(s, c, -w) for s, c, w in terms]
    batch = space_batch([(s, 1) for s, _, _ in terms], patch=grid.patch)
    try:
        batch.set_coefficients(np.concatenate([np.asarray(c, dtype=np.float64).ravel() for _, c, _ in terms]))
        return batch.subset_error_norms(grid.points_per_dir, grid.weights_per_dir,
                                        [(i, w) for i, (_, _, w) in enumerate(terms)], sid)
    finally:
        batch.close()


def error_norms(*args):
    """(L2 error, H1-seminorm error).  Two forms:

    * ``error_norms(solution_eval, reference_eval, grid)`` -- the reference
      signature (analysis.py:262-270) with the evaluators above;
    * ``error_norms(plan, components, problem, grid)`` -- the combined
      solution against the problem's closed form, one device pass reusing
      the components' own handle when possible.
    """
    if len(args) == 3:
        return _evaluator_error_norms(*args)
    plan, components, problem, grid = args
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


# study drivers (reference analysis.py:273-528), batched on the device
from .studies import (ConvergenceRecord, GammaSweepRow, convergence_study, fit_rate,  # noqa: E402
                      gamma_sweep, read_convergence_csv, write_convergence_csv, write_gamma_csv)

__all__ += [
    "annulus_solution_3d", "annulus_forcing_3d", "annulus_gradient_3d", "constant_forcing_problem",
    "Evaluator", "analytic_evaluator", "spline_evaluator", "combined_evaluator", "error_norms",
    "fit_rate", "ConvergenceRecord", "convergence_study", "write_convergence_csv", "read_convergence_csv",
    "GammaSweepRow", "gamma_sweep", "write_gamma_csv",
]
