"""Host-side knot vectors (exact metadata only; no basis evaluation here).

The device rebuilds the open knot vector from breakpoints and evaluates all
basis functions; the host only produces the breakpoints, with the same
numpy expressions as the reference so they are bitwise identical:

* ``KnotVector``            -- reference splines.py:25-80
* ``make_open_knot_vector`` -- splines.py:83-110
* ``grade_point``           -- splines.py:113-130
* ``dyadic_level_knots``    -- splines.py:133-146
* ``one_sided_level_knots`` -- BASELINE cfg4 radical grading x_j = (j/n)^gamma
  toward one end (not in the reference)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "KnotVector",
    "make_open_knot_vector",
    "grade_point",
    "dyadic_level_knots",
    "one_sided_level_knots",
]


@dataclass(frozen=True)
class KnotVector:
    """Open knot vector on [0, 1] with its degree (validated like the reference)."""

    degree: int
    knots: np.ndarray
    breakpoints: np.ndarray = field(init=False, repr=False, compare=False)
    multiplicities: np.ndarray = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        p = int(self.degree)
        if p < 1:
            raise ValueError(f"degree must be >= 1, got {p}")
        k = np.ascontiguousarray(self.knots, dtype=np.float64)
        if k.ndim != 1 or k.size < 2 * (p + 1):
            raise ValueError("knot vector too short for an open vector")
        if np.any(np.diff(k) < 0):
            raise ValueError("knots must be nondecreasing")
        if k[0] != 0.0 or k[-1] != 1.0:
            raise ValueError("knot vector must span [0, 1]")
        uniq, counts = np.unique(k, return_counts=True)
        if counts[0] != p + 1 or counts[-1] != p + 1:
            raise ValueError("end knots must have multiplicity degree + 1")
        if uniq.size > 2 and counts[1:-1].max() > p + 1:
            raise ValueError("interior knot multiplicity exceeds degree + 1")
        object.__setattr__(self, "degree", p)
        object.__setattr__(self, "knots", k)
        object.__setattr__(self, "breakpoints", uniq)
        object.__setattr__(self, "multiplicities", counts)

    @property
    def n(self) -> int:
        return self.knots.size - self.degree - 1

    @property
    def n_elements(self) -> int:
        return self.breakpoints.size - 1

    @property
    def interior_multiplicity(self) -> int | None:
        """Common multiplicity of the interior breakpoints (None if none / mixed)."""
        inner = self.multiplicities[1:-1]
        if inner.size == 0 or np.any(inner != inner[0]):
            return None
        return int(inner[0])

    def element_spans(self) -> np.ndarray:
        k = self.knots
        return np.nonzero(k[:-1] < k[1:])[0]

    def element_offsets(self) -> np.ndarray:
        return self.element_spans() - self.degree


def make_open_knot_vector(degree, breakpoints, regularity) -> KnotVector:
    """Open vector over ``breakpoints`` with interior multiplicity degree - regularity."""
    p, r = int(degree), int(regularity)
    if p < 1:
        raise ValueError(f"degree must be >= 1, got {p}")
    if not -1 <= r <= p - 1:
        raise ValueError(f"regularity must be in [-1, {p - 1}], got {r}")
    b = np.asarray(breakpoints, dtype=np.float64)
    if b.ndim != 1 or b.size < 2:
        raise ValueError("need at least two breakpoints")
    if np.any(np.diff(b) <= 0):
        raise ValueError("breakpoints must be strictly increasing")
    if b[0] != 0.0 or b[-1] != 1.0:
        raise ValueError("breakpoints must start at 0 and end at 1")
    inner = np.repeat(b[1:-1], p - r)
    return KnotVector(p, np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)]))


def grade_point(t, gamma):
    """Symmetric radical grading of [0, 1] (same float expressions as the reference)."""
    if gamma < 1.0:
        raise ValueError(f"grading exponent must be >= 1, got {gamma}")
    t = np.asarray(t, dtype=np.float64)
    if np.any(t < 0.0) or np.any(t > 1.0):
        raise ValueError("grading input must lie in [0, 1]")
    scale = 2.0 ** (gamma - 1.0)
    graded = np.where(t <= 0.5, scale * t**gamma, 1.0 - scale * (1.0 - t) ** gamma)
    return float(graded) if graded.ndim == 0 else graded


def dyadic_level_knots(level, degree, regularity, grading=1.0) -> KnotVector:
    """2**level graded elements on [0, 1]; exact endpoints."""
    lv = int(level)
    if lv < 0:
        raise ValueError(f"level must be >= 0, got {lv}")
    b = grade_point(np.linspace(0.0, 1.0, 2**lv + 1), grading)
    b[0], b[-1] = 0.0, 1.0
    return make_open_knot_vector(degree, b, regularity)


def one_sided_level_knots(level, degree, regularity, gamma=3.0, toward="low") -> KnotVector:
    """2**level elements with breakpoints (j/n)**gamma graded toward one end.

    ``toward="high"`` mirrors them, 1 - ((n-j)/n)**gamma, which is exact in
    FP64 for n = 2**level (level <= 17).
    """
    n = 2 ** int(level)
    j = np.arange(n + 1, dtype=np.float64)
    if toward == "low":
        b = (j / n) ** gamma
    elif toward == "high":
        b = 1.0 - ((n - j) / n) ** gamma
    else:
        raise ValueError("toward must be 'low' or 'high'")
    b[0], b[-1] = 0.0, 1.0
    return make_open_knot_vector(degree, b, regularity)
