"""Combination plans, component solutions and the combine step.

* ``CombinationPlan`` / ``simplex_set`` / ``combination_coefficients`` /
  ``is_downward_closed`` / ``general_coefficients``: host integer logic,
  bit-exact with the reference (combination.py:48-159).
* ``baseline_plan``: BASELINE's "i_k >= 1" sets = the reference simplex
  plan shifted by +1.
* ``ComponentSolution`` / ``solve_component`` (163-200) and
  ``evaluate_combined`` (209-236) run on the device; the scattered-point
  ``evaluate_combined_points`` replaces the reference's per-point idiom
  (tests/test_acceptance.py:224-230).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from math import comb

import numpy as np

__all__ = [
    "CombinationPlan", "ComponentSolution", "simplex_set", "combination_coefficients",
    "is_downward_closed", "general_coefficients", "baseline_plan", "solve_component",
    "evaluate_combined", "evaluate_combined_points",
]


@dataclass(frozen=True)
class CombinationPlan:
    """Lexicographically sorted (beta, integer coefficient) terms summing to 1."""

    d: int
    terms: tuple
    level: int | None = None

    def __post_init__(self):
        terms = tuple((tuple(int(b) for b in beta), int(c)) for beta, c in self.terms)
        if not terms:
            raise ValueError("a combination plan needs at least one term")
        seen = set()
        for beta, c in terms:
            if len(beta) != self.d:
                raise ValueError(f"index {beta} does not have {self.d} entries")
            if min(beta) < 0:
                raise ValueError(f"negative level in index {beta}")
            if c == 0:
                raise ValueError(f"zero coefficient stored for {beta}")
            if beta in seen:
                raise ValueError("duplicate indices in plan")
            seen.add(beta)
        terms = tuple(sorted(terms))
        total = sum(c for _, c in terms)
        if total != 1:
            raise ValueError(f"plan coefficients sum to {total}, expected 1")
        object.__setattr__(self, "terms", terms)

    @property
    def betas(self) -> list:
        return [b for b, _ in self.terms]

    @property
    def coefficients(self) -> dict:
        return dict(self.terms)

    def __len__(self) -> int:
        return len(self.terms)


def simplex_set(d: int, level: int) -> list:
    if d < 1:
        raise ValueError(f"dimension must be >= 1, got {d}")
    if level < 0:
        raise ValueError(f"level must be >= 0, got {level}")
    return sorted(b for b in itertools.product(range(level + 1), repeat=d) if sum(b) <= level)


def combination_coefficients(d: int, level: int) -> CombinationPlan:
    """(-1)^t C(d-1, t) on the top d layers t = level - |beta| in {0..d-1}."""
    terms = [(b, (-1) ** (level - sum(b)) * comb(d - 1, level - sum(b)))
             for b in simplex_set(d, level) if level - sum(b) <= d - 1]
    return CombinationPlan(d, tuple(terms), level=level)


def is_downward_closed(index_set) -> bool:
    members = {tuple(b) for b in index_set}
    return all(beta[:k] + (beta[k] - 1,) + beta[k + 1:] in members
               for beta in members for k in range(len(beta)) if beta[k] > 0)


def general_coefficients(index_set) -> CombinationPlan:
    """Signed count of binary upward shifts inside a downward-closed set."""
    betas = sorted({tuple(int(b) for b in beta) for beta in index_set})
    if not betas:
        raise ValueError("index set is empty")
    d = len(betas[0])
    if any(len(b) != d for b in betas):
        raise ValueError("index set mixes dimensions")
    if any(x < 0 for b in betas for x in b):
        raise ValueError("index set contains negative levels")
    if not is_downward_closed(betas):
        raise ValueError("index set is not downward closed")
    members = set(betas)
    terms = []
    for beta in betas:
        c = sum((-1) ** sum(k) for k in itertools.product((0, 1), repeat=d)
                if tuple(b + kk for b, kk in zip(beta, k)) in members)
        if c:
            terms.append((beta, c))
    return CombinationPlan(d, tuple(terms))


def baseline_plan(d: int, w: int) -> CombinationPlan:
    """BASELINE plan: i_k >= 1, w-d+1 <= |i| <= w, c = (-1)^{w-|i|} C(d-1, w-|i|)."""
    base = combination_coefficients(d, w - d)
    return CombinationPlan(d, tuple((tuple(b + 1 for b in beta), c) for beta, c in base.terms), level=w)


@dataclass
class ComponentSolution:
    """Solution on one component space; ``coefficients`` are full C order."""

    beta: tuple
    space: object
    coefficients: np.ndarray
    solve_time: float
    _batch: object = field(default=None, repr=False, compare=False)
    _index: int = field(default=-1, repr=False, compare=False)

    @property
    def n_dofs(self) -> int:
        return self.space.n_dofs

    def eval_grid(self, points_per_dir, gradient=False):
        b = self._batch
        if b is not None and getattr(b, "h", None):
            return b.combine_grid(points_per_dir, gradient=gradient, comp=self._index)
        return self.space.eval_grid(self.coefficients, points_per_dir, gradient)


def solve_component(problem, beta, quad_points=None) -> ComponentSolution:
    """One-term batch of run_plan (reference combination.py:183-200)."""
    from .scheduler import solve_terms

    sols, _ = solve_terms(((tuple(int(b) for b in beta), 1),), problem, quad_points)
    return sols[0]


def _lookup(components) -> dict:
    if isinstance(components, dict):
        return {tuple(k): v for k, v in components.items()}
    return {tuple(c.beta): c for c in components}


def _combine_batch(plan, components, patch=None):
    """A device handle holding the plan's components (reused when possible)."""
    from .assembly import space_batch

    lookup = _lookup(components)
    chosen = []
    for beta, c in plan.terms:
        if beta not in lookup:
            raise KeyError(f"no component solution supplied for index {beta}")
        chosen.append((lookup[beta], c))
    first = chosen[0][0]
    b = getattr(first, "_batch", None)
    if (b is not None and getattr(b, "h", None) and len(b.spec.terms) == len(chosen)
            and all(getattr(s, "_batch", None) is b and s._index == i for i, (s, _) in enumerate(chosen))
            and tuple(c for _, c in b.spec.terms) == tuple(c for _, c in chosen)
            and (patch is None or b.spec.patch is patch)):
        return b, False
    batch = space_batch([(s.space, c) for s, c in chosen], patch=patch)
    batch.set_coefficients(np.concatenate([np.asarray(s.coefficients, dtype=np.float64).ravel()
                                           for s, _ in chosen]))
    return batch, True


def evaluate_combined(plan, components, points_per_dir, gradient=False):
    """Plan-order signed sum on a tensor grid (deterministic, device)."""
    batch, owned = _combine_batch(plan, components)
    try:
        return batch.combine_grid(points_per_dir, gradient=gradient, comp=-1)
    finally:
        if owned:
            batch.close()


def evaluate_combined_points(plan, components, points) -> np.ndarray:
    """Combined solution at scattered parametric points (n, d)."""
    batch, owned = _combine_batch(plan, components)
    try:
        return batch.combine_points(np.asarray(points, dtype=np.float64))
    finally:
        if owned:
            batch.close()


# surplus / profit (reference combination.py:239-302), batched on the device
from .studies import ProfitRow, profit_table, surplus_norm  # noqa: E402,F401
