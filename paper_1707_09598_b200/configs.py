"""The five BASELINE.json configurations as (problem, plan, points, grid).

Inputs are synthetic and fully defined by SURVEY.md section 8(d): random
evaluation points come from ``np.random.default_rng(seed).random((N, d))``;
cfg3-5 points and all error grids are the survey's proposals (BASELINE.json
does not specify them).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import analysis as A
from .assembly import QuadGrid
from .combination import CombinationPlan, baseline_plan
from .geometry import quarter_annulus, unit_hypercube

__all__ = ["Config", "get_config", "CONFIG_NAMES"]

CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg5", "cfg5_tensor")


@dataclass
class Config:
    name: str
    problem: A.BenchmarkProblem
    plan: CombinationPlan
    n_points: int
    seed: int
    grid_levels: tuple
    quad_points: int

    def points(self, n=None) -> np.ndarray:
        d = self.plan.d
        return np.random.default_rng(self.seed).random((self.n_points if n is None else n, d))

    def grid(self) -> QuadGrid:
        return QuadGrid(self.problem.patch, self.grid_levels, self.quad_points, self.problem.grading)


def get_config(name: str) -> Config:
    if name == "cfg1":
        prob = A.BenchmarkProblem("cfg1_square_sin", unit_hypercube(2), A.sin_product_forcing, 2, 1,
                                  solution=A.sin_product_solution, solution_gradient=A.sin_product_gradient)
        return Config(name, prob, baseline_plan(2, 6), 4096, 0, (5, 5), 3)
    if name == "cfg2":
        prob = A.BenchmarkProblem("cfg2_cube_sin", unit_hypercube(3), A.sin_product_forcing, 3, 2,
                                  solution=A.sin_product_solution, solution_gradient=A.sin_product_gradient)
        return Config(name, prob, baseline_plan(3, 7), 32768, 1, (5, 5, 5), 4)
    if name == "cfg3":
        prob = A.BenchmarkProblem("cfg3_annulus", quarter_annulus(2), A.annulus_polar_forcing, 3, 2,
                                  solution=A.annulus_polar_solution, solution_gradient=A.annulus_polar_gradient)
        return Config(name, prob, baseline_plan(2, 8), 4096, 2, (7, 7), 4)
    if name in ("cfg5", "cfg5_tensor"):
        prob = A.BenchmarkProblem("cfg5_cube_exp", unit_hypercube(3), A.exp_bubble_forcing, 4, 3,
                                  solution=A.exp_bubble_solution, solution_gradient=A.exp_bubble_gradient)
        plan = baseline_plan(3, 12) if name == "cfg5" else CombinationPlan(3, (((6, 6, 6), 1),), level=6)
        return Config(name, prob, plan, 32768, 4, (6, 6, 6), 5)
    raise KeyError(f"unknown config {name!r}; expected one of {CONFIG_NAMES}")


@dataclass
class MultipatchConfig:
    """BASELINE cfg4: the L-shape, p=2 C1, combination
    technique w=9 (15 components), uniform or one-sided graded knots,
    4096 random parametric points per patch (seed 3), per-patch (8,8) error
    grid with q=3 on the same knots."""

    name: str
    problem: object
    plan: CombinationPlan
    n_points: int = 4096
    seed: int = 3
    grid_levels: tuple = (8, 8)
    quad_points: int = 3

    def points(self, n=None) -> np.ndarray:
        return np.random.default_rng(self.seed).random((self.n_points if n is None else n, 2))


def get_multipatch_config(name: str = "cfg4") -> MultipatchConfig:
    from .multipatch import lshape_problem

    if name not in ("cfg4", "cfg4_graded"):
        raise KeyError(f"unknown multipatch config {name!r}")
    return MultipatchConfig(name, lshape_problem(graded=name == "cfg4_graded"), baseline_plan(2, 9))   # w = 9 (BASELINE configs[3])
