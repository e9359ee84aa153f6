"""B200-native batched sparse-grid combination-technique IGA hot path.

Drop-in for the reference package's plan driver (``run_plan``), component
solve (``solve_component``) and combine (``evaluate_combined``); every
component of a plan is assembled, solved and combined by hand-written
sm_100a FP64 kernels in ``libsgiga.so`` (C ABI: include/sgiga.h).
"""
from .analysis import BenchmarkProblem, error_norms
from .assembly import DiscreteSpace, QuadGrid, assemble_poisson
from .combination import (CombinationPlan, ComponentSolution, baseline_plan,
                          combination_coefficients, evaluate_combined,
                          evaluate_combined_points, general_coefficients, solve_component)
from .errors import EmptyInteriorError, InvalidGeometryError, LinearSolveError
from .geometry import NurbsPatch, quarter_annulus, unit_hypercube
from .pipeline import Batch, gauss_rule
from .scheduler import RunReport, optimized_makespan, run_plan

__version__ = "0.1.0"

__all__ = [
    "BenchmarkProblem", "error_norms", "DiscreteSpace", "QuadGrid", "assemble_poisson",
    "CombinationPlan", "ComponentSolution", "baseline_plan", "combination_coefficients",
    "evaluate_combined", "evaluate_combined_points", "general_coefficients", "solve_component",
    "EmptyInteriorError", "InvalidGeometryError", "LinearSolveError", "NurbsPatch",
    "quarter_annulus", "unit_hypercube", "Batch", "gauss_rule", "RunReport",
    "optimized_makespan", "run_plan", "backend",
]


def backend() -> str:
    """The only backend: the CUDA library (there is no CPU fallback)."""
    return "cuda-sm_100a"
