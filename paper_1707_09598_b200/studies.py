"""Batched study drivers on the device pipeline (SURVEY.md section 8(f),
rows 3 and 4).

* Surplus / profit (reference combination.py:239-302): every component of a
  profit box is solved in ONE batch; each hierarchical surplus (the signed
  sum over the 2^d componentwise-lower binary neighbours) is integrated on
  its ``QuadGrid`` by one device pass (``sgiga_subset_error_norms`` against
  zero), accumulating the neighbours in the reference's order
  (combination.py:269-272).
* Convergence studies (analysis.py:273-528): all levels of a study -- and
  the overkill tensor reference when the problem has no closed form -- are
  solved in ONE batch; each level's L2 / H1-seminorm error is one device
  pass over its plan's terms (minus the closed form, or minus the overkill
  component).  ``gamma_sweep`` reuses it per grading and method.

Per-component solve times are apportioned from the batch wall time by the
modelled cost, as ``run_plan`` does (scheduler.RunReport).
"""
from __future__ import annotations

import csv
import itertools
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "ProfitRow", "surplus_norm", "profit_table",
    "fit_rate", "ConvergenceRecord", "convergence_study", "write_convergence_csv",
    "read_convergence_csv", "GammaSweepRow", "gamma_sweep", "write_gamma_csv",
]


# ---- surplus / profit --------------------------------------------------------
def _binary_shifts(beta):
    """(sign, lower) for the componentwise-lower binary neighbours with all
    levels >= 0, in itertools.product((0, 1), ...) order (beta itself first)."""
    for k in itertools.product((0, 1), repeat=len(beta)):
        lower = tuple(b - kk for b, kk in zip(beta, k))
        if min(lower) >= 0:
            yield (-1) ** sum(k), lower


@dataclass(frozen=True)
class ProfitRow:
    """Surplus-to-cost record of one component index."""

    beta: tuple
    surplus_l2: float
    dofs: int

    @property
    def profit(self) -> float:
        return self.surplus_l2 / self.dofs


def _surplus_on(batch, index, problem, beta, q):
    from .assembly import QuadGrid

    grid = QuadGrid(problem.patch, beta, q, problem.grading)
    terms = [(index[lower], float(sign)) for sign, lower in _binary_shifts(beta)]
    l2, _ = batch.subset_error_norms(grid.points_per_dir, grid.weights_per_dir, terms, None)
    return l2


def surplus_norm(problem, beta, cache=None, quad_points=None):
    """L2 norm of the hierarchical surplus at ``beta`` and the dofs of the
    ``beta`` component (reference combination.py:247-272).  ``cache``
    (a dict) receives the component solutions keyed by index."""
    from .scheduler import solve_terms

    beta = tuple(int(b) for b in beta)
    if cache is None:
        cache = {}
    q = quad_points if quad_points is not None else problem.degree + 1
    lowers = [lower for _, lower in _binary_shifts(beta)]
    sols, (batch, _) = solve_terms(tuple((lw, 1) for lw in lowers), problem, quad_points)
    index = {lw: i for i, lw in enumerate(lowers)}
    norm = _surplus_on(batch, index, problem, beta, q)
    for lw, s in zip(lowers, sols):
        cache.setdefault(lw, s)
    return float(norm), cache[beta].n_dofs


def profit_table(problem, beta_max, quad_points=None) -> list:
    """Profit rows for every index 0 <= beta <= beta_max (reference
    combination.py:287-302); the whole box is one device batch."""
    from .scheduler import solve_terms

    d = len(problem.patch.knotvectors)
    if np.isscalar(beta_max):
        beta_max = (int(beta_max),) * d
    beta_max = tuple(int(b) for b in beta_max)
    if len(beta_max) != d or any(b < 0 for b in beta_max):
        raise ValueError(f"invalid profit box bound {beta_max}")
    q = quad_points if quad_points is not None else problem.degree + 1
    box = list(itertools.product(*(range(b + 1) for b in beta_max)))
    sols, (batch, _) = solve_terms(tuple((b, 1) for b in box), problem, quad_points)
    index = {b: i for i, b in enumerate(box)}
    return [ProfitRow(beta, float(_surplus_on(batch, index, problem, beta, q)), sols[index[beta]].n_dofs)
            for beta in box]


# ---- convergence studies -----------------------------------------------------
def fit_rate(levels, errors):
    """Least-squares rate of errors ~ C 2^(-rate * level) and the per-step
    rates (reference analysis.py:273-291)."""
    lv = np.asarray(levels, dtype=np.float64)
    er = np.asarray(errors, dtype=np.float64)
    if lv.shape != er.shape or lv.ndim != 1:
        raise ValueError("levels and errors must be matching 1D sequences")
    if lv.size < 3:
        raise ValueError("rate fit needs at least three levels")
    if np.any(er <= 0.0):
        raise ValueError("errors must be positive for a log fit")
    slope = np.polyfit(lv, np.log2(er), 1)[0]
    return float(-slope), np.log2(er[:-1] / er[1:])


@dataclass(frozen=True)
class ConvergenceRecord:
    """One (method, level) row of a convergence study."""

    method: str
    d: int
    degree: int
    regularity: int
    grading: float
    level: int
    n_components: int
    dofs_total: int
    dofs_max_component: int
    l2_error: float
    h1_semi_error: float
    time_serial_s: float
    times_cores: dict = field(default_factory=dict)

    @property
    def h(self) -> float:
        return 2.0 ** (-self.level)


def _plan_for(method: str, d: int, level: int):
    from .combination import CombinationPlan, combination_coefficients

    if method == "tensor":
        return CombinationPlan(d, (((level,) * d, 1),), level=level)
    if method == "sparse":
        return combination_coefficients(d, level)
    raise ValueError(f"method must be 'tensor' or 'sparse', got {method!r}")


def convergence_study(problem, method, levels, cores=(), workers=1, quad_points=None, reference_margin=2):
    """Errors of ``method`` over ``levels`` against the closed-form solution,
    or against an overkill tensor solution ``reference_margin`` levels above
    the finest level (reference analysis.py:325-386).  Every level's plan and
    the overkill component are solved in one batch; the overkill solve stays
    out of the timing columns."""
    from .analysis import solution_id_of
    from .assembly import QuadGrid
    from .scheduler import _lpt_makespan, solve_terms

    levels = [int(j) for j in levels]
    if not levels:
        raise ValueError("no levels requested")
    if any(j < 0 for j in levels):
        raise ValueError("levels must be >= 0")
    if int(workers) < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    d = len(problem.patch.knotvectors)
    q = quad_points if quad_points is not None else problem.degree + 1
    plans = [_plan_for(method, d, lv) for lv in levels]
    keys = []
    for plan in plans:
        for beta, _ in plan.terms:
            if beta not in keys:
                keys.append(beta)
    sid = solution_id_of(problem.solution) if problem.solution is not None else None
    ref_beta = None
    if problem.solution is None:
        ref_level = max(levels) + int(reference_margin)
        ref_beta = (ref_level,) * d
        if ref_beta not in keys:
            keys.append(ref_beta)
    elif sid is None:
        raise ValueError("convergence_study on the device needs a registered closed-form solution")
    sols, (batch, wall) = solve_terms(tuple((b, 1) for b in keys), problem, quad_points)
    index = {b: i for i, b in enumerate(keys)}
    if ref_beta is not None:
        ref_grid = QuadGrid(problem.patch, ref_beta, q, problem.grading)
    records = []
    for level, plan in zip(levels, plans):
        terms = [(index[beta], float(c)) for beta, c in plan.terms]
        if ref_beta is None:
            grid = QuadGrid(problem.patch, (level,) * d, q, problem.grading)
            l2, h1 = batch.subset_error_norms(grid.points_per_dir, grid.weights_per_dir, terms, sid)
        else:
            terms.append((index[ref_beta], -1.0))
            l2, h1 = batch.subset_error_norms(ref_grid.points_per_dir, ref_grid.weights_per_dir, terms, None)
        comp = [(beta, sols[index[beta]].n_dofs, sols[index[beta]].solve_time) for beta, _ in plan.terms]
        ordered = sorted(comp, key=lambda it: (-it[2], it[0]))
        records.append(ConvergenceRecord(
            method=method, d=d, degree=problem.degree, regularity=problem.regularity,
            grading=problem.grading, level=level, n_components=len(plan),
            dofs_total=int(sum(n for _, n, _ in comp)), dofs_max_component=int(max(n for _, n, _ in comp)),
            l2_error=float(l2), h1_semi_error=float(h1), time_serial_s=float(sum(t for _, _, t in comp)),
            times_cores={int(c): _lpt_makespan([t for _, _, t in ordered], int(c)) for c in cores}))
    return records


_CONV_HEADER = ["method", "d", "p", "r", "gamma", "J", "h", "n_components", "dofs_total",
                "dofs_max_component", "l2_error", "h1_semi_error", "time_serial_s"]


def write_convergence_csv(path, records, cores=()) -> None:
    """Fixed column layout of the reference (analysis.py:389-431)."""
    cores = [int(c) for c in cores]
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(_CONV_HEADER + [f"time_cores_{c}_s" for c in cores])
        for r in records:
            w.writerow([r.method, r.d, r.degree, r.regularity, repr(r.grading), r.level, repr(r.h),
                        r.n_components, r.dofs_total, r.dofs_max_component, repr(r.l2_error),
                        repr(r.h1_semi_error), repr(r.time_serial_s)] + [repr(r.times_cores[c]) for c in cores])


def read_convergence_csv(path):
    """Inverse of write_convergence_csv: (records, cores)."""
    with open(path, newline="", encoding="utf-8") as fh:
        rd = csv.reader(fh)
        header = next(rd)
        cores = [int(n[len("time_cores_"):-len("_s")]) for n in header if n.startswith("time_cores_")]
        recs = []
        for row in rd:
            v = dict(zip(header, row))
            recs.append(ConvergenceRecord(
                method=v["method"], d=int(v["d"]), degree=int(v["p"]), regularity=int(v["r"]),
                grading=float(v["gamma"]), level=int(v["J"]), n_components=int(v["n_components"]),
                dofs_total=int(v["dofs_total"]), dofs_max_component=int(v["dofs_max_component"]),
                l2_error=float(v["l2_error"]), h1_semi_error=float(v["h1_semi_error"]),
                time_serial_s=float(v["time_serial_s"]),
                times_cores={c: float(v[f"time_cores_{c}_s"]) for c in cores}))
    return recs, cores


@dataclass(frozen=True)
class GammaSweepRow:
    """Fitted rates of one (grading, method) pair."""

    gamma: float
    method: str
    d: int
    degree: int
    regularity: int
    l2_rate: float
    h1_semi_rate: float


def gamma_sweep(d, gammas, levels, methods=("sparse", "tensor"), degree=3, regularity=None, workers=1,
                fit_from=None):
    """Rates of the constant-forcing annulus problem across gradings
    (reference analysis.py:485-528): (rows, records)."""
    from .analysis import constant_forcing_problem

    gammas = [float(g) for g in gammas]
    if not gammas:
        raise ValueError("no gradings requested")
    rows, all_records = [], []
    for gamma in gammas:
        problem = constant_forcing_problem(d, gamma, degree, regularity)
        for method in methods:
            recs = convergence_study(problem, method, levels, workers=workers)
            all_records.extend(recs)
            use = [r for r in recs if fit_from is None or r.level >= fit_from]
            lv = [r.level for r in use]
            l2_rate, _ = fit_rate(lv, [r.l2_error for r in use])
            h1_rate, _ = fit_rate(lv, [r.h1_semi_error for r in use])
            rows.append(GammaSweepRow(gamma, method, d, problem.degree, problem.regularity, l2_rate, h1_rate))
    return rows, all_records


def write_gamma_csv(path, rows) -> None:
    """Rate table: gamma, method, d, p, r, l2_rate, h1_semi_rate."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["gamma", "method", "d", "p", "r", "l2_rate", "h1_semi_rate"])
        for r in rows:
            w.writerow([repr(r.gamma), r.method, r.d, r.degree, r.regularity, repr(r.l2_rate),
                        repr(r.h1_semi_rate)])

