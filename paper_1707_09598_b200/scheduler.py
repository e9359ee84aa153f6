"""Drop-in ``run_plan``: the whole plan is one batched device pipeline.

Reference: scheduler.py:26-96.  ``run_plan(plan, problem, workers=1,
quad_points=None) -> (solutions, RunReport)`` keeps its signature and
invariants (plan order, sum of component times == serial_time, times > 0).
Components are solved together, so each component's ``solve_time`` is the
measured batch time apportioned by a modelled cost (assembly metric bytes +
PCG bytes x iterations); ``RunReport.wall_time`` is the measured wall time.
``workers`` is validated like the reference and otherwise unused (one GPU).
"""
from __future__ import annotations

import csv
import heapq
import time

import numpy as np

from . import _lib
from .analysis import forcing_id_of
from .pipeline import Batch, PlanSpec, knot_tables_for

__all__ = ["RunReport", "optimized_makespan", "lpt_partition", "run_plan", "solve_terms",
           "write_timing_csv", "DEFAULT_RTOL", "PlanSession", "make_spec"]

DEFAULT_RTOL = 1e-13   # north star: CG to 1e-13 relative residual


def _lpt_makespan(ordered_times, cores: int) -> float:
    if cores < 1:
        raise ValueError(f"core count must be >= 1, got {cores}")
    free = [0.0] * cores
    for t in ordered_times:
        if t < 0.0:
            raise ValueError("job times must be nonnegative")
        heapq.heappush(free, heapq.heappop(free) + float(t))
    return max(free)


def optimized_makespan(times, cores: int) -> float:
    """Longest-processing-time-first makespan (reference scheduler.py:39-42)."""
    return _lpt_makespan(sorted((float(t) for t in times), reverse=True), cores)


def lpt_partition(costs, parts: int) -> list:
    """LPT assignment of jobs to ``parts`` bins (the multi-GPU partitioner);
    ties broken by job index so every rank computes the same answer."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, b) for b in range(parts)]
    bins = [[] for _ in range(parts)]
    for i in order:
        load, b = heapq.heappop(heap)
        bins[b].append(i)
        heapq.heappush(heap, (load + float(costs[i]), b))
    return [sorted(b) for b in bins]


class RunReport:
    """Timing summary: components = ((beta, dofs, seconds), ...) in plan order."""

    def __init__(self, components, wall_time, phase_ms=None, iterations=None):
        self.components = tuple(components)
        self.wall_time = float(wall_time)
        self.phase_ms = phase_ms
        self.iterations = iterations

    @property
    def serial_time(self) -> float:
        return float(sum(t for _, _, t in self.components))

    @property
    def total_dofs(self) -> int:
        return int(sum(n for _, n, _ in self.components))

    @property
    def max_component_dofs(self) -> int:
        return int(max(n for _, n, _ in self.components))

    def optimized_time(self, cores: int) -> float:
        ordered = sorted(self.components, key=lambda it: (-it[2], it[0]))
        return _lpt_makespan([t for _, _, t in ordered], cores)


def make_spec(terms, problem, quad_points=None, knot_rule=None) -> PlanSpec:
    patch = problem.patch
    d = len(patch.knotvectors)
    q = int(quad_points) if quad_points is not None else int(problem.degree) + 1
    tables = knot_tables_for(terms, d, problem.degree, problem.regularity, problem.grading, knot_rule)
    return PlanSpec(d, int(problem.degree), int(problem.regularity), q, tuple(terms), tables, patch,
                    forcing_id_of(problem.forcing))


def solve_terms(terms, problem, quad_points=None, rtol=DEFAULT_RTOL, maxit=0, knot_rule=None,
                keep_batch=True):
    """Assemble + solve a list of (beta, coef) terms in one batch."""
    from .assembly import DiscreteSpace
    from .combination import ComponentSolution
    from .splines import dyadic_level_knots

    t0 = time.perf_counter()
    spec = make_spec(terms, problem, quad_points, knot_rule)
    batch = Batch(spec, host_forcing=problem.forcing if spec.forcing_id == _lib.FORCING_HOST else None)
    batch.assemble()
    batch.solve(rtol=rtol, maxit=maxit)
    flat = batch.coefficients()
    wall = time.perf_counter() - t0
    cost = batch.component_cost()
    share = wall * cost / cost.sum()
    sols = []
    for i, (beta, _) in enumerate(terms):
        if knot_rule is not None:
            kvs = tuple(knot_rule(k, int(lv)) for k, lv in enumerate(beta))
        else:
            kvs = tuple(dyadic_level_knots(lv, problem.degree, problem.regularity, problem.grading) for lv in beta)
        sols.append(ComponentSolution(tuple(beta), DiscreteSpace(kvs), batch.component_coefficients(flat, i).copy(),
                                      float(share[i]), batch if keep_batch else None, i))
    if not keep_batch:
        batch.close()
    return sols, (batch, wall)


def run_plan(plan, problem, workers=1, quad_points=None):
    """Solve every component of ``plan``; returns (solutions, RunReport)."""
    workers = int(workers)
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    t0 = time.perf_counter()
    sols, (batch, _) = solve_terms(tuple(plan.terms), problem, quad_points)
    wall = time.perf_counter() - t0
    ms, _ = batch.phase_stats()
    report = RunReport(tuple((s.beta, s.n_dofs, s.solve_time) for s in sols), wall,
                       phase_ms=tuple(float(x) for x in ms), iterations=tuple(int(i) for i in batch.iters))
    return sols, report


class PlanSession:
    """A device handle kept across repeated solves of one plan shape.

    ``run(points)`` is the end-to-end call: host->device copy of the
    points, assemble, PCG, combine, device->host copy of the combined
    values -- one library call (sgiga_run), one stream synchronisation; from
    the second call on with the same arguments it replays a captured CUDA
    graph.  The problem descriptor is uploaded once, when the session opens
    (``update(problem)`` re-uploads a same-shape problem).
    """

    def __init__(self, plan, problem, quad_points=None, rtol=DEFAULT_RTOL, stream=None):
        self.plan = plan
        self.problem = problem
        self.rtol = float(rtol)
        self.spec = make_spec(tuple(plan.terms), problem, quad_points)
        self.batch = Batch(self.spec, stream=stream,
                           host_forcing=problem.forcing if self.spec.forcing_id == _lib.FORCING_HOST else None)

    @property
    def h2d_input_bytes(self) -> int:
        return int(sum(a.nbytes for a in self.batch._keep.values()))

    def update(self, problem) -> None:
        """Re-upload a problem of the same shape (new geometry weights,
        forcing, ...); an identical descriptor keeps the captured graph."""
        spec = make_spec(tuple(self.plan.terms), problem, self.spec.quad_points)
        self.batch.upload(spec)
        self.problem, self.spec = problem, spec

    def run(self, points) -> np.ndarray:
        return self.batch.run(points, self.rtol)

    def submit(self, points, out) -> None:
        """Pipelined form of run(): enqueue a pass on page-locked host
        buffers (``points`` in, combined values into ``out``) and return;
        passes run back to back on the device.  ``wait()`` synchronises and
        raises the reference's exceptions for the last submitted pass."""
        self.batch.run_host_async(points, out, self.rtol)

    def wait(self) -> None:
        self.batch.run_wait()

    def close(self):
        self.batch.close()


def write_timing_csv(path, report: RunReport, cores=()) -> None:
    """Same layout as the reference (scheduler.py:99-125)."""
    if not report.components:
        raise ValueError("report has no components")
    d = len(report.components[0][0])
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow([f"beta_{i + 1}" for i in range(d)] + ["dofs", "time_s"])
        for beta, dofs, t in report.components:
            w.writerow([*beta, dofs, repr(t)])
        pad = [""] * (d - 1)
        w.writerow(["serial", *pad, report.total_dofs, repr(report.serial_time)])
        for c in cores:
            w.writerow([f"cores_{int(c)}", *pad, report.total_dofs, repr(report.optimized_time(int(c)))])
