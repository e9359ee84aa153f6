"""Multi-GPU combination technique: components sharded over ranks.

SURVEY.md section 8(e): the components of a plan are independent
(reference PAPER.md:121-126), so each rank solves an LPT-balanced subset --
the reference's own ``optimized_makespan`` rule (scheduler.py:39-42) applied
to a modelled cost -- with no data-path collective.  The only exchange is at
the combine: one all-gather of per-component point values, then the
plan-order sum on every rank, which keeps the reference's bitwise
determinism across worker counts (tests/test_scheduler.py:103-110); an NCCL
sum-all-reduce would not fix the summation order.

One process per GPU (torchrun); the device plumbing is torch.distributed
(NCCL on GPUs, gloo on CPU for the tests).
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .scheduler import lpt_partition

__all__ = ["component_cost_model", "plan_partition", "ordered_combine", "combine_distributed",
           "run_plan_distributed"]


def component_cost_model(terms, degree: int, d: int) -> np.ndarray:
    """Modelled cost per component: stencil bytes x an iteration estimate.

    Jacobi-PCG iterations grow like the square root of the condition
    number, i.e. like 2**max(beta) on these meshes; the stencil has
    prod(min(m_k, 2p+1)) slots per interior row.
    """
    W = 2 * degree + 1
    out = []
    for beta, _ in terms:
        m = np.array([2**b + degree - 2 for b in beta], dtype=np.float64)
        rows = float(np.prod(np.maximum(m, 0)))
        slots = float(np.prod(np.minimum(np.maximum(m, 1), W)))
        out.append(rows * (8.0 * slots + 104.0) * (1.0 + 2.0 ** max(beta)))
    return np.array(out)


def plan_partition(plan, world: int, degree: int) -> list:
    """Component indices per rank (deterministic LPT)."""
    return lpt_partition(component_cost_model(plan.terms, degree, plan.d), world)


def ordered_combine(plan, values: np.ndarray) -> np.ndarray:
    """sum_beta c_beta v_beta in plan order: vals = c*v, then vals += c*v
    (reference combination.py:227-233).  ``values`` is (n_comp, npts)."""
    acc = None
    for (beta, c), v in zip(plan.terms, values):
        term = float(c) * v
        acc = term if acc is None else acc + term
    return acc


def _allgather_padded(local: np.ndarray, counts: Sequence[int], group=None, device=None):
    """All-gather (n_i, npts) blocks of different n_i via padding to max n_i."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    nmax = max(counts)
    npts = local.shape[1]
    buf = torch.zeros((nmax, npts), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.as_tensor(local, dtype=torch.float64, device=device)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return [o[:n].cpu().numpy() for o, n in zip(outs, counts)]


def combine_distributed(plan, npts: int, local_values_fn: Callable, degree: int, group=None, device=None):
    """Each rank evaluates its components (``local_values_fn(indices) ->
    (len(indices), npts)``); one all-gather; ordered sum on every rank."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    parts = plan_partition(plan, world, degree)
    mine = parts[rank]
    local = np.asarray(local_values_fn(mine), dtype=np.float64).reshape(len(mine), npts)
    blocks = _allgather_padded(local, [len(p) for p in parts], group, device)
    full = np.empty((len(plan.terms), npts))
    for idx, blk in zip(parts, blocks):
        full[idx] = blk
    return ordered_combine(plan, full)


def run_plan_distributed(plan, problem, points, quad_points=None, rtol=1e-13, group=None):
    """Multi-GPU drop-in for run_plan + scattered combine (one rank per GPU).

    Returns the combined values at ``points`` on every rank, bitwise equal
    to the single-GPU ``evaluate_combined_points``.
    """
    import torch

    from .pipeline import Batch
    from .scheduler import make_spec

    pts = np.ascontiguousarray(points, dtype=np.float64)
    device = torch.device("cuda", torch.cuda.current_device())

    def local(indices):
        if not indices:
            return np.zeros((0, pts.shape[0]))
        terms = tuple(plan.terms[i] for i in indices)
        b = Batch(make_spec(terms, problem, quad_points))
        try:
            b.assemble()
            b.solve(rtol=rtol)
            return b.combine_points(pts, per_component=True)
        finally:
            b.close()

    return combine_distributed(plan, pts.shape[0], local, problem.degree, group, device)
