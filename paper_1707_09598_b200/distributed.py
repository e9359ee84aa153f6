"""Multi-GPU combination technique: one plan's components sharded over ranks.

SURVEY.md section 8(e): the components of a plan are independent
(reference PAPER.md:121-126), so each rank assembles and solves an
LPT-balanced subset -- the reference's own ``optimized_makespan`` rule
(scheduler.py:39-42) applied to a modelled cost -- with no data-path
collective.  The only exchange is at the combine:

* every rank evaluates its components at the points into a DEVICE buffer
  (``sgiga_run_components_async``: assemble + solve + per-component combine,
  no host round trip);
* one NCCL ``all_gather_into_tensor`` of those buffers (padded to the
  largest shard) over NVLink;
* the plan-order sum ``sgiga_plan_order_sum`` on every rank, with the exact
  operations and order of the single-GPU combine (vals = c*v; vals += c*v,
  reference combination.py:227-233).

A component's per-point values do not depend on which other components
share its batch (fixed per-component reduction orders; tested), so the
distributed result is bitwise equal to the single-GPU one -- the
reference's worker-count invariance (tests/test_scheduler.py:103-110).  An
NCCL sum all-reduce would not fix the summation order.

One process per GPU (torchrun); torch.distributed is the plumbing (NCCL on
GPUs, gloo on CPU for the host-logic tests).
"""
from __future__ import annotations

import ctypes as ct
from typing import Callable, Sequence

import numpy as np

from .scheduler import lpt_partition

__all__ = ["component_cost_model", "plan_partition", "plan_rows", "ordered_combine", "combine_distributed",
           "allgather_padded", "DistributedPlan", "run_plan_distributed"]

# modelling constants (measured on the B200, bench.py / profiles/r02):
ASM_RATE = 40.0e12      # canonical sum-factorised FP64 FLOP/s of the tiled 3-D assembly, thin cross-section
ASM_RATE_LONG = 30.0e12 # ... cross-sections with no axis of <= 4 elements (cfg5 per-class timeline)
ASM_RATE_2D = 4.0e12    # ... of the 2-D assembly (cfg3 x1024)
HBM_RATE = 4.0e12       # bytes/s the FD / line-FD PCG streams its stencils at
JACOBI_ITER = 2.0       # Jacobi-PCG iterations grow ~ 2**max(level) (conditioning of K)
FD_MMAX = 72            # axes the FD preconditioner diagonalises (csrc/sgiga_internal.cuh)


def component_cost_model(terms, degree: int, d: int) -> np.ndarray:
    """Modelled device seconds per component.

    * assembly: canonical sum-factorised FLOPs F_el = 2 d^2 sum_k P^(d+k+1)
      + 2 d P^(d+1) per element at the measured rate of the
      tiled kernel for the component's cross-section class -- on cfg5 the
      assembly is ~75 % of a pass and scales with the element count
      2^|beta|, not with the solver;
    * solve: FD-preconditioned components (every axis but the longest
      within the FD range) converge in 1-2 iterations: ~3 stencil sweeps
      (iterations + true residual) plus the line factors; the others run
      Jacobi-PCG whose iteration count grows like 2^max(beta).
    """
    P = degree + 1
    W = 2 * degree + 1
    F_el = 2 * d * d * sum(P ** (d + k + 1) for k in range(1, d + 1)) + 2 * d * P ** (d + 1)
    out = []
    for beta, _ in terms:
        nel = float(np.prod([2.0 ** b for b in beta]))
        # the tiled kernel covers a thin cross-section axis whole (the stream
        # axis is the longest one); long x long cross-sections run slower
        thin = d == 3 and min(sorted(beta)[:-1]) <= 2
        rate = (ASM_RATE if thin else ASM_RATE_LONG) if d == 3 else ASM_RATE_2D
        m = np.array([2 ** b + degree - 2 for b in beta], dtype=np.float64)
        rows = float(np.prod(np.maximum(m, 0)))
        slots = float(np.prod(np.minimum(np.maximum(m, 1), W)))
        stencil = 8.0 * slots * rows
        t_asm = nel * F_el / rate
        others = np.sort(m)[:-1] if d > 1 else np.array([])
        if np.all(others <= FD_MMAX):
            sweeps = 3.0 + (8.0 * rows * P / stencil if stencil else 0.0)   # + line factors
        else:
            sweeps = JACOBI_ITER ** max(beta)
        out.append(t_asm + sweeps * (stencil + 104.0 * rows) / HBM_RATE)
    return np.array(out)


def plan_partition(plan, world: int, degree: int) -> list:
    """Component indices per rank (deterministic LPT on the cost model)."""
    return lpt_partition(component_cost_model(plan.terms, degree, plan.d), world)


def plan_rows(parts: Sequence[Sequence[int]], nmax: int, n_comp: int) -> np.ndarray:
    """Row of every plan component in the all-gathered [world * nmax, npts]
    buffer: rank r's k-th component sits at row r * nmax + k."""
    rows = np.full(n_comp, -1, dtype=np.int64)
    for r, idx in enumerate(parts):
        for k, c in enumerate(idx):
            rows[c] = r * nmax + k
    if np.any(rows < 0):
        raise ValueError("partition does not cover the plan")
    return rows


def ordered_combine(plan, values: np.ndarray) -> np.ndarray:
    """Host restatement of the plan-order sum (reference combination.py:
    227-233): vals = c*v, then vals += c*v.  ``values`` is (n_comp, npts)."""
    acc = None
    for (beta, c), v in zip(plan.terms, values):
        term = float(c) * v
        acc = term if acc is None else acc + term
    return acc


def allgather_padded(local, counts: Sequence[int], group=None):
    """All-gather (n_r, npts) blocks of different n_r: each rank pads to
    max(counts) rows, one ``all_gather_into_tensor``; returns the
    [world * nmax, npts] tensor (same device as ``local``)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    nmax = max(counts)
    npts = local.shape[1]
    buf = torch.zeros((nmax, npts), dtype=torch.float64, device=local.device)
    if local.shape[0]:
        buf[: local.shape[0]].copy_(local)
    out = torch.empty((world * nmax, npts), dtype=torch.float64, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out


def combine_distributed(plan, npts: int, local_values_fn: Callable, degree: int, group=None, device=None):
    """Host-side variant (CPU tensors / gloo): each rank evaluates its
    components (``local_values_fn(indices) -> (len(indices), npts)``), one
    padded all-gather, the plan-order sum on every rank (numpy)."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    parts = plan_partition(plan, world, degree)
    mine = parts[rank]
    local = np.asarray(local_values_fn(mine), dtype=np.float64).reshape(len(mine), npts)
    counts = [len(p) for p in parts]
    gathered = allgather_padded(torch.as_tensor(local, device=device), counts, group).cpu().numpy()
    rows = plan_rows(parts, max(counts), len(plan.terms))
    return ordered_combine(plan, gathered[rows])


class DistributedPlan:
    """One rank's share of a plan split over ``world`` GPUs (device path).

    ``step(pts)`` = assemble + solve the rank's components, evaluate them at
    the device points ``pts`` (per component), all-gather over NCCL, plan-
    order sum on the device: returns the combined values (device tensor),
    bitwise equal to the single-GPU combine.  No host round trip of values.
    """

    def __init__(self, plan, problem, quad_points=None, rtol=1e-13, group=None):
        import torch
        import torch.distributed as dist

        from . import _lib
        from .pipeline import Batch
        from .scheduler import make_spec

        self.plan, self.rtol, self.group = plan, rtol, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.parts = plan_partition(plan, self.world, problem.degree)
        self.mine = self.parts[self.rank]
        self.counts = [len(p) for p in self.parts]
        self.nmax = max(self.counts)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.lib = _lib.load()
        self.batch = Batch(make_spec(tuple(plan.terms[i] for i in self.mine), problem, quad_points)) \
            if self.mine else None
        rows = plan_rows(self.parts, self.nmax, len(plan.terms))
        self.d_rows = torch.as_tensor(rows, device=self.device)
        self.d_coef = torch.as_tensor(np.array([c for _, c in plan.terms], dtype=np.int32), device=self.device)
        self._bufs = {}

    def _buffers(self, npts):
        import torch
        if npts not in self._bufs:
            self._bufs[npts] = (torch.zeros((self.nmax, npts), dtype=torch.float64, device=self.device),
                                torch.empty((self.world * self.nmax, npts), dtype=torch.float64, device=self.device),
                                torch.empty(npts, dtype=torch.float64, device=self.device))
        return self._bufs[npts]

    def step(self, pts_dev):
        """pts_dev: (npts, d) float64 CUDA tensor, contiguous."""
        import torch
        import torch.distributed as dist

        from . import _lib

        npts = int(pts_dev.shape[0])
        local, gathered, out = self._buffers(npts)
        cur = torch.cuda.current_stream(self.device)
        if self.batch is not None:
            bs = torch.cuda.ExternalStream(self.batch.stream_ptr, device=self.device)
            bs.wait_stream(cur)                          # points / buffers ready
            self.batch.run_components_async(pts_dev.data_ptr(), npts, local.data_ptr(), self.rtol)
            self.batch.run_wait()                        # convergence verdict (raises LinearSolveError)
            cur.wait_stream(bs)
        dist.all_gather_into_tensor(gathered, local, group=self.group)
        _lib.check(self.lib.sgiga_plan_order_sum(ct.c_void_p(cur.cuda_stream), len(self.plan.terms), npts,
                                                 ct.c_void_p(self.d_coef.data_ptr()),
                                                 ct.c_void_p(self.d_rows.data_ptr()),
                                                 ct.c_void_p(gathered.data_ptr()), ct.c_void_p(out.data_ptr())))
        return out

    def close(self):
        if self.batch is not None:
            self.batch.close()
            self.batch = None


def run_plan_distributed(plan, problem, points, quad_points=None, rtol=1e-13, group=None):
    """Multi-GPU drop-in for run_plan + scattered combine (one rank per GPU).

    Returns the combined values at ``points`` (numpy) on every rank, bitwise
    equal to the single-GPU ``evaluate_combined_points``.
    """
    import torch

    pts = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64),
                          device=torch.device("cuda", torch.cuda.current_device()))
    dp = DistributedPlan(plan, problem, quad_points, rtol, group)
    try:
        return dp.step(pts).cpu().numpy()
    finally:
        dp.close()
