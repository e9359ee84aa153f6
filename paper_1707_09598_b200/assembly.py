"""Discrete spaces, quadrature grids and single-space assembly (GPU-backed).

Host mirrors of the reference objects (assembly.py): ``DiscreteSpace``
(50-127), ``QuadGrid`` (141-183, per-axis points/weights only -- the mapped
points live on the device), ``AssembledSystem`` (193-206) and
``assemble_poisson`` (357-390), which here runs the batched device
assembly on a one-term plan and exports the interior CSR.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import EmptyInteriorError
from .pipeline import Batch, PlanSpec, gauss_rule
from .splines import KnotVector, dyadic_level_knots

__all__ = [
    "EmptyInteriorError", "gauss_rule", "DiscreteSpace", "QuadGrid", "AssembledSystem",
    "assemble_poisson", "space_batch",
]


@dataclass(frozen=True)
class DiscreteSpace:
    """Tensor-product B-spline space on [0,1]^d (host metadata)."""

    knotvectors: tuple

    def __post_init__(self):
        kvs = tuple(self.knotvectors)
        if not 1 <= len(kvs) <= 3:
            raise ValueError("space dimension must be 1, 2 or 3")
        for kv in kvs:
            if not hasattr(kv, "knots") or not hasattr(kv, "degree"):
                raise TypeError("knotvectors must be KnotVector instances")
        object.__setattr__(self, "knotvectors", kvs)

    @classmethod
    def from_levels(cls, levels, degree, regularity, grading=1.0):
        return cls(tuple(dyadic_level_knots(lv, degree, regularity, grading) for lv in levels))

    @property
    def d(self) -> int:
        return len(self.knotvectors)

    @property
    def dims(self) -> tuple:
        return tuple(int(np.asarray(kv.knots).size - kv.degree - 1) for kv in self.knotvectors)

    @property
    def n_dofs(self) -> int:
        return int(np.prod(self.dims))

    def interior_mask(self) -> np.ndarray:
        mask = np.zeros(self.dims, dtype=bool)
        mask[tuple(slice(1, n - 1) for n in self.dims)] = True
        return mask

    def interior_dofs(self) -> np.ndarray:
        return np.flatnonzero(self.interior_mask().ravel())

    def boundary_dofs(self) -> np.ndarray:
        return np.flatnonzero(~self.interior_mask().ravel())

    def eval_grid(self, coeffs, points_per_dir, gradient=False):
        """Device evaluation of one coefficient vector on a tensor grid."""
        coeffs = np.asarray(coeffs, dtype=np.float64)
        if coeffs.size != self.n_dofs:
            raise ValueError(f"coefficient vector has {coeffs.size} entries, space has {self.n_dofs}")
        batch = space_batch([(self, 1)])
        try:
            batch.set_coefficients(coeffs.ravel())
            return batch.combine_grid(points_per_dir, gradient=gradient, comp=0)
        finally:
            batch.close()


def _regularity_of(kvs) -> int:
    """Common C^r of a set of knot vectors (device supports one r per batch)."""
    p = kvs[0].degree
    mus = set()
    for kv in kvs:
        if kv.degree != p:
            raise ValueError("all directions / components must share one degree on the device path")
        k = np.asarray(kv.knots)
        uniq, counts = np.unique(k, return_counts=True)
        mus.update(int(c) for c in counts[1:-1])
    if len(mus) > 1:
        raise ValueError("mixed interior knot multiplicities are not supported on the device path")
    return p - (mus.pop() if mus else 1)


def space_batch(space_coef_pairs, patch=None, forcing_id=_lib.FORCING_ZERO, quad_points=None,
                host_forcing=None) -> Batch:
    """A handle whose terms are given by explicit spaces (knot tables keyed by
    pseudo-levels: one id per distinct knot vector and axis)."""
    from .geometry import unit_hypercube

    spaces = [s for s, _ in space_coef_pairs]
    d = spaces[0].d
    kvs_all = [kv for s in spaces for kv in s.knotvectors]
    p = kvs_all[0].degree
    r = _regularity_of(kvs_all)
    ids = [dict() for _ in range(d)]
    tables, terms = {}, []
    for s, c in space_coef_pairs:
        if s.d != d:
            raise ValueError("spaces of one batch must share the dimension")
        beta = []
        for k, kv in enumerate(s.knotvectors):
            bp = np.unique(np.asarray(kv.knots, dtype=np.float64))
            key = bp.tobytes()
            if key not in ids[k]:
                ids[k][key] = len(ids[k])
                tables[(k, ids[k][key])] = bp
            beta.append(ids[k][key])
        terms.append((tuple(beta), int(c)))
    spec = PlanSpec(d, p, r, int(quad_points or p + 1), tuple(terms), tables,
                    patch if patch is not None else unit_hypercube(d), forcing_id)
    return Batch(spec, host_forcing=host_forcing)


class QuadGrid:
    """Tensor Gauss grid on the graded dyadic cells of ``levels``.

    Per-axis points and weights are built with the reference's numpy
    expressions (assembly.py:161-169); mapping, det J and the error
    quadrature run on the device (``analysis.error_norms``).
    """

    def __init__(self, patch, levels, quad_points, grading=1.0):
        d = patch.dim if hasattr(patch, "dim") else len(patch.knotvectors)
        levels = tuple(int(lv) for lv in levels)
        if len(levels) != d:
            raise ValueError(f"expected {d} levels, got {len(levels)}")
        gn, gw = gauss_rule(quad_points)
        pts, wts = [], []
        for lv in levels:
            bp = dyadic_level_knots(lv, 1, 0, grading).breakpoints
            h = np.diff(bp)
            pts.append((bp[:-1, None] + h[:, None] * gn[None, :]).ravel())
            wts.append((h[:, None] * gw[None, :]).ravel())
        self.patch = patch
        self.levels = levels
        self.grading = float(grading)
        self.quad_points = int(quad_points)
        self.points_per_dir = pts
        self.weights_per_dir = wts
        self.grid_shape = tuple(p.size for p in pts)

    @property
    def n_points(self) -> int:
        return int(np.prod(self.grid_shape))


@dataclass
class AssembledSystem:
    matrix: object
    rhs: np.ndarray
    space: DiscreteSpace
    interior: np.ndarray

    def expand(self, interior_coeffs) -> np.ndarray:
        full = np.zeros(self.space.n_dofs)
        full[self.interior] = interior_coeffs
        return full


def assemble_poisson(space: DiscreteSpace, patch, forcing, quad_points=None, kernel=None) -> AssembledSystem:
    """Device assembly of one space; returns the interior CSR and load."""
    from .analysis import forcing_id_of

    if kernel is not None:
        raise NotImplementedError("the device path assembles with its own kernels (kernel= is a CPU hook)")
    interior = space.interior_dofs()
    if interior.size == 0:
        raise EmptyInteriorError(f"space of shape {space.dims} has no interior degrees of freedom")
    fid = forcing_id_of(forcing)
    batch = space_batch([(space, 1)], patch=patch, forcing_id=fid, quad_points=quad_points,
                        host_forcing=forcing if fid == _lib.FORCING_HOST else None)
    try:
        batch.assemble()
        mat, rhs = batch.export_csr(0)
    finally:
        batch.close()
    return AssembledSystem(mat, rhs, space, interior)
