"""Batched device pipeline: one plan -> one libsgiga handle.

``Batch`` owns the C-ABI handle of one combination plan and exposes the
three phases (assemble, solve, combine) plus the parity exports.  The host
only prepares exact metadata (integer plan, breakpoints, Gauss nodes from
numpy, the homogeneous control net); everything else runs on the GPU.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .geometry import homogeneous_net
from .splines import dyadic_level_knots

__all__ = ["gauss_rule", "Batch", "PlanSpec", "make_desc", "knot_tables_for"]


def gauss_rule(q: int):
    """Gauss-Legendre on [0, 1] (reference assembly.py:41-46, same numpy calls)."""
    if not 1 <= q <= 10:
        raise ValueError(f"quadrature points per direction must be in [1, 10], got {q}")
    nodes, weights = np.polynomial.legendre.leggauss(q)
    return 0.5 * (nodes + 1.0), 0.5 * weights


@dataclass
class PlanSpec:
    """Everything a handle needs, in host arrays."""

    d: int
    degree: int
    regularity: int
    quad_points: int
    terms: tuple            # ((beta, coef), ...) in plan order
    knot_tables: dict       # (axis, key) -> breakpoints; key = level (or table id)
    patch: object           # NurbsPatch-like
    forcing_id: int
    flags: int = 0          # sgiga_flags (include/sgiga.h), e.g. 1 = assembly only


def knot_tables_for(terms, d, degree, regularity, grading=1.0, knot_rule: Callable | None = None):
    """(axis, level) -> breakpoints for every level a plan uses."""
    tables = {}
    for beta, _ in terms:
        for k, lv in enumerate(beta):
            if (k, lv) in tables:
                continue
            if knot_rule is not None:
                kv = knot_rule(k, int(lv))
            else:
                kv = dyadic_level_knots(int(lv), degree, regularity, grading)
            tables[(k, lv)] = np.ascontiguousarray(kv.breakpoints, dtype=np.float64)
    return tables


def make_desc(spec: PlanSpec):
    """struct sgiga_problem_desc for ``spec`` (+ the arrays it points into)."""
    d, n = spec.d, len(spec.terms)
    levels = np.array([list(b) for b, _ in spec.terms], dtype=np.int32).reshape(n, d)
    coefs = np.array([c for _, c in spec.terms], dtype=np.int32)
    max_level = max([int(k[1]) for k in spec.knot_tables] + [int(levels.max()) if levels.size else 0])
    L = max_level + 1
    bp_off = -np.ones(d * L, dtype=np.int64)
    bp_cnt = np.zeros(d * L, dtype=np.int32)
    chunks, pos = [], 0
    for (k, lv), bp in sorted(spec.knot_tables.items()):
        bp_off[k * L + lv] = pos
        bp_cnt[k * L + lv] = bp.size
        chunks.append(bp)
        pos += bp.size
    bps = np.ascontiguousarray(np.concatenate(chunks) if chunks else np.zeros(1))
    gn, gw = gauss_rule(spec.quad_points)
    kvs = spec.patch.knotvectors
    keep = dict(
        levels=levels, coefs=coefs, bp_off=bp_off, bp_cnt=bp_cnt, bps=bps,
        gn=np.ascontiguousarray(gn), gw=np.ascontiguousarray(gw),
        gdeg=np.array([kv.degree for kv in kvs], dtype=np.int32),
        gnk=np.array([np.asarray(kv.knots).size for kv in kvs], dtype=np.int32),
        gk=np.ascontiguousarray(np.concatenate([np.asarray(kv.knots, dtype=np.float64) for kv in kvs])),
        hw=np.ascontiguousarray(homogeneous_net(spec.patch).ravel()),
    )
    K = keep
    desc = _lib.ProblemDesc(
        d, spec.degree, spec.regularity, spec.quad_points, n,
        _lib.ptr(K["levels"], ct.c_int32), _lib.ptr(K["coefs"], ct.c_int32),
        _lib.ptr(K["gn"], ct.c_double), _lib.ptr(K["gw"], ct.c_double),
        max_level, _lib.ptr(K["bp_off"], ct.c_int64), _lib.ptr(K["bp_cnt"], ct.c_int32),
        _lib.ptr(K["bps"], ct.c_double), _lib.ptr(K["gdeg"], ct.c_int32),
        _lib.ptr(K["gnk"], ct.c_int32), _lib.ptr(K["gk"], ct.c_double),
        _lib.ptr(K["hw"], ct.c_double), spec.forcing_id, int(spec.flags),
    )
    return desc, keep


class Batch:
    """Device state of one plan (create -> assemble -> solve -> combine)."""

    def __init__(self, spec: PlanSpec, stream=None, host_forcing: Callable | None = None):
        self.lib = _lib.load()
        self.spec = spec
        self.host_forcing = host_forcing
        self._build_desc(spec)
        h = ct.c_void_p()
        _lib.check(self.lib.sgiga_create(ct.byref(self.desc), stream, ct.byref(h)))
        self.h = h
        n = len(spec.terms)
        dims = np.zeros((n, spec.d), dtype=np.int32)
        offs = np.zeros(n + 1, dtype=np.int64)
        _lib.check(self.lib.sgiga_component_info(self.h, _lib.ptr(dims, ct.c_int32), _lib.ptr(offs, ct.c_int64)))
        self.dims = dims
        self.dof_offsets = offs
        sizes = [ct.c_int64() for _ in range(4)]
        _lib.check(self.lib.sgiga_batch_sizes(self.h, *[ct.byref(s) for s in sizes]))
        self.total_qp, self.total_rows, self.total_dofs, self.total_slots = (int(s.value) for s in sizes)
        self.iters = None
        self.relres = None

    def _build_desc(self, spec: PlanSpec):
        self.desc, self._keep = make_desc(spec)

    @property
    def n_comp(self) -> int:
        return len(self.spec.terms)

    @property
    def stream_ptr(self) -> int:
        return int(self.lib.sgiga_stream(self.h) or 0)

    def upload(self, spec: PlanSpec | None = None):
        """Host->device copy of the problem descriptor (same shape); with
        ``spec`` a new problem replaces the handle's (new forcing, weights,
        ...).  Uploading a byte-identical descriptor is a no-op."""
        if spec is not None:
            desc, keep = make_desc(spec)
            _lib.check(self.lib.sgiga_upload(self.h, ct.byref(desc)))
            self.spec, self.desc, self._keep = spec, desc, keep
            return
        _lib.check(self.lib.sgiga_upload(self.h, ct.byref(self.desc)))

    # ---- phases -------------------------------------------------------------
    def _host_forcing_density(self):
        if self.spec.forcing_id == _lib.FORCING_HOST:
            x = np.empty((self.total_qp, self.spec.d))
            _lib.check(self.lib.sgiga_quad_points_physical(self.h, _lib.ptr(x, ct.c_double)))
            f = np.ascontiguousarray(np.asarray(self.host_forcing(x), dtype=np.float64))
            if f.ndim == 0:
                f = np.full(self.total_qp, float(f))
            if f.shape != (self.total_qp,):
                raise ValueError(f"forcing returned shape {f.shape} for {self.total_qp} points")
            _lib.check(self.lib.sgiga_set_forcing_density(self.h, _lib.ptr(f, ct.c_double)))

    def assemble(self):
        self._host_forcing_density()
        _lib.check(self.lib.sgiga_assemble(self.h))

    def solve(self, rtol: float = 1e-13, maxit: int = 0):
        n = self.n_comp
        it = np.zeros(n, dtype=np.int32)
        rr = np.zeros(n, dtype=np.float64)
        code = self.lib.sgiga_solve(self.h, float(rtol), int(maxit), _lib.ptr(it, ct.c_int32), _lib.ptr(rr, ct.c_double))
        self.iters, self.relres = it, rr
        _lib.check(code)
        return it, rr

    def run(self, pts: np.ndarray | None = None, rtol: float = 1e-13, maxit: int = 0):
        """assemble + solve + combine at ``pts`` in ONE library call (one
        stream synchronisation): run_plan + evaluate_combined
        (scheduler.py:74-96, combination.py:209-236).  Returns the combined
        values (empty when ``pts`` is None)."""
        self._host_forcing_density()
        n = self.n_comp
        it = np.zeros(n, dtype=np.int32)
        rr = np.zeros(n, dtype=np.float64)
        if pts is None:
            pts = np.zeros((0, self.spec.d))
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != self.spec.d:
            raise ValueError(f"points must have shape (n, {self.spec.d})")
        # the [0, 1]^d range check runs on the device (combine kernels ->
        # ValueError through the status word), not as a host pass over pts
        out = np.empty(pts.shape[0])
        code = self.lib.sgiga_run(self.h, float(rtol), int(maxit), pts.ctypes.data, pts.shape[0],
                                  out.ctypes.data, 0, _lib.ptr(it, ct.c_int32), _lib.ptr(rr, ct.c_double))
        self.iters, self.relres = it, rr
        _lib.check(code)
        return out

    def run_device(self, pts_ptr: int, npts: int, out_ptr: int, rtol: float = 1e-13, maxit: int = 0):
        """As run(), with the points and the output resident in HBM."""
        self._host_forcing_density()
        n = self.n_comp
        it = np.zeros(n, dtype=np.int32)
        rr = np.zeros(n, dtype=np.float64)
        code = self.lib.sgiga_run(self.h, float(rtol), int(maxit), pts_ptr, int(npts), out_ptr, 1,
                                  _lib.ptr(it, ct.c_int32), _lib.ptr(rr, ct.c_double))
        self.iters, self.relres = it, rr
        _lib.check(code)

    def run_device_async(self, pts_ptr: int, npts: int, out_ptr: int, rtol: float = 1e-13, maxit: int = 0):
        """Enqueue one run_device pass without synchronising (passes pipeline
        back to back on the device); run_wait() reports the last one."""
        self._host_forcing_density()
        _lib.check(self.lib.sgiga_run_async(self.h, float(rtol), int(maxit), pts_ptr, int(npts), out_ptr))

    def run_components_async(self, pts_ptr: int, npts: int, out_ptr: int, rtol: float = 1e-13, maxit: int = 0):
        """Enqueue assemble + solve + PER-COMPONENT combine (out = n_comp x
        npts device doubles, coefficients not applied) without synchronising:
        the local half of a plan split over ranks."""
        self._host_forcing_density()
        _lib.check(self.lib.sgiga_run_components_async(self.h, float(rtol), int(maxit), pts_ptr, int(npts), out_ptr))

    def run_host_async(self, pts: np.ndarray, out: np.ndarray, rtol: float = 1e-13, maxit: int = 0):
        """Enqueue one end-to-end pass with page-locked HOST buffers (H2D of
        ``pts`` and D2H into ``out`` inside the pass) without synchronising;
        ``out`` is valid after run_wait(), which reports the last pass."""
        self._host_forcing_density()
        if pts.ndim != 2 or pts.shape[1] != self.spec.d or out.shape != (pts.shape[0],):
            raise ValueError(f"points must have shape (n, {self.spec.d}) and out shape (n,)")
        if not (pts.flags.c_contiguous and out.flags.c_contiguous and pts.dtype == np.float64
                and out.dtype == np.float64):
            raise ValueError("points and out must be C-contiguous float64")
        _lib.check(self.lib.sgiga_run_host_async(self.h, float(rtol), int(maxit), pts.ctypes.data,
                                                 pts.shape[0], out.ctypes.data))

    def run_wait(self):
        n = self.n_comp
        it = np.zeros(n, dtype=np.int32)
        rr = np.zeros(n, dtype=np.float64)
        code = self.lib.sgiga_run_wait(self.h, _lib.ptr(it, ct.c_int32), _lib.ptr(rr, ct.c_double))
        self.iters, self.relres = it, rr
        _lib.check(code)

    def coefficients(self) -> np.ndarray:
        out = np.empty(self.total_dofs)
        _lib.check(self.lib.sgiga_coefficients(self.h, _lib.ptr(out, ct.c_double)))
        return out

    def set_coefficients(self, full: np.ndarray):
        full = np.ascontiguousarray(full, dtype=np.float64)
        if full.size != self.total_dofs:
            raise ValueError(f"expected {self.total_dofs} coefficients, got {full.size}")
        _lib.check(self.lib.sgiga_set_coefficients(self.h, _lib.ptr(full, ct.c_double)))

    def component_coefficients(self, flat: np.ndarray, c: int) -> np.ndarray:
        return flat[self.dof_offsets[c]:self.dof_offsets[c + 1]]

    def combine_points(self, pts: np.ndarray, per_component: bool = False) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != self.spec.d:
            raise ValueError(f"points must have shape (n, {self.spec.d})")
        n = pts.shape[0]   # range check on the device (ValueError via the status word)
        out = np.empty((self.n_comp, n) if per_component else n)
        _lib.check(self.lib.sgiga_combine_points(self.h, pts.ctypes.data, n, out.ctypes.data,
                                                 -1 if per_component else 0))
        return out

    def combine_points_device(self, pts_ptr: int, npts: int, out_ptr: int, per_component=False):
        """Inputs/outputs already resident in HBM (raw device pointers)."""
        _lib.check(self.lib.sgiga_combine_points(self.h, pts_ptr, npts, out_ptr, -2 if per_component else 1))

    def combine_grid(self, points_per_dir: Sequence[np.ndarray], gradient=False, comp: int = -1):
        d = self.spec.d
        if len(points_per_dir) != d:
            raise ValueError(f"expected {d} point arrays, got {len(points_per_dir)}")
        arrs = [np.atleast_1d(np.asarray(p, dtype=np.float64)).ravel() for p in points_per_dir]
        for a in arrs:
            if a.size and (a.min() < 0.0 or a.max() > 1.0):
                raise ValueError("evaluation points must lie in [0, 1]")
        npd = np.array([a.size for a in arrs], dtype=np.int64)
        cat = np.ascontiguousarray(np.concatenate(arrs))
        shape = tuple(int(x) for x in npd)
        vals = np.empty(shape)
        grads = np.empty(shape + (d,)) if gradient else None
        _lib.check(self.lib.sgiga_combine_grid(
            self.h, _lib.ptr(cat, ct.c_double), _lib.ptr(npd, ct.c_int64), int(comp),
            _lib.ptr(vals, ct.c_double), _lib.ptr(grads, ct.c_double) if gradient else None))
        return (vals, grads) if gradient else vals

    def error_norms(self, points_per_dir, weights_per_dir, solution_id: int):
        arrs = [np.asarray(p, dtype=np.float64).ravel() for p in points_per_dir]
        wts = [np.asarray(w, dtype=np.float64).ravel() for w in weights_per_dir]
        npd = np.array([a.size for a in arrs], dtype=np.int64)
        cp = np.ascontiguousarray(np.concatenate(arrs))
        cw = np.ascontiguousarray(np.concatenate(wts))
        out = np.zeros(2)
        _lib.check(self.lib.sgiga_error_norms(self.h, _lib.ptr(cp, ct.c_double), _lib.ptr(cw, ct.c_double),
                                              _lib.ptr(npd, ct.c_int64), int(solution_id), _lib.ptr(out, ct.c_double)))
        return float(out[0]), float(out[1])

    def subset_error_norms(self, points_per_dir, weights_per_dir, terms, solution_id=None):
        """L2 / H1-seminorm of sum_t w_t u_{c_t} (minus the closed form
        ``solution_id``; None = against zero) on a tensor quadrature grid;
        ``terms`` = [(component index, weight), ...] in accumulation order."""
        arrs = [np.asarray(p, dtype=np.float64).ravel() for p in points_per_dir]
        wts = [np.asarray(w, dtype=np.float64).ravel() for w in weights_per_dir]
        npd = np.array([a.size for a in arrs], dtype=np.int64)
        cp = np.ascontiguousarray(np.concatenate(arrs))
        cw = np.ascontiguousarray(np.concatenate(wts))
        tc = np.ascontiguousarray([int(c) for c, _ in terms], dtype=np.int32)
        tw = np.ascontiguousarray([float(w) for _, w in terms], dtype=np.float64)
        out = np.zeros(2)
        _lib.check(self.lib.sgiga_subset_error_norms(
            self.h, _lib.ptr(cp, ct.c_double), _lib.ptr(cw, ct.c_double), _lib.ptr(npd, ct.c_int64),
            len(tc), _lib.ptr(tc, ct.c_int32), _lib.ptr(tw, ct.c_double),
            -1 if solution_id is None else int(solution_id), _lib.ptr(out, ct.c_double)))
        return float(out[0]), float(out[1])

    def export_csr(self, comp: int):
        """Interior CSR + rhs of one component (reference row order)."""
        import scipy.sparse as sps

        nnz = ct.c_int64()
        _lib.check(self.lib.sgiga_export_csr(self.h, int(comp), ct.byref(nnz), None, None, None, None))
        rows = int(np.prod(self.dims[comp] - 2)) if np.all(self.dims[comp] > 2) else 0
        indptr = np.zeros(rows + 1, dtype=np.int64)
        indices = np.zeros(max(1, nnz.value), dtype=np.int32)
        data = np.zeros(max(1, nnz.value))
        rhs = np.zeros(max(1, rows))
        _lib.check(self.lib.sgiga_export_csr(self.h, int(comp), ct.byref(nnz), _lib.ptr(indptr, ct.c_int64),
                                             _lib.ptr(indices, ct.c_int32), _lib.ptr(data, ct.c_double),
                                             _lib.ptr(rhs, ct.c_double)))
        n = int(nnz.value)
        mat = sps.csr_matrix((data[:n], indices[:n], indptr), shape=(rows, rows))
        return mat, rhs[:rows]

    def basis_table(self, axis: int, level: int):
        """Kernel 1's device output for one (axis, level): (vals, ders, pts,
        wts) shaped like assembly._direction_tables (assembly.py:209-234)."""
        nel = ct.c_int32(0)
        _lib.check(self.lib.sgiga_basis_table(self.h, axis, level, ct.byref(nel), None, None, None, None))
        n, q, P = nel.value, self.spec.quad_points, self.spec.degree + 1
        vals, ders = np.empty((n, q, P)), np.empty((n, q, P))
        pts, wts = np.empty(n * q), np.empty(n * q)
        _lib.check(self.lib.sgiga_basis_table(self.h, axis, level, ct.byref(nel), _lib.ptr(vals, ct.c_double),
                                              _lib.ptr(ders, ct.c_double), _lib.ptr(pts, ct.c_double),
                                              _lib.ptr(wts, ct.c_double)))
        return vals, ders, pts, wts

    def phase_stats(self):
        ms = np.zeros(3, dtype=np.float32)
        ln = np.zeros(3, dtype=np.int64)
        _lib.check(self.lib.sgiga_phase_stats(self.h, _lib.ptr(ms, ct.c_float), _lib.ptr(ln, ct.c_int64)))
        return ms, ln

    def close(self):
        if getattr(self, "h", None):
            self.lib.sgiga_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # modelled per-component cost used to apportion the batch time
    def component_cost(self) -> np.ndarray:
        n = self.n_comp
        rows = np.prod(np.maximum(self.dims - 2, 0), axis=1).astype(np.float64)
        W = 2 * self.spec.degree + 1
        slots = np.prod(np.minimum(np.maximum(self.dims - 2, 1), W), axis=1).astype(np.float64)
        its = self.iters.astype(np.float64) if self.iters is not None else np.ones(n)
        return (8.0 * slots * rows + 104.0 * rows) * (its + 1.0) + 1.0
