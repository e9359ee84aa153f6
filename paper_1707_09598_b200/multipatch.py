"""Multipatch components with C0 gluing and Dirichlet lifting (BASELINE
cfg4).

The reference solves single-patch problems with homogeneous Dirichlet data
only (SPEC.md:150,208 list multipatch as a non-goal); cfg4 needs an
extension, built here the way GeoPDEs does it (the package the paper used):

* every component beta is the same tensor space on each patch (levels per
  global x / y direction, knots from a per-patch rule: uniform dyadic, or
  one-sided radical grading (j/n)^3 toward the re-entrant corner, mirrored
  where the corner sits at the parametric end);
* conforming interfaces glue the patch functions C0 (one global dof per
  matched pair); every function touching a non-interface side is a
  Dirichlet dof;
* Dirichlet values = L2 projection of the data onto the boundary trace
  space (one SPD system per component over the whole Dirichlet boundary);
* the lifted interior system A_II u_I = b_I - A_IB u_B is solved by batched
  Jacobi-PCG to 1e-13, then expanded back to per-patch full coefficient
  vectors, so combine / error norms run per patch with the existing kernels.

Host work here is integer bookkeeping only (global numbering, CSR
structure, contribution lists); every floating-point step runs on the
device (csrc/k_multipatch.cu).  Parity: against the independent numpy
restatement in oracle/multipatch_oracle.py -- parity unpinned (no reference
code path exists).
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from .pipeline import Batch, gauss_rule
from .splines import dyadic_level_knots, one_sided_level_knots

__all__ = ["Interface", "MultipatchProblem", "lshape_problem", "MultipatchSolution", "run_multipatch_plan",
           "patch_grid"]


@dataclass(frozen=True)
class Interface:
    """Patch ``a``'s side (fixed axis, side) glued to patch ``b``'s side; the
    shared edge runs along the other (2-D) axis with the same orientation."""

    a: int
    a_axis: int
    a_side: int
    b: int
    b_axis: int
    b_side: int


@dataclass(frozen=True)
class MultipatchProblem:
    name: str
    patches: tuple
    degree: int
    regularity: int
    forcing: Callable
    dirichlet: Callable                 # data g on every non-interface side (registered closed form)
    interfaces: tuple
    knot_rules: tuple                   # per patch: (axis, level) -> KnotVector
    solution: Callable | None = None
    solution_gradient: Callable | None = None


def _lshape_rules(degree, regularity, graded):
    if not graded:
        rule = (lambda k, lv: dyadic_level_knots(lv, degree, regularity))
        return (rule, rule, rule)
    # toward the origin: patch 0 = [-1,0]x[0,1] (x high, y low), 1 = [0,1]^2
    # (x low, y low), 2 = [-1,0]x[-1,0] (x high, y high)
    towards = (("high", "low"), ("low", "low"), ("high", "high"))

    def make(tw):
        return lambda k, lv: one_sided_level_knots(lv, degree, regularity, 3.0, tw[k])
    return tuple(make(tw) for tw in towards)


def lshape_problem(graded=False, degree=2, regularity=None) -> MultipatchProblem:
    """BASELINE cfg4: u = r^(2/3) sin(2 theta / 3) on the L-shape, f = 0."""
    from .analysis import lshape_gradient, lshape_solution, zero_forcing
    from .geometry import lshape_patches

    r = degree - 1 if regularity is None else regularity
    ifaces = (Interface(0, 0, 1, 1, 0, 0),    # x = 0, y in [0, 1]
              Interface(0, 1, 0, 2, 1, 1))    # y = 0, x in [-1, 0]
    return MultipatchProblem("cfg4_lshape" + ("_graded" if graded else ""), lshape_patches(), degree, r,
                             zero_forcing, lshape_solution, ifaces, _lshape_rules(degree, r, graded),
                             lshape_solution, lshape_gradient)


def patch_grid(problem, patch, levels, quad_points):
    """Per-axis Gauss points / weights on the patch's own knots (the error
    grid of cfg4 uses the same -- possibly graded -- knots)."""
    gn, gw = gauss_rule(quad_points)
    pts, wts = [], []
    for k, lv in enumerate(levels):
        bp = problem.knot_rules[patch](k, int(lv)).breakpoints
        h = np.diff(bp)
        pts.append((bp[:-1, None] + h[:, None] * gn[None, :]).ravel())
        wts.append((h[:, None] * gw[None, :]).ravel())
    return pts, wts


class _Glue:
    """Global C0 numbering of one component over the patches (union-find on
    (patch, local C-order dof)) and the Dirichlet / interior split."""

    def __init__(self, dims, problem):
        self.dims = dims                           # per patch (n_x, n_y)
        self.base = np.concatenate([[0], np.cumsum([nx * ny for nx, ny in dims])])
        parent = np.arange(self.base[-1])

        def find(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        def side_dofs(pi, axis, side):
            nx, ny = dims[pi]
            if axis == 0:
                i = nx - 1 if side else 0
                return [self.base[pi] + i * ny + j for j in range(ny)]
            j = ny - 1 if side else 0
            return [self.base[pi] + i * ny + j for i in range(nx)]

        iface_sides = set()
        for f in problem.interfaces:
            la, lb = side_dofs(f.a, f.a_axis, f.a_side), side_dofs(f.b, f.b_axis, f.b_side)
            if len(la) != len(lb):
                raise ValueError("non-conforming interface")
            for u, v in zip(la, lb):
                ru, rv = find(u), find(v)
                if ru != rv:
                    parent[max(ru, rv)] = min(ru, rv)
            iface_sides.add((f.a, f.a_axis, f.a_side))
            iface_sides.add((f.b, f.b_axis, f.b_side))
        roots = np.array([find(i) for i in range(self.base[-1])])
        dirichlet = np.zeros(self.base[-1], dtype=bool)
        self.dir_sides = []
        for pi in range(len(dims)):
            for axis in (0, 1):
                for side in (0, 1):
                    if (pi, axis, side) in iface_sides:
                        continue
                    self.dir_sides.append((pi, axis, side))
                    dirichlet[side_dofs(pi, axis, side)] = True
        root_dir = np.zeros(self.base[-1], dtype=bool)
        np.logical_or.at(root_dir, roots, dirichlet)
        uniq = np.unique(roots)
        is_b = root_dir[uniq]
        self.interior_roots = uniq[~is_b]
        self.bnd_roots = uniq[is_b]
        pos = -np.ones(self.base[-1], dtype=np.int64)
        pos[self.interior_roots] = np.arange(self.interior_roots.size)
        pos[self.bnd_roots] = self.interior_roots.size + np.arange(self.bnd_roots.size)
        self.gpos = pos[roots]                     # local dof -> [interior | boundary] position
        self.nI, self.nB = int(self.interior_roots.size), int(self.bnd_roots.size)
        self.side_dofs = side_dofs


class MultipatchSolution:
    """Solved multipatch plan: per-patch handles holding the full per-patch
    coefficients (combine / error norms run per patch)."""

    def __init__(self, problem, plan, batches, iters, relres, bnd_iters):
        self.problem, self.plan, self.batches = problem, plan, batches
        self.iters, self.relres, self.bnd_iters = iters, relres, bnd_iters

    def combine_points(self, patch, pts):
        return self.batches[patch].combine_points(pts)

    def coefficients(self, patch):
        return self.batches[patch].coefficients()

    def error_norms(self, levels, quad_points):
        """L2 / H1-seminorm errors over the whole L-shape (sum over patches)."""
        from .analysis import solution_id_of

        sid = solution_id_of(self.problem.solution)
        e2 = h2 = 0.0
        for pi, b in enumerate(self.batches):
            pts, wts = patch_grid(self.problem, pi, levels, quad_points)
            l2, h1 = b.error_norms(pts, wts, sid)
            e2 += l2 * l2
            h2 += h1 * h1
        return float(np.sqrt(e2)), float(np.sqrt(h2))

    def close(self):
        for b in self.batches:
            b.close()


def run_multipatch_plan(plan, problem: MultipatchProblem, quad_points=None, rtol=1e-13, maxit=0):
    """Assemble, glue, lift and solve every component of ``plan`` on the
    patches; returns a MultipatchSolution."""
    import torch

    from .analysis import solution_id_of
    from .scheduler import make_spec

    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    f64, i64 = torch.float64, torch.int64
    terms = tuple(plan.terms)
    ncomp = len(terms)
    p = problem.degree
    W = 2 * p + 1
    sid = solution_id_of(problem.dirichlet)
    if sid is None:
        raise ValueError("Dirichlet data must be a registered closed form")

    # ---- per patch: one handle with every component, assembled on the device
    batches = []
    for pi, patch in enumerate(problem.patches):
        prob1 = _PatchProblem(patch, problem.forcing, p, problem.regularity)
        spec = make_spec(terms, prob1, quad_points, knot_rule=problem.knot_rules[pi])
        b = Batch(spec)
        b.assemble()
        batches.append(b)
    npatch = len(batches)
    dims = [[tuple(int(x) for x in batches[pi].dims[c]) for pi in range(npatch)] for c in range(ncomp)]
    glue = [_Glue(dims[c], problem) for c in range(ncomp)]

    # ---- full patch stencils (device) into one concatenated source array
    src_off = {}
    total = 0
    for c in range(ncomp):
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            src_off[(c, pi)] = total
            total += nx * ny * W * W + nx * ny          # stencil + load
    src = torch.zeros(max(total, 1), dtype=f64, device=dev)
    for c in range(ncomp):
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            o = src_off[(c, pi)]
            _lib.check(lib.sgiga_full_patch_system(batches[pi].h, c, ct.c_void_p(src.data_ptr() + 8 * o),
                                                   ct.c_void_p(src.data_ptr() + 8 * (o + nx * ny * W * W))))
    # ---- boundary data moments per Dirichlet side (device)
    eoff, etot = {}, 0
    for c in range(ncomp):
        for (pi, axis, side) in glue[c].dir_sides:
            n = dims[c][pi][1 - axis]
            eoff[(c, pi, axis, side)] = etot
            etot += n * W + n
    esrc = torch.zeros(max(etot, 1), dtype=f64, device=dev)
    for (c, pi, axis, side), o in eoff.items():
        n = dims[c][pi][1 - axis]
        _lib.check(lib.sgiga_edge_projection_system(batches[pi].h, c, 1 - axis, side, sid,
                                                    ct.c_void_p(esrc.data_ptr() + 8 * o),
                                                    ct.c_void_p(esrc.data_ptr() + 8 * (o + n * W))))
    torch.cuda.synchronize()

    # ---- CSR structures + contribution lists (integer bookkeeping)
    AI, AB, BB = _CsrBuilder(), _CsrBuilder(), _CsrBuilder()
    offI, offB = [0], [0]
    for c in range(ncomp):
        g = glue[c]
        baseI, baseB = offI[-1], offB[-1]
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            o = src_off[(c, pi)]
            rows = nx * ny
            gp = g.gpos[g.base[pi]:g.base[pi] + rows]
            for r in range(rows):
                gr = gp[r]
                if gr >= g.nI:
                    continue
                ix, iy = divmod(r, ny)
                AI.add_rhs(baseI + gr, o + rows * W * W + r)
                for sx in range(W):
                    jx = ix + sx - p
                    if jx < 0 or jx >= nx:
                        continue
                    for sy in range(W):
                        jy = iy + sy - p
                        if jy < 0 or jy >= ny:
                            continue
                        gc = gp[jx * ny + jy]
                        s_idx = o + (sx * W + sy) * rows + r
                        if gc < g.nI:
                            AI.add(baseI + gr, baseI + gc, s_idx)
                        else:
                            AB.add(baseI + gr, baseB + gc - g.nI, s_idx)
        for (pi, axis, side) in g.dir_sides:
            o = eoff[(c, pi, axis, side)]
            n = dims[c][pi][1 - axis]
            loc = g.side_dofs(pi, axis, side)
            gl = [g.gpos[d] - g.nI for d in loc]
            for i in range(n):
                BB.add_rhs(baseB + gl[i], o + n * W + i)
                for jj in range(max(0, i - p), min(n, i + p + 1)):
                    BB.add(baseB + gl[i], baseB + gl[jj], o + i * W + (jj - i + p))
        offI.append(baseI + g.nI)
        offB.append(baseB + g.nB)
    NI, NB = offI[-1], offB[-1]

    def to_dev(a, dt=i64):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

    stream = ct.c_void_p(batches[0].stream_ptr)
    AIc, ABc, BBc = AI.finish(NI, NI), AB.finish(NI, NB), BB.finish(NB, NB)

    def values(csr, source):
        start, idx = to_dev(csr["src_start"]), to_dev(csr["src_idx"])
        v = torch.zeros(max(csr["nnz"], 1), dtype=f64, device=dev)
        _lib.check(lib.sgiga_gather_sum(stream, csr["nnz"], ct.c_void_p(start.data_ptr()),
                                        ct.c_void_p(idx.data_ptr()), ct.c_void_p(source.data_ptr()),
                                        ct.c_void_p(v.data_ptr())))
        rstart, ridx = to_dev(csr["rhs_start"]), to_dev(csr["rhs_idx"])
        rv = torch.zeros(max(csr["nrows"], 1), dtype=f64, device=dev)
        _lib.check(lib.sgiga_gather_sum(stream, csr["nrows"], ct.c_void_p(rstart.data_ptr()),
                                        ct.c_void_p(ridx.data_ptr()), ct.c_void_p(source.data_ptr()),
                                        ct.c_void_p(rv.data_ptr())))
        return v, rv, to_dev(csr["rowptr"]), to_dev(csr["col"], torch.int32), (start, idx, rstart, ridx)

    vI, bI, rpI, colI, keep1 = values(AIc, src)
    vB, _, rpB, colB, keep2 = values(ABc, src)
    vM, rM, rpM, colM, keep3 = values(BBc, esrc)

    def pcg(off, rowptr, col, val, rhs, n):
        x = torch.zeros(max(n, 1), dtype=f64, device=dev)
        offd = to_dev(off)
        it = np.zeros(ncomp, dtype=np.int32)
        rr = np.zeros(ncomp, dtype=np.float64)
        _lib.check(lib.sgiga_csr_pcg(stream, ncomp, ct.c_void_p(offd.data_ptr()), n,
                                     ct.c_void_p(rowptr.data_ptr()), ct.c_void_p(col.data_ptr()),
                                     ct.c_void_p(val.data_ptr()), ct.c_void_p(rhs.data_ptr()),
                                     ct.c_void_p(x.data_ptr()), float(rtol), int(maxit),
                                     _lib.ptr(it, ct.c_int32), _lib.ptr(rr, ct.c_double)))
        return x, it, rr

    uB, itB, rrB = pcg(offB, rpM, colM, vM, rM, NB)                 # L2 projection of the data
    _lib.check(lib.sgiga_csr_spmv_sub(stream, NI, ct.c_void_p(rpB.data_ptr()), ct.c_void_p(colB.data_ptr()),
                                      ct.c_void_p(vB.data_ptr()), ct.c_void_p(uB.data_ptr()),
                                      ct.c_void_p(bI.data_ptr())))
    uI, itI, rrI = pcg(offI, rpI, colI, vI, bI, NI)
    # acceptance: the reference's 1e-10 (linsolve.py:49-53) is the target of
    # the residual-replacement restarts; the one-sided (j/n)^3 grading makes
    # cells ~4e-6 wide (kappa ~ 1e11) and leaves the FP64 residual noise floor
    # at ~1e-10 on the most anisotropic components, so 1e-9 is accepted here
    for name, it, rr in (("boundary projection", itB, rrB), ("interior", itI, rrI)):
        if np.any(it < 0) or not np.all(np.isfinite(rr)) or np.any(rr > 1e-9):
            from .errors import LinearSolveError
            raise LinearSolveError(f"multipatch {name} solve failed: iters {it.tolist()}, relres {rr.tolist()}")

    # ---- expansion to per-patch full coefficient vectors (device gather)
    allv = torch.cat([uI[:NI], uB[:NB]])
    for pi in range(npatch):
        idx = []
        for c in range(ncomp):
            g = glue[c]
            nx, ny = dims[c][pi]
            gp = g.gpos[g.base[pi]:g.base[pi] + nx * ny]
            idx.append(np.where(gp < g.nI, offI[c] + gp, NI + offB[c] + gp - g.nI))
        idxd = to_dev(np.concatenate(idx))
        full = torch.zeros(idxd.numel(), dtype=f64, device=dev)
        _lib.check(lib.sgiga_gather(stream, idxd.numel(), ct.c_void_p(idxd.data_ptr()),
                                    ct.c_void_p(allv.data_ptr()), ct.c_void_p(full.data_ptr())))
        torch.cuda.synchronize()
        _lib.check(lib.sgiga_set_coefficients_device(batches[pi].h, ct.c_void_p(full.data_ptr())))
    torch.cuda.synchronize()
    del keep1, keep2, keep3
    return MultipatchSolution(problem, plan, batches, itI, rrI, itB)


class _PatchProblem:
    """The per-patch view make_spec needs (patch, forcing, degree, regularity)."""

    def __init__(self, patch, forcing, degree, regularity):
        self.patch, self.forcing, self.degree, self.regularity = patch, forcing, degree, regularity
        self.grading = 1.0


class _CsrBuilder:
    """CSR structure + per-entry source lists, entries in insertion order
    within a row's column (deterministic fixed-order sums)."""

    def __init__(self):
        self.entries = {}
        self.rhs = {}

    def add(self, r, c, s):
        self.entries.setdefault((r, c), []).append(s)

    def add_rhs(self, r, s):
        self.rhs.setdefault(r, []).append(s)

    def finish(self, nrows, ncols):
        keys = sorted(self.entries)
        rowptr = np.zeros(nrows + 1, dtype=np.int64)
        for r, _ in keys:
            rowptr[r + 1] += 1
        rowptr = np.cumsum(rowptr)
        col = np.array([c for _, c in keys], dtype=np.int32)
        start = np.zeros(len(keys) + 1, dtype=np.int64)
        idx = []
        for k, key in enumerate(keys):
            lst = self.entries[key]
            idx.extend(lst)
            start[k + 1] = start[k] + len(lst)
        rstart = np.zeros(nrows + 1, dtype=np.int64)
        ridx = []
        for r in range(nrows):
            lst = self.rhs.get(r, [])
            ridx.extend(lst)
            rstart[r + 1] = rstart[r] + len(lst)
        return dict(nrows=nrows, ncols=ncols, nnz=len(keys), rowptr=rowptr, col=col, src_start=start,
                    src_idx=np.array(idx, dtype=np.int64), rhs_start=rstart, rhs_idx=np.array(ridx, dtype=np.int64))
