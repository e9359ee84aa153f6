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

__all__ = ["Interface", "MultipatchProblem", "lshape_problem", "MultipatchSolution", "MultipatchSession",
           "run_multipatch_plan", "multipatch_structures", "patch_grid"]


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

    def __init__(self, problem, plan, batches, iters, relres, bnd_iters, owner=None):
        self.problem, self.plan, self.batches = problem, plan, batches
        self.iters, self.relres, self.bnd_iters = iters, relres, bnd_iters
        self._owner = owner

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
        if self._owner is not None:
            self._owner.close()
            self._owner = None
        else:
            for b in self.batches:
                b.close()


def _csr_from_entries(rows, cols, srcs, seq, rrows, rsrcs, rseq, nrows, ncols):
    """CSR structure + per-entry source lists from flat entry arrays: keys
    sorted by (row, col), each key's sources in insertion order (seq), so the
    device sums them in a fixed order (deterministic)."""
    o = np.lexsort((seq, cols, rows))
    rows, cols, srcs = rows[o], cols[o], srcs[o]
    new = np.ones(rows.size, dtype=bool)
    new[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    key_first = np.nonzero(new)[0]
    nnz = int(key_first.size)
    start = np.append(key_first, rows.size).astype(np.int64)
    krow, kcol = rows[key_first], cols[key_first]
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(rowptr, krow + 1, 1)
    rowptr = np.cumsum(rowptr)
    ro = np.lexsort((rseq, rrows))
    rrows, rsrcs = rrows[ro], rsrcs[ro]
    rstart = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(rstart, rrows + 1, 1)
    rstart = np.cumsum(rstart)
    return dict(nrows=nrows, ncols=ncols, nnz=nnz, rowptr=rowptr, col=kcol.astype(np.int32), src_start=start,
                src_idx=srcs.astype(np.int64), rhs_start=rstart, rhs_idx=rsrcs.astype(np.int64))


def multipatch_structures(dims, glue, p):
    """Integer bookkeeping of a multipatch plan (host, once): the source
    layout of the device-computed full patch stencils / loads and Dirichlet
    edge moments, and the CSR structures of the glued interior (AI),
    interior-boundary (AB) and boundary-projection (BB) systems with their
    fixed-order contribution lists.  ``dims[c][pi]`` = (n_x, n_y) of
    component c on patch pi, ``glue[c]`` its ``_Glue``."""
    ncomp, npatch = len(dims), len(dims[0])
    W = 2 * p + 1
    # source layout: per (component, patch) full stencil [W*W][rows] + load [rows]
    src_off, total = {}, 0
    for c in range(ncomp):
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            src_off[(c, pi)] = total
            total += nx * ny * W * W + nx * ny
    eoff, etot = {}, 0
    for c in range(ncomp):
        for (pi, axis, side) in glue[c].dir_sides:
            n = dims[c][pi][1 - axis]
            eoff[(c, pi, axis, side)] = etot
            etot += n * W + n

    # ---- CSR structures + contribution lists, vectorised (numpy)
    AIl, ABl, BBl = ([], [], [], []), ([], [], [], []), ([], [], [], [])
    AIr, BBr = ([], [], []), ([], [], [])
    seq0 = 0
    offI, offB = [0], [0]
    for c in range(ncomp):
        g = glue[c]
        baseI, baseB = offI[-1], offB[-1]
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            o = src_off[(c, pi)]
            rows = nx * ny
            gp = g.gpos[g.base[pi]:g.base[pi] + rows]
            r = np.arange(rows)
            ix, iy = r // ny, r % ny
            inter = gp < g.nI
            AIr[0].append(baseI + gp[inter])
            AIr[1].append(o + rows * W * W + r[inter])
            AIr[2].append(seq0 + r[inter] * (W * W + 1))
            sx, sy = np.meshgrid(np.arange(W), np.arange(W), indexing="ij")
            sx, sy = sx.ravel(), sy.ravel()
            jx = ix[:, None] + sx[None, :] - p
            jy = iy[:, None] + sy[None, :] - p
            ok = inter[:, None] & (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny)
            gr = np.broadcast_to(gp[:, None], ok.shape)[ok]
            gc = gp[np.clip(jx, 0, nx - 1) * ny + np.clip(jy, 0, ny - 1)][ok]
            sidx = (o + (sx * W + sy)[None, :] * rows + r[:, None])[ok]
            sq = (seq0 + r[:, None] * (W * W + 1) + 1 + np.arange(W * W)[None, :])[ok]
            mI = gc < g.nI
            for tgt, m, cbase in ((AIl, mI, baseI), (ABl, ~mI, baseB - g.nI)):
                tgt[0].append(baseI + gr[m])
                tgt[1].append(cbase + gc[m])
                tgt[2].append(sidx[m])
                tgt[3].append(sq[m])
            seq0 += rows * (W * W + 1)
        for (pi, axis, side) in g.dir_sides:
            o = eoff[(c, pi, axis, side)]
            n = dims[c][pi][1 - axis]
            gl = np.array([g.gpos[d] - g.nI for d in g.side_dofs(pi, axis, side)], dtype=np.int64)
            i = np.arange(n)
            BBr[0].append(baseB + gl)
            BBr[1].append(o + n * W + i)
            BBr[2].append(seq0 + i * (2 * p + 2))
            jj = i[:, None] + np.arange(-p, p + 1)[None, :]
            ok = (jj >= 0) & (jj < n)
            BBl[0].append(np.broadcast_to((baseB + gl)[:, None], ok.shape)[ok])
            BBl[1].append(baseB + gl[np.clip(jj, 0, n - 1)][ok])
            BBl[2].append((o + i[:, None] * W + (jj - i[:, None] + p))[ok])
            BBl[3].append((seq0 + i[:, None] * (2 * p + 2) + 1 + np.arange(2 * p + 1)[None, :])[ok])
            seq0 += n * (2 * p + 2)
        offI.append(baseI + g.nI)
        offB.append(baseB + g.nB)
    NI, NB = offI[-1], offB[-1]
    cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, dtype=np.int64))
    AIc = _csr_from_entries(*(cat(x) for x in AIl), *(cat(x) for x in AIr), NI, NI)
    ABc = _csr_from_entries(*(cat(x) for x in ABl), np.zeros(0, np.int64), np.zeros(0, np.int64),
                            np.zeros(0, np.int64), NI, NB)
    BBc = _csr_from_entries(*(cat(x) for x in BBl), *(cat(x) for x in BBr), NB, NB)
    return dict(src_off=src_off, eoff=eoff, src_total=total, esrc_total=etot, AI=AIc, AB=ABc, BB=BBc,
                NI=NI, NB=NB, offI=offI, offB=offB)


class MultipatchSession:
    """cfg4 driver with the integer bookkeeping done ONCE: per-patch handles
    (one per patch, every component), the global C0 numbering of every
    component, the CSR structures of the glued interior / interior-boundary /
    boundary-projection systems with their fixed-order contribution lists,
    all uploaded to the device at construction (the multipatch analogue of
    the handle's component table).  ``solve()`` then runs device work only:
    per-patch assembly, full patch stencils, Dirichlet edge moments, the
    gathered-sum values, two batched CSR PCG solves and the expansion back
    to per-patch coefficients."""

    def __init__(self, plan, problem: MultipatchProblem, quad_points=None, rtol=1e-13, maxit=0):
        import torch

        from .analysis import solution_id_of
        from .scheduler import make_spec

        self.lib = lib = _lib.load()
        self.plan, self.problem, self.rtol, self.maxit = plan, problem, rtol, maxit
        self.dev = dev = torch.device("cuda", torch.cuda.current_device())
        f64, i64 = torch.float64, torch.int64
        terms = tuple(plan.terms)
        self.ncomp = ncomp = len(terms)
        p = problem.degree
        self.p, self.W = p, 2 * p + 1
        W = self.W
        self.sid = solution_id_of(problem.dirichlet)
        if self.sid is None:
            raise ValueError("Dirichlet data must be a registered closed form")
        import dataclasses
        self.batches = []
        for pi, patch in enumerate(problem.patches):
            prob1 = _PatchProblem(patch, problem.forcing, p, problem.regularity)
            spec = make_spec(terms, prob1, quad_points, knot_rule=problem.knot_rules[pi])
            # the patch handles only assemble (gluing and solves run here): no
            # FD preconditioner set-up on their side streams
            self.batches.append(Batch(dataclasses.replace(spec, flags=_lib.FLAG_ASSEMBLY_ONLY)))
        self.npatch = npatch = len(self.batches)
        dims = [[tuple(int(x) for x in self.batches[pi].dims[c]) for pi in range(npatch)] for c in range(ncomp)]
        glue = [_Glue(dims[c], problem) for c in range(ncomp)]
        self.dims = dims
        st = multipatch_structures(dims, glue, p)
        self.src_off, self.eoff = st["src_off"], st["eoff"]
        AIc, ABc, BBc = st["AI"], st["AB"], st["BB"]
        NI, NB, offI, offB = st["NI"], st["NB"], st["offI"], st["offB"]
        self.src = torch.zeros(max(st["src_total"], 1), dtype=f64, device=dev)
        self.esrc = torch.zeros(max(st["esrc_total"], 1), dtype=f64, device=dev)
        self.NI, self.NB, self.offI, self.offB = NI, NB, offI, offB

        def to_dev(a, dt=i64):
            return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)

        self._csr = {}
        for name, csr in (("I", AIc), ("B", ABc), ("M", BBc)):
            self._csr[name] = dict(
                nnz=csr["nnz"], nrows=csr["nrows"], start=to_dev(csr["src_start"]), idx=to_dev(csr["src_idx"]),
                rstart=to_dev(csr["rhs_start"]), ridx=to_dev(csr["rhs_idx"]), rowptr=to_dev(csr["rowptr"]),
                col=to_dev(csr["col"], torch.int32), val=torch.zeros(max(csr["nnz"], 1), dtype=f64, device=dev),
                rhs=torch.zeros(max(csr["nrows"], 1), dtype=f64, device=dev))
        self.d_offI, self.d_offB = to_dev(offI), to_dev(offB)
        self.xI = torch.zeros(max(NI, 1), dtype=f64, device=dev)
        self.xB = torch.zeros(max(NB, 1), dtype=f64, device=dev)
        self.allv = torch.zeros(NI + NB, dtype=f64, device=dev)
        # per-patch expansion maps (global position -> full per-patch vectors)
        self.expand_idx, self.full = [], []
        for pi in range(npatch):
            idx = []
            for c in range(ncomp):
                g = glue[c]
                nx, ny = dims[c][pi]
                gp = g.gpos[g.base[pi]:g.base[pi] + nx * ny]
                idx.append(np.where(gp < g.nI, offI[c] + gp, NI + offB[c] + gp - g.nI))
            idxd = to_dev(np.concatenate(idx))
            self.expand_idx.append(idxd)
            self.full.append(torch.zeros(idxd.numel(), dtype=f64, device=dev))
        # Dirichlet edges per patch handle (batched edge-moment launches)
        self.edge_lists = []
        for pi in range(npatch):
            rows = [(c, 1 - axis, side, o) for (c, pj, axis, side), o in self.eoff.items() if pj == pi]
            if not rows:
                self.edge_lists.append(None)
                continue
            e = to_dev(np.array([r[:3] for r in rows], dtype=np.int32), torch.int32)
            o = to_dev(np.array([r[3] for r in rows], dtype=np.int64))
            maxq = max(self.batches[pi].spec.quad_points * 2 ** int(plan.terms[r[0]][0][r[1]]) for r in rows)
            self.edge_lists.append((e, o, len(rows), maxq))
        self.stream = ct.c_void_p(self.batches[0].stream_ptr)
        torch.cuda.synchronize()

    def _values(self, name, source):
        lib, cs, st = self.lib, self._csr[name], self.stream
        _lib.check(lib.sgiga_gather_sum(st, cs["nnz"], ct.c_void_p(cs["start"].data_ptr()),
                                        ct.c_void_p(cs["idx"].data_ptr()), ct.c_void_p(source.data_ptr()),
                                        ct.c_void_p(cs["val"].data_ptr())))
        _lib.check(lib.sgiga_gather_sum(st, cs["nrows"], ct.c_void_p(cs["rstart"].data_ptr()),
                                        ct.c_void_p(cs["ridx"].data_ptr()), ct.c_void_p(source.data_ptr()),
                                        ct.c_void_p(cs["rhs"].data_ptr())))

    def _pcg(self, name, off, x, rhs, n):
        cs = self._csr[name]
        it = np.zeros(self.ncomp, dtype=np.int32)
        rr = np.zeros(self.ncomp, dtype=np.float64)
        x.zero_()
        _lib.check(self.lib.sgiga_csr_pcg(self.stream, self.ncomp, ct.c_void_p(off.data_ptr()), n,
                                          ct.c_void_p(cs["rowptr"].data_ptr()), ct.c_void_p(cs["col"].data_ptr()),
                                          ct.c_void_p(cs["val"].data_ptr()), ct.c_void_p(rhs.data_ptr()),
                                          ct.c_void_p(x.data_ptr()), float(self.rtol), int(self.maxit),
                                          _lib.ptr(it, ct.c_int32), _lib.ptr(rr, ct.c_double)))
        return it, rr

    def solve(self) -> "MultipatchSession":
        """One device pass: assemble, glue, lift, solve, expand."""
        import torch

        lib, W = self.lib, self.W
        for b in self.batches:
            b.assemble()
        for c in range(self.ncomp):
            for pi in range(self.npatch):
                nx, ny = self.dims[c][pi]
                o = self.src_off[(c, pi)]
                _lib.check(lib.sgiga_full_patch_system(self.batches[pi].h, c, ct.c_void_p(self.src.data_ptr() + 8 * o),
                                                       ct.c_void_p(self.src.data_ptr() + 8 * (o + nx * ny * W * W))))
        for pi, el in enumerate(self.edge_lists):
            if el is None:
                continue
            e, o, ne, maxq = el
            _lib.check(lib.sgiga_edge_projection_batch(self.batches[pi].h, ne, ct.c_void_p(e.data_ptr()),
                                                       ct.c_void_p(o.data_ptr()), maxq, self.sid,
                                                       ct.c_void_p(self.esrc.data_ptr())))
        torch.cuda.synchronize()   # the patch handles' streams -> the solve stream
        self._values("I", self.src)
        self._values("B", self.src)
        self._values("M", self.esrc)
        itB, rrB = self._pcg("M", self.d_offB, self.xB, self._csr["M"]["rhs"], self.NB)   # L2 projection of the data
        cI, cB = self._csr["I"], self._csr["B"]
        _lib.check(lib.sgiga_csr_spmv_sub(self.stream, self.NI, ct.c_void_p(cB["rowptr"].data_ptr()),
                                          ct.c_void_p(cB["col"].data_ptr()), ct.c_void_p(cB["val"].data_ptr()),
                                          ct.c_void_p(self.xB.data_ptr()), ct.c_void_p(cI["rhs"].data_ptr())))
        itI, rrI = self._pcg("I", self.d_offI, self.xI, cI["rhs"], self.NI)
        # acceptance: the reference's 1e-10 (linsolve.py:49-53) is the target of
        # the residual-replacement restarts; the one-sided (j/n)^3 grading makes
        # cells ~4e-6 wide (kappa ~ 1e11) and leaves the FP64 residual noise
        # floor at ~1e-10 on the most anisotropic components, so 1e-9 is accepted
        for name, it, rr in (("boundary projection", itB, rrB), ("interior", itI, rrI)):
            if np.any(it < 0) or not np.all(np.isfinite(rr)) or np.any(rr > 1e-9):
                from .errors import LinearSolveError
                raise LinearSolveError(f"multipatch {name} solve failed: iters {it.tolist()}, relres {rr.tolist()}")
        # ---- expansion to per-patch full coefficient vectors (device gather)
        self.allv[: self.NI].copy_(self.xI[: self.NI])
        self.allv[self.NI:].copy_(self.xB[: self.NB])
        torch.cuda.synchronize()
        for pi in range(self.npatch):
            idxd, full = self.expand_idx[pi], self.full[pi]
            _lib.check(lib.sgiga_gather(self.stream, idxd.numel(), ct.c_void_p(idxd.data_ptr()),
                                        ct.c_void_p(self.allv.data_ptr()), ct.c_void_p(full.data_ptr())))
            torch.cuda.synchronize()
            _lib.check(lib.sgiga_set_coefficients_device(self.batches[pi].h, ct.c_void_p(full.data_ptr())))
        torch.cuda.synchronize()
        self.iters, self.relres, self.bnd_iters = itI, rrI, itB
        return self

    def solution(self) -> MultipatchSolution:
        return MultipatchSolution(self.problem, self.plan, self.batches, self.iters, self.relres, self.bnd_iters,
                                  owner=self)

    def close(self):
        for b in self.batches:
            b.close()
        self.batches = []


def run_multipatch_plan(plan, problem: MultipatchProblem, quad_points=None, rtol=1e-13, maxit=0):
    """Assemble, glue, lift and solve every component of ``plan`` on the
    patches (one-shot MultipatchSession); returns a MultipatchSolution."""
    sess = MultipatchSession(plan, problem, quad_points, rtol, maxit)
    try:
        sess.solve()
    except Exception:
        sess.close()
        raise
    return sess.solution()


class _PatchProblem:
    """The per-patch view make_spec needs (patch, forcing, degree, regularity)."""

    def __init__(self, patch, forcing, degree, regularity):
        self.patch, self.forcing, self.degree, self.regularity = patch, forcing, degree, regularity
        self.grading = 1.0
