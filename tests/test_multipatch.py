"""Multipatch extension (BASELINE cfg4).

PARITY UNPINNED: the reference has no multipatch code path; the device
path is checked against the independent CPU restatement
(oracle/multipatch_oracle.py) and against exact reproduction of a
biquadratic solution (non-zero Dirichlet data, so the lifting is exercised).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2
from paper_1707_09598_b200 import analysis as A
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.combination import baseline_plan
from paper_1707_09598_b200.multipatch import (Interface, MultipatchProblem, _Glue, _lshape_rules,
                                              _PatchProblem, lshape_problem, run_multipatch_plan)
from paper_1707_09598_b200.scheduler import make_spec


def poly_problem(graded=False):
    """u = x(1-x) y(1-y) on the L-shape: in the p=2 space, u != 0 on the boundary."""
    base = lshape_problem(graded=graded)
    return MultipatchProblem("lshape_poly", base.patches, 2, 1, A.cube_forcing, A.cube_solution,
                             base.interfaces, _lshape_rules(2, 1, graded), A.cube_solution, A.cube_gradient)


def specs_for(problem, plan, q=3):
    return [make_spec(tuple(plan.terms), _PatchProblem(pt, problem.forcing, problem.degree, problem.regularity),
                      q, knot_rule=problem.knot_rules[pi]) for pi, pt in enumerate(problem.patches)]


def physical(patch_index, pts):
    x0, x1, y0, y1 = ((-1, 0, 0, 1), (0, 1, 0, 1), (-1, 0, -1, 0))[patch_index]
    return np.stack([x0 + (x1 - x0) * pts[:, 0], y0 + (y1 - y0) * pts[:, 1]], axis=1)


# ---- host logic (CPU) ----------------------------------------------------------
def test_lshape_glue_counts():
    prob = lshape_problem()
    # level (1, 1), p = 2: 4 x 4 functions per patch; two glued sides of 4
    g = _Glue([(4, 4)] * 3, prob)
    assert g.nI + g.nB == 48 - 8
    # interior: patch-interior 2x2 per patch + the interface functions that
    # touch no Dirichlet side (2 per interface; the shared corner sits on the
    # re-entrant Dirichlet edges)
    assert g.nI == 3 * 4 + 2 + 2
    assert sorted(g.dir_sides) == sorted([(0, 0, 0), (0, 1, 1), (1, 0, 1), (1, 1, 0), (1, 1, 1),
                                          (2, 0, 0), (2, 0, 1), (2, 1, 0)])
    with pytest.raises(ValueError):
        _Glue([(4, 4), (4, 5), (4, 4)], prob)   # the x = 0 interface would join 4 and 5 functions


def test_graded_rules_conform_on_interfaces():
    prob = lshape_problem(graded=True)
    for f in prob.interfaces:
        ea, eb = 1 - f.a_axis, 1 - f.b_axis
        for lv in range(1, 7):
            ka, kb = prob.knot_rules[f.a](ea, lv), prob.knot_rules[f.b](eb, lv)
            assert np.array_equal(ka.breakpoints, kb.breakpoints)
    # graded toward the origin: patch 1 = [0,1]^2 refines at parametric 0
    bp = prob.knot_rules[1](0, 4).breakpoints
    assert bp[1] - bp[0] < bp[-1] - bp[-2]


def test_oracle_reproduces_biquadratic():
    from oracle import multipatch_oracle as MO

    prob = poly_problem()
    plan = baseline_plan(2, 3)
    specs = specs_for(prob, plan)
    coefs = MO.run_plan(specs, prob, 3)
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    for pi in range(3):
        pts = rng.random((64, 2))
        v = O.Oracle(specs[pi]).combine_points(pts, coefs=coefs[pi])
        assert np.max(np.abs(v - A.cube_solution(physical(pi, pts)))) < 1e-12


# ---- device (GPU) --------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("graded", [False, True])
def test_gpu_reproduces_biquadratic(graded):
    prob = poly_problem(graded)
    sol = run_multipatch_plan(baseline_plan(2, 5), prob)
    try:
        rng = np.random.default_rng(6)
        for pi in range(3):
            pts = rng.random((500, 2))
            v = sol.combine_points(pi, pts)
            assert np.max(np.abs(v - A.cube_solution(physical(pi, pts)))) < 1e-11
        l2, h1 = sol.error_norms((4, 4), 3)
        # solver-tolerance level (graded cells near the corner are ~3e-5 wide)
        assert l2 < 1e-11 and h1 < 1e-8
    finally:
        sol.close()


@pytest.mark.gpu
@pytest.mark.parametrize("graded", [False, True])
def test_gpu_matches_multipatch_oracle(graded):
    from oracle import multipatch_oracle as MO
    from oracle import oracle as O

    prob = lshape_problem(graded=graded)
    plan = baseline_plan(2, 5)
    sol = run_multipatch_plan(plan, prob)
    try:
        specs = specs_for(prob, plan)
        ref = MO.run_plan(specs, prob, 3)
        pts = np.random.default_rng(3).random((400, 2))
        for pi in range(3):
            assert rel_l2(sol.coefficients(pi), ref[pi]) <= 1e-10
            v = sol.combine_points(pi, pts)
            assert rel_l2(v, O.Oracle(specs[pi]).combine_points(pts, coefs=ref[pi])) <= 1e-9
        assert np.all(sol.iters > 0)
    finally:
        sol.close()


@pytest.mark.gpu
def test_cfg4_full_runs_and_grading_helps():
    errs = {}
    for name in ("cfg4", "cfg4_graded"):
        cfg = configs.get_multipatch_config(name)
        sol = run_multipatch_plan(cfg.plan, cfg.problem)
        try:
            assert len(cfg.plan) == 15
            errs[name] = sol.error_norms((6, 6), cfg.quad_points)
            v = sol.combine_points(1, cfg.points(256))
            assert np.all(np.isfinite(v))
        finally:
            sol.close()
    # the r^(2/3) corner singularity: one-sided grading toward it lowers the error
    assert errs["cfg4_graded"][0] < errs["cfg4"][0]
    assert errs["cfg4"][0] < 1e-2


def test_interface_dataclass():
    f = Interface(0, 0, 1, 1, 0, 0)
    assert (f.a, f.b) == (0, 1)


def _loop_structures(dims, glue, p):
    """Straightforward restatement of the cfg4 bookkeeping (the round-1 loop
    builder): per-entry source lists in insertion order, keys sorted."""
    W = 2 * p + 1
    ncomp, npatch = len(dims), len(dims[0])
    src_off, total = {}, 0
    for c in range(ncomp):
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            src_off[(c, pi)] = total
            total += nx * ny * W * W + nx * ny
    eoff, etot = {}, 0
    for c in range(ncomp):
        for (pi, axis, side) in glue[c].dir_sides:
            eoff[(c, pi, axis, side)] = etot
            etot += dims[c][pi][1 - axis] * (W + 1)
    mats = {"AI": ({}, {}), "AB": ({}, {}), "BB": ({}, {})}
    offI, offB = [0], [0]
    for c in range(ncomp):
        g = glue[c]
        baseI, baseB = offI[-1], offB[-1]
        for pi in range(npatch):
            nx, ny = dims[c][pi]
            o, rows = src_off[(c, pi)], nx * ny
            gp = g.gpos[g.base[pi]:g.base[pi] + rows]
            for r in range(rows):
                gr = gp[r]
                if gr >= g.nI:
                    continue
                ix, iy = divmod(r, ny)
                mats["AI"][1].setdefault(baseI + gr, []).append(o + rows * W * W + r)
                for sx in range(W):
                    for sy in range(W):
                        jx, jy = ix + sx - p, iy + sy - p
                        if not (0 <= jx < nx and 0 <= jy < ny):
                            continue
                        gc = gp[jx * ny + jy]
                        s_idx = o + (sx * W + sy) * rows + r
                        if gc < g.nI:
                            mats["AI"][0].setdefault((baseI + gr, baseI + gc), []).append(s_idx)
                        else:
                            mats["AB"][0].setdefault((baseI + gr, baseB + gc - g.nI), []).append(s_idx)
        for (pi, axis, side) in g.dir_sides:
            o, n = eoff[(c, pi, axis, side)], dims[c][pi][1 - axis]
            gl = [g.gpos[d] - g.nI for d in g.side_dofs(pi, axis, side)]
            for i in range(n):
                mats["BB"][1].setdefault(baseB + gl[i], []).append(o + n * W + i)
                for jj in range(max(0, i - p), min(n, i + p + 1)):
                    mats["BB"][0].setdefault((baseB + gl[i], baseB + gl[jj]), []).append(o + i * W + (jj - i + p))
        offI.append(baseI + g.nI)
        offB.append(baseB + g.nB)
    return mats, offI, offB, total, etot


@pytest.mark.parametrize("graded", [False, True])
def test_vectorised_multipatch_structures_match_loop_builder(graded):
    """The vectorised bookkeeping of the cfg4 session equals the per-entry
    loop builder: same CSR keys, same source lists in the same order (so the
    device's fixed-order sums are unchanged)."""
    from paper_1707_09598_b200.multipatch import _Glue, multipatch_structures

    cfg = configs.get_multipatch_config("cfg4_graded" if graded else "cfg4")
    prob, p = cfg.problem, cfg.problem.degree
    dims = [[tuple(prob.knot_rules[pi](k, beta[k]).n for k in range(2)) for pi in range(3)]
            for beta in cfg.plan.betas]
    glue = [_Glue(d, prob) for d in dims]
    st = multipatch_structures(dims, glue, p)
    mats, offI, offB, total, etot = _loop_structures(dims, glue, p)
    assert st["offI"] == offI and st["offB"] == offB
    assert st["src_total"] == total and st["esrc_total"] == etot
    for name in ("AI", "AB", "BB"):
        csr = st[name]
        ent, rhs = mats[name]
        keys = sorted(ent)
        assert csr["nnz"] == len(keys)
        rows = np.repeat(np.arange(csr["nrows"]), np.diff(csr["rowptr"]))
        assert [(int(r), int(c)) for r, c in zip(rows, csr["col"])] == keys
        for k, key in enumerate(keys):
            s, e = csr["src_start"][k], csr["src_start"][k + 1]
            assert csr["src_idx"][s:e].tolist() == ent[key]
        for r in range(csr["nrows"]):
            s, e = csr["rhs_start"][r], csr["rhs_start"][r + 1]
            assert csr["rhs_idx"][s:e].tolist() == rhs.get(r, [])
