"""GPU parity, round 2: kernel-1 tables, solver failure semantics, cfg4
per-patch systems, gamma sweep, batch-composition independence and the
pass-pipelining invariants.  Needs a B200: run with ``-m gpu``.

Goldens come from the reference itself (tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as ct
import hashlib

import numpy as np
import pytest

from conftest import normwise, probe_vector, rel_l2
from paper_1707_09598_b200 import _lib, configs
from paper_1707_09598_b200 import analysis as A
from paper_1707_09598_b200.errors import LinearSolveError
from paper_1707_09598_b200.geometry import unit_hypercube
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import PlanSession, make_spec

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------------------
# kernel 1 on the device vs the reference's _direction_tables, bitwise
# ---------------------------------------------------------------------------
def test_basis_tables_device_bitwise(golden):
    """assembly._direction_tables (assembly.py:209-234): values, derivatives,
    Gauss points and weights of every golden knot vector, read back from the
    device tables kernel 1 wrote -- bit for bit."""
    g = golden("basis")
    for i in range(int(g["ncases"])):
        p, r, lv, gr = (float(x) for x in g[f"c{i}_meta"])
        p, r, lv = int(p), int(r), int(lv)
        prob = A.BenchmarkProblem(f"basis{i}", unit_hypercube(1), A.constant_one, p, r, grading=gr)
        b = Batch(make_spec((((lv,), 1),), prob, p + 1))
        try:
            b.assemble()
            vals, ders, pts, wts = b.basis_table(0, lv)
        finally:
            b.close()
        assert np.array_equal(vals, g[f"c{i}_vals"]), f"case {i}: values"
        assert np.array_equal(ders, g[f"c{i}_ders"]), f"case {i}: derivatives"
        assert np.array_equal(pts, g[f"c{i}_pts"]), f"case {i}: Gauss points"
        assert np.array_equal(wts, g[f"c{i}_wts"]), f"case {i}: weights"


def test_basis_tables_device_bitwise_3d_plan():
    """The same tables inside a 3-D plan: every (axis, level) of cfg2 equals
    the 1-D evaluation of the same knot vector (dedup by (axis, level))."""
    cfg = configs.get_config("cfg2")
    b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    try:
        b.assemble()
        for lv in sorted({beta[0] for beta in cfg.plan.betas}):
            one = Batch(make_spec((((lv,), 1),), A.BenchmarkProblem("t", unit_hypercube(1), A.constant_one, 3, 2),
                                  cfg.quad_points))
            try:
                one.assemble()
                ref = one.basis_table(0, lv)
            finally:
                one.close()
            for axis in range(3):
                if any(beta[axis] == lv for beta in cfg.plan.betas):
                    got = b.basis_table(axis, lv)
                    assert all(np.array_equal(x, y) for x, y in zip(got, ref))
    finally:
        b.close()


# ---------------------------------------------------------------------------
# solver failure semantics (linsolve.py:47-53) driven through the device
# ---------------------------------------------------------------------------
def test_not_converged_raises_linear_solve_error(monkeypatch):
    """Jacobi-PCG capped at one iteration cannot reach 1e-13: the device
    verdict must surface as LinearSolveError (linsolve.py:49-53)."""
    monkeypatch.setenv("SGIGA_NO_FD", "1")
    cfg = configs.get_config("cfg2")
    b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    try:
        b.assemble()
        with pytest.raises(LinearSolveError, match="did not converge"):
            b.solve(rtol=1e-13, maxit=1)
        # the handle stays usable: a full solve afterwards converges
        it, rr = b.solve(rtol=1e-13)
        assert np.all(rr <= 1e-10) and np.all(it >= 1)
    finally:
        b.close()


def test_fd_path_not_converged_raises():
    """Same verdict on the FD-preconditioned path (annulus: P != A, needs
    more than one iteration)."""
    cfg = configs.get_config("cfg3")
    b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    try:
        b.assemble()
        with pytest.raises(LinearSolveError):
            b.solve(rtol=1e-13, maxit=1)
    finally:
        b.close()


def test_non_finite_forcing_raises_linear_solve_error():
    """A forcing that yields NaN makes the solution non-finite: LinearSolveError
    (linsolve.py:47-48), through the one-call pass as well."""
    def nan_forcing(x):
        f = np.ones(x.shape[0])
        f[::7] = np.nan
        return f

    prob = A.BenchmarkProblem("nan", unit_hypercube(2), nan_forcing, 2, 1)
    spec = make_spec((((3, 2), 1), ((2, 3), 1)), prob, 3)
    b = Batch(spec, host_forcing=nan_forcing)
    try:
        b.assemble()
        with pytest.raises(LinearSolveError, match="non-finite"):
            b.solve(rtol=1e-13)
        with pytest.raises(LinearSolveError):
            b.run(np.random.default_rng(0).random((64, 2)))
    finally:
        b.close()


def test_pipelined_failure_is_sticky():
    """A pipelined pass that failed before the last one is still reported by
    the wait (the status of pass k must not be overwritten by
    pass k+1)."""
    cfg = configs.get_config("cfg1")
    b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    pts = np.ascontiguousarray(cfg.points(256))
    import torch
    pin = torch.empty(pts.shape, dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(pts))
    outs = [torch.empty(256, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    try:
        b.run_host_async(pin.numpy(), outs[0].numpy(), rtol=1e-30, maxit=1)   # cannot converge
        b.run_host_async(pin.numpy(), outs[1].numpy(), rtol=1e-13)            # converges
        with pytest.raises(LinearSolveError, match="earlier pipelined pass"):
            b.run_wait()
        # consumed: the next verdict is clean
        b.run_host_async(pin.numpy(), outs[1].numpy(), rtol=1e-13)
        b.run_wait()
    finally:
        b.close()


def test_failed_pass_leaves_no_stale_sort_state():
    """a pass rejected after the point sort was enqueued must
    not corrupt the next sorted combine (stale cell cursors)."""
    cfg = configs.get_config("cfg2")
    pts = cfg.points(4096)
    spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
    ref = Batch(spec)
    b = Batch(spec)
    try:
        want = ref.run(pts)
        with pytest.raises(ValueError):
            b.run(pts, rtol=0.0)
        with pytest.raises(LinearSolveError):
            b.run(pts, rtol=1e-30, maxit=1)
        got = b.run(pts)
        assert np.array_equal(got, want)
        got2 = b.run(pts)
        assert np.array_equal(got2, want)
    finally:
        ref.close()
        b.close()


def test_sessions_do_not_share_scratch():
    """two sessions with passes in flight on the same host
    thread stage points / values in their OWN buffers."""
    import torch
    c1, c2 = configs.get_config("cfg1"), configs.get_config("cfg3")
    s1 = PlanSession(c1.plan, c1.problem, c1.quad_points)
    s2 = PlanSession(c2.plan, c2.problem, c2.quad_points)
    try:
        p1, p2 = c1.points(2048), c2.points(4096)
        w1, w2 = s1.run(p1), s2.run(p2)
        pins = []
        for p in (p1, p2):
            t = torch.empty(p.shape, dtype=torch.float64, pin_memory=True)
            t.copy_(torch.from_numpy(p))
            pins.append(t)
        o1 = torch.empty(len(p1), dtype=torch.float64, pin_memory=True)
        o2 = torch.empty(len(p2), dtype=torch.float64, pin_memory=True)
        for _ in range(3):
            s1.submit(pins[0].numpy(), o1.numpy())
            s2.submit(pins[1].numpy(), o2.numpy())
        s1.wait()
        s2.wait()
        assert np.array_equal(o1.numpy(), w1) and np.array_equal(o2.numpy(), w2)
    finally:
        s1.close()
        s2.close()


# ---------------------------------------------------------------------------
# a component's bits do not depend on the batch it is solved in (the
# multi-GPU shard of a plan computes what the full plan computes)
# ---------------------------------------------------------------------------
def test_subset_batch_bitwise_equals_full_batch():
    cfg = configs.get_config("cfg5")
    terms = tuple(cfg.plan.terms)
    pts = cfg.points(1024)
    full = Batch(make_spec(terms, cfg.problem, cfg.quad_points))
    pick = [0, 7, 29, 64, 100, 135]
    sub = Batch(make_spec(tuple(terms[i] for i in pick), cfg.problem, cfg.quad_points))
    try:
        full.assemble()
        full.solve()
        vf = full.combine_points(pts, per_component=True)
        sub.assemble()
        sub.solve()
        vs = sub.combine_points(pts, per_component=True)
        cf, cs = full.coefficients(), sub.coefficients()
        for k, i in enumerate(pick):
            assert np.array_equal(vs[k], vf[i]), f"component {terms[i][0]}"
            assert np.array_equal(sub.component_coefficients(cs, k), full.component_coefficients(cf, i))
    finally:
        full.close()
        sub.close()


# ---------------------------------------------------------------------------
# gamma_sweep (reference analysis.py:485-528)
# ---------------------------------------------------------------------------
def test_gamma_sweep_matches_reference(golden):
    g = golden("gamma")
    rows, recs = A.gamma_sweep(2, [1.0, 2.0], [1, 2, 3], methods=("sparse", "tensor"), degree=2)
    assert [r.gamma for r in rows] == list(g["rows_gamma"])
    assert [r.method for r in rows] == [str(x) for x in g["rows_method"]]
    np.testing.assert_allclose([r.l2_rate for r in rows], g["rows_l2_rate"], rtol=1e-6)
    np.testing.assert_allclose([r.h1_semi_rate for r in rows], g["rows_h1_rate"], rtol=1e-6)
    assert [r.level for r in recs] == list(g["rec_level"])
    assert [r.n_components for r in recs] == list(g["rec_ncomp"])
    assert [r.dofs_total for r in recs] == list(g["rec_dofs"])
    np.testing.assert_allclose([r.l2_error for r in recs], g["rec_l2"], rtol=1e-6)
    np.testing.assert_allclose([r.h1_semi_error for r in recs], g["rec_h1"], rtol=1e-6)


# ---------------------------------------------------------------------------
# cfg4: per-patch single-patch systems pinned to the reference
# ---------------------------------------------------------------------------
def _digest(indptr, indices):
    h = hashlib.sha256()
    h.update(np.asarray(indptr, dtype=np.int64).tobytes())
    h.update(np.asarray(indices, dtype=np.int64).tobytes())
    return h.hexdigest()


def _full_patch_csr(lib, b, c, nx, ny, p):
    """sgiga_full_patch_system (device, boundary rows included) -> CSR in the
    reference's C order, exact zeros dropped, sorted columns."""
    import scipy.sparse as sps
    import torch
    W = 2 * p + 1
    rows = nx * ny
    dst = torch.zeros(rows * W * W + rows, dtype=torch.float64, device="cuda")
    _lib.check(lib.sgiga_full_patch_system(b.h, c, ct.c_void_p(dst.data_ptr()),
                                           ct.c_void_p(dst.data_ptr() + 8 * rows * W * W)))
    torch.cuda.synchronize()
    st = dst[: rows * W * W].cpu().numpy().reshape(W, W, nx, ny)
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    r_l, c_l, v_l = [], [], []
    for sx in range(W):
        for sy in range(W):
            jx, jy = ix + sx - p, iy + sy - p
            ok = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny) & (st[sx, sy] != 0.0)
            r_l.append((ix * ny + iy)[ok])
            c_l.append((jx * ny + jy)[ok])
            v_l.append(st[sx, sy][ok])
    m = sps.csr_matrix((np.concatenate(v_l), (np.concatenate(r_l), np.concatenate(c_l))), shape=(rows, rows))
    m.sort_indices()
    return m


@pytest.mark.parametrize("graded", [False, True])
def test_cfg4_patch_systems_match_reference(golden, graded):
    """Each cfg4 patch's single-patch system on its own (one-sided graded)
    knots: the full stiffness the multipatch path glues (reference
    full_stiffness, assembly.py:393-398) and the homogeneous-Dirichlet
    interior system (assemble_poisson, assembly.py:357-390) -- patterns
    bit-exact, values <= 1e-12 norm-wise.  Gluing / lifting stay unpinned."""
    from paper_1707_09598_b200.multipatch import _PatchProblem, lshape_problem
    g = golden("cfg4")
    cfg = configs.get_multipatch_config("cfg4_graded" if graded else "cfg4")
    prob = lshape_problem(graded=graded)
    assert [tuple(b) for b in g["betas"]] == list(cfg.plan.betas)
    lib = _lib.load()
    tag = "g" if graded else "u"
    p = prob.degree
    for pi, patch in enumerate(prob.patches):
        spec = make_spec(tuple(cfg.plan.terms), _PatchProblem(patch, prob.forcing, p, prob.regularity), None,
                         knot_rule=prob.knot_rules[pi])
        b = Batch(spec)
        try:
            b.assemble()
            for c in range(len(cfg.plan)):
                key = f"{tag}{c}_{pi}"
                nx, ny = (int(x) for x in b.dims[c])
                m = _full_patch_csr(lib, b, c, nx, ny, p)
                assert m.nnz == int(g[f"{key}_nnz"]), key
                assert _digest(m.indptr, m.indices) == str(g[f"{key}_digest"]), key
                assert normwise(m @ probe_vector(7 * c + pi, m.shape[0]), g[f"{key}_Av"]) <= 1e-12, key
                if f"{key}_data" in g:
                    assert normwise(m.data, g[f"{key}_data"]) <= 1e-12
                A_, _ = b.export_csr(c)
                A_.sort_indices()
                assert A_.nnz == int(g[f"{key}_int_nnz"]), key
                assert _digest(A_.indptr, A_.indices) == str(g[f"{key}_int_digest"]), key
                assert normwise(A_ @ probe_vector(7 * c + pi + 3, A_.shape[0]), g[f"{key}_int_Av"]) <= 1e-12
        finally:
            b.close()


# ---------------------------------------------------------------------------
# cfg2: every permutation class of the plan (one stored component each)
# ---------------------------------------------------------------------------
def test_cfg2_permutation_classes_match_reference(golden):
    g = golden("cfg2")
    cfg = configs.get_config("cfg2")
    b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    try:
        b.assemble()
        classes = {tuple(sorted(beta)) for beta in cfg.plan.betas}
        seen = {tuple(sorted(cfg.plan.betas[int(i)])) for i in g["stored"]}
        assert classes <= seen
        for i in g["stored"]:
            A_, rhs = b.export_csr(int(i))
            assert A_.nnz == int(g[f"k{i}_nnz"])
            assert normwise(A_ @ probe_vector(i, A_.shape[0]), g[f"k{i}_Av"]) <= 1e-12
            assert normwise(rhs, g[f"k{i}_rhs"]) <= 1e-12
    finally:
        b.close()


# ---------------------------------------------------------------------------
# cfg5's comparison point: the full tensor-grid solve at 2^6 per direction
# ---------------------------------------------------------------------------
@pytest.mark.slow
def test_cfg5_tensor_matches_reference(golden):
    """CombinationPlan(3, (((6,6,6),1),)) (reference analysis.py:317-320):
    287 496 interior rows, 189 M nnz.  Element matrices and load from the
    reference's own kernel; the golden solution is the LABELLED scipy
    Jacobi-PCG restatement at rtol 1e-13 (reference spsolve is infeasible,
    SURVEY 8(c)); see tests/golden/make_golden_tensor.py."""
    g = golden("cfg5_tensor")
    cfg = configs.get_config("cfg5_tensor")
    b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
    try:
        b.assemble()
        A_, rhs = b.export_csr(0)
        assert A_.shape[0] == int(g["rows"]) and A_.nnz == int(g["nnz"])
        mx = float(g["maxabs"])
        for k, r in enumerate(g["full_rows"]):
            s, e = A_.indptr[r], A_.indptr[r + 1]
            assert np.array_equal(A_.indices[s:e], g[f"row{k}_cols"]), f"row {r} pattern"
            assert np.max(np.abs(A_.data[s:e] - g[f"row{k}_vals"])) <= 1e-12 * mx
        Av = A_ @ np.random.default_rng(1234).standard_normal(A_.shape[0])
        dots = [np.random.default_rng(5000 + k).standard_normal(A_.shape[0]) for k in range(3)]
        assert normwise(Av[g["sample_rows"]], g["Av_sample"]) <= 1e-12
        assert abs(np.linalg.norm(Av) - g["Av_norm"]) <= 1e-12 * g["Av_norm"]
        np.testing.assert_allclose([w @ Av for w in dots], g["Av_dots"], rtol=0, atol=1e-11 * g["Av_norm"] * 600)
        assert normwise(rhs[g["sample_rows"]], g["b_sample"]) <= 1e-12
        np.testing.assert_allclose([w @ rhs for w in dots], g["b_dots"], rtol=0, atol=1e-11 * g["b_norm"] * 600)
        del A_
        it, rr = b.solve(rtol=1e-13)
        assert rr[0] <= 1e-12 and 1 <= it[0] <= int(g["cg_iterations"])
        coef = b.coefficients()
        assert abs(np.linalg.norm(coef) - g["coef_norm"]) <= 1e-9 * g["coef_norm"]
        assert normwise(coef[g["coef_sample_idx"]], g["coef_sample"]) <= 1e-9
        vals = b.combine_points(g["points"])
        assert rel_l2(vals, g["combined"]) <= 1e-9
        sid = A.solution_id_of(cfg.problem.solution)
        l2, h1 = b.error_norms(cfg.grid().points_per_dir, cfg.grid().weights_per_dir, sid)
        np.testing.assert_allclose([l2, h1], g["errors"], rtol=5e-4)   # 3 significant digits
    finally:
        b.close()


def test_distributed_plan_step_world1_bitwise():
    """DistributedPlan (the per-step form bench.py --gpus N uses: per-component
    values on the device, NCCL all-gather, device plan-order sum) at world 1
    equals the single-GPU combine bitwise, step after step."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1707_09598_b200.combination import evaluate_combined_points
    from paper_1707_09598_b200.distributed import DistributedPlan
    from paper_1707_09598_b200.scheduler import run_plan

    cfg = configs.get_config("cfg2")
    pts = cfg.points(4096)
    sols, _ = run_plan(cfg.plan, cfg.problem)
    ref = evaluate_combined_points(cfg.plan, sols, pts)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        dp = DistributedPlan(cfg.plan, cfg.problem, cfg.quad_points)
        pd = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
        for _ in range(3):
            assert np.array_equal(dp.step(pd).cpu().numpy(), ref)
        dp.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("graded", [False, True])
def test_batched_edge_projection_matches_per_edge(graded):
    """sgiga_edge_projection_batch (one launch per patch, per-point map /
    tangent / Dirichlet data shared) == sgiga_edge_projection_system per
    edge, bitwise (same operations, same order)."""
    import dataclasses

    import torch

    from paper_1707_09598_b200.analysis import solution_id_of
    from paper_1707_09598_b200.multipatch import _PatchProblem, lshape_problem
    prob = lshape_problem(graded=graded)
    cfg = configs.get_multipatch_config("cfg4_graded" if graded else "cfg4")
    lib = _lib.load()
    sid = solution_id_of(prob.dirichlet)
    p, W = prob.degree, 2 * prob.degree + 1
    for pi, patch in enumerate(prob.patches):
        spec = make_spec(tuple(cfg.plan.terms), _PatchProblem(patch, prob.forcing, p, prob.regularity), None,
                         knot_rule=prob.knot_rules[pi])
        b = Batch(dataclasses.replace(spec, flags=_lib.FLAG_ASSEMBLY_ONLY))
        try:
            b.assemble()
            edges, offs, tot, maxq = [], [], 0, 0
            for c in range(len(cfg.plan)):
                for axis in (0, 1):
                    for side in (0, 1):
                        n = int(b.dims[c][1 - axis])
                        edges.append((c, 1 - axis, side))
                        offs.append(tot)
                        tot += n * W + n
                        maxq = max(maxq, 3 * 2 ** int(cfg.plan.betas[c][1 - axis]))
            ref = torch.zeros(tot, dtype=torch.float64, device="cuda")
            for (c, ax, side), o in zip(edges, offs):
                n = int(b.dims[c][ax])
                _lib.check(lib.sgiga_edge_projection_system(b.h, c, ax, side, sid,
                                                            ct.c_void_p(ref.data_ptr() + 8 * o),
                                                            ct.c_void_p(ref.data_ptr() + 8 * (o + n * W))))
            got = torch.zeros(tot, dtype=torch.float64, device="cuda")
            e = torch.as_tensor(np.array(edges, dtype=np.int32), device="cuda")
            od = torch.as_tensor(np.array(offs, dtype=np.int64), device="cuda")
            _lib.check(lib.sgiga_edge_projection_batch(b.h, len(edges), ct.c_void_p(e.data_ptr()),
                                                       ct.c_void_p(od.data_ptr()), maxq, sid,
                                                       ct.c_void_p(got.data_ptr())))
            torch.cuda.synchronize()
            assert torch.equal(got, ref)
        finally:
            b.close()


# ---------------------------------------------------------------------------
# fused true residual of the line-FD PCG on Kronecker box systems
# ---------------------------------------------------------------------------
def test_fused_true_residual_matches_host_residual():
    """On box geometries the line-FD PCG reports ||b - A x|| / ||b|| without a
    sweep of its own: b - (A x_k + alpha A p_k), both products taken in the
    iteration's sweep (k_pcg_fdl<.., FUSED>), plus the rounding bound
    u || |A| |x_k| || of the last update.  The reported value must bound the
    residual of the stored coefficients recomputed on the host in extended
    precision from the exported CSR (linsolve.py:49-53), and exceed it by no
    more than twice that rounding bound."""
    cfg = configs.get_config("cfg5")
    terms = (((8, 2, 2), 1), ((5, 4, 3), 1), ((2, 7, 3), -2))
    spec = make_spec(terms, cfg.problem, cfg.quad_points)
    b = Batch(spec)
    try:
        b.assemble()
        it, rr = b.solve(rtol=1e-13)
        assert np.all(it >= 2), it          # the fused product was exercised
        full = b.coefficients()
        for c in range(b.n_comp):
            A_, rhs = b.export_csr(c)
            x = b.component_coefficients(full, c).reshape(tuple(b.dims[c]))
            x = x[tuple(slice(1, -1) for _ in range(spec.d))].ravel()
            # extended-precision A x row by row (scipy has no longdouble SpMV)
            prod = A_.data.astype(np.longdouble) * x[A_.indices].astype(np.longdouble)
            Ax = np.add.reduceat(prod, A_.indptr[:-1])
            nb = np.linalg.norm(rhs.astype(np.longdouble))
            ref = float(np.linalg.norm(Ax - rhs.astype(np.longdouble)) / nb)
            bound = float(2.0 ** -53 * np.linalg.norm(abs(A_) @ np.abs(x)) / nb)
            assert ref <= 1e-12                 # recurrence 1e-13; linsolve.py accepts 1e-10
            assert ref <= rr[c] * (1 + 1e-6) + 1e-17, (c, rr[c], ref, bound)
            assert rr[c] <= ref + 2.0 * bound + 1e-17, (c, rr[c], ref, bound)
    finally:
        b.close()
