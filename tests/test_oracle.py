"""Pin the CPU oracle (oracle/sgiga_oracle.c) to the reference.

Every check compares the oracle with golden vectors that the reference
itself produced (tests/golden/make_golden.py) or with the reference's own
known-answer tests.  CPU only.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import normwise, probe_vector, rel_l2
from oracle import oracle as O
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.scheduler import make_spec
from paper_1707_09598_b200.splines import dyadic_level_knots


def test_basis_tables_bitwise(golden):
    g = golden("basis")
    for i in range(int(g["ncases"])):
        p, r, lv, gam = g[f"c{i}_meta"]
        p, r, lv = int(p), int(r), int(lv)
        kv = dyadic_level_knots(lv, p, r, gam)
        assert np.array_equal(kv.knots, g[f"c{i}_knots"]), "host knots must be bitwise"
        vals, ders, offs, pts, wts = O.direction_tables(p, r, kv.breakpoints, p + 1, g[f"c{i}_gn"], g[f"c{i}_gw"])
        assert np.array_equal(vals, g[f"c{i}_vals"])
        assert np.array_equal(ders, g[f"c{i}_ders"])
        assert np.array_equal(offs, g[f"c{i}_offs"])
        assert np.array_equal(pts, g[f"c{i}_pts"])
        assert np.array_equal(wts, g[f"c{i}_wts"])
        for x, f, tab in zip(g[f"c{i}_xs"], g[f"c{i}_first"], g[f"c{i}_tab"]):
            first, t = O.eval_basis(kv.knots, p, x, 1)
            assert first == f
            assert np.array_equal(t, tab)


def test_known_basis_values():
    # reference tests/test_splines.py:141-152 (hat and uniform quadratic)
    from paper_1707_09598_b200.splines import make_open_knot_vector

    kv = make_open_knot_vector(1, [0.0, 0.5, 1.0], 0)
    first, t = O.eval_basis(kv.knots, 1, 0.25, 0)
    assert first == 0 and np.allclose(t[0], [0.5, 0.5])
    kv = make_open_knot_vector(2, [0.0, 1 / 3, 2 / 3, 1.0], 1)
    _, t = O.eval_basis(kv.knots, 2, 0.5, 0)
    assert np.allclose(t[0], [0.125, 0.75, 0.125])
    # right endpoint uses the left limit (splines.py:255-256)
    for p, r in ((1, 0), (2, 1), (3, 2)):
        kv = dyadic_level_knots(2, p, r)
        first, t = O.eval_basis(kv.knots, p, 1.0, 0)
        assert first + p + 1 == kv.n and t[0][-1] == 1.0


def test_partition_of_unity():
    rng = np.random.default_rng(101)
    for _ in range(40):
        p = int(rng.integers(1, 5))
        r = int(rng.integers(0, p))
        kv = dyadic_level_knots(int(rng.integers(0, 6)), p, r, float(rng.choice([1.0, 2.0, 3.0])))
        for x in rng.random(25):
            _, t = O.eval_basis(kv.knots, p, float(x), 1)
            assert np.all(t[0] >= -1e-14)
            assert abs(t[0].sum() - 1.0) < 1e-12
            assert abs(t[1].sum()) < 1e-10


def test_element_kernel_matches_reference(golden):
    g = golden("kernel")
    for d in (1, 2, 3):
        a = np.zeros_like(g[f"d{d}_out_a"])
        b = np.zeros_like(g[f"d{d}_out_b"])
        O.local_poisson_systems(*(g[f"d{d}_{k}"] for k in ("values", "derivs", "elem_index", "qp_index",
                                                           "fn_index", "metric", "load")), a, b)
        np.testing.assert_allclose(a, g[f"d{d}_out_a"], atol=1e-13)
        np.testing.assert_allclose(b, g[f"d{d}_out_b"], atol=1e-13)


def test_element_kernel_rejects_d9():
    d = 9
    with pytest.raises(ValueError):
        O.local_poisson_systems(np.zeros((d, 1, 1, 1)), np.zeros((d, 1, 1, 1)), np.zeros((1, d), np.int64),
                                np.zeros((1, d), np.int32), np.zeros((1, d), np.int32), np.zeros((1, 1, d, d)),
                                np.zeros((1, 1)), np.zeros((1, 1, 1)), np.zeros((1, 1)))


def test_interval_hat_system():
    # reference tests/test_assembly.py:99-103: A = [[4]], b = [0.5]
    from paper_1707_09598_b200.analysis import BenchmarkProblem, constant_one
    from paper_1707_09598_b200.geometry import unit_hypercube

    prob = BenchmarkProblem("hat", unit_hypercube(1), constant_one, 1, 0)
    orc = O.Oracle(make_spec((((1,), 1),), prob))
    A, b = orc.assemble_csr(0)
    np.testing.assert_allclose(A.toarray(), [[4.0]], atol=1e-13)
    np.testing.assert_allclose(b, [0.5], atol=1e-14)


def _config_oracle(name):
    cfg = configs.get_config(name)
    spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
    return cfg, O.Oracle(spec)


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg2"])
def test_config_assembly_matches_reference(golden, name):
    g = golden(name)
    cfg, orc = _config_oracle(name)
    assert np.array_equal(np.array(cfg.plan.betas), g["betas"])
    assert np.array_equal(np.array([c for _, c in cfg.plan.terms]), g["coefs"])
    for i in g["stored"]:
        A, b = orc.assemble_csr(int(i))
        A.sort_indices()
        assert A.nnz == int(g[f"k{i}_nnz"])
        if f"k{i}_indptr" in g:
            assert np.array_equal(A.indptr, g[f"k{i}_indptr"])
            assert np.array_equal(A.indices, g[f"k{i}_indices"])
            assert normwise(A.data, g[f"k{i}_data"]) <= 1e-12
        assert normwise(A @ probe_vector(i, A.shape[0]), g[f"k{i}_Av"]) <= 1e-12
        assert normwise(b, g[f"k{i}_rhs"]) <= 1e-12


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg2"])
def test_config_solution_and_combine(golden, name):
    g = golden(name)
    cfg, orc = _config_oracle(name)
    coefs = orc.run_plan(O.SOLVER_DIRECT)
    assert rel_l2(coefs, g["coefficients"]) <= 1e-11
    vals = orc.combine_points(g["points"])
    assert rel_l2(vals, g["combined"]) <= 1e-9
    grid = cfg.grid()
    sid = __import__("paper_1707_09598_b200.analysis", fromlist=["x"]).solution_id_of(cfg.problem.solution)
    l2, h1 = orc.error_norms(grid.points_per_dir, grid.weights_per_dir, sid)
    np.testing.assert_allclose([l2, h1], g["errors"], rtol=5e-4)   # 3 significant digits


def test_pcg_restatement_agrees_with_direct(golden):
    g = golden("cfg1")
    cfg, orc = _config_oracle("cfg1")
    direct = orc.run_plan(O.SOLVER_DIRECT)
    pcg = orc.run_plan(O.SOLVER_PCG, rtol=1e-13)
    assert rel_l2(pcg, direct) <= 1e-11
    assert np.all(orc.relres <= 1e-12)
