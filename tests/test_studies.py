"""Surplus / profit and convergence-study drivers
against the reference's own results (tests/golden/studies.npz, written by
tests/golden/make_golden.py from the reference's profit_table and
convergence_study)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1707_09598_b200 import analysis as A
from paper_1707_09598_b200 import combination as C
from paper_1707_09598_b200 import studies as S


# ---- host logic (CPU) ----------------------------------------------------------
def test_binary_shifts_order_and_signs():
    got = list(S._binary_shifts((2, 0, 1)))
    # itertools.product order, beta itself first, negative levels dropped
    assert got == [(1, (2, 0, 1)), (-1, (2, 0, 0)), (-1, (1, 0, 1)), (1, (1, 0, 0))]
    assert list(S._binary_shifts((0, 0))) == [(1, (0, 0))]


def test_fit_rate_and_errors():
    lv = [1, 2, 3, 4]
    err = [2.0 ** (-3 * j) * 5 for j in lv]
    rate, steps = S.fit_rate(lv, err)
    assert rate == pytest.approx(3.0)
    assert np.allclose(steps, 3.0)
    with pytest.raises(ValueError):
        S.fit_rate([1, 2], [1.0, 0.5])
    with pytest.raises(ValueError):
        S.fit_rate([1, 2, 3], [1.0, 0.0, 0.5])


def test_convergence_csv_round_trip(tmp_path):
    recs = [S.ConvergenceRecord("sparse", 2, 2, 1, 1.0, j, 3 * j, 10 * j, 4 * j, 1.0 / j, 2.0 / j, 0.1 * j,
                                {1: 0.1 * j, 4: 0.05 * j}) for j in (1, 2, 3)]
    path = tmp_path / "conv.csv"
    S.write_convergence_csv(path, recs, cores=(1, 4))
    back, cores = S.read_convergence_csv(path)
    assert cores == [1, 4] and back == recs
    assert recs[1].h == 0.25
    rows = [S.GammaSweepRow(2.0, "sparse", 2, 3, 2, 3.9, 2.9)]
    S.write_gamma_csv(tmp_path / "g.csv", rows)
    assert (tmp_path / "g.csv").read_text().splitlines()[0] == "gamma,method,d,p,r,l2_rate,h1_semi_rate"


def test_profit_and_study_argument_errors():
    prob = A.polynomial_cube_problem(2)
    with pytest.raises(ValueError):
        C.profit_table(prob, (1, -1))
    with pytest.raises(ValueError):
        C.profit_table(prob, (1, 1, 1))
    with pytest.raises(ValueError):
        A.convergence_study(prob, "sparse", [])
    with pytest.raises(ValueError):
        A.convergence_study(prob, "sparse", [-1])
    with pytest.raises(ValueError):
        S._plan_for("dense", 2, 3)
    row = C.ProfitRow((1, 2), 0.5, 10)
    assert row.profit == 0.05


# ---- device (GPU) --------------------------------------------------------------
PROFIT_CASES = {
    "annulus2_p2": (lambda: A.regular_annulus_problem(2, degree=2), 2),
    "cube3_p2": (lambda: A.polynomial_cube_problem(3, degree=2), (1, 1, 2)),
    "const2_p2_g2": (lambda: A.constant_forcing_problem(2, grading=2.0, degree=2), 2),
}


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(PROFIT_CASES))
def test_profit_table_matches_reference(golden, key):
    g = golden("studies")
    make, bmax = PROFIT_CASES[key]
    rows = C.profit_table(make(), bmax)
    assert np.array_equal(np.array([r.beta for r in rows]), g[f"profit_{key}_beta"])
    assert np.array_equal(np.array([r.dofs for r in rows]), g[f"profit_{key}_dofs"])
    ref = g[f"profit_{key}_l2"]
    got = np.array([r.surplus_l2 for r in rows])
    # surpluses span many orders of magnitude; the tiny ones are solve noise
    scale = ref.max()
    assert np.all(np.abs(got - ref) <= 1e-7 * ref + 1e-11 * scale), (got, ref)


@pytest.mark.gpu
def test_surplus_norm_single_index_and_cache(golden):
    g = golden("studies")
    prob = A.regular_annulus_problem(2, degree=2)
    cache = {}
    norm, dofs = C.surplus_norm(prob, (2, 1), cache)
    betas = [tuple(b) for b in g["profit_annulus2_p2_beta"]]
    i = betas.index((2, 1))
    assert dofs == int(g["profit_annulus2_p2_dofs"][i])
    assert norm == pytest.approx(float(g["profit_annulus2_p2_l2"][i]), rel=1e-7)
    assert set(cache) == {(2, 1), (2, 0), (1, 1), (1, 0)}


STUDIES = {
    "annulus2_sparse": (lambda: A.regular_annulus_problem(2, degree=2), "sparse"),
    "annulus2_tensor": (lambda: A.regular_annulus_problem(2, degree=2), "tensor"),
    "const2_sparse": (lambda: A.constant_forcing_problem(2, grading=1.0, degree=2), "sparse"),
}


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(STUDIES))
def test_convergence_study_matches_reference(golden, key):
    g = golden("studies")
    make, method = STUDIES[key]
    levels = [int(x) for x in g[f"conv_{key}_levels"]]
    recs = A.convergence_study(make(), method, levels, cores=(1, 2))
    assert [r.n_components for r in recs] == list(g[f"conv_{key}_ncomp"])
    assert [r.dofs_total for r in recs] == list(g[f"conv_{key}_dofs"])
    # L2 / H1 to 3 significant digits (Appendix A), in practice ~1e-9
    assert np.allclose([r.l2_error for r in recs], g[f"conv_{key}_l2"], rtol=1e-6, atol=0)
    assert np.allclose([r.h1_semi_error for r in recs], g[f"conv_{key}_h1"], rtol=1e-6, atol=0)
    assert all(r.time_serial_s > 0 and r.times_cores[1] == pytest.approx(r.time_serial_s) for r in recs)


@pytest.mark.gpu
def test_evaluator_error_norms_match_plan_form():
    from paper_1707_09598_b200 import configs

    cfg = configs.get_config("cfg1")
    from paper_1707_09598_b200.scheduler import run_plan

    sols, _ = run_plan(cfg.plan, cfg.problem)
    grid = cfg.grid()
    a = A.error_norms(cfg.plan, sols, cfg.problem, grid)
    b = A.error_norms(A.combined_evaluator(cfg.plan, sols),
                      A.analytic_evaluator(cfg.problem.solution, cfg.problem.solution_gradient), grid)
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    # spline vs spline: a component against itself is zero
    s0 = sols[0]
    z = A.error_norms(A.spline_evaluator(s0.space, s0.coefficients),
                      A.spline_evaluator(s0.space, s0.coefficients), grid)
    assert z == (0.0, 0.0)


@pytest.mark.gpu
def test_gamma_sweep_runs_and_fits():
    rows, recs = A.gamma_sweep(2, [1.0], [1, 2, 3], methods=("sparse",), degree=2)
    assert len(rows) == 1 and len(recs) == 3
    assert rows[0].l2_rate > 0 and rows[0].h1_semi_rate > 0
