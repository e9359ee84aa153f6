"""Host-side logic: plans, knots, quadrature, scheduling, forcing registry."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1707_09598_b200 import analysis as A
from paper_1707_09598_b200 import _lib
from paper_1707_09598_b200.combination import (CombinationPlan, baseline_plan, combination_coefficients,
                                               general_coefficients, is_downward_closed)
from paper_1707_09598_b200.pipeline import gauss_rule
from paper_1707_09598_b200.scheduler import RunReport, lpt_partition, optimized_makespan
from paper_1707_09598_b200.splines import (KnotVector, dyadic_level_knots, grade_point,
                                           one_sided_level_knots)


@pytest.mark.parametrize("d,w,n", [(2, 6, 9), (3, 7, 31), (2, 8, 13), (2, 9, 15), (3, 12, 136)])
def test_baseline_plan_counts(d, w, n):
    plan = baseline_plan(d, w)
    assert len(plan) == n
    assert sum(c for _, c in plan.terms) == 1
    assert plan.betas == sorted(plan.betas)
    for beta, c in plan.terms:
        t = w - sum(beta)
        assert min(beta) >= 1 and 0 <= t <= d - 1
        from math import comb
        assert c == (-1) ** t * comb(d - 1, t)


def test_combination_coefficients_layers():
    plan = combination_coefficients(3, 4)
    assert set(plan.coefficients.values()) == {1, -2}
    assert sum(plan.coefficients.values()) == 1
    small = combination_coefficients(2, 1)
    assert small.terms == (((0, 0), -1), ((0, 1), 1), ((1, 0), 1))


def test_general_coefficients_matches_simplex():
    for d, lv in ((2, 3), (3, 2)):
        from paper_1707_09598_b200.combination import simplex_set
        assert general_coefficients(simplex_set(d, lv)).terms == combination_coefficients(d, lv).terms
    with pytest.raises(ValueError):
        general_coefficients([(1, 0)])
    assert not is_downward_closed([(1, 1), (0, 0)])


def test_plan_validation():
    with pytest.raises(ValueError):
        CombinationPlan(2, (((0, 0), 2),))
    with pytest.raises(ValueError):
        CombinationPlan(2, ())
    with pytest.raises(ValueError):
        CombinationPlan(2, (((0, 0), 1), ((0, 0), 0)))
    p = CombinationPlan(2, (((1, 0), 1), ((0, 1), 1), ((0, 0), -1)))
    assert p.betas == [(0, 0), (0, 1), (1, 0)]


def test_knots_exact():
    for lv in range(0, 13):
        kv = dyadic_level_knots(lv, 3, 2)
        assert np.array_equal(kv.breakpoints, np.arange(2**lv + 1) / 2**lv)
        assert kv.n == 2**lv + 3
    kv = dyadic_level_knots(3, 2, 0)
    assert kv.n == 1 + 2 + 7 * 2 + 1 - 1 or kv.n == 2 + 1 + 7 * 2
    g = grade_point(np.linspace(0, 1, 9), 3.0)
    assert g[0] == 0.0 and g[-1] == 1.0 and np.all(np.diff(g) > 0)
    os_ = one_sided_level_knots(4, 2, 1, 3.0)
    n = 16
    assert np.array_equal(os_.breakpoints, (np.arange(n + 1) / n) ** 3)
    hi = one_sided_level_knots(4, 2, 1, 3.0, toward="high")
    assert np.allclose(hi.breakpoints, 1 - os_.breakpoints[::-1], atol=0)
    with pytest.raises(ValueError):
        KnotVector(2, (0.0, 0.0, 0.5, 1.0, 1.0))


def test_gauss_rule():
    n, w = gauss_rule(2)
    np.testing.assert_allclose(n, [0.5 - 1 / (2 * np.sqrt(3)), 0.5 + 1 / (2 * np.sqrt(3))])
    np.testing.assert_allclose(w, [0.5, 0.5])
    for q in range(1, 11):
        n, w = gauss_rule(q)
        assert abs(w.sum() - 1) < 1e-14
        k = 2 * q - 1
        assert abs(np.sum(w * n**k) - 1 / (k + 1)) < 1e-13
    with pytest.raises(ValueError):
        gauss_rule(11)


def test_makespan_and_partition():
    assert optimized_makespan([4.0, 3.0, 2.0, 1.0], 2) == pytest.approx(5.0)
    assert optimized_makespan([], 3) == 0.0
    with pytest.raises(ValueError):
        optimized_makespan([1.0], 0)
    parts = lpt_partition([5, 1, 4, 2, 3], 2)
    assert sorted(sum(parts, [])) == [0, 1, 2, 3, 4]
    assert lpt_partition([5, 1, 4, 2, 3], 2) == parts      # deterministic
    rep = RunReport((((1, 1), 10, 0.5), ((1, 2), 20, 0.25)), 1.0)
    assert rep.serial_time == 0.75 and rep.total_dofs == 30 and rep.max_component_dofs == 20
    assert rep.optimized_time(1) == pytest.approx(0.75)
    assert rep.optimized_time(2) == pytest.approx(0.5)


def _fd_laplacian(u, x, h=1e-4):
    out = np.zeros(x.shape[0])
    for m in range(x.shape[1]):
        e = np.zeros(x.shape[1]); e[m] = h
        out += (u(x + e) - 2 * u(x) + u(x - e)) / h**2
    return out


@pytest.mark.parametrize("u,f,g,d", [
    (A.sin_product_solution, A.sin_product_forcing, A.sin_product_gradient, 2),
    (A.sin_product_solution, A.sin_product_forcing, A.sin_product_gradient, 3),
    (A.exp_bubble_solution, A.exp_bubble_forcing, A.exp_bubble_gradient, 3),
    (A.cube_solution, A.cube_forcing, A.cube_gradient, 3),
    (A.annulus_solution_2d, A.annulus_forcing_2d, A.annulus_gradient_2d, 2),
])
def test_closed_forms_consistent(u, f, g, d):
    x = np.random.default_rng(3).uniform(0.2, 0.8, size=(50, d))
    np.testing.assert_allclose(-_fd_laplacian(u, x), f(x), atol=2e-5 * max(1, np.abs(f(x)).max()))
    h = 1e-6
    fd = np.stack([(u(x + h * np.eye(d)[m]) - u(x - h * np.eye(d)[m])) / (2 * h) for m in range(d)], axis=-1)
    np.testing.assert_allclose(g(x), fd, atol=1e-7)


def test_annulus_polar_closed_form():
    r = np.random.default_rng(4).uniform(1.1, 1.9, 40)
    th = np.random.default_rng(5).uniform(0.1, 1.4, 40)
    x = np.stack([r * np.cos(th), r * np.sin(th)], axis=1)
    np.testing.assert_allclose(A.annulus_polar_solution(x), (r**2 - 1) * (r**2 - 4) * np.sin(2 * th), atol=1e-12)
    np.testing.assert_allclose(-_fd_laplacian(A.annulus_polar_solution, x), A.annulus_polar_forcing(x), atol=1e-4)


def test_forcing_registry():
    assert A.forcing_id_of(A.sin_product_forcing) == _lib.FORCING_SIN_PRODUCT
    assert A.forcing_id_of(lambda x: x[:, 0]) == _lib.FORCING_HOST
    assert A.forcing_id_of(None) == _lib.FORCING_ZERO

    def fake():
        pass
    fake.__module__, fake.__qualname__ = "sparseiga.analysis", "annulus_forcing_2d"
    assert A.forcing_id_of(fake) == _lib.FORCING_ANNULUS_2D
