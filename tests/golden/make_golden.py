"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py [--cfg5]

It imports ``sparseiga`` from a scratch copy of /root/reference/pkg with the
Cython kernel built (falls back to the in-place sources with the numpy
kernel), evaluates the reference's own API on the BASELINE configurations'
inputs (SURVEY.md section 8(d) recipes) and writes small .npz fixtures next
to this script.  The fixtures pin both the CPU oracle (tests/test_oracle.py)
and the GPU path (tests/test_gpu_parity.py); nothing at test time reads
/root/reference.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
SCRATCH = Path("/tmp/sgiga_refpkg")


def import_reference():
    if not (SCRATCH / "src").exists():
        shutil.copytree(REF, SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       capture_output=True)
    sys.path.insert(0, str(SCRATCH / "src"))
    import sparseiga  # noqa: F401

    return sparseiga


def shifted_plan(combination, d, w):
    base = combination.combination_coefficients(d, w - d)
    return combination.CombinationPlan(d, tuple((tuple(b + 1 for b in beta), c) for beta, c in base.terms))


def per_point(ref_comb, plan, comps, pts):
    """The reference's scattered-point idiom (tests/test_acceptance.py:224-230)."""
    out = np.zeros(len(pts))
    for i, x in enumerate(pts):
        grid = tuple(np.array([c]) for c in x)
        out[i] = np.ravel(ref_comb.evaluate_combined(plan, comps, grid))[0]
    return out


def csr_digest(m):
    h = hashlib.sha256()
    h.update(np.asarray(m.indptr, dtype=np.int64).tobytes())
    h.update(np.asarray(m.indices, dtype=np.int64).tobytes())
    return h.hexdigest()


def gen_basis(sg):
    from sparseiga import assembly, splines

    cases = [(1, 0, 2, 1.0), (2, 1, 3, 1.0), (3, 2, 4, 1.0), (4, 3, 5, 1.0), (2, 0, 3, 1.0),
             (3, 1, 2, 1.0), (3, 2, 3, 2.0), (2, 1, 4, 3.0), (4, 1, 2, 1.0)]
    out = {}
    rng = np.random.default_rng(7)
    for i, (p, r, lv, g) in enumerate(cases):
        kv = splines.dyadic_level_knots(lv, p, r, g)
        gn, gw = assembly.gauss_rule(p + 1)
        vals, ders, offs, pts, wts = assembly._direction_tables(kv, gn, gw)
        xs = np.concatenate([[0.0, 1.0], kv.breakpoints[1:-1], rng.random(20)])
        firsts, tabs = [], []
        for x in xs:
            f, t = splines.eval_basis(kv, x, max_deriv=1)
            firsts.append(f)
            tabs.append(t)
        out[f"c{i}_meta"] = np.array([p, r, lv, g])
        out[f"c{i}_knots"] = kv.knots
        out[f"c{i}_bp"] = kv.breakpoints
        out[f"c{i}_gn"], out[f"c{i}_gw"] = gn, gw
        out[f"c{i}_vals"], out[f"c{i}_ders"] = vals, ders
        out[f"c{i}_offs"], out[f"c{i}_pts"], out[f"c{i}_wts"] = offs, pts, wts
        out[f"c{i}_xs"], out[f"c{i}_first"], out[f"c{i}_tab"] = xs, np.array(firsts), np.array(tabs)
    out["ncases"] = np.array(len(cases))
    np.savez_compressed(HERE / "basis.npz", **out)


def gen_kernel(sg):
    from sparseiga._kernels import _compiled, _fallback, kernel_backend

    kern = _compiled if kernel_backend() == "compiled" else _fallback
    rng = np.random.default_rng(59)
    out = {"backend": np.array(kernel_backend())}
    for d in (1, 2, 3):
        chunk, q, kmax, max_nel = 3, 4, 3, 5
        n_loc = 3**d
        values = rng.standard_normal((d, max_nel, q, kmax))
        derivs = rng.standard_normal((d, max_nel, q, kmax))
        elem_index = rng.integers(0, max_nel, size=(chunk, d)).astype(np.int64)
        qp_index = np.stack([v.ravel() for v in np.meshgrid(*([np.arange(q)] * d), indexing="ij")], axis=1).astype(np.int32)
        fn_index = np.stack([v.ravel() for v in np.meshgrid(*([np.arange(3)] * d), indexing="ij")], axis=1).astype(np.int32)
        metric = rng.standard_normal((chunk, q**d, d, d))
        metric = metric + metric.transpose(0, 1, 3, 2)
        load = rng.standard_normal((chunk, q**d))
        a, b = np.zeros((chunk, n_loc, n_loc)), np.zeros((chunk, n_loc))
        kern.local_poisson_systems(values, derivs, elem_index, qp_index, fn_index, metric, load, a, b)
        for k, v in dict(values=values, derivs=derivs, elem_index=elem_index, qp_index=qp_index,
                         fn_index=fn_index, metric=metric, load=load, out_a=a, out_b=b).items():
            out[f"d{d}_{k}"] = v
    np.savez_compressed(HERE / "kernel.npz", **out)


CFG = {
    # name: (d, p, w, patch, forcing/solution factory, q, npts, seed, grid levels, store all csr)
    "cfg1": (2, 2, 6, "square", "sin", 3, 4096, 0, (5, 5), True),
    "cfg2": (3, 3, 7, "cube", "sin", 4, 32768, 1, (5, 5, 5), False),
    "cfg3": (2, 3, 8, "annulus", "polar", 4, 4096, 2, (7, 7), True),
    "cfg5": (3, 4, 12, "cube", "expbubble", 5, 32768, 4, (6, 6, 6), False),
}


def sin_u(x):
    return np.prod(np.sin(np.pi * x), axis=-1)


def sin_f(x):
    return (x.shape[-1] * np.pi**2) * sin_u(x)


def sin_g(x):
    s, c = np.sin(np.pi * x), np.cos(np.pi * x)
    return np.stack([np.pi * c[..., m] * np.prod(np.delete(s, m, axis=-1), axis=-1)
                     for m in range(x.shape[-1])], axis=-1)


def polar_u(x):
    s = x[..., 0] ** 2 + x[..., 1] ** 2
    return 2 * x[..., 0] * x[..., 1] * (s - 5 + 4 / s)


def polar_f(x):
    s = x[..., 0] ** 2 + x[..., 1] ** 2
    return 32 * x[..., 0] * x[..., 1] / (s * s) - 24 * x[..., 0] * x[..., 1]


def polar_g(x):
    xx, yy = x[..., 0], x[..., 1]
    s = xx**2 + yy**2
    h, hp = s - 5 + 4 / s, 1 - 4 / s**2
    return np.stack([2 * yy * h + 4 * xx**2 * yy * hp, 2 * xx * h + 4 * xx * yy**2 * hp], axis=-1)


def exp_u(x):
    return np.exp(x.sum(-1)) * np.prod(x * (1 - x), axis=-1)


def exp_f(x):
    b = x * (1 - x)
    return np.exp(x.sum(-1)) * sum(x[..., m] * (x[..., m] + 3) * np.prod(np.delete(b, m, axis=-1), axis=-1)
                                   for m in range(x.shape[-1]))


def exp_g(x):
    b = x * (1 - x)
    e = np.exp(x.sum(-1))
    return np.stack([e * (b[..., m] + 1 - 2 * x[..., m]) * np.prod(np.delete(b, m, axis=-1), axis=-1)
                     for m in range(x.shape[-1])], axis=-1)


def closed_forms(kind):
    """Module-level callables (picklable for the reference's worker pool)."""
    return {"sin": (sin_u, sin_f, sin_g), "polar": (polar_u, polar_f, polar_g),
            "expbubble": (exp_u, exp_f, exp_g)}[kind]


def gen_config(name, comps_to_store=None, n_points=512, workers=1):
    from sparseiga import analysis, assembly, combination, geometry, linsolve, scheduler

    d, p, w, patch_kind, kind, q, npts, seed, glev, all_csr = CFG[name]
    patch = {"square": geometry.unit_hypercube(2), "cube": geometry.unit_hypercube(3),
             "annulus": geometry.quarter_annulus(2)}[patch_kind]
    u, f, g = closed_forms(kind)
    problem = analysis.BenchmarkProblem(name, patch, f, p, p - 1, solution=u, solution_gradient=g)
    plan = shifted_plan(combination, d, w)
    out = {"betas": np.array(plan.betas, dtype=np.int32), "coefs": np.array([c for _, c in plan.terms], dtype=np.int32)}
    t0 = time.perf_counter()
    sols, report = scheduler.run_plan(plan, problem, workers=workers)
    out["run_plan_wall"] = np.array(time.perf_counter() - t0)
    out["coefficients"] = np.concatenate([s.coefficients for s in sols])
    out["dims"] = np.array([s.space.dims for s in sols], dtype=np.int32)
    store = range(len(sols)) if all_csr else (comps_to_store or [])
    rng_v = np.random.default_rng(1234)
    for i in store:
        beta = plan.betas[i]
        space = assembly.DiscreteSpace.from_levels(beta, p, p - 1)
        sysm = assembly.assemble_poisson(space, patch, f)
        m = sysm.matrix.tocsr()
        m.sort_indices()
        out[f"k{i}_nnz"] = np.array(m.nnz)
        out[f"k{i}_digest"] = np.array(csr_digest(m))
        out[f"k{i}_rhs"] = sysm.rhs
        v = rng_v.standard_normal(m.shape[0])
        out[f"k{i}_v"] = v
        out[f"k{i}_Av"] = m @ v
        out[f"k{i}_maxabs"] = np.array(np.abs(m.data).max())
        if m.nnz <= 30000:
            out[f"k{i}_indptr"], out[f"k{i}_indices"], out[f"k{i}_data"] = m.indptr, m.indices, m.data
    out["stored"] = np.array(list(store), dtype=np.int32)
    pts = np.random.default_rng(seed).random((npts, d))[:n_points]
    t0 = time.perf_counter()
    out["points"] = pts
    out["combined"] = per_point(combination, plan, sols, pts)
    out["combine_wall"] = np.array(time.perf_counter() - t0)
    grid = assembly.QuadGrid(patch, glev, q)
    t0 = time.perf_counter()
    l2, h1 = analysis.error_norms(analysis.combined_evaluator(plan, sols),
                                  analysis.analytic_evaluator(u, g), grid)
    out["errors"] = np.array([l2, h1])
    out["errors_wall"] = np.array(time.perf_counter() - t0)
    if name == "cfg5":
        # 1.4 M coefficients are too big for a fixture: keep the stored
        # components in full and a per-component checksum (norm, seeded dot)
        coef = out.pop("coefficients")
        off = np.concatenate([[0], np.cumsum(np.prod(out["dims"], axis=1))])
        vs = [coef[off[c]:off[c + 1]] for c in range(len(off) - 1)]
        out["coef_norms"] = np.array([np.linalg.norm(v) for v in vs])
        out["coef_dots"] = np.array([np.random.default_rng(1000 + c).standard_normal(v.size) @ v
                                     for c, v in enumerate(vs)])
        for i in out["stored"]:
            out[f"k{i}_coef"] = vs[i]
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, "components", len(plan), "L2/H1", l2, h1, flush=True)


def gen_studies():
    """Surplus / profit tables and convergence studies
    computed by the reference's own drivers."""
    from sparseiga import analysis, combination

    out = {}
    cases = {
        "annulus2_p2": (analysis.regular_annulus_problem(2, degree=2), 2),
        "cube3_p2": (analysis.polynomial_cube_problem(3, degree=2), (1, 1, 2)),
        "const2_p2_g2": (analysis.constant_forcing_problem(2, grading=2.0, degree=2), 2),
    }
    for key, (prob, bmax) in cases.items():
        rows = combination.profit_table(prob, bmax)
        out[f"profit_{key}_beta"] = np.array([r.beta for r in rows], dtype=np.int32)
        out[f"profit_{key}_l2"] = np.array([r.surplus_l2 for r in rows])
        out[f"profit_{key}_dofs"] = np.array([r.dofs for r in rows], dtype=np.int64)
    studies = {
        "annulus2_sparse": (analysis.regular_annulus_problem(2, degree=2), "sparse", [1, 2, 3, 4]),
        "annulus2_tensor": (analysis.regular_annulus_problem(2, degree=2), "tensor", [1, 2, 3]),
        "const2_sparse": (analysis.constant_forcing_problem(2, grading=1.0, degree=2), "sparse", [1, 2, 3]),
    }
    for key, (prob, method, levels) in studies.items():
        recs = analysis.convergence_study(prob, method, levels)
        out[f"conv_{key}_levels"] = np.array(levels, dtype=np.int32)
        out[f"conv_{key}_l2"] = np.array([r.l2_error for r in recs])
        out[f"conv_{key}_h1"] = np.array([r.h1_semi_error for r in recs])
        out[f"conv_{key}_dofs"] = np.array([r.dofs_total for r in recs], dtype=np.int64)
        out[f"conv_{key}_ncomp"] = np.array([r.n_components for r in recs], dtype=np.int32)
    np.savez_compressed(HERE / "studies.npz", **out)
    print("studies", sorted(k for k in out if k.endswith("_l2")), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg5", action="store_true", help="also run cfg5 (minutes, 8 workers)")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    sg = import_reference()
    print("reference backend:", sg.kernel_backend())
    if args.only in (None, "basis"):
        gen_basis(sg)
    if args.only in (None, "kernel"):
        gen_kernel(sg)
    if args.only in (None, "cfg1"):
        gen_config("cfg1")
    if args.only in (None, "cfg3"):
        gen_config("cfg3")
    if args.only in (None, "cfg2"):
        # largest component by nnz (3,2,2) and the slowest-converging (5,1,1)
        from sparseiga import combination
        plan = shifted_plan(combination, 3, 7)
        pick = [plan.betas.index(b) for b in ((3, 2, 2), (5, 1, 1), (1, 1, 5), (2, 3, 2))]
        gen_config("cfg2", comps_to_store=pick)
    if args.only in (None, "studies"):
        gen_studies()
    if args.cfg5 or args.only == "cfg5":
        from sparseiga import combination
        plan = shifted_plan(combination, 3, 12)
        pick = [plan.betas.index(b) for b in ((1, 1, 10), (4, 4, 4), (10, 1, 1))]
        gen_config("cfg5", comps_to_store=pick, n_points=256, workers=os.cpu_count())


if __name__ == "__main__":
    main()
