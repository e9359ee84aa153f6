"""Golden fixture for the cfg5 comparison point: the full tensor-grid solve
at 2^6 elements per direction (BASELINE configs[4], reference plan
``CombinationPlan(3, (((6,6,6),1),))``, analysis.py:317-320).

Run in the build container only (needs /root/reference, ~20-40 min on 8
cores):

    python tests/golden/make_golden_tensor.py [--workers 8]

What comes from where:

* Basis tables, geometry, metric and load: the reference's own functions
  and expressions (``assembly._direction_tables``, ``NurbsPatch.eval_grid``,
  ``np.linalg.inv`` + the einsum of assembly.py:286-294,
  ``_group_elements``).
* Element matrices: the reference's compiled element kernel
  ``local_poisson_systems`` (_kernels/_compiled.pyx:17-90) on every one of
  the 262 144 elements.
* Global accumulation: the reference's ``_assemble_full`` adds a COO->CSR
  per 2-element chunk into a running CSR (131 072 CSR additions of a
  189 M-nnz matrix: infeasible), so the element matrices are summed here
  into a banded (row, offset) array instead -- elements are processed in
  5^3 colour classes (elements 5 apart in every direction share no
  function), so a vectorised scatter never collides.  Same additions,
  different (rounding-level) order.
* Solve: the reference's ``spsolve`` is infeasible at 287 496 rows
  (SURVEY 8(c)); the coefficients come from the LABELLED restatement
  SURVEY 8(d) prescribes -- scipy Jacobi-preconditioned CG, rtol 1e-13 --
  and the reference's acceptance check ||Ax-b|| <= 1e-10 ||b||
  (linsolve.py:49-53) is applied to it.
* Combined values: the reference's per-point idiom (test_acceptance.py:
  224-230) on a one-term plan; errors: the reference's ``error_norms`` on
  ``QuadGrid((6,6,6), 5)``.

The fixture keeps checksums (norms, seeded dot products) plus seeded
samples of A v, b and x, 64 complete matrix rows and 4096 combined values
-- the full vectors would be 7 MB.
"""
from __future__ import annotations

import argparse
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import exp_f, exp_g, exp_u, import_reference, per_point_parallel  # noqa: E402

LEVEL, P = 6, 4
_S = {}


def _colour_batch(args):
    """Element matrices of one colour class (slice of it), reference kernel."""
    from sparseiga._kernels import local_poisson_systems
    idx = args
    em = np.ascontiguousarray(_S["elem_multi"][idx])
    nc = len(idx)
    n_loc = _S["n_loc"]
    out_a = np.zeros((nc, n_loc, n_loc))
    out_b = np.zeros((nc, n_loc))
    local_poisson_systems(_S["values"], _S["derivs"], em, _S["qp_index"], _S["fn_index"],
                          np.ascontiguousarray(_S["metric_el"][idx]), np.ascontiguousarray(_S["load_el"][idx]),
                          out_a, out_b)
    return idx, out_a, out_b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--maxiter", type=int, default=20000)
    args = ap.parse_args()
    sg = import_reference()
    print("reference backend:", sg.kernel_backend(), flush=True)
    from scipy import sparse as sps
    from scipy.sparse import linalg as spla
    from sparseiga import analysis, assembly, combination, geometry
    from sparseiga.assembly import _direction_tables, _group_elements, _outer_product, gauss_rule

    T0 = time.perf_counter()
    d, p = 3, P
    q = p + 1
    patch = geometry.unit_hypercube(3)
    space = assembly.DiscreteSpace.from_levels((LEVEL,) * 3, p, p - 1)
    gnodes, gweights = gauss_rule(q)
    tabs = [_direction_tables(kv, gnodes, gweights) for kv in space.knotvectors]
    nels = [t[0].shape[0] for t in tabs]
    kmax, max_nel = p + 1, max(nels)
    values = np.zeros((d, max_nel, q, kmax))
    derivs = np.zeros((d, max_nel, q, kmax))
    for axis, (v, dv, _, _, _) in enumerate(tabs):
        values[axis, : nels[axis]] = v
        derivs[axis, : nels[axis]] = dv
    # assembly.py:286-294, verbatim expressions of the reference
    x, jac, det = patch.eval_grid([t[3] for t in tabs], jacobian=True, check=True)
    wgrid = _outer_product([t[4] for t in tabs])
    jinv = np.linalg.inv(jac.reshape(-1, d, d)).reshape(jac.shape)
    metric = np.einsum("...mi,...ni->...mn", jinv, jinv) * (det * wgrid)[..., None, None]
    rhs_density = np.asarray(exp_f(x.reshape(-1, d)), dtype=np.float64).reshape(det.shape)
    load = rhs_density * det * wgrid
    del x, jac, jinv
    n_qp = q**d
    n_elems = int(np.prod(nels))
    loc_dims = (p + 1,) * d
    n_loc = int(np.prod(loc_dims))
    _S.update(values=values, derivs=derivs, n_loc=n_loc,
              metric_el=_group_elements(metric, nels, q), load_el=_group_elements(load, nels, q),
              qp_index=np.stack(np.unravel_index(np.arange(n_qp), (q,) * d), axis=1).astype(np.int32),
              fn_index=np.stack(np.unravel_index(np.arange(n_loc), loc_dims), axis=1).astype(np.int32),
              elem_multi=np.stack(np.unravel_index(np.arange(n_elems), nels), axis=1).astype(np.int64))
    del metric, load
    print(f"tables/geometry/metric {time.perf_counter() - T0:.1f} s", flush=True)

    # banded accumulation: full dofs n^3 (n = 68), offsets (2p+1)^3
    dims = space.dims
    W = 2 * p + 1
    nfull = int(np.prod(dims))
    band = np.zeros((nfull, W**3))
    rhs = np.zeros(nfull)
    fn = _S["fn_index"].astype(np.int64)
    # slot of the (a, b) local pair: (j - i + p) per axis, i = e + a
    off = fn[None, :, :] - fn[:, None, :] + p                     # [a, b, d]
    slot_ab = (off[..., 0] * W + off[..., 1]) * W + off[..., 2]   # [a, b]
    strides = np.array([dims[1] * dims[2], dims[2], 1], dtype=np.int64)
    em = _S["elem_multi"]
    colour = (em[:, 0] % q) * q * q + (em[:, 1] % q) * q + em[:, 2] % q
    jobs = []
    for c in range(q**3):
        idx = np.nonzero(colour == c)[0]
        for part in np.array_split(idx, max(1, len(idx) // 256)):
            jobs.append(part)
    t0 = time.perf_counter()
    done = 0
    with mp.get_context("fork").Pool(args.workers) as pool:
        for idx, out_a, out_b in pool.imap(_colour_batch, jobs, chunksize=1):
            rows = ((em[idx][:, None, :] + fn[None, :, :]) * strides).sum(-1)   # [E, a] global function
            lin = rows[:, :, None] * (W**3) + slot_ab[None, :, :]
            band.reshape(-1)[lin.reshape(-1)] += out_a.reshape(-1)   # no collisions inside a colour
            rhs[rows.reshape(-1)] += out_b.reshape(-1)
            done += len(idx)
            if done % 32768 < len(idx):
                print(f"  elements {done}/{n_elems}  {time.perf_counter() - t0:.0f} s", flush=True)
    t_asm = time.perf_counter() - t0
    print(f"element kernel + accumulation {t_asm:.1f} s", flush=True)
    del _S["metric_el"], _S["load_el"]

    # interior system in the reference's C order (assembly.py:84-96, 389)
    interior = space.interior_dofs()
    m = [n - 2 for n in dims]
    nint = int(np.prod(m))
    imulti = np.stack(np.unravel_index(np.arange(nint), m), axis=1) + 1                # full index
    frow = (imulti * strides).sum(-1)
    assert np.array_equal(frow, interior)
    sl = np.stack(np.unravel_index(np.arange(W**3), (W,) * 3), axis=1) - p            # [slot, d]
    cols_multi = imulti[:, None, :] + sl[None, :, :]                                   # [row, slot, d]
    ok = np.all((cols_multi >= 1) & (cols_multi <= np.array(m)), axis=-1)
    mstr = np.array([m[1] * m[2], m[2], 1], dtype=np.int64)
    cols = ((cols_multi - 1) * mstr).sum(-1)
    vals = band[frow]
    keep = ok & (vals != 0.0)          # csr addition drops exact zeros
    counts = keep.sum(1)
    indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    A = sps.csr_matrix((vals[keep], cols[keep].astype(np.int32), indptr), shape=(nint, nint))
    A.sort_indices()
    b = rhs[interior]
    del band, vals, cols, cols_multi, ok, keep
    print(f"interior system: {nint} rows, nnz {A.nnz}", flush=True)

    out = {"dims": np.array(dims, dtype=np.int32), "nnz": np.array(A.nnz), "rows": np.array(nint)}
    rng = np.random.default_rng(2024)
    vprobe = np.random.default_rng(1234).standard_normal(nint)
    Av = A @ vprobe
    dots = [np.random.default_rng(5000 + k).standard_normal(nint) for k in range(3)]
    out["Av_norm"] = np.array(np.linalg.norm(Av))
    out["Av_dots"] = np.array([w @ Av for w in dots])
    out["b_norm"] = np.array(np.linalg.norm(b))
    out["b_dots"] = np.array([w @ b for w in dots])
    samp = np.sort(rng.choice(nint, 4096, replace=False))
    out["sample_rows"] = samp
    out["Av_sample"] = Av[samp]
    out["b_sample"] = b[samp]
    full_rows = np.sort(rng.choice(nint, 64, replace=False))
    out["full_rows"] = full_rows
    for k, r in enumerate(full_rows):
        s, e = A.indptr[r], A.indptr[r + 1]
        out[f"row{k}_cols"] = A.indices[s:e].astype(np.int32)
        out[f"row{k}_vals"] = A.data[s:e]
    out["maxabs"] = np.array(np.abs(A.data).max())
    out["asm_s"] = np.array(t_asm)

    # labelled restatement of the solve: scipy Jacobi-PCG, rtol 1e-13
    dinv = 1.0 / A.diagonal()
    M = spla.LinearOperator(A.shape, matvec=lambda r: dinv * r, dtype=np.float64)
    it = [0]

    def cb(_):
        it[0] += 1
        if it[0] % 100 == 0:
            print(f"  cg it {it[0]}", flush=True)

    t0 = time.perf_counter()
    xs, info = spla.cg(A, b, rtol=1e-13, atol=0.0, maxiter=args.maxiter, M=M, callback=cb)
    t_cg = time.perf_counter() - t0
    relres = float(np.linalg.norm(A @ xs - b) / np.linalg.norm(b))
    print(f"jacobi-pcg info {info} iterations {it[0]} true relres {relres:.3e} ({t_cg:.0f} s)", flush=True)
    assert info == 0 and relres <= 1e-10, "linsolve.py:49-53 acceptance"
    full = np.zeros(nfull)
    full[interior] = xs
    out["cg_iterations"] = np.array(it[0])
    out["cg_relres"] = np.array(relres)
    out["cg_s"] = np.array(t_cg)
    out["coef_norm"] = np.array(np.linalg.norm(full))
    out["coef_dots"] = np.array([np.random.default_rng(6000 + k).standard_normal(nfull) @ full for k in range(3)])
    csamp = np.sort(rng.choice(nfull, 4096, replace=False))
    out["coef_sample_idx"] = csamp
    out["coef_sample"] = full[csamp]

    # combined values at the cfg5 points (seed 4), reference per-point idiom
    plan = combination.CombinationPlan(3, (((LEVEL,) * 3, 1),), level=LEVEL)
    sol = combination.ComponentSolution((LEVEL,) * 3, space, full, 1.0)
    pts = np.random.default_rng(4).random((32768, 3))[:4096]
    out["points"] = pts
    out["combined"] = per_point_parallel(plan, [sol], pts, args.workers)
    grid = assembly.QuadGrid(patch, (6, 6, 6), q)
    l2, h1 = analysis.error_norms(analysis.combined_evaluator(plan, [sol]),
                                  analysis.analytic_evaluator(exp_u, exp_g), grid)
    out["errors"] = np.array([l2, h1])
    print("tensor L2/H1", l2, h1, f"total {time.perf_counter() - T0:.0f} s", flush=True)
    np.savez_compressed(HERE / "cfg5_tensor.npz", **out)


if __name__ == "__main__":
    main()
