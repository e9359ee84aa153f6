/*
 * sgiga.h -- C ABI of the B200-native batched sparse-grid IGA hot path.
 *
 * One handle = one combination plan on one GPU: every anisotropic
 * tensor-product component of the plan is assembled, solved and combined in
 * a single batched device pipeline (hand-written sm_100a FP64 kernels).
 * Plain C types only; no torch / CUDA types in the signatures (the stream is
 * passed as an opaque pointer).
 *
 * Reference interfaces replaced (paths relative to the reference package
 * pkg/src/sparseiga/):
 *   sgiga_create/sgiga_assemble/sgiga_solve/sgiga_coefficients
 *       -> scheduler.run_plan (scheduler.py:74-96) driving
 *          combination.solve_component (combination.py:183-200), i.e.
 *          DiscreteSpace.from_levels (assembly.py:64-70),
 *          assemble_poisson (assembly.py:357-390) and
 *          linsolve.solve_spd (linsolve.py:16-54), per component.
 *   sgiga_combine_points / sgiga_combine_grid
 *       -> combination.evaluate_combined (combination.py:209-236) and the
 *          per-point idiom of tests/test_acceptance.py:224-230.
 *   sgiga_error_norms
 *       -> analysis.error_norms + combined_evaluator + analytic_evaluator
 *          (analysis.py:226-270) on an assembly.QuadGrid (assembly.py:141-183).
 *   sgiga_export_csr
 *       -> AssembledSystem.matrix / .rhs (assembly.py:193-206, 389-390),
 *          for parity checks only.
 *   sgiga_local_poisson_systems
 *       -> _kernels.local_poisson_systems (_kernels/_compiled.pyx:17-90,
 *          _kernels/_fallback.py:13-65), the reference's element-kernel
 *          plugin point (assembly.py:273-274, 330-340).
 *
 * Error codes map to the reference exception classes (see the enum).
 * Every call is synchronous with respect to the host unless stated; a
 * handle is bound to one stream and is not thread-safe.
 */
#ifndef SGIGA_H
#define SGIGA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum sgiga_status {
    SGIGA_OK = 0,
    SGIGA_ERR_VALUE = -1,    /* ValueError: malformed descriptor / argument  */
    SGIGA_ERR_GEOMETRY = -2, /* geometry.InvalidGeometryError: det J <= 0     */
    SGIGA_ERR_SOLVE = -3,    /* linsolve.LinearSolveError: non-finite /       */
                             /*   not converged / residual above tolerance    */
    SGIGA_ERR_EMPTY = -4,    /* assembly.EmptyInteriorError                   */
    SGIGA_ERR_CUDA = -5,     /* CUDA runtime failure (no device, OOM, fault)  */
    SGIGA_ERR_STATE = -6,    /* call order (e.g. combine before solve)        */
    SGIGA_ERR_KEY = -7       /* KeyError: component missing                   */
};

/* ---- device forcing / exact-solution registry ----------------------------
 * The reference passes the forcing as a Python callable evaluated at
 * physical quadrature points (assembly.py:237-245, 290-292).  Closed forms
 * that the benchmark configurations use run on the device; anything else is
 * evaluated by the host on device-computed points (SGIGA_FORCING_HOST). */
enum sgiga_forcing {
    SGIGA_FORCING_HOST = -1,          /* density supplied per quad point      */
    SGIGA_FORCING_ZERO = 0,           /* f = 0 (full_stiffness, cfg4)         */
    SGIGA_FORCING_SIN_PRODUCT = 1,    /* u = prod sin(pi x_k), f = d pi^2 u    */
    SGIGA_FORCING_ANNULUS_POLAR = 2,  /* u = (r^2-1)(r^2-4) sin 2theta (cfg3) */
    SGIGA_FORCING_EXP_BUBBLE = 3,     /* u = e^{x+y+z} prod x_k(1-x_k) (cfg5) */
    SGIGA_FORCING_CUBE_POLY = 4,      /* analysis.cube_forcing (analysis.py:146-152) */
    SGIGA_FORCING_ANNULUS_2D = 5,     /* analysis.annulus_forcing_2d (112-117) */
    SGIGA_FORCING_ANNULUS_3D = 6,     /* analysis.annulus_forcing_3d (134-136) */
    SGIGA_FORCING_CONSTANT_ONE = 7,   /* analysis.constant_one (139-140)       */
    SGIGA_FORCING_LSHAPE = 8          /* u = r^{2/3} sin(2theta/3), f = 0      */
};

/* ---- problem + plan descriptor (host pointers) ---------------------------
 * Mirrors BenchmarkProblem (analysis.py:52-77) + NurbsPatch
 * (geometry.py:34-71) + CombinationPlan (combination.py:49-90).
 *
 * Analysis knot vectors are given per (axis, level) as breakpoints; the
 * open knot vector is rebuilt on the device with interior multiplicity
 * degree - regularity exactly as make_open_knot_vector (splines.py:83-110).
 * Breakpoints and Gauss nodes are produced by the host with the same numpy
 * expressions as the reference (dyadic_level_knots splines.py:133-146,
 * gauss_rule assembly.py:41-46), so they are bitwise identical.           */
typedef struct sgiga_problem_desc {
    int32_t d;                  /* 1..3                                       */
    int32_t degree;             /* p >= 1 (<= 4 on the device path)           */
    int32_t regularity;         /* r in [0, p-1] (C^r joins)                  */
    int32_t quad_points;        /* q Gauss points per element and direction   */
    int32_t n_comp;             /* number of plan terms                       */
    const int32_t* levels;      /* [n_comp*d], lexicographic plan order       */
    const int32_t* coefs;       /* [n_comp] integer combination coefficients  */
    const double* gauss_nodes;  /* [q] on [0,1]                               */
    const double* gauss_weights;/* [q], sum 1                                 */
    int32_t max_level;          /* levels are in [0, max_level]               */
    const int64_t* bp_offset;   /* [d*(max_level+1)] into breakpoints, -1 = unused */
    const int32_t* bp_count;    /* [d*(max_level+1)] number of breakpoints (nel+1) */
    const double* breakpoints;  /* concatenated breakpoint tables             */
    /* geometry (NurbsPatch): per-axis knot vectors + homogeneous net        */
    const int32_t* geo_degree;  /* [d]                                        */
    const int32_t* geo_nknots;  /* [d]                                        */
    const double* geo_knots;    /* concatenated [sum geo_nknots]              */
    const double* geo_hw;       /* [n_1*...*n_d*(d+1)] C order: (w*P, w)      */
    int32_t forcing_id;         /* enum sgiga_forcing                         */
    int32_t flags;              /* SGIGA_FLAG_*                               */
} sgiga_problem_desc;

/* descriptor flags */
enum sgiga_flags {
    SGIGA_FLAG_ASSEMBLY_ONLY = 1   /* the handle only assembles (the multipatch driver glues and solves
                                      on its own): no FD preconditioner set-up is enqueued            */
};

typedef struct sgiga_handle sgiga_handle;

/* Create a handle for one plan: validates the descriptor, builds the
 * component table and allocates all device buffers.  stream may be NULL
 * (the library creates its own).  Nothing is computed yet.              */
int sgiga_create(const sgiga_problem_desc* desc, void* stream, sgiga_handle** out);

/* Re-upload the host descriptor arrays (same shape as at create time):
 * the per-step host->device copy of the problem inputs.                  */
int sgiga_upload(sgiga_handle* h, const sgiga_problem_desc* desc);

/* Number of quadrature points of the whole batch and, for
 * SGIGA_FORCING_HOST, the two-phase host forcing protocol:
 * sgiga_quad_points_physical copies the mapped points x (npts*d) to the
 * host, sgiga_set_forcing_density uploads f(x) (npts).                   */
int sgiga_batch_sizes(sgiga_handle* h, int64_t* total_qp, int64_t* total_rows,
                      int64_t* total_dofs, int64_t* total_slots);
int sgiga_quad_points_physical(sgiga_handle* h, double* x_out);
int sgiga_set_forcing_density(sgiga_handle* h, const double* f);

/* Per-component metadata: dims n_k (C-order full space, [n_comp*d]),
 * offsets of each component's full coefficient vector ([n_comp+1]).     */
int sgiga_component_info(sgiga_handle* h, int32_t* dims, int64_t* dof_offsets);

/* Phase 1: basis tables, geometry/metric/load, stencil assembly (+ D^-1). */
int sgiga_assemble(sgiga_handle* h);

/* Phase 2: batched Jacobi-PCG on all components to ||r||/||b|| <= rtol,
 * then the reference's acceptance check ||Ax-b|| <= 1e-10 ||b||
 * (linsolve.py:49-53).  iters_out / relres_out may be NULL.             */
int sgiga_solve(sgiga_handle* h, double rtol, int32_t maxit,
                int32_t* iters_out, double* relres_out);

/* Full C-order coefficient vectors with zero boundary, concatenated in
 * plan order (AssembledSystem.expand, assembly.py:202-206).             */
int sgiga_coefficients(sgiga_handle* h, double* out);
/* Replace the device coefficients (e.g. components supplied by a user). */
int sgiga_set_coefficients(sgiga_handle* h, const double* full_coefs);

/* Phase 3: sum_beta c_beta u_beta at scattered parametric points
 * (npts x d, C order), accumulated in plan order.
 *   device = 0 : host pointers (H2D/D2H inside the call), out[npts]
 *   device = 1 : device pointers (inputs resident in HBM), out[npts]
 *   device = -1: host pointers, per-component values out[n_comp*npts]
 *   device = -2: device pointers, per-component values out[n_comp*npts]
 * (per-component mode feeds the multi-GPU ordered combine).             */
int sgiga_combine_points(sgiga_handle* h, const double* pts, int64_t npts,
                         double* out, int32_t device);

/* The whole plan in one call: assemble, solve, combine at npts points
 * (device = 0 host / 1 device pointers, as sgiga_combine_points), all
 * enqueued on the handle's stream with ONE synchronisation at the end.
 * Replaces run_plan + evaluate_combined (scheduler.py:74-96,
 * combination.py:209-236).  Errors are reported as by the three phase
 * calls (the first failing phase wins); npts = 0 skips the combine.     */
int sgiga_run(sgiga_handle* h, double rtol, int32_t maxit, const double* pts,
              int64_t npts, double* out, int32_t device, int32_t* iters_out,
              double* relres_out);

/* Asynchronous form of sgiga_run with device-resident points / output:
 * sgiga_run_async enqueues the whole pass on the handle's stream and
 * returns without synchronising (back-to-back passes pipeline on the
 * device); sgiga_run_wait synchronises and reports the LAST enqueued pass
 * exactly as sgiga_run does (status, iterations, relative residuals).     */
int sgiga_run_async(sgiga_handle* h, double rtol, int32_t maxit, const double* pts_dev,
                    int64_t npts, double* out_dev);
int sgiga_run_wait(sgiga_handle* h, int32_t* iters_out, double* relres_out);
/* Asynchronous end-to-end pass with HOST buffers: the page-locked points are
 * copied host->device inside the pass (point-sort side stream) and the
 * combined values device->host into the page-locked output after the
 * combine; returns after enqueueing.  Passes pipeline back to back (the
 * host may submit pass k+1 while pass k runs); the output buffer of a pass
 * must stay untouched until sgiga_run_wait, which reports the LAST pass.
 * Same computation and result as sgiga_run(..., device = 0).            */
int sgiga_run_host_async(sgiga_handle* h, double rtol, int32_t maxit, const double* pts_pinned,
                         int64_t npts, double* out_pinned);

/* Tensor grid variant: per-axis parameter arrays concatenated; vals has
 * prod(npts) entries (C order), grads (optional, may be NULL) prod*d.
 * comp = -1 combines the plan; comp >= 0 evaluates that component alone
 * (DiscreteSpace.eval_grid, assembly.py:101-127).                        */
int sgiga_combine_grid(sgiga_handle* h, const double* pts_per_dir,
                       const int64_t* npts_per_dir, int32_t comp,
                       double* vals, double* grads);

/* L2 and H1-seminorm error of the combined solution against the device
 * closed-form solution on a tensor Gauss grid (per-axis points/weights as
 * QuadGrid builds them).  out[0] = L2, out[1] = H1 seminorm.            */
/* Same quadrature for an explicit signed term list: the field
 * sum_t weights[t] * u_{comps[t]} (accumulated in the given order, as the
 * reference's surplus, combination.py:269-272) against the closed-form
 * solution_id, or against zero when solution_id < 0 (then out = the L2 norm
 * and H1 seminorm of the field itself).  Serves surplus_norm / profit_table
 * (combination.py:247-302) and the study drivers' per-level errors
 * (analysis.py:325-386), several plans sharing one solved batch.         */
int sgiga_subset_error_norms(sgiga_handle* h, const double* pts_per_dir,
                             const double* wts_per_dir, const int64_t* npts_per_dir,
                             int32_t n_terms, const int32_t* comps, const double* weights,
                             int32_t solution_id, double* out);

int sgiga_error_norms(sgiga_handle* h, const double* pts_per_dir,
                      const double* wts_per_dir, const int64_t* npts_per_dir,
                      int32_t solution_id, double* out);

/* sgiga_run_async with per-component output: out_dev[c * npts + i] = value
 * of component c (plan order, coefficient NOT applied) at point i -- the
 * local half of a plan split over ranks (distributed.py).  No sync; the
 * verdict comes from sgiga_run_wait.                                      */
int sgiga_run_components_async(sgiga_handle* h, double rtol, int32_t maxit, const double* pts_dev,
                               int64_t npts, double* out_dev);

/* Batched sgiga_edge_projection_system: one launch for nedge edges of this
 * patch handle.  d_edges [nedge][3] = (component, running axis, side),
 * d_offsets [nedge] = offset of the edge's band [n][2p+1] in d_base (its
 * rhs [n] follows the band); max_edge_qp >= nel*q of every edge.  Device
 * arrays; enqueued on the handle's stream.                                */
int sgiga_edge_projection_batch(sgiga_handle* h, int32_t nedge, const int32_t* d_edges, const int64_t* d_offsets,
                                int32_t max_edge_qp, int32_t solution_id, double* d_base);

/* Multi-GPU combine: out[pt] = sum_c coef[c] * src[row[c]][pt]
 * over the plan's terms in plan order, with the exact operations of the
 * single-GPU combine (vals = c*v; vals += c*v, combination.py:227-233), so
 * a plan split over ranks reproduces the one-GPU values bitwise after the
 * per-component values (rows of npts doubles) are all-gathered.  Device
 * pointers; enqueued on `stream`, no synchronisation.                    */
int sgiga_plan_order_sum(void* stream, int32_t nterm, int64_t npts, const int32_t* d_coef,
                         const int64_t* d_row, const double* d_src, double* d_out);

/* Parity export of kernel 1's output for one (axis, level) knot vector, as
 * assembly._direction_tables (assembly.py:209-234) returns it: basis values
 * and first derivatives [nel][q][p+1], Gauss points xi [nel*q] and weights
 * h*w_g [nel*q].  nel_out receives the element count; pass NULL arrays to
 * query it.  The tables are the ones the last assembly pass computed on the
 * device (SGIGA_ERR_STATE before any assembly).                           */
int sgiga_basis_table(sgiga_handle* h, int32_t axis, int32_t level, int32_t* nel_out, double* vals,
                      double* ders, double* pts, double* wts);

/* Parity export of one component: interior CSR (C-order rows, sorted
 * columns, exact zeros dropped as scipy's csr addition does) and rhs.
 * Call with indices/data NULL to get nnz first.                          */
int sgiga_export_csr(sgiga_handle* h, int32_t comp, int64_t* nnz_out,
                     int64_t* indptr, int32_t* indices, double* data,
                     double* rhs);

/* Device time (ms) of the last assemble / solve / combine calls and the
 * number of kernel launches each issued.                                 */
int sgiga_phase_stats(sgiga_handle* h, float* ms3, int64_t* launches3);

/* Device time (ms, CUDA events on the handle's stream) of the last launch
 * of each kernel group: [0] basis tables, [1] metric/load, [2] stencil
 * assembly, [3] small-component PCG, [4] large-component PCG (all
 * iterations), [5] residual check + expand, [6] combine / grid evaluation. */
int sgiga_kernel_times(sgiga_handle* h, float* ms7);

/* FP64 operations the last stencil assembly executed (FMA = 2), counted
 * on the host from the launch's work decomposition (the tiled 3-D kernel;
 * 0 when the plan ran another assembly kernel).  The bench reports it
 * beside the canonical sum-factorised count of SURVEY 8(d).              */
int sgiga_assembly_flops(sgiga_handle* h, double* executed);

/* Which stencil assembly the last pass ran (measurement only; the bench
 * picks the roofline that bounds it): 0 = one-row-per-CTA / 2-D block /
 * generic kernels (FP64 bound), 1 = tiled 3-D kernel (FP64 bound), 2 =
 * Kronecker box assembly (axis-aligned box geometries: 1-D bands, one store
 * pass over the stencil -- HBM-store bound).                              */
int sgiga_assembly_kind(sgiga_handle* h, int32_t* kind);

/* Per-component PCG iteration counts of the last solve.                 */
int sgiga_iterations(sgiga_handle* h, int32_t* iters);

/* ---- multipatch pieces (BASELINE cfg4; no reference
 * code path exists -- SPEC.md:150,208 -- so these extend the single-patch
 * discretisation of assembly.py:357-390 the GeoPDEs way).  All pointers
 * named d_* are DEVICE pointers; launches go to the handle's / the given
 * stream; the caller orchestrates (paper_1707_09598_b200/multipatch.py).
 *
 * Full-patch stiffness of component comp of an assembled patch handle:
 * every function (boundary rows included), rows in reference C order over
 * n_1 x ... x n_d, (2p+1)^d relative-offset slots (last axis fastest, zero
 * outside the patch): d_vals[slot*rows + row]; load vector d_rhs[rows].   */
int sgiga_full_patch_system(sgiga_handle* h, int32_t comp, double* d_vals, double* d_rhs);

/* Dirichlet data moments on one edge of a 2-D patch: the edge runs along
 * parametric axis `axis` with the other coordinate = side (0/1).  Banded
 * 1-D mass d_band[i*(2p+1) + j-i+p] = int B_i B_j |dx/dxi| and
 * d_rhs[i] = int g B_i |dx/dxi|, g = device closed form solution_id.     */
int sgiga_edge_projection_system(sgiga_handle* h, int32_t comp, int32_t axis, int32_t side,
                                 int32_t solution_id, double* d_band, double* d_rhs);

/* d_dst[k] = sum_{t=d_start[k]}^{d_start[k+1]-1} d_src[d_idx[t]] (fixed order). */
int sgiga_gather_sum(void* stream, int64_t n, const int64_t* d_start, const int64_t* d_idx,
                     const double* d_src, double* d_dst);
/* d_dst[k] = d_idx[k] >= 0 ? d_src[d_idx[k]] : 0.                         */
int sgiga_gather(void* stream, int64_t n, const int64_t* d_idx, const double* d_src, double* d_dst);
/* d_y[r] -= sum_k val[k] x[col[k]] over CSR row r.                         */
int sgiga_csr_spmv_sub(void* stream, int64_t nrows, const int64_t* d_rowptr, const int32_t* d_col,
                       const double* d_val, const double* d_x, double* d_y);
/* Batched Jacobi-PCG: system s = rows [d_off[s], d_off[s+1]) of one CSR
 * over the concatenated vector; ||r|| <= rtol ||b||; iters_out < 0 flags
 * non-convergence; relres_out = true residual (host arrays, synchronises). */
int sgiga_csr_pcg(void* stream, int32_t nsys, const int64_t* d_off, int64_t nrows_total,
                  const int64_t* d_rowptr, const int32_t* d_col, const double* d_val, const double* d_b,
                  double* d_x, double rtol, int32_t maxit, int32_t* iters_out, double* relres_out);
/* Device-to-device sgiga_set_coefficients (full C-order vectors).        */
int sgiga_set_coefficients_device(sgiga_handle* h, const double* d_full);

/* The CUDA stream (cudaStream_t) every launch of this handle goes to. */
void* sgiga_stream(sgiga_handle* h);

int sgiga_destroy(sgiga_handle* h);
const char* sgiga_last_error(void);
int sgiga_device_count(int32_t* n);

/* B4: GPU mirror of _kernels.local_poisson_systems (host arrays, same
 * shapes and accumulate-into-outputs contract as _compiled.pyx:17-90):
 *   values, derivs  [d, max_nel, n_q, kmax]
 *   elem_index      [n_chunk, d]  int64
 *   qp_index        [n_qp, d]     int32
 *   fn_index        [n_loc, d]    int32
 *   metric          [n_chunk, n_qp, d, d]
 *   load            [n_chunk, n_qp]
 *   out_a (+=)      [n_chunk, n_loc, n_loc]
 *   out_b (+=)      [n_chunk, n_loc]
 * Returns SGIGA_ERR_VALUE when d > 8 (_compiled.pyx:38-39).              */
int sgiga_local_poisson_systems(int32_t d, int32_t max_nel, int32_t n_q, int32_t kmax,
                                int64_t n_chunk, int32_t n_qp, int32_t n_loc,
                                const double* values, const double* derivs,
                                const int64_t* elem_index, const int32_t* qp_index,
                                const int32_t* fn_index, const double* metric,
                                const double* load, double* out_a, double* out_b);

#ifdef __cplusplus
}
#endif

#endif /* SGIGA_H */
