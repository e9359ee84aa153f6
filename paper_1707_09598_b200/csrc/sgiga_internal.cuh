// sgiga_internal.cuh -- shared device data model of the batched pipeline.
//
// One handle holds one combination plan.  Every component (anisotropic
// tensor-product B-spline space) gets an entry in a device-resident
// component table; all per-component arrays (metric/load at quadrature
// points, the stencil matrix, the PCG vectors, the full coefficient
// vectors) are concatenated batch-wide and addressed through offsets.
//
// Internal row order: each component orders its interior rows in C order
// over an internal axis permutation ax[0..d-1] whose LAST axis is the
// stream axis of the assembly kernel (the longest one), so the rows a
// pencil produces are contiguous.  Only the boundary kernels (expand,
// CSR export) translate to the reference's C order over the original
// axes (assembly.py:84-96, 313-316).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sgiga.h"

namespace sgiga {

constexpr int MAXD = 3;
constexpr int PMAX = 5;   // p + 1 <= 5 (degree <= 4) on the device path
constexpr int QMAX = 10;  // gauss_rule accepts q <= 10 (assembly.py:43)
constexpr int WMAX = 2 * PMAX - 1;  // stencil slots per axis (2p+1)
constexpr int GEO_PMAX = 8;         // geometry degree <= 7
// 2-D components whose longest axis exceeds this run the line-FD PCG along
// it (only the short axis is diagonalised), not the full FD: the largest
// eigen-problems (m ~ 33..72, Jacobi, one SM) were the critical path of cfg1 / cfg3
constexpr int FD_FULL_MMAX2 = 24;
constexpr int FD_MMAX = 72;         // FD preconditioner: interior functions per diagonalised axis (smem eigen)
constexpr int64_t FDG_MIN_ROWS = 65536;   // FD components at least this large: whole-GPU PCG (k_pcg_grid.cu)
constexpr int FDG_MAX_CTAS = 1024;        // cooperative grid cap (partial-sum buffer size)
constexpr int COMBINE_SORT_BITS = 12;                      // cell sort of the combine points
constexpr int COMBINE_SORT_BINS = 1 << COMBINE_SORT_BITS;

// device error flags (bit mask in Handle::d_err)
enum : int { ERRF_GEOMETRY = 1, ERRF_NONFINITE = 2, ERRF_SPAN = 4, ERRF_POINTS = 16 };   // 8: cluster shape

struct TabInfo {        // one analysis knot vector = (axis, level)
    int axis, level;
    int nel, nk, n;     // elements, knots, functions
    int uniform;        // 1: breakpoints are exactly j/nel with nel a power of two
    int64_t bp_off;     // breakpoints (nel+1) in d_bp
    int64_t knot_off;   // knots in d_knots
    int64_t val_off;    // basis values [nel][q][P]; derivs at +nel*q*P
    int64_t qp_off;     // quad points xi [nel*q] in d_qx, weights in d_qw
    int64_t geo_off;    // geometry basis at quad points: [nel*q][2][GEO_PMAX]
};

struct CompInfo {
    int lv[MAXD];       // level per original axis
    int n[MAXD];        // full function count per original axis
    int m[MAXD];        // interior count (n - 2)
    int nel[MAXD];
    int tab[MAXD];      // TabInfo index per original axis
    int ax[MAXD];       // internal axis order (outer -> inner), ax[d-1] = stream
    int S[MAXD];        // stencil slots per ORIGINAL axis
    int absm[MAXD];     // 1 = absolute column slots (m <= 2p+1), 0 = relative
    int coef;           // combination coefficient
    int small;          // 1 = solved by the one-CTA PCG path
    int64_t rows;       // prod m
    int64_t nslots;     // prod S
    int64_t rs[MAXD];   // internal row stride of ORIGINAL axis k
    int64_t ss[MAXD];   // internal slot stride of ORIGINAL axis k
    int64_t halo;       // vector padding on both sides
    int64_t vec_off;    // position of internal row 0 in the padded vectors
    int64_t mat_off;    // stencil values: mat_off + slot*rows + row
    int64_t qp_off;     // metric/load: qp_off + comp*nqp + qp (storage order s,a,b)
    int64_t nqp;        // prod nel*q
    int64_t qs[MAXD];   // qp storage stride of ORIGINAL axis k
    int64_t dof_off;    // full coefficient vector offset
    int64_t ndofs;
    int64_t so_off;     // slot column-offset table: col = rowbase(row) + off[slot]
    int64_t chunk_off;  // first PCG chunk (large path)
    int nchunks;
    int fd;             // 1 = solved by the FD-preconditioned one-CTA CG (k_fd.cu)
    int tile3;          // 1 = assembled by the tiled 3-D kernel (k_assembly_tile.cu; per component:
                        //     the choice never depends on the batch the component is in)
};

struct GeoInfo {
    int d;
    int deg[MAXD], nk[MAXD], n[MAXD];
    int64_t knot_off[MAXD];
};

struct CgState;
// k_status fused into the last CTA of the tiled combine (sgiga_run passes)
struct StatusFuse {
    const CgState* st;
    const double* relres;
    int ncomp;
    CgState* hst;
    double* hrel;
    int* herr;
    int* hsticky;       // failure word OR-ed over pipelined passes (mapped host memory)
    unsigned* ticket;   // nullptr: not fused
};


struct Pencil {         // one CTA of the assembly kernel
    int comp;
    int ia, ib;         // full function index along tile axes ax[d-2], ax[d-3]
    int r0, r1;         // full function row range [r0, r1) along the stream axis
};

// one CTA of the tiled 3-D assembly (k_assembly_tile.cu): a block of the
// cross-section (rows a0 .. a0+na-1 along a = ax[1], b0 .. b0+nb-1 along
// b = ax[0], full function indices) times a segment [r0, r1) of the stream
// axis ax[2]; xa / xb = the component's union plane-window extents (points),
// xap = the TMA box's inner extent (the plane buffer's row stride); cw =
// stage-2 columns per work item (1 or 2)
struct Tile3 {
    int comp;
    int a0, na, b0, nb;
    int r0, r1;
    int xa, xap, xb;
    int cw;
};
#ifndef SGIGA_TILE3_G12
#define SGIGA_TILE3_G12 256
#endif
constexpr int TILE3_G12 = SGIGA_TILE3_G12;     // stage-1/2 threads (warps 0 .. G12/32 - 1)
constexpr int TILE3_G3 = 128;                  // stage-3 threads (the last 4 warps, one per TMEM lane quadrant)
constexpr int TILE3_THREADS = TILE3_G12 + TILE3_G3;
// TMEM columns of one stage-3 work item: the ring -- P physical stream rows
// (row R at R mod P) of 2p+1 doubles -- and the current element's P x P
// partial block, two 32-bit columns per double (p = 4: 90 + 50 columns,
// 3 items per thread; p = 3: 56 + 32, 5 items)
__host__ __device__ constexpr int tile3_ring_cols(int P) { return 2 * P * (2 * P - 1); }
__host__ __device__ constexpr int tile3_r3_cols(int P) { return 2 * P * P; }   // at the slot start (16-aligned)
__host__ __device__ constexpr int tile3_slot_cols(int P) { return (tile3_r3_cols(P) + tile3_ring_cols(P) + 15) & ~15; }
__host__ __device__ constexpr int tile3_nslot(int P) { return 512 / tile3_slot_cols(P); }   // rings per stage-3 thread

constexpr int ASM2_BA = 8;   // 2-D assembly: tile rows per block (k_assembly2d.cu)
struct Block2 {         // one CTA of the 2-D assembly kernel
    int comp;
    int walk;           // original axis the block walks along; the other is tiled
    int ia0, na;        // tile rows [ia0, ia0 + na) (full indices)
    int r0, r1;         // walk rows [r0, r1) (full indices)
};

struct Chunk {          // PCG row block of a large component
    int comp;
    int row0;
    int nrow;
    int idx;            // chunk index within the component
};

struct CgState {
    double rho, alpha, beta, bb, rr;
    int it, active, conv, pad;
    unsigned int cnt1, cnt2;
};

// a component's pass failed (linsolve.py:47-53 verdict, evaluated on the
// device so pipelined passes can OR it into a sticky word)
__device__ __forceinline__ bool cg_failed(const CgState& s, double rel) {
    if (s.bb == 0.0) return false;   // empty interior / zero right-hand side
    return !isfinite(rel) || !s.conv || rel > 1e-10;
}

// ---- Cox-de Boor (NURBS book A2.3) with the reference's rounding -------
// splines.py:172-224.  __dadd_rn/__dmul_rn keep nvcc from contracting
// into FMAs, so tables are bitwise equal to the reference's numpy scalars.
__device__ __forceinline__ void ders_basis_funs(int i, double xi, int p, int nders,
                                                const double* __restrict__ knots,
                                                double* ders /* [(nders+1)*(p+1)] */) {
    double ndu[PMAX + 3][PMAX + 3];
    double left[PMAX + 3], right[PMAX + 3], a[2][PMAX + 3];
    ndu[0][0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = __dsub_rn(xi, knots[i + 1 - j]);
        right[j] = __dsub_rn(knots[i + j], xi);
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            ndu[j][r] = __dadd_rn(right[r + 1], left[j - r]);
            double temp = __ddiv_rn(ndu[r][j - 1], ndu[j][r]);
            ndu[r][j] = __dadd_rn(saved, __dmul_rn(right[r + 1], temp));
            saved = __dmul_rn(left[j - r], temp);
        }
        ndu[j][j] = saved;
    }
    for (int j = 0; j <= p; ++j) ders[j] = ndu[j][p];
    if (nders == 0) return;
    for (int k = 1; k <= nders; ++k)
        for (int j = 0; j <= p; ++j) ders[k * (p + 1) + j] = 0.0;
    int kmax = nders < p ? nders : p;
    for (int r = 0; r <= p; ++r) {
        int s1 = 0, s2 = 1;
        a[0][0] = 1.0;
        for (int k = 1; k <= kmax; ++k) {
            double dd = 0.0;
            int rk = r - k, pk = p - k;
            if (r >= k) {
                a[s2][0] = __ddiv_rn(a[s1][0], ndu[pk + 1][rk]);
                dd = __dmul_rn(a[s2][0], ndu[rk][pk]);
            }
            int j1 = (rk >= -1) ? 1 : -rk;
            int j2 = (r - 1 <= pk) ? k - 1 : p - r;
            for (int j = j1; j <= j2; ++j) {
                a[s2][j] = __ddiv_rn(__dsub_rn(a[s1][j], a[s1][j - 1]), ndu[pk + 1][rk + j]);
                dd = __dadd_rn(dd, __dmul_rn(a[s2][j], ndu[rk + j][pk]));
            }
            if (r <= pk) {
                a[s2][k] = __ddiv_rn(-a[s1][k - 1], ndu[pk + 1][r]);
                dd = __dadd_rn(dd, __dmul_rn(a[s2][k], ndu[r][pk]));
            }
            ders[k * (p + 1) + r] = dd;
            int t = s1; s1 = s2; s2 = t;
        }
    }
    double fac = (double)p;
    for (int k = 1; k <= kmax; ++k) {
        for (int j = 0; j <= p; ++j) ders[k * (p + 1) + j] = __dmul_rn(ders[k * (p + 1) + j], fac);
        fac = __dmul_rn(fac, (double)(p - k));
    }
}

// Same recurrence with a compile-time degree: fully unrolled, register
// resident, identical rounding (values + first derivatives only).
template <int p>
__device__ __forceinline__ void ders_basis_funs_t(int i, double xi, const double* __restrict__ knots,
                                                  double* N, double* dN) {
    double ndu[p + 1][p + 1];
    double left[p + 1], right[p + 1];
    ndu[0][0] = 1.0;
#pragma unroll
    for (int j = 1; j <= p; ++j) {
        left[j] = __dsub_rn(xi, knots[i + 1 - j]);
        right[j] = __dsub_rn(knots[i + j], xi);
        double saved = 0.0;
#pragma unroll
        for (int r = 0; r < j; ++r) {
            ndu[j][r] = __dadd_rn(right[r + 1], left[j - r]);
            double temp = __ddiv_rn(ndu[r][j - 1], ndu[j][r]);
            ndu[r][j] = __dadd_rn(saved, __dmul_rn(right[r + 1], temp));
            saved = __dmul_rn(left[j - r], temp);
        }
        ndu[j][j] = saved;
    }
#pragma unroll
    for (int j = 0; j <= p; ++j) N[j] = ndu[j][p];
    if (dN == nullptr) return;
    // first derivatives (k = 1 of A2.3): a[s2][0] = 1/ndu[p][r-1], ...
#pragma unroll
    for (int r = 0; r <= p; ++r) {
        double d = 0.0;
        if (r >= 1) d = __dmul_rn(__ddiv_rn(1.0, ndu[p][r - 1]), ndu[r - 1][p - 1]);
        if (r <= p - 1) d = __dadd_rn(d, __dmul_rn(__ddiv_rn(-1.0, ndu[p][r]), ndu[r][p - 1]));
        dN[r] = __dmul_rn(d, (double)p);
    }
}

// _find_span (splines.py:149-169) on a full knot vector.
__device__ __forceinline__ int find_span(const double* __restrict__ k, int nk, int p, double xi,
                                         bool left) {
    int n = nk - p - 1, lo = 0, hi = nk;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        bool go = left ? (k[mid] < xi) : (k[mid] <= xi);
        if (go) lo = mid + 1; else hi = mid;
    }
    int i = lo - 1;
    if (i < p) i = p;
    if (i > n - 1) i = n - 1;
    while (k[i] == k[i + 1]) i = left ? i - 1 : i + 1;
    return i;
}

// ---- launchers (defined in the .cu files) -------------------------------
struct Handle;

cudaError_t launch_basis_tables(Handle* h);
cudaError_t launch_metric(Handle* h);
cudaError_t launch_assembly(Handle* h);
int run_pcg(Handle* h, double rtol, int maxit);
int launch_pcg_cluster(Handle* h, double rtol, int maxit);
cudaError_t launch_residual_check(Handle* h);
cudaError_t launch_solve_prologue(Handle* h, cudaStream_t stream);
cudaError_t launch_fd_eigen(Handle* h, cudaStream_t s);
cudaError_t launch_pcg_fd(Handle* h, double rtol, int maxit, cudaStream_t stream = nullptr);
cudaError_t launch_pcg_fdl(Handle* h, double rtol, int maxit);
cudaError_t launch_fd_setup(Handle* h, cudaStream_t s);
cudaError_t launch_pcg_fdg(Handle* h, double rtol, int maxit);
size_t fd_comp_smem(const CompInfo& C, int d);
cudaError_t launch_status(Handle* h);
cudaError_t launch_expand(Handle* h);
cudaError_t launch_combine_points(Handle* h, const double* d_pts, int64_t npts, double* d_out,
                                  int per_component, bool* status_fused = nullptr);
// cell sort of the combine points on stream s; *sorted = false when the
// point set is not sorted (too small / too large / SGIGA_COMBINE_NOSORT)
cudaError_t launch_combine_sort(Handle* h, const double* d_pts, int64_t npts, cudaStream_t s, bool* sorted);
cudaError_t launch_combine_grid(Handle* h, const double* d_pts, const int64_t* npd, int comp,
                                double* d_vals, double* d_grads);
cudaError_t launch_error_norms(Handle* h, const double* d_pts, const double* d_wts,
                               const int64_t* npd, int solution_id, double* d_partials,
                               int64_t* nblocks, const int* d_tcomp = nullptr, const double* d_tw = nullptr,
                               int nterm = 0);

}  // namespace sgiga
