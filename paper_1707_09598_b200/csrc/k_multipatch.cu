// k_multipatch.cu -- device pieces of the multipatch path (BASELINE cfg4:
// three bilinear patches glued C0, non-homogeneous Dirichlet lifting,
// one-sided graded knots).  SURVEY.md section 8(f) row 1.
//
// The reference has no multipatch code path:
// this extends its single-patch discretisation (assembly.py:357-390) the way
// GeoPDEs does -- per-patch FULL stiffness (every function, boundary rows
// included), a global C0 dof map across conforming interfaces, Dirichlet
// values by L2 projection of the data onto the boundary trace space, and the
// lifted interior system  A_II u_I = b_I - A_IB u_B.  Parity is against the
// repository's own restatement (oracle/multipatch_oracle.py): unpinned.
//
// The host (paper_1707_09598_b200/multipatch.py) only builds integer maps
// (global numbering, CSR structure, contribution lists); every floating-point
// step runs here:
//   * k_full_patch      -- full-patch stencil (relative offsets, C-order rows)
//                          and load vector of one component of a patch handle
//   * k_edge_projection -- 1-D mass band and data moments on one patch edge
//   * k_gather_sum      -- CSR values = fixed-order sums of contributions
//   * k_csr_pcg         -- batched Jacobi-PCG, one CTA per system
//   * k_csr_spmv_sub, k_gather -- lifting and expansion
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "forcing.cuh"
#include "handle.cuh"

namespace sgiga {

constexpr int MP_THREADS = 256;

// ---- full-patch stencil -------------------------------------------------------
// entry (row i, offset o) = sum over the elements of both supports and their
// quadrature points of sum_{m,n} G_mn dB_i/dxi_m dB_j/dxi_n   (j = i + o);
// the load entry (o = 0 slot thread) = sum B_i L.  One thread per entry.
template <int D>
__global__ void __launch_bounds__(MP_THREADS)
k_full_patch(const CompInfo* __restrict__ comps, int c, const TabInfo* __restrict__ tabs,
             const double* __restrict__ vals, const double* __restrict__ Gbuf, int p, int mu, int q,
             double* __restrict__ out_vals, double* __restrict__ out_rhs) {
    const CompInfo& C = comps[c];
    const int W = 2 * p + 1, P = p + 1;
    int64_t rows = 1, nslots = 1;
    for (int k = 0; k < D; ++k) { rows *= C.n[k]; nslots *= W; }
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= rows * nslots) return;
    const int64_t slot = gid / rows, row = gid % rows;
    int ii[D], jj[D], elo[D], ehi[D];
    bool ok = true;
    {
        int64_t r = row, s = slot;
        for (int k = D - 1; k >= 0; --k) {
            ii[k] = (int)(r % C.n[k]); r /= C.n[k];
            const int o = (int)(s % W) - p; s /= W;
            jj[k] = ii[k] + o;
            if (jj[k] < 0 || jj[k] >= C.n[k]) ok = false;
        }
    }
    const bool center = slot == (nslots - 1) / 2;
    double acc = 0.0, accL = 0.0;
    if (ok) {
        for (int k = 0; k < D; ++k) {
            const int num = max(ii[k], jj[k]) - p;
            elo[k] = num <= 0 ? 0 : (num + mu - 1) / mu;
            ehi[k] = min(min(ii[k], jj[k]) / mu, C.nel[k] - 1);
            if (elo[k] > ehi[k]) ok = false;
        }
    }
    if (ok) {
        const double* Gc = Gbuf + C.qp_off;
        const int ncg = D * (D + 1) / 2;
        int e[D], g[D];
        for (int k = 0; k < D; ++k) e[k] = elo[k];
        while (true) {
            for (int k = 0; k < D; ++k) g[k] = 0;
            while (true) {
                // basis values / derivatives of i and j on every axis at this point
                double bi[D], di[D], bj[D], dj[D];
                int64_t lin = 0;
                for (int k = 0; k < D; ++k) {
                    const TabInfo& T = tabs[C.tab[k]];
                    const int64_t nq = (int64_t)T.nel * q;
                    const int64_t base = ((int64_t)e[k] * q + g[k]) * P;
                    const double* v = vals + T.val_off;
                    bi[k] = v[base + ii[k] - e[k] * mu];
                    di[k] = v[nq * P + base + ii[k] - e[k] * mu];
                    bj[k] = v[base + jj[k] - e[k] * mu];
                    dj[k] = v[nq * P + base + jj[k] - e[k] * mu];
                    lin += ((int64_t)e[k] * q + g[k]) * C.qs[k];
                }
                for (int m = 0; m < D; ++m) {
                    double gm = 1.0;
                    for (int k = 0; k < D; ++k) gm *= (k == m) ? di[k] : bi[k];
                    for (int n = 0; n < D; ++n) {
                        double gn = 1.0;
                        for (int k = 0; k < D; ++k) gn *= (k == n) ? dj[k] : bj[k];
                        acc += Gc[(int64_t)sym_index(D, m, n) * C.nqp + lin] * gm * gn;
                    }
                }
                if (center) {
                    double b = 1.0;
                    for (int k = 0; k < D; ++k) b *= bi[k];
                    accL += Gc[(int64_t)ncg * C.nqp + lin] * b;
                }
                int k = D - 1;   // next quadrature point (odometer)
                while (k >= 0 && ++g[k] == q) { g[k] = 0; --k; }
                if (k < 0) break;
            }
            int k = D - 1;       // next element
            while (k >= 0 && ++e[k] > ehi[k]) { e[k] = elo[k]; --k; }
            if (k < 0) break;
        }
    }
    out_vals[slot * rows + row] = acc;
    if (center) out_rhs[row] = accL;
}

// ---- boundary data projection: one edge of a 2-D patch ------------------------
// the edge runs along parametric axis `axis`, the other axis is fixed at
// `side` (0 or 1).  band[i*(2p+1) + (j-i+p)] = int B_i B_j |dx/dxi|,
// rhs[i] = int g(x) B_i |dx/dxi|, g = the device closed form `sol_id`.
__global__ void __launch_bounds__(MP_THREADS)
k_edge_projection(const CompInfo* __restrict__ comps, int c, const TabInfo* __restrict__ tabs,
                  const double* __restrict__ vals, const double* __restrict__ qx,
                  const double* __restrict__ qw, const GeoInfo* __restrict__ geo,
                  const double* __restrict__ gknots, const double* __restrict__ hw, int p, int mu,
                  int q, int axis, int side, int sol_id, double* __restrict__ band,
                  double* __restrict__ rhs) {
    const CompInfo& C = comps[c];
    const TabInfo T = tabs[C.tab[axis]];
    const int n = T.n, W = 2 * p + 1, P = p + 1;
    const int64_t nq = (int64_t)T.nel * q;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * (W + 1); idx += gridDim.x * blockDim.x) {
        const int i = idx / (W + 1), o = idx % (W + 1) - p;   // o == p + 1: the rhs entry
        const bool is_rhs = o == p + 1;
        const int j = is_rhs ? i : i + o;
        double acc = 0.0;
        if (j >= 0 && j < n) {
            const int num = max(i, j) - p;
            const int elo = num <= 0 ? 0 : (num + mu - 1) / mu;
            const int ehi = min(min(i, j) / mu, T.nel - 1);
            for (int e = elo; e <= ehi; ++e)
                for (int g = 0; g < q; ++g) {
                    const int64_t qi = (int64_t)e * q + g;
                    const double* v = vals + T.val_off + qi * P;
                    const double bi = v[i - e * mu], bj = v[j - e * mu];
                    // map and tangent at (xi_axis, side)
                    double xi[2];
                    xi[axis] = qx[T.qp_off + qi];
                    xi[1 - axis] = (double)side;
                    const GeoInfo G = *geo;
                    int first[2];
                    double bv[2][GEO_PMAX + 1], bd[2][GEO_PMAX + 1];
                    for (int k = 0; k < 2; ++k) {
                        const double* kk = gknots + G.knot_off[k];
                        const int span = find_span(kk, G.nk[k], G.deg[k], xi[k], xi[k] == 1.0);
                        double tab[2 * (GEO_PMAX + 1)];
                        ders_basis_funs(span, xi[k], G.deg[k], 1, kk, tab);
                        first[k] = span - G.deg[k];
                        for (int a = 0; a <= G.deg[k]; ++a) { bv[k][a] = tab[a]; bd[k][a] = tab[G.deg[k] + 1 + a]; }
                    }
                    double hom[3] = {0, 0, 0}, dh[3] = {0, 0, 0};   // along `axis`
                    for (int a = 0; a <= G.deg[0]; ++a)
                        for (int b = 0; b <= G.deg[1]; ++b) {
                            const int64_t L = (int64_t)(first[0] + a) * G.n[1] + (first[1] + b);
                            const double pv = bv[0][a] * bv[1][b];
                            const double pd = axis == 0 ? bd[0][a] * bv[1][b] : bv[0][a] * bd[1][b];
                            for (int cc = 0; cc < 3; ++cc) {
                                hom[cc] += pv * hw[L * 3 + cc];
                                dh[cc] += pd * hw[L * 3 + cc];
                            }
                        }
                    double x[2], t2 = 0.0;
                    for (int cc = 0; cc < 2; ++cc) {
                        x[cc] = hom[cc] / hom[2];
                        const double tc = (dh[cc] - x[cc] * dh[2]) / hom[2];
                        t2 += tc * tc;
                    }
                    const double wj = qw[T.qp_off + qi] * sqrt(t2);
                    if (is_rhs) {
                        double u, gr[2];
                        solution_value<2>(sol_id, x, u, gr);
                        acc += wj * u * bi;
                    } else {
                        acc += wj * bi * bj;
                    }
                }
        }
        if (is_rhs) rhs[i] = acc;
        else band[(int64_t)i * W + (o + p)] = acc;
    }
}

// the same moments for MANY edges of one patch handle in one launch: one
// CTA per edge; the per-quadrature-point quantities (map, tangent length,
// Dirichlet data) are computed once per point into shared memory instead of
// once per (band entry, point)
__global__ void __launch_bounds__(MP_THREADS)
k_edge_projection_batch(const CompInfo* __restrict__ comps, const TabInfo* __restrict__ tabs,
                        const double* __restrict__ vals, const double* __restrict__ qx,
                        const double* __restrict__ qw, const GeoInfo* __restrict__ geo,
                        const double* __restrict__ gknots, const double* __restrict__ hw, int p, int mu,
                        int q, const int* __restrict__ edges, const int64_t* __restrict__ offs, int sol_id,
                        double* __restrict__ base) {
    extern __shared__ double esm[];
    const int c = edges[3 * blockIdx.x], axis = edges[3 * blockIdx.x + 1], side = edges[3 * blockIdx.x + 2];
    const CompInfo& C = comps[c];
    const TabInfo T = tabs[C.tab[axis]];
    const int n = T.n, W = 2 * p + 1, P = p + 1, nq = T.nel * q;
    double* sw = esm;        // w_j |dx/dxi|
    double* sg = esm + nq;   // w_j |dx/dxi| g(x)
    const GeoInfo G = *geo;
    for (int qi = threadIdx.x; qi < nq; qi += MP_THREADS) {
        double xi[2];
        xi[axis] = qx[T.qp_off + qi];
        xi[1 - axis] = (double)side;
        int first[2];
        double bv[2][GEO_PMAX + 1], bd[2][GEO_PMAX + 1];
        for (int k = 0; k < 2; ++k) {
            const double* kk = gknots + G.knot_off[k];
            const int span = find_span(kk, G.nk[k], G.deg[k], xi[k], xi[k] == 1.0);
            double tab[2 * (GEO_PMAX + 1)];
            ders_basis_funs(span, xi[k], G.deg[k], 1, kk, tab);
            first[k] = span - G.deg[k];
            for (int a = 0; a <= G.deg[k]; ++a) { bv[k][a] = tab[a]; bd[k][a] = tab[G.deg[k] + 1 + a]; }
        }
        double hom[3] = {0, 0, 0}, dh[3] = {0, 0, 0};   // along `axis`
        for (int a = 0; a <= G.deg[0]; ++a)
            for (int b = 0; b <= G.deg[1]; ++b) {
                const int64_t L = (int64_t)(first[0] + a) * G.n[1] + (first[1] + b);
                const double pv = bv[0][a] * bv[1][b];
                const double pd = axis == 0 ? bd[0][a] * bv[1][b] : bv[0][a] * bd[1][b];
                for (int cc = 0; cc < 3; ++cc) {
                    hom[cc] += pv * hw[L * 3 + cc];
                    dh[cc] += pd * hw[L * 3 + cc];
                }
            }
        double x[2], t2 = 0.0;
        for (int cc = 0; cc < 2; ++cc) {
            x[cc] = hom[cc] / hom[2];
            const double tc = (dh[cc] - x[cc] * dh[2]) / hom[2];
            t2 += tc * tc;
        }
        const double wj = qw[T.qp_off + qi] * sqrt(t2);
        double u, gr[2];
        solution_value<2>(sol_id, x, u, gr);
        sw[qi] = wj;
        sg[qi] = wj * u;
    }
    __syncthreads();
    double* band = base + offs[blockIdx.x];
    double* rhs = band + (int64_t)n * W;
    for (int idx = threadIdx.x; idx < n * (W + 1); idx += MP_THREADS) {
        const int i = idx / (W + 1), o = idx % (W + 1) - p;   // o == p + 1: the rhs entry
        const bool is_rhs = o == p + 1;
        const int j = is_rhs ? i : i + o;
        double acc = 0.0;
        if (j >= 0 && j < n) {
            const int num = max(i, j) - p;
            const int elo = num <= 0 ? 0 : (num + mu - 1) / mu;
            const int ehi = min(min(i, j) / mu, T.nel - 1);
            for (int e = elo; e <= ehi; ++e)
                for (int g = 0; g < q; ++g) {
                    const int qi = e * q + g;
                    const double* v = vals + T.val_off + (int64_t)qi * P;
                    const double bi = v[i - e * mu];
                    acc += is_rhs ? sg[qi] * bi : sw[qi] * bi * v[j - e * mu];
                }
        }
        if (is_rhs) rhs[i] = acc;
        else band[(int64_t)i * W + (o + p)] = acc;
    }
}

// ---- sparse helpers --------------------------------------------------------------
__global__ void k_gather_sum(int64_t n, const int64_t* __restrict__ start, const int64_t* __restrict__ idx,
                             const double* __restrict__ src, double* __restrict__ dst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double s = 0.0;
    for (int64_t t = start[k]; t < start[k + 1]; ++t) s += src[idx[t]];   // fixed order
    dst[k] = s;
}

__global__ void k_gather(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    dst[k] = idx[k] >= 0 ? src[idx[k]] : 0.0;
}

__global__ void k_csr_spmv_sub(int64_t nrows, const int64_t* __restrict__ rowptr, const int* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ x,
                               double* __restrict__ y) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    double s = 0.0;
    for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) s += val[k] * x[col[k]];
    y[r] -= s;
}

__device__ __forceinline__ double mp_block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < MP_THREADS / 32; ++w) s += red[w];
    return s;
}

// batched Jacobi-PCG on CSR systems (rows [off[s], off[s+1]) of one
// concatenated matrix; columns index the concatenated vector)
__global__ void __launch_bounds__(MP_THREADS)
k_csr_pcg(const int64_t* __restrict__ off, const int64_t* __restrict__ rowptr, const int* __restrict__ col,
          const double* __restrict__ val, const double* __restrict__ b, double* __restrict__ x,
          double* __restrict__ work, double rtol2, int maxit, int* __restrict__ iters,
          double* __restrict__ relres) {
    __shared__ double red[MP_THREADS / 32];
    const int s = blockIdx.x, tid = threadIdx.x;
    const int64_t r0 = off[s], r1 = off[s + 1], n = r1 - r0, N = off[gridDim.x];
    double* rr = work;            // [N] each: r, z, p, q, dinv
    double* zz = work + N;
    double* pp = work + 2 * N;
    double* qq = work + 3 * N;
    double* di = work + 4 * N;
    double bbl = 0.0;
    for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) {
        double dg = 0.0;
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) if (col[k] == i) dg = val[k];
        di[i] = dg != 0.0 ? 1.0 / dg : 0.0;
        x[i] = 0.0;
        rr[i] = b[i];
        zz[i] = di[i] * b[i];
        pp[i] = zz[i];
        bbl += b[i] * b[i];
    }
    const double bb = mp_block_sum(bbl, red);
    double rzl = 0.0;
    for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) rzl += rr[i] * zz[i];
    double rz = mp_block_sum(rzl, red);
    int it = 0, restarts = 0;
    bool conv = bb == 0.0 || n == 0;
    // residual replacement: once the recursive residual has converged, the
    // true one is checked; if rounding drift (strongly graded meshes) left
    // it above 1e-10, CG restarts from b - A x (at most 3 times)
    while (true) {
    while (!conv && it < maxit) {
        double pql = 0.0;
        for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) {
            double y = 0.0;
            for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) y += val[k] * pp[col[k]];
            qq[i] = y;
            pql += pp[i] * y;
        }
        const double alpha = rz / mp_block_sum(pql, red);
        double rrl = 0.0;
        for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) {
            x[i] += alpha * pp[i];
            rr[i] -= alpha * qq[i];
            zz[i] = di[i] * rr[i];
            rrl += rr[i] * rr[i];
        }
        const double rrs = mp_block_sum(rrl, red);
        ++it;
        if (rrs <= rtol2 * bb) { conv = true; break; }
        double rzl2 = 0.0;
        for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) rzl2 += rr[i] * zz[i];
        const double rzn = mp_block_sum(rzl2, red);
        const double beta = rzn / rz;
        rz = rzn;
        for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) pp[i] = zz[i] + beta * pp[i];
        __syncthreads();
    }
    // true residual (linsolve.py:49-53 acceptance)
    double eel = 0.0;
    for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) {
        double y = 0.0;
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) y += val[k] * x[col[k]];
        const double e = b[i] - y;
        rr[i] = e;
        eel += e * e;
    }
    const double ee = mp_block_sum(eel, red);
    if (!conv || bb == 0.0 || ee <= 1e-20 * bb || restarts >= 3 || it >= maxit) {
        if (tid == 0) {
            iters[s] = conv ? it : -it - 1;
            relres[s] = bb > 0.0 ? sqrt(ee / bb) : sqrt(ee);
        }
        return;
    }
    ++restarts;
    conv = false;
    double rzl3 = 0.0;
    for (int64_t i = r0 + tid; i < r1; i += MP_THREADS) {
        zz[i] = di[i] * rr[i];
        pp[i] = zz[i];
        rzl3 += rr[i] * zz[i];
    }
    rz = mp_block_sum(rzl3, red);
    }
}

// the same batched Jacobi-PCG with every vector of a system in SHARED
// memory and 1024 threads per system: the CSR matrix streams from L2/L1,
// the gathers p[col] hit shared memory (the global-memory variant above is
// the fallback for systems too large for a CTA)
constexpr int MPS_THREADS = 1024;

__device__ __forceinline__ double mps_block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < MPS_THREADS / 32; ++w) s += red[w];
    return s;
}

__global__ void __launch_bounds__(MPS_THREADS)
k_csr_pcg_smem(const int64_t* __restrict__ off, const int64_t* __restrict__ rowptr, const int* __restrict__ col,
               const double* __restrict__ val, const double* __restrict__ b, double* __restrict__ x,
               double rtol2, int maxit, int* __restrict__ iters, double* __restrict__ relres) {
    extern __shared__ double ps[];
    __shared__ double red[MPS_THREADS / 32];
    const int s = blockIdx.x, tid = threadIdx.x;
    const int64_t r0 = off[s], r1 = off[s + 1];
    const int n = (int)(r1 - r0);
    double* xs = ps;              // [n] each: x, r, z, p, q, dinv
    double* rr = xs + n;
    double* zz = rr + n;
    double* pp = zz + n;
    double* qq = pp + n;
    double* di = qq + n;
    double bbl = 0.0;
    for (int i = tid; i < n; i += MPS_THREADS) {
        const int64_t gi = r0 + i;
        double dg = 0.0;
        for (int64_t k = rowptr[gi]; k < rowptr[gi + 1]; ++k) if (col[k] == gi) dg = val[k];
        di[i] = dg != 0.0 ? 1.0 / dg : 0.0;
        const double bi = b[gi];
        xs[i] = 0.0;
        rr[i] = bi;
        zz[i] = di[i] * bi;
        pp[i] = zz[i];
        bbl += bi * bi;
    }
    const double bb = mps_block_sum(bbl, red);
    double rzl = 0.0;
    for (int i = tid; i < n; i += MPS_THREADS) rzl += rr[i] * zz[i];
    double rz = mps_block_sum(rzl, red);
    int it = 0, restarts = 0;
    bool conv = bb == 0.0 || n == 0;
    // out = A v: SPL lanes per row (a row's entries are read as contiguous
    // runs across the lanes -- many independent loads in flight, the matrix
    // streams from L2 every iteration), lane partials reduced by a fixed
    // butterfly; returns this thread's share of (w, out) for the dot product
    // four row groups per pass: their loads are all in flight before the
    // first is consumed (the L2 latency, not the bandwidth, bounds one SM)
    constexpr int SPL = 8, RPP = 4, RW = MPS_THREADS / SPL;
    auto spmv = [&](const double* v, double* out, const double* w) -> double {
        const int sub = tid & (SPL - 1);
        double dot = 0.0;
        for (int i0 = 0; i0 < n; i0 += RPP * RW) {
            double y[RPP];
            int64_t k[RPP], ke[RPP];
#pragma unroll
            for (int u = 0; u < RPP; ++u) {
                const int i = i0 + u * RW + tid / SPL;
                y[u] = 0.0;
                k[u] = ke[u] = 0;
                if (i < n) {
                    k[u] = __ldg(rowptr + r0 + i) + sub;
                    ke[u] = __ldg(rowptr + r0 + i + 1);
                }
            }
            bool more = true;
            while (more) {
                more = false;
#pragma unroll
                for (int u = 0; u < RPP; ++u)
                    if (k[u] < ke[u]) {
                        y[u] += __ldg(val + k[u]) * v[__ldg(col + k[u]) - r0];
                        k[u] += SPL;
                        more = more || k[u] < ke[u];
                    }
            }
#pragma unroll
            for (int u = 0; u < RPP; ++u) {
#pragma unroll
                for (int o = SPL / 2; o > 0; o >>= 1) y[u] += __shfl_xor_sync(0xffffffffu, y[u], o);
                const int i = i0 + u * RW + tid / SPL;
                if (i < n && sub == 0) {
                    out[i] = y[u];
                    if (w) dot += w[i] * y[u];
                }
            }
        }
        return dot;
    };
    // residual replacement as in k_csr_pcg (at most 3 restarts from b - A x)
    while (true) {
        while (!conv && it < maxit) {
            const double pql = spmv(pp, qq, pp);
            const double alpha = rz / mps_block_sum(pql, red);
            double rrl = 0.0, rzl2 = 0.0;
            for (int i = tid; i < n; i += MPS_THREADS) {
                xs[i] += alpha * pp[i];
                const double ri = rr[i] - alpha * qq[i];
                const double zi = di[i] * ri;
                rr[i] = ri;
                zz[i] = zi;
                rrl += ri * ri;
                rzl2 += ri * zi;
            }
            const double rrs = mps_block_sum(rrl, red);
            const double rzn = mps_block_sum(rzl2, red);
            ++it;
            if (rrs <= rtol2 * bb) { conv = true; break; }
            const double beta = rzn / rz;
            rz = rzn;
            for (int i = tid; i < n; i += MPS_THREADS) pp[i] = zz[i] + beta * pp[i];
            __syncthreads();
        }
        __syncthreads();
        spmv(xs, qq, nullptr);   // true residual (linsolve.py:49-53 acceptance)
        __syncthreads();
        double eel = 0.0;
        for (int i = tid; i < n; i += MPS_THREADS) {
            const double e = b[r0 + i] - qq[i];
            rr[i] = e;
            eel += e * e;
        }
        const double ee = mps_block_sum(eel, red);
        if (!conv || bb == 0.0 || ee <= 1e-20 * bb || restarts >= 3 || it >= maxit) {
            for (int i = tid; i < n; i += MPS_THREADS) x[r0 + i] = xs[i];
            if (tid == 0) {
                iters[s] = conv ? it : -it - 1;
                relres[s] = bb > 0.0 ? sqrt(ee / bb) : sqrt(ee);
            }
            return;
        }
        ++restarts;
        conv = false;
        double rzl3 = 0.0;
        for (int i = tid; i < n; i += MPS_THREADS) {
            zz[i] = di[i] * rr[i];
            pp[i] = zz[i];
            rzl3 += rr[i] * zz[i];
        }
        rz = mps_block_sum(rzl3, red);
    }
}

// ---- the batched CSR Jacobi-PCG on a thread-block CLUSTER per system -----
// (the one-SM kernels above are L2-latency bound: the whole matrix streams
// through one SM every iteration).  K = 8 CTAs per system, contiguous row
// slices; every CTA keeps its slice of the CSR matrix in shared memory and a
// full copy of u, the only gathered vector.  Chronopoulos-Gear PCG (one
// reduction of (r.u, w.u, r.r) per iteration, the scheme of k_pcg_cluster.cu)
// with the same residual-replacement restarts as k_csr_pcg; partials summed
// in fixed (rank, warp) order by every CTA: deterministic.
constexpr int MPC_THREADS = 512, MPC_WARPS = MPC_THREADS / 32, MPC_K = 8, MPC_SPL = 4;

__global__ void __launch_bounds__(MPC_THREADS, 1)
k_csr_pcg_cl(const int64_t* __restrict__ off, const int64_t* __restrict__ rowptr, const int* __restrict__ col,
             const double* __restrict__ val, const double* __restrict__ b, double* __restrict__ x,
             double rtol2, int maxit, int* __restrict__ iters, double* __restrict__ relres) {
    namespace cgs = cooperative_groups;
    cgs::cluster_group cluster = cgs::this_cluster();
    const int K = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
    extern __shared__ double cs[];
    const int sys = blockIdx.x / K, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = off[sys];
    const int n = (int)(off[sys + 1] - r0);
    const int RLmax = (n + K - 1) / K;
    const int lo = min(n, rank * RLmax), hi = min(n, lo + RLmax), RL = hi - lo;
    const int64_t k0 = rowptr[r0 + lo], nnzl = rowptr[r0 + hi] - k0;
    double* cred = cs;                                 // [3][MPC_K][MPC_WARPS]
    double* xs = cred + 3 * MPC_K * MPC_WARPS;         // own rows: x r u w p s d
    double* rs_ = xs + RLmax;
    double* us = rs_ + RLmax;
    double* ws = us + RLmax;
    double* pv = ws + RLmax;
    double* sv = pv + RLmax;
    double* ds = sv + RLmax;
    double* uf = ds + RLmax;                           // [n] full copy of u
    double* lv = uf + n;                               // [nnzl] own CSR values
    int* lc = reinterpret_cast<int*>(lv + nnzl);       // [nnzl] columns (system-local)
    int* lp = lc + nnzl;                               // [RL + 1] row starts (slice-local)
    for (int64_t k = tid; k < nnzl; k += MPC_THREADS) {
        lv[k] = val[k0 + k];
        lc[k] = (int)(col[k0 + k] - r0);
    }
    for (int i = tid; i <= RL; i += MPC_THREADS) lp[i] = (int)(rowptr[r0 + lo + i] - k0);
    __syncthreads();
    for (int il = tid; il < RL; il += MPC_THREADS) {   // Jacobi diagonal
        const int gi = lo + il;
        double dg = 0.0;
        for (int k = lp[il]; k < lp[il + 1]; ++k) if (lc[k] == gi) dg = lv[k];
        ds[il] = dg != 0.0 ? 1.0 / dg : 0.0;
        xs[il] = 0.0;
    }
    // broadcast own u slice into every rank's full copy
    auto bcast = [&](const double* src) {
        for (int il = tid; il < RL; il += MPC_THREADS) {
            const double v = src[il];
            for (int r = 0; r < K; ++r) cluster.map_shared_rank(uf, r)[lo + il] = v;
        }
    };
    auto sum3 = [&](double* v) {   // cluster-wide fixed-order sum of three values
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double a = __shfl_xor_sync(0xffffffffu, v[0], o);
            const double b2 = __shfl_xor_sync(0xffffffffu, v[1], o);
            const double c2 = __shfl_xor_sync(0xffffffffu, v[2], o);
            v[0] += a; v[1] += b2; v[2] += c2;
        }
        if (lane < K) {
            double* dst = cluster.map_shared_rank(cred, lane);
#pragma unroll
            for (int k = 0; k < 3; ++k) dst[(k * MPC_K + rank) * MPC_WARPS + warp] = v[k];
        }
        cluster.sync();
        const int np = K * MPC_WARPS;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double s = 0.0;
            for (int j = lane; j < np; j += 32) s += cred[k * MPC_K * MPC_WARPS + j];
            v[k] = s;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double a = __shfl_xor_sync(0xffffffffu, v[0], o);
            const double b2 = __shfl_xor_sync(0xffffffffu, v[1], o);
            const double c2 = __shfl_xor_sync(0xffffffffu, v[2], o);
            v[0] += a; v[1] += b2; v[2] += c2;
        }
    };
    // ws = A uf on own rows (MPC_SPL lanes per row, fixed butterfly), then the
    // partials of (r.u, w.u, r.r)
    auto spmv_dots = [&](double* dots) {
        const int sub = tid & (MPC_SPL - 1);
        for (int i0 = 0; i0 < RL; i0 += MPC_THREADS / MPC_SPL) {
            const int il = i0 + tid / MPC_SPL;
            double y = 0.0;
            if (il < RL)
                for (int k = lp[il] + sub; k < lp[il + 1]; k += MPC_SPL) y += lv[k] * uf[lc[k]];
#pragma unroll
            for (int o = MPC_SPL / 2; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
            if (il < RL && sub == 0) ws[il] = y;
        }
        __syncthreads();
        dots[0] = dots[1] = dots[2] = 0.0;
        for (int il = tid; il < RL; il += MPC_THREADS) {
            const double ri = rs_[il], ui = us[il];
            dots[0] += ri * ui;
            dots[1] += ws[il] * ui;
            dots[2] += ri * ri;
        }
    };
    // (re)start from the residual in rs_: u = D r, w = A u, scalars
    double dots[3], gamma = 0.0, alpha = 0.0, beta = 0.0, bb = 0.0;
    auto start = [&]() {
        for (int il = tid; il < RL; il += MPC_THREADS) us[il] = ds[il] * rs_[il];
        bcast(us);
        cluster.sync();
        spmv_dots(dots);
        sum3(dots);
        gamma = dots[0];
        alpha = dots[1] != 0.0 ? gamma / dots[1] : 0.0;
        beta = 0.0;
        for (int il = tid; il < RL; il += MPC_THREADS) { pv[il] = us[il]; sv[il] = ws[il]; }
        return dots[2];
    };
    for (int il = tid; il < RL; il += MPC_THREADS) rs_[il] = b[r0 + lo + il];
    __syncthreads();
    bb = start();
    int it = 0, restarts = 0;
    bool conv = bb == 0.0 || n == 0;
    double ee = 0.0;
    while (true) {
        while (!conv && it < maxit) {
            for (int il = tid; il < RL; il += MPC_THREADS) {
                xs[il] += alpha * pv[il];
                const double ri = rs_[il] - alpha * sv[il];
                rs_[il] = ri;
                us[il] = ds[il] * ri;
            }
            bcast(us);
            cluster.sync();   // u complete on every rank; cred free
            spmv_dots(dots);
            sum3(dots);
            ++it;
            if (dots[2] <= rtol2 * bb) { conv = true; break; }
            const double g_new = dots[0];
            beta = g_new / gamma;
            alpha = g_new / (dots[1] - beta * g_new / alpha);
            gamma = g_new;
            for (int il = tid; il < RL; il += MPC_THREADS) {
                pv[il] = us[il] + beta * pv[il];
                sv[il] = ws[il] + beta * sv[il];
            }
        }
        // true residual (linsolve.py:49-53 acceptance): x broadcast like u
        cluster.sync();
        bcast(xs);
        cluster.sync();
        spmv_dots(dots);   // ws = A x
        double ev[3] = {0.0, 0.0, 0.0};
        for (int il = tid; il < RL; il += MPC_THREADS) {
            const double e = b[r0 + lo + il] - ws[il];
            rs_[il] = e;
            ev[0] += isfinite(xs[il]) ? e * e : __longlong_as_double(0x7ff8000000000000ULL);
        }
        sum3(ev);
        ee = ev[0];
        if (!conv || bb == 0.0 || ee <= 1e-20 * bb || restarts >= 3 || it >= maxit) break;
        ++restarts;   // residual replacement from b - A x
        conv = false;
        cluster.sync();
        start();
    }
    for (int il = tid; il < RL; il += MPC_THREADS) x[r0 + lo + il] = xs[il];
    if (tid == 0 && rank == 0) {
        iters[sys] = conv ? it : -it - 1;
        relres[sys] = bb > 0.0 ? sqrt(ee / bb) : sqrt(ee);
    }
    cluster.sync();   // no CTA exits while others may still write into its smem
}

}  // namespace sgiga

using namespace sgiga;

extern "C" {

int sgiga_full_patch_system(sgiga_handle* hh, int32_t comp, double* d_vals, double* d_rhs) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !d_vals || !d_rhs) return SGIGA_ERR_VALUE;
    if (comp < 0 || comp >= h->ncomp) { set_error("component index out of range"); return SGIGA_ERR_KEY; }
    if (!h->assembled) { set_error("full patch system before assemble"); return SGIGA_ERR_STATE; }
    const CompInfo& C = h->comps[comp];
    int64_t rows = 1, ns = 1;
    for (int k = 0; k < h->d; ++k) { rows *= C.n[k]; ns *= 2 * h->p + 1; }
    const int64_t n = rows * ns;
    const unsigned blocks = (unsigned)((n + MP_THREADS - 1) / MP_THREADS);
    if (h->d == 1) k_full_patch<1><<<blocks, MP_THREADS, 0, h->stream>>>(h->d_comps, comp, h->d_tabs, h->d_tabvals, h->d_G, h->p, h->mu, h->q, d_vals, d_rhs);
    else if (h->d == 2) k_full_patch<2><<<blocks, MP_THREADS, 0, h->stream>>>(h->d_comps, comp, h->d_tabs, h->d_tabvals, h->d_G, h->p, h->mu, h->q, d_vals, d_rhs);
    else k_full_patch<3><<<blocks, MP_THREADS, 0, h->stream>>>(h->d_comps, comp, h->d_tabs, h->d_tabvals, h->d_G, h->p, h->mu, h->q, d_vals, d_rhs);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}

int sgiga_edge_projection_system(sgiga_handle* hh, int32_t comp, int32_t axis, int32_t side,
                                 int32_t solution_id, double* d_band, double* d_rhs) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !d_band || !d_rhs) return SGIGA_ERR_VALUE;
    if (h->d != 2) { set_error("edge projection: 2-D patches only"); return SGIGA_ERR_VALUE; }
    if (comp < 0 || comp >= h->ncomp || axis < 0 || axis > 1 || side < 0 || side > 1) {
        set_error("edge projection: bad component / axis / side");
        return SGIGA_ERR_VALUE;
    }
    if (!h->tables_ready) { set_error("edge projection before the basis tables"); return SGIGA_ERR_STATE; }
    const int n = h->comps[comp].n[axis];
    const unsigned blocks = (unsigned)((n * (2 * h->p + 2) + MP_THREADS - 1) / MP_THREADS);
    k_edge_projection<<<blocks, MP_THREADS, 0, h->stream>>>(h->d_comps, comp, h->d_tabs, h->d_tabvals, h->d_qx,
                                                            h->d_qw, h->d_geo, h->d_geo_knots, h->d_geo_hw,
                                                            h->p, h->mu, h->q, axis, side, solution_id, d_band,
                                                            d_rhs);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}

int sgiga_edge_projection_batch(sgiga_handle* hh, int32_t nedge, const int32_t* d_edges, const int64_t* d_offsets,
                                int32_t max_edge_qp, int32_t solution_id, double* d_base) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || (nedge > 0 && (!d_edges || !d_offsets || !d_base))) return SGIGA_ERR_VALUE;
    if (h->d != 2) { set_error("edge projection: 2-D patches only"); return SGIGA_ERR_VALUE; }
    if (nedge == 0) return SGIGA_OK;
    if (!h->tables_ready) { set_error("edge projection before the basis tables"); return SGIGA_ERR_STATE; }
    const size_t smem = sizeof(double) * 2 * (size_t)std::max(max_edge_qp, 1);
    if (smem > 200 * 1024) { set_error("edge projection: too many quadrature points per edge"); return SGIGA_ERR_VALUE; }
    SG_CUDA(cudaFuncSetAttribute(k_edge_projection_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_edge_projection_batch<<<(unsigned)nedge, MP_THREADS, smem, h->stream>>>(
        h->d_comps, h->d_tabs, h->d_tabvals, h->d_qx, h->d_qw, h->d_geo, h->d_geo_knots, h->d_geo_hw, h->p, h->mu,
        h->q, d_edges, d_offsets, solution_id, d_base);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}

int sgiga_gather_sum(void* stream, int64_t n, const int64_t* d_start, const int64_t* d_idx,
                     const double* d_src, double* d_dst) {
    if (n <= 0) return SGIGA_OK;
    k_gather_sum<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d_start, d_idx, d_src, d_dst);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}

int sgiga_gather(void* stream, int64_t n, const int64_t* d_idx, const double* d_src, double* d_dst) {
    if (n <= 0) return SGIGA_OK;
    k_gather<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, d_idx, d_src, d_dst);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}

int sgiga_csr_spmv_sub(void* stream, int64_t nrows, const int64_t* d_rowptr, const int32_t* d_col,
                       const double* d_val, const double* d_x, double* d_y) {
    if (nrows <= 0) return SGIGA_OK;
    k_csr_spmv_sub<<<(unsigned)((nrows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nrows, d_rowptr, d_col,
                                                                                      d_val, d_x, d_y);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}

int sgiga_csr_pcg(void* stream, int32_t nsys, const int64_t* d_off, int64_t nrows_total,
                  const int64_t* d_rowptr, const int32_t* d_col, const double* d_val, const double* d_b,
                  double* d_x, double rtol, int32_t maxit, int32_t* iters_out, double* relres_out) {
    if (nsys <= 0) return SGIGA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    {   // systems small enough for shared memory: the cluster kernel, else the
        // one-SM shared-memory kernel
        std::vector<int64_t> off(nsys + 1);
        SG_CUDA(cudaMemcpyAsync(off.data(), d_off, sizeof(int64_t) * (nsys + 1), cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaStreamSynchronize(s));
        int64_t nmax = 0;
        for (int i = 0; i < nsys; ++i) nmax = std::max(nmax, off[i + 1] - off[i]);
        std::vector<int64_t> rp(nrows_total + 1);
        SG_CUDA(cudaMemcpyAsync(rp.data(), d_rowptr, sizeof(int64_t) * (nrows_total + 1), cudaMemcpyDeviceToHost, s));
        SG_CUDA(cudaStreamSynchronize(s));
        int64_t cl_need = 0;
        for (int i = 0; i < nsys; ++i) {
            const int64_t n = off[i + 1] - off[i], RLm = (n + MPC_K - 1) / MPC_K;
            for (int r = 0; r < MPC_K; ++r) {
                const int64_t lo = std::min(n, r * RLm), hi = std::min(n, lo + RLm);
                const int64_t nnzl = rp[off[i] + hi] - rp[off[i] + lo];
                const int64_t bytes = 8 * (3 * MPC_K * MPC_WARPS + 7 * RLm + n + nnzl) + 4 * (nnzl + RLm + 1) + 16;
                cl_need = std::max(cl_need, bytes);
            }
        }
        if (cl_need <= 200 * 1024) {
            int* dit = nullptr;
            double* drr = nullptr;
            SG_CUDA(cudaMalloc(&dit, sizeof(int) * nsys));
            SG_CUDA(cudaMalloc(&drr, sizeof(double) * nsys));
            cudaError_t e = cudaFuncSetAttribute(k_csr_pcg_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_need);
            if (e == cudaSuccess) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)(nsys * MPC_K));
                cfg.blockDim = dim3(MPC_THREADS);
                cfg.dynamicSmemBytes = (size_t)cl_need;
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = MPC_K;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                e = cudaLaunchKernelEx(&cfg, k_csr_pcg_cl, d_off, d_rowptr, (const int*)d_col, d_val, d_b, d_x,
                                       rtol * rtol, maxit > 0 ? maxit : 1000000, dit, drr);
            }
            if (e == cudaSuccess) e = cudaMemcpyAsync(iters_out, dit, sizeof(int) * nsys, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(relres_out, drr, sizeof(double) * nsys, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            cudaFree(dit); cudaFree(drr);
            SG_CUDA(e);
            return SGIGA_OK;
        }
        const size_t smem = sizeof(double) * 6 * (size_t)std::max<int64_t>(nmax, 1);
        if (smem <= 200 * 1024) {
            int* dit = nullptr;
            double* drr = nullptr;
            SG_CUDA(cudaMalloc(&dit, sizeof(int) * nsys));
            SG_CUDA(cudaMalloc(&drr, sizeof(double) * nsys));
            cudaError_t e = cudaFuncSetAttribute(k_csr_pcg_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess) {
                k_csr_pcg_smem<<<(unsigned)nsys, MPS_THREADS, smem, s>>>(d_off, d_rowptr, d_col, d_val, d_b, d_x,
                                                                       rtol * rtol, maxit > 0 ? maxit : 1000000, dit, drr);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaMemcpyAsync(iters_out, dit, sizeof(int) * nsys, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(relres_out, drr, sizeof(double) * nsys, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            cudaFree(dit); cudaFree(drr);
            SG_CUDA(e);
            return SGIGA_OK;
        }
    }
    double* work = nullptr;
    int* dit = nullptr;
    double* drr = nullptr;
    SG_CUDA(cudaMalloc(&work, sizeof(double) * 5 * std::max<int64_t>(nrows_total, 1)));
    SG_CUDA(cudaMalloc(&dit, sizeof(int) * nsys));
    SG_CUDA(cudaMalloc(&drr, sizeof(double) * nsys));
    k_csr_pcg<<<(unsigned)nsys, MP_THREADS, 0, s>>>(d_off, d_rowptr, d_col, d_val, d_b, d_x, work,
                                                     rtol * rtol, maxit > 0 ? maxit : 1000000, dit, drr);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(iters_out, dit, sizeof(int) * nsys, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(relres_out, drr, sizeof(double) * nsys, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(work); cudaFree(dit); cudaFree(drr);
    SG_CUDA(e);
    return SGIGA_OK;
}

int sgiga_set_coefficients_device(sgiga_handle* hh, const double* d_full) {
    Handle* h = reinterpret_cast<Handle*>(hh);
    if (!h || !d_full) return SGIGA_ERR_VALUE;
    SG_CUDA(cudaMemcpyAsync(h->d_coef, d_full, sizeof(double) * h->total_dofs, cudaMemcpyDeviceToDevice, h->stream));
    SG_CUDA(cudaStreamSynchronize(h->stream));
    h->have_coefs = true;
    return SGIGA_OK;
}

}  // extern "C"
