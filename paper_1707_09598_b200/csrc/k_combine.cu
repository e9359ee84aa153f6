// k_combine.cu -- kernel 4: the combination step sum_beta c_beta u_beta at
// scattered points or on tensor grids (with parametric gradients), and the
// L2 / H1-seminorm error quadrature against a device closed form.
//
// Reference: combination.evaluate_combined (combination.py:209-236) with
// DiscreteSpace.eval_grid / _tensor_apply (assembly.py:101-138), the
// per-point idiom of tests/test_acceptance.py:224-230, and
// analysis.error_norms / _push_gradient (analysis.py:235-270).
//
// One thread per point, templated on (D, p) so the Cox-de Boor tables and
// the coefficient window stay in registers.  Components are visited in plan
// (lexicographic) order -- the accumulation order the reference guarantees
// -- and an axis' 1-D basis is recomputed only when its level changes
// between consecutive components.  The span of a uniform dyadic knot vector
// is closed-form (floor(xi*2^l), exact), graded ones use a binary search
// with the reference's side rule (splines.py:149-169, 255-257).
#include <cstdlib>

#include "forcing.cuh"
#include "handle.cuh"

namespace sgiga {

template <int P, bool GRAD>
__device__ __forceinline__ int axis_basis(const TabInfo& T, const double* __restrict__ knots,
                                          int mu, double xi, double* bv, double* bd) {
    constexpr int p = P - 1;
    const double* k = knots + T.knot_off;
    int span;
    if (T.uniform) {
        int e = (int)(xi * (double)T.nel);   // exact: nel is a power of two
        if (e > T.nel - 1) e = T.nel - 1;
        span = p + e * mu;
    } else {
        span = find_span(k, T.nk, p, xi, xi == 1.0);
    }
    ders_basis_funs_t<p>(span, xi, k, bv, GRAD ? bd : nullptr);
    return span - p;
}

// the P contiguous coefficients at row[0..P) by ceil((P+1)/2) aligned 16-byte
// loads (the coefficient buffer is padded by 2 doubles past its end)
template <int P>
__device__ __forceinline__ void load_row_v(const double* row, double* c) {
    constexpr int NV = (P + 2) / 2;
    const uintptr_t a = reinterpret_cast<uintptr_t>(row);
    const bool odd = (a & 8) != 0;
    const double2* r2 = reinterpret_cast<const double2*>(a & ~(uintptr_t)15);
    double w[2 * NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const double2 v = __ldg(r2 + i);
        w[2 * i] = v.x;
        w[2 * i + 1] = v.y;
    }
#pragma unroll
    for (int l = 0; l < P; ++l) c[l] = odd ? w[l + 1] : w[l];
}

// VEC: coefficient rows by 16-byte loads (coef must be the padded d_coef);
// same values, same operations
template <int D, int P, bool GRAD, bool VEC = false>
__device__ __forceinline__ void eval_component(const CompInfo& C, const double* __restrict__ coef,
                                               const int* first, const double (*Bv)[P],
                                               const double (*Bd)[P], double& v, double* g) {
    const double* cf = coef + C.dof_off;
    if constexpr (D == 1) {
        double sv = 0.0, sd = 0.0;
#pragma unroll
        for (int a = 0; a < P; ++a) {
            double c = cf[first[0] + a];
            sv += Bv[0][a] * c;
            if (GRAD) sd += Bd[0][a] * c;
        }
        v = sv;
        if (GRAD) g[0] = sd;
    } else if constexpr (D == 2) {
        const int n1 = C.n[1];
        double v0 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int a = 0; a < P; ++a) {
            const double* row = cf + (int64_t)(first[0] + a) * n1 + first[1];
            double tv = 0.0, td = 0.0;
            double cr[P];
            if constexpr (VEC) load_row_v<P>(row, cr);
#pragma unroll
            for (int b = 0; b < P; ++b) {
                double c = VEC ? cr[b] : __ldg(row + b);
                tv += Bv[1][b] * c;
                if (GRAD) td += Bd[1][b] * c;
            }
            v0 += Bv[0][a] * tv;
            if (GRAD) { g0 += Bd[0][a] * tv; g1 += Bv[0][a] * td; }
        }
        v = v0;
        if (GRAD) { g[0] = g0; g[1] = g1; }
    } else {
        const int n1 = C.n[1], n2 = C.n[2];
        double v0 = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
#pragma unroll
        for (int a = 0; a < P; ++a) {
            double uv = 0.0, u1 = 0.0, u2 = 0.0;
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double* row = cf + ((int64_t)(first[0] + a) * n1 + (first[1] + b)) * n2 + first[2];
                double tv = 0.0, td = 0.0;
                double cr[P];
                if constexpr (VEC) load_row_v<P>(row, cr);
#pragma unroll
                for (int l = 0; l < P; ++l) {
                    double c = VEC ? cr[l] : __ldg(row + l);
                    tv += Bv[2][l] * c;
                    if (GRAD) td += Bd[2][l] * c;
                }
                uv += Bv[1][b] * tv;
                if (GRAD) { u1 += Bd[1][b] * tv; u2 += Bv[1][b] * td; }
            }
            v0 += Bv[0][a] * uv;
            if (GRAD) { g0 += Bd[0][a] * uv; g1 += Bv[0][a] * u1; g2 += Bv[0][a] * u2; }
        }
        v = v0;
        if (GRAD) { g[0] = g0; g[1] = g1; g[2] = g2; }
    }
}

// sum over components [c_lo, c_hi) in plan order at one parametric point
template <int D, int P, bool GRAD>
__device__ __forceinline__ void combine_at(const CompInfo* __restrict__ comps, int c_lo, int c_hi,
                                           bool weighted, const TabInfo* __restrict__ tabs,
                                           const double* __restrict__ knots, int mu,
                                           const double* __restrict__ coef, const double* xi,
                                           double& acc, double* gacc, double* per_comp,
                                           int64_t per_stride) {
    int cur[D], first[D];
    double Bv[D][P], Bd[D][P];
#pragma unroll
    for (int k = 0; k < D; ++k) cur[k] = -1;
    bool started = false;
    acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) gacc[k] = 0.0;
    for (int c = c_lo; c < c_hi; ++c) {
        const CompInfo& C = comps[c];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            int t = C.tab[k];
            if (t != cur[k]) {
                cur[k] = t;
                first[k] = axis_basis<P, GRAD>(tabs[t], knots, mu, xi[k], Bv[k], Bd[k]);
            }
        }
        double v, g[D];
        eval_component<D, P, GRAD>(C, coef, first, Bv, Bd, v, g);
        if (per_comp) { per_comp[(int64_t)c * per_stride] = v; continue; }
        double cf = weighted ? (double)C.coef : 1.0;
        // vals = c*v, then vals += c*v in plan order (combination.py:227-233)
        if (!started) {
            acc = cf * v;
#pragma unroll
            for (int k = 0; k < D; ++k) gacc[k] = cf * g[k];
            started = true;
        } else {
            acc = __dadd_rn(acc, cf * v);
#pragma unroll
            for (int k = 0; k < D; ++k) gacc[k] = __dadd_rn(gacc[k], cf * g[k]);
        }
    }
}

// explicit signed term list (component index, weight) in the given order:
// acc = w0 v0, acc += w_t v_t -- the reference's surplus accumulation
// (combination.py:269-272) and, with the plan's terms, evaluate_combined
template <int D, int P, bool GRAD>
__device__ __forceinline__ void combine_terms(const CompInfo* __restrict__ comps,
                                              const int* __restrict__ tcomp, const double* __restrict__ tw,
                                              int nterm, const TabInfo* __restrict__ tabs,
                                              const double* __restrict__ knots, int mu,
                                              const double* __restrict__ coef, const double* xi,
                                              double& acc, double* gacc) {
    int cur[D], first[D];
    double Bv[D][P], Bd[D][P];
#pragma unroll
    for (int k = 0; k < D; ++k) cur[k] = -1;
    acc = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) gacc[k] = 0.0;
    for (int t = 0; t < nterm; ++t) {
        const CompInfo& C = comps[tcomp[t]];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            int tb = C.tab[k];
            if (tb != cur[k]) {
                cur[k] = tb;
                first[k] = axis_basis<P, GRAD>(tabs[tb], knots, mu, xi[k], Bv[k], Bd[k]);
            }
        }
        double v, g[D];
        eval_component<D, P, GRAD>(C, coef, first, Bv, Bd, v, g);
        const double cf = tw[t];
        if (t == 0) {
            acc = cf * v;
#pragma unroll
            for (int k = 0; k < D; ++k) gacc[k] = cf * g[k];
        } else {
            acc = __dadd_rn(acc, cf * v);
#pragma unroll
            for (int k = 0; k < D; ++k) gacc[k] = __dadd_rn(gacc[k], cf * g[k]);
        }
    }
}

template <int D, int P>
__global__ void __launch_bounds__(128)
k_combine_points(const CompInfo* __restrict__ comps, int ncomp, const TabInfo* __restrict__ tabs,
                 const double* __restrict__ knots, int mu, const double* __restrict__ coef,
                 const double* __restrict__ pts, int64_t npts, double* __restrict__ out,
                 int per_component, int* __restrict__ err) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts) return;
    double xi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        xi[k] = pts[t * D + k];
        if (!(xi[k] >= 0.0 && xi[k] <= 1.0)) atomicOr(err, ERRF_POINTS);   // evaluation points in [0,1]^d
    }
    double acc, g[D];
    combine_at<D, P, false>(comps, 0, ncomp, true, tabs, knots, mu, coef, xi, acc, g,
                            per_component ? out + t : nullptr, npts);
    if (!per_component) out[t] = acc;
}

// Scattered-point combine, tiled: a CTA owns NPT points and splits the work
// three ways so every thread has independent work (one thread per point
// leaves an SM with a handful of warps, latency-bound):
//   A. one item per (basis table = (axis, level), point): span + Cox-de Boor
//      values into shared memory (pt innermost: conflict-free) -- each
//      table is evaluated once per point, not once per component;
//   B. one item per (component, point): the P^D tensor contraction with the
//      component's coefficient window -> V[c][pt];
//   C. one thread per point: the plan-order sum acc = c0 v0, acc += c v
//      (combination.py:227-233) -- the same operations, in the same order,
//      as combine_at, so the result is bitwise the per-thread kernel's.
constexpr int CP_THREADS = 256;   // tiled combine, large plans (64 points per CTA)
constexpr int CP_THREADS_S = 128; // small plans (32 points per CTA): more CTAs per SM

template <int D, int P, int NTH>
__global__ void __launch_bounds__(NTH)
k_combine_points_tiled(const CompInfo* __restrict__ comps, int ncomp, const TabInfo* __restrict__ tabs,
                       int ntab, const double* __restrict__ knots, int mu, const double* __restrict__ coef,
                       const double* __restrict__ pts, int64_t npts, const int* __restrict__ perm,
                       double* __restrict__ out, int per_component, int npt, int* __restrict__ hist,
                       int* __restrict__ err, StatusFuse sf) {
    extern __shared__ double csm[];
    double* Bt = csm;                                   // [ntab][P][npt]
    double* V = Bt + (size_t)ntab * P * npt;            // [ncomp][npt]
    int* first = reinterpret_cast<int*>(V + (per_component ? 0 : (size_t)ncomp * npt));   // [ntab][npt]
    int* gidx = first + (size_t)ntab * npt;             // [npt] point index (cell order -> input order)
    const int tid = threadIdx.x;
    const int64_t p0 = (int64_t)blockIdx.x * npt;
    const int nloc = npts - p0 < npt ? (int)(npts - p0) : npt;
    for (int pt = tid; pt < nloc; pt += NTH) gidx[pt] = perm ? perm[p0 + pt] : (int)(p0 + pt);
    if (hist && blockIdx.x == 0)   // the sort is done: leave its cursors zero for the next call
        for (int i = tid; i < COMBINE_SORT_BINS; i += NTH) hist[i] = 0;
    __syncthreads();
    for (int it = tid; it < ntab * npt; it += NTH) {
        const int pt = it % npt, t = it / npt;
        if (pt >= nloc) continue;
        const TabInfo T = tabs[t];
        const double xi = pts[(int64_t)gidx[pt] * D + T.axis];
        if (!(xi >= 0.0 && xi <= 1.0)) atomicOr(err, ERRF_POINTS);   // evaluation points in [0,1]^d
        double bv[P];
        first[t * npt + pt] = axis_basis<P, false>(T, knots, mu, xi, bv, nullptr);
#pragma unroll
        for (int j = 0; j < P; ++j) Bt[(t * P + j) * npt + pt] = bv[j];
    }
    __syncthreads();
    for (int it = tid; it < ncomp * npt; it += NTH) {
        const int pt = it % npt, c = it / npt;
        if (pt >= nloc) continue;
        const CompInfo& C = comps[c];
        double Bv[D][P];
        int fs[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const int t = C.tab[k];
            fs[k] = first[t * npt + pt];
#pragma unroll
            for (int j = 0; j < P; ++j) Bv[k][j] = Bt[(t * P + j) * npt + pt];
        }
        double v, g[D];
        eval_component<D, P, false, true>(C, coef, fs, Bv, Bv, v, g);
        if (per_component) out[(int64_t)c * npts + gidx[pt]] = v;
        else V[c * npt + pt] = v;
    }
    if (per_component) return;
    __syncthreads();
    for (int pt = tid; pt < nloc; pt += NTH) {
        double acc = 0.0;
        for (int c = 0; c < ncomp; ++c) {
            const double cv = (double)comps[c].coef * V[c * npt + pt];
            acc = (c == 0) ? cv : __dadd_rn(acc, cv);
        }
        out[gidx[pt]] = acc;
    }
    if (sf.ticket) {   // the pass's status (k_status) by the CTA that finishes last
        __shared__ bool last;
        __threadfence();
        __syncthreads();
        if (tid == 0) last = atomicAdd(sf.ticket, 1u) == gridDim.x - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            int fail = 0;
            for (int c = tid; c < sf.ncomp; c += NTH) {
                const CgState s = sf.st[c];
                const double rel = sf.relres[c];
                sf.hst[c] = s;
                sf.hrel[c] = rel;
                fail |= cg_failed(s, rel);
            }
            fail = __syncthreads_or(fail);
            if (tid == 0) {
                const int e = *reinterpret_cast<volatile int*>(err);
                *sf.herr = e;
                *sf.hsticky |= (fail ? 1 : 0) | (e ? 2 : 0);
                *sf.ticket = 0u;
            }
            __threadfence_system();
        }
    }
}

// ---- cell sort of the points (locality of the coefficient windows) --------
// key = row-major cell index on a 2^bits-per-axis grid; a counting sort
// gives a permutation of the points in cell order.  The order inside a cell
// depends on atomic timing, but every point's value is computed by the same
// operations wherever it lands, so the output stays bitwise deterministic.
constexpr int SORT_BITS = COMBINE_SORT_BITS;   // 4096 cells
template <int D>
__device__ __forceinline__ int cell_key(const double* x) {
    constexpr int b = SORT_BITS / D, n = 1 << b;
    int key = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        int c = (int)(x[k] * (double)n);
        c = c < 0 ? 0 : (c > n - 1 ? n - 1 : c);
        key = key * n + c;
    }
    return key;
}

template <int D>
__global__ void k_cell_hist(const double* __restrict__ pts, int64_t npts, int* __restrict__ hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npts) atomicAdd(&hist[cell_key<D>(pts + i * D)], 1);
}

// exclusive scan of the 4096 bin counts, one CTA of 1024 threads
__global__ void __launch_bounds__(1024) k_cell_scan(int* __restrict__ hist) {
    __shared__ int ws[32];
    constexpr int PER = (1 << SORT_BITS) / 1024;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int v[PER], s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) { v[j] = hist[tid * PER + j]; s += v[j]; }
    int inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int w = ws[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        ws[lane] = w;
    }
    __syncthreads();
    int run = inc - s + (wid ? ws[wid - 1] : 0);
#pragma unroll
    for (int j = 0; j < PER; ++j) { hist[tid * PER + j] = run; run += v[j]; }
}

template <int D>
__global__ void k_cell_scatter(const double* __restrict__ pts, int64_t npts, int* __restrict__ cursor,
                               int* __restrict__ perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npts) perm[atomicAdd(&cursor[cell_key<D>(pts + i * D)], 1)] = (int)i;
}

template <int D, int P>
__global__ void __launch_bounds__(128)
k_combine_grid(const CompInfo* __restrict__ comps, int ncomp, const TabInfo* __restrict__ tabs,
               const double* __restrict__ knots, int mu, const double* __restrict__ coef,
               const double* __restrict__ pts, int64_t n0, int64_t n1, int64_t n2, int comp,
               double* __restrict__ vals, double* __restrict__ grads) {
    int64_t N = n0 * (D > 1 ? n1 : 1) * (D > 2 ? n2 : 1);
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    int64_t npd[3] = {n0, n1, n2}, off[3] = {0, n0, n0 + n1};
    double xi[D];
    int64_t rem = t;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) { xi[k] = pts[off[k] + rem % npd[k]]; rem /= npd[k]; }
    double acc, g[D];
    int lo = comp >= 0 ? comp : 0, hi = comp >= 0 ? comp + 1 : ncomp;
    if (grads) {
        combine_at<D, P, true>(comps, lo, hi, comp < 0, tabs, knots, mu, coef, xi, acc, g, nullptr, 0);
#pragma unroll
        for (int k = 0; k < D; ++k) grads[t * D + k] = g[k];
    } else {
        combine_at<D, P, false>(comps, lo, hi, comp < 0, tabs, knots, mu, coef, xi, acc, g, nullptr, 0);
    }
    vals[t] = acc;
}

// geometry map at one parametric point (geometry.py:87-132)
template <int D>
__device__ __forceinline__ double geo_point(const GeoInfo& G, const double* __restrict__ gknots,
                                            const double* __restrict__ hw, const double* xi,
                                            double* x, double (*Ji)[D]) {
    int first[D];
    double bv[D][GEO_PMAX + 1], bd[D][GEO_PMAX + 1];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double* kk = gknots + G.knot_off[k];
        int span = find_span(kk, G.nk[k], G.deg[k], xi[k], xi[k] == 1.0);
        double tab[2 * (GEO_PMAX + 1)];
        ders_basis_funs(span, xi[k], G.deg[k], 1, kk, tab);
        first[k] = span - G.deg[k];
        for (int j = 0; j <= G.deg[k]; ++j) { bv[k][j] = tab[j]; bd[k][j] = tab[G.deg[k] + 1 + j]; }
    }
    double hom[D + 1], dh[D][D + 1];
#pragma unroll
    for (int c = 0; c <= D; ++c) {
        hom[c] = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) dh[m][c] = 0.0;
    }
    int c0 = G.deg[0] + 1, c1 = D > 1 ? G.deg[D > 1 ? 1 : 0] + 1 : 1, c2 = D > 2 ? G.deg[D - 1] + 1 : 1;
    for (int i = 0; i < c0; ++i)
        for (int j = 0; j < c1; ++j)
            for (int l = 0; l < c2; ++l) {
                int idx[3] = {i, j, l};
                int64_t L = 0;
                double prod = 1.0, pm[D];
#pragma unroll
                for (int k = 0; k < D; ++k) L = L * G.n[k] + (first[k] + idx[k]);
#pragma unroll
                for (int k = 0; k < D; ++k) prod *= bv[k][idx[k]];
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    double t = 1.0;
#pragma unroll
                    for (int k = 0; k < D; ++k) t *= (k == m) ? bd[k][idx[k]] : bv[k][idx[k]];
                    pm[m] = t;
                }
#pragma unroll
                for (int c = 0; c <= D; ++c) {
                    double hv = hw[L * (D + 1) + c];
                    hom[c] += prod * hv;
#pragma unroll
                    for (int m = 0; m < D; ++m) dh[m][c] += pm[m] * hv;
                }
            }
    double J[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = hom[i] / hom[D];
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
        for (int i = 0; i < D; ++i) J[i][m] = (dh[m][i] - x[i] * dh[m][D]) / hom[D];
    double det;
    if constexpr (D == 1) {
        det = J[0][0];
        Ji[0][0] = 1.0 / det;
    } else if constexpr (D == 2) {
        det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        Ji[0][0] = J[1][1] / det; Ji[0][1] = -J[0][1] / det;
        Ji[1][0] = -J[1][0] / det; Ji[1][1] = J[0][0] / det;
    } else {
        double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        double c01 = J[1][0] * J[2][2] - J[1][2] * J[2][0];
        double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        det = J[0][0] * c00 - J[0][1] * c01 + J[0][2] * c02;
        Ji[0][0] = c00 / det;
        Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
        Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
        Ji[1][0] = -c01 / det;
        Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
        Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
        Ji[2][0] = c02 / det;
        Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
        Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    }
    return det;
}

constexpr int ERR_THREADS = 256;

template <int D, int P>
__global__ void __launch_bounds__(ERR_THREADS)
k_error_norms(const CompInfo* __restrict__ comps, int ncomp, const TabInfo* __restrict__ tabs,
              const double* __restrict__ knots, int mu, const double* __restrict__ coef,
              const GeoInfo* __restrict__ geo, const double* __restrict__ gknots,
              const double* __restrict__ hw, const double* __restrict__ pts,
              const double* __restrict__ wts, int64_t n0, int64_t n1, int64_t n2, int sol_id,
              double* __restrict__ partials, int* __restrict__ err, const int* __restrict__ tcomp,
              const double* __restrict__ tw, int nterm) {
    __shared__ double red[2][ERR_THREADS / 32];
    int64_t N = n0 * (D > 1 ? n1 : 1) * (D > 2 ? n2 : 1);
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double e2 = 0.0, h2 = 0.0;
    if (t < N) {
        int64_t npd[3] = {n0, n1, n2}, off[3] = {0, n0, n0 + n1};
        double xi[D], w = 1.0;
        int64_t rem = t, jj[D];
#pragma unroll
        for (int k = D - 1; k >= 0; --k) { jj[k] = rem % npd[k]; xi[k] = pts[off[k] + jj[k]]; rem /= npd[k]; }
#pragma unroll
        for (int k = 0; k < D; ++k) w = (k == 0) ? wts[off[0] + jj[0]] : w * wts[off[k] + jj[k]];
        double x[D], Ji[D][D];
        const GeoInfo G = *geo;
        double det = geo_point<D>(G, gknots, hw, xi, x, Ji);
        if (!(det > 0.0)) atomicOr(err, ERRF_GEOMETRY);
        double acc, g[D];
        if (tcomp) combine_terms<D, P, true>(comps, tcomp, tw, nterm, tabs, knots, mu, coef, xi, acc, g);
        else combine_at<D, P, true>(comps, 0, ncomp, true, tabs, knots, mu, coef, xi, acc, g, nullptr, 0);
        double ue = 0.0, ge[D];
#pragma unroll
        for (int i = 0; i < D; ++i) ge[i] = 0.0;
        if (sol_id >= 0) solution_value<D>(sol_id, x, ue, ge);   // < 0: norms of the combination itself
        double dv = acc - ue, dg2 = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {   // J^-T grad (analysis.py:235-237)
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s += Ji[k][i] * g[k];
            double e = s - ge[i];
            dg2 += e * e;
        }
        double wd = w * det;   // QuadGrid.weights = wgrid * det (assembly.py:178)
        e2 = wd * (dv * dv);
        h2 = wd * dg2;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
    }
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { red[0][wid] = e2; red[1][wid] = h2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < ERR_THREADS / 32; ++i) { a += red[0][i]; b += red[1][i]; }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

// ordered final sum of the block partials (one CTA)
__global__ void k_sum_partials(const double* __restrict__ partials, int64_t nblocks,
                               double* __restrict__ out) {
    __shared__ double red[2][32];
    double a = 0.0, b = 0.0;
    for (int64_t i = threadIdx.x; i < nblocks; i += blockDim.x) {
        a += partials[2 * i];
        b += partials[2 * i + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { red[0][wid] = a; red[1][wid] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { s0 += red[0][i]; s1 += red[1][i]; }
        out[0] = sqrt(s0);
        out[1] = sqrt(s1);
    }
}

// (d, p) dispatch: D in 1..3, P = p + 1 in 2..5
#define SGIGA_DISPATCH_DP(d, P, MACRO)                                   \
    switch ((d) * 10 + (P)) {                                            \
    case 12: MACRO(1, 2); break; case 13: MACRO(1, 3); break;            \
    case 14: MACRO(1, 4); break; case 15: MACRO(1, 5); break;            \
    case 22: MACRO(2, 2); break; case 23: MACRO(2, 3); break;            \
    case 24: MACRO(2, 4); break; case 25: MACRO(2, 5); break;            \
    case 32: MACRO(3, 2); break; case 33: MACRO(3, 3); break;            \
    case 34: MACRO(3, 4); break; case 35: MACRO(3, 5); break;            \
    default: return cudaErrorInvalidValue;                               \
    }

cudaError_t launch_combine_sort(Handle* h, const double* d_pts, int64_t npts, cudaStream_t s, bool* sorted) {
    *sorted = false;
    if (npts < 2048 || npts >= (int64_t)1 << 31 || h->opt.combine_nosort) return cudaSuccess;
    cudaError_t e;
    if ((size_t)npts > h->cperm_cap) {
        if (h->d_cperm) cudaFree(h->d_cperm);
        h->d_cperm = nullptr;
        h->cperm_cap = 0;
        if ((e = cudaMalloc(&h->d_cperm, sizeof(int) * npts)) != cudaSuccess) return e;
        h->cperm_cap = (size_t)npts;
    }
    // the histogram is zeroed on the sort's own stream by every sort: a pass
    // that never reached its combine (an error after the sort was enqueued,
    // the per-thread combine) must not leave stale cursors behind
    if ((e = cudaMemsetAsync(h->d_chist, 0, sizeof(int) * COMBINE_SORT_BINS, s)) != cudaSuccess) return e;
    const unsigned sb = (unsigned)((npts + 255) / 256);
    if (h->d == 1) k_cell_hist<1><<<sb, 256, 0, s>>>(d_pts, npts, h->d_chist);
    else if (h->d == 2) k_cell_hist<2><<<sb, 256, 0, s>>>(d_pts, npts, h->d_chist);
    else k_cell_hist<3><<<sb, 256, 0, s>>>(d_pts, npts, h->d_chist);
    k_cell_scan<<<1, 1024, 0, s>>>(h->d_chist);
    if (h->d == 1) k_cell_scatter<1><<<sb, 256, 0, s>>>(d_pts, npts, h->d_chist, h->d_cperm);
    else if (h->d == 2) k_cell_scatter<2><<<sb, 256, 0, s>>>(d_pts, npts, h->d_chist, h->d_cperm);
    else k_cell_scatter<3><<<sb, 256, 0, s>>>(d_pts, npts, h->d_chist, h->d_cperm);
    *sorted = true;
    return cudaGetLastError();
}

cudaError_t launch_combine_points(Handle* h, const double* d_pts, int64_t npts, double* d_out,
                                  int per_component, bool* status_fused) {
    if (status_fused) *status_fused = false;
    if (npts == 0) return cudaSuccess;
    StatusFuse sf{};
    if (status_fused && !per_component && h->d_ticket) {
        sf = StatusFuse{h->d_cg, h->d_relres, h->ncomp, h->dh_cg, h->dh_rel, h->dh_err, h->dh_sticky, h->d_ticket};
        *status_fused = true;
    }
    const int ntab = (int)h->tabs.size(), P = h->p + 1;
    // points per CTA: as many as fit ~100 KB of shared memory (2 CTAs/SM), <= 64
    auto smem_of = [&](int n) {
        return (size_t)n * (ntab * P * sizeof(double) + ntab * sizeof(int) +
                            (per_component ? 0 : (size_t)h->ncomp * sizeof(double)));
    };
    // small plans (<= 64 components, degree <= 3): 32 points / 128 threads per
    // CTA (more resident CTAs); larger: 64 points / 256 threads (measured)
    const bool small_cta = h->ncomp <= 64 && h->p <= 3;
    int npt = small_cta ? 32 : 64;
    // <= 40 KB per CTA: the (component, point) contractions are gather-latency
    // bound, so more resident CTAs (5 per SM) beat more points per CTA
    while (npt > 1 && smem_of(npt) > 40 * 1024) npt >>= 1;
    if (smem_of(npt) > 200 * 1024 || h->opt.combine_perthread) {   // huge plans: one thread per point
        unsigned blocks = (unsigned)((npts + 127) / 128);
#define LAUNCH_CP(DD, PP)                                                                     \
    k_combine_points<DD, PP><<<blocks, 128, 0, h->stream>>>(h->d_comps, h->ncomp, h->d_tabs,   \
                                                            h->d_knots, h->mu, h->d_coef,     \
                                                            d_pts, npts, d_out, per_component, h->d_err)
        SGIGA_DISPATCH_DP(h->d, h->p + 1, LAUNCH_CP)
#undef LAUNCH_CP
        h->launches[2]++;
        if (status_fused) *status_fused = false;
        return cudaGetLastError();
    }
    const size_t smem = smem_of(npt) + sizeof(int) * npt;
    const unsigned blocks = (unsigned)((npts + npt - 1) / npt);
    // cell sort (enough points per cell to matter, int32 indices): done here,
    // or already enqueued on the side stream by sgiga_run (h->cs_ready)
    const int* perm = nullptr;
    if (h->cs_ready) {
        perm = h->d_cperm;
        h->cs_ready = false;
        h->launches[2] += 3;
    } else {
        bool sorted = false;
        cudaError_t e = launch_combine_sort(h, d_pts, npts, h->stream, &sorted);
        if (e != cudaSuccess) return e;
        if (sorted) {
            perm = h->d_cperm;
            h->launches[2] += 3;
        }
    }
#define LAUNCH_CPT(DD, PP)                                                                          \
    {                                                                                               \
        if (small_cta) {                                                                            \
            cudaError_t e_ = cudaFuncSetAttribute(k_combine_points_tiled<DD, PP, CP_THREADS_S>,     \
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            if (e_ != cudaSuccess) return e_;                                                       \
            k_combine_points_tiled<DD, PP, CP_THREADS_S><<<blocks, CP_THREADS_S, smem, h->stream>>>( \
                h->d_comps, h->ncomp, h->d_tabs, ntab, h->d_knots, h->mu, h->d_coef, d_pts, npts, perm, \
                d_out, per_component, npt, perm ? h->d_chist : nullptr, h->d_err, sf);             \
        } else {                                                                                    \
            cudaError_t e_ = cudaFuncSetAttribute(k_combine_points_tiled<DD, PP, CP_THREADS>,       \
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            if (e_ != cudaSuccess) return e_;                                                       \
            k_combine_points_tiled<DD, PP, CP_THREADS><<<blocks, CP_THREADS, smem, h->stream>>>(   \
                h->d_comps, h->ncomp, h->d_tabs, ntab, h->d_knots, h->mu, h->d_coef, d_pts, npts, perm, \
                d_out, per_component, npt, perm ? h->d_chist : nullptr, h->d_err, sf);             \
        }                                                                                           \
    }
    SGIGA_DISPATCH_DP(h->d, h->p + 1, LAUNCH_CPT)
#undef LAUNCH_CPT
    h->launches[2]++;
    return cudaGetLastError();
}

cudaError_t launch_combine_grid(Handle* h, const double* d_pts, const int64_t* npd, int comp,
                                double* d_vals, double* d_grads) {
    int64_t N = 1;
    for (int k = 0; k < h->d; ++k) N *= npd[k];
    if (N == 0) return cudaSuccess;
    unsigned blocks = (unsigned)((N + 127) / 128);
    int64_t n1 = h->d > 1 ? npd[1] : 1, n2 = h->d > 2 ? npd[2] : 1;
#define LAUNCH_CG(DD, PP)                                                                      \
    k_combine_grid<DD, PP><<<blocks, 128, 0, h->stream>>>(h->d_comps, h->ncomp, h->d_tabs,      \
                                                          h->d_knots, h->mu, h->d_coef, d_pts,  \
                                                          npd[0], n1, n2, comp, d_vals, d_grads)
    SGIGA_DISPATCH_DP(h->d, h->p + 1, LAUNCH_CG)
#undef LAUNCH_CG
    h->launches[2]++;
    return cudaGetLastError();
}

cudaError_t launch_error_norms(Handle* h, const double* d_pts, const double* d_wts,
                               const int64_t* npd, int solution_id, double* d_partials,
                               int64_t* nblocks, const int* d_tcomp, const double* d_tw, int nterm) {
    int64_t N = 1;
    for (int k = 0; k < h->d; ++k) N *= npd[k];
    int64_t nb = (N + ERR_THREADS - 1) / ERR_THREADS;
    *nblocks = nb;
    int64_t n1 = h->d > 1 ? npd[1] : 1, n2 = h->d > 2 ? npd[2] : 1;
#define LAUNCH_EN(DD, PP)                                                                      \
    k_error_norms<DD, PP><<<(unsigned)nb, ERR_THREADS, 0, h->stream>>>(                        \
        h->d_comps, h->ncomp, h->d_tabs, h->d_knots, h->mu, h->d_coef, h->d_geo,               \
        h->d_geo_knots, h->d_geo_hw, d_pts, d_wts, npd[0], n1, n2, solution_id, d_partials,    \
        h->d_err, d_tcomp, d_tw, nterm)
    SGIGA_DISPATCH_DP(h->d, h->p + 1, LAUNCH_EN)
#undef LAUNCH_EN
    k_sum_partials<<<1, 1024, 0, h->stream>>>(d_partials, nb, d_partials + 2 * nb);
    h->launches[2] += 2;
    return cudaGetLastError();
}

}  // namespace sgiga

// ---- multi-GPU combine: plan-order sum of gathered per-component values ----
// out[pt] = sum_c coef_c * src[row_c][pt] with the single-GPU combine's
// exact operations and order (vals = c*v; vals += c*v, combination.py:
// 227-233): a plan split over ranks reproduces the one-GPU values bit for
// bit once every rank's per-component values are all-gathered.
namespace sgiga {
__global__ void k_plan_order_sum(int nterm, int64_t npts, const int* __restrict__ coef,
                                 const int64_t* __restrict__ row, const double* __restrict__ src,
                                 double* __restrict__ out) {
    const int64_t pt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pt >= npts) return;
    double acc = 0.0;
    for (int c = 0; c < nterm; ++c) {
        const double cv = (double)coef[c] * src[row[c] * npts + pt];
        acc = (c == 0) ? cv : __dadd_rn(acc, cv);
    }
    out[pt] = acc;
}
}  // namespace sgiga

extern "C" int sgiga_plan_order_sum(void* stream, int32_t nterm, int64_t npts, const int32_t* d_coef,
                                    const int64_t* d_row, const double* d_src, double* d_out) {
    using namespace sgiga;
    if (nterm < 1 || npts < 0 || !d_coef || !d_row || !d_src || !d_out) {
        set_error("sgiga_plan_order_sum: bad argument");
        return SGIGA_ERR_VALUE;
    }
    if (npts == 0) return SGIGA_OK;
    k_plan_order_sum<<<(unsigned)((npts + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nterm, npts, d_coef, d_row,
                                                                                         d_src, d_out);
    SG_CUDA(cudaGetLastError());
    return SGIGA_OK;
}
