// k_tables.cu -- kernel 1 (knots + Cox-de Boor basis tables at Gauss
// points, staged per (axis, level)) and the fused per-quadrature-point
// geometry / metric / load kernel.
//
// Reference: splines.make_open_knot_vector (splines.py:83-110),
// assembly._direction_tables (assembly.py:209-234), NurbsPatch.eval_grid
// (geometry.py:87-132), metric + load (assembly.py:286-294).
#include "forcing.cuh"
#include "handle.cuh"

namespace sgiga {

// ---- open knot vectors from breakpoints ---------------------------------
// ---- basis + geometry-basis tables at every (table, element, node) -------
__global__ void k_basis_tables(const TabInfo* __restrict__ tabs, int ntab,
                               const int64_t* __restrict__ tab_qp_cum, int p, int mu, int q,
                               const double* __restrict__ gauss, const double* __restrict__ bp,
                               const double* __restrict__ knots, const GeoInfo* __restrict__ geo,
                               const double* __restrict__ gknots, double* __restrict__ vals,
                               double* __restrict__ qx, double* __restrict__ qw,
                               double* __restrict__ geob, int* __restrict__ geofirst,
                               int* __restrict__ err) {
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= tab_qp_cum[ntab]) return;
    int lo = 0, hi = ntab;  // table of this thread
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (tab_qp_cum[mid] <= gid) lo = mid; else hi = mid;
    }
    const TabInfo T = tabs[lo];
    int local = (int)(gid - tab_qp_cum[lo]);
    int e = local / q, g = local % q;
    const double* b = bp + T.bp_off;
    double a0 = b[e], h = __dsub_rn(b[e + 1], a0);
    double xi = __dadd_rn(a0, __dmul_rn(h, gauss[g]));   // assembly.py:224
    double w = __dmul_rn(h, gauss[q + g]);                // assembly.py:233
    int P = p + 1;
    double tab[2 * (PMAX + 2)];
    ders_basis_funs(p + e * mu, xi, p, 1, knots + T.knot_off, tab);
    double* vv = vals + T.val_off;
    int64_t nq = (int64_t)T.nel * q;
    for (int j = 0; j < P; ++j) {
        vv[(int64_t)local * P + j] = tab[j];
        vv[nq * P + (int64_t)local * P + j] = tab[P + j];
    }
    qx[T.qp_off + local] = xi;
    qw[T.qp_off + local] = w;
    // geometry basis of this axis at xi (collocation_matrix, splines.py:262-274)
    const GeoInfo G = *geo;
    int ax = T.axis, pg = G.deg[ax];
    const double* gk = gknots + G.knot_off[ax];
    int span = find_span(gk, G.nk[ax], pg, xi, xi == 1.0);
    double gt[2 * (GEO_PMAX + 1)];
    ders_basis_funs(span, xi, pg, 1, gk, gt);
    double* gb = geob + (T.geo_off + local) * (2 * GEO_PMAX);
    for (int j = 0; j <= pg; ++j) {
        gb[j] = gt[j];
        gb[GEO_PMAX + j] = gt[pg + 1 + j];
    }
    geofirst[T.geo_off + local] = span - pg;
    if (!(xi > 0.0 && xi < 1.0)) atomicOr(err, ERRF_SPAN);
}

// ---- fused geometry -> metric + load --------------------------------------
// One thread per (component, quadrature point), storage order (s, a, b).
// GP > 0: every geometry axis has degree GP - 1 (compile-time contraction
// loops); the homogeneous control net is staged in shared memory when it
// fits (nsh > 0 doubles).  Same operations in the same order for every GP:
// the metric does not depend on the instantiation.
// resident CTAs per SM: as many as the registers allow without (or with a
// negligible) spill -- the kernel is latency-bound (global loads, divisions);
// cfg5 (D 3, degree-1 box, diagonal metric): 2 CTAs 1.74 ms, 3 1.32, 4 1.23
constexpr int metric_minb(int D, int GP, bool DG) {
    return D < 3 ? ((D == 2 && GP == 4 && !DG) ? 3 : 4) : (GP == 2 ? (DG ? 4 : 3) : 2);
}
template <int D, int GP, bool DG>
__global__ void __launch_bounds__(256, metric_minb(D, GP, DG))
k_metric(const CompInfo* __restrict__ comps, int ncomp,
                         const int64_t* __restrict__ qp_cum, const TabInfo* __restrict__ tabs,
                         const double* __restrict__ qx, const double* __restrict__ qw,
                         const double* __restrict__ geob, const int* __restrict__ geofirst,
                         const GeoInfo* __restrict__ geo, const double* __restrict__ hw_g,
                         int q, int forcing_id, const double* __restrict__ hostf,
                         double* __restrict__ xphys, double* __restrict__ Gout,
                         int* __restrict__ err, const int* __restrict__ cta_comp, int nsh) {
    extern __shared__ double s_hw[];
    const double* hw = hw_g;
    if (nsh > 0) {
        for (int i = threadIdx.x; i < nsh; i += blockDim.x) s_hw[i] = hw_g[i];
        __syncthreads();
        hw = s_hw;
    }
    // the component of the CTA's first point from the per-CTA table (no
    // search, no barrier); a thread past that component's end searches itself
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= qp_cum[ncomp]) return;
    int lo = cta_comp[blockIdx.x];
    int64_t base = qp_cum[lo];
    if (gid >= qp_cum[lo + 1]) {
        int l2 = lo, h2 = ncomp;
        while (h2 - l2 > 1) {
            int mid = (l2 + h2) >> 1;
            if (qp_cum[mid] <= gid) l2 = mid; else h2 = mid;
        }
        lo = l2;
        base = qp_cum[lo];
    }
    unsigned qsk[D], nqk[D];
    int64_t toff[D], goff[D];
    {
        const CompInfo& C1 = comps[lo];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            qsk[k] = (unsigned)C1.qs[k];
            nqk[k] = (unsigned)C1.nel[k] * (unsigned)q;
            const TabInfo& T = tabs[C1.tab[k]];
            toff[k] = T.qp_off;
            goff[k] = T.geo_off;
        }
    }
    const CompInfo& C = comps[lo];
    // per-component quadrature index < 2^31 (a component with more points
    // would need > 16 GB of metric): 32-bit index arithmetic
    const unsigned lin = (unsigned)(gid - base);
    double w = 1.0;
    const double* bv[D];
    int first[D];
    unsigned Qa[D];
#pragma unroll
    for (int k = 0; k < D; ++k) Qa[k] = (lin / qsk[k]) % nqk[k];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        first[k] = geofirst[goff[k] + Qa[k]];
        bv[k] = geob + (goff[k] + Qa[k]) * (2 * GEO_PMAX);
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double wk = qw[toff[k] + Qa[k]];
        w = (k == 0) ? wk : __dmul_rn(w, wk);   // _outer_product, assembly.py:186-190
    }
    // homogeneous contraction (geometry.py:114, 124) over active functions
    double hom[D + 1], dh[D][D + 1];
#pragma unroll
    for (int c = 0; c <= D; ++c) {
        hom[c] = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) dh[m][c] = 0.0;
    }
    int gn[D];
#pragma unroll
    for (int k = 0; k < D; ++k) gn[k] = geo->n[k];
    const int c0 = GP > 0 ? GP : geo->deg[0] + 1;
    const int c1 = D > 1 ? (GP > 0 ? GP : geo->deg[1] + 1) : 1;
    const int c2 = D > 2 ? (GP > 0 ? GP : geo->deg[2] + 1) : 1;
    // compile-time degree: the point's geometry basis values / derivatives
    // in registers, read as 16-byte pairs (same values, same operations)
    constexpr int GR = GP > 0 ? GP : 1;
    double gvb[D][GR], gdb[D][GR];
    if constexpr (GP > 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
#pragma unroll
            for (int i = 0; i + 1 < GP; i += 2) {
                const double2 v2 = __ldg(reinterpret_cast<const double2*>(bv[k] + i));
                const double2 d2 = __ldg(reinterpret_cast<const double2*>(bv[k] + GEO_PMAX + i));
                gvb[k][i] = v2.x; gvb[k][i + 1] = v2.y;
                gdb[k][i] = d2.x; gdb[k][i + 1] = d2.y;
            }
            if constexpr (GP & 1) {
                gvb[k][GP - 1] = __ldg(bv[k] + GP - 1);
                gdb[k][GP - 1] = __ldg(bv[k] + GEO_PMAX + GP - 1);
            }
        }
    }
    auto BV = [&](int k, int i) { if constexpr (GP > 0) return gvb[k][i]; else return bv[k][i]; };
    auto BD = [&](int k, int i) { if constexpr (GP > 0) return gdb[k][i]; else return bv[k][GEO_PMAX + i]; };
    if constexpr (D == 3) {
        // sum-factorised: contract axis 0 (values and derivatives), then axis
        // 1, then axis 2 -- 2(D+1)(c0 c1 c2 + 1.5 c1 c2 + 2 c2) FMAs instead of
        // a product per control point (rounding-level reordering of einsum)
        const int L0 = first[0] * gn[1], L1 = first[1];
#pragma unroll
        for (int l = 0; l < c2; ++l) {
            double Bvv[D + 1], Bdv[D + 1], Bvd[D + 1];
#pragma unroll
            for (int c = 0; c <= D; ++c) Bvv[c] = Bdv[c] = Bvd[c] = 0.0;
#pragma unroll
            for (int j = 0; j < c1; ++j) {
                double Av[D + 1], Ad[D + 1];
#pragma unroll
                for (int c = 0; c <= D; ++c) Av[c] = Ad[c] = 0.0;
#pragma unroll
                for (int i = 0; i < c0; ++i) {
                    const double b0 = BV(0, i), d0 = BD(0, i);
                    const double* h = hw + (int64_t)(((L0 + i * gn[1]) + (L1 + j)) * gn[2] + first[2] + l) * (D + 1);
#pragma unroll
                    for (int c = 0; c <= D; ++c) {
                        Av[c] = fma(b0, h[c], Av[c]);
                        Ad[c] = fma(d0, h[c], Ad[c]);
                    }
                }
                const double b1 = BV(1, j), d1 = BD(1, j);
#pragma unroll
                for (int c = 0; c <= D; ++c) {
                    Bvv[c] = fma(b1, Av[c], Bvv[c]);
                    Bdv[c] = fma(b1, Ad[c], Bdv[c]);
                    Bvd[c] = fma(d1, Av[c], Bvd[c]);
                }
            }
            const double b2 = BV(2, l), d2 = BD(2, l);
#pragma unroll
            for (int c = 0; c <= D; ++c) {
                hom[c] = fma(b2, Bvv[c], hom[c]);
                dh[0][c] = fma(b2, Bdv[c], dh[0][c]);
                dh[1][c] = fma(b2, Bvd[c], dh[1][c]);
                dh[2][c] = fma(d2, Bvv[c], dh[2][c]);
            }
        }
    } else
#pragma unroll
    for (int i = 0; i < c0; ++i)
#pragma unroll
        for (int j = 0; j < c1; ++j)
#pragma unroll
            for (int l = 0; l < c2; ++l) {
                int idx[3] = {i, j, l};
                int L = 0;
                double v[D], dv[D];
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    L = L * gn[k] + (first[k] + idx[k]);
                    v[k] = BV(k, idx[k]);
                    dv[k] = BD(k, idx[k]);
                }
                double prod = v[0];
#pragma unroll
                for (int k = 1; k < D; ++k) prod = __dmul_rn(prod, v[k]);
                double pm[D];
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    double t = (m == 0) ? dv[0] : v[0];
#pragma unroll
                    for (int k = 1; k < D; ++k) t = __dmul_rn(t, (k == m) ? dv[k] : v[k]);
                    pm[m] = t;
                }
#pragma unroll
                for (int c = 0; c <= D; ++c) {
                    double hv = hw[L * (D + 1) + c];
                    hom[c] = __dadd_rn(hom[c], __dmul_rn(prod, hv));
#pragma unroll
                    for (int m = 0; m < D; ++m) dh[m][c] = __dadd_rn(dh[m][c], __dmul_rn(pm[m], hv));
                }
            }
    // two divisions per point (1/W, 1/det), the rest multiplications by the
    // reciprocals: rounding-level differences from the reference's per-entry
    // divisions (A and b stay within the 1e-12 norm-wise contract)
    double x[D], J[D][D];
    const double invW = __ddiv_rn(1.0, hom[D]);
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = __dmul_rn(hom[i], invW);
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
        for (int i = 0; i < D; ++i)   // quotient rule, geometry.py:126
            // diagonal metric (axis-aligned box, DG): the off-diagonal terms are
            // exact zeros in the general evaluation too -- same diagonal bits
            J[i][m] = (DG && i != m) ? 0.0 : __dmul_rn(__dsub_rn(dh[m][i], __dmul_rn(x[i], dh[m][D])), invW);
    double det, Ji[D][D];
    if constexpr (D == 1) {
        det = J[0][0];
        Ji[0][0] = __ddiv_rn(1.0, J[0][0]);
    } else if constexpr (D == 2) {
        det = __dsub_rn(__dmul_rn(J[0][0], J[1][1]), __dmul_rn(J[0][1], J[1][0]));
        const double id = __ddiv_rn(1.0, det);
        Ji[0][0] = __dmul_rn(J[1][1], id);
        Ji[0][1] = __dmul_rn(-J[0][1], id);
        Ji[1][0] = __dmul_rn(-J[1][0], id);
        Ji[1][1] = __dmul_rn(J[0][0], id);
    } else {
        // cofactors in the oracle's order (oracle/sgiga_oracle.c det_small / inv_small)
        auto mm = [&](int i, int j) { return J[i][j]; };
        auto cof = [&](int a, int b, int c, int e) {
            return __dsub_rn(__dmul_rn(mm(a / 3, a % 3), mm(b / 3, b % 3)), __dmul_rn(mm(c / 3, c % 3), mm(e / 3, e % 3)));
        };
        double c00 = cof(4, 8, 5, 7), c01 = cof(3, 8, 5, 6), c02 = cof(3, 7, 4, 6);
        det = __dadd_rn(__dsub_rn(__dmul_rn(J[0][0], c00), __dmul_rn(J[0][1], c01)), __dmul_rn(J[0][2], c02));
        const double id = __ddiv_rn(1.0, det);
        Ji[0][0] = __dmul_rn(c00, id);
        Ji[0][1] = __dmul_rn(cof(2, 7, 1, 8), id);
        Ji[0][2] = __dmul_rn(cof(1, 5, 2, 4), id);
        Ji[1][0] = __dmul_rn(cof(5, 6, 3, 8), id);
        Ji[1][1] = __dmul_rn(cof(0, 8, 2, 6), id);
        Ji[1][2] = __dmul_rn(cof(2, 3, 0, 5), id);
        Ji[2][0] = __dmul_rn(cof(3, 7, 4, 6), id);
        Ji[2][1] = __dmul_rn(cof(1, 6, 0, 7), id);
        Ji[2][2] = __dmul_rn(cof(0, 4, 1, 3), id);
    }
    if (!(det > 0.0)) atomicOr(err, ERRF_GEOMETRY);   // geometry.py:128-131
    int64_t nqp = C.nqp;
    double* Gc = Gout + C.qp_off;
    double dw = __dmul_rn(det, w);
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
        for (int n = m; n < D; ++n) {    // (Jinv Jinv^T) * (det * w), assembly.py:288-289
            if (DG && n != m) continue;   // exact zeros, set once per layout
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) s = __dadd_rn(s, __dmul_rn(Ji[m][i], Ji[n][i]));
            Gc[(int64_t)sym_index(D, m, n) * nqp + lin] = __dmul_rn(s, dw);
        }
    double f;
    if (forcing_id == SGIGA_FORCING_HOST) {
        f = hostf ? hostf[gid] : 0.0;
        if (xphys)
#pragma unroll
            for (int i = 0; i < D; ++i) xphys[gid * D + i] = x[i];
    } else {
        f = forcing_value<D>(forcing_id, x);
    }
    // load = f * det * w (assembly.py:292)
    Gc[(int64_t)(D * (D + 1) / 2) * nqp + lin] = __dmul_rn(__dmul_rn(f, det), w);
}

// ---- metric + load of an axis-aligned box (metric_diagonal) ---------------
// The map is x_k = c0_k + L_k xi_k per axis, so J = diag(L), det = L0 L1 L2
// and G_kk = det / L_k^2 * w are closed forms (geometry.py:114-132 and
// assembly.py:286-294 evaluated symbolically for this patch class): per point
// only the weight product w = w0 w1 w2 (assembly.py:186-190, same order) and
// the forcing remain.  g[k] = det / L_k^2 and det are per-patch constants
// folded on the host; the off-diagonal entries are the exact zeros set once
// per layout.  Rounding-level differences from the general contraction
// (k_metric), which SGIGA_NO_BOX_METRIC keeps.  Write-bound: 4 doubles per
// quadrature point.
__global__ void __launch_bounds__(256) k_metric_box(
    const CompInfo* __restrict__ comps, int ncomp, const int64_t* __restrict__ qp_cum,
    const TabInfo* __restrict__ tabs, const double* __restrict__ qx, const double* __restrict__ qw,
    int q, int forcing_id, const double* __restrict__ hostf, double* __restrict__ xphys,
    double* __restrict__ Gout, int* __restrict__ err, const int* __restrict__ cta_comp, double3 c0,
    double3 L, double3 g, double det, int load_only) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid == 0 && !(det > 0.0)) atomicOr(err, ERRF_GEOMETRY);   // geometry.py:128-131
    if (gid >= qp_cum[ncomp]) return;
    int lo = cta_comp[blockIdx.x];
    if (gid >= qp_cum[lo + 1]) {
        int l2 = lo, h2 = ncomp;
        while (h2 - l2 > 1) {
            int mid = (l2 + h2) >> 1;
            if (qp_cum[mid] <= gid) l2 = mid; else h2 = mid;
        }
        lo = l2;
    }
    const CompInfo& C = comps[lo];
    const unsigned lin = (unsigned)(gid - qp_cum[lo]);
    double w = 1.0, x[3];
    const double c0k[3] = {c0.x, c0.y, c0.z}, Lk[3] = {L.x, L.y, L.z};
    // storage order (s, b, a), a = ax[1] innermost: two divisions per point
    const int ka = C.ax[1], kb = C.ax[0];
    const unsigned nqa = (unsigned)C.nel[ka] * (unsigned)q, nqb = (unsigned)C.nel[kb] * (unsigned)q;
    const unsigned t1 = lin / nqa, Qs = t1 / nqb;
    const unsigned Qa_ = lin - t1 * nqa, Qb_ = t1 - Qs * nqb;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const unsigned Qa = k == ka ? Qa_ : (k == kb ? Qb_ : Qs);
        const int64_t t = tabs[C.tab[k]].qp_off + Qa;
        const double wk = qw[t];
        w = (k == 0) ? wk : __dmul_rn(w, wk);
        x[k] = __fma_rn(Lk[k], qx[t], c0k[k]);
    }
    const int64_t nqp = C.nqp;
    double* Gc = Gout + C.qp_off;
    if (!load_only) {   // the Kronecker assembly (k_assembly_box.cu) reads the load only
        Gc[(int64_t)sym_index(3, 0, 0) * nqp + lin] = __dmul_rn(g.x, w);
        Gc[(int64_t)sym_index(3, 1, 1) * nqp + lin] = __dmul_rn(g.y, w);
        Gc[(int64_t)sym_index(3, 2, 2) * nqp + lin] = __dmul_rn(g.z, w);
    }
    double f;
    if (forcing_id == SGIGA_FORCING_HOST) {
        f = hostf ? hostf[gid] : 0.0;
        if (xphys)
#pragma unroll
            for (int i = 0; i < 3; ++i) xphys[gid * 3 + i] = x[i];
    } else {
        f = forcing_value<3>(forcing_id, x);
    }
    Gc[(int64_t)6 * nqp + lin] = __dmul_rn(__dmul_rn(f, det), w);
}

// NPT consecutive points (along the innermost quadrature axis) per thread:
// one index decomposition (two divisions) per NPT points, the rest by
// increment-with-carry; the load is stored as 16-byte vectors.  Requires every
// component's point count to be a multiple of NPT and the load rows 16-byte
// aligned (the launcher checks; true for every box plan with >= 2 elements
// per axis).  Per point the operations and their order are k_metric_box's.
template <int NPT>
__global__ void __launch_bounds__(256) k_metric_box_v(
    const CompInfo* __restrict__ comps, int ncomp, const int64_t* __restrict__ qp_cum,
    const TabInfo* __restrict__ tabs, const double* __restrict__ qx, const double* __restrict__ qw,
    int q, int forcing_id, const double* __restrict__ hostf, double* __restrict__ xphys,
    double* __restrict__ Gout, int* __restrict__ err, const int* __restrict__ cta_comp, double3 c0,
    double3 L, double3 g, double det, int load_only) {
    static_assert(NPT % 2 == 0, "vector stores");
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * NPT;
    if (gid == 0 && !(det > 0.0)) atomicOr(err, ERRF_GEOMETRY);   // geometry.py:128-131
    if (gid >= qp_cum[ncomp]) return;
    int lo = cta_comp[blockIdx.x * NPT];   // (table per 256 points)
    if (gid >= qp_cum[lo + 1]) {
        int l2 = lo, h2 = ncomp;
        while (h2 - l2 > 1) {
            int mid = (l2 + h2) >> 1;
            if (qp_cum[mid] <= gid) l2 = mid; else h2 = mid;
        }
        lo = l2;
    }
    const CompInfo& C = comps[lo];
    const unsigned lin = (unsigned)(gid - qp_cum[lo]);
    const double c0k[3] = {c0.x, c0.y, c0.z}, Lk[3] = {L.x, L.y, L.z};
    const int ka = C.ax[1], kb = C.ax[0];
    const unsigned nqa = (unsigned)C.nel[ka] * (unsigned)q, nqb = (unsigned)C.nel[kb] * (unsigned)q;
    const unsigned t1 = lin / nqa;
    unsigned Qs = t1 / nqb, Qa_ = lin - t1 * nqa, Qb_ = t1 - Qs * nqb;
    int64_t toff[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) toff[k] = tabs[C.tab[k]].qp_off;
    const int64_t nqp = C.nqp;
    double* Gc = Gout + C.qp_off;
    double fv[NPT];
#pragma unroll
    for (int j = 0; j < NPT; ++j) {
        double w = 1.0, x[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const unsigned Qa = k == ka ? Qa_ : (k == kb ? Qb_ : Qs);
            const int64_t t = toff[k] + Qa;
            const double wk = qw[t];
            w = (k == 0) ? wk : __dmul_rn(w, wk);
            x[k] = __fma_rn(Lk[k], qx[t], c0k[k]);
        }
        if (!load_only) {
            Gc[(int64_t)sym_index(3, 0, 0) * nqp + lin + j] = __dmul_rn(g.x, w);
            Gc[(int64_t)sym_index(3, 1, 1) * nqp + lin + j] = __dmul_rn(g.y, w);
            Gc[(int64_t)sym_index(3, 2, 2) * nqp + lin + j] = __dmul_rn(g.z, w);
        }
        double f;
        if (forcing_id == SGIGA_FORCING_HOST) {
            f = hostf ? hostf[gid + j] : 0.0;
            if (xphys)
#pragma unroll
                for (int i = 0; i < 3; ++i) xphys[(gid + j) * 3 + i] = x[i];
        } else {
            f = forcing_value<3>(forcing_id, x);
        }
        fv[j] = __dmul_rn(__dmul_rn(f, det), w);
        if (++Qa_ == nqa) {
            Qa_ = 0;
            if (++Qb_ == nqb) { Qb_ = 0; ++Qs; }
        }
    }
    double2* o = reinterpret_cast<double2*>(Gc + (int64_t)6 * nqp + lin);
#pragma unroll
    for (int j = 0; j < NPT; j += 2) o[j / 2] = make_double2(fv[j], fv[j + 1]);
}

void box_constants(const Handle* h, double* c0, double* L, double* g, double* det) {
    // control points: coordinate k of corner (a, b, c) depends on index k only
    auto hw = [&](int a, int b, int c, int comp) { return h->geo_hw[(size_t)((a * 2 + b) * 2 + c) * 4 + comp]; };
    c0[0] = hw(0, 0, 0, 0); c0[1] = hw(0, 0, 0, 1); c0[2] = hw(0, 0, 0, 2);
    L[0] = hw(1, 0, 0, 0) - c0[0]; L[1] = hw(0, 1, 0, 1) - c0[1]; L[2] = hw(0, 0, 1, 2) - c0[2];
    *det = L[0] * (L[1] * L[2]);
    for (int k = 0; k < 3; ++k) {
        const double il = 1.0 / L[k];
        g[k] = (il * il) * *det;
    }
}

// tab_qp_cum / qp_cum live right after d_gauss (see handle.cu)
extern int64_t* tab_qp_cum_ptr(Handle* h);
extern int64_t* comp_qp_cum_ptr(Handle* h);

cudaError_t launch_basis_tables(Handle* h) {
    int nt = (int)h->tabs.size();
    int64_t n = h->total_tabqp;
    int blocks = (int)((n + 127) / 128);
    k_basis_tables<<<blocks, 128, 0, h->stream>>>(
        h->d_tabs, nt, tab_qp_cum_ptr(h), h->p, h->mu, h->q, h->d_gauss, h->d_bp, h->d_knots,
        h->d_geo, h->d_geo_knots, h->d_tabvals, h->d_qx, h->d_qw, h->d_geob, h->d_geofirst,
        h->d_err);
    h->launches[0]++;
    return cudaGetLastError();
}

cudaError_t launch_metric(Handle* h) {
    int64_t n = h->total_qp;
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    const double* hostf = (h->forcing_id == SGIGA_FORCING_HOST) ? h->d_hostf : nullptr;
    // geometry degree of every axis (compile-time loops for degree 1..3) and
    // the control net in shared memory when it is at most 24 KB
    int gp = h->geo.deg[0] + 1;
    for (int k = 1; k < h->d; ++k)
        if (h->geo.deg[k] + 1 != gp) gp = 0;
    if (gp > (h->d == 3 ? 3 : 4)) gp = 0;   // (3-D, degree 3: register spills -- runtime loops)
    const int nsh = h->geo_hw.size() <= 3072 ? (int)h->geo_hw.size() : 0;
    const size_t shb = sizeof(double) * (size_t)nsh;
    // axis-aligned box geometry (3-D): the off-diagonal metric entries are
    // exact zeros -- written once per layout, the pass writes the diagonal
    const bool dg = h->d == 3 && metric_diagonal(h);
    if (dg && !h->metric_offdiag_zeroed) {
        cudaError_t e0 = cudaMemsetAsync(h->d_G, 0, sizeof(double) * (size_t)h->nG() * h->total_qp, h->stream);
        if (e0 != cudaSuccess) return e0;
        h->metric_offdiag_zeroed = true;
    }
    if (dg && !h->opt.no_box_metric) {
        double c0[3], L[3], g[3], det;
        box_constants(h, c0, L, g, &det);
        constexpr int NPT = 4;
        bool vec = true;   // NPT points per thread: no group straddles a component, 16-byte aligned load rows
        for (const CompInfo& C : h->comps)
            if (C.nqp % NPT != 0 || ((C.qp_off + 6 * C.nqp) & 1)) { vec = false; break; }
        if (vec)
            k_metric_box_v<NPT><<<(unsigned)((n + 256 * NPT - 1) / (256 * NPT)), 256, 0, h->stream>>>(
                h->d_comps, h->ncomp, comp_qp_cum_ptr(h), h->d_tabs, h->d_qx, h->d_qw, h->q, h->forcing_id,
                hostf, h->d_xphys, h->d_G, h->d_err, h->d_mcomp, make_double3(c0[0], c0[1], c0[2]),
                make_double3(L[0], L[1], L[2]), make_double3(g[0], g[1], g[2]), det, box_assembly_ready(h) ? 1 : 0);
        else
        k_metric_box<<<(unsigned)blocks, 256, 0, h->stream>>>(
            h->d_comps, h->ncomp, comp_qp_cum_ptr(h), h->d_tabs, h->d_qx, h->d_qw, h->q, h->forcing_id,
            hostf, h->d_xphys, h->d_G, h->d_err, h->d_mcomp, make_double3(c0[0], c0[1], c0[2]),
            make_double3(L[0], L[1], L[2]), make_double3(g[0], g[1], g[2]), det, box_assembly_ready(h) ? 1 : 0);
        h->launches[0]++;
        return cudaGetLastError();
    }
#define LAUNCH_METRIC(DD, GG)                                                                \
    if (dg && DD == 3) k_metric<DD, GG, true><<<(unsigned)blocks, 256, shb, h->stream>>>(     \
        h->d_comps, h->ncomp, comp_qp_cum_ptr(h), h->d_tabs, h->d_qx, h->d_qw, h->d_geob,    \
        h->d_geofirst, h->d_geo, h->d_geo_hw, h->q, h->forcing_id, hostf, h->d_xphys, h->d_G, \
        h->d_err, h->d_mcomp, nsh);                                                          \
    else k_metric<DD, GG, false><<<(unsigned)blocks, 256, shb, h->stream>>>(                   \
        h->d_comps, h->ncomp, comp_qp_cum_ptr(h), h->d_tabs, h->d_qx, h->d_qw, h->d_geob,    \
        h->d_geofirst, h->d_geo, h->d_geo_hw, h->q, h->forcing_id, hostf, h->d_xphys, h->d_G, \
        h->d_err, h->d_mcomp, nsh)
#define LAUNCH_METRIC_D(DD)                                                                   \
    switch (gp) {                                                                             \
        case 2: LAUNCH_METRIC(DD, 2); break;                                                  \
        case 3: LAUNCH_METRIC(DD, 3); break;                                                  \
        case 4: if (DD < 3) { LAUNCH_METRIC(DD, 4); break; } [[fallthrough]];                \
        default: LAUNCH_METRIC(DD, 0); break;                                                 \
    }
    if (h->d == 1) { LAUNCH_METRIC_D(1) }
    else if (h->d == 2) { LAUNCH_METRIC_D(2) }
    else { LAUNCH_METRIC_D(3) }
#undef LAUNCH_METRIC_D
#undef LAUNCH_METRIC
    h->launches[0]++;
    return cudaGetLastError();
}

}  // namespace sgiga
