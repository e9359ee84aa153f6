/*
 * sgiga_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's assemble -> solve -> combine
 * path (sparseiga v0.1.0, paths relative to pkg/src/sparseiga/).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the timed CPU
 * baseline -- never as part of the product path.
 *
 * Pinning: tests/test_oracle.py checks every function here against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py)
 * and against the reference's own known-answer tests.
 *
 * Third-party arithmetic the reference delegates:
 *   numpy leggauss      -> Gauss nodes are an INPUT (host numpy, bitwise).
 *   numpy linalg.det/inv-> closed-form 2x2/3x3 cofactors (rounding-level).
 *   scipy spsolve       -> SuperLU is replaced by a banded Cholesky on the
 *                          axis order that minimises the band (a direct
 *                          SPD solve, rounding-level equal), or, labelled,
 *                          by Jacobi-PCG (SPEC.md:231 allows either).
 * Compile with -ffp-contract=off so no FMA changes the reference's
 * rounding (the reference's Cython kernel is plain gcc -O2 on x86-64).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>
#include <time.h>

#include "../include/sgiga.h"

#define MAXD 3
#define MAXP 12

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------------
 * knot vectors: make_open_knot_vector (splines.py:83-110)
 * ---------------------------------------------------------------------- */
typedef struct {
    int p, nk, n, nel, mu;
    double* knots; /* owned */
    const double* bp;
} okv;

static void okv_build(okv* kv, int p, int r, const double* bp, int nbp) {
    int mu = p - r, nel = nbp - 1, i, j, pos = 0;
    kv->p = p;
    kv->mu = mu;
    kv->nel = nel;
    kv->bp = bp;
    kv->nk = 2 * (p + 1) + (nel - 1) * mu;
    kv->n = kv->nk - p - 1;
    kv->knots = (double*)malloc(sizeof(double) * kv->nk);
    for (i = 0; i <= p; ++i) kv->knots[pos++] = 0.0;
    for (i = 1; i < nel; ++i)
        for (j = 0; j < mu; ++j) kv->knots[pos++] = bp[i];
    for (i = 0; i <= p; ++i) kv->knots[pos++] = 1.0;
}

static void okv_free(okv* kv) { free(kv->knots); }

/* _find_span (splines.py:149-169) */
static int find_span(const double* k, int nk, int p, double xi, int left) {
    int n = nk - p - 1, lo = 0, hi = nk, i;
    /* searchsorted: first index with k[idx] > xi (right) / >= xi (left) */
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        int go_right = left ? (k[mid] < xi) : (k[mid] <= xi);
        if (go_right) lo = mid + 1; else hi = mid;
    }
    i = lo - 1;
    if (i < p) i = p;
    if (i > n - 1) i = n - 1;
    while (k[i] == k[i + 1]) i = left ? i - 1 : i + 1;
    return i;
}

/* _ders_basis_funs (splines.py:172-224): NURBS book A2.3; ders is
 * [(nders+1) x (p+1)] row-major. */
static void ders_basis_funs(int i, double xi, int p, int nders, const double* knots,
                            double* ders) {
    double ndu[MAXP + 1][MAXP + 1], left[MAXP + 1], right[MAXP + 1], a[2][MAXP + 1];
    int j, r, k;
    ndu[0][0] = 1.0;
    for (j = 1; j <= p; ++j) {
        double saved = 0.0;
        left[j] = xi - knots[i + 1 - j];
        right[j] = knots[i + j] - xi;
        for (r = 0; r < j; ++r) {
            double temp;
            ndu[j][r] = right[r + 1] + left[j - r];
            temp = ndu[r][j - 1] / ndu[j][r];
            ndu[r][j] = saved + right[r + 1] * temp;
            saved = left[j - r] * temp;
        }
        ndu[j][j] = saved;
    }
    for (k = 0; k <= nders; ++k)
        for (j = 0; j <= p; ++j) ders[k * (p + 1) + j] = 0.0;
    for (j = 0; j <= p; ++j) ders[j] = ndu[j][p];
    if (nders == 0) return;
    for (r = 0; r <= p; ++r) {
        int s1 = 0, s2 = 1, kmax = nders < p ? nders : p;
        a[0][0] = 1.0;
        for (k = 1; k <= kmax; ++k) {
            double d = 0.0;
            int rk = r - k, pk = p - k, j1, j2, jj, tmp;
            if (r >= k) {
                a[s2][0] = a[s1][0] / ndu[pk + 1][rk];
                d = a[s2][0] * ndu[rk][pk];
            }
            j1 = (rk >= -1) ? 1 : -rk;
            j2 = (r - 1 <= pk) ? k - 1 : p - r;
            for (jj = j1; jj <= j2; ++jj) {
                a[s2][jj] = (a[s1][jj] - a[s1][jj - 1]) / ndu[pk + 1][rk + jj];
                d += a[s2][jj] * ndu[rk + jj][pk];
            }
            if (r <= pk) {
                a[s2][k] = -a[s1][k - 1] / ndu[pk + 1][r];
                d += a[s2][k] * ndu[r][pk];
            }
            ders[k * (p + 1) + r] = d;
            tmp = s1; s1 = s2; s2 = tmp;
        }
    }
    {
        double fac = (double)p;
        int kmax = nders < p ? nders : p;
        for (k = 1; k <= kmax; ++k) {
            for (j = 0; j <= p; ++j) ders[k * (p + 1) + j] *= fac;
            fac *= (double)(p - k);
        }
    }
}

/* eval_basis (splines.py:227-259): returns the first active index. */
int orc_eval_basis(int p, int nk, const double* knots, double xi, int max_deriv,
                   int side, double* table) {
    int left = (side < 0) ? (xi == 1.0) : side; /* -1 = default rule */
    int i = find_span(knots, nk, p, xi, left);
    ders_basis_funs(i, xi, p, max_deriv, knots, table);
    return i - p;
}

/* _direction_tables (assembly.py:209-234) for one knot vector.  vals/ders
 * are [nel][q][p+1]; offsets [nel]; pts/wts [nel*q]. */
int orc_direction_tables(int p, int r, int nbp, const double* bp, int q,
                         const double* gn, const double* gw, double* vals,
                         double* ders, int32_t* offsets, double* pts, double* wts) {
    okv kv;
    double tab[2 * (MAXP + 1)];
    int e, g, a, bad = 0;
    okv_build(&kv, p, r, bp, nbp);
    for (e = 0; e < kv.nel; ++e) {
        double lo = bp[e], hi = bp[e + 1], h = hi - lo;
        offsets[e] = e * kv.mu;
        for (g = 0; g < q; ++g) {
            double xi = lo + h * gn[g];
            int first = orc_eval_basis(p, kv.nk, kv.knots, xi, 1, -1, tab);
            if (first != e * kv.mu) bad = 1;
            for (a = 0; a <= p; ++a) {
                vals[((size_t)e * q + g) * (p + 1) + a] = tab[a];
                ders[((size_t)e * q + g) * (p + 1) + a] = tab[p + 1 + a];
            }
            pts[e * q + g] = xi;
            wts[e * q + g] = h * gw[g];
        }
    }
    okv_free(&kv);
    return bad ? SGIGA_ERR_VALUE : SGIGA_OK;
}

/* ------------------------------------------------------------------------
 * closed forms (analysis.py:83-167 and SURVEY.md Appendix B)
 * ---------------------------------------------------------------------- */
static double forcing_eval(int id, int d, const double* x) {
    const double pi = 3.141592653589793;
    int k, m;
    switch (id) {
    case SGIGA_FORCING_ZERO: return 0.0;
    case SGIGA_FORCING_SIN_PRODUCT: {
        double u = 1.0;
        for (k = 0; k < d; ++k) u *= sin(pi * x[k]);
        return ((double)d * (pi * pi)) * u;
    }
    case SGIGA_FORCING_ANNULUS_POLAR: {
        double xx = x[0], yy = x[1], s = xx * xx + yy * yy;
        return 32.0 * xx * yy / (s * s) - 24.0 * xx * yy;
    }
    case SGIGA_FORCING_EXP_BUBBLE: {
        double b[MAXD], e = 0.0, tot = 0.0;
        for (k = 0; k < d; ++k) { b[k] = x[k] * (1.0 - x[k]); e += x[k]; }
        for (m = 0; m < d; ++m) {
            double t = x[m] * (x[m] + 3.0);
            for (k = 0; k < d; ++k) if (k != m) t *= b[k];
            tot += t;
        }
        return exp(e) * tot;
    }
    case SGIGA_FORCING_CUBE_POLY: {
        double b[MAXD], tot = 0.0;
        for (k = 0; k < d; ++k) b[k] = x[k] * (1.0 - x[k]);
        for (m = 0; m < d; ++m) {
            double t = 1.0;
            for (k = 0; k < d; ++k) if (k != m) t *= b[k];
            tot += 2.0 * t;
        }
        return tot;
    }
    case SGIGA_FORCING_ANNULUS_2D:
    case SGIGA_FORCING_ANNULUS_3D: {
        double xx = x[0], yy = x[1], x2 = xx * xx, y2 = yy * yy;
        double f2 = 2.0 * xx * (x2 * x2 + 22.0 * x2 * y2 - 5.0 * x2 + 21.0 * y2 * y2 - 45.0 * y2 + 4.0);
        if (id == SGIGA_FORCING_ANNULUS_2D) return f2;
        {
            double r2 = x2 + y2, u2 = -(r2 - 1.0) * (r2 - 4.0) * xx * y2;
            return (f2 + pi * pi * u2) * sin(pi * x[2]);
        }
    }
    case SGIGA_FORCING_CONSTANT_ONE: return 1.0;
    case SGIGA_FORCING_LSHAPE: return 0.0;
    default: return 0.0;
    }
}

/* value and physical gradient of the exact solution */
static void solution_eval(int id, int d, const double* x, double* u, double* g) {
    const double pi = 3.141592653589793;
    int k, m;
    for (k = 0; k < d; ++k) g[k] = 0.0;
    *u = 0.0;
    switch (id) {
    case SGIGA_FORCING_SIN_PRODUCT: {
        double s[MAXD], c[MAXD];
        for (k = 0; k < d; ++k) { s[k] = sin(pi * x[k]); c[k] = cos(pi * x[k]); }
        *u = 1.0;
        for (k = 0; k < d; ++k) *u *= s[k];
        for (m = 0; m < d; ++m) {
            double t = pi * c[m];
            for (k = 0; k < d; ++k) if (k != m) t *= s[k];
            g[m] = t;
        }
        return;
    }
    case SGIGA_FORCING_ANNULUS_POLAR: {
        double xx = x[0], yy = x[1], s = xx * xx + yy * yy;
        double h = s - 5.0 + 4.0 / s, hp = 1.0 - 4.0 / (s * s);
        *u = 2.0 * xx * yy * h;
        g[0] = 2.0 * yy * h + 4.0 * xx * xx * yy * hp;
        g[1] = 2.0 * xx * h + 4.0 * xx * yy * yy * hp;
        return;
    }
    case SGIGA_FORCING_EXP_BUBBLE: {
        double b[MAXD], e = 0.0;
        for (k = 0; k < d; ++k) { b[k] = x[k] * (1.0 - x[k]); e += x[k]; }
        e = exp(e);
        *u = e;
        for (k = 0; k < d; ++k) *u *= b[k];
        for (m = 0; m < d; ++m) {
            double t = e * (b[m] + 1.0 - 2.0 * x[m]);
            for (k = 0; k < d; ++k) if (k != m) t *= b[k];
            g[m] = t;
        }
        return;
    }
    case SGIGA_FORCING_CUBE_POLY: {
        double b[MAXD];
        for (k = 0; k < d; ++k) b[k] = x[k] * (1.0 - x[k]);
        *u = 1.0;
        for (k = 0; k < d; ++k) *u *= b[k];
        for (m = 0; m < d; ++m) {
            double t = 1.0 - 2.0 * x[m];
            for (k = 0; k < d; ++k) if (k != m) t *= b[k];
            g[m] = t;
        }
        return;
    }
    case SGIGA_FORCING_ANNULUS_2D:
    case SGIGA_FORCING_ANNULUS_3D: {
        double xx = x[0], yy = x[1], x2 = xx * xx, y2 = yy * yy, r2 = x2 + y2;
        double u2 = -(r2 - 1.0) * (r2 - 4.0) * xx * y2;
        double gx = -5.0 * x2 * x2 * y2 - 6.0 * x2 * y2 * y2 + 15.0 * x2 * y2 - y2 * y2 * y2 + 5.0 * y2 * y2 - 4.0 * y2;
        double gy = -2.0 * x2 * x2 * xx * yy - 8.0 * x2 * xx * y2 * yy + 10.0 * x2 * xx * yy
                    - 6.0 * xx * y2 * y2 * yy + 20.0 * xx * y2 * yy - 8.0 * xx * yy;
        if (id == SGIGA_FORCING_ANNULUS_2D) { *u = u2; g[0] = gx; g[1] = gy; return; }
        {
            double sz = sin(pi * x[2]), cz = cos(pi * x[2]);
            *u = u2 * sz; g[0] = gx * sz; g[1] = gy * sz; g[2] = u2 * pi * cz;
        }
        return;
    }
    case SGIGA_FORCING_LSHAPE: {
        double r = sqrt(x[0] * x[0] + x[1] * x[1]), th = atan2(x[1], x[0]);
        if (th < 0.0) th += 2.0 * pi;
        if (r == 0.0) return;
        {
            double rr = pow(r, 2.0 / 3.0), s = sin(2.0 * th / 3.0), c = cos(2.0 * th / 3.0);
            double dr = (2.0 / 3.0) * rr / r * s, dth = rr * (2.0 / 3.0) * c;
            *u = rr * s;
            g[0] = dr * cos(th) - dth * sin(th) / r;
            g[1] = dr * sin(th) + dth * cos(th) / r;
        }
        return;
    }
    default: return;
    }
}

int orc_forcing(int id, int d, int64_t npts, const double* x, double* f) {
    int64_t i;
    for (i = 0; i < npts; ++i) f[i] = forcing_eval(id, d, x + i * d);
    return SGIGA_OK;
}

int orc_solution(int id, int d, int64_t npts, const double* x, double* u, double* g) {
    int64_t i;
    for (i = 0; i < npts; ++i) solution_eval(id, d, x + i * d, u + i, g + i * d);
    return SGIGA_OK;
}

/* ------------------------------------------------------------------------
 * geometry: NurbsPatch.eval_grid (geometry.py:87-132)
 * ---------------------------------------------------------------------- */
typedef struct {
    int d, deg[MAXD], nk[MAXD], n[MAXD];
    const double* knots[MAXD];
    const double* hw;
} ogeo;

static void geo_from_desc(const sgiga_problem_desc* D, ogeo* g) {
    int k;
    size_t off = 0;
    g->d = D->d;
    for (k = 0; k < D->d; ++k) {
        g->deg[k] = D->geo_degree[k];
        g->nk[k] = D->geo_nknots[k];
        g->n[k] = g->nk[k] - g->deg[k] - 1;
        g->knots[k] = D->geo_knots + off;
        off += g->nk[k];
    }
    g->hw = D->geo_hw;
}

static double det_small(int d, const double* J) {
    if (d == 1) return J[0];
    if (d == 2) return J[0] * J[3] - J[1] * J[2];
    return J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
           J[2] * (J[3] * J[7] - J[4] * J[6]);
}

static void inv_small(int d, const double* J, double det, double* Ji) {
    if (d == 1) { Ji[0] = 1.0 / J[0]; return; }
    if (d == 2) {
        Ji[0] = J[3] / det; Ji[1] = -J[1] / det;
        Ji[2] = -J[2] / det; Ji[3] = J[0] / det;
        return;
    }
    Ji[0] = (J[4] * J[8] - J[5] * J[7]) / det;
    Ji[1] = (J[2] * J[7] - J[1] * J[8]) / det;
    Ji[2] = (J[1] * J[5] - J[2] * J[4]) / det;
    Ji[3] = (J[5] * J[6] - J[3] * J[8]) / det;
    Ji[4] = (J[0] * J[8] - J[2] * J[6]) / det;
    Ji[5] = (J[2] * J[3] - J[0] * J[5]) / det;
    Ji[6] = (J[3] * J[7] - J[4] * J[6]) / det;
    Ji[7] = (J[1] * J[6] - J[0] * J[7]) / det;
    Ji[8] = (J[0] * J[4] - J[1] * J[3]) / det;
}

/* Map one parametric point: x [d], J [d*d] with J[i*d+m] = dx_i/dxi_m,
 * det.  The homogeneous sums run over active functions in C order as the
 * reference's dense einsum does over nonzero entries. */
static void geo_map(const ogeo* G, const double* xi, double* x, double* J, double* det) {
    int d = G->d, k, i, j, l, w;
    int first[MAXD];
    double tab[MAXD][2 * (MAXP + 1)];
    double hom[MAXD + 1], dh[MAXD][MAXD + 1];
    int cnt[MAXD] = {1, 1, 1};
    for (k = 0; k < d; ++k) {
        first[k] = orc_eval_basis(G->deg[k], G->nk[k], G->knots[k], xi[k], 1, -1, tab[k]);
        cnt[k] = G->deg[k] + 1;
    }
    for (w = 0; w <= d; ++w) {
        hom[w] = 0.0;
        for (k = 0; k < d; ++k) dh[k][w] = 0.0;
    }
    for (i = 0; i < cnt[0]; ++i)
        for (j = 0; j < (d > 1 ? cnt[1] : 1); ++j)
            for (l = 0; l < (d > 2 ? cnt[2] : 1); ++l) {
                size_t lin;
                int m;
                double bv[MAXD], bd[MAXD];
                int idx[MAXD] = {i, j, l};
                lin = 0;
                for (k = 0; k < d; ++k) {
                    lin = lin * G->n[k] + (size_t)(first[k] + idx[k]);
                    bv[k] = tab[k][idx[k]];
                    bd[k] = tab[k][G->deg[k] + 1 + idx[k]];
                }
                for (w = 0; w <= d; ++w) {
                    double h = G->hw[lin * (d + 1) + w], prod = bv[0];
                    for (k = 1; k < d; ++k) prod = prod * bv[k];
                    hom[w] += prod * h;
                    for (m = 0; m < d; ++m) {
                        double pm = (m == 0) ? bd[0] : bv[0];
                        for (k = 1; k < d; ++k) pm = pm * ((k == m) ? bd[k] : bv[k]);
                        dh[m][w] += pm * h;
                    }
                }
            }
    for (i = 0; i < d; ++i) x[i] = hom[i] / hom[d];
    for (k = 0; k < d; ++k)
        for (i = 0; i < d; ++i) J[i * d + k] = (dh[k][i] - x[i] * dh[k][d]) / hom[d];
    *det = det_small(d, J);
}

/* eval_grid(jacobian=True) on a tensor grid: x [N*d], J [N*d*d], det [N] */
int orc_geometry_grid(const sgiga_problem_desc* D, const double* pts, const int64_t* npd,
                      double* x, double* J, double* det) {
    ogeo G;
    int d = D->d, k;
    int64_t N = 1, t, off[MAXD];
    geo_from_desc(D, &G);
    off[0] = 0;
    for (k = 0; k < d; ++k) { N *= npd[k]; if (k) off[k] = off[k - 1] + npd[k - 1]; }
    for (t = 0; t < N; ++t) {
        double xi[MAXD];
        int64_t rem = t;
        for (k = d - 1; k >= 0; --k) { xi[k] = pts[off[k] + rem % npd[k]]; rem /= npd[k]; }
        geo_map(&G, xi, x + t * d, J + t * d * d, det + t);
    }
    for (t = 0; t < N; ++t) if (!(det[t] > 0.0)) return SGIGA_ERR_GEOMETRY;
    return SGIGA_OK;
}

/* ------------------------------------------------------------------------
 * element kernel: _kernels/_compiled.pyx:17-90 (loop order preserved)
 * ---------------------------------------------------------------------- */
int orc_local_poisson_systems(int d, int max_nel, int n_q, int kmax, int64_t n_chunk,
                              int n_qp, int n_loc, const double* values,
                              const double* derivs, const int64_t* elem_index,
                              const int32_t* qp_index, const int32_t* fn_index,
                              const double* metric, const double* load, double* out_a,
                              double* out_b) {
    int64_t c;
    double *val, *grad, *half;
    if (d > 8) return SGIGA_ERR_VALUE;
    val = (double*)malloc(sizeof(double) * n_loc);
    grad = (double*)malloc(sizeof(double) * n_loc * d);
    half = (double*)malloc(sizeof(double) * n_loc * d);
#define TAB(T, l, e, q, f) T[(((size_t)(l) * max_nel + (e)) * n_q + (q)) * kmax + (f)]
    for (c = 0; c < n_chunk; ++c) {
        int q, a, b, l, m, n;
        for (q = 0; q < n_qp; ++q) {
            double w;
            for (a = 0; a < n_loc; ++a) {
                double va[8], da[8], v, g;
                for (l = 0; l < d; ++l) {
                    int64_t e_l = elem_index[c * d + l];
                    int q_l = qp_index[q * d + l];
                    va[l] = TAB(values, l, e_l, q_l, fn_index[a * d + l]);
                    da[l] = TAB(derivs, l, e_l, q_l, fn_index[a * d + l]);
                }
                v = 1.0;
                for (l = 0; l < d; ++l) v *= va[l];
                val[a] = v;
                for (m = 0; m < d; ++m) {
                    g = da[m];
                    for (l = 0; l < d; ++l) if (l != m) g *= va[l];
                    grad[a * d + m] = g;
                }
            }
            w = load[c * n_qp + q];
            for (a = 0; a < n_loc; ++a) out_b[c * n_loc + a] += val[a] * w;
            for (a = 0; a < n_loc; ++a)
                for (n = 0; n < d; ++n) {
                    double s = 0.0;
                    for (m = 0; m < d; ++m)
                        s += grad[a * d + m] * metric[((c * n_qp + q) * d + m) * d + n];
                    half[a * d + n] = s;
                }
            for (a = 0; a < n_loc; ++a)
                for (b = a; b < n_loc; ++b) {
                    double s = 0.0;
                    for (n = 0; n < d; ++n) s += half[a * d + n] * grad[b * d + n];
                    out_a[(c * n_loc + a) * n_loc + b] += s;
                }
        }
        for (a = 0; a < n_loc; ++a)
            for (b = a + 1; b < n_loc; ++b)
                out_a[(c * n_loc + b) * n_loc + a] = out_a[(c * n_loc + a) * n_loc + b];
    }
#undef TAB
    free(val); free(grad); free(half);
    return SGIGA_OK;
}

/* ------------------------------------------------------------------------
 * one component: DiscreteSpace.from_levels (assembly.py:64-70) +
 * _assemble_full (assembly.py:264-354) + interior extraction (389-390)
 * ---------------------------------------------------------------------- */
typedef struct {
    int d, p, q;
    okv kv[MAXD];
    int n[MAXD], m[MAXD], nel[MAXD];
    int64_t ndofs, nrows;
    /* interior CSR (rows in C order over interior multi-indices) */
    int64_t nnz;
    int64_t* indptr;
    int32_t* indices;
    double* data;
    double* rhs;
    /* per-axis interior column ranges, indexed by full row index */
    int* clo[MAXD];
    int* ccnt[MAXD];
} ocomp;

static const double* bp_table(const sgiga_problem_desc* D, int axis, int level, int* nbp) {
    int idx = axis * (D->max_level + 1) + level;
    *nbp = D->bp_count[idx];
    return D->breakpoints + D->bp_offset[idx];
}

static void comp_setup(const sgiga_problem_desc* D, int c, ocomp* C) {
    int k;
    memset(C, 0, sizeof(*C));
    C->d = D->d;
    C->p = D->degree;
    C->q = D->quad_points;
    C->ndofs = 1;
    C->nrows = 1;
    for (k = 0; k < D->d; ++k) {
        int nbp, i;
        const double* bp = bp_table(D, k, D->levels[c * D->d + k], &nbp);
        okv_build(&C->kv[k], D->degree, D->regularity, bp, nbp);
        C->n[k] = C->kv[k].n;
        C->m[k] = C->n[k] - 2 > 0 ? C->n[k] - 2 : 0;
        C->nel[k] = C->kv[k].nel;
        C->ndofs *= C->n[k];
        C->nrows *= C->m[k];
        C->clo[k] = (int*)malloc(sizeof(int) * C->n[k]);
        C->ccnt[k] = (int*)malloc(sizeof(int) * C->n[k]);
        for (i = 0; i < C->n[k]; ++i) {
            /* elements containing function i: e*mu <= i <= e*mu + p */
            int mu = C->kv[k].mu, p = C->p;
            int ef = (i - p) <= 0 ? 0 : (i - p + mu - 1) / mu;
            int el = i / mu;
            int lo, hi;
            if (el > C->nel[k] - 1) el = C->nel[k] - 1;
            lo = ef * mu;
            hi = el * mu + p;
            if (lo < 1) lo = 1;
            if (hi > C->n[k] - 2) hi = C->n[k] - 2;
            C->clo[k][i] = lo;
            C->ccnt[k][i] = hi >= lo ? hi - lo + 1 : 0;
        }
    }
}

static void comp_free(ocomp* C) {
    int k;
    for (k = 0; k < C->d; ++k) { okv_free(&C->kv[k]); free(C->clo[k]); free(C->ccnt[k]); }
    free(C->indptr); free(C->indices); free(C->data); free(C->rhs);
}

/* build the interior CSR pattern: Kronecker product of per-axis ranges */
static void comp_pattern(ocomp* C) {
    int d = C->d, k;
    int64_t row, pos = 0;
    C->indptr = (int64_t*)malloc(sizeof(int64_t) * (C->nrows + 1));
    C->indptr[0] = 0;
    for (row = 0; row < C->nrows; ++row) {
        int64_t rem = row, cnt = 1;
        for (k = d - 1; k >= 0; --k) { int i = 1 + (int)(rem % C->m[k]); rem /= C->m[k]; cnt *= C->ccnt[k][i]; }
        C->indptr[row + 1] = C->indptr[row] + cnt;
    }
    C->nnz = C->indptr[C->nrows];
    C->indices = (int32_t*)malloc(sizeof(int32_t) * (C->nnz ? C->nnz : 1));
    C->data = (double*)calloc(C->nnz ? C->nnz : 1, sizeof(double));
    C->rhs = (double*)calloc(C->nrows ? C->nrows : 1, sizeof(double));
    for (row = 0; row < C->nrows; ++row) {
        int r[MAXD], cur[MAXD];
        int64_t rem = row, t, cnt = C->indptr[row + 1] - C->indptr[row];
        for (k = d - 1; k >= 0; --k) { r[k] = 1 + (int)(rem % C->m[k]); rem /= C->m[k]; }
        for (k = 0; k < d; ++k) cur[k] = 0;
        for (t = 0; t < cnt; ++t) {
            int64_t col = 0;
            for (k = 0; k < d; ++k) col = col * C->m[k] + (C->clo[k][r[k]] + cur[k] - 1);
            C->indices[pos++] = (int32_t)col;
            for (k = d - 1; k >= 0; --k) {
                if (++cur[k] < C->ccnt[k][r[k]]) break;
                cur[k] = 0;
            }
        }
    }
}

/* position of interior (row multi-index ri, col multi-index ci) in CSR */
static int64_t comp_pos(const ocomp* C, const int* ri, const int* ci) {
    int k;
    int64_t row = 0, within = 0;
    for (k = 0; k < C->d; ++k) row = row * C->m[k] + (ri[k] - 1);
    for (k = 0; k < C->d; ++k) within = within * C->ccnt[k][ri[k]] + (ci[k] - C->clo[k][ri[k]]);
    return C->indptr[row] + within;
}

static int comp_assemble(const sgiga_problem_desc* D, int forcing_id, const double* host_f,
                         ocomp* C) {
    int d = C->d, p = C->p, q = C->q, P = p + 1, k, e, g, a;
    int n_qp = 1, n_loc = 1;
    double *vals[MAXD], *ders[MAXD], *pts[MAXD], *wts[MAXD];
    int32_t* offs[MAXD];
    int64_t Nq[MAXD], nel_tot = 1, el;
    double *values, *derivs, *metric, *load, *out_a, *out_b;
    int64_t *elem_index;
    int32_t *qp_index, *fn_index;
    int max_nel = 0, status = SGIGA_OK;
    ogeo G;
    geo_from_desc(D, &G);
    comp_pattern(C);
    for (k = 0; k < d; ++k) {
        int nel = C->nel[k];
        vals[k] = (double*)malloc(sizeof(double) * nel * q * P);
        ders[k] = (double*)malloc(sizeof(double) * nel * q * P);
        pts[k] = (double*)malloc(sizeof(double) * nel * q);
        wts[k] = (double*)malloc(sizeof(double) * nel * q);
        offs[k] = (int32_t*)malloc(sizeof(int32_t) * nel);
        if (orc_direction_tables(p, p - C->kv[k].mu, nel + 1, C->kv[k].bp, q, D->gauss_nodes,
                                 D->gauss_weights, vals[k], ders[k], offs[k], pts[k], wts[k]))
            status = SGIGA_ERR_VALUE;
        Nq[k] = (int64_t)nel * q;
        nel_tot *= nel;
        if (nel > max_nel) max_nel = nel;
        n_qp *= q;
        n_loc *= P;
    }
    /* padded tables [d, max_nel, q, kmax] (assembly.py:278-284) */
    values = (double*)calloc((size_t)d * max_nel * q * P, sizeof(double));
    derivs = (double*)calloc((size_t)d * max_nel * q * P, sizeof(double));
    for (k = 0; k < d; ++k)
        for (e = 0; e < C->nel[k]; ++e)
            for (g = 0; g < q; ++g)
                for (a = 0; a < P; ++a) {
                    size_t dst = (((size_t)k * max_nel + e) * q + g) * P + a;
                    values[dst] = vals[k][((size_t)e * q + g) * P + a];
                    derivs[dst] = ders[k][((size_t)e * q + g) * P + a];
                }
    qp_index = (int32_t*)malloc(sizeof(int32_t) * n_qp * d);
    fn_index = (int32_t*)malloc(sizeof(int32_t) * n_loc * d);
    for (g = 0; g < n_qp; ++g) { int rem = g; for (k = d - 1; k >= 0; --k) { qp_index[g * d + k] = rem % q; rem /= q; } }
    for (a = 0; a < n_loc; ++a) { int rem = a; for (k = d - 1; k >= 0; --k) { fn_index[a * d + k] = rem % P; rem /= P; } }
    elem_index = (int64_t*)malloc(sizeof(int64_t) * d);
    metric = (double*)malloc(sizeof(double) * n_qp * d * d);
    load = (double*)malloc(sizeof(double) * n_qp);
    out_a = (double*)malloc(sizeof(double) * n_loc * n_loc);
    out_b = (double*)malloc(sizeof(double) * n_loc);
    /* element loop in C order (elem_multi, assembly.py:309-311) */
    for (el = 0; el < nel_tot && status == SGIGA_OK; ++el) {
        int ei[MAXD];
        int64_t rem = el;
        for (k = d - 1; k >= 0; --k) { ei[k] = (int)(rem % C->nel[k]); rem /= C->nel[k]; elem_index[k] = ei[k]; }
        for (g = 0; g < n_qp; ++g) {
            double xi[MAXD], x[MAXD], J[MAXD * MAXD], Ji[MAXD * MAXD], det, w;
            int64_t gq[MAXD], flat = 0;
            int mm, nn, ii;
            for (k = 0; k < d; ++k) {
                gq[k] = (int64_t)ei[k] * q + qp_index[g * d + k];
                xi[k] = pts[k][gq[k]];
                flat = flat * Nq[k] + gq[k];
            }
            geo_map(&G, xi, x, J, &det);
            if (!(det > 0.0)) { status = SGIGA_ERR_GEOMETRY; break; }
            /* wgrid = outer product of per-axis weights (assembly.py:186-190, 287) */
            w = wts[0][gq[0]];
            for (k = 1; k < d; ++k) w = w * wts[k][gq[k]];
            inv_small(d, J, det, Ji);
            /* metric = (Jinv Jinv^T) * (det * w) (assembly.py:288-289) */
            for (mm = 0; mm < d; ++mm)
                for (nn = 0; nn < d; ++nn) {
                    double s = 0.0;
                    for (ii = 0; ii < d; ++ii) s += Ji[mm * d + ii] * Ji[nn * d + ii];
                    metric[(g * d + mm) * d + nn] = s * (det * w);
                }
            /* load = f(x) * det * w (assembly.py:290-292) */
            {
                double f = (forcing_id == SGIGA_FORCING_HOST) ? host_f[flat] : forcing_eval(forcing_id, d, x);
                load[g] = f * det * w;
            }
        }
        if (status != SGIGA_OK) break;
        memset(out_a, 0, sizeof(double) * n_loc * n_loc);
        memset(out_b, 0, sizeof(double) * n_loc);
        orc_local_poisson_systems(d, max_nel, q, P, 1, n_qp, n_loc, values, derivs, elem_index,
                                  qp_index, fn_index, metric, load, out_a, out_b);
        /* scatter (assembly.py:341-352), keeping interior x interior only */
        for (a = 0; a < n_loc; ++a) {
            int ri[MAXD], inter = 1, b;
            for (k = 0; k < d; ++k) {
                ri[k] = offs[k][ei[k]] + fn_index[a * d + k];
                if (ri[k] < 1 || ri[k] > C->n[k] - 2) inter = 0;
            }
            if (!inter) continue;
            {
                int64_t row = 0;
                for (k = 0; k < d; ++k) row = row * C->m[k] + (ri[k] - 1);
                C->rhs[row] += out_b[a];
            }
            for (b = 0; b < n_loc; ++b) {
                int ci[MAXD], cin = 1;
                for (k = 0; k < d; ++k) {
                    ci[k] = offs[k][ei[k]] + fn_index[b * d + k];
                    if (ci[k] < 1 || ci[k] > C->n[k] - 2) cin = 0;
                }
                if (!cin) continue;
                C->data[comp_pos(C, ri, ci)] += out_a[a * n_loc + b];
            }
        }
    }
    for (k = 0; k < d; ++k) { free(vals[k]); free(ders[k]); free(pts[k]); free(wts[k]); free(offs[k]); }
    free(values); free(derivs); free(qp_index); free(fn_index); free(elem_index);
    free(metric); free(load); free(out_a); free(out_b);
    return status;
}

/* ------------------------------------------------------------------------
 * solves
 * ---------------------------------------------------------------------- */
static double spmv_resid(const ocomp* C, const double* x, double* tmp) {
    int64_t i, j;
    double s2 = 0.0;
    for (i = 0; i < C->nrows; ++i) {
        double s = 0.0;
        for (j = C->indptr[i]; j < C->indptr[i + 1]; ++j) s += C->data[j] * x[C->indices[j]];
        if (tmp) tmp[i] = s;
        s -= C->rhs[i];
        s2 += s * s;
    }
    return sqrt(s2);
}

/* Direct SPD solve: band Cholesky on the axis order with the largest
 * interior extent outermost (the band that C order would give is
 * p * prod(other extents)). */
static int solve_direct(const ocomp* C, double* x) {
    int d = C->d, k, perm[MAXD], i2;
    int64_t N = C->nrows, bw = 0, i, j, t, pstr[MAXD];
    int64_t *old2new;
    double *L, *y;
    for (k = 0; k < d; ++k) perm[k] = k;
    for (k = 0; k < d; ++k)
        for (i2 = k + 1; i2 < d; ++i2)
            if (C->m[perm[i2]] > C->m[perm[k]]) { int tmp = perm[k]; perm[k] = perm[i2]; perm[i2] = tmp; }
    /* stride of original axis a in the permuted order */
    {
        int64_t s = 1;
        for (k = d - 1; k >= 0; --k) { pstr[perm[k]] = s; s *= C->m[perm[k]]; }
    }
    old2new = (int64_t*)malloc(sizeof(int64_t) * N);
    for (i = 0; i < N; ++i) {
        int64_t rem = i, nw = 0;
        for (k = d - 1; k >= 0; --k) { nw += (rem % C->m[k]) * pstr[k]; rem /= C->m[k]; }
        old2new[i] = nw;
    }
    for (i = 0; i < N; ++i)
        for (j = C->indptr[i]; j < C->indptr[i + 1]; ++j) {
            int64_t dd = old2new[i] - old2new[C->indices[j]];
            if (dd > bw) bw = dd;
        }
    L = (double*)calloc((size_t)N * (bw + 1), sizeof(double)); /* L[i][i-j] */
    for (i = 0; i < N; ++i)
        for (j = C->indptr[i]; j < C->indptr[i + 1]; ++j) {
            int64_t ni = old2new[i], nj = old2new[C->indices[j]];
            if (nj <= ni) L[ni * (bw + 1) + (ni - nj)] = C->data[j];
        }
    for (i = 0; i < N; ++i) {
        int64_t j0 = i - bw < 0 ? 0 : i - bw;
        for (j = j0; j <= i; ++j) {
            int64_t k0 = (i - bw > j - bw ? i - bw : j - bw);
            double s = L[i * (bw + 1) + (i - j)];
            if (k0 < 0) k0 = 0;
            for (t = k0; t < j; ++t) s -= L[i * (bw + 1) + (i - t)] * L[j * (bw + 1) + (j - t)];
            if (j == i) {
                if (!(s > 0.0)) { free(L); free(old2new); return SGIGA_ERR_SOLVE; }
                L[i * (bw + 1)] = sqrt(s);
            } else {
                L[i * (bw + 1) + (i - j)] = s / L[j * (bw + 1)];
            }
        }
    }
    y = (double*)malloc(sizeof(double) * N);
    for (i = 0; i < N; ++i) y[old2new[i]] = C->rhs[i];
    for (i = 0; i < N; ++i) {
        int64_t j0 = i - bw < 0 ? 0 : i - bw;
        double s = y[i];
        for (j = j0; j < i; ++j) s -= L[i * (bw + 1) + (i - j)] * y[j];
        y[i] = s / L[i * (bw + 1)];
    }
    for (i = N - 1; i >= 0; --i) {
        int64_t j1 = i + bw > N - 1 ? N - 1 : i + bw;
        double s = y[i];
        for (j = i + 1; j <= j1; ++j) s -= L[j * (bw + 1) + (j - i)] * y[j];
        y[i] = s / L[i * (bw + 1)];
    }
    for (i = 0; i < N; ++i) x[i] = y[old2new[i]];
    free(L); free(y); free(old2new);
    return SGIGA_OK;
}

/* Jacobi-preconditioned CG, labelled alternative. */
static int solve_pcg(const ocomp* C, double rtol, int maxit, double* x, int* iters) {
    int64_t N = C->nrows, i, j;
    double *r = malloc(sizeof(double) * N), *z = malloc(sizeof(double) * N);
    double *pv = malloc(sizeof(double) * N), *qv = malloc(sizeof(double) * N);
    double *dinv = malloc(sizeof(double) * N);
    double bn = 0.0, rho = 0.0;
    int it = 0, ok = 0;
    for (i = 0; i < N; ++i) {
        for (j = C->indptr[i]; j < C->indptr[i + 1]; ++j)
            if (C->indices[j] == i) dinv[i] = 1.0 / C->data[j];
        x[i] = 0.0;
        r[i] = C->rhs[i];
        z[i] = dinv[i] * r[i];
        pv[i] = z[i];
        bn += r[i] * r[i];
        rho += r[i] * z[i];
    }
    bn = sqrt(bn);
    if (bn == 0.0) ok = 1;
    while (!ok && it < maxit) {
        double pq = 0.0, alpha, rr = 0.0, rn = 0.0, beta;
        for (i = 0; i < N; ++i) {
            double s = 0.0;
            for (j = C->indptr[i]; j < C->indptr[i + 1]; ++j) s += C->data[j] * pv[C->indices[j]];
            qv[i] = s;
            pq += pv[i] * s;
        }
        alpha = rho / pq;
        for (i = 0; i < N; ++i) {
            x[i] += alpha * pv[i];
            r[i] -= alpha * qv[i];
            rn += r[i] * r[i];
        }
        ++it;
        if (sqrt(rn) <= rtol * bn) { ok = 1; break; }
        for (i = 0; i < N; ++i) { z[i] = dinv[i] * r[i]; rr += r[i] * z[i]; }
        beta = rr / rho;
        rho = rr;
        for (i = 0; i < N; ++i) pv[i] = z[i] + beta * pv[i];
    }
    *iters = it;
    free(r); free(z); free(pv); free(qv); free(dinv);
    return ok ? SGIGA_OK : SGIGA_ERR_SOLVE;
}

/* ------------------------------------------------------------------------
 * public entry points
 * ---------------------------------------------------------------------- */
int orc_component_dims(const sgiga_problem_desc* D, int c, int32_t* n) {
    int k;
    for (k = 0; k < D->d; ++k) {
        int nbp;
        bp_table(D, k, D->levels[c * D->d + k], &nbp);
        n[k] = D->degree + 1 + (nbp - 2) * (D->degree - D->regularity);
    }
    return SGIGA_OK;
}

/* Assemble one component and return its interior CSR + rhs (two-call
 * protocol: indptr/indices/data NULL -> only nnz and nrows). */
int orc_assemble_csr(const sgiga_problem_desc* D, int c, const double* host_f,
                     int64_t* nrows, int64_t* nnz, int64_t* indptr, int32_t* indices,
                     double* data, double* rhs) {
    ocomp C;
    int st;
    int64_t i, j, out = 0;
    comp_setup(D, c, &C);
    if (C.nrows == 0) { comp_free(&C); *nrows = 0; *nnz = 0; return SGIGA_ERR_EMPTY; }
    st = comp_assemble(D, D->forcing_id, host_f, &C);
    if (st) { comp_free(&C); return st; }
    *nrows = C.nrows;
    /* drop exact zeros (scipy csr + csr, assembly.py:349-351) */
    for (i = 0; i < C.nnz; ++i) out += (C.data[i] != 0.0);
    *nnz = out;
    if (indptr && indices && data) {
        int64_t pos = 0;
        indptr[0] = 0;
        for (i = 0; i < C.nrows; ++i) {
            for (j = C.indptr[i]; j < C.indptr[i + 1]; ++j)
                if (C.data[j] != 0.0) { indices[pos] = C.indices[j]; data[pos] = C.data[j]; ++pos; }
            indptr[i + 1] = pos;
        }
    }
    if (rhs) memcpy(rhs, C.rhs, sizeof(double) * C.nrows);
    comp_free(&C);
    return SGIGA_OK;
}

/* solve_component (combination.py:183-200): full C-order coefficients.
 * solver 0 = direct, 1 = Jacobi-PCG(rtol). */
static int run_component(const sgiga_problem_desc* D, int c, int solver, double rtol,
                         double* coefs, double* relres, int* iters) {
    ocomp C;
    int st = SGIGA_OK, k;
    int64_t i;
    double *x;
    comp_setup(D, c, &C);
    memset(coefs, 0, sizeof(double) * C.ndofs);
    *iters = 0;
    *relres = 0.0;
    if (C.nrows == 0) { comp_free(&C); return SGIGA_OK; } /* combination.py:194-195 */
    st = comp_assemble(D, D->forcing_id, NULL, &C);
    if (st) { comp_free(&C); return st; }
    x = (double*)calloc(C.nrows, sizeof(double));
    {
        double bn = 0.0;
        for (i = 0; i < C.nrows; ++i) bn += C.rhs[i] * C.rhs[i];
        bn = sqrt(bn);
        if (bn > 0.0) {
            st = solver == 0 ? solve_direct(&C, x) : solve_pcg(&C, rtol, 1000000, x, iters);
            if (!st) {
                double res = spmv_resid(&C, x, NULL);
                *relres = res / bn;
                for (i = 0; i < C.nrows; ++i) if (!isfinite(x[i])) st = SGIGA_ERR_SOLVE;
                if (res > 1e-10 * bn) st = SGIGA_ERR_SOLVE; /* linsolve.py:49-53 */
            }
        }
    }
    /* expand (assembly.py:202-206) */
    for (i = 0; i < C.nrows; ++i) {
        int64_t rem = i, full = 0, mul = 1;
        int ri[MAXD];
        for (k = C.d - 1; k >= 0; --k) { ri[k] = 1 + (int)(rem % C.m[k]); rem /= C.m[k]; }
        for (k = C.d - 1; k >= 0; --k) { full += ri[k] * mul; mul *= C.n[k]; }
        coefs[full] = x[i];
    }
    free(x);
    comp_free(&C);
    return st;
}

int64_t orc_total_dofs(const sgiga_problem_desc* D, int64_t* offsets) {
    int c, k;
    int64_t tot = 0;
    for (c = 0; c < D->n_comp; ++c) {
        int32_t n[MAXD];
        int64_t nd = 1;
        orc_component_dims(D, c, n);
        for (k = 0; k < D->d; ++k) nd *= n[k];
        if (offsets) offsets[c] = tot;
        tot += nd;
    }
    if (offsets) offsets[D->n_comp] = tot;
    return tot;
}

/* run_plan (scheduler.py:74-96): all components, OpenMP over components
 * (the reference uses one process per component), longest-first. */
int orc_run_plan(const sgiga_problem_desc* D, int nthreads, int solver, double rtol,
                 double* coefs, double* times, double* relres, int32_t* iters) {
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (D->n_comp + 1));
    int* order = (int*)malloc(sizeof(int) * D->n_comp);
    int64_t* cost = (int64_t*)malloc(sizeof(int64_t) * D->n_comp);
    int c, status = SGIGA_OK, i, j;
    orc_total_dofs(D, off);
    for (c = 0; c < D->n_comp; ++c) { order[c] = c; cost[c] = off[c + 1] - off[c]; }
    for (i = 0; i < D->n_comp; ++i)
        for (j = i + 1; j < D->n_comp; ++j)
            if (cost[order[j]] > cost[order[i]]) { int t = order[i]; order[i] = order[j]; order[j] = t; }
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (i = 0; i < D->n_comp; ++i) {
        int cc = order[i], it = 0, st;
        double rr = 0.0, t0 = now_s();
        st = run_component(D, cc, solver, rtol, coefs + off[cc], &rr, &it);
        if (times) times[cc] = now_s() - t0;
        if (relres) relres[cc] = rr;
        if (iters) iters[cc] = it;
        if (st) {
#pragma omp critical
            { if (status == SGIGA_OK) status = st; }
        }
    }
    free(off); free(order); free(cost);
    return status;
}

/* value (and parametric gradient) of one component at one point */
static void comp_point(const sgiga_problem_desc* D, const okv* kv, const int* n,
                       const double* coef, const double* xi, int grad, double* v, double* g) {
    int d = D->d, p = D->degree, P = p + 1, k, a0, a1, a2, first[MAXD];
    double tab[MAXD][2 * (MAXP + 1)];
    for (k = 0; k < d; ++k)
        first[k] = orc_eval_basis(p, kv[k].nk, kv[k].knots, xi[k], grad ? 1 : 0, -1, tab[k]);
    *v = 0.0;
    if (grad) for (k = 0; k < d; ++k) g[k] = 0.0;
    for (a0 = 0; a0 < P; ++a0)
        for (a1 = 0; a1 < (d > 1 ? P : 1); ++a1)
            for (a2 = 0; a2 < (d > 2 ? P : 1); ++a2) {
                int idx[MAXD] = {a0, a1, a2}, m;
                int64_t lin = 0;
                double c, b = 1.0;
                for (k = 0; k < d; ++k) lin = lin * n[k] + (first[k] + idx[k]);
                c = coef[lin];
                for (k = 0; k < d; ++k) b = b * tab[k][idx[k]];
                *v += b * c;
                if (grad)
                    for (m = 0; m < d; ++m) {
                        double bm = 1.0;
                        for (k = 0; k < d; ++k) bm = bm * (k == m ? tab[k][P + idx[k]] : tab[k][idx[k]]);
                        g[m] += bm * c;
                    }
            }
}

typedef struct { okv kv[MAXD]; int n[MAXD]; } ospace;

static ospace* spaces_build(const sgiga_problem_desc* D) {
    ospace* S = (ospace*)malloc(sizeof(ospace) * D->n_comp);
    int c, k;
    for (c = 0; c < D->n_comp; ++c)
        for (k = 0; k < D->d; ++k) {
            int nbp;
            const double* bp = bp_table(D, k, D->levels[c * D->d + k], &nbp);
            okv_build(&S[c].kv[k], D->degree, D->regularity, bp, nbp);
            S[c].n[k] = S[c].kv[k].n;
        }
    return S;
}

static void spaces_free(const sgiga_problem_desc* D, ospace* S) {
    int c, k;
    for (c = 0; c < D->n_comp; ++c) for (k = 0; k < D->d; ++k) okv_free(&S[c].kv[k]);
    free(S);
}

/* evaluate_combined at scattered points via the per-point idiom
 * (test_acceptance.py:224-230), accumulation in plan order
 * (combination.py:219-233). comp >= 0 evaluates that component only. */
int orc_combine_points(const sgiga_problem_desc* D, const double* coefs, int comp,
                       const double* pts, int64_t npts, int nthreads, double* out) {
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (D->n_comp + 1));
    ospace* S = spaces_build(D);
    int64_t t;
    orc_total_dofs(D, off);
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (t = 0; t < npts; ++t) {
        int c;
        double acc = 0.0, v, g[MAXD];
        int started = 0;
        for (c = 0; c < D->n_comp; ++c) {
            if (comp >= 0 && c != comp) continue;
            comp_point(D, S[c].kv, S[c].n, coefs + off[c], pts + t * D->d, 0, &v, g);
            if (comp >= 0) { acc = v; break; }
            v = (double)D->coefs[c] * v;
            acc = started ? acc + v : v;
            started = 1;
        }
        out[t] = acc;
    }
    spaces_free(D, S);
    free(off);
    return SGIGA_OK;
}

/* tensor-grid evaluation with optional parametric gradients */
int orc_combine_grid(const sgiga_problem_desc* D, const double* coefs, int comp,
                     const double* pts, const int64_t* npd, int nthreads, double* vals,
                     double* grads) {
    int d = D->d, k;
    int64_t N = 1, t, poff[MAXD];
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (D->n_comp + 1));
    ospace* S = spaces_build(D);
    orc_total_dofs(D, off);
    poff[0] = 0;
    for (k = 0; k < d; ++k) { N *= npd[k]; if (k) poff[k] = poff[k - 1] + npd[k - 1]; }
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (t = 0; t < N; ++t) {
        double xi[MAXD], acc = 0.0, gacc[MAXD] = {0, 0, 0}, v, g[MAXD];
        int64_t rem = t;
        int c, kk, started = 0;
        for (kk = d - 1; kk >= 0; --kk) { xi[kk] = pts[poff[kk] + rem % npd[kk]]; rem /= npd[kk]; }
        for (c = 0; c < D->n_comp; ++c) {
            double cf;
            if (comp >= 0 && c != comp) continue;
            comp_point(D, S[c].kv, S[c].n, coefs + off[c], xi, grads != NULL, &v, g);
            cf = comp >= 0 ? 1.0 : (double)D->coefs[c];
            if (!started) { acc = cf * v; for (kk = 0; kk < d; ++kk) gacc[kk] = cf * g[kk]; }
            else { acc += cf * v; for (kk = 0; kk < d; ++kk) gacc[kk] += cf * g[kk]; }
            started = 1;
        }
        vals[t] = acc;
        if (grads) for (kk = 0; kk < d; ++kk) grads[t * d + kk] = gacc[kk];
    }
    spaces_free(D, S);
    free(off);
    return SGIGA_OK;
}

/* error_norms (analysis.py:262-270) of the combined solution against the
 * closed form, on a QuadGrid (assembly.py:141-183) given by per-axis
 * points and weights. out = {L2, H1-seminorm}. */
int orc_error_norms(const sgiga_problem_desc* D, const double* coefs, const double* pts,
                    const double* wts, const int64_t* npd, int solution_id, int nthreads,
                    double* out) {
    int d = D->d, k;
    int64_t N = 1, t, poff[MAXD];
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (D->n_comp + 1));
    ospace* S = spaces_build(D);
    ogeo G;
    double l2 = 0.0, h1 = 0.0;
    int bad = 0;
    geo_from_desc(D, &G);
    orc_total_dofs(D, off);
    poff[0] = 0;
    for (k = 0; k < d; ++k) { N *= npd[k]; if (k) poff[k] = poff[k - 1] + npd[k - 1]; }
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(+ : l2, h1) reduction(| : bad)
    for (t = 0; t < N; ++t) {
        double xi[MAXD], x[MAXD], J[9], Ji[9], det, w, acc = 0.0, gacc[MAXD] = {0, 0, 0};
        double v, g[MAXD], ue, ge[MAXD], dv, dg2 = 0.0;
        int64_t rem = t;
        int c, kk, ii, started = 0;
        for (kk = d - 1; kk >= 0; --kk) {
            int64_t j = rem % npd[kk];
            xi[kk] = pts[poff[kk] + j];
            rem /= npd[kk];
        }
        /* wgrid * det (assembly.py:171-178) */
        {
            int64_t r2 = t, jj[MAXD];
            for (kk = d - 1; kk >= 0; --kk) { jj[kk] = r2 % npd[kk]; r2 /= npd[kk]; }
            w = wts[poff[0] + jj[0]];
            for (kk = 1; kk < d; ++kk) w = w * wts[poff[kk] + jj[kk]];
        }
        geo_map(&G, xi, x, J, &det);
        if (!(det > 0.0)) bad |= 1;
        inv_small(d, J, det, Ji);
        for (c = 0; c < D->n_comp; ++c) {
            double cf = (double)D->coefs[c];
            comp_point(D, S[c].kv, S[c].n, coefs + off[c], xi, 1, &v, g);
            if (!started) { acc = cf * v; for (kk = 0; kk < d; ++kk) gacc[kk] = cf * g[kk]; }
            else { acc += cf * v; for (kk = 0; kk < d; ++kk) gacc[kk] += cf * g[kk]; }
            started = 1;
        }
        solution_eval(solution_id, d, x, &ue, ge);
        dv = acc - ue;
        /* push gradient by J^{-T} (analysis.py:235-237) */
        for (ii = 0; ii < d; ++ii) {
            double s = 0.0, e;
            for (kk = 0; kk < d; ++kk) s += Ji[kk * d + ii] * gacc[kk];
            e = s - ge[ii];
            dg2 += e * e;
        }
        l2 += (w * det) * (dv * dv);
        h1 += (w * det) * dg2;
    }
    spaces_free(D, S);
    free(off);
    out[0] = sqrt(l2);
    out[1] = sqrt(h1);
    return bad ? SGIGA_ERR_GEOMETRY : SGIGA_OK;
}

/* one-component solve statistics used by the tests: PCG iteration count */
int orc_component_pcg(const sgiga_problem_desc* D, int c, double rtol, double* coefs,
                      int32_t* iters, double* relres) {
    int it = 0, st;
    st = run_component(D, c, 1, rtol, coefs, relres, &it);
    *iters = it;
    return st;
}
