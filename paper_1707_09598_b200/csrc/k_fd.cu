// k_fd.cu -- fast-diagonalisation (FD) preconditioned CG for the small
// components: the preconditioner is the exact inverse of the parametric
// Kronecker-sum operator
//     P = sum_k c_k (M_1 x .. x K_k x .. x M_d),
// applied as  P^-1 = (U_1 x .. x U_d) diag(1 / sum_k c_k lambda_k)(U_1 x .. x U_d)^T
// with  K_k U_k = M_k U_k Lambda_k,  U_k^T M_k U_k = I  (the 1-D interior
// stiffness / mass pencil of each axis' knot vector).  c_k = integral of the
// metric entry G_kk over the patch (sum over the quadrature points), so for
// the identity geometry (unit hypercube, constant metric) P == A and CG
// converges in one or two iterations; for a smooth map P is spectrally
// equivalent to A independently of h and p (Sangalli & Tani, SIAM J. Sci.
// Comput. 2016).  The reference solves the same systems with SuperLU
// (linsolve.py:16-54); any solver meeting its residual contract may replace
// it, and the true residual ||A x - b|| / ||b|| is checked here on exit.
//
// Kernel 3a (k_fd_eigen): one CTA per distinct 1-D knot vector -- interior
// M and K from the quadrature tables (band only), banded Cholesky M = L L^T,
// C = L^-1 K L^-T, cyclic parallel Jacobi C = Q Lambda Q^T, U = L^-T Q.
// Kernel 3b (k_pcg_fd): one CTA per component, every vector in shared
// memory, SpMV from the slot-major stencil, P^-1 as 2d mode products.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "handle.cuh"

namespace sgiga {

#ifndef SGIGA_FDL_UNR
#define SGIGA_FDL_UNR 16
#endif
#ifndef SGIGA_FDL_UNR2
#define SGIGA_FDL_UNR2 32
#endif
#ifndef SGIGA_FDL_FUSED_UNR1
#define SGIGA_FDL_FUSED_UNR1 0
#endif
#ifndef SGIGA_FDL_FUSED_MINB
#define SGIGA_FDL_FUSED_MINB 2
#endif
// the fused-residual instantiation: 2 CTAs per SM (128 registers) and 32
// stencil loads in flight in the double-product sweep -- at 3 CTAs / 80
// registers ptxas serialises the load batch (measured: cfg5 pass 3.58 -> 3.46
// ms; 24 loads 3.49, 1 CTA x 64 loads 4.27, first sweep at 32 loads 3.47)
constexpr int FDL_UNR2 = SGIGA_FDL_UNR2;   // the double-product sweep's loads in flight (even)
constexpr int FDL_UNR = SGIGA_FDL_UNR;   // line-FD SpMV: stencil loads in flight per thread (even)

constexpr int FD_THREADS = 512;
constexpr int EIG_THREADS = 512;
constexpr int EIG_ITEMS = ((FD_MMAX / 2) * (FD_MMAX / 2) + (FD_MMAX / 2) * FD_MMAX + EIG_THREADS - 1) / EIG_THREADS;
constexpr int FD_LD = FD_MMAX + 1;   // padded row stride of the eigen work arrays
// staged quadrature tables of one knot vector: 2 nel q (p+1) + nel q <= 74 * 10 * 11
constexpr int FD_TAB_MAX = 8192;

template <int NT = FD_THREADS>
__device__ __forceinline__ double fd_block_sum(double v, double* red) {
    // fixed-order block sum (deterministic): warp tree, then warp partials in order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    return s;
}

// ---- 3a: generalized eigen-decomposition of the 1-D interior pencils ------
// Persymmetric pencils (symmetric knot vectors, e.g. uniform): M and K
// commute with the exchange J, so the pencil splits exactly into its even
// (dimension ceil(m/2)) and odd (floor(m/2)) halves, solved side by side --
// half the Jacobi steps, a quarter of the work per step.  Both halves sit
// block-diagonally in one m x m array, so the banded Cholesky and the
// substitutions run unchanged (each half is banded with bandwidth p).
// Jacobi step = rotations of every pair of the round-robin pairings (one per
// half) then ONE pass of fused two-sided 2x2 block updates J_k^T C_kl J_l
// (every entry of C belongs to exactly one (pair k, pair l) block: race-free)
// plus the column rotations of V: two barriers per step.
__device__ __forceinline__ double fd_block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < EIG_THREADS / 32; ++w) s = fmax(s, red[w]);
    return s;
}

__global__ void __launch_bounds__(EIG_THREADS)
k_fd_eigen(const TabInfo* __restrict__ tabs, const int* __restrict__ uniq,
           const int64_t* __restrict__ uoff, const int64_t* __restrict__ loff,
           const double* __restrict__ vals, const double* __restrict__ qw, int p, int mu, int q,
           double* __restrict__ dU, double* __restrict__ dL, long long* __restrict__ prof) {
    extern __shared__ double fsm[];
    long long t0 = clock64();
    auto stamp = [&](int k) { if (prof && threadIdx.x == 0) prof[blockIdx.x * 8 + k] = clock64() - t0; };
    constexpr int NPMAX = FD_MMAX / 2 + 1;
    __shared__ double rc[NPMAX + 1], rs[NPMAX + 1], red[EIG_THREADS / 32], rdg[FD_MMAX];
    __shared__ int rp[NPMAX + 1], rq[NPMAX + 1];
    const int t = uniq[blockIdx.x];
    const TabInfo T = tabs[t];
    const int m = T.n - 2, tid = threadIdx.x, P = p + 1;
    double* L = fsm;                       // M, then its Cholesky factor (lower)
    double* Cm = L + FD_MMAX * FD_LD;      // K, then L^-1 K L^-T, then Lambda
    double* V = Cm + FD_MMAX * FD_LD;      // Jacobi rotations, then U
    double* tb = V + FD_MMAX * FD_LD;      // staged basis values | derivatives | weights
    const int nq = T.nel * q;
    {   // one coalesced copy of this knot vector's quadrature tables
        const double* bvg = vals + T.val_off;
        const double* wg = qw + T.qp_off;
        const int nv = 2 * nq * P;
        for (int i = tid; i < nv; i += EIG_THREADS) tb[i] = bvg[i];
        for (int i = tid; i < nq; i += EIG_THREADS) tb[nv + i] = wg[i];
    }
    const double* bv = tb;
    const double* bd = bv + nq * P;
    const double* w = bd + nq * P;
    __syncthreads();

    // interior mass / stiffness (global functions 1..n-2), band |i-j| <= p
    double dmx = 0.0, amx = 0.0;
    for (int idx = tid; idx < m * m; idx += EIG_THREADS) {
        const int i = idx / m, j = idx % m, gi = i + 1, gj = j + 1;
        double mv = 0.0, kv = 0.0;
        if (abs(gi - gj) <= p) {
            const int num = max(gi, gj) - p;
            const int elo = num <= 0 ? 0 : (num + mu - 1) / mu;
            const int ehi = min(min(gi, gj) / mu, T.nel - 1);
            for (int e = elo; e <= ehi; ++e) {
                const int a = gi - e * mu, b = gj - e * mu;
                for (int g = 0; g < q; ++g) {
                    const int base = (e * q + g) * P;
                    const double wq = w[e * q + g];
                    mv += wq * bv[base + a] * bv[base + b];
                    kv += wq * bd[base + a] * bd[base + b];
                }
            }
        }
        L[i * FD_LD + j] = mv;
        Cm[i * FD_LD + j] = kv;
    }
    __syncthreads();
    // persymmetry test (relative to the largest entry; K dominates the scale)
    for (int idx = tid; idx < m * m; idx += EIG_THREADS) {
        const int i = idx / m, j = idx % m, ii = m - 1 - i, jj = m - 1 - j;
        dmx = fmax(dmx, fmax(fabs(L[i * FD_LD + j] - L[ii * FD_LD + jj]),
                             fabs(Cm[i * FD_LD + j] - Cm[ii * FD_LD + jj]) * 1e-6));
        amx = fmax(amx, fmax(fabs(L[i * FD_LD + j]), fabs(Cm[i * FD_LD + j]) * 1e-6));
    }
    dmx = fd_block_max(dmx, red);
    amx = fd_block_max(amx, red);
    const bool sym = m >= 2 && dmx <= 1e-13 * amx;
    const int h = m / 2, ms = sym ? m - h : m, ma = sym ? h : 0;
    const double r2 = 0.70710678118654752440;
    // column c of the even / odd basis S: entries (index, weight)
    auto sbasis = [&](int c, int* ix, double* wt) -> int {   // c < ms
        if (c < h) { ix[0] = c; wt[0] = r2; ix[1] = m - 1 - c; wt[1] = r2; return 2; }
        ix[0] = h; wt[0] = 1.0; return 1;                      // the middle function (m odd)
    };
    if (sym) {   // L, Cm <- S^T M S (+) A^T M A, block-diagonal (V as scratch)
        for (int pass = 0; pass < 2; ++pass) {
            double* X = pass ? Cm : L;
            for (int idx = tid; idx < m * m; idx += EIG_THREADS) {
                const int i = idx / m, j = idx % m;
                double v = 0.0;
                if (i < ms && j < ms) {
                    int ia[2], ja[2];
                    double wa[2], wb[2];
                    const int na = sbasis(i, ia, wa), nb = sbasis(j, ja, wb);
                    for (int x = 0; x < na; ++x)
                        for (int y = 0; y < nb; ++y) v += wa[x] * wb[y] * X[ia[x] * FD_LD + ja[y]];
                } else if (i >= ms && j >= ms) {
                    const int a = i - ms, b = j - ms, a2 = m - 1 - a, b2 = m - 1 - b;
                    v = 0.5 * ((X[a * FD_LD + b] - X[a * FD_LD + b2]) - (X[a2 * FD_LD + b] - X[a2 * FD_LD + b2]));
                }
                V[i * FD_LD + j] = v;
            }
            __syncthreads();
            for (int idx = tid; idx < m * m; idx += EIG_THREADS) X[(idx / m) * FD_LD + idx % m] = V[(idx / m) * FD_LD + idx % m];
            __syncthreads();
        }
    }
    stamp(0);
    // banded Cholesky M = L L^T of each diagonal block (one warp per block,
    // the two persymmetric halves side by side); rdg = 1 / diag(L)
    {
        const int warp = tid >> 5, lane = tid & 31;
        const int nblk = sym && ma > 0 ? 2 : 1;
        if (warp < nblk) {
            const int b0 = warp ? ms : 0, b1 = warp ? m : ms;
            // lane -> (i, j) of the p x p trailing update, 1 <= j <= i <= p
            int ui = 0, uj = 0;
            {
                int c = lane;
                for (int i = 1; i <= p && ui == 0; ++i) { if (c < i) { ui = i; uj = c + 1; } else c -= i; }
            }
            for (int k = b0; k < b1; ++k) {
                const double d = sqrt(L[k * FD_LD + k]);
                const double rd = 1.0 / d;
                const bool wc = lane >= 1 && lane <= p && k + lane < b1, wu = ui > 0 && k + ui < b1;
                const double cv = wc ? L[(k + lane) * FD_LD + k] : 0.0;
                double li = 0.0, lj = 0.0, tv = 0.0;
                if (wu) { li = L[(k + ui) * FD_LD + k] * rd; lj = L[(k + uj) * FD_LD + k] * rd; tv = L[(k + ui) * FD_LD + k + uj]; }
                __syncwarp();
                if (lane == 0) { L[k * FD_LD + k] = d; rdg[k] = rd; }
                if (wc) L[(k + lane) * FD_LD + k] = cv * rd;
                if (wu) L[(k + ui) * FD_LD + k + uj] = tv - li * lj;
                __syncwarp();
            }
        }
        for (int idx = tid; idx < m * m; idx += EIG_THREADS)   // V = I (Jacobi accumulator)
            V[(idx / m) * FD_LD + idx % m] = (idx / m == idx % m) ? 1.0 : 0.0;
    }
    __syncthreads();
    stamp(1);
    // X = L^-1 K (column j per thread), then C = X L^-T (row r per thread):
    // forward substitutions with the last p results in registers
    if (tid < m) {
        const int j = tid;
        const int b0 = (sym && j >= ms) ? ms : 0, b1 = (sym && j < ms) ? ms : m;
        double xw[PMAX - 1] = {};
        for (int i = b0; i < b1; ++i) {
            double s = Cm[i * FD_LD + j];
#pragma unroll
            for (int l = PMAX - 2; l >= 0; --l)   // xw[l] = X[i-1-l][j]
                if (l < p && i - 1 - l >= b0) s -= L[i * FD_LD + i - 1 - l] * xw[l];
            s *= rdg[i];
#pragma unroll
            for (int l = PMAX - 2; l > 0; --l) xw[l] = xw[l - 1];
            xw[0] = s;
            Cm[i * FD_LD + j] = s;
        }
    }
    __syncthreads();
    if (tid < m) {
        const int r = tid;
        const int b0 = (sym && r >= ms) ? ms : 0, b1 = (sym && r < ms) ? ms : m;
        double xw[PMAX - 1] = {};
        for (int i = b0; i < b1; ++i) {
            double s = Cm[r * FD_LD + i];
#pragma unroll
            for (int l = PMAX - 2; l >= 0; --l)
                if (l < p && i - 1 - l >= b0) s -= L[i * FD_LD + i - 1 - l] * xw[l];
            s *= rdg[i];
#pragma unroll
            for (int l = PMAX - 2; l > 0; --l) xw[l] = xw[l - 1];
            xw[0] = s;
            Cm[r * FD_LD + i] = s;
        }
    }
    __syncthreads();
    for (int idx = tid; idx < m * m; idx += EIG_THREADS) {   // symmetrise
        const int i = idx / m, j = idx % m;
        if (i < j) {
            const double a = 0.5 * (Cm[i * FD_LD + j] + Cm[j * FD_LD + i]);
            Cm[i * FD_LD + j] = a;
            Cm[j * FD_LD + i] = a;
        }
    }
    __syncthreads();
    stamp(2);
    // cyclic parallel Jacobi: one round-robin pairing per half (block b at
    // offset ob, size sb, padded to nb even; local index sb is a dummy)
    const int o1 = ms, s0 = ms, s1 = ma;
    const int n0 = s0 + (s0 & 1), n1 = s1 + (s1 & 1), np0 = n0 / 2, np1 = n1 / 2, npt = np0 + np1;
    const int nsteps = max(n0, n1) - 1;
    // C stays exactly symmetric: only the blocks k <= l are computed, the
    // (l, k) block is written as the transpose of (k, l)
    const int nc0 = np0 * (np0 + 1) / 2, nc1 = np1 * (np1 + 1) / 2, ncs = nc0 + nc1;
    const int nitems = ncs + np0 * s0 + np1 * s1;
    auto tri = [](int r, int n, int& k, int& l) {   // r-th (k, l), k <= l < n, row-major
        k = 0;
        while (r >= n - k) { r -= n - k; ++k; }
        l = k + r;
    };
    int nsweep = 0;
    long long acc_rot = 0, acc_upd = 0;   // probe (SGIGA_FD_PROFILE)
    // this thread's update items, decoded once: (pair k, pair l) blocks of C
    // (same half), then (pair k, row i of its half) rotations of V
    int dk_[EIG_ITEMS], dl_[EIG_ITEMS];
#pragma unroll
    for (int u = 0; u < EIG_ITEMS; ++u) {
        const int idx = tid + u * EIG_THREADS;
        dk_[u] = 0; dl_[u] = 0;
        if (idx < nc0) tri(idx, np0, dk_[u], dl_[u]);
        else if (idx < ncs) { tri(idx - nc0, np1, dk_[u], dl_[u]); dk_[u] += np0; dl_[u] += np0; }
        else if (idx < ncs + np0 * s0) { const int r = idx - ncs; dk_[u] = r / s0; dl_[u] = r % s0; }
        else if (idx < nitems) { const int r = idx - ncs - np0 * s0; dk_[u] = np0 + r / s1; dl_[u] = o1 + r % s1; }
    }
    // stop at ||offdiag|| <= 1e-13 ||diag||: below that the off-diagonal is
    // rounding noise of the rotations (~eps * lambda_max per entry); the
    // preconditioner only needs the eigen-pairs to a few digits short of eps
    for (int sweep = 0; sweep < 15 && m > 1; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int idx = tid; idx < m * m; idx += EIG_THREADS) {
            const int i = idx / m, j = idx % m;
            const double v = Cm[i * FD_LD + j];
            if (i == j) dia += v * v; else off += v * v;
        }
        off = fd_block_sum<EIG_THREADS>(off, red);
        dia = fd_block_sum<EIG_THREADS>(dia, red);
        if (off <= 1e-26 * dia) break;
        ++nsweep;
        for (int st = 0; st < nsteps; ++st) {
            long long tr0 = (prof && tid == 0) ? clock64() : 0;
            if (tid < npt) {   // rotation of pair tid (its half's round-robin pairing, step st)
                const int b = tid < np0 ? 0 : 1, k = b ? tid - np0 : tid;
                const int nb = b ? n1 : n0, sb = b ? s1 : s0, ob = b ? o1 : 0;
                int pi = -1, qi = -1;
                double c = 1.0, sn = 0.0;
                if (st < nb - 1) {
                    int a, bb;
                    if (k == 0) { a = nb - 1; bb = st; }
                    else {   // (st + k) mod (nb-1), (st - k) mod (nb-1) without integer division
                        a = st + k; if (a >= nb - 1) a -= nb - 1;
                        bb = st - k; if (bb < 0) bb += nb - 1;
                    }
                    const int lo = min(a, bb), hi = max(a, bb);
                    if (hi < sb) { pi = ob + lo; qi = ob + hi; }
                    else if (lo < sb) { pi = ob + lo; }   // paired with the dummy
                }
                if (qi >= 0) {
                    const double apq = Cm[pi * FD_LD + qi];
                    const double app = Cm[pi * FD_LD + pi], aqq = Cm[qi * FD_LD + qi];
                    if (apq != 0.0 && apq * apq > 1e-36 * fabs(app * aqq)) {
                        // t = tan of the rotation = sgn(phi) psi / (|phi| + hypot(phi, psi)),
                        // phi = aqq - app, psi = 2 apq; c = 1/sqrt(1+t^2), s = t c, written
                        // without divisions: with D = |phi| + hypot, c = D / hypot(D, psi)
                        const double phi = aqq - app, psi = 2.0 * apq;
                        const double dd = fabs(phi) + sqrt(fma(phi, phi, psi * psi));
                        const double ir = rsqrt(fma(dd, dd, psi * psi));
                        c = dd * ir;
                        sn = copysign(1.0, phi) * psi * ir;
                    }
                }
                rp[tid] = pi; rq[tid] = qi; rc[tid] = c; rs[tid] = sn;
            }
            __syncthreads();
            long long tr1 = (prof && tid == 0) ? clock64() : 0;
#pragma unroll
            for (int u = 0; u < EIG_ITEMS; ++u) {
                const int idx = tid + u * EIG_THREADS;
                if (idx >= nitems) break;
                if (idx < ncs) {   // block (pair k rows) x (pair l columns)
                    const int k = dk_[u], l = dl_[u];
                    const double sk = rs[k], sl = rs[l];
                    if (sk == 0.0 && sl == 0.0) continue;
                    const int pk = rp[k], qk = rq[k], pl = rp[l], ql = rq[l];
                    const double ck = rc[k], cl = rc[l];
                    const bool hq = qk >= 0, hl = ql >= 0;   // (pk, pl exist: a rotating pair has both)
                    double a = Cm[pk * FD_LD + pl];
                    double b = hl ? Cm[pk * FD_LD + ql] : 0.0;
                    double c = hq ? Cm[qk * FD_LD + pl] : 0.0;
                    double d = (hq && hl) ? Cm[qk * FD_LD + ql] : 0.0;
                    // rows: J_k^T, then columns: J_l
                    const double a1 = ck * a - sk * c, b1 = ck * b - sk * d;
                    const double c1 = sk * a + ck * c, d1 = sk * b + ck * d;
                    a = cl * a1 - sl * b1; b = sl * a1 + cl * b1;
                    c = cl * c1 - sl * d1; d = sl * c1 + cl * d1;
                    if (k == l) { b = 0.0; c = 0.0; }   // the annihilated pair
                    Cm[pk * FD_LD + pl] = a;
                    if (hl) Cm[pk * FD_LD + ql] = b;
                    if (hq) Cm[qk * FD_LD + pl] = c;
                    if (hq && hl) Cm[qk * FD_LD + ql] = d;
                    if (k != l) {   // the transposed block (l, k)
                        Cm[pl * FD_LD + pk] = a;
                        if (hl) Cm[ql * FD_LD + pk] = b;
                        if (hq) Cm[pl * FD_LD + qk] = c;
                        if (hq && hl) Cm[ql * FD_LD + qk] = d;
                    }
                } else {               // V J_k, row i
                    const int k = dk_[u], i = dl_[u];
                    const double sk = rs[k];
                    if (sk == 0.0) continue;
                    const int pk = rp[k], qk = rq[k];
                    const double ck = rc[k];
                    const double va = V[i * FD_LD + pk], vb = V[i * FD_LD + qk];
                    V[i * FD_LD + pk] = ck * va - sk * vb;
                    V[i * FD_LD + qk] = sk * va + ck * vb;
                }
            }
            __syncthreads();
            if (prof && tid == 0) { acc_rot += tr1 - tr0; acc_upd += clock64() - tr1; }
        }
    }
    stamp(3);
    if (prof && tid == 0) {
        prof[blockIdx.x * 8 + 5] = nsweep;
        prof[blockIdx.x * 8 + 6] = m + (sym ? 1000 : 0);
        prof[blockIdx.x * 8 + 7] = acc_rot;
        prof[blockIdx.x * 8 + 4] = acc_upd;
    }
    // U' = L^-T Q (column j per thread, back substitution in its diagonal block)
    if (tid < m) {
        const int j = tid;
        const int b0 = (sym && j >= ms) ? ms : 0, b1 = (sym && j < ms) ? ms : m;
        double xw[PMAX - 1] = {};
        for (int i = b1 - 1; i >= b0; --i) {
            double s = V[i * FD_LD + j];
#pragma unroll
            for (int l = PMAX - 2; l >= 0; --l)   // xw[l] = U'[i+1+l][j]
                if (l < p && i + 1 + l < b1) s -= L[(i + 1 + l) * FD_LD + i] * xw[l];
            s *= rdg[i];
#pragma unroll
            for (int l = PMAX - 2; l > 0; --l) xw[l] = xw[l - 1];
            xw[0] = s;
            V[i * FD_LD + j] = s;
        }
    }
    __syncthreads();
    // back to the original basis: u = S u' (even half) or A u' (odd half)
    double* U = dU + uoff[t];
    for (int idx = tid; idx < m * m; idx += EIG_THREADS) {
        const int a = idx / m, j = idx % m;   // eigenvector a, entry j
        double v;
        if (!sym) v = V[j * FD_LD + a];
        else if (a < ms) v = (j < h) ? r2 * V[j * FD_LD + a] : (j >= m - h ? r2 * V[(m - 1 - j) * FD_LD + a] : V[h * FD_LD + a]);
        else v = (j < h) ? r2 * V[(ms + j) * FD_LD + a] : (j >= m - h ? -r2 * V[(ms + m - 1 - j) * FD_LD + a] : 0.0);
        U[idx] = v;
    }
    for (int a = tid; a < m; a += EIG_THREADS) dL[loff[t] + a] = Cm[a * FD_LD + a];
}

// ---- 3b: FD-preconditioned CG, one CTA per component -----------------------
__device__ __forceinline__ int fd_row_base(const CompInfo& C, int d, int row) {
    int rb = row;
    for (int k = 0; k < d; ++k)
        if (C.absm[k]) rb -= ((row / (int)C.rs[k]) % C.m[k]) * (int)C.rs[k];
    return rb;
}

// full C-order coefficient vector of component C from its internal-order
// interior solution x (thread t of nt): interior dofs get x, boundary dofs 0
template <int D>
__device__ __forceinline__ void fd_expand(const CompInfo& C, const double* __restrict__ x,
                                          double* __restrict__ coef, int t, int nt) {
    int n[D], rs[D];
#pragma unroll
    for (int k = 0; k < D; ++k) { n[k] = C.n[k]; rs[k] = (int)C.rs[k]; }
    double* cf = coef + C.dof_off;
    const int nd = (int)C.ndofs;
    for (int f = t; f < nd; f += nt) {
        int rem = f, row = 0;
        bool inter = true;
#pragma unroll
        for (int k = D - 1; k >= 0; --k) {
            const int ik = rem % n[k];
            rem /= n[k];
            if (ik < 1 || ik > n[k] - 2) inter = false;
            else row += (ik - 1) * rs[k];
        }
        cf[f] = inter ? x[row] : 0.0;
    }
}

// SpMV of the FD kernel: q = A v, v halo-padded in shared memory.  np
// threads per row (slot classes t = part mod np), consecutive threads on
// consecutive rows so the stencil loads coalesce, 16 independent loads in
// flight per thread; the np partial sums are added in fixed order.  Out of
// line: both call sites (the PCG loop and the true residual) get the same
// load batching.
template <int D>
__device__ __noinline__ void fd_spmv(const CompInfo& C, const double* __restrict__ val, const int* __restrict__ offs,
                                     const double* __restrict__ ph, double* __restrict__ qs,
                                     double* __restrict__ qp, int R, int NS, int np) {
    const int tid = threadIdx.x;
    for (int w = tid; w < R * np; w += FD_THREADS) {
        const int part = w / R, row = w - part * R;
        const int rb = fd_row_base(C, D, row);
        double y0 = 0.0, y1 = 0.0;
        int t = part;
        for (; t + 15 * np < NS; t += 16 * np) {
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = __ldg(val + (size_t)(t + u * np) * R + row);
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
                y0 += v[u] * ph[rb + offs[t + u * np]];
                y1 += v[u + 1] * ph[rb + offs[t + (u + 1) * np]];
            }
        }
        for (; t < NS; t += np) y0 += __ldg(val + (size_t)t * R + row) * ph[rb + offs[t]];
        if (np == 1) qs[row] = y0 + y1;
        else qp[w] = y0 + y1;
    }
    __syncthreads();
    if (np == 1) return;
    for (int row = tid; row < R; row += FD_THREADS) {
        double y = qp[row];
        for (int k = 1; k < np; ++k) y += qp[k * R + row];
        qs[row] = y;
    }
    __syncthreads();
}

template <int D>
__global__ void __launch_bounds__(FD_THREADS, 1)
k_pcg_fd(const CompInfo* __restrict__ comps, const int* __restrict__ list,
         const int* __restrict__ slotoff, const double* __restrict__ stencil,
         const double* __restrict__ rhs, const double* __restrict__ Gbuf,
         const int64_t* __restrict__ uoff, const int64_t* __restrict__ loff,
         const double* __restrict__ dU, const double* __restrict__ dL, const double* __restrict__ ckg,
         double* __restrict__ xout, double* __restrict__ coef, CgState* __restrict__ st,
         double* __restrict__ relres, double rtol2, int maxit, long long* __restrict__ prof) {
    extern __shared__ double fsm[];
    const long long t0 = clock64();
    auto stamp = [&](int k) { if (prof && threadIdx.x == 0) prof[blockIdx.x * 8 + k] = clock64() - t0; };
    __shared__ double red[FD_THREADS / 32];
    const int c = list[blockIdx.x];
    const CompInfo& C = comps[c];
    const int R = (int)C.rows, H = (int)C.halo, NS = (int)C.nslots, tid = threadIdx.x;
    int mk[D], rsk[D];
    int64_t us[D], ls[D];
    int ntot_u = 0, ntot_l = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        mk[k] = C.m[k];
        rsk[k] = (int)C.rs[k];
        us[k] = ntot_u; ntot_u += mk[k] * mk[k];
        ls[k] = ntot_l; ntot_l += mk[k];
    }
    double* xs = fsm;
    double* rs_ = xs + R;
    double* zs = rs_ + R;
    double* qs = zs + R;
    double* ts = qs + R;
    double* pe = ts + R;              // p with zero halos [H + R + H]
    double* ph = pe + H;
    double* Us = pe + R + 2 * H;      // U_k, k = 0..D-1
    double* Ls = Us + ntot_u;         // lambda_k
    double* qp = Ls + ntot_l;         // SpMV partial sums [FD_THREADS]
    int* offs = reinterpret_cast<int*>(qp + FD_THREADS);
    const double* b = rhs + C.vec_off;
    const double* val = stencil + C.mat_off;

    for (int i = tid; i < NS; i += FD_THREADS) offs[i] = slotoff[C.so_off + i];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const int t = C.tab[k];
        for (int i = tid; i < mk[k] * mk[k]; i += FD_THREADS) Us[us[k] + i] = dU[uoff[t] + i];
        for (int i = tid; i < mk[k]; i += FD_THREADS) Ls[ls[k] + i] = dL[loff[t] + i];
    }
    for (int i = tid; i < H; i += FD_THREADS) { pe[i] = 0.0; pe[H + R + i] = 0.0; }
    // c_k = sum over the quadrature points of G_kk (the patch integral of the
    // metric's diagonal; 1 for the identity map), from k_fd_metric_scale
    double ck[D];
#pragma unroll
    for (int k = 0; k < D; ++k) ck[k] = ckg[c * MAXD + k];
    // z = P^-1 v  (v -> ts -> zs -> ... ; 2D mode products, result in zs)
    auto mode = [&](const double* src, double* dst, int k, bool trans) {
        const int m = mk[k], s = rsk[k];
        const double* U = Us + us[k];
        for (int row = tid; row < R; row += FD_THREADS) {
            const int a = (row / s) % m, base = row - a * s;
            double acc = 0.0;
            if (trans) {
                for (int j = 0; j < m; ++j) acc += U[a * m + j] * src[base + j * s];
            } else {
                for (int j = 0; j < m; ++j) acc += U[j * m + a] * src[base + j * s];
            }
            dst[row] = acc;
        }
        __syncthreads();
    };
    auto scale = [&](double* v) {
        for (int row = tid; row < R; row += FD_THREADS) {
            double den = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) den += ck[k] * Ls[ls[k] + (row / rsk[k]) % mk[k]];
            v[row] /= den;
        }
        __syncthreads();
    };
    auto precond = [&](const double* v) {   // -> zs
        double* bufs[2] = {ts, zs};
        const double* src = v;
        int w = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) { mode(src, bufs[w], k, true); src = bufs[w]; w ^= 1; }
        scale(const_cast<double*>(src));
#pragma unroll
        for (int k = D - 1; k >= 0; --k) { mode(src, bufs[w], k, false); src = bufs[w]; w ^= 1; }
    };
    // q = A v for v held in ph (halo-padded), see fd_spmv
    const int np = max(1, min(8, FD_THREADS / max(R, 1)));
    auto spmv = [&]() { fd_spmv<D>(C, val, offs, ph, qs, qp, R, NS, np); };

    double bbl = 0.0;
    for (int i = tid; i < R; i += FD_THREADS) {
        const double bi = b[i];
        xs[i] = 0.0;
        rs_[i] = bi;
        bbl += bi * bi;
    }
    const double bb = fd_block_sum(bbl, red);
    int it = 0, conv = (bb == 0.0);
    stamp(1);
    if (!conv) {
        precond(rs_);
        stamp(2);
        double rzl = 0.0;
        for (int i = tid; i < R; i += FD_THREADS) { ph[i] = zs[i]; rzl += rs_[i] * zs[i]; }
        double rz = fd_block_sum(rzl, red);
        while (it < maxit) {
            spmv();
            if (it == 0) stamp(3);
            double pql = 0.0;
            for (int i = tid; i < R; i += FD_THREADS) pql += ph[i] * qs[i];
            const double alpha = rz / fd_block_sum(pql, red);
            double rrl = 0.0;
            for (int i = tid; i < R; i += FD_THREADS) {
                xs[i] += alpha * ph[i];
                const double ri = rs_[i] - alpha * qs[i];
                rs_[i] = ri;
                rrl += ri * ri;
            }
            const double rr = fd_block_sum(rrl, red);
            ++it;
            if (rr <= rtol2 * bb) { conv = 1; break; }
            precond(rs_);
            double rzl2 = 0.0;
            for (int i = tid; i < R; i += FD_THREADS) rzl2 += rs_[i] * zs[i];
            const double rzn = fd_block_sum(rzl2, red);
            const double beta = rzn / rz;
            rz = rzn;
            for (int i = tid; i < R; i += FD_THREADS) ph[i] = zs[i] + beta * ph[i];
            __syncthreads();
        }
    }
    stamp(4);
    // true residual ||A x - b|| / ||b|| (linsolve.py:49-53)
    for (int i = tid; i < R; i += FD_THREADS) {
        ph[i] = xs[i];
        xout[C.vec_off + i] = xs[i];
    }
    __syncthreads();
    spmv();
    stamp(5);
    double eel = 0.0;
    for (int i = tid; i < R; i += FD_THREADS) {
        const double e = qs[i] - b[i];
        eel += isfinite(xs[i]) ? e * e : __longlong_as_double(0x7ff8000000000000ULL);
    }
    const double ee = fd_block_sum(eel, red);
    if (tid == 0) {
        st[c].it = it;
        st[c].conv = conv;
        st[c].active = 0;
        st[c].bb = bb;
        relres[c] = bb > 0.0 ? sqrt(ee / bb) : (ee == 0.0 ? 0.0 : ee);
    }
    // the component's full coefficient vector in the reference's C order,
    // zero on the boundary (AssembledSystem.expand, assembly.py:202-206)
    fd_expand<D>(C, xs, coef, tid, FD_THREADS);
    stamp(6);
    if (prof && tid == 0) prof[blockIdx.x * 8 + 7] = R * 1000 + NS;
}

// ---- 3e: line-FD preconditioned CG for components with ONE long axis -------
// P = c_s K_s x M_o + M_s x (sum_o c_o K_o x M_rest): the (at most two) other
// axes are diagonalised with their 1-D eigen-pairs (k_fd_eigen), leaving one
// banded SPD system (c_s K_s + mu M_s) per line along the stream axis (the
// longest; contiguous in the internal row order), mu = sum_o c_o lambda_o.
// For the identity map P == A again -- cfg5's (1,1,10) components converge
// in one or two iterations instead of ~27 000 Jacobi-PCG iterations -- and
// no eigen-decomposition of the long axis (up to 1026 functions) is needed:
// its pencil is only factorised per line by banded Cholesky.  One CTA per
// component, vectors in the batch's global PCG arrays (L2-resident).
constexpr int FDL_THREADS = 256;
constexpr int PM = PMAX - 1;   // largest degree: register windows of the banded line factors

// ---- FD set-up, off the critical path (side stream, overlapping the
// assembly; k_fd_setup_enqueue) ----------------------------------------------
// c_k = patch integral of G_kk (sum over the quadrature points) of every FD /
// line-FD component: one CTA per (component, axis), fixed-order block sum
template <int D>
__global__ void __launch_bounds__(256)
k_fd_metric_scale(const CompInfo* __restrict__ comps, const int* __restrict__ list_a, int na,
                  const int* __restrict__ list_b, const double* __restrict__ Gbuf, double* __restrict__ ckg) {
    __shared__ double red[8];
    const int c = blockIdx.x < na ? list_a[blockIdx.x] : list_b[blockIdx.x - na];
    const int k = blockIdx.y, tid = threadIdx.x;
    const CompInfo& C = comps[c];
    const double* g = Gbuf + C.qp_off + (int64_t)sym_index(D, k, k) * C.nqp;
    const int64_t n = C.nqp;
    double s0 = 0.0, s1 = 0.0;
    int64_t i = tid;
    for (; i + 7 * 256 < n; i += 8 * 256) {   // 8 loads in flight
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(g + i + u * 256);
#pragma unroll
        for (int u = 0; u < 8; u += 2) { s0 += v[u]; s1 += v[u + 1]; }
    }
    for (; i < n; i += 256) s0 += g[i];
    const double tot = fd_block_sum<256>(s0 + s1, red);
    if (tid == 0) ckg[c * MAXD + k] = tot;
}

// the same c_k for the whole-GPU FD components (millions of points each):
// FDG_SCALE_CHUNKS CTAs per (component, axis) write fixed-order partials,
// one CTA per (component, axis) sums them in chunk order (deterministic)
constexpr int FDG_SCALE_CHUNKS = 256;
template <int D>
__global__ void __launch_bounds__(256)
k_fd_metric_scale_part(const CompInfo* __restrict__ comps, const int* __restrict__ list,
                       const double* __restrict__ Gbuf, double* __restrict__ part) {
    __shared__ double red[8];
    const int ci = blockIdx.y, k = blockIdx.z, chunk = blockIdx.x, tid = threadIdx.x;
    const CompInfo& C = comps[list[ci]];
    const double* g = Gbuf + C.qp_off + (int64_t)sym_index(D, k, k) * C.nqp;
    const int64_t n = C.nqp, per = (n + FDG_SCALE_CHUNKS - 1) / FDG_SCALE_CHUNKS;
    const int64_t lo = chunk * per, hi = lo + per < n ? lo + per : n;
    double s0 = 0.0, s1 = 0.0;
    int64_t i = lo + tid;
    for (; i + 256 < hi; i += 512) { s0 += __ldg(g + i); s1 += __ldg(g + i + 256); }
    for (; i < hi; i += 256) s0 += g[i];
    const double tot = fd_block_sum<256>(s0 + s1, red);
    if (tid == 0) part[((int64_t)ci * MAXD + k) * FDG_SCALE_CHUNKS + chunk] = tot;
}

__global__ void __launch_bounds__(256)
k_fd_metric_scale_fin(const int* __restrict__ list, const double* __restrict__ part, double* __restrict__ ckg) {
    __shared__ double red[8];
    const int ci = blockIdx.x, k = blockIdx.y, tid = threadIdx.x;
    const double v = part[((int64_t)ci * MAXD + k) * FDG_SCALE_CHUNKS + tid];
    const double tot = fd_block_sum<256>(v, red);
    if (tid == 0) ckg[list[ci] * MAXD + k] = tot;
}
static_assert(FDG_SCALE_CHUNKS == 256, "one partial per thread of the finishing CTA");

// banded interior K_s, M_s of a line-FD component's stream axis (lower band,
// [i][k] = entry (i, i - k)), one CTA per component
template <int D>
__global__ void __launch_bounds__(256)
k_fdl_bands(const CompInfo* __restrict__ comps, const int* __restrict__ list, const TabInfo* __restrict__ tabs,
            const double* __restrict__ vals, const double* __restrict__ qw, int p, int mu, int q,
            const int64_t* __restrict__ fdl_off, double* __restrict__ fdl) {
    const int c = list[blockIdx.x];
    const CompInfo& C = comps[c];
    const int P1 = p + 1, s = C.ax[D - 1], ms = C.m[s];
    double* Kb = fdl + fdl_off[c];
    double* Mb = Kb + (int64_t)ms * P1;
    const TabInfo T = tabs[C.tab[s]];
    const int64_t nq = (int64_t)T.nel * q;
    const double* bv = vals + T.val_off;
    const double* bd = bv + nq * P1;
    const double* w = qw + T.qp_off;
    for (int idx = threadIdx.x; idx < ms * P1; idx += 256) {
        const int i = idx / P1, kk = idx % P1, j = i - kk, gi = i + 1, gj = j + 1;
        double mv = 0.0, kv = 0.0;
        if (j >= 0) {
            const int num = gi - p;   // gi >= gj
            const int elo = num <= 0 ? 0 : (num + mu - 1) / mu;
            const int ehi = min(gj / mu, T.nel - 1);
            for (int e = elo; e <= ehi; ++e) {
                const int a = gi - e * mu, bb = gj - e * mu;
                for (int g = 0; g < q; ++g) {
                    const int64_t base = ((int64_t)e * q + g) * P1;
                    const double wg = w[(int64_t)e * q + g];
                    mv += wg * bv[base + a] * bv[base + bb];
                    kv += wg * bd[base + a] * bd[base + bb];
                }
            }
        }
        Kb[idx] = kv;
        Mb[idx] = mv;
    }
}

// one banded Cholesky per line, c_s K_s + mu_L M_s = F F^T with
// mu_L = sum over the other axes of c_k lambda_k(line): one thread per line,
// the last p factor rows in registers.  Stored per row i: [0] = 1 / F(i,i),
// [k] = F(i, i-k), k = 1..p.  Grid (line blocks, component).  The
// component's K_s / M_s bands are staged in shared memory first: the row
// recurrence then waits on shared-memory, not L2, latency (cfg3: 106 us ->
// the serial chain of its longest line).
template <int D>
__global__ void __launch_bounds__(64)
k_fdl_factor(const CompInfo* __restrict__ comps, const int* __restrict__ list, int p,
             const int64_t* __restrict__ loff, const double* __restrict__ dL, const double* __restrict__ ckg,
             const int64_t* __restrict__ fdl_off, double* __restrict__ fdl, int staged) {
    const int c = list[blockIdx.y];
    const CompInfo& C = comps[c];
    const int P1 = p + 1, s = C.ax[D - 1], ms = C.m[s];
    int nlines = 1;
#pragma unroll
    for (int o = 0; o < D - 1; ++o) nlines *= C.m[C.ax[o]];
    const int L = blockIdx.x * 64 + threadIdx.x;
    if (blockIdx.x * 64 >= nlines) return;
    extern __shared__ double fband[];   // [K_s band | M_s band], ms * P1 each (when staged)
    const double* Kb = fdl + fdl_off[c];
    if (staged) {
        for (int i = threadIdx.x; i < 2 * ms * P1; i += blockDim.x) fband[i] = Kb[i];
        __syncthreads();
        Kb = fband;
    }
    if (L >= nlines) return;
    double muL = 0.0;
    {
        int rem = L;
#pragma unroll
        for (int o = D - 2; o >= 0; --o) {
            const int ax = C.ax[o], io = rem % C.m[ax];
            rem /= C.m[ax];
            muL += ckg[c * MAXD + ax] * dL[loff[C.tab[ax]] + io];
        }
    }
    const double cs = ckg[c * MAXD + s];
    const double* Mb = Kb + ms * P1;
    double* F = fdl + fdl_off[c] + 2 * (int64_t)ms * P1 + (int64_t)L * ms * P1;
    double Fw[PM][PM + 1], Rw[PM];   // Fw[d][k] = F(i-1-d, i-1-d-k)
#pragma unroll
    for (int d = 0; d < PM; ++d) {
        Rw[d] = 0.0;
#pragma unroll
        for (int k = 0; k <= PM; ++k) Fw[d][k] = 0.0;
    }
    for (int i = 0; i < ms; ++i) {
        double Fi[PM + 1];
#pragma unroll
        for (int k = 0; k <= PM; ++k) Fi[k] = 0.0;
#pragma unroll
        for (int kk = PM; kk >= 1; --kk) {   // F(i, j), j = i - kk, increasing j
            if (kk <= p && kk <= i) {
                double sv = cs * Kb[i * P1 + kk] + muL * Mb[i * P1 + kk];
#pragma unroll
                for (int ll = PM; ll > kk; --ll)   // l = i - ll < j
                    if (ll <= p && ll <= i) sv -= Fi[ll] * Fw[kk - 1][ll - kk];
                Fi[kk] = sv * Rw[kk - 1];
            }
        }
        double dv = cs * Kb[i * P1] + muL * Mb[i * P1];
#pragma unroll
        for (int ll = PM; ll >= 1; --ll)
            if (ll <= p && ll <= i) dv -= Fi[ll] * Fi[ll];
        const double r = 1.0 / sqrt(dv);
        F[i * P1] = r;
#pragma unroll
        for (int kk = 1; kk <= PM; ++kk)
            if (kk <= p) F[i * P1 + kk] = Fi[kk];
#pragma unroll
        for (int d = PM - 1; d >= 1; --d) {
            Rw[d] = Rw[d - 1];
#pragma unroll
            for (int k = 0; k <= PM; ++k) Fw[d][k] = Fw[d - 1][k];
        }
        Rw[0] = r;
#pragma unroll
        for (int k = 0; k <= PM; ++k) Fw[0][k] = Fi[k];
    }
}

template <int D, int PL, bool FUSED>   // PL = p (compile-time: the line scan's p x p state lives in registers); FUSED: true residual inside the sweeps
__global__ void __launch_bounds__(FDL_THREADS, FUSED ? SGIGA_FDL_FUSED_MINB : 3)
k_pcg_fdl(const CompInfo* __restrict__ comps, const int* __restrict__ list, const int* __restrict__ slotoff,
          const double* __restrict__ stencil, const double* __restrict__ rhs, int p,
          const int64_t* __restrict__ uoff, const double* __restrict__ dU, const double* __restrict__ ckg,
          const int64_t* __restrict__ fdl_off, const double* __restrict__ fdl, double* __restrict__ xg,
          double* __restrict__ rg, double* __restrict__ zg, double* __restrict__ pg, double* __restrict__ qg,
          double* __restrict__ tg, CgState* __restrict__ st, double* __restrict__ relres, double rtol2,
          int maxit, double* __restrict__ coef) {
    // one thread-block cluster of K CTAs per component: rows, lines and
    // vector work split over the K*FDL_THREADS threads, phases separated by
    // cluster barriers (release / acquire: the global-memory vectors written
    // by one CTA are visible to the others after it), dot products reduced
    // through distributed shared memory in fixed rank order
    namespace cgs = cooperative_groups;
    cgs::cluster_group cluster = cgs::this_cluster();
    __shared__ double red[FDL_THREADS / 32], cpart[2];
    const int K = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
    const int c = list[blockIdx.x / K];
    const CompInfo& C = comps[c];
    const int R = (int)C.rows, NS = (int)C.nslots, tid = threadIdx.x, P1 = p + 1;
    const int gt = rank * FDL_THREADS + tid, GT = K * FDL_THREADS;
    int slot = 0;
    auto csum = [&](double v) -> double {   // cluster-wide fixed-order sum
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        if (tid == 0) {
            double sacc = 0.0;
#pragma unroll
            for (int w = 0; w < FDL_THREADS / 32; ++w) sacc += red[w];
            cpart[slot] = sacc;
        }
        cluster.sync();
        double tot = 0.0;
        for (int r = 0; r < K; ++r) tot += *cluster.map_shared_rank(&cpart[slot], r);
        slot ^= 1;
        return tot;
    };
    const int s = C.ax[D - 1], ms = C.m[s];
    constexpr int NO = D - 1;                      // other axes: C.ax[0 .. D-2]
    int oax[NO > 0 ? NO : 1], om[NO > 0 ? NO : 1], ors[NO > 0 ? NO : 1];
    int nlines = 1;
#pragma unroll
    for (int o = 0; o < NO; ++o) {
        oax[o] = C.ax[o];
        om[o] = C.m[oax[o]];
        ors[o] = (int)C.rs[oax[o]];
        nlines *= om[o];
    }
    double* x = xg + C.vec_off;
    double* r = rg + C.vec_off;
    double* z = zg + C.vec_off;
    double* pp = pg + C.vec_off;   // zero halos on both sides (SpMV gathers)
    double* qq = qg + C.vec_off;
    double* t = tg + C.vec_off;
    const double* b = rhs + C.vec_off;
    const double* val = stencil + C.mat_off;
    // slot column offsets staged in shared memory (the SpMV's gathers then
    // depend on one global load, not two)
    __shared__ double lsF[FDL_THREADS / 32][32 * (PM + 1)], lsy[FDL_THREADS / 32][32];
    __shared__ int soffs[WMAX * WMAX * WMAX];
    for (int i = tid; i < NS; i += FDL_THREADS) soffs[i] = slotoff[C.so_off + i];
    __syncthreads();
    const int* offs = soffs;
    const double* Fac = fdl + fdl_off[c] + 2 * (int64_t)ms * P1;   // k_fdl_factor

    // mode product over other axis o (global buffers)
    auto mode = [&](const double* src, double* dst, int o, bool trans) {
        const int m = om[o], sr = ors[o];
        const double* U = dU + uoff[C.tab[oax[o]]];
        for (int row = gt; row < R; row += GT) {
            const int a = (row / sr) % m, base = row - a * sr;
            double acc = 0.0;
            if (trans) {
                for (int j = 0; j < m; ++j) acc += U[a * m + j] * src[base + j * sr];
            } else {
                for (int j = 0; j < m; ++j) acc += U[j * m + a] * src[base + j * sr];
            }
            dst[row] = acc;
        }
        cluster.sync();
    };
    // in place, every line L = rows [L*ms, (L+1)*ms): forward then backward
    // banded substitution, ONE WARP per line, parallel over the line: lane l
    // owns a segment of CH = ceil(ms / 32) rows.  A row of the recurrence is
    // an affine map of the state S = the last p results (companion matrix
    // A_i, first row a_k = -F(i,i)^-1 F(i, i-k)); each lane
    //   1. composes its segment's rows into one p x p affine map (M, v),
    //   2. receives its entry state from its predecessor lane: a chain of
    //      32 mat-vec steps (S_next = M S + v, one shuffle round each),
    //   3. reruns the plain recurrence over its rows from that state.
    // The sequential depth drops from ms rows to ~2 CH + 32 steps (cfg3's
    // 129-row lines: 5 + 32 + 5; cfg5's 1026-row lines: 33 + 32 + 33).
    // The scan reassociates rounding only; P^-1 stays a fixed linear map
    // (a preconditioner -- the CG's true residual is checked on exit).
    auto line_solve_scan = [&](double* y) {
        const int warp = tid >> 5, lane = tid & 31;
        const int gw = rank * (FDL_THREADS / 32) + warp, GW = K * (FDL_THREADS / 32);
        const int CH = (ms + 31) >> 5;
        const int i0 = min(ms, lane * CH), i1 = min(ms, i0 + CH);
        for (int L = gw; L < nlines; L += GW) {
            const double* F = Fac + (int64_t)L * ms * P1;
            double* yl = y + (int64_t)L * ms;
            double M[PL][PL], v[PL], S[PL];
            auto compose = [&](const double* a, double bd) {   // (M, v) <- A_i (M, v)
                double r0[PL], v0 = bd;
#pragma unroll
                for (int j = 0; j < PL; ++j) {
                    double acc = 0.0;
#pragma unroll
                    for (int k = 0; k < PL; ++k) acc = fma(a[k], M[k][j], acc);
                    r0[j] = acc;
                }
#pragma unroll
                for (int k = 0; k < PL; ++k) v0 = fma(a[k], v[k], v0);
#pragma unroll
                for (int r = PL - 1; r >= 1; --r) {
                    v[r] = v[r - 1];
#pragma unroll
                    for (int j = 0; j < PL; ++j) M[r][j] = M[r - 1][j];
                }
#pragma unroll
                for (int j = 0; j < PL; ++j) M[0][j] = r0[j];
                v[0] = v0;
            };
            auto reset = [&]() {
#pragma unroll
                for (int r = 0; r < PL; ++r) {
                    v[r] = 0.0;
                    S[r] = 0.0;
#pragma unroll
                    for (int j = 0; j < PL; ++j) M[r][j] = r == j ? 1.0 : 0.0;
                }
            };
            auto chain = [&](int from, int step) {   // lane from -> from + step -> ...
                for (int l = from; l + step >= 0 && l + step < 32; l += step) {
                    double E[PL];
#pragma unroll
                    for (int r = 0; r < PL; ++r) {
                        double acc = v[r];
#pragma unroll
                        for (int k = 0; k < PL; ++k) acc = fma(M[r][k], S[k], acc);
                        E[r] = acc;
                    }
#pragma unroll
                    for (int r = 0; r < PL; ++r) {
                        const double e = __shfl_sync(0xffffffffu, E[r], l);
                        if (lane == l + step) S[r] = e;
                    }
                }
            };
            // forward: y(i) = (y(i) - sum_k F(i, i-k) y(i-k)) / F(i, i); S[k] = y(i-k)
            reset();
            for (int i = i0; i < i1; ++i) {
                const double d = F[(int64_t)i * P1];
                double a[PL];
#pragma unroll
                for (int k = 0; k < PL; ++k) a[k] = (k < p && k < i) ? -d * F[(int64_t)i * P1 + k + 1] : 0.0;
                compose(a, d * yl[i]);
            }
            chain(0, 1);
            for (int i = i0; i < i1; ++i) {
                double sv = yl[i];
#pragma unroll
                for (int k = PL - 1; k >= 0; --k)
                    if (k < p && k < i) sv -= F[(int64_t)i * P1 + k + 1] * S[k];
                sv *= F[(int64_t)i * P1];
#pragma unroll
                for (int r = PL - 1; r >= 1; --r) S[r] = S[r - 1];
                S[0] = sv;
                yl[i] = sv;
            }
            __syncwarp();
            // backward: x(i) = (y(i) - sum_k F(i+k, i) x(i+k)) / F(i, i); S[k] = x(i+k)
            reset();
            for (int i = i1 - 1; i >= i0; --i) {
                const double d = F[(int64_t)i * P1];
                double a[PL];
#pragma unroll
                for (int k = 0; k < PL; ++k)
                    a[k] = (k < p && i + k + 1 < ms) ? -d * F[(int64_t)(i + k + 1) * P1 + k + 1] : 0.0;
                compose(a, d * yl[i]);
            }
            chain(31, -1);
            for (int i = i1 - 1; i >= i0; --i) {
                double sv = yl[i];
#pragma unroll
                for (int k = PL - 1; k >= 0; --k)
                    if (k < p && i + k + 1 < ms) sv -= F[(int64_t)(i + k + 1) * P1 + k + 1] * S[k];
                sv *= F[(int64_t)i * P1];
#pragma unroll
                for (int r = PL - 1; r >= 1; --r) S[r] = S[r - 1];
                S[0] = sv;
                yl[i] = sv;
            }
            __syncwarp();
        }
        cluster.sync();
    };
    // serial variant (degree 4, and lines enough to fill the cluster's warps):
    // ONE WARP per line, the lanes stage 32 factor rows
    // (and y) into shared memory -- the next 32 already in flight in
    // registers -- while lane 0 runs the serial recurrence from shared memory
    // with the last p results (forward) / the p pending column sums
    // (backward, column-oriented) in registers
    auto line_solve_serial = [&](double* y) {
        const int warp = tid >> 5, lane = tid & 31;
        const int gw = rank * (FDL_THREADS / 32) + warp, GW = K * (FDL_THREADS / 32);
        double* sF = lsF[warp];
        double* sy = lsy[warp];
        const int nch = (ms + 31) / 32;
        for (int L = gw; L < nlines; L += GW) {
            const double* F = Fac + (int64_t)L * ms * P1;
            double* yl = y + (int64_t)L * ms;
            double rf[PM + 1], ry = 0.0;
            auto ld = [&](int i0) {
                const int i = i0 + lane;
#pragma unroll
                for (int k = 0; k <= PM; ++k) rf[k] = (i < ms && k <= p) ? F[(int64_t)i * P1 + k] : 0.0;
                ry = i < ms ? yl[i] : 0.0;
            };
            // forward: y(i) = (y(i) - sum_k F(i, i-k) y(i-k)) / F(i, i)
            double yw[PM];
#pragma unroll
            for (int k = 0; k < PM; ++k) yw[k] = 0.0;
            ld(0);
            for (int ch = 0; ch < nch; ++ch) {
                const int i0 = ch * 32, n = min(32, ms - i0);
#pragma unroll
                for (int k = 0; k <= PM; ++k) sF[lane * (PM + 1) + k] = rf[k];
                sy[lane] = ry;
                __syncwarp();
                if (ch + 1 < nch) ld(i0 + 32);
                if (lane == 0) {
                    for (int ii = 0; ii < n; ++ii) {
                        const int i = i0 + ii;
                        double sv = sy[ii];
#pragma unroll
                        for (int k = PM; k >= 1; --k)
                            if (k <= p && k <= i) sv -= sF[ii * (PM + 1) + k] * yw[k - 1];
                        sv *= sF[ii * (PM + 1)];
                        sy[ii] = sv;
#pragma unroll
                        for (int d = PM - 1; d >= 1; --d) yw[d] = yw[d - 1];
                        yw[0] = sv;
                    }
                }
                __syncwarp();
                if (lane < n) yl[i0 + lane] = sy[lane];
                __syncwarp();
            }
            // backward, column-oriented: acw[d] = pending sum_k F(i+k, i) y(i+k)
            // of row i - d
            double acw[PM];
#pragma unroll
            for (int k = 0; k < PM; ++k) acw[k] = 0.0;
            ld((nch - 1) * 32);
            for (int ch = nch - 1; ch >= 0; --ch) {
                const int i0 = ch * 32, n = min(32, ms - i0);
#pragma unroll
                for (int k = 0; k <= PM; ++k) sF[lane * (PM + 1) + k] = rf[k];
                sy[lane] = ry;
                __syncwarp();
                if (ch > 0) ld(i0 - 32);
                if (lane == 0) {
                    for (int ii = n - 1; ii >= 0; --ii) {
                        const double sv = (sy[ii] - acw[0]) * sF[ii * (PM + 1)];
                        sy[ii] = sv;
#pragma unroll
                        for (int d = 0; d < PM - 1; ++d) acw[d] = acw[d + 1];
                        acw[PM - 1] = 0.0;
#pragma unroll
                        for (int k = 1; k <= PM; ++k)
                            if (k <= p) acw[k - 1] += sF[ii * (PM + 1) + k] * sv;
                    }
                }
                __syncwarp();
                if (lane < n) yl[i0 + lane] = sy[lane];
                __syncwarp();
            }
        }
        cluster.sync();
    };
    // the scan when the lines leave most of the cluster's warps idle (2-D:
    // a few long lines, the serial chain is the critical path); with lines
    // for every warp the serial recurrence is cheaper (no second pass over
    // the factors).  Degree 4: serial only (the scan's 4 x 4 state spills).
    auto line_solve = [&](double* y) {
        if constexpr (PL >= 4) line_solve_serial(y);
        else if (nlines < K * (FDL_THREADS / 32)) line_solve_scan(y);
        else line_solve_serial(y);
    };
    auto precond = [&]() {   // z = P^-1 r
        if constexpr (D == 3) {
            mode(r, t, 0, true);
            mode(t, z, 1, true);
            line_solve(z);
            mode(z, t, 1, false);
            mode(t, z, 0, false);
        } else if constexpr (D == 2) {
            mode(r, t, 0, true);
            line_solve(t);
            mode(t, z, 0, false);
        } else {
            for (int i = gt; i < R; i += GT) z[i] = r[i];
            cluster.sync();
            line_solve(z);
        }
    };
    constexpr int UNR1 = (FUSED && SGIGA_FDL_FUSED_UNR1) ? FDL_UNR2 : FDL_UNR;
    auto spmv = [&](const double* v, double* out) {   // out = A v (v halo-padded)
        for (int row = gt; row < R; row += GT) {
            const int rb = fd_row_base(C, D, row);
            double y0 = 0.0, y1 = 0.0;
            int tt = 0;
            for (; tt + UNR1 - 1 < NS; tt += UNR1) {   // UNR1 independent stencil loads in flight
                double vv[UNR1];
#pragma unroll
                for (int u = 0; u < UNR1; ++u) vv[u] = __ldg(val + (size_t)(tt + u) * R + row);
#pragma unroll
                for (int u = 0; u < UNR1; u += 2) {
                    y0 += vv[u] * v[rb + offs[tt + u]];
                    y1 += vv[u + 1] * v[rb + offs[tt + u + 1]];
                }
            }
            for (; tt < NS; ++tt) y0 += __ldg(val + (size_t)tt * R + row) * v[rb + offs[tt]];
            out[row] = y0 + y1;
        }
        cluster.sync();
    };
    // out = A v and out2 = A u in ONE sweep of the stored stencil (the sweep
    // is bound by the stencil's HBM read; the second gather hits L1/L2).
    // out is accumulated exactly as in spmv (same operations and order).
    // absl accumulates sum_rows (|A| |u|)_row^2 (rounding bound of the fused
    // true residual, see below).
    double absl = 0.0;
    auto spmv2 = [&](const double* v, const double* u, double* out, double* out2) {
        absl = 0.0;
        for (int row = gt; row < R; row += GT) {
            const int rb = fd_row_base(C, D, row);
            double y0 = 0.0, y1 = 0.0, w0 = 0.0, w1 = 0.0, s0 = 0.0, s1 = 0.0;
            int tt = 0;
            for (; tt + FDL_UNR2 - 1 < NS; tt += FDL_UNR2) {
                double vv[FDL_UNR2];
#pragma unroll
                for (int k = 0; k < FDL_UNR2; ++k) vv[k] = __ldg(val + (size_t)(tt + k) * R + row);
#pragma unroll
                for (int k = 0; k < FDL_UNR2; k += 2) {
                    const int c0 = rb + offs[tt + k], c1 = rb + offs[tt + k + 1];
                    y0 += vv[k] * v[c0];
                    y1 += vv[k + 1] * v[c1];
                    const double u0 = u[c0], u1 = u[c1];
                    w0 += vv[k] * u0;
                    w1 += vv[k + 1] * u1;
                    s0 += fabs(vv[k]) * fabs(u0);
                    s1 += fabs(vv[k + 1]) * fabs(u1);
                }
            }
            for (; tt < NS; ++tt) {
                const double a = __ldg(val + (size_t)tt * R + row);
                const int c0 = rb + offs[tt];
                y0 += a * v[c0];
                w0 += a * u[c0];
                s0 += fabs(a) * fabs(u[c0]);
            }
            out[row] = y0 + y1;
            out2[row] = w0 + w1;
            absl += (s0 + s1) * (s0 + s1);
        }
        cluster.sync();
    };

    double bbl = 0.0;
    for (int i = gt; i < R; i += GT) {
        const double bi = b[i];
        x[i] = 0.0;
        r[i] = bi;
        bbl += bi * bi;
    }
    const double bb = csum(bbl);
    // True residual ||b - A x|| / ||b|| (linsolve.py:49-53).
    // FUSED (the launcher sets it when the FD preconditioner is the exact
    // inverse up to rounding -- Kronecker box systems, 1-3 iterations): no
    // sweep of its own.  From the second iteration on, the iteration's sweep
    // multiplies the stencil with BOTH p_k and x_k (spmv2), and after x_{k+1} =
    // x_k + alpha p_k the residual is taken as b - (A x_k + alpha A p_k) -- two
    // direct products with the stored stencil, not the CG recurrence (x_0 = 0:
    // in the first iteration A x_1 = alpha A p_0 is the recurrence's own
    // product).  The iterates are bitwise those of the plain loop.  What this
    // form cannot see is the rounding of the last update x_{k+1} = fl(x_k +
    // alpha p_k), |delta| <= u |x_{k+1}|: its image A delta is bounded by
    // u || |A| |x_k| ||_2 (first order; the same sweep accumulates |A| |x_k|),
    // and the bound is ADDED to the reported residual -- relres is an upper
    // bound of the residual of the stored x.  Otherwise (tens of iterations)
    // one separate sweep after the loop is cheaper.
    int it = 0, conv = (bb == 0.0);
    double eel = 0.0;
    if (!conv) {
        precond();
        double rzl = 0.0;
        for (int i = gt; i < R; i += GT) { pp[i] = z[i]; rzl += r[i] * z[i]; }
        double rz = csum(rzl);
        while (it < maxit) {
            if (!FUSED || it == 0) spmv(pp, qq);
            else spmv2(pp, x, qq, t);   // t = A x_k (the preconditioner's scratch is free here)
            double pql = 0.0;
            for (int i = gt; i < R; i += GT) pql += pp[i] * qq[i];
            const double alpha = rz / csum(pql);
            double rrl = 0.0;
            eel = 0.0;
            for (int i = gt; i < R; i += GT) {
                const double xi = x[i] + alpha * pp[i];
                x[i] = xi;
                const double ri = r[i] - alpha * qq[i];
                r[i] = ri;
                rrl += ri * ri;
                if constexpr (FUSED) {
                    const double e = it == 0 ? ri : (b[i] - t[i]) - alpha * qq[i];
                    eel += isfinite(xi) ? e * e : __longlong_as_double(0x7ff8000000000000ULL);
                }
            }
            const double rr = csum(rrl);
            ++it;
            if (rr <= rtol2 * bb) { conv = 1; break; }
            precond();
            double rzl2 = 0.0;
            for (int i = gt; i < R; i += GT) rzl2 += r[i] * z[i];
            const double rzn = csum(rzl2);
            const double beta = rzn / rz;
            rz = rzn;
            for (int i = gt; i < R; i += GT) pp[i] = z[i] + beta * pp[i];
            cluster.sync();
        }
    }
    if constexpr (!FUSED) {   // x is copied into the halo-padded p buffer for the gather
        for (int i = gt; i < R; i += GT) pp[i] = x[i];
        cluster.sync();
        spmv(pp, qq);
        eel = 0.0;
        for (int i = gt; i < R; i += GT) {
            const double e = qq[i] - b[i];
            eel += isfinite(x[i]) ? e * e : __longlong_as_double(0x7ff8000000000000ULL);
        }
    }
    const double ee = csum(eel);
    double rbound = 0.0;   // u || |A| |x_k| ||_2, u = 2^-53
    if constexpr (FUSED) rbound = 0x1p-53 * sqrt(csum(it > 1 ? absl : 0.0));
    if (gt == 0) {
        st[c].it = it;
        st[c].conv = conv;
        st[c].active = 0;
        st[c].bb = bb;
        relres[c] = bb > 0.0 ? (FUSED ? (sqrt(ee) + rbound) / sqrt(bb) : sqrt(ee / bb)) : (ee == 0.0 ? 0.0 : ee);
    }
    // full C-order coefficients (x complete: the last cluster barrier is in csum)
    fd_expand<D>(C, x, coef, gt, GT);
    cluster.sync();   // no CTA exits while others may still read its cpart
}

cudaError_t launch_pcg_fdl(Handle* h, double rtol, int maxit) {
    const int n = (int)h->fdl_comps.size();
    if (n == 0) return cudaSuccess;
    // cluster CTAs per component: a constant, so a component's reduction
    // order (and its bits) never depends on which other components share
    // the batch (a rank's subset of a plan computes what the full plan does)
    const int K = 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n * K));
    cfg.blockDim = dim3(FDL_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const double rt2 = rtol * rtol;
    cudaError_t e;
#define LAUNCH_FDL(DD)                                                                                       \
    e = cudaLaunchKernelEx(&cfg, k_pcg_fdl<DD, PP, FZ>, (const CompInfo*)h->d_comps, (const int*)h->d_fdl_list, \
                           (const int*)h->d_slotoff, (const double*)h->d_stencil, (const double*)h->d_rhs,  \
                           h->p, (const int64_t*)h->d_fd_uoff, (const double*)h->d_fdU,                    \
                           (const double*)h->d_ck, (const int64_t*)h->d_fdl_off, (const double*)h->d_fdl,  \
                           h->d_x, h->d_r, h->d_z, h->d_p, h->d_q, h->d_q2, h->d_cg, h->d_relres, rt2, maxit, \
                           h->d_coef)
#define LAUNCH_FDL_P(DD)                                 \
    switch (h->p) {                                      \
        case 1: { constexpr int PP = 1; LAUNCH_FDL(DD); } break; \
        case 2: { constexpr int PP = 2; LAUNCH_FDL(DD); } break; \
        case 3: { constexpr int PP = 3; LAUNCH_FDL(DD); } break; \
        default: { constexpr int PP = 4; LAUNCH_FDL(DD); } break; \
    }
    // Kronecker box systems (3-D): exact FD inverse, fused true residual
    if (h->d == 1) { constexpr bool FZ = false; LAUNCH_FDL_P(1); }
    else if (h->d == 2) { constexpr bool FZ = false; LAUNCH_FDL_P(2); }
    else if (h->box_state > 0) { constexpr bool FZ = true; LAUNCH_FDL_P(3); }
    else { constexpr bool FZ = false; LAUNCH_FDL_P(3); }
#undef LAUNCH_FDL_P
#undef LAUNCH_FDL
    h->launches[1]++;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// side-stream kernels are launched with the device's highest scheduling
// priority as a launch attribute (kept in captured graph nodes, unlike the
// stream's priority): their few CTAs get SMs as soon as assembly CTAs retire
template <typename... KArgs, typename... Args>
static cudaError_t launch_hi(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = hi;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// FD set-up after the metric (stream s, forked from the main stream after
// k_metric, joined before the solve): c_k of every FD / line-FD component,
// then the line-FD stream-axis bands and per-line factors
cudaError_t launch_fd_box_scale(Handle* h, cudaStream_t s);

cudaError_t launch_fd_setup(Handle* h, cudaStream_t s) {
    const int nf = (int)h->fd_comps.size(), nl = (int)h->fdl_comps.size(), ng = (int)h->fdg_comps.size();
    const bool box = h->box_state > 0;   // Kronecker assembly: c_k in closed form, no metric sums
    if (box && nf + nl + ng > 0) {
        cudaError_t e = launch_fd_box_scale(h, s);
        if (e != cudaSuccess) return e;
    }
    if (ng > 0 && !box) {   // c_k of the whole-GPU FD components: chunked two-level sum
        const dim3 gp(FDG_SCALE_CHUNKS, (unsigned)ng, (unsigned)h->d);
#define LAUNCH_SCALE_G(DD)                                                                                       \
    launch_hi(k_fd_metric_scale_part<DD>, gp, dim3(256), 0, s, (const CompInfo*)h->d_comps, (const int*)h->d_fdg_list, \
              (const double*)h->d_G, h->d_fdg_ckpart)
        if (h->d == 1) { LAUNCH_SCALE_G(1); }
        else if (h->d == 2) { LAUNCH_SCALE_G(2); }
        else { LAUNCH_SCALE_G(3); }
#undef LAUNCH_SCALE_G
        launch_hi(k_fd_metric_scale_fin, dim3((unsigned)ng, (unsigned)h->d), dim3(256), 0, s,
                  (const int*)h->d_fdg_list, (const double*)h->d_fdg_ckpart, h->d_ck);
        h->launches[0] += 2;
    }
    if (nf + nl == 0) return cudaGetLastError();
    const dim3 g1((unsigned)(nf + nl), (unsigned)h->d);
    if (!box) {
#define LAUNCH_SCALE(DD)                                                                              \
    launch_hi(k_fd_metric_scale<DD>, g1, dim3(256), 0, s, h->d_comps, h->d_fdlist, nf, h->d_fdl_list, h->d_G, h->d_ck)
    if (h->d == 1) { LAUNCH_SCALE(1); }
    else if (h->d == 2) { LAUNCH_SCALE(2); }
    else { LAUNCH_SCALE(3); }
#undef LAUNCH_SCALE
    h->launches[0]++;
    }
    if (nl == 0) return cudaGetLastError();
    int maxlines = 1;
    for (int c : h->fdl_comps) {
        const CompInfo& C = h->comps[c];
        int lines = 1;
        for (int o = 0; o < h->d - 1; ++o) lines *= C.m[C.ax[o]];
        maxlines = std::max(maxlines, lines);
    }
    const dim3 g3((unsigned)((maxlines + 63) / 64), (unsigned)nl);
    int maxms = 1;
    for (int c : h->fdl_comps) maxms = std::max(maxms, h->comps[c].m[h->comps[c].ax[h->d - 1]]);
    // staged only while small: a large staging buffer would keep the 3-D
    // assembly's CTAs (this kernel runs beside it on the side stream) off
    // the SM for the factor's duration
    const size_t fsm0 = sizeof(double) * 2 * (size_t)maxms * (h->p + 1);
    const int staged = fsm0 <= 24 * 1024;
    const size_t fsm = staged ? fsm0 : 0;
#define LAUNCH_FACT(DD)                                                                                     \
    launch_hi(k_fdl_bands<DD>, dim3((unsigned)nl), dim3(256), 0, s, h->d_comps, h->d_fdl_list, h->d_tabs,   \
              h->d_tabvals, h->d_qw, h->p, h->mu, h->q, h->d_fdl_off, h->d_fdl);                          \
    cudaFuncSetAttribute(k_fdl_factor<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);         \
    launch_hi(k_fdl_factor<DD>, g3, dim3(64), fsm, s, h->d_comps, h->d_fdl_list, h->p, h->d_fd_loff, h->d_fdL, \
              h->d_ck, h->d_fdl_off, h->d_fdl, staged)
    if (h->d == 1) { LAUNCH_FACT(1); }
    else if (h->d == 2) { LAUNCH_FACT(2); }
    else { LAUNCH_FACT(3); }
#undef LAUNCH_FACT
    h->launches[0] += 2;
    return cudaGetLastError();
}

size_t fd_eigen_smem() { return sizeof(double) * (3 * FD_MMAX * FD_LD + FD_TAB_MAX); }

size_t fd_comp_smem(const CompInfo& C, int d) {
    int64_t u = 0, l = 0;
    for (int k = 0; k < d; ++k) { u += (int64_t)C.m[k] * C.m[k]; l += C.m[k]; }
    return sizeof(double) * (size_t)(6 * C.rows + 2 * C.halo + u + l + FD_THREADS) + sizeof(int) * (size_t)(C.nslots + 1);
}

cudaError_t launch_fd_eigen(Handle* h, cudaStream_t s) {
    if (h->fd_uniq.empty()) return cudaSuccess;
    const size_t smem = fd_eigen_smem();
    cudaError_t e = cudaFuncSetAttribute(k_fd_eigen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int nu = (int)h->fd_uniq.size();
    long long* prof = nullptr;
    if (h->opt.fd_profile) {   // per-CTA phase cycles (probe only)
        if ((e = cudaMalloc(&prof, sizeof(long long) * 8 * nu)) != cudaSuccess) return e;
        cudaMemsetAsync(prof, 0, sizeof(long long) * 8 * nu, s);
    }
    if ((e = launch_hi(k_fd_eigen, dim3((unsigned)nu), dim3(EIG_THREADS), smem, s, h->d_tabs, h->d_fd_uniq,
                       h->d_fd_uoff, h->d_fd_loff, h->d_tabvals, h->d_qw, h->p, h->mu, h->q, h->d_fdU, h->d_fdL,
                       prof)) != cudaSuccess)
        return e;
    h->launches[0]++;
    if (prof) {
        std::vector<long long> t(8 * nu);
        cudaMemcpyAsync(t.data(), prof, sizeof(long long) * t.size(), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        for (int b = 0; b < nu; ++b)
            fprintf(stderr, "fd-eigen cta %d m=%lld sweeps=%lld cycles: build=%lld chol=%lld C=%lld jacobi=%lld upd=%lld rot=%lld\n",
                    b, t[8 * b + 6], t[8 * b + 5], t[8 * b], t[8 * b + 1], t[8 * b + 2], t[8 * b + 3], t[8 * b + 4], t[8 * b + 7]);
        cudaFree(prof);
    }
    return cudaGetLastError();
}

cudaError_t launch_pcg_fd(Handle* h, double rtol, int maxit, cudaStream_t stream) {
    if (!stream) stream = h->stream;
    const int n = (int)h->fd_comps.size();
    if (n == 0) return cudaSuccess;
    size_t smem = 0;
    for (int c : h->fd_comps) smem = std::max(smem, fd_comp_smem(h->comps[c], h->d));
    cudaError_t e;
    long long* prof = nullptr;
    if (h->opt.fd_profile) {   // per-CTA phase cycles (probe only)
        if ((e = cudaMalloc(&prof, sizeof(long long) * 8 * n)) != cudaSuccess) return e;
        cudaMemsetAsync(prof, 0, sizeof(long long) * 8 * n, stream);
    }
#define LAUNCH_FD(DD)                                                                                 \
    e = cudaFuncSetAttribute(k_pcg_fd<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
    if (e != cudaSuccess) return e;                                                                   \
    k_pcg_fd<DD><<<(unsigned)n, FD_THREADS, smem, stream>>>(                                       \
        h->d_comps, h->d_fdlist, h->d_slotoff, h->d_stencil, h->d_rhs, h->d_G, h->d_fd_uoff,          \
        h->d_fd_loff, h->d_fdU, h->d_fdL, h->d_ck, h->d_x, h->d_coef, h->d_cg, h->d_relres, rtol * rtol, maxit, prof)
    if (h->d == 1) { LAUNCH_FD(1); }
    else if (h->d == 2) { LAUNCH_FD(2); }
    else { LAUNCH_FD(3); }
#undef LAUNCH_FD
    h->launches[1]++;
    if (prof) {
        std::vector<long long> t(8 * n);
        cudaMemcpyAsync(t.data(), prof, sizeof(long long) * t.size(), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        for (int b = 0; b < n; ++b)
            fprintf(stderr, "pcg-fd cta %d R=%lld NS=%lld cycles: prologue=%lld b=%lld precond=%lld spmv1=%lld "
                    "loop=%lld spmv2=%lld end=%lld\n", b, t[8 * b + 7] / 1000, t[8 * b + 7] % 1000, t[8 * b],
                    t[8 * b + 1], t[8 * b + 2], t[8 * b + 3], t[8 * b + 4], t[8 * b + 5], t[8 * b + 6]);
        cudaFree(prof);
    }
    return cudaGetLastError();
}

}  // namespace sgiga
