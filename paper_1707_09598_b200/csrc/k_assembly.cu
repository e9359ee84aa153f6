// k_assembly.cu -- kernel 2: sum-factorised stiffness + load assembly
// straight into the per-component stencil layout (no COO/CSR, no atomics,
// deterministic).
//
// Reference: assembly._assemble_full (assembly.py:264-354) with the element
// kernel _kernels/_compiled.pyx:17-90, interior extraction assembly.py:389.
//
// Formulation.  For interior row i and column j = i + o of component c,
//   A(i,j) = sum_{m,n} sum_{quad pts x} G_mn(x) prod_k T^k_{t_k(m,n)}(i_k, j_k, x_k)
// where G = det*w*J^-1 J^-T is precomputed per quadrature point (k_metric)
// and T^k_t is the product of 1-D basis values/derivatives of i_k and j_k
// (t_k = 2*[m==k] + [n==k]).  Instead of the element-by-element local
// matrices of the reference, the contraction runs over the *global*
// quadrature grid one axis at a time: a CTA owns a pencil of rows (fixed
// (i_a, i_b) along the two tile axes, a range of rows along the stream
// axis s) and streams over the quadrature planes x_s:
//   stage 1: contract axis b  S1[pair][x_a][s_b]
//   stage 2: contract axis a  S2[t_s][s_a][s_b]   (pairs grouped by t_s)
//   stage 3: rank-1 update of the P alive rows of the current element
//            along s into a ring of accumulators; completed rows are
//            flushed (several at once, coalesced along s) to the stencil.
// Per element this needs about D^2 q^3 P^2 + D^2 q^2 P^2 W + 4 q P^2 W^2
// FMAs instead of the reference's D^2 q^D P^{2D}.
#include "handle.cuh"

namespace sgiga {

constexpr int FLUSH_ROWS = 4;   // rows written per flush (32 B runs)
constexpr int ASM_THREADS = 256;

struct AxisWin {        // one tile axis of a pencil
    int present;        // 0 = virtual axis (D < 3 / D < 2)
    int tab;            // TabInfo index
    int i;              // full function index of the pencil row
    int e0, ne;         // support elements [e0, e0+ne)
    int N;              // window quadrature points = ne*q
    int S;              // slots
    int absm;
    int64_t qs;         // qp storage stride
    int64_t rs, ss;     // row / slot strides
};

__device__ __forceinline__ double basis_at(const double* __restrict__ vals, const TabInfo& T,
                                           int P, int q, int mu, int fn, int e, int g, int der) {
    int loc = fn - e * mu;
    if (loc < 0 || loc >= P) return 0.0;
    int64_t nq = (int64_t)T.nel * q;
    return vals[T.val_off + (der ? nq * P : 0) + ((int64_t)e * q + g) * P + loc];
}

template <int D>
__global__ void __launch_bounds__(ASM_THREADS)
k_assemble_pencil(const CompInfo* __restrict__ comps, const TabInfo* __restrict__ tabs,
                  const Pencil* __restrict__ pencils, const double* __restrict__ vals, int p,
                  int mu, int q, const double* __restrict__ Gbuf, double* __restrict__ stencil,
                  double* __restrict__ rhs, double* __restrict__ dinv) {
    extern __shared__ double sm[];
    const Pencil pc = pencils[blockIdx.x];
    const CompInfo& C = comps[pc.comp];
    const int P = p + 1, tid = threadIdx.x, nth = blockDim.x;
    const int s = C.ax[D - 1];
    const TabInfo Ts = tabs[C.tab[s]];

    // ---- tile-axis windows (virtual axes have N = S = 1) ----------------
    AxisWin A, B;
    auto setup = [&](AxisWin& W, int present, int k, int i) {
        W.present = present;
        if (!present) {
            W.tab = 0; W.i = 0; W.e0 = 0; W.ne = 1; W.N = 1; W.S = 1; W.absm = 1;
            W.qs = 0; W.rs = 0; W.ss = 0;
            return;
        }
        const TabInfo& T = tabs[C.tab[k]];
        W.tab = C.tab[k];
        W.i = i;
        int ef = (i - p) <= 0 ? 0 : (i - p + mu - 1) / mu;
        int el = i / mu;
        if (el > T.nel - 1) el = T.nel - 1;
        W.e0 = ef;
        W.ne = el - ef + 1;
        W.N = W.ne * q;
        W.S = C.S[k];
        W.absm = C.absm[k];
        W.qs = C.qs[k];
        W.rs = C.rs[k];
        W.ss = C.ss[k];
    };
    setup(A, D >= 2, D >= 2 ? C.ax[D - 2] : 0, pc.ia);
    setup(B, D >= 3, D >= 3 ? C.ax[D - 3] : 0, pc.ib);
    const int Ss = C.S[s];
    const int SAB = A.S * B.S;
    const int RING = FLUSH_ROWS + P - 1;
    const int nG = D * (D + 1) / 2 + 1;
    const int NPAIR = D * D;

    // ---- shared memory carve-up -------------------------------------------
    double* Ta = sm;                          // [4][A.S][A.N]
    double* Tb = Ta + 4 * A.S * A.N;          // [4][B.S][B.N]
    double* phiA = Tb + 4 * B.S * B.N;        // [A.N]  value of i_a
    double* phiB = phiA + A.N;                // [B.N]
    double* Gw = phiB + B.N;                  // [nG][A.N][B.N]
    double* S1 = Gw + nG * A.N * B.N;         // [NPAIR][A.N][B.S]
    double* SL1 = S1 + NPAIR * A.N * B.S;     // [A.N]
    double* S2 = SL1 + A.N;                   // [4][SAB] + 1 (load)
    double* Bs = S2 + 4 * SAB + 1;            // [2][q][P] stream element tables
    double* Acc = Bs + 2 * q * P;             // [RING][Ss][SAB]
    double* AccL = Acc + RING * Ss * SAB;     // [RING]

    // ---- 1-D pair tables of the tile axes --------------------------------
    auto build_T = [&](const AxisWin& W, double* T, double* phi) {
        if (!W.present) {
            if (tid == 0) { T[0] = 1.0; T[1] = 0.0; T[2] = 0.0; T[3] = 0.0; phi[0] = 1.0; }
            return;
        }
        const TabInfo& TT = tabs[W.tab];
        int tot = 4 * W.S * W.N;
        for (int idx = tid; idx < tot; idx += nth) {
            int x = idx % W.N, rest = idx / W.N;
            int sl = rest % W.S, t = rest / W.S;
            int e = W.e0 + x / q, g = x % q;
            int j = W.absm ? sl + 1 : W.i + sl - p;     // column function
            double v = 0.0;
            if (j >= 1 && j <= TT.n - 2) {
                double a = basis_at(vals, TT, P, q, mu, W.i, e, g, t >> 1);
                double b = basis_at(vals, TT, P, q, mu, j, e, g, t & 1);
                v = a * b;
            }
            T[idx] = v;
        }
        for (int x = tid; x < W.N; x += nth)
            phi[x] = basis_at(vals, TT, P, q, mu, W.i, W.e0 + x / q, x % q, 0);
    };
    build_T(A, Ta, phiA);
    build_T(B, Tb, phiB);
    for (int idx = tid; idx < RING * Ss * SAB; idx += nth) Acc[idx] = 0.0;
    for (int idx = tid; idx < RING; idx += nth) AccL[idx] = 0.0;
    __syncthreads();

    // pair tables (compile-time D)
    int g_of[D * D], ts_of[D * D], ta_of[D * D], tb_of[D * D];
    {
        int ka = D >= 2 ? C.ax[D - 2] : -1, kb = D >= 3 ? C.ax[D - 3] : -1;
#pragma unroll
        for (int m = 0; m < D; ++m)
#pragma unroll
            for (int n = 0; n < D; ++n) {
                int pr = m * D + n;
                g_of[pr] = sym_index(D, m, n);
                ts_of[pr] = 2 * (m == s) + (n == s);
                ta_of[pr] = 2 * (m == ka) + (n == ka);
                tb_of[pr] = 2 * (m == kb) + (n == kb);
            }
    }

    const int n_s = Ts.n;
    const int r0 = pc.r0, r1 = pc.r1;
    int e_first = (r0 - p) <= 0 ? 0 : (r0 - p + mu - 1) / mu;
    int e_last = (r1 - 1) / mu;
    if (e_last > Ts.nel - 1) e_last = Ts.nel - 1;
    int pend_lo = r0;
    const double* Gc = Gbuf + C.qp_off;
    const int64_t nqp = C.nqp;
    const int64_t qa0 = (int64_t)A.e0 * q, qb0 = (int64_t)B.e0 * q;
    const int64_t row_base = (A.present ? (A.i - 1) * A.rs : 0) + (B.present ? (B.i - 1) * B.rs : 0);
    const int64_t slot_base_rows = C.rows;

    for (int e = e_first; e <= e_last; ++e) {
        // stream-axis element tables
        for (int idx = tid; idx < 2 * q * P; idx += nth) {
            int der = idx / (q * P), rem = idx % (q * P);
            int g = rem / P, j = rem % P;
            int64_t nq = (int64_t)Ts.nel * q;
            Bs[idx] = vals[Ts.val_off + (der ? nq * P : 0) + ((int64_t)e * q + g) * P + j];
        }
        const int off_e = e * mu;
        for (int g = 0; g < q; ++g) {
            const int64_t Qs = (int64_t)e * q + g;
            // ---- load the metric plane window ------------------------------
            const int plane = A.N * B.N;
            for (int idx = tid; idx < nG * plane; idx += nth) {
                int c = idx / plane, rem = idx % plane;
                int xa = rem / B.N, xb = rem % B.N;
                int64_t lin = Qs * C.qs[s] + (qa0 + xa) * A.qs + (qb0 + xb) * B.qs;
                Gw[idx] = Gc[(int64_t)c * nqp + lin];
            }
            __syncthreads();
            // ---- stage 1: contract axis b ----------------------------------
            {
                int tot = NPAIR * A.N * B.S;
                for (int idx = tid; idx < tot; idx += nth) {
                    int sb = idx % B.S, rest = idx / B.S;
                    int xa = rest % A.N, pr = rest / A.N;
                    const double* gp = Gw + (g_of[pr] * A.N + xa) * B.N;
                    const double* tp = Tb + (tb_of[pr] * B.S + sb) * B.N;
                    double acc = 0.0;
                    for (int xb = 0; xb < B.N; ++xb) acc += gp[xb] * tp[xb];
                    S1[idx] = acc;
                }
                for (int xa = tid; xa < A.N; xa += nth) {
                    const double* gp = Gw + ((nG - 1) * A.N + xa) * B.N;
                    double acc = 0.0;
                    for (int xb = 0; xb < B.N; ++xb) acc += gp[xb] * phiB[xb];
                    SL1[xa] = acc;
                }
            }
            __syncthreads();
            // ---- stage 2: contract axis a, group pairs by stream type -----
            {
                int tot = 4 * SAB;
                for (int idx = tid; idx < tot; idx += nth) {
                    int sab = idx % SAB, ts = idx / SAB;
                    int sa = sab / B.S, sb = sab % B.S;
                    double acc = 0.0;
#pragma unroll
                    for (int pr = 0; pr < D * D; ++pr) {
                        if (ts_of[pr] != ts) continue;
                        const double* s1 = S1 + pr * A.N * B.S + sb;
                        const double* tp = Ta + (ta_of[pr] * A.S + sa) * A.N;
                        for (int xa = 0; xa < A.N; ++xa) acc += s1[xa * B.S] * tp[xa];
                    }
                    S2[idx] = acc;
                }
                if (tid == nth - 1) {
                    double acc = 0.0;
                    for (int xa = 0; xa < A.N; ++xa) acc += SL1[xa] * phiA[xa];
                    S2[4 * SAB] = acc;
                }
            }
            __syncthreads();
            // ---- stage 3: accumulate the alive rows of element e ----------
            {
                int tot = P * P * SAB;
                for (int idx = tid; idx < tot; idx += nth) {
                    int sab = idx % SAB, rest = idx / SAB;
                    int bl = rest % P, al = rest / P;
                    int i = off_e + al, j = off_e + bl;
                    if (i < r0 || i >= r1) continue;
                    if (j < 1 || j > n_s - 2) continue;
                    int os = C.absm[s] ? j - 1 : j - i + p;
                    double va = Bs[g * P + al], da = Bs[q * P + g * P + al];
                    double vb = Bs[g * P + bl], db = Bs[q * P + g * P + bl];
                    double v = va * vb * S2[sab] + va * db * S2[SAB + sab] +
                               da * vb * S2[2 * SAB + sab] + da * db * S2[3 * SAB + sab];
                    Acc[((i % RING) * Ss + os) * SAB + sab] += v;
                }
                for (int al = tid; al < P; al += nth) {
                    int i = off_e + al;
                    if (i < r0 || i >= r1) continue;
                    AccL[i % RING] += Bs[g * P + al] * S2[4 * SAB];
                }
            }
            __syncthreads();
        }
        // ---- flush completed rows ------------------------------------------
        int done_hi = (e == Ts.nel - 1) ? n_s : (e + 1) * mu;
        if (done_hi > r1) done_hi = r1;
        int npend = done_hi - pend_lo;
        if (npend > 0 && (npend >= FLUSH_ROWS || e == e_last)) {
            // rhs and D^-1 of the pending rows
            for (int t = tid; t < npend; t += nth) {
                int i = pend_lo + t;
                int64_t row = row_base + (int64_t)(i - 1) * C.rs[s];
                int os = C.absm[s] ? i - 1 : p;
                int sa = A.present ? (A.absm ? A.i - 1 : p) : 0;
                int sb = B.present ? (B.absm ? B.i - 1 : p) : 0;
                double dg = Acc[((i % RING) * Ss + os) * SAB + sa * B.S + sb];
                rhs[C.vec_off + row] = AccL[i % RING];
                dinv[C.vec_off + row] = 1.0 / dg;
                AccL[i % RING] = 0.0;
            }
            __syncthreads();
            int tot = npend * Ss * SAB;
            for (int idx = tid; idx < tot; idx += nth) {
                int t = idx % npend, sl = idx / npend;
                int sab = sl % SAB, os = sl / SAB;
                int sa = sab / B.S, sb = sab % B.S;
                int i = pend_lo + t;
                int64_t row = row_base + (int64_t)(i - 1) * C.rs[s];
                int64_t slot = (int64_t)os * C.ss[s] + sa * A.ss + sb * B.ss;
                double* a = &Acc[((i % RING) * Ss + os) * SAB + sab];
                stencil[C.mat_off + slot * slot_base_rows + row] = *a;
                *a = 0.0;
            }
            pend_lo = done_hi;
            __syncthreads();
        }
    }
}

size_t assembly_smem_bytes(const Handle* h) {
    int P = h->p + 1, q = h->q, W = 2 * h->p + 1, D = h->d;
    int NA = D >= 2 ? P * q : 1, NB = D >= 3 ? P * q : 1;
    int SA = D >= 2 ? W : 1, SB = D >= 3 ? W : 1, SS = W;
    int RING = FLUSH_ROWS + P - 1;
    int nG = D * (D + 1) / 2 + 1;
    size_t n = 4 * SA * NA + 4 * SB * NB + NA + NB + (size_t)nG * NA * NB + D * D * NA * SB + NA +
               4 * SA * SB + 1 + 2 * q * P + (size_t)RING * SS * SA * SB + RING;
    return n * sizeof(double);
}

bool launch_assembly_fast(Handle* h, cudaError_t* err, int npencils);
bool launch_assembly_2d(Handle* h, cudaError_t* err);
bool launch_assembly_tile(Handle* h, cudaError_t* err);
bool launch_assembly_box(Handle* h, cudaError_t* err);

cudaError_t launch_assembly(Handle* h) {
    int np = (int)h->pencils.size();
    if (np == 0) return cudaSuccess;
    cudaError_t fe = cudaSuccess;
    if (!h->force_generic_assembly && launch_assembly_2d(h, &fe))     // 2-D blocks, q = p+1
        return fe == cudaSuccess ? cudaGetLastError() : fe;
    h->asm_tiled = false;
    if (launch_assembly_box(h, &fe))   // axis-aligned box: Kronecker stiffness + factorised load
        return fe == cudaSuccess ? cudaGetLastError() : fe;
    if (!h->force_generic_assembly && launch_assembly_tile(h, &fe)) {   // 3-D tiles, q = p+1, p = 3, 4
        h->asm_tiled = true;
        if (fe != cudaSuccess) return fe;
        // the components below the tile threshold: one row per CTA
        if (h->n_pencils_other > 0 && launch_assembly_fast(h, &fe, h->n_pencils_other))
            return fe == cudaSuccess ? cudaGetLastError() : fe;
        return cudaGetLastError();
    }
    if (!h->force_generic_assembly && launch_assembly_fast(h, &fe, np))   // maximal regularity, q = p+1
        return fe == cudaSuccess ? cudaGetLastError() : fe;
    size_t smem = assembly_smem_bytes(h);
    cudaError_t e;
#define LAUNCH_ASM(DD)                                                                        \
    e = cudaFuncSetAttribute(k_assemble_pencil<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                      \
    if (e != cudaSuccess) return e;                                                           \
    k_assemble_pencil<DD><<<np, ASM_THREADS, smem, h->stream>>>(                              \
        h->d_comps, h->d_tabs, h->d_pencils, h->d_tabvals, h->p, h->mu, h->q, h->d_G,         \
        h->d_stencil, h->d_rhs, h->d_dinv)
    if (h->d == 1) { LAUNCH_ASM(1); }
    else if (h->d == 2) { LAUNCH_ASM(2); }
    else { LAUNCH_ASM(3); }
#undef LAUNCH_ASM
    h->launches[0]++;
    return cudaGetLastError();
}

}  // namespace sgiga
