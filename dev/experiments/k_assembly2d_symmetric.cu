// k_assembly2d.cu -- kernel 2 for 2-D components (maximal regularity,
// q = p + 1): a CTA owns a BLOCK of up to BA tile rows x a segment of the
// stream axis and walks the segment one stream ELEMENT (Q quadrature lines)
// per barrier interval.
//
// Reference: assembly._assemble_full (assembly.py:264-354) with the element
// kernel local_poisson_systems (_kernels/_compiled.pyx:48-90):
//   A_ij = sum_q grad(B_i) . G(q) . grad(B_j),   b_i = sum_q B_i L(q),
// G = det w J^-1 J^-T, L = f det w (assembly.py:286-294, computed per
// quadrature point by k_metric).
//
// Sum factorisation over the tensor quadrature grid (tile axis a, stream
// axis s), pair types t = (m, n) in {(s,s), (s,a), (a,s), (a,a)}:
//   stage 1 (contract x_a): thread (tile element e_a, local row la, type t)
//     keeps its Q x P pair-table slice Bu(la) Bv(lb) in registers (fixed for
//     the whole block) and, per stream line g, contracts the element's Q
//     metric values (broadcast loads) into the P values of row i_a = e_a + la,
//     offsets o_a = lb - la; they land in the row-indexed layout
//     S1[g][t][i_a][o_a][la] (each slot written by exactly one thread);
//   stage 2 (contract x_s): thread (row i_a, offset o_a, line phase h) sums
//     S1 over la (one 16-byte-vector read per t), and accumulates the P x P
//     (stream row, stream column) block of the current stream element in
//     registers; the line phases are reduced by shuffles at the element's end
//     and the block is folded into a shared ring of stream rows; completed
//     rows are flushed F at a time (F consecutive stream rows = contiguous
//     runs in the stencil, whose rows are stream-axis fastest).
// Stage 1 of element k and stage 2 of element k-1 run on disjoint thread
// groups in the same interval (double-buffered S1), the metric lines and
// stream basis tables of elements k+1, k+2 stream in by cp.async meanwhile:
// ONE __syncthreads per stream element.  Deterministic (fixed-order sums),
// no atomics, every stencil entry written exactly once.
#include <cstdio>

#include "handle.cuh"

namespace sgiga {

template <int P, int BA_>
struct Asm2Cfg {
    static constexpr int p = P - 1, Q = P, W = 2 * P - 1;
    static constexpr int BA = BA_;                  // tile rows per block
    static constexpr int NEA = BA + p;              // tile elements of the window
    static constexpr int NXA = NEA * Q;             // tile quadrature points per line
    static constexpr int F = 4;                     // stream rows per flush
    static constexpr int RING = F + P;              // alive stream rows
    static constexpr int NG = 4;                    // G_00, G_01, G_11, load
#ifndef SGIGA_A2_NQ
#define SGIGA_A2_NQ 0
#endif
    // lanes per stage-2 item (power of two; each lane sums lines g = lane mod NQ)
    // (cfg3 x1024, Q = 4: NQ 4 / 2 / 1 = 5.64 / 5.07 / 5.59 ms; cfg1 x1024, Q = 3: 0.46 / 0.42 / 0.40 ms)
    static constexpr int NQ = SGIGA_A2_NQ > 0 ? SGIGA_A2_NQ : (Q <= 3 ? 1 : 2);
    // symmetry A(i, j) = A(j, i): only the tile offsets o_a = j_a - i_a >= 0
    // are assembled (P of the W); the o_a < 0 entries are the twins'
    static constexpr int NPR = (P + 1) / 2;         // stage-1 local-row pairs (la, P-1-la)
    static constexpr int N1 = NEA * NPR * 4;        // stage-1 items (e_a, pair, t)
    static constexpr int N1L = NEA * P;             // stage-1 load items (e_a, la)
    static constexpr int N2 = BA * P * NQ;          // stage-2 items (i_a, o_a, line phase)
    static constexpr int N2L = BA;                  // stage-2 load items (i_a)
    static constexpr int NT = 32 * (((N1 + N1L > N2 + N2L ? N1 + N1L : N2 + N2L) + 31) / 32);
    // shared memory (doubles)
    static constexpr int sGe = Q * NXA + 2;         // one entry's Q lines (+2: bank skew between entries)
    static constexpr int sB = 2 * Q * P;            // stream basis values + derivatives of the element
    static constexpr int sG = (NG * sGe + sB + 1) & ~1;   // one buffer (16-byte aligned)
    // four buffers for a prefetch distance of 2: the buffer element k+2 is
    // copied into (start of interval k) is neither element k's (stage 1) nor
    // element k-1's (its stream basis tables feed stage 2 in interval k)
    static constexpr int NGB = 4;
    static constexpr int oG = 0;                    // [NGB][NG][Q][NXA] + [2][Q][P]
    // S1[g][t][i_a][o_a][la]: row blocks and line blocks padded by 16 bytes
    // (the stage-2 reads of a warp's rows and line phases fall on different banks)
    static constexpr int IAS = P * P;
    static constexpr int S1G = 4 * BA * IAS + 2;
    static constexpr int nS1 = Q * S1G;
    static constexpr int oS1 = oG + NGB * sG;       // [2][Q][S1G]
    static constexpr int nSL = Q * BA * P;
    static constexpr int oSL = oS1 + 2 * nS1;       // [2][Q][BA][P]
    static constexpr int ACW = P * W;               // ring entries of a row: (o_a >= 0, o_s)
    static constexpr int oAcc = oSL + 2 * nSL;      // [RING][BA][P][W]
    static constexpr int oAccL = oAcc + RING * BA * ACW;   // [RING][BA]
    static constexpr int total = oAccL + RING * BA;
    // resident CTAs per SM: shared memory (228 KB per SM, 1 KB reserved per
    // CTA) and a register budget of >= 96 per thread
    static constexpr int SMEM_CTAS = (228 * 1024) / (total * 8 + 1024);
    static constexpr int REG_CTAS = 65536 / (NT * 96);
    static constexpr int MINB0 = SMEM_CTAS < REG_CTAS ? SMEM_CTAS : REG_CTAS;
#ifndef SGIGA_A2_MINB
#define SGIGA_A2_MINB 0
#endif
    static constexpr int MINB = SGIGA_A2_MINB > 0 ? SGIGA_A2_MINB : (MINB0 < 1 ? 1 : (MINB0 > 4 ? 4 : MINB0));
};

__device__ __forceinline__ void cp_async8_2d(double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}

template <int P, int BA_>
__global__ void __launch_bounds__(Asm2Cfg<P, BA_>::NT, Asm2Cfg<P, BA_>::MINB)
k_assemble2d(const CompInfo* __restrict__ comps, const TabInfo* __restrict__ tabs,
             const Block2* __restrict__ blocks, const double* __restrict__ vals,
             const double* __restrict__ Gbuf, double* __restrict__ stencil, double* __restrict__ rhs,
             double* __restrict__ dinv, long long* __restrict__ prof) {
    using F = Asm2Cfg<P, BA_>;
    constexpr int p = F::p, Q = F::Q, W = F::W, NXA = F::NXA, BA = F::BA, NQ = F::NQ, NT = F::NT;
    constexpr int IAS = F::IAS, ACW = F::ACW;
    extern __shared__ __align__(16) double sm[];
    double* Acc = sm + F::oAcc;
    double* AccL = sm + F::oAccL;
    // probe (SGIGA_ASM_PROFILE=1): sampled blocks record their cycles
    const int psl = (prof && (blockIdx.x % 256) == 0 && blockIdx.x / 256 < 64) ? (int)(blockIdx.x / 256) : -1;
    long long pt0 = psl >= 0 ? clock64() : 0, pc = 0, p1 = 0, p2 = 0, pf = 0;

    const Block2 bk = blocks[blockIdx.x];
    const CompInfo& C = comps[bk.comp];
    const int tid = threadIdx.x;
    // walk axis ks (chosen per component on the host, independent of the
    // stencil's row order), tile axis ka = the other one
    const int ks = bk.walk, ka = 1 - ks;
    const TabInfo Ta = tabs[C.tab[ka]], Ts = tabs[C.tab[ks]];
    const int nel_a = Ta.nel, nel_s = Ts.nel;
    const int na = bk.na, e0 = bk.ia0 - p;          // window element el <-> tile element e0 + el
    const int r0 = bk.r0, r1 = bk.r1;               // walk rows [r0, r1) (full indices)
    const int ef = r0 - p < 0 ? 0 : r0 - p;
    const int elast = r1 - 1 > nel_s - 1 ? nel_s - 1 : r1 - 1;
    const int nelem = elast - ef + 1;
    const int64_t nqp = C.nqp, qs_s = C.qs[ks], qs_a = C.qs[ka];
    const double* Gc = Gbuf + C.qp_off;
    const int64_t nqa = (int64_t)nel_a * Q, nqs = (int64_t)nel_s * Q;
    // metric entries (packed symmetric, sym_index) per pair type
    const int g_ss = sym_index(2, ks, ks), g_as = sym_index(2, ka, ks), g_aa = sym_index(2, ka, ka);

    // ---- zero everything that is accumulated or partially written: plane
    // buffers (out-of-patch points stay zero), S1 / SL (slots no thread owns
    // stay zero), the accumulator ring ----------------------------------------
    for (int i = tid; i < F::total; i += NT) sm[i] = 0.0;
    __syncthreads();
    const int xa_lo = e0 < 0 ? -e0 * Q : 0;                          // valid window points [xa_lo, xa_hi)
    const int xa_hi = (e0 + F::NEA > nel_a ? nel_a - e0 : F::NEA) * Q;
    const int nx = xa_hi - xa_lo;
    const double* bsv = vals + Ts.val_off;          // walk-axis basis: values [nel][Q][P], derivs at + nqs * P
    // this thread's share of every element copy, decoded once: smem offset
    // and offset from the element's first metric point (>= 0) or, encoded
    // negative, from its walk-axis basis tables; every element copies alike
    constexpr int MAXC = (F::NG * Q * NXA + F::sB + NT - 1) / NT;
    int c_sm[MAXC];
    int64_t c_gl[MAXC];
    {
        const int n = F::NG * Q * nx;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            const int i = tid + c * NT;
            c_sm[c] = -1;
            c_gl[c] = 0;
            if (i < n) {
                const int x = i % nx, r = i / nx, g = r % Q, ent = r / Q;
                c_sm[c] = ent * F::sGe + g * NXA + xa_lo + x;
                c_gl[c] = (int64_t)ent * nqp + (int64_t)g * qs_s + (int64_t)(e0 * Q + xa_lo + x) * qs_a;
            } else if (i < n + F::sB) {
                const int b = i - n, der = b / (Q * P), rem = b % (Q * P);
                c_sm[c] = F::NG * F::sGe + b;
                c_gl[c] = -1 - ((der ? nqs * P : 0) + rem);
            }
        }
    }
    auto load_elem = [&](int es, int buf) {
        double* Gw = sm + F::oG + buf * F::sG;
        const double* gbase = Gc + (int64_t)es * Q * qs_s;
        const double* bbase = bsv + (int64_t)es * Q * P;
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
            if (c_sm[c] >= 0) cp_async8_2d(&Gw[c_sm[c]], c_gl[c] >= 0 ? gbase + c_gl[c] : bbase + (-1 - c_gl[c]));
        asm volatile("cp.async.commit_group;\n");
    };
    // the first two elements are in flight while the register tables are built
    if (nelem > 0) load_elem(ef, 0);
    if (nelem > 1) load_elem(ef + 1, 1);

    // ---- stage-1 item (every thread one), pair-table slice in registers -----
    // item (t, el, pr): local rows la1 = pr and la2 = P-1-pr of tile element
    // el, their P+1 non-negative offsets: k < K1 -> (la1, lb = la1 + k),
    // k >= K1 -> (la2, lb = la2 + k - K1)  (the middle row of odd P alone)
    const bool s1_on = tid < F::N1, s1_load = tid >= F::N1 && tid < F::N1 + F::N1L;
    int s1_el, s1_la1, s1_la2, s1_t = 0;
    if (s1_on) {
        const int pr = tid % F::NPR;
        s1_el = (tid / F::NPR) % F::NEA;
        s1_t = tid / (F::NPR * F::NEA);
        s1_la1 = pr;
        s1_la2 = P - 1 - pr;
    } else {
        const int j = tid - F::N1;
        s1_la1 = s1_la2 = j % P;
        s1_el = (j / P) % F::NEA;
    }
    const int K1 = P - s1_la1;
    const int s1_e = e0 + s1_el;
    const int s1_ia1 = s1_el + s1_la1 - p, s1_ia2 = s1_el + s1_la2 - p;   // local rows they feed
    const bool e_ok = (s1_on || s1_load) && s1_e >= 0 && s1_e < nel_a;
    const bool v1 = e_ok && s1_ia1 >= 0 && s1_ia1 < na;
    const bool v2 = e_ok && s1_on && s1_la2 != s1_la1 && s1_ia2 >= 0 && s1_ia2 < na;
    double T[Q][P + 1];   // (s1_on) Bu(la) Bv(lb) at the element's Q points; (s1_load) value(la) in T[g][0]
#pragma unroll
    for (int g = 0; g < Q; ++g)
#pragma unroll
        for (int k = 0; k <= P; ++k) T[g][k] = 0.0;
    if (v1 || v2) {
        const double* bv = vals + Ta.val_off + (int64_t)s1_e * Q * P;
        const double* bd = bv + nqa * P;
        const int u = s1_t >> 1, v = s1_t & 1;
#pragma unroll
        for (int g = 0; g < Q; ++g) {
            if (s1_on) {
                const double a1 = u ? bd[g * P + s1_la1] : bv[g * P + s1_la1];
                const double a2 = u ? bd[g * P + s1_la2] : bv[g * P + s1_la2];
#pragma unroll
                for (int k = 0; k <= P; ++k) {
                    const bool first = k < K1;
                    const int lb = first ? s1_la1 + k : s1_la2 + k - K1;
                    if (lb < P) T[g][k] = (first ? a1 : a2) * (v ? bd[g * P + lb] : bv[g * P + lb]);
                }
            } else {
                T[g][0] = bv[g * P + s1_la1];
            }
        }
    }
    const int s1_gent = s1_t == 0 ? g_ss : (s1_t == 3 ? g_aa : g_as);

    // ---- stage-2 item (every thread one): (tile row, offset o_a >= 0, line phase)
    const int s2_ia = tid < F::N2 ? tid / (NQ * P) : tid - F::N2;   // local tile row (full row bk.ia0 + s2_ia)
    const int s2_oj = (tid / NQ) % P, s2_g = tid % NQ;              // offset o_a, first line
    const bool s2_on = tid < F::N2 && s2_ia < na && s2_g < Q;
    const bool s2_load = tid >= F::N2 && tid < F::N2 + F::N2L && s2_ia < na;
    double R[P][P], RL[P];
#pragma unroll
    for (int a = 0; a < P; ++a) {
        RL[a] = 0.0;
#pragma unroll
        for (int b = 0; b < P; ++b) R[a][b] = 0.0;
    }
    // flush bookkeeping: rows [r0, next_flush) are written
    int next_flush = r0;
    const int64_t rows_c = C.rows, ss_a = C.ss[ka], ss_s = C.ss[ks], rs_a = C.rs[ka], rs_s = C.rs[ks];
    const int64_t rbase = (int64_t)(bk.ia0 - 1) * rs_a;
    const int absm_a = C.absm[ka], absm_s = C.absm[ks], n_a = C.n[ka], n_s = C.n[ks];
    if (nelem > 1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const long long pt1 = psl >= 0 ? clock64() : 0;

    for (int k = 0; k <= nelem; ++k) {
        long long pk = psl >= 0 ? clock64() : 0;
        if (k + 2 < nelem) load_elem(ef + k + 2, (k + 2) % F::NGB);
        if (psl >= 0) { const long long t = clock64(); pc += t - pk; pk = t; }
        if (k < nelem && (v1 || v2)) {   // ---- stage 1, element ef + k ----
            const double* Gw = sm + F::oG + (k % F::NGB) * F::sG;
            if (s1_on) {
                double* S1w = sm + F::oS1 + (k & 1) * F::nS1 + s1_t * BA * IAS;
                double* out1 = S1w + s1_ia1 * IAS + s1_la1;   // + o_a * P
                double* out2 = S1w + s1_ia2 * IAS + s1_la2;
                const double* gl = Gw + s1_gent * F::sGe + s1_el * Q;
#pragma unroll
                for (int g = 0; g < Q; ++g) {
                    double acc[P + 1];
#pragma unroll
                    for (int kk = 0; kk <= P; ++kk) acc[kk] = 0.0;
#pragma unroll
                    for (int ga = 0; ga < Q; ++ga) {
                        const double gv = gl[g * NXA + ga];
#pragma unroll
                        for (int kk = 0; kk <= P; ++kk) acc[kk] = fma(gv, T[ga][kk], acc[kk]);
                    }
#pragma unroll
                    for (int kk = 0; kk <= P; ++kk) {
                        const bool first = kk < K1;
                        if (first ? v1 : (v2 && s1_la2 + kk - K1 < P))
                            (first ? out1 + kk * P : out2 + (kk - K1) * P)[g * F::S1G] = acc[kk];
                    }
                }
            } else {
                double* out = sm + F::oSL + (k & 1) * F::nSL + s1_ia1 * P + s1_la1;
                const double* gl = Gw + (F::NG - 1) * F::sGe + s1_el * Q;
#pragma unroll
                for (int g = 0; g < Q; ++g) {
                    double acc = 0.0;
#pragma unroll
                    for (int ga = 0; ga < Q; ++ga) acc = fma(gl[g * NXA + ga], T[ga][0], acc);
                    out[g * BA * P] = acc;
                }
            }
        }
        if (psl >= 0) { const long long t = clock64(); p1 += t - pk; pk = t; }
        if (k >= 1) {   // ---- stage 2 of walk element es (its S1 was written in interval k-1) ----
            const int es = ef + k - 1;
            const double* S1r = sm + F::oS1 + ((k - 1) & 1) * F::nS1;
            const double* SLr = sm + F::oSL + ((k - 1) & 1) * F::nSL;
            const double* Bv = sm + F::oG + ((k - 1) % F::NGB) * F::sG + F::NG * F::sGe;   // [Q][P] values
            const double* Bd = Bv + Q * P;                                                  // derivatives
            if (s2_on) {   // lines g = s2_g (mod NQ) of the element: S_t = sum_la S1, then the P x P block
#pragma unroll
                for (int gi = 0; gi < (Q + NQ - 1) / NQ; ++gi) {
                    const int g = s2_g + gi * NQ;
                    if (NQ * ((Q + NQ - 1) / NQ) != Q && g >= Q) break;
                    double S[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const double* src = S1r + g * F::S1G + (t * BA + s2_ia) * IAS + s2_oj * P;
                        if constexpr (P % 2 == 0) {
                            double a0 = 0.0, a1 = 0.0;
#pragma unroll
                            for (int la = 0; la < P; la += 2) {
                                const double2 v = *reinterpret_cast<const double2*>(src + la);
                                a0 += v.x;
                                a1 += v.y;
                            }
                            S[t] = a0 + a1;
                        } else {
                            double a = 0.0;
#pragma unroll
                            for (int la = 0; la < P; ++la) a += src[la];
                            S[t] = a;
                        }
                    }
                    double vb[P], db[P];
#pragma unroll
                    for (int l = 0; l < P; ++l) {
                        vb[l] = Bv[g * P + l];
                        db[l] = Bd[g * P + l];
                    }
#pragma unroll
                    for (int ls = 0; ls < P; ++ls) {
                        // pair types along s: (s,s) D D, (s,a) D V, (a,s) V D, (a,a) V V
                        const double c0 = db[ls] * S[1] + vb[ls] * S[3];   // x V(ms)
                        const double c1 = db[ls] * S[0] + vb[ls] * S[2];   // x D(ms)
#pragma unroll
                        for (int ms = 0; ms < P; ++ms)
                            R[ls][ms] = gi == 0 ? fma(c0, vb[ms], c1 * db[ms]) : R[ls][ms] + fma(c0, vb[ms], c1 * db[ms]);
                    }
                }
            } else if (s2_load) {
#pragma unroll
                for (int g = 0; g < Q; ++g) {
                    double sl = 0.0;
#pragma unroll
                    for (int la = 0; la < P; ++la) sl += SLr[(g * BA + s2_ia) * P + la];
#pragma unroll
                    for (int ls = 0; ls < P; ++ls) RL[ls] = fma(sl, Bv[g * P + ls], RL[ls]);
                }
#pragma unroll
                for (int ls = 0; ls < P; ++ls) {
                    const int is = es + ls;
                    if (is >= r0 && is < r1) AccL[(is % F::RING) * BA + s2_ia] += RL[ls];
                    RL[ls] = 0.0;
                }
            }
            // the element's line phases are summed across the NQ lanes of an
            // item (fixed butterfly order; lanes of missing lines carry zeros)
#pragma unroll
            for (int ls = 0; ls < P; ++ls)
#pragma unroll
                for (int ms = 0; ms < P; ++ms) {
#pragma unroll
                    for (int o = 1; o < NQ; o <<= 1) {
                        const double y = __shfl_xor_sync(0xffffffffu, R[ls][ms], o);
                        R[ls][ms] = (s2_g & o) ? y + R[ls][ms] : R[ls][ms] + y;
                    }
                }
            if (s2_on && s2_g == 0) {
#pragma unroll
                for (int ls = 0; ls < P; ++ls) {
                    const int is = es + ls;
                    if (is >= r0 && is < r1) {
                        double* acc = Acc + (((is % F::RING) * BA + s2_ia) * P + s2_oj) * W + p - ls;
#pragma unroll
                        for (int ms = 0; ms < P; ++ms) acc[ms] += R[ls][ms];
                    }
                }
            }
#pragma unroll
            for (int ls = 0; ls < P; ++ls)   // lanes without a line must bring zeros to the next sum
#pragma unroll
                for (int ms = 0; ms < P; ++ms) R[ls][ms] = 0.0;
            if (psl >= 0) { const long long t = clock64(); p2 += t - pk; pk = t; }
            // ---- flush the completed walk rows, F at a time: every live entry
            // (o_a > 0, or o_a = 0 and o_s >= 0) to its own slot and the twin
            // row's mirrored slot; the structural zeros are in place (memset
            // once per layout) ----
            const int done = es == elast ? r1 - 1 : (es < r1 - 1 ? es : r1 - 1);
            if (done >= next_flush && (done - next_flush + 1 >= F::F || es == elast)) {
                __syncthreads();
                const int nf = done - next_flush + 1;
                const int grp = tid >> 5, ln = tid & 31;
                constexpr int NGRP = NT / 32;
                for (int lnx = ln; lnx < na * nf; lnx += 32) {
                    // lane <-> (tile row, walk row), consecutive lanes along
                    // the axis that is contiguous in the stencil's row order
                    int ial, f;
                    if (rs_s == 1) { ial = lnx / nf; f = lnx - ial * nf; }
                    else { f = lnx / na; ial = lnx - f * na; }
                    const int ia = bk.ia0 + ial, is = next_flush + f;
                    const int64_t row = rbase + (int64_t)ial * rs_a + (int64_t)(is - 1) * rs_s;
                    const double* accr = Acc + ((is % F::RING) * BA + ial) * ACW;
                    double* dst = stencil + C.mat_off;
                    for (int e = grp; e < ACW; e += NGRP) {
                        const int oa = e / W, os = e % W - p;
                        const int ja = ia + oa, js = is + os;
                        if ((oa == 0 && os < 0) || ja > n_a - 2 || js < 1 || js > n_s - 2) continue;
                        const double v = accr[e];
                        const int64_t sa = absm_a ? ja - 1 : oa + p, sst = absm_s ? js - 1 : os + p;
                        dst[row + (sa * ss_a + sst * ss_s) * rows_c] = v;
                        if (oa != 0 || os != 0) {
                            const int64_t saM = absm_a ? ia - 1 : p - oa, sstM = absm_s ? is - 1 : p - os;
                            dst[row + oa * rs_a + os * rs_s + (saM * ss_a + sstM * ss_s) * rows_c] = v;
                        }
                    }
                    if (grp == NGRP - 1) {
                        const int slot = (is % F::RING) * BA + ial;
                        rhs[C.vec_off + row] = AccL[slot];
                        dinv[C.vec_off + row] = 1.0 / accr[p];
                    }
                }
                __syncthreads();
                for (int it = tid; it < nf * BA * ACW; it += NT) {
                    const int f = it / (BA * ACW), rem = it - f * (BA * ACW);
                    Acc[((next_flush + f) % F::RING) * BA * ACW + rem] = 0.0;
                }
                for (int it = tid; it < nf * BA; it += NT)
                    AccL[((next_flush + it / BA) % F::RING) * BA + it % BA] = 0.0;
                next_flush = done + 1;
            }
            if (psl >= 0) { const long long t = clock64(); pf += t - pk; pk = t; }
        }
        if (k + 2 < nelem) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
    }
    if (psl >= 0 && tid == 0) {
        prof[psl * 8 + 0] = pt1 - pt0;       // setup
        prof[psl * 8 + 1] = p1;              // stage 1
        prof[psl * 8 + 2] = clock64() - pt1; // loop total
        prof[psl * 8 + 3] = nelem + 1;
        prof[psl * 8 + 4] = p2;              // stage 2
        prof[psl * 8 + 5] = bk.na;
        prof[psl * 8 + 6] = pc;              // copy issue
        prof[psl * 8 + 7] = pf;              // flush
    }
}

template <int P, int BA>
static bool launch2(Handle* h, cudaError_t* err) {
    using F = Asm2Cfg<P, BA>;
    const size_t smem = sizeof(double) * F::total;
    *err = cudaFuncSetAttribute(k_assemble2d<P, BA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (*err != cudaSuccess) return true;
    if (!h->stencil_zeroed) {   // structural zeros once per layout: the kernel writes live entries only
        *err = cudaMemsetAsync(h->d_stencil, 0, sizeof(double) * (size_t)h->total_slots, h->stream);
        if (*err != cudaSuccess) return true;
        h->stencil_zeroed = true;
    }
    long long* prof = nullptr;
    if (h->opt.asm_profile) {
        cudaMalloc(&prof, 64 * 8 * sizeof(long long));
        cudaMemsetAsync(prof, 0, 64 * 8 * sizeof(long long), h->stream);
    }
    k_assemble2d<P, BA><<<(unsigned)h->blocks2.size(), F::NT, smem, h->stream>>>(
        h->d_comps, h->d_tabs, h->d_blocks2, h->d_tabvals, h->d_G, h->d_stencil, h->d_rhs, h->d_dinv, prof);
    *err = cudaGetLastError();
    if (prof) {
        long long t[64 * 8];
        cudaStreamSynchronize(h->stream);
        cudaMemcpy(t, prof, sizeof t, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 64; ++i)
            if (t[i * 8 + 3])
                fprintf(stderr, "asm2d-profile block %d: na %lld intervals %lld setup %lld loop %lld (%.0f/interval) "
                        "stage1 %lld stage2 %lld (copy issue %lld, flush %lld)\n", i * 256, t[i * 8 + 5], t[i * 8 + 3], t[i * 8 + 0],
                        t[i * 8 + 2], (double)t[i * 8 + 2] / t[i * 8 + 3], t[i * 8 + 1], t[i * 8 + 4], t[i * 8 + 6], t[i * 8 + 7]);
        cudaFree(prof);
    }
    return true;
}

// returns false when the handle has no 2-D block list (not d = 2, not
// maximal regularity with q = p + 1): the caller falls back to the pencils
bool launch_assembly_2d(Handle* h, cudaError_t* err) {
    if (h->d != 2 || h->blocks2.empty()) return false;
    h->launches[0] += 1;
    switch (h->p + 1) {   // tile rows per block: ASM2_BA (4 and 16 measured slower on cfg1 / cfg3)
    case 2: return launch2<2, ASM2_BA>(h, err);
    case 3: return launch2<3, ASM2_BA>(h, err);
    case 4: return launch2<4, ASM2_BA>(h, err);
    case 5: return launch2<5, ASM2_BA>(h, err);
    default: return false;
    }
}

}  // namespace sgiga
