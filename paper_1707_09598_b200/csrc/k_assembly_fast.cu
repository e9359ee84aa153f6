// k_assembly_fast.cu -- kernel 2, fast path: maximal-regularity spaces
// (interior multiplicity 1) with q = p + 1, compile-time (D, P, Q).
//
// Same global sum factorisation as k_assembly.cu (see the derivation
// there), expressed in *relative* offsets o = j - i in [-p, p] so every
// support range is compile-time:
//   * a pencil row i's support window is elements i-p .. i (t = 0..p),
//     window point x = t*Q + g; on element i-p+t the row function has local
//     index p-t and the column function j = i + (t+k) - p has local index k,
//     so T[type][x][k] (k = 0..p) holds exactly the nonzero (slot, point)
//     pairs -- slot s = t + k.  Window elements outside the patch (rows near
//     the boundary, short axes) are skipped by predication, never computed;
//   * the metric plane window is double-buffered so the next plane streams
//     in while the current one is contracted: in 3-D with Q even by ONE TMA
//     tensor copy per plane (per-component 4-D tensor map, out-of-patch
//     points zero-filled, mbarrier completion), otherwise by cp.async of the
//     valid points from per-thread copy lists (the invalid ones stay zero);
//   * 3-D planes are software-pipelined: stage 1 of plane j and stage 3 of
//     plane j-1 run on disjoint thread groups in one barrier interval;
//   * stage 1 (contract tile axis b): warp half <-> pair (m,n), lane <-> x_a,
//     W register accumulators, P FMAs per metric value loaded;
//   * stage 2 (contract tile axis a): (pair, s_b, t) items, then a
//     fixed-order sum over the pairs of each stream type and over t;
//   * stage 3: rank-1 update of the P alive rows of the current stream
//     element; completed rows are flushed, mapping relative offsets to the
//     stencil's storage slots (absolute or relative), zeros elsewhere.
// Deterministic, no atomics; every stencil entry is written exactly once.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "handle.cuh"

namespace sgiga {


__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ long long clk64() {   // ordered w.r.t. memory ops and barriers
    long long t;
    asm volatile("mov.u64 %0, %%clock64;\n" : "=l"(t)::"memory");
    return t;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;\n"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n"); }

template <int D, int P, int Q, bool TM = false>
struct FastCfg {
    static constexpr int p = P - 1;
    static constexpr int W = 2 * P - 1;               // relative slots per axis
    static constexpr int RP = (P + 1) & ~1;            // pair-table row stride (16-byte rows: double2 loads)
    static constexpr int NX = P * Q;                   // window points per tile axis
    static constexpr int NA = D >= 2 ? NX : 1;
    static constexpr int NB = D >= 3 ? NX : 1;
    static constexpr int WA = D >= 2 ? W : 1;
    static constexpr int WB = D >= 3 ? W : 1;
    static constexpr int WAB = WA * WB;
    static constexpr int NG = D * (D + 1) / 2 + 1;     // metric entries + load
    static constexpr int NPAIR = D * D;
    static constexpr int PPW = NX <= 16 ? 2 : 1;       // pairs per warp in stage 1
    // 3-D stage 1 works on 5 metric groups (+ the load unit): pairs that share
    // a pair-table row of axis b are contracted by one lane from one row load,
    // and (a,s) / (s,a) share one S1 slot (same metric entry, same row)
    static constexpr bool GRP = D == 3 && P >= 5;       // grouped stage 1 (P = 4: one pair per unit measured faster)
    static constexpr int NGRP = GRP ? 5 : NPAIR;
    static constexpr int NU1 = NGRP + 1;
    static constexpr int S1T = 32 * ((NU1 + PPW - 1) / PPW);
    // 3-D: three-stage software pipeline on disjoint thread groups -- in one
    // barrier interval G1 runs stage 1 of plane j, G2 stage 2 of plane j-1
    // and G3 stage 3 of plane j-2 (+ the row flushes); S1/SL1/S2 are double
    // buffered, G2/G3 take two items per thread.  2-D: one 352-thread group,
    // stages separated by barriers.
    static constexpr bool PIPE = D == 3;
    // stage-2 output slots: the 4 stream types, type 0 (4 pairs in 3-D) split
    // in two halves, + the load term
    static constexpr bool SPLIT = D == 3;
    static constexpr int NT2 = SPLIT ? 5 : 4;
    // stage-2 outputs: 3-D -- one (s_a, s_b) block per pair (summed by stream
    // type in stage 3) + the load term; 2-D -- NT2 slots + load
    static constexpr int S2C = PIPE && P >= 5 ? 2 : 1;  // stage-2 s_b columns per thread (register budget)
    // 3-D: S2[pair][s_a][S2R] rows padded to an even length, so a stage-2
    // thread's two adjacent s_b columns leave as ONE 16-byte store (lanes on
    // distinct bank quads); even buffer stride
    static constexpr int S2R = PIPE && S2C == 2 ? ((WB + 1) & ~1) : WB;
    static constexpr int S2B = WA * S2R;               // one pair block
    static constexpr int NI2 = PIPE ? ((NPAIR * S2B + 2) & ~1) : NT2 * WAB + 1;
    static constexpr int LOAD2P = PIPE ? NPAIR * S2B : NT2 * WAB;   // the load term's slot
    static constexpr int NSB2 = (WB + S2C - 1) / S2C;  // stage-2 column groups (s_b .. s_b + S2C - 1)
    static constexpr int S2T = PIPE ? 32 * ((NPAIR * NSB2 + 1 + 31) / 32) : 0;   // one (pair, s_b pair) each
    static constexpr int S3T = PIPE ? 32 * ((WAB + P + 31) / 32) : 0;         // one (s_a, s_b) column / load row each
    static constexpr int NT = PIPE ? S1T + S2T + S3T : 352;
    // resident CTAs per SM (launch bounds)
    static constexpr int MINB = PIPE && P >= 5 ? 1 : 2;
    static constexpr int NBUF = PIPE ? 2 : 1;          // S1 / SL1 / S2 buffers
    // plane windows by one TMA tensor copy per plane (TM: the component's
    // 4-D tensor map exists -- every global stride a multiple of 16 bytes);
    // the smem rows are then NX padded to an even count (box inner extent)
    static constexpr bool TMA = TM && PIPE;
    static constexpr int NAP = D >= 2 ? (TMA ? ((NX + 1) & ~1) : (NX | 1)) : 1;   // smem row stride of a plane
    static constexpr int RING = P;                     // alive rows of the accumulator ring
    static constexpr int nGw = NG * NB * NAP;          // one plane buffer
    static constexpr int sGw = (nGw + 15) & ~15;       // buffer stride (128-byte aligned TMA destination)
    // S1 rows [pair][xa][S1W]: 3-D pads W to even so stage 2 reads two
    // adjacent s_b columns with one 16-byte load
    static constexpr int S1W = S2C == 2 ? ((W + 1) & ~1) : W;
    static constexpr int nS1 = NPAIR * NA * (PIPE ? S1W : WB);
    // shared-memory layout (doubles)
    static constexpr int oGw = 0;                      // [NGB][NG][NB][NAP]
    // plane buffers: TMA -- prefetch distance GPD = 2 planes (three buffers,
    // the next two planes in flight while one is contracted); cp.async -- 1
    static constexpr int GPD = TMA ? 2 : 1;
    static constexpr int NGB = GPD + 1;
    static constexpr int oTa = oGw + NGB * sGw;        // [4][NA][RP]
    static constexpr int oTb = oTa + 4 * NA * RP;      // [4][NB][RP]
    static constexpr int oPhiA = oTb + 4 * NB * RP;    // [NA]
    static constexpr int oPhiB = oPhiA + NA;           // [NB]
    static constexpr int oS1 = oPhiB + NB;             // [NBUF][NPAIR][NA][WB]
    static constexpr int oSL1 = oS1 + NBUF * nS1;      // [NBUF][NA]
    static constexpr int oS2 = oSL1 + NBUF * NA;       // [NBUF][NI2]
    static constexpr int oBs = oS2 + NBUF * NI2;       // [2][2][Q][P]
    static constexpr int oAcc = oBs + 4 * Q * P;       // [RING][W][WAB]
    static constexpr int oAccL = oAcc + RING * W * WAB;
    static constexpr int total = oAccL + RING;
};

template <int D, int P, int Q, bool TM>
size_t fast_smem_bytes() { return sizeof(double) * FastCfg<D, P, Q, TM>::total; }

template <int D, int P, int Q, bool TM>
__global__ void __launch_bounds__(FastCfg<D, P, Q, TM>::NT, FastCfg<D, P, Q, TM>::MINB)
k_assemble_fast(const CompInfo* __restrict__ comps, const TabInfo* __restrict__ tabs,
                const Pencil* __restrict__ pencils, const double* __restrict__ vals,
                const double* __restrict__ Gbuf, double* __restrict__ stencil,
                double* __restrict__ rhs, double* __restrict__ dinv, long long* __restrict__ prof,
                const CUtensorMap* __restrict__ tmaps) {
    using F = FastCfg<D, P, Q, TM>;
    constexpr int NT = F::NT;
    constexpr int p = F::p, W = F::W;
    extern __shared__ __align__(128) double sm[];
    double* Ta = sm + F::oTa;
    double* Tb = sm + F::oTb;
    double* phiA = sm + F::oPhiA;
    double* phiB = sm + F::oPhiB;
    double* S1 = sm + F::oS1;
    double* SL1 = sm + F::oSL1;
    double* S2 = sm + F::oS2;
    double* Bs = sm + F::oBs;
    double* Acc = sm + F::oAcc;
    double* AccL = sm + F::oAccL;

    const Pencil pc = pencils[blockIdx.x];
    const CompInfo& C = comps[pc.comp];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s = C.ax[D - 1];
    const int ka = D >= 2 ? C.ax[D - 2] : 0, kb = D >= 3 ? C.ax[D - 3] : 0;
    const TabInfo Ts = tabs[C.tab[s]];
    const int nel_a = D >= 2 ? tabs[C.tab[ka]].nel : 1, nel_b = D >= 3 ? tabs[C.tab[kb]].nel : 1;
    // valid window elements t in [t_lo, t_hi) of the two tile axes
    const int ta_lo = D >= 2 ? max(0, p - pc.ia) : 0, ta_hi = D >= 2 ? min(P, nel_a + p - pc.ia) : 1;
    const int tb_lo = D >= 3 ? max(0, p - pc.ib) : 0, tb_hi = D >= 3 ? min(P, nel_b + p - pc.ib) : 1;

    // ---- 1-D pair tables of the tile axes (relative coordinates) ----------
    auto build_T = [&](int k, int i, double* T, double* phi, int NXk) {
        const TabInfo& TT = tabs[C.tab[k]];
        const int64_t nq = (int64_t)TT.nel * Q;
        for (int idx = tid; idx < 4 * NXk * F::RP; idx += NT) {
            int kk = idx % F::RP, x = (idx / F::RP) % NXk, type = idx / (F::RP * NXk);
            int t = x / Q, g = x % Q, e = i - p + t;
            double v = 0.0;
            if (kk < P && e >= 0 && e < TT.nel) {
                const double* base = vals + TT.val_off + ((int64_t)e * Q + g) * P;
                double a = (type >> 1) ? base[nq * P + (p - t)] : base[p - t];
                double b = (type & 1) ? base[nq * P + kk] : base[kk];
                v = a * b;
            }
            T[idx] = v;
        }
        for (int x = tid; x < NXk; x += NT) {
            int t = x / Q, g = x % Q, e = i - p + t;
            phi[x] = (e >= 0 && e < TT.nel) ? vals[TT.val_off + ((int64_t)e * Q + g) * P + (p - t)] : 0.0;
        }
    };
    if (D >= 2) build_T(ka, pc.ia, Ta, phiA, F::NA);
    else if (tid == 0) { Ta[0] = 1.0; Ta[1] = Ta[2] = Ta[3] = 0.0; phiA[0] = 1.0; }
    if (D >= 3) build_T(kb, pc.ib, Tb, phiB, F::NB);
    else if (tid == 0) { Tb[0] = 1.0; Tb[1] = Tb[2] = Tb[3] = 0.0; phiB[0] = 1.0; }
    for (int idx = tid; idx < F::RING * W * F::WAB + F::RING; idx += NT) Acc[idx] = 0.0;
    // cp.async variant: invalid window points stay zero in the plane buffers
    // (the TMA unit zero-fills them itself)
    if constexpr (!F::TMA)
        for (int idx = tid; idx < F::NGB * F::sGw; idx += NT) sm[F::oGw + idx] = 0.0;
    __shared__ __align__(8) uint64_t fast_mbar[3];   // TMA variant: one barrier per plane buffer
    if (F::TMA && tid == 0) {
        mbar_init(&fast_mbar[0], 1);
        mbar_init(&fast_mbar[1], 1);
        mbar_init(&fast_mbar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        // the first GPD planes are issued here, in flight while the pencil's
        // tables and flush maps are built (short pencils: the pipeline fill)
        const int ef = pc.r0 - p < 0 ? 0 : pc.r0 - p;
        const int el = pc.r1 - 1 > Ts.nel - 1 ? Ts.nel - 1 : pc.r1 - 1;
        const int np0 = (el - ef + 1) * Q;
        const int x0u = (pc.ia - p) * Q, x1 = (pc.ib - p) * Q, x0 = x0u - (x0u & 1);
        for (int jj = 0; jj < F::GPD && jj < np0; ++jj) {
            double* Gw = sm + F::oGw + jj * F::sGw;
            mbar_expect_tx(&fast_mbar[jj], (uint32_t)(F::nGw * 8));
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                ::"r"(smem_u32(Gw)), "l"(tmaps + pc.comp), "r"(x0), "r"(x1), "r"(ef * Q + jj), "r"(0),
                  "r"(smem_u32(&fast_mbar[jj]))
                : "memory");
        }
    }
    __syncthreads();

    // ---- metric plane window (a innermost in global and shared memory) ----
    const double* Gc = Gbuf + C.qp_off;
    const int64_t nqp = C.nqp;
    const int64_t qs_s = C.qs[s], qs_b = D >= 3 ? C.qs[kb] : 0;
    const int xa_lo = D >= 2 ? ta_lo * Q : 0, nxa = D >= 2 ? (ta_hi - ta_lo) * Q : 1;   // valid xa run
    const int xb_lo = D >= 3 ? tb_lo * Q : 0, nxb = D >= 3 ? (tb_hi - tb_lo) * Q : 1;
    const int64_t Xa0 = D >= 2 ? (int64_t)(pc.ia - p) * Q + xa_lo : 0;   // first valid global a index
    const int64_t Xb0 = D >= 3 ? (int64_t)(pc.ib - p) * Q + xb_lo : 0;
    // every plane copies the same (entry, xb, xa) window: each thread's share
    // (smem offset, offset from the plane's first valid point) is decoded
    // once per pencil, so a plane costs a few instructions per copy
    constexpr int MAXC0 = (F::NG * F::NB * F::NA + NT - 1) / NT;
    constexpr bool PRE = !F::TMA && MAXC0 <= 8;   // else: row teams, one division per row
    constexpr int MAXC = PRE ? MAXC0 : 1;
    int c_sm[MAXC], c_gl[MAXC];
    constexpr int LPR = F::NA <= 16 ? 16 : 32, NTEAM = NT / LPR;
    const int team = tid / LPR, tl_ = tid % LPR;
    if constexpr (PRE) {
        const int per_row = nxa, ntot = F::NG * nxb * nxa;
#pragma unroll
        for (int k = 0; k < MAXC; ++k) {
            const int idx = tid + k * NT;
            c_sm[k] = -1;
            c_gl[k] = 0;
            if (idx < ntot) {
                const int xa = idx % per_row, r = idx / per_row;
                const int xb = r % nxb, gi = r / nxb;
                c_sm[k] = (gi * F::NB + xb_lo + xb) * F::NAP + xa_lo + xa;
                c_gl[k] = (int)((int64_t)gi * nqp + (int64_t)xb * qs_b + xa);
            }
        }
    }
    // TMA variant: ONE 4-D tensor copy per plane -- box (x_a, x_b, 1, entry)
    // of the component's metric tensor map, out-of-patch window points
    // zero-filled by the TMA unit -- armed and issued by one thread, completion
    // counted on the buffer's mbarrier (phase bit per buffer in mb_phase)
    uint32_t mb_phase = 0;
    const CUtensorMap* tmap = F::TMA ? tmaps + pc.comp : nullptr;
    // the innermost box start must be 16-byte aligned: an odd window start
    // (Q odd) is rounded down one point and the plane is read shifted by tsh
    const int tx0u = D >= 2 ? (pc.ia - p) * Q : 0, tx1 = D >= 3 ? (pc.ib - p) * Q : 0;
    const int tsh = F::TMA ? (tx0u & 1) : 0, tx0 = tx0u - tsh;
    auto load_plane_tma = [&](int64_t Qs, int buf) {
        if (tid != 0) return;
        double* Gw = sm + F::oGw + buf * F::sGw;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(&fast_mbar[buf], (uint32_t)(F::nGw * 8));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
            ::"r"(smem_u32(Gw)), "l"(tmap), "r"(tx0), "r"(tx1), "r"((int)Qs), "r"(0), "r"(smem_u32(&fast_mbar[buf]))
            : "memory");
    };
    auto wait_plane_tma = [&](int buf) {
        const uint32_t par = (mb_phase >> buf) & 1u;
        while (!mbar_try_wait(&fast_mbar[buf], par)) {
        }
        mb_phase ^= 1u << buf;
    };
    auto load_plane = [&](int64_t Qs, int buf) {
        double* Gw = sm + F::oGw + buf * F::sGw;
        const double* base = Gc + Qs * qs_s + Xa0 + Xb0 * qs_b;
        if constexpr (PRE) {
#pragma unroll
            for (int k = 0; k < MAXC; ++k)
                if (c_sm[k] >= 0) cp_async8(&Gw[c_sm[k]], base + c_gl[k]);
        } else if (tl_ < nxa) {
            const int rows = F::NG * nxb;
            for (int r = team; r < rows; r += NTEAM) {
                const int gi = r / nxb, xb = r - gi * nxb;
                cp_async8(&Gw[(gi * F::NB + xb_lo + xb) * F::NAP + xa_lo + tl_],
                          base + (int64_t)gi * nqp + (int64_t)xb * qs_b + tl_);
            }
        }
        cp_async_commit();
    };

    constexpr int NPAIR = F::NPAIR;
    const int r0 = pc.r0, r1 = pc.r1;
    const int e_first = r0 - p < 0 ? 0 : r0 - p;
    const int e_last = r1 - 1 > Ts.nel - 1 ? Ts.nel - 1 : r1 - 1;
    const int64_t nq_s = (int64_t)Ts.nel * Q;
    const int64_t row_base = (D >= 2 ? (int64_t)(pc.ia - 1) * C.rs[ka] : 0) +
                             (D >= 3 ? (int64_t)(pc.ib - 1) * C.rs[kb] : 0);
    // flush maps of the tile axes: storage slot (ca, cb) -> relative accumulator
    // index oa*WB + ob (-1 if the column is outside the band / on the boundary)
    // and its storage-slot stride part
    __shared__ int flt_rel[WMAX * WMAX], flt_slot[WMAX * WMAX];
    const int Ss = C.S[s], Sa = D >= 2 ? C.S[ka] : 1, Sb = D >= 3 ? C.S[kb] : 1, SAB = Sa * Sb;
    const int absm_s = C.absm[s], n_s = C.n[s];
    const int64_t ss_s = C.ss[s], rs_s = C.rs[s], rows_c = C.rows;
    for (int cab = tid; cab < SAB; cab += NT) {
        const int ca = cab / Sb, cb = cab % Sb;
        auto rel = [&](int k, int ik, int sk) -> int {
            const int j = C.absm[k] ? sk + 1 : ik + sk - p, o = j - ik;
            return (j < 1 || j > C.n[k] - 2 || o < -p || o > p) ? -1 : o + p;
        };
        const int oa = D >= 2 ? rel(ka, pc.ia, ca) : 0, ob = D >= 3 ? rel(kb, pc.ib, cb) : 0;
        flt_rel[cab] = (oa < 0 || ob < 0) ? -1 : oa * F::WB + ob;
        flt_slot[cab] = (int)((D >= 2 ? (int64_t)ca * C.ss[ka] : 0) + (D >= 3 ? (int64_t)cb * C.ss[kb] : 0));
    }
    int tsp[NPAIR], tap[NPAIR];   // stream / tile-a type of each (m, n) pair
#pragma unroll
    for (int pr = 0; pr < NPAIR; ++pr) {
        tsp[pr] = 2 * ((pr / D) == s) + ((pr % D) == s);
        tap[pr] = 2 * ((pr / D) == ka) + ((pr % D) == ka);
    }
    // this thread's stage-2 item (one per thread: 4 W^2 + 1 <= NT)
    constexpr int NT2 = F::NT2, LOAD2 = NT2 * F::WAB;
    static_assert(F::PIPE || LOAD2 + 1 <= NT, "one stage-2 item per thread (2-D)");
    const int i2_it = tid;
    const bool i2_on = D >= 2 && i2_it < LOAD2 + 1, i2_load = i2_it == LOAD2;
    const int i2_slot = i2_it / F::WAB, i2_sab = i2_it % F::WAB;
    const int i2_ts = i2_slot == 4 ? 0 : i2_slot;
    int i2_mask = 0;   // pairs this item sums (slots 0 / 4 take the first / last half of type 0)
    {
        int c0 = 0;
#pragma unroll
        for (int pr = 0; pr < NPAIR; ++pr) {
            if (tsp[pr] != i2_ts) continue;
            const bool take = !F::SPLIT || i2_ts != 0 || ((i2_slot == 4) == (c0 >= 2));
            if (i2_ts == 0) ++c0;
            if (take) i2_mask |= 1 << pr;
        }
    }
    const int i2_sa = i2_sab / F::WB, i2_sb = i2_sab % F::WB;
    const int i2_tl = max(ta_lo, i2_sa - p), i2_th = min(ta_hi - 1, i2_sa);

    int buf = 0;
    if constexpr (F::PIPE) {
        // interval j (j = 0 .. nplanes+1), ONE barrier at its end:
        //   start: issue plane j+1 into buffer (j+1)&1 (TMA: one thread);
        //   G1: wait plane j, stage 1 of plane j -> S1/SL1[j&1];
        //   G2: stage 2 of plane j-1: S1/SL1[(j-1)&1] -> S2[(j-1)&1];
        //   G3: stage 3 of plane j-2 from S2[(j-2)&1]; when plane j-2 closes
        //       element ep, row ep is complete: G3 flushes it and zeroes its
        //       ring slot (two G3-only named barriers) before the next row
        //       that maps to the slot receives its first update at j+1.
        constexpr int S1T = F::S1T, S2T = F::S2T, S3T = F::S3T;
        const bool inG1 = tid < S1T, inG2 = !inG1 && tid < S1T + S2T, inG3 = tid >= S1T + S2T;
        const int g2t = tid - S1T, g3t = tid - S1T - S2T;
        const int nplanes = (e_last - e_first + 1) * Q;
        // this G2 thread's stage-2 column: (pair, s_b) -> all s_a
        const bool s2_on = inG2 && g2t < NPAIR * F::NSB2 + 1, s2_load = g2t == NPAIR * F::NSB2;
        const int s2_pr = g2t / F::NSB2, s2_sb = F::S2C * (g2t % F::NSB2);   // columns s2_sb .. + S2C - 1
        int s2_sp = 0, s2_ta = 0;   // S1 / Ta offsets of the pair
#pragma unroll
        for (int pr = 0; pr < NPAIR; ++pr)
            if (pr == s2_pr) {
                // (s, a) and (a, s) contract the same metric entry with the same
                // b-row: stage 1 writes the (a, s) slot only
                const int prs = F::GRP && pr == s * D + ka ? ka * D + s : pr;
                s2_sp = prs * F::NA * F::S1W + s2_sb;
                s2_ta = tap[pr] * F::NA * F::RP;
            }
        // stage 3 sums the pair blocks of each stream type (fixed pair order):
        // type 0 = pairs without s, 1 = (m, s), 2 = (s, n), 3 = (s, s)
        const int ty_off[9] = {(ka * D + ka) * F::S2B, (ka * D + kb) * F::S2B, (kb * D + ka) * F::S2B,
                               (kb * D + kb) * F::S2B, (ka * D + s) * F::S2B,  (kb * D + s) * F::S2B,
                               (s * D + ka) * F::S2B,  (s * D + kb) * F::S2B,  (s * D + s) * F::S2B};
        auto load_bs = [&](int e) {   // G3: stream basis values/derivatives of element e
            double* Bd = Bs + (e & 1) * 2 * Q * P;
            for (int idx = g3t; idx < 2 * Q * P; idx += S3T) {
                const int der = idx / (Q * P), rem = idx % (Q * P);
                cp_async8(&Bd[idx], vals + Ts.val_off + (der ? nq_s * P : 0) + (int64_t)e * Q * P + rem);
            }
        };   // (cp.async: completed by the G3 wait at the end of the NEXT interval)
        auto flush3 = [&](int i) {   // G3: row i -> stencil / rhs / dinv
            const int64_t row = row_base + (int64_t)(i - 1) * rs_s;
            const double* accr = Acc + ((i % F::RING) * W) * F::WAB;
            double* dst = stencil + C.mat_off + row;
            for (int it = g3t; it < Ss * SAB; it += S3T) {
                const int cab = it % SAB, cs = it / SAB;
                const int j = absm_s ? cs + 1 : i + cs - p, o = j - i;   // stream-axis column
                const int oab = flt_rel[cab];
                const bool ok = oab >= 0 && j >= 1 && j <= n_s - 2 && o >= -p && o <= p;
                const double v = ok ? accr[(o + p) * F::WAB + oab] : 0.0;
                dst[((int64_t)cs * ss_s + flt_slot[cab]) * rows_c] = v;
            }
            if (g3t == 0) {
                rhs[C.vec_off + row] = AccL[i % F::RING];
                dinv[C.vec_off + row] = 1.0 / accr[p * F::WAB + p * F::WB + p];
            }
        };
        double R3[P][P], RL3 = 0.0;   // G3: the current element's sums (registers)
#pragma unroll
        for (int al = 0; al < P; ++al)
#pragma unroll
            for (int bl = 0; bl < P; ++bl) R3[al][bl] = 0.0;
        auto bar3 = [&]() { asm volatile("bar.sync 1, %0;\n" ::"r"(S3T) : "memory"); };
        if (nplanes > 0) {
            if (inG3) {
                load_bs(e_first);
                cp_async_commit();
                cp_async_wait_all();
            }
            if constexpr (F::TMA) {
                // (the first GPD planes were issued at kernel entry)
            } else {
                load_plane((int64_t)e_first * Q, 0);
                cp_async_wait_all();
            }
            __syncthreads();
        }
        // phase profile (SGIGA_ASM_PROFILE=1): block 0's group leaders record
        // their own work and the whole interval (work + barrier wait)
        const bool prf = prof != nullptr && blockIdx.x == 0 && (tid & 31) == 0;   // every warp's lane 0
        long long pw = 0, pt = 0, p0 = prf ? clk64() : 0;
        for (int j = 0; nplanes > 0 && j < nplanes + 2; ++j) {
            if (j + F::GPD < nplanes) {
                if constexpr (F::TMA) load_plane_tma((int64_t)e_first * Q + j + F::GPD, (j + F::GPD) % F::NGB);
                else load_plane((int64_t)e_first * Q + j + 1, (j + 1) % F::NGB);
            }
            if (inG1) {
                if (j < nplanes) {   // ---- stage 1 (plane j): contract tile axis b ----
                    if constexpr (F::TMA) wait_plane_tma(j % F::NGB);
                    const double* Gw = sm + F::oGw + (j % F::NGB) * F::sGw + tsh;
                    double* S1w = S1 + (j & 1) * F::nS1;
                    const int half = F::PPW == 2 ? (lane >> 4) : 0;
                    const int xa = F::PPW == 2 ? (lane & 15) : lane;
                    // GRP: warps -> units so the heavy (two-pair) units sit on SM
                    // sub-partitions (warp % 4) apart from stage 2's two warps
                    // (6, 7): {T, T, S, T, S, load}
                    const int unit = F::GRP ? (warp == 1 ? 2 : warp == 2 ? 1 : warp) : warp * F::PPW + half;
                    const int prr = unit < F::NGRP ? 0 : (unit == F::NGRP ? NPAIR : NPAIR + 1);   // load unit -> NPAIR
                    if (unit < F::NGRP && xa < F::NA) {
                        // groups in axis roles (a = ka, b = kb, s): {aa, ss}, {as}, {ab, sb},
                        // {ba, bs}, {bb}; both pairs of a group have the same b-type
                        int m0 = unit / D, n0 = unit % D, m1 = -1, n1 = -1;
                        if constexpr (F::GRP) switch (unit) {
                            case 0: m0 = ka; n0 = ka; m1 = s; n1 = s; break;
                            case 1: m0 = ka; n0 = s; break;
                            case 2: m0 = ka; n0 = kb; m1 = s; n1 = kb; break;
                            case 3: m0 = kb; n0 = ka; m1 = kb; n1 = s; break;
                            default: m0 = kb; n0 = kb; break;
                        }
                        const bool two = m1 >= 0;
                        const int tb = 2 * (m0 == kb) + (n0 == kb);
                        const double* gcol0 = Gw + sym_index(D, m0, n0) * F::NB * F::NAP + xa;
                        const double* gcol1 = Gw + (two ? sym_index(D, m1, n1) : 0) * F::NB * F::NAP + xa;
                        const double* tr = Tb + tb * F::NB * F::RP;
                        double acc[W], acd[W];
#pragma unroll
                        for (int q2 = 0; q2 < W; ++q2) acc[q2] = acd[q2] = 0.0;
#pragma unroll
                        for (int t = 0; t < P; ++t) {
                            if (t < tb_lo || t >= tb_hi) continue;
#pragma unroll
                            for (int g2 = 0; g2 < Q; ++g2) {
                                const int x = t * Q + g2;
                                const double gv = gcol0[x * F::NAP];
                                const double gw = two ? gcol1[x * F::NAP] : 0.0;
                                double tv[F::RP];   // warp-uniform row: RP/2 broadcast 16-byte loads
#pragma unroll
                                for (int k2 = 0; k2 < F::RP / 2; ++k2) {
                                    const double2 v2 = *reinterpret_cast<const double2*>(tr + x * F::RP + 2 * k2);
                                    tv[2 * k2] = v2.x;
                                    tv[2 * k2 + 1] = v2.y;
                                }
#pragma unroll
                                for (int k = 0; k < P; ++k) {
                                    acc[t + k] += gv * tv[k];
                                    if (two) acd[t + k] += gw * tv[k];
                                }
                            }
                        }
                        // 16-byte stores when the rows are even (lanes on distinct bank quads)
                        auto store_row = [&](double* o, const double* a) {
                            if constexpr (F::S1W % 2 == 0) {
#pragma unroll
                                for (int q2 = 0; q2 < W; q2 += 2)
                                    *reinterpret_cast<double2*>(o + q2) = make_double2(a[q2], q2 + 1 < W ? a[q2 + 1] : 0.0);
                            } else {
#pragma unroll
                                for (int q2 = 0; q2 < W; ++q2) o[q2] = a[q2];
                            }
                        };
                        store_row(S1w + ((m0 * D + n0) * F::NA + xa) * F::S1W, acc);
                        if (two) store_row(S1w + ((m1 * D + n1) * F::NA + xa) * F::S1W, acd);
                    } else if (prr == NPAIR && xa < F::NA) {   // load: SL1 = sum_xb L phiB
                        const double* gcol = Gw + (F::NG - 1) * F::NB * F::NAP + xa;
                        double acc = 0.0;
#pragma unroll
                        for (int x = 0; x < F::NB; ++x) acc += gcol[x * F::NAP] * phiB[x];
                        SL1[(j & 1) * F::NA + xa] = acc;
                    }
                }
            } else if (inG2) {
                if (j >= 1 && j <= nplanes) {   // ---- stage 2 (plane j-1): contract tile axis a ----
                    const int b2 = (j - 1) & 1;
                    const double* S1r = S1 + b2 * F::nS1;
                    double* S2w = S2 + b2 * F::NI2;
                    if (s2_load) {   // load: SL2 = sum_xa SL1 phiA
                        const double* sl = SL1 + b2 * F::NA;
                        double acc = 0.0;
#pragma unroll
                        for (int x = 0; x < F::NA; ++x) acc += sl[x] * phiA[x];
                        S2w[F::LOAD2P] = acc;
                    } else if (s2_on) {
                        // S2[pair][s_a][s_b] = sum_xa S1[pair][xa][s_b] Ta[xa][s_a - t(xa)],
                        // two adjacent s_b columns per thread: one 16-byte S1 load and
                        // one pair-table row feed 2P FMAs
                        double acc[W], acd[W];
#pragma unroll
                        for (int q2 = 0; q2 < W; ++q2) acc[q2] = acd[q2] = 0.0;
                        const double* sp = S1r + s2_sp;
                        const double* ta = Ta + s2_ta;
#pragma unroll
                        for (int t = 0; t < P; ++t) {
                            if (t < ta_lo || t >= ta_hi) continue;
#pragma unroll
                            for (int g2 = 0; g2 < Q; ++g2) {
                                const int xa = t * Q + g2;
                                double2 v;
                                if constexpr (F::S2C == 2) v = *reinterpret_cast<const double2*>(sp + xa * F::S1W);
                                else v.x = sp[xa * F::S1W];
                                double tv[F::RP];
#pragma unroll
                                for (int k2 = 0; k2 < F::RP / 2; ++k2) {
                                    const double2 v2 = *reinterpret_cast<const double2*>(ta + xa * F::RP + 2 * k2);
                                    tv[2 * k2] = v2.x;
                                    tv[2 * k2 + 1] = v2.y;
                                }
#pragma unroll
                                for (int k = 0; k < P; ++k) {
                                    if constexpr (F::S2C == 2) {
                                        acc[t + k] += v.x * tv[k];
                                        acd[t + k] += v.y * tv[k];
                                    } else if (xa & 1) {   // one column: even / odd points in two chains
                                        acd[t + k] += v.x * tv[k];
                                    } else {
                                        acc[t + k] += v.x * tv[k];
                                    }
                                }
                            }
                        }
                        double* o2 = S2w + s2_pr * F::S2B + s2_sb;
                        if constexpr (F::S2C == 1) {
#pragma unroll
                            for (int sa = 0; sa < W; ++sa) o2[sa * F::S2R] = acc[sa] + acd[sa];
                        } else {   // columns s_b, s_b + 1 (the pad column for the last s_b)
#pragma unroll
                            for (int sa = 0; sa < W; ++sa)
                                *reinterpret_cast<double2*>(o2 + sa * F::S2R) = make_double2(acc[sa], acd[sa]);
                        }
                    }
                }
            } else {
                if (j < nplanes && j > 0 && j % Q == 0) load_bs(e_first + j / Q);
                if (j >= 2) {   // ---- stage 3 (plane j-2): rank-1 updates ----
                    // thread (s_a, s_b) keeps the P x P (row al, column bl) sums
                    // of the current stream element in registers and folds them
                    // into the shared ring once per element
                    const int jp = j - 2, ep = e_first + jp / Q, gp = jp % Q;
                    const double* Bp = Bs + (ep & 1) * 2 * Q * P + gp * P;   // values; derivatives at +Q*P
                    const double* S2r = S2 + (jp & 1) * F::NI2;
                    if (g3t < F::WAB) {
                        // stream types: 0 = pairs without s, 1 = (m, s), 2 = (s, n), 3 = (s, s)
                        const double* q = S2r + (g3t / F::WB) * F::S2R + g3t % F::WB;
                        const double s0 = ((q[ty_off[0]] + q[ty_off[1]]) + q[ty_off[2]]) + q[ty_off[3]];
                        const double s1 = q[ty_off[4]] + q[ty_off[5]], s2v = q[ty_off[6]] + q[ty_off[7]];
                        const double s3 = q[ty_off[8]];
                        double vb[P], db[P];
#pragma unroll
                        for (int bl = 0; bl < P; ++bl) {
                            vb[bl] = Bp[bl];
                            db[bl] = Bp[Q * P + bl];
                        }
#pragma unroll
                        for (int al = 0; al < P; ++al) {
                            const double c0 = vb[al] * s0 + db[al] * s2v, c1 = vb[al] * s1 + db[al] * s3;
#pragma unroll
                            for (int bl = 0; bl < P; ++bl) R3[al][bl] += vb[bl] * c0 + db[bl] * c1;
                        }
                    } else if (g3t < F::WAB + P) {
                        RL3 += Bp[g3t - F::WAB] * S2r[F::LOAD2P];
                    }
                    if (gp == Q - 1) {   // element ep complete
                        if (g3t < F::WAB) {
#pragma unroll
                            for (int al = 0; al < P; ++al) {
                                const int i = ep + al;
                                if (i >= r0 && i < r1) {
                                    double* acc = Acc + ((i % F::RING) * W) * F::WAB + g3t;
#pragma unroll
                                    for (int bl = 0; bl < P; ++bl) acc[(bl - al + p) * F::WAB] += R3[al][bl];
                                }
#pragma unroll
                                for (int bl = 0; bl < P; ++bl) R3[al][bl] = 0.0;
                            }
                        } else if (g3t < F::WAB + P) {
                            const int i = ep + g3t - F::WAB;
                            if (i >= r0 && i < r1) AccL[i % F::RING] += RL3;
                            RL3 = 0.0;
                        }
                        bar3();
                        if (ep < e_last) {
                            if (ep >= r0 && ep < r1) {
                                flush3(ep);
                                bar3();
                                double* accz = Acc + ((ep % F::RING) * W) * F::WAB;
                                for (int it = g3t; it < W * F::WAB; it += S3T) accz[it] = 0.0;
                                if (g3t == 0) AccL[ep % F::RING] = 0.0;
                            }
                        } else {
                            for (int i = (ep > r0 ? ep : r0); i < r1; ++i) flush3(i);
                        }
                    }
                }
            }
            if (prf) pw += clk64() - p0;
            if constexpr (!F::TMA) cp_async_wait_all();
            else if (inG3) {   // one (possibly empty) group per interval: wait for all but this one
                cp_async_commit();
                cp_async_wait_prev();
            }
            __syncthreads();
            if (prf) {
                const long long t1 = clk64();
                pt += t1 - p0;
                p0 = t1;
            }
        }
        if (prf) {
            const int g = inG1 ? 0 : (inG2 ? 1 : 2);
            if (tid == 0 || tid == S1T || tid == S1T + S2T) {
                prof[2 * g] = pw;
                prof[2 * g + 1] = pt;
            }
            if (g == 0 && tid == 0) prof[6] = nplanes + 2;
            prof[8 + (tid >> 5)] = pw;   // per-warp work
        }
    } else {
    const bool pr = prof != nullptr && blockIdx.x == 0 && tid == 0;   // phase profile
    long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tc = 0;
    load_plane((int64_t)e_first * Q, 0);
    for (int e = e_first; e <= e_last; ++e) {
        for (int idx = tid; idx < 2 * Q * P; idx += NT) {
            int der = idx / (Q * P), rem = idx % (Q * P);
            Bs[idx] = vals[Ts.val_off + (der ? nq_s * P : 0) + (int64_t)e * Q * P + rem];
        }
        for (int g = 0; g < Q; ++g) {
            if (pr) tc = clock64();
            // issue the next plane, then wait for the current one
            const bool more = (g + 1 < Q) || (e < e_last);
            if (more) {
                load_plane(g + 1 < Q ? (int64_t)e * Q + g + 1 : (int64_t)(e + 1) * Q, buf ^ 1);
                cp_async_wait_prev();
            } else {
                cp_async_wait_all();
            }
            __syncthreads();
            if (pr) { long long t = clock64(); tp[0] += t - tc; tc = t; }
            const double* Gw = sm + F::oGw + buf * F::sGw;
            // ---- stage 1: contract tile axis b ------------------------------
            if constexpr (D == 3) {
                const int half = F::PPW == 2 ? (lane >> 4) : 0;
                const int xa = F::PPW == 2 ? (lane & 15) : lane;
                const int pr = warp * F::PPW + half;
                if (pr < NPAIR && xa < F::NA) {
                    const int gidx = sym_index(D, pr / D, pr % D);
                    const int tb = 2 * ((pr / D) == kb) + ((pr % D) == kb);
                    double acc[W];
#pragma unroll
                    for (int j = 0; j < W; ++j) acc[j] = 0.0;
                    const double* gcol = Gw + gidx * F::NB * F::NAP + xa;
                    const double* tr = Tb + tb * F::NB * F::RP;
#pragma unroll
                    for (int t = 0; t < P; ++t) {
                        if (t < tb_lo || t >= tb_hi) continue;
#pragma unroll
                        for (int g2 = 0; g2 < Q; ++g2) {
                            const int x = t * Q + g2;
                            const double gv = gcol[x * F::NAP];
#pragma unroll
                            for (int k = 0; k < P; ++k) acc[t + k] += gv * tr[x * F::RP + k];
                        }
                    }
                    double* out = S1 + (pr * F::NA + xa) * W;
#pragma unroll
                    for (int j = 0; j < W; ++j) out[j] = acc[j];
                } else if (pr == NPAIR && xa < F::NA) {   // load: SL1 = sum_xb L phiB
                    const double* gcol = Gw + (F::NG - 1) * F::NB * F::NAP + xa;
                    double acc = 0.0;
#pragma unroll
                    for (int x = 0; x < F::NB; ++x) acc += gcol[x * F::NAP] * phiB[x];
                    SL1[xa] = acc;
                }
                __syncthreads();
            }
            if (pr) { long long t = clock64(); tp[1] += t - tc; tc = t; }
            // ---- stage 2: contract tile axis a ------------------------------
            if constexpr (D >= 2) {
                // one pass: S2[ts][sa][sb] = sum over the pairs of stream type ts,
                // window elements t with k = sa - t in [0, p], and their Q points
                // the item (decoded once per pencil, see i2_*) is the same for
                // every plane: compile-time (t, g2) loops with predication give
                // immediate-offset loads, ~3 instructions per FMA
                if (i2_on) {
                    if (i2_load) {   // load: SL2 = sum_xa SL1 phiA
                        double acc = 0.0;
#pragma unroll
                        for (int x = 0; x < F::NA; ++x)
                            acc += (D == 3 ? SL1[x] : Gw[(F::NG - 1) * F::NAP + x]) * phiA[x];
                        S2[LOAD2] = acc;
                    } else {
                        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                        for (int prr = 0; prr < NPAIR; ++prr) {
                            if (!((i2_mask >> prr) & 1)) continue;
                            const double* sp = D == 3 ? S1 + prr * F::NA * W + i2_sb
                                                      : Gw + sym_index(D, prr / D, prr % D) * F::NAP;
                            const int sstr = D == 3 ? W : 1;
                            const double* tp0 = Ta + tap[prr] * F::NA * F::RP + i2_sa;
#pragma unroll
                            for (int t = 0; t < P; ++t) {
                                if (t < i2_tl || t > i2_th) continue;
#pragma unroll
                                for (int g2 = 0; g2 < Q; ++g2) {
                                    const int xa = t * Q + g2;
                                    const double v = sp[xa * sstr] * tp0[xa * F::RP - t];
                                    if (g2 & 1) acc1 += v; else acc0 += v;
                                }
                            }
                        }
                        S2[i2_it] = acc0 + acc1;
                    }
                }
                if (pr) { long long t = clock64(); tp[2] += t - tc; tc = t; }
            } else {
                if (tid < 4) S2[tid] = (tid == 3) ? Gw[0] : 0.0;
                if (tid == 0) S2[4] = Gw[(F::NG - 1) * F::NB * F::NAP];
            }
            __syncthreads();
            if (pr) { long long t = clock64(); tp[3] += t - tc; tc = t; }
            // ---- stage 3: rank-1 update of the alive rows of element e ------
            for (int it = tid; it < P * F::WAB; it += NT) {
                const int sab = it % F::WAB, al = it / F::WAB;
                const int i = e + al;
                if (i < r0 || i >= r1) continue;
                const double va = Bs[g * P + al], da = Bs[Q * P + g * P + al];
                const double s0 = F::SPLIT ? S2[sab] + S2[4 * F::WAB + sab] : S2[sab];
                const double s1 = S2[F::WAB + sab], s2v = S2[2 * F::WAB + sab], s3 = S2[3 * F::WAB + sab];
                const double c0 = va * s0 + da * s2v, c1 = va * s1 + da * s3;
                double* acc = Acc + ((i % F::RING) * W) * F::WAB + sab;
#pragma unroll
                for (int bl = 0; bl < P; ++bl) {
                    const double vb = Bs[g * P + bl], db = Bs[Q * P + g * P + bl];
                    acc[(bl - al + p) * F::WAB] += vb * c0 + db * c1;
                }
            }
            if (tid < P) {
                const int i = e + tid;
                if (i >= r0 && i < r1) AccL[i % F::RING] += Bs[g * P + tid] * S2[LOAD2];
            }
            buf ^= 1;
            if (pr) { long long t = clock64(); tp[4] += t - tc; tc = t; tp[6] += 1; }
        }
        __syncthreads();
        if (pr) tc = clock64();
        // ---- flush: row e completes with element e; the last element also
        // completes the trailing rows of the segment.  Every storage slot of
        // a flushed row is written (zeros where the relative offset is out
        // of the band or the column is on the boundary). ----------------------
        const int lo = (e == e_last) ? (e > r0 ? e : r0) : e;
        const int hi = (e == e_last) ? r1 : (e + 1 < r1 ? e + 1 : r1);
        for (int i = (lo > r0 ? lo : r0); i < hi; ++i) {
            const int64_t row = row_base + (int64_t)(i - 1) * rs_s;
            double* accr = Acc + ((i % F::RING) * W) * F::WAB;
            double* dst = stencil + C.mat_off + row;
            for (int it = tid; it < Ss * SAB; it += NT) {
                const int cab = it % SAB, cs = it / SAB;
                const int j = absm_s ? cs + 1 : i + cs - p, o = j - i;   // stream-axis column
                const int oab = flt_rel[cab];
                const bool ok = oab >= 0 && j >= 1 && j <= n_s - 2 && o >= -p && o <= p;
                const double v = ok ? accr[(o + p) * F::WAB + oab] : 0.0;
                dst[((int64_t)cs * ss_s + flt_slot[cab]) * rows_c] = v;
            }
            if (tid == 0) {
                const int dsab = D >= 2 ? (p * F::WB + (D >= 3 ? p : 0)) : 0;
                rhs[C.vec_off + row] = AccL[i % F::RING];
                dinv[C.vec_off + row] = 1.0 / accr[p * F::WAB + dsab];
            }
            __syncthreads();
            for (int it = tid; it < W * F::WAB; it += NT) accr[it] = 0.0;
            if (tid == 0) AccL[i % F::RING] = 0.0;
            __syncthreads();
        }
        if (pr) { tp[5] += clock64() - tc; tp[7] += 1; }
    }
    if (pr)
        for (int k = 0; k < 8; ++k) prof[k] = tp[k];
    }
}

// dispatch: returns false when (d, p, q, mu) has no fast instantiation
// Per-component 4-D tensor maps of the metric buffer for the TMA plane
// copies: dims (x_a, x_b, x_s, entry) with element strides (1, N_a, N_a N_b,
// nqp) -- the qp storage order of build_tables (a innermost) -- and box
// (NX, NX, 1, NG).  Built once per handle (host encode, one H2D copy);
// false when the driver entry point or an encode is unavailable.
static bool build_tmaps(Handle* h, int NX) {
    if (h->tmaps_state != 0) return h->tmaps_state > 0;
    h->tmaps_state = -1;
    if (h->d != 3) return false;
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &qres) != cudaSuccess ||
        qres != cudaDriverEntryPointSuccess || !fnp) {
        cudaGetLastError();
        return false;
    }
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    EncodeFn encode = reinterpret_cast<EncodeFn>(fnp);
    std::vector<CUtensorMap> maps(h->ncomp);
    const int q = h->q, NG = h->nG();
    for (int c = 0; c < h->ncomp; ++c) {
        const CompInfo& C = h->comps[c];
        const int s = C.ax[2], a = C.ax[1], b = C.ax[0];
        const cuuint64_t Na = (cuuint64_t)C.nel[a] * q, Nb = (cuuint64_t)C.nel[b] * q, Ns = (cuuint64_t)C.nel[s] * q;
        if (C.qs[a] != 1 || C.qs[b] != (int64_t)Na || C.qs[s] != (int64_t)(Na * Nb)) return false;
        const cuuint64_t dims[4] = {Na, Nb, Ns, (cuuint64_t)NG};
        const cuuint64_t strides[3] = {Na * 8, Na * Nb * 8, (cuuint64_t)C.nqp * 8};
        // box rows padded to an even count (16-byte inner extent); every
        // global stride must be a multiple of 16 bytes as well
        const cuuint32_t box[4] = {(cuuint32_t)((NX + 1) & ~1), (cuuint32_t)NX, 1, (cuuint32_t)NG};
        if (strides[0] % 16 || strides[1] % 16 || strides[2] % 16 || (C.qp_off * 8) % 16) return false;
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (encode(&maps[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)(h->d_G + C.qp_off), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    if (!h->d_tmaps && cudaMalloc(&h->d_tmaps, sizeof(CUtensorMap) * h->ncomp) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (cudaMemcpyAsync(h->d_tmaps, maps.data(), sizeof(CUtensorMap) * h->ncomp, cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    h->tmaps_state = 1;
    return true;
}

bool launch_assembly_fast(Handle* h, cudaError_t* err, int npencils) {
    if (h->mu != 1 || h->q != h->p + 1 || h->pencils.empty()) return false;
    if (npencils <= 0) return true;
    const int key = h->d * 10 + (h->p + 1);
    const bool no_tma = h->opt.no_tma;
    const bool tma = h->d == 3 && !no_tma &&
                     build_tmaps(h, (h->p + 1) * h->q);
    size_t smem = 0;
    const void* fn = nullptr;
    int nthreads = 352;
    switch (key) {
#define CASE(DD, PP)                                                                 \
    case DD * 10 + PP:                                                               \
        if (tma && FastCfg<DD, PP, PP, true>::TMA) {                                 \
            smem = fast_smem_bytes<DD, PP, PP, true>();                              \
            fn = (const void*)k_assemble_fast<DD, PP, PP, true>;                     \
            nthreads = FastCfg<DD, PP, PP, true>::NT;                                \
        } else {                                                                     \
            smem = fast_smem_bytes<DD, PP, PP, false>();                             \
            fn = (const void*)k_assemble_fast<DD, PP, PP, false>;                    \
            nthreads = FastCfg<DD, PP, PP, false>::NT;                               \
        }                                                                            \
        break;
        CASE(1, 2) CASE(1, 3) CASE(1, 4) CASE(1, 5)
        CASE(2, 2) CASE(2, 3) CASE(2, 4) CASE(2, 5)
        CASE(3, 2) CASE(3, 3) CASE(3, 4) CASE(3, 5)
#undef CASE
    default: return false;
    }
    *err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (*err != cudaSuccess) return true;
    long long* prof = nullptr;
    if (h->opt.asm_profile) {
        cudaMalloc(&prof, 40 * sizeof(long long));
        cudaMemsetAsync(prof, 0, 40 * sizeof(long long), h->stream);
    }
    void* args[] = {(void*)&h->d_comps, (void*)&h->d_tabs, (void*)&h->d_pencils, (void*)&h->d_tabvals,
                    (void*)&h->d_G, (void*)&h->d_stencil, (void*)&h->d_rhs, (void*)&h->d_dinv,
                    (void*)&prof, (void*)&h->d_tmaps};
    *err = cudaLaunchKernel(fn, dim3((unsigned)npencils), dim3(nthreads), args, smem, h->stream);
    if (prof) {
        long long t[40];
        cudaStreamSynchronize(h->stream);
        cudaMemcpy(t, prof, sizeof t, cudaMemcpyDeviceToHost);
        const double n = t[6] > 0 ? (double)t[6] : 1.0;
        if (h->d == 3) {
            fprintf(stderr, "asm-profile per-warp work cycles/interval:");
            for (int w = 0; w < nthreads / 32; ++w) fprintf(stderr, " %.0f", t[8 + w] / n);
            fprintf(stderr, "\n");
        }
        if (h->d == 3)
            fprintf(stderr, "asm-profile block0 intervals=%lld cycles/interval: G1 work=%.0f total=%.0f | G2 work=%.0f"
                    " total=%.0f | G3 work=%.0f total=%.0f\n", t[6], t[0] / n, t[1] / n, t[2] / n, t[3] / n, t[4] / n,
                    t[5] / n);
        else
        fprintf(stderr, "asm-profile block0 planes=%lld elements=%lld cycles/plane: load-wait=%.0f stage1=%.0f "
                "stage2a=%.0f stage2b=%.0f stage3=%.0f ; flush/element=%.0f\n", t[6], t[7], t[0] / n, t[1] / n,
                t[2] / n, t[3] / n, t[4] / n, t[5] / (t[7] > 0 ? (double)t[7] : 1.0));
        cudaFree(prof);
    }
    h->launches[0] += 1;
    return true;
}

}  // namespace sgiga
