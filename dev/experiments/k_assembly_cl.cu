// k_assembly_cl.cu -- kernel 2, 3-D cluster path (maximal regularity,
// q = p + 1, P = p + 1 in 3..5).
//
// Same sum factorisation and three-group plane pipeline as k_assembly_fast
// (see the derivation there and in k_assembly.cu), but the CK = p pencils
// (ia0 .. ia0 + CK - 1, ib) of one stream segment run as ONE thread-block
// cluster, one pencil per CTA, sharing stage 1 through distributed shared
// memory:
//   * the pencils' a-windows overlap: pencil ia reads window elements
//     ia - p .. ia, so the cluster's union is the CK + p = 2 CK elements
//     ia0 - p .. ia0 + CK - 1.  CTA k OWNS two of them (ia0 - p + 2k,
//     ia0 - p + 2k + 1): its TMA plane copy is only those 2Q points along a
//     (x all NX points along b), and its stage 1 contracts axis b for them
//     only -- the 5x-redundant stage 1 of the one-pencil-per-CTA kernel
//     (every x_a point contracted by all P pencils whose window holds it)
//     drops to 1x (+ the cluster's edge);
//   * stage 2 of pencil ia reads the stage-1 rows S1[pair][x_a][o_b] of its
//     P window elements from their owners' shared memory
//     (ld.shared::cluster, addresses mapped once per pencil);
//   * stage 3 and the row flushes stay CTA-local (the pencil's own rows);
//   * one cluster barrier (arrive.release / wait.acquire) ends every plane
//     interval instead of __syncthreads: it publishes interval j's S1 to the
//     neighbours and frees the buffer they read in interval j;
//   * CTAs whose pencil row lies beyond the axis (the last cluster of an
//     axis whose length is not a multiple of CK) still own window elements:
//     they run stage 1 only.
// The smaller plane windows (2Q instead of PQ points along a) and S1 rows
// halve the shared memory of a CTA, so two CTAs (two clusters' pencils)
// share an SM.
// Deterministic: every S1 / S2 value is computed by one thread in a fixed
// order, exactly as in the one-CTA kernel; every stencil entry is written
// once.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "handle.cuh"

namespace sgiga {

namespace {
__device__ __forceinline__ uint32_t cl_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cl_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(cl_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void cl_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(cl_smem(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool cl_mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(cl_smem(bar)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// volatile without a memory clobber: kept in program order w.r.t. the
// cluster barriers (also volatile), free to be scheduled among the FMAs
__device__ __forceinline__ double2 cl_ld2(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ double cl_ld1(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// interval barrier: a RELAXED arrive (an arrive.release is a fence over every
// outstanding access of the thread -- the flush's global stores included);
// the threads whose shared-memory writes others read next interval fence
// first: stage 1 (S1, read by the cluster) at cluster scope, stage 2 (S2,
// read by stage 3 of this CTA) at CTA scope
__device__ __forceinline__ void cl_sync_relaxed(int scope) {
    if (scope == 2) asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
    else if (scope == 1) asm volatile("fence.acq_rel.cta;\n" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ long long cl_clk() {
    long long t;
    asm volatile("mov.u64 %0, %%clock64;\n" : "=l"(t)::"memory");
    return t;
}
}  // namespace

template <int P, int Q, int NGB_>
struct ClCfg {
    static constexpr int D = 3;
    static constexpr int p = P - 1, W = 2 * P - 1;
    static constexpr int CK = p;                         // CTAs (pencils) per cluster
    static constexpr int RP = (P + 1) & ~1;              // pair-table row stride (double2 rows)
    static constexpr int NX = P * Q;                     // pencil window points per tile axis
    static constexpr int NA = NX, NB = NX;
    static constexpr int NXO = 2 * Q;                    // owned points along a (two elements)
    // plane row stride = TMA box inner extent: even (16-byte rows) and, for
    // odd Q, one point more on each side (an odd first point is read from
    // the preceding even one, shifted by tsh)
    static constexpr int NAPO = ((NXO + 1) & ~1) + ((Q & 1) ? 2 : 0);
    static constexpr int WB = W, WAB = W * W;
    static constexpr int NG = 7;                          // metric entries + load
    static constexpr int NPAIR = 9;
    static constexpr int NGRP = 5;                        // stage-1 metric groups (see k_assembly_fast)
    static constexpr int N1 = NGRP * NXO + NXO;           // stage-1 items (+ load items)
    static constexpr int S1T = 32 * ((N1 + 31) / 32);
    static constexpr int NSB2 = (W + 1) / 2;              // stage-2 column pairs
    static constexpr int S2T = 32 * ((NPAIR * NSB2 + 1 + 31) / 32);
    static constexpr int S3T = 32 * ((WAB + P + 31) / 32);
    static constexpr int NT = S1T + S2T + S3T;
    static constexpr int NGB = NGB_;                      // plane buffers (prefetch distance NGB - 1)
    static constexpr int GPD = NGB - 1;
    static constexpr int MINB = NGB <= 2 ? 2 : 1;         // resident CTAs per SM
    static constexpr int S1W = (W + 1) & ~1;
    static constexpr int nS1 = NPAIR * NXO * S1W;
    static constexpr int NI2 = NPAIR * WAB + 1;
    static constexpr int RING = P;
    static constexpr int nGw = NG * NB * NAPO;
    static constexpr int sGw = (nGw + 15) & ~15;
    static constexpr int ev(int x) { return (x + 1) & ~1; }
    static constexpr int oGw = 0;
    static constexpr int oTa = oGw + NGB * sGw;          // [4][NA][RP]
    static constexpr int oTb = oTa + 4 * NA * RP;        // [4][NB][RP]
    static constexpr int oPhiA = oTb + 4 * NB * RP;      // [NA]
    static constexpr int oPhiB = ev(oPhiA + NA);         // [NB]
    static constexpr int oS1 = ev(oPhiB + NB);           // [2][NPAIR][NXO][S1W]
    static constexpr int oSL1 = oS1 + 2 * nS1;           // [2][NXO]
    static constexpr int oS2 = ev(oSL1 + 2 * NXO);       // [2][NI2]
    static constexpr int oBs = ev(oS2 + 2 * NI2);        // [2][2][Q][P]
    static constexpr int oAcc = ev(oBs + 4 * Q * P);     // [RING][W][WAB]
    static constexpr int oAccL = oAcc + RING * W * WAB;  // [RING]
    static constexpr int total = oAccL + RING;
};

template <int P, int Q, int NGB>
size_t cl_smem_bytes() { return sizeof(double) * ClCfg<P, Q, NGB>::total; }

template <int P, int Q, int NGB>
__global__ void __launch_bounds__(ClCfg<P, Q, NGB>::NT, ClCfg<P, Q, NGB>::MINB)
k_assemble_cl(const CompInfo* __restrict__ comps, const TabInfo* __restrict__ tabs,
              const Pencil* __restrict__ pencils, const double* __restrict__ vals,
              double* __restrict__ stencil, double* __restrict__ rhs, double* __restrict__ dinv,
              long long* __restrict__ prof, const CUtensorMap* __restrict__ tmaps, int probe) {
    using F = ClCfg<P, Q, NGB>;
    constexpr int D = 3, NT = F::NT, p = F::p, W = F::W, NPAIR = F::NPAIR;
    constexpr int S1T = F::S1T, S2T = F::S2T, S3T = F::S3T;
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
    __shared__ __align__(8) uint64_t mbar[NGB];
    __shared__ int flt_rel[WMAX * WMAX], flt_slot[WMAX * WMAX];

    const Pencil pc = pencils[blockIdx.x];
    const CompInfo& C = comps[pc.comp];
    const int tid = threadIdx.x;
    const int crank = (int)cl_rank();
    const int s = C.ax[2], ka = C.ax[1], kb = C.ax[0];
    const TabInfo Ts = tabs[C.tab[s]];
    const int nel_a = tabs[C.tab[ka]].nel, nel_b = tabs[C.tab[kb]].nel;
    const bool live = pc.ia >= 1 && pc.ia <= C.m[ka];     // else: stage 1 of the owned elements only
    const int ia0 = pc.ia - crank;
    const int eo0 = ia0 - p + 2 * crank;                   // first owned element along a
    const int ta_lo = max(0, p - pc.ia), ta_hi = min(P, nel_a + p - pc.ia);
    const int tb_lo = max(0, p - pc.ib), tb_hi = min(P, nel_b + p - pc.ib);
    const int r0 = pc.r0, r1 = pc.r1;
    const int e_first = r0 - p < 0 ? 0 : r0 - p;
    const int e_last = r1 - 1 > Ts.nel - 1 ? Ts.nel - 1 : r1 - 1;
    const int nplanes = (e_last - e_first + 1) * Q;
    // TMA box start: owned points along a (odd start rounded down, read shifted)
    const int tx0u = eo0 * Q, tsh = tx0u & 1, tx0 = tx0u - tsh, tx1 = (pc.ib - p) * Q;
    const CUtensorMap* tmap = tmaps + pc.comp;
    auto issue_plane = [&](int plane, int b) {   // one thread
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        cl_mbar_expect_tx(&mbar[b], (uint32_t)(F::nGw * 8));
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
            ::"r"(cl_smem(sm + F::oGw + b * F::sGw)), "l"(tmap), "r"(tx0), "r"(tx1), "r"(plane), "r"(0),
              "r"(cl_smem(&mbar[b]))
            : "memory");
    };
    if (tid == 0) {
        for (int b = 0; b < NGB; ++b) cl_mbar_init(&mbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int jj = 0; jj < F::GPD && jj < nplanes; ++jj) issue_plane(e_first * Q + jj, jj);
    }

    // ---- 1-D pair tables of the tile axes (relative coordinates) ----------
    auto build_T = [&](int k, int i, double* T, double* phi) {
        const TabInfo& TT = tabs[C.tab[k]];
        const int64_t nq = (int64_t)TT.nel * Q;
        for (int idx = tid; idx < 4 * F::NX * F::RP; idx += NT) {
            const int kk = idx % F::RP, x = (idx / F::RP) % F::NX, type = idx / (F::RP * F::NX);
            const int t = x / Q, g = x % Q, e = i - p + t;
            double v = 0.0;
            if (kk < P && e >= 0 && e < TT.nel) {
                const double* base = vals + TT.val_off + ((int64_t)e * Q + g) * P;
                const double a = (type >> 1) ? base[nq * P + (p - t)] : base[p - t];
                const double b = (type & 1) ? base[nq * P + kk] : base[kk];
                v = a * b;
            }
            T[idx] = v;
        }
        for (int x = tid; x < F::NX; x += NT) {
            const int t = x / Q, g = x % Q, e = i - p + t;
            phi[x] = (e >= 0 && e < TT.nel) ? vals[TT.val_off + ((int64_t)e * Q + g) * P + (p - t)] : 0.0;
        }
    };
    if (live) build_T(ka, pc.ia, Ta, phiA);
    build_T(kb, pc.ib, Tb, phiB);
    for (int idx = tid; idx < F::RING * W * F::WAB + F::RING; idx += NT) Acc[idx] = 0.0;

    const int64_t nq_s = (int64_t)Ts.nel * Q;
    const int64_t row_base = (int64_t)(pc.ia - 1) * C.rs[ka] + (int64_t)(pc.ib - 1) * C.rs[kb];
    const int Ss = C.S[s], Sa = C.S[ka], Sb = C.S[kb], SAB = Sa * Sb;
    const int absm_s = C.absm[s], n_s = C.n[s];
    const int64_t ss_s = C.ss[s], rows_c = C.rows;
    if (live)
        for (int cab = tid; cab < SAB; cab += NT) {
            const int ca = cab / Sb, cb = cab % Sb;
            auto rel = [&](int k, int ik, int sk) -> int {
                const int j = C.absm[k] ? sk + 1 : ik + sk - p, o = j - ik;
                return (j < 1 || j > C.n[k] - 2 || o < -p || o > p) ? -1 : o + p;
            };
            const int oa = rel(ka, pc.ia, ca), ob = rel(kb, pc.ib, cb);
            flt_rel[cab] = (oa < 0 || ob < 0) ? -1 : oa * F::WB + ob;
            flt_slot[cab] = (int)((int64_t)ca * C.ss[ka] + (int64_t)cb * C.ss[kb]);
        }

    const bool inG1 = tid < S1T, inG2 = !inG1 && tid < S1T + S2T, inG3 = tid >= S1T + S2T;
    const int g2t = tid - S1T, g3t = tid - S1T - S2T;

    // ---- stage-1 item: (metric group, owned point xo) or (load, xo) -------
    // warp 0 takes the three two-pair groups, warp 1 the single ones + load
    const int u_idx = tid / F::NXO, xo = tid % F::NXO;
    int m0 = 0, n0 = 0, m1 = -1, n1 = -1;
    {
        constexpr int uord[5] = {0, 2, 3, 1, 4};
        const int unit = u_idx < F::NGRP ? uord[u_idx] : 0;
        switch (unit) {
            case 0: m0 = ka; n0 = ka; m1 = s; n1 = s; break;
            case 1: m0 = ka; n0 = s; break;
            case 2: m0 = ka; n0 = kb; m1 = s; n1 = kb; break;
            case 3: m0 = kb; n0 = ka; m1 = kb; n1 = s; break;
            default: m0 = kb; n0 = kb; break;
        }
    }
    const bool two = m1 >= 0;
    const int g1_tb = 2 * (m0 == kb) + (n0 == kb);
    const int g1_e0 = sym_index(D, m0, n0), g1_e1 = two ? sym_index(D, m1, n1) : 0;
    const int g1_o0 = (m0 * D + n0) * F::NXO + xo, g1_o1 = two ? (m1 * D + n1) * F::NXO + xo : 0;

    // ---- stage-2 item: (pair, s_b column pair) or the load; window element
    // t of the pencil is owned by cluster rank (crank + t) / 2 ---------------
    const bool s2_on = live && inG2 && g2t < NPAIR * F::NSB2 + 1, s2_load = g2t == NPAIR * F::NSB2;
    const int s2_pr = g2t / F::NSB2, s2_sb = 2 * (g2t % F::NSB2);
    int s2_ta = 0, s2_prs = 0;
    {
#pragma unroll
        for (int pr = 0; pr < NPAIR; ++pr)
            if (pr == s2_pr) {
                s2_prs = pr == s * D + ka ? ka * D + s : pr;   // (s, a) shares the (a, s) S1 slot
                s2_ta = (2 * ((pr / D) == ka) + ((pr % D) == ka)) * F::NA * F::RP;
            }
    }
    uint32_t s2_base[P];
#pragma unroll
    for (int t = 0; t < P; ++t) {
        const int own = crank + t, o = own >> 1, lo = own & 1;
        const uint32_t local = s2_load ? cl_smem(SL1 + lo * Q)
                                       : cl_smem(S1 + ((s2_prs * F::NXO) + lo * Q) * F::S1W + s2_sb);
        s2_base[t] = (probe & 1) ? local : cl_mapa(local, (uint32_t)(o < F::CK ? o : 0));
    }

    // ---- stage 3 (as k_assembly_fast) --------------------------------------
    const int ty_off[9] = {(ka * D + ka) * F::WAB, (ka * D + kb) * F::WAB, (kb * D + ka) * F::WAB,
                           (kb * D + kb) * F::WAB, (ka * D + s) * F::WAB,  (kb * D + s) * F::WAB,
                           (s * D + ka) * F::WAB,  (s * D + kb) * F::WAB,  (s * D + s) * F::WAB};
    auto load_bs = [&](int e) {
        double* Bd = Bs + (e & 1) * 2 * Q * P;
        for (int idx = g3t; idx < 2 * Q * P; idx += S3T) {
            const int der = idx / (Q * P), rem = idx % (Q * P);
            Bd[idx] = vals[Ts.val_off + (der ? nq_s * P : 0) + (int64_t)e * Q * P + rem];
        }
    };
    auto flush3 = [&](int i) {
        const int64_t row = row_base + (int64_t)(i - 1) * C.rs[s];
        const double* accr = Acc + ((i % F::RING) * W) * F::WAB;
        double* dst = stencil + C.mat_off + row;
        for (int it = g3t; it < Ss * SAB; it += S3T) {
            const int cab = it % SAB, cs = it / SAB;
            const int j = absm_s ? cs + 1 : i + cs - p, o = j - i;
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
    double R3[P][P], RL3 = 0.0;
#pragma unroll
    for (int al = 0; al < P; ++al)
#pragma unroll
        for (int bl = 0; bl < P; ++bl) R3[al][bl] = 0.0;
    auto bar3 = [&]() { asm volatile("bar.sync 1, %0;\n" ::"r"(S3T) : "memory"); };

    if (live && inG3 && nplanes > 0) load_bs(e_first);
    cl_sync();   // tables, maps, barrier init visible; every CTA of the cluster running

    const bool prf = prof != nullptr && blockIdx.x == 0 && (tid == 0 || tid == S1T || tid == S1T + S2T);
    long long pw = 0, pt = 0, p0 = prf ? cl_clk() : 0;
    uint32_t mb_phase = 0;
    for (int j = 0; j < nplanes + 2 && nplanes > 0; ++j) {
        if (tid == 0 && j + F::GPD < nplanes) issue_plane(e_first * Q + j + F::GPD, (j + F::GPD) % NGB);
        if (inG1) {
            if (j < nplanes) {   // ---- stage 1 (plane j), owned points ----
                const int b = j % NGB;
                {
                    const uint32_t par = (mb_phase >> b) & 1u;
                    while (!cl_mbar_try_wait(&mbar[b], par)) {
                    }
                    mb_phase ^= 1u << b;
                }
                const double* Gw = sm + F::oGw + b * F::sGw + tsh;
                double* S1w = S1 + (j & 1) * F::nS1;
                if (u_idx < F::NGRP) {
                    const double* gcol0 = Gw + g1_e0 * F::NB * F::NAPO + xo;
                    const double* gcol1 = Gw + g1_e1 * F::NB * F::NAPO + xo;
                    const double* tr = Tb + g1_tb * F::NB * F::RP;
                    double acc[W], acd[W];
#pragma unroll
                    for (int q2 = 0; q2 < W; ++q2) acc[q2] = acd[q2] = 0.0;
#pragma unroll
                    for (int t = 0; t < P; ++t) {
                        if (t < tb_lo || t >= tb_hi) continue;
#pragma unroll
                        for (int g2 = 0; g2 < Q; ++g2) {
                            const int x = t * Q + g2;
                            const double gv = gcol0[x * F::NAPO];
                            const double gw = two ? gcol1[x * F::NAPO] : 0.0;
                            double tv[F::RP];
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
                    double* out = S1w + g1_o0 * F::S1W;
#pragma unroll
                    for (int q2 = 0; q2 < W; ++q2) out[q2] = acc[q2];
                    if (two) {
                        double* o1 = S1w + g1_o1 * F::S1W;
#pragma unroll
                        for (int q2 = 0; q2 < W; ++q2) o1[q2] = acd[q2];
                    }
                } else if (u_idx == F::NGRP) {   // load: SL1 = sum_xb L phiB
                    const double* gcol = Gw + (F::NG - 1) * F::NB * F::NAPO + xo;
                    double acc = 0.0;
#pragma unroll
                    for (int x = 0; x < F::NB; ++x) acc += gcol[x * F::NAPO] * phiB[x];
                    SL1[(j & 1) * F::NXO + xo] = acc;
                }
            }
        } else if (inG2) {
            if (s2_on && j >= 1 && j <= nplanes) {   // ---- stage 2 (plane j-1) ----
                const int b2 = (j - 1) & 1;
                double* S2w = S2 + b2 * F::NI2;
                if (s2_load) {
                    const uint32_t boff = (uint32_t)(b2 * F::NXO * 8);
                    double acc = 0.0;
#pragma unroll
                    for (int t = 0; t < P; ++t) {
                        if (t < ta_lo || t >= ta_hi) continue;
#pragma unroll
                        for (int g2 = 0; g2 < Q; ++g2) acc += cl_ld1(s2_base[t] + boff + g2 * 8) * phiA[t * Q + g2];
                    }
                    S2w[F::NI2 - 1] = acc;
                } else {
                    const uint32_t boff = (uint32_t)(b2 * F::nS1 * 8);
                    const double* ta = Ta + s2_ta;
                    double acc[W], acd[W];
#pragma unroll
                    for (int q2 = 0; q2 < W; ++q2) acc[q2] = acd[q2] = 0.0;
#pragma unroll
                    for (int t = 0; t < P; ++t) {
                        if (t < ta_lo || t >= ta_hi) continue;
                        double2 v[Q];
#pragma unroll
                        for (int g2 = 0; g2 < Q; ++g2) v[g2] = cl_ld2(s2_base[t] + boff + g2 * F::S1W * 8);
#pragma unroll
                        for (int g2 = 0; g2 < Q; ++g2) {
                            const int xa = t * Q + g2;
                            double tv[F::RP];
#pragma unroll
                            for (int k2 = 0; k2 < F::RP / 2; ++k2) {
                                const double2 v2 = *reinterpret_cast<const double2*>(ta + xa * F::RP + 2 * k2);
                                tv[2 * k2] = v2.x;
                                tv[2 * k2 + 1] = v2.y;
                            }
#pragma unroll
                            for (int k = 0; k < P; ++k) {
                                acc[t + k] += v[g2].x * tv[k];
                                acd[t + k] += v[g2].y * tv[k];
                            }
                        }
                    }
                    double* o2 = S2w + s2_pr * F::WAB + s2_sb;
#pragma unroll
                    for (int sa = 0; sa < W; ++sa) o2[sa * F::WB] = acc[sa];
                    if (s2_sb + 1 < F::WB) {
#pragma unroll
                        for (int sa = 0; sa < W; ++sa) o2[sa * F::WB + 1] = acd[sa];
                    }
                }
            }
        } else if (live) {
            if (j < nplanes && j > 0 && j % Q == 0) load_bs(e_first + j / Q);
            if (j >= 2) {   // ---- stage 3 (plane j-2) ----
                const int jp = j - 2, ep = e_first + jp / Q, gp = jp % Q;
                const double* Bp = Bs + (ep & 1) * 2 * Q * P + gp * P;
                const double* S2r = S2 + (jp & 1) * F::NI2;
                if (g3t < F::WAB) {
                    const double* q = S2r + g3t;
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
                    RL3 += Bp[g3t - F::WAB] * S2r[F::NI2 - 1];
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
        if (prf) pw += cl_clk() - p0;
        cl_sync_relaxed(inG1 ? 2 : (inG2 ? 1 : 0));
        if (prf) {
            const long long t1 = cl_clk();
            pt += t1 - p0;
            p0 = t1;
        }
    }
    if (prf) {
        const int g = inG1 ? 0 : (inG2 ? 1 : 2);
        prof[2 * g] = pw;
        prof[2 * g + 1] = pt;
        if (g == 0) prof[6] = nplanes + 2;
    }
}

// 4-D tensor maps of the metric buffer with the cluster kernel's box
// (NAPO owned points along a, NX along b, one plane, all entries)
static bool build_tmaps_cl(Handle* h, int box_a, int NX) {
    if (h->tmaps_cl_state != 0) return h->tmaps_cl_state > 0;
    h->tmaps_cl_state = -1;
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
        const cuuint32_t box[4] = {(cuuint32_t)box_a, (cuuint32_t)NX, 1, (cuuint32_t)NG};
        if (strides[0] % 16 || strides[1] % 16 || strides[2] % 16 || (C.qp_off * 8) % 16) return false;
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (encode(&maps[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)(h->d_G + C.qp_off), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    if (!h->d_tmaps_cl && cudaMalloc(&h->d_tmaps_cl, sizeof(CUtensorMap) * h->ncomp) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (cudaMemcpyAsync(h->d_tmaps_cl, maps.data(), sizeof(CUtensorMap) * h->ncomp, cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    h->tmaps_cl_state = 1;
    return true;
}

template <int P, int NGB>
static bool launch_cl(Handle* h, cudaError_t* err) {
    using F = ClCfg<P, P, NGB>;
    if (!build_tmaps_cl(h, F::NAPO, F::NX)) return false;
    const size_t smem = cl_smem_bytes<P, P, NGB>();
    auto fn = k_assemble_cl<P, P, NGB>;
    *err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (*err != cudaSuccess) return true;
    long long* prof = nullptr;
    if (h->opt.asm_profile) {
        cudaMalloc(&prof, 8 * sizeof(long long));
        cudaMemsetAsync(prof, 0, 8 * sizeof(long long), h->stream);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)h->clpencils.size());
    cfg.blockDim = dim3(F::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = F::CK;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(h->d_tmaps_cl);
    *err = cudaLaunchKernelEx(&cfg, fn, (const CompInfo*)h->d_comps, (const TabInfo*)h->d_tabs,
                              (const Pencil*)h->d_clpencils, (const double*)h->d_tabvals, h->d_stencil, h->d_rhs,
                              h->d_dinv, prof, tm, getenv("SGIGA_CL_PROBE") ? atoi(getenv("SGIGA_CL_PROBE")) : 0);
    if (prof) {
        long long t[8];
        cudaStreamSynchronize(h->stream);
        cudaMemcpy(t, prof, sizeof t, cudaMemcpyDeviceToHost);
        const double n = t[6] > 0 ? (double)t[6] : 1.0;
        fprintf(stderr, "asm-profile (cluster) block0 intervals=%lld cycles/interval: G1 work=%.0f total=%.0f | "
                "G2 work=%.0f total=%.0f | G3 work=%.0f total=%.0f\n", t[6], t[0] / n, t[1] / n, t[2] / n,
                t[3] / n, t[4] / n, t[5] / n);
        cudaFree(prof);
    }
    h->launches[0] += 1;
    return true;
}

// false when the cluster path does not apply (then k_assemble_fast runs)
bool launch_assembly_cl(Handle* h, cudaError_t* err) {
    if (h->d != 3 || h->mu != 1 || h->q != h->p + 1 || h->clpencils.empty() || h->opt.no_tma ||
        h->opt.no_asm_cluster)
        return false;
    const bool one = h->opt.asm_cl_ngb3;
    switch (h->p + 1) {
        case 3: return one ? launch_cl<3, 3>(h, err) : launch_cl<3, 2>(h, err);
        case 4: return one ? launch_cl<4, 3>(h, err) : launch_cl<4, 2>(h, err);
        case 5: return one ? launch_cl<5, 3>(h, err) : launch_cl<5, 2>(h, err);
        default: return false;
    }
}

}  // namespace sgiga
