// k_assembly_tile.cu -- kernel 2 for 3-D components (maximal regularity,
// q = p + 1, degree 3 or 4): tiled cross-sections, warp-specialised.
//
// Reference: the element loop of _assemble_full / local_poisson_systems
// (S/assembly.py:264-354, S/_kernels/_compiled.pyx:48-90) restated as a
// global sum factorisation into the implicit-column stencil (derivation in
// k_assembly.cu).  Where k_assembly_fast.cu gives every cross-section row
// (i_a, i_b) its own CTA, a CTA here owns a TILE of rows -- na rows along
// a = ax[1] times nb rows along b = ax[0] -- and a segment of the stream
// axis s = ax[2]:
//   * one TMA tensor copy per quadrature plane brings the UNION window of
//     the tile's rows, so a thin axis (2 or 4 elements: most of a sparse
//     grid's components) is read once per plane instead of once per row, and
//     stage 1 -- which does not depend on i_a -- is computed once for all
//     na rows;
//   * warps 0..11 (G12), plane j:  stage 1 (contract b) -> S1[ib][pair slot][xa][w_b],
//     named barrier, stage 2 (contract a) -> S2[row][unit][c_a][c_b] (pairs summed
//     per unit of the stream-direction type stage 3 needs, storage columns);
//   * warps 12..15 (G3), plane j-1 in the same barrier interval: stage 3 --
//     one work item per (row, storage column (c_a, c_b)); the P alive stream
//     rows of an item (a ring of 35 doubles for p = 4) live in TENSOR MEMORY
//     (tcgen05.ld / .st, each G3 warp in its own TMEM lane quadrant, up to
//     7 rings per thread), so the ring costs no registers between planes and
//     the tile size is not capped by the register file; completed stream rows
//     go straight to the stencil.
// One CTA barrier per plane.  Deterministic, no atomics, each stencil entry
// written once; a row's value does not depend on the tiling.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "handle.cuh"

namespace sgiga {

#ifndef SGIGA_TILE3_NS2
#define SGIGA_TILE3_NS2 3
#endif
#ifndef SGIGA_TILE3_NPB
#define SGIGA_TILE3_NPB 2
#endif
constexpr int TILE3_NPB = SGIGA_TILE3_NPB;   // TMA plane buffers (prefetch distance NPB)
#ifndef SGIGA_TILE3_NS1
#define SGIGA_TILE3_NS1 2
#endif
constexpr int TILE3_NS1 = SGIGA_TILE3_NS1;   // stage-1 output buffers (2: one G12 barrier per plane)
constexpr int TILE3_NS2 = SGIGA_TILE3_NS2;   // S2 buffers between the stage-2 and stage-3 warps

namespace {

__device__ __forceinline__ uint32_t t3_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one double (two TMEM columns) of this thread's lane
__device__ __forceinline__ double tm_ld2_issue(uint32_t a, uint32_t& lo, uint32_t& hi) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(lo), "=r"(hi) : "r"(a));
    return 0.0;
}
__device__ __forceinline__ void tm_st2(uint32_t a, double v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n"
                 ::"r"(a), "r"((uint32_t)__double2loint(v)), "r"((uint32_t)__double2hiint(v)) : "memory");
}
// n consecutive TMEM columns (n even, 16-column chunks + pairs) of this thread's lane
template <int N>
__device__ __forceinline__ void tm_ldn(uint32_t a, uint32_t* r) {
#pragma unroll
    for (int c = 0; c + 16 <= N; c += 16)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                     "%13, %14, %15}, [%16];\n"
                     : "=r"(r[c]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]), "=r"(r[c + 5]),
                       "=r"(r[c + 6]), "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]), "=r"(r[c + 10]), "=r"(r[c + 11]),
                       "=r"(r[c + 12]), "=r"(r[c + 13]), "=r"(r[c + 14]), "=r"(r[c + 15])
                     : "r"(a + c));
#pragma unroll
    for (int c = N & ~15; c < N; c += 2)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(r[c]), "=r"(r[c + 1]) : "r"(a + c));
}
template <int N>
__device__ __forceinline__ void tm_stn(uint32_t a, const uint32_t* r) {
#pragma unroll
    for (int c = 0; c + 16 <= N; c += 16)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                     "%13, %14, %15, %16};\n"
                     ::"r"(a + c), "r"(r[c]), "r"(r[c + 1]), "r"(r[c + 2]), "r"(r[c + 3]), "r"(r[c + 4]), "r"(r[c + 5]),
                       "r"(r[c + 6]), "r"(r[c + 7]), "r"(r[c + 8]), "r"(r[c + 9]), "r"(r[c + 10]), "r"(r[c + 11]),
                       "r"(r[c + 12]), "r"(r[c + 13]), "r"(r[c + 14]), "r"(r[c + 15])
                     : "memory");
#pragma unroll
    for (int c = N & ~15; c < N; c += 2)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(a + c), "r"(r[c]), "r"(r[c + 1])
                     : "memory");
}
// 8 doubles = 16 TMEM columns of this thread's lane, the 32-bit halves
// paired inside the asm (no register copies between the TMEM and FP64 views)
__device__ __forceinline__ void tm_ld_d8(uint32_t a, double* d) {
    asm volatile("{\n .reg .b32 r<16>;\n"
                 " tcgen05.ld.sync.aligned.32x32b.x16.b32 {r0, r1, r2, r3, r4, r5, r6, r7, r8, r9, r10, r11, r12, r13, "
                 "r14, r15}, [%8];\n"
                 " mov.b64 %0, {r0, r1};\n mov.b64 %1, {r2, r3};\n mov.b64 %2, {r4, r5};\n mov.b64 %3, {r6, r7};\n"
                 " mov.b64 %4, {r8, r9};\n mov.b64 %5, {r10, r11};\n mov.b64 %6, {r12, r13};\n"
                 " mov.b64 %7, {r14, r15};\n}\n"
                 : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3]), "=d"(d[4]), "=d"(d[5]), "=d"(d[6]), "=d"(d[7])
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld_d1(uint32_t a, double& d) {
    asm volatile("{\n .reg .b32 r<2>;\n tcgen05.ld.sync.aligned.32x32b.x2.b32 {r0, r1}, [%1];\n"
                 " mov.b64 %0, {r0, r1};\n}\n" : "=d"(d) : "r"(a));
}
__device__ __forceinline__ void tm_st_d8(uint32_t a, const double* d) {
    asm volatile("{\n .reg .b32 r<16>;\n"
                 " mov.b64 {r0, r1}, %1;\n mov.b64 {r2, r3}, %2;\n mov.b64 {r4, r5}, %3;\n mov.b64 {r6, r7}, %4;\n"
                 " mov.b64 {r8, r9}, %5;\n mov.b64 {r10, r11}, %6;\n mov.b64 {r12, r13}, %7;\n"
                 " mov.b64 {r14, r15}, %8;\n"
                 " tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {r0, r1, r2, r3, r4, r5, r6, r7, r8, r9, r10, r11, r12, "
                 "r13, r14, r15};\n}\n"
                 ::"r"(a), "d"(d[0]), "d"(d[1]), "d"(d[2]), "d"(d[3]), "d"(d[4]), "d"(d[5]), "d"(d[6]), "d"(d[7])
                 : "memory");
}
// the element partial R3 (P*P doubles at the slot start)
template <int P>
__device__ __forceinline__ void tm_ld_r3(uint32_t a, double (*r3)[P]) {
    double* d = &r3[0][0];
#pragma unroll
    for (int c = 0; c + 8 <= P * P; c += 8) tm_ld_d8(a + 2 * c, d + c);
#pragma unroll
    for (int c = (P * P) & ~7; c < P * P; ++c) tm_ld_d1(a + 2 * c, d[c]);
}
template <int P>
__device__ __forceinline__ void tm_st_r3(uint32_t a, double (*r3)[P]) {
    double* d = &r3[0][0];
#pragma unroll
    for (int c = 0; c + 8 <= P * P; c += 8) tm_st_d8(a + 2 * c, d + c);
#pragma unroll
    for (int c = (P * P) & ~7; c < P * P; ++c) tm_st2(a + 2 * c, d[c]);
}
// stencil store that asks L2 to keep the line (the 8-byte entries of one
// 32-byte sector arrive over four stream rows; an early eviction of the
// partial sector costs a DRAM read-modify-write)
__device__ __forceinline__ void st_keep(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(t3_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, q;\n}\n" : "=r"(ok) : "r"(t3_smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

template <int P>
struct TCfg {
    static constexpr int p = P - 1, Q = P, W = 2 * P - 1;
    static constexpr int RP = (P + 1) & ~1;     // pair-table row (16-byte pair loads)
    static constexpr int PQ = P * Q;            // window points of one row
    // symmetry: stage 2 reads only w_b >= p & ~1 (o_b >= 0, even start for
    // aligned pair loads), so stage 1 keeps the columns WBS1 .. W-1 only
    static constexpr int WBS1 = p & ~1;
    static constexpr int S1W = (W - WBS1 + 1) & ~1;   // S1 row (w_b pairs by 16-byte loads)
    static constexpr int NC2 = (W + 1) / 2;     // stage-2 column pairs
    static constexpr int NG = 7;                // 6 metric entries + load
    static constexpr int NU = 5;                // stage-2 units
    static constexpr int SC = tile3_slot_cols(P);     // TMEM columns per stage-3 item
    static constexpr int R3C = tile3_r3_cols(P);      // its element partial (slot start)
    static constexpr int NSLOT = tile3_nslot(P);
    static constexpr int RC = 2 * W;                  // TMEM columns per physical stream row
};

// per-CTA shared-memory layout (doubles)
struct TLay {
    int est, sGw, oTa, oTb, oPhiA, oPhiB, oS1, s1slot, oSL1, oS2, s2sz, oRL, oList, total;
};

// dg: diagonal metric (axis-aligned box geometry): 4 plane entries (G_aa,
// G_bb, G_ss, load), 3 stage-1 slots, 3 stage-2 units
__host__ __device__ inline TLay tile3_layout(int P, int na, int nb, int xa, int xap, int xb, int n3, bool dg) {
    const int Q = P, W = 2 * P - 1, RP = (P + 1) & ~1, PQ = P * Q, S1W = (W - ((P - 1) & ~1) + 1) & ~1;
    const int rows = na * nb;
    TLay L;
    // plane buffer: 7 dense entries (one TMA box) or 4 entries at a 128-byte
    // aligned stride (four TMA boxes, each destination 128-byte aligned)
    L.est = dg ? ((xb * xap + 15) & ~15) : xb * xap;
    L.sGw = ((dg ? 4 : 7) * L.est + 15) & ~15;
    L.oTa = TILE3_NPB * L.sGw;
    L.oTb = L.oTa + na * 4 * PQ * RP;
    L.oPhiA = L.oTb + nb * 4 * PQ * RP;
    L.oPhiB = L.oPhiA + na * PQ;
    L.oS1 = (L.oPhiB + nb * PQ + 1) & ~1;
    L.s1slot = xa * S1W + 2;
    L.oSL1 = L.oS1 + TILE3_NS1 * nb * (dg ? 3 : 8) * L.s1slot;   // TILE3_NS1 stage-1 buffers
    L.oS2 = (L.oSL1 + TILE3_NS1 * nb * xa + 1) & ~1;
    L.s2sz = (dg ? 3 : 5) * n3 + rows;           // [row][unit][c_a][c_b] + load [row]
    L.oRL = L.oS2 + TILE3_NS2 * L.s2sz;
    L.oList = L.oRL + rows * P;                  // stage-3 item list (ints): computed items first
    L.total = L.oList + (n3 + 1) / 2;
    return L;
}

// Symmetry: A(i, j) = A(j, i), so a stage-3 work item -- a cross-section row
// and one storage column (c_a, c_b) -- is computed only for non-negative
// cross-section offsets (o_b > 0, or o_b = 0 and o_a >= 0) and writes the
// mirrored entries of the twin row too; for (o_a, o_b) = (0, 0) only the
// stream offsets o_s >= 0 are written (and mirrored).  Categories of a
// storage column: computed (POS, POS0 = the (0, 0) column), NEG (its
// in-band entries come from twins; only its structural zeros are written
// here), DEAD (outside the band or on the boundary: zeros).
enum : int { T3_DEAD = 0, T3_NEG = 1, T3_POS = 2, T3_POS0 = 3 };
__host__ __device__ inline int tile3_category(int ia, int ib, int ca, int cb, int absa, int absb, int ma, int mb,
                                              int p) {
    const int ja = absa ? ca + 1 : ia + ca - p, jb = absb ? cb + 1 : ib + cb - p;
    const int oa = ja - ia, ob = jb - ib;
    if (!(ja >= 1 && ja <= ma && oa >= -p && oa <= p && jb >= 1 && jb <= mb && ob >= -p && ob <= p)) return T3_DEAD;
    if (ob > 0 || (ob == 0 && oa > 0)) return T3_POS;
    if (ob == 0 && oa == 0) return T3_POS0;
    return T3_NEG;
}

// stage-1 pair slots: aa, as(=sa), ss, ab, sb, ba, bs, bb -- b-type of each
// (2 (m == b) + (n == b): derivative of the row / column function along b)
__device__ __constant__ int c_t3_btype[8] = {0, 0, 0, 1, 1, 2, 2, 3};
// stage-2 units (pairs summed per stream type; type 0 split in two):
//   u0 {aa, ab}, u1 {ba, bb}, u2 {as, bs} (type 1), u3 {sa, sb} (type 2), u4 {ss}
// (S1 slot, a-type) of the two pairs of each unit (u4: one pair)
__device__ __constant__ int c_t3_uslot[5][2] = {{0, 3}, {5, 7}, {1, 6}, {1, 4}, {2, 2}};
__device__ __constant__ int c_t3_uat[5][2] = {{3, 2}, {1, 0}, {2, 0}, {1, 0}, {0, 0}};

// diagonal-metric mode: stage-1 slot -> (plane entry, b-type): aa (0, 0), ss (2, 0), bb (1, 3), load (3);
// stage-2 units: aa (S1 slot 0, a-type 3), bb (slot 2, a-type 0), ss (slot 1, a-type 0)
__device__ __constant__ int c_t3d_btype[3] = {0, 0, 3};
__device__ __constant__ int c_t3d_uslot[3] = {0, 2, 1};
__device__ __constant__ int c_t3d_uat[3] = {3, 0, 0};

template <int P, bool DG>
__global__ void __launch_bounds__(TILE3_THREADS, 1)
k_assemble_tile(const CompInfo* __restrict__ comps, const TabInfo* __restrict__ tabs,
                const Tile3* __restrict__ tiles, const double* __restrict__ vals,
                double* __restrict__ stencil, double* __restrict__ rhs, double* __restrict__ dinv,
                const CUtensorMap* __restrict__ tmaps, long long* __restrict__ prof) {
    using F = TCfg<P>;
    // general metric: 7 plane entries, 8 stage-1 pair slots + load, 5 stage-2
    // units; diagonal metric (G_ab = G_as = G_bs = 0 exactly): 4 / 3 + 1 / 3
    constexpr int NGE = DG ? 4 : 7, NS1 = DG ? 3 : 8, NI1 = NS1 + 1, NU = DG ? 3 : 5;
    constexpr int p = F::p, Q = F::Q, W = F::W, RP = F::RP, PQ = F::PQ, S1W = F::S1W, WBS1 = F::WBS1;
    constexpr int NC2 = F::NC2, G12 = TILE3_G12, NT = TILE3_THREADS;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar[TILE3_NPB];
    // S2 hand-off between the groups: full[b] (G12 wrote plane buffer b),
    // empty[b] (G3 consumed it) -- no CTA-wide barrier per plane, so a slow
    // stage-3 plane (an element's flush) does not stall stages 1/2
    __shared__ __align__(8) uint64_t s2full[TILE3_NS2], s2empty[TILE3_NS2];
    __shared__ int s_ent[8];
    __shared__ uint32_t s_tmem;
    // the tile, its component and tables staged in shared memory: values the
    // compiler rematerialises under register pressure reload from there
    __shared__ Tile3 sT;
    __shared__ CompInfo sC;
    __shared__ TabInfo sTab[3];
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid == 0) sT = tiles[blockIdx.x];
    __syncthreads();
    if (tid == 0) sC = comps[sT.comp];
    __syncthreads();
    if (tid < 3) sTab[tid] = tabs[sC.tab[sC.ax[tid == 0 ? 1 : (tid == 1 ? 0 : 2)]]];
    __syncthreads();
    const Tile3& T = sT;
    const CompInfo& C = sC;
    const int ka = C.ax[1], kb = C.ax[0], ks = C.ax[2];
    const TabInfo& TA = sTab[0];
    const TabInfo& TB = sTab[1];
    const TabInfo& TS = sTab[2];
    const int nel_a = TA.nel, nel_b = TB.nel, nel_s = TS.nel;
    const int na = T.na, nb = T.nb, rows = na * nb;
    const int EA0 = max(0, T.a0 - p), EB0 = max(0, T.b0 - p);
    const int EA1 = min(nel_a - 1, T.a0 + na - 1);
    const int XAv = (EA1 - EA0 + 1) * Q;                   // valid union extent along a
    const int r0 = T.r0, r1 = T.r1;
    const int e_first = max(0, r0 - p), e_last = min(r1 - 1, nel_s - 1);
    const int nE = e_last - e_first + 1;
    const int nplanes = nE > 0 ? nE * Q : 0;
    if (nplanes == 0) return;   // uniform over the CTA
    const int Sa = C.S[ka], Sb = C.S[kb], SAB = Sa * Sb;
    const int n3 = rows * SAB;
    const TLay L = tile3_layout(P, na, nb, T.xa, T.xap, T.xb, n3, DG);
    const int xap = T.xap, xb = T.xb;
    double* Ta = sm + L.oTa;
    double* Tb = sm + L.oTb;
    double* phiA = sm + L.oPhiA;
    double* phiB = sm + L.oPhiB;
    double* const S1b = sm + L.oS1;
    double* const SL1b = sm + L.oSL1;
    double* S1 = S1b;
    double* SL1 = SL1b;
    double* S2 = sm + L.oS2;
    double* RLs = sm + L.oRL;
    // odd Q: the box's inner start must be 16-byte aligned -- an odd window
    // start is rounded down one point and the plane is read shifted by tsh
    const int tsh = (Q & 1) ? ((EA0 * Q) & 1) : 0;
    const int tx0 = EA0 * Q - tsh, tx1 = EB0 * Q;
    const CUtensorMap* tmap = tmaps + T.comp;
    const uint32_t pbytes = (uint32_t)(NGE * xb * xap * 8);

    auto issue_plane = [&](int j) {   // one thread: plane j -> buffer j % NPB
        const int b = j % TILE3_NPB;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(t3_smem_u32(&bar[b])),
                     "r"(pbytes) : "memory");
        if constexpr (!DG) {   // one copy: box (x_a, x_b, 1 plane, 7 entries)
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                ::"r"(t3_smem_u32(sm + b * L.sGw)), "l"(tmap), "r"(tx0), "r"(tx1), "r"(e_first * Q + j), "r"(0),
                  "r"(t3_smem_u32(&bar[b]))
                : "memory");
        } else {               // four copies of box (x_a, x_b, 1, 1): G_aa, G_bb, G_ss, load
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int ent = k == 0 ? sym_index(3, ka, ka) : (k == 1 ? sym_index(3, kb, kb) : (k == 2 ? sym_index(3, ks, ks) : 6));
                asm volatile(
                    "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                    ::"r"(t3_smem_u32(sm + b * L.sGw + k * L.est)), "l"(tmap), "r"(tx0), "r"(tx1),
                      "r"(e_first * Q + j), "r"(ent), "r"(t3_smem_u32(&bar[b]))
                    : "memory");
            }
        }
    };
    if (tid == 0) {
        for (int b = 0; b < TILE3_NPB; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(t3_smem_u32(&bar[b])) : "memory");
        for (int b = 0; b < TILE3_NS2; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(t3_smem_u32(&s2full[b])), "r"(G12) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(t3_smem_u32(&s2empty[b])), "r"(TILE3_G3)
                         : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int jj = 0; jj < TILE3_NPB && jj < nplanes; ++jj) issue_plane(jj);
    }
    if (tid < 8) {   // plane entry of each stage-1 pair slot: aa as ss ab sb ba bs bb
        const int mm = tid == 2 || tid == 4 ? ks : (tid >= 5 ? kb : ka);
        const int nn = tid == 0 || tid == 5 ? ka : (tid == 3 || tid == 4 || tid == 7 ? kb : ks);
        s_ent[tid] = DG ? (tid == 0 ? 0 : (tid == 1 ? 2 : 1)) : sym_index(3, mm, nn);   // DG: aa ss bb -> 0 2 1
    }
    if (warp == G12 / 32) {   // first G3 warp: the whole tensor memory (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                     ::"r"(t3_smem_u32(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }

    // ---- 1-D pair tables of the tile rows (relative window coordinates):
    // T[row][type][x = t Q + g][k] = (row fn p-t)^(type>>1)' (e, g) * (fn k)^(type&1)' (e, g),
    // e = i - p + t; phi[row][x] = row function value (load) -------------
    auto build_T = [&](const TabInfo& TT, int i0, int nr, double* Tt, double* phi) {
        const int64_t nq = (int64_t)TT.nel * Q;
        for (int idx = tid; idx < nr * 4 * PQ * RP; idx += NT) {
            const int kk = idx % RP, x = (idx / RP) % PQ, type = (idx / (RP * PQ)) % 4, r = idx / (RP * PQ * 4);
            const int t = x / Q, g = x % Q, e = i0 + r - p + t;
            double v = 0.0;
            if (kk < P && e >= 0 && e < TT.nel) {
                const double* base = vals + TT.val_off + ((int64_t)e * Q + g) * P;
                const double a = (type >> 1) ? base[nq * P + (p - t)] : base[p - t];
                const double b = (type & 1) ? base[nq * P + kk] : base[kk];
                v = a * b;
            }
            Tt[idx] = v;
        }
        for (int idx = tid; idx < nr * PQ; idx += NT) {
            const int x = idx % PQ, r = idx / PQ, t = x / Q, g = x % Q, e = i0 + r - p + t;
            phi[idx] = (e >= 0 && e < TT.nel) ? vals[TT.val_off + ((int64_t)e * Q + g) * P + (p - t)] : 0.0;
        }
    };
    build_T(TA, T.a0, na, Ta, phiA);
    build_T(TB, T.b0, nb, Tb, phiB);
    for (int idx = tid; idx < rows * P; idx += NT) RLs[idx] = 0.0;
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

    // ---- stage 3 (G3): rings in tensor memory --------------------------------
    const bool inG3 = tid >= G12;
    const int g3t = tid - G12;   // 0..127: TMEM lane 32 (warp % 4) + lane
    const uint32_t tbase = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    // item list: computed columns first (packed r*SAB + c_a*Sb + c_b, bit 30 =
    // POS0), then the others (bit 30 = DEAD); built once per tile
    __shared__ int s_cnt[2];
    int* s_list = reinterpret_cast<int*>(sm + L.oList);
    if (tid < 2) s_cnt[tid] = 0;
    __syncthreads();
    for (int it = tid; it < n3; it += NT) {
        const int cb = it % Sb, ca = (it / Sb) % Sa, r = it / SAB;
        const int cat = tile3_category(T.a0 + r % na, T.b0 + r / na, ca, cb, C.absm[ka], C.absm[kb], C.m[ka],
                                       C.m[kb], p);
        if (cat >= T3_POS) s_list[atomicAdd(&s_cnt[0], 1)] = it | (cat == T3_POS0 ? 1 << 30 : 0);
        else s_list[n3 - 1 - atomicAdd(&s_cnt[1], 1)] = it | (cat == T3_DEAD ? 1 << 30 : 0);
    }
    __syncthreads();
    const int npos = s_cnt[0];
    const int n3r = npos + rows;   // + one load-ring item per row (shared memory)
    const int nslot = (n3r + TILE3_G3 - 1) / TILE3_G3;   // <= NSLOT (host-checked)
    const int64_t rs_s = C.rs[ks], ss_s = C.ss[ks], rows_c = C.rows;
    const int absm_s = C.absm[ks], m_s = C.m[ks], S_s = C.S[ks];
    const int64_t nq_s = (int64_t)nel_s * Q;
    uint64_t l2keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(l2keep));
    if (inG3) {   // rings start at zero
        for (int k = 0; k < nslot; ++k)
#pragma unroll
            for (int c = 0; c < F::SC; c += 2) tm_st2(tbase + k * F::SC + c, 0.0);
        tm_wait_st();
    }

    // each stage-3 item's S2 offset (-1: dead column -- outside the band or on
    // the boundary -- whose stencil entries are written as zeros)
    int s2off[F::NSLOT];
#pragma unroll
    for (int k = 0; k < F::NSLOT; ++k) {
        const int i = g3t + TILE3_G3 * k;
        s2off[k] = -1;
        if (inG3 && i < npos) {
            const int it = s_list[i] & ((1 << 30) - 1);
            const int cb = it % Sb, ca = (it / Sb) % Sa, r = it / SAB;
            s2off[k] = (r * NU) * SAB + ca * Sb + cb;
        }
    }
    const bool prf = prof != nullptr && blockIdx.x == 0;
    long long gt0 = 0;
    if (prof != nullptr && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    long long pc0 = 0, pc1 = 0, pc2 = 0, pc3 = 0;
    const int n1 = nb * NI1 * XAv;
    // stage-2 work items (row, unit, column group): an absolute b axis (thin:
    // m_b <= 2p+1) enumerates its storage columns c_b only (w_b = c_b + 1 - i_b + p),
    // a relative one its 2p+1 offsets, one or two per item
    const int cw = T.cw;
    const int absm_b = C.absm[kb];
    // (symmetry: only columns with o_b >= 0, i.e. w_b >= p; a relative axis
    // starts its column groups at the even w_b = p & ~1 for aligned pair loads)
    const int wbs = cw == 2 ? (p & ~1) : p;
    const int ncol2 = absm_b ? Sb : (W - wbs + cw - 1) / cw;
    const int n2 = rows * NU * ncol2;
    if (!inG3) {
        for (int j = 0; j < nplanes; ++j) {
            const long long c0 = prf ? clock64() : 0;
            {
                // ---- wait for plane j ----------------------------------------
                {
                    const uint32_t par = (uint32_t)((j / TILE3_NPB) & 1);
                    const uint32_t ba = t3_smem_u32(&bar[j % TILE3_NPB]);
                    uint32_t ok = 0;
                    while (!ok)
                        asm volatile("{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
                                     " selp.u32 %0, 1, 0, q;\n}\n" : "=r"(ok) : "r"(ba), "r"(par) : "memory");
                }
                const double* Gw = sm + (j % TILE3_NPB) * L.sGw + tsh;
                if constexpr (TILE3_NS1 > 1) {   // plane j's stage-1 buffer
                    S1 = S1b + (j % TILE3_NS1) * (nb * NS1 * L.s1slot);
                    SL1 = SL1b + (j % TILE3_NS1) * (nb * T.xa);
                }
                // ---- stage 1: contract b -> S1[ib][slot][xa][w_b], SL1[ib][xa] --
                for (int it = tid; it < n1; it += G12) {
                    const int xa = it % XAv, q = it / XAv, sig = q % NI1, rb = q / NI1;
                    const int ib = T.b0 + rb;
                    const int tlo = max(0, p - ib), thi = min(P, nel_b + p - ib);
                    const int xoff = (ib - p - EB0) * Q;   // union row of the row's window point x = 0
                    if (sig < NS1) {
                        const double* gp = Gw + s_ent[sig] * L.est + xoff * xap + xa;
                        const double* tr = Tb + (rb * 4 + (DG ? c_t3d_btype[sig] : c_t3_btype[sig])) * PQ * RP;
                        double acc[W];
#pragma unroll
                        for (int w = 0; w < W; ++w) acc[w] = 0.0;
#pragma unroll
                        for (int t = 0; t < P; ++t) {
                            if (t < tlo || t >= thi) continue;
#pragma unroll
                            for (int g = 0; g < Q; ++g) {
                                const int x = t * Q + g;
                                const double gv = gp[x * xap];
                                double tv[RP];
#pragma unroll
                                for (int k2 = 0; k2 < RP / 2; ++k2) {
                                    const double2 v2 = *reinterpret_cast<const double2*>(tr + x * RP + 2 * k2);
                                    tv[2 * k2] = v2.x;
                                    tv[2 * k2 + 1] = v2.y;
                                }
#pragma unroll
                                for (int k = 0; k < P; ++k)
                                    if (t + k >= WBS1) acc[t + k] = fma(gv, tv[k], acc[t + k]);
                            }
                        }
                        double* o = S1 + (rb * NS1 + sig) * L.s1slot + xa * S1W - WBS1;
#pragma unroll
                        for (int w = WBS1; w < W; w += 2)
                            *reinterpret_cast<double2*>(o + w) = make_double2(acc[w], w + 1 < W ? acc[w + 1] : 0.0);
                    } else {
                        const double* gp = Gw + (NGE - 1) * L.est + xoff * xap + xa;
                        const double* ph = phiB + rb * PQ;
                        double acc = 0.0;
#pragma unroll
                        for (int t = 0; t < P; ++t) {
                            if (t < tlo || t >= thi) continue;
#pragma unroll
                            for (int g = 0; g < Q; ++g) acc = fma(gp[(t * Q + g) * xap], ph[t * Q + g], acc);
                        }
                        SL1[rb * T.xa + xa] = acc;
                    }
                }
                asm volatile("bar.sync 1, %0;\n" ::"r"(G12) : "memory");
                if (tid == 0 && j + TILE3_NPB < nplanes) issue_plane(j + TILE3_NPB);   // buffer j % NPB is free now
                // ---- stage 2: contract a -> S2[row][unit][c_a][c_b], S2L[row] -----
                const int jb = j % TILE3_NS2, ju = j / TILE3_NS2;   // S2 buffer and its use count
                if (ju >= 1) mb_wait(&s2empty[jb], (uint32_t)((ju - 1) & 1));   // stage 3 done with plane j - NS2
                double* S2w = S2 + jb * L.s2sz;
                auto stage2 = [&](auto CWc) {
                    constexpr int CW = decltype(CWc)::value;
                    for (int it = tid; it < n2 + rows; it += G12) {
                        if (it < n2) {
                            const int cg = it % ncol2, u = (it / ncol2) % NU, r = it / (ncol2 * NU);
                            const int ra = r % na, rb = r / na, ia = T.a0 + ra, ib = T.b0 + rb;
                            const int wb0 = absm_b ? cg + 1 - ib + p : wbs + CW * cg;   // first w_b of the item
                            if (wb0 < 0 || wb0 >= W) continue;   // column outside the band: dead stage-3 items
                            if (absm_b && wb0 < p) continue;     // o_b < 0: computed by the twin row
                            const int tlo = max(0, p - ia), thi = min(P, nel_a + p - ia);
                            const int xoff = (ia - p - EA0) * Q;
                            double acc0[W], acc1[W];
#pragma unroll
                            for (int w = 0; w < W; ++w) acc0[w] = acc1[w] = 0.0;
#pragma unroll
                            for (int pr = 0; pr < 2; ++pr) {
                                if (pr == 1 && (DG || u == 4)) break;
                                const int sl1 = DG ? c_t3d_uslot[u] : c_t3_uslot[u][pr];
                                const int at = DG ? c_t3d_uat[u] : c_t3_uat[u][pr];
                                const double* sp = S1 + (rb * NS1 + sl1) * L.s1slot + xoff * S1W + (wb0 - WBS1);
                                const double* ta = Ta + (ra * 4 + at) * PQ * RP;
#pragma unroll
                                for (int t = 0; t < P; ++t) {
                                    if (t < tlo || t >= thi) continue;
#pragma unroll
                                    for (int g = 0; g < Q; ++g) {
                                        const int x = t * Q + g;
                                        double2 v;
                                        if constexpr (CW == 2) v = *reinterpret_cast<const double2*>(sp + x * S1W);
                                        else v.x = sp[x * S1W];
                                        double tv[RP];
#pragma unroll
                                        for (int k2 = 0; k2 < RP / 2; ++k2) {
                                            const double2 v2 = *reinterpret_cast<const double2*>(ta + x * RP + 2 * k2);
                                            tv[2 * k2] = v2.x;
                                            tv[2 * k2 + 1] = v2.y;
                                        }
#pragma unroll
                                        for (int k = 0; k < P; ++k) {
                                            acc0[t + k] = fma(v.x, tv[k], acc0[t + k]);
                                            if constexpr (CW == 2) acc1[t + k] = fma(v.y, tv[k], acc1[t + k]);
                                        }
                                    }
                                }
                            }
                            // relative (w_a, w_b) -> storage columns (c_a, c_b)
                            double* o = S2w + (r * NU + u) * SAB;
#pragma unroll
                            for (int cc = 0; cc < CW; ++cc) {
                                const int wb = wb0 + cc;
                                const int cb = absm_b ? wb - p + ib - 1 : wb;
                                if (wb >= W || cb < 0 || cb >= Sb) continue;
#pragma unroll
                                for (int wa = 0; wa < W; ++wa) {
                                    const int ca = C.absm[ka] ? wa - p + ia - 1 : wa;
                                    if (ca >= 0 && ca < Sa) o[ca * Sb + cb] = cc == 0 ? acc0[wa] : acc1[wa];
                                }
                            }
                        } else {
                            const int r = it - n2, ra = r % na, rb = r / na, ia = T.a0 + ra;
                            const int tlo = max(0, p - ia), thi = min(P, nel_a + p - ia);
                            const double* sl = SL1 + rb * T.xa + (ia - p - EA0) * Q;
                            const double* ph = phiA + ra * PQ;
                            double acc = 0.0;
#pragma unroll
                            for (int t = 0; t < P; ++t) {
                                if (t < tlo || t >= thi) continue;
#pragma unroll
                                for (int g = 0; g < Q; ++g) acc = fma(sl[t * Q + g], ph[t * Q + g], acc);
                            }
                            S2w[NU * n3 + r] = acc;
                        }
                    }
                };
                if (cw == 2) stage2(std::integral_constant<int, 2>{});
                else stage2(std::integral_constant<int, 1>{});
                mb_arrive(&s2full[jb]);                               // plane j's S2 is written
                // S1 read: stage 1 of j+1 may write it (two S1 buffers: the
                // barrier after stage 1 of j+1 orders it before plane j+2's writes)
                if constexpr (TILE3_NS1 == 1) asm volatile("bar.sync 1, %0;\n" ::"r"(G12) : "memory");
            }
            if (prf && tid == 0) { pc0 += clock64() - c0; pc3 += 1; }
        }
    } else {
        for (int jj = 0; jj < nplanes; ++jj) {
            const long long c0 = prf ? clock64() : 0;
            const int jb = jj % TILE3_NS2;
            mb_wait(&s2full[jb], (uint32_t)((jj / TILE3_NS2) & 1));
            // ---- stage 3 (plane jj): stream axis, rank-1 updates ---------------------
            const int el = jj / Q, g = jj - el * Q, e = e_first + el;
            const double* S2r = S2 + jb * L.s2sz;
            double vb[P], db[P];
            {
                const double* bp = vals + TS.val_off + ((int64_t)e * Q + g) * P;
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    vb[k] = __ldg(bp + k);
                    db[k] = __ldg(bp + nq_s * P + k);
                }
            }
            const bool last_pt = g == Q - 1;
            const int nfl = e < e_last ? 1 : P;   // the last element completes rows e .. e + p
            const int emod = e % P;
#pragma unroll 1
            for (int k = 0; k < nslot; ++k) {
                const int i = g3t + TILE3_G3 * k;
                const uint32_t t3 = tbase + k * F::SC;    // element partial R3[al][bl]
                const uint32_t ta = t3 + F::R3C;          // ring: physical row h at ta + h * RC
                // R3 accumulates this element's Q planes; at the element's last
                // plane it is added to the ring window it touches -- stream row
                // e + al (physical row (e + al) mod P), offsets w = p - al .. 2p - al
                // (two-level sum: element partials, then elements, as the
                // reference's element-by-element assembly)
                double r3[P][P];
                tm_ld_r3<P>(t3, r3);
                tm_wait_ld();
                const bool item = i < npos;
                int s2o = s2off[0];   // (register select, no local-memory indexing)
#pragma unroll
                for (int kk = 1; kk < F::NSLOT; ++kk) s2o = k == kk ? s2off[kk] : s2o;
                if (s2o >= 0) {   // live item
                    const double* s2p = S2r + s2o;
                    // stream types 0 (no s), 1 (m, s), 2 (s, n), 3 (s, s); a diagonal
                    // metric has no type-1/2 pairs (their sums are exactly zero)
                    const double s0 = s2p[0] + s2p[SAB];
                    const double s1 = DG ? 0.0 : s2p[2 * SAB], s2v = DG ? 0.0 : s2p[3 * SAB];
                    const double s3 = DG ? s2p[2 * SAB] : s2p[4 * SAB];
#pragma unroll
                    for (int al = 0; al < P; ++al) {
                        const double c0 = DG ? vb[al] * s0 : fma(vb[al], s0, db[al] * s2v);
                        const double c1 = DG ? db[al] * s3 : fma(vb[al], s1, db[al] * s3);
#pragma unroll
                        for (int bl = 0; bl < P; ++bl) r3[al][bl] = fma(vb[bl], c0, fma(db[bl], c1, r3[al][bl]));
                    }
                }
                if (!last_pt) {
                    tm_st_r3<P>(t3, r3);
                } else {   // window row by row (registers): ring += R3, R3 = 0
#pragma unroll
                    for (int al = 0; al < P; ++al) {
                        const int h = emod + al < P ? emod + al : emod + al - P;
                        uint32_t wlo[P], whi[P];
#pragma unroll
                        for (int bl = 0; bl < P; ++bl) tm_ld2_issue(ta + h * F::RC + 2 * (bl - al + p), wlo[bl], whi[bl]);
                        tm_wait_ld();
#pragma unroll
                        for (int bl = 0; bl < P; ++bl) {
                            tm_st2(ta + h * F::RC + 2 * (bl - al + p), __hiloint2double((int)whi[bl], (int)wlo[bl]) + r3[al][bl]);
                            tm_st2(t3 + 2 * (al * P + bl), 0.0);
                        }
                    }
                }
                // (tcgen05 ops are warp-collective: the flush's TMEM traffic runs on
                // every lane, the global stores only for real items)
                if (last_pt) {   // element e complete: flush row e (+ the trailing rows), zero them
                    tm_wait_st();
                    const int le = item ? s_list[i] : 0;
                    const bool pos0 = (le >> 30) & 1;
                    const int it = le & ((1 << 30) - 1);
                    const int cb = it % Sb, ca = (it / Sb) % Sa, r = it / SAB;
                    const int ia = T.a0 + r % na, ib = T.b0 + r / na;
                    const int ja = C.absm[ka] ? ca + 1 : ia + ca - p, jb = C.absm[kb] ? cb + 1 : ib + cb - p;
                    const int64_t rowbase = (int64_t)(ia - 1) * C.rs[ka] + (int64_t)(ib - 1) * C.rs[kb];
                    const int64_t slotab = (int64_t)ca * C.ss[ka] + (int64_t)cb * C.ss[kb];
                    // the twin row (ja, jb) and this row's column slots in it
                    const int64_t rowbaseM = (int64_t)(ja - 1) * C.rs[ka] + (int64_t)(jb - 1) * C.rs[kb];
                    const int caM = C.absm[ka] ? ia - 1 : 2 * p - ca, cbM = C.absm[kb] ? ib - 1 : 2 * p - cb;
                    const int64_t slotabM = (int64_t)caM * C.ss[ka] + (int64_t)cbM * C.ss[kb];
                    for (int f = 0; f < nfl; ++f) {
                        const int h = emod + f < P ? emod + f : emod + f - P;
                        uint32_t rl[W], rh[W];
#pragma unroll
                        for (int w = 0; w < W; ++w) tm_ld2_issue(ta + h * F::RC + 2 * w, rl[w], rh[w]);
                        tm_wait_ld();
                        const int irow = e + f;
                        if (item && irow >= r0 && irow < r1) {
                            const int64_t row = rowbase + (int64_t)(irow - 1) * rs_s;
                            double* dst = stencil + C.mat_off + row;
#pragma unroll
                            for (int w = 0; w < W; ++w) {
                                const int jc = irow + w - p;
                                const bool inr = jc >= 1 && jc <= m_s;
                                const double v = __hiloint2double((int)rh[w], (int)rl[w]);
                                // own entry (the (0,0) column's o_s < 0 entries are its twins'
                                // mirrors; structural zeros are in place: stencil_zeroed)
                                if (inr && !(pos0 && w < p)) {
                                    const int cs = absm_s ? jc - 1 : w;
                                    st_keep(dst + ((int64_t)cs * ss_s + slotab) * rows_c, v, l2keep);
                                }
                                // mirrored entry A(twin, this row)
                                if (inr && !(pos0 && w <= p)) {
                                    const int csM = absm_s ? irow - 1 : 2 * p - w;
                                    st_keep(stencil + C.mat_off + rowbaseM + (int64_t)(jc - 1) * rs_s +
                                                ((int64_t)csM * ss_s + slotabM) * rows_c, v, l2keep);
                                }
                            }
                            if (pos0) dinv[C.vec_off + row] = 1.0 / __hiloint2double((int)rh[p], (int)rl[p]);
                        }
#pragma unroll
                        for (int w = 0; w < W; ++w) tm_st2(ta + h * F::RC + 2 * w, 0.0);   // becomes stream row e + f + P
                    }
                }
                if (!item && i < n3r) {   // load ring of row r (shared memory)
                    const int rr = i - npos;
                    double* RL = RLs + rr * P;
                    const double sl = S2r[NU * n3 + rr];
#pragma unroll
                    for (int al = 0; al < P; ++al) RL[al] = fma(vb[al], sl, RL[al]);
                    if (last_pt) {
                        const int ia2 = T.a0 + rr % na, ib2 = T.b0 + rr / na;
                        const int64_t rowbase = (int64_t)(ia2 - 1) * C.rs[ka] + (int64_t)(ib2 - 1) * C.rs[kb];
                        for (int f = 0; f < nfl; ++f) {
                            const int irow = e + f;
                            if (irow >= r0 && irow < r1) rhs[C.vec_off + rowbase + (int64_t)(irow - 1) * rs_s] = RL[0];
#pragma unroll
                            for (int al = 0; al < p; ++al) RL[al] = RL[al + 1];
                            RL[p] = 0.0;
                        }
                    }
                }
            }
            tm_wait_st();   // this plane's rings are in TMEM before the next plane loads them
            mb_arrive(&s2empty[jb]);                                  // plane jj's S2 is consumed
            if (prf && tid == G12) pc2 += clock64() - c0;
        }
    }
    __syncthreads();
    if (prf) {
        if (tid == 0) { prof[0] = pc0; prof[1] = pc1; }
        if (tid == G12) { prof[2] = pc2; prof[3] = pc3; }
    }
    if (prof != nullptr && tid == 0) {   // per-CTA timeline: start, end (ns), SM
        long long gt1;
        unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        prof[8 + 3 * blockIdx.x] = gt0;
        prof[9 + 3 * blockIdx.x] = gt1;
        prof[10 + 3 * blockIdx.x] = smid;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == G12 / 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(s_tmem) : "memory");
}

}  // namespace

bool tile3_eligible(const Handle* h) {
    return h->d == 3 && h->mu == 1 && h->q == h->p + 1 && (h->p == 3 || h->p == 4) && !h->opt.no_tma &&
           !h->opt.asm_pencil && !h->opt.generic_assembly && !h->force_generic_assembly;
}

// The metric G = det w J^-1 J^-T is diagonal -- G_ab = G_as = G_bs = 0.0
// exactly as k_metric computes them -- when the geometry is an axis-aligned
// box: degree 1 on [0, 1] per axis (basis derivatives exactly -1, +1, so the
// off-diagonal Jacobian sums cancel exactly), unit weights, control point
// coordinate i a function of index i only.  The tiled kernel then skips the
// off-diagonal pairs (their contributions are exact zeros: same bits).
bool metric_diagonal(const Handle* h) {
    if (h->d != 3 || h->opt.no_diag_metric) return false;
    for (int k = 0; k < 3; ++k) {
        if (h->geo.deg[k] != 1 || h->geo.n[k] != 2 || h->geo.nk[k] != 4) return false;
        const double* kv = h->geo_knots.data() + h->geo.knot_off[k];
        if (!(kv[0] == 0.0 && kv[1] == 0.0 && kv[2] == 1.0 && kv[3] == 1.0)) return false;
    }
    auto hw = [&](int a, int b, int c, int comp) { return h->geo_hw[(size_t)((a * 2 + b) * 2 + c) * 4 + comp]; };
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int c = 0; c < 2; ++c) {
                if (hw(a, b, c, 3) != 1.0) return false;
                if (hw(a, b, c, 0) != hw(a, 0, 0, 0) || hw(a, b, c, 1) != hw(0, b, 0, 1) ||
                    hw(a, b, c, 2) != hw(0, 0, c, 2))
                    return false;
            }
    return true;
}

#ifndef SGIGA_TILE3_C3
#define SGIGA_TILE3_C3 260.0    // cost model: cycles of one stage-3 item slot per plane
#endif
#ifndef SGIGA_TILE3_O12
#define SGIGA_TILE3_O12 300.0   // ... fixed cycles of the G12 part of an interval
#endif
#ifndef SGIGA_TILE3_OVH
#define SGIGA_TILE3_OVH 150.0   // ... fixed cycles of an interval
#endif
// Tile shapes, stream segments and tensor maps (host, once per component
// table).  Per component the tile (na x nb rows) minimises a per-row model of
// one barrier interval -- max(G12: stage 1 + stage 2, G3: stage 3), each
// stage max(work-item rounds x item length, FMAs / throughput) -- subject to
// the tensor-memory ring capacity and the shared-memory budget; the stream
// segment length minimises the estimated makespan max(longest tile, total /
// SMs); tiles are issued longest first.
static bool build_tiles3(Handle* h) {
    if (h->tiles3_state != 0) return h->tiles3_state > 0;
    h->tiles3_state = -1;
    if (!tile3_eligible(h)) return false;
    const int p = h->p, P = p + 1, Q = h->q, W = 2 * p + 1, NC2 = (W + 1) / 2;
    const int NSLOT = tile3_nslot(P);
    const size_t SMEM_CAP = 225 * 1024;
    const bool dg = metric_diagonal(h);
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
    const int segs[] = {96, 64, 48, 32, 24, 16, 12, 8};
    constexpr int NSEG = 8;

    struct Shape { int na, nb, ta, tb, xa, xap, xb, cw; double plane; };
    std::vector<Shape> shp(h->ncomp);
    std::vector<CUtensorMap> maps(h->ncomp);
    for (int c = 0; c < h->ncomp; ++c) {
        const CompInfo& C = h->comps[c];
        if (!C.rows || !C.tile3) continue;
        const int ka = C.ax[1], kb = C.ax[0], ks = C.ax[2];
        const int ma = C.m[ka], mb = C.m[kb], Sa = C.S[ka], Sb = C.S[kb];
        const int nel_a = C.nel[ka], nel_b = C.nel[kb];
        const int Ir = Sa * Sb;
        double best = 1e300;
        Shape bs{};
        for (int ta = 1; ta <= ma; ++ta) {
            const int na = (ma + ta - 1) / ta;
            if (ta > 1 && (ma + ta - 2) / (ta - 1) == na) continue;
            for (int tb = 1; tb <= mb; ++tb) {
                const int nb = (mb + tb - 1) / tb;
                if (tb > 1 && (mb + tb - 2) / (tb - 1) == nb) continue;
                const int rows = na * nb, n3 = rows * Ir;
                // computed (POS) stage-3 items of the fullest tile of this shape
                int npos = 0;
                for (int tbi = 0; tbi < tb; ++tbi)
                    for (int tai = 0; tai < ta; ++tai) {
                        const int a0 = 1 + (int)((int64_t)tai * ma / ta), a1 = 1 + (int)((int64_t)(tai + 1) * ma / ta);
                        const int b0 = 1 + (int)((int64_t)tbi * mb / tb), b1 = 1 + (int)((int64_t)(tbi + 1) * mb / tb);
                        int cnt = 0;
                        for (int ib = b0; ib < b1; ++ib)
                            for (int ia = a0; ia < a1; ++ia)
                                for (int ca = 0; ca < Sa; ++ca)
                                    for (int cb = 0; cb < Sb; ++cb)
                                        cnt += tile3_category(ia, ib, ca, cb, C.absm[ka], C.absm[kb], ma, mb, p) >= T3_POS;
                        npos = std::max(npos, cnt);
                    }
                if (npos + rows > TILE3_G3 * NSLOT) continue;
                const int xa = std::min(na + p, nel_a) * Q, xb = std::min(nb + p, nel_b) * Q;
                const int xap = (Q & 1) ? ((xa + 2) & ~1) : ((xa + 1) & ~1);
                if (xap > 256 || xb > 256) continue;
                const TLay L = tile3_layout(P, na, nb, xa, xap, xb, n3, dg);
                if ((size_t)L.total * 8 > SMEM_CAP) continue;
                const double xbw = std::min(P, nel_b) * Q, xaw = std::min(P, nel_a) * Q;
                // one barrier interval, in cycles: a work item's chain at ~2
                // cycles per FMA, the SM's sustained FP64 rate ~32 FMA / cycle
                auto stage = [&](double items, double nthr, double per_item) {
                    return std::max(std::ceil(items / nthr) * per_item * 2.0, items * per_item / 32.0);
                };
#ifndef SGIGA_TILE3_CW
                const int cw = C.absm[kb] || rows * 5 * W <= TILE3_G12 ? 1 : 2;
#else
                const int cw = C.absm[kb] ? 1 : SGIGA_TILE3_CW;
#endif
                const int wbs = cw == 2 ? (p & ~1) : p;
                const double n2 = (double)rows * 5 * (C.absm[kb] ? (Sb + 1) / 2 : (W - wbs + cw - 1) / cw);
                const double t12 = stage((double)nb * (dg ? 4 : 9) * xa, TILE3_G12, xbw * P) +
                                   stage(n2 * (dg ? 0.6 : 1.0), TILE3_G12, (dg ? 1.0 : 2.0) * xaw * P * cw) +
                                   SGIGA_TILE3_O12;
                const double t3 = std::ceil((npos + rows) / (double)TILE3_G3) * SGIGA_TILE3_C3 +
                                  (double)n3 / TILE3_G3 * 20.0;
                const double cost = std::max(t12, t3) + SGIGA_TILE3_OVH;
                const double per_row = cost / rows;
                if (per_row < best * 0.999) {
                    best = per_row;
                    bs = Shape{na, nb, ta, tb, xa, xap, xb, cw, cost};
                }
            }
        }
        if (best >= 1e299) return false;
        shp[c] = bs;
        const cuuint64_t Na = (cuuint64_t)C.nel[ka] * Q, Nb = (cuuint64_t)C.nel[kb] * Q, Ns = (cuuint64_t)C.nel[ks] * Q;
        if (C.qs[ka] != 1 || C.qs[kb] != (int64_t)Na || C.qs[ks] != (int64_t)(Na * Nb)) return false;
        const cuuint64_t dims[4] = {Na, Nb, Ns, (cuuint64_t)h->nG()};
        const cuuint64_t strides[3] = {Na * 8, Na * Nb * 8, (cuuint64_t)C.nqp * 8};
        const cuuint32_t box[4] = {(cuuint32_t)bs.xap, (cuuint32_t)bs.xb, 1, dg ? 1u : (cuuint32_t)h->nG()};
        if (strides[0] % 16 || strides[1] % 16 || strides[2] % 16 || (C.qp_off * 8) % 16) return false;
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (encode(&maps[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)(h->d_G + C.qp_off), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    // stream segment length: makespan model over the SMs (one CTA each)
    int nsm = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const double setup_planes = 6.0;
    int SEG = segs[0];
    {
        double bestspan = 1e300;
        for (int si = 0; si < NSEG; ++si) {
            const int cand = segs[si];
            double tot = 0, mx = 0;
            for (int c = 0; c < h->ncomp; ++c) {
                const CompInfo& C = h->comps[c];
                if (!C.rows || !C.tile3) continue;
                const int ks = C.ax[2], ms = C.m[ks], nel_s = C.nel[ks];
                const double ntile = (double)shp[c].ta * shp[c].tb;
                for (int r0 = 1; r0 < 1 + ms; r0 += cand) {
                    const int r1 = std::min(1 + ms, r0 + cand);
                    const int ne = std::min(r1 - 1, nel_s - 1) - std::max(0, r0 - p) + 1;
                    const double cost = (ne * Q + setup_planes) * shp[c].plane;
                    tot += cost * ntile;
                    mx = std::max(mx, cost);
                }
            }
            const double span = std::max(mx, tot / nsm);
            if (span < bestspan * 0.97) { bestspan = span; SEG = cand; }
        }
    }

    std::vector<Tile3> tl;
    std::vector<double> tcost;
    size_t smem = 0;
    for (int c = 0; c < h->ncomp; ++c) {
        const CompInfo& C = h->comps[c];
        if (!C.rows || !C.tile3) continue;
        const Shape& S = shp[c];
        const int ka = C.ax[1], kb = C.ax[0], ks = C.ax[2];
        const int ma = C.m[ka], mb = C.m[kb], ms = C.m[ks], nel_s = C.nel[ks];
        for (int tb = 0; tb < S.tb; ++tb) {
            const int b0 = 1 + (int)((int64_t)tb * mb / S.tb), b1 = 1 + (int)((int64_t)(tb + 1) * mb / S.tb);
            for (int ta = 0; ta < S.ta; ++ta) {
                const int a0 = 1 + (int)((int64_t)ta * ma / S.ta), a1 = 1 + (int)((int64_t)(ta + 1) * ma / S.ta);
                for (int r0 = 1; r0 < 1 + ms; r0 += SEG) {
                    Tile3 t;
                    t.comp = c;
                    t.a0 = a0; t.na = a1 - a0; t.b0 = b0; t.nb = b1 - b0;
                    t.r0 = r0; t.r1 = std::min(1 + ms, r0 + SEG);
                    t.xa = S.xa; t.xap = S.xap; t.xb = S.xb; t.cw = S.cw;
                    const int ne = std::min(t.r1 - 1, nel_s - 1) - std::max(0, t.r0 - p) + 1;
                    const TLay L = tile3_layout(P, t.na, t.nb, t.xa, t.xap, t.xb,
                                                t.na * t.nb * C.S[C.ax[1]] * C.S[C.ax[0]], dg);
                    smem = std::max(smem, (size_t)L.total * 8);
                    tl.push_back(t);
                    tcost.push_back((ne * Q + setup_planes) * S.plane);
                }
            }
        }
    }
    if (tl.empty() || smem > SMEM_CAP) return false;
    // FP64 operations the launch executes (FMA = 2): per plane, stage 1 --
    // 8 pair slots x valid a-window x valid b-window x P (+ load), stage 2 --
    // 9 pairs x executed w_b columns x valid a-window x P (+ load), stage 3 --
    // per live column 2 P^2 + 2 P FMAs + 2 P products + 1 sum (+ load ring),
    // and per element the ring fold (P^2 adds)
    double flops = 0.0;
    for (const Tile3& t : tl) {
        const CompInfo& C = h->comps[t.comp];
        const int ka = C.ax[1], kb = C.ax[0], ks = C.ax[2];
        const int nel_a = C.nel[ka], nel_b = C.nel[kb], nel_s = C.nel[ks];
        const int ne = std::min(t.r1 - 1, nel_s - 1) - std::max(0, t.r0 - p) + 1;
        if (ne <= 0) continue;
        auto win = [&](int i, int nel) { return (std::min(nel - 1, i) - std::max(0, i - p) + 1) * Q; };
        const int EA0 = std::max(0, t.a0 - p), EA1 = std::min(nel_a - 1, t.a0 + t.na - 1);
        const double XAv = (double)(EA1 - EA0 + 1) * Q;
        double s1 = 0.0, s2 = 0.0, s3 = 0.0;
        for (int rb = 0; rb < t.nb; ++rb) {   // stage 1: only the kept columns t + k >= p & ~1
            const int ib = t.b0 + rb;
            double fk = 0.0;
            for (int tt = std::max(0, p - ib); tt < std::min(P, nel_b + p - ib); ++tt)
                fk += Q * (P - std::max(0, (p & ~1) - tt));
            s1 += XAv * ((dg ? 3.0 : 8.0) * fk + win(ib, nel_b)) * 2.0;
        }
        const int Sa = C.S[ka], Sb = C.S[kb];
        for (int rb = 0; rb < t.nb; ++rb)
            for (int ra = 0; ra < t.na; ++ra) {
                const int ia = t.a0 + ra, ib = t.b0 + rb;
                int ncol = 0;   // stage-2 columns executed (o_b >= 0; pair groups padded)
                if (C.absm[kb]) {
                    for (int cb = 0; cb < Sb; ++cb) ncol += cb + 1 - ib >= 0 && cb + 1 - ib <= p;
                } else {
                    const int wbs = t.cw == 2 ? (p & ~1) : p;
                    ncol = t.cw * ((W - wbs + t.cw - 1) / t.cw);
                }
                s2 += ((dg ? 3.0 : 9.0) * ncol * P + 1.0) * win(ia, nel_a) * 2.0;
                for (int ca = 0; ca < Sa; ++ca)
                    for (int cb = 0; cb < Sb; ++cb)
                        if (tile3_category(ia, ib, ca, cb, C.absm[ka], C.absm[kb], C.m[ka], C.m[kb], p) >= T3_POS)
                            s3 += (2.0 * (2.0 * P * P + 2.0 * P) + 2.0 * P + 1.0) + (double)P * P / Q;
                s3 += 2.0 * P;   // load ring
            }
        flops += (s1 + s2 + s3) * ne * Q;
    }
    h->tiles3_flops = flops;
    std::vector<int> order(tl.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return tcost[x] > tcost[y]; });
    h->tiles3.resize(tl.size());
    for (size_t i = 0; i < order.size(); ++i) h->tiles3[i] = tl[order[i]];
    if (h->d_tiles3) { cudaFree(h->d_tiles3); h->d_tiles3 = nullptr; }
    if (h->d_tmaps3) { cudaFree(h->d_tmaps3); h->d_tmaps3 = nullptr; }
    if (cudaMalloc(&h->d_tiles3, sizeof(Tile3) * h->tiles3.size()) != cudaSuccess ||
        cudaMalloc(&h->d_tmaps3, sizeof(CUtensorMap) * h->ncomp) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (cudaMemcpyAsync(h->d_tiles3, h->tiles3.data(), sizeof(Tile3) * h->tiles3.size(), cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess ||
        cudaMemcpyAsync(h->d_tmaps3, maps.data(), sizeof(CUtensorMap) * h->ncomp, cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    h->tiles3_smem = smem;
    h->tiles3_dg = dg;
    h->asm_seg = SEG;
    h->tiles3_state = 1;
    return true;
}

// returns false when the plan has no tiled instantiation (the caller then
// runs k_assemble_fast)
bool launch_assembly_tile(Handle* h, cudaError_t* err) {
    if (!build_tiles3(h)) return false;
    const void* fn = nullptr;
    switch ((h->p + 1) * 2 + (h->tiles3_dg ? 1 : 0)) {
        case 8: fn = (const void*)k_assemble_tile<4, false>; break;
        case 9: fn = (const void*)k_assemble_tile<4, true>; break;
        case 10: fn = (const void*)k_assemble_tile<5, false>; break;
        case 11: fn = (const void*)k_assemble_tile<5, true>; break;
        default: return false;
    }
    *err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->tiles3_smem);
    if (*err != cudaSuccess) return true;
    // the kernel writes only the band's live entries: the structural zeros of
    // the stencil (columns outside the band or on the boundary) are set once
    // per layout (the buffer is rewritten by every pass, the zeros never change)
    if (!h->stencil_zeroed) {
        *err = cudaMemsetAsync(h->d_stencil, 0, sizeof(double) * (size_t)h->total_slots, h->stream);
        if (*err != cudaSuccess) return true;
        h->stencil_zeroed = true;
    }
    long long* prof = nullptr;
    const size_t nprof = 8 + 3 * h->tiles3.size();
    if (h->opt.asm_profile) {
        cudaMalloc(&prof, nprof * sizeof(long long));
        cudaMemsetAsync(prof, 0, nprof * sizeof(long long), h->stream);
    }
    void* args[] = {(void*)&h->d_comps, (void*)&h->d_tabs, (void*)&h->d_tiles3, (void*)&h->d_tabvals,
                    (void*)&h->d_stencil, (void*)&h->d_rhs, (void*)&h->d_dinv, (void*)&h->d_tmaps3, (void*)&prof};
    *err = cudaLaunchKernel(fn, dim3((unsigned)h->tiles3.size()), dim3(TILE3_THREADS), args, h->tiles3_smem,
                            h->stream);
    if (prof) {
        std::vector<long long> tv(nprof);
        long long* t = tv.data();
        cudaStreamSynchronize(h->stream);
        cudaMemcpy(t, prof, nprof * sizeof(long long), cudaMemcpyDeviceToHost);
        {   // timeline: makespan, SM busy fraction, busy time per tile class
            long long t0 = t[8], t1 = t[9];
            double busy = 0;
            std::vector<double> cls(64, 0.0);
            std::vector<int> ncls(64, 0);
            for (size_t b = 0; b < h->tiles3.size(); ++b) {
                t0 = std::min(t0, t[8 + 3 * b]);
                t1 = std::max(t1, t[9 + 3 * b]);
                const double d = (double)(t[9 + 3 * b] - t[8 + 3 * b]);
                busy += d;
                const Tile3& tt = h->tiles3[b];
                const CompInfo& C = h->comps[tt.comp];
                const int la = std::min(7, 31 - __builtin_clz(std::max(1, C.nel[C.ax[1]])));
                const int lb = std::min(7, 31 - __builtin_clz(std::max(1, C.nel[C.ax[0]])));
                cls[la * 8 + lb] += d;
                ncls[la * 8 + lb] += 1;
            }
            int nsm = 148;
            fprintf(stderr, "asm-tile timeline: makespan %.3f ms, SM busy %.1f%%; busy ms by (log2 nel_a, log2 nel_b):",
                    (t1 - t0) * 1e-6, 100.0 * busy / ((double)nsm * (t1 - t0)));
            for (int c = 0; c < 64; ++c)
                if (ncls[c]) fprintf(stderr, " (%d,%d):%.2f/%d", c / 8, c % 8, cls[c] * 1e-6 / nsm, ncls[c]);
            fprintf(stderr, "\n");
        }
        const double n = t[3] > 0 ? (double)t[3] : 1.0;
        const Tile3& t0 = h->tiles3[0];
        fprintf(stderr, "asm-tile block0 comp=%d rows=%dx%d cw=%d intervals=%lld cycles/interval: G12 work=%.0f "
                "barrier=%.0f | G3 work=%.0f ; tiles=%zu seg=%d smem=%zu\n", t0.comp, t0.na, t0.nb, t0.cw, t[3],
                t[0] / n, t[1] / n, t[2] / n, h->tiles3.size(), h->asm_seg, h->tiles3_smem);
        cudaFree(prof);
    }
    h->launches[0] += 1;
    return true;
}

}  // namespace sgiga
