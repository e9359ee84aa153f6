// k_assembly_box.cu -- kernel 2 for axis-aligned box geometries (3-D):
// the stiffness by Kronecker factors, the load by a three-stage sum
// factorisation.
//
// Reference: _assemble_full / local_poisson_systems (S/assembly.py:264-354,
// S/_kernels/_compiled.pyx:48-90) with the metric of assembly.py:286-294.
// On a box (metric_diagonal: degree-1 axis-separable map, unit weights) the
// map is x_k = c0_k + L_k xi_k, so G = det w J^-1 J^-T = diag(g_k w) with the
// per-patch constants g_k = det / L_k^2 and the tensor-product weight
// w = w_0 w_1 w_2.  The quadrature sum of the stiffness then factorises
// exactly (same points, same weights, regrouped):
//   A(i, j) = sum_k g_k  K_k(i_k, j_k) prod_{l != k} M_l(i_l, j_l),
//   M(i, j) = sum_e sum_g w N_i N_j,   K(i, j) = sum_e sum_g w N_i' N_j'
// (1-D banded tables per analysis knot vector, k_box_tables), and the
// assembly is one pass writing the band's live stencil entries -- bound by
// the HBM store bandwidth of the stencil itself (8 B per live entry).  The
// load b_i = sum_x f(x) det w(x) N_i(x) keeps the forcing at every
// quadrature point (k_metric_box writes f det w) and is contracted one axis
// at a time (a, then b, then the stream axis s: k_rhs_box_stage x3).
// Rounding-level differences from the element-by-element sums; the matrix is
// exactly symmetric (the 1-D tables are, and every entry is the same
// expression of its factors).  SGIGA_NO_BOX_ASM keeps the tiled kernel.
#include <algorithm>
#include <vector>

#include "handle.cuh"

namespace sgiga {

namespace {

constexpr int BOX_THREADS = 256;
#ifndef SGIGA_BOX_MINB
#define SGIGA_BOX_MINB 2   // resident CTAs per SM of k_stencil_box: 2 (109 registers, no spills) measured best -- cfg5 assembly 1.09 / 1.04 / 1.17 / 1.28 ms at 3 / 2 / 4 / 6
#endif

struct BoxStage {
    int tab;             // TabInfo of the contracted axis
    int cdim;            // contracted output dim (extent = interior functions)
    int n[3];            // output extents in thread order (n[2] fastest)
    int pad;
    int64_t in_off, out_off;
    int64_t in_str[3];   // input stride per output dim (contracted: of the quadrature index)
    int64_t out_str[3];
};
struct BoxWork {         // one CTA: BOX_THREADS consecutive outputs of an entry
    int ent, pad;
    int64_t first;
};

// M and K band of every interior function: box1d[2 (tcum[t] + i W + o) + {0, 1}],
// column j = i + o - p (zero outside [0, m)).  The element range and the
// products are symmetric in (i, j): M(i, j) and M(j, i) are the same bits.
__global__ void k_box_tables(const TabInfo* __restrict__ tabs, int ntab, const int64_t* __restrict__ tcum,
                             int p, int mu, int q, const double* __restrict__ vals, const double* __restrict__ qw,
                             double* __restrict__ box1d) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= tcum[ntab]) return;
    int lo = 0, hi = ntab;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tcum[mid] <= gid) lo = mid; else hi = mid;
    }
    const TabInfo T = tabs[lo];
    const int W = 2 * p + 1, P = p + 1;
    const int64_t loc = gid - tcum[lo];
    const int i = (int)(loc / W), o = (int)(loc % W), m = T.n - 2, j = i + o - p;
    double M = 0.0, K = 0.0;
    if (j >= 0 && j < m) {
        const int f = i + 1, g = j + 1, fl = min(f, g), fh = max(f, g);
        // elements whose active functions [e mu, e mu + p] hold both
        const int e0 = fh - p <= 0 ? 0 : (fh - p + mu - 1) / mu;
        const int e1 = min(T.nel - 1, fl / mu);
        const int64_t nq = (int64_t)T.nel * q;
        const double* V = vals + T.val_off;
        const double* Dv = V + nq * P;
        for (int e = e0; e <= e1; ++e)
            for (int gq = 0; gq < q; ++gq) {
                const int64_t x = (int64_t)e * q + gq;
                const double w = qw[T.qp_off + x];
                const int lf = f - e * mu, lg = g - e * mu;
                M = __fma_rn(w, __dmul_rn(V[x * P + lf], V[x * P + lg]), M);
                K = __fma_rn(w, __dmul_rn(Dv[x * P + lf], Dv[x * P + lg]), K);
            }
    }
    box1d[2 * gid] = M;
    box1d[2 * gid + 1] = K;
}

// One thread per interior row (PCG chunks: 256 rows of one component), all
// live band entries of the row.  Internal axis order j = 0 (outer) .. 2
// (stream, slot stride 1): consecutive threads = consecutive stream rows,
// so every store instruction of a warp writes one contiguous 256-byte run.
template <int P>
__global__ void __launch_bounds__(BOX_THREADS, SGIGA_BOX_MINB)
k_stencil_box(const CompInfo* __restrict__ comps, const Chunk* __restrict__ chunks,
              const int64_t* __restrict__ tcum, const double* __restrict__ box1d, double3 gk,
              double* __restrict__ stencil, double* __restrict__ dinv) {
    constexpr int p = P - 1, W = 2 * p + 1;
    const Chunk ch = chunks[blockIdx.x];
    if ((int)threadIdx.x >= ch.nrow) return;
    const CompInfo& C = comps[ch.comp];
    const int row = ch.row0 + (int)threadIdx.x;
    const int64_t R = C.rows;
    // the row's band along the stream axis in registers (the unrolled inner
    // loop); the two outer factors are read per iteration (L1 hits) -- only
    // the inner loop is unrolled: a fully unrolled W^3 body overflowed the
    // instruction cache (85 % no_instruction stalls)
    double Ms[W], Ks[W], g[3];
    int ik[3], mk[3], absk[3];
    int64_t ssk[3];
    const double2* bb[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int k = C.ax[j];
        mk[j] = C.m[k];
        absk[j] = C.absm[k];
        ssk[j] = C.ss[k];
        ik[j] = (row / (int)C.rs[k]) % mk[j];
        bb[j] = reinterpret_cast<const double2*>(box1d) + tcum[C.tab[k]] + (int64_t)ik[j] * W;
        g[j] = k == 0 ? gk.x : (k == 1 ? gk.y : gk.z);
    }
#pragma unroll
    for (int o = 0; o < W; ++o) {
        const double2 v = __ldg(bb[2] + o);
        Ms[o] = v.x;
        Ks[o] = v.y;
    }
    double* out = stencil + C.mat_off + row;
#pragma unroll 1
    for (int o0 = 0; o0 < W; ++o0) {
        const int c0 = ik[0] + o0 - p;
        if (c0 < 0 || c0 >= mk[0]) continue;   // structural zero (set once per layout)
        const int64_t t0 = (int64_t)(absk[0] ? c0 : o0) * ssk[0];
        const double2 f0 = __ldg(bb[0] + o0);
#pragma unroll 1
        for (int o1 = 0; o1 < W; ++o1) {
            const int c1 = ik[1] + o1 - p;
            if (c1 < 0 || c1 >= mk[1]) continue;
            const int64_t t1 = t0 + (int64_t)(absk[1] ? c1 : o1) * ssk[1];
            const double2 f1 = __ldg(bb[1] + o1);
            // A = (g_0 K_0 M_1 + g_1 M_0 K_1) M_2 + g_2 M_0 M_1 K_2: the same
            // expression of the (symmetric) factors for every entry
            const double ab = __dadd_rn(__dmul_rn(g[0], __dmul_rn(f0.y, f1.x)), __dmul_rn(g[1], __dmul_rn(f0.x, f1.y)));
            const double cc = __dmul_rn(g[2], __dmul_rn(f0.x, f1.x));
            double* o = out + t1 * R;
            const bool diag01 = o0 == p && o1 == p;
#pragma unroll
            for (int o2 = 0; o2 < W; ++o2) {
                const int c2 = ik[2] + o2 - p;
                if (c2 < 0 || c2 >= mk[2]) continue;
                const double v = __fma_rn(ab, Ms[o2], __dmul_rn(cc, Ks[o2]));
                o[(int64_t)(absk[2] ? c2 : o2) * R] = v;
                if (o2 == p && diag01) dinv[C.vec_off + row] = 1.0 / v;
            }
        }
    }
}

// One axis of the load's sum factorisation: out[u] = sum over the
// quadrature points x of the support of interior function u[cdim]
// of in[...x...] N_{u[cdim]+1}(x).
// QT = quadrature points per element at compile time (0: run-time q): the
// g loop is unrolled, QT loads in flight per thread instead of one (same
// operations and order).
template <int QT>
__global__ void __launch_bounds__(BOX_THREADS)
k_rhs_box_stage(const BoxStage* __restrict__ ents, const BoxWork* __restrict__ work,
                const TabInfo* __restrict__ tabs, const double* __restrict__ vals, int p, int mu, int q,
                const double* __restrict__ in, double* __restrict__ out) {
    const BoxWork wk = work[blockIdx.x];
    const BoxStage& S = ents[wk.ent];
    const int64_t u = wk.first + threadIdx.x;
    const int n1 = S.n[1], n2 = S.n[2];
    const int64_t tot = (int64_t)S.n[0] * n1 * n2;
    if (u >= tot) return;
    int uu[3];
    if (tot <= 0x7fffffff) {   // 32-bit index arithmetic (always, in practice)
        const unsigned ul = (unsigned)u, t1 = ul / (unsigned)n2;
        uu[2] = (int)(ul - t1 * (unsigned)n2);
        uu[0] = (int)(t1 / (unsigned)n1);
        uu[1] = (int)(t1 - (unsigned)uu[0] * (unsigned)n1);
    } else {
        uu[2] = (int)(u % n2);
        uu[1] = (int)((u / n2) % n1);
        uu[0] = (int)(u / ((int64_t)n1 * n2));
    }
    const int cd = S.cdim;
    int64_t ib = S.in_off, ob = S.out_off;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        ob += uu[d] * S.out_str[d];
        if (d != cd) ib += uu[d] * S.in_str[d];
    }
    const TabInfo& T = tabs[S.tab];
    const int P = p + 1, f = (cd == 0 ? uu[0] : (cd == 1 ? uu[1] : uu[2])) + 1;   // (no dynamic register index)
    const int e0 = f - p <= 0 ? 0 : (f - p + mu - 1) / mu;
    const int e1 = min(T.nel - 1, f / mu);
    const double* V = vals + T.val_off;
    const int64_t cs = S.in_str[cd];
    const int qq = QT ? QT : q;
    double acc = 0.0;
    for (int e = e0; e <= e1; ++e) {
        const double* ip = in + ib + (int64_t)e * qq * cs;
        const double* vp = V + (int64_t)e * qq * P + f - e * mu;
        if constexpr (QT > 0) {
            double a[QT], b[QT];
#pragma unroll
            for (int g = 0; g < QT; ++g) { a[g] = ip[g * cs]; b[g] = vp[g * P]; }
#pragma unroll
            for (int g = 0; g < QT; ++g) acc = __fma_rn(a[g], b[g], acc);
        } else {
            for (int g = 0; g < qq; ++g) acc = __fma_rn(ip[g * cs], vp[g * P], acc);
        }
    }
    out[ob] = acc;
}

}  // namespace

bool box_assembly_eligible(const Handle* h) {
    return h->d == 3 && !h->opt.no_box_asm && !h->opt.no_box_metric && !h->opt.asm_pencil &&
           !h->opt.generic_assembly && !h->force_generic_assembly && h->p >= 1 && h->p <= 4 && metric_diagonal(h);
}

// host tables of the box path (once per layout): band offsets per knot
// vector, the three load stages per component and their CTA work lists,
// the stage buffers
static bool build_box(Handle* h) {
    if (h->box_state != 0) return h->box_state > 0;
    h->box_state = -1;
    if (!box_assembly_eligible(h)) return false;
    const int p = h->p, W = 2 * p + 1, q = h->q, ntab = (int)h->tabs.size();
    std::vector<int64_t> tcum(ntab + 1, 0);
    for (int t = 0; t < ntab; ++t) tcum[t + 1] = tcum[t] + (int64_t)std::max(0, h->tabs[t].n - 2) * W;
    std::vector<BoxStage> ents;
    std::vector<BoxWork> work[3];
    int64_t x1 = 0, x2 = 0;
    const int nG = h->nG();
    for (int c = 0; c < h->ncomp; ++c) {
        const CompInfo& C = h->comps[c];
        if (C.rows == 0) continue;
        const int b = C.ax[0], a = C.ax[1], s = C.ax[2];
        const int nqa = C.nel[a] * q, nqb = C.nel[b] * q, nqs = C.nel[s] * q;
        const int ma = C.m[a], mb = C.m[b], ms = C.m[s];
        BoxStage A{}, B{}, S3{};
        A.tab = C.tab[a]; A.cdim = 2;
        A.n[0] = nqs; A.n[1] = nqb; A.n[2] = ma;
        A.in_off = C.qp_off + (int64_t)(nG - 1) * C.nqp;   // the load entry f det w
        A.in_str[0] = C.qs[s]; A.in_str[1] = C.qs[b]; A.in_str[2] = C.qs[a];
        A.out_off = x1;
        A.out_str[0] = (int64_t)nqb * ma; A.out_str[1] = ma; A.out_str[2] = 1;
        B.tab = C.tab[b]; B.cdim = 1;
        B.n[0] = nqs; B.n[1] = mb; B.n[2] = ma;
        B.in_off = x1;
        B.in_str[0] = (int64_t)nqb * ma; B.in_str[1] = ma; B.in_str[2] = 1;
        B.out_off = x2;
        B.out_str[0] = (int64_t)mb * ma; B.out_str[1] = ma; B.out_str[2] = 1;
        S3.tab = C.tab[s]; S3.cdim = 2;
        S3.n[0] = mb; S3.n[1] = ma; S3.n[2] = ms;
        S3.in_off = x2;
        S3.in_str[0] = ma; S3.in_str[1] = 1; S3.in_str[2] = (int64_t)mb * ma;
        S3.out_off = C.vec_off;
        S3.out_str[0] = C.rs[b]; S3.out_str[1] = C.rs[a]; S3.out_str[2] = C.rs[s];
        x1 += (int64_t)nqs * nqb * ma;
        x2 += (int64_t)nqs * mb * ma;
        const BoxStage st[3] = {A, B, S3};
        for (int k = 0; k < 3; ++k) {
            const int e = (int)ents.size();
            ents.push_back(st[k]);
            const int64_t n = (int64_t)st[k].n[0] * st[k].n[1] * st[k].n[2];
            for (int64_t f = 0; f < n; f += BOX_THREADS) work[k].push_back(BoxWork{e, 0, f});
        }
    }
    for (int k = 0; k < 3; ++k) h->box_nwork[k] = (int)work[k].size();
    std::vector<BoxWork> wall;
    for (int k = 0; k < 3; ++k) wall.insert(wall.end(), work[k].begin(), work[k].end());
    auto al = [](void** p, size_t bytes) { return cudaMalloc(p, std::max<size_t>(bytes, 16)) == cudaSuccess; };
    if (!al((void**)&h->d_box1d, sizeof(double) * 2 * tcum[ntab]) ||
        !al((void**)&h->d_box_tcum, sizeof(int64_t) * tcum.size()) ||
        !al(&h->d_box_stage, sizeof(BoxStage) * ents.size()) || !al(&h->d_box_work, sizeof(BoxWork) * wall.size()) ||
        !al((void**)&h->d_box_x1, sizeof(double) * x1) || !al((void**)&h->d_box_x2, sizeof(double) * x2)) {
        cudaGetLastError();
        return false;
    }
    if (cudaMemcpyAsync(h->d_box_tcum, tcum.data(), sizeof(int64_t) * tcum.size(), cudaMemcpyHostToDevice,
                        h->stream) != cudaSuccess ||
        (!ents.empty() && cudaMemcpyAsync(h->d_box_stage, ents.data(), sizeof(BoxStage) * ents.size(),
                                          cudaMemcpyHostToDevice, h->stream) != cudaSuccess) ||
        (!wall.empty() && cudaMemcpyAsync(h->d_box_work, wall.data(), sizeof(BoxWork) * wall.size(),
                                          cudaMemcpyHostToDevice, h->stream) != cudaSuccess) ||
        cudaStreamSynchronize(h->stream) != cudaSuccess)
        return false;
    h->box_tab_total = tcum[ntab];
    h->box_state = 1;
    return true;
}

bool box_assembly_ready(Handle* h) { return build_box(h); }

// FD metric scales c_k of a box: G_kk = g_k w exactly, and the quadrature
// weights sum to the unit parameter volume, so c_k = sum_x G_kk(x) = g_k
// (the FD preconditioner is then the exact inverse of the Kronecker
// stiffness up to rounding); replaces k_fd_metric_scale's quadrature sums
__global__ void k_fd_box_scale(int n, double3 g, double* __restrict__ ckg) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k = i % MAXD;
    ckg[i] = k == 0 ? g.x : (k == 1 ? g.y : (k == 2 ? g.z : 0.0));
}

cudaError_t launch_fd_box_scale(Handle* h, cudaStream_t s) {
    double c0[3], L[3], g[3], det;
    box_constants(h, c0, L, g, &det);
    const int n = h->ncomp * MAXD;
    if (n > 0) k_fd_box_scale<<<(n + 127) / 128, 128, 0, s>>>(n, make_double3(g[0], g[1], g[2]), h->d_ck);
    h->launches[0]++;
    return cudaGetLastError();
}

void free_box(Handle* h) {
    void* ptrs[] = {h->d_box1d, h->d_box_tcum, h->d_box_stage, h->d_box_work, h->d_box_x1, h->d_box_x2};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    h->d_box1d = nullptr; h->d_box_tcum = nullptr; h->d_box_stage = nullptr; h->d_box_work = nullptr;
    h->d_box_x1 = nullptr; h->d_box_x2 = nullptr;
    h->box_state = 0;
}

bool launch_assembly_box(Handle* h, cudaError_t* err) {
    if (!build_box(h)) return false;
    // only live entries are written: the structural zeros are set once per layout
    if (!h->stencil_zeroed) {
        *err = cudaMemsetAsync(h->d_stencil, 0, sizeof(double) * (size_t)h->total_slots, h->stream);
        if (*err != cudaSuccess) return true;
        h->stencil_zeroed = true;
    }
    const int ntab = (int)h->tabs.size();
    if (h->box_tab_total > 0)
        k_box_tables<<<(unsigned)((h->box_tab_total + 127) / 128), 128, 0, h->stream>>>(
            h->d_tabs, ntab, h->d_box_tcum, h->p, h->mu, h->q, h->d_tabvals, h->d_qw, h->d_box1d);
    double c0[3], L[3], g[3], det;
    box_constants(h, c0, L, g, &det);
    const unsigned nch = (unsigned)h->chunks.size();
    if (nch > 0) {
        const double3 gk = make_double3(g[0], g[1], g[2]);
        switch (h->p + 1) {
            case 2: k_stencil_box<2><<<nch, BOX_THREADS, 0, h->stream>>>(h->d_comps, h->d_chunks, h->d_box_tcum, h->d_box1d, gk, h->d_stencil, h->d_dinv); break;
            case 3: k_stencil_box<3><<<nch, BOX_THREADS, 0, h->stream>>>(h->d_comps, h->d_chunks, h->d_box_tcum, h->d_box1d, gk, h->d_stencil, h->d_dinv); break;
            case 4: k_stencil_box<4><<<nch, BOX_THREADS, 0, h->stream>>>(h->d_comps, h->d_chunks, h->d_box_tcum, h->d_box1d, gk, h->d_stencil, h->d_dinv); break;
            default: k_stencil_box<5><<<nch, BOX_THREADS, 0, h->stream>>>(h->d_comps, h->d_chunks, h->d_box_tcum, h->d_box1d, gk, h->d_stencil, h->d_dinv); break;
        }
    }
    const BoxStage* ents = (const BoxStage*)h->d_box_stage;
    const BoxWork* w = (const BoxWork*)h->d_box_work;
    const double* ins[3] = {h->d_G, h->d_box_x1, h->d_box_x2};
    double* outs[3] = {h->d_box_x1, h->d_box_x2, h->d_rhs};
    int64_t wo = 0;
    for (int k = 0; k < 3; ++k) {
        if (h->box_nwork[k] > 0) {
#define RHS_STAGE(QT)                                                                       \
    k_rhs_box_stage<QT><<<(unsigned)h->box_nwork[k], BOX_THREADS, 0, h->stream>>>(          \
        ents, w + wo, h->d_tabs, h->d_tabvals, h->p, h->mu, h->q, ins[k], outs[k])
            switch (h->q) {
                case 2: RHS_STAGE(2); break;
                case 3: RHS_STAGE(3); break;
                case 4: RHS_STAGE(4); break;
                case 5: RHS_STAGE(5); break;
                default: RHS_STAGE(0); break;
            }
#undef RHS_STAGE
        }
        wo += h->box_nwork[k];
    }
    h->launches[0] += 5;
    *err = cudaGetLastError();
    return true;
}

}  // namespace sgiga
