// k_pcg.cu -- kernel 3: batched Jacobi-preconditioned CG over all
// components of a plan, plus the post-solve residual acceptance check and
// the expansion to full coefficient vectors.
//
// Reference: linsolve.solve_spd (linsolve.py:16-54) -- a direct SuperLU
// solve; SPEC.md:231 allows Jacobi-CG instead.  Residual acceptance
// ||Ax-b|| <= 1e-10 ||b|| (linsolve.py:49-53), zero-rhs shortcut (43-45),
// expand with zero boundary (assembly.py:202-206).
//
// Two regimes:
//  * small components (rows <= SMALL_ROWS): one CTA per component runs the
//    whole CG loop with all vectors in shared memory (no grid syncs);
//  * large components: row chunks of 256, three fused kernels per
//    iteration, per-component scalars reduced by the last chunk to finish
//    (fixed chunk order -> deterministic), iterations replayed as CUDA
//    graphs with the convergence test on the device.
#include "handle.cuh"

namespace sgiga {

constexpr int SMALL_ROWS = 2048;
constexpr int SMALL_THREADS = 1024;
constexpr int CHUNK_ROWS = 256;
constexpr int GRAPH_ITERS = 16;

// column offset of slot component s_k along original axis k for row index r_k
__device__ __forceinline__ int64_t col_contrib(const CompInfo& C, int k, int sk, int rk, int p) {
    return (int64_t)(C.absm[k] ? (sk - rk) : (sk - p)) * C.rs[k];
}

// y(row) = sum_slots A(row, slot) * v(col(row, slot)); v indexed from the
// component's padded base.  Slots split across `lanes` threads.
template <int D>
__device__ __forceinline__ double spmv_row(const CompInfo& C, const double* __restrict__ val,
                                           const double* __restrict__ v, int64_t row, int p,
                                           int lane, int lanes) {
    int r[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < D; ++k) r[k] = (int)((row / C.rs[k]) % C.m[k]);
    int S0 = C.S[0], S1 = D > 1 ? C.S[1] : 1, S2 = D > 2 ? C.S[2] : 1;
    int64_t ns = (int64_t)S0 * S1 * S2;
    double acc = 0.0;
    for (int64_t t = lane; t < ns; t += lanes) {
        int s2 = (int)(t % S2), s1 = (int)((t / S2) % S1), s0 = (int)(t / ((int64_t)S1 * S2));
        int64_t col = row + col_contrib(C, 0, s0, r[0], p);
        int64_t slot = (int64_t)s0 * C.ss[0];
        if (D > 1) { col += col_contrib(C, 1, s1, r[1], p); slot += (int64_t)s1 * C.ss[1]; }
        if (D > 2) { col += col_contrib(C, 2, s2, r[2], p); slot += (int64_t)s2 * C.ss[2]; }
        acc += __ldg(&val[slot * C.rows + row]) * v[col];
    }
    return acc;
}

// deterministic block reduction of NV values (fixed shuffle tree + fixed
// warp order); result broadcast to all threads.
template <int NV>
__device__ __forceinline__ void block_sum(double* v, double* red /* [32*NV] */) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) red[k * 32 + w] = v[k];
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = lane < nw ? red[k * 32 + lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) red[k * 32] = t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = red[k * 32];
    __syncthreads();
}

// ---------------------------------------------------------------------------
// small path: whole PCG in one CTA
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SMALL_THREADS)
k_pcg_small(const CompInfo* __restrict__ comps, const int* __restrict__ list,
            const double* __restrict__ stencil, const double* __restrict__ rhs,
            const double* __restrict__ dinv, double* __restrict__ xout, CgState* __restrict__ st,
            int p, double rtol2, int maxit) {
    extern __shared__ double sm[];
    const int c = list[blockIdx.x];
    const CompInfo C = comps[c];
    const int64_t R = C.rows, H = C.halo;
    double* xs = sm;
    double* rs_ = xs + R;
    double* zs = rs_ + R;
    double* ds = zs + R;
    double* qv = ds + R;
    double* pe = qv + R;          // [H + R + H]
    double* red = pe + R + 2 * H; // [32*2]
    double* ps = pe + H;
    const double* val = stencil + C.mat_off;
    const double* b = rhs + C.vec_off;
    const double* di = dinv + C.vec_off;
    const int tid = threadIdx.x, nth = blockDim.x;
    int lanes = 1;
    while (lanes < 32 && lanes * 2 * R <= nth) lanes *= 2;
    const int groups = nth / lanes, grp = tid / lanes, lane = tid % lanes;

    double v2[2] = {0.0, 0.0};
    for (int64_t i = tid; i < H; i += nth) { pe[i] = 0.0; pe[H + R + i] = 0.0; }
    for (int64_t i = tid; i < R; i += nth) {
        double bi = b[i], d = di[i], z = d * bi;
        xs[i] = 0.0; rs_[i] = bi; ds[i] = d; zs[i] = z; ps[i] = z;
        v2[0] += bi * z;
        v2[1] += bi * bi;
    }
    block_sum<2>(v2, red);
    double rho = v2[0], bb = v2[1];
    int it = 0, conv = (bb == 0.0);
    while (!conv && it < maxit) {
        // q = A p ; p.q
        double pq[1] = {0.0};
        for (int64_t base = 0; base < R; base += groups) {   // warp-uniform trip count
            int64_t row = base + grp;
            double y = row < R ? spmv_row<D>(C, val, ps, row, p, lane, lanes) : 0.0;
            for (int o = lanes >> 1; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
            if (lane == 0 && row < R) { qv[row] = y; pq[0] += ps[row] * y; }
        }
        block_sum<1>(pq, red);
        double alpha = rho / pq[0];
        double w[2] = {0.0, 0.0};
        for (int64_t i = tid; i < R; i += nth) {
            double xi = xs[i] + alpha * ps[i];
            double ri = rs_[i] - alpha * qv[i];
            double zi = ds[i] * ri;
            xs[i] = xi; rs_[i] = ri; zs[i] = zi;
            w[0] += ri * ri;
            w[1] += ri * zi;
        }
        block_sum<2>(w, red);
        ++it;
        if (w[0] <= rtol2 * bb) { conv = 1; break; }
        double beta = w[1] / rho;
        rho = w[1];
        for (int64_t i = tid; i < R; i += nth) ps[i] = zs[i] + beta * ps[i];
        __syncthreads();
    }
    for (int64_t i = tid; i < R; i += nth) xout[C.vec_off + i] = xs[i];
    if (tid == 0) {
        st[c].it = it;
        st[c].conv = conv;
        st[c].active = 0;
        st[c].bb = bb;
    }
}

// ---------------------------------------------------------------------------
// large path: chunked kernels
// ---------------------------------------------------------------------------
struct ChunkCtx {
    const CompInfo* comps;
    const Chunk* chunks;
    const double* stencil;
    const double* rhs;
    const double* dinv;
    double *x, *r, *z, *p, *q;
    CgState* st;
    double* part;
    int* active_count;
    int p_deg;
    double rtol2;
    int maxit;
};

// last chunk of a component to finish reduces the partials (chunk order)
template <int NV>
__device__ __forceinline__ bool finish_component(const ChunkCtx& X, const Chunk& ch,
                                                 const CompInfo& C, double* v, double* out,
                                                 unsigned int* cnt, double* red) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) X.part[(C.chunk_off + ch.idx) * 3 + k] = v[k];
        __threadfence();
        unsigned int prev = atomicAdd(cnt, 1u);
        last = (prev == (unsigned)C.nchunks - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    // ordered final sum by warp 0
    if (threadIdx.x < 32) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int j = threadIdx.x; j < C.nchunks; j += 32)
                s += ((volatile double*)X.part)[(C.chunk_off + j) * 3 + k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            out[k] = s;
        }
    }
    if (threadIdx.x == 0) *cnt = 0;
    return true;
}

__global__ void k_cg_init(ChunkCtx X) {
    __shared__ double red[64];
    const Chunk ch = X.chunks[blockIdx.x];
    const CompInfo& C = X.comps[ch.comp];
    if (C.small) return;
    int64_t row = ch.row0 + threadIdx.x;
    double v[2] = {0.0, 0.0};
    if (threadIdx.x < ch.nrow) {
        int64_t i = C.vec_off + row;
        double bi = X.rhs[i], z = X.dinv[i] * bi;
        X.x[i] = 0.0; X.r[i] = bi; X.z[i] = z; X.p[i] = z;
        v[0] = bi * z; v[1] = bi * bi;
    }
    block_sum<2>(v, red);
    double out[2];
    if (finish_component<2>(X, ch, C, v, out, &X.st[ch.comp].cnt1, red) && threadIdx.x == 0) {
        CgState& s = X.st[ch.comp];
        s.rho = out[0]; s.bb = out[1]; s.it = 0;
        s.conv = (out[1] == 0.0);
        s.active = !s.conv;
        if (s.active) atomicAdd(X.active_count, 1);
    }
}

template <int D>
__global__ void k_cg_spmv(ChunkCtx X) {
    __shared__ double red[64];
    const Chunk ch = X.chunks[blockIdx.x];
    const CompInfo& C = X.comps[ch.comp];
    if (C.small || !X.st[ch.comp].active) return;
    int64_t row = ch.row0 + threadIdx.x;
    double v[1] = {0.0};
    if (threadIdx.x < ch.nrow) {
        double y = spmv_row<D>(C, X.stencil + C.mat_off, X.p + C.vec_off, row, X.p_deg, 0, 1);
        X.q[C.vec_off + row] = y;
        v[0] = X.p[C.vec_off + row] * y;
    }
    block_sum<1>(v, red);
    double out[1];
    if (finish_component<1>(X, ch, C, v, out, &X.st[ch.comp].cnt1, red) && threadIdx.x == 0) {
        CgState& s = X.st[ch.comp];
        s.alpha = s.rho / out[0];
    }
}

__global__ void k_cg_update(ChunkCtx X) {
    __shared__ double red[64];
    const Chunk ch = X.chunks[blockIdx.x];
    const CompInfo& C = X.comps[ch.comp];
    if (C.small || !X.st[ch.comp].active) return;
    const double alpha = X.st[ch.comp].alpha;
    double v[2] = {0.0, 0.0};
    if (threadIdx.x < ch.nrow) {
        int64_t i = C.vec_off + ch.row0 + threadIdx.x;
        double ri = X.r[i] - alpha * X.q[i];
        X.x[i] += alpha * X.p[i];
        double zi = X.dinv[i] * ri;
        X.r[i] = ri; X.z[i] = zi;
        v[0] = ri * ri; v[1] = ri * zi;
    }
    block_sum<2>(v, red);
    double out[2];
    if (finish_component<2>(X, ch, C, v, out, &X.st[ch.comp].cnt2, red) && threadIdx.x == 0) {
        CgState& s = X.st[ch.comp];
        s.it += 1;
        if (out[0] <= X.rtol2 * s.bb) {
            s.conv = 1; s.active = 0;
            atomicSub(X.active_count, 1);
        } else if (s.it >= X.maxit) {
            s.active = 0;
            atomicSub(X.active_count, 1);
        } else {
            s.beta = out[1] / s.rho;
            s.rho = out[1];
        }
    }
}

__global__ void k_cg_pupdate(ChunkCtx X) {
    const Chunk ch = X.chunks[blockIdx.x];
    const CompInfo& C = X.comps[ch.comp];
    if (C.small || !X.st[ch.comp].active) return;
    const double beta = X.st[ch.comp].beta;
    if (threadIdx.x < ch.nrow) {
        int64_t i = C.vec_off + ch.row0 + threadIdx.x;
        X.p[i] = X.z[i] + beta * X.p[i];
    }
}

// ---- residual check: relres_c = ||A x - b|| / ||b|| ----------------------
template <int D>
__global__ void k_residual(ChunkCtx X, double* relres) {
    __shared__ double red[64];
    const Chunk ch = X.chunks[blockIdx.x];
    const CompInfo& C = X.comps[ch.comp];
    int64_t row = ch.row0 + threadIdx.x;
    double v[2] = {0.0, 0.0};
    if (threadIdx.x < ch.nrow) {
        double y = spmv_row<D>(C, X.stencil + C.mat_off, X.x + C.vec_off, row, X.p_deg, 0, 1);
        double bi = X.rhs[C.vec_off + row], e = y - bi, xv = X.x[C.vec_off + row];
        v[0] = e * e;
        v[1] = bi * bi;
        if (!isfinite(xv)) v[0] = __longlong_as_double(0x7ff8000000000000ULL);
    }
    block_sum<2>(v, red);
    double out[2];
    if (finish_component<2>(X, ch, C, v, out, &X.st[ch.comp].cnt1, red) && threadIdx.x == 0)
        relres[ch.comp] = out[1] > 0.0 ? sqrt(out[0] / out[1]) : (out[0] == 0.0 ? 0.0 : out[0]);
}

// ---- expand interior solution to full C-order coefficients ---------------
template <int D>
__global__ void k_expand(const CompInfo* __restrict__ comps, int ncomp,
                         const int64_t* __restrict__ dof_cum, const double* __restrict__ x,
                         double* __restrict__ coef) {
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= dof_cum[ncomp]) return;
    int lo = 0, hi = ncomp;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (dof_cum[mid] <= gid) lo = mid; else hi = mid;
    }
    const CompInfo& C = comps[lo];
    int64_t f = gid - dof_cum[lo], rem = f, row = 0;
    bool inter = true;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
        int ik = (int)(rem % C.n[k]);
        rem /= C.n[k];
        if (ik < 1 || ik > C.n[k] - 2) inter = false;
        else row += (int64_t)(ik - 1) * C.rs[k];
    }
    coef[C.dof_off + f] = inter ? x[C.vec_off + row] : 0.0;
}

static ChunkCtx make_ctx(Handle* h, double rtol, int maxit) {
    ChunkCtx X;
    X.comps = h->d_comps; X.chunks = h->d_chunks; X.stencil = h->d_stencil;
    X.rhs = h->d_rhs; X.dinv = h->d_dinv;
    X.x = h->d_x; X.r = h->d_r; X.z = h->d_z; X.p = h->d_p; X.q = h->d_q;
    X.st = h->d_cg; X.part = h->d_part; X.active_count = h->d_active_count;
    X.p_deg = h->p; X.rtol2 = rtol * rtol; X.maxit = maxit;
    return X;
}

extern int64_t* comp_dof_cum_ptr(Handle* h);

size_t small_smem_bytes(const Handle* h) {
    int64_t mx = 0;
    for (int c : h->small_comps) {
        const CompInfo& C = h->comps[c];
        int64_t b = 6 * C.rows + 2 * C.halo;
        if (b > mx) mx = b;
    }
    return (size_t)(mx + 64) * sizeof(double);
}

int run_pcg(Handle* h, double rtol, int maxit) {
    ChunkCtx X = make_ctx(h, rtol, maxit);
    int nch = (int)h->chunks.size();
    SG_CUDA(cudaMemsetAsync(h->d_active_count, 0, sizeof(int), h->stream));
    if (!h->small_comps.empty()) {
        size_t smem = small_smem_bytes(h);
#define LAUNCH_SMALL(DD)                                                                         \
    SG_CUDA(cudaFuncSetAttribute(k_pcg_small<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                 (int)smem));                                                    \
    k_pcg_small<DD><<<(unsigned)h->small_comps.size(), SMALL_THREADS, smem, h->stream>>>(        \
        h->d_comps, h->d_small, h->d_stencil, h->d_rhs, h->d_dinv, h->d_x, h->d_cg, h->p,        \
        rtol * rtol, maxit)
        h->kstart(3);
        if (h->d == 1) { LAUNCH_SMALL(1); }
        else if (h->d == 2) { LAUNCH_SMALL(2); }
        else { LAUNCH_SMALL(3); }
#undef LAUNCH_SMALL
        h->kstop(3);
        SG_CUDA(cudaGetLastError());
        h->launches[1]++;
    }
    if (!h->large_comps.empty()) {
        h->kstart(4);
        k_cg_init<<<nch, CHUNK_ROWS, 0, h->stream>>>(X);
        SG_CUDA(cudaGetLastError());
        h->launches[1]++;
        // capture GRAPH_ITERS iterations once, replay until all converged
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        SG_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < GRAPH_ITERS; ++k) {
            if (h->d == 1) k_cg_spmv<1><<<nch, CHUNK_ROWS, 0, h->stream>>>(X);
            else if (h->d == 2) k_cg_spmv<2><<<nch, CHUNK_ROWS, 0, h->stream>>>(X);
            else k_cg_spmv<3><<<nch, CHUNK_ROWS, 0, h->stream>>>(X);
            k_cg_update<<<nch, CHUNK_ROWS, 0, h->stream>>>(X);
            k_cg_pupdate<<<nch, CHUNK_ROWS, 0, h->stream>>>(X);
        }
        SG_CUDA(cudaStreamEndCapture(h->stream, &graph));
        SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        int max_rounds = maxit / GRAPH_ITERS + 2;
        for (int round = 0; round < max_rounds; ++round) {
            SG_CUDA(cudaGraphLaunch(exec, h->stream));
            h->launches[1] += 3 * GRAPH_ITERS;
            SG_CUDA(cudaMemcpyAsync(h->h_pinned_flag, h->d_active_count, sizeof(int),
                                    cudaMemcpyDeviceToHost, h->stream));
            SG_CUDA(cudaStreamSynchronize(h->stream));
            if (*h->h_pinned_flag <= 0) break;
        }
        h->kstop(4);
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
    }
    return SGIGA_OK;
}

cudaError_t launch_residual_check(Handle* h) {
    ChunkCtx X = make_ctx(h, 0.0, 0);
    int nch = (int)h->chunks.size();
    if (h->d == 1) k_residual<1><<<nch, CHUNK_ROWS, 0, h->stream>>>(X, h->d_relres);
    else if (h->d == 2) k_residual<2><<<nch, CHUNK_ROWS, 0, h->stream>>>(X, h->d_relres);
    else k_residual<3><<<nch, CHUNK_ROWS, 0, h->stream>>>(X, h->d_relres);
    h->launches[1]++;
    return cudaGetLastError();
}

cudaError_t launch_expand(Handle* h) {
    int64_t n = h->total_dofs;
    unsigned blocks = (unsigned)((n + 255) / 256);
    if (h->d == 1) k_expand<1><<<blocks, 256, 0, h->stream>>>(h->d_comps, h->ncomp, comp_dof_cum_ptr(h), h->d_x, h->d_coef);
    else if (h->d == 2) k_expand<2><<<blocks, 256, 0, h->stream>>>(h->d_comps, h->ncomp, comp_dof_cum_ptr(h), h->d_x, h->d_coef);
    else k_expand<3><<<blocks, 256, 0, h->stream>>>(h->d_comps, h->ncomp, comp_dof_cum_ptr(h), h->d_x, h->d_coef);
    h->launches[1]++;
    return cudaGetLastError();
}

}  // namespace sgiga
