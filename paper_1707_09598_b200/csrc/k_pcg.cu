// k_pcg.cu -- kernel 3: batched Jacobi-preconditioned CG over all
// components of a plan, plus the post-solve residual acceptance check and
// the expansion to full coefficient vectors.
//
// Reference: linsolve.solve_spd (linsolve.py:16-54) -- a direct SuperLU
// solve; SPEC.md:231 allows Jacobi-CG instead.  Residual acceptance
// ||Ax-b|| <= 1e-10 ||b|| (linsolve.py:49-53), zero-rhs shortcut (43-45),
// expand with zero boundary (assembly.py:202-206).
//
// Stencil SpMV: column of (row, slot) = rowbase(row) + off[slot], with
// rowbase = row - sum_{absolute axes} r_k rs_k and off[] a per-component
// table (handle.cu), so the inner loop is two loads and one FMA.
//
// Two regimes:
//  * small components (rows <= 2048): one CTA per component runs the whole
//    CG loop; vectors (and the matrix, when it fits) live in shared memory;
//    3 barriers per iteration, double-buffered deterministic reductions.
//  * large components: 256-row chunks, two fused kernels per iteration
//    (SpMV with the direction update folded in, then the x/r/z update),
//    per-component scalars reduced by the last chunk to finish in fixed
//    chunk order (deterministic), iterations replayed as a CUDA graph with
//    the convergence test on the device.
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "handle.cuh"

namespace sgiga {

constexpr int SMALL_THREADS = 1024;
constexpr int CHUNK_ROWS = 256;
constexpr int GRAPH_ITERS = 16;   // even: p buffers alternate per iteration

// shared memory (in doubles) of one small-path CTA: reductions, 6 vectors
// (p with halo), the slot-offset table; the matrix is appended when it fits
__host__ __device__ inline int64_t small_vec_doubles(int64_t R, int64_t H, int64_t NS) {
    // red, x r z d q, p+halo, offs (int), rowbase (int), SpMV partials, pad
    return 128 + 6 * R + 2 * H + (NS + 1) / 2 + 1 + (R + 1) / 2 + 1 + (R > 1024 ? R : 1024) + 2;
}

__device__ __forceinline__ int rowbase_of(const CompInfo& C, int d, int row) {
    int rb = row;
    for (int k = 0; k < d; ++k)
        if (C.absm[k]) rb -= ((row / (int)C.rs[k]) % C.m[k]) * (int)C.rs[k];
    return rb;
}

// warp-level deterministic sum, then a fixed-order sum over the block's
// warp partials read by every thread (one barrier; `red` must not be
// rewritten before another barrier has passed -> callers double-buffer).
template <int NV>
__device__ __forceinline__ void block_sum_1sync(double* v, double* red) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) red[k * 32 + w] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = lane < nw ? red[k * 32 + lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        v[k] = t;
    }
}

// ---------------------------------------------------------------------------
// small path: whole PCG in one CTA
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(SMALL_THREADS)
k_pcg_small(const CompInfo* __restrict__ comps, const int* __restrict__ list,
            const int* __restrict__ slotoff, const double* __restrict__ stencil,
            const double* __restrict__ rhs, const double* __restrict__ dinv,
            double* __restrict__ xout, CgState* __restrict__ st, double rtol2, int maxit,
            int smem_doubles) {
    extern __shared__ double sm[];
    const int c = list[blockIdx.x];
    const CompInfo& Cg = comps[c];
    const int R = (int)Cg.rows, H = (int)Cg.halo, NS = (int)Cg.nslots;
    // leading slots staged in shared memory, the rest streamed from L2/HBM
    const int NSS = (int)min((int64_t)NS, (smem_doubles - small_vec_doubles(R, H, NS)) / R);
    double* red = sm;                     // [2][64] double-buffered reductions
    double* xs = red + 128;
    double* rs_ = xs + R;
    double* zs = rs_ + R;
    double* ds = zs + R;
    double* qv = ds + R;
    double* pe = qv + R;                  // [H + R + H]
    double* ps = pe + H;
    int* offs = reinterpret_cast<int*>(pe + R + 2 * H);        // [NS]
    double* msm = sm + small_vec_doubles(R, H, NS);              // [NSS*R]
    const double* gval = stencil + Cg.mat_off;
    const double* b = rhs + Cg.vec_off;
    const double* di = dinv + Cg.vec_off;
    const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nth >> 5, nrb = (R + 31) >> 5;
    const int NG = nrb <= nwarps ? nwarps / nrb : 1;    // slot groups per row block
    int* rbv = offs + NS + (NS & 1);                     // [R] rowbase per row
    double* parts = reinterpret_cast<double*>(rbv + R + (R & 1));   // [NG][R]

    for (int i = tid; i < NS; i += nth) offs[i] = slotoff[Cg.so_off + i];
    for (int i = tid; i < R; i += nth) rbv[i] = rowbase_of(Cg, D, i);
    for (int i = tid; i < NSS * R; i += nth) msm[i] = gval[i];
    for (int i = tid; i < H; i += nth) { pe[i] = 0.0; pe[H + R + i] = 0.0; }
    double v2[2] = {0.0, 0.0};
    for (int i = tid; i < R; i += nth) {
        double bi = b[i], dd = di[i], z = dd * bi;
        xs[i] = 0.0; rs_[i] = bi; ds[i] = dd; zs[i] = z; ps[i] = z;
        v2[0] += bi * z;
        v2[1] += bi * bi;
    }
    block_sum_1sync<2>(v2, red);
    double rho = v2[0];
    const double bb = v2[1];
    int it = 0, conv = (bb == 0.0), par = 1;
    __syncthreads();
    while (!conv && it < maxit) {
        // SpMV, slot-parallel: warp (row block, slot group g) streams slots
        // t = g, g+NG, ... over 32 consecutive rows (coalesced, conflict-free)
        for (int w = warp; w < nrb * NG; w += nwarps) {
            const int rbk = w % nrb, g = w / nrb, row = rbk * 32 + lane;
            double y0 = 0.0, y1 = 0.0;
            if (row < R) {
                const int rb = rbv[row];
                int t = g;
                for (; t + NG < NSS; t += 2 * NG) {
                    y0 += msm[t * R + row] * ps[rb + offs[t]];
                    y1 += msm[(t + NG) * R + row] * ps[rb + offs[t + NG]];
                }
                if (t < NSS) { y0 += msm[t * R + row] * ps[rb + offs[t]]; t += NG; }
                const double* gv = gval + row;
                for (; t + NG < NS; t += 2 * NG) {
                    double a0 = __ldg(gv + (size_t)t * R), a1 = __ldg(gv + (size_t)(t + NG) * R);
                    y0 += a0 * ps[rb + offs[t]];
                    y1 += a1 * ps[rb + offs[t + NG]];
                }
                if (t < NS) y0 += __ldg(gv + (size_t)t * R) * ps[rb + offs[t]];
                parts[g * R + row] = y0 + y1;
            }
        }
        __syncthreads();
        double pq[1] = {0.0};
        for (int i = tid; i < R; i += nth) {
            double y = parts[i];
            for (int g = 1; g < NG; ++g) y += parts[g * R + i];   // fixed order
            qv[i] = y;
            pq[0] += ps[i] * y;
        }
        block_sum_1sync<1>(pq, red + 64 * par);
        par ^= 1;
        const double alpha = rho / pq[0];
        double w[2] = {0.0, 0.0};
        for (int i = tid; i < R; i += nth) {
            double ri = rs_[i] - alpha * qv[i];
            xs[i] += alpha * ps[i];
            double zi = ds[i] * ri;
            rs_[i] = ri; zs[i] = zi;
            w[0] += ri * ri;
            w[1] += ri * zi;
        }
        block_sum_1sync<2>(w, red + 64 * par);
        par ^= 1;
        ++it;
        if (w[0] <= rtol2 * bb) { conv = 1; break; }
        const double beta = w[1] / rho;
        rho = w[1];
        for (int i = tid; i < R; i += nth) ps[i] = zs[i] + beta * ps[i];
        __syncthreads();   // p complete before the next SpMV
    }
    for (int i = tid; i < R; i += nth) xout[Cg.vec_off + i] = xs[i];
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
    const int* slotoff;
    const double* stencil;
    const double* rhs;
    const double* dinv;
    double *x, *r, *z, *q;
    double *p0, *p1;      // alternating direction buffers
    CgState* st;
    double* part;
    int* active_count;
    const int* alist;     // active chunk list (compacted between graph replays)
    const int* acount;    // its length
    double rtol2;
    int maxit;
};

// in-place, order-preserving compaction of the active chunk list (one CTA)
__global__ void __launch_bounds__(1024) k_cg_compact(const Chunk* __restrict__ chunks,
                                                     const CgState* __restrict__ st,
                                                     int* __restrict__ alist, int* __restrict__ acount,
                                                     int* __restrict__ host_counts) {
    __shared__ int wsum[32];
    __shared__ int base;
    const int n = *acount, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) base = 0;
    __syncthreads();
    for (int t0 = 0; t0 < n; t0 += 1024) {
        const int i = t0 + tid;
        const int c = i < n ? alist[i] : -1;
        const int keep = (c >= 0 && st[chunks[c].comp].active) ? 1 : 0;
        int incl = keep;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        int wbase = 0;
        for (int k = 0; k < w; ++k) wbase += wsum[k];
        const int pos = base + wbase + incl - keep;
        __syncthreads();   // every thread has read alist[i] and wsum
        if (keep) alist[pos] = c;
        if (tid == 1023) base = pos + keep;
        __syncthreads();
    }
    if (tid == 0) { *acount = base; host_counts[0] = base; }
}

// last chunk of a component to finish reduces the partials (chunk order)
template <int NV>
__device__ __forceinline__ bool finish_component(const ChunkCtx& X, const Chunk& ch,
                                                 const CompInfo& C, const double* v, double* out,
                                                 unsigned int* cnt) {
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
    double v[2] = {0.0, 0.0};
    if (threadIdx.x < ch.nrow) {
        int64_t i = C.vec_off + ch.row0 + threadIdx.x;
        double bi = X.rhs[i], z = X.dinv[i] * bi;
        X.x[i] = 0.0; X.r[i] = bi; X.z[i] = z; X.p0[i] = 0.0; X.p1[i] = 0.0;
        v[0] = bi * z; v[1] = bi * bi;
    }
    block_sum_1sync<2>(v, red);
    double out[2];
    if (finish_component<2>(X, ch, C, v, out, &X.st[ch.comp].cnt1) && threadIdx.x == 0) {
        CgState& s = X.st[ch.comp];
        s.rho = out[0]; s.bb = out[1]; s.it = 0; s.beta = 0.0;
        s.conv = (out[1] == 0.0);
        s.active = !s.conv;
        if (s.active) atomicAdd(X.active_count, 1);
    }
}

// p_new = z + beta p_old (own rows, written to pn); q = A p_new with p_new
// formed on the fly at gathered columns; partial p_new . q.
// L lanes per row: L = 1 in the bulk (enough rows in flight), L = 2 / 4
// when the active set is small (latency-bound tail: more loads in flight).
template <int D, int L>
__global__ void __launch_bounds__(CHUNK_ROWS * L) k_cg_spmv(ChunkCtx X, int parity) {
    __shared__ double red[64];
    if ((int)blockIdx.x >= *X.acount) return;
    const Chunk ch = X.chunks[X.alist[blockIdx.x]];
    const CompInfo& C = X.comps[ch.comp];
    if (C.small || !X.st[ch.comp].active) return;
    const double* po = (parity ? X.p1 : X.p0) + C.vec_off;
    double* pn = (parity ? X.p0 : X.p1) + C.vec_off;
    const double* z = X.z + C.vec_off;
    const double beta = X.st[ch.comp].beta;
    const int R = (int)C.rows, NS = (int)C.nslots;
    const int* offs = X.slotoff + C.so_off;
    const double* val = X.stencil + C.mat_off;
    const int lr = threadIdx.x / L, ln = threadIdx.x % L;
    double v[1] = {0.0};
    double y = 0.0;
    const int row = ch.row0 + lr;
    if (lr < ch.nrow) {
        const int rb = rowbase_of(C, D, row);
        const double* vr = val + row;
#pragma unroll 4
        for (int t = ln; t < NS; t += L) {
            int col = rb + __ldg(offs + t);
            y += __ldg(vr + (size_t)t * R) * (z[col] + beta * po[col]);
        }
    }
#pragma unroll
    for (int o = L >> 1; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (lr < ch.nrow && ln == 0) {
        double pr = z[row] + beta * po[row];
        pn[row] = pr;
        X.q[C.vec_off + row] = y;
        v[0] = pr * y;
    }
    block_sum_1sync<1>(v, red);
    double out[1];
    if (finish_component<1>(X, ch, C, v, out, &X.st[ch.comp].cnt1) && threadIdx.x == 0) {
        CgState& s = X.st[ch.comp];
        s.alpha = s.rho / out[0];
    }
}

__global__ void __launch_bounds__(CHUNK_ROWS) k_cg_update(ChunkCtx X, int parity) {
    __shared__ double red[64];
    if ((int)blockIdx.x >= *X.acount) return;
    const Chunk ch = X.chunks[X.alist[blockIdx.x]];
    const CompInfo& C = X.comps[ch.comp];
    if (C.small || !X.st[ch.comp].active) return;
    const double alpha = X.st[ch.comp].alpha;
    const double* pn = (parity ? X.p0 : X.p1);
    double v[2] = {0.0, 0.0};
    if (threadIdx.x < ch.nrow) {
        int64_t i = C.vec_off + ch.row0 + threadIdx.x;
        double ri = X.r[i] - alpha * X.q[i];
        X.x[i] += alpha * pn[i];
        double zi = X.dinv[i] * ri;
        X.r[i] = ri; X.z[i] = zi;
        v[0] = ri * ri; v[1] = ri * zi;
    }
    block_sum_1sync<2>(v, red);
    double out[2];
    if (finish_component<2>(X, ch, C, v, out, &X.st[ch.comp].cnt2) && threadIdx.x == 0) {
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

// ---- residual check: relres_c = ||A x - b|| / ||b|| ----------------------
template <int D>
__global__ void k_residual(ChunkCtx X, double* relres, int skip_small) {
    __shared__ double red[64];
    const Chunk ch = X.chunks[blockIdx.x];
    const CompInfo& C = X.comps[ch.comp];
    if (C.fd || (skip_small && C.small)) return;   // the FD / cluster PCG kernels checked these
    double v[2] = {0.0, 0.0};
    if (threadIdx.x < ch.nrow) {
        int row = ch.row0 + threadIdx.x;
        int rb = rowbase_of(C, D, row);
        const int R = (int)C.rows, NS = (int)C.nslots;
        const int* offs = X.slotoff + C.so_off;
        const double* vr = X.stencil + C.mat_off + row;
        const double* xv = X.x + C.vec_off;
        double y = 0.0;
        for (int t = 0; t < NS; ++t) y += vr[(size_t)t * R] * xv[rb + offs[t]];
        double bi = X.rhs[C.vec_off + row], e = y - bi;
        v[0] = e * e;
        v[1] = bi * bi;
        if (!isfinite(xv[row])) v[0] = __longlong_as_double(0x7ff8000000000000ULL);
    }
    block_sum_1sync<2>(v, red);
    double out[2];
    if (finish_component<2>(X, ch, C, v, out, &X.st[ch.comp].cnt1) && threadIdx.x == 0)
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
    if (C.fd) return;   // the FD / line-FD kernels write their components' coefficients
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
    X.comps = h->d_comps; X.chunks = h->d_chunks; X.slotoff = h->d_slotoff;
    X.alist = nullptr; X.acount = nullptr;
    X.stencil = h->d_stencil; X.rhs = h->d_rhs; X.dinv = h->d_dinv;
    X.x = h->d_x; X.r = h->d_r; X.z = h->d_z; X.q = h->d_q;
    X.p0 = h->d_p; X.p1 = h->d_q2;
    X.st = h->d_cg; X.part = h->d_part; X.active_count = h->d_active_count;
    X.rtol2 = rtol * rtol; X.maxit = maxit;
    return X;
}

extern int64_t* comp_dof_cum_ptr(Handle* h);

size_t small_smem_bytes(const Handle* h, int64_t* smem_doubles) {
    const int64_t limit = (224 * 1024) / 8;
    int64_t total = 0;
    for (int c : h->small_comps) {
        const CompInfo& C = h->comps[c];
        int64_t v = small_vec_doubles(C.rows, C.halo, C.nslots);
        total = std::max(total, std::min(limit, v + C.rows * C.nslots));
    }
    *smem_doubles = total;
    return (size_t)total * sizeof(double);
}

int run_pcg(Handle* h, double rtol, int maxit) {
    ChunkCtx X = make_ctx(h, rtol, maxit);
    int nch = (int)h->chunks.size();
    const bool no_cluster = h->opt.no_cluster;
    h->small_checked = false;
    const bool any_fd = !h->fd_comps.empty() || !h->fdl_comps.empty() || !h->fdg_comps.empty();
    if (any_fd) {   // FD-preconditioned CG (k_fd.cu), which also checks its true residuals
        if (h->fd_pending) {
            SG_CUDA(cudaStreamWaitEvent(h->stream, h->fd_join, 0));
            h->fd_pending = false;
        }
        h->kstart(3);
        if (!h->fd_comps.empty() && !h->fdl_comps.empty()) {
            // the one-CTA FD solves (few, long CTAs) run on the high-priority
            // side stream beside the line-FD clusters instead of before them
            SG_CUDA(cudaEventRecord(h->pcg_fork, h->stream));
            SG_CUDA(cudaStreamWaitEvent(h->stream2, h->pcg_fork, 0));
            SG_CUDA(launch_pcg_fd(h, rtol, maxit, h->stream2));   // small: everything in shared memory
            SG_CUDA(cudaEventRecord(h->pcg_join, h->stream2));
            SG_CUDA(launch_pcg_fdl(h, rtol, maxit));              // one long axis: banded line solves
            SG_CUDA(cudaStreamWaitEvent(h->stream, h->pcg_join, 0));
        } else {
            SG_CUDA(launch_pcg_fd(h, rtol, maxit));    // small: everything in shared memory
            SG_CUDA(launch_pcg_fdl(h, rtol, maxit));   // one long axis: banded line solves
        }
        SG_CUDA(launch_pcg_fdg(h, rtol, maxit));       // large, every axis FD: whole-GPU cooperative PCG
        if (h->small_comps.empty()) h->kstop(3);
    }
    if (!h->small_comps.empty() && !no_cluster) {
        h->small_checked = true;   // the cluster kernel also computes the true residual
        if (!any_fd) h->kstart(3);
        int st = launch_pcg_cluster(h, rtol, maxit);   // k_pcg_cluster.cu
        h->kstop(3);
        if (st) return st;
    } else if (!h->small_comps.empty()) {
        int64_t total = 0;
        size_t smem = small_smem_bytes(h, &total);
        int cap = (int)total;   // a CTA stages its matrix iff its vectors + matrix fit
        if (!any_fd) h->kstart(3);
#define LAUNCH_SMALL(DD)                                                                         \
    SG_CUDA(cudaFuncSetAttribute(k_pcg_small<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                 (int)smem));                                                    \
    k_pcg_small<DD><<<(unsigned)h->small_comps.size(), SMALL_THREADS, smem, h->stream>>>(        \
        h->d_comps, h->d_small, h->d_slotoff, h->d_stencil, h->d_rhs, h->d_dinv, h->d_x,         \
        h->d_cg, rtol * rtol, maxit, cap)
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
        // active chunk list: every chunk of a large component, plan order
        std::vector<int> al;
        for (int c : h->large_comps)
            for (int i = 0; i < h->comps[c].nchunks; ++i) al.push_back((int)h->comps[c].chunk_off + i);
        int ncur = (int)al.size();
        SG_CUDA(cudaMemcpyAsync(h->d_alist, al.data(), sizeof(int) * al.size(), cudaMemcpyHostToDevice, h->stream));
        SG_CUDA(cudaMemcpyAsync(h->d_active_count + 1, &ncur, sizeof(int), cudaMemcpyHostToDevice, h->stream));
        X.alist = h->d_alist;
        X.acount = h->d_active_count + 1;
        // capture GRAPH_ITERS iterations over `grid` chunks; replay until all
        // converged; re-capture with a smaller grid whenever the active set
        // (compacted on the device after every replay) halves
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        auto capture = [&](int grid) -> int {
            if (exec) { cudaGraphExecDestroy(exec); exec = nullptr; }
            if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
            SG_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < GRAPH_ITERS; ++k) {
                int par = k & 1;
                const int lanes = grid <= 2 * 148 ? 4 : (grid <= 6 * 148 ? 2 : 1);
#define SPMV(DD, LL) k_cg_spmv<DD, LL><<<grid, CHUNK_ROWS * LL, 0, h->stream>>>(X, par)
#define SPMV_L(DD) { if (lanes == 4) SPMV(DD, 4); else if (lanes == 2) SPMV(DD, 2); else SPMV(DD, 1); }
                if (h->d == 1) SPMV_L(1)
                else if (h->d == 2) SPMV_L(2)
                else SPMV_L(3)
#undef SPMV_L
#undef SPMV
                k_cg_update<<<grid, CHUNK_ROWS, 0, h->stream>>>(X, par);
            }
            k_cg_compact<<<1, 1024, 0, h->stream>>>(h->d_chunks, h->d_cg, h->d_alist, h->d_active_count + 1,
                                                     h->d_active_count + 2);
            SG_CUDA(cudaStreamEndCapture(h->stream, &graph));
            SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
            return SGIGA_OK;
        };
        int grid = ncur;
        int st = capture(grid);
        if (st) return st;
        int max_rounds = maxit / GRAPH_ITERS + 2;
        const bool trace = h->opt.pcg_trace;
        cudaEvent_t tev0 = nullptr, tev1 = nullptr;
        if (trace) { cudaEventCreate(&tev0); cudaEventCreate(&tev1); cudaEventRecord(tev0, h->stream); }
        for (int round = 0; round < max_rounds; ++round) {
            if (trace && (round & 63) == 0) {
                cudaEventRecord(tev1, h->stream);
                cudaEventSynchronize(tev1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, tev0, tev1);
                fprintf(stderr, "pcg-trace it=%d ms=%.3f active_comps=%d grid=%d\n", round * GRAPH_ITERS, ms,
                        round ? h->h_pinned_flag[0] : (int)h->large_comps.size(), grid);
            }
            SG_CUDA(cudaGraphLaunch(exec, h->stream));
            h->launches[1] += 2 * GRAPH_ITERS + 1;
            SG_CUDA(cudaMemcpyAsync(h->h_pinned_flag, h->d_active_count, 3 * sizeof(int),
                                    cudaMemcpyDeviceToHost, h->stream));
            SG_CUDA(cudaStreamSynchronize(h->stream));
            const int active_comps = h->h_pinned_flag[0], active_chunks = h->h_pinned_flag[2];
            if (active_comps <= 0 || active_chunks <= 0) break;
            if (2 * active_chunks <= grid) {
                grid = active_chunks;
                if ((st = capture(grid))) return st;
            }
        }
        h->kstop(4);
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        // the converged x of every component is in d_x regardless of parity
    }
    return SGIGA_OK;
}

// ---- per-solve prologue / per-call status (single small launches that
// replace memset and copy nodes) --------------------------------------------
__global__ void k_solve_prologue(CgState* __restrict__ st, int ncomp, int* __restrict__ active_count) {
    int* w = reinterpret_cast<int*>(st);
    const int n = ncomp * (int)(sizeof(CgState) / sizeof(int));
    for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = 0;
    if (threadIdx.x < 4) active_count[threadIdx.x] = 0;
}

// solver state, true residuals and the error flags -> mapped host memory
__global__ void k_status(const CgState* __restrict__ st, const double* __restrict__ relres,
                         const int* __restrict__ err, int ncomp, CgState* hst, double* hrel, int* herr,
                         int* hsticky) {
    int fail = 0;
    for (int c = threadIdx.x; c < ncomp; c += blockDim.x) {
        const CgState s = st[c];
        hst[c] = s;
        hrel[c] = relres[c];
        fail |= cg_failed(s, relres[c]);
    }
    fail = __syncthreads_or(fail);
    if (threadIdx.x == 0) {
        *herr = *err;
        *hsticky |= (fail ? 1 : 0) | (*err ? 2 : 0);
    }
    __threadfence_system();
}

cudaError_t launch_solve_prologue(Handle* h, cudaStream_t stream) {
    k_solve_prologue<<<1, 256, 0, stream>>>(h->d_cg, h->ncomp, h->d_active_count);
    h->launches[1]++;
    return cudaGetLastError();
}

cudaError_t launch_status(Handle* h) {
    k_status<<<1, 256, 0, h->stream>>>(h->d_cg, h->d_relres, h->d_err, h->ncomp, h->dh_cg, h->dh_rel, h->dh_err,
                                       h->dh_sticky);
    h->launches[1]++;
    return cudaGetLastError();
}

cudaError_t launch_residual_check(Handle* h) {
    ChunkCtx X = make_ctx(h, 0.0, 0);
    int nch = (int)h->chunks.size();
    if (nch == 0 || ((h->small_checked || h->small_comps.empty()) && h->large_comps.empty())) return cudaSuccess;
    const int sk = h->small_checked ? 1 : 0;
    if (h->d == 1) k_residual<1><<<nch, CHUNK_ROWS, 0, h->stream>>>(X, h->d_relres, sk);
    else if (h->d == 2) k_residual<2><<<nch, CHUNK_ROWS, 0, h->stream>>>(X, h->d_relres, sk);
    else k_residual<3><<<nch, CHUNK_ROWS, 0, h->stream>>>(X, h->d_relres, sk);
    h->launches[1]++;
    return cudaGetLastError();
}

cudaError_t launch_expand(Handle* h) {
    int64_t n = h->total_dofs;
    if (n == 0) return cudaSuccess;
    bool any = false;   // components not expanded by the FD kernels (incl. empty interiors)
    for (const CompInfo& C : h->comps) any = any || !C.fd;
    if (!any) return cudaSuccess;
    unsigned blocks = (unsigned)((n + 255) / 256);
    if (h->d == 1) k_expand<1><<<blocks, 256, 0, h->stream>>>(h->d_comps, h->ncomp, comp_dof_cum_ptr(h), h->d_x, h->d_coef);
    else if (h->d == 2) k_expand<2><<<blocks, 256, 0, h->stream>>>(h->d_comps, h->ncomp, comp_dof_cum_ptr(h), h->d_x, h->d_coef);
    else k_expand<3><<<blocks, 256, 0, h->stream>>>(h->d_comps, h->ncomp, comp_dof_cum_ptr(h), h->d_x, h->d_coef);
    h->launches[1]++;
    return cudaGetLastError();
}

}  // namespace sgiga
