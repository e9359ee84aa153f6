// k_pcg_cluster.cu -- kernel 3, small components (<= 2048 interior rows):
// the whole Jacobi-PCG loop of a component in one thread-block cluster.
//
// Reference: linsolve.solve_spd (linsolve.py:16-54); Jacobi-CG is the
// alternative SPEC.md:231 allows.  This is the Chronopoulos-Gear form of
// preconditioned CG (same iterates as textbook PCG in exact arithmetic)
// whose three dot products (r.u, w.u, r.r) share ONE reduction per
// iteration, so the latency chain per iteration is: update -> broadcast u
// -> cluster barrier -> SpMV w = A u + dots -> cluster barrier.
//
// Layout: K CTAs (SMs) per component, contiguous row slices; every CTA
// holds its slice of the stencil matrix in shared memory (slot-major) and a
// full copy of u (the only gathered vector); the new u slice and the per-warp
// dot partials are written into every rank's shared memory through DSMEM.
// All ranks sum the partials in the same fixed (rank, warp) order, so the
// scalars are identical on every CTA and deterministic run to run.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "handle.cuh"

namespace sgiga {

constexpr int CL_THREADS = 256;
constexpr int CL_WARPS = CL_THREADS / 32;

__device__ __forceinline__ int row_base_abs(const CompInfo& C, int d, int row) {
    int rb = row;
    for (int k = 0; k < d; ++k)
        if (C.absm[k]) rb -= ((row / (int)C.rs[k]) % C.m[k]) * (int)C.rs[k];
    return rb;
}

// shared memory (doubles) besides the staged matrix
__host__ __device__ inline int64_t cg1_vec_doubles(int64_t R, int64_t RL, int64_t H, int64_t NS) {
    // cluster partials [3][8 ranks][8 warps], x r u w p s d (own rows),
    // u full copy (+halo), offs (int), rowbase (int), SpMV partials, pad
    return 3 * 8 * CL_WARPS + 7 * RL + R + 2 * H + (NS + 1) / 2 + 1 + (RL + 1) / 2 + 1 +
           (RL > 256 ? RL * 2 : 512) + 2;
}

template <int D>
__global__ void __launch_bounds__(CL_THREADS, 1)
k_pcg_cg1(const CompInfo* __restrict__ comps, const int* __restrict__ list,
          const int* __restrict__ slotoff, const double* __restrict__ stencil,
          const double* __restrict__ rhs, const double* __restrict__ dinv,
          double* __restrict__ xout, CgState* __restrict__ st, double rtol2, int maxit,
          int smem_doubles, int nlist, int* errflag, long long* prof, int prof_slot,
          double* __restrict__ relres) {
    namespace cgs = cooperative_groups;
    cgs::cluster_group cluster = cgs::this_cluster();
    const int K = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
    extern __shared__ double sm[];
    if (K != (int)(gridDim.x / (unsigned)nlist) || (int)(blockIdx.x % K) != rank) {
        if (threadIdx.x == 0) atomicOr(errflag, 8);   // cluster shape not as launched
        return;
    }
    const int c = list[blockIdx.x / K];
    const CompInfo& Cg = comps[c];
    const int R = (int)Cg.rows, H = (int)Cg.halo, NS = (int)Cg.nslots;
    const int RLmax = (R + K - 1) / K;
    const int lo = min(R, rank * RLmax), hi = min(R, lo + RLmax), RL = hi - lo;
    const int64_t vec = cg1_vec_doubles(R, RLmax, H, NS);
    const int NSS = RL > 0 ? (int)min((int64_t)NS, (smem_doubles - vec) / max(RL, 1)) : 0;
    double* cred = sm;                        // [3][8][CL_WARPS]
    double* xs = cred + 3 * 8 * CL_WARPS;     // own rows ...
    double* rs_ = xs + RLmax;
    double* us = rs_ + RLmax;
    double* ws = us + RLmax;
    double* pv = ws + RLmax;
    double* sv = pv + RLmax;
    double* ds = sv + RLmax;
    double* ue = ds + RLmax;                  // [H + R + H] full copy of u
    double* uf = ue + H;
    int* offs = reinterpret_cast<int*>(ue + R + 2 * H);
    int* rbv = offs + NS + (NS & 1);
    double* parts = reinterpret_cast<double*>(rbv + RLmax + (RLmax & 1));
    double* msm = sm + vec;                   // [NSS][RL] own rows, slot-major
    const double* gval = stencil + Cg.mat_off;
    const double* b = rhs + Cg.vec_off;
    const double* di = dinv + Cg.vec_off;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nrb = (RL + 31) >> 5;
    const int NG = nrb == 0 ? 1 : (nrb <= CL_WARPS ? CL_WARPS / nrb : 1);

    for (int i = tid; i < NS; i += CL_THREADS) offs[i] = slotoff[Cg.so_off + i];
    for (int i = tid; i < RL; i += CL_THREADS) rbv[i] = row_base_abs(Cg, D, lo + i);
    for (int i = tid; i < NSS * RL; i += CL_THREADS) {
        const int t = i / RL, il = i % RL;
        msm[i] = gval[(size_t)t * R + lo + il];
    }
    for (int i = tid; i < H; i += CL_THREADS) { ue[i] = 0.0; ue[H + R + i] = 0.0; }
    for (int i = tid; i < R; i += CL_THREADS) uf[i] = di[i] * b[i];   // u0 = D^-1 b everywhere
    for (int il = tid; il < RL; il += CL_THREADS) {
        const int i = lo + il;
        xs[il] = 0.0; rs_[il] = b[i]; ds[il] = di[i]; us[il] = di[i] * b[i];
    }
    __syncthreads();

    // Register-resident matrix: when every warp owns exactly one (row block,
    // slot group), its first MAXS slots (values + column offsets) are loaded
    // once and reused for the whole solve -- the SpMV then issues all its
    // gathers back to back instead of a dependent smem chain per slot.
    constexpr int MAXS = 32;
    const bool reg_mode = nrb <= CL_WARPS && warp < nrb * NG;
    const int my_il = (warp % max(nrb, 1)) * 32 + lane, my_g = warp / max(nrb, 1);
    double vreg[MAXS];
    int oreg[MAXS];
#pragma unroll
    for (int j = 0; j < MAXS; ++j) {
        const int t = my_g + j * NG;
        const bool ok = reg_mode && my_il < RL && t < NS;
        vreg[j] = ok ? (t < NSS ? msm[t * RL + my_il] : gval[(size_t)t * R + lo + my_il]) : 0.0;
        oreg[j] = ok ? offs[t] : 0;
    }

    // w = A u on own rows (slot-parallel), then the three dot partials
    auto spmv_dots = [&](double* dots) {
        if (reg_mode) {
            if (my_il < RL) {
                const int rb = rbv[my_il];
                double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
#pragma unroll
                for (int j = 0; j < MAXS; j += 4) {
                    y0 += vreg[j] * uf[rb + oreg[j]];
                    y1 += vreg[j + 1] * uf[rb + oreg[j + 1]];
                    y2 += vreg[j + 2] * uf[rb + oreg[j + 2]];
                    y3 += vreg[j + 3] * uf[rb + oreg[j + 3]];
                }
                for (int t = my_g + MAXS * NG; t < NS; t += NG)   // slots beyond the register cache
                    y0 += (t < NSS ? msm[t * RL + my_il] : __ldg(gval + (size_t)t * R + lo + my_il)) *
                          uf[rb + offs[t]];
                parts[my_g * RL + my_il] = (y0 + y1) + (y2 + y3);
            }
        } else
        for (int w = warp; w < nrb * NG; w += CL_WARPS) {
            const int rbk = w % nrb, g = w / nrb, il = rbk * 32 + lane;
            if (il < RL) {
                const int rb = rbv[il];
                double y0 = 0.0, y1 = 0.0;
                int t = g;
                for (; t + NG < NSS; t += 2 * NG) {
                    y0 += msm[t * RL + il] * uf[rb + offs[t]];
                    y1 += msm[(t + NG) * RL + il] * uf[rb + offs[t + NG]];
                }
                if (t < NSS) { y0 += msm[t * RL + il] * uf[rb + offs[t]]; t += NG; }
                const double* gv = gval + lo + il;
                for (; t + NG < NS; t += 2 * NG) {
                    double a0 = __ldg(gv + (size_t)t * R), a1 = __ldg(gv + (size_t)(t + NG) * R);
                    y0 += a0 * uf[rb + offs[t]];
                    y1 += a1 * uf[rb + offs[t + NG]];
                }
                if (t < NS) y0 += __ldg(gv + (size_t)t * R) * uf[rb + offs[t]];
                parts[g * RL + il] = y0 + y1;
            }
        }
        __syncthreads();
        dots[0] = dots[1] = dots[2] = 0.0;
        for (int il = tid; il < RL; il += CL_THREADS) {
            double y = parts[il];
            for (int g = 1; g < NG; ++g) y += parts[g * RL + il];   // fixed order
            ws[il] = y;
            const double ri = rs_[il], ui = us[il];
            dots[0] += ri * ui;   // gamma = r.u
            dots[1] += y * ui;    // delta = w.u
            dots[2] += ri * ri;   // r.r
        }
    };
    // cluster-wide sum: warp partials -> every rank's cred[v][rank][warp]
    // (DSMEM), one cluster barrier, fixed-order sum by every thread
    auto cluster_sum3 = [&](double* v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {   // three independent shuffle trees, interleaved
            const double a = __shfl_xor_sync(0xffffffffu, v[0], o);
            const double b2 = __shfl_xor_sync(0xffffffffu, v[1], o);
            const double c2 = __shfl_xor_sync(0xffffffffu, v[2], o);
            v[0] += a; v[1] += b2; v[2] += c2;
        }
        if (lane < K) {
            double* dst = cluster.map_shared_rank(cred, lane);
#pragma unroll
            for (int k = 0; k < 3; ++k) dst[(k * 8 + rank) * CL_WARPS + warp] = v[k];
        }
        cluster.sync();
        // fixed-order tree over the K*CL_WARPS partials: strided per-lane sums + xor shuffles
        const int np = K * CL_WARPS;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double* src = cred + k * 8 * CL_WARPS;
            double s = 0.0;
            for (int j = lane; j < np; j += 32) s += src[j];
            v[k] = s;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double a = __shfl_xor_sync(0xffffffffu, v[0], o);
            const double b2 = __shfl_xor_sync(0xffffffffu, v[1], o);
            const double c2 = __shfl_xor_sync(0xffffffffu, v[2], o);
            v[0] += a; v[1] += b2; v[2] += c2;
        }
    };

    double dots[3];
    spmv_dots(dots);
    cluster_sum3(dots);
    const double bb = dots[2];
    double gamma = dots[0], alpha = gamma / dots[1], beta = 0.0;
    for (int il = tid; il < RL; il += CL_THREADS) { pv[il] = us[il]; sv[il] = ws[il]; }
    int it = 0, conv = (bb == 0.0);
    // optional phase profile (SGIGA_PCG_PROFILE=<plan index>): clock64 sums
    // of thread 0, rank 0 of that component into prof[0..5]
    const bool pr = prof != nullptr && (int)(blockIdx.x / K) == prof_slot && rank == 0 && tid == 0;
    long long tp[6] = {0, 0, 0, 0, 0, 0};
    while (!conv && it < maxit) {
        long long c0 = pr ? clock64() : 0;
        // x += alpha p; r -= alpha s; u = D r; broadcast the u slice
        for (int il = tid; il < RL; il += CL_THREADS) {
            xs[il] += alpha * pv[il];
            const double ri = rs_[il] - alpha * sv[il];
            const double ui = ds[il] * ri;
            rs_[il] = ri;
            us[il] = ui;
            for (int r = 0; r < K; ++r) cluster.map_shared_rank(uf, r)[lo + il] = ui;
        }
        long long c1 = pr ? clock64() : 0;
        cluster.sync();   // u complete on every rank; cred free
        long long c2 = pr ? clock64() : 0;
        spmv_dots(dots);
        long long c3 = pr ? clock64() : 0;
        cluster_sum3(dots);
        long long c4 = pr ? clock64() : 0;
        if (pr) { tp[0] += c1 - c0; tp[1] += c2 - c1; tp[2] += c3 - c2; tp[3] += c4 - c3; tp[5] += 1; }
        ++it;
        if (dots[2] <= rtol2 * bb) { conv = 1; break; }
        const double g_new = dots[0];
        beta = g_new / gamma;
        alpha = g_new / (dots[1] - beta * g_new / alpha);
        gamma = g_new;
        for (int il = tid; il < RL; il += CL_THREADS) {
            pv[il] = us[il] + beta * pv[il];
            sv[il] = ws[il] + beta * sv[il];
        }
        if (pr) tp[4] += clock64() - c4;
        // (the next u broadcast waits for the cluster barrier above; pv/sv are CTA-local)
    }
    if (pr)
        for (int k = 0; k < 6; ++k) prof[k] = tp[k];
    // acceptance check of the reference (linsolve.py:49-53): the TRUE
    // residual ||A x - b|| / ||b||, with the register-resident matrix: x is
    // broadcast like u (every rank finished reading uf and cred above)
    for (int il = tid; il < RL; il += CL_THREADS) {
        xout[Cg.vec_off + lo + il] = xs[il];
        for (int r = 0; r < K; ++r) cluster.map_shared_rank(uf, r)[lo + il] = xs[il];
    }
    cluster.sync();
    spmv_dots(dots);   // ws = A x
    double ev[3] = {0.0, 0.0, 0.0};
    for (int il = tid; il < RL; il += CL_THREADS) {
        const double e = ws[il] - b[lo + il];
        ev[0] += isfinite(xs[il]) ? e * e : __longlong_as_double(0x7ff8000000000000ULL);
    }
    cluster_sum3(ev);
    if (tid == 0 && rank == 0) {
        st[c].it = it;
        st[c].conv = conv;
        st[c].active = 0;
        st[c].bb = bb;
        relres[c] = bb > 0.0 ? sqrt(ev[0] / bb) : (ev[0] == 0.0 ? 0.0 : ev[0]);
    }
    cluster.sync();   // no CTA exits while others may still write into its smem
}

int launch_pcg_cluster(Handle* h, double rtol, int maxit) {
    const int ns = (int)h->small_comps.size();
    if (ns == 0) return SGIGA_OK;
    // cluster CTAs per component: a constant, so a component's reduction
    // order (and its bits) never depends on which other components share
    // the batch (a rank's subset of a plan computes what the full plan does)
    const int K = 8;
    const int64_t limit = (224 * 1024) / 8;
    int64_t total = 0;
    for (int c : h->small_comps) {
        const CompInfo& C = h->comps[c];
        const int64_t RL = (C.rows + K - 1) / K;
        const int64_t v = cg1_vec_doubles(C.rows, RL, C.halo, C.nslots);
        total = std::max(total, std::min(limit, v + RL * C.nslots));
    }
    const size_t smem = (size_t)total * sizeof(double);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(ns * K));
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = h->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const double rt2 = rtol * rtol;
    const int sd = (int)total;
    const int pslot = h->opt.pcg_profile ? 0 : -1;
    long long* dprof = nullptr;
    if (pslot >= 0) {
        SG_CUDA(cudaMalloc(&dprof, 8 * sizeof(long long)));
        SG_CUDA(cudaMemsetAsync(dprof, 0, 8 * sizeof(long long), h->stream));
    }
#define LAUNCH_CG1(DD)                                                                        \
    SG_CUDA(cudaFuncSetAttribute(k_pcg_cg1<DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                 (int)smem));                                                 \
    SG_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_cg1<DD>, (const CompInfo*)h->d_comps,               \
                               (const int*)h->d_small, (const int*)h->d_slotoff,              \
                               (const double*)h->d_stencil, (const double*)h->d_rhs,          \
                               (const double*)h->d_dinv, h->d_x, h->d_cg, rt2, maxit, sd, ns, \
                               h->d_err, dprof, pslot, h->d_relres))
    if (h->d == 1) { LAUNCH_CG1(1); }
    else if (h->d == 2) { LAUNCH_CG1(2); }
    else { LAUNCH_CG1(3); }
#undef LAUNCH_CG1
    h->launches[1]++;
    if (dprof) {
        long long t[8];
        SG_CUDA(cudaMemcpyAsync(t, dprof, sizeof t, cudaMemcpyDeviceToHost, h->stream));
        SG_CUDA(cudaStreamSynchronize(h->stream));
        const double n = t[5] > 0 ? (double)t[5] : 1.0;
        fprintf(stderr, "pcg-profile comp-slot=%d K=%d iters=%lld cycles/iter: update=%.0f sync=%.0f "
                "spmv+dots=%.0f reduce=%.0f scalars+pupdate=%.0f\n", pslot, K, t[5], t[0] / n, t[1] / n,
                t[2] / n, t[3] / n, t[4] / n);
        cudaFree(dprof);
    }
    return SGIGA_OK;
}

}  // namespace sgiga
