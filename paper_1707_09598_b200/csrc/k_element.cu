// k_element.cu -- B4: GPU mirror of the reference's element-kernel plugin
// point _kernels.local_poisson_systems (_kernels/_compiled.pyx:17-90,
// _kernels/_fallback.py:13-65).  Same arrays, same accumulate-into-outputs
// contract; one thread per (element, a, b >= a) entry, mirrored at the end
// like _compiled.pyx:87-90.  This is a parity hook for the reference's own
// random-input agreement test (tests/test_kernels.py:19-55); the fast
// assembly path is k_assembly.cu.
#include <algorithm>
#include <vector>

#include "handle.cuh"

namespace sgiga {

struct ElemArgs {
    int d, max_nel, n_q, kmax, n_qp, n_loc;
    int64_t n_chunk;
    const double *values, *derivs, *metric, *load;
    const int64_t* elem_index;
    const int32_t *qp_index, *fn_index;
    double *out_a, *out_b;
};

__device__ __forceinline__ void local_val_grad(const ElemArgs& A, int64_t c, int q, int a,
                                               double& v, double* g) {
    double va[8], da[8];
    for (int l = 0; l < A.d; ++l) {
        int64_t e = A.elem_index[c * A.d + l];
        int ql = A.qp_index[q * A.d + l];
        int fl = A.fn_index[a * A.d + l];
        size_t idx = (((size_t)l * A.max_nel + e) * A.n_q + ql) * A.kmax + fl;
        va[l] = A.values[idx];
        da[l] = A.derivs[idx];
    }
    v = 1.0;
    for (int l = 0; l < A.d; ++l) v *= va[l];
    for (int m = 0; m < A.d; ++m) {
        double t = da[m];
        for (int l = 0; l < A.d; ++l) if (l != m) t *= va[l];
        g[m] = t;
    }
}

__global__ void k_local_systems(ElemArgs A) {
    int64_t npair = (int64_t)A.n_loc * A.n_loc;
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= A.n_chunk * npair) return;
    int64_t c = gid / npair;
    int a = (int)((gid % npair) / A.n_loc), b = (int)(gid % A.n_loc);
    if (b < a) return;
    double s_ab = 0.0, s_b = 0.0;
    for (int q = 0; q < A.n_qp; ++q) {
        double va, vb, ga[8], gb[8];
        local_val_grad(A, c, q, a, va, ga);
        local_val_grad(A, c, q, b, vb, gb);
        const double* G = A.metric + (c * A.n_qp + q) * A.d * A.d;
        double s = 0.0;
        for (int n = 0; n < A.d; ++n) {
            double half = 0.0;
            for (int m = 0; m < A.d; ++m) half += ga[m] * G[m * A.d + n];
            s += half * gb[n];
        }
        s_ab += s;
        if (b == a) s_b += va * A.load[c * A.n_qp + q];
    }
    double* oa = A.out_a + c * npair;
    oa[(int64_t)a * A.n_loc + b] += s_ab;
    if (b == a) A.out_b[c * A.n_loc + a] += s_b;
}

__global__ void k_local_mirror(ElemArgs A) {
    int64_t npair = (int64_t)A.n_loc * A.n_loc;
    int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= A.n_chunk * npair) return;
    int64_t c = gid / npair;
    int a = (int)((gid % npair) / A.n_loc), b = (int)(gid % A.n_loc);
    if (b >= a) return;
    double* oa = A.out_a + c * npair;
    oa[(int64_t)a * A.n_loc + b] = oa[(int64_t)b * A.n_loc + a];
}

}  // namespace sgiga

using namespace sgiga;

extern "C" int sgiga_local_poisson_systems(int32_t d, int32_t max_nel, int32_t n_q, int32_t kmax,
                                           int64_t n_chunk, int32_t n_qp, int32_t n_loc,
                                           const double* values, const double* derivs,
                                           const int64_t* elem_index, const int32_t* qp_index,
                                           const int32_t* fn_index, const double* metric,
                                           const double* load, double* out_a, double* out_b) {
    if (d > 8) { set_error("kernel supports at most 8 directions"); return SGIGA_ERR_VALUE; }
    if (d < 1 || n_chunk < 0 || n_qp < 0 || n_loc < 0) { set_error("bad shapes"); return SGIGA_ERR_VALUE; }
    if (n_chunk == 0 || n_loc == 0) return SGIGA_OK;
    size_t ntab = (size_t)d * max_nel * n_q * kmax;
    size_t sizes[] = {ntab, ntab, (size_t)n_chunk * n_qp * d * d, (size_t)n_chunk * n_qp,
                      (size_t)n_chunk * n_loc * n_loc, (size_t)n_chunk * n_loc};
    const double* hsrc[] = {values, derivs, metric, load, out_a, out_b};
    double* dbuf[6] = {};
    int64_t* dei = nullptr;
    int32_t *dqi = nullptr, *dfi = nullptr;
    int st = SGIGA_OK;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 6 && e == cudaSuccess; ++i) {
        e = cudaMalloc(&dbuf[i], std::max<size_t>(sizes[i], 1) * sizeof(double));
        if (e == cudaSuccess && sizes[i])
            e = cudaMemcpy(dbuf[i], hsrc[i], sizes[i] * sizeof(double), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMalloc(&dei, sizeof(int64_t) * n_chunk * d);
    if (e == cudaSuccess) e = cudaMalloc(&dqi, sizeof(int32_t) * std::max(1, n_qp * d));
    if (e == cudaSuccess) e = cudaMalloc(&dfi, sizeof(int32_t) * n_loc * d);
    if (e == cudaSuccess) e = cudaMemcpy(dei, elem_index, sizeof(int64_t) * n_chunk * d, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n_qp) e = cudaMemcpy(dqi, qp_index, sizeof(int32_t) * n_qp * d, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dfi, fn_index, sizeof(int32_t) * n_loc * d, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        ElemArgs A;
        A.d = d; A.max_nel = max_nel; A.n_q = n_q; A.kmax = kmax; A.n_qp = n_qp; A.n_loc = n_loc;
        A.n_chunk = n_chunk;
        A.values = dbuf[0]; A.derivs = dbuf[1]; A.metric = dbuf[2]; A.load = dbuf[3];
        A.out_a = dbuf[4]; A.out_b = dbuf[5];
        A.elem_index = dei; A.qp_index = dqi; A.fn_index = dfi;
        int64_t n = n_chunk * (int64_t)n_loc * n_loc;
        unsigned blocks = (unsigned)((n + 127) / 128);
        k_local_systems<<<blocks, 128>>>(A);
        k_local_mirror<<<blocks, 128>>>(A);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpy(out_a, dbuf[4], sizes[4] * sizeof(double), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemcpy(out_b, dbuf[5], sizes[5] * sizeof(double), cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); st = SGIGA_ERR_CUDA; }
    for (double* p : dbuf) if (p) cudaFree(p);
    if (dei) cudaFree(dei);
    if (dqi) cudaFree(dqi);
    if (dfi) cudaFree(dfi);
    return st;
}
