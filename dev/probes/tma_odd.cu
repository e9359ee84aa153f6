// Probe (not product): does a 4-D TMA tile copy with an even-padded inner box
// (26 doubles) and odd start coordinates work?  nvcc -arch=sm_100a tma_odd.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const CUtensorMap* tm, int x0, int x1, int x2, double* out, int nbytes, int off) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    double* dst = sm + off;
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(nbytes) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(su32(dst)), "l"(tm), "r"(x0), "r"(x1), "r"(x2), "r"(0),
                     "r"(su32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < nbytes / 8; i += blockDim.x) out[i] = dst[i];
}
int main() {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fnp; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fnp;
    const int cases[][6] = {  // NX(box1), box0, Na, x0, P-style off(doubles), threads
        {16, 16, 16, -12, 0, 352}, {25, 26, 20, -20, 0, 352}, {25, 26, 20, 0, 0, 352},
        {25, 26, 40, 4, 0, 608}, {25, 26, 20, -20, 4560, 608}, {25, 26, 40, 5, 0, 352}};
    for (auto& c : cases) {
        const int NX = c[0], B0 = c[1], Na = c[2], x0 = c[3], off = c[4], nt = c[5];
        const int Nb = Na, Ns = 10, NG = 7;
        size_t nqp = (size_t)Na * Nb * Ns;
        std::vector<double> h(nqp * NG);
        for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
        double* d; cudaMalloc(&d, h.size() * 8); cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        CUtensorMap m;
        cuuint64_t dims[4] = {(cuuint64_t)Na, (cuuint64_t)Nb, (cuuint64_t)Ns, (cuuint64_t)NG};
        cuuint64_t str[3] = {(cuuint64_t)Na * 8, (cuuint64_t)Na * Nb * 8, nqp * 8};
        cuuint32_t box[4] = {(cuuint32_t)B0, (cuuint32_t)NX, 1, (cuuint32_t)NG}, es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUtensorMap* dm; cudaMalloc(&dm, sizeof m); cudaMemcpy(dm, &m, sizeof m, cudaMemcpyHostToDevice);
        const int nbytes = B0 * NX * NG * 8;
        double* dout; cudaMalloc(&dout, nbytes);
        int smem = (off + B0 * NX * NG) * 8;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<1, nt, smem>>>(dm, x0, -3, 2, dout, nbytes, off);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> o(nbytes / 8);
        int bad = -1;
        if (e == cudaSuccess) {
            cudaMemcpy(o.data(), dout, nbytes, cudaMemcpyDeviceToHost);
            for (int g = 0; g < NG && bad < 0; ++g)
                for (int y = 0; y < NX && bad < 0; ++y)
                    for (int x = 0; x < B0; ++x) {
                        int X = x0 + x, Y = -3 + y;
                        double ref = (X >= 0 && X < Na && Y >= 0 && Y < Nb) ? h[g * nqp + 2 * Na * Nb + Y * Na + X] : 0.0;
                        if (o[(g * NX + y) * B0 + x] != ref) { bad = (g * NX + y) * B0 + x; break; }
                    }
        }
        printf("NX=%d box0=%d Na=%d x0=%d off=%d nt=%d encode=%d err=%s bad=%d\n", NX, B0, Na, x0, off, nt, (int)r,
               cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
        cudaFree(d); cudaFree(dm); cudaFree(dout);
    }
    return 0;
}
