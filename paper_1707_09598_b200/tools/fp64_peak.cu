// fp64_peak.cu -- sustained DFMA micro-benchmark: the FP64 roofline
// denominator (MEASURED_PEAKS.json has none).
// Each thread runs 16 independent FMA chains; grid = 148 SMs x 8 CTAs.
#include <cuda_runtime.h>
#include <cstdint>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;   // keep the chains alive
}

// legacy FP64 tensor-core MMA (DMMA, mma.sync m8n8k4): is it faster than
// DFMA on this part?  (north star: tensor cores only if they profit)
__global__ void k_dmma(double* out, int iters, double a0, double b0) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = threadIdx.x * 1e-9; }
    double a = a0 + threadIdx.x * 1e-12, b = b0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

extern "C" int sgiga_dmma_peak(double* tflops) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d_out;
    if (cudaMalloc(&d_out, sizeof(double)) != cudaSuccess) return -5;
    int blocks = sms * 4, threads = 256, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dmma<<<blocks, threads>>>(d_out, 16, 1e-3, 1e-3);
    float ms = 0.f;
    double best = 0.0;
    for (int rep = 0; rep < 20; ++rep) {
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(d_out, iters, 1e-3, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 512.0 * 8.0 * (double)iters * blocks * (threads / 32);
        double tf = fl / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
        if (ms < 50.f) iters *= 2;
    }
    *tflops = best;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_out);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}

extern "C" int sgiga_fp64_peak(double seconds_target, double* tflops, double* ms_out) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d_out;
    if (cudaMalloc(&d_out, sizeof(double)) != cudaSuccess) return -5;
    int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(d_out, 64, 0.999999, 1e-7);   // warm-up
    float ms = 0.f;
    double best = 0.0;
    for (int rep = 0; rep < 50; ++rep) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(d_out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16.0 * (double)iters * blocks * threads;
        double tf = fl / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
        if (ms * 1e-3 * (rep + 1) > seconds_target) break;
        if (ms < 50.f) iters *= 2;
    }
    *tflops = best;
    if (ms_out) *ms_out = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_out);
    return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
