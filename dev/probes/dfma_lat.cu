// DFMA dependent-issue latency and per-SMSP throughput on the B200
#include <cstdio>
template <int CH>
__global__ void k(double* out, long long* cyc, int n) {
    double a[CH];
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
    const double x = 1.0000001, y = 0.999999;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = fma(a[c], x, y);
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < CH; ++c) s += a[c];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8); long long h;
    const int n = 4096;
#define RUN(CH, W) k<CH><<<1, 32 * W>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
    printf("chains/thread %2d warps %2d: %.2f cycles per dependent step, %.2f cycles per warp-DFMA (per SM)\n", CH, W, (double)h / n, (double)h / (n * (double)CH * W));
    RUN(1, 1) RUN(2, 1) RUN(4, 1) RUN(8, 1) RUN(16, 1)
    RUN(1, 4) RUN(4, 4) RUN(8, 4) RUN(1, 8) RUN(4, 8) RUN(8, 8) RUN(4, 16) RUN(8, 16)
    return 0;
}
