// micro-benchmark: cost of cluster.sync() vs __syncthreads() in a loop
// (352 threads per CTA, clusters of 4, one CTA per SM)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(4, 1, 1) k_cl(long long* out, int iters) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    double a = threadIdx.x;
    for (int i = 0; i < iters; ++i) { a = a * 1.0000001 + 0.5; cl.sync(); }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
    if (a == -1) out[1] = 1;
}
__global__ void k_cta(long long* out, int iters) {
    long long t0 = clock64();
    double a = threadIdx.x;
    for (int i = 0; i < iters; ++i) { a = a * 1.0000001 + 0.5; __syncthreads(); }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
    if (a == -1) out[1] = 1;
}
__global__ void __cluster_dims__(4, 1, 1) k_split(long long* out, int iters) {
    long long t0 = clock64();
    double a = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        a = a * 1.0000001 + 0.5;
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
    if (a == -1) out[1] = 1;
}
int main() {
    long long* d; cudaMalloc(&d, 16); long long h;
    for (int rep = 0; rep < 2; ++rep) {
        k_cta<<<148, 352>>>(d, 10000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("__syncthreads: %lld cycles\n", h);
        k_cl<<<148, 352>>>(d, 10000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("cluster.sync (4): %lld cycles\n", h);
        k_split<<<148, 352>>>(d, 10000); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); printf("split arrive/wait (4): %lld cycles\n", h);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
