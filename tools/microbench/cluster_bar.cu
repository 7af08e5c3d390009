// Latency of a 2-CTA cluster barrier (barrier.cluster.arrive + wait) vs a CTA barrier, 128 threads per CTA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) k_cluster(int iters, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}
__global__ void k_cta(int iters, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}
int main() {
    long long* d;
    long long h[4];
    cudaMalloc(&d, 64);
    k_cluster<<<2, 128>>>(10000, d);
    cudaDeviceSynchronize();
    k_cluster<<<2, 128>>>(10000, d);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("cluster barrier: %lld cycles (%s)\n", h[0], cudaGetErrorString(cudaGetLastError()));
    k_cta<<<1, 128>>>(10000, d);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("cta barrier: %lld cycles\n", h[0]);
    return 0;
}
