// Are the FP64 tensor (DMMA) and FP64 FMA pipes independent? (development aid)
// Per-SM throughput of DMMA.8x8x4 alone, DFMA alone, and both interleaved, 8 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters, double s) {
    double acc[8][2], f[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc[i][0] = s * i; acc[i][1] = s + i; }
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = s * (i + 1);
    const double a = s * threadIdx.x, b = s - threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], a, b);
        }
        if (MODE != 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
        }
    }
    long long t1 = clock64();
    double z = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) z += acc[i][0] + acc[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) z += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = z;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1 << 20] = (double)(t1 - t0) / iters;
}
template <int M> void run(double* d, const char* name) {
    k<M><<<148, 256>>>(d, 4000, 1e-9);
    cudaDeviceSynchronize();
    double h; cudaMemcpy(&h, d + (1 << 20), 8, cudaMemcpyDeviceToHost);
    // per iteration per warp: 8 DMMA (8*256 FMA) and/or 64 DFMA (64*32 FMA); 8 warps per SM
    const double fma_dmma = (M != 1) ? 8.0 * 256 * 8 : 0, fma_dfma = (M != 0) ? 64.0 * 32 * 8 : 0;
    printf("%-28s %.1f cycles/iter -> DMMA %.1f FMA/clk/SM, DFMA %.1f FMA/clk/SM\n", name, h, fma_dmma / h,
           fma_dfma / h);
}
int main() {
    double* d; cudaMalloc(&d, ((1 << 20) + 8) * 8);
    run<0>(d, "DMMA only");
    run<1>(d, "DFMA only");
    run<2>(d, "DMMA + DFMA interleaved");
    return 0;
}
