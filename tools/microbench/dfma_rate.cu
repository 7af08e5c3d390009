// Issue rate of the rotation-update DFMA pattern for ONE warp and for 4 warps per SMSP
// (development aid): x' = fma(cm1, x, fma(c, y, x)), y' = fma(cm1, y, fma(-c, x, y)) over
// 2 rows x 16 column pairs, parameters in registers.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void apply2(double& x, double& y, double cm1, double c) {
    const double tx = fma(c, y, x);
    const double ty = fma(-c, x, y);
    x = fma(cm1, x, tx);
    y = fma(cm1, y, ty);
}
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(double* out, int iters, double seed) {
    double x0[32], x1[32], cm[16], cc[16];
#pragma unroll
    for (int i = 0; i < 32; ++i) { x0[i] = seed * (i + threadIdx.x); x1[i] = seed * (i - threadIdx.x); }
#pragma unroll
    for (int q = 0; q < 16; ++q) { cm[q] = -1e-3 * seed * q; cc[q] = 1e-2 * seed * (q + 1); }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                apply2(x0[2 * q], x0[2 * q + 1], cm[q], cc[q]);
                apply2(x1[2 * q], x1[2 * q + 1], cm[q], cc[q]);
            }
        } else {  // independent FMAs with one shared operand: pipe-rate reference
#pragma unroll
            for (int i = 0; i < 32; ++i) { x0[i] = fma(cc[i & 15], x0[i], cm[i & 15]); x1[i] = fma(cc[i & 15], x1[i], cm[i & 15]); }
#pragma unroll
            for (int i = 0; i < 32; ++i) { x0[i] = fma(cc[i & 15], x0[i], cm[i & 15]); x1[i] = fma(cc[i & 15], x1[i], cm[i & 15]); }
        }
    }
    long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += x0[i] + x1[i];
    out[blockIdx.x * 128 + threadIdx.x] = acc;
    if (threadIdx.x == 0) out[100000 + blockIdx.x] = (double)(t1 - t0) / iters / 128.0;  // cycles per DFMA (warp)
}
template <int M> void run(double* d, int threads, const char* name) {
    k<M><<<1, threads>>>(d, 2000, 1e-3);
    cudaDeviceSynchronize();
    double h; cudaMemcpy(&h, d + 100000, 8, cudaMemcpyDeviceToHost);
    printf("%-48s threads %3d: %.2f cycles per warp-DFMA (per warp)\n", name, threads, h);
}
int main() {
    double* d; cudaMalloc(&d, 200000 * 8);
    run<0>(d, 32, "apply2 pattern (2 rows x 16 pairs)");
    run<0>(d, 64, "apply2 pattern (2 rows x 16 pairs)");
    run<0>(d, 128, "apply2 pattern (2 rows x 16 pairs)");
    run<1>(d, 32, "independent fma, shared operands");
    run<1>(d, 128, "independent fma, shared operands");
    return 0;
}
