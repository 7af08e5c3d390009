// Single-warp shared-memory throughput on B200: cycles per LDS.128 / LDS.64 / STS.64 when ONE warp
// issues 16 independent accesses back to back (the 32x32 kernel's parameter loads and transposes).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench/lds_warp.cu -o tools/microbench/lds_warp
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
    __shared__ __align__(16) double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 1e-3;
    __syncthreads();
    const int lane = threadIdx.x & 31, half = lane >> 4;
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int o = (it * 64) & 1023;
        if (MODE == 0) {  // LDS.128, two addresses (half-warp broadcast): the parameter loads
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 v = *reinterpret_cast<const double2*>(&buf[o + 2 * q + 32 * half]);
                acc[q] += v.x * v.y;
            }
        } else if (MODE == 1) {  // LDS.128, distinct per lane (the transpose reads)
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double2 v = *reinterpret_cast<const double2*>(&buf[o + 68 * (q & 7) + 2 * lane + (q >> 3) * 1024]);
                acc[q] += v.x * v.y;
            }
        } else if (MODE == 2) {  // STS.64 distinct (the transpose writes)
#pragma unroll
            for (int q = 0; q < 16; ++q) buf[2048 + 34 * q + lane] = acc[q] + it;
        } else if (MODE == 3) {  // LDS.64 broadcast-pair
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] += buf[o + q + 32 * half];
        } else if (MODE == 4) {  // SHFL.IDX of a double (2 x SHFL32) from lane q of the half
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] += __shfl_sync(0xffffffffu, acc[(q + 1) & 15] + it, q + 16 * half);
        } else {  // mixed: 8 LDS.128 + 8 double shuffles
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double2 v = *reinterpret_cast<const double2*>(&buf[o + 2 * q + 32 * half]);
                acc[q] += v.x * v.y;
            }
#pragma unroll
            for (int q = 8; q < 16; ++q) acc[q] += __shfl_sync(0xffffffffu, acc[(q + 1) & 15] + it, q + 16 * half);
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += acc[q];
    if (s == 12345.0) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
    double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 1024);
    const int iters = 2000;
    k<MODE><<<1, 32 * warps>>>(out, cyc, 10);
    k<MODE><<<1, 32 * warps>>>(out, cyc, iters);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-40s warps/CTA %2d: %.2f cycles per access instruction per warp\n", name, warps, (double)c / (iters * 16.0));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    for (int w : {1, 2, 4, 8}) {
        run<0>("LDS.128 half-warp broadcast", w);
        run<1>("LDS.128 distinct", w);
        run<2>("STS.64 distinct", w);
        run<3>("LDS.64 half-warp broadcast", w);
        run<4>("SHFL.IDX double (2 x 32-bit)", w);
        run<5>("8 LDS.128 + 8 double SHFL", w);
    }
    return 0;
}
