// Latency pieces of the transpose reduction used by the register kernels (development aid).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int RSTR = 34;
template <int MODE>
__global__ void k(double* out, int iters) {
    __shared__ __align__(16) double red[4][16 * RSTR];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, hl = lane & 15, half = lane >> 4;
    double* r = red[w];
    double v = lane * 1e-3, acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double s;
        if (MODE == 0) {  // 16 STS, syncwarp, 8 LDS.128, tree
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q * RSTR + lane] = v + q;
            __syncwarp();
            const double2* p = reinterpret_cast<const double2*>(r + hl * RSTR + 16 * half);
            double2 a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3], a4 = p[4], a5 = p[5], a6 = p[6], a7 = p[7];
            s = (((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y))) +
                (((a4.x + a4.y) + (a5.x + a5.y)) + ((a6.x + a6.y) + (a7.x + a7.y)));
            __syncwarp();
        } else if (MODE == 1) {  // 1 STS, syncwarp, 1 LDS
            r[lane] = v;
            __syncwarp();
            s = r[lane ^ 1];
            __syncwarp();
        } else if (MODE == 2) {  // DADD tree of 16 values, no smem
            double a[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) a[q] = v * (q + 1);
            s = (((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))) +
                (((a[8] + a[9]) + (a[10] + a[11])) + ((a[12] + a[13]) + (a[14] + a[15])));
        } else if (MODE == 3) {  // dependent DADD chain of 8
            s = v;
#pragma unroll
            for (int q = 0; q < 8; ++q) s = s + 1.0;
        } else if (MODE == 4) {  // shuffle pair
            s = __shfl_xor_sync(0xffffffffu, v, 1);
        } else if (MODE == 5) {  // 16 STS + sync + 1 LDS
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q * RSTR + lane] = v + q;
            __syncwarp();
            s = r[hl * RSTR + 16 * half];
            __syncwarp();
        } else if (MODE == 6) {  // 1 STS + sync + 8 LDS.128 + tree
            r[hl * RSTR + 16 * half] = v;
            __syncwarp();
            const double2* p = reinterpret_cast<const double2*>(r + hl * RSTR + 16 * half);
            double2 a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3], a4 = p[4], a5 = p[5], a6 = p[6], a7 = p[7];
            s = (((a0.x + a0.y) + (a1.x + a1.y)) + ((a2.x + a2.y) + (a3.x + a3.y))) +
                (((a4.x + a4.y) + (a5.x + a5.y)) + ((a6.x + a6.y) + (a7.x + a7.y)));
            __syncwarp();
        } else if (MODE == 7) {  // 8 STS.128 + sync + 1 LDS
#pragma unroll
            for (int q = 0; q < 8; ++q) reinterpret_cast<double2*>(r + 2 * q * RSTR)[lane] = make_double2(v + q, v - q);
            __syncwarp();
            s = r[hl * RSTR + 16 * half];
            __syncwarp();
        } else if (MODE == 9) {  // butterfly shuffle reduction of 16 doubles over 16 lanes
            double a[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) a[q] = v * (q + 1);
#pragma unroll
            for (int m = 8, n = 16; m >= 1; m >>= 1, n >>= 1) {
                const bool up = (hl & m) != 0;
#pragma unroll
                for (int i = 0; i < n / 2; ++i) {
                    const double lo = a[i], hi = a[i + n / 2];
                    const double send = up ? lo : hi, keep = up ? hi : lo;
                    a[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
                }
            }
            s = a[0];
        } else {  // 16 STS, no sync, no reload: issue cost
#pragma unroll
            for (int q = 0; q < 16; ++q) r[q * RSTR + lane] = v + q;
            s = v + 1.0;
        }
        v = s * 1e-9;
        acc += s;
    }
    long long t1 = clock64();
    if (lane == 0) out[w] = (double)(t1 - t0) / iters;
    if (acc == 12345.0) out[1000] = acc;
}
template <int M> void run(double* d, const char* name) {
    k<M><<<1, 128>>>(d, 10000); cudaDeviceSynchronize(); double h4[4]; cudaMemcpy(h4, d, 32, cudaMemcpyDeviceToHost); k<M><<<1, 32>>>(d, 10000);
    cudaDeviceSynchronize();
    double h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("%-40s %.1f cycles/round (4 warps)  %.1f (1 warp)\n", name, h4[0], h[0]);
}
int main() {
    double* d; cudaMalloc(&d, 8192 * 8);
    run<0>(d, "16 STS + sync + 8 LDS.128 + tree");
    run<1>(d, "1 STS + sync + 1 LDS");
    run<2>(d, "16 DMUL + DADD tree (depth 4)");
    run<3>(d, "8 dependent DADD");
    run<4>(d, "1 SHFL (double)");
    run<5>(d, "16 STS + sync + 1 LDS");
    run<6>(d, "1 STS + sync + 8 LDS.128 + tree");
    run<7>(d, "8 STS.128 + sync + 1 LDS");
    run<8>(d, "16 STS (no reload)");
    run<9>(d, "16 DMUL + butterfly SHFL reduction");
    return 0;
}
