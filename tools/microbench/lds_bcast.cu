// LDS.128 / LDS.64 broadcast cost on B200: cycles per warp-instruction per SM for address patterns
// (full-warp broadcast, two half-warp addresses in the same / different banks, distinct per lane).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench/lds_bcast.cu -o tools/microbench/lds_bcast
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT, int W>
__global__ void k(double* out, int iters) {
    __shared__ __align__(16) double buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = i * 1e-3;
    __syncthreads();
    const int lane = threadIdx.x & 31, half = lane >> 4;
    int base;
    if (PAT == 0) base = 0;                       // one address for the warp
    else if (PAT == 1) base = half * 32;          // two addresses, 256 B apart (same banks)
    else if (PAT == 2) base = half * 2;           // two addresses, 16 B apart (different banks)
    else base = lane * 2;                         // distinct, conflict-free
    double acc0 = 0, acc1 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int off = ((q * 64 + it * 8) & 1023) + base;
            if (W == 128) {
                const double2 v = *reinterpret_cast<const double2*>(&buf[off]);
                acc0 += v.x; acc1 += v.y;
            } else {
                acc0 += buf[off];
            }
        }
    }
    if (acc0 + acc1 == 12345.0) out[threadIdx.x] = acc0;
}

template <int PAT, int W>
void run(const char* name) {
    double* out; cudaMalloc(&out, 4096 * 8);
    const int iters = 4096, blocks = 148 * 4, threads = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<PAT, W><<<blocks, threads>>>(out, 16);
    cudaEventRecord(a);
    k<PAT, W><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double instr_per_sm = (double)blocks / 148 * threads / 32 * iters * 16;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-34s LDS.%d: %.2f cycles per warp-instruction per SM\n", name, W, cyc / instr_per_sm);
    cudaFree(out);
}

int main() {
    run<0, 128>("full-warp broadcast");
    run<1, 128>("2 addresses, same banks");
    run<2, 128>("2 addresses, different banks");
    run<3, 128>("distinct per lane");
    run<0, 64>("full-warp broadcast");
    run<1, 64>("2 addresses, same banks");
    run<2, 64>("2 addresses, different banks");
    run<3, 64>("distinct per lane");
    return 0;
}
