// peak.cu -- FMA-pipe peak microbenchmark (roofline denominator).
//
// MEASURED_PEAKS.json carries HBM and bf16 only; the Jacobi kernels are bound
// by the FP64 (FP32 for single) FMA pipe, so bench.py measures that pipe's
// peak on the same box, same clocks: 8 independent FMA chains per thread,
// enough warps to saturate every SM.
#include <cuda_runtime.h>

#include "bsvd_b200.h"

namespace {

template <class F>
__global__ void __launch_bounds__(256) k_fma_peak(int iters, F seed, F* out) {
    F a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
      a7 = a0 + 7;
    const F b = (F)0.999999, c = (F)1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
            a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
        }
    }
    const F s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == (F)-1) out[blockIdx.x] = s;  // keep the chains alive
}

}  // namespace

extern "C" int bsvd_bench_fma_peak(int dtype, int blocks, int iters, void* out, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == BSVD_D) k_fma_peak<double><<<blocks, 256, 0, st>>>(iters, 1.0, static_cast<double*>(out));
    else if (dtype == BSVD_S) k_fma_peak<float><<<blocks, 256, 0, st>>>(iters, 1.0f, static_cast<float*>(out));
    else return BSVD_ERR_ARG;
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}
