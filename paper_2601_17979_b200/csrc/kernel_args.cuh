// kernel_args.cuh -- argument blocks shared by the launchers and kernels.
#pragma once

#include "finalize.cuh"

namespace bsvd {

// One uniform-shape batch, as seen by every solver kernel.
template <class T>
struct SolveArgs {
    using R = typename tr<T>::R;
    const T* A;          // user input, m x n column-major
    int64_t lda, strideA;
    int m, n;            // user shape
    int trans;           // 1: solve A^H (m < n), factors swapped on output
    int bm, bn;          // working shape (bm >= bn)
    T* U;
    int64_t ldu, strideU;
    R* S;
    int64_t strideS;
    T* V;
    int64_t ldv, strideV;
    int want_v;          // caller wants V
    int need_v;          // V accumulated (want_v or trans)
    double tol;          // k * u
    int max_sweeps;
    int nb;              // blocked path block width
    int inner_budget;    // inner sweeps per block pair (inner_sweeps or 100)
    int batch;
    T* work;             // global residency for W/V (and Gram/Delta) when smem is too small
    int64_t work_stride; // elements per problem
    int resident;        // bit0: W in smem, bit1: V in smem, bit2: scratch in smem
    int group;           // lanes per column pair (general unblocked kernel)
    int kernel;          // variant id for telemetry
    bsvd_info* info;
};

// Kernel variant ids (bsvd_info.kernel).  Ids of retired round-1/round-2 experiments are not reused
// (profiles/r2_c1_kernel_experiments.md).
enum {
    KV_UNBLOCKED_GENERAL = 1,
    KV_BLOCKED_GENERAL = 2,
    KV_BLOCKED_DMMA = 8,        // blocked FP64, nb = 16, Gram/update on DMMA tensor cores
    KV_BLOCKED_DMMA_VG = 9,     // same, V kept in global memory (L2), 3 CTAs/SM
    KV_BLOCKED_DMMA_512 = 10,   // same, 512-thread CTAs (16 warps) for one-CTA-per-SM sizes
    KV_UNBLOCKED_REG32B = 12,   // 32x32 FP64 second generation: unrolled ring, maintained norms, two-FMA
    KV_UNBLOCKED_REG16B = 24,   // 16x16 FP32 second generation: 2 problems per warp, row per lane
    KV_HEEVJ = 31,              // batched Hermitian Jacobi eigensolver (bsvd_heevj_batched)
    KV_BLOCKED_REG = 30,        // blocked FP64: block pairs register-resident (kernel (2) on X), V P on DMMA
    KV_CREG32 = 32,             // complex FP64, n = 32, m <= 256: CTA per problem, rows in registers, V in smem
    KV_UNBLOCKED_REG16C = 34,   // 16x16 FP32 third generation: 4 problems per warp, 2 rows per lane
    KV_CREGB = 51,              // complex FP64 blocked (n > 32): block pairs through the complex register iteration
    KV_CREG32_TMA = 45,         // KV_CREG32 with the bulk-copy (TMA) loader: 1-3 % slower, opt-in
                                //   (profiles/r2_tma_loader.md)
    KV_UNBLOCKED_REG32G = 42,   // KV_UNBLOCKED_REG32B with scaled (fast) rotations: one FMA per updated element
    KV_UNBLOCKED_REG32F = 52,   // KV_UNBLOCKED_REG32G, one problem per warp with V in lockstep (small batches)
};

template <class T>
BSVD_DEV void load_problem(const SolveArgs<T>& a, int prob, T* W, int ldw, T* Vw, int ldvw, int* bad) {
    const T* Ap = a.A + (size_t)prob * a.strideA;
    const int tid = threadIdx.x, nt = blockDim.x;
    int nonfinite = 0;
    // kernel (1): coalesced column-major loads; the transpose route reads A
    // along its own columns and scatters the conjugate into W (src/svd.py:346-347)
    const int total = a.m * a.n;
    for (int e = tid; e < total; e += nt) {
        const int r = e % a.m, c = e / a.m;
        const T x = Ap[r + (size_t)c * a.lda];
        nonfinite |= !finiteT(x);
        if (a.trans) W[c + (size_t)r * ldw] = conjT(x);
        else W[r + (size_t)c * ldw] = x;
    }
    if (a.need_v) {
        for (int e = tid; e < a.bn * a.bn; e += nt) {
            const int r = e % a.bn, c = e / a.bn;
            Vw[r + (size_t)c * ldvw] = (r == c) ? one<T>() : zero<T>();
        }
    }
    if (nonfinite) atomicOr(bad, 1);
}

template <class T>
BSVD_DEV FinalOut<T> final_out(const SolveArgs<T>& a, int prob) {
    FinalOut<T> o;
    o.U = a.U + (size_t)prob * a.strideU;
    o.ldu = a.ldu;
    o.S = a.S + (size_t)prob * a.strideS;
    o.V = a.V ? a.V + (size_t)prob * a.strideV : nullptr;
    o.ldv = a.ldv;
    o.trans = a.trans != 0;
    o.want_v = a.want_v != 0;
    return o;
}

}  // namespace bsvd
