// finalize.cu -- kernel (5) as a standalone pass for the register-resident
// solvers: the raw converged working copy W (bm x bn) and V (bn x bn) sit in
// the workspace; one CTA per problem stages them in shared memory and runs
// the shared finalisation routine (finalize.cuh: sigma in float64, tiny-column
// completion, stable descending sort, permuted U/V, transpose swap).
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {

template <class T>
__device__ __forceinline__ void finalize_one_ws(const SolveArgs<T>& a, int prob, unsigned char* smem) {
    using R = typename tr<T>::R;
    const int bm = a.bm, bn = a.bn;
    const T* src = a.work + (size_t)prob * a.work_stride;
    T* W = reinterpret_cast<T*>(smem);
    T* Vw = a.need_v ? W + (size_t)bm * bn : nullptr;
    size_t off = ((size_t)bm * bn + (a.need_v ? (size_t)bn * bn : 0)) * sizeof(T);
    off = (off + 15) & ~size_t(15);
    R* sig = reinterpret_cast<R*>(smem + off);
    off += ((size_t)bn * sizeof(R) + 15) & ~size_t(15);
    int* perm = reinterpret_cast<int*>(smem + off);
    off += ((size_t)bn * sizeof(int) + 15) & ~size_t(15);
    int* flag = reinterpret_cast<int*>(smem + off);
    const int total = bm * bn + (a.need_v ? bn * bn : 0);
    for (int e = threadIdx.x; e < total; e += blockDim.x) W[e] = src[e];
    __syncthreads();
    finalize_block<T>(W, bm, bm, bn, Vw, bn, sig, perm, flag, final_out(a, prob));
}

template <class T>
__device__ __forceinline__ bool flag_set(const SolveArgs<T>& a, int prob) {
    const T f = a.work[(size_t)prob * a.work_stride + a.work_stride - 1];
    if constexpr (tr<T>::cplx) return f.re != 0;
    else return f != 0;
}

// FLAGGED: the pass after a solver that finalised most problems itself.  One thread per problem reads its
// flag (CTA c covers problems 128 c .. 128 c + 127), and the CTA finalises the flagged ones in turn --
// instead of one CTA per problem that mostly exits at once (C2: 7.3 us for 10,000 empty CTAs).
template <class T, bool FLAGGED = false>
__global__ void __launch_bounds__(128) k_finalize_ws(SolveArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    if constexpr (FLAGGED) {
        __shared__ int list[128];
        __shared__ int cnt;
        if (threadIdx.x == 0) cnt = 0;
        __syncthreads();
        const int p = blockIdx.x * 128 + threadIdx.x;
        if (p < a.batch && flag_set(a, p)) list[atomicAdd(&cnt, 1)] = p;
        __syncthreads();
        const int nf = cnt;
        for (int j = 0; j < nf; ++j) {
            finalize_one_ws(a, list[j], smem);
            __syncthreads();  // the staging buffer is reused for the next flagged problem
        }
    } else {
        finalize_one_ws(a, blockIdx.x, smem);
    }
}

template <class T, bool FLAGGED>
static int launch_finalize_impl(SolveArgs<T> a, cudaStream_t st) {
    const size_t es = sizeof(T);
    size_t smem = ((size_t)a.bm * a.bn + (a.need_v ? (size_t)a.bn * a.bn : 0)) * es;
    smem = ((smem + 15) & ~size_t(15)) + (((size_t)a.bn * sizeof(typename tr<T>::R) + 15) & ~size_t(15)) +
           (((size_t)a.bn * 4 + 15) & ~size_t(15)) + 16;
    auto k = k_finalize_ws<T, FLAGGED>;
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return BSVD_ERR_CUDA;
    }
    k<<<FLAGGED ? (a.batch + 127) / 128 : a.batch, 128, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template <class T>
int launch_finalize_ws(SolveArgs<T> a, cudaStream_t st) {
    return launch_finalize_impl<T, false>(a, st);
}
template <class T>
int launch_finalize_flagged(SolveArgs<T> a, cudaStream_t st) {
    return launch_finalize_impl<T, true>(a, st);
}
template int launch_finalize_flagged<double>(SolveArgs<double>, cudaStream_t);
template int launch_finalize_flagged<float>(SolveArgs<float>, cudaStream_t);

// Finalisation in place in the workspace (global / L2): for solvers whose W
// and V live in the workspace and are too large to stage in shared memory.
template <class T>
__global__ void __launch_bounds__(256) k_finalize_gm(SolveArgs<T> a) {
    using R = typename tr<T>::R;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x;
    T* W = a.work + (size_t)prob * a.work_stride;
    T* Vw = a.need_v ? W + (size_t)a.bm * a.bn : nullptr;
    R* sig = reinterpret_cast<R*>(smem);
    int* perm = reinterpret_cast<int*>(smem + (((size_t)a.bn * sizeof(R) + 15) & ~size_t(15)));
    int* flag = perm + ((a.bn + 3) & ~3);
    finalize_block<T>(W, a.bm, a.bm, a.bn, Vw, a.bn, sig, perm, flag, final_out(a, prob));
}

template <class T>
int launch_finalize_gm(SolveArgs<T> a, cudaStream_t st) {
    const size_t smem = (((size_t)a.bn * sizeof(typename tr<T>::R) + 15) & ~size_t(15)) +
                        (size_t)((a.bn + 3) & ~3) * 4 + 16;
    k_finalize_gm<T><<<a.batch, 256, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

// The finalize operator on caller buffers (finalize(work_a, v), src/svd.py:278-303): W (m x n, ldw) and
// V (vrows x n, ldv) staged in shared memory, U / sigma / permuted V written to the outputs.
template <class T>
__global__ void __launch_bounds__(128) k_finalize_ext(int m, int n, int vrows, const T* W, int64_t ldw, int64_t sW,
                                                      const T* V, int64_t ldv, int64_t sV, T* U, int64_t ldu,
                                                      int64_t sU, typename tr<T>::R* S, int64_t sS, T* Vo,
                                                      int64_t ldvo, int64_t svo) {
    using R = typename tr<T>::R;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x;
    T* Ws = reinterpret_cast<T*>(smem);
    T* Vs = Ws + (size_t)m * n;
    size_t off = ((size_t)m * n + (size_t)vrows * n) * sizeof(T);
    off = (off + 15) & ~size_t(15);
    R* sig = reinterpret_cast<R*>(smem + off);
    off += ((size_t)n * sizeof(R) + 15) & ~size_t(15);
    int* perm = reinterpret_cast<int*>(smem + off);
    off += ((size_t)n * sizeof(int) + 15) & ~size_t(15);
    int* flag = reinterpret_cast<int*>(smem + off);
    const T* Wp = W + (size_t)prob * sW;
    for (int e = threadIdx.x; e < m * n; e += blockDim.x) Ws[e] = Wp[(e % m) + (size_t)(e / m) * ldw];
    if (V) {
        const T* Vp = V + (size_t)prob * sV;
        for (int e = threadIdx.x; e < vrows * n; e += blockDim.x) Vs[e] = Vp[(e % vrows) + (size_t)(e / vrows) * ldv];
    }
    __syncthreads();
    FinalOut<T> o;
    o.U = U + (size_t)prob * sU;
    o.ldu = ldu;
    o.S = S + (size_t)prob * sS;
    o.V = V ? Vo + (size_t)prob * svo : nullptr;
    o.ldv = ldvo;
    o.trans = false;
    o.want_v = V != nullptr;
    finalize_block<T>(Ws, m, m, n, V ? Vs : nullptr, vrows, sig, perm, flag, o, vrows);
}

size_t finalize_ext_smem(int esize, int rsize, int m, int n, int vrows) {
    size_t smem = ((size_t)m * n + (size_t)vrows * n) * esize;
    return ((smem + 15) & ~size_t(15)) + (((size_t)n * rsize + 15) & ~size_t(15)) + (((size_t)n * 4 + 15) & ~size_t(15)) +
           16;
}

template <class T>
int launch_finalize_ext(int m, int n, int vrows, int batch, const void* W, int64_t ldw, int64_t sW, const void* V,
                        int64_t ldv, int64_t sV, void* U, int64_t ldu, int64_t sU, void* S, int64_t sS, void* Vo,
                        int64_t ldvo, int64_t svo, size_t smem_limit, cudaStream_t st) {
    const size_t smem = finalize_ext_smem(sizeof(T), sizeof(typename tr<T>::R), m, n, V ? vrows : 0);
    if (smem > smem_limit) return BSVD_ERR_UNSUPPORTED;
    auto k = k_finalize_ext<T>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<batch, 128, smem, st>>>(m, n, V ? vrows : 0, static_cast<const T*>(W), ldw, sW, static_cast<const T*>(V), ldv,
                                sV, static_cast<T*>(U), ldu, sU, static_cast<typename tr<T>::R*>(S), sS,
                                static_cast<T*>(Vo), ldvo, svo);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}
#define BSVD_FIN_EXT(T)                                                                                          \
    template int launch_finalize_ext<T>(int, int, int, int, const void*, int64_t, int64_t, const void*, int64_t, \
                                        int64_t, void*, int64_t, int64_t, void*, int64_t, void*, int64_t, int64_t, \
                                        size_t, cudaStream_t);
BSVD_FIN_EXT(float)
BSVD_FIN_EXT(double)
BSVD_FIN_EXT(cx<float>)
BSVD_FIN_EXT(cx<double>)

template int launch_finalize_gm<double>(SolveArgs<double>, cudaStream_t);
template int launch_finalize_gm<cx<double>>(SolveArgs<cx<double>>, cudaStream_t);

template int launch_finalize_ws<float>(SolveArgs<float>, cudaStream_t);
template int launch_finalize_ws<double>(SolveArgs<double>, cudaStream_t);
template int launch_finalize_ws<cx<float>>(SolveArgs<cx<float>>, cudaStream_t);
template int launch_finalize_ws<cx<double>>(SolveArgs<cx<double>>, cudaStream_t);

}  // namespace bsvd
