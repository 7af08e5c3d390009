// launch.h -- internal planning/launch interface between api.cu and the kernels.
#pragma once

#include <type_traits>

#include <cuda_runtime.h>
#include <stddef.h>

#include "kernel_args.cuh"

namespace bsvd {

struct Plan {
    int kernel;         // KV_* variant
    int resident;       // residency bits (see SolveArgs::resident)
    size_t smem;        // dynamic shared memory per CTA
    size_t work_elems;  // global workspace elements per problem
    int threads;        // CTA size
    int group;          // lanes per pair (general unblocked)
    int grid;           // CTAs (0 = one per problem)
    int aux;            // kernel-specific (creg32: columns staged by the bulk-copy loader)
};

Plan plan_unblocked_general(int esize, int rsize, int bm, int bn, int need_v, size_t smem_limit);
Plan plan_blocked_general(int esize, int rsize, int bm, int bn, int nb, int need_v, size_t smem_limit);
Plan plan_blocked_dmma(int dtype, int bm, int bn, int nb, int need_v, bool contiguous, size_t smem_limit,
                       int variant);
int launch_blocked_dmma(SolveArgs<double> a, const Plan& p, cudaStream_t st);

template <class T>
int launch_unblocked_general(SolveArgs<T> a, const Plan& p, cudaStream_t st);
template <class T>
int launch_blocked_general(SolveArgs<T> a, const Plan& p, cudaStream_t st);
bool is_reg32b(int kv);
Plan plan_unblocked_reg32b(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant, int max_sweeps);
int split_tail(int batch, int sms, int override);  // 32x32 FP64: problems of a batch run as kernel 52's tail
int launch_unblocked_reg32b(SolveArgs<double> a, const Plan& p, cudaStream_t st);

template <class T>
int launch_finalize_ws(SolveArgs<T> a, cudaStream_t st);
template <class T>
int launch_finalize_gm(SolveArgs<T> a, cudaStream_t st);
template <class T>
int launch_finalize_flagged(SolveArgs<T> a, cudaStream_t st);
template <class T>
int launch_qr(SolveArgs<T> a, T* R, T* refl, T* phase, cudaStream_t st);
template <class T>
int launch_applyq(int bm, int bn, int batch, const T* refl, const T* phase, const T* UR, T* Out, int64_t ldo,
                  int64_t so, cudaStream_t st);
int launch_qr_path(bsvd_info* info, int batch, int bits, cudaStream_t st);
size_t qr_smem(int esize, int bm, int bn);
bool qr_reg_ok(int esize, bool cplx, int bm, int bn);
template <class T>
int launch_finalize_ext(int m, int n, int vrows, int batch, const void* W, int64_t ldw, int64_t sW, const void* V,
                        int64_t ldv, int64_t sV, void* U, int64_t ldu, int64_t sU, void* S, int64_t sS, void* Vo,
                        int64_t ldvo, int64_t svo, size_t smem_limit, cudaStream_t st);
template <class T>
int launch_householder_qr(int m, int n, int batch, const void* A, int64_t lda, int64_t sA, void* Q, int64_t ldq,
                          int64_t sQ, void* R, int64_t ldr, int64_t sR, void* work, size_t smem_limit, cudaStream_t st);
size_t householder_qr_work_bytes(int esize, int m, int n, int batch);
template <bool CX>
int launch_qr_col(SolveArgs<typename std::conditional<CX, cx<double>, double>::type> a,
                  typename std::conditional<CX, cx<double>, double>::type* R,
                  typename std::conditional<CX, cx<double>, double>::type* refl,
                  typename std::conditional<CX, cx<double>, double>::type* phase, cudaStream_t st);
template <bool CX>
int launch_applyq_col(int bm, int bn, int batch, const typename std::conditional<CX, cx<double>, double>::type* refl,
                      const typename std::conditional<CX, cx<double>, double>::type* phase,
                      const typename std::conditional<CX, cx<double>, double>::type* UR,
                      typename std::conditional<CX, cx<double>, double>::type* Out, int64_t ldo, int64_t so,
                      cudaStream_t st);
size_t heevj_workspace(int dtype, int n, int batch, size_t smem_limit);
int launch_heevj(int dtype, int n, int batch, const void* G, int64_t ldg, int64_t sG, void* D, int64_t sD, void* M,
                 int64_t ldm, int64_t sM, int m_init, double k, int max_sweeps, bsvd_info* info, void* work,
                 size_t work_bytes, size_t smem_limit, cudaStream_t st);
int launch_verify(int dtype, int m, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* U,
                  int64_t ldu, int64_t sU, const void* S, int64_t sS, const void* V, int64_t ldv, int64_t sV,
                  const double* Sref, int64_t sR, double* out, cudaStream_t st);
Plan plan_blocked_reg(int dtype, int bm, int bn, int nb, int need_v, bool contiguous, int inner_sweeps, int variant = 0);
int launch_blocked_reg(SolveArgs<double> a, const Plan& p, cudaStream_t st);
Plan plan_unblocked_reg16b(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant);
int launch_unblocked_reg16b(SolveArgs<float> a, const Plan& p, cudaStream_t st);
Plan plan_unblocked_reg16c(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant);
int launch_unblocked_reg16c(SolveArgs<float> a, const Plan& p, cudaStream_t st);
Plan plan_creg32(int dtype, int bm, int bn, int need_v, bool contiguous, int blocked, int nb, int variant,
                 size_t smem_limit);
int launch_creg32(SolveArgs<cx<double>> a, const Plan& p, cudaStream_t st);
Plan plan_cregb(int dtype, int bm, int bn, int need_v, bool trans, int nb);
int launch_cregb(SolveArgs<cx<double>> a, const Plan& p, cudaStream_t st);

int group_for_rows(int bm);
int threads_for(int bn, int G);

// kernel-level operators (bsvd_*_batched entry points)
template <class T>
int launch_onesided_raw(T* A, int64_t lda, int64_t sa, int m, int n, int batch, T* V, int64_t ldv, int64_t sv,
                        int vrows, double tol, int max_sweeps, int64_t* rot, int32_t* sw, cudaStream_t st);
template <class T>
int launch_gram_raw(const T* A, int64_t lda, int64_t sa, int m, int wi, int wj, int batch, T* G, int64_t ldg,
                    int64_t sg, cudaStream_t st);
template <class T>
int launch_fused_raw(T* B, int64_t ldb, int64_t sb, int m, int w, int batch, const T* J, int64_t ldj, int64_t sj,
                     int delta, cudaStream_t st);

}  // namespace bsvd
