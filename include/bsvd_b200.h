/*
 * bsvd_b200.h -- C-ABI of the B200-native batched one-sided Jacobi SVD.
 *
 * This is the drop-in boundary for the reference's hot path
 *   batch_svd(problems, opts, state)            /root/reference/pkg/src/bsvd/batch.py:85-157
 * and the kernel operator API it drives through
 *   Backend(onesided_sweeps, eig_sweeps, fused_pair_update)
 *                                               /root/reference/pkg/src/bsvd/backend.py:30-35
 *   onesided_sweeps   src/_kernels_numba.py:85-138   (unblocked sweeps, per problem)
 *   eig_sweeps        src/_kernels_numba.py:17-82    (inner Gram eigensolve, blocked path)
 *   fused_pair_update src/_kernels_numba.py:141-175  (W += W * Delta, V += V * Delta)
 *   compute_gram      src/svd.py:144-179
 *   _finalize_factors src/svd.py:243-275
 * The reference calls those once per problem per sweep from Python; here one
 * call solves a whole uniform-shape batch on the device (all sweeps, the
 * per-problem convergence test of src/batch.py:62-82 and finalisation).
 *
 * Conventions: plain pointers and sizes, no torch or CUDA types.  All array
 * pointers are DEVICE pointers; matrices are column-major (src/core.py:1-7),
 * complex values interleaved (re, im).  `stream` is a cudaStream_t passed as
 * void* (NULL = legacy default stream).  Calls are stream-ordered, reentrant,
 * never allocate, never synchronise, and use the current device.
 */
#ifndef BSVD_B200_H
#define BSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSVD_ABI_VERSION 1

/* element types; codes equal src/fileio.py:49-54 (s, d, c, z) */
typedef enum { BSVD_S = 0, BSVD_D = 1, BSVD_C = 2, BSVD_Z = 3 } bsvd_dtype;

/* solver routes (src/svd.py:559-582): dispatch = svd_dispatch, the others force
   (FORCE_QR = svd_qr_preprocessed: Householder QR first whatever the aspect ratio) */
enum { BSVD_DISPATCH = 0, BSVD_FORCE_UNBLOCKED = 1, BSVD_FORCE_BLOCKED = 2, BSVD_FORCE_QR = 3 };

/* JacobiOptions (src/svd.py:58-91) as a POD. */
typedef struct {
    double k;           /* rotation-guard multiplier, tol = k*u              */
    int max_sweeps;     /* max_nsweeps                                       */
    int nb;             /* block width of the blocked path                   */
    int inner_sweeps;   /* inner eigensolver sweeps per block pair (0 = 100) */
    int masking;        /* accepted for parity; every problem exits on its own quiet sweep */
    int want_v;         /* compute_right_vectors                             */
    int route;          /* BSVD_DISPATCH / BSVD_FORCE_*                      */
    int fused_updates;  /* accepted for parity; updates are always fused     */
    int row_block;      /* accepted for parity (tiling is the kernel's own)  */
    int kernel;         /* 0 = auto; >0 forces a kernel variant (tests/bench) */
    int use_qr;         /* use_qr_preprocess: dispatch takes the "qr+" route when m >= 3n (QR_RATIO) */
    int reserved[2];    /* [0]: 32x32 FP64 kernel 52 (0 = automatic: one-wave batches and the tail of larger ones; > 0 = that
                           many tail problems; < 0 = off, kernel 42 alone; experimental); [1]: 0 */
} bsvd_opts;

/* Per-problem telemetry, written by the device (mirrors SolveInfo / BatchState). */
typedef struct {
    int32_t converged;      /* quiet sweep reached within max_sweeps              */
    int32_t outer_sweeps;   /* sweeps up to and including the quiet one           */
    int64_t rotations;      /* SolveInfo.inner_rotations                          */
    int64_t gram_calls;     /* blocked path: Gram formations                      */
    int64_t update_calls;   /* blocked path: pair updates applied                 */
    int32_t last_rotations; /* rotations applied in the final sweep               */
    int32_t path;           /* 1 unblocked, 2 blocked (| 0x100 transposed, | 0x200 qr) */
    int32_t status;         /* 0 ok, 1 non-finite input                           */
    int32_t kernel;         /* kernel variant that ran                            */
} bsvd_info;

/* Status codes returned by the calls. */
enum {
    BSVD_OK = 0,
    BSVD_ERR_ARG = -1,       /* bad dtype / shape / stride / option   */
    BSVD_ERR_WORKSPACE = -2, /* work_bytes smaller than required      */
    BSVD_ERR_CUDA = -3,      /* kernel launch failed                  */
    BSVD_ERR_UNSUPPORTED = -4
};

/*
 * Batched economy SVD of `batch` matrices A_b (m x n, any m, n >= 0):
 *   A_b = U_b diag(S_b) V_b^H,  k = min(m, n)
 * A_b  at A + b*strideA, leading dimension lda >= m        (input, not modified)
 * U_b  at U + b*strideU, m x k, ldu >= m                   (output)
 * S_b  at S + b*strideS, k real values, descending         (output; real dtype)
 * V_b  at V + b*strideV, n x k, ldv >= n, or V == NULL      (output if want_v)
 * info: device array of `batch` bsvd_info (may be NULL).
 * Wide inputs (m < n) are solved through A^H with U and V swapped
 * ("transpose+" route, src/svd.py:346-347, :531-536).
 * work: device scratch of bsvd_workspace_bytes(...) bytes (may be 0 bytes).
 * Strides and leading dimensions are in elements.
 */
int bsvd_gesvj_batched(int dtype, int m, int n, int batch,
                       const void* A, int64_t lda, int64_t strideA,
                       void* U, int64_t ldu, int64_t strideU,
                       void* S, int64_t strideS,
                       void* V, int64_t ldv, int64_t strideV,
                       const bsvd_opts* opts, bsvd_info* info,
                       void* work, size_t work_bytes, void* stream);

/*
 * Host-buffer variant: the same solve with A, U, S, V and info in HOST memory
 * (pinned for full PCIe bandwidth; dense packing required: lda = m,
 * strideA = m*n, ldu = m, strideU = m*k, strideS = k, ldv = n, strideV = n*k).
 * The batch is cut into chunks of `chunk` problems that are pipelined over
 * the caller's `nstreams` streams (H2D of one chunk, the solve of another and
 * the D2H of a third overlap); work is ordered after prior work on
 * streams[0], and streams[0] is ordered after all of it on return, so the call
 * behaves like one stream-ordered operation on streams[0].  `work` is DEVICE
 * scratch of bsvd_host_workspace_bytes(...) bytes (staging for nstreams
 * chunks plus their solver workspace).  Chunks on different streams solve
 * concurrently, so when the chunks in flight (one per stream) exceed two
 * waves of kernel 52 (16 problems per SM) a 32x32 FP64 batch solves with
 * kernel 42 alone (the throughput kernel; factors bitwise those of the
 * one-call solve).  Asynchronous: synchronise streams[0]
 * before reading the outputs.  Replaces the reference's per-problem host loop
 * batch_svd -> _ProblemRun (src/batch.py:85-157) for host-resident batches.
 */
int bsvd_gesvj_batched_host(int dtype, int m, int n, int batch,
                            const void* A, void* U, void* S, void* V,
                            const bsvd_opts* opts, bsvd_info* info,
                            int chunk, void* work, size_t work_bytes,
                            void* const* streams, int nstreams);

/*
 * bsvd_gesvj_batched_host for a LIST of host matrices (the reference's batch_svd input, a list of
 * column-major m x n problems, src/batch.py:85-157): A_ptrs[b] points at problem b (m*n contiguous
 * column-major elements, any host memory); A_stage is page-locked host memory of batch*m*n elements
 * that receives the packed batch.  `pack_threads` host threads pack chunk after chunk while the
 * pipeline transfers and solves the chunks already packed, so packing overlaps the device work.
 * Outputs, streams and workspace as for bsvd_gesvj_batched_host; returns after every chunk is packed
 * and enqueued (A_ptrs may be released then; A_stage only after streams[0] completes).
 */
int bsvd_gesvj_batched_host_gather(int dtype, int m, int n, int batch,
                                   const void* const* A_ptrs, void* A_stage, int pack_threads,
                                   void* U, void* S, void* V,
                                   const bsvd_opts* opts, bsvd_info* info,
                                   int chunk, void* work, size_t work_bytes,
                                   void* const* streams, int nstreams);

/* Device scratch needed by bsvd_gesvj_batched_host for (chunk, nstreams). */
size_t bsvd_host_workspace_bytes(int dtype, int m, int n, int chunk, int nstreams, const bsvd_opts* opts);

/*
 * Batched Hermitian eigensolver by cyclic Jacobi rotations (the reference's
 * standalone jacobi_hermitian_eig, src/eig.py:90-148, on eig_sweeps
 * src/_kernels_numba.py:17-82).  G_b: n x n Hermitian (DEVICE, ldg; only the
 * upper triangle and the real part of the diagonal are read), D_b: n real
 * eigenvalues (unsorted, like the reference), M_b: n x n eigenvector matrix
 * (ldm) with G ~= M diag(D) M^H; when m_init != 0 M_b holds the starting
 * matrix and the rotations are accumulated into it (the reference's eigvecs=
 * argument), else it starts as the identity.  Guard k*u*sqrt(|d_i||d_j|),
 * at most max_sweeps sweeps; info (may be NULL): outer_sweeps = sweeps_run
 * (quiet sweep included), rotations, converged.  work: DEVICE scratch of
 * bsvd_heevj_workspace_bytes(...) bytes (0 when G and M fit in shared memory).
 */
/*
 * eig_sweeps(g, d, m, pairs, starts, tol, max_sweeps, delta) (src/_kernels_numba.py:17-82), the
 * reference's Backend operator, batch-granular and in place: G_b n x n (only the off-diagonal is read;
 * rotated in place, pivots zeroed, diagonal untouched), D_b the n real pivots (in/out), M_b n x n
 * accumulator (in/out; delta != 0: M accumulates P - I including the identity columns' terms, start
 * it at zero).  Absolute guard tol (= k u).  info: sweeps run, rotations, converged.  Workspace as
 * bsvd_heevj_workspace_bytes.  Disjoint pairs of an iteration are applied together (2 x 2 block
 * updates), so results match the sequential reference to rounding.
 */
int bsvd_eig_sweeps_batched(int dtype, int n, int batch, void* G, int64_t ldg, int64_t strideG, void* D,
                            int64_t strideD, void* M, int64_t ldm, int64_t strideM, double tol, int max_sweeps,
                            int delta, bsvd_info* info, void* work, size_t work_bytes, void* stream);
int bsvd_heevj_batched(int dtype, int n, int batch, const void* G, int64_t ldg, int64_t strideG,
                       void* D, int64_t strideD, void* M, int64_t ldm, int64_t strideM, int m_init,
                       double k, int max_sweeps, bsvd_info* info, void* work, size_t work_bytes, void* stream);
size_t bsvd_heevj_workspace_bytes(int dtype, int n, int batch);

/*
 * On-device accuracy metrics of a solved batch (the reference's verify.py:44-84,
 * float64 accumulation), written to out[4*b .. 4*b+3] (DEVICE doubles):
 *   e1 = |A - U diag(S) V^H|_1 / (n |A|_1)   (NaN when V is NULL)
 *   e2 = |I - U^H U|_1 / m,  e3 = |I - V^H V|_1 / n   (e3 NaN without V)
 *   e4 = |S - Sref|_F / min(m, n)             (NaN when Sref is NULL; Sref float64)
 * All pointers DEVICE, column-major, the layouts of bsvd_gesvj_batched's outputs.
 */
int bsvd_verify_batched(int dtype, int m, int n, int batch,
                        const void* A, int64_t lda, int64_t strideA,
                        const void* U, int64_t ldu, int64_t strideU,
                        const void* S, int64_t strideS,
                        const void* V, int64_t ldv, int64_t strideV,
                        const double* Sref, int64_t strideSref, double* out, void* stream);

/* Device scratch needed by bsvd_gesvj_batched for this problem class (any lda >= m). */
size_t bsvd_workspace_bytes(int dtype, int m, int n, int batch, const bsvd_opts* opts);

/* Kernel variant the auto-dispatch would pick (for telemetry/tests); the choice may depend on the
 * batch size (16x16 FP32 switches to the quarter-warp kernel from 3,500 problems): the _batched form
 * answers for `batch` problems, the plain form for batch = 0. */
int bsvd_select_kernel(int dtype, int m, int n, const bsvd_opts* opts);
int bsvd_select_kernel_batched(int dtype, int m, int n, int batch, const bsvd_opts* opts);

/* Fill opts with the reference defaults (JacobiOptions(), src/svd.py:70-78). */
void bsvd_default_opts(bsvd_opts* opts);

const char* bsvd_strerror(int code);
int bsvd_abi_version(void);

/*
 * Kernel-level operator entry points, batch-granular versions of the
 * reference's Backend plugin functions (src/backend.py:30-35).  Each works on
 * `batch` independent problems in place on the device and returns per-problem
 * rotation counts in rotations[] (device int64, may be NULL).
 *
 * bsvd_onesided_sweeps_batched ~ onesided_sweeps(a, v, pairs, starts, tol, max_sweeps);
 *   sweeps[b] = sweeps run, bit 30 set when the last sweep was quiet (converged).
 *   a: m x n (lda), v: vrows x n (ldv) or NULL (vrows = 0).
 * bsvd_gram_batched ~ compute_gram(ai, aj) with ai = a[:, 0:wi], aj = a[:, wi:wi+wj]
 *   g: (wi+wj) x (wi+wj), ldg.
 * bsvd_fused_pair_update_batched ~ fused_pair_update(bi, bj, j, row_block, delta)
 *   b: m x (wi+wj) (ldb) holding [bi bj] side by side, j: w x w (ldj).
 */
int bsvd_onesided_sweeps_batched(int dtype, int m, int n, int batch, void* a, int64_t lda,
                                 int64_t stride_a, int vrows, void* v, int64_t ldv,
                                 int64_t stride_v, double tol, int max_sweeps,
                                 int64_t* rotations, int32_t* sweeps, void* stream);
int bsvd_gram_batched(int dtype, int m, int wi, int wj, int batch, const void* a, int64_t lda,
                      int64_t stride_a, void* g, int64_t ldg, int64_t stride_g, void* stream);
int bsvd_fused_pair_update_batched(int dtype, int m, int w, int batch, void* b, int64_t ldb,
                                   int64_t stride_b, const void* j, int64_t ldj, int64_t stride_j,
                                   int delta, void* stream);

/*
 * finalize(work_a, v) (src/svd.py:278-303; _finalize_factors src/svd.py:243-275) as a batched
 * operator: W m x n (ldw, m >= n) -> sigma (float64 column norms cast to the real dtype),
 * U = W / sigma with orthogonal completion of columns below tiny/u, stable descending order;
 * V (vrows x n, ldv) or NULL is permuted alike into Vout.  Inputs are not modified.
 */
int bsvd_finalize_batched(int dtype, int m, int n, int batch, const void* W, int64_t ldw, int64_t stride_w,
                          int vrows, const void* V, int64_t ldv, int64_t stride_v, void* U, int64_t ldu,
                          int64_t stride_u, void* S, int64_t stride_s, void* Vout, int64_t ldvo,
                          int64_t stride_vout, void* stream);

/*
 * householder_qr(a) (src/core.py:118-168) as a batched operator: A m x n (m >= n) -> Q m x n with
 * orthonormal columns and R n x n upper triangular with a real non-negative diagonal (the
 * reference's sign convention), A = Q R.  Device workspace: bsvd_householder_qr_workspace_bytes.
 */
size_t bsvd_householder_qr_workspace_bytes(int dtype, int m, int n, int batch);
int bsvd_householder_qr_batched(int dtype, int m, int n, int batch, const void* a, int64_t lda,
                                int64_t stride_a, void* q, int64_t ldq, int64_t stride_q, void* r, int64_t ldr,
                                int64_t stride_r, void* work, size_t work_bytes, void* stream);

/*
 * Host helper for the list API: dst[i * bytes .. ] = src[i][0 .. bytes) for i < count, over
 * nthreads host threads (packs a list of column-major matrices into the pinned batch layout).
 */
int bsvd_pack_host(const void* const* src, int count, size_t bytes, void* dst, int nthreads);

/*
 * Diagnostics: FMA-pipe peak microbenchmark used as the roofline denominator
 * (dtype BSVD_D or BSVD_S).  Launches blocks x 256 threads, each running
 * iters x 128 dependent-free FMAs; out: device scratch of `blocks` elements.
 * Flops = 2 * 128 * 256 * blocks * iters.
 */
int bsvd_bench_fma_peak(int dtype, int blocks, int iters, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BSVD_B200_H */
