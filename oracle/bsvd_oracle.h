/*
 * bsvd_oracle.h -- CPU restatement of the reference batched one-sided Jacobi SVD.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels and the "port" CPU baseline timed by bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_2601_17979_b200) never links it.
 *
 * Every routine restates a function of the reference package
 * /root/reference/pkg/src/bsvd (cited as src/<file>:<line> in the .cpp).
 * Pinning: tests/test_oracle.py checks it against golden vectors produced by
 * the reference itself (tests/golden/make_golden.py).
 */
#ifndef BSVD_ORACLE_H
#define BSVD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes follow src/fileio.py:49-54 (s, d, c, z) */
enum { ORC_S = 0, ORC_D = 1, ORC_C = 2, ORC_Z = 3 };

/* force codes: 0 = svd_dispatch, 1 = svd_unblocked, 2 = svd_blocked, 3 = svd_qr_preprocessed */
typedef struct {
    double k;            /* JacobiOptions.k            src/svd.py:70 */
    int max_nsweeps;     /* JacobiOptions.max_nsweeps  src/svd.py:71 */
    int nb;              /* JacobiOptions.nb           src/svd.py:72 */
    int inner_sweeps;    /* JacobiOptions.inner_sweeps src/svd.py:73 */
    int want_v;          /* compute_right_vectors      src/svd.py:76 */
    int fused_updates;   /* JacobiOptions.fused_updates src/svd.py:77 */
    int row_block;       /* JacobiOptions.row_block    src/svd.py:78 */
    int force;           /* 0 dispatch, 1 unblocked, 2 blocked, 3 qr */
    int use_qr;          /* JacobiOptions.use_qr_preprocess src/svd.py:75 */
} orc_opts;

/* path codes */
enum { ORC_PATH_EMPTY = 0, ORC_PATH_UNBLOCKED = 1, ORC_PATH_BLOCKED = 2 };

typedef struct {
    int32_t converged;        /* SolveInfo.converged        */
    int32_t outer_sweeps;     /* SolveInfo.outer_sweeps     */
    int64_t inner_rotations;  /* SolveInfo.inner_rotations  */
    int32_t path;             /* ORC_PATH_*                 */
    int32_t transposed;       /* "transpose+" prefix        */
    int64_t gram_calls;       /* WorkCounters (per problem, standalone run) */
    int64_t eig_calls;
    int64_t update_calls;
    int32_t status;           /* 0 ok, <0 error */
    int32_t qr;               /* "qr+" route taken          */
} orc_info;

/*
 * Solve one problem (standalone svd_* semantics, src/svd.py:550-582).
 * a: m x n column-major, leading dimension m.  Outputs with k = min(m, n):
 *   u: m x k column-major (ld m), s: k real values, v: n x k (ld n) or NULL.
 * Returns 0 on success, negative on argument error.
 */
int orc_solve(int dtype, int m, int n, const void* a, void* u, void* s, void* v,
              const orc_opts* opts, orc_info* info);

/* Batch of equal-shape problems, contiguous (stride m*n / m*k / k / n*k).
 * nthreads <= 0 uses all available threads (OpenMP). */
int orc_solve_batch(int dtype, int m, int n, int batch, const void* a, void* u, void* s,
                    void* v, const orc_opts* opts, orc_info* info, int nthreads);

/* Kernel-level restatements (one problem, one call), for unit tests. */
/* onesided_sweeps, src/_kernels_numba.py:85-138.  Returns rotations; *sweeps and *conv out. */
int64_t orc_onesided_sweeps(int dtype, int m, int n, void* a, int vrows, void* v, double tol,
                            int max_sweeps, int* sweeps, int* conv);
/* eig_sweeps, src/_kernels_numba.py:17-82.  g: w x w, d: w (real), mm: mrows x w */
int64_t orc_eig_sweeps(int dtype, int w, void* g, void* d, int mrows, void* mm, double tol,
                       int max_sweeps, int delta, int* sweeps, int* conv);
/* compute_gram, src/svd.py:144-179: g = [Ai Aj]^H [Ai Aj], w = wi + wj */
void orc_compute_gram(int dtype, int m, int wi, int wj, const void* ai, const void* aj, void* g);
/* fused_pair_update, src/_kernels_numba.py:141-175 */
void orc_fused_pair_update(int dtype, int m, int wi, int wj, void* bi, void* bj, const void* j,
                           int row_block, int delta);
/* round_robin_schedule, src/ordering.py:32-75.  pairs: 2*P ints, starts: T+1 ints.
 * Returns P (number of pairs); *n_iter receives T. Arrays must hold ell*ell entries. */
int orc_schedule(int ell, int* pairs, int* starts, int* n_iter);

int orc_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
