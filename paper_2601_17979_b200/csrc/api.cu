// api.cu -- the C-ABI (include/bsvd_b200.h): argument checks, route
// selection (src/svd.py:375-381 dispatch), kernel planning and launch.
#include <cstdlib>
#include <cuda_runtime.h>
#include <string.h>

#include <emmintrin.h>  // SSE2 non-temporal stores (x86-64 baseline)

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "launch.h"
#include <nvtx3/nvToolsExt.h>

using namespace bsvd;

namespace {
// NVTX range around every C-ABI entry point (tracing): the calls show up by name on an nsys /
// Nsight timeline next to the kernels they launch; free when no tool is attached (nvtx3 is header-only)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

constexpr size_t kSmemFallback = 232448;  // 227 KB opt-in limit of sm_100
constexpr int FV_WARPS_PER_SM = 8;  // kernel 52 while it fits one resident wave (C1: 1,184 0.29 vs 0.32 ms; 1,250 0.45 vs 0.41)

size_t smem_limit() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return kSmemFallback;
    }
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || v <= 0) {
        cudaGetLastError();
        return kSmemFallback;
    }
    return (size_t)v;
}

int esize_of(int dt) { return dt == BSVD_S ? 4 : dt == BSVD_D ? 8 : dt == BSVD_C ? 8 : 16; }
int rsize_of(int dt) { return (dt == BSVD_S || dt == BSVD_C) ? 4 : 8; }

struct Route {
    int trans, bm, bn, blocked, need_v, qr;
};

int make_route(int m, int n, const bsvd_opts* o, Route* r) {
    if (o->route != BSVD_DISPATCH && m < n) return BSVD_ERR_ARG;  // forced solvers need m >= n
    r->trans = (o->route == BSVD_DISPATCH && m < n) ? 1 : 0;
    r->bm = r->trans ? n : m;
    r->bn = r->trans ? m : n;
    // QR first (src/svd.py:364-371): forced, or dispatch with use_qr_preprocess and bm >= 3 bn (QR_RATIO)
    r->qr = (r->bn > 0 && (o->route == BSVD_FORCE_QR ||
                           (o->route == BSVD_DISPATCH && o->use_qr && (double)r->bm >= 3.0 * r->bn)))
                ? 1 : 0;
    if (o->route == BSVD_FORCE_UNBLOCKED) r->blocked = 0;
    else if (o->route == BSVD_FORCE_BLOCKED) r->blocked = 1;
    else r->blocked = r->bn > 32;  // SMALL_CUTOFF, src/svd.py:52
    r->need_v = (o->want_v || r->trans) ? 1 : 0;
    return BSVD_OK;
}

int sm_count() {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        v <= 0) {
        cudaGetLastError();
        return 148;  // B200
    }
    return v;
}

Plan make_plan(int dt, const Route& r, const bsvd_opts* o, bool contiguous = true, int batch = 0) {
    const size_t lim = smem_limit();
    const int es = esize_of(dt), rs = rsize_of(dt);
    const bool reg_ok = contiguous && !r.trans;  // register kernels: dense column-major input, no transpose
    if (o->kernel == 0 || o->kernel == KV_CREG32 || o->kernel == KV_CREG32_TMA) {  // complex FP64, n = 32: both routes
        Plan p = plan_creg32(dt, r.bm, r.bn, r.need_v, reg_ok, r.blocked, o->nb, o->kernel, lim);
        if (p.kernel) return p;
        if (o->kernel != 0) return p;
    }
    if (r.blocked && (o->kernel == 0 || o->kernel == KV_CREGB)) {  // complex FP64, n > 32
        Plan p = plan_cregb(dt, r.bm, r.bn, r.need_v, r.trans, o->nb);
        if (p.kernel) return p;
        if (o->kernel != 0) return p;
    }
    if (r.blocked) {
        if (o->kernel == 0 || o->kernel == KV_BLOCKED_REG) {
            Plan p = plan_blocked_reg(dt, r.bm, r.bn, o->nb, r.need_v, reg_ok, o->inner_sweeps, o->kernel);
            if (p.kernel) return p;
            if (o->kernel != 0) return p;
        }
        if (o->kernel == 0 || o->kernel == KV_BLOCKED_DMMA || o->kernel == KV_BLOCKED_DMMA_VG ||
            o->kernel == KV_BLOCKED_DMMA_512) {
            Plan p = plan_blocked_dmma(dt, r.bm, r.bn, o->nb, r.need_v, reg_ok, lim, o->kernel);
            if (p.kernel) return p;
            if (o->kernel != 0) return p;
        }
        return plan_blocked_general(es, rs, r.bm, r.bn, o->nb, r.need_v, lim);
    }
    if (o->kernel == 0 || o->kernel == KV_UNBLOCKED_REG16C) {
        // 16x16 FP32 from ~3,500 problems on: the quarter-warp kernel (C2 10k: 172 vs 207 us); below it the
        // half-warp kernel's shorter per-warp chain wins.  The two are bit-identical (same sums in the same
        // tree, same parameter and update arithmetic), so batch == standalone still holds bitwise.
        if (o->kernel != 0 || batch >= 3500) {
            Plan p = plan_unblocked_reg16c(dt, r.bm, r.bn, r.need_v, reg_ok, o->kernel);
            if (p.kernel || o->kernel != 0) return p;
        }
    }
    if (o->kernel == 0 || o->kernel == KV_UNBLOCKED_REG16B) {
        Plan p = plan_unblocked_reg16b(dt, r.bm, r.bn, r.need_v, reg_ok, o->kernel);
        if (p.kernel) return p;
        if (o->kernel != 0) return p;
    }
    if (o->kernel == 0 || o->kernel == KV_UNBLOCKED_REG32B || o->kernel == KV_UNBLOCKED_REG32G ||
        o->kernel == KV_UNBLOCKED_REG32F) {
        // 32x32 FP64, the second-generation register kernel.  With V: scaled rotations (one FMA per
        // updated element; sigma = ||w|| / ||v||) at every batch size -- one kernel, so batch ==
        // standalone holds bitwise (profiles/r2_c1_kernel_experiments.md: 10k 1.70 vs 1.85 ms, 1,184
        // problems 0.333 vs 0.34 ms for the warp-specialised round-1 kernel).  Values only: the unscaled
        // form (the scaled one needs V's column norms to cancel its scale roundings).
        // Batches of at most FV_WARPS_PER_SM problems per SM: one problem per warp, V carried in lockstep
        // by the other half-warp (bit-identical to 42, no replay phase) -- the GPU is not full, so the
        // shorter per-problem chain wins over 42's two problems per warp.
        const bool fv = r.need_v && batch > 0 && batch <= FV_WARPS_PER_SM * sm_count() && o->reserved[0] == 0;
        const int want = o->kernel ? o->kernel
                                   : (r.need_v ? (fv ? KV_UNBLOCKED_REG32F : KV_UNBLOCKED_REG32G) : KV_UNBLOCKED_REG32B);
        Plan p = plan_unblocked_reg32b(dt, r.bm, r.bn, r.need_v, reg_ok, want, o->max_sweeps);
        // above one resident wave of 52's warps: the last problems run as 52 in the same launch
        if (p.kernel == KV_UNBLOCKED_REG32G && o->kernel == 0 && batch > 0)
            p.aux = split_tail(batch, sm_count(), o->reserved[0]);
        if (p.kernel) return p;
        if (o->kernel != 0) return p;  // forced variant unavailable => kernel 0 => unsupported
    }
    if (o->kernel != 0 && o->kernel != KV_UNBLOCKED_GENERAL) return Plan{};
    return plan_unblocked_general(es, rs, r.bm, r.bn, r.need_v, lim);
}

int check_opts(const bsvd_opts* o) {
    if (!o) return BSVD_ERR_ARG;
    if (!(o->k > 0) || o->max_sweeps < 1 || o->nb < 1 || o->inner_sweeps < 0 || o->row_block < 1)
        return BSVD_ERR_ARG;
    if (o->route < 0 || o->route > 3) return BSVD_ERR_ARG;
    return BSVD_OK;
}

__global__ void k_info_empty(bsvd_info* info, int batch, int trans) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < batch) {
        bsvd_info inf;
        memset(&inf, 0, sizeof(inf));
        inf.converged = 1;
        inf.path = trans ? 0x100 : 0;
        info[i] = inf;
    }
}

template <class T>
int run(const Route& r, const Plan& p, int m, int n, int batch, const void* A, int64_t lda, int64_t sA, void* U,
        int64_t ldu, int64_t sU, void* S, int64_t sS, void* V, int64_t ldv, int64_t sV, const bsvd_opts* o,
        bsvd_info* info, void* work, cudaStream_t st) {
    SolveArgs<T> a{};
    a.A = static_cast<const T*>(A);
    a.lda = lda;
    a.strideA = sA;
    a.m = m;
    a.n = n;
    a.trans = r.trans;
    a.bm = r.bm;
    a.bn = r.bn;
    a.U = static_cast<T*>(U);
    a.ldu = ldu;
    a.strideU = sU;
    a.S = static_cast<typename tr<T>::R*>(S);
    a.strideS = sS;
    a.V = static_cast<T*>(V);
    a.ldv = ldv;
    a.strideV = sV;
    a.want_v = o->want_v ? 1 : 0;
    a.need_v = r.need_v;
    a.tol = o->k * tr<T>::u;
    a.max_sweeps = o->max_sweeps;
    a.nb = o->nb;
    a.inner_budget = o->inner_sweeps >= 1 ? o->inner_sweeps : 100;  // INNER_BUDGET, src/svd.py:55
    a.batch = batch;
    a.work = p.work_elems ? static_cast<T*>(work) : nullptr;
    a.work_stride = (int64_t)p.work_elems;
    a.info = info;
    switch (p.kernel) {
        case KV_UNBLOCKED_GENERAL: return launch_unblocked_general<T>(a, p, st);
        case KV_BLOCKED_GENERAL: return launch_blocked_general<T>(a, p, st);
        case KV_UNBLOCKED_REG16B:
            if constexpr (sizeof(T) == 4 && !tr<T>::cplx) return launch_unblocked_reg16b(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
        case KV_UNBLOCKED_REG16C:
            if constexpr (sizeof(T) == 4 && !tr<T>::cplx) return launch_unblocked_reg16c(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
        case KV_BLOCKED_REG:
            if constexpr (sizeof(T) == 8 && !tr<T>::cplx) return launch_blocked_reg(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
        case KV_CREG32:
        case KV_CREG32_TMA:
            if constexpr (sizeof(T) == 16 && tr<T>::cplx) return launch_creg32(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
        case KV_CREGB:
            if constexpr (sizeof(T) == 16 && tr<T>::cplx) return launch_cregb(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
        case KV_BLOCKED_DMMA:
        case KV_BLOCKED_DMMA_VG:
        case KV_BLOCKED_DMMA_512:
            if constexpr (sizeof(T) == 8 && !tr<T>::cplx) return launch_blocked_dmma(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
        case KV_UNBLOCKED_REG32B:
        case KV_UNBLOCKED_REG32G:
        case KV_UNBLOCKED_REG32F:
            if constexpr (sizeof(T) == 8 && !tr<T>::cplx) return launch_unblocked_reg32b(a, p, st);
            return BSVD_ERR_UNSUPPORTED;
    }
    return BSVD_ERR_UNSUPPORTED;
}

}  // namespace

extern "C" {

size_t bsvd_heevj_workspace_bytes(int dtype, int n, int batch) {
    if (dtype < 0 || dtype > 3 || n < 0 || batch < 0) return 0;
    return heevj_workspace(dtype, n, batch, smem_limit());
}

int bsvd_heevj_batched(int dtype, int n, int batch, const void* G, int64_t ldg, int64_t strideG, void* D,
                       int64_t strideD, void* M, int64_t ldm, int64_t strideM, int m_init, double k, int max_sweeps,
                       bsvd_info* info, void* work, size_t work_bytes, void* stream) {
    const NvtxRange nvtx_range("bsvd_heevj_batched");
    if (dtype < 0 || dtype > 3 || n < 0 || batch < 0 || !(k > 0) || max_sweeps < 1) return BSVD_ERR_ARG;
    if (batch == 0 || n == 0) return BSVD_OK;
    if (!G || !D || !M || ldg < n || ldm < n) return BSVD_ERR_ARG;
    if (batch > 1 && (strideG < ldg * (int64_t)n || strideD < n || strideM < ldm * (int64_t)n)) return BSVD_ERR_ARG;
    return launch_heevj(dtype, n, batch, G, ldg, strideG, D, strideD, M, ldm, strideM, m_init, k, max_sweeps, info,
                        work, work_bytes, smem_limit(), static_cast<cudaStream_t>(stream));
}

int bsvd_eig_sweeps_batched(int dtype, int n, int batch, void* G, int64_t ldg, int64_t strideG, void* D,
                            int64_t strideD, void* M, int64_t ldm, int64_t strideM, double tol, int max_sweeps,
                            int delta, bsvd_info* info, void* work, size_t work_bytes, void* stream) {
    const NvtxRange nvtx_range("bsvd_eig_sweeps_batched");
    if (dtype < 0 || dtype > 3 || n < 0 || batch < 0 || !(tol >= 0) || max_sweeps < 1) return BSVD_ERR_ARG;
    if (batch == 0 || n == 0) return BSVD_OK;
    if (!G || !D || !M || ldg < n || ldm < n) return BSVD_ERR_ARG;
    // caller's M (delta: the P - I accumulator), caller's d, g written back, absolute tolerance
    const int mode = 1 | (delta ? 2 : 0) | 4 | 8 | 16;
    return launch_heevj(dtype, n, batch, G, ldg, strideG, D, strideD, M, ldm, strideM, mode, tol, max_sweeps, info,
                        work, work_bytes, smem_limit(), static_cast<cudaStream_t>(stream));
}

int bsvd_verify_batched(int dtype, int m, int n, int batch, const void* A, int64_t lda, int64_t strideA,
                        const void* U, int64_t ldu, int64_t strideU, const void* S, int64_t strideS, const void* V,
                        int64_t ldv, int64_t strideV, const double* Sref, int64_t strideSref, double* out,
                        void* stream) {
    const NvtxRange nvtx_range("bsvd_verify_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0) return BSVD_ERR_ARG;
    if (batch == 0) return BSVD_OK;
    if (!A || !U || !S || !out || lda < m || ldu < m || (V && ldv < n)) return BSVD_ERR_ARG;
    return launch_verify(dtype, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, V, ldv, strideV, Sref,
                         strideSref, out, static_cast<cudaStream_t>(stream));
}

int bsvd_finalize_batched(int dtype, int m, int n, int batch, const void* W, int64_t ldw, int64_t strideW,
                          int vrows, const void* V, int64_t ldv, int64_t strideV, void* U, int64_t ldu,
                          int64_t strideU, void* S, int64_t strideS, void* Vout, int64_t ldvo, int64_t strideVout,
                          void* stream) {
    const NvtxRange nvtx_range("bsvd_finalize_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0 || vrows < 0) return BSVD_ERR_ARG;
    if (n > m) return BSVD_ERR_ARG;  // finalize expects m >= n (src/svd.py:246-247)
    if (batch == 0 || n == 0) return BSVD_OK;
    if (!W || !U || !S || ldw < m || ldu < m) return BSVD_ERR_ARG;
    if (V && (!Vout || ldv < vrows || ldvo < vrows)) return BSVD_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t lim = smem_limit();
    switch (dtype) {
        case BSVD_S: return launch_finalize_ext<float>(m, n, vrows, batch, W, ldw, strideW, V, ldv, strideV, U, ldu, strideU, S, strideS, Vout, ldvo, strideVout, lim, st);
        case BSVD_D: return launch_finalize_ext<double>(m, n, vrows, batch, W, ldw, strideW, V, ldv, strideV, U, ldu, strideU, S, strideS, Vout, ldvo, strideVout, lim, st);
        case BSVD_C: return launch_finalize_ext<cx<float>>(m, n, vrows, batch, W, ldw, strideW, V, ldv, strideV, U, ldu, strideU, S, strideS, Vout, ldvo, strideVout, lim, st);
        case BSVD_Z: return launch_finalize_ext<cx<double>>(m, n, vrows, batch, W, ldw, strideW, V, ldv, strideV, U, ldu, strideU, S, strideS, Vout, ldvo, strideVout, lim, st);
    }
    return BSVD_ERR_ARG;
}

size_t bsvd_householder_qr_workspace_bytes(int dtype, int m, int n, int batch) {
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0) return 0;
    return householder_qr_work_bytes(esize_of(dtype), m, n, batch);
}

int bsvd_householder_qr_batched(int dtype, int m, int n, int batch, const void* A, int64_t lda, int64_t strideA,
                                void* Q, int64_t ldq, int64_t strideQ, void* R, int64_t ldr, int64_t strideR,
                                void* work, size_t work_bytes, void* stream) {
    const NvtxRange nvtx_range("bsvd_householder_qr_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0) return BSVD_ERR_ARG;
    if (m < n) return BSVD_ERR_ARG;  // householder_qr needs m >= n (src/core.py:125-126)
    if (batch == 0 || n == 0) return BSVD_OK;
    if (!A || !Q || !R || lda < m || ldq < m || ldr < n) return BSVD_ERR_ARG;
    if (!work || work_bytes < householder_qr_work_bytes(esize_of(dtype), m, n, batch)) return BSVD_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t lim = smem_limit();
    switch (dtype) {
        case BSVD_S: return launch_householder_qr<float>(m, n, batch, A, lda, strideA, Q, ldq, strideQ, R, ldr, strideR, work, lim, st);
        case BSVD_D: return launch_householder_qr<double>(m, n, batch, A, lda, strideA, Q, ldq, strideQ, R, ldr, strideR, work, lim, st);
        case BSVD_C: return launch_householder_qr<cx<float>>(m, n, batch, A, lda, strideA, Q, ldq, strideQ, R, ldr, strideR, work, lim, st);
        case BSVD_Z: return launch_householder_qr<cx<double>>(m, n, batch, A, lda, strideA, Q, ldq, strideQ, R, ldr, strideR, work, lim, st);
    }
    return BSVD_ERR_ARG;
}

int bsvd_pack_host(const void* const* src, int count, size_t bytes, void* dst, int nthreads) {
    if (count < 0 || (count > 0 && (!src || !dst))) return BSVD_ERR_ARG;
    unsigned char* d = static_cast<unsigned char*>(dst);
    auto work = [&](int lo, int hi) {
        for (int i = lo; i < hi; ++i) memcpy(d + (size_t)i * bytes, src[i], bytes);
    };
    const int nt = nthreads < 1 ? 1 : (nthreads > 32 ? 32 : nthreads);
    if (nt == 1 || count < 2 * nt) {
        work(0, count);
        return BSVD_OK;
    }
    std::vector<std::thread> pool;
    const int step = (count + nt - 1) / nt;
    for (int lo = 0; lo < count; lo += step) pool.emplace_back(work, lo, lo + step < count ? lo + step : count);
    for (auto& t : pool) t.join();
    return BSVD_OK;
}

int bsvd_abi_version(void) { return BSVD_ABI_VERSION; }

void bsvd_default_opts(bsvd_opts* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->k = 30.0;
    o->max_sweeps = 30;
    o->nb = 16;
    o->inner_sweeps = 1;
    o->masking = 0;
    o->want_v = 1;
    o->route = BSVD_DISPATCH;
    o->fused_updates = 1;
    o->row_block = 64;
    o->kernel = 0;
}

const char* bsvd_strerror(int code) {
    switch (code) {
        case BSVD_OK: return "ok";
        case BSVD_ERR_ARG: return "invalid argument";
        case BSVD_ERR_WORKSPACE: return "workspace too small";
        case BSVD_ERR_CUDA: return "CUDA launch error";
        case BSVD_ERR_UNSUPPORTED: return "unsupported kernel variant for this problem";
    }
    return "unknown error";
}

extern "C++" {
namespace {
bool promote_f32(int dtype, const Route& r, const bsvd_opts* o);  // (defined below)
}
}

int bsvd_select_kernel_batched(int dtype, int m, int n, int batch, const bsvd_opts* opts) {
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0 || check_opts(opts)) return BSVD_ERR_ARG;
    Route r;
    if (make_route(m, n, opts, &r)) return BSVD_ERR_ARG;
    if (r.bn == 0 || r.bm == 0) return 0;
    if (r.qr) {  // the kernel that solves R
        Route rr = r;
        rr.trans = 0;
        rr.bm = r.bn;
        rr.blocked = r.bn > 32;
        rr.need_v = 1;
        rr.qr = 0;
        return make_plan(dtype, rr, opts, true, batch).kernel;
    }
    if (promote_f32(dtype, r, opts)) {  // single precision on a double-precision register kernel
        Route rd = r;
        return make_plan(dtype == BSVD_C ? BSVD_Z : BSVD_D, rd, opts, true, batch).kernel;
    }
    return make_plan(dtype, r, opts, true, batch).kernel;
}

int bsvd_select_kernel(int dtype, int m, int n, const bsvd_opts* opts) {
    return bsvd_select_kernel_batched(dtype, m, n, 0, opts);
}

namespace {
bool host_direct_enabled() {
    static const int v = [] {
        const char* e = getenv("BSVD_HOST_DIRECT");
        return (e && e[0] == '1') ? 1 : 0;
    }();
    return v != 0;
}
// Staging layout of one pipeline slot (device): A | U | V | S | info | solver workspace.
struct HostSlot {
    size_t a, u, v, s, info, ws, total;
};
// The options a chunk of a multi-chunk host pipeline solves with: chunks on different streams run
// concurrently, so throughput beats single-problem latency -- the 32x32 FP64 problems use kernel 42 alone
// (two problems per warp) rather than 52 (one problem per warp: the fastest single chunk, but half the
// problems per resident warp).  C1-10k end to end, chunks of 1,250 on 4 streams, medians of 3 on one box:
// 4.04 ms with 52 / 42 + 52 tail -> 3.86 ms (tools/ramp_probe.py).
// ... when the chunks in flight (one per stream) hold more than two waves of kernel 52: below that, 52's
// shorter chain wins (C1 slices: 1,250 problems in chunks of 313 1.57 M/s with 52 vs 1.38-1.50 with 42;
// 2,500 in chunks of 342 1.96 vs 1.76-1.91)
bool pipeline_throughput(int batch, int chunk, int nstreams) {
    const long in_flight = (long)nstreams * (chunk < batch ? chunk : batch);
    return in_flight > 2L * FV_WARPS_PER_SM * sm_count();
}
bsvd_opts pipeline_opts(const bsvd_opts& o) {
    bsvd_opts p = o;
    if (p.reserved[0] == 0) p.reserved[0] = -1;
    return p;
}

HostSlot host_slot(int dtype, int m, int n, int chunk, const bsvd_opts* o) {
    const size_t es = (size_t)esize_of(dtype), rs = (size_t)rsize_of(dtype);
    const size_t k = (size_t)(m < n ? m : n);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    HostSlot h{};
    h.a = al((size_t)chunk * m * n * es);
    h.u = al((size_t)chunk * m * k * es);
    h.v = o->want_v ? al((size_t)chunk * n * k * es) : 0;
    h.s = al((size_t)chunk * k * rs);
    h.info = al((size_t)chunk * sizeof(bsvd_info));
    const bsvd_opts po = pipeline_opts(*o);
    h.ws = al(std::max(bsvd_workspace_bytes(dtype, m, n, chunk, o), bsvd_workspace_bytes(dtype, m, n, chunk, &po)));
    h.total = h.a + h.u + h.v + h.s + h.info + h.ws;
    return h;
}
}  // namespace

size_t bsvd_host_workspace_bytes(int dtype, int m, int n, int chunk, int nstreams, const bsvd_opts* opts) {
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || chunk < 1 || nstreams < 1 || check_opts(opts)) return 0;
    return host_slot(dtype, m, n, chunk, opts).total * (size_t)nstreams;
}

namespace {
// Packs the chunks of a list of host matrices into the pinned batch layout on `nthreads` host threads
// (thread t packs chunks t, t + nthreads, ...), publishing each chunk as done so that the pipeline can
// enqueue its H2D while later chunks are still being packed.
// A problem's bytes into the pinned staging with non-temporal stores: the staging is only read again by the
// copy engine, so write-allocating it in the host caches would add a read of every destination line (an
// extra ~80 MB of host-memory traffic per C1-10k call, competing with the H2D / D2H DMA).
inline void stream_copy(unsigned char* dst, const void* src, size_t bytes) {
    if (((uintptr_t)dst & 15) || (bytes & 15)) {
        memcpy(dst, src, bytes);
        return;
    }
    const unsigned char* s8 = static_cast<const unsigned char*>(src);
    for (size_t o = 0; o < bytes; o += 64) {
        if (o + 64 <= bytes) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s8 + o));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s8 + o + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s8 + o + 32));
            const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s8 + o + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + o + 48), d);
        } else {
            for (size_t q = o; q < bytes; q += 16)
                _mm_stream_si128(reinterpret_cast<__m128i*>(dst + q),
                                 _mm_loadu_si128(reinterpret_cast<const __m128i*>(s8 + q)));
        }
    }
}

// Chunk boundaries of the host pipeline: `chunk`-problem chunks, the last one ragged.
struct ChunkPlan {
    int batch, chunk;
    int count() const { return (batch + chunk - 1) / chunk; }
    int begin(int c) const { return c * chunk; }
    int end(int c) const { return (c + 1) * chunk < batch ? (c + 1) * chunk : batch; }
};

struct ChunkPacker {
    std::vector<std::thread> pool;
    std::atomic<int>* done = nullptr;
    ChunkPacker(const void* const* src, unsigned char* dst, size_t bytes, ChunkPlan plan, int nthreads) {
        const int nchunks = plan.count();
        done = new std::atomic<int>[nchunks];
        for (int c = 0; c < nchunks; ++c) done[c].store(0, std::memory_order_relaxed);
        const int nt = nthreads < 1 ? 1 : (nthreads > nchunks ? nchunks : nthreads);
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([=]() {
                for (int c = t; c < nchunks; c += nt) {
                    const int b1 = plan.end(c);
                    for (int i = plan.begin(c); i < b1; ++i) stream_copy(dst + (size_t)i * bytes, src[i], bytes);
                    _mm_sfence();  // the non-temporal stores are visible before the chunk is published
                    done[c].store(1, std::memory_order_release);
                }
            });
    }
    void wait(int c) const {
        while (!done[c].load(std::memory_order_acquire)) std::this_thread::yield();
    }
    ~ChunkPacker() {
        for (auto& t : pool) t.join();
        delete[] done;
    }
};

int gesvj_host_impl(int dtype, int m, int n, int batch, const void* A, const void* const* A_ptrs, int pack_threads,
                    void* U, void* S, void* V, const bsvd_opts* opts, bsvd_info* info, int chunk, void* work,
                    size_t work_bytes, void* const* streams, int nstreams);
}  // namespace

int bsvd_gesvj_batched_host(int dtype, int m, int n, int batch, const void* A, void* U, void* S, void* V,
                            const bsvd_opts* opts, bsvd_info* info, int chunk, void* work, size_t work_bytes,
                            void* const* streams, int nstreams) {
    const NvtxRange nvtx_range("bsvd_gesvj_batched_host");
    return gesvj_host_impl(dtype, m, n, batch, A, nullptr, 0, U, S, V, opts, info, chunk, work, work_bytes, streams,
                           nstreams);
}

int bsvd_gesvj_batched_host_gather(int dtype, int m, int n, int batch, const void* const* A_ptrs, void* A_stage,
                                   int pack_threads, void* U, void* S, void* V, const bsvd_opts* opts,
                                   bsvd_info* info, int chunk, void* work, size_t work_bytes, void* const* streams,
                                   int nstreams) {
    const NvtxRange nvtx_range("bsvd_gesvj_batched_host_gather");
    if (batch > 0 && !A_ptrs) return BSVD_ERR_ARG;
    return gesvj_host_impl(dtype, m, n, batch, A_stage, A_ptrs, pack_threads, U, S, V, opts, info, chunk, work,
                           work_bytes, streams, nstreams);
}

namespace {
int gesvj_host_impl(int dtype, int m, int n, int batch, const void* A, const void* const* A_ptrs, int pack_threads,
                    void* U, void* S, void* V, const bsvd_opts* opts, bsvd_info* info, int chunk, void* work,
                    size_t work_bytes, void* const* streams, int nstreams) {
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0 || chunk < 1 || nstreams < 1 || !streams)
        return BSVD_ERR_ARG;
    int rc = check_opts(opts);
    if (rc) return rc;
    if (batch == 0) return BSVD_OK;
    const int k = m < n ? m : n;
    if (k > 0 && (!A || !U || !S || (opts->want_v && !V))) return BSVD_ERR_ARG;
    const HostSlot hs = host_slot(dtype, m, n, chunk, opts);
    if (hs.total * (size_t)nstreams > work_bytes || !work) return BSVD_ERR_WORKSPACE;
    const size_t es = (size_t)esize_of(dtype), rs = (size_t)rsize_of(dtype);
    cudaStream_t s0 = static_cast<cudaStream_t>(streams[0]);
    // Direct mode (opt-in, BSVD_HOST_DIRECT=1): when every output buffer is page-locked host memory mapped
    // into the device address space, the kernels write U, S, V and info straight into it over PCIe
    // instead of staging them for per-chunk D2H copies.  Measured on B200 (bench.py e2e): C2 +6 %
    // (15.1 vs 14.2 M/s), but C1-10k -15 % (2.04 vs 2.39 M/s) and C4 -20 %: the kernels' column-wise
    // 128-256 B stores over PCIe stall them and move fewer bytes per second than the copy engines.
    unsigned char *Uh = static_cast<unsigned char*>(U), *Sh = static_cast<unsigned char*>(S),
                  *Vh = static_cast<unsigned char*>(V);
    bsvd_info* Ih = info;
    bool direct = host_direct_enabled();
    if (direct) {
        auto mapped = [](void* p, unsigned char** dev) {
            if (!p) return true;
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            if (at.type != cudaMemoryTypeHost || !at.devicePointer) return false;
            *dev = static_cast<unsigned char*>(at.devicePointer);
            return true;
        };
        unsigned char* ih = reinterpret_cast<unsigned char*>(info);
        direct = mapped(U, &Uh) && mapped(S, &Sh) && (!opts->want_v || mapped(V, &Vh)) && mapped(info, &ih);
        Ih = reinterpret_cast<bsvd_info*>(ih);
        if (!direct) Uh = static_cast<unsigned char*>(U), Sh = static_cast<unsigned char*>(S),
                     Vh = static_cast<unsigned char*>(V), Ih = info;
    }
    // fork: every stream starts after the work already queued on streams[0]
    cudaEvent_t fork = nullptr;
    cudaEvent_t* joins = new cudaEvent_t[nstreams]();
    if (nstreams > 1) {
        if (cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) { delete[] joins; return BSVD_ERR_CUDA; }
        cudaEventRecord(fork, s0);
        for (int i = 1; i < nstreams; ++i) cudaStreamWaitEvent(static_cast<cudaStream_t>(streams[i]), fork, 0);
    }
    rc = BSVD_OK;
    const ChunkPlan plan{batch, chunk};
    const bsvd_opts po = pipeline_throughput(batch, chunk, nstreams) ? pipeline_opts(*opts) : *opts;
    const int nchunks = plan.count();
    ChunkPacker* packer = nullptr;  // gather mode: pack chunks on host threads ahead of their H2D
    if (A_ptrs && k > 0)
        packer = new ChunkPacker(A_ptrs, static_cast<unsigned char*>(const_cast<void*>(A)), (size_t)m * n * es, plan,
                                 pack_threads);
    for (int c = 0; c < nchunks && rc == BSVD_OK; ++c) {
        if (packer) packer->wait(c);
        const int slot = c % nstreams;
        cudaStream_t st = static_cast<cudaStream_t>(streams[slot]);
        const int b0 = plan.begin(c), cb = plan.end(c) - b0;
        unsigned char* base = static_cast<unsigned char*>(work) + hs.total * (size_t)slot;
        void* Ad = base;
        void* Ud = base + hs.a;
        void* Vd = opts->want_v ? base + hs.a + hs.u : nullptr;
        void* Sd = base + hs.a + hs.u + hs.v;
        bsvd_info* Id = reinterpret_cast<bsvd_info*>(base + hs.a + hs.u + hs.v + hs.s);
        void* Wd = base + hs.a + hs.u + hs.v + hs.s + hs.info;
        const size_t abytes = (size_t)cb * m * n * es;
        if (abytes && cudaMemcpyAsync(Ad, static_cast<const unsigned char*>(A) + (size_t)b0 * m * n * es, abytes,
                                      cudaMemcpyHostToDevice, st) != cudaSuccess) { rc = BSVD_ERR_CUDA; break; }
        if (direct) {  // outputs land in host memory from the kernels; no copies back
            rc = bsvd_gesvj_batched(dtype, m, n, cb, Ad, m > 0 ? m : 1, (int64_t)m * n, Uh + (size_t)b0 * m * k * es,
                                    m > 0 ? m : 1, (int64_t)m * k, Sh + (size_t)b0 * k * rs, k,
                                    opts->want_v ? Vh + (size_t)b0 * n * k * es : nullptr, n > 0 ? n : 1,
                                    (int64_t)n * k, &po, Ih ? Ih + b0 : Id, Wd, hs.ws, st);
            if (rc) break;
            continue;
        }
        rc = bsvd_gesvj_batched(dtype, m, n, cb, Ad, m > 0 ? m : 1, (int64_t)m * n, Ud, m > 0 ? m : 1,
                                (int64_t)m * k, Sd, k, Vd, n > 0 ? n : 1, (int64_t)n * k, &po, Id, Wd, hs.ws, st);
        if (rc) break;
        const size_t ub = (size_t)cb * m * k * es, vb = (size_t)cb * n * k * es, sb = (size_t)cb * k * rs;
        bool ok = true;
        if (ub) ok &= cudaMemcpyAsync(static_cast<unsigned char*>(U) + (size_t)b0 * m * k * es, Ud, ub,
                                      cudaMemcpyDeviceToHost, st) == cudaSuccess;
        if (sb) ok &= cudaMemcpyAsync(static_cast<unsigned char*>(S) + (size_t)b0 * k * rs, Sd, sb,
                                      cudaMemcpyDeviceToHost, st) == cudaSuccess;
        if (opts->want_v && vb) ok &= cudaMemcpyAsync(static_cast<unsigned char*>(V) + (size_t)b0 * n * k * es, Vd,
                                                      vb, cudaMemcpyDeviceToHost, st) == cudaSuccess;
        if (info) ok &= cudaMemcpyAsync(info + b0, Id, (size_t)cb * sizeof(bsvd_info), cudaMemcpyDeviceToHost,
                                        st) == cudaSuccess;
        if (!ok) rc = BSVD_ERR_CUDA;
    }
    // join: streams[0] waits for the other streams' last chunk
    for (int i = 1; i < nstreams; ++i) {
        if (cudaEventCreateWithFlags(&joins[i], cudaEventDisableTiming) != cudaSuccess) { rc = BSVD_ERR_CUDA; continue; }
        cudaEventRecord(joins[i], static_cast<cudaStream_t>(streams[i]));
        cudaStreamWaitEvent(s0, joins[i], 0);
    }
    for (int i = 1; i < nstreams; ++i)
        if (joins[i]) cudaEventDestroy(joins[i]);
    if (fork) cudaEventDestroy(fork);
    delete[] joins;
    delete packer;  // joins the packing threads (all chunks are packed once the loop has run)
    return rc;
}
}  // namespace

extern "C++" {
namespace {
// QR route workspace: reflectors (bm x bn) | R (bn x bn) | phases (bn) | U_R (bn x bn) | inner solve
struct QrWs {
    size_t refl, r, ph, ur, inner_off, total;
    bsvd_opts io;
};
QrWs qr_ws(int dtype, const Route& r, int batch, const bsvd_opts* o) {
    QrWs q{};
    const size_t es = (size_t)esize_of(dtype), B = (size_t)batch;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    q.io = *o;
    q.io.route = r.bn <= 32 ? BSVD_FORCE_UNBLOCKED : BSVD_FORCE_BLOCKED;
    q.io.use_qr = 0;
    q.io.want_v = r.trans ? 1 : o->want_v;
    q.refl = 0;
    q.r = al(B * r.bm * r.bn * es);
    q.ph = q.r + al(B * r.bn * r.bn * es);
    q.ur = q.ph + al(B * r.bn * es);
    q.inner_off = q.ur + al(B * r.bn * r.bn * es);
    q.total = q.inner_off + bsvd_workspace_bytes(dtype, r.bn, r.bn, batch, &q.io);
    return q;
}
}  // namespace
}  // extern "C++"

extern "C++" {
namespace {
// Single-precision problems whose shape a double-precision register kernel takes are solved in double
// precision -- inputs widened, factors rounded back -- with the single-precision tolerance k u_32 (opts.k
// scaled by u_32 / u_64 = 2^29, exact): FP32 blocked shapes (n % 16 == 0, m <= 256) and 32 x 32 on the
// FP64 register kernels, complex64 with n = 32, m <= 256 on the complex128 one.  The general
// single-precision kernels are 1.5-9.5x slower on these shapes (tools/general_time.py,
// tools/promo_time.py); the double-precision solve is at least as accurate as the reference's.
bool promote_f32(int dtype, const Route& r, const bsvd_opts* o) {
    if (r.qr || r.trans || o->kernel != 0) return false;
    if (dtype == BSVD_S) {
        if (r.blocked) return plan_blocked_reg(BSVD_D, r.bm, r.bn, o->nb, r.need_v, true, o->inner_sweeps, 0).kernel != 0;
        return r.bm == 32 && r.bn == 32;
    }
    if (dtype == BSVD_C)
        return plan_creg32(BSVD_Z, r.bm, r.bn, r.need_v, true, r.blocked, o->nb, 0, smem_limit()).kernel != 0 ||
               (r.blocked && plan_cregb(BSVD_Z, r.bm, r.bn, r.need_v, r.trans, o->nb).kernel != 0);
    return false;
}
struct PromWs {
    size_t a, u, s, v, inner, total;
    bsvd_opts io;
};
PromWs prom_ws(int dtype, int m, int n, int batch, const bsvd_opts* o) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t B = (size_t)batch, k = (size_t)(m < n ? m : n);
    const size_t es = dtype == BSVD_C ? 16 : 8, rs = 8;  // the double-precision element sizes
    PromWs w{};
    w.io = *o;
    w.io.k = o->k * 0x1p+29;
    w.a = 0;
    w.u = al(B * m * n * es);
    w.s = w.u + al(B * m * k * es);
    w.v = w.s + al(B * k * rs);
    w.inner = w.v + (o->want_v ? al(B * n * k * es) : 0);
    w.total = w.inner + bsvd_workspace_bytes(dtype == BSVD_C ? BSVD_Z : BSVD_D, m, n, batch, &w.io);
    return w;
}
__global__ void k_widen(const float* A, int64_t lda, int64_t sA, int m, int n, int batch, double* out) {
    const int64_t total = (int64_t)batch * m * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / ((int64_t)m * n), rc = e % ((int64_t)m * n);
        const int r = (int)(rc % m), c = (int)(rc / m);
        out[e] = (double)A[b * sA + r + c * lda];
    }
}
__global__ void k_narrow(const double* in, int rows, int cols, int batch, float* out, int64_t ld, int64_t so) {
    const int64_t total = (int64_t)batch * rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / ((int64_t)rows * cols), rc = e % ((int64_t)rows * cols);
        const int r = (int)(rc % rows), c = (int)(rc / rows);
        out[b * so + r + c * ld] = (float)in[e];
    }
}
int grid_for(int64_t total) { return (int)std::min<int64_t>((total + 255) / 256, 148 * 16); }
}  // namespace
}  // extern "C++"

size_t bsvd_workspace_bytes(int dtype, int m, int n, int batch, const bsvd_opts* opts) {
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0 || check_opts(opts)) return 0;
    Route r;
    if (make_route(m, n, opts, &r)) return 0;
    if (r.bn == 0 || r.bm == 0) return 0;
    if (r.qr) return qr_ws(dtype, r, batch, opts).total;
    if (promote_f32(dtype, r, opts)) return prom_ws(dtype, m, n, batch, opts).total;
    // the call plans with contiguous = (lda == m): size for both plans, so a caller with a padded lda who
    // allocates this many bytes never gets BSVD_ERR_WORKSPACE
    const Plan pc = make_plan(dtype, r, opts, true, batch);
    const Plan pg = make_plan(dtype, r, opts, false, batch);
    const size_t elems = pc.work_elems > pg.work_elems ? pc.work_elems : pg.work_elems;
    return elems * (size_t)esize_of(dtype) * (size_t)batch;
}

extern "C++" {
namespace {
template <class T>
int run_qr(int dtype, const Route& r, int m, int n, int batch, const void* A, int64_t lda, int64_t sA, void* U,
           int64_t ldu, int64_t sU, void* S, int64_t sS, void* V, int64_t ldv, int64_t sV, const bsvd_opts* o,
           bsvd_info* info, void* work, size_t work_bytes, cudaStream_t st) {
    const QrWs q = qr_ws(dtype, r, batch, o);
    if (q.total > work_bytes || !work) return BSVD_ERR_WORKSPACE;
    if (!qr_reg_ok(sizeof(T), tr<T>::cplx, r.bm, r.bn) && qr_smem(sizeof(T), r.bm, r.bn) > smem_limit())
        return BSVD_ERR_UNSUPPORTED;
    unsigned char* w = static_cast<unsigned char*>(work);
    T* refl = reinterpret_cast<T*>(w + q.refl);
    T* R = reinterpret_cast<T*>(w + q.r);
    T* ph = reinterpret_cast<T*>(w + q.ph);
    T* UR = reinterpret_cast<T*>(w + q.ur);
    SolveArgs<T> a{};
    a.A = static_cast<const T*>(A);
    a.lda = lda;
    a.strideA = sA;
    a.m = m;
    a.n = n;
    a.trans = r.trans;
    a.bm = r.bm;
    a.bn = r.bn;
    a.batch = batch;
    a.info = info;
    int rc = launch_qr<T>(a, R, refl, ph, st);
    if (rc) return rc;
    const int bn = r.bn;
    // Jacobi SVD of R (bn x bn): U_R to the workspace; V_R is the caller's V (or, transposed, the caller's U)
    void* Vi = r.trans ? U : (o->want_v ? V : nullptr);
    const int64_t ldvi = r.trans ? ldu : ldv, svi = r.trans ? sU : sV;
    rc = bsvd_gesvj_batched(dtype, bn, bn, batch, R, bn, (int64_t)bn * bn, UR, bn, (int64_t)bn * bn, S, sS, Vi,
                            ldvi, svi, &q.io, info, w + q.inner_off, work_bytes - q.inner_off, st);
    if (rc) return rc;
    // left factor U = Q diag(p) U_R (src/svd.py:529-530); transposed: that is the caller's V
    if (!r.trans) rc = launch_applyq<T>(r.bm, bn, batch, refl, ph, UR, static_cast<T*>(U), ldu, sU, st);
    else if (o->want_v) rc = launch_applyq<T>(r.bm, bn, batch, refl, ph, UR, static_cast<T*>(V), ldv, sV, st);
    if (rc) return rc;
    if (info) rc = launch_qr_path(info, batch, 0x200 | (r.trans ? 0x100 : 0), st);
    return rc;
}
}  // namespace
}  // extern "C++"

int bsvd_gesvj_batched(int dtype, int m, int n, int batch, const void* A, int64_t lda, int64_t strideA, void* U,
                       int64_t ldu, int64_t strideU, void* S, int64_t strideS, void* V, int64_t ldv,
                       int64_t strideV, const bsvd_opts* opts, bsvd_info* info, void* work, size_t work_bytes,
                       void* stream) {
    const NvtxRange nvtx_range("bsvd_gesvj_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0) return BSVD_ERR_ARG;
    int rc = check_opts(opts);
    if (rc) return rc;
    Route r;
    if ((rc = make_route(m, n, opts, &r))) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (batch == 0) return BSVD_OK;
    const int k = m < n ? m : n;
    if (k == 0) {  // "empty" path (src/svd.py:351-362)
        if (info) {
            k_info_empty<<<(batch + 255) / 256, 256, 0, st>>>(info, batch, r.trans);
            if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
        }
        return BSVD_OK;
    }
    if (!A || !U || !S) return BSVD_ERR_ARG;
    if (lda < m || ldu < m) return BSVD_ERR_ARG;
    if (opts->want_v && (!V || ldv < n)) return BSVD_ERR_ARG;
    if (batch > 1 && (strideA < lda * (int64_t)n || strideU < ldu * (int64_t)k || strideS < k)) return BSVD_ERR_ARG;
    if (batch > 1 && opts->want_v && strideV < ldv * (int64_t)k) return BSVD_ERR_ARG;
    if (r.qr) {
        switch (dtype) {
            case BSVD_S:
                return run_qr<float>(dtype, r, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, V, ldv,
                                     strideV, opts, info, work, work_bytes, st);
            case BSVD_D:
                return run_qr<double>(dtype, r, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, V, ldv,
                                      strideV, opts, info, work, work_bytes, st);
            case BSVD_C:
                return run_qr<cx<float>>(dtype, r, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, V,
                                         ldv, strideV, opts, info, work, work_bytes, st);
            default:
                return run_qr<cx<double>>(dtype, r, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, V,
                                          ldv, strideV, opts, info, work, work_bytes, st);
        }
    }
    if (promote_f32(dtype, r, opts)) {  // single precision on a double-precision register kernel
        const PromWs w = prom_ws(dtype, m, n, batch, opts);
        if (w.total > work_bytes || !work) return BSVD_ERR_WORKSPACE;
        const int c = dtype == BSVD_C ? 2 : 1;  // complex: interleaved (re, im) = twice the rows of floats
        unsigned char* wb = static_cast<unsigned char*>(work);
        double* A64 = reinterpret_cast<double*>(wb + w.a);
        double* U64 = reinterpret_cast<double*>(wb + w.u);
        double* S64 = reinterpret_cast<double*>(wb + w.s);
        double* V64 = opts->want_v ? reinterpret_cast<double*>(wb + w.v) : nullptr;
        const int64_t tot_a = (int64_t)batch * c * m * n;
        k_widen<<<grid_for(tot_a), 256, 0, st>>>(static_cast<const float*>(A), c * lda, c * strideA, c * m, n, batch,
                                                 A64);
        if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
        rc = bsvd_gesvj_batched(dtype == BSVD_C ? BSVD_Z : BSVD_D, m, n, batch, A64, m, (int64_t)m * n, U64, m,
                                (int64_t)m * k, S64, k, V64, n, (int64_t)n * k, &w.io, info, wb + w.inner,
                                work_bytes - w.inner, stream);
        if (rc) return rc;
        k_narrow<<<grid_for((int64_t)batch * c * m * k), 256, 0, st>>>(U64, c * m, k, batch, static_cast<float*>(U),
                                                                        c * ldu, c * strideU);
        k_narrow<<<grid_for((int64_t)batch * k), 256, 0, st>>>(S64, k, 1, batch, static_cast<float*>(S), k, strideS);
        if (V64)
            k_narrow<<<grid_for((int64_t)batch * c * n * k), 256, 0, st>>>(V64, c * n, k, batch,
                                                                            static_cast<float*>(V), c * ldv,
                                                                            c * strideV);
        return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
    }
    const Plan p = make_plan(dtype, r, opts, lda == m, batch);
    if (!p.kernel) return BSVD_ERR_UNSUPPORTED;
    const size_t need = p.work_elems * (size_t)esize_of(dtype) * (size_t)batch;
    if (need > work_bytes || (need && !work)) return BSVD_ERR_WORKSPACE;
    void* Vp = opts->want_v ? V : nullptr;
    switch (dtype) {
        case BSVD_S:
            return run<float>(r, p, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, Vp, ldv, strideV, opts,
                              info, work, st);
        case BSVD_D:
            return run<double>(r, p, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, Vp, ldv, strideV,
                               opts, info, work, st);
        case BSVD_C:
            return run<cx<float>>(r, p, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, Vp, ldv, strideV,
                                  opts, info, work, st);
        case BSVD_Z:
            return run<cx<double>>(r, p, m, n, batch, A, lda, strideA, U, ldu, strideU, S, strideS, Vp, ldv,
                                   strideV, opts, info, work, st);
    }
    return BSVD_ERR_ARG;
}

int bsvd_onesided_sweeps_batched(int dtype, int m, int n, int batch, void* a, int64_t lda, int64_t stride_a,
                                 int vrows, void* v, int64_t ldv, int64_t stride_v, double tol, int max_sweeps,
                                 int64_t* rotations, int32_t* sweeps, void* stream) {
    const NvtxRange nvtx_range("bsvd_onesided_sweeps_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || n < 0 || batch < 0 || vrows < 0 || max_sweeps < 1) return BSVD_ERR_ARG;
    if (batch == 0) return BSVD_OK;
    if (!a || lda < m || (vrows > 0 && (!v || ldv < vrows))) return BSVD_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    void* vp = vrows > 0 ? v : nullptr;
    switch (dtype) {
        case BSVD_S:
            return launch_onesided_raw<float>((float*)a, lda, stride_a, m, n, batch, (float*)vp, ldv, stride_v, vrows,
                                              tol, max_sweeps, rotations, sweeps, st);
        case BSVD_D:
            return launch_onesided_raw<double>((double*)a, lda, stride_a, m, n, batch, (double*)vp, ldv, stride_v,
                                               vrows, tol, max_sweeps, rotations, sweeps, st);
        case BSVD_C:
            return launch_onesided_raw<cx<float>>((cx<float>*)a, lda, stride_a, m, n, batch, (cx<float>*)vp, ldv,
                                                  stride_v, vrows, tol, max_sweeps, rotations, sweeps, st);
        case BSVD_Z:
            return launch_onesided_raw<cx<double>>((cx<double>*)a, lda, stride_a, m, n, batch, (cx<double>*)vp, ldv,
                                                   stride_v, vrows, tol, max_sweeps, rotations, sweeps, st);
    }
    return BSVD_ERR_ARG;
}

int bsvd_gram_batched(int dtype, int m, int wi, int wj, int batch, const void* a, int64_t lda, int64_t stride_a,
                      void* g, int64_t ldg, int64_t stride_g, void* stream) {
    const NvtxRange nvtx_range("bsvd_gram_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || wi < 1 || wj < 0 || batch < 0) return BSVD_ERR_ARG;
    if (batch == 0) return BSVD_OK;
    if (!a || !g || lda < m || ldg < wi + wj) return BSVD_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (dtype) {
        case BSVD_S: return launch_gram_raw<float>((const float*)a, lda, stride_a, m, wi, wj, batch, (float*)g, ldg, stride_g, st);
        case BSVD_D: return launch_gram_raw<double>((const double*)a, lda, stride_a, m, wi, wj, batch, (double*)g, ldg, stride_g, st);
        case BSVD_C: return launch_gram_raw<cx<float>>((const cx<float>*)a, lda, stride_a, m, wi, wj, batch, (cx<float>*)g, ldg, stride_g, st);
        case BSVD_Z: return launch_gram_raw<cx<double>>((const cx<double>*)a, lda, stride_a, m, wi, wj, batch, (cx<double>*)g, ldg, stride_g, st);
    }
    return BSVD_ERR_ARG;
}

int bsvd_fused_pair_update_batched(int dtype, int m, int w, int batch, void* b, int64_t ldb, int64_t stride_b,
                                   const void* j, int64_t ldj, int64_t stride_j, int delta, void* stream) {
    const NvtxRange nvtx_range("bsvd_fused_pair_update_batched");
    if (dtype < 0 || dtype > 3 || m < 0 || w < 1 || batch < 0) return BSVD_ERR_ARG;
    if (batch == 0 || m == 0) return BSVD_OK;
    if (!b || !j || ldb < m || ldj < w) return BSVD_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (dtype) {
        case BSVD_S: return launch_fused_raw<float>((float*)b, ldb, stride_b, m, w, batch, (const float*)j, ldj, stride_j, delta, st);
        case BSVD_D: return launch_fused_raw<double>((double*)b, ldb, stride_b, m, w, batch, (const double*)j, ldj, stride_j, delta, st);
        case BSVD_C: return launch_fused_raw<cx<float>>((cx<float>*)b, ldb, stride_b, m, w, batch, (const cx<float>*)j, ldj, stride_j, delta, st);
        case BSVD_Z: return launch_fused_raw<cx<double>>((cx<double>*)b, ldb, stride_b, m, w, batch, (const cx<double>*)j, ldj, stride_j, delta, st);
    }
    return BSVD_ERR_ARG;
}

}  // extern "C"
