// unblocked_reg.cu -- kernel (2), register-resident fast path for 32x32 FP64.
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule (src/ordering.py:32-75); the working copy
// lives in registers instead of memory:
//
//  * A warp owns TWO problems; half-warp h (16 lanes) owns problem h and every
//    lane holds two full rows (rows l and l+16, 2 x 32 doubles).  The 16
//    disjoint column pairs of a schedule iteration sit in fixed register slots
//    (2k, 2k+1); instead of indexing columns by the schedule, the columns MOVE
//    one position along the tournament ring (bot0 -> top1 -> ... -> top15 ->
//    bot15 -> ... -> bot1 -> bot0) after every iteration, so every register
//    index is a compile-time constant.  After the 31 iterations of a sweep the
//    columns are back in natural order.
//  * Dot products: each lane forms the 48 partials (g_ii, g_jj, g_ji for 16
//    pairs over its two rows) and transposes them through shared memory; lane
//    k of each half then sums pair k's 16 partials and evaluates the guard
//    (F4) and the rotation (F5) in float64 with call-free rcp/rsqrt refinement
//    (common.cuh), so no ABI call forces the resident rows to spill.
//  * Phase alternation instead of a V warp: during a sweep the warp holds W
//    and logs every rotation (c - 1, w s) to an L2-resident log; after the
//    sweep it parks W in the workspace, pulls V into the same registers,
//    replays the logged rotations (cp.async double-buffered, throughput-bound
//    FP64 with plenty of ILP), parks V and resumes W.  Warps in the latency-
//    bound W phase interleave with warps in the throughput-bound V phase.
//  * Per-problem convergence: a problem stops after its first quiet sweep
//    (src/svd.py:427-430); its half keeps stepping with identity rotations
//    while the partner problem runs (a quiet sweep never writes, F7).
//  * The data are pre-scaled by an exact power of two (max |a| in [0.5, 1)),
//    undone on output: rotations are scale-invariant and the scaling is
//    exact, so the rotation sequence is unchanged; it keeps the squared
//    column norms far from under/overflow.
//  * Raw W and V go to the workspace; finalize.cu forms sigma, normalises,
//    sorts and permutes (kernel 5).
#include "kernel_args.cuh"
#include "launch.h"
#include "rotation.cuh"

namespace bsvd {
namespace reg32 {

constexpr int N = 32;      // columns
constexpr int H = 16;      // column pairs per iteration
constexpr int NIT = 31;    // iterations per sweep
constexpr int RSTR = 34;   // doubles per row of the dot-product transpose buffer (bank padding)
constexpr int LOG_ELEMS = NIT * H * 2 + 32;  // doubles per problem: rotation log (31 x 16 Par) + masks

// ring position -> register slot (slot 2k = top[k], slot 2k+1 = bot[k])
__host__ __device__ constexpr int ring_slot(int q) {
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}

struct __align__(16) Par {
    double cm1, c;  // x <- x + (cm1 x + c y);  y <- y + (cm1 y - c x)
};

struct WarpSmem {
    double red[3 * H * RSTR];  // dot-product transpose
    Par pub[2][H];             // this iteration's rotations, [half][pair]
    Par stage[2][2][H];        // V replay: double-buffered log rows [buf][half][pair]
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// advance every column one ring position (compile-time register moves)
__device__ __forceinline__ void ring_rotate(double (&x)[N]) {
    const double t = x[ring_slot(NIT - 1)];
#pragma unroll
    for (int q = NIT - 1; q >= 1; --q) x[ring_slot(q)] = x[ring_slot(q - 1)];
    x[ring_slot(0)] = t;
}

// column index at ring position r after t rotations (ell = 32)
__device__ __forceinline__ int col_at(int r, int t) {
    int q = r - t;
    if (q < 0) q += NIT;
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}

// Reference form (F5): x + (cm1 x + c y), one full-scale rounding.
__device__ __forceinline__ void apply(double& x, double& y, double cm1, double c) {
    const double nx = x + fma(cm1, x, c * y);
    const double ny = y + fma(cm1, y, -(c * x));
    x = nx;
    y = ny;
}
// Two-FMA form: (x + c y) + cm1 x with the shrink term fused (no rounded c = 1
// + cm1 ever formed, so the small-angle bias F5 guards against cannot arise);
// two full-scale roundings instead of one.  Opt-in (KV_UNBLOCKED_REG32_F2).
__device__ __forceinline__ void apply2(double& x, double& y, double cm1, double c) {
    const double tx = fma(c, y, x);
    const double ty = fma(-c, x, y);
    x = fma(cm1, x, tx);
    y = fma(cm1, y, ty);
}
template <bool F2>
__device__ __forceinline__ void applyv(double& x, double& y, double cm1, double c) {
    if constexpr (F2) apply2(x, y, cm1, c); else apply(x, y, cm1, c);
}

__device__ __forceinline__ void rotation(double d, double g, double& s_out, double& cm1_out) {
    double t;
    rotation_tsc(d, g, t, s_out, cm1_out);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

template <int NW, int MAXREG, bool F2>
__global__ void __launch_bounds__(NW * 32) __maxnreg__(MAXREG) k_reg32(SolveArgs<double> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
    const int half = lane >> 4, hl = lane & 15;
    const int prob = (blockIdx.x * NW + warp) * 2 + half;
    const bool live = prob < a.batch;
    const int r0 = hl, r1 = hl + 16;
    const size_t pstride = (size_t)a.work_stride;
    double* wsW = a.work + (size_t)(live ? prob : 0) * pstride;  // W 32x32, V 32x32, then the log
    double* wsV = wsW + N * N;
    Par* logp = reinterpret_cast<Par*>(wsW + 2 * N * N);           // [31][16]
    uint32_t* logm = reinterpret_cast<uint32_t*>(logp + NIT * H);  // [31]
    const bool want_v = a.need_v != 0;

    double x0[N], x1[N];
    int bad = 0;
    double amax = 0.0;
    {
        const double* Ap = a.A + (size_t)(live ? prob : 0) * a.strideA;  // plan requires lda == 32
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] = live ? Ap[r0 + c * N] : 0.0;
            x1[c] = live ? Ap[r1 + c * N] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < N; ++c) {
            bad |= !isfinite(x0[c]) | !isfinite(x1[c]);
            amax = fmax(amax, fmax(fabs(x0[c]), fabs(x1[c])));
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int ex = prescale_exponent(amax);
    {
        const double scale = pow2(-ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] *= scale;
            x1[c] *= scale;
        }
    }
    if (a.reserved_stagger > 0) __nanosleep((unsigned)((warp % 3) * a.reserved_stagger));
    const double tol = a.tol;
    int sweeps = 0, last = 0, done = live ? 0 : 1;
    long long rot_total = 0;
    bool v_started = false;  // V still identity until the first replay

#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        int my_rot = 0;
        unsigned any_mask = 0;
        // ======================= W phase: one sweep =======================
#pragma unroll 1
        for (int t = 0; t < NIT; ++t) {
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double xa0 = x0[2 * k], xb0 = x0[2 * k + 1], xa1 = x1[2 * k], xb1 = x1[2 * k + 1];
                sm.red[(3 * k + 0) * RSTR + lane] = fma(xa1, xa1, xa0 * xa0);
                sm.red[(3 * k + 1) * RSTR + lane] = fma(xb1, xb1, xb0 * xb0);
                sm.red[(3 * k + 2) * RSTR + lane] = fma(xb1, xa1, xb0 * xa0);
            }
            __syncwarp();
            double g[3];
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const double2* row = reinterpret_cast<const double2*>(sm.red + (3 * hl + e) * RSTR + 16 * half);
                double2 p0 = row[0], p1 = row[1], p2 = row[2], p3 = row[3];
                double s0 = p0.x + p0.y, s1 = p1.x + p1.y, s2 = p2.x + p2.y, s3 = p3.x + p3.y;
                p0 = row[4];
                p1 = row[5];
                p2 = row[6];
                p3 = row[7];
                s0 += p0.x + p0.y;
                s1 += p1.x + p1.y;
                s2 += p2.x + p2.y;
                s3 += p3.x + p3.y;
                g[e] = (s0 + s1) + (s2 + s3);
            }
            // lane hl holds pair k = hl: slots (2k, 2k+1) = (top[k], bot[k])
            const int k = hl;
            const int ctop = (k == 0) ? 0 : col_at(k, t);
            const int cbot = col_at(k == 0 ? 0 : 2 * H - 1 - k, t);
            const bool flip = ctop > cbot;  // reference pair (i, j) = (min, max)
            const double gii = flip ? g[1] : g[0];
            const double gjj = flip ? g[0] : g[1];
            const double gji = g[2];
            const double absg = fabs(gji);
            Par par;
            par.cm1 = 0.0;
            par.c = 0.0;
            const bool rot = !done && !(absg <= 0.0) && !(absg < tol * fsqrt(gii * gjj));
            if (rot) {
                double s, cm1;
                rotation(gii - gjj, absg, s, cm1);
                const double ws = gji >= 0.0 ? s : -s;  // conj(g_ji)/|g_ji| * s for real data
                par.cm1 = cm1;
                par.c = flip ? -ws : ws;  // x = top slot, y = bot slot; i = min(top, bot)
            }
            my_rot += rot ? 1 : 0;
            const unsigned mask = __ballot_sync(0xffffffffu, rot);
            any_mask |= mask;
            sm.pub[half][k] = par;
            if (want_v && live) {  // a dead half aliases problem 0's workspace: never write
                logp[t * H + k] = par;
                if (hl == 0) logm[t] = (mask >> (16 * half)) & 0xFFFFu;
            }
            __syncwarp();
            if (mask) {
                // branch-free: identity rotations (cm1 = c = 0) are exact no-ops
#pragma unroll
                for (int q = 0; q < H; ++q) {
                    const Par pq = sm.pub[half][q];
                    applyv<F2>(x0[2 * q], x0[2 * q + 1], pq.cm1, pq.c);
                    applyv<F2>(x1[2 * q], x1[2 * q + 1], pq.cm1, pq.c);
                }
            }
            __syncwarp();
            ring_rotate(x0);
            ring_rotate(x1);
        }
        // ---- sweep end: per-problem rotation count over the half warp ----
        int tot = my_rot;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (!done) {
            sweeps = sw + 1;
            last = tot;
            rot_total += tot;
            if (tot == 0) done = 1;
        }
        const int partner_done = __shfl_xor_sync(0xffffffffu, done, 16);  // all lanes, unconditionally
        const bool both_done = done && partner_done;
        // ======================= V phase: replay the sweep =======================
        if (want_v && any_mask) {
            if (live) {
#pragma unroll
                for (int c = 0; c < N; ++c) {  // park W
                    wsW[r0 + c * N] = x0[c];
                    wsW[r1 + c * N] = x1[c];
                }
            }
            if (v_started) {
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    x0[c] = wsV[r0 + c * N];
                    x1[c] = wsV[r1 + c * N];
                }
            } else {  // V = I before the first replay
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    x0[c] = (c == r0) ? 1.0 : 0.0;
                    x1[c] = (c == r1) ? 1.0 : 0.0;
                }
                v_started = true;
            }
            __syncwarp();  // this warp's log writes are visible to all its lanes
            // mask words of this half's problem: lane hl holds iterations hl and hl + 16
            const uint32_t ma = logm[hl];
            const uint32_t mb = (hl + 16 < NIT) ? logm[hl + 16] : 0u;
            cp_async16(&sm.stage[0][half][hl], &logp[hl]);
            cp_commit();
#pragma unroll 1
            for (int t = 0; t < NIT; ++t) {
                if (t + 1 < NIT) cp_async16(&sm.stage[(t + 1) & 1][half][hl], &logp[(t + 1) * H + hl]);
                cp_commit();
                const uint32_t own = __shfl_sync(0xffffffffu, t < 16 ? ma : mb, 16 * half + (t & 15));
                const uint32_t both = own | __shfl_xor_sync(0xffffffffu, own, 16);
                cp_wait<1>();
                __syncwarp();
                if (both) {
                    const Par* st = sm.stage[t & 1][half];
#pragma unroll
                    for (int q = 0; q < H; ++q) {
                        const Par pq = st[q];
                        applyv<F2>(x0[2 * q], x0[2 * q + 1], pq.cm1, pq.c);
                        applyv<F2>(x1[2 * q], x1[2 * q + 1], pq.cm1, pq.c);
                    }
                }
                __syncwarp();
                ring_rotate(x0);
                ring_rotate(x1);
            }
            cp_wait<0>();
            if (live) {
#pragma unroll
                for (int c = 0; c < N; ++c) {  // park V
                    wsV[r0 + c * N] = x0[c];
                    wsV[r1 + c * N] = x1[c];
                }
            }
            __syncwarp();
#pragma unroll
            for (int c = 0; c < N; ++c) {
                x0[c] = wsW[r0 + c * N];
                x1[c] = wsW[r1 + c * N];
            }
        }
        if (both_done) break;
    }
    if (live) {
        const double unscale = pow2(ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            wsW[r0 + c * N] = x0[c] * unscale;
            wsW[r1 + c * N] = x1[c] * unscale;
        }
        if (want_v && !v_started) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsV[r0 + c * N] = (c == r0) ? 1.0 : 0.0;
                wsV[r1 + c * N] = (c == r1) ? 1.0 : 0.0;
            }
        }
    }
    const unsigned badm = __ballot_sync(0xffffffffu, bad != 0);
    if (live && hl == 0 && a.info) {
        bsvd_info inf;
        inf.converged = done;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = 0;
        inf.update_calls = 0;
        inf.last_rotations = last;
        inf.path = 1;
        inf.status = ((badm >> (16 * half)) & 0xFFFFu) ? 1 : 0;
        inf.kernel = a.kernel;
        a.info[prob] = inf;
    }
}

}  // namespace reg32

// register-budget variants: (warps per CTA, min CTAs per SM) -> registers per thread
//   KV_UNBLOCKED_REG32    (4, 3): 168 regs, 12 warps/SM (default)
//   KV_UNBLOCKED_REG32_R2 (2, 5): 204 regs, 10 warps/SM
//   KV_UNBLOCKED_REG32_R3 (1, 9): 227 regs,  9 warps/SM
//   KV_UNBLOCKED_REG32_O3 (4, 2): 255 regs,  8 warps/SM
static int variant_nw(int kv) {
    switch (kv) {
        case KV_UNBLOCKED_REG32_R2: return 2;
        case KV_UNBLOCKED_REG32_R3: return 1;
        default: return 4;
    }
}

Plan plan_unblocked_reg(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_D && bm == 32 && bn == 32 && lda_ok) {
        const bool known = variant == KV_UNBLOCKED_REG32 || variant == KV_UNBLOCKED_REG32_O3 ||
                           variant == KV_UNBLOCKED_REG32_R2 || variant == KV_UNBLOCKED_REG32_R3 ||
                           variant == KV_UNBLOCKED_REG32_F2;
        p.kernel = known ? variant : KV_UNBLOCKED_REG32;
        p.threads = variant_nw(p.kernel) * 32;
        p.smem = variant_nw(p.kernel) * sizeof(reg32::WarpSmem);
        p.work_elems = 2 * 32 * 32 + reg32::LOG_ELEMS;
        p.grid = 0;
        p.resident = 0;
        (void)need_v;
    }
    return p;
}

template <int NW, int MAXREG, bool F2 = false>
static int launch_variant(SolveArgs<double> a, cudaStream_t st) {
    const int per_cta = 2 * NW;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    const size_t smem = NW * sizeof(reg32::WarpSmem);
    auto k = reg32::k_reg32<NW, MAXREG, F2>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<grid, NW * 32, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_unblocked_reg_d32(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    int rc;
    switch (p.kernel) {
        case KV_UNBLOCKED_REG32_O3: rc = launch_variant<4, 255>(a, st); break;
        case KV_UNBLOCKED_REG32_R2: rc = launch_variant<2, 200>(a, st); break;
        case KV_UNBLOCKED_REG32_R3: rc = launch_variant<1, 224>(a, st); break;
        case KV_UNBLOCKED_REG32_F2: rc = launch_variant<4, 168, true>(a, st); break;
        default: rc = launch_variant<4, 168>(a, st); break;
    }
    if (rc) return rc;
    return launch_finalize_ws<double>(a, st);
}

}  // namespace bsvd
