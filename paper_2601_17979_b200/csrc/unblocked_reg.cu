// unblocked_reg.cu -- kernel (2), register-resident fast path for 32x32 FP64.
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule (src/ordering.py:32-75), with the working
// copy held in registers instead of shared memory:
//
//  * A warp owns TWO problems; half-warp h (16 lanes) owns problem h, and each
//    lane holds two full rows of W (rows l and l+16, 2 x 32 doubles).  The
//    16 disjoint column pairs of a schedule iteration sit in fixed register
//    slots (2k, 2k+1); instead of indexing columns by the schedule, the
//    columns are MOVED between slots after every iteration along the
//    tournament ring (bot0 -> top1 -> ... -> top15 -> bot15 -> ... -> bot1 ->
//    bot0), so every register index is a compile-time constant.  After 31
//    iterations (one sweep) the slots are back in natural column order.
//  * The 48 dot products of an iteration (g_ii, g_jj, g_ji for 16 pairs) are
//    formed per lane over its two rows and reduced over the 16 lanes with a
//    transposing xor butterfly (45 shuffles instead of 48 x 4): after the last
//    level lane k of each half holds the full sums of pair k and evaluates the
//    rotation (guard F4, parameters F5) in float64 exactly like the reference.
//  * Parameters go through a 4-deep shared-memory ring guarded by mbarriers to
//    a V warp that holds the two problems' V rows the same way and applies
//    the identical rotations (warp specialisation: the V update never waits
//    on the dot-product/parameter chain).
//  * A problem stops after its first quiet sweep (per-problem convergence on
//    the device); the warp keeps stepping its partner problem, whose quiet
//    sweeps are exact no-ops (F7).
//  * The raw converged W and V go to a workspace; the finalisation kernel
//    (finalize.cu) forms sigma, normalises, sorts and permutes.
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {
namespace reg32 {

constexpr int N = 32;       // columns
constexpr int H = 16;       // column pairs per iteration
constexpr int NIT = 31;     // iterations per sweep
constexpr int RING = 4;     // parameter ring depth (iterations)
constexpr int WPAIRS = 2;   // (A warp, V warp) pairs per CTA -> 4 problems per CTA
constexpr int RSTR = 34;    // doubles per row of the dot-product transpose buffer (bank padding)

// ring position -> register slot (slot 2k = top[k], slot 2k+1 = bot[k])
__host__ __device__ constexpr int ring_slot(int q) {
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}

struct __align__(16) Par {
    double cm1, c;  // x <- x + (cm1 x + c y);  y <- y + (cm1 y - c x)
};
struct __align__(16) Slot {
    Par p[2][H];      // [problem half][pair]
    unsigned mask;    // rotation bits: pair k of half h at bit 16h + k
    int stop;
    int pad[2];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

// advance every column one ring position (compile-time register moves)
__device__ __forceinline__ void ring_rotate(double (&x)[N]) {
    const double t = x[ring_slot(NIT - 1)];
#pragma unroll
    for (int q = NIT - 1; q >= 1; --q) x[ring_slot(q)] = x[ring_slot(q - 1)];
    x[ring_slot(0)] = t;
}

// value (column index) at ring position r after t rotations, ell = 32
__device__ __forceinline__ int col_at(int r, int t) {
    int q = r - t;
    if (q < 0) q += NIT;
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}

__device__ __forceinline__ void apply(double& x, double& y, double cm1, double c) {
    const double nx = x + fma(cm1, x, c * y);
    const double ny = y + fma(cm1, y, -(c * x));
    x = nx;
    y = ny;
}

template <bool WANT_V, int MINB>
__global__ void __launch_bounds__(WANT_V ? 128 : 64, WANT_V ? MINB : 2 * MINB) k_reg32(SolveArgs<double> a) {
    __shared__ Slot ring[WPAIRS][RING];
    __shared__ uint64_t full[WPAIRS][RING], empty_[WPAIRS][RING];
    __shared__ __align__(16) double redbuf[WPAIRS][3 * H * RSTR];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int half = lane >> 4, hl = lane & 15;
    const int wp = warp % WPAIRS;           // warp pair
    const bool is_v = warp >= WPAIRS;
    const int prob = blockIdx.x * (2 * WPAIRS) + wp * 2 + half;
    const bool live = prob < a.batch;
    if (threadIdx.x == 0) {
        for (int w = 0; w < WPAIRS; ++w)
            for (int s = 0; s < RING; ++s) {
                mbar_init(&full[w][s], 32);
                mbar_init(&empty_[w][s], 32);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int r0 = hl, r1 = hl + 16;
    double* wsW = a.work + (size_t)(live ? prob : 0) * a.work_stride;
    double* wsV = wsW + N * N;

    if (!is_v) {
        // ---------------- A warp: dots, rotation parameters, W update ----------------
        double* red = redbuf[wp];
        double x0[N], x1[N];
        const double* Ap = a.A + (size_t)(live ? prob : 0) * a.strideA;
        int bad = 0;
        double amax = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] = live ? Ap[r0 + c * N] : 0.0;  // plan requires lda == 32
            x1[c] = live ? Ap[r1 + c * N] : 0.0;
            bad |= !isfinite(x0[c]) | !isfinite(x1[c]);
            amax = fmax(amax, fmax(fabs(x0[c]), fabs(x1[c])));
        }
        // exact power-of-two pre-scaling to max|a| in [0.5, 1): rotations are
        // scale invariant and the scaling is exact, so the iteration is the same;
        // it keeps the call-free div/sqrt operands in range (undone on output)
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        int ex = (int)((__double_as_longlong(amax) >> 52) & 0x7ff) - 1022;
        if (!(amax > 0.0) || !isfinite(amax)) ex = 0;
        ex = max(-1021, min(1022, ex));
        const double scale = __longlong_as_double((long long)(1023 - ex) << 52);
        const double unscale = __longlong_as_double((long long)(1023 + ex) << 52);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] *= scale;
            x1[c] *= scale;
        }
        const double tol = a.tol;
        int sweeps = 0, last = 0, done = live ? 0 : 1;
        long long rot_total = 0;
        uint32_t it = 0;
#pragma unroll 1
        for (int sw = 0; sw < a.max_sweeps; ++sw) {
            int my_rot = 0;
#pragma unroll 1
            for (int t = 0; t < NIT; ++t) {
                // ---- dot products: 16 pairs x 3 values per lane over its two rows,
                //      transposed through shared memory: lane k of each half then sums
                //      the 16 partials of pair k (conflict-free LDS.128, 34-double rows)
#pragma unroll
                for (int k = 0; k < H; ++k) {
                    const double xa0 = x0[2 * k], xb0 = x0[2 * k + 1], xa1 = x1[2 * k], xb1 = x1[2 * k + 1];
                    red[(3 * k + 0) * RSTR + lane] = fma(xa1, xa1, xa0 * xa0);
                    red[(3 * k + 1) * RSTR + lane] = fma(xb1, xb1, xb0 * xb0);
                    red[(3 * k + 2) * RSTR + lane] = fma(xb1, xa1, xb0 * xa0);
                }
                __syncwarp();
                double g[3];
#pragma unroll
                for (int e = 0; e < 3; ++e) {
                    const double2* row = reinterpret_cast<const double2*>(red + (3 * hl + e) * RSTR + 16 * half);
                    double2 p0 = row[0], p1 = row[1], p2 = row[2], p3 = row[3];
                    double s0 = p0.x + p0.y, s1 = p1.x + p1.y, s2 = p2.x + p2.y, s3 = p3.x + p3.y;
                    p0 = row[4]; p1 = row[5]; p2 = row[6]; p3 = row[7];
                    s0 += p0.x + p0.y;
                    s1 += p1.x + p1.y;
                    s2 += p2.x + p2.y;
                    s3 += p3.x + p3.y;
                    g[e] = (s0 + s1) + (s2 + s3);
                }
                // lane hl now holds pair k = hl: slots (2k, 2k+1) = (top[k], bot[k])
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
                bool rot = false;
                if (!(absg <= 0.0) && !(absg < tol * fsqrt(gii * gjj))) {
                    rot = true;
                    const double w = copysign(1.0, gji);  // conj(g_ji)/|g_ji| for real data
                    const RotParams p = rot_params_fast(gii - gjj, 2.0 * absg);
                    const double ws = w * p.s;
                    par.cm1 = p.cm1;
                    // x = top slot, y = bot slot; i = min(top, bot)
                    par.c = flip ? -ws : ws;
                }
                rot = rot && !done;
                if (!rot) {
                    par.cm1 = 0.0;
                    par.c = 0.0;
                }
                my_rot += rot ? 1 : 0;
                const unsigned mask = __ballot_sync(0xffffffffu, rot);
                // ---- publish to the ring (V warp) ----
                const uint32_t s = it % RING;
                if (WANT_V && it >= RING) mbar_wait(&empty_[wp][s], ((it / RING) - 1) & 1);
                Slot& sl = ring[wp][s];
                sl.p[half][k] = par;
                if (lane == 0) {
                    sl.mask = mask;
                    sl.stop = 0;
                }
                __syncwarp();
                if (WANT_V) mbar_arrive(&full[wp][s]);
                // ---- W update: pairs rotating in either half; identity params elsewhere ----
#pragma unroll
                for (int q = 0; q < H; ++q) {
                    if (mask & (0x10001u << q)) {
                        const Par pq = sl.p[half][q];
                        apply(x0[2 * q], x0[2 * q + 1], pq.cm1, pq.c);
                        apply(x1[2 * q], x1[2 * q + 1], pq.cm1, pq.c);
                    }
                }
                if (!WANT_V) __syncwarp();  // the slot is rewritten next iteration
                ring_rotate(x0);
                ring_rotate(x1);
                ++it;
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
            const int other = __shfl_xor_sync(0xffffffffu, done, 16);
            if (done && other) break;
        }
        // stop marker for the V warp
        if (WANT_V) {
            const uint32_t s = it % RING;
            if (it >= RING) mbar_wait(&empty_[wp][s], ((it / RING) - 1) & 1);
            if (lane == 0) ring[wp][s].stop = 1;
            __syncwarp();
            mbar_arrive(&full[wp][s]);
        }
        if (live) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsW[r0 + c * N] = x0[c] * unscale;
                wsW[r1 + c * N] = x1[c] * unscale;
            }
            const unsigned badm = __ballot_sync(0xffffffffu, bad != 0);
            if (hl == 0 && a.info) {
                bsvd_info inf;
                inf.converged = done;
                inf.outer_sweeps = sweeps;
                inf.rotations = rot_total;
                inf.gram_calls = 0;
                inf.update_calls = 0;
                inf.last_rotations = last;
                inf.path = 1;
                inf.status = (badm >> (16 * half)) & 0xFFFFu ? 1 : 0;
                inf.kernel = MINB == 3 ? KV_UNBLOCKED_REG32_O3 : KV_UNBLOCKED_REG32;
                a.info[prob] = inf;
            }
        }
    } else if (WANT_V) {
        // ---------------- V warp: replay the rotations on V ----------------
        double y0[N], y1[N];
#pragma unroll
        for (int c = 0; c < N; ++c) {
            y0[c] = (c == r0) ? 1.0 : 0.0;
            y1[c] = (c == r1) ? 1.0 : 0.0;
        }
#pragma unroll 1
        for (uint32_t it = 0;; ++it) {
            const uint32_t s = it % RING;
            mbar_wait(&full[wp][s], (it / RING) & 1);
            const Slot& sl = ring[wp][s];
            if (sl.stop) break;
            const unsigned mask = sl.mask;
#pragma unroll
            for (int q = 0; q < H; ++q) {
                if (mask & (0x10001u << q)) {
                    const Par pq = sl.p[half][q];
                    apply(y0[2 * q], y0[2 * q + 1], pq.cm1, pq.c);
                    apply(y1[2 * q], y1[2 * q + 1], pq.cm1, pq.c);
                }
            }
            __syncwarp();
            mbar_arrive(&empty_[wp][s]);
            ring_rotate(y0);
            ring_rotate(y1);
        }
        if (live) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsV[r0 + c * N] = y0[c];
                wsV[r1 + c * N] = y1[c];
            }
        }
    }
}

}  // namespace reg32

Plan plan_unblocked_reg(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_D && bm == 32 && bn == 32 && lda_ok) {
        p.kernel = variant == KV_UNBLOCKED_REG32_O3 ? KV_UNBLOCKED_REG32_O3 : KV_UNBLOCKED_REG32;
        p.threads = need_v ? 128 : 64;
        p.smem = 0;
        p.work_elems = 2 * 32 * 32;
        p.grid = 0;
        p.resident = 0;
    }
    return p;
}

int launch_unblocked_reg_d32(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = 2 * 32 * 32;
    const int per_cta = 2 * reg32::WPAIRS;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    if (p.kernel == KV_UNBLOCKED_REG32_O3) {
        if (a.need_v) reg32::k_reg32<true, 3><<<grid, 128, 0, st>>>(a);
        else reg32::k_reg32<false, 3><<<grid, 64, 0, st>>>(a);
    } else {
        if (a.need_v) reg32::k_reg32<true, 2><<<grid, 128, 0, st>>>(a);
        else reg32::k_reg32<false, 2><<<grid, 64, 0, st>>>(a);
    }
    if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
    return launch_finalize_ws<double>(a, st);
}

}  // namespace bsvd
