// unblocked_reg16.cu -- kernel (2), register-resident fast path for 16x16 FP32
// (BASELINE config C2).
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule for ell = 16 (15 iterations x 8 pairs per
// sweep), per-problem exit after the first quiet sweep.
//
// Mapping: a warp owns FOUR problems; quarter-warp q (8 lanes) owns problem q
// and every lane holds rows l and l+8 of W (and of V) in registers.  As in the
// 32-column kernel the column pairs sit in fixed register slots and columns
// move one ring position per iteration (static register indices).  The 24
// per-lane dot-product partials are reduced over the 8 lanes with a
// transposing xor butterfly (21 shuffles), after which lane k of each quarter
// holds pair k's sums and evaluates the rotation; the parameters are
// broadcast back with shuffles.  Everything stays in FP32 registers with FMA:
// the reference forms the rotation and the update in float64 and rounds on
// store (F6); here the norms, parameters and updates run in float32 (one to
// two extra roundings per update, measured accuracy in DESIGN.md), which keeps
// the kernel on the 128-lane FP32 pipe.  Data are pre-scaled by an exact power
// of two so squared norms cannot over/underflow.  Raw W and V go to the
// workspace; finalize.cu (sigma in float64) completes the factorisation.
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {
namespace reg16 {

constexpr int N = 16;     // columns
constexpr int H = 8;      // pairs per iteration
constexpr int NIT = 15;   // iterations per sweep
constexpr int NW = 4;     // warps per CTA (16 problems)

__host__ __device__ constexpr int ring_slot(int q) {
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}

__device__ __forceinline__ void ring_rotate(float (&x)[N]) {
    const float t = x[ring_slot(NIT - 1)];
#pragma unroll
    for (int q = NIT - 1; q >= 1; --q) x[ring_slot(q)] = x[ring_slot(q - 1)];
    x[ring_slot(0)] = t;
}

__device__ __forceinline__ int col_at(int r, int t) {
    int q = r - t;
    if (q < 0) q += NIT;
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}

__device__ __forceinline__ float rsqrt_nr(float x) {  // 1/sqrt(x), one Newton step on the MUFU seed
    const float r = rsqrtf(x);
    return fmaf(0.5f * r, fmaf(-x * r, r, 1.0f), r);
}
__device__ __forceinline__ float rcp_nr(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.0f), r);
}

__device__ __forceinline__ float pow2f(int e) {  // 2^e, e in [-126, 127]
    return __int_as_float((127 + e) << 23);
}

// Reference rotation formulas (F5) in float32 on exponent-normalised (d, g):
// t = sgn(d) 2g / (|d| + sqrt(d^2 + 4 g^2)), c = 1/sqrt(1 + t^2), s = t c, c - 1 = -s^2 / (1 + c).
__device__ __forceinline__ void rotation_f32(float d, float g, float& s_out, float& cm1_out) {
    const float mx = fmaxf(fabsf(d), g);
    const int e = ((__float_as_int(mx) >> 23) & 0xff) - 127;
    const float sc = pow2f(-max(-126, min(126, e)));
    const float dn = d * sc, gn = g * sc;
    const float q = fmaf(dn, dn, 4.0f * gn * gn);
    const float rq = rsqrt_nr(q);
    const float sq = q * rq;
    const float den = fabsf(dn) + sq;
    float t = 2.0f * gn * rcp_nr(den);
    t = d >= 0.0f ? t : -t;
    const float c = rsqrt_nr(fmaf(t, t, 1.0f));
    const float s = t * c;
    s_out = s;
    cm1_out = -(s * s) * rcp_nr(1.0f + c);
}

__device__ __forceinline__ void apply(float& x, float& y, float cm1, float c) {
    const float nx = x + fmaf(cm1, x, c * y);
    const float ny = y + fmaf(cm1, y, -(c * x));
    x = nx;
    y = ny;
}

template <bool WANT_V>
__global__ void __launch_bounds__(NW * 32) k_reg16(SolveArgs<float> a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int quarter = lane >> 3, ql = lane & 7;
    const int prob = (blockIdx.x * NW + warp) * 4 + quarter;
    const bool live = prob < a.batch;
    const int bm = a.bm;  // rows (<= 16); missing rows are zero
    const int r0 = ql, r1 = ql + 8;
    float x0[N], x1[N], y0[N], y1[N];
    int bad = 0;
    float amax = 0.0f;
    {
        const float* Ap = a.A + (size_t)(live ? prob : 0) * a.strideA;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] = (live && r0 < bm) ? Ap[r0 + (size_t)c * a.lda] : 0.0f;
            x1[c] = (live && r1 < bm) ? Ap[r1 + (size_t)c * a.lda] : 0.0f;
            bad |= !isfinite(x0[c]) | !isfinite(x1[c]);
            amax = fmaxf(amax, fmaxf(fabsf(x0[c]), fabsf(x1[c])));
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    int ex = ((__float_as_int(amax) >> 23) & 0xff) - 126;
    if (!(amax > 0.0f) || !isfinite(amax)) ex = 0;
    ex = max(-100, min(100, ex));
    {
        const float sc = pow2f(-ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] *= sc;
            x1[c] *= sc;
        }
    }
    if (WANT_V) {
#pragma unroll
        for (int c = 0; c < N; ++c) {
            y0[c] = (c == r0) ? 1.0f : 0.0f;
            y1[c] = (c == r1) ? 1.0f : 0.0f;
        }
    }
    const float tol = (float)a.tol;
    int sweeps = 0, last = 0, done = live ? 0 : 1;
    long long rot_total = 0;
    const int qbase = lane & ~7;
    const bool b2 = (ql >> 2) & 1, b1 = (ql >> 1) & 1, b0 = ql & 1;

#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        int my_rot = 0;
#pragma unroll 1
        for (int t = 0; t < NIT; ++t) {
            // ---- dot products over this lane's two rows, pairs k = 0..7 ----
            float v[H][3];
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const float xa0 = x0[2 * k], xb0 = x0[2 * k + 1], xa1 = x1[2 * k], xb1 = x1[2 * k + 1];
                v[k][0] = fmaf(xa1, xa1, xa0 * xa0);
                v[k][1] = fmaf(xb1, xb1, xb0 * xb0);
                v[k][2] = fmaf(xb1, xa1, xb0 * xa0);
            }
            // ---- transposing butterfly over the 8 lanes of the quarter ----
            float k1[4][3];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int e = 0; e < 3; ++e) {
                    const float keep = b2 ? v[k + 4][e] : v[k][e];
                    const float send = b2 ? v[k][e] : v[k + 4][e];
                    k1[k][e] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
            float k2[2][3];
#pragma unroll
            for (int k = 0; k < 2; ++k)
#pragma unroll
                for (int e = 0; e < 3; ++e) {
                    const float keep = b1 ? k1[k + 2][e] : k1[k][e];
                    const float send = b1 ? k1[k][e] : k1[k + 2][e];
                    k2[k][e] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
                }
            float g[3];
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const float keep = b0 ? k2[1][e] : k2[0][e];
                const float send = b0 ? k2[0][e] : k2[1][e];
                g[e] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
            }
            // lane ql holds pair k = ql: slots (2k, 2k+1) = (top[k], bot[k])
            const int k = ql;
            const int ctop = (k == 0) ? 0 : col_at(k, t);
            const int cbot = col_at(k == 0 ? 0 : 2 * H - 1 - k, t);
            const bool flip = ctop > cbot;
            const float gii = flip ? g[1] : g[0];
            const float gjj = flip ? g[0] : g[1];
            const float gji = g[2];
            const float absg = fabsf(gji);
            float cm1 = 0.0f, cc = 0.0f;
            const float lim = tol * (sqrtf(gii) * sqrtf(gjj));
            const bool rot = !done && !(absg <= 0.0f) && !(absg < lim);
            if (rot) {
                float s;
                rotation_f32(gii - gjj, absg, s, cm1);
                const float ws = gji >= 0.0f ? s : -s;
                cc = flip ? -ws : ws;
            }
            my_rot += rot ? 1 : 0;
            const unsigned mask = __ballot_sync(0xffffffffu, rot);
            if (mask) {
#pragma unroll
                for (int q = 0; q < H; ++q) {
                    const float pc = __shfl_sync(0xffffffffu, cm1, qbase + q);
                    const float pcc = __shfl_sync(0xffffffffu, cc, qbase + q);
                    apply(x0[2 * q], x0[2 * q + 1], pc, pcc);
                    apply(x1[2 * q], x1[2 * q + 1], pc, pcc);
                    if (WANT_V) {
                        apply(y0[2 * q], y0[2 * q + 1], pc, pcc);
                        apply(y1[2 * q], y1[2 * q + 1], pc, pcc);
                    }
                }
            }
            ring_rotate(x0);
            ring_rotate(x1);
            if (WANT_V) {
                ring_rotate(y0);
                ring_rotate(y1);
            }
        }
        int tot = my_rot;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (!done) {
            sweeps = sw + 1;
            last = tot;
            rot_total += tot;
            if (tot == 0) done = 1;
        }
        const int all_done = __all_sync(0xffffffffu, done != 0);
        if (all_done) break;
    }
    const unsigned badm = __ballot_sync(0xffffffffu, bad != 0);
    if (live) {
        float* wsW = a.work + (size_t)prob * a.work_stride;
        float* wsV = wsW + bm * N;
        const float us = pow2f(ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            if (r0 < bm) wsW[r0 + c * bm] = x0[c] * us;
            if (r1 < bm) wsW[r1 + c * bm] = x1[c] * us;
        }
        if (WANT_V) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsV[r0 + c * N] = y0[c];
                wsV[r1 + c * N] = y1[c];
            }
        }
        if (ql == 0 && a.info) {
            bsvd_info inf;
            inf.converged = done;
            inf.outer_sweeps = sweeps;
            inf.rotations = rot_total;
            inf.gram_calls = 0;
            inf.update_calls = 0;
            inf.last_rotations = last;
            inf.path = 1;
            inf.status = ((badm >> (8 * quarter)) & 0xFFu) ? 1 : 0;
            inf.kernel = KV_UNBLOCKED_REG16F;
            a.info[prob] = inf;
        }
    }
}

}  // namespace reg16

Plan plan_unblocked_reg16(int dtype, int bm, int bn, int need_v, bool lda_ok) {
    Plan p{};
    if (dtype == BSVD_S && bn == 16 && bm >= 16 && bm <= 16 && lda_ok) {
        p.kernel = KV_UNBLOCKED_REG16F;
        p.threads = reg16::NW * 32;
        p.work_elems = (size_t)bm * 16 + (need_v ? 16 * 16 : 0);
    }
    return p;
}

int launch_unblocked_reg16(SolveArgs<float> a, const Plan& p, cudaStream_t st) {
    a.kernel = KV_UNBLOCKED_REG16F;
    a.work_stride = (int64_t)p.work_elems;
    const int per_cta = 4 * reg16::NW;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    if (a.need_v) reg16::k_reg16<true><<<grid, reg16::NW * 32, 0, st>>>(a);
    else reg16::k_reg16<false><<<grid, reg16::NW * 32, 0, st>>>(a);
    if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
    return launch_finalize_ws<float>(a, st);
}

}  // namespace bsvd
