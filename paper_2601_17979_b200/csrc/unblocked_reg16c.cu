// unblocked_reg16c.cu -- kernel (2), third-generation register-resident
// 16x16 FP32 path (BASELINE config C2).
//
// Same iteration, schedule and arithmetic as unblocked_reg16b.cu (the
// iteration of src/_kernels_numba.py:85-138 on the round-robin ring of
// src/ordering.py:32-75, per-problem exit after the first quiet sweep), with
// a quarter-warp per problem: a warp owns FOUR problems, lane l of quarter q
// holds rows l and l + 8 of problem q's W and V (32 + 32 floats).  Per
// problem-iteration this removes the redundancy of gen. 2, where two lanes
// evaluate every rotation and every lane holds one row:
//  * each lane pre-sums its two rows' products, so the transposing xor
//    butterfly over the 8 lanes of a quarter is 4 + 2 + 1 shuffles and lane l
//    ends with pair l's g_ji alone (no duplicate parameter chain).  The
//    pre-sum (rounded products, no FMA contraction) is gen. 2's xor-8 level
//    and the remaining levels are its xor 4, 2, 1, so every dot product, and
//    with it every rotation, has gen. 2's bits: the two kernels are
//    bit-identical and the default switches between them on the batch size
//    without breaking batch == standalone (reference tests/test_batch.py:19-28);
//  * the rotation update is the same 4 FMAs per row and column pair, on twice
//    the rows per lane, so the FMA count per problem is unchanged while the
//    reduction / parameter / publish overhead per problem halves.
// The fused finalisation sums sigma in float64 in finalize_block's tree
// (rows l, l + 8 pre-summed in-lane = its xor-8 level, then xor 4, 2, 1), so
// sigma and U are the bits of the standalone pass; problems with a
// sigma < tiny/u column are flagged to it (orthogonal completion).
#include "kernel_args.cuh"
#include "launch.h"
#include "ring16.cuh"

namespace bsvd {
namespace reg16c {

using namespace ring16;

struct __align__(16) QSmem {  // one problem (quarter-warp)
    float2 pub[H];            // this iteration's rotations (cm1, c) by pair
    float nrm[N];             // maintained squared column norms
    float sig[N];             // finalisation: sigma by column
    int rk[N];                // finalisation: rank by column
    int ex, bad, sweeps, last, rot;  // per-problem bookkeeping, kept here to free registers for the rows
};

// Transposing xor butterfly over the 8 lanes of a quarter: lane ql ends with the quarter's total
// of v[ql] (4 + 2 + 1 shuffles).
__device__ __forceinline__ float reduce8q(const float (&v)[H], int ql) {
    const bool b2 = ql & 4, b1 = ql & 2, b0 = ql & 1;
    float a4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float keep = b2 ? v[i + 4] : v[i], send = b2 ? v[i] : v[i + 4];
        a4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    float a2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float keep = b1 ? a4[i + 2] : a4[i], send = b1 ? a4[i] : a4[i + 2];
        a2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    const float keep = b0 ? a2[1] : a2[0], send = b0 ? a2[0] : a2[1];
    return keep + __shfl_xor_sync(0xffffffffu, send, 1);
}

// any bit of a quarter set -> all 8 bits of that quarter (a problem's masks never depend on its neighbours)
__device__ __forceinline__ uint32_t quarter_spread(uint32_t b) {
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) r |= ((b >> (8 * q)) & 0xFFu) ? (0xFFu << (8 * q)) : 0u;
    return r;
}

// the two-FMA update (ring16::apply2) on rows l and l + 8 at once: packed FP32 FMAs (FFMA2, one issue
// slot for two FMAs, the coefficient broadcast from one register); per half identical to apply2
__device__ __forceinline__ void apply2x2(float2& x, float2& y, float cm1, float c) {
    const float2 cc = make_float2(c, c), nc = make_float2(-c, -c), mm = make_float2(cm1, cm1);
    const float2 tx = __ffma2_rn(cc, y, x);
    const float2 ty = __ffma2_rn(nc, x, y);
    x = __ffma2_rn(mm, x, tx);
    y = __ffma2_rn(mm, y, ty);
}

struct St {
    int my_rot;
    bool full;       // some lane of the warp takes fresh norms this iteration
    uint32_t fmask;  // lanes whose problem takes them
};

// the same update written to other registers (the ring shift folded into it, see iter)
__device__ __forceinline__ void apply2x2_to(float2 x, float2 y, float2& nx, float2& ny, float cm1, float c) {
    const float2 cc = make_float2(c, c), nc = make_float2(-c, -c), mm = make_float2(cm1, cm1);
    const float2 tx = __ffma2_rn(cc, y, x);
    const float2 ty = __ffma2_rn(nc, x, y);
    nx = __ffma2_rn(mm, x, tx);
    ny = __ffma2_rn(mm, y, ty);
}

template <int u, bool WANT_V, int SH = 0>
__device__ __forceinline__ void iter(float2 (&X)[N], float2 (&Y)[N], QSmem& sm,
                                     const uint32_t* ctab, int t, int lane, int ql, bool done, float tol2,
                                     float tol, St& st) {
    float v[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
        const float2 pr = __fmul2_rn(X[BS(q, u)], X[TS(q, u)]);
        v[q] = __fadd_rn(pr.x, pr.y);
    }
    const float g = reduce8q(v, ql);
    const uint32_t code = ctab[t * H + ql];
    const int ct = code & 0xff, cb = (code >> 8) & 0xff;
    const bool flip = (code >> 16) != 0;
    float gt = sm.nrm[ct], gb = sm.nrm[cb];
    if (st.full) {
        float a[H];  // one set of partials at a time
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const float2 pa = __fmul2_rn(X[TS(q, u)], X[TS(q, u)]);
            a[q] = __fadd_rn(pa.x, pa.y);
        }
        const float ft = reduce8q(a, ql);
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const float2 pb = __fmul2_rn(X[BS(q, u)], X[BS(q, u)]);
            a[q] = __fadd_rn(pb.x, pb.y);
        }
        const float fb = reduce8q(a, ql);
        if ((st.fmask >> lane) & 1u) {
            gt = ft;
            gb = fb;
        }
    }
    const float absg = fabsf(g);
    const bool rot = rot_guard(absg, gt, gb, tol2, tol) && !done && absg > 0.0f;
    const float d = gt - gb;
    float s, cm1, tabs;
    rot_abs(fabsf(d), absg, s, cm1, tabs);
    const bool eneg = d < 0.0f || (d == 0.0f && flip);  // sgn(0) = +1 in (i, j) orientation
    const float c = rot ? xor_signf(s, (g < 0.0f) != eneg) : 0.0f;
    cm1 = rot ? cm1 : 0.0f;
    const float dtg = rot ? xor_signf(tabs * absg, eneg) : 0.0f;
    const float nt = gt + dtg, nb = gb - dtg;
    const bool shrink = rot && (nt < 0.25f * gt || nb < 0.25f * gb);
    __syncwarp();  // every lane has read last iteration's pub[]
    sm.pub[ql] = make_float2(cm1, c);
    sm.nrm[ct] = nt;  // lane ql alone owns columns ct, cb of its problem this iteration
    sm.nrm[cb] = nb;
    st.my_rot += rot ? 1 : 0;
    const unsigned mask = __ballot_sync(0xffffffffu, rot);
    {
        const uint32_t sb = __ballot_sync(0xffffffffu, shrink);
        st.fmask = quarter_spread(sb);
        st.full = sb != 0u;
    }
    __syncwarp();
    if constexpr (SH == 0) {
        if (mask) {
            // two pairs' parameters per 16-byte load, fetched just before use (4 live registers, not 16)
            const float4* pp = reinterpret_cast<const float4*>(sm.pub);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float4 pr = pp[i];
                apply2x2(X[TS(2 * i, u)], X[BS(2 * i, u)], pr.x, pr.y);
                if (WANT_V) apply2x2(Y[TS(2 * i, u)], Y[BS(2 * i, u)], pr.x, pr.y);
                apply2x2(X[TS(2 * i + 1, u)], X[BS(2 * i + 1, u)], pr.z, pr.w);
                if (WANT_V) apply2x2(Y[TS(2 * i + 1, u)], Y[BS(2 * i + 1, u)], pr.z, pr.w);
            }
        }
    } else {
        // last iteration of an unrolled group, branch-free: the ring shift by SH is folded into the
        // update (every slot is in one pair; pairs that do not rotate have zero parameters and copy
        // exactly), so the loop back-edge moves no registers
        const float4* pp = reinterpret_cast<const float4*>(sm.pub);
        float2 X2[N], Y2[N];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 pr = pp[i];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int q = 2 * i + h;
                const float pc = h ? pr.z : pr.x, ps = h ? pr.w : pr.y;
                apply2x2_to(X[TS(q, u)], X[BS(q, u)], X2[dst_slot(TS(q, u), SH)], X2[dst_slot(BS(q, u), SH)], pc, ps);
                if (WANT_V)
                    apply2x2_to(Y[TS(q, u)], Y[BS(q, u)], Y2[dst_slot(TS(q, u), SH)], Y2[dst_slot(BS(q, u), SH)], pc,
                                ps);
            }
        }
#pragma unroll
        for (int c = 0; c < N; ++c) {
            X[c] = X2[c];
            if (WANT_V) Y[c] = Y2[c];
        }
    }
}

template <int SH, bool WANT_V>
__device__ __forceinline__ void shift_all(float2 (&X)[N], float2 (&Y)[N]) {
    ring_shift<SH>(X);
    if (WANT_V) ring_shift<SH>(Y);
}

// iterations t0 + u .. t0 + U - 1 with compile-time register slots
template <int U, int u, bool WANT_V>
__device__ __forceinline__ void group(float2 (&X)[N], float2 (&Y)[N], QSmem& sm,
                                      const uint32_t* ctab, int t0, int lane, int ql, bool done, float tol2,
                                      float tol, St& st) {
    iter<u, WANT_V>(X, Y, sm, ctab, t0 + u, lane, ql, done, tol2, tol, st);
    if constexpr (u + 1 < U) group<U, u + 1, WANT_V>(X, Y, sm, ctab, t0, lane, ql, done, tol2, tol, st);
}

template <int NW, int MINB, int U, bool WANT_V>
__global__ void __launch_bounds__(NW * 32, MINB) k_reg16c(SolveArgs<float> a) {
    __shared__ QSmem qsm[NW * 4];
    __shared__ uint32_t ctab[NIT * H];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int qt = lane >> 3, ql = lane & 7;
    for (int e = threadIdx.x; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    __syncthreads();
    QSmem& sm = qsm[warp * 4 + qt];
    const int prob = (blockIdx.x * NW + warp) * 4 + qt;
    const bool live = prob < a.batch;
    float2 X[N], Y[N];  // rows (l, l + 8) of W and V: packed pairs for the FFMA2 update
    int bad = 0;
    float amax = 0.0f;
    {
        const float* Ap = a.A + (size_t)(live ? prob : 0) * a.strideA;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            X[c].x = live ? Ap[ql + (size_t)c * a.lda] : 0.0f;
            X[c].y = live ? Ap[ql + 8 + (size_t)c * a.lda] : 0.0f;
            bad |= !isfinite(X[c].x) || !isfinite(X[c].y);
            amax = fmaxf(amax, fmaxf(fabsf(X[c].x), fabsf(X[c].y)));
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    int ex = ((__float_as_int(amax) >> 23) & 0xff) - 126;
    if (!(amax > 0.0f) || !isfinite(amax)) ex = 0;
    ex = max(-100, min(100, ex));
    {
        const unsigned bm = __ballot_sync(0xffffffffu, bad != 0);
        if (ql == 0) {
            sm.ex = ex;
            sm.bad = ((bm >> (8 * qt)) & 0xFFu) ? 1 : 0;
            sm.sweeps = 0;
            sm.last = 0;
            sm.rot = 0;
        }
    }
    {
        const float sc = pow2f(-ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            X[c] = __fmul2_rn(X[c], make_float2(sc, sc));
            Y[c] = make_float2((c == ql) ? 1.0f : 0.0f, (c == ql + 8) ? 1.0f : 0.0f);
        }
    }
    const float tol = (float)a.tol, tol2 = tol * tol;
    int done = live ? 0 : 1;
#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        St st;
        st.my_rot = 0;
        st.full = true;
        st.fmask = 0xffffffffu;
        if constexpr (U == 2) {
#pragma unroll 1
            for (int gi = 0; gi < 8; ++gi) {
                iter<0, WANT_V>(X, Y, sm, ctab, 2 * gi, lane, ql, done != 0, tol2, tol, st);
                if (gi == 7) {
                    shift_all<1, WANT_V>(X, Y);
                    break;
                }
                iter<1, WANT_V, 2>(X, Y, sm, ctab, 2 * gi + 1, lane, ql, done != 0, tol2, tol, st);
            }
        } else {  // U divides 15: the ring moves once per U iterations
#pragma unroll 1
            for (int gi = 0; gi < NIT / U; ++gi) {
                group<U, 0, WANT_V>(X, Y, sm, ctab, U * gi, lane, ql, done != 0, tol2, tol, st);
                shift_all<U, WANT_V>(X, Y);
            }
        }
        int tot = st.my_rot;  // lane ql counts pair ql of its problem
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (!done) {
            if (ql == 0) {
                sm.sweeps = sw + 1;
                sm.last = tot;
                sm.rot += tot;
            }
            if (tot == 0) done = 1;
        }
        if (__all_sync(0xffffffffu, done != 0)) break;
    }
    // ======== kernel (5) fused: sigma (float64 sums in finalize_block's order), order, U, V ========
    float* wsW = a.work + (size_t)(live ? prob : 0) * a.work_stride;
    float* wsV = wsW + N * N;
    __syncwarp();
    const float us = pow2f(sm.ex);
    bool fused;
    {
        // per half of the columns: rows l, l + 8 pre-summed in-lane (finalize_block's xor-8 level; its
        // xor-16 level adds zero rows), then a transposing xor butterfly (4, 2, 1) -> lane ql ends with
        // columns ql and ql + 8 (eight doubles live at a time instead of sixteen: no spills at 96 registers)
        const bool b2 = ql & 4, b1 = ql & 2, b0 = ql & 1;
        double colsum[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double v[8], a4[4], a2[2];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double w0 = (double)(X[8 * h + i].x * us), w1 = (double)(X[8 * h + i].y * us);
                v[i] = w0 * w0 + w1 * w1;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double keep = b2 ? v[i + 4] : v[i], send = b2 ? v[i] : v[i + 4];
                a4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const double keep = b1 ? a4[i + 2] : a4[i], send = b1 ? a4[i] : a4[i + 2];
                a2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
            }
            const double keep = b0 ? a2[1] : a2[0], send = b0 ? a2[0] : a2[1];
            colsum[h] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
        const float sg0 = (float)__dsqrt_rn(colsum[0]);  // sigma of columns ql, ql + 8, cast like the reference
        const float sg1 = (float)__dsqrt_rn(colsum[1]);
        const bool hole = !((double)sg0 >= dtiny<float>()) || !((double)sg1 >= dtiny<float>());
        const unsigned hm = __ballot_sync(0xffffffffu, hole);
        fused = ((hm >> (8 * qt)) & 0xFFu) == 0u;
        const int c0 = ql, c1 = ql + 8;
        sm.sig[c0] = sg0;
        sm.sig[c1] = sg1;
        __syncwarp();
        int r0 = 0, r1 = 0;  // stable descending ranks (finalize.cuh step 4)
#pragma unroll
        for (int c2 = 0; c2 < N; ++c2) {
            const float s2 = sm.sig[c2];
            r0 += sig_before(s2, sg0) || (c2 < c0 && sig_tie(s2, sg0));
            r1 += sig_before(s2, sg1) || (c2 < c1 && sig_tie(s2, sg1));
        }
        sm.rk[c0] = r0;
        sm.rk[c1] = r1;
        __syncwarp();
        if (live && fused) {
            const FinalOut<float> o = final_out(a, prob);
            o.S[r0] = sg0;
            o.S[r1] = sg1;
#pragma unroll
            for (int c = 0; c < N; ++c) {
                const size_t col = (size_t)sm.rk[c] * o.ldu;
                const float sc = sm.sig[c], rs = __frcp_rn(sc);
                o.U[ql + col] = div_by_sigma_f(X[c].x * us, sc, rs);
                o.U[ql + 8 + col] = div_by_sigma_f(X[c].y * us, sc, rs);
            }
            if (WANT_V && o.want_v && o.V) {
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const size_t col = (size_t)sm.rk[c] * o.ldv;
                    o.V[ql + col] = Y[c].x;
                    o.V[ql + 8 + col] = Y[c].y;
                }
            }
        }
    }
    if (live) {
        if (ql == 0) wsW[a.work_stride - 1] = fused ? 0.0f : 1.0f;  // flag for the standalone pass
        if (!fused) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsW[ql + c * N] = X[c].x * us;
                wsW[ql + 8 + c * N] = X[c].y * us;
            }
            if (WANT_V) {
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    wsV[ql + c * N] = Y[c].x;
                    wsV[ql + 8 + c * N] = Y[c].y;
                }
            }
        }
        if (ql == 0 && a.info) {
            bsvd_info inf;
            inf.converged = done;
            inf.outer_sweeps = sm.sweeps;
            inf.rotations = sm.rot;
            inf.gram_calls = 0;
            inf.update_calls = 0;
            inf.last_rotations = sm.last;
            inf.path = 1;
            inf.status = sm.bad;
            inf.kernel = a.kernel;
            a.info[prob] = inf;
        }
    }
}

// C2's 10,000 problems are 2,500 warps = 16.9 per SM: MINB keeps the register count at <= 112 so
// that 18 warps fit an SM and the launch is one wave
template <int NW, int MINB, int U>
void launch_nw(const SolveArgs<float>& a, cudaStream_t st) {
    const int per_cta = 4 * NW;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    if (a.need_v) k_reg16c<NW, MINB, U, true><<<grid, NW * 32, 0, st>>>(a);
    else k_reg16c<NW, MINB, U, false><<<grid, NW * 32, 0, st>>>(a);
}

}  // namespace reg16c

Plan plan_unblocked_reg16c(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_S && bn == 16 && bm == 16 && lda_ok) {
        (void)variant;
        p.kernel = KV_UNBLOCKED_REG16C;
        p.threads = 32;
        p.work_elems = (size_t)bm * 16 + (need_v ? 16 * 16 : 0) + 1;  // + the finalisation flag
    }
    return p;
}

int launch_unblocked_reg16c(SolveArgs<float> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    // one-warp CTAs, ring unrolled by 2 (round 1 measured the ring unrolled by 3 / 5 -- fewer register
    // moves, but longer bodies spill at the 96-register cap -- and 2-warp CTAs: all slower)
    reg16c::launch_nw<1, 18, 2>(a, st);
    if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
    return launch_finalize_flagged<float>(a, st);  // only problems the fused finalisation left over
}

}  // namespace bsvd
