// unblocked_reg16b.cu -- kernel (2), second-generation register-resident
// 16x16 FP32 path (BASELINE config C2).
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule for n = 16 (15 iterations x 8 pairs per
// sweep, src/ordering.py:32-75), per-problem exit after the first quiet sweep.
//
// Mapping: a warp owns TWO problems, half-warp h owns problem h and lane l of
// the half holds row l of W and row l of V (16 + 16 floats), so 5,000 warps
// carry C2's 10,000 problems at ~30 warps per SM.  The gen. 1 kernel
// (unblocked_reg16.cu: four problems per warp, two rows per lane, three dot
// products per pair, ring moved every iteration, rotations broadcast by
// shuffles) is a one-wave launch whose time is one warp's dependency chain;
// here each warp carries half the rows and the chain is shortened the way
// unblocked_reg32b.cu does it for FP64:
//  * tournament ring unrolled by 2 (compile-time register slots, one ring
//    move per two iterations);
//  * maintained column norms (one fresh dot product g_ji per pair;
//    norms recomputed at sweep start and after a >4x shrink);
//  * transposing xor-butterfly reduction of the 8 g_ji partials over the 16
//    lanes (8 shuffles), rotations published through shared memory;
//  * half-angle rotation parameters on MUFU seeds with one Newton step each,
//    two-FMA update with c - 1 carried separately (F5).
// Parameters and updates run in float32 like gen. 1 (the reference forms them
// in float64, F6; measured accuracy in DESIGN.md).  Raw W and V go to the
// workspace and finalize.cu (sigma in float64) completes the factorisation.
#include "kernel_args.cuh"
#include "launch.h"
#include "ring16.cuh"

namespace bsvd {
namespace reg16b {

constexpr int NW = 4;    // warps per CTA (8 problems)
using namespace ring16;

struct __align__(16) WarpSmem {
    float2 pub[2][H];   // this iteration's rotations (cm1, c) [half][pair]
    float nrm[2][N];    // maintained squared column norms [half][column]
    float sig[2][N];    // finalisation: sigma by column
    int rk[2][N];       // finalisation: rank by column
};

// Transposing butterfly over the 16 lanes of a half: v[0..NV) per lane -> lane l ends with the
// half's total of value index vidx(l) = (l >> 1) (NV = 8) -- 4 + 2 + 1 + 1 shuffles.
__device__ __forceinline__ float reduce8(float (&v)[8], int hl) {
    const bool b3 = hl & 8, b2 = hl & 4, b1 = hl & 2;
    float a4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float keep = b3 ? v[i + 4] : v[i], send = b3 ? v[i] : v[i + 4];
        a4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float a2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float keep = b2 ? a4[i + 2] : a4[i], send = b2 ? a4[i] : a4[i + 2];
        a2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const float keep = b1 ? a2[1] : a2[0], send = b1 ? a2[0] : a2[1];
    const float a1 = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    return a1 + __shfl_xor_sync(0xffffffffu, a1, 1);
}

struct St {
    int my_rot;
    bool full;       // some lane of the warp takes fresh norms this iteration
    uint32_t fmask;  // lanes whose problem takes them (per half: a problem's bits never depend on its partner)
};

template <int u, bool WANT_V>
__device__ __forceinline__ void iter(float (&x)[N], float (&y)[N], WarpSmem& sm, const uint32_t* ctab, int t,
                                     int lane, int half, int hl, bool done, float tol2, float tol, St& st) {
    const int k = hl >> 1;  // pair this lane reduces / evaluates (two lanes per pair)
    float v[8];
#pragma unroll
    for (int q = 0; q < H; ++q) v[q] = x[BS(q, u)] * x[TS(q, u)];
    const float g = reduce8(v, hl);
    const uint32_t code = ctab[t * H + k];
    const int ct = code & 0xff, cb = (code >> 8) & 0xff;
    const bool flip = (code >> 16) != 0;
    float gt = sm.nrm[half][ct], gb = sm.nrm[half][cb];
    if (st.full) {
        float a[8], b[8];
#pragma unroll
        for (int q = 0; q < H; ++q) {
            a[q] = x[TS(q, u)] * x[TS(q, u)];
            b[q] = x[BS(q, u)] * x[BS(q, u)];
        }
        const float ft = reduce8(a, hl), fb = reduce8(b, hl);
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
    __syncwarp();  // every lane has read nrm[]
    if ((hl & 1) == 0) {
        sm.pub[half][k] = make_float2(cm1, c);
        sm.nrm[half][ct] = nt;
        sm.nrm[half][cb] = nb;
        st.my_rot += rot ? 1 : 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, rot);
    {
        const uint32_t sb = __ballot_sync(0xffffffffu, shrink);
        st.fmask = ((sb & 0xFFFFu) ? 0xFFFFu : 0u) | ((sb >> 16) ? 0xFFFF0000u : 0u);
        st.full = sb != 0u;
    }
    __syncwarp();
    if (mask) {
        const float4* pp = reinterpret_cast<const float4*>(sm.pub[half]);
        float4 pr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pr[i] = pp[i];
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const float pc = (q & 1) ? pr[q >> 1].z : pr[q >> 1].x;
            const float pcc = (q & 1) ? pr[q >> 1].w : pr[q >> 1].y;
            apply2(x[TS(q, u)], x[BS(q, u)], pc, pcc);
            if (WANT_V) apply2(y[TS(q, u)], y[BS(q, u)], pc, pcc);
        }
    }
}

template <bool WANT_V, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) k_reg16b(SolveArgs<float> a) {
    __shared__ WarpSmem wsm[NW];
    __shared__ uint32_t ctab[NIT * H];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = lane >> 4, hl = lane & 15;
    for (int e = threadIdx.x; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    __syncthreads();
    WarpSmem& sm = wsm[warp];
    const int prob = (blockIdx.x * NW + warp) * 2 + half;
    const bool live = prob < a.batch;
    float x[N], y[N];
    int bad = 0;
    float amax = 0.0f;
    {
        const float* Ap = a.A + (size_t)(live ? prob : 0) * a.strideA;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x[c] = live ? Ap[hl + (size_t)c * a.lda] : 0.0f;
            bad |= !isfinite(x[c]);
            amax = fmaxf(amax, fabsf(x[c]));
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    int ex = ((__float_as_int(amax) >> 23) & 0xff) - 126;
    if (!(amax > 0.0f) || !isfinite(amax)) ex = 0;
    ex = max(-100, min(100, ex));
    {
        const float sc = pow2f(-ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x[c] *= sc;
            y[c] = (c == hl) ? 1.0f : 0.0f;
        }
    }
    const float tol = (float)a.tol, tol2 = tol * tol;
    int sweeps = 0, last = 0, done = live ? 0 : 1;
    long long rot_total = 0;
#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        St st;
        st.my_rot = 0;
        st.full = true;
        st.fmask = 0xffffffffu;
#pragma unroll 1
        for (int gi = 0; gi < 8; ++gi) {
            iter<0, WANT_V>(x, y, sm, ctab, 2 * gi, lane, half, hl, done != 0, tol2, tol, st);
            if (gi == 7) {
                ring_shift<1>(x);
                if (WANT_V) ring_shift<1>(y);
                break;
            }
            iter<1, WANT_V>(x, y, sm, ctab, 2 * gi + 1, lane, half, hl, done != 0, tol2, tol, st);
            ring_shift<2>(x);
            if (WANT_V) ring_shift<2>(y);
        }
        int tot = st.my_rot;  // even lanes of the half count the half's 8 pairs
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (!done) {
            sweeps = sw + 1;
            last = tot;
            rot_total += tot;
            if (tot == 0) done = 1;
        }
        if (__all_sync(0xffffffffu, done != 0)) break;
    }
    // ======== kernel (5) fused: sigma (float64 sums in finalize_block's order), order, U, V ========
    float* wsW = a.work + (size_t)(live ? prob : 0) * a.work_stride;
    float* wsV = wsW + N * N;
    const float us = pow2f(ex);
    bool fused;
    {
        // lane hl ends with column hl's sum: transposing xor butterfly (8, 4, 2, 1) = the tree of
        // finalize_block's xor reduction over the rows (rows 16..31 of that warp are zero)
        double v[N];
#pragma unroll
        for (int c = 0; c < N; ++c) {
            const double w = (double)(x[c] * us);
            v[c] = w * w;
        }
        const bool b3 = hl & 8, b2 = hl & 4, b1 = hl & 2, b0 = hl & 1;
        double a8[8], a4[4], a2[2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double keep = b3 ? v[i + 8] : v[i], send = b3 ? v[i] : v[i + 8];
            a8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double keep = b2 ? a8[i + 4] : a8[i], send = b2 ? a8[i] : a8[i + 4];
            a4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double keep = b1 ? a4[i + 2] : a4[i], send = b1 ? a4[i] : a4[i + 2];
            a2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        const double keep = b0 ? a2[1] : a2[0], send = b0 ? a2[0] : a2[1];
        const double tot = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        const float sg = (float)__dsqrt_rn(tot);  // sigma of column hl, cast like the reference
        const bool hole = !((double)sg >= dtiny<float>());
        const unsigned hm = __ballot_sync(0xffffffffu, hole);
        fused = ((hm >> (16 * half)) & 0xFFFFu) == 0u;
        sm.sig[half][hl] = sg;
        __syncwarp();
        int r = 0;  // stable descending rank (finalize.cuh step 4)
#pragma unroll
        for (int c2 = 0; c2 < N; ++c2) {
            const float s2 = sm.sig[half][c2];
            r += sig_before(s2, sg) || (c2 < hl && sig_tie(s2, sg));
        }
        sm.rk[half][hl] = r;
        __syncwarp();
        if (live && fused) {
            const FinalOut<float> o = final_out(a, prob);
            o.S[r] = sg;
#pragma unroll
            for (int c = 0; c < N; ++c) {
                const float sc = sm.sig[half][c];
                o.U[hl + (size_t)sm.rk[half][c] * o.ldu] = div_by_sigma_f(x[c] * us, sc, __frcp_rn(sc));
            }
            if (WANT_V && o.want_v && o.V) {
#pragma unroll
                for (int c = 0; c < N; ++c) o.V[hl + (size_t)sm.rk[half][c] * o.ldv] = y[c];
            }
        }
    }
    const unsigned badm = __ballot_sync(0xffffffffu, bad != 0);
    if (live) {
        if (hl == 0) wsW[a.work_stride - 1] = fused ? 0.0f : 1.0f;  // flag for the standalone pass
        if (!fused) {
#pragma unroll
            for (int c = 0; c < N; ++c) wsW[hl + c * N] = x[c] * us;
            if (WANT_V) {
#pragma unroll
                for (int c = 0; c < N; ++c) wsV[hl + c * N] = y[c];
            }
        }
        if (hl == 0 && a.info) {
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
}

}  // namespace reg16b

Plan plan_unblocked_reg16b(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_S && bn == 16 && bm == 16 && lda_ok) {
        (void)variant;
        p.kernel = KV_UNBLOCKED_REG16B;
        p.threads = reg16b::NW * 32;
        p.work_elems = (size_t)bm * 16 + (need_v ? 16 * 16 : 0) + 1;  // + the finalisation flag
    }
    return p;
}

int launch_unblocked_reg16b(SolveArgs<float> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    const int per_cta = 2 * reg16b::NW;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    // (a 56-register cap for 9 CTAs = 36 warps per SM measured slower in round 1: the V kernel spills)
    if (a.need_v) reg16b::k_reg16b<true, 1><<<grid, reg16b::NW * 32, 0, st>>>(a);
    else reg16b::k_reg16b<false, 1><<<grid, reg16b::NW * 32, 0, st>>>(a);
    if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
    return launch_finalize_flagged<float>(a, st);  // only problems the fused finalisation left over
}

}  // namespace bsvd
