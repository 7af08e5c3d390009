// unblocked_reg32f.cu -- kernel (2), fourth-generation register-resident
// 32x32 FP64 path (the north-star C1 shape): ONE problem per warp, lane l
// holds row l of W AND row l of V, both in registers for the whole solve.
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule (src/ordering.py:32-75) and the same
// per-pair arithmetic as unblocked_reg32c.cu (maintained column norms
// recomputed at sweep start and after a >4x shrink, guard |g| >= k u
// sqrt(g_ii g_jj), half-angle rotation parameters, two-FMA update with c - 1
// carried separately, update fused with the next iteration's partial dot
// products, finalisation fused at the end).
//
// What changes against gen. 2 (unblocked_reg32b.cu) and gen. 3 (reg32c):
//  * No V phase.  Gen. 2/3 rotate W for a whole sweep, park W in the
//    workspace, load V and replay a rotation log onto it: 16 KB of L2 traffic
//    per problem and sweep (the 2.5x DRAM write-back of the C1 profile) and a
//    second, chain-free but separate phase.  Here V's row rides in the same
//    lane (64 more registers), so the workspace is touched only by the rare
//    hole fallback.
//  * V lags W by one iteration.  The V rotations of iteration t - 1 are
//    issued inside iteration t's reduction -> guard -> rotation-parameter
//    chain (same basic block: the compiler interleaves 64 independent DFMAs
//    into a ~400-cycle dependency chain), so the warp's own instruction
//    stream hides most of its chain; the last iteration of a sweep is
//    flushed at the sweep end.  Parameters are double-buffered in shared
//    memory by iteration parity.
//  * Optional per-pair skip (SKIP): a pair the guard does not rotate is a
//    warp-uniform branch here (one problem per warp), so its 4 W FMAs per
//    lane are not issued.
// One problem per warp keeps every warp independent (no CTA barrier after
// set-up): a converged problem's warp leaves at once.
#include "kernel_args.cuh"
#include "launch.h"
#include "ring32.cuh"

namespace bsvd {
namespace r32f {

using namespace ring32;

struct WarpSmem {
    double red[2 * H * RSTR];  // transpose buffer: rows 0..15 g partials (rows 0..31: norms, finalisation)
    Par pub[2][H];             // rotations of the iterations of parity 0 / 1
    double nrm[N];             // maintained squared column norms
};

struct St {
    int my_rot;  // rotations of pair (lane & 15) in this sweep, counted by lanes < 16
    bool full;   // this iteration reads fresh norms
};

template <int u>
__device__ __forceinline__ void cross(const double (&x)[N], double* red, int lane, int k) {
    red[k * RSTR + lane] = x[BS(k, u)] * x[TS(k, u)];
}

// V rotations of the iteration at offset u (register naming of the current group) from pub
template <int u>
__device__ __forceinline__ void v_apply(double (&v)[N], const Par* pub) {
#pragma unroll
    for (int q = 0; q < H; ++q) {
        const Par p = pub[q];
        apply2(v[TS(q, u)], v[BS(q, u)], p.cm1, p.c);
    }
}

// rotation parameters without a data-dependent branch: the rare rescale for pairs of columns
// below 2^-500 is an exact power-of-two factor chosen by a select
__device__ __forceinline__ void rot_abs_sel(double dabs, double g, double& s, double& cm1, double& tabs) {
    const double sc = fmax(dabs, g) < 0x1p-500 ? 0x1p+600 : 1.0;
    rot_abs_core(dabs * sc, g * sc, s, cm1, tabs);
}

template <int u, bool WANTV, bool SKIP>
__device__ __forceinline__ void w_iter(double (&x)[N], double (&v)[N], WarpSmem& sm, const uint32_t* ctab, int t,
                                       int lane, double tol, double tol2, St& st) {
    const int k = lane & 15, half = lane >> 4;
    const uint32_t code = ctab[t * H + k];
    __syncwarp();
    const int ct = code & 0xff, cb = (code >> 8) & 0xff;
    const bool flip = (code >> 16) != 0;
    const double g = sum32(sm.red, k, half);
    double gt, gb;
    if (st.full) {  // fresh squared norms through the same buffer (sweep start, after a >4x shrink)
        __syncwarp();
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const double a = x[TS(q, u)], b = x[BS(q, u)];
            sm.red[q * RSTR + lane] = a * a;
            sm.red[(H + q) * RSTR + lane] = b * b;
        }
        __syncwarp();
        gt = sum32(sm.red, k, half);
        gb = sum32(sm.red, H + k, half);
    } else {
        gt = sm.nrm[ct];
        gb = sm.nrm[cb];
    }
    const double absg = fabs(g);
    // guard (F4): rotate unless |g| <= 0 or |g| < tol sqrt(gii gjj); squared comparison,
    // exact-sqrt fallback where g^2 could underflow
    const double p = gt * gb;
    const bool rsq = !(absg * absg < tol2 * p);
    const bool rex = !(absg < tol * fsqrt(p));
    const bool rot = (absg < 0x1p-400 ? rex : rsq) && absg > 0.0;
    const double d = gt - gb;
    double s, cm1, tabs;
    rot_abs_sel(fabs(d), absg, s, cm1, tabs);
    // V rotations of the previous iteration (offset u - 1; identity at a sweep start), issued into the
    // parameter chain above
    if constexpr (WANTV) v_apply<u - 1>(v, sm.pub[u ^ 1]);
    const bool eneg = d < 0.0 || (d == 0.0 && flip);  // sgn(0) = +1 in (i, j) orientation
    Par par;
    par.cm1 = rot ? cm1 : 0.0;
    par.c = rot ? xor_sign(s, (g < 0.0) != eneg) : 0.0;  // x = top slot, y = bottom slot
    const double dtg = rot ? xor_sign(tabs * absg, eneg) : 0.0;
    const double nt = gt + dtg, nb = gb - dtg;
    const bool shrink = rot && (nt < 0.25 * gt || nb < 0.25 * gb);
    __syncwarp();  // every lane has read red[], nrm[] and pub[u ^ 1]
    if (lane < H) {
        sm.pub[u][k] = par;
        sm.nrm[ct] = nt;
        sm.nrm[cb] = nb;
        st.my_rot += rot ? 1 : 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, rot) & 0xFFFFu;
    st.full = __ballot_sync(0xffffffffu, shrink) != 0u;
    __syncwarp();
    constexpr int un = u + 1;  // offset of iteration t + 1 (pre-shift naming)
    if (mask) {
#pragma unroll
        for (int q = 0; q < H; ++q) {
            if (!SKIP || ((mask >> q) & 1u)) {
                const Par cur = sm.pub[u][q];
                apply2(x[TS(q, u)], x[BS(q, u)], cur.cm1, cur.c);
            }
            if (q >= 1) cross<un>(x, sm.red, lane, q - 1);  // next pair q-1 needs this iteration's pairs q-2, q
        }
        cross<un>(x, sm.red, lane, H - 1);
    } else {
#pragma unroll
        for (int q = 0; q < H; ++q) cross<un>(x, sm.red, lane, q);
    }
}

template <bool WANTV, bool SKIP>
__device__ __forceinline__ void w_sweep(double (&x)[N], double (&v)[N], WarpSmem& sm, const uint32_t* ctab,
                                        int lane, double tol, double tol2, St& st) {
    if (WANTV && lane < H) sm.pub[1][lane] = Par{0.0, 0.0};  // "iteration -1": identity (exact no-op)
#pragma unroll
    for (int k = 0; k < H; ++k) cross<0>(x, sm.red, lane, k);  // first iteration; st.full set by the caller
#pragma unroll 1
    for (int gi = 0; gi < 16; ++gi) {
        const int t0 = 2 * gi;
        w_iter<0, WANTV, SKIP>(x, v, sm, ctab, t0, lane, tol, tol2, st);
        if (gi == 15) {
            ring_shift<1>(x);
            if constexpr (WANTV) ring_shift<1>(v);
            break;
        }
        w_iter<1, WANTV, SKIP>(x, v, sm, ctab, t0 + 1, lane, tol, tol2, st);
        ring_shift<2>(x);
        if constexpr (WANTV) ring_shift<2>(v);
    }
    if constexpr (WANTV) {  // flush: V rotations of iteration 30 (offset 0, ring moved by one since)
        __syncwarp();
        v_apply<-1>(v, sm.pub[0]);
    }
}

template <int NW, int MINB, bool WANTV, bool SKIP>
__global__ void __launch_bounds__(NW * 32, MINB) k_reg32f(SolveArgs<double> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
    uint32_t* ctab = reinterpret_cast<uint32_t*>(smem_raw + NW * sizeof(WarpSmem));
    for (int e = threadIdx.x; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    __syncthreads();
    const int prob = blockIdx.x * NW + warp;
    if (prob >= a.batch) return;  // warps are independent from here on
    const size_t pstride = (size_t)a.work_stride;
    double* wsW = a.work + (size_t)prob * pstride;  // hole fallback only: W 32x32, V 32x32, flag
    double* wsV = wsW + N * N;

    double x[N], v[N];
    int bad = 0;
    double amax = 0.0;
    {
        const double* Ap = a.A + (size_t)prob * a.strideA;  // plan requires lda == 32
#pragma unroll
        for (int c = 0; c < N; ++c) x[c] = Ap[lane + c * N];
#pragma unroll
        for (int c = 0; c < N; ++c) {
            bad |= !isfinite(x[c]);
            amax = fmax(amax, fabs(x[c]));
        }
    }
#pragma unroll
    for (int c = 0; c < N; ++c) v[c] = (c == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int ex = prescale_exponent(amax);
    {
        const double scale = pow2(-ex);
#pragma unroll
        for (int c = 0; c < N; ++c) x[c] *= scale;
    }
    const double tol = a.tol, tol2 = a.tol * a.tol;
    int sweeps = 0, last = 0, done = 0;
    long long rot_total = 0;

#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        St st;
        st.my_rot = 0;
        st.full = true;
        w_sweep<WANTV, SKIP>(x, v, sm, ctab, lane, tol, tol2, st);
        int tot = st.my_rot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        sweeps = sw + 1;
        last = tot;
        rot_total += tot;
        if (tot == 0) {
            done = 1;
            break;
        }
    }
    // ======== kernel (5) fused: sigma, order, U = W / sigma, V permuted (holes -> standalone pass) ========
    double* flagp = wsW + pstride - 1;
    const double unscale = pow2(ex);
    bool fused;
    {
        __syncwarp();
#pragma unroll
        for (int c = 0; c < N; ++c) sm.red[c * RSTR + lane] = __dmul_rn(x[c], x[c]);
        __syncwarp();
        // lane c: column c; sum in finalize_block's xor-butterfly order (rows (i, i + 16) first)
        double pp[H];
#pragma unroll
        for (int i = 0; i < H; ++i) pp[i] = __dadd_rn(sm.red[lane * RSTR + i], sm.red[lane * RSTR + i + H]);
        const double ss = __dsqrt_rn(sum16_butterfly(pp));  // sigma of the scaled W (exact power-of-two scale)
        const double sg = ss * unscale;
        const bool tiny = !(sg >= dtiny<double>() && ss >= 0x1p-480 && ss <= 0x1p+960);  // as unblocked_reg32b.cu
        fused = __ballot_sync(0xffffffffu, tiny) == 0u;
        __syncwarp();
        double2* sr = reinterpret_cast<double2*>(sm.pub);  // [32] (scaled sigma, reciprocal)
        int* rk = reinterpret_cast<int*>(sm.nrm);          // [32] rank by column
        sr[lane] = make_double2(ss, rcp_refined(ss));
        __syncwarp();
        int r = 0;  // stable descending rank (finalize.cuh step 4)
#pragma unroll 8
        for (int c2 = 0; c2 < N; ++c2) {
            const double s2 = sr[c2].x;
            r += sig_before(s2, ss) || (c2 < lane && sig_tie(s2, ss));
        }
        rk[lane] = r;
        __syncwarp();
        if (fused) {
            const FinalOut<double> o = final_out(a, prob);
            o.S[r] = sg;
            double* u = o.U + lane;
#pragma unroll
            for (int c = 0; c < N; ++c) {  // U = W / sigma: reciprocal, then one residual correction
                const int rc = rk[c];
                const double2 t = sr[c];
                u[(size_t)rc * o.ldu] = div_by_sigma(x[c], t.x, t.y);
            }
            if (WANTV && o.want_v && o.V) {
#pragma unroll
                for (int c = 0; c < N; ++c) o.V[lane + (size_t)rk[c] * o.ldv] = v[c];
            }
        }
        if (lane == 0) *flagp = fused ? 0.0 : 1.0;
    }
    if (!fused) {
#pragma unroll
        for (int c = 0; c < N; ++c) wsW[lane + c * N] = x[c] * unscale;
        if (WANTV) {
#pragma unroll
            for (int c = 0; c < N; ++c) wsV[lane + c * N] = v[c];
        }
    }
    const unsigned badm = __ballot_sync(0xffffffffu, bad != 0);
    if (lane == 0 && a.info) {
        bsvd_info inf;
        inf.converged = done;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = 0;
        inf.update_calls = 0;
        inf.last_rotations = last;
        inf.path = 1;
        inf.status = badm ? 1 : 0;
        inf.kernel = a.kernel;
        a.info[prob] = inf;
    }
}

inline size_t smem_bytes(int nw) { return (size_t)nw * sizeof(WarpSmem) + NIT * H * 4; }

}  // namespace r32f

bool is_reg32f(int kv) { return kv >= KV_UNBLOCKED_REG32F && kv <= KV_UNBLOCKED_REG32F_LAST; }

Plan plan_unblocked_reg32f(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_D && bm == 32 && bn == 32 && lda_ok) {
        p.kernel = is_reg32f(variant) ? variant : KV_UNBLOCKED_REG32F;
        p.threads = 128;
        p.smem = r32f::smem_bytes(4);
        p.work_elems = 2 * 32 * 32 + 2;  // W, V for the hole fallback; flag in the last element
        p.grid = 0;
        p.resident = 0;
        (void)need_v;
    }
    return p;
}

template <int NW, int MINB, bool SKIP>
static int launch_r32f(SolveArgs<double> a, cudaStream_t st) {
    const int grid = (a.batch + NW - 1) / NW;
    const size_t smem = r32f::smem_bytes(NW);
    auto k = a.need_v ? r32f::k_reg32f<NW, MINB, true, SKIP> : r32f::k_reg32f<NW, MINB, false, SKIP>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<grid, NW * 32, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_unblocked_reg32f(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    int rc;
    switch (p.kernel - KV_UNBLOCKED_REG32F) {
        case 1: rc = launch_r32f<4, 2, true>(a, st); break;   // per-pair skip of unrotated W pairs
        case 2: rc = launch_r32f<4, 3, false>(a, st); break;  // 168-register cap, 12 warps/SM
        case 3: rc = launch_r32f<2, 4, false>(a, st); break;  // 2-warp CTAs
        default: rc = launch_r32f<4, 2, false>(a, st); break; // 255 registers, 8 warps/SM
    }
    if (rc) return rc;
    return launch_finalize_flagged<double>(a, st);  // only problems the fused finalisation left over
}

}  // namespace bsvd
