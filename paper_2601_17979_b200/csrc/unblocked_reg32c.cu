// unblocked_reg32c.cu -- kernel (2), third-generation register-resident
// 32x32 FP64 path (the north-star C1 shape): ONE problem per warp, lane l
// holds row l, so a problem's working copy is 32 doubles per lane.
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule (src/ordering.py:32-75) and the same
// numerics as unblocked_reg32b.cu (maintained column norms recomputed at sweep
// start and after a >4x shrink, two-FMA update with c - 1 carried separately,
// half-angle rotation parameters, update fused with the next iteration's
// partial products, V by phase alternation from a per-sweep rotation log,
// finalisation fused at the end with holes flagged to k_finalize_ws).
//
// Why another layout: gen. 2 (two problems per warp, two rows per lane)
// needs 128 registers for the rows and runs two warps per SMSP, and a W
// iteration is a ~1,500-cycle dependency chain (transpose reduction, the
// rsqrt -> rsqrt -> rcp parameter chain, publish, update) that two warps
// cannot hide: the FP64 pipe sits at ~46 %.  Here the rows take 64
// registers, so three (168 regs) or four (128 regs) warps share an SMSP and
// hide each other's chains; the price is that both half-warps evaluate the
// same 16 rotations (the parameter chain is per problem, not per two).
// Each warp is independent (no CTA barrier after set-up): a converged problem
// leaves at once instead of idling beside its partner.
#include "kernel_args.cuh"
#include "launch.h"
#include "ring32.cuh"

namespace bsvd {
namespace r32c {

using namespace ring32;
constexpr int LOG_ELEMS = NIT * H * 2 + 32;  // doubles per problem: rotation log (31 x 16 Par) + padding

struct WarpSmem {
    double red[2 * H * RSTR];  // transpose buffer: rows 0..15 g partials (rows 0..31: norms, finalisation)
    Par pub[H];                // this iteration's rotations
    Par stage[2][H];           // V replay: double-buffered log rows
    double nrm[N];             // maintained squared column norms
};

struct St {
    int my_rot;       // rotations of pair (lane & 15) in this sweep, counted by lanes < 16
    uint32_t itbits;  // bit t: some pair rotated in iteration t
    bool full;        // this iteration reads fresh norms
};

// g_ji partial of pair k at offset u from this lane's row
template <int u>
__device__ __forceinline__ void cross(const double (&x)[N], double* red, int lane, int k) {
    red[k * RSTR + lane] = x[BS(k, u)] * x[TS(k, u)];
}

template <int u, int PD>
__device__ __forceinline__ void w_iter(double (&x)[N], WarpSmem& sm, const uint32_t* ctab, int t, int lane,
                                       double tol, double tol2, Par* logl, St& st) {
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
    bool rot = !(absg * absg < tol2 * p);
    if (absg < 0x1p-400 && absg > 0.0) rot = !(absg < tol * fsqrt(p));
    rot = rot && absg > 0.0;
    const double d = gt - gb;
    double s, cm1, tabs;
    rot_abs(fabs(d), absg, s, cm1, tabs);
    const bool eneg = d < 0.0 || (d == 0.0 && flip);  // sgn(0) = +1 in (i, j) orientation
    Par par;
    par.cm1 = rot ? cm1 : 0.0;
    par.c = rot ? xor_sign(s, (g < 0.0) != eneg) : 0.0;  // x = top slot, y = bottom slot
    const double dtg = rot ? xor_sign(tabs * absg, eneg) : 0.0;
    const double nt = gt + dtg, nb = gb - dtg;
    const bool shrink = rot && (nt < 0.25 * gt || nb < 0.25 * gb);
    __syncwarp();  // every lane has read red[] and nrm[]
    if (lane < H) {
        sm.pub[k] = par;
        if (logl) logl[t * H] = par;
        sm.nrm[ct] = nt;
        sm.nrm[cb] = nb;
        st.my_rot += rot ? 1 : 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, rot);
    st.full = __ballot_sync(0xffffffffu, shrink) != 0u;
    st.itbits |= (mask != 0u ? 1u : 0u) << t;
    __syncwarp();
    constexpr int un = u + 1;  // offset of iteration t + 1 (pre-shift naming)
    if (mask) {
        Par pq[PD];  // rotations PD ahead
#pragma unroll
        for (int q = 0; q < PD; ++q) pq[q] = sm.pub[q];
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const Par cur = pq[q % PD];
            if (q + PD < H) pq[q % PD] = sm.pub[q + PD];
            apply2(x[TS(q, u)], x[BS(q, u)], cur.cm1, cur.c);
            if (q >= 1) cross<un>(x, sm.red, lane, q - 1);  // next pair q-1 needs this iteration's pairs q-2, q
        }
        cross<un>(x, sm.red, lane, H - 1);
    } else {
#pragma unroll
        for (int q = 0; q < H; ++q) cross<un>(x, sm.red, lane, q);
    }
}

template <int u, int PD>
__device__ __forceinline__ void v_iter(double (&x)[N], WarpSmem& sm, int t, int lane, const Par* logl,
                                       uint32_t itbits) {
    if (t + 1 < NIT && lane < H) cp_async16(&sm.stage[(t + 1) & 1][lane], logl + (t + 1) * H);
    cp_commit();
    cp_wait<1>();
    __syncwarp();
    if ((itbits >> t) & 1u) {
        const Par* stp = sm.stage[t & 1];
        Par pr[PD];
#pragma unroll
        for (int q = 0; q < PD; ++q) pr[q] = stp[q];
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const Par pq = pr[q % PD];
            if (q + PD < H) pr[q % PD] = stp[q + PD];
            apply2(x[TS(q, u)], x[BS(q, u)], pq.cm1, pq.c);
        }
    }
    __syncwarp();
}

template <int PD>
__device__ __forceinline__ void w_sweep(double (&x)[N], WarpSmem& sm, const uint32_t* ctab, int lane, double tol,
                                        double tol2, Par* logl, St& st) {
#pragma unroll
    for (int k = 0; k < H; ++k) cross<0>(x, sm.red, lane, k);  // first iteration; st.full set by the caller
#pragma unroll 1
    for (int gi = 0; gi < 16; ++gi) {
        const int t0 = 2 * gi;
        w_iter<0, PD>(x, sm, ctab, t0, lane, tol, tol2, logl, st);
        if (gi == 15) {
            ring_shift<1>(x);
            break;
        }
        w_iter<1, PD>(x, sm, ctab, t0 + 1, lane, tol, tol2, logl, st);
        ring_shift<2>(x);
    }
}

template <int PD>
__device__ __forceinline__ void v_sweep(double (&x)[N], WarpSmem& sm, int lane, const Par* logl, uint32_t itbits) {
#pragma unroll 1
    for (int gi = 0; gi < 16; ++gi) {
        const int t0 = 2 * gi;
        v_iter<0, PD>(x, sm, t0, lane, logl, itbits);
        if (gi == 15) {
            ring_shift<1>(x);
            break;
        }
        v_iter<1, PD>(x, sm, t0 + 1, lane, logl, itbits);
        ring_shift<2>(x);
    }
}

template <int NW, int MINB, int PD>
__global__ void __launch_bounds__(NW * 32, MINB) k_reg32c(SolveArgs<double> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
    uint32_t* ctab = reinterpret_cast<uint32_t*>(smem_raw + NW * sizeof(WarpSmem));
    for (int e = threadIdx.x; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    __syncthreads();
    const int prob = blockIdx.x * NW + warp;
    if (prob >= a.batch) return;  // warps are independent from here on
    if (a.reserved_stagger > 0) __nanosleep((unsigned)((warp & 3) * a.reserved_stagger));  // experiment
    const size_t pstride = (size_t)a.work_stride;
    double* wsW = a.work + (size_t)prob * pstride;  // W 32x32 (parking), V 32x32, then the log
    double* wsV = wsW + N * N;
    const bool want_v = a.need_v != 0;
    Par* logl = want_v ? reinterpret_cast<Par*>(wsW + 2 * N * N) + (lane & 15) : nullptr;
    Par* logw = (want_v && lane < H) ? logl : nullptr;

    double x[N];
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
    bool v_started = false;

#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        St st;
        st.my_rot = 0;
        st.itbits = 0;
        st.full = true;
        w_sweep<PD>(x, sm, ctab, lane, tol, tol2, logw, st);
        int tot = st.my_rot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        sweeps = sw + 1;
        last = tot;
        rot_total += tot;
        if (tot == 0) done = 1;
        // ---- V phase: replay the sweep's rotations onto V ----
        if (want_v && st.itbits) {
#pragma unroll
            for (int c = 0; c < N; ++c) wsW[lane + c * N] = x[c];  // park W
            if (v_started) {
#pragma unroll
                for (int c = 0; c < N; ++c) x[c] = wsV[lane + c * N];
            } else {
#pragma unroll
                for (int c = 0; c < N; ++c) x[c] = (c == lane) ? 1.0 : 0.0;
                v_started = true;
            }
            __syncwarp();  // the log rows written by lanes < 16 are visible to the warp
            if (lane < H) cp_async16(&sm.stage[0][lane], logl);
            cp_commit();
            v_sweep<PD>(x, sm, lane, logl, st.itbits);
            cp_wait<0>();
#pragma unroll
            for (int c = 0; c < N; ++c) wsV[lane + c * N] = x[c];  // park V
            __syncwarp();
#pragma unroll
            for (int c = 0; c < N; ++c) x[c] = wsW[lane + c * N];
        }
        if (done) break;
    }
    // ======== kernel (5) fused: sigma, order, U = W / sigma, V permuted (holes -> standalone pass) ========
    double* flagp = wsW + pstride - 1;
    const double unscale = pow2(ex);
    bool fused;
    {
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
        double2* sr = reinterpret_cast<double2*>(sm.stage);  // [32] (scaled sigma, reciprocal)
        int* rk = reinterpret_cast<int*>(sm.nrm);            // [32] rank by column
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
            if (o.want_v && o.V) {
                if (v_started) {
#pragma unroll
                    for (int c = 0; c < N; ++c) x[c] = wsV[lane + c * N];  // all loads before the stores
                } else {
#pragma unroll
                    for (int c = 0; c < N; ++c) x[c] = (c == lane) ? 1.0 : 0.0;
                }
#pragma unroll
                for (int c = 0; c < N; ++c) o.V[lane + (size_t)rk[c] * o.ldv] = x[c];
            }
        }
        if (lane == 0) *flagp = fused ? 0.0 : 1.0;
    }
    if (!fused) {
#pragma unroll
        for (int c = 0; c < N; ++c) wsW[lane + c * N] = x[c] * unscale;
        if (want_v && !v_started) {
#pragma unroll
            for (int c = 0; c < N; ++c) wsV[lane + c * N] = (c == lane) ? 1.0 : 0.0;
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

}  // namespace r32c

bool is_reg32c(int kv) { return kv >= KV_UNBLOCKED_REG32C && kv <= KV_UNBLOCKED_REG32C_LAST; }

Plan plan_unblocked_reg32c(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_D && bm == 32 && bn == 32 && lda_ok) {
        p.kernel = is_reg32c(variant) ? variant : KV_UNBLOCKED_REG32C;
        p.threads = 128;
        p.smem = r32c::smem_bytes(4);
        p.work_elems = 2 * 32 * 32 + r32c::LOG_ELEMS;
        p.grid = 0;
        p.resident = 0;
        (void)need_v;
    }
    return p;
}

template <int NW, int MINB, int PD>
static int launch_r32c(SolveArgs<double> a, cudaStream_t st) {
    const int grid = (a.batch + NW - 1) / NW;
    const size_t smem = r32c::smem_bytes(NW);
    auto k = r32c::k_reg32c<NW, MINB, PD>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<grid, NW * 32, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_unblocked_reg32c(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    int rc;
    switch (p.kernel - KV_UNBLOCKED_REG32C) {
        case 1: rc = launch_r32c<4, 3, 8>(a, st); break;   // 168 regs, 12 warps/SM
        case 2: rc = launch_r32c<4, 4, 2>(a, st); break;   // 128 regs, depth 2
        case 3: rc = launch_r32c<4, 3, 16>(a, st); break;  // 168 regs, all rotations ahead
        default: rc = launch_r32c<4, 4, 4>(a, st); break;  // 128 regs, 16 warps/SM
    }
    if (rc) return rc;
    return launch_finalize_flagged<double>(a, st);  // only problems the fused finalisation left over
}

}  // namespace bsvd
