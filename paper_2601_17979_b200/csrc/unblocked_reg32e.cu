// unblocked_reg32e.cu -- kernel (2), warp-specialised register-resident
// 32x32 FP64 path (the north-star C1 shape).
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule (src/ordering.py:32-75); numerics of
// unblocked_reg32b.cu (maintained column norms recomputed every sweep and
// after a >4x shrink, two-FMA update with c - 1 carried separately,
// half-angle rotation parameters).
//
// Each pair of problems is owned by TWO warps of the CTA:
//
//  * the W warp holds W (lane hl: rows hl and hl + 16 of both problems' 32
//    columns, half-warp h = problem h) and runs the latency-bound part:
//    g_ji dot products, the transpose reduction, the rotation parameters,
//    the guard and the in-register update of W;
//  * the V warp holds V the same way and applies the published rotations of
//    every iteration as they appear -- pure FP64 throughput work that fills
//    the W warp's dependency stalls on the same SM sub-partition.
//
// The rotations travel through a shared-memory ring of RING iteration slots
// guarded by mbarriers (full: W -> V, empty: V -> W).  Nothing is parked in
// global memory between sweeps and there is no replay phase; W and V leave
// the registers once, at the end, for finalize.cu (sigma, U, the order).
// W warps get the higher warp ids so the scheduler's high-id-first arbitration
// favours the critical chain.
#include "kernel_args.cuh"
#include "launch.h"
#include "rotation.cuh"

namespace bsvd {
namespace r32e {

constexpr int N = 32;      // columns
constexpr int H = 16;      // column pairs per iteration
constexpr int NIT = 31;    // iterations per sweep (ring length)
constexpr int RSTR = 34;   // doubles per row of the transpose buffer (bank padding)
constexpr int RING = 4;    // rotation slots between the W and the V warp of a pair

__host__ __device__ constexpr int ring_slot(int q) {  // ring position -> register slot at t = 0
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}
__host__ __device__ constexpr int md(int a) { return ((a % NIT) + NIT) % NIT; }
__host__ __device__ constexpr int TS(int k, int u) { return k == 0 ? 0 : ring_slot(md(k - u)); }
__host__ __device__ constexpr int BS(int k, int u) { return ring_slot(md((k == 0 ? 0 : NIT - k) - u)); }

struct __align__(16) Par {
    double cm1, c;  // x <- x + (cm1 x + c y);  y <- y + (cm1 y - c x)
};

struct Slot {
    Par pub[2][H];   // rotations of one iteration [problem half][pair]
    uint32_t ctrl;   // bit 0: some rotation is not the identity; bit 1: stop
    uint32_t pad[3];
};

struct PairSmem {
    double red[N * RSTR];  // W warp: transpose buffer [row][lane]
    double nrm[2][N];      // W warp: maintained squared column norms [half][column]
    Slot ring[RING];
    uint64_t full[RING];   // W -> V: slot written (32 arrivals)
    uint64_t empty[RING];  // V -> W: slot consumed (32 arrivals)
};

constexpr uint32_t CTRL_ROT = 1u, CTRL_STOP = 2u;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <int SH>
__device__ __forceinline__ void ring_shift(double (&x)[N]) {
    if constexpr (md(SH) != 0) {
        double y[NIT];
#pragma unroll
        for (int q = 0; q < NIT; ++q) y[q] = x[ring_slot(q)];
#pragma unroll
        for (int q = 0; q < NIT; ++q) x[ring_slot(q)] = y[md(q - SH)];
    }
}

__device__ __forceinline__ void apply2(double& x, double& y, double cm1, double c) {
    const double tx = fma(c, y, x);
    const double ty = fma(-c, x, y);
    x = fma(cm1, x, tx);
    y = fma(cm1, y, ty);
}

template <int u>
__device__ __forceinline__ void rotate_all(double (&x0)[N], double (&x1)[N], const Par* pub) {
#pragma unroll
    for (int q = 0; q < H; ++q) {
        const Par pq = pub[q];
        apply2(x0[TS(q, u)], x0[BS(q, u)], pq.cm1, pq.c);
        apply2(x1[TS(q, u)], x1[BS(q, u)], pq.cm1, pq.c);
    }
}

__device__ __forceinline__ double sum16(const double* p) {  // 16 consecutive doubles, fixed tree
    const double2* r = reinterpret_cast<const double2*>(p);
    const double2 p0 = r[0], p1 = r[1], p2 = r[2], p3 = r[3], p4 = r[4], p5 = r[5], p6 = r[6], p7 = r[7];
    const double s0 = (p0.x + p0.y) + (p1.x + p1.y), s1 = (p2.x + p2.y) + (p3.x + p3.y);
    const double s2 = (p4.x + p4.y) + (p5.x + p5.y), s3 = (p6.x + p6.y) + (p7.x + p7.y);
    return (s0 + s1) + (s2 + s3);
}

__device__ __forceinline__ double xor_sign(double x, bool neg) {
    return __longlong_as_double(__double_as_longlong(x) ^ ((long long)neg << 63));
}

// Per (t, k): column ids ct, cb (reference orientation via flip): ct | cb << 8 | flip << 16.
__host__ __device__ inline uint32_t pair_code(int t, int k) {
    int qt = k - t, qb = (k == 0 ? 0 : NIT - k) - t;
    qt += qt < 0 ? NIT : 0;
    qb += qb < 0 ? NIT : 0;
    const int ct = (k == 0) ? 0 : ring_slot(qt);
    const int cb = ring_slot(qb);
    return (uint32_t)ct | ((uint32_t)cb << 8) | ((ct > cb) ? (1u << 16) : 0u);
}

// |d|, g -> s = sin(th) >= 0, c - 1, |t| (half-angle form, rotation.cuh)
__device__ __forceinline__ void rot_abs(double dabs, double g, double& s, double& cm1, double& tabs) {
    const double mx = fmax(dabs, g);
    const double sc = mx < 0x1p-500 ? 0x1p+600 : 1.0;  // exact rescale of tiny pairs
    const double dn = dabs * sc, gn = g * sc;
    const double q = fma(4.0 * gn, gn, dn * dn);  // the gen. 2 kernel's association: identical bits
    const double ir = rsqrt_cubic(q);
    const double c2 = fma(0.5 * dn, ir, 0.5);
    const double ic = rsqrt_cubic(c2);
    const double c = c2 * ic;
    s = (gn * ir) * ic;
    cm1 = -(s * s) * rcp_cubic(1.0 + c);
    tabs = s * ic;
}

struct WState {
    int my_rot;     // rotations of this lane's pair in the sweep
    bool any;       // some rotation in this sweep (either problem)
    bool full;      // this iteration recomputes the norms of some problem of the pair
    uint32_t fmask; // lanes whose problem takes the fresh norms (per half)
    uint32_t g;     // global iteration counter (ring slot / phase)
};

// ---------------------------------------------------------------- W warp --
template <int u, bool SYNC>
__device__ __forceinline__ void w_iter(double (&x0)[N], double (&x1)[N], PairSmem& sm, const uint32_t* ctab, int t,
                                       int lane, int half, int hl, bool done, double tol, double tol2, WState& st) {
    if (st.full) {
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const double a0 = x0[TS(k, u)], b0 = x0[BS(k, u)], a1 = x1[TS(k, u)], b1 = x1[BS(k, u)];
            sm.red[(2 * k) * RSTR + lane] = fma(a1, a1, a0 * a0);
            sm.red[(2 * k + 1) * RSTR + lane] = fma(b1, b1, b0 * b0);
        }
        __syncwarp();
        const double ft = sum16(sm.red + (2 * hl) * RSTR + 16 * half);
        const double fb = sum16(sm.red + (2 * hl + 1) * RSTR + 16 * half);
        const uint32_t code = ctab[t * H + hl];
        if ((st.fmask >> lane) & 1u) {
            sm.nrm[half][code & 0xff] = ft;
            sm.nrm[half][(code >> 8) & 0xff] = fb;
        }
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const double a0 = x0[TS(k, u)], b0 = x0[BS(k, u)], a1 = x1[TS(k, u)], b1 = x1[BS(k, u)];
        sm.red[k * RSTR + lane] = fma(b1, a1, b0 * a0);
    }
    const uint32_t code = ctab[t * H + hl];
    __syncwarp();
    const int ct = code & 0xff, cb = (code >> 8) & 0xff;
    const double gt = sm.nrm[half][ct], gb = sm.nrm[half][cb];
    const double g = sum16(sm.red + hl * RSTR + 16 * half);
    const double absg = fabs(g);
    // guard (F4): rotate unless |g| <= 0 or |g| < tol sqrt(gii gjj)
    const double p = gt * gb;
    bool rot = !(absg * absg < tol2 * p);
    if (absg < 0x1p-400) rot = !(absg < tol * fsqrt(p));  // g^2 could underflow
    rot = rot && !done && absg > 0.0;
    const double d = gt - gb;
    double s, cm1, tabs;
    rot_abs(fabs(d), absg, s, cm1, tabs);
    // sign of tau in slot orientation: sgn(d); for d == 0 the reference's
    // sgn(0) = +1 in (i, j) orientation
    const bool eneg = d < 0.0 || (d == 0.0 && (code >> 16) != 0);
    Par par;
    par.cm1 = rot ? cm1 : 0.0;
    par.c = rot ? xor_sign(s, (g < 0.0) != eneg) : 0.0;  // x = top slot, y = bot slot
    const double dtg = rot ? xor_sign(tabs * absg, eneg) : 0.0;
    const double nt = gt + dtg, nb = gb - dtg;
    sm.nrm[half][ct] = nt;
    sm.nrm[half][cb] = nb;
    const bool shrink = rot && (nt < 0.25 * gt || nb < 0.25 * gb);
    st.my_rot += rot ? 1 : 0;
    const unsigned mask = __ballot_sync(0xffffffffu, rot);
    {  // a >4x shrink in a problem makes that problem's next iteration recompute its norms
        const uint32_t sb = __ballot_sync(0xffffffffu, shrink);
        st.fmask = ((sb & 0xFFFFu) ? 0xFFFFu : 0u) | ((sb >> 16) ? 0xFFFF0000u : 0u);
        st.full = sb != 0u;
    }
    st.any |= mask != 0u;
    const uint32_t s_idx = st.g % RING;
    Slot& slot = sm.ring[s_idx];
    if (SYNC && st.g >= RING) mbar_wait(&sm.empty[s_idx], ((st.g / RING) - 1) & 1);
    slot.pub[half][hl] = par;
    if (lane == 0) slot.ctrl = mask ? CTRL_ROT : 0u;
    __syncwarp();
    if (SYNC) mbar_arrive(&sm.full[s_idx]);
    ++st.g;
    if (mask) rotate_all<u>(x0, x1, slot.pub[half]);
}

template <int U, bool SYNC>
__device__ __forceinline__ void w_sweep(double (&x0)[N], double (&x1)[N], PairSmem& sm, const uint32_t* ctab,
                                        int lane, int half, int hl, bool done, double tol, double tol2, WState& st) {
    constexpr int NG = (NIT + U - 1) / U;
    constexpr int R = NIT - (NG - 1) * U;  // iterations in the last group
#pragma unroll 1
    for (int gi = 0; gi < NG; ++gi) {
        const int t0 = gi * U;
        const bool last = gi == NG - 1;
        w_iter<0, SYNC>(x0, x1, sm, ctab, t0, lane, half, hl, done, tol, tol2, st);
        if constexpr (U >= 2) {
            if (R == 1 && last) { ring_shift<1>(x0); ring_shift<1>(x1); break; }
            w_iter<1 % U, SYNC>(x0, x1, sm, ctab, t0 + 1, lane, half, hl, done, tol, tol2, st);
        }
        if constexpr (U >= 3) {
            if (R == 2 && last) { ring_shift<2>(x0); ring_shift<2>(x1); break; }
            w_iter<2 % U, SYNC>(x0, x1, sm, ctab, t0 + 2, lane, half, hl, done, tol, tol2, st);
        }
        if constexpr (U >= 4) {
            if (R == 3 && last) { ring_shift<3>(x0); ring_shift<3>(x1); break; }
            w_iter<3 % U, SYNC>(x0, x1, sm, ctab, t0 + 3, lane, half, hl, done, tol, tol2, st);
        }
        ring_shift<U>(x0);
        ring_shift<U>(x1);
    }
}

// ---------------------------------------------------------------- V warp --
template <int u>
__device__ __forceinline__ void v_iter(double (&x0)[N], double (&x1)[N], PairSmem& sm, int half, uint32_t& g) {
    const uint32_t s_idx = g % RING;
    mbar_wait(&sm.full[s_idx], (g / RING) & 1);
    const Slot& slot = sm.ring[s_idx];
    if (slot.ctrl & CTRL_ROT) rotate_all<u>(x0, x1, slot.pub[half]);
    __syncwarp();
    mbar_arrive(&sm.empty[s_idx]);
    ++g;
}

template <int U>
__device__ __forceinline__ void v_sweep(double (&x0)[N], double (&x1)[N], PairSmem& sm, int half, uint32_t& g) {
    constexpr int NG = (NIT + U - 1) / U;
    constexpr int R = NIT - (NG - 1) * U;
#pragma unroll 1
    for (int gi = 0; gi < NG; ++gi) {
        const bool last = gi == NG - 1;
        v_iter<0>(x0, x1, sm, half, g);
        if constexpr (U >= 2) {
            if (R == 1 && last) { ring_shift<1>(x0); ring_shift<1>(x1); break; }
            v_iter<1 % U>(x0, x1, sm, half, g);
        }
        if constexpr (U >= 3) {
            if (R == 2 && last) { ring_shift<2>(x0); ring_shift<2>(x1); break; }
            v_iter<2 % U>(x0, x1, sm, half, g);
        }
        if constexpr (U >= 4) {
            if (R == 3 && last) { ring_shift<3>(x0); ring_shift<3>(x1); break; }
            v_iter<3 % U>(x0, x1, sm, half, g);
        }
        ring_shift<U>(x0);
        ring_shift<U>(x1);
    }
}

// NP problem pairs per CTA: warps [0, NP) are V warps, [NP, 2 NP) W warps.
template <int NP, int MINB, int UW, int UV>
__global__ void __launch_bounds__(2 * NP * 32, MINB) k_reg32e(SolveArgs<double> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool is_w = warp >= NP;
    const int pr = is_w ? warp - NP : warp;
    PairSmem& sm = reinterpret_cast<PairSmem*>(smem_raw)[pr];
    uint32_t* ctab = reinterpret_cast<uint32_t*>(smem_raw + NP * sizeof(PairSmem));
    const int half = lane >> 4, hl = lane & 15;
    const int prob = (blockIdx.x * NP + pr) * 2 + half;
    const bool live = prob < a.batch;
    const int r0 = hl, r1 = hl + 16;
    double* wsW = a.work + (size_t)(live ? prob : 0) * (size_t)a.work_stride;  // W 32x32, then V 32x32
    double* wsV = wsW + N * N;
    const bool want_v = a.need_v != 0;
    for (int e = threadIdx.x; e < NIT * H; e += 2 * NP * 32) ctab[e] = pair_code(e / H, e % H);
    if (threadIdx.x < NP * RING) {
        PairSmem& ps = reinterpret_cast<PairSmem*>(smem_raw)[threadIdx.x / RING];
        mbar_init(&ps.full[threadIdx.x % RING], 32);
        mbar_init(&ps.empty[threadIdx.x % RING], 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");  // init visible before first use
    }
    __syncthreads();

    if (!is_w) {
        // ============================ V warp ============================
        if (!want_v) return;
        double x0[N], x1[N];
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] = (c == r0) ? 1.0 : 0.0;
            x1[c] = (c == r1) ? 1.0 : 0.0;
        }
        uint32_t g = 0;
#pragma unroll 1
        for (;;) {
            mbar_wait(&sm.full[g % RING], (g / RING) & 1);  // peek at the sweep's first slot
            if (sm.ring[g % RING].ctrl & CTRL_STOP) break;
            v_sweep<UV>(x0, x1, sm, half, g);
        }
        if (live) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsV[r0 + c * N] = x0[c];
                wsV[r1 + c * N] = x1[c];
            }
        }
        return;
    }

    // ============================ W warp ============================
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
    const double tol = a.tol, tol2 = a.tol * a.tol;
    int sweeps = 0, last = 0, done = live ? 0 : 1;
    long long rot_total = 0;
    WState st;
    st.g = 0;
#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        st.my_rot = 0;
        st.any = false;
        st.full = true;  // fresh norms at the start of every sweep
        st.fmask = 0xffffffffu;
        if (want_v) w_sweep<UW, true>(x0, x1, sm, ctab, lane, half, hl, done != 0, tol, tol2, st);
        else w_sweep<UW, false>(x0, x1, sm, ctab, lane, half, hl, done != 0, tol, tol2, st);
        int tot = st.my_rot;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (!done) {
            sweeps = sw + 1;
            last = tot;
            rot_total += tot;
            if (tot == 0) done = 1;
        }
        const int partner_done = __shfl_xor_sync(0xffffffffu, done, 16);
        if (done && partner_done) break;
    }
    if (want_v) {  // release the V warp
        const uint32_t s_idx = st.g % RING;
        if (st.g >= RING) mbar_wait(&sm.empty[s_idx], ((st.g / RING) - 1) & 1);
        if (lane == 0) sm.ring[s_idx].ctrl = CTRL_STOP;
        __syncwarp();
        mbar_arrive(&sm.full[s_idx]);
    }
    if (live) {
        const double unscale = pow2(ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            wsW[r0 + c * N] = x0[c] * unscale;
            wsW[r1 + c * N] = x1[c] * unscale;
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

}  // namespace r32e

bool is_reg32e(int kv) { return kv >= KV_UNBLOCKED_REG32E && kv <= KV_UNBLOCKED_REG32E_LAST; }

static size_t r32e_smem(int np) { return np * sizeof(r32e::PairSmem) + r32e::NIT * r32e::H * 4; }

Plan plan_unblocked_reg32e(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant) {
    Plan p{};
    if (dtype == BSVD_D && bm == 32 && bn == 32 && lda_ok) {
        p.kernel = is_reg32e(variant) ? variant : KV_UNBLOCKED_REG32E;
        p.threads = 256;
        p.smem = r32e_smem(4);
        p.work_elems = 2 * 32 * 32;
        p.grid = 0;
        p.resident = 0;
        (void)need_v;
    }
    return p;
}

template <int NP, int MINB, int UW, int UV>
static int launch_r32e(SolveArgs<double> a, cudaStream_t st) {
    const int per_cta = 2 * NP;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    const size_t smem = r32e_smem(NP);
    auto k = r32e::k_reg32e<NP, MINB, UW, UV>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<grid, 2 * NP * 32, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_unblocked_reg32e(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    int rc;
    switch (p.kernel) {
        case KV_UNBLOCKED_REG32E + 1: rc = launch_r32e<6, 1, 2, 2>(a, st); break;  // 12 warps/SM, 168 regs
        case KV_UNBLOCKED_REG32E + 2: rc = launch_r32e<4, 1, 2, 4>(a, st); break;  // V unroll 4
        case KV_UNBLOCKED_REG32E + 3: rc = launch_r32e<2, 3, 2, 2>(a, st); break;  // 4-warp CTAs, 12 warps/SM
        default: rc = launch_r32e<4, 1, 2, 2>(a, st); break;                       // 8 warps/SM, 255 regs
    }
    if (rc) return rc;
    return launch_finalize_ws<double>(a, st);
}

}  // namespace bsvd
