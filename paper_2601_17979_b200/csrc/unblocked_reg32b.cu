// unblocked_reg32b.cu -- kernel (2), second-generation register-resident
// 32x32 FP64 path (the north-star C1 shape).
//
// Same iteration as onesided_sweeps (src/_kernels_numba.py:85-138) on the
// reference's round-robin schedule (src/ordering.py:32-75), re-organised for
// FP64-pipe throughput.  Layout is that of unblocked_reg.cu (a warp owns two
// problems; half-warp h owns problem h; lane hl holds rows hl and hl + 16 of
// all 32 columns in registers; the 16 pairs of an iteration sit in fixed
// register slots), with four changes:
//
//  * U-fold unrolled ring.  The tournament moves every column one ring
//    position per iteration.  Unrolling U iterations makes the slot of each
//    pair a compile-time function of the offset inside the group, so the
//    registers move once per group (by pi^U, one 31-cycle = 32 moves) instead
//    of once per iteration.
//  * Maintained column norms.  g_ii and g_jj are carried per column (in
//    shared memory, indexed by column id) and updated exactly like the
//    reference's two-sided eigen-update d_i += t|g|, d_j -= t|g|
//    (src/_kernels_numba.py:60-62); only g_ji is a fresh dot product.  The
//    norms are recomputed from the data in the first iteration of every sweep
//    and in any iteration that follows a >4x shrink of a norm (cancellation
//    guard, as LAPACK xGESVJ does).  A quiet sweep therefore decides
//    convergence on freshly computed norms, like the reference.
//  * Two-FMA rotation update x' = fma(cm1, x, fma(ws, y, x)): c - 1 is still
//    carried separately (F5), one FP64 instruction per flop of the update.
//  * Short-latency rotation parameters (rotation_half, rotation.cuh).
//
// Deviations are numerical only (same schedule, same guard, same rotation
// formula up to rounding); tools/acc_cmp.py and tests/test_gpu_parity.py hold
// the kernel to the parity contract.  V is replayed from a per-sweep rotation
// log exactly as in unblocked_reg.cu; finalize.cu forms sigma, U, the order.
#include <algorithm>

#include "kernel_args.cuh"
#include "launch.h"
#include "rotation.cuh"

namespace bsvd {
namespace r32b {

constexpr int N = 32;      // columns
constexpr int H = 16;      // column pairs per iteration
constexpr int NIT = 31;    // iterations per sweep (ring length)
constexpr int RSTR = 34;   // doubles per row of the dot-product transpose buffer (bank padding)
constexpr int LOG_ELEMS = NIT * H * 2 + 32;  // doubles per problem: rotation log (31 x 16 Par) + masks
constexpr int SB = H + 2;  // slot-state offset of the bottom columns (bank padding)
constexpr int SLS = 40;    // slot-state doubles per half
// slot that pair k's top / bottom column occupies in the next iteration: tops move right (the top of
// pair 15 becomes its bottom), bottoms move left (the bottom of pair 1 becomes pair 0's bottom, whose
// previous bottom becomes the top of pair 1), the fixed column stays the top of pair 0
__host__ __device__ constexpr int next_top(int k) { return k == 0 ? 0 : (k == H - 1 ? SB + H - 1 : k + 1); }
__host__ __device__ constexpr int next_bot(int k) { return k == 0 ? 1 : (k == 1 ? SB : SB + k - 1); }

__host__ __device__ constexpr int ring_slot(int q) {  // ring position -> register slot at t = 0
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}
__host__ __device__ constexpr int md(int a) { return ((a % NIT) + NIT) % NIT; }
__host__ __device__ constexpr int ring_pos(int s) {  // inverse of ring_slot (s >= 1)
    return s == 1 ? 0 : ((s & 1) == 0 ? s / 2 : 2 * H - 1 - (s - 1) / 2);
}
// slot that register slot s moves to under a ring shift by SH (the fixed column, slot 0, stays)
__host__ __device__ constexpr int dst_slot(int s, int SH) { return s == 0 ? 0 : ring_slot(md(ring_pos(s) + SH)); }
// register slot of pair k's top / bottom column at offset u inside an unrolled group
__host__ __device__ constexpr int TS(int k, int u) { return k == 0 ? 0 : ring_slot(md(k - u)); }
__host__ __device__ constexpr int BS(int k, int u) { return ring_slot(md((k == 0 ? 0 : NIT - k) - u)); }

struct __align__(16) Par {
    double cm1, c;  // x <- x + (cm1 x + c y);  y <- y + (cm1 y - c x)
};

struct WarpSmem {
    double red[3 * H * RSTR];  // dot-product transpose
    Par pub[2][H];             // this iteration's rotations, [half][pair]
    Par stage[2][2][H];        // V replay: double-buffered log rows [buf][half][pair]
    // per-column state indexed by pair slot (top of pair k: k, bottom: SB + k) and moved along the
    // tournament each iteration, so that lane k's reads and writes are bank-conflict free (indexed by
    // column id they were 3.9 wavefronts per access instead of 2, profiles/r2_ncu_c1_k42.txt)
    double nrm[2][SLS];        // maintained squared column norms [half][slot]
    double dsc[2][SLS];        // FG: column scale factors d (true column = d * stored column) [half][slot]
    double rds[2][SLS];        // FG: 1 / d
    double dv[2][N];           // FG: d at the end of the W sweep, applied to V after its replay
    double vn[2][N];           // FG: column norms of V after its latest replay (1 before the first)
    double sgs[2][N];          // FG finalisation: sigma of the scaled problem = ||w|| / ||v||
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

// move every column SH ring positions forward (compile-time register moves)
template <int SH>
__device__ __forceinline__ void ring_shift(double (&x)[N]) {
    // x[slot(q)] <- x[slot(q - SH)] for every ring position; 31 is prime, so the
    // permutation is one cycle: follow it with a single temporary (32 moves)
    if constexpr (md(SH) != 0) {
        const double t = x[ring_slot(0)];
#pragma unroll
        for (int i = 0; i < NIT - 1; ++i) x[ring_slot(md(-i * SH))] = x[ring_slot(md(-(i + 1) * SH))];
        x[ring_slot(md(-(NIT - 1) * SH))] = t;
    }
}

__device__ __forceinline__ void apply2(double& x, double& y, double cm1, double c) {
    const double tx = fma(c, y, x);
    const double ty = fma(-c, x, y);
    x = fma(cm1, x, tx);
    y = fma(cm1, y, ty);
}

// Scaled (fast) rotation on stored columns (FG): with a_x = d_x p_x and a_y = d_y p_y the rotation
//   a_x' = c a_x + S a_y,  a_y' = c a_y - S a_x        (S = +-s, the reference's update)
// is p_x' = p_x + alpha p_y,  p_y' = p_y + beta p_x   with alpha = T d_y / d_x, beta = -T d_x / d_y,
// T = S / c (the signed tangent), and d_x' = c d_x, d_y' = c d_y: one FMA per element instead of two.
__device__ __forceinline__ void apply_fg(double& x, double& y, double alpha, double beta) {
    const double xo = x;
    x = fma(alpha, y, x);
    y = fma(beta, xo, y);
}
template <bool FG>
__device__ __forceinline__ void apply_any(double& x, double& y, double p0, double p1) {
    if constexpr (FG) apply_fg(x, y, p0, p1);
    else apply2(x, y, p0, p1);
}
// the same update with the ring shift folded in: results go straight to their post-shift registers
// (nx, ny are slots of a second array), so the loop back-edge needs no register moves
template <bool FG>
__device__ __forceinline__ void apply_to(double x, double y, double& nx, double& ny, double p0, double p1) {
    if constexpr (FG) {
        nx = fma(p0, y, x);
        ny = fma(p1, x, y);
    } else {
        const double tx = fma(p1, y, x);
        const double ty = fma(-p1, x, y);
        nx = fma(p0, x, tx);
        ny = fma(p0, y, ty);
    }
}

__device__ __forceinline__ double sum16(const double* p) {  // 16 consecutive doubles, fixed tree
    const double2* r = reinterpret_cast<const double2*>(p);
    const double2 p0 = r[0], p1 = r[1], p2 = r[2], p3 = r[3], p4 = r[4], p5 = r[5], p6 = r[6], p7 = r[7];
    const double s0 = (p0.x + p0.y) + (p1.x + p1.y), s1 = (p2.x + p2.y) + (p3.x + p3.y);
    const double s2 = (p4.x + p4.y) + (p5.x + p5.y), s3 = (p6.x + p6.y) + (p7.x + p7.y);
    return (s0 + s1) + (s2 + s3);
}

// 16 consecutive doubles summed in the order of a 16-8-4-2-1 xor butterfly over rows (i, i + 16) first:
// the column-norm order of finalize_block (finalize.cuh step 1), so the fused and the standalone
// finalisation give the same sigma bits.

__device__ __forceinline__ double sum16_butterfly(const double* p) {
    double t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i] = p[i] + p[i + 8];
#pragma unroll
    for (int i = 0; i < 4; ++i) t[i] = t[i] + t[i + 4];
    return (t[0] + t[2]) + (t[1] + t[3]);
}

// partial dot products of this lane's two rows for the 16 pairs at offset u
template <int u, bool FULL>
__device__ __forceinline__ void partials(const double (&x0)[N], const double (&x1)[N], double* red, int lane) {
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const double a0 = x0[TS(k, u)], b0 = x0[BS(k, u)], a1 = x1[TS(k, u)], b1 = x1[BS(k, u)];
        if constexpr (FULL) {
            red[(3 * k + 0) * RSTR + lane] = fma(a1, a1, a0 * a0);
            red[(3 * k + 1) * RSTR + lane] = fma(b1, b1, b0 * b0);
            red[(3 * k + 2) * RSTR + lane] = fma(b1, a1, b0 * a0);
        } else {
            red[k * RSTR + lane] = fma(b1, a1, b0 * a0);
        }
    }
}

// Development probes (tools/microbench/wchain.cu defines R32_PROBE_ON): clock
// deltas between stage boundaries of the W iteration, warp 0 of block 0.
#ifdef R32_PROBE_ON
__device__ unsigned long long g_r32_probe[16];
#define R32P(i, v) r32_probe(i, v, st)
#else
#define R32P(i, v)
#endif

struct IterState {
    long long tl;       // last probe clock (R32_PROBE_ON only)
    int my_rot;         // rotations of this lane's pair in the sweep
    uint32_t itbits;    // bit t: some pair of either problem rotated in iteration t
    bool full;          // this iteration recomputes the norms of some problem of the warp
    uint32_t fmask;     // ballot of the lanes whose problem takes the fresh norms (per half: a
                        // problem's numerics never depend on the problem sharing its warp)
};

#ifdef R32_PROBE_ON
__device__ __forceinline__ void r32_probe_t(int i, double v, long long& tl) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64; // %1" : "=l"(c) : "d"(v) : "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (i > 0) atomicAdd(&g_r32_probe[i], (unsigned long long)(c - tl));
        else atomicAdd(&g_r32_probe[0], 1ull);
    }
    tl = c;
}
#define R32PT(i, v, tl) r32_probe_t(i, v, tl)
#else
#define R32PT(i, v, tl)
#endif
#ifdef R32_PROBE_ON
__device__ __forceinline__ void r32_probe(int i, double v, IterState& st) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64; // %1" : "=l"(c) : "d"(v) : "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (i > 0) atomicAdd(&g_r32_probe[i], (unsigned long long)(c - st.tl));
        else atomicAdd(&g_r32_probe[0], 1ull);
    }
    st.tl = c;
}
#endif

// Column ids of pair k at iteration t, packed ct | cb << 8 | flip << 16
// (built once per CTA in shared memory; reference orientation i < j).
__host__ __device__ inline uint32_t pair_code(int t, int k) {
    int qt = k - t, qb = (k == 0 ? 0 : NIT - k) - t;
    qt += qt < 0 ? NIT : 0;
    qb += qb < 0 ? NIT : 0;
    const int ct = (k == 0) ? 0 : ring_slot(qt);
    const int cb = ring_slot(qb);
    return (uint32_t)ct | ((uint32_t)cb << 8) | ((ct > cb) ? (1u << 16) : 0u);
}

__device__ __forceinline__ double xor_sign(double x, bool neg) {
    return __longlong_as_double(__double_as_longlong(x) ^ ((long long)neg << 63));
}

// |d|, g -> s = sin(th) >= 0, c - 1, |t| (rotation_half without the signs).
// Fast path without rescaling (the data are pre-scaled to max |a| in
// [0.5, 1), so d^2 + 4 g^2 only underflows for pairs of columns below
// 2^-250); the exact rescale is a rare fix-up after the fact.
__device__ __forceinline__ void rot_abs_core(double dabs, double g, double& s, double& cm1, double& tabs) {
    const double q = fma(4.0 * g, g, dabs * dabs);
    const double ir = rsqrt_cubic(q);
    const double gi = g * ir;
    const double c2 = fma(0.5 * dabs, ir, 0.5);
    const double ic = rsqrt_cubic(c2);
    const double c = c2 * ic;
    s = gi * ic;
    cm1 = -(s * s) * rcp_cubic(1.0 + c);
    tabs = s * ic;
}
__device__ __forceinline__ void rot_abs(double dabs, double g, double& s, double& cm1, double& tabs) {
    rot_abs_core(dabs, g, s, cm1, tabs);
    if (fmax(dabs, g) < 0x1p-500) rot_abs_core(dabs * 0x1p+600, g * 0x1p+600, s, cm1, tabs);
}
// FG: |t|, c and 1/c of the same half-angle chain (no 1 / (1 + c): c - 1 is not needed)
__device__ __forceinline__ void rot_fg_core(double dabs, double g, double& tabs, double& c, double& ic) {
    const double q = fma(4.0 * g, g, dabs * dabs);
    const double ir = rsqrt_cubic(q);
    const double gi = g * ir;
    const double c2 = fma(0.5 * dabs, ir, 0.5);
    ic = rsqrt_cubic(c2);
    c = c2 * ic;
    tabs = (gi * ic) * ic;
}
__device__ __forceinline__ void rot_fg(double dabs, double g, double& tabs, double& c, double& ic) {
    rot_fg_core(dabs, g, tabs, c, ic);
    if (fmax(dabs, g) < 0x1p-500) rot_fg_core(dabs * 0x1p+600, g * 0x1p+600, tabs, c, ic);
}

// g_ji partial product of next pair k (offset u) from this lane's two rows
template <int u>
__device__ __forceinline__ void cross_partial(const double (&x0)[N], const double (&x1)[N], double* red, int lane,
                                              int k) {
    red[k * RSTR + lane] = fma(x1[BS(k, u)], x1[TS(k, u)], x0[BS(k, u)] * x0[TS(k, u)]);
}
// squared-norm partials of next pairs' top / bottom columns (full iterations), rows H + 2k, H + 2k + 1
template <int u>
__device__ __forceinline__ void norm_partials(const double (&x0)[N], const double (&x1)[N], double* red, int lane) {
#pragma unroll
    for (int k = 0; k < H; ++k) {
        const double a0 = x0[TS(k, u)], b0 = x0[BS(k, u)], a1 = x1[TS(k, u)], b1 = x1[BS(k, u)];
        red[(H + 2 * k) * RSTR + lane] = fma(a1, a1, a0 * a0);
        red[(H + 2 * k + 1) * RSTR + lane] = fma(b1, b1, b0 * b0);
    }
}
// partials of the iteration at offset u (sweep start: always full)
template <int u>
__device__ __forceinline__ void all_partials(const double (&x0)[N], const double (&x1)[N], double* red, int lane,
                                             bool full) {
#pragma unroll
    for (int k = 0; k < H; ++k) cross_partial<u>(x0, x1, red, lane, k);
    if (full) norm_partials<u>(x0, x1, red, lane);
}

// One W iteration at offset u of the unrolled group; t = global iteration
// (0..30).  On entry red[] holds this iteration's partial products; the
// update is fused with the partials of iteration t + 1 (offset u + 1 in the
// pre-shift register naming: next pair k = columns of this iteration's pairs
// k - 1 and k + 1), so they are ready when the next reduction starts.
template <int u, int PD, bool FG = false, int SH = 0, bool FV = false>
__device__ __forceinline__ void w_iter(double (&x0)[N], double (&x1)[N], WarpSmem& sm, const uint32_t* ctab, int t,
                                       int lane, int half, int hl, bool done, double tol, double tol2,
                                       Par* logl, IterState& st) {
    R32P(0, x0[TS(0, u)]);
    const uint32_t code = ctab[t * H + hl];
    __syncwarp();
    // ---- lane hl owns pair k = hl of its half's problem ----
    const int k = hl;
    const int ct = code & 0xff, cb = (code >> 8) & 0xff;
    const bool flip = (code >> 16) != 0;
    double gt, gb;
    (void)ct;
    (void)cb;
    double sct = 1.0, scb = 1.0, rst = 1.0, rsb = 1.0;  // FG: scale factors of the pair's columns
    if constexpr (FG) {
        sct = sm.dsc[half][k];
        scb = sm.dsc[half][SB + k];
        rst = sm.rds[half][k];
        rsb = sm.rds[half][SB + k];
    }
    if (st.full && ((st.fmask >> lane) & 1u)) {
        gt = sum16(sm.red + (H + 2 * k) * RSTR + 16 * half);
        gb = sum16(sm.red + (H + 2 * k + 1) * RSTR + 16 * half);
        if constexpr (FG) {
            gt *= sct * sct;
            gb *= scb * scb;
        }
    } else {
        gt = sm.nrm[half][k];
        gb = sm.nrm[half][SB + k];
    }
    double g = sum16(sm.red + k * RSTR + 16 * half);
    if constexpr (FG) g *= sct * scb;  // dot product of the true columns
    const double absg = fabs(g);
    R32P(1, g);
    // guard (F4): rotate unless |g| <= 0 or |g| < tol sqrt(gii gjj); squared
    // comparison, exact-sqrt fallback where g^2 could underflow
    const double p = gt * gb;
    bool rot = !(absg * absg < tol2 * p);
    if (absg < 0x1p-400 && absg > 0.0) rot = !(absg < tol * fsqrt(p));
    rot = rot && !done && absg > 0.0;
    const double d = gt - gb;
    double s, cm1, tabs, cc = 1.0, icc = 1.0;
    if constexpr (FG) rot_fg(fabs(d), absg, tabs, cc, icc);
    else rot_abs(fabs(d), absg, s, cm1, tabs);
    // sign of tau in slot orientation: sgn(d), and for d == 0 the reference's
    // sgn(0) = +1 taken in (i, j) orientation
    const bool eneg = d < 0.0 || (d == 0.0 && flip);
    Par par;
    if constexpr (FG) {
        const double T = xor_sign(tabs, (g < 0.0) != eneg);  // signed tangent S / c
        par.cm1 = rot ? T * (scb * rst) : 0.0;                // alpha (x = top slot)
        par.c = rot ? -T * (sct * rsb) : 0.0;                 // beta (y = bottom slot)
    } else {
        par.cm1 = rot ? cm1 : 0.0;
        par.c = rot ? xor_sign(s, (g < 0.0) != eneg) : 0.0;  // x = top slot, y = bot slot
    }
    R32P(2, par.cm1);
    sm.pub[half][k] = par;
    // FV (one problem per warp: W rows in half 0, V rows in half 1): only half 0's rotations are real;
    // half 1 evaluates pairs of V's columns in lockstep and discards them
    const unsigned mask = __ballot_sync(0xffffffffu, rot) & (FV ? 0xFFFFu : 0xFFFFFFFFu);
    if (logl) logl[t * H] = par;
    __syncwarp();
    R32P(6, sm.pub[half][0].c);
    const double dtg = rot ? xor_sign(tabs * absg, eneg) : 0.0;
    const double nt = gt + dtg, nb = gb - dtg;
    {  // the pair's column state moves to the columns' slots of iteration t + 1
        const int dt = next_top(k), db = next_bot(k);
        sm.nrm[half][dt] = nt;
        sm.nrm[half][db] = nb;
        if constexpr (FG) {
            sm.dsc[half][dt] = rot ? cc * sct : sct;
            sm.dsc[half][db] = rot ? cc * scb : scb;
            sm.rds[half][dt] = rot ? icc * rst : rst;
            sm.rds[half][db] = rot ? icc * rsb : rsb;
        }
    }
    const bool shrink = rot && (nt < 0.25 * gt || nb < 0.25 * gb);
    st.my_rot += rot ? 1 : 0;
    {  // a >4x shrink in a problem makes that problem's next iteration recompute its norms
        const uint32_t sb = __ballot_sync(0xffffffffu, shrink) & (FV ? 0xFFFFu : 0xFFFFFFFFu);
        st.fmask = ((sb & 0xFFFFu) ? 0xFFFFu : 0u) | ((sb >> 16) ? 0xFFFF0000u : 0u);
        st.full = sb != 0u;
    }
    st.itbits |= (mask != 0u ? 1u : 0u) << t;
    constexpr int un = u + 1;  // offset of iteration t + 1 (pre-shift naming)
    if (SH != 0 || mask) {
        // rotations PD ahead (PD = 16: all first) -- the loop interleaves stores to red[]
        const int ph = FV ? 0 : half;  // FV: V's rows (half 1) take W's rotations
        Par pq[PD];
#pragma unroll
        for (int q = 0; q < PD; ++q) pq[q] = sm.pub[ph][q];
        if constexpr (SH == 0) {
#pragma unroll
            for (int q = 0; q < H; ++q) {
                const Par cur = pq[q % PD];
                if (q + PD < H) pq[q % PD] = sm.pub[ph][q + PD];
                apply_any<FG>(x0[TS(q, u)], x0[BS(q, u)], cur.cm1, cur.c);
                apply_any<FG>(x1[TS(q, u)], x1[BS(q, u)], cur.cm1, cur.c);
                if (q >= 1) cross_partial<un>(x0, x1, sm.red, lane, q - 1);  // needs pairs q-2, q
            }
            cross_partial<un>(x0, x1, sm.red, lane, H - 1);
            if (st.full) norm_partials<un>(x0, x1, sm.red, lane);
        } else {
            // last iteration of an unrolled group, branch-free: the ring shift by SH = un is folded into
            // the update (every slot belongs to one pair, so every post-shift register is written by an
            // FMA; a pair that does not rotate has zero parameters and its FMAs copy exactly), so the
            // loop back-edge needs no register moves; iteration t + 1 is at offset 0 of the new naming
            static_assert(SH == un, "the folded shift must bring the next iteration to offset 0");
            double y0[N], y1[N];
#pragma unroll
            for (int q = 0; q < H; ++q) {
                const Par cur = pq[q % PD];
                if (q + PD < H) pq[q % PD] = sm.pub[ph][q + PD];
                apply_to<FG>(x0[TS(q, u)], x0[BS(q, u)], y0[dst_slot(TS(q, u), SH)], y0[dst_slot(BS(q, u), SH)],
                             cur.cm1, cur.c);
                apply_to<FG>(x1[TS(q, u)], x1[BS(q, u)], y1[dst_slot(TS(q, u), SH)], y1[dst_slot(BS(q, u), SH)],
                             cur.cm1, cur.c);
                if (q >= 1) cross_partial<0>(y0, y1, sm.red, lane, q - 1);
            }
            cross_partial<0>(y0, y1, sm.red, lane, H - 1);
#pragma unroll
            for (int c = 0; c < N; ++c) {
                x0[c] = y0[c];
                x1[c] = y1[c];
            }
            if (st.full) norm_partials<0>(x0, x1, sm.red, lane);
        }
    } else {
#pragma unroll
        for (int q = 0; q < H; ++q) cross_partial<un>(x0, x1, sm.red, lane, q);
        if (st.full) norm_partials<un>(x0, x1, sm.red, lane);
    }
    R32P(3, x1[BS(H - 1, u)]);
}

// One V replay iteration at offset u (log row t is staged in sm.stage[t & 1]).
template <int u, int PD, bool FG = false, int SH = 0>
__device__ __forceinline__ void v_iter(double (&x0)[N], double (&x1)[N], WarpSmem& sm, int t, int half, int hl,
                                       const Par* logl, uint32_t itbits, long long& tl) {
    R32PT(7, x0[TS(0, u)], tl);
    if (t + 1 < NIT) cp_async16(&sm.stage[(t + 1) & 1][half][hl], logl + (t + 1) * H);
    cp_commit();
    cp_wait<1>();
    __syncwarp();
    R32PT(8, sm.stage[t & 1][half][0].c, tl);
    const bool go = (itbits >> t) & 1u;
    if (SH != 0 || go) {  // (the log holds zero parameters for pairs that did not rotate)
        const Par* stp = sm.stage[t & 1][half];
        Par pr[PD];  // rotations PD ahead, then independent FMAs
#pragma unroll
        for (int q = 0; q < PD; ++q) pr[q] = stp[q];
        if constexpr (SH == 0) {
#pragma unroll
            for (int q = 0; q < H; ++q) {
                const Par pq = pr[q % PD];
                if (q + PD < H) pr[q % PD] = stp[q + PD];
                apply_any<FG>(x0[TS(q, u)], x0[BS(q, u)], pq.cm1, pq.c);
                apply_any<FG>(x1[TS(q, u)], x1[BS(q, u)], pq.cm1, pq.c);
            }
        } else {  // ring shift folded into the update (see w_iter)
            double y0[N], y1[N];
#pragma unroll
            for (int q = 0; q < H; ++q) {
                const Par pq = pr[q % PD];
                if (q + PD < H) pr[q % PD] = stp[q + PD];
                apply_to<FG>(x0[TS(q, u)], x0[BS(q, u)], y0[dst_slot(TS(q, u), SH)], y0[dst_slot(BS(q, u), SH)],
                             pq.cm1, pq.c);
                apply_to<FG>(x1[TS(q, u)], x1[BS(q, u)], y1[dst_slot(TS(q, u), SH)], y1[dst_slot(BS(q, u), SH)],
                             pq.cm1, pq.c);
            }
#pragma unroll
            for (int c = 0; c < N; ++c) {
                x0[c] = y0[c];
                x1[c] = y1[c];
            }
        }
    }
    R32PT(9, x1[BS(H - 1, u)], tl);
    __syncwarp();
}

template <int U, int PD, bool FG = false, bool FV = false>
__device__ __forceinline__ void w_sweep(double (&x0)[N], double (&x1)[N], WarpSmem& sm, const uint32_t* ctab,
                                        int lane, int half, int hl, bool done, double tol, double tol2, Par* logl,
                                        IterState& st) {
    constexpr int NG = (NIT + U - 1) / U;
    constexpr int R = NIT - (NG - 1) * U;  // iterations in the last group
    static_assert(U == 2 && R == 1, "ring unrolled by 2: 15 groups of two iterations and one single");
    all_partials<0>(x0, x1, sm.red, lane, true);  // first iteration of a sweep: fresh norms
#pragma unroll 1
    for (int gi = 0; gi < NG; ++gi) {
        const int t0 = gi * U;
        w_iter<0, PD, FG, 0, FV>(x0, x1, sm, ctab, t0, lane, half, hl, done, tol, tol2, logl, st);
        if (gi == NG - 1) {  // once per sweep: the shift by one that closes the ring
            ring_shift<1>(x0);
            ring_shift<1>(x1);
            break;
        }
        // the second iteration of the group writes its results straight into the shifted registers
        w_iter<1, PD, FG, 2, FV>(x0, x1, sm, ctab, t0 + 1, lane, half, hl, done, tol, tol2, logl, st);
    }
}

template <int U, int PD, bool FG = false>
__device__ __forceinline__ void v_sweep(double (&x0)[N], double (&x1)[N], WarpSmem& sm, int half, int hl,
                                        const Par* logl, uint32_t itbits, long long& tl) {
    constexpr int NG = (NIT + U - 1) / U;
    constexpr int R = NIT - (NG - 1) * U;
    static_assert(U == 2 && R == 1, "ring unrolled by 2");
#pragma unroll 1
    for (int gi = 0; gi < NG; ++gi) {
        const int t0 = gi * U;
        v_iter<0, PD, FG>(x0, x1, sm, t0, half, hl, logl, itbits, tl);
        if (gi == NG - 1) {
            ring_shift<1>(x0);
            ring_shift<1>(x1);
            break;
        }
        v_iter<1, PD, FG, 2>(x0, x1, sm, t0 + 1, half, hl, logl, itbits, tl);
    }
}

// FV (fused V, kernel id 52): one problem per warp for batches that leave SM sub-partitions idle.  Half 0
// holds W's rows (hl, hl + 16) and half 1 the same rows of V, which take W's rotations in lockstep (the
// same parameters, the same FMAs as the replay, so the same bits): no rotation log, no replay phase, no
// parking of W and V in global memory.  Half 1 evaluates pairs of V's columns and discards them.
template <int NW, int MINB, int U, int UV, int PD, bool FG = false, bool FV = false>
__device__ __forceinline__ void reg32b_body(const SolveArgs<double>& a, int cta) {
    static_assert(!FV || FG, "the fused-V mode is built on the scaled rotations");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
    const int half = lane >> 4, hl = lane & 15;
    const int ph = FV ? 0 : half;  // the half whose problem this lane's results belong to
    const int prob = FV ? cta * NW + warp : (cta * NW + warp) * 2 + half;
    const bool live = prob < a.batch;
    const int r0 = hl, r1 = hl + 16;
    const size_t pstride = (size_t)a.work_stride;
    double* wsW = a.work + (size_t)(live ? prob : 0) * pstride;  // W 32x32, V 32x32, then the log
    double* wsV = wsW + N * N;
    Par* logp = reinterpret_cast<Par*>(wsW + 2 * N * N);           // [31][16]
    const bool want_v = a.need_v != 0;
    // this lane's column of the rotation log; a dead half never writes (it
    // aliases problem 0's workspace) but may read
    Par* logl = want_v && !FV ? logp + hl : nullptr;
    Par* logw = live ? logl : nullptr;
    uint32_t* ctab = reinterpret_cast<uint32_t*>(smem_raw + NW * sizeof(WarpSmem));
    for (int e = threadIdx.x; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    if constexpr (FG) {  // unit scales (the warp's own slots; lane hl: pair hl's two slots, columns 2 hl, 2 hl + 1)
        sm.dsc[half][hl] = sm.dsc[half][SB + hl] = 1.0;
        sm.rds[half][hl] = sm.rds[half][SB + hl] = 1.0;
        sm.vn[half][2 * hl] = sm.vn[half][2 * hl + 1] = 1.0;
    }
    __syncthreads();

    double x0[N], x1[N];
    int bad = 0;
    double amax = 0.0;
    {
        const double* Ap = a.A + (size_t)(live ? prob : 0) * a.strideA;  // plan requires lda == 32
        const bool ld = live && !(FV && half);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] = ld ? __ldcs(Ap + r0 + c * N) : 0.0;  // read once: evict-first, keep L2 for the workspace
            x1[c] = ld ? __ldcs(Ap + r1 + c * N) : 0.0;
        }
        if (FV && half) {  // V = I
#pragma unroll
            for (int c = 0; c < N; ++c) {
                x0[c] = (c == r0) ? 1.0 : 0.0;
                x1[c] = (c == r1) ? 1.0 : 0.0;
            }
        }
#pragma unroll
        for (int c = 0; c < N; ++c) {
            bad |= !isfinite(x0[c]) | !isfinite(x1[c]);
            amax = fmax(amax, fmax(fabs(x0[c]), fabs(x1[c])));
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int ex = FV ? __shfl_sync(0xffffffffu, prescale_exponent(amax), 0) : prescale_exponent(amax);
    {
        const double scale = (FV && half) ? 1.0 : pow2(-ex);
#pragma unroll
        for (int c = 0; c < N; ++c) {
            x0[c] *= scale;
            x1[c] *= scale;
        }
    }
    const double tol = a.tol, tol2 = a.tol * a.tol;
    int sweeps = 0, last = 0, done = live ? 0 : 1;
    long long rot_total = 0;
    bool v_started = false;  // V still identity until the first replay

#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        IterState st;
        st.my_rot = 0;
        st.itbits = 0;
        st.full = true;  // fresh norms at the start of every sweep
        st.fmask = 0xffffffffu;
        w_sweep<U, PD, FG, FV>(x0, x1, sm, ctab, lane, half, hl, done != 0, tol, tol2, logw, st);
        if constexpr (FG) {
            // back to true columns at the sweep end (the ring is back in place: slot c = column c), so
            // every sweep starts from unit scales and the finalisation sees W and V themselves
            // the state is in the slots of iteration 0 again: lane hl holds the scales of columns
            // code(0, hl); d by column id into dv, then unit scales for the next sweep
            __syncwarp();
            {
                const uint32_t c0 = ctab[hl];
                sm.dv[half][c0 & 0xff] = sm.dsc[half][hl];
                sm.dv[half][(c0 >> 8) & 0xff] = sm.dsc[half][SB + hl];
                sm.dsc[half][hl] = sm.dsc[half][SB + hl] = 1.0;
                sm.rds[half][hl] = sm.rds[half][SB + hl] = 1.0;
            }
            __syncwarp();
            if (st.itbits) {  // (FV: V's rows take the same scales, as after the replay)
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const double dc = sm.dv[ph][c];
                    x0[c] *= dc;
                    x1[c] *= dc;
                }
            }
            __syncwarp();
            if (FV && want_v && st.itbits) {  // column norms of V (half 1's rows), as after the replay
#pragma unroll
                for (int c = 0; c < N; ++c)
                    sm.red[c * RSTR + lane] = __dadd_rn(__dmul_rn(x0[c], x0[c]), __dmul_rn(x1[c], x1[c]));
                __syncwarp();
                const double na = __dsqrt_rn(sum16_butterfly(sm.red + (2 * hl) * RSTR + 16));
                const double nb = __dsqrt_rn(sum16_butterfly(sm.red + (2 * hl + 1) * RSTR + 16));
                __syncwarp();
                if (half) {
                    sm.vn[0][2 * hl] = na;
                    sm.vn[0][2 * hl + 1] = nb;
                }
                __syncwarp();
            }
        }
        // ---- sweep end: per-problem rotation count over the half warp ----
        int tot = st.my_rot;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if constexpr (FV) tot = __shfl_sync(0xffffffffu, tot, 0);  // half 1's count is not a problem's
        if (!done) {
            sweeps = sw + 1;
            last = tot;
            rot_total += tot;
            if (tot == 0) done = 1;
        }
        const int partner_done = __shfl_xor_sync(0xffffffffu, done, 16);
        const bool both_done = done && partner_done;
        // ======================= V phase: replay the sweep =======================
        if (!FV && want_v && st.itbits) {
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
            cp_async16(&sm.stage[0][half][hl], logl);
            cp_commit();
            v_sweep<UV, PD, FG>(x0, x1, sm, half, hl, logl, st.itbits, st.tl);
            cp_wait<0>();
            if constexpr (FG) {
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const double dc = sm.dv[half][c];
                    x0[c] *= dc;
                    x1[c] *= dc;
                }
                // column norms of V (the scale roundings W and V share; the finalisation divides them out)
                __syncwarp();
#pragma unroll
                for (int c = 0; c < N; ++c)
                    sm.red[c * RSTR + lane] = __dadd_rn(__dmul_rn(x0[c], x0[c]), __dmul_rn(x1[c], x1[c]));
                __syncwarp();
                sm.vn[half][2 * hl] = __dsqrt_rn(sum16_butterfly(sm.red + (2 * hl) * RSTR + 16 * half));
                sm.vn[half][2 * hl + 1] = __dsqrt_rn(sum16_butterfly(sm.red + (2 * hl + 1) * RSTR + 16 * half));
                __syncwarp();
            }
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
    // ======== kernel (5) fused (phase-alternating path): sigma, order, U = W / sigma, V permuted ========
    // A problem with a column below tiny/u (orthogonal completion, finalize.cuh step 3) is left to
    // the standalone finalisation pass: W and V go to the workspace with its flag set.
    double* flagp = wsW + pstride - 1;  // last double of the problem's workspace (log padding)
    bool fused = false;
    {
        const double unscale = pow2(ex);
#pragma unroll
        for (int c = 0; c < N; ++c) sm.red[c * RSTR + lane] = __dadd_rn(__dmul_rn(x0[c], x0[c]), __dmul_rn(x1[c], x1[c]));
        __syncwarp();
        // lane hl: columns 2 hl, 2 hl + 1.  Sigma of the scaled W (ssa); the power-of-two scale is
        // exact, so sa = ssa * 2^ex and x / ssa are the unscaled sigma and quotient.
        const double wna = __dsqrt_rn(sum16_butterfly(sm.red + (2 * hl) * RSTR + 16 * ph));
        const double wnb = __dsqrt_rn(sum16_butterfly(sm.red + (2 * hl + 1) * RSTR + 16 * ph));
        // FG: sigma = ||w|| / ||v|| (the column-scale roundings W and V share cancel); U = W / ||w||
        double ssa = wna, ssb = wnb;
        bool vok = true;
        if constexpr (FG) {
            const double va = sm.vn[ph][2 * hl], vb = sm.vn[ph][2 * hl + 1];
            ssa = div_by_sigma(wna, va, rcp_refined(va));
            ssb = div_by_sigma(wnb, vb, rcp_refined(vb));
            vok = va >= 0.5 && va <= 2.0 && vb >= 0.5 && vb <= 2.0;
        }
        const double sa = ssa * unscale, sb = ssb * unscale;
        // holes (sigma < tiny/u), scaled sigmas outside the reciprocal's safe range, and columns whose
        // scaled squares may have left the normal range (sigma < 2^-480 of the problem's scale: the
        // standalone pass rescales per column, like the reference's underflow-safe norms) take the
        // standalone pass
        const bool tiny = !(sa >= dtiny<double>() && sb >= dtiny<double>() && wna >= 0x1p-480 && wnb >= 0x1p-480 &&
                            wna <= 0x1p+960 && wnb <= 0x1p+960 && vok);
        const unsigned tm = __ballot_sync(0xffffffffu, tiny);
        fused = ((tm >> (16 * ph)) & 0xFFFFu) == 0u;
        __syncwarp();
        // [half][32] (scaled sigma, reciprocal) and rank by column, in rows 32.. of red
        double2* sr = reinterpret_cast<double2*>(sm.red + 32 * RSTR) + 32 * ph;
        int* rk = reinterpret_cast<int*>(sm.red + 32 * RSTR + 128) + 32 * ph;
        const bool own = !(FV && half);  // FV: half 0 alone fills the shared tables, half 1 (V) reads them
        if (own) {
            sr[2 * hl] = make_double2(wna, rcp_refined(wna));
            sr[2 * hl + 1] = make_double2(wnb, rcp_refined(wnb));
            if constexpr (FG) {
                sm.sgs[half][2 * hl] = ssa;
                sm.sgs[half][2 * hl + 1] = ssb;
            }
        }
        __syncwarp();
        int ra = 0, rb = 0;  // stable descending ranks (finalize.cuh step 4)
        if (own) {
#pragma unroll 8
            for (int c2 = 0; c2 < N; ++c2) {
                const double s2 = FG ? sm.sgs[half][c2] : sr[c2].x;
                ra += sig_before(s2, ssa) || (c2 < 2 * hl && sig_tie(s2, ssa));
                rb += sig_before(s2, ssb) || (c2 < 2 * hl + 1 && sig_tie(s2, ssb));
            }
            rk[2 * hl] = ra;
            rk[2 * hl + 1] = rb;
        }
        __syncwarp();
        if (live && fused) {
            const FinalOut<double> o = final_out(a, prob);
            if (own) {
                o.S[ra] = sa;
                o.S[rb] = sb;
                double* u0 = o.U + r0;
                double* u1 = o.U + r1;
#pragma unroll
                for (int c = 0; c < N; ++c) {  // U = W / sigma: reciprocal, then one residual correction
                    const int rc = rk[c];
                    const double2 t = sr[c];
                    __stcs(u0 + (size_t)rc * o.ldu, div_by_sigma(x0[c], t.x, t.y));  // streaming: not re-read
                    __stcs(u1 + (size_t)rc * o.ldu, div_by_sigma(x1[c], t.x, t.y));
                }
            }
            if (o.want_v && o.V && (!FV || half)) {
                // all 64 loads ahead of the stores (the compiler cannot prove o.V and wsV disjoint,
                // so interleaving would serialise one L2 round trip per element); FV: V is in registers
                if (!FV && v_started) {
#pragma unroll
                    for (int c = 0; c < N; ++c) {
                        x0[c] = wsV[r0 + c * N];
                        x1[c] = wsV[r1 + c * N];
                    }
                } else if (!FV) {
#pragma unroll
                    for (int c = 0; c < N; ++c) {
                        x0[c] = (c == r0) ? 1.0 : 0.0;
                        x1[c] = (c == r1) ? 1.0 : 0.0;
                    }
                }
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const int rc = rk[c];
                    double y0 = x0[c], y1 = x1[c];
                    if constexpr (FG) {
                        const double vv = sm.vn[ph][c], rv = rcp_refined(vv);
                        y0 = div_by_sigma(y0, vv, rv);
                        y1 = div_by_sigma(y1, vv, rv);
                    }
                    __stcs(o.V + r0 + (size_t)rc * o.ldv, y0);
                    __stcs(o.V + r1 + (size_t)rc * o.ldv, y1);
                }
            }
        }
        if (live && (FV ? lane : hl) == 0) *flagp = fused ? 0.0 : 1.0;
    }
    if (live && !fused) {
        const double unscale = pow2(ex);
        if constexpr (FV) {  // W / ||v|| (half 0), V / ||v|| (half 1) by column for the standalone pass
            double* dst = half ? wsV : wsW;
            const double us = half ? 1.0 : unscale;
            if (!half || want_v) {
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const double vv = sm.vn[0][c], rv = rcp_refined(vv);
                    dst[r0 + c * N] = div_by_sigma(x0[c], vv, rv) * us;
                    dst[r1 + c * N] = div_by_sigma(x1[c], vv, rv) * us;
                }
            }
        } else if constexpr (FG) {  // W / ||v||, V / ||v|| by column for the standalone pass
#pragma unroll
            for (int c = 0; c < N; ++c) {
                const double vv = sm.vn[half][c], rv = rcp_refined(vv);
                wsW[r0 + c * N] = div_by_sigma(x0[c], vv, rv) * unscale;
                wsW[r1 + c * N] = div_by_sigma(x1[c], vv, rv) * unscale;
            }
            if (want_v && v_started) {
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    x0[c] = wsV[r0 + c * N];
                    x1[c] = wsV[r1 + c * N];
                }
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const double vv = sm.vn[half][c], rv = rcp_refined(vv);
                    wsV[r0 + c * N] = div_by_sigma(x0[c], vv, rv);
                    wsV[r1 + c * N] = div_by_sigma(x1[c], vv, rv);
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsW[r0 + c * N] = x0[c] * unscale;
                wsW[r1 + c * N] = x1[c] * unscale;
            }
        }
        if (!FV && want_v && !v_started) {
#pragma unroll
            for (int c = 0; c < N; ++c) {
                wsV[r0 + c * N] = (c == r0) ? 1.0 : 0.0;
                wsV[r1 + c * N] = (c == r1) ? 1.0 : 0.0;
            }
        }
    }
    if (!FV && live && fused) {
        // the problem is finished and its workspace (W / V parking, rotation log) is dead: drop its L2
        // lines instead of letting them be written back to DRAM (they were ~60 % of the kernel's DRAM
        // traffic); the line holding the finalisation flag, which the standalone pass reads, is kept
        // (FV never touches its workspace before the flag)
        __syncwarp();
        const uintptr_t lo = ((uintptr_t)wsW + 127) & ~(uintptr_t)127;
        const uintptr_t hi = (uintptr_t)flagp & ~(uintptr_t)127;
        for (uintptr_t l = lo + (uintptr_t)hl * 128; l < hi; l += 16 * 128)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
    }
    const unsigned badm = __ballot_sync(0xffffffffu, bad != 0);
    if (live && (FV ? lane : hl) == 0 && a.info) {
        bsvd_info inf;
        inf.converged = done;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = 0;
        inf.update_calls = 0;
        inf.last_rotations = last;
        inf.path = 1;
        inf.status = ((badm >> (16 * ph)) & 0xFFFFu) ? 1 : 0;
        inf.kernel = a.kernel;
        a.info[prob] = inf;
    }
}

template <int NW, int MINB, int U, int UV, int PD, bool FG = false, bool FV = false>
__global__ void __launch_bounds__(NW * 32, MINB) k_reg32b(SolveArgs<double> a) {
    reg32b_body<NW, MINB, U, UV, PD, FG, FV>(a, blockIdx.x);
}

// Batches above one resident wave: the head as 42 (two problems per warp) and a tail of whole problems
// as 52 (one problem per warp, V in lockstep) in ONE launch, head CTAs first, so the last partial wave
// runs the shorter single-problem chain instead of leaving SM sub-partitions idle (bit-identical: 42 and
// 52 give the same bits).  `tail` is `head` with every per-problem pointer advanced past the head.
template <int NW, int MINB, int U, int UV, int PD>
__global__ void __launch_bounds__(NW * 32, MINB) k_reg32b_split(SolveArgs<double> head, SolveArgs<double> tail,
                                                               int head_ctas) {
    if ((int)blockIdx.x < head_ctas) reg32b_body<NW, MINB, U, UV, PD, true, false>(head, blockIdx.x);
    else reg32b_body<NW, MINB, U, UV, PD, true, true>(tail, blockIdx.x - head_ctas);
}

}  // namespace r32b

bool is_reg32b(int kv) { return kv == KV_UNBLOCKED_REG32B || kv == KV_UNBLOCKED_REG32G || kv == KV_UNBLOCKED_REG32F; }

Plan plan_unblocked_reg32b(int dtype, int bm, int bn, int need_v, bool lda_ok, int variant, int max_sweeps) {
    Plan p{};
    (void)max_sweeps;
    if (dtype == BSVD_D && bm == 32 && bn == 32 && lda_ok) {
        p.kernel = is_reg32b(variant) ? variant : KV_UNBLOCKED_REG32B;
        p.threads = 128;
        p.smem = 4 * sizeof(r32b::WarpSmem) + r32b::NIT * r32b::H * 4;
        p.work_elems = 2 * 32 * 32 + r32b::LOG_ELEMS;  // W, V, one sweep's rotation log, flag
        p.grid = 0;
        p.resident = 0;
        (void)need_v;
    }
    return p;
}

template <int NW, int MINB, int U, int UV, int PD, bool FG, bool FV = false>
static int launch_r32b(SolveArgs<double> a, cudaStream_t st) {
    const int per_cta = FV ? NW : 2 * NW;
    const int grid = (a.batch + per_cta - 1) / per_cta;
    const size_t smem = NW * sizeof(r32b::WarpSmem) + r32b::NIT * r32b::H * 4;
    auto k = r32b::k_reg32b<NW, MINB, U, UV, PD, FG, FV>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<grid, NW * 32, smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

// head (42) + tail (52) in one launch; tail problems = p.aux (make_plan: split_tail)
static int launch_r32b_split(SolveArgs<double> a, int tail, cudaStream_t st) {
    constexpr int NW = 4;
    SolveArgs<double> h = a, t = a;
    const int nh = a.batch - tail;
    h.batch = nh;
    h.kernel = KV_UNBLOCKED_REG32G;
    t.batch = tail;
    t.kernel = KV_UNBLOCKED_REG32F;
    t.A = a.A + (size_t)nh * a.strideA;
    t.U = a.U + (size_t)nh * a.strideU;
    t.S = a.S + (size_t)nh * a.strideS;
    if (a.V) t.V = a.V + (size_t)nh * a.strideV;
    t.work = a.work + (size_t)nh * a.work_stride;
    if (a.info) t.info = a.info + nh;
    const int head_ctas = (nh + 2 * NW - 1) / (2 * NW), tail_ctas = (tail + NW - 1) / NW;
    const size_t smem = NW * sizeof(r32b::WarpSmem) + r32b::NIT * r32b::H * 4;
    auto k = r32b::k_reg32b_split<NW, 2, 2, 2, 8>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<head_ctas + tail_ctas, NW * 32, smem, st>>>(h, t, head_ctas);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

// tail problems for a batch of `batch` on `sms` SMs (0: no split): above one resident wave of 42's warps
// a tail of 2 problems per SM (4 from 48 problems per SM on); between one wave of 52's warps and one of
// 42's, up to 4 per SM as long as every warp of the launch stays resident (measured on B200, tools/tail_split.py: 1,250 0.43 -> 0.40 ms, 2,500 0.66 -> 0.58 ms, 5,000
// 1.00 -> 0.97 ms, 10,000 1.69 -> 1.65 ms); `override` (bsvd_opts.reserved[0], experimental): > 0 forces
// that tail, < 0 disables the split
int split_tail(int batch, int sms, int override) {
    if (override < 0) return 0;
    if (override > 0) return override <= batch ? override : 0;
    if (batch <= 8 * sms) return 0;  // kernel 52 alone
    int x = batch < 48 * sms ? 2 * sms : 4 * sms;  // (tools/tail_split.py: 5,000 best at 296, 10,000 at 592)
    if (batch <= 16 * sms) x = std::min(4 * sms, 15 * sms - batch);  // keep head warps + tail warps resident
    x &= ~3;
    return x >= 2 * sms ? x : 0;
}

// 4 warps per CTA, 2 CTAs per SM (255 registers: 8 warps, 16 problems per SM), ring unrolled by 2.
// Round-1 variants measured slower and retired: a 168-register cap (12 warps/SM, spills), the V ring
// unrolled by 4, a shuffle-butterfly g_ji reduction, a split W kernel + V replay kernel.
int launch_unblocked_reg32b(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    if (p.kernel == KV_UNBLOCKED_REG32G && p.aux > 0 && p.aux <= a.batch) {
        const int rc = launch_r32b_split(a, p.aux, st);
        if (rc) return rc;
        return launch_finalize_flagged<double>(a, st);
    }
    // (kernel 52 alone runs its own instantiation: 3-4 % faster below one wave than the split kernel's
    // one-problem-per-warp body with an empty head, _abtest A/B on B200, although that one spills less)
    const int rc = p.kernel == KV_UNBLOCKED_REG32G   ? launch_r32b<4, 2, 2, 2, 8, true>(a, st)  // scaled rotations
                   : p.kernel == KV_UNBLOCKED_REG32F ? launch_r32b<4, 2, 2, 2, 8, true, true>(a, st)  // + V in lockstep
                                                     : launch_r32b<4, 2, 2, 2, 16, false>(a, st);
    if (rc) return rc;
    return launch_finalize_flagged<double>(a, st);  // only problems the fused finalisation left over
}

}  // namespace bsvd
