// creg32.cu -- kernel (2)/(3), complex FP64 (c128) register-resident Jacobi for
// n = 32 columns and m <= 256 rows (BASELINE config C4: 256 x 32 c128, both the
// reference's dispatch route and its blocked Gram route, and the 32 x 32 R
// factor of the QR-preprocessed route).
//
// Reference iteration (onesided_sweeps, src/_kernels_numba.py:85-138): for
// each of the 31 iterations of the round-robin schedule (src/ordering.py:
// 32-75) and each of its 16 disjoint pairs (i < j):
//   g_ji = sum_r conj(a_rj) a_ri,  skip if |g_ji| <= 0 or |g_ji| < tol sqrt(g_ii g_jj)
//   w = conj(g_ji)/|g_ji|, tau = (g_ii - g_jj)/(2|g_ji|), t, s, c - 1 (F5)
//   a_i <- a_i + (cm1 a_i + s conj(w) a_j),  a_j <- a_j + (cm1 a_j - s w a_i)
// For n = 32 with nb = 16 the blocked route (_sweep_blocked, src/svd.py:
// 481-522) has exactly one block pair, the whole matrix: its Gram eigensolve
// (eig_sweeps on G = W^H W, src/_kernels_numba.py:17-82) applies the same
// rotation sequence two-sidedly to G, and W <- W (I + Delta), V <- V (I + Delta)
// (fused_pair_update, src/_kernels_numba.py:141-175) -- so one kernel serves
// both routes; only the telemetry (gram/update calls, path) and the inner
// sweep budget differ.
//
// B200 mapping: one CTA per problem, NW = ceil(m / 32) warps, lane l of warp w
// holds row 32 w + l of W (32 complex = 64 doubles) in registers with the
// tournament ring in compile-time register slots (unrolled by 2, as in
// unblocked_reg32b.cu).  Per iteration: each lane forms its row's 16
// conj(x_b) x_t partials, a smem transpose reduces them over the warp, the NW
// warp sums go through a parity-double-buffered smem slot and ONE named
// barrier, and every warp then evaluates all 16 rotations itself (identical
// bits in every warp: same sums, same order), so no second barrier is needed.
// Column norms are maintained (d_i +- t|g|, recomputed at sweep start and after
// a >4x shrink).  Rotation parameters use the half-angle chain of
// rotation.cuh without ever forming |g|: A = +-(1/r)(1/c) p and
// t|g| = |g|^2 (1/r)(1/c)^2, so the complex phase costs no division.
// V never leaves shared memory: since V starts as I and only ever gets
// right-multiplied by the rotations, V = P, the running product, updated
// every iteration by all threads (one (row, pair) task each) in smem.
#include <algorithm>

#include "kernel_args.cuh"
#include "launch.h"
#include "rotation.cuh"
#include "tma.cuh"

namespace bsvd {
namespace creg {

constexpr int N = 32;      // columns
constexpr int H = 16;      // pairs per iteration
constexpr int NIT = 31;    // iterations per sweep
constexpr int MAXW = 8;    // warps per CTA (m <= 256)

__host__ __device__ constexpr int ring_slot(int q) {
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}
__host__ __device__ constexpr int md(int a) { return ((a % NIT) + NIT) % NIT; }
__host__ __device__ constexpr int ring_pos(int s) {  // inverse of ring_slot (s >= 1)
    return s == 1 ? 0 : ((s & 1) == 0 ? s / 2 : 2 * H - 1 - (s - 1) / 2);
}
// slot that register slot s moves to under a ring shift by SH (the fixed column, slot 0, stays)
__host__ __device__ constexpr int dst_slot(int s, int SH) { return s == 0 ? 0 : ring_slot(md(ring_pos(s) + SH)); }
__host__ __device__ constexpr int TS(int k, int u) { return k == 0 ? 0 : ring_slot(md(k - u)); }
__host__ __device__ constexpr int BS(int k, int u) { return ring_slot(md((k == 0 ? 0 : NIT - k) - u)); }

__host__ __device__ inline uint32_t pair_code(int t, int k) {
    int qt = k - t, qb = (k == 0 ? 0 : NIT - k) - t;
    qt += qt < 0 ? NIT : 0;
    qb += qb < 0 ? NIT : 0;
    const int ct = (k == 0) ? 0 : ring_slot(qt);
    const int cb = ring_slot(qb);
    return (uint32_t)ct | ((uint32_t)cb << 8) | ((ct > cb) ? (1u << 16) : 0u);
}

struct __align__(16) Par {
    double cm1, ar, ai, pad;  // x_t += cm1 x_t + A x_b;  x_b += cm1 x_b - conj(A) x_t
};

constexpr int RS2 = 33;    // double2 transpose buffer row stride (conflict-free 16-byte reads)

struct WarpSmem {
    double2 red[H * RS2];      // transpose buffer: pair q's (re, im) partials of the 32 lanes, row q
    double pub[3 * H];         // this iteration's rotations, dense (cm1, ar, ai) triples: 2 pairs = 3 x 16 B
    double nrm[N];             // maintained squared column norms (identical in every warp)
};

struct CtaSmem {
    double gsum[2][MAXW][4 * H];   // cross-warp partial sums [parity][warp][value]
    int misc[4];                   // [0] bad input, [2..3] amax bits (8-byte aligned)
};
struct PSmem {
    double2 P[N * N];              // running rotation product (= V), column-major, (re, im) interleaved
};

// totals over the warp's 32 lanes of both components of transpose row `row` (identical bits on both
// halves; each component summed in the tree of sum16 over consecutive lanes, then across the halves)
__device__ __forceinline__ double2 sum32x2(const double2* red, int row, int half) {
    const double2* r = red + row * RS2 + 16 * half;
    double2 p[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) p[i] = r[i];
    double sx[4], sy[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        sx[j] = (p[4 * j].x + p[4 * j + 1].x) + (p[4 * j + 2].x + p[4 * j + 3].x);
        sy[j] = (p[4 * j].y + p[4 * j + 1].y) + (p[4 * j + 2].y + p[4 * j + 3].y);
    }
    const double tx = (sx[0] + sx[1]) + (sx[2] + sx[3]);
    const double ty = (sy[0] + sy[1]) + (sy[2] + sy[3]);
    const double ox = __shfl_xor_sync(0xffffffffu, tx, 16), oy = __shfl_xor_sync(0xffffffffu, ty, 16);
    return half ? make_double2(ox + tx, oy + ty) : make_double2(tx + ox, ty + oy);
}
__device__ __forceinline__ void bar_named(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int SH>
__device__ __forceinline__ void ring_shift(double (&x)[N]) {
    if constexpr (md(SH) != 0) {
        const double t = x[ring_slot(0)];
#pragma unroll
        for (int i = 0; i < NIT - 1; ++i) x[ring_slot(md(-i * SH))] = x[ring_slot(md(-(i + 1) * SH))];
        x[ring_slot(md(-(NIT - 1) * SH))] = t;
    }
}

// x_t += cm1 x_t + A x_b,  x_b += cm1 x_b - conj(A) x_t   (old values on every right-hand side)
__device__ __forceinline__ void capply(double& tr, double& ti, double& br, double& bi, const Par& p) {
    const double ntr = fma(p.cm1, tr, fma(p.ar, br, fma(-p.ai, bi, tr)));
    const double nti = fma(p.cm1, ti, fma(p.ar, bi, fma(p.ai, br, ti)));
    const double nbr = fma(p.cm1, br, fma(-p.ar, tr, fma(-p.ai, ti, br)));
    const double nbi = fma(p.cm1, bi, fma(-p.ar, ti, fma(p.ai, tr, bi)));
    tr = ntr;
    ti = nti;
    br = nbr;
    bi = nbi;
}
// the same update written to other registers (the ring shift folded into it, see iter)
__device__ __forceinline__ void capply_to(double tr, double ti, double br, double bi, double& ntr, double& nti,
                                          double& nbr, double& nbi, const Par& p) {
    ntr = fma(p.cm1, tr, fma(p.ar, br, fma(-p.ai, bi, tr)));
    nti = fma(p.cm1, ti, fma(p.ar, bi, fma(p.ai, br, ti)));
    nbr = fma(p.cm1, br, fma(-p.ar, tr, fma(-p.ai, ti, br)));
    nbi = fma(p.cm1, bi, fma(-p.ar, ti, fma(p.ai, tr, bi)));
}

// Half-angle rotation for (|d|, p = g_tb): kk = (1/r)(1/c) with r = sqrt(d^2 + 4|p|^2),
// so that A = +-kk p, cm1 = -|s|^2 / (1 + c), dn = t |g| = |p|^2 kk / c.
__device__ __forceinline__ void cparams_core(double dabs, double pr, double pi, double& cm1, double& kk, double& dn) {
    const double q2 = fma(pr, pr, pi * pi);
    const double q = fma(4.0, q2, dabs * dabs);
    const double ir = rsqrt_cubic(q);
    const double c2 = fma(0.5 * dabs, ir, 0.5);
    const double ic = rsqrt_cubic(c2);
    const double c = c2 * ic;
    kk = ir * ic;
    cm1 = -(q2 * kk * kk) * rcp_cubic(1.0 + c);
    dn = q2 * kk * ic;
}
// -> cm1, (ar, ai) = kk p (the rotation's off-diagonal before its sign), dn
__device__ __forceinline__ void cparams(double dabs, double pr, double pi, double& cm1, double& ar, double& ai,
                                       double& dn) {
    double kk;
    cparams_core(dabs, pr, pi, cm1, kk, dn);
    ar = kk * pr;
    ai = kk * pi;
    if (fmax(dabs, fmax(fabs(pr), fabs(pi))) < 0x1p-500) {  // exact power-of-two rescale of tiny inputs
        // kk p = kk' (2^600 p) with kk' of the rescaled inputs: kk itself (~1/|p|) overflows for
        // subnormal p (columns graded over more than the exponent range), 2^600 p does not
        const double sr = pr * 0x1p+600, si = pi * 0x1p+600;
        cparams_core(dabs * 0x1p+600, sr, si, cm1, kk, dn);
        ar = kk * sr;
        ai = kk * si;
        dn *= 0x1p-600;
    }
}

struct Ctx {
    WarpSmem* sm;
    CtaSmem* cs;
    PSmem* ps;                 // smem P (SP kernels)
    const uint32_t* ctab;
    int lane, half, k, warp;
    int nww;                   // warps holding rows of W (the rest hold V rows / padding)
    bool wrow;                 // this lane holds a row of W
    double tol, tol2;
    bool want_p;
};

struct IState {
    int my_rot;  // rotations of pair k in this sweep (lanes < 16)
    bool full;   // this iteration reads fresh norms
    int par;     // cross-warp buffer parity
};

// SH != 0: the last iteration of an unrolled group with the ring shift by SH folded into the W update
// (results go straight to their post-shift registers; branch-free: pairs that do not rotate have zero
// parameters and copy exactly), so the loop back-edge moves no registers
// DELTA (k_cregb): the shared-memory P holds Delta = P - I, updated as Delta J + (J - I) (the reference's
// delta mode), J - I = [[cm1, -conj(A)], [A, cm1]] on (top, bottom) for the task rows ct and cb
template <int u, int NW, bool SP, int SH = 0, bool DELTA = false>
__device__ __forceinline__ void iter(double (&xr)[N], double (&xi)[N], const Ctx& c, int t, IState& st) {
    WarpSmem& sm = *c.sm;
    // ---- partial products of this lane's row: p_q = conj(x_b) x_t (V / padding lanes keep 0) ----
    if (SP || c.wrow) {  // SP: every lane is a W (or zero padding) row
#pragma unroll
        for (int q = 0; q < H; ++q) {
            const double tr = xr[TS(q, u)], ti = xi[TS(q, u)], br = xr[BS(q, u)], bi = xi[BS(q, u)];
            sm.red[q * RS2 + c.lane] = make_double2(fma(bi, ti, br * tr), fma(-bi, tr, br * ti));
        }
    }
    const uint32_t code = c.ctab[t * H + c.k];
    __syncwarp();
    double v[4];
    {
        const double2 g = sum32x2(sm.red, c.k, c.half);
        v[0] = g.x;
        v[1] = g.y;
    }
    int nval = 2;
    if (st.full) {  // fresh squared norms through the same buffer (rare: sweep start, >4x shrink)
        __syncwarp();
        if (SP || c.wrow) {
#pragma unroll
            for (int q = 0; q < H; ++q) {
                const double tr = xr[TS(q, u)], ti = xi[TS(q, u)], br = xr[BS(q, u)], bi = xi[BS(q, u)];
                sm.red[q * RS2 + c.lane] = make_double2(fma(ti, ti, tr * tr), fma(bi, bi, br * br));
            }
        }
        __syncwarp();
        const double2 gn = sum32x2(sm.red, c.k, c.half);
        v[2] = gn.x;
        v[3] = gn.y;
        nval = 4;
    }
    if constexpr (NW > 1) {  // sum over the CTA's warps: one barrier, fixed warp order
        double* g = c.cs->gsum[st.par][0];
        if (c.lane < H && (SP || c.warp < c.nww))
            for (int x = 0; x < nval; ++x) g[c.warp * 4 * H + x * H + c.k] = v[x];
        bar_named(NW * 32);
        for (int x = 0; x < nval; ++x) {
            double s = g[x * H + c.k];
#pragma unroll
            for (int w = 1; w < NW; ++w)
                if (SP || w < c.nww) s += g[w * 4 * H + x * H + c.k];
            v[x] = s;
        }
        st.par ^= 1;
    }
    // ---- rotation of pair k (every warp, identical bits) ----
    const int ct = code & 0xff, cb = (code >> 8) & 0xff;
    const bool flip = (code >> 16) != 0;
    const double pr = v[0], pi = v[1];
    const double gt = st.full ? v[2] : sm.nrm[ct];
    const double gb = st.full ? v[3] : sm.nrm[cb];
    const double q2 = fma(pr, pr, pi * pi);
    const double pp = gt * gb;
    const double pm = fmax(fabs(pr), fabs(pi));
    bool rot = !(q2 < c.tol2 * pp);
    if (pm < 0x1p-400 && pm > 0.0) {  // |g| from the rescaled components (squares would underflow)
        const double sr = pr * 0x1p+600, si = pi * 0x1p+600;
        rot = !(fsqrt(fma(sr, sr, si * si)) < c.tol * fsqrt(pp) * 0x1p+600);
    }
    rot = rot && pm > 0.0;
    const double d = gt - gb;
    double cm1, ar, ai, dn;
    cparams(fabs(d), pr, pi, cm1, ar, ai, dn);
    const bool eneg = d < 0.0 || (d == 0.0 && flip);
    Par par;
    par.cm1 = rot ? cm1 : 0.0;
    par.ar = rot ? (eneg ? -ar : ar) : 0.0;
    par.ai = rot ? (eneg ? -ai : ai) : 0.0;
    par.pad = 0.0;
    const double dtg = rot ? (eneg ? -dn : dn) : 0.0;
    const double nt = gt + dtg, nb = gb - dtg;
    const bool shrink = rot && (nt < 0.25 * gt || nb < 0.25 * gb);
    __syncwarp();  // every lane has read nrm[] and red[] of this iteration
    if (c.lane < H) {
        sm.pub[3 * c.k] = par.cm1;
        sm.pub[3 * c.k + 1] = par.ar;
        sm.pub[3 * c.k + 2] = par.ai;
        sm.nrm[ct] = nt;
        sm.nrm[cb] = nb;
        st.my_rot += rot ? 1 : 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, rot);
    st.full = __ballot_sync(0xffffffffu, shrink) != 0u;
    __syncwarp();
    if (SH == 0 && !mask) return;
    // ---- W update in registers (two pairs' parameters per three 16-byte loads) ----
    if constexpr (SH == 0) {
#pragma unroll
        for (int q = 0; q < H; q += 2) {
            const double2* pp = reinterpret_cast<const double2*>(sm.pub + 3 * q);
            const double2 a = pp[0], b = pp[1], d = pp[2];
            Par p0, p1;
            p0.cm1 = a.x;
            p0.ar = a.y;
            p0.ai = b.x;
            p1.cm1 = b.y;
            p1.ar = d.x;
            p1.ai = d.y;
            capply(xr[TS(q, u)], xi[TS(q, u)], xr[BS(q, u)], xi[BS(q, u)], p0);
            capply(xr[TS(q + 1, u)], xi[TS(q + 1, u)], xr[BS(q + 1, u)], xi[BS(q + 1, u)], p1);
        }
    } else {
        double yr[N], yi[N];
#pragma unroll
        for (int q = 0; q < H; q += 2) {
            const double2* pp = reinterpret_cast<const double2*>(sm.pub + 3 * q);
            const double2 a = pp[0], b = pp[1], d = pp[2];
            Par p0, p1;
            p0.cm1 = a.x;
            p0.ar = a.y;
            p0.ai = b.x;
            p1.cm1 = b.y;
            p1.ar = d.x;
            p1.ai = d.y;
            capply_to(xr[TS(q, u)], xi[TS(q, u)], xr[BS(q, u)], xi[BS(q, u)], yr[dst_slot(TS(q, u), SH)],
                      yi[dst_slot(TS(q, u), SH)], yr[dst_slot(BS(q, u), SH)], yi[dst_slot(BS(q, u), SH)], p0);
            capply_to(xr[TS(q + 1, u)], xi[TS(q + 1, u)], xr[BS(q + 1, u)], xi[BS(q + 1, u)],
                      yr[dst_slot(TS(q + 1, u), SH)], yi[dst_slot(TS(q + 1, u), SH)], yr[dst_slot(BS(q + 1, u), SH)],
                      yi[dst_slot(BS(q + 1, u), SH)], p1);
        }
#pragma unroll
        for (int col = 0; col < N; ++col) {
            xr[col] = yr[col];
            xi[col] = yi[col];
        }
        if (!mask) return;
    }
    // ---- P (= V) update in smem: task (row = lane, pair q) for q = warp, warp + NW, ... ----
    if (SP && c.want_p) {
        double2* P = c.ps->P;
        for (int q = c.warp; q < H; q += NW) {
            Par pq;
            pq.cm1 = sm.pub[3 * q];
            pq.ar = sm.pub[3 * q + 1];
            pq.ai = sm.pub[3 * q + 2];
            if (pq.cm1 == 0.0 && pq.ar == 0.0 && pq.ai == 0.0) continue;  // skipped pair (warp-uniform)
            const uint32_t cq = c.ctab[t * H + q];
            const int a0 = (cq & 0xff) * N + c.lane, b0 = ((cq >> 8) & 0xff) * N + c.lane;
            const double2 ta = P[a0], tb = P[b0];  // 16-byte accesses: 32 lanes, one column, conflict-free
            double tr = ta.x, ti = ta.y, br = tb.x, bi = tb.y;
            capply(tr, ti, br, bi, pq);
            if (DELTA) {
                const int ctq = cq & 0xff, cbq = (cq >> 8) & 0xff;
                if (c.lane == ctq) {
                    tr += pq.cm1;
                    br -= pq.ar;
                    bi += pq.ai;
                } else if (c.lane == cbq) {
                    tr += pq.ar;
                    ti += pq.ai;
                    br += pq.cm1;
                }
            }
            P[a0] = make_double2(tr, ti);
            P[b0] = make_double2(br, bi);
        }
    }
}

// one sweep (31 iterations, ring unrolled by 2); returns with the columns in natural order
template <int NW, bool SP, bool DELTA = false>
__device__ __forceinline__ void sweep(double (&xr)[N], double (&xi)[N], const Ctx& c, IState& st) {
    st.full = true;
#pragma unroll 1
    for (int gi = 0; gi < 16; ++gi) {
        const int t0 = 2 * gi;
        iter<0, NW, SP, 0, DELTA>(xr, xi, c, t0, st);
        if (gi == 15) {
            ring_shift<1>(xr);
            ring_shift<1>(xi);
            break;
        }
        iter<1, NW, SP, 2, DELTA>(xr, xi, c, t0 + 1, st);  // writes straight into the registers shifted by two
    }
}

__host__ __device__ inline size_t smem_bytes(int nw, bool sp) {
    return (size_t)nw * sizeof(WarpSmem) + sizeof(CtaSmem) + (sp ? sizeof(PSmem) : 0) + NIT * H * 4;
}
// TMA loader: staging for one whole problem (m x 32 complex) plus its mbarrier, behind the rest
__host__ __device__ inline size_t stage_offset(int nw, bool sp) { return (smem_bytes(nw, sp) + 127) & ~(size_t)127; }
// columns staged: as many as fit beside the kernel's own shared memory (C4, 256 x 32 with V as P in
// smem: 31 of 32; the last column is then read directly)
inline int staged_cols(int nw, bool sp, int m, size_t limit) {
    const size_t col = (size_t)m * sizeof(cx<double>);
    const size_t base = stage_offset(nw, sp) + 16;
    return limit <= base ? 0 : (int)std::min<size_t>(N, (limit - base) / col);
}
inline size_t smem_bytes_tma(int nw, bool sp, int m, int ncs) {
    return stage_offset(nw, sp) + (size_t)m * ncs * sizeof(cx<double>) + 16;
}

// NW warps; SP: V as the smem product P (m > 224), else V rows ride along in registers below
// W's rows (rows m .. m + 31 of the CTA, rotated like W, excluded from the dot products).
// TMA (variant 45): kernel (1) stages the problem into shared memory with one bulk copy per column
// (cp.async.bulk -> UBLKCP) completing on an mbarrier; without TMA (default): coalesced LDG.  One CTA
// per problem either way.
template <int NW, bool SP, bool TMA>
__global__ void __launch_bounds__(NW * 32, (8 / NW) > 0 ? (8 / NW) : 1)
    k_creg32(SolveArgs<cx<double>> a, int blocked, int ncs) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int m = a.bm;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    WarpSmem* wsm = reinterpret_cast<WarpSmem*>(smem);
    CtaSmem* cs = reinterpret_cast<CtaSmem*>(smem + NW * sizeof(WarpSmem));
    PSmem* ps = reinterpret_cast<PSmem*>(smem + NW * sizeof(WarpSmem) + sizeof(CtaSmem));
    uint32_t* ctab =
        reinterpret_cast<uint32_t*>(smem + NW * sizeof(WarpSmem) + sizeof(CtaSmem) + (SP ? sizeof(PSmem) : 0));
    cx<double>* stg = reinterpret_cast<cx<double>*>(smem + stage_offset(NW, SP));
    uint64_t* mbar = reinterpret_cast<uint64_t*>(stg + (size_t)m * ncs);
    const bool want_p = a.need_v != 0;
    for (int e = tid; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    const uint32_t stage_bytes = (uint32_t)(m * sizeof(cx<double>));
    // warp 0 puts problem q's first ncs columns in flight (lane = column)
    auto issue = [&](int q) {
        if (lane == 0) tma::mbar_arrive_expect(mbar, stage_bytes * ncs);
        __syncwarp();
        if (lane < ncs)
            tma::bulk_g2s(stg + (size_t)lane * m, a.A + (size_t)q * a.strideA + (size_t)lane * a.lda, stage_bytes,
                          mbar);
    };
    if constexpr (TMA) {
        if (tid == 0) {
            tma::mbar_init(mbar, 1);
            tma::fence_mbar_init();
        }
        __syncthreads();
        if (warp == 0 && blockIdx.x < a.batch) issue(blockIdx.x);
    }
    uint32_t phase = 0;
#pragma unroll 1
    for (int prob = blockIdx.x; prob < a.batch; prob = a.batch) {  // one problem per CTA
        for (int e = lane; e < H * RS2; e += 32) wsm[warp].red[e] = make_double2(0.0, 0.0);  // V / padding lanes stay 0
        if (tid < 4) cs->misc[tid] = 0;
        if (SP && want_p)
            for (int e = tid; e < N * N; e += NW * 32) {
                const int r = e % N, col = e / N;
                ps->P[col * N + r] = make_double2((r == col) ? 1.0 : 0.0, 0.0);
            }
        // ---- kernel (1): this lane's row of A, exact power-of-two prescale ----
        const int row = warp * 32 + lane;
        const bool live = row < m;
        const int vrow = (!SP && want_p && row >= m && row < m + N) ? row - m : -1;  // row of V this lane holds
        double xr[N], xi[N];
        double amax = 0.0;
        int bad = 0;
        if constexpr (TMA) {
            tma::mbar_wait(mbar, phase);
            phase ^= 1u;
        }
        {
            const cx<double>* Ap = a.A + (size_t)prob * a.strideA;
#pragma unroll
            for (int col = 0; col < N; ++col) {
                cx<double> z{0.0, 0.0};
                if (live) z = (TMA && col < ncs) ? stg[row + (size_t)col * m] : Ap[row + (size_t)col * a.lda];
                xr[col] = z.re;
                xi[col] = z.im;
                bad |= !(isfinite(z.re) && isfinite(z.im));
                amax = fmax(amax, fmax(fabs(z.re), fabs(z.im)));
            }
        }
        __syncthreads();  // (TMA) every lane has its row: the staging buffer is free
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        }
        if (lane == 0) {
            if (bad) atomicOr(&cs->misc[0], 1);
            atomicMax(reinterpret_cast<unsigned long long*>(&cs->misc[2]),
                      (unsigned long long)__double_as_longlong(amax));
        }
        __syncthreads();
        const int ex = prescale_exponent(__longlong_as_double(*reinterpret_cast<long long*>(&cs->misc[2])));
        {
            const double sc = pow2(-ex);
#pragma unroll
            for (int col = 0; col < N; ++col) {
                xr[col] = vrow >= 0 ? (col == vrow ? 1.0 : 0.0) : xr[col] * sc;  // V = I
                xi[col] *= sc;
            }
        }
        Ctx c;
        c.sm = &wsm[warp];
        c.cs = cs;
        c.ctab = ctab;
        c.lane = lane;
        c.half = lane >> 4;
        c.k = lane & 15;
        c.warp = warp;
        c.ps = ps;
        c.nww = (m + 31) / 32;
        c.wrow = live;
        c.tol = a.tol;
        c.tol2 = a.tol * a.tol;
        c.want_p = want_p;
        const int budget = blocked ? a.inner_budget : 1;
        int sweeps = 0, last = 0, conv = 0;
        long long rot_total = 0, grams = 0, updates = 0;
        IState st;
        st.par = 0;
#pragma unroll 1
        for (int sw = 0; sw < a.max_sweeps; ++sw) {
            int bp_rot = 0;
#pragma unroll 1
            for (int isw = 0; isw < budget; ++isw) {
                st.my_rot = 0;
                sweep<NW, SP>(xr, xi, c, st);
                int r = st.my_rot;  // lanes 0..15: counts of pairs 0..15 (identical in every warp)
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
                r = __shfl_sync(0xffffffffu, r, 0);
                bp_rot += r;
                if (r == 0) break;
            }
            ++grams;
            updates += bp_rot ? 1 : 0;
            sweeps = sw + 1;
            last = bp_rot;
            rot_total += bp_rot;
            if (bp_rot == 0) {
                conv = 1;
                break;
            }
        }
        // ---- raw W (unscaled) and V = P to the workspace for the finalisation pass ----
        cx<double>* W = a.work + (size_t)prob * (size_t)a.work_stride;
        if (live) {
            const double us = pow2(ex);
#pragma unroll
            for (int col = 0; col < N; ++col) W[row + (size_t)col * m] = cx<double>{xr[col] * us, xi[col] * us};
        }
        if (SP && want_p) {
            __syncthreads();
            cx<double>* V = W + (size_t)m * N;
            for (int e = tid; e < N * N; e += NW * 32) {
                const int r = e % N, col = e / N;
                const double2 z = ps->P[col * N + r];
                V[e] = cx<double>{z.x, z.y};
            }
        }
        if (vrow >= 0) {
            cx<double>* V = W + (size_t)m * N;
#pragma unroll
            for (int col = 0; col < N; ++col) V[vrow + (size_t)col * N] = cx<double>{xr[col], xi[col]};
        }
        if (tid == 0 && a.info) {
            bsvd_info inf;
            inf.converged = conv;
            inf.outer_sweeps = sweeps;
            inf.rotations = rot_total;
            inf.gram_calls = blocked ? grams : 0;
            inf.update_calls = blocked ? updates : 0;
            inf.last_rotations = last;
            inf.path = blocked ? 2 : 1;
            inf.status = cs->misc[0] ? 1 : 0;
            inf.kernel = a.kernel;
            a.info[prob] = inf;
        }
        __syncthreads();  // shared state (red, misc, P, gsum) is re-initialised for the next problem
    }
}

// Blocked complex FP64, n > 32 (n % 16 == 0, m <= 256): the outer round-robin over the l = n / 16 column
// blocks of _sweep_blocked (src/svd.py:481-522); each block pair X = [Wi Wj] (m x 32) is solved by this
// file's register iteration in its P-in-shared-memory form (the inner eigensolve of the block pair's
// Gram is one-sided Jacobi on X itself: the same rotations, G never formed), then X is written back and
// [Vi Vj] <- [Vi Vj] P (the fused update of src/_kernels_numba.py:141-175) row by row from the
// workspace.  One CTA per problem, block pairs of an outer iteration in turn; W and V live in the
// (L2-resident) workspace, finalised by the standalone pass.
// DELTA (more than 4 column blocks or inner sweeps != 1): P accumulates Delta = P - I and both W and V are
// updated once per round as M + M Delta from the unrotated workspace copy (one rounding per round instead of
// one per rotation on W; c128 128x128 Frobenius-mass drift 35.9u -> see profiles)
template <int NW, bool DELTA = false>
__global__ void __launch_bounds__(NW * 32, (8 / NW) > 0 ? (8 / NW) : 1) k_cregb(SolveArgs<cx<double>> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int m = a.bm, n = a.bn, prob = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    WarpSmem* wsm = reinterpret_cast<WarpSmem*>(smem);
    CtaSmem* cs = reinterpret_cast<CtaSmem*>(smem + NW * sizeof(WarpSmem));
    PSmem* ps = reinterpret_cast<PSmem*>(smem + NW * sizeof(WarpSmem) + sizeof(CtaSmem));
    uint32_t* ctab = reinterpret_cast<uint32_t*>(smem + NW * sizeof(WarpSmem) + sizeof(CtaSmem) + sizeof(PSmem));
    const bool want_p = a.need_v != 0;
    const int ell = n / 16, Sb = ell + (ell & 1), nib = Sb - 1, hb = Sb / 2;
    cx<double>* W = a.work + (size_t)prob * (size_t)a.work_stride;  // m x n, then V n x n
    cx<double>* V = W + (size_t)m * n;
    for (int e = tid; e < NIT * H; e += NW * 32) ctab[e] = pair_code(e / H, e % H);
    if (tid < 4) cs->misc[tid] = 0;
    __syncthreads();
    // ---- kernel (1): A -> W with an exact power-of-two prescale, V = I ----
    {
        const cx<double>* Ap = a.A + (size_t)prob * a.strideA;
        double amax = 0.0;
        int bad = 0;
        for (int e = tid; e < m * n; e += NW * 32) {
            const cx<double> z = Ap[(e % m) + (size_t)(e / m) * a.lda];
            bad |= !(isfinite(z.re) && isfinite(z.im));
            amax = fmax(amax, fmax(fabs(z.re), fabs(z.im)));
        }
        if (bad) atomicOr(&cs->misc[0], 1);
        atomicMax(reinterpret_cast<unsigned long long*>(&cs->misc[2]), (unsigned long long)__double_as_longlong(amax));
        __syncthreads();
        const double sc = pow2(-prescale_exponent(__longlong_as_double(*reinterpret_cast<long long*>(&cs->misc[2]))));
        for (int e = tid; e < m * n; e += NW * 32) {
            const cx<double> z = Ap[(e % m) + (size_t)(e / m) * a.lda];
            W[e] = cx<double>{z.re * sc, z.im * sc};
        }
        if (want_p)
            for (int e = tid; e < n * n; e += NW * 32) V[e] = cx<double>{(e % n) == (e / n) ? 1.0 : 0.0, 0.0};
        __syncthreads();
    }
    const int ex = prescale_exponent(__longlong_as_double(*reinterpret_cast<long long*>(&cs->misc[2])));
    const int row = warp * 32 + lane;
    const bool live = row < m;
    Ctx c;
    c.sm = &wsm[warp];
    c.cs = cs;
    c.ctab = ctab;
    c.lane = lane;
    c.half = lane >> 4;
    c.k = lane & 15;
    c.warp = warp;
    c.ps = ps;
    c.nww = (m + 31) / 32;
    c.wrow = live;
    c.tol = a.tol;
    c.tol2 = a.tol * a.tol;
    c.want_p = want_p;
    const int budget = a.inner_budget;
    int sweeps = 0, last = 0, conv = 0;
    long long rot_total = 0, grams = 0, updates = 0;
    double xr[N], xi[N];
#pragma unroll 1
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        long long sweep_rot = 0;
#pragma unroll 1
        for (int tb = 0; tb < nib; ++tb) {
#pragma unroll 1
            for (int g = 0; g < hb; ++g) {
                int bi = 0, bj = 0;
                if (!rr_pair(tb, g, Sb, ell, bi, bj)) continue;  // phantom block (odd l)
                auto col = [&](int x) { return x < 16 ? bi * 16 + x : bj * 16 + x - 16; };
                // X = [Wi Wj]: this lane's row; P = I; transpose buffers cleared (padding lanes read 0)
#pragma unroll
                for (int x = 0; x < N; ++x) {
                    const cx<double> z = live ? W[row + (size_t)col(x) * m] : cx<double>{0.0, 0.0};
                    xr[x] = z.re;
                    xi[x] = z.im;
                }
                for (int e = lane; e < H * RS2; e += 32) wsm[warp].red[e] = make_double2(0.0, 0.0);
                if (want_p || DELTA)
                    for (int e = tid; e < N * N; e += NW * 32)
                        ps->P[e] = make_double2((!DELTA && (e % N) == (e / N)) ? 1.0 : 0.0, 0.0);
                __syncthreads();
                IState st;
                st.par = 0;
                int bp_rot = 0;
#pragma unroll 1
                for (int isw = 0; isw < budget; ++isw) {
                    st.my_rot = 0;
                    sweep<NW, true, DELTA>(xr, xi, c, st);
                    int r = st.my_rot;  // lanes 0..15: counts of pairs 0..15 (identical in every warp)
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
                    r = __shfl_sync(0xffffffffu, r, 0);
                    bp_rot += r;
                    if (r == 0) break;
                }
                ++grams;
                sweep_rot += bp_rot;
                if (bp_rot) {
                    ++updates;
                    if (!DELTA && live) {
#pragma unroll
                        for (int x = 0; x < N; ++x) W[row + (size_t)col(x) * m] = cx<double>{xr[x], xi[x]};
                    }
                    // [Mi Mj] <- [Mi Mj] P (V) or [Mi Mj] + [Mi Mj] Delta (DELTA: W and V), one row per thread
                    // (the rows of X are free registers now)
                    auto rows_update = [&](cx<double>* M, int ld, int nrows) {
                        for (int vr = tid; vr < nrows; vr += NW * 32) {
#pragma unroll
                            for (int x = 0; x < N; ++x) {
                                const cx<double> z = M[vr + (size_t)col(x) * ld];
                                xr[x] = z.re;
                                xi[x] = z.im;
                            }
#pragma unroll 4
                            for (int y = 0; y < N; ++y) {
                                double sr = 0.0, si = 0.0;
#pragma unroll
                                for (int x = 0; x < N; ++x) {
                                    const double2 p = ps->P[y * N + x];  // P[x][y], column-major
                                    sr = fma(xr[x], p.x, fma(-xi[x], p.y, sr));
                                    si = fma(xr[x], p.y, fma(xi[x], p.x, si));
                                }
                                M[vr + (size_t)col(y) * ld] = DELTA ? cx<double>{xr[y] + sr, xi[y] + si} : cx<double>{sr, si};
                            }
                        }
                    };
                    if (want_p || DELTA) __syncthreads();  // P complete
                    if (DELTA) rows_update(W, m, m);
                    if (want_p) rows_update(V, n, n);
                }
                __syncthreads();  // the next block pair reads the columns written here
            }
        }
        sweeps = sw + 1;
        last = (int)sweep_rot;
        rot_total += sweep_rot;
        if (sweep_rot == 0) {
            conv = 1;
            break;
        }
    }
    {
        const double us = pow2(ex);
        for (int e = tid; e < m * n; e += NW * 32) W[e] = cx<double>{W[e].re * us, W[e].im * us};
    }
    if (tid == 0 && a.info) {
        bsvd_info inf;
        inf.converged = conv;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = grams;
        inf.update_calls = updates;
        inf.last_rotations = last;
        inf.path = 2;
        inf.status = cs->misc[0] ? 1 : 0;
        inf.kernel = a.kernel;
        a.info[prob] = inf;
    }
}

}  // namespace creg

Plan plan_creg32(int dtype, int bm, int bn, int need_v, bool contiguous, int blocked, int nb, int variant,
                 size_t smem_limit) {
    Plan p{};
    if (dtype != BSVD_Z || bn != 32 || bm < 32 || bm > 256 || !contiguous) return p;
    if (blocked && nb != 16) return p;  // one block pair = the whole matrix only when nb = 16
    const int rows = bm + (need_v ? 32 : 0);  // V rows ride in registers when they fit
    const bool sp = rows > 256;
    const int nw = ((sp ? bm : rows) + 31) / 32;
    p.kernel = variant == KV_CREG32_TMA ? KV_CREG32_TMA : KV_CREG32;
    p.threads = nw * 32;
    p.group = nw | (sp ? 0x100 : 0);
    p.smem = creg::smem_bytes(nw, sp);
    if (p.kernel == KV_CREG32_TMA) {
        p.aux = creg::staged_cols(nw, sp, bm, smem_limit);
        p.smem = creg::smem_bytes_tma(nw, sp, bm, p.aux);
    }
    p.work_elems = (size_t)bm * bn + (need_v ? (size_t)bn * bn : 0);
    p.grid = 0;
    p.resident = blocked ? 1 : 0;  // route flag for the launcher
    return p;
}

Plan plan_cregb(int dtype, int bm, int bn, int need_v, bool trans, int nb) {
    Plan p{};
    if (dtype != BSVD_Z || trans || nb != 16 || bn <= 32 || bn % 16 != 0 || bm < bn || bm > 256) return p;
    const int nw = (bm + 31) / 32;
    p.kernel = KV_CREGB;
    p.threads = nw * 32;
    p.group = nw;
    p.smem = creg::smem_bytes(nw, true);
    p.work_elems = (size_t)bm * bn + (need_v ? (size_t)bn * bn : 0);
    return p;
}

template <int NW>
static int launch_cb(SolveArgs<cx<double>> a, const Plan& p, cudaStream_t st) {
    // delta mode as in the real blocked kernel: more than 4 column blocks or inner sweeps other than one
    auto k = (a.bn > 64 || a.inner_budget != 1) ? creg::k_cregb<NW, true> : creg::k_cregb<NW, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<a.batch, NW * 32, p.smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_cregb(SolveArgs<cx<double>> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    int rc;
    switch (p.group) {
        case 2: rc = launch_cb<2>(a, p, st); break;
        case 3: rc = launch_cb<3>(a, p, st); break;
        case 4: rc = launch_cb<4>(a, p, st); break;
        case 5: rc = launch_cb<5>(a, p, st); break;
        case 6: rc = launch_cb<6>(a, p, st); break;
        case 7: rc = launch_cb<7>(a, p, st); break;
        case 8: rc = launch_cb<8>(a, p, st); break;
        default: return BSVD_ERR_UNSUPPORTED;
    }
    if (rc) return rc;
    return launch_finalize_gm<cx<double>>(a, st);
}

template <int NW, bool SP>
static int launch_c(SolveArgs<cx<double>> a, const Plan& p, cudaStream_t st) {
    auto k = p.kernel == KV_CREG32_TMA ? creg::k_creg32<NW, SP, true> : creg::k_creg32<NW, SP, false>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<a.batch, NW * 32, p.smem, st>>>(a, p.resident, p.aux);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_creg32(SolveArgs<cx<double>> a, const Plan& p, cudaStream_t st) {
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    int rc;
    switch (p.group) {
        case 1: rc = launch_c<1, false>(a, p, st); break;
        case 2: rc = launch_c<2, false>(a, p, st); break;
        case 3: rc = launch_c<3, false>(a, p, st); break;
        case 4: rc = launch_c<4, false>(a, p, st); break;
        case 5: rc = launch_c<5, false>(a, p, st); break;
        case 6: rc = launch_c<6, false>(a, p, st); break;
        case 7: rc = launch_c<7, false>(a, p, st); break;
        case 8: rc = launch_c<8, false>(a, p, st); break;
        case 8 | 0x100: rc = launch_c<8, true>(a, p, st); break;
        default: return BSVD_ERR_UNSUPPORTED;
    }
    if (rc) return rc;
    return launch_finalize_gm<cx<double>>(a, st);
}

}  // namespace bsvd
