// blocked_dmma.cu -- kernel (3), blocked one-sided Jacobi on FP64 tensor cores.
//
// Restates _sweep_blocked (src/svd.py:481-522) for real float64, nb = 16
// (w = 2 nb = 32), n a multiple of 16: per block pair (i, j) of the
// round-robin schedule over ell = n/16 blocks (src/ordering.py:32-75)
//   compute_gram  G = [Wi Wj]^T [Wi Wj]            (src/svd.py:144-179)
//   _eig_delta    inner sweep(s) of two-sided Jacobi on G with
//                 Delta = P - I accumulation        (src/eig.py:151-174,
//                                                    src/_kernels_numba.py:17-82)
//   fused update  [Wi Wj] += [Wi Wj] Delta, V too   (src/_kernels_numba.py:141-175)
// and a sweep whose pairs all had zero inner rotations ends the problem.
//
// B200 mapping (one CTA of 256 threads per problem):
//  * W (and V when it fits) resident in shared memory for the whole solve,
//    column-major with a padded leading dimension (bank spread of DMMA
//    fragment loads); V of larger problems stays in global memory (L2).
//  * The ell/2 block pairs of a schedule iteration are disjoint (F9) and run
//    concurrently, one warp group per pair (named barriers per group).
//  * Gram and update are DMMA m8n8k4 tiles (mma.sync ... f64: SASS DMMA.8x8x4,
//    the FP64 tensor pipe): the Gram as the 10 upper 8x8 tiles of X^T X over
//    the m rows, mirrored exactly; the update as 8-row blocks x 4 column tiles
//    with the accumulator initialised to the block itself (the "+W" of
//    W + W Delta fused into the MMA, one rounding per element chain).
//  * The inner eigensolve keeps G and Delta in shared memory: the 16 disjoint
//    rotations of an inner iteration get their parameters from 16 lanes
//    (call-free rotation_tsc), then the group updates every 2x2 block of G
//    (rotation p on its rows, then q on its columns -- the reference's order
//    for p < q -- mirror written exactly) and the Delta columns.
//  * Data are pre-scaled by an exact power of two (undone before finalize).
#include "kernel_args.cuh"
#include "launch.h"
#include "rotation.cuh"

namespace bsvd {
namespace bdmma {

constexpr int WB = 32;    // Gram width 2 nb
constexpr int HB = 16;    // inner pairs per iteration
constexpr int GLD = 34;   // leading dimension of G / Delta in smem (16-byte column shift: conflict-free LDS.128)

struct InnerPar {
    double cm1, ws;  // real: wsc == ws
    int i, j, rot, pad;
};

struct GroupSmem {
    double G[WB * GLD];
    double D[WB * GLD];
    double d[WB];
    InnerPar prm[2][HB];  // rotation parameters, double-buffered by iteration parity
    int cnt[2];           // inner rotations per inner sweep (by sweep parity)
    int pad[2];
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// x <- x + (cm1 x + b y), y <- y + (cm1 y - a x)   (rot_pair with real ws/wsc)
__device__ __forceinline__ void rot2(double& x, double& y, double cm1, double a, double b) {
    const double nx = x + fma(cm1, x, b * y);
    const double ny = y + fma(cm1, y, -(a * x));
    x = nx;
    y = ny;
}

// Rotation of inner pair (i, j) from g = G[i][j] (reference eig_sweeps guard and
// formulas, src/_kernels_numba.py:35-60): zeroes the pivot and updates d when it rotates.
__device__ __forceinline__ void inner_params(GroupSmem& S, int i, int j, double g, double tol, InnerPar& pr,
                                             int* cnt) {
    pr.i = i;
    pr.j = j;
    pr.rot = 0;
    pr.cm1 = 0.0;
    pr.ws = 0.0;
    const double absg = fabs(g);
    const double di = S.d[i], dj = S.d[j];
    if (!(absg <= 0.0) && !(absg < tol * fsqrt(fabs(di) * fabs(dj)))) {
        double t, s, cm1;
        rotation_tsc(di - dj, absg, t, s, cm1);
        pr.rot = 1;
        pr.cm1 = cm1;
        pr.ws = g >= 0.0 ? s : -s;  // w s, w = g_ij / |g_ij|
        const double td = t * absg;
        S.d[i] = di + td;
        S.d[j] = dj - td;
        S.G[i + j * GLD] = 0.0;  // g_ij = g_ji = 0 after the rotation
        S.G[j + i * GLD] = 0.0;
        atomicAdd(cnt, 1);
    }
}

// One group's inner eigensolve on G (zero diagonal) / d, accumulating Delta
// (initialised to 0).  Returns the inner rotations of the counted sweeps.
//
// One barrier per inner iteration.  The ring of the tournament makes pair k'
// of iteration t+1 draw its two columns from pairs (k'-1, k'+1) of iteration t
// (k' = 0: (0,1), k' = 15: (14,15)), so the thread owning 2x2 block
// (k'-1, k'+1) evaluates pair k''s rotation right after updating that block;
// parameters are double-buffered by iteration parity.  An evaluation past the
// last counted sweep only touches G and d, which are discarded (Delta is what
// leaves the eigensolve), so speculating one iteration ahead is exact.
// Delta columns: thread -> (pair p = gtid % 16, a contiguous chunk of rows),
// 16-byte shared-memory accesses, parameters loaded once per iteration.
template <int GT>
__device__ __noinline__ long long inner_eig(GroupSmem& S, int gtid, int bar_id, int budget, double tol) {
    constexpr int NCH = GT / 16;        // row chunks per pair
    constexpr int RPC = WB / NCH;       // rows per chunk (16, 8, 4 or 2)
    constexpr int NOWN = (120 + GT - 1) / GT;
    if (gtid < HB) {
        int i, j;
        rr_pair(0, gtid, WB, WB, i, j);
        InnerPar pr;
        inner_params(S, i, j, S.G[i + j * GLD], tol, pr, &S.cnt[0]);
        S.prm[0][gtid] = pr;
    }
    group_bar(bar_id, GT);
    int bp[NOWN], bq[NOWN];
#pragma unroll
    for (int o = 0; o < NOWN; ++o) {
        const int blk = gtid + o * GT;
        bp[o] = -1;
        bq[o] = -1;
        if (blk < 120) {
            int P = 0, rem = blk;
            while (rem >= 15 - P) {
                rem -= 15 - P;
                ++P;
            }
            bp[o] = P;
            bq[o] = P + 1 + rem;
        }
    }
    const int dp = gtid & 15, r0 = (gtid >> 4) * RPC;  // Delta task
    long long pair_rot = 0;
    int it = 0;
    for (int isw = 0; isw < budget; ++isw) {
        for (int tw = 0; tw < WB - 1; ++tw, ++it) {
            const InnerPar* cur = S.prm[it & 1];
            InnerPar* nxt = S.prm[(it + 1) & 1];
            const int tn = (tw + 1 == WB - 1) ? 0 : tw + 1;  // next iteration in the ring
            int* ncnt = &S.cnt[(tw + 1 == WB - 1 ? isw + 1 : isw) & 1];
#pragma unroll
            for (int ob = 0; ob < NOWN; ++ob) {
                const int P = bp[ob], Q = bq[ob];
                if (P < 0) continue;
                const int nk = (P == 0 && Q == 1) ? 0 : (P == 14 && Q == 15) ? 15 : (Q == P + 2 ? P + 1 : -1);
                const InnerPar Pp = cur[P], Qp = cur[Q];
                if (!Pp.rot && !Qp.rot && nk < 0) continue;
                double x00 = S.G[Pp.i + Qp.i * GLD], x01 = S.G[Pp.i + Qp.j * GLD];
                double x10 = S.G[Pp.j + Qp.i * GLD], x11 = S.G[Pp.j + Qp.j * GLD];
                if (Pp.rot) {  // rows i_p, j_p: g_iq + (cm1 g_iq + ws g_jq), g_jq + (cm1 g_jq - wsc g_iq)
                    rot2(x00, x10, Pp.cm1, Pp.ws, Pp.ws);
                    rot2(x01, x11, Pp.cm1, Pp.ws, Pp.ws);
                }
                if (Qp.rot) {  // columns i_q, j_q
                    rot2(x00, x01, Qp.cm1, Qp.ws, Qp.ws);
                    rot2(x10, x11, Qp.cm1, Qp.ws, Qp.ws);
                }
                if (Pp.rot || Qp.rot) {
                    S.G[Pp.i + Qp.i * GLD] = x00;
                    S.G[Qp.i + Pp.i * GLD] = x00;
                    S.G[Pp.i + Qp.j * GLD] = x01;
                    S.G[Qp.j + Pp.i * GLD] = x01;
                    S.G[Pp.j + Qp.i * GLD] = x10;
                    S.G[Qp.i + Pp.j * GLD] = x10;
                    S.G[Pp.j + Qp.j * GLD] = x11;
                    S.G[Qp.j + Pp.j * GLD] = x11;
                }
                if (nk >= 0) {
                    int i, j;
                    rr_pair(tn, nk, WB, WB, i, j);
                    const bool ri = (i == Pp.i) || (i == Pp.j);  // i among the block's rows?
                    const int rr = ri ? i : j, cc = ri ? j : i;
                    const double g = (rr == Pp.i) ? ((cc == Qp.i) ? x00 : x01) : ((cc == Qp.i) ? x10 : x11);
                    InnerPar pr;
                    inner_params(S, i, j, g, tol, pr, ncnt);
                    nxt[nk] = pr;
                }
            }
            {
                const InnerPar Pd = cur[dp];
                if (Pd.rot) {
                    double* ci = &S.D[r0 + Pd.i * GLD];
                    double* cj = &S.D[r0 + Pd.j * GLD];
                    double xi[RPC], xj[RPC];
#pragma unroll
                    for (int v = 0; v < RPC; v += 2) {
                        const double2 a2 = *reinterpret_cast<const double2*>(ci + v);
                        const double2 b2 = *reinterpret_cast<const double2*>(cj + v);
                        xi[v] = a2.x;
                        xi[v + 1] = a2.y;
                        xj[v] = b2.x;
                        xj[v + 1] = b2.y;
                    }
#pragma unroll
                    for (int v = 0; v < RPC; ++v) {
                        rot2(xi[v], xj[v], Pd.cm1, Pd.ws, Pd.ws);  // Delta_:i + (cm1 Delta_:i + wsc Delta_:j) ...
                        const int r = r0 + v;
                        if (r == Pd.i) {  // identity contribution of P = I + Delta
                            xi[v] += Pd.cm1;
                            xj[v] -= Pd.ws;
                        }
                        if (r == Pd.j) {
                            xi[v] += Pd.ws;
                            xj[v] += Pd.cm1;
                        }
                    }
#pragma unroll
                    for (int v = 0; v < RPC; v += 2) {
                        *reinterpret_cast<double2*>(ci + v) = make_double2(xi[v], xi[v + 1]);
                        *reinterpret_cast<double2*>(cj + v) = make_double2(xj[v], xj[v + 1]);
                    }
                }
            }
            // counter of sweep isw+1 (= isw-1): every thread read it before phase (isw, 0)'s barrier
            if (tw == 1 && gtid == 0) S.cnt[(isw + 1) & 1] = 0;
            group_bar(bar_id, GT);
        }
        const int irot = S.cnt[isw & 1];
        pair_rot += irot;
        if (irot == 0) break;
    }
    return pair_rot;
}

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_blocked_dmma(SolveArgs<double> a) {
    constexpr int NWARP = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x;
    const int bm = a.bm, bn = a.bn;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;  // MMA fragment coordinates
    const int ldW = bm + 4, ldV = bn + 4;
    const bool v_smem = (a.resident & 2) != 0;
    const int ell = bn / 16;
    const int Sb = ell + (ell & 1), hb = Sb / 2, nib = Sb - 1;
    int ngp = 1;
    while (ngp < hb && ngp < NWARP && ngp < 8) ngp <<= 1;  // groups (power of two; named barriers 1..8)
    const int wg = NWARP / ngp;                  // warps per group
    const int grp = warp / wg, wig = warp % wg;
    const int gthreads = wg * 32, gtid = tid - grp * gthreads;

    size_t off = 0;
    double* W = reinterpret_cast<double*>(smem);
    off += (size_t)bn * ldW * sizeof(double);
    double* Vw = nullptr;
    int ldv_w = ldV;
    if (a.need_v) {
        if (v_smem) {
            Vw = reinterpret_cast<double*>(smem + off);
            off += (size_t)bn * ldV * sizeof(double);
        } else {
            Vw = a.work + (size_t)prob * a.work_stride;
            ldv_w = bn;
        }
    }
    off = (off + 15) & ~size_t(15);
    GroupSmem* gs = reinterpret_cast<GroupSmem*>(smem + off);
    off += (size_t)ngp * sizeof(GroupSmem);
    off = (off + 15) & ~size_t(15);
    double* sig = reinterpret_cast<double*>(smem + off);
    off += (size_t)bn * sizeof(double);
    int* perm = reinterpret_cast<int*>(smem + off);
    off += ((size_t)bn * sizeof(int) + 15) & ~size_t(15);
    int* misc = reinterpret_cast<int*>(smem + off);  // [0] sweep rot, [1] flag, [2] bad, [3] gram, [4] upd
    unsigned long long* amax_bits = reinterpret_cast<unsigned long long*>(misc + 6);
    if (tid < 6) misc[tid] = 0;
    if (tid == 0) *amax_bits = 0ull;
    __syncthreads();

    // ---- load W (kernel (1)), V = I, pre-scale by an exact power of two ----
    {
        const double* Ap = a.A + (size_t)prob * a.strideA;
        int bad = 0;
        double amax = 0.0;
        for (int e = tid; e < bm * bn; e += NT) {
            const int r = e % bm, c = e / bm;
            const double x = Ap[r + (size_t)c * a.lda];
            bad |= !isfinite(x);
            amax = fmax(amax, fabs(x));
            W[r + c * ldW] = x;
        }
        if (bad) atomicOr(&misc[2], 1);
        // non-negative doubles order like their bit patterns
        atomicMax(amax_bits, (unsigned long long)__double_as_longlong(amax));
        if (Vw)
            for (int e = tid; e < bn * bn; e += NT) {
                const int r = e % bn, c = e / bn;
                Vw[r + c * ldv_w] = (r == c) ? 1.0 : 0.0;
            }
    }
    __syncthreads();
    const int ex = prescale_exponent(__longlong_as_double((long long)*amax_bits));
    {
        const double sc = pow2(-ex);
        for (int e = tid; e < bm * bn; e += NT) W[e % bm + (e / bm) * ldW] *= sc;
    }
    __syncthreads();

    const double tol = a.tol;
    GroupSmem& S = gs[grp];
    const int bar_id = 1 + grp;
    int sweeps = 0, last = 0;
    bool conv = false;
    long long rot_total = 0;

    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        for (int tb = 0; tb < nib; ++tb) {
            for (int slot = grp; slot < hb; slot += ngp) {
                int bi, bj;
                if (!rr_pair(tb, slot, Sb, ell, bi, bj)) continue;  // phantom (odd ell): group idles
                const int i0 = bi * 16, j0 = bj * 16;
                auto wcol = [&](int x) -> double* { return W + (size_t)(x < 16 ? i0 + x : j0 + x - 16) * ldW; };
                // ---- 1. Gram on DMMA: 10 upper 8x8 tiles of X^T X ----
                for (int ti = wig; ti < 10; ti += wg) {
                    const int P = ti < 4 ? 0 : (ti < 7 ? 1 : (ti < 9 ? 2 : 3));
                    const int Q = ti < 4 ? ti : (ti < 7 ? ti - 3 : (ti < 9 ? ti - 5 : 3));
                    const double* xp = wcol(8 * P + g8);
                    const double* xq = wcol(8 * Q + g8);
                    double c0 = 0.0, c1 = 0.0;
                    for (int k = 0; k < bm; k += 4) dmma(c0, c1, xp[k + t4], xq[k + t4]);
                    // D[g8][2 t4 + e] = G[8P + g8][8Q + 2 t4 + e]
                    const int r = 8 * P + g8;
                    const int cA = 8 * Q + 2 * t4;
                    const double cv[2] = {c0, c1};
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int c = cA + e;
                        if (r == c) {
                            S.d[r] = cv[e];
                            S.G[r + c * GLD] = 0.0;
                        } else {
                            S.G[r + c * GLD] = cv[e];
                            S.G[c + r * GLD] = cv[e];  // exact mirror
                        }
                    }
                }
                for (int e = gtid; e < WB * WB; e += gthreads) S.D[(e & 31) + (e >> 5) * GLD] = 0.0;
                if (gtid == 0) {
                    S.cnt[0] = 0;
                    S.cnt[1] = 0;
                }
                group_bar(bar_id, gthreads);
                // ---- 2. inner eigensolve (inner_budget sweeps, early exit) ----
                long long pair_rot = 0;
                switch (gthreads) {
                    case 512: pair_rot = inner_eig<512>(S, gtid, bar_id, a.inner_budget, tol); break;
                    case 256: pair_rot = inner_eig<256>(S, gtid, bar_id, a.inner_budget, tol); break;
                    case 128: pair_rot = inner_eig<128>(S, gtid, bar_id, a.inner_budget, tol); break;
                    case 64: pair_rot = inner_eig<64>(S, gtid, bar_id, a.inner_budget, tol); break;
                    default: pair_rot = inner_eig<32>(S, gtid, bar_id, a.inner_budget, tol); break;
                }
                group_bar(bar_id, gthreads);  // every thread has read the counters before they are reused
                if (gtid == 0) {
                    atomicAdd(&misc[3], 1);
                    if (pair_rot) {
                        atomicAdd(&misc[0], (int)min(pair_rot, (long long)0x3fffffff));
                        atomicAdd(&misc[4], 1);
                    }
                }
                if (pair_rot) {
                    // ---- 3. fused update on DMMA: [Bi Bj] += [Bi Bj] Delta (W, then V) ----
                    for (int pass = 0; pass < (Vw ? 2 : 1); ++pass) {
                        double* B = pass == 0 ? W : Vw;
                        const int rows = pass == 0 ? bm : bn;
                        const int ld = pass == 0 ? ldW : ldv_w;
                        auto bcol = [&](int x) -> double* {
                            return B + (size_t)(x < 16 ? i0 + x : j0 + x - 16) * ld;
                        };
                        for (int rb = wig; rb < rows / 8; rb += wg) {
                            const int r0 = rb * 8;
                            double c[4][2];
#pragma unroll
                            for (int C = 0; C < 4; ++C) {
                                c[C][0] = bcol(8 * C + 2 * t4)[r0 + g8];
                                c[C][1] = bcol(8 * C + 2 * t4 + 1)[r0 + g8];
                            }
                            double af[8];
#pragma unroll
                            for (int ks = 0; ks < 8; ++ks) af[ks] = bcol(4 * ks + t4)[r0 + g8];
#pragma unroll
                            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
                                for (int C = 0; C < 4; ++C)
                                    dmma(c[C][0], c[C][1], af[ks], S.D[(4 * ks + t4) + (8 * C + g8) * GLD]);
#pragma unroll
                            for (int C = 0; C < 4; ++C) {
                                bcol(8 * C + 2 * t4)[r0 + g8] = c[C][0];
                                bcol(8 * C + 2 * t4 + 1)[r0 + g8] = c[C][1];
                            }
                        }
                    }
                }
                group_bar(bar_id, gthreads);  // G / Delta reused by this group's next slot
            }
            __syncthreads();  // every pair of this schedule iteration is updated
        }
        const int srot = misc[0];
        __syncthreads();
        if (tid == 0) misc[0] = 0;
        sweeps = sw + 1;
        last = srot;
        if (srot == 0) {
            conv = true;
            break;
        }
        rot_total += srot;
    }
    // ---- unscale and finalise (kernel 5) ----
    {
        const double us = pow2(ex);
        for (int e = tid; e < bm * bn; e += NT) W[e % bm + (e / bm) * ldW] *= us;
    }
    __syncthreads();
    finalize_block<double>(W, ldW, bm, bn, Vw, ldv_w, sig, perm, &misc[1], final_out(a, prob));
    if (tid == 0 && a.info) {
        bsvd_info inf;
        inf.converged = conv ? 1 : 0;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = misc[3];
        inf.update_calls = misc[4];
        inf.last_rotations = last;
        inf.path = 2;
        inf.status = misc[2] ? 1 : 0;
        inf.kernel = a.kernel;
        a.info[prob] = inf;
    }
}

size_t smem_bytes(int bm, int bn, bool v_smem, int nwarp) {
    const int ell = bn / 16;
    const int hb = (ell + (ell & 1)) / 2;
    int ngp = 1;
    while (ngp < hb && ngp < nwarp && ngp < 8) ngp <<= 1;
    size_t off = (size_t)bn * (bm + 4) * 8;
    if (v_smem) off += (size_t)bn * (bn + 4) * 8;
    off = (off + 15) & ~size_t(15);
    off += (size_t)ngp * sizeof(GroupSmem);
    off = (off + 15) & ~size_t(15);
    off += (size_t)bn * 8 + (((size_t)bn * 4 + 15) & ~size_t(15)) + 64;
    return off;
}

}  // namespace bdmma

// variants: KV_BLOCKED_DMMA    256 threads, <=128 regs, V in smem when it fits
//           KV_BLOCKED_DMMA_VG 256 threads, <= 85 regs (3 CTAs/SM), V in L2
//           KV_BLOCKED_DMMA_512 512 threads (16 warps for one-CTA-per-SM problems), V in smem if it fits
Plan plan_blocked_dmma(int dtype, int bm, int bn, int nb, int need_v, bool contiguous, size_t smem_limit,
                       int variant) {
    Plan p{};
    if (dtype != BSVD_D || nb != 16 || bn % 16 != 0 || bn < 32 || bm % 8 != 0 || !contiguous) return p;
    int kv = variant;
    if (kv != KV_BLOCKED_DMMA && kv != KV_BLOCKED_DMMA_VG && kv != KV_BLOCKED_DMMA_512) {
        // auto: 64x64-class problems run 3 CTAs/SM with V in L2; larger ones take 16 warps in one CTA
        kv = (bdmma::smem_bytes(bm, bn, false, 8) * 3 <= (size_t)228 * 1024) ? KV_BLOCKED_DMMA_VG
                                                                              : KV_BLOCKED_DMMA_512;
    }
    const int nwarp = kv == KV_BLOCKED_DMMA_512 ? 16 : 8;
    const size_t with_v = bdmma::smem_bytes(bm, bn, need_v != 0, nwarp);
    const size_t without_v = bdmma::smem_bytes(bm, bn, false, nwarp);
    const bool v_global = kv == KV_BLOCKED_DMMA_VG;
    if (need_v && !v_global && with_v <= smem_limit) {
        p.resident = 3;
        p.smem = with_v;
        p.work_elems = 0;
    } else if (without_v <= smem_limit) {
        p.resident = 1;
        p.smem = without_v;
        p.work_elems = need_v ? (size_t)bn * bn : 0;
    } else {
        return p;
    }
    p.kernel = kv;
    p.threads = nwarp * 32;
    return p;
}

template <int NT, int MINB>
static int launch_bd(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    auto k = bdmma::k_blocked_dmma<NT, MINB>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    // the occupancy of this kernel is shared-memory bound: ask for the largest carveout
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    k<<<a.batch, NT, p.smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_blocked_dmma(SolveArgs<double> a, const Plan& p, cudaStream_t st) {
    a.resident = p.resident;
    a.kernel = p.kernel;
    a.work_stride = (int64_t)p.work_elems;
    switch (p.kernel) {
        case KV_BLOCKED_DMMA_VG: return launch_bd<256, 3>(a, p, st);
        case KV_BLOCKED_DMMA_512: return launch_bd<512, 1>(a, p, st);
        default: return launch_bd<256, 2>(a, p, st);
    }
}

}  // namespace bsvd
