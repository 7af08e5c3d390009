// qr_reg.cu -- register-resident Householder QR and Q application for the
// "qr+" route on FP64 data (real and complex) with n <= 32, m <= 256: the
// tall-skinny shape of BASELINE config C4 (256 x 32 c128).
//
// Same algorithm and conventions as qr.cu (householder_qr, src/core.py:118-168;
// U = Q diag(p) U_R, src/svd.py:529-530): for k = 0 .. n-1
//   x = b[k:, k]; ||x|| in float64; phase = x0/|x0| (1 if x0 = 0);
//   v = x + phase ||x|| e1, v /= ||v||;  b[k:, k+1:] -= 2 v (v^H b[k:, k+1:]);
//   b[k, k] = -phase ||x||   (zero x or zero v: no reflector, v = 0 stored)
// and the left factor as H_0 ... H_{n-1} [diag(p) U_R; 0].
//
// B200 mapping: one CTA per problem, NW = ceil(m / 32) warps, lane l of warp w
// holds row 32 w + l of the working matrix (32 columns, real or complex) in
// registers; the column loop is fully unrolled so every register index is a
// compile-time constant and reflector k only touches columns j > k.  Per
// reflector: the column norm is an xor-butterfly warp sum plus one cross-warp
// slot (the diagonal entry rides along), and v^H b[:, j] for all trailing
// columns is a smem transpose per warp plus one cross-warp slot; every warp
// forms the same totals in the same order, so each reflector costs two
// barriers and no smem round trip of the matrix itself (the smem kernels in
// qr.cu stage all of b and synchronise ~6 times per column).
#include <type_traits>

#include "kernel_args.cuh"
#include "launch.h"
#include "rotation.cuh"

namespace bsvd {
namespace qreg {

constexpr int N = 32;
constexpr int RSTR = 34;
constexpr int MAXV = 64;  // values per reduction (32 complex columns)
constexpr int MAXW = 8;

struct WarpSm {
    double red[MAXV * RSTR];  // transpose buffer: one row per reduced value
    double pub[MAXV];         // CTA totals of the current reduction
};
struct CtaSm {
    double g[2][MAXW][MAXV + 4];  // cross-warp partials [parity][warp][value]; slots MAXV.. for the norm step
    double diag[2 * N];           // diagonal of R before the sign convention (re, im)
    int misc[4];
};

__device__ __forceinline__ double sum16(const double* p) {
    const double2* r = reinterpret_cast<const double2*>(p);
    const double2 p0 = r[0], p1 = r[1], p2 = r[2], p3 = r[3], p4 = r[4], p5 = r[5], p6 = r[6], p7 = r[7];
    const double s0 = (p0.x + p0.y) + (p1.x + p1.y), s1 = (p2.x + p2.y) + (p3.x + p3.y);
    const double s2 = (p4.x + p4.y) + (p5.x + p5.y), s3 = (p6.x + p6.y) + (p7.x + p7.y);
    return (s0 + s1) + (s2 + s3);
}
__device__ __forceinline__ double sum32(const double* red, int row, int half) {
    const double s = sum16(red + row * RSTR + 16 * half);
    const double o = __shfl_xor_sync(0xffffffffu, s, 16);
    return half ? o + s : s + o;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ void bar_cta(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

// CTA totals of red rows [0, NV) (written by the caller, who also did __syncwarp) into sm.pub
template <int NV, int NW>
__device__ __forceinline__ void reduce_publish(WarpSm& sm, CtaSm& cs, int lane, int warp, int& par) {
    const int half = lane >> 4, k16 = lane & 15;
    constexpr int NI = (NV + 15) / 16;
    double t[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) t[i] = sum32(sm.red, k16 + 16 * i, half);  // every lane: sum32 shuffles
    if constexpr (NW > 1) {
        if (lane < 16) {
#pragma unroll
            for (int i = 0; i < NI; ++i)
                if (k16 + 16 * i < NV) cs.g[par][warp][k16 + 16 * i] = t[i];
        }
        bar_cta(NW * 32);
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            if (k16 + 16 * i < NV) {
                double s = cs.g[par][0][k16 + 16 * i];
#pragma unroll
                for (int w = 1; w < NW; ++w) s += cs.g[par][w][k16 + 16 * i];
                t[i] = s;
            }
        }
        par ^= 1;
    }
    if (lane < 16) {
#pragma unroll
        for (int i = 0; i < NI; ++i)
            if (k16 + 16 * i < NV) sm.pub[k16 + 16 * i] = t[i];
    }
    __syncwarp();
}

// x / |x| for a complex (xr, xi), 1 for 0
__device__ __forceinline__ void cphase(double xr, double xi, double& pr, double& pi) {
    const double a2 = fma(xr, xr, xi * xi);
    if (a2 > 0.0) {
        const double inv = fdiv(1.0, fsqrt(a2));  // call-free (a CALL would spill the resident row)
        pr = xr * inv;
        pi = xi * inv;
    } else {
        pr = 1.0;
        pi = 0.0;
    }
}

template <bool CX>
struct Row {
    double re[N];
    double im[CX ? N : 1];
};

// one reflector (compile-time column K; the 32 steps are fully unrolled so reflector K only touches the
// 31 - K trailing columns -- measured faster than a rolled body with the active column shifted into a
// fixed slot, which does ~1.5x the reduction work)
template <bool CX, int NW, int K>
__device__ __forceinline__ void qr_step(Row<CX>& x, WarpSm& sm, CtaSm& cs, int lane, int warp, int row, int bm,
                                        int bn, bool live, int& par, double* vk) {
    if (K >= bn) return;
    // ---- ||b[K:, K]||^2 and the diagonal entry b[K, K] ----
    double a2 = 0.0;
    if (live && row >= K) a2 = CX ? fma(x.re[K], x.re[K], x.im[CX ? K : 0] * x.im[CX ? K : 0]) : x.re[K] * x.re[K];
    a2 = warp_sum(a2);
    double* g = cs.g[par][0];
    if (lane == 0) g[warp * (MAXV + 4) + MAXV] = a2;
    if (row == K) {
        cs.diag[2 * K] = x.re[K];
        cs.diag[2 * K + 1] = CX ? x.im[CX ? K : 0] : 0.0;
    }
    bar_cta(NW * 32);
    double s = g[MAXV];
#pragma unroll
    for (int w = 1; w < NW; ++w) s += g[w * (MAXV + 4) + MAXV];
    const double ar = cs.diag[2 * K], ai = cs.diag[2 * K + 1];
    par ^= 1;
    const double nx = fsqrt(s);
    double pr, pi;
    if (CX) {
        cphase(ar, ai, pr, pi);
    } else {
        pr = ar > 0.0 ? 1.0 : -1.0;  // unit_phase of a real: sign, 1 for 0 (src/core.py:135-137)
        if (!(ar * ar > 0.0)) pr = 1.0;
        pi = 0.0;
    }
    const double v0r = fma(pr, nx, ar), v0i = fma(pi, nx, ai);
    const double vn = fsqrt(fmax(s - fma(ar, ar, ai * ai), 0.0) + fma(v0r, v0r, v0i * v0i));
    const bool skip = !(nx > 0.0) || !(vn > 0.0);
    const double iv = skip ? 0.0 : fdiv(1.0, vn);
    double vr = 0.0, vi = 0.0;
    if (live && row == K) {
        vr = v0r * iv;
        vi = v0i * iv;
    } else if (live && row > K) {
        vr = x.re[K] * iv;
        vi = CX ? x.im[CX ? K : 0] * iv : 0.0;
    }
    if (live) {
        if (CX) reinterpret_cast<double2*>(vk)[row + (size_t)K * bm] = make_double2(vr, vi);
        else vk[row + (size_t)K * bm] = vr;
    }
    if (skip) return;  // CTA-uniform
    // ---- w_j = v^H b[:, j] for j > K ----
    constexpr int NC = N - 1 - K;          // trailing columns
    constexpr int NV = NC * (CX ? 2 : 1);  // reduced values
    if constexpr (NC > 0) {
#pragma unroll
        for (int j = K + 1; j < N; ++j) {
            const int c = j - K - 1;
            if (CX) {  // conj(v) b_j
                sm.red[(2 * c) * RSTR + lane] = fma(vi, x.im[CX ? j : 0], vr * x.re[j]);
                sm.red[(2 * c + 1) * RSTR + lane] = fma(-vi, x.re[j], vr * x.im[CX ? j : 0]);
            } else {
                sm.red[c * RSTR + lane] = vr * x.re[j];
            }
        }
        __syncwarp();
        reduce_publish<NV, NW>(sm, cs, lane, warp, par);
        // ---- b_j -= 2 v w_j ----
#pragma unroll
        for (int j = K + 1; j < N; ++j) {
            const int c = j - K - 1;
            if (CX) {
                const double2 w = reinterpret_cast<const double2*>(sm.pub)[c];
                const double wr = 2.0 * w.x, wi = 2.0 * w.y;
                x.re[j] = fma(-vr, wr, fma(vi, wi, x.re[j]));
                x.im[CX ? j : 0] = fma(-vr, wi, fma(-vi, wr, x.im[CX ? j : 0]));
            } else {
                x.re[j] = fma(-vr, 2.0 * sm.pub[c], x.re[j]);
            }
        }
        __syncwarp();  // pub / red reusable
    }
    if (row == K) {  // exact diagonal (src/core.py:142)
        x.re[K] = -pr * nx;
        if (CX) x.im[CX ? K : 0] = -pi * nx;
    }
}

template <bool CX, int NW, int K>
__device__ __forceinline__ void qr_all(Row<CX>& x, WarpSm& sm, CtaSm& cs, int lane, int warp, int row, int bm, int bn,
                                       bool live, int& par, double* vk) {
    if constexpr (K < N) {
        qr_step<CX, NW, K>(x, sm, cs, lane, warp, row, bm, bn, live, par, vk);
        qr_all<CX, NW, K + 1>(x, sm, cs, lane, warp, row, bm, bn, live, par, vk);
    }
}

template <bool CX>
using Elt = typename std::conditional<CX, cx<double>, double>::type;

template <bool CX, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_qr_reg(SolveArgs<Elt<CX>> a, Elt<CX>* R, Elt<CX>* refl,
                                                      Elt<CX>* phase) {
    using T = Elt<CX>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bm = a.bm, bn = a.bn;
    WarpSm& sm = reinterpret_cast<WarpSm*>(smem)[warp];
    CtaSm& cs = *reinterpret_cast<CtaSm*>(smem + NW * sizeof(WarpSm));
    const int row = warp * 32 + lane;
    const bool live = row < bm;
    const T* Ap = a.A + (size_t)prob * a.strideA;
    Row<CX> x;
    int bad = 0;
#pragma unroll
    for (int c = 0; c < N; ++c) {  // kernel (1): b = A, or A^H on the transpose route
        double re = 0.0, im = 0.0;
        if (live && c < bn) {
            const T z = a.trans ? Ap[c + (size_t)row * a.lda] : Ap[row + (size_t)c * a.lda];
            if constexpr (CX) {
                re = z.re;
                im = a.trans ? -z.im : z.im;
            } else {
                re = z;
            }
        }
        bad |= !(isfinite(re) && isfinite(im));
        x.re[c] = re;
        if (CX) x.im[CX ? c : 0] = im;
    }
    if (tid == 0) cs.misc[0] = 0;
    __syncthreads();
    if (bad) atomicOr(&cs.misc[0], 1);
    int par = 0;
    double* vk = reinterpret_cast<double*>(refl + (size_t)prob * bm * bn);
    qr_all<CX, NW, 0>(x, sm, cs, lane, warp, row, bm, bn, live, par, vk);
    // ---- sign convention: p_k = r_kk/|r_kk|, R row k *= conj(p_k), diagonal |r_kk| ----
    if (warp == 0) {
#pragma unroll
        for (int c = 0; c < N; ++c)
            if (lane == c) {
                cs.diag[2 * c] = x.re[c];
                cs.diag[2 * c + 1] = CX ? x.im[CX ? c : 0] : 0.0;
            }
    }
    __syncthreads();
    if (warp == 0 && lane < bn) {
        const double dr = cs.diag[2 * lane], di = cs.diag[2 * lane + 1];
        double pr, pi;
        if (CX) {
            cphase(dr, di, pr, pi);
        } else {
            pr = dr > 0.0 ? 1.0 : -1.0;
            if (!(dr * dr > 0.0)) pr = 1.0;
            pi = 0.0;
        }
        T* Rp = R + (size_t)prob * bn * bn;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            if (c >= bn) break;
            double yr = 0.0, yi = 0.0;
            if (c == lane) {
                yr = fsqrt(fma(dr, dr, di * di));
            } else if (c > lane) {  // x conj(p)
                const double xr = x.re[c], xi = CX ? x.im[CX ? c : 0] : 0.0;
                yr = fma(xr, pr, xi * pi);
                yi = fma(xi, pr, -xr * pi);
            }
            if constexpr (CX) Rp[lane + (size_t)c * bn] = T{yr, yi};
            else Rp[lane + (size_t)c * bn] = yr;
        }
        if constexpr (CX) phase[(size_t)prob * bn + lane] = T{pr, pi};
        else phase[(size_t)prob * bn + lane] = pr;
    }
    if (tid == 0 && a.info) a.info[prob].status = cs.misc[0];  // provisional; the inner solve rewrites info
}

// Out = H_0 ... H_{bn-1} [diag(p) U_R; 0]
template <bool CX, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_applyq_reg(int bm, int bn, const Elt<CX>* refl,
                                                          const Elt<CX>* phase, const Elt<CX>* UR, Elt<CX>* Out,
                                                          int64_t ldo, int64_t so) {
    using T = Elt<CX>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    WarpSm& sm = reinterpret_cast<WarpSm*>(smem)[warp];
    CtaSm& cs = *reinterpret_cast<CtaSm*>(smem + NW * sizeof(WarpSm));
    const int row = warp * 32 + lane;
    const bool live = row < bm;
    const T* Vk = refl + (size_t)prob * bm * bn;
    Row<CX> y;
    {
        double pr = 0.0, pi = 0.0;
        if (row < bn) {
            if constexpr (CX) {
                const T p = phase[(size_t)prob * bn + row];
                pr = p.re;
                pi = p.im;
            } else {
                pr = phase[(size_t)prob * bn + row];
            }
        }
        const T* U = UR + (size_t)prob * bn * bn;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            double ur = 0.0, ui = 0.0;
            if (row < bn && c < bn) {
                if constexpr (CX) {
                    const T z = U[row + (size_t)c * bn];
                    ur = z.re;
                    ui = z.im;
                } else {
                    ur = U[row + (size_t)c * bn];
                }
            }
            y.re[c] = fma(pr, ur, -pi * ui);  // p_r u_rc
            if (CX) y.im[CX ? c : 0] = fma(pr, ui, pi * ur);
        }
    }
    int par = 0;
    // reflectors in reverse order; v_k for this row prefetched one step ahead
    double vr = 0.0, vi = 0.0;
    if (live && bn > 0) {
        if constexpr (CX) {
            const T z = Vk[row + (size_t)(bn - 1) * bm];
            vr = z.re;
            vi = z.im;
        } else {
            vr = Vk[row + (size_t)(bn - 1) * bm];
        }
    }
#pragma unroll 1
    for (int k = bn - 1; k >= 0; --k) {
        double nr = 0.0, ni = 0.0;
        if (live && k > 0) {
            if constexpr (CX) {
                const T z = Vk[row + (size_t)(k - 1) * bm];
                nr = z.re;
                ni = z.im;
            } else {
                nr = Vk[row + (size_t)(k - 1) * bm];
            }
        }
        // w_j = v^H y_j (all columns)
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (CX) {
                sm.red[(2 * j) * RSTR + lane] = fma(vi, y.im[CX ? j : 0], vr * y.re[j]);
                sm.red[(2 * j + 1) * RSTR + lane] = fma(-vi, y.re[j], vr * y.im[CX ? j : 0]);
            } else {
                sm.red[j * RSTR + lane] = vr * y.re[j];
            }
        }
        __syncwarp();
        reduce_publish<(CX ? 2 * N : N), NW>(sm, cs, lane, warp, par);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (CX) {
                const double2 w = reinterpret_cast<const double2*>(sm.pub)[j];
                const double wr = 2.0 * w.x, wi = 2.0 * w.y;
                y.re[j] = fma(-vr, wr, fma(vi, wi, y.re[j]));
                y.im[CX ? j : 0] = fma(-vr, wi, fma(-vi, wr, y.im[CX ? j : 0]));
            } else {
                y.re[j] = fma(-vr, 2.0 * sm.pub[j], y.re[j]);
            }
        }
        __syncwarp();
        vr = nr;
        vi = ni;
    }
    if (live) {
        T* O = Out + (size_t)prob * so;
#pragma unroll
        for (int c = 0; c < N; ++c) {
            if (c >= bn) break;
            if constexpr (CX) O[row + (size_t)c * ldo] = T{y.re[c], y.im[CX ? c : 0]};
            else O[row + (size_t)c * ldo] = y.re[c];
        }
    }
}

inline size_t smem_bytes(int nw) { return (size_t)nw * sizeof(WarpSm) + sizeof(CtaSm); }

}  // namespace qreg

bool qr_reg_ok(int esize, bool cplx, int bm, int bn) {
    return esize == (cplx ? 16 : 8) && bn >= 1 && bn <= 32 && bm <= 256 && bm >= bn;
}

template <bool CX, int NW>
static int launch_qr_reg_nw(SolveArgs<qreg::Elt<CX>> a, qreg::Elt<CX>* R, qreg::Elt<CX>* refl,
                            qreg::Elt<CX>* phase, cudaStream_t st) {
    const size_t smem = qreg::smem_bytes(NW);
    auto k = qreg::k_qr_reg<CX, NW>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<a.batch, NW * 32, smem, st>>>(a, R, refl, phase);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template <bool CX, int NW>
static int launch_applyq_reg_nw(int bm, int bn, int batch, const qreg::Elt<CX>* refl, const qreg::Elt<CX>* phase,
                                const qreg::Elt<CX>* UR, qreg::Elt<CX>* Out, int64_t ldo, int64_t so,
                                cudaStream_t st) {
    const size_t smem = qreg::smem_bytes(NW);
    auto k = qreg::k_applyq_reg<CX, NW>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<batch, NW * 32, smem, st>>>(bm, bn, refl, phase, UR, Out, ldo, so);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template <bool CX>
int launch_qr_reg(SolveArgs<qreg::Elt<CX>> a, qreg::Elt<CX>* R, qreg::Elt<CX>* refl, qreg::Elt<CX>* phase,
                  cudaStream_t st) {
    switch ((a.bm + 31) / 32) {
        case 1: return launch_qr_reg_nw<CX, 1>(a, R, refl, phase, st);
        case 2: return launch_qr_reg_nw<CX, 2>(a, R, refl, phase, st);
        case 3: case 4: return launch_qr_reg_nw<CX, 4>(a, R, refl, phase, st);
        default: return launch_qr_reg_nw<CX, 8>(a, R, refl, phase, st);
    }
}

template <bool CX>
int launch_applyq_reg(int bm, int bn, int batch, const qreg::Elt<CX>* refl, const qreg::Elt<CX>* phase,
                      const qreg::Elt<CX>* UR, qreg::Elt<CX>* Out, int64_t ldo, int64_t so, cudaStream_t st) {
    switch ((bm + 31) / 32) {
        case 1: return launch_applyq_reg_nw<CX, 1>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
        case 2: return launch_applyq_reg_nw<CX, 2>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
        case 3: case 4: return launch_applyq_reg_nw<CX, 4>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
        default: return launch_applyq_reg_nw<CX, 8>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
    }
}

template int launch_qr_reg<false>(SolveArgs<double>, double*, double*, double*, cudaStream_t);
template int launch_qr_reg<true>(SolveArgs<cx<double>>, cx<double>*, cx<double>*, cx<double>*, cudaStream_t);
template int launch_applyq_reg<false>(int, int, int, const double*, const double*, const double*, double*, int64_t,
                                      int64_t, cudaStream_t);
template int launch_applyq_reg<true>(int, int, int, const cx<double>*, const cx<double>*, const cx<double>*,
                                     cx<double>*, int64_t, int64_t, cudaStream_t);

}  // namespace bsvd
