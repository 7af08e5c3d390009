// qr_col.cu -- column-distributed Householder QR and Q application for the
// "qr+" route on FP64 data (real and complex), n <= 32, m <= 256: BASELINE
// config C4 (256 x 32 c128) on the QR route.
//
// Same algorithm and conventions as qr.cu (householder_qr,
// src/core.py:118-168; U = Q diag(p) U_R, src/svd.py:529-530).
//
// Layout: one CTA of NWC warps per problem (QR: 16, two columns per warp --
// measured 2.06 ms vs 2.49 ms with 8 on C4; Q application: 8, four columns
// per warp -- 1.26 ms vs 2.62 ms with 16, which spills); column c of the
// working matrix belongs to warp c % NWC (interleaved so the trailing work
// stays balanced as k advances), and lane l of that warp holds rows
// l, l + 32, ..., l + 32 (RPL - 1) of its columns in registers.  Every dot
// product v^H b_j is then a warp-local sum (a lane-local partial over the
// lane's rows plus a shuffle all-reduce), so a reflector costs one CTA
// barrier (the owner warp publishes v through a double-buffered smem slot)
// and no shared-memory transpose of partial sums -- a row-distributed
// register kernel (one row per lane, an earlier version of this file) moved
// every partial product of every trailing column through smem and was
// load/store bound (C4: 3.3 + 2.4 ms vs 2.06 + 1.26 ms here).  Applying Q needs no barrier at
// all: the reflectors are known, each warp applies all of them to its own
// columns.
#include <type_traits>

#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {
namespace qcol {

constexpr int N = 32;   // columns (max)

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// x / |x| for a complex (xr, xi), 1 for 0
__device__ __forceinline__ void cphase(double xr, double xi, double& pr, double& pi) {
    const double a2 = fma(xr, xr, xi * xi);
    if (a2 > 0.0) {
        const double inv = fdiv(1.0, fsqrt(a2));
        pr = xr * inv;
        pi = xi * inv;
    } else {
        pr = 1.0;
        pi = 0.0;
    }
}

template <bool CX>
using Elt = typename std::conditional<CX, cx<double>, double>::type;

template <bool CX>
__device__ __forceinline__ void ld(const Elt<CX>* p, double& re, double& im) {
    if constexpr (CX) {
        const cx<double> z = *p;
        re = z.re;
        im = z.im;
    } else {
        re = *p;
        im = 0.0;
    }
}
template <bool CX>
__device__ __forceinline__ void st(Elt<CX>* p, double re, double im) {
    if constexpr (CX) *p = cx<double>{re, im};
    else *p = re;
}

template <bool CX, int RPL, int CPW>
struct Cols {
    double re[CPW][RPL];
    double im[CPW][CX ? RPL : 1];
};

struct __align__(16) QSmem {
    double v[2][2 * 256];  // published reflector, double-buffered [parity][row (re, im)]
    double diag[2 * N];    // R's diagonal before the sign convention
    int skip[2];
    int bad;
};

// ---- b_j -= 2 v (v^H b_j) for this warp's columns c > k (all warp-uniform branches) ----
template <bool CX, int RPL, int NWC>
__device__ __forceinline__ void apply_reflector(Cols<CX, RPL, N / NWC>& x, const double (&vr)[RPL],
                                                const double (&vi)[RPL], int warp, int kmin) {
    constexpr int CPW = N / NWC;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + NWC * i;
        if (c <= kmin) continue;
        double wr = 0.0, wi = 0.0;  // conj(v) . b_c over this lane's rows
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            if (CX) {
                wr = fma(vr[p], x.re[i][p], fma(vi[p], x.im[i][CX ? p : 0], wr));
                wi = fma(vr[p], x.im[i][CX ? p : 0], fma(-vi[p], x.re[i][p], wi));
            } else {
                wr = fma(vr[p], x.re[i][p], wr);
            }
        }
        wr = 2.0 * wsum(wr);
        if (CX) wi = 2.0 * wsum(wi);
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            if (CX) {
                x.re[i][p] = fma(-vr[p], wr, fma(vi[p], wi, x.re[i][p]));
                x.im[i][CX ? p : 0] = fma(-vr[p], wi, fma(-vi[p], wr, x.im[i][CX ? p : 0]));
            } else {
                x.re[i][p] = fma(-vr[p], wr, x.re[i][p]);
            }
        }
    }
}

template <bool CX, int RPL, int NWC>
__global__ void __launch_bounds__(NWC * 32, (NWC == 16 || (CX && RPL == 8)) ? 1 : 2) k_qr_col(
    SolveArgs<Elt<CX>> a, Elt<CX>* R, Elt<CX>* refl, Elt<CX>* phase) {
    using T = Elt<CX>;
    constexpr int CPW = N / NWC;
    __shared__ QSmem sm;
    const int prob = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bm = a.bm, bn = a.bn;
    const T* Ap = a.A + (size_t)prob * a.strideA;
    Cols<CX, RPL, CPW> x;
    int bad = 0;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + NWC * i;
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            const int r = lane + 32 * p;
            double re = 0.0, im = 0.0;
            if (c < bn && r < bm) {  // kernel (1): b = A, or A^H on the transpose route
                ld<CX>(a.trans ? Ap + c + (size_t)r * a.lda : Ap + r + (size_t)c * a.lda, re, im);
                if (CX && a.trans) im = -im;
            }
            bad |= !(isfinite(re) && isfinite(im));
            x.re[i][p] = re;
            if (CX) x.im[i][CX ? p : 0] = im;
        }
    }
    if (tid == 0) sm.bad = 0;
    __syncthreads();
    if (bad) atomicOr(&sm.bad, 1);
    double* vk = reinterpret_cast<double*>(refl + (size_t)prob * bm * bn);
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
#pragma unroll 1
        for (int w = 0; w < NWC; ++w) {
            const int k = w + NWC * i;  // column k lives in slot i of warp w
            if (k >= bn) break;
            const int par = k & 1;
            if (warp == w) {
                // ---- reflector for column k (owner warp only) ----
                double s = 0.0, ar = 0.0, ai = 0.0;
#pragma unroll
                for (int p = 0; p < RPL; ++p) {
                    const int r = lane + 32 * p;
                    const double re = x.re[i][p], im = CX ? x.im[i][CX ? p : 0] : 0.0;
                    if (r >= k) s = fma(re, re, fma(im, im, s));
                    if (r == k) {
                        ar = re;
                        ai = im;
                    }
                }
                s = wsum(s);
                ar = __shfl_sync(0xffffffffu, ar, k & 31);
                ai = __shfl_sync(0xffffffffu, ai, k & 31);
                const double nx = fsqrt(s);
                double pr, pi;
                if (CX) {
                    cphase(ar, ai, pr, pi);
                } else {
                    pr = ar > 0.0 ? 1.0 : -1.0;  // unit_phase of a real: sign, 1 for 0
                    if (!(ar * ar > 0.0)) pr = 1.0;
                    pi = 0.0;
                }
                const double v0r = fma(pr, nx, ar), v0i = fma(pi, nx, ai);
                const double vn = fsqrt(fmax(s - fma(ar, ar, ai * ai), 0.0) + fma(v0r, v0r, v0i * v0i));
                const bool skip = !(nx > 0.0) || !(vn > 0.0);
                const double iv = skip ? 0.0 : fdiv(1.0, vn);
#pragma unroll
                for (int p = 0; p < RPL; ++p) {
                    const int r = lane + 32 * p;
                    double vr = 0.0, vi = 0.0;
                    if (r == k) {
                        vr = v0r * iv;
                        vi = v0i * iv;
                    } else if (r > k) {
                        vr = x.re[i][p] * iv;
                        vi = CX ? x.im[i][CX ? p : 0] * iv : 0.0;
                    }
                    sm.v[par][2 * r] = vr;
                    sm.v[par][2 * r + 1] = vi;
                    if (r < bm) {
                        if (CX) reinterpret_cast<double2*>(vk)[r + (size_t)k * bm] = make_double2(vr, vi);
                        else vk[r + (size_t)k * bm] = vr;
                    }
                    if (r == k && !skip) {  // exact diagonal (src/core.py:142)
                        x.re[i][p] = -pr * nx;
                        if (CX) x.im[i][CX ? p : 0] = -pi * nx;
                    }
                }
                if (lane == 0) sm.skip[par] = skip ? 1 : 0;
            }
            __syncthreads();  // v of column k published (double buffer: one barrier per reflector)
            if (!sm.skip[par]) {
                double vr[RPL], vi[RPL];
#pragma unroll
                for (int p = 0; p < RPL; ++p) {
                    const int r = lane + 32 * p;
                    vr[p] = sm.v[par][2 * r];
                    vi[p] = sm.v[par][2 * r + 1];
                }
                apply_reflector<CX, RPL, NWC>(x, vr, vi, warp, k);
            }
        }
    }
    // ---- sign convention: p_k = r_kk/|r_kk|, R row k *= conj(p_k), diagonal |r_kk| ----
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + NWC * i;
        if (c < bn && c < 32 * RPL) {
#pragma unroll
            for (int p = 0; p < RPL; ++p)
                if (lane + 32 * p == c) {
                    sm.diag[2 * c] = x.re[i][p];
                    sm.diag[2 * c + 1] = CX ? x.im[i][CX ? p : 0] : 0.0;
                }
        }
    }
    __syncthreads();
    T* Rp = R + (size_t)prob * bn * bn;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + NWC * i;
        if (c >= bn) continue;
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            const int r = lane + 32 * p;
            if (r >= bn) continue;
            double yr = 0.0, yi = 0.0;
            const double dr = sm.diag[2 * r], di = sm.diag[2 * r + 1];
            if (r == c) {
                yr = fsqrt(fma(dr, dr, di * di));
            } else if (r < c) {  // x conj(p_r)
                double pr, pi;
                if (CX) {
                    cphase(dr, di, pr, pi);
                } else {
                    pr = dr > 0.0 ? 1.0 : -1.0;
                    if (!(dr * dr > 0.0)) pr = 1.0;
                    pi = 0.0;
                }
                const double xr = x.re[i][p], xi = CX ? x.im[i][CX ? p : 0] : 0.0;
                yr = fma(xr, pr, xi * pi);
                yi = fma(xi, pr, -xr * pi);
            }
            st<CX>(Rp + r + (size_t)c * bn, yr, yi);
        }
    }
    if (tid < bn) {
        const double dr = sm.diag[2 * tid], di = sm.diag[2 * tid + 1];
        double pr, pi;
        if (CX) {
            cphase(dr, di, pr, pi);
        } else {
            pr = dr > 0.0 ? 1.0 : -1.0;
            if (!(dr * dr > 0.0)) pr = 1.0;
            pi = 0.0;
        }
        st<CX>(phase + (size_t)prob * bn + tid, pr, pi);
    }
    if (tid == 0 && a.info) a.info[prob].status = sm.bad;  // provisional; the inner solve rewrites info
}

// Out = H_0 ... H_{bn-1} [diag(p) U_R; 0]: each warp applies every reflector to its own columns
template <bool CX, int RPL, int NWC>
__global__ void __launch_bounds__(NWC * 32, (NWC == 16 || (CX && RPL == 8)) ? 1 : 2) k_applyq_col(
    int bm, int bn, const Elt<CX>* refl, const Elt<CX>* phase, const Elt<CX>* UR, Elt<CX>* Out, int64_t ldo,
    int64_t so) {
    using T = Elt<CX>;
    constexpr int CPW = N / NWC;
    const int prob = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const T* Vk = refl + (size_t)prob * bm * bn;
    const T* U = UR + (size_t)prob * bn * bn;
    const T* Pp = phase + (size_t)prob * bn;
    Cols<CX, RPL, CPW> y;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + NWC * i;
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            const int r = lane + 32 * p;
            double yr = 0.0, yi = 0.0;
            if (c < bn && r < bn) {  // p_r u_rc
                double ur, ui, pr, pi;
                ld<CX>(U + r + (size_t)c * bn, ur, ui);
                ld<CX>(Pp + r, pr, pi);
                yr = fma(pr, ur, -pi * ui);
                yi = fma(pr, ui, pi * ur);
            }
            y.re[i][p] = yr;
            if (CX) y.im[i][CX ? p : 0] = yi;
        }
    }
    double nr[RPL], ni[RPL];  // reflector k prefetched one step ahead
    auto load_v = [&](int k) {
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            const int r = lane + 32 * p;
            nr[p] = 0.0;
            ni[p] = 0.0;
            if (r < bm && r >= k) ld<CX>(Vk + r + (size_t)k * bm, nr[p], ni[p]);
        }
    };
    if (bn > 0) load_v(bn - 1);
#pragma unroll 1
    for (int k = bn - 1; k >= 0; --k) {
        double vr[RPL], vi[RPL];
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            vr[p] = nr[p];
            vi[p] = ni[p];
        }
        if (k > 0) load_v(k - 1);
        apply_reflector<CX, RPL, NWC>(y, vr, vi, warp, -1);  // every column: Q acts on all of [diag(p) U_R; 0]
    }
    T* O = Out + (size_t)prob * so;
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
        const int c = warp + NWC * i;
        if (c >= bn) continue;
#pragma unroll
        for (int p = 0; p < RPL; ++p) {
            const int r = lane + 32 * p;
            if (r < bm) st<CX>(O + r + (size_t)c * ldo, y.re[i][p], CX ? y.im[i][CX ? p : 0] : 0.0);
        }
    }
}

}  // namespace qcol

bool qr_reg_ok(int esize, bool cplx, int bm, int bn) {  // shapes the column-distributed kernels take
    return esize == (cplx ? 16 : 8) && bn >= 1 && bn <= 32 && bm <= 256 && bm >= bn;
}

template <bool CX, int RPL, int NWC = 16>
static int qcol_qr(SolveArgs<qcol::Elt<CX>> a, qcol::Elt<CX>* R, qcol::Elt<CX>* refl, qcol::Elt<CX>* phase,
                   cudaStream_t st) {
    qcol::k_qr_col<CX, RPL, NWC><<<a.batch, NWC * 32, 0, st>>>(a, R, refl, phase);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}
template <bool CX, int RPL, int NWC = 8>
static int qcol_applyq(int bm, int bn, int batch, const qcol::Elt<CX>* refl, const qcol::Elt<CX>* phase,
                       const qcol::Elt<CX>* UR, qcol::Elt<CX>* Out, int64_t ldo, int64_t so, cudaStream_t st) {
    qcol::k_applyq_col<CX, RPL, NWC><<<batch, NWC * 32, 0, st>>>(bm, bn, refl, phase, UR, Out, ldo, so);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template <bool CX>
int launch_qr_col(SolveArgs<qcol::Elt<CX>> a, qcol::Elt<CX>* R, qcol::Elt<CX>* refl, qcol::Elt<CX>* phase,
                  cudaStream_t st) {
    const int rpl = (a.bm + 31) / 32;
    if (rpl <= 1) return qcol_qr<CX, 1>(a, R, refl, phase, st);
    if (rpl <= 2) return qcol_qr<CX, 2>(a, R, refl, phase, st);
    if (rpl <= 4) return qcol_qr<CX, 4>(a, R, refl, phase, st);
    return qcol_qr<CX, 8>(a, R, refl, phase, st);
}
template <bool CX>
int launch_applyq_col(int bm, int bn, int batch, const qcol::Elt<CX>* refl, const qcol::Elt<CX>* phase,
                      const qcol::Elt<CX>* UR, qcol::Elt<CX>* Out, int64_t ldo, int64_t so, cudaStream_t st) {
    const int rpl = (bm + 31) / 32;
    if (rpl <= 1) return qcol_applyq<CX, 1>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
    if (rpl <= 2) return qcol_applyq<CX, 2>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
    if (rpl <= 4) return qcol_applyq<CX, 4>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
    return qcol_applyq<CX, 8>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
}

template int launch_qr_col<false>(SolveArgs<double>, double*, double*, double*, cudaStream_t);
template int launch_qr_col<true>(SolveArgs<cx<double>>, cx<double>*, cx<double>*, cx<double>*, cudaStream_t);
template int launch_applyq_col<false>(int, int, int, const double*, const double*, const double*, double*, int64_t,
                                      int64_t, cudaStream_t);
template int launch_applyq_col<true>(int, int, int, const cx<double>*, const cx<double>*, const cx<double>*,
                                     cx<double>*, int64_t, int64_t, cudaStream_t);

}  // namespace bsvd
