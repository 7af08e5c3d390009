// verify.cu -- on-device accuracy metrics e1-e4 for whole batches
// (src/verify.py:44-84; thresholds k*u, src/verify.py:39-41), one CTA per
// problem, float64 accumulation:
//   e1 = |A - U diag(s) V^H|_1 / (n |A|_1)          (max absolute column sum)
//   e2 = |I - U^H U|_1 / m,  e3 = |I - V^H V|_1 / n
//   e4 = |s - s_ref|_F / min(m, n)                    (NaN when no reference)
// so a 10k-problem parity check does not bottleneck on host numpy.
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {
namespace vfy {

template <class T>
BSVD_DEV cx<double> ld(const T* p) {
    if constexpr (tr<T>::cplx) return cx<double>{(double)p->re, (double)p->im};
    else return cx<double>{(double)*p, 0.0};
}
BSVD_DEV cx<double> cmul(cx<double> a, cx<double> b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
BSVD_DEV cx<double> cconj(cx<double> a) { return {a.re, -a.im}; }
BSVD_DEV double cabs(cx<double> a) { return hypot(a.re, a.im); }

BSVD_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// max over columns of sum_i |X_ij| where X = I - Y^H Y (Y: rows x k, ld ldy)
template <class T>
BSVD_DEV double ortho_colmax(const T* Y, int64_t ldy, int rows, int k, int warp, int lane, int nw) {
    double mx = 0.0;
    for (int j = warp; j < k; j += nw) {
        double cs = 0.0;
        for (int i = 0; i < k; ++i) {
            double gr = 0.0, gi = 0.0;
            for (int r = lane; r < rows; r += 32) {
                const cx<double> p = cmul(cconj(ld(Y + r + (size_t)i * ldy)), ld(Y + r + (size_t)j * ldy));
                gr += p.re;
                gi += p.im;
            }
            gr = warp_sum(gr);
            gi = warp_sum(gi);
            cs += hypot((i == j ? 1.0 : 0.0) - gr, -gi);
        }
        mx = fmax(mx, cs);
    }
    return mx;
}

template <class T>
__global__ void __launch_bounds__(256) k_verify(int m, int n, const T* A, int64_t lda, int64_t sA, const T* U,
                                                int64_t ldu, int64_t sU, const typename tr<T>::R* S, int64_t sS,
                                                const T* V, int64_t ldv, int64_t sV, const double* Sref,
                                                int64_t sR, double* out) {
    __shared__ double red[3][8];
    const int prob = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int k = m < n ? m : n;
    const T* Ap = A + (size_t)prob * sA;
    const T* Up = U + (size_t)prob * sU;
    const T* Vp = V ? V + (size_t)prob * sV : nullptr;
    const typename tr<T>::R* Sp = S + (size_t)prob * sS;
    // e1: residual and |A|_1 column maxima
    double rmax = 0.0, amax = 0.0;
    for (int j = warp; j < n; j += nw) {
        double rs = 0.0, as = 0.0;
        for (int i = lane; i < m; i += 32) {
            const cx<double> a = ld(Ap + i + (size_t)j * lda);
            cx<double> rec{0.0, 0.0};
            if (Vp)
                for (int l = 0; l < k; ++l) {
                    const cx<double> us = ld(Up + i + (size_t)l * ldu);
                    const double s = (double)Sp[l];
                    const cx<double> t = cmul(us, cconj(ld(Vp + j + (size_t)l * ldv)));
                    rec.re += s * t.re;
                    rec.im += s * t.im;
                }
            rs += cabs(cx<double>{a.re - rec.re, a.im - rec.im});
            as += cabs(a);
        }
        rmax = fmax(rmax, warp_sum(rs));
        amax = fmax(amax, warp_sum(as));
    }
    const double o2 = ortho_colmax(Up, ldu, m, k, warp, lane, nw);
    const double o3 = Vp ? ortho_colmax(Vp, ldv, n, k, warp, lane, nw) : 0.0;
    if (lane == 0) {
        red[0][warp] = rmax;
        red[1][warp] = amax;
        red[2][warp] = o2;
    }
    __syncthreads();
    double e1n = 0.0, e1d = 0.0, e2 = 0.0;
    for (int w = 0; w < nw; ++w) {
        e1n = fmax(e1n, red[0][w]);
        e1d = fmax(e1d, red[1][w]);
        e2 = fmax(e2, red[2][w]);
    }
    __syncthreads();
    if (lane == 0) red[0][warp] = o3;
    __syncthreads();
    if (tid == 0) {
        double e3 = 0.0;
        for (int w = 0; w < nw; ++w) e3 = fmax(e3, red[0][w]);
        double* o = out + (size_t)prob * 4;
        const double den = (double)n * e1d;
        o[0] = Vp ? (den == 0.0 ? (e1n == 0.0 ? 0.0 : INFINITY) : e1n / den) : NAN;
        o[1] = m ? e2 / m : 0.0;
        o[2] = (Vp && n) ? e3 / n : (Vp ? 0.0 : NAN);
        if (Sref) {
            double ss = 0.0;
            for (int l = 0; l < k; ++l) {
                const double dl = (double)Sp[l] - Sref[(size_t)prob * sR + l];
                ss += dl * dl;
            }
            o[3] = k ? sqrt(ss) / k : 0.0;
        } else {
            o[3] = NAN;
        }
    }
}

template <class T>
int launch(int m, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* U, int64_t ldu, int64_t sU,
           const void* S, int64_t sS, const void* V, int64_t ldv, int64_t sV, const double* Sref, int64_t sR,
           double* out, cudaStream_t st) {
    k_verify<T><<<batch, 256, 0, st>>>(m, n, static_cast<const T*>(A), lda, sA, static_cast<const T*>(U), ldu, sU,
                                       static_cast<const typename tr<T>::R*>(S), sS, static_cast<const T*>(V), ldv,
                                       sV, Sref, sR, out);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

}  // namespace vfy

int launch_verify(int dtype, int m, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* U,
                  int64_t ldu, int64_t sU, const void* S, int64_t sS, const void* V, int64_t ldv, int64_t sV,
                  const double* Sref, int64_t sR, double* out, cudaStream_t st) {
    switch (dtype) {
        case BSVD_S: return vfy::launch<float>(m, n, batch, A, lda, sA, U, ldu, sU, S, sS, V, ldv, sV, Sref, sR, out, st);
        case BSVD_D: return vfy::launch<double>(m, n, batch, A, lda, sA, U, ldu, sU, S, sS, V, ldv, sV, Sref, sR, out, st);
        case BSVD_C:
            return vfy::launch<cx<float>>(m, n, batch, A, lda, sA, U, ldu, sU, S, sS, V, ldv, sV, Sref, sR, out, st);
        case BSVD_Z:
            return vfy::launch<cx<double>>(m, n, batch, A, lda, sA, U, ldu, sU, S, sS, V, ldv, sV, Sref, sR, out, st);
    }
    return BSVD_ERR_ARG;
}

}  // namespace bsvd
