// qr.cu -- the "qr+" route: batched Householder QR pre-processing of tall
// problems and the back-transformation of the left factor.
//
// householder_qr (src/core.py:118-168) per problem, one CTA each, the working
// matrix b (A, or A^H on the transpose route) staged in shared memory:
//   for k: x = b[k:, k]; ||x|| (float64); phase = x0/|x0| (1 if x0 = 0);
//          v = x + phase ||x|| e1, v /= ||v||; b[k:, k:] -= 2 v (v^H b[k:, k:]);
//          b[k, k] = -phase ||x||, b[k+1:, k] = 0   (zero x or zero v: no reflector)
//   sign convention: p_k = r_kk/|r_kk|, R row k *= conj(p_k), Q column k *= p_k.
// The reflectors v_k (zero when skipped) and the phases p_k go to the
// workspace; Q is never formed.  The Jacobi solve then runs on the n x n R
// (src/svd.py:364-371) and the left factor is U = Q diag(p) U_R (src/svd.py:
// 529-530), applied as H_0 ... H_{n-1} [diag(p) U_R; 0] (the reflectors in
// reverse order, like LAPACK's ormqr) by k_applyq.
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {
namespace qr {

template <class T>
BSVD_DEV T mulT(T a, T b) {
    if constexpr (tr<T>::cplx) return T{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    else return a * b;
}
template <class T>
BSVD_DEV T conjT_(T a) {
    if constexpr (tr<T>::cplx) return T{a.re, -a.im};
    else return a;
}
template <class T>
BSVD_DEV T subT(T a, T b) {
    if constexpr (tr<T>::cplx) return T{a.re - b.re, a.im - b.im};
    else return a - b;
}
template <class T>
BSVD_DEV T addT(T a, T b) {
    if constexpr (tr<T>::cplx) return T{a.re + b.re, a.im + b.im};
    else return a + b;
}
template <class T>
BSVD_DEV T scaleT(T a, double s) {
    if constexpr (tr<T>::cplx) return T{(decltype(a.re))(a.re * s), (decltype(a.re))(a.im * s)};
    else return (T)(a * s);
}
template <class T>
BSVD_DEV double abs2T(T a) {
    if constexpr (tr<T>::cplx) return (double)a.re * a.re + (double)a.im * a.im;
    else return (double)a * a;
}
template <class T>
BSVD_DEV T fromRe(double x) {
    if constexpr (tr<T>::cplx) return T{(decltype(T{}.re))x, 0};
    else return (T)x;
}
// x / |x| (1 for x = 0), computed in float64
template <class T>
BSVD_DEV T unit_phase(T x) {
    const double a2 = abs2T(x);
    if (!(a2 > 0.0)) return fromRe<T>(1.0);
    if constexpr (tr<T>::cplx) {
        const double inv = 1.0 / sqrt(a2);
        return T{(decltype(x.re))(x.re * inv), (decltype(x.re))(x.im * inv)};
    } else {
        return x > 0 ? (T)1 : (T)-1;
    }
}

// CTA sum of a double (blockDim multiple of 32, <= 1024); all threads get the result
BSVD_DEV double cta_sum(double v, double* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) scratch[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += scratch[i];  // fixed order: identical on every thread
    return s;
}

template <class T>
__global__ void __launch_bounds__(256) k_qr(SolveArgs<T> a, T* R, T* refl, T* phase) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x;
    const int bm = a.bm, bn = a.bn, tid = threadIdx.x, nt = blockDim.x;
    const int ldb = bm + 1;                     // padded: thread (segment, column) accesses spread over banks
    T* B = reinterpret_cast<T*>(smem);          // bm x bn, ld bm + 1
    T* vs = B + (size_t)ldb * bn;               // reflector k
    const int nseg = nt / bn;
    T* part = vs + bm;                          // partial dots [segments][bn]
    T* wv = part + (size_t)nseg * bn;           // 2 w_j
    const size_t soff = ((size_t)((bm + 1) * bn + bm + nseg * bn + bn) * sizeof(T) + 15) & ~size_t(15);
    double* scratch = reinterpret_cast<double*>(smem + soff);
    int* flag = reinterpret_cast<int*>(scratch + 32);
    T* Vk = refl + (size_t)prob * bm * bn;
    const T* Ap = a.A + (size_t)prob * a.strideA;
    int bad = 0;
    for (int e = tid; e < bm * bn; e += nt) {  // kernel (1): b = A, or A^H on the transpose route
        const int r = e % bm, c = e / bm;
        const T x = a.trans ? conjT_(Ap[c + (size_t)r * a.lda]) : Ap[r + (size_t)c * a.lda];
        bad |= !finiteT(x);
        B[r + (size_t)c * ldb] = x;
    }
    if (tid == 0) *flag = 0;
    __syncthreads();
    if (bad) atomicOr(flag, 1);
    const int j = tid % bn, sg = tid / bn;
    for (int k = 0; k < bn; ++k) {
        double s = 0.0;
        for (int r = k + tid; r < bm; r += nt) s += abs2T(B[r + (size_t)k * ldb]);
        s = cta_sum(s, scratch);
        const double norm_x = sqrt(s);
        const T alpha = B[k + (size_t)k * ldb];
        const T ph = unit_phase(alpha);
        const T v0 = addT(alpha, scaleT(ph, norm_x));
        const double vn = sqrt(fmax(s - abs2T(alpha), 0.0) + abs2T(v0));
        const bool skip = !(norm_x > 0.0) || !(vn > 0.0);
        const double iv = skip ? 0.0 : 1.0 / vn;
        for (int r = tid; r < bm; r += nt) {  // v (zero when skipped) -> workspace and smem
            T v = fromRe<T>(0.0);
            if (r == k) v = scaleT(v0, iv);
            else if (r > k) v = scaleT(B[r + (size_t)k * ldb], iv);
            Vk[r + (size_t)k * bm] = v;
            vs[r] = v;
        }
        __syncthreads();
        const int len = bm - k, seg = (len + nseg - 1) / nseg;
        const int r0 = k + sg * seg, r1 = min(bm, r0 + seg);
        const bool act = !skip && sg < nseg && j > k;
        if (act) {  // trailing columns j > k: w_j = v^H b[k:, j]
            double wr = 0.0, wi = 0.0;
            for (int r = r0; r < r1; ++r) {
                const T p = mulT(conjT_(vs[r]), B[r + (size_t)j * ldb]);
                if constexpr (tr<T>::cplx) {
                    wr += p.re;
                    wi += p.im;
                } else {
                    wr += p;
                }
            }
            if constexpr (tr<T>::cplx) part[sg * bn + j] = T{(decltype(T{}.re))wr, (decltype(T{}.re))wi};
            else part[sg * bn + j] = (T)wr;
        }
        __syncthreads();
        if (!skip && tid < bn && tid > k) {
            double wr = 0.0, wi = 0.0;
            for (int q = 0; q < nseg; ++q) {
                if constexpr (tr<T>::cplx) {
                    wr += part[q * bn + tid].re;
                    wi += part[q * bn + tid].im;
                } else {
                    wr += part[q * bn + tid];
                }
            }
            if constexpr (tr<T>::cplx) wv[tid] = T{(decltype(T{}.re))(2.0 * wr), (decltype(T{}.re))(2.0 * wi)};
            else wv[tid] = (T)(2.0 * wr);
        }
        __syncthreads();
        if (act) {  // b[k:, j] -= 2 v w_j
            const T w2 = wv[j];
            for (int r = r0; r < r1; ++r) B[r + (size_t)j * ldb] = subT(B[r + (size_t)j * ldb], mulT(vs[r], w2));
        }
        if (tid == 0 && !skip) B[k + (size_t)k * ldb] = scaleT(ph, -norm_x);  // exact value (src/core.py:142)
        __syncthreads();
    }
    // sign convention and R out (bn x bn, ld bn, zeros below the diagonal)
    T* Rp = R + (size_t)prob * bn * bn;
    T* Pp = phase + (size_t)prob * bn;
    for (int e = tid; e < bn * bn; e += nt) {
        const int r = e % bn, c = e / bn;
        T x = fromRe<T>(0.0);
        if (r <= c) {
            const T dkk = B[r + (size_t)r * ldb];
            const T p = unit_phase(dkk);
            x = (r == c) ? fromRe<T>(sqrt(abs2T(dkk))) : mulT(B[r + (size_t)c * ldb], conjT_(p));
        }
        Rp[e] = x;
    }
    for (int k = tid; k < bn; k += nt) Pp[k] = unit_phase(B[k + (size_t)k * ldb]);
    if (tid == 0 && a.info) a.info[prob].status = *flag;  // provisional; the inner solve rewrites info
}

// Out (bm x bn, ld ldo) = H_0 ... H_{bn-1} [diag(p) U_R; 0].  Y staged in shared memory with a
// padded leading dimension; thread (segment s, column j) owns rows [s*seg, (s+1)*seg) of column j:
// partial v^H Y[:, j] per segment -> smem -> summed per column -> rank-1 update of the own rows.
template <class T>
__global__ void __launch_bounds__(256) k_applyq(int bm, int bn, const T* refl, const T* phase, const T* UR,
                                                T* Out, int64_t ldo, int64_t so) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int ldy = bm + 1;
    T* Y = reinterpret_cast<T*>(smem);                 // bm x bn, ld bm + 1
    T* vs = Y + (size_t)ldy * bn;                      // reflector k (bm)
    T* part = vs + bm;                                 // partial dots [segments][bn]
    T* wv = part + (size_t)(nt / bn + 1) * bn;         // 2 w_j per column
    const T* Vk = refl + (size_t)prob * bm * bn;
    const T* Pp = phase + (size_t)prob * bn;
    const T* U = UR + (size_t)prob * bn * bn;
    for (int e = tid; e < bm * bn; e += nt) {
        const int r = e % bm, c = e / bm;
        Y[r + (size_t)c * ldy] = r < bn ? mulT(Pp[r], U[r + (size_t)c * bn]) : fromRe<T>(0.0);
    }
    const int nseg = nt / bn;                          // row segments per column (threads beyond idle)
    const int j = tid % bn, sg = tid / bn;
    for (int k = bn - 1; k >= 0; --k) {
        const T* v = Vk + (size_t)k * bm;
        for (int r = k + tid; r < bm; r += nt) vs[r] = v[r];
        __syncthreads();
        const int len = bm - k, seg = (len + nseg - 1) / nseg;
        const int r0 = k + sg * seg, r1 = min(bm, r0 + seg);
        if (sg < nseg) {
            double wr = 0.0, wi = 0.0;
            for (int r = r0; r < r1; ++r) {
                const T p = mulT(conjT_(vs[r]), Y[r + (size_t)j * ldy]);
                if constexpr (tr<T>::cplx) {
                    wr += p.re;
                    wi += p.im;
                } else {
                    wr += p;
                }
            }
            if constexpr (tr<T>::cplx) part[sg * bn + j] = T{(decltype(T{}.re))wr, (decltype(T{}.re))wi};
            else part[sg * bn + j] = (T)wr;
        }
        __syncthreads();
        if (tid < bn) {
            double wr = 0.0, wi = 0.0;
            for (int q = 0; q < nseg; ++q) {
                if constexpr (tr<T>::cplx) {
                    wr += part[q * bn + tid].re;
                    wi += part[q * bn + tid].im;
                } else {
                    wr += part[q * bn + tid];
                }
            }
            if constexpr (tr<T>::cplx) wv[tid] = T{(decltype(T{}.re))(2.0 * wr), (decltype(T{}.re))(2.0 * wi)};
            else wv[tid] = (T)(2.0 * wr);
        }
        __syncthreads();
        if (sg < nseg) {
            const T w2 = wv[j];
            for (int r = r0; r < r1; ++r) Y[r + (size_t)j * ldy] = subT(Y[r + (size_t)j * ldy], mulT(vs[r], w2));
        }
        __syncthreads();
    }
    T* O = Out + (size_t)prob * so;
    for (int e = tid; e < bm * bn; e += nt) O[(e % bm) + (size_t)(e / bm) * ldo] = Y[(e % bm) + (size_t)(e / bm) * ldy];
}

__global__ void k_qr_path(bsvd_info* info, int batch, int bits) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < batch) info[i].path |= bits;
}

}  // namespace qr

int qr_threads(int bn) { return bn > 256 ? 0 : 256; }  // 256 / bn row segments per column, rest idle
size_t qr_smem(int esize, int bm, int bn) {
    const int nt = qr_threads(bn);
    if (!nt) return ~(size_t)0;
    return ((((size_t)(bm + 1) * bn + bm + (size_t)(nt / bn) * bn + bn) * esize + 15) & ~size_t(15)) + 32 * 8 + 16;
}

template <class T>
int launch_qr(SolveArgs<T> a, T* R, T* refl, T* phase, cudaStream_t st) {
    if constexpr (std::is_same<T, double>::value || std::is_same<T, cx<double>>::value) {
        if (qr_reg_ok(sizeof(T), tr<T>::cplx, a.bm, a.bn)) return launch_qr_col<tr<T>::cplx>(a, R, refl, phase, st);
    }
    const size_t smem = qr_smem(sizeof(T), a.bm, a.bn);
    if (smem > 232448) return BSVD_ERR_UNSUPPORTED;
    auto k = qr::k_qr<T>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<a.batch, qr_threads(a.bn), smem, st>>>(a, R, refl, phase);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template <class T>
int launch_applyq(int bm, int bn, int batch, const T* refl, const T* phase, const T* UR, T* Out, int64_t ldo,
                  int64_t so, cudaStream_t st) {
    if constexpr (std::is_same<T, double>::value || std::is_same<T, cx<double>>::value) {
        if (qr_reg_ok(sizeof(T), tr<T>::cplx, bm, bn))
            return launch_applyq_col<tr<T>::cplx>(bm, bn, batch, refl, phase, UR, Out, ldo, so, st);
    }
    if (bn > 256) return BSVD_ERR_UNSUPPORTED;
    const int nt = 256;  // 256 / bn row segments per column; the remaining threads only stage data
    const size_t smem = ((size_t)(bm + 1) * bn + bm + (size_t)(nt / bn + 1) * bn + bn) * sizeof(T);
    auto k = qr::k_applyq<T>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BSVD_ERR_CUDA;
    k<<<batch, nt, smem, st>>>(bm, bn, refl, phase, UR, Out, ldo, so);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

int launch_qr_path(bsvd_info* info, int batch, int bits, cudaStream_t st) {
    qr::k_qr_path<<<(batch + 255) / 256, 256, 0, st>>>(info, batch, bits);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

// householder_qr(a) (src/core.py:118-168) as a batched operator: reflectors + R by launch_qr, then
// Q = H_0 ... H_{n-1} [diag(p); 0] (the sign convention folded in), R copied to the caller's layout.
namespace qr {
template <class T>
__global__ void k_eye_copy(int n, int batch, T* eye, const T* Rw, T* R, int64_t ldr, int64_t sR) {
    const int prob = blockIdx.x;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
        const int r = e % n, c = e / n;
        eye[(size_t)prob * n * n + e] = fromRe<T>(r == c ? 1.0 : 0.0);
        R[(size_t)prob * sR + r + (size_t)c * ldr] = Rw[(size_t)prob * n * n + e];
    }
}
}  // namespace qr

size_t householder_qr_work_bytes(int esize, int m, int n, int batch) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t B = (size_t)batch, es = (size_t)esize;
    return al(B * m * n * es) + al(B * n * es) + 2 * al(B * n * n * es);
}

template <class T>
int launch_householder_qr(int m, int n, int batch, const void* A, int64_t lda, int64_t sA, void* Q, int64_t ldq,
                          int64_t sQ, void* R, int64_t ldr, int64_t sR, void* work, size_t smem_limit, cudaStream_t st) {
    if (!qr_reg_ok(sizeof(T), tr<T>::cplx, m, n) && qr_smem(sizeof(T), m, n) > smem_limit) return BSVD_ERR_UNSUPPORTED;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t B = (size_t)batch, es = sizeof(T);
    unsigned char* w = static_cast<unsigned char*>(work);
    T* refl = reinterpret_cast<T*>(w);
    T* ph = reinterpret_cast<T*>(w + al(B * m * n * es));
    T* Rw = reinterpret_cast<T*>(w + al(B * m * n * es) + al(B * n * es));
    T* eye = reinterpret_cast<T*>(w + al(B * m * n * es) + al(B * n * es) + al(B * n * n * es));
    SolveArgs<T> a{};
    a.A = static_cast<const T*>(A);
    a.lda = lda;
    a.strideA = sA;
    a.m = m;
    a.n = n;
    a.bm = m;
    a.bn = n;
    a.batch = batch;
    int rc = launch_qr<T>(a, Rw, refl, ph, st);
    if (rc) return rc;
    qr::k_eye_copy<T><<<batch, 128, 0, st>>>(n, batch, eye, Rw, static_cast<T*>(R), ldr, sR);
    if (cudaPeekAtLastError() != cudaSuccess) return BSVD_ERR_CUDA;
    return launch_applyq<T>(m, n, batch, refl, ph, eye, static_cast<T*>(Q), ldq, sQ, st);
}

#define BSVD_QR_INST(T)                                                                                   \
    template int launch_qr<T>(SolveArgs<T>, T*, T*, T*, cudaStream_t);                                    \
    template int launch_applyq<T>(int, int, int, const T*, const T*, const T*, T*, int64_t, int64_t,      \
                                  cudaStream_t);                                                          \
    template int launch_householder_qr<T>(int, int, int, const void*, int64_t, int64_t, void*, int64_t,    \
                                          int64_t, void*, int64_t, int64_t, void*, size_t, cudaStream_t);
BSVD_QR_INST(float)
BSVD_QR_INST(double)
BSVD_QR_INST(cx<float>)
BSVD_QR_INST(cx<double>)

}  // namespace bsvd
