// common.cuh -- element types, rotation arithmetic and the round-robin
// schedule shared by every B200 kernel of the batched Jacobi SVD.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "bsvd_b200.h"

namespace bsvd {

// ---------------------------------------------------------------------------
// Element types.  Complex values are interleaved (re, im) like numpy
// (SPEC.md:96), so a cx<double> is a 16-byte aligned double2.
// ---------------------------------------------------------------------------
template <class F>
struct alignas(2 * sizeof(F)) cx {
    F re, im;
};

// tr<T>: R = real field, W = float64 work type of the rotation arithmetic
// (the reference computes rotation parameters and updates in float64 for
// every storage type, src/_kernels_numba.py:1-7 and SURVEY F6).
template <class T>
struct tr;
template <>
struct tr<float> {
    using R = float;
    using W = double;
    static constexpr bool cplx = false;
    static constexpr double u = 0x1p-24;
    static constexpr int code = BSVD_S;
};
template <>
struct tr<double> {
    using R = double;
    using W = double;
    static constexpr bool cplx = false;
    static constexpr double u = 0x1p-53;
    static constexpr int code = BSVD_D;
};
template <>
struct tr<cx<float>> {
    using R = float;
    using W = cx<double>;
    static constexpr bool cplx = true;
    static constexpr double u = 0x1p-24;
    static constexpr int code = BSVD_C;
};
template <>
struct tr<cx<double>> {
    using R = double;
    using W = cx<double>;
    static constexpr bool cplx = true;
    static constexpr double u = 0x1p-53;
    static constexpr int code = BSVD_Z;
};

#define BSVD_HD __host__ __device__ __forceinline__
#define BSVD_DEV __device__ __forceinline__

template <class T>
BSVD_HD T zero() {
    return T{};
}
template <class T>
BSVD_HD T one() {
    T x{};
    if constexpr (tr<T>::cplx) x.re = 1; else x = 1;
    return x;
}

// |z| in the storage precision (reference: abs(), src/_kernels_numba.py:104-109)
BSVD_DEV float absT(float x) { return fabsf(x); }
BSVD_DEV double absT(double x) { return fabs(x); }
BSVD_DEV float absT(cx<float> z) { return hypotf(z.re, z.im); }
BSVD_DEV double absT(cx<double> z) { return hypot(z.re, z.im); }

// |z|^2 accumulated in float64 (column norms; re^2 + im^2 on GPU)
BSVD_DEV double norm2d(float x) { double d = x; return d * d; }
BSVD_DEV double norm2d(double x) { return x * x; }
BSVD_DEV double norm2d(cx<float> z) { double a = z.re, b = z.im; return fma(a, a, b * b); }
BSVD_DEV double norm2d(cx<double> z) { return fma(z.re, z.re, z.im * z.im); }
// largest |component| and |x * sd|^2 (sd a power of two) for the FP64 column norms of finalize.cuh
BSVD_DEV double abs_component(double x) { return fabs(x); }
BSVD_DEV double abs_component(cx<double> z) { return fmax(fabs(z.re), fabs(z.im)); }
BSVD_DEV double abs_component(float x) { return fabs((double)x); }
BSVD_DEV double abs_component(cx<float> z) { return fmax(fabs((double)z.re), fabs((double)z.im)); }
BSVD_DEV double norm2d_scaled(double x, double sd) { const double y = x * sd; return y * y; }
BSVD_DEV double norm2d_scaled(cx<double> z, double sd) {
    const double a = z.re * sd, b = z.im * sd;
    return fma(a, a, b * b);
}
BSVD_DEV double norm2d_scaled(float x, double sd) { return norm2d(x) * (sd * sd); }
BSVD_DEV double norm2d_scaled(cx<float> z, double sd) { return norm2d(z) * (sd * sd); }

BSVD_DEV float conjT(float x) { return x; }
BSVD_DEV double conjT(double x) { return x; }
template <class F>
BSVD_DEV cx<F> conjT(cx<F> z) { return {z.re, -z.im}; }

// storage-precision multiply-accumulate: acc + conj(a) * b
BSVD_DEV float cmac(float acc, float a, float b) { return fmaf(a, b, acc); }
BSVD_DEV double cmac(double acc, double a, double b) { return fma(a, b, acc); }
template <class F>
BSVD_DEV cx<F> cmac(cx<F> acc, cx<F> a, cx<F> b) {
    // conj(a) * b = (ar*br + ai*bi) + i (ar*bi - ai*br)
    acc.re = fma(a.re, b.re, fma(a.im, b.im, acc.re));
    acc.im = fma(a.re, b.im, fma(-a.im, b.re, acc.im));
    return acc;
}
// storage-precision multiply-accumulate without conjugation: acc + a * b
BSVD_DEV float mac(float acc, float a, float b) { return fmaf(a, b, acc); }
BSVD_DEV double mac(double acc, double a, double b) { return fma(a, b, acc); }
template <class F>
BSVD_DEV cx<F> mac(cx<F> acc, cx<F> a, cx<F> b) {
    acc.re = fma(a.re, b.re, fma(-a.im, b.im, acc.re));
    acc.im = fma(a.re, b.im, fma(a.im, b.re, acc.im));
    return acc;
}
BSVD_DEV float addT(float a, float b) { return a + b; }
BSVD_DEV double addT(double a, double b) { return a + b; }
template <class F>
BSVD_DEV cx<F> addT(cx<F> a, cx<F> b) { return {a.re + b.re, a.im + b.im}; }

// complex / real componentwise (numba complex division by a real, F4)
BSVD_DEV float divR(float a, float b) { return a / b; }
BSVD_DEV double divR(double a, double b) { return a / b; }
template <class F>
BSVD_DEV cx<F> divR(cx<F> a, F b) { return {a.re / b, a.im / b}; }

BSVD_DEV double wide(float x) { return (double)x; }
BSVD_DEV double wide(double x) { return x; }
BSVD_DEV cx<double> wide(cx<float> z) { return {(double)z.re, (double)z.im}; }
BSVD_DEV cx<double> wide(cx<double> z) { return z; }
BSVD_DEV void store(float* p, double x) { *p = (float)x; }
BSVD_DEV void store(double* p, double x) { *p = x; }
BSVD_DEV void store(cx<float>* p, cx<double> z) { *p = cx<float>{(float)z.re, (float)z.im}; }
BSVD_DEV void store(cx<double>* p, cx<double> z) { *p = z; }
template <class T, class Wt>
BSVD_DEV T narrow(Wt w) {
    T x;
    store(&x, w);
    return x;
}

BSVD_DEV double scaleW(double c, double x) { return c * x; }
BSVD_DEV cx<double> scaleW(double c, cx<double> x) { return {c * x.re, c * x.im}; }
BSVD_DEV double conjW(double a) { return a; }
BSVD_DEV cx<double> conjW(cx<double> a) { return {a.re, -a.im}; }

// The reference's rotation update with c - 1 carried separately (F5):
//   x_i <- x_i + (cm1 x_i + wsc x_j),  x_j <- x_j + (cm1 x_j - ws x_i)
BSVD_DEV void rot_pair(double& xi, double& xj, double cm1, double ws, double wsc) {
    const double ni = xi + fma(cm1, xi, wsc * xj);
    const double nj = xj + fma(cm1, xj, -(ws * xi));
    xi = ni;
    xj = nj;
}
BSVD_DEV void rot_pair(cx<double>& xi, cx<double>& xj, double cm1, cx<double> ws, cx<double> wsc) {
    // wsc * xj and ws * xi as full complex products in float64
    const double a_re = fma(wsc.re, xj.re, -(wsc.im * xj.im));
    const double a_im = fma(wsc.re, xj.im, wsc.im * xj.re);
    const double b_re = fma(ws.re, xi.re, -(ws.im * xi.im));
    const double b_im = fma(ws.re, xi.im, ws.im * xi.re);
    cx<double> ni{xi.re + fma(cm1, xi.re, a_re), xi.im + fma(cm1, xi.im, a_im)};
    cx<double> nj{xj.re + fma(cm1, xj.re, -b_re), xj.im + fma(cm1, xj.im, -b_im)};
    xi = ni;
    xj = nj;
}

// Rotation parameters of the 2x2 Hermitian problem (src/_kernels_numba.py:116-127):
// tau = (gii - gjj) / (2|g|); t = sgn(tau) / (|tau| + sqrt(1 + tau^2));
// h = sqrt(1 + t^2); s = t / h; cm1 = -t^2 / (h (1 + h)).  IEEE div/sqrt.
struct RotParams {
    double t, s, cm1;
};
BSVD_DEV RotParams rot_params(double num, double absg2) {
    const double tau = num / absg2;
    const double sgn = tau >= 0.0 ? 1.0 : -1.0;
    const double t = sgn / (fabs(tau) + sqrt(fma(tau, tau, 1.0)));
    const double h = sqrt(fma(t, t, 1.0));
    RotParams p;
    p.t = t;
    p.s = t / h;
    p.cm1 = -(t * t) / (h * (1.0 + h));
    return p;
}

// ---------------------------------------------------------------------------
// Call-free float64 division / square root for register-resident kernels.
// CUDA's IEEE '/' and sqrt() branch to a slow-path subroutine; the CALL makes
// the register allocator spill every live value around it, which wrecks a
// kernel that keeps its working copy in registers.  These versions refine the
// MUFU approximations with Newton steps in DFMA and a final residual
// correction (result within 1 ulp of the IEEE value), and handle 0, tiny
// (pre-scaled by exact powers of two) and infinite operands with selects.
// ---------------------------------------------------------------------------
BSVD_DEV double rcp_approx(double b) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    return r;
}
BSVD_DEV double rsqrt_approx(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
// 1/b by three Newton steps on the MUFU seed (b normal, 1/b normal); scale-invariant under exact
// powers of two, so a prescaled kernel and the standalone finalisation get the same bits.
BSVD_DEV double rcp_refined(double b) {
    double r = rcp_approx(b);
#pragma unroll
    for (int i = 0; i < 3; ++i) r = fma(r, fma(-b, r, 1.0), r);
    return r;
}
// x / s as U = W / sigma is formed everywhere in FP64 (finalize.cuh and the fused finalisations):
// reciprocal, product, one residual correction (within 1 ulp of the IEEE quotient; identical bits
// whichever kernel finalises a problem)
BSVD_DEV double div_by_sigma(double x, double s, double rs) {
    const double q = x * rs;
    return fma(fma(-s, q, x), rs, q);
}
// FP32 U = W / sigma, everywhere the same (finalize.cuh and the fused finalisations of the 16x16 kernels):
// the correctly rounded reciprocal, the product, one residual correction (within 1 ulp of the IEEE
// quotient; a third of the instructions of an IEEE division, which was ~7 % of the C2 kernel)
BSVD_DEV float div_by_sigma_f(float x, float s, float rs) {
    const float q = x * rs;
    return fmaf(fmaf(-s, q, x), rs, q);
}
// a / b for b > 0 (b may be tiny or +inf); a finite.
BSVD_DEV double fdiv(double a, double b) {
    const bool sm = b < 0x1p-960;
    const double as = sm ? a * 0x1p+1000 : a;
    const double bs = sm ? b * 0x1p+1000 : b;
    double r = rcp_approx(bs);
    double e = fma(-bs, r, 1.0);
    r = fma(r, e, r);
    e = fma(-bs, r, 1.0);
    r = fma(r, e, r);
    e = fma(-bs, r, 1.0);
    r = fma(r, e, r);
    const double q = as * r;
    const double rem = fma(-bs, q, as);
    const double qr = fma(rem, r, q);
    return isinf(bs) ? 0.0 * as : (isinf(q) ? q : qr);
}
// sqrt(x) for x >= 0 (x may be 0, tiny or +inf).
BSVD_DEV double fsqrt(double x) {
    const bool tiny = x < 0x1p-960;
    const double xs = tiny ? x * 0x1p+1000 : x;
    double y = rsqrt_approx(xs);
    double e = fma(-(xs * y), y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-(xs * y), y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-(xs * y), y, 1.0);
    y = fma(0.5 * y, e, y);
    double s = xs * y;
    const double rr = fma(-s, s, xs);
    s = fma(rr, 0.5 * y, s);
    s = tiny ? s * 0x1p-500 : s;
    return (x == 0.0 || isinf(x)) ? x : s;
}
// rot_params with the call-free primitives (same formula, <= 1 ulp per op).
BSVD_DEV RotParams rot_params_fast(double num, double absg2) {
    const double tau = fdiv(num, absg2);
    const double sgn = tau >= 0.0 ? 1.0 : -1.0;
    const double t = fdiv(sgn, fabs(tau) + fsqrt(fma(tau, tau, 1.0)));
    const double h = fsqrt(fma(t, t, 1.0));
    RotParams p;
    p.t = t;
    p.s = fdiv(t, h);
    p.cm1 = -fdiv(t * t, h * (1.0 + h));
    return p;
}

// ---------------------------------------------------------------------------
// Round-robin tournament schedule (src/ordering.py:32-75) in closed form.
// Slots other than top[0] form a ring [bot0, top1..top_{h-1}, bot_{h-1}..bot1]
// of length S-1; every iteration each value advances one ring position.
// Pair k of iteration t is (top_t[k], bot_t[k]) sorted; a pair touching the
// phantom index (odd ell) is dropped.  Verified against the reference
// schedule in tests/test_host.py.
// ---------------------------------------------------------------------------
BSVD_HD int rr_val(int q, int S) {  // initial value at ring position q
    const int h = S >> 1;
    if (q == 0) return 1;
    if (q <= h - 1) return 2 * q;
    return 2 * (2 * h - 1 - q) + 1;
}
BSVD_HD int rr_at(int r, int t, int S) {  // value at ring position r after t rotations
    const int L = S - 1;
    int q = (r - (t % L)) % L;
    if (q < 0) q += L;
    return rr_val(q, S);
}
// S = ell rounded up to even.  Returns false for a phantom pair.
BSVD_HD bool rr_pair(int t, int k, int S, int ell, int& i, int& j) {
    const int h = S >> 1;
    const int a = (k == 0) ? 0 : rr_at(k, t, S);
    const int b = rr_at(k == 0 ? 0 : 2 * h - 1 - k, t, S);
    i = a < b ? a : b;
    j = a < b ? b : a;
    return j < ell;
}

// ---------------------------------------------------------------------------
// Warp helpers
// ---------------------------------------------------------------------------
BSVD_DEV float shfl_xor(float v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
BSVD_DEV double shfl_xor(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
template <class F>
BSVD_DEV cx<F> shfl_xor(cx<F> v, int m) {
    return {__shfl_xor_sync(0xffffffffu, v.re, m), __shfl_xor_sync(0xffffffffu, v.im, m)};
}
BSVD_DEV int64_t shfl_xor(int64_t v, int m) { return __shfl_xor_sync(0xffffffffu, (long long)v, m); }

// smallest reliably normalisable column norm, finfo(rdt).tiny / u (src/svd.py:253)
template <class T>
BSVD_HD double dtiny() {
    if constexpr (sizeof(typename tr<T>::R) == 4) return 1.1754943508222875e-38 / 0x1p-24;
    else return 2.2250738585072014e-308 / 0x1p-53;
}

BSVD_DEV bool finiteT(float x) { return isfinite(x); }
BSVD_DEV bool finiteT(double x) { return isfinite(x); }
template <class F>
BSVD_DEV bool finiteT(cx<F> z) { return isfinite(z.re) && isfinite(z.im); }

}  // namespace bsvd
