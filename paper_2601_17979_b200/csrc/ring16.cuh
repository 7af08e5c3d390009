// ring16.cuh -- shared pieces of the 16x16 FP32 register kernels: the
// tournament ring for n = 16 in compile-time register slots
// (src/ordering.py:32-75), the FP32 half-angle rotation parameters and the
// two-FMA update (see unblocked_reg16b.cu for the derivation).
#pragma once

#include <cstdint>

namespace bsvd {
namespace ring16 {

constexpr int N = 16;    // columns
constexpr int H = 8;     // pairs per iteration
constexpr int NIT = 15;  // iterations per sweep

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

// ring move by SH positions; 15 = 3 x 5 is not prime, so follow every cycle of the permutation
template <int SH, typename T>
__device__ __forceinline__ void ring_shift(T (&x)[N]) {
    if constexpr (md(SH) != 0) {
        T y[NIT];
#pragma unroll
        for (int q = 0; q < NIT; ++q) y[q] = x[ring_slot(q)];
#pragma unroll
        for (int q = 0; q < NIT; ++q) x[ring_slot(q)] = y[md(q - SH)];
    }
}

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
__device__ __forceinline__ float rsqrt_nr(float x) {
    const float r = rsqrtf(x);
    return fmaf(0.5f * r, fmaf(-x * r, r, 1.0f), r);
}
__device__ __forceinline__ float rcp_nr(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return fmaf(r, fmaf(-x, r, 1.0f), r);
}
// |d|, g -> s = sin(th) >= 0, c - 1, |t| (half-angle form of the reference formula, rotation.cuh)
__device__ __forceinline__ void rot_abs_core(float dabs, float g, float& s, float& cm1, float& tabs) {
    const float q = fmaf(4.0f * g, g, dabs * dabs);
    const float ir = rsqrt_nr(q);
    const float c2 = fmaf(0.5f * dabs, ir, 0.5f);
    const float ic = rsqrt_nr(c2);
    const float c = c2 * ic;
    s = (g * ir) * ic;
    cm1 = -(s * s) * rcp_nr(1.0f + c);
    tabs = s * ic;
}
// |d|, |g| < 2^-50: the float32 squares of the chain above underflow (exactly rank-deficient inputs
// leave rounding-noise columns that keep rotating among themselves and shrink towards the subnormal
// range).  The parameters are ratios, so (|d|, g) are first normalised by an exact power of two taken
// through float64 (2^-e itself overflows float32 for subnormal inputs) -- no IEEE division / square
// root, whose slow paths would cost registers in the hot loop.
__device__ __forceinline__ void rot_abs_tiny(float dabs, float g, float& s, float& cm1, float& tabs) {
    const double mx = (double)fmaxf(dabs, g);
    const int e = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1023;
    const double sc = __longlong_as_double((long long)(1023 - max(-1000, min(1000, e))) << 52);
    rot_abs_core((float)((double)dabs * sc), (float)((double)g * sc), s, cm1, tabs);
}
__device__ __forceinline__ void rot_abs(float dabs, float g, float& s, float& cm1, float& tabs) {
    rot_abs_core(dabs, g, s, cm1, tabs);
    if (fmaxf(dabs, g) < 0x1p-50f) rot_abs_tiny(dabs, g, s, cm1, tabs);
}
// rotate iff |g| >= tol sqrt(g_ii g_jj) (src/_kernels_numba.py guard, F4): squared in float32, and
// squared in float64 for |g| < 2^-60 where the float32 squares and products underflow
__device__ __forceinline__ bool rot_guard(float absg, float gt, float gb, float tol2, float tol) {
    bool rot = !(absg * absg < tol2 * (gt * gb));
    if (absg < 0x1p-60f && absg > 0.0f) {
        const double ag = absg, td = tol;
        rot = !(ag * ag < (td * td) * ((double)gt * (double)gb));
    }
    return rot;
}
__device__ __forceinline__ float xor_signf(float x, bool neg) {
    return __int_as_float(__float_as_int(x) ^ ((int)neg << 31));
}
__device__ __forceinline__ void apply2(float& x, float& y, float cm1, float c) {
    const float tx = fmaf(c, y, x);
    const float ty = fmaf(-c, x, y);
    x = fmaf(cm1, x, tx);
    y = fmaf(cm1, y, ty);
}

}  // namespace ring16
}  // namespace bsvd
