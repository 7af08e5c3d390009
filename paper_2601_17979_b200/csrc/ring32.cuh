// ring32.cuh -- shared pieces of the 32-column register kernels: the
// tournament ring in compile-time register slots (src/ordering.py:32-75), the
// rotation record, the two-FMA update and the short-latency rotation
// parameters (same formulas as unblocked_reg32b.cu, see there for the
// derivation and the numerical notes).
#pragma once

#include "rotation.cuh"

namespace bsvd {
namespace ring32 {

constexpr int N = 32;     // columns
constexpr int H = 16;     // column pairs per iteration
constexpr int NIT = 31;   // iterations per sweep (ring length)
constexpr int RSTR = 34;  // doubles per row of a transpose buffer (even: double2 reads; bank padding)

__host__ __device__ constexpr int ring_slot(int q) {  // ring position -> register slot at t = 0
    return q == 0 ? 1 : (q <= H - 1 ? 2 * q : 2 * (2 * H - 1 - q) + 1);
}
__host__ __device__ constexpr int md(int a) { return ((a % NIT) + NIT) % NIT; }
// register slot of pair k's top / bottom column at offset u inside an unrolled group
__host__ __device__ constexpr int TS(int k, int u) { return k == 0 ? 0 : ring_slot(md(k - u)); }
__host__ __device__ constexpr int BS(int k, int u) { return ring_slot(md((k == 0 ? 0 : NIT - k) - u)); }

// column ids of pair k at iteration t: ct | cb << 8 | (ct > cb) << 16 (reference orientation i < j)
__host__ __device__ inline uint32_t pair_code(int t, int k) {
    int qt = k - t, qb = (k == 0 ? 0 : NIT - k) - t;
    qt += qt < 0 ? NIT : 0;
    qb += qb < 0 ? NIT : 0;
    const int ct = (k == 0) ? 0 : ring_slot(qt);
    const int cb = ring_slot(qb);
    return (uint32_t)ct | ((uint32_t)cb << 8) | ((ct > cb) ? (1u << 16) : 0u);
}

struct __align__(16) Par {
    double cm1, c;  // x <- x + (cm1 x + c y);  y <- y + (cm1 y - c x)
};

// move every column SH ring positions forward: 31 is prime, one cycle, one temporary
template <int SH>
__device__ __forceinline__ void ring_shift(double (&x)[N]) {
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

__device__ __forceinline__ double sum16(const double* p) {  // 16 consecutive doubles, fixed tree
    const double2* r = reinterpret_cast<const double2*>(p);
    const double2 p0 = r[0], p1 = r[1], p2 = r[2], p3 = r[3], p4 = r[4], p5 = r[5], p6 = r[6], p7 = r[7];
    const double s0 = (p0.x + p0.y) + (p1.x + p1.y), s1 = (p2.x + p2.y) + (p3.x + p3.y);
    const double s2 = (p4.x + p4.y) + (p5.x + p5.y), s3 = (p6.x + p6.y) + (p7.x + p7.y);
    return (s0 + s1) + (s2 + s3);
}
// total over a warp's 32 lanes of transpose row `row` (identical bits on both half-warps)
__device__ __forceinline__ double sum32(const double* red, int row, int half) {
    const double s = sum16(red + row * RSTR + 16 * half);
    const double o = __shfl_xor_sync(0xffffffffu, s, 16);
    return half ? o + s : s + o;
}

__device__ __forceinline__ double xor_sign(double x, bool neg) {
    return __longlong_as_double(__double_as_longlong(x) ^ ((long long)neg << 63));
}

// |d|, g -> s = sin(th) >= 0, c - 1, |t| (half-angle chain rsqrt -> rsqrt -> rcp, cubic steps)
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

// 16 consecutive doubles summed in the order of a 16-8-4-2-1 xor butterfly (p_i = v_i + v_{i+16} given):
// the column-norm order of finalize_block, so fused and standalone finalisation give the same sigma bits
__device__ __forceinline__ double sum16_butterfly(const double* p) {
    double t[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t[i] = p[i] + p[i + 8];
#pragma unroll
    for (int i = 0; i < 4; ++i) t[i] = t[i] + t[i + 4];
    return (t[0] + t[2]) + (t[1] + t[3]);
}

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

}  // namespace ring32
}  // namespace bsvd
