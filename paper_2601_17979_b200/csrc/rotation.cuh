// rotation.cuh -- call-free float64 Jacobi rotation parameters.
//
// Same formula as the reference (src/_kernels_numba.py:40-52, :116-127; F5):
//   tau = (a_ii - a_jj) / (2|a_ij|);  t = sgn(tau) / (|tau| + sqrt(1 + tau^2)),  sgn(0) = +1
//   h = sqrt(1 + t^2);  s = t / h;  c - 1 = -t^2 / (h (1 + h))
// evaluated as t = sgn(d) 2g / (|d| + sqrt(d^2 + 4 g^2)) on exponent-normalised
// (d, g) and c = 1/sqrt(1 + t^2), s = t c, c - 1 = -s^2 / (1 + c) (algebraically
// identical), with MUFU rcp/rsqrt seeds refined by Newton steps in DFMA and a
// final residual correction: every result within ~1 ulp, no slow-path CALL
// (a CALL makes the register allocator spill all live registers around it).
#pragma once

#include "common.cuh"

namespace bsvd {

BSVD_DEV double pow2(int e) {  // 2^e for e in [-1022, 1023]
    return __longlong_as_double((long long)(1023 + e) << 52);
}

// (d = a_ii - a_jj, g = |a_ij| > 0) -> t, s, cm1 = c - 1
BSVD_DEV void rotation_tsc(double d, double g, double& t_out, double& s_out, double& cm1_out) {
    const double mx = fmax(fabs(d), g);
    const int e = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1023;
    const double sc = pow2(-max(-1022, min(1022, e)));
    const double dn = d * sc, gn = g * sc;  // exact
    const double q = fma(dn, dn, 4.0 * gn * gn);
    double r = rsqrt_approx(q);
    double ee = fma(-(q * r), r, 1.0);
    r = fma(0.5 * r, ee, r);
    ee = fma(-(q * r), r, 1.0);
    r = fma(0.5 * r, ee, r);
    double sq = q * r;
    sq = fma(fma(-sq, sq, q), 0.5 * r, sq);
    const double den = fabs(dn) + sq;
    double rd = rcp_approx(den);
    double e2 = fma(-den, rd, 1.0);
    rd = fma(rd, e2, rd);
    e2 = fma(-den, rd, 1.0);
    rd = fma(rd, e2, rd);
    const double num = 2.0 * gn;
    double t = num * rd;
    t = fma(fma(-den, t, num), rd, t);
    t = d >= 0.0 ? t : -t;  // sgn(0) = +1
    const double h2 = fma(t, t, 1.0);
    double c = rsqrt_approx(h2);
    ee = fma(-(h2 * c), c, 1.0);
    c = fma(0.5 * c, ee, c);
    ee = fma(-(h2 * c), c, 1.0);
    c = fma(0.5 * c, ee, c);
    ee = fma(-(h2 * c), c, 1.0);
    c = fma(0.5 * c, ee, c);
    const double s = t * c;
    const double op = 1.0 + c;
    double ro = rcp_approx(op);
    e2 = fma(-op, ro, 1.0);
    ro = fma(ro, e2, ro);
    e2 = fma(-op, ro, 1.0);
    ro = fma(ro, e2, ro);
    const double s2 = s * s;
    double cm = s2 * ro;
    cm = fma(fma(-op, cm, s2), ro, cm);
    t_out = t;
    s_out = s;
    cm1_out = -cm;
}

// Short-latency variant of rotation_tsc for the register kernels, where the
// parameter chain sits on every iteration's critical path.  Half-angle form
// of the same rotation:
//   r = sqrt(d^2 + 4 g^2),  cos 2th = |d| / r,  c^2 = (1 + cos 2th) / 2,
//   s = g / (r c),  t = s / c (signed like tau),  c - 1 = -s^2 / (1 + c),
// with MUFU seeds and one cubic (third-order) Newton step each, so the chain
// is rsqrt -> rsqrt -> rcp (~250 cycles) instead of rsqrt -> rcp -> rsqrt ->
// rcp with two or three quadratic steps each.  No cancellation anywhere
// (c^2 >= 1/2, 1 + c >= 1.7); results within a few ulp of the reference
// formula (tests/test_gpu_parity.py holds the solver to the parity contract).
BSVD_DEV double rsqrt_cubic(double q) {  // 1/sqrt(q), q normal and > 0
    const double y = rsqrt_approx(q);
    const double e = fma(-(q * y), y, 1.0);       // 1 - q y^2
    return fma(y * e, fma(0.375, e, 0.5), y);    // y (1 + e/2 + 3e^2/8)
}
BSVD_DEV double rcp_cubic(double b) {  // 1/b, b normal
    const double y = rcp_approx(b);
    const double e = fma(-b, y, 1.0);
    return fma(y, fma(e, e, e), y);  // y (1 + e + e^2)
}
BSVD_DEV void rotation_half(double d, double g, double& t_out, double& s_out, double& cm1_out) {
    const double mx = fmax(fabs(d), g);
    const int e = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1023;
    const double sc = pow2(-max(-1020, min(1020, e)));
    const double dn = fabs(d) * sc, gn = g * sc;  // exact; max(dn, gn) in [1, 2)
    const double g2 = gn + gn;
    const double q = fma(dn, dn, g2 * g2);       // in [1, 20)
    const double ir = rsqrt_cubic(q);            // 1 / r
    const double c2 = fma(0.5 * dn, ir, 0.5);    // (1 + |d|/r) / 2 in [1/2, 1]
    const double ic = rsqrt_cubic(c2);           // 1 / c
    const double c = c2 * ic;
    const double s = (gn * ir) * ic;             // sin(th) >= 0
    const double ro = rcp_cubic(1.0 + c);
    cm1_out = -(s * s) * ro;
    const double sg = d >= 0.0 ? s : -s;         // sgn(tau), sgn(0) = +1
    s_out = sg;
    t_out = sg * ic;
}

// exact power-of-two exponent that brings amax into [0.5, 1) (0 for 0/inf/nan)
BSVD_DEV int prescale_exponent(double amax) {
    int ex = (int)((__double_as_longlong(amax) >> 52) & 0x7ff) - 1022;
    if (!(amax > 0.0) || !isfinite(amax)) ex = 0;
    return max(-1021, min(1021, ex));
}

}  // namespace bsvd
