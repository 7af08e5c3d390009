// bsvd_oracle.cpp -- CPU restatement of the reference one-sided Jacobi SVD.
//
// TEST INFRASTRUCTURE ONLY (see bsvd_oracle.h).  This is the checker the GPU
// kernels are compared against and the "port" CPU baseline; it is never part
// of the product path.
//
// Faithfulness notes.  The reference's hot kernels are numba functions compiled
// without fastmath, i.e. strict IEEE with no FMA contraction.  This file is
// compiled with -ffp-contract=off and reproduces numba's type promotions
// (SURVEY F6): for single-precision data the column norms accumulate in float64
// from float32 products, the cross term accumulates in the storage precision,
// and the rotation parameters and the update arithmetic run in float64 with a
// rounding store.  Complex |z| is libm hypot, as numba lowers abs(complex).
// With those rules the unblocked path reproduces the reference bit for bit on
// the golden vectors (tests/test_oracle.py).  compute_gram and the two-stage
// update use numpy/OpenBLAS in the reference, which no restatement can match
// bitwise; they are sequential sums here and are pinned by tolerance.
#include "bsvd_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

template <class F>
struct cx {
    F re, im;
};

template <class T>
struct tr;
template <>
struct tr<float> {
    using R = float;
    using W = double;
    static constexpr bool cplx = false;
    static constexpr double u = 0x1p-24;
};
template <>
struct tr<double> {
    using R = double;
    using W = double;
    static constexpr bool cplx = false;
    static constexpr double u = 0x1p-53;
};
template <>
struct tr<cx<float>> {
    using R = float;
    using W = cx<double>;
    static constexpr bool cplx = true;
    static constexpr double u = 0x1p-24;
};
template <>
struct tr<cx<double>> {
    using R = double;
    using W = cx<double>;
    static constexpr bool cplx = true;
    static constexpr double u = 0x1p-53;
};

// ---- scalar helpers reproducing numba's lowering -------------------------
inline float absv(float x) { return std::fabs(x); }
inline double absv(double x) { return std::fabs(x); }
inline float absv(cx<float> z) { return ::hypotf(z.re, z.im); }     // numba abs(complex64)
inline double absv(cx<double> z) { return ::hypot(z.re, z.im); }    // numba abs(complex128)

inline float conjv(float x) { return x; }
inline double conjv(double x) { return x; }
template <class F>
inline cx<F> conjv(cx<F> z) { return {z.re, -z.im}; }

template <class T>
inline T zero() { return T{}; }

// storage-precision arithmetic (numba complex_mul: ac-bd, ad+bc)
inline float mulT(float a, float b) { return a * b; }
inline double mulT(double a, double b) { return a * b; }
template <class F>
inline cx<F> mulT(cx<F> a, cx<F> b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline float addT(float a, float b) { return a + b; }
inline double addT(double a, double b) { return a + b; }
template <class F>
inline cx<F> addT(cx<F> a, cx<F> b) { return {a.re + b.re, a.im + b.im}; }

// complex / real -> componentwise (CPython/numba complex division with b.imag == 0)
inline float divR(float a, float b) { return a / b; }
inline double divR(double a, double b) { return a / b; }
template <class F>
inline cx<F> divR(cx<F> a, F b) { return {a.re / b, a.im / b}; }

// widening to the float64 work type, rounding store back
inline double wide(float x) { return (double)x; }
inline double wide(double x) { return x; }
inline cx<double> wide(cx<float> z) { return {(double)z.re, (double)z.im}; }
inline cx<double> wide(cx<double> z) { return z; }
template <class T>
inline T narrow(double x);
template <>
inline float narrow<float>(double x) { return (float)x; }
template <>
inline double narrow<double>(double x) { return x; }
template <class T>
inline T narrowc(cx<double> z);
template <>
inline cx<float> narrowc<cx<float>>(cx<double> z) { return {(float)z.re, (float)z.im}; }
template <>
inline cx<double> narrowc<cx<double>>(cx<double> z) { return z; }
inline float narrowT(double x, float*) { return (float)x; }
inline double narrowT(double x, double*) { return x; }
inline cx<float> narrowT(cx<double> z, cx<float>*) { return {(float)z.re, (float)z.im}; }
inline cx<double> narrowT(cx<double> z, cx<double>*) { return z; }
template <class T, class Wt>
inline T nar(Wt w) { return narrowT(w, (T*)nullptr); }

// float64 work-type arithmetic
inline double scaleW(double c, double x) { return c * x; }
inline cx<double> scaleW(double c, cx<double> x) { return {c * x.re, c * x.im}; }
inline double mulW(double a, double b) { return a * b; }
inline cx<double> mulW(cx<double> a, cx<double> b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
inline double addW(double a, double b) { return a + b; }
inline cx<double> addW(cx<double> a, cx<double> b) { return {a.re + b.re, a.im + b.im}; }
inline double subW(double a, double b) { return a - b; }
inline cx<double> subW(cx<double> a, cx<double> b) { return {a.re - b.re, a.im - b.im}; }
inline double conjW(double a) { return a; }
inline cx<double> conjW(cx<double> a) { return {a.re, -a.im}; }
inline double addScalar(double a, double c) { return a + c; }
inline cx<double> addScalar(cx<double> a, double c) { return {a.re + c, a.im}; }

template <class T>
inline T one() {
    T x{};
    if constexpr (tr<T>::cplx) x.re = 1; else x = 1;
    return x;
}
template <class T>
inline double realpart(T x) {
    if constexpr (tr<T>::cplx) return (double)x.re; else return (double)x;
}

// ---- round-robin schedule  (src/ordering.py:32-75) -----------------------
struct Sched {
    std::vector<int> pairs;   // 2*P
    std::vector<int> starts;  // T+1
    int n_iter = 0;
};

Sched make_schedule(int ell) {
    Sched s;
    int size = (ell % 2 == 0) ? ell : ell + 1;
    int half = size / 2;
    std::vector<int> top, bot;
    for (int x = 0; x < size; x += 2) top.push_back(x);
    for (int x = 1; x < size; x += 2) bot.push_back(x);
    s.starts.push_back(0);
    for (int it = 0; it < size - 1; ++it) {
        for (int k = 0; k < half; ++k) {
            int t = top[k], b = bot[k];
            int i = t < b ? t : b, j = t < b ? b : t;
            if (j < ell) {
                s.pairs.push_back(i);
                s.pairs.push_back(j);
            }
        }
        s.starts.push_back((int)s.pairs.size() / 2);
        if (half > 1) {
            // top, bot = [top[0], bot[0]] + top[1:-1], bot[1:] + [top[-1]]
            std::vector<int> nt, nb;
            nt.push_back(top[0]);
            nt.push_back(bot[0]);
            for (int k = 1; k < half - 1; ++k) nt.push_back(top[k]);
            for (int k = 1; k < half; ++k) nb.push_back(bot[k]);
            nb.push_back(top[half - 1]);
            top = nt;
            bot = nb;
        }
    }
    s.n_iter = size - 1;
    return s;
}

// ---- onesided_sweeps  (src/_kernels_numba.py:85-138) ---------------------
template <class T>
int64_t onesided(int m, T* a, int lda, int vrows, T* v, int ldv, const Sched& sc, double tol,
                 int max_sweeps, int* sweeps_out, int* conv_out) {
    using R = typename tr<T>::R;
    using W = typename tr<T>::W;
    int sweeps = 0;
    int64_t rotations = 0;
    bool converged = false;
    while (!converged && sweeps < max_sweeps) {
        converged = true;
        sweeps += 1;
        for (int it = 0; it < sc.n_iter; ++it) {
            for (int p = sc.starts[it]; p < sc.starts[it + 1]; ++p) {
                const int i = sc.pairs[2 * p], j = sc.pairs[2 * p + 1];
                T* ci = a + (size_t)i * lda;
                T* cj = a + (size_t)j * lda;
                double gii = 0.0, gjj = 0.0;
                T gji = zero<T>();
                for (int r = 0; r < m; ++r) {
                    const T ai = ci[r], aj = cj[r];
                    const R ti = absv(ai), tj = absv(aj);
                    gii += (double)(R)(ti * ti);  // product in storage precision (F6)
                    gjj += (double)(R)(tj * tj);
                    gji = addT(gji, mulT(conjv(aj), ai));
                }
                const R absg = absv(gji);
                if (absg <= (R)0) continue;
                if ((double)absg < tol * std::sqrt(gii * gjj)) continue;
                converged = false;
                rotations += 1;
                const T w = divR(conjv(gji), absg);
                const double tau = (gii - gjj) / (2.0 * (double)absg);
                const double sgn = tau >= 0.0 ? 1.0 : -1.0;
                const double t = sgn / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                const double h = std::sqrt(1.0 + t * t);
                const double s = t / h;
                const double cm1 = -(t * t) / (h * (1.0 + h));
                const W ws = scaleW(s, wide(w));
                const W wsc = scaleW(s, wide(conjv(w)));
                for (int r = 0; r < m; ++r) {
                    const W ai = wide(ci[r]), aj = wide(cj[r]);
                    ci[r] = nar<T>(addW(ai, addW(scaleW(cm1, ai), mulW(wsc, aj))));
                    cj[r] = nar<T>(addW(aj, subW(scaleW(cm1, aj), mulW(ws, ai))));
                }
                T* vi = v + (size_t)i * ldv;
                T* vj = v + (size_t)j * ldv;
                for (int r = 0; r < vrows; ++r) {
                    const W xi = wide(vi[r]), xj = wide(vj[r]);
                    vi[r] = nar<T>(addW(xi, addW(scaleW(cm1, xi), mulW(wsc, xj))));
                    vj[r] = nar<T>(addW(xj, subW(scaleW(cm1, xj), mulW(ws, xi))));
                }
            }
        }
    }
    if (sweeps_out) *sweeps_out = sweeps;
    if (conv_out) *conv_out = converged ? 1 : 0;
    return rotations;
}

// ---- eig_sweeps  (src/_kernels_numba.py:17-82) ---------------------------
template <class T>
int64_t eig_sweeps(int n, T* g, int ldg, typename tr<T>::R* d, int mrows, T* mm, int ldm,
                   const Sched& sc, double tol, int max_sweeps, bool delta, int* sweeps_out,
                   int* conv_out) {
    using R = typename tr<T>::R;
    using W = typename tr<T>::W;
    int sweeps = 0;
    int64_t rotations = 0;
    bool converged = false;
    while (!converged && sweeps < max_sweeps) {
        converged = true;
        sweeps += 1;
        for (int it = 0; it < sc.n_iter; ++it) {
            for (int p = sc.starts[it]; p < sc.starts[it + 1]; ++p) {
                const int i = sc.pairs[2 * p], j = sc.pairs[2 * p + 1];
                const T gij = g[i + (size_t)j * ldg];
                const R absg = absv(gij);
                if (absg <= (R)0) continue;
                const R prod = (R)(std::fabs(d[i]) * std::fabs(d[j]));  // storage-real precision
                const R sq = std::sqrt(prod);
                if ((double)absg < tol * (double)sq) continue;
                converged = false;
                rotations += 1;
                const T w = divR(gij, absg);
                const R ddiff = (R)(d[i] - d[j]);
                const double tau = (double)ddiff / (2.0 * (double)absg);
                const double sgn = tau >= 0.0 ? 1.0 : -1.0;
                const double t = sgn / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                const double h = std::sqrt(1.0 + t * t);
                const double s = t / h;
                const double cm1 = -(t * t) / (h * (1.0 + h));
                const W ws = scaleW(s, wide(w));
                const W wsc = scaleW(s, wide(conjv(w)));
                for (int q = 0; q < n; ++q) {
                    if (q == i || q == j) continue;
                    const W riq = wide(g[i + (size_t)q * ldg]);
                    const W rjq = wide(g[j + (size_t)q * ldg]);
                    const W niq = addW(riq, addW(scaleW(cm1, riq), mulW(ws, rjq)));
                    const W njq = addW(rjq, subW(scaleW(cm1, rjq), mulW(wsc, riq)));
                    g[i + (size_t)q * ldg] = nar<T>(niq);
                    g[j + (size_t)q * ldg] = nar<T>(njq);
                    g[q + (size_t)i * ldg] = nar<T>(conjW(niq));
                    g[q + (size_t)j * ldg] = nar<T>(conjW(njq));
                }
                g[i + (size_t)j * ldg] = zero<T>();
                g[j + (size_t)i * ldg] = zero<T>();
                const double td = t * (double)absg;
                d[i] = (R)((double)d[i] + td);
                d[j] = (R)((double)d[j] - td);
                for (int r = 0; r < mrows; ++r) {
                    const W vi = wide(mm[r + (size_t)i * ldm]);
                    const W vj = wide(mm[r + (size_t)j * ldm]);
                    mm[r + (size_t)i * ldm] = nar<T>(addW(vi, addW(scaleW(cm1, vi), mulW(wsc, vj))));
                    mm[r + (size_t)j * ldm] = nar<T>(addW(vj, subW(scaleW(cm1, vj), mulW(ws, vi))));
                }
                if (delta) {
                    T* mii = &mm[i + (size_t)i * ldm];
                    T* mji = &mm[j + (size_t)i * ldm];
                    T* mij = &mm[i + (size_t)j * ldm];
                    T* mjj = &mm[j + (size_t)j * ldm];
                    *mii = nar<T>(addScalar(wide(*mii), cm1));
                    *mji = nar<T>(addW(wide(*mji), wsc));
                    *mij = nar<T>(subW(wide(*mij), ws));
                    *mjj = nar<T>(addScalar(wide(*mjj), cm1));
                }
            }
        }
    }
    if (sweeps_out) *sweeps_out = sweeps;
    if (conv_out) *conv_out = converged ? 1 : 0;
    return rotations;
}

// ---- compute_gram  (src/svd.py:144-179) ----------------------------------
// Upper triangle by sequential sums in storage precision, strict lower mirrored
// as the conjugate, diagonal forced real.
template <class T>
void gram(int m, int wi, int wj, const T* ai, int ldai, const T* aj, int ldaj, T* g, int ldg) {
    const int wt = wi + wj;
    auto col = [&](int c) -> const T* {
        return c < wi ? ai + (size_t)c * ldai : aj + (size_t)(c - wi) * ldaj;
    };
    for (int b = 0; b < wt; ++b) {
        const T* xb = col(b);
        for (int a = 0; a <= b; ++a) {
            const T* xa = col(a);
            T acc = zero<T>();
            for (int r = 0; r < m; ++r) acc = addT(acc, mulT(conjv(xa[r]), xb[r]));
            g[a + (size_t)b * ldg] = acc;
            g[b + (size_t)a * ldg] = conjv(acc);
        }
        T dg = g[b + (size_t)b * ldg];
        if constexpr (tr<T>::cplx) dg.im = 0;
        g[b + (size_t)b * ldg] = dg;
    }
}

// ---- fused_pair_update  (src/_kernels_numba.py:141-175) ------------------
// Rows are independent, so the row_block tiling does not change the result.
template <class T>
void fused_update(int m, int wi, int wj, T* bi, int ldi, T* bj, int ldj, const T* J, int ldJ,
                  bool delta, bool twostage) {
    const int wt = wi + wj;
    std::vector<T> buf(wt), acc(wt);
    for (int r = 0; r < m; ++r) {
        for (int k = 0; k < wi; ++k) buf[k] = bi[r + (size_t)k * ldi];
        for (int k = 0; k < wj; ++k) buf[wi + k] = bj[r + (size_t)k * ldj];
        for (int q = 0; q < wt; ++q) {
            T z;
            if (!twostage) {
                z = mulT(buf[0], J[0 + (size_t)q * ldJ]);
                for (int k = 1; k < wt; ++k) z = addT(z, mulT(buf[k], J[k + (size_t)q * ldJ]));
            } else {
                // src/svd.py:213-221: t = bi @ D[:wi] ; t += bj @ D[wi:]
                T z1 = mulT(buf[0], J[0 + (size_t)q * ldJ]);
                for (int k = 1; k < wi; ++k) z1 = addT(z1, mulT(buf[k], J[k + (size_t)q * ldJ]));
                T z2 = mulT(buf[wi], J[wi + (size_t)q * ldJ]);
                for (int k = wi + 1; k < wt; ++k) z2 = addT(z2, mulT(buf[k], J[k + (size_t)q * ldJ]));
                z = addT(z1, z2);
            }
            acc[q] = delta ? addT(buf[q], z) : z;
        }
        for (int q = 0; q < wi; ++q) bi[r + (size_t)q * ldi] = acc[q];
        for (int q = 0; q < wj; ++q) bj[r + (size_t)q * ldj] = acc[wi + q];
    }
}

// ---- numpy pairwise summation (np.sum over a contiguous column) ----------
double pairwise_sum(const double* a, long n) {
    if (n < 8) {
        double res = 0.0;
        for (long i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        long i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

// numpy's SIMD complex absolute (larger * sqrt(fma(ratio, ratio, 1)))
inline double np_cabs(double re, double im) {
    re = std::fabs(re);
    im = std::fabs(im);
    const double larger = std::max(re, im), smaller = std::min(re, im);
    if (larger == 0.0) return 0.0;
    const double ratio = smaller / larger;
    return std::sqrt(std::fma(ratio, ratio, 1.0)) * larger;
}

// ---- _finalize_factors  (src/svd.py:224-275) -----------------------------
template <class T>
void finalize(int m, int n, T* w, int ldw, T* v, int ldv, int vrows, typename tr<T>::R* sigma) {
    using R = typename tr<T>::R;
    const double u_r = tr<T>::u;
    std::vector<double> sq(m);
    std::vector<R> sig(n);
    for (int c = 0; c < n; ++c) {
        const T* col = w + (size_t)c * ldw;
        for (int r = 0; r < m; ++r) {
            if constexpr (tr<T>::cplx) {
                const double a = np_cabs((double)col[r].re, (double)col[r].im);
                sq[r] = a * a;
            } else {
                const double a = std::fabs((double)col[r]);
                sq[r] = a * a;
            }
        }
        sig[c] = (R)std::sqrt(pairwise_sum(sq.data(), m));
    }
    const double dtiny = (double)std::numeric_limits<R>::min() / u_r;
    std::vector<int> zero_cols, formed;
    for (int c = 0; c < n; ++c) {
        T* col = w + (size_t)c * ldw;
        if ((double)sig[c] < dtiny) {
            sig[c] = 0;
            zero_cols.push_back(c);
        } else {
            const R sc = sig[c];
            if constexpr (tr<T>::cplx) {
                const R scl = (R)1 / sc;  // numpy complex / real: multiply by reciprocal
                for (int r = 0; r < m; ++r) col[r] = {col[r].re * scl, col[r].im * scl};
            } else {
                for (int r = 0; r < m; ++r) col[r] = col[r] / sc;
            }
            formed.push_back(c);
        }
    }
    // _orthogonal_completion  src/svd.py:224-240
    for (int hole : zero_cols) {
        std::vector<double> load(m, 0.0);
        for (int c : formed)
            for (int r = 0; r < m; ++r) {
                const T x = w[r + (size_t)c * ldw];
                double ax;
                if constexpr (tr<T>::cplx) ax = np_cabs(x.re, x.im); else ax = std::fabs((double)x);
                load[r] += ax * ax;
            }
        int kmin = 0;
        for (int r = 1; r < m; ++r)
            if (load[r] < load[kmin]) kmin = r;
        std::vector<typename tr<T>::W> x(m);
        for (int r = 0; r < m; ++r) x[r] = wide(zero<T>());
        x[kmin] = wide(one<T>());
        for (int pass = 0; pass < 2; ++pass) {
            for (int c : formed) {
                const T* uc = w + (size_t)c * ldw;
                typename tr<T>::W dot = wide(zero<T>());
                for (int r = 0; r < m; ++r) dot = addW(dot, mulW(conjW(wide(uc[r])), x[r]));
                for (int r = 0; r < m; ++r) x[r] = subW(x[r], mulW(wide(uc[r]), dot));
            }
        }
        double nrm = 0.0;
        for (int r = 0; r < m; ++r) {
            if constexpr (tr<T>::cplx) nrm += x[r].re * x[r].re + x[r].im * x[r].im;
            else nrm += x[r] * x[r];
        }
        nrm = std::sqrt(nrm);
        for (int r = 0; r < m; ++r) {
            if constexpr (tr<T>::cplx) w[r + (size_t)hole * ldw] = nar<T>(typename tr<T>::W{x[r].re / nrm, x[r].im / nrm});
            else w[r + (size_t)hole * ldw] = nar<T>(x[r] / nrm);
        }
        formed.push_back(hole);
    }
    // stable descending sort, permute U and V  (np.argsort(-sigma, kind="stable"))
    std::vector<int> order(n);
    for (int c = 0; c < n; ++c) order[c] = c;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return -sig[a] < -sig[b]; });
    bool ident = true;
    for (int c = 0; c < n; ++c) ident = ident && order[c] == c;
    if (!ident) {
        std::vector<T> tmp((size_t)m * n);
        for (int c = 0; c < n; ++c)
            for (int r = 0; r < m; ++r) tmp[r + (size_t)c * m] = w[r + (size_t)order[c] * ldw];
        for (int c = 0; c < n; ++c)
            for (int r = 0; r < m; ++r) w[r + (size_t)c * ldw] = tmp[r + (size_t)c * m];
        if (v) {
            std::vector<T> tv((size_t)vrows * n);
            for (int c = 0; c < n; ++c)
                for (int r = 0; r < vrows; ++r) tv[r + (size_t)c * vrows] = v[r + (size_t)order[c] * ldv];
            for (int c = 0; c < n; ++c)
                for (int r = 0; r < vrows; ++r) v[r + (size_t)c * ldv] = tv[r + (size_t)c * vrows];
        }
    }
    for (int c = 0; c < n; ++c) sigma[c] = sig[order[c]];
}

// ---- householder_qr  (src/core.py:118-168) --------------------------------
// Reduced non-pivoted QR by Householder reflections in the working precision;
// norms in float64 (np.linalg.norm's BLAS order is not reproduced: this part
// of the restatement is pinned by tolerance, like the reference's own tests).
template <class T>
double norm2v(const T* x, int len) {
    double s = 0.0;
    for (int i = 0; i < len; ++i) {
        if constexpr (tr<T>::cplx) s += (double)x[i].re * x[i].re + (double)x[i].im * x[i].im;
        else s += (double)x[i] * x[i];
    }
    return std::sqrt(s);
}
template <class T>
T scaleT(T x, double c) {
    if constexpr (tr<T>::cplx) return {(decltype(x.re))(x.re * c), (decltype(x.re))(x.im * c)};
    else return (T)(x * c);
}
template <class T>
T subT(T a, T b) {
    if constexpr (tr<T>::cplx) return {a.re - b.re, a.im - b.im};
    else return a - b;
}
template <class T>
T phase_of(T x) {  // x / |x|, 1 for x == 0
    if constexpr (tr<T>::cplx) {
        const double a = std::hypot((double)x.re, (double)x.im);
        if (a == 0.0) return one<T>();
        return {(decltype(x.re))(x.re / a), (decltype(x.re))(x.im / a)};
    } else {
        return x == 0 ? (T)1 : (x > 0 ? (T)1 : (T)-1);
    }
}
// a (m x n, ld m) -> q (m x n), r (n x n); requires m >= n
template <class T>
void householder_qr(int m, int n, const T* a, std::vector<T>& q, std::vector<T>& r_out) {
    std::vector<T> r(a, a + (size_t)m * n);
    std::vector<std::pair<int, std::vector<T>>> refl;
    for (int k = 0; k < n; ++k) {
        T* x = r.data() + k + (size_t)k * m;
        const int len = m - k;
        const double norm_x = norm2v(x, len);
        if (norm_x == 0.0) continue;
        const T ph = phase_of(x[0]);
        std::vector<T> v(x, x + len);
        v[0] = addT(v[0], scaleT(ph, norm_x));
        const double vn = norm2v(v.data(), len);
        if (vn == 0.0) continue;
        for (auto& e : v) e = scaleT(e, 1.0 / vn);
        for (int j = k; j < n; ++j) {  // r[k:, k:] -= 2 outer(v, v^H r[k:, k:])
            T* cj = r.data() + k + (size_t)j * m;
            T w = zero<T>();
            for (int i = 0; i < len; ++i) w = addT(w, mulT(conjv(v[i]), cj[i]));
            const T w2 = scaleT(w, 2.0);
            for (int i = 0; i < len; ++i) cj[i] = subT(cj[i], mulT(v[i], w2));
        }
        x[0] = scaleT(ph, -norm_x);
        for (int i = 1; i < len; ++i) x[i] = zero<T>();
        refl.push_back({k, std::move(v)});
    }
    q.assign((size_t)m * n, zero<T>());
    for (int k = 0; k < n; ++k) q[k + (size_t)k * m] = one<T>();
    for (auto it = refl.rbegin(); it != refl.rend(); ++it) {
        const int k = it->first, len = m - k;
        const std::vector<T>& v = it->second;
        for (int j = 0; j < n; ++j) {
            T* cj = q.data() + k + (size_t)j * m;
            T w = zero<T>();
            for (int i = 0; i < len; ++i) w = addT(w, mulT(conjv(v[i]), cj[i]));
            const T w2 = scaleT(w, 2.0);
            for (int i = 0; i < len; ++i) cj[i] = subT(cj[i], mulT(v[i], w2));
        }
    }
    for (int k = 0; k < n; ++k) {  // diag(r) real >= 0
        const T dkk = r[k + (size_t)k * m];
        const T p = phase_of(dkk);
        bool is_zero;
        if constexpr (tr<T>::cplx) is_zero = dkk.re == 0 && dkk.im == 0; else is_zero = dkk == 0;
        if (is_zero) continue;
        for (int j = k; j < n; ++j) r[k + (size_t)j * m] = mulT(r[k + (size_t)j * m], conjv(p));
        for (int i = 0; i < m; ++i) q[i + (size_t)k * m] = mulT(q[i + (size_t)k * m], p);
        if constexpr (tr<T>::cplx) r[k + (size_t)k * m] = {(decltype(dkk.re))std::hypot((double)dkk.re, (double)dkk.im), 0};
        else r[k + (size_t)k * m] = (T)std::fabs((double)dkk);
    }
    r_out.assign((size_t)n * n, zero<T>());
    for (int j = 0; j < n; ++j)
        for (int i = 0; i <= j; ++i) r_out[i + (size_t)j * n] = r[i + (size_t)j * m];
}

// ---- _ProblemRun + _run_standalone  (src/svd.py:312-556) -----------------
template <class T>
int solve(int m, int n, const T* a, T* u, typename tr<T>::R* s, T* vout, const orc_opts* o,
          orc_info* info) {
    using R = typename tr<T>::R;
    std::memset(info, 0, sizeof(*info));
    if (o->force != 0 && m < n) {
        info->status = -2;  // ShapeError: forced solver requires m >= n
        return -2;
    }
    const bool transposed = o->force == 0 && m < n;
    const int bm = transposed ? n : m, bn = transposed ? m : n;
    info->transposed = transposed ? 1 : 0;
    if (bm == 0 || bn == 0) {
        info->converged = 1;
        info->path = ORC_PATH_EMPTY;
        return 0;
    }
    // W = fmatrix(b), b = a^H when transposed  (src/svd.py:346-373)
    std::vector<T> W((size_t)bm * bn);
    for (int c = 0; c < bn; ++c)
        for (int r = 0; r < bm; ++r)
            W[r + (size_t)c * bm] = transposed ? conjv(a[c + (size_t)r * m]) : a[r + (size_t)c * m];
    // QR first (src/svd.py:364-371): forced, or dispatch with use_qr_preprocess and bm >= 3 bn
    const bool use_qr = o->force == 3 || (o->force == 0 && o->use_qr && (double)bm >= 3.0 * bn);
    std::vector<T> Q;
    const int bm_in = bm;
    int bmw = bm;
    if (use_qr) {
        std::vector<T> Rm;
        householder_qr<T>(bm, bn, W.data(), Q, Rm);
        W = Rm;
        bmw = bn;
        info->qr = 1;
    }
    bool blocked;
    if (o->force == 1) blocked = false;
    else if (o->force == 2) blocked = true;
    else blocked = bn > 32;  // SMALL_CUTOFF  src/svd.py:52, :375-378
    info->path = blocked ? ORC_PATH_BLOCKED : ORC_PATH_UNBLOCKED;
    const bool need_v = o->want_v || transposed;
    std::vector<T> V;
    int vrows = 0;
    if (need_v) {
        vrows = bn;
        V.assign((size_t)bn * bn, zero<T>());
        for (int c = 0; c < bn; ++c) V[c + (size_t)c * bn] = one<T>();
    }
    const double tol = o->k * tr<T>::u;
    const int inner_budget = o->inner_sweeps >= 1 ? o->inner_sweeps : 100;  // INNER_BUDGET

    Sched sc;
    std::vector<std::pair<int, int>> blocks;
    if (!blocked) {
        if (bn >= 2) sc = make_schedule(bn);
    } else {
        const int nb = o->nb;
        const int ell = (bn + nb - 1) / nb;
        for (int b = 0; b < ell; ++b) blocks.push_back({b * nb, std::min((b + 1) * nb, bn)});
        if (ell >= 2) sc = make_schedule(ell);
    }
    std::vector<Sched> inner_sched(2 * o->nb + 1);
    auto inner_for = [&](int w) -> const Sched& {
        if ((int)inner_sched.size() <= w) inner_sched.resize(w + 1);
        if (inner_sched[w].starts.empty()) inner_sched[w] = make_schedule(w);
        return inner_sched[w];
    };

    bool converged = false;
    int outer = 0;
    int64_t inner_rot = 0, gram_calls = 0, eig_calls = 0, update_calls = 0;
    std::vector<T> G, D;
    std::vector<R> d;
    T* Vp = need_v ? V.data() : nullptr;
    while (!converged && outer < o->max_nsweeps) {
        bool quiet = true;
        if (!blocked) {
            if (bn >= 2) {  // _sweep_unblocked  src/svd.py:433-447
                int sw, cv;
                const int64_t rot = onesided<T>(bmw, W.data(), bmw, vrows, Vp, bn, sc, tol, 1, &sw, &cv);
                eig_calls += 1;
                inner_rot += rot;
                quiet = rot == 0;
            }
        } else if (blocks.size() == 1) {  // _sweep_single_block  src/svd.py:461-479
            const int w = bn;
            G.assign((size_t)w * w, zero<T>());
            gram<T>(bmw, w, 0, W.data(), bmw, W.data(), bmw, G.data(), w);
            gram_calls += 1;
            d.assign(w, 0);
            for (int c = 0; c < w; ++c) d[c] = (R)realpart(G[c + (size_t)c * w]);
            for (int c = 0; c < w; ++c) G[c + (size_t)c * w] = zero<T>();
            D.assign((size_t)w * w, zero<T>());
            int64_t rot = 0;
            if (w >= 2) {
                int sw, cv;
                rot = eig_sweeps<T>(w, G.data(), w, d.data(), w, D.data(), w, inner_for(w), tol,
                                    inner_budget, true, &sw, &cv);
            }
            eig_calls += 1;
            inner_rot += rot;
            if (rot != 0) {
                quiet = false;
                fused_update<T>(bmw, w, 0, W.data(), bmw, W.data(), bmw, D.data(), w, true, false);
                if (need_v) fused_update<T>(bn, w, 0, V.data(), bn, V.data(), bn, D.data(), w, true, false);
                update_calls += 1;
            }
        } else {  // _sweep_blocked  src/svd.py:481-522
            const int P = (int)sc.pairs.size() / 2;
            for (int p = 0; p < P; ++p) {
                const int bi = sc.pairs[2 * p], bj = sc.pairs[2 * p + 1];
                const int i0 = blocks[bi].first, i1 = blocks[bi].second;
                const int j0 = blocks[bj].first, j1 = blocks[bj].second;
                const int wi = i1 - i0, wj = j1 - j0, w = wi + wj;
                T* Wi = W.data() + (size_t)i0 * bmw;
                T* Wj = W.data() + (size_t)j0 * bmw;
                G.assign((size_t)w * w, zero<T>());
                gram<T>(bmw, wi, wj, Wi, bmw, Wj, bmw, G.data(), w);
                gram_calls += 1;
                // _eig_delta  src/eig.py:151-174
                d.assign(w, 0);
                for (int c = 0; c < w; ++c) d[c] = (R)realpart(G[c + (size_t)c * w]);
                for (int c = 0; c < w; ++c) G[c + (size_t)c * w] = zero<T>();
                D.assign((size_t)w * w, zero<T>());
                int sw, cv;
                const int64_t rot = eig_sweeps<T>(w, G.data(), w, d.data(), w, D.data(), w, inner_for(w),
                                                  tol, inner_budget, true, &sw, &cv);
                eig_calls += 1;
                inner_rot += rot;
                if (rot == 0) continue;
                quiet = false;
                const bool two = !o->fused_updates;
                fused_update<T>(bmw, wi, wj, Wi, bmw, Wj, bmw, D.data(), w, true, two);
                if (need_v)
                    fused_update<T>(bn, wi, wj, V.data() + (size_t)i0 * bn, bn, V.data() + (size_t)j0 * bn,
                                    bn, D.data(), w, true, two);
                update_calls += 1;
            }
        }
        outer += 1;
        if (quiet) converged = true;
    }
    finalize<T>(bmw, bn, W.data(), bmw, Vp, bn, vrows, s);
    if (use_qr) {  // U = Q @ Uhat  (src/svd.py:529-530)
        std::vector<T> Uf((size_t)bm_in * bn, zero<T>());
        for (int j = 0; j < bn; ++j)
            for (int l = 0; l < bn; ++l) {
                const T wl = W[l + (size_t)j * bn];
                for (int i = 0; i < bm_in; ++i)
                    Uf[i + (size_t)j * bm_in] = addT(Uf[i + (size_t)j * bm_in], mulT(Q[i + (size_t)l * bm_in], wl));
            }
        W.swap(Uf);
    }
    // outputs: k = bn.  U is m x k, V is n x k.
    if (!transposed) {
        std::memcpy(u, W.data(), sizeof(T) * (size_t)bm * bn);
        if (vout && o->want_v) std::memcpy(vout, V.data(), sizeof(T) * (size_t)bn * bn);
    } else {
        std::memcpy(u, V.data(), sizeof(T) * (size_t)bn * bn);       // m x m
        if (vout && o->want_v) std::memcpy(vout, W.data(), sizeof(T) * (size_t)bm * bn);  // n x m
    }
    info->converged = converged ? 1 : 0;
    info->outer_sweeps = outer;
    info->inner_rotations = inner_rot;
    info->gram_calls = gram_calls;
    info->eig_calls = eig_calls;
    info->update_calls = update_calls;
    return 0;
}

template <class T>
int solve_batch(int m, int n, int batch, const T* a, T* u, typename tr<T>::R* s, T* v,
                const orc_opts* o, orc_info* info, int nthreads) {
    const int k = std::min(m, n);
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(min : err)
#endif
    for (int b = 0; b < batch; ++b) {
        const int rc = solve<T>(m, n, a + (size_t)b * m * n, u + (size_t)b * m * k, s + (size_t)b * k,
                                v ? v + (size_t)b * n * k : nullptr, o, &info[b]);
        if (rc < err) err = rc;
    }
    return err;
}

}  // namespace

extern "C" {

int orc_solve(int dtype, int m, int n, const void* a, void* u, void* s, void* v,
              const orc_opts* opts, orc_info* info) {
    if (m < 0 || n < 0 || !opts || !info) return -1;
    switch (dtype) {
        case ORC_S: return solve<float>(m, n, (const float*)a, (float*)u, (float*)s, (float*)v, opts, info);
        case ORC_D: return solve<double>(m, n, (const double*)a, (double*)u, (double*)s, (double*)v, opts, info);
        case ORC_C: return solve<cx<float>>(m, n, (const cx<float>*)a, (cx<float>*)u, (float*)s, (cx<float>*)v, opts, info);
        case ORC_Z: return solve<cx<double>>(m, n, (const cx<double>*)a, (cx<double>*)u, (double*)s, (cx<double>*)v, opts, info);
    }
    return -1;
}

int orc_solve_batch(int dtype, int m, int n, int batch, const void* a, void* u, void* s, void* v,
                    const orc_opts* opts, orc_info* info, int nthreads) {
    if (m < 0 || n < 0 || batch < 0 || !opts || !info) return -1;
    switch (dtype) {
        case ORC_S: return solve_batch<float>(m, n, batch, (const float*)a, (float*)u, (float*)s, (float*)v, opts, info, nthreads);
        case ORC_D: return solve_batch<double>(m, n, batch, (const double*)a, (double*)u, (double*)s, (double*)v, opts, info, nthreads);
        case ORC_C: return solve_batch<cx<float>>(m, n, batch, (const cx<float>*)a, (cx<float>*)u, (float*)s, (cx<float>*)v, opts, info, nthreads);
        case ORC_Z: return solve_batch<cx<double>>(m, n, batch, (const cx<double>*)a, (cx<double>*)u, (double*)s, (cx<double>*)v, opts, info, nthreads);
    }
    return -1;
}

int64_t orc_onesided_sweeps(int dtype, int m, int n, void* a, int vrows, void* v, double tol,
                            int max_sweeps, int* sweeps, int* conv) {
    if (n < 2) {
        if (sweeps) *sweeps = 0;
        if (conv) *conv = 0;
        return 0;
    }
    Sched sc = make_schedule(n);
    switch (dtype) {
        case ORC_S: return onesided<float>(m, (float*)a, m, vrows, (float*)v, vrows, sc, tol, max_sweeps, sweeps, conv);
        case ORC_D: return onesided<double>(m, (double*)a, m, vrows, (double*)v, vrows, sc, tol, max_sweeps, sweeps, conv);
        case ORC_C: return onesided<cx<float>>(m, (cx<float>*)a, m, vrows, (cx<float>*)v, vrows, sc, tol, max_sweeps, sweeps, conv);
        case ORC_Z: return onesided<cx<double>>(m, (cx<double>*)a, m, vrows, (cx<double>*)v, vrows, sc, tol, max_sweeps, sweeps, conv);
    }
    return -1;
}

int64_t orc_eig_sweeps(int dtype, int w, void* g, void* d, int mrows, void* mm, double tol,
                       int max_sweeps, int delta, int* sweeps, int* conv) {
    if (w < 2) {
        if (sweeps) *sweeps = 0;
        if (conv) *conv = 0;
        return 0;
    }
    Sched sc = make_schedule(w);
    switch (dtype) {
        case ORC_S: return eig_sweeps<float>(w, (float*)g, w, (float*)d, mrows, (float*)mm, mrows, sc, tol, max_sweeps, delta, sweeps, conv);
        case ORC_D: return eig_sweeps<double>(w, (double*)g, w, (double*)d, mrows, (double*)mm, mrows, sc, tol, max_sweeps, delta, sweeps, conv);
        case ORC_C: return eig_sweeps<cx<float>>(w, (cx<float>*)g, w, (float*)d, mrows, (cx<float>*)mm, mrows, sc, tol, max_sweeps, delta, sweeps, conv);
        case ORC_Z: return eig_sweeps<cx<double>>(w, (cx<double>*)g, w, (double*)d, mrows, (cx<double>*)mm, mrows, sc, tol, max_sweeps, delta, sweeps, conv);
    }
    return -1;
}

void orc_compute_gram(int dtype, int m, int wi, int wj, const void* ai, const void* aj, void* g) {
    const int w = wi + wj;
    switch (dtype) {
        case ORC_S: gram<float>(m, wi, wj, (const float*)ai, m, (const float*)aj, m, (float*)g, w); break;
        case ORC_D: gram<double>(m, wi, wj, (const double*)ai, m, (const double*)aj, m, (double*)g, w); break;
        case ORC_C: gram<cx<float>>(m, wi, wj, (const cx<float>*)ai, m, (const cx<float>*)aj, m, (cx<float>*)g, w); break;
        case ORC_Z: gram<cx<double>>(m, wi, wj, (const cx<double>*)ai, m, (const cx<double>*)aj, m, (cx<double>*)g, w); break;
    }
}

void orc_fused_pair_update(int dtype, int m, int wi, int wj, void* bi, void* bj, const void* j,
                           int row_block, int delta) {
    (void)row_block;
    const int w = wi + wj;
    switch (dtype) {
        case ORC_S: fused_update<float>(m, wi, wj, (float*)bi, m, (float*)bj, m, (const float*)j, w, delta, false); break;
        case ORC_D: fused_update<double>(m, wi, wj, (double*)bi, m, (double*)bj, m, (const double*)j, w, delta, false); break;
        case ORC_C: fused_update<cx<float>>(m, wi, wj, (cx<float>*)bi, m, (cx<float>*)bj, m, (const cx<float>*)j, w, delta, false); break;
        case ORC_Z: fused_update<cx<double>>(m, wi, wj, (cx<double>*)bi, m, (cx<double>*)bj, m, (const cx<double>*)j, w, delta, false); break;
    }
}

int orc_schedule(int ell, int* pairs, int* starts, int* n_iter) {
    if (ell < 2) return -1;
    Sched s = make_schedule(ell);
    std::memcpy(pairs, s.pairs.data(), sizeof(int) * s.pairs.size());
    std::memcpy(starts, s.starts.data(), sizeof(int) * s.starts.size());
    *n_iter = s.n_iter;
    return (int)s.pairs.size() / 2;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

}  // extern "C"
