// finalize.cuh -- kernel (5): finalisation fused into the solver kernels.
//
// Restates _finalize_factors (src/svd.py:243-275) and _orthogonal_completion
// (src/svd.py:224-240) as a CTA-cooperative device routine that runs on the
// converged working copy while it is still resident (smem or L2):
//   sigma_c = sqrt(sum_r |w_rc|^2) accumulated in float64, cast to the real dtype;
//   sigma_c < tiny/u -> sigma_c = 0 and U column by orthogonal completion;
//   U_c = W_c / sigma_c (complex: times the reciprocal, as numpy divides);
//   stable descending order, U and V permuted alike, then the transpose route
//   swaps the factors (src/svd.py:531-536).
#pragma once

#include "common.cuh"

namespace bsvd {

template <class T>
struct FinalOut {
    T* U;                      // m x k, ldu (already offset to this problem)
    int64_t ldu;
    typename tr<T>::R* S;      // k
    T* V;                      // n x k, ldv, or nullptr
    int64_t ldv;
    bool trans;                // W holds (A^H) factors: U_out = V_fac, V_out = U_fac
    bool want_v;
};

template <class T>
BSVD_DEV T scale_by_sigma(T x, typename tr<T>::R s) {
    if constexpr (tr<T>::cplx) {
        const typename tr<T>::R r = (typename tr<T>::R)1 / s;  // numpy complex / real
        return T{x.re * r, x.im * r};
    } else if constexpr (sizeof(T) == 8) {
        return div_by_sigma(x, s, rcp_refined(s));  // the fused finalisations' formula, bit for bit
    } else {
        return div_by_sigma_f(x, s, __frcp_rn(s));  // the 16x16 kernels' fused formula, bit for bit
    }
}

// `before(a, b)`: a sorts before b under argsort(-sigma, stable) (NaN last).
template <class R>
BSVD_DEV bool sig_before(R a, R b) {
    if (isnan(b)) return !isnan(a);
    return a > b;
}
template <class R>
BSVD_DEV bool sig_tie(R a, R b) {
    return (isnan(a) && isnan(b)) || a == b;
}

// All threads of the CTA must call.  W: bm x bn (ldw), Vw: bn x bn (ldvw) or null.
// sig, perm: smem scratch of bn entries; flag: smem int.
template <class T>
__device__ void finalize_block(T* W, int ldw, int bm, int bn, T* Vw, int ldvw,
                               typename tr<T>::R* sig, int* perm, int* flag,
                               const FinalOut<T>& o, int vrows = -1) {
    if (vrows < 0) vrows = bn;  // rows of Vw (the standalone finalize operator allows any)
    using R = typename tr<T>::R;
    using Wt = typename tr<T>::W;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    // 1. column norms in float64.  FP64 columns are first scaled by a power of two from their largest
    // component (the reference's np.linalg.norm is underflow/overflow-safe; plain squares of a column
    // at 1e-200 vanish): exact, so the bits are those of the plain sum wherever its squares are
    // representable -- and those of the register kernels' fused finalisation, which sums the squares
    // of the problem-scaled W.  FP32 squares are exact and in range in float64.
    for (int c = warp; c < bn; c += nw) {
        double acc = 0.0;
        if constexpr (sizeof(R) == 8) {
            double mx = 0.0;
            for (int r = lane; r < bm; r += 32) mx = fmax(mx, abs_component(W[r + (size_t)c * ldw]));
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            int e = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1023;
            if (!(mx > 0.0) || !isfinite(mx)) e = 0;
            e = max(-1021, min(1021, e));
            const double sd = __longlong_as_double((long long)(1023 - e) << 52);
            for (int r = lane; r < bm; r += 32) acc += norm2d_scaled(W[r + (size_t)c * ldw], sd);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) sig[c] = (R)(sqrt(acc) * __longlong_as_double((long long)(1023 + e) << 52));
        } else {
            for (int r = lane; r < bm; r += 32) acc += norm2d(W[r + (size_t)c * ldw]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) sig[c] = (R)sqrt(acc);
        }
    }
    if (tid == 0) *flag = 0;
    __syncthreads();
    const double tiny = dtiny<T>();
    // 2. normalise formed columns; detect holes
    for (int e = tid; e < bm * bn; e += nt) {
        const int r = e % bm, c = e / bm;
        const R sc = sig[c];
        if ((double)sc < tiny) {
            if (r == 0) atomicOr(flag, 1);
        } else {
            W[r + (size_t)c * ldw] = scale_by_sigma(W[r + (size_t)c * ldw], sc);
        }
    }
    __syncthreads();
    // 3. orthogonal completion of the holes (rare: rank-deficient / zero columns)
    if (*flag) {
        for (int c = tid; c < bn; c += nt)
            if ((double)sig[c] < tiny) sig[c] = 0;
        __syncthreads();
        if (warp == 0) {
            for (int hole = 0; hole < bn; ++hole) {
                if (sig[hole] != 0) continue;
                // formed = nonzero columns ascending, then holes < `hole` ascending
                // load[r] = sum_formed |u_rc|^2 ; k = first argmin
                double best = CUDART_INF;
                int bestr = 0x7fffffff;
                for (int r = lane; r < bm; r += 32) {
                    double ld = 0.0;
                    for (int c = 0; c < bn; ++c)
                        if (sig[c] != 0) ld += norm2d(W[r + (size_t)c * ldw]);
                    for (int c = 0; c < hole; ++c)
                        if (sig[c] == 0) ld += norm2d(W[r + (size_t)c * ldw]);
                    if (ld < best || (ld == best && r < bestr)) { best = ld; bestr = r; }
                }
                for (int off = 16; off > 0; off >>= 1) {
                    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                    const int orr = __shfl_xor_sync(0xffffffffu, bestr, off);
                    if (ob < best || (ob == best && orr < bestr)) { best = ob; bestr = orr; }
                }
                T* x = W + (size_t)hole * ldw;
                for (int r = lane; r < bm; r += 32) x[r] = (r == bestr) ? one<T>() : zero<T>();
                __syncwarp();
                for (int pass = 0; pass < 2; ++pass) {
                    for (int stage = 0; stage < 2; ++stage) {
                        for (int c = 0; c < (stage == 0 ? bn : hole); ++c) {
                            const bool use = stage == 0 ? (sig[c] != 0) : (sig[c] == 0);
                            if (!use) continue;
                            const T* uc = W + (size_t)c * ldw;
                            Wt dot{};
                            for (int r = lane; r < bm; r += 32) {
                                const Wt a = wide(conjT(uc[r])), b = wide(x[r]);
                                if constexpr (tr<T>::cplx) {
                                    dot.re += a.re * b.re - a.im * b.im;
                                    dot.im += a.re * b.im + a.im * b.re;
                                } else {
                                    dot += a * b;
                                }
                            }
#pragma unroll
                            for (int off = 16; off > 0; off >>= 1) {
                                if constexpr (tr<T>::cplx) {
                                    dot.re += __shfl_xor_sync(0xffffffffu, dot.re, off);
                                    dot.im += __shfl_xor_sync(0xffffffffu, dot.im, off);
                                } else {
                                    dot += __shfl_xor_sync(0xffffffffu, dot, off);
                                }
                            }
                            for (int r = lane; r < bm; r += 32) {
                                const Wt a = wide(uc[r]);
                                Wt xr = wide(x[r]);
                                if constexpr (tr<T>::cplx) {
                                    xr.re -= a.re * dot.re - a.im * dot.im;
                                    xr.im -= a.re * dot.im + a.im * dot.re;
                                } else {
                                    xr -= a * dot;
                                }
                                store(&x[r], xr);
                            }
                            __syncwarp();
                        }
                    }
                }
                double nrm = 0.0;
                for (int r = lane; r < bm; r += 32) nrm += norm2d(x[r]);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, off);
                nrm = sqrt(nrm);
                for (int r = lane; r < bm; r += 32) {
                    Wt xr = wide(x[r]);
                    if constexpr (tr<T>::cplx) { xr.re /= nrm; xr.im /= nrm; } else { xr /= nrm; }
                    store(&x[r], xr);
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }
    // 4. stable descending ranks
    for (int c = tid; c < bn; c += nt) {
        const R sc = sig[c];
        int rank = 0;
        for (int c2 = 0; c2 < bn; ++c2) {
            const R s2 = sig[c2];
            rank += sig_before(s2, sc) || (c2 < c && sig_tie(s2, sc));
        }
        perm[rank] = c;
    }
    __syncthreads();
    // 5. permuted outputs (transpose route swaps the factors)
    T* Uo = o.trans ? o.V : o.U;
    const int64_t ldUo = o.trans ? o.ldv : o.ldu;
    const bool writeW = o.trans ? o.want_v : true;
    if (writeW && Uo) {
        for (int e = tid; e < bm * bn; e += nt) {
            const int r = e % bm, c = e / bm;
            Uo[r + (size_t)c * ldUo] = W[r + (size_t)perm[c] * ldw];
        }
    }
    T* Vo = o.trans ? o.U : o.V;
    const int64_t ldVo = o.trans ? o.ldu : o.ldv;
    const bool writeV = o.trans ? true : o.want_v;
    if (writeV && Vo && Vw) {
        for (int e = tid; e < vrows * bn; e += nt) {
            const int r = e % vrows, c = e / vrows;
            Vo[r + (size_t)c * ldVo] = Vw[r + (size_t)perm[c] * ldvw];
        }
    }
    for (int c = tid; c < bn; c += nt) o.S[c] = sig[perm[c]];
}

}  // namespace bsvd
