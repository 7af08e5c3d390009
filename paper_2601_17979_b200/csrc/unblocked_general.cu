// unblocked_general.cu -- kernel (2), general form: one CTA per problem.
//
// Restates onesided_sweeps (src/_kernels_numba.py:85-138) driven sweep by
// sweep as in _ProblemRun.sweep / _sweep_unblocked (src/svd.py:417-447), with
// the batch driver's per-problem convergence test (src/batch.py:62-82) done
// on the device: a CTA stops after its first zero-rotation sweep.
//
// Mapping: the working copy W (bm x bn) and V (bn x bn) stay resident in
// shared memory when they fit (else in a global workspace, L2-resident).
// Each iteration of the round-robin schedule has floor(bn/2) disjoint column
// pairs (F9); a group of G lanes owns one pair: the three dot products are
// lane-strided over rows and combined with an xor butterfly (every lane ends
// with bit-identical sums, so all lanes derive identical rotation
// parameters), then the rotation is applied to the pair's rows of W and V.
// One __syncthreads separates schedule iterations.  This is the shape-generic
// path (any m >= n, any dtype); the 32-column FP64 fast path lives in
// unblocked_reg.cu.
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {

// One problem's unblocked sweeps on a resident working copy (all CTA threads).
// W: bm x bn (ldw), Vw: vrows x bn (ldv) or null.  misc[0] is a zeroed smem
// counter.  Semantics of onesided_sweeps(max_sweeps) + _ProblemRun.sweep:
// stops after the first zero-rotation sweep, which is counted.
template <class T>
__device__ void onesided_sweeps_dev(T* W, int64_t ldw, int bm, int bn, T* Vw, int64_t ldv, int vrows,
                                    double tol, int max_sweeps, int G, int* misc, int& sweeps,
                                    long long& rot_total, int& last, bool& conv) {
    using R = typename tr<T>::R;
    using Wt = typename tr<T>::W;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int gid = tid / G, lg = tid % G, ngroups = nt / G;
    const int S = bn + (bn & 1), h = S >> 1, n_it = S - 1;
    sweeps = 0;
    last = 0;
    conv = false;
    rot_total = 0;
    if (bn < 2) {
        // no pairs: one quiet sweep (src/svd.py:434-436)
        conv = true;
        sweeps = 1;
        return;
    }
    for (int sw = 0; sw < max_sweeps; ++sw) {
        int my_rot = 0;
        for (int t = 0; t < n_it; ++t) {
            for (int k0 = 0; k0 < h; k0 += ngroups) {
                const int k = k0 + gid;
                int i = 0, j = 0;
                const bool valid = (k < h) && rr_pair(t, k, S, bn, i, j);
                double gii = 0.0, gjj = 0.0;
                T gji = zero<T>();
                if (valid) {
                    const T* ci = W + (size_t)i * ldw;
                    const T* cj = W + (size_t)j * ldw;
                    for (int r = lg; r < bm; r += G) {
                        const T x = ci[r], y = cj[r];
                        gii += norm2d(x);
                        gjj += norm2d(y);
                        gji = cmac(gji, y, x);  // += conj(a_j) a_i
                    }
                }
                for (int o = G >> 1; o > 0; o >>= 1) {
                    gii += shfl_xor(gii, o);
                    gjj += shfl_xor(gjj, o);
                    gji = addT(gji, shfl_xor(gji, o));
                }
                if (valid) {
                    const R absg = absT(gji);
                    // guard F4: |g| > 0 and |g| >= tol sqrt(gii gjj)
                    if (!(absg <= (R)0) && !((double)absg < tol * sqrt(gii * gjj))) {
                        const T w = divR(conjT(gji), absg);
                        const RotParams p = rot_params(gii - gjj, 2.0 * (double)absg);
                        const Wt ws = scaleW(p.s, wide(w));
                        const Wt wsc = scaleW(p.s, wide(conjT(w)));
                        T* ci = W + (size_t)i * ldw;
                        T* cj = W + (size_t)j * ldw;
                        for (int r = lg; r < bm; r += G) {
                            Wt xi = wide(ci[r]), xj = wide(cj[r]);
                            rot_pair(xi, xj, p.cm1, ws, wsc);
                            store(&ci[r], xi);
                            store(&cj[r], xj);
                        }
                        if (Vw) {
                            T* vi = Vw + (size_t)i * ldv;
                            T* vj = Vw + (size_t)j * ldv;
                            for (int r = lg; r < vrows; r += G) {
                                Wt xi = wide(vi[r]), xj = wide(vj[r]);
                                rot_pair(xi, xj, p.cm1, ws, wsc);
                                store(&vi[r], xi);
                                store(&vj[r], xj);
                            }
                        }
                        my_rot += (lg == 0);
                    }
                }
            }
            __syncthreads();
        }
        int v = my_rot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&misc[0], v);
        __syncthreads();
        const int total = misc[0];
        __syncthreads();
        if (tid == 0) misc[0] = 0;
        sweeps = sw + 1;
        last = total;
        if (total == 0) {
            conv = true;
            break;
        }
        rot_total += total;
    }
}

template <class T>
__global__ void __launch_bounds__(512) k_unblocked_general(SolveArgs<T> a) {
    using R = typename tr<T>::R;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x;
    const int bm = a.bm, bn = a.bn;
    const int tid = threadIdx.x;
    T* gws = a.work ? a.work + (size_t)prob * a.work_stride : nullptr;
    size_t off = 0;
    T* W;
    T* Vw = nullptr;
    if (a.resident & 1) {
        W = reinterpret_cast<T*>(smem);
        off += (size_t)bm * bn * sizeof(T);
    } else {
        W = gws;
    }
    if (a.need_v) {
        if (a.resident & 2) {
            Vw = reinterpret_cast<T*>(smem + off);
            off += (size_t)bn * bn * sizeof(T);
        } else {
            Vw = gws + (size_t)bm * bn;
        }
    }
    off = (off + 15) & ~size_t(15);
    R* sig = reinterpret_cast<R*>(smem + off);
    off += ((size_t)bn * sizeof(R) + 15) & ~size_t(15);
    int* perm = reinterpret_cast<int*>(smem + off);
    off += ((size_t)bn * sizeof(int) + 15) & ~size_t(15);
    int* misc = reinterpret_cast<int*>(smem + off);  // [0] rotations, [1] flag, [2] bad input
    if (tid < 4) misc[tid] = 0;
    __syncthreads();
    load_problem(a, prob, W, bm, Vw, bn, &misc[2]);
    __syncthreads();
    int sweeps, last;
    long long rot_total;
    bool conv;
    onesided_sweeps_dev<T>(W, bm, bm, bn, Vw, bn, bn, a.tol, a.max_sweeps, a.group, misc, sweeps, rot_total,
                           last, conv);
    finalize_block<T>(W, bm, bm, bn, Vw, bn, sig, perm, &misc[1], final_out(a, prob));
    if (tid == 0 && a.info) {
        bsvd_info inf;
        inf.converged = conv ? 1 : 0;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = 0;
        inf.update_calls = 0;
        inf.last_rotations = last;
        inf.path = 1 | (a.trans ? 0x100 : 0);
        inf.status = misc[2] ? 1 : 0;
        inf.kernel = KV_UNBLOCKED_GENERAL;
        a.info[prob] = inf;
    }
}

// Kernel-level operator: onesided_sweeps on `batch` problems in place (global memory).
template <class T>
__global__ void __launch_bounds__(512) k_onesided_raw(T* A, int64_t lda, int64_t sa, int m, int n, T* V,
                                                       int64_t ldv, int64_t sv, int vrows, double tol,
                                                       int max_sweeps, int G, int64_t* rotations,
                                                       int32_t* sweeps_out) {
    __shared__ int misc[4];
    if (threadIdx.x < 4) misc[threadIdx.x] = 0;
    __syncthreads();
    const int prob = blockIdx.x;
    int sweeps, last;
    long long rot_total;
    bool conv;
    onesided_sweeps_dev<T>(A + (size_t)prob * sa, lda, m, n, V ? V + (size_t)prob * sv : nullptr, ldv, vrows,
                           tol, max_sweeps, G, misc, sweeps, rot_total, last, conv);
    if (threadIdx.x == 0) {
        if (rotations) rotations[prob] = rot_total;
        if (sweeps_out) sweeps_out[prob] = ((n < 2) ? 0 : sweeps) | ((conv && n >= 2) ? (1 << 30) : 0);
    }
}

int group_for_rows(int bm) {
    if (bm >= 128) return 32;
    if (bm >= 64) return 16;
    if (bm >= 24) return 8;
    if (bm >= 8) return 4;
    return 2;
}

int threads_for(int bn, int G) {
    const int h = (bn + 1) / 2;
    int threads = h * G;
    threads = (threads + 31) / 32 * 32;
    if (threads < 64) threads = 64;
    if (threads > 512) threads = 512;
    return threads;
}

template <class T>
int launch_onesided_raw(T* A, int64_t lda, int64_t sa, int m, int n, int batch, T* V, int64_t ldv, int64_t sv,
                        int vrows, double tol, int max_sweeps, int64_t* rot, int32_t* sw, cudaStream_t st) {
    const int G = group_for_rows(m > vrows ? m : vrows);
    k_onesided_raw<T><<<batch, threads_for(n, G), 0, st>>>(A, lda, sa, m, n, V, ldv, sv, vrows, tol, max_sweeps,
                                                            G, rot, sw);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}
template int launch_onesided_raw<float>(float*, int64_t, int64_t, int, int, int, float*, int64_t, int64_t, int,
                                        double, int, int64_t*, int32_t*, cudaStream_t);
template int launch_onesided_raw<double>(double*, int64_t, int64_t, int, int, int, double*, int64_t, int64_t, int,
                                         double, int, int64_t*, int32_t*, cudaStream_t);
template int launch_onesided_raw<cx<float>>(cx<float>*, int64_t, int64_t, int, int, int, cx<float>*, int64_t,
                                            int64_t, int, double, int, int64_t*, int32_t*, cudaStream_t);
template int launch_onesided_raw<cx<double>>(cx<double>*, int64_t, int64_t, int, int, int, cx<double>*, int64_t,
                                             int64_t, int, double, int, int64_t*, int32_t*, cudaStream_t);

// --------------------------------------------------------------------------
// planning and launch
// --------------------------------------------------------------------------
static inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

Plan plan_unblocked_general(int esize, int rsize, int bm, int bn, int need_v, size_t smem_limit) {
    Plan p{};
    const size_t wb = (size_t)bm * bn * esize;
    const size_t vb = need_v ? (size_t)bn * bn * esize : 0;
    const size_t fixed = al16((size_t)bn * rsize) + al16((size_t)bn * 4) + 64;
    if (al16(wb + vb) + fixed <= smem_limit) {
        p.resident = 3;
        p.smem = al16(wb + vb) + fixed;
        p.work_elems = 0;
    } else if (al16(wb) + fixed <= smem_limit) {
        p.resident = 1;
        p.smem = al16(wb) + fixed;
        p.work_elems = (size_t)bm * bn + (need_v ? (size_t)bn * bn : 0);
    } else {
        p.resident = 0;
        p.smem = fixed;
        p.work_elems = (size_t)bm * bn + (need_v ? (size_t)bn * bn : 0);
    }
    const int G = group_for_rows(bm);
    const int threads = threads_for(bn, G);
    p.group = G;
    p.threads = threads;
    p.kernel = KV_UNBLOCKED_GENERAL;
    return p;
}

template <class T>
int launch_unblocked_general(SolveArgs<T> a, const Plan& p, cudaStream_t st) {
    a.resident = p.resident;
    a.group = p.group;
    a.kernel = KV_UNBLOCKED_GENERAL;
    auto kern = k_unblocked_general<T>;
    if (p.smem > 48 * 1024) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
            return BSVD_ERR_CUDA;
    }
    kern<<<a.batch, p.threads, p.smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template int launch_unblocked_general<float>(SolveArgs<float>, const Plan&, cudaStream_t);
template int launch_unblocked_general<double>(SolveArgs<double>, const Plan&, cudaStream_t);
template int launch_unblocked_general<cx<float>>(SolveArgs<cx<float>>, const Plan&, cudaStream_t);
template int launch_unblocked_general<cx<double>>(SolveArgs<cx<double>>, const Plan&, cudaStream_t);

}  // namespace bsvd
