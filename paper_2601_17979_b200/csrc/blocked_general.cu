// blocked_general.cu -- kernel (3), general form: blocked one-sided Jacobi,
// one CTA per problem.
//
// Restates _sweep_blocked / _sweep_single_block (src/svd.py:461-522): per
// block pair (round-robin over ell = ceil(bn/nb) blocks, src/ordering.py),
//   compute_gram   G = [Wi Wj]^H [Wi Wj]       (src/svd.py:144-179)
//   _eig_delta     inner_budget sweeps of two-sided Jacobi on G, accumulating
//                  Delta = P - I              (src/eig.py:151-174,
//                                               src/_kernels_numba.py:17-82)
//   fused update   [Wi Wj] += [Wi Wj] Delta, same on V
//                                              (src/_kernels_numba.py:141-175)
// A sweep with zero inner rotations ends the problem (src/svd.py:417-431).
//
// The inner eigensolve runs the floor(w/2) disjoint rotations of a schedule
// iteration in parallel: each thread owns one 2x2 block (p < q) of G and
// applies rotation p to its rows and then rotation q to its columns, the same
// order the reference's sequential loop uses, and writes the conjugate mirror,
// so G stays exactly Hermitian.  This is the shape-generic path (any nb, any
// dtype); W, V, G and Delta live in shared memory when they fit.
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {

template <class T>
struct InnerRot {
    typename tr<T>::W ws, wsc;
    double cm1;
    int i, j;  // j < 0: unpaired index this iteration
    int rot;
};

template <class T>
__global__ void __launch_bounds__(256) k_blocked_general(SolveArgs<T> a) {
    using R = typename tr<T>::R;
    using Wt = typename tr<T>::W;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x;
    const int bm = a.bm, bn = a.bn, nb = a.nb;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int wmax = bn < 2 * nb ? bn : 2 * nb;
    const int hmax = (wmax + 1) / 2;
    constexpr int RT = 32;  // update row tile
    T* gws = a.work ? a.work + (size_t)prob * a.work_stride : nullptr;
    size_t goff = 0;
    size_t off = 0;
    auto take = [&](size_t elems, bool in_smem) -> T* {
        T* p;
        if (in_smem) {
            p = reinterpret_cast<T*>(smem + off);
            off = (off + elems * sizeof(T) + 15) & ~size_t(15);
        } else {
            p = gws + goff;
            goff += elems;
        }
        return p;
    };
    T* W = take((size_t)bm * bn, a.resident & 1);
    T* Vw = a.need_v ? take((size_t)bn * bn, a.resident & 2) : nullptr;
    T* G = take((size_t)wmax * wmax, a.resident & 4);
    T* D = take((size_t)wmax * wmax, a.resident & 4);
    T* Tl = take((size_t)RT * wmax, a.resident & 4);
    R* d = reinterpret_cast<R*>(smem + off);
    off = (off + (size_t)wmax * sizeof(R) + 15) & ~size_t(15);
    InnerRot<T>* prm = reinterpret_cast<InnerRot<T>*>(smem + off);
    off = (off + (size_t)hmax * sizeof(InnerRot<T>) + 15) & ~size_t(15);
    R* sig = reinterpret_cast<R*>(smem + off);
    off = (off + (size_t)bn * sizeof(R) + 15) & ~size_t(15);
    int* perm = reinterpret_cast<int*>(smem + off);
    off = (off + (size_t)bn * sizeof(int) + 15) & ~size_t(15);
    int* misc = reinterpret_cast<int*>(smem + off);  // [0] inner rot counter, [1] flag, [2] bad
    if (tid < 4) misc[tid] = 0;
    __syncthreads();
    load_problem(a, prob, W, bm, Vw, bn, &misc[2]);
    __syncthreads();

    const int ell = (bn + nb - 1) / nb;
    const int Sb = ell + (ell & 1), hb = ell >= 2 ? Sb / 2 : 1, nib = ell >= 2 ? Sb - 1 : 1;
    int sweeps = 0, last = 0;
    bool conv = false;
    long long rot_total = 0, gram_calls = 0, update_calls = 0;
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
        long long sweep_rot = 0;
        for (int tb = 0; tb < nib; ++tb) {
            for (int kb = 0; kb < hb; ++kb) {
                int i0, wi, j0, wj;
                if (ell >= 2) {
                    int bi, bj;
                    if (!rr_pair(tb, kb, Sb, ell, bi, bj)) continue;
                    i0 = bi * nb;
                    wi = min(nb, bn - i0);
                    j0 = bj * nb;
                    wj = min(nb, bn - j0);
                } else {
                    i0 = 0;
                    wi = bn;
                    j0 = 0;
                    wj = 0;
                }
                const int w = wi + wj;
                auto colp = [&](T* base, int ld, int x) -> T* {
                    return base + (size_t)(x < wi ? i0 + x : j0 + x - wi) * ld;
                };
                // 1. Gram, upper triangle + conjugate mirror, real diagonal
                for (int e = tid; e < w * w; e += nt) {
                    const int ra = e % w, cb = e / w;
                    if (ra > cb) continue;
                    const T* xa = colp(W, bm, ra);
                    const T* xb = colp(W, bm, cb);
                    T acc = zero<T>();
                    for (int r = 0; r < bm; ++r) acc = cmac(acc, xa[r], xb[r]);
                    if (ra == cb) {
                        if constexpr (tr<T>::cplx) d[ra] = acc.re; else d[ra] = acc;
                        G[ra + (size_t)cb * w] = zero<T>();
                    } else {
                        G[ra + (size_t)cb * w] = acc;
                        G[cb + (size_t)ra * w] = conjT(acc);
                    }
                }
                for (int e = tid; e < w * w; e += nt) D[e] = zero<T>();
                __syncthreads();
                gram_calls += 1;
                // 2. inner Jacobi sweeps with Delta accumulation
                long long pair_rot = 0;
                if (w >= 2) {
                    const int Sw = w + (w & 1), hw = Sw / 2, nitw = Sw - 1;
                    for (int isw = 0; isw < a.inner_budget; ++isw) {
                        for (int tw = 0; tw < nitw; ++tw) {
                            for (int p = tid; p < hw; p += nt) {
                                int i, j;
                                const bool v = rr_pair(tw, p, Sw, w, i, j);
                                InnerRot<T> pr;
                                pr.i = i;
                                pr.j = v ? j : -1;
                                pr.rot = 0;
                                pr.cm1 = 0.0;
                                pr.ws = Wt{};
                                pr.wsc = Wt{};
                                if (v) {
                                    const T gij = G[i + (size_t)j * w];
                                    const R absg = absT(gij);
                                    const R sq = sqrt((R)(fabs(d[i]) * fabs(d[j])));
                                    if (!(absg <= (R)0) && !((double)absg < a.tol * (double)sq)) {
                                        const T wph = divR(gij, absg);
                                        const R dd = d[i] - d[j];
                                        const RotParams q = rot_params((double)dd, 2.0 * (double)absg);
                                        pr.rot = 1;
                                        pr.cm1 = q.cm1;
                                        pr.ws = scaleW(q.s, wide(wph));
                                        pr.wsc = scaleW(q.s, wide(conjT(wph)));
                                        const double td = q.t * (double)absg;
                                        d[i] = (R)((double)d[i] + td);
                                        d[j] = (R)((double)d[j] - td);
                                        atomicAdd(&misc[0], 1);
                                    }
                                }
                                prm[p] = pr;
                            }
                            __syncthreads();
                            // G <- J^H G J over 2x2 blocks (p < q), mirror kept exact
                            for (int e = tid; e < hw * hw; e += nt) {
                                const int p = e / hw, q = e % hw;
                                const InnerRot<T> P = prm[p];
                                if (p == q) {
                                    if (P.rot) {
                                        G[P.i + (size_t)P.j * w] = zero<T>();
                                        G[P.j + (size_t)P.i * w] = zero<T>();
                                    }
                                    continue;
                                }
                                if (p > q) continue;
                                const InnerRot<T> Q = prm[q];
                                if (!P.rot && !Q.rot) continue;
                                const int np = P.j >= 0 ? 2 : 1, nq = Q.j >= 0 ? 2 : 1;
                                const int ip[2] = {P.i, P.j}, iq[2] = {Q.i, Q.j};
                                Wt x[2][2];
                                for (int u = 0; u < np; ++u)
                                    for (int v2 = 0; v2 < nq; ++v2) x[u][v2] = wide(G[ip[u] + (size_t)iq[v2] * w]);
                                if (P.rot)  // rows i_p, j_p: x_i + (cm1 x_i + ws x_j), x_j + (cm1 x_j - wsc x_i)
                                    for (int v2 = 0; v2 < nq; ++v2) rot_pair(x[0][v2], x[1][v2], P.cm1, P.wsc, P.ws);
                                if (Q.rot)  // columns i_q, j_q: x_i + (cm1 x_i + wsc x_j), x_j + (cm1 x_j - ws x_i)
                                    for (int u = 0; u < np; ++u) rot_pair(x[u][0], x[u][1], Q.cm1, Q.ws, Q.wsc);
                                for (int u = 0; u < np; ++u)
                                    for (int v2 = 0; v2 < nq; ++v2) {
                                        store(&G[ip[u] + (size_t)iq[v2] * w], x[u][v2]);
                                        store(&G[iq[v2] + (size_t)ip[u] * w], conjW(x[u][v2]));
                                    }
                            }
                            // Delta columns of every rotated pair, then the identity terms
                            for (int e = tid; e < w * hw; e += nt) {
                                const int r = e % w, p = e / w;
                                const InnerRot<T> P = prm[p];
                                if (!P.rot) continue;
                                Wt xi = wide(D[r + (size_t)P.i * w]), xj = wide(D[r + (size_t)P.j * w]);
                                rot_pair(xi, xj, P.cm1, P.ws, P.wsc);
                                if (r == P.i) {
                                    if constexpr (tr<T>::cplx) xi.re += P.cm1; else xi += P.cm1;
                                    if constexpr (tr<T>::cplx) { xj.re -= P.ws.re; xj.im -= P.ws.im; } else xj -= P.ws;
                                }
                                if (r == P.j) {
                                    if constexpr (tr<T>::cplx) { xi.re += P.wsc.re; xi.im += P.wsc.im; } else xi += P.wsc;
                                    if constexpr (tr<T>::cplx) xj.re += P.cm1; else xj += P.cm1;
                                }
                                store(&D[r + (size_t)P.i * w], xi);
                                store(&D[r + (size_t)P.j * w], xj);
                            }
                            __syncthreads();
                        }
                        const int irot = misc[0];
                        __syncthreads();
                        if (tid == 0) misc[0] = 0;
                        pair_rot += irot;
                        if (irot == 0) break;
                    }
                }
                if (pair_rot == 0) continue;
                sweep_rot += pair_rot;
                update_calls += 1;
                // 3. fused update [Bi Bj] += [Bi Bj] Delta in row tiles (W, then V)
                for (int pass = 0; pass < (a.need_v ? 2 : 1); ++pass) {
                    T* B = pass == 0 ? W : Vw;
                    const int rows = pass == 0 ? bm : bn;
                    for (int r0 = 0; r0 < rows; r0 += RT) {
                        const int rt = min(RT, rows - r0);
                        for (int e = tid; e < rt * w; e += nt) {
                            const int rr = e % rt, x = e / rt;
                            Tl[rr + x * RT] = colp(B, rows, x)[r0 + rr];
                        }
                        __syncthreads();
                        for (int e = tid; e < rt * w; e += nt) {
                            const int rr = e % rt, q = e / rt;
                            T z = zero<T>();
                            for (int k = 0; k < w; ++k) z = mac(z, Tl[rr + k * RT], D[k + (size_t)q * w]);
                            colp(B, rows, q)[r0 + rr] = addT(Tl[rr + q * RT], z);
                        }
                        __syncthreads();
                    }
                }
            }
        }
        sweeps = sw + 1;
        last = (int)sweep_rot;
        if (sweep_rot == 0) {
            conv = true;
            break;
        }
        rot_total += sweep_rot;
    }
    finalize_block<T>(W, bm, bm, bn, Vw, bn, sig, perm, &misc[1], final_out(a, prob));
    if (tid == 0 && a.info) {
        bsvd_info inf;
        inf.converged = conv ? 1 : 0;
        inf.outer_sweeps = sweeps;
        inf.rotations = rot_total;
        inf.gram_calls = gram_calls;
        inf.update_calls = update_calls;
        inf.last_rotations = last;
        inf.path = 2 | (a.trans ? 0x100 : 0);
        inf.status = misc[2] ? 1 : 0;
        inf.kernel = KV_BLOCKED_GENERAL;
        a.info[prob] = inf;
    }
}

static inline size_t al16b(size_t x) { return (x + 15) & ~size_t(15); }

Plan plan_blocked_general(int esize, int rsize, int bm, int bn, int nb, int need_v, size_t smem_limit) {
    Plan p{};
    const int wmax = bn < 2 * nb ? bn : 2 * nb;
    const int hmax = (wmax + 1) / 2;
    const size_t wb = al16b((size_t)bm * bn * esize);
    const size_t vb = need_v ? al16b((size_t)bn * bn * esize) : 0;
    const size_t sb = 2 * al16b((size_t)wmax * wmax * esize) + al16b((size_t)32 * wmax * esize);
    const size_t rotsz = 64;  // >= sizeof(InnerRot<T>) for every T
    const size_t fixed = al16b((size_t)wmax * rsize) + al16b((size_t)hmax * rotsz) + al16b((size_t)bn * rsize) +
                         al16b((size_t)bn * 4) + 64;
    size_t work = 0;
    int res = 0;
    size_t used = fixed;
    // scratch first (hot), then W, then V
    if (used + sb <= smem_limit) { res |= 4; used += sb; } else work += sb / esize + 16;
    if (used + wb <= smem_limit) { res |= 1; used += wb; } else work += (size_t)bm * bn;
    if (need_v) {
        if (used + vb <= smem_limit) { res |= 2; used += vb; } else work += (size_t)bn * bn;
    }
    p.resident = res;
    p.smem = used;
    p.work_elems = work ? work + 64 : 0;
    p.threads = 256;
    p.kernel = KV_BLOCKED_GENERAL;
    return p;
}

template <class T>
int launch_blocked_general(SolveArgs<T> a, const Plan& p, cudaStream_t st) {
    a.resident = p.resident;
    a.kernel = KV_BLOCKED_GENERAL;
    auto kern = k_blocked_general<T>;
    if (p.smem > 48 * 1024) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem) != cudaSuccess)
            return BSVD_ERR_CUDA;
    }
    kern<<<a.batch, p.threads, p.smem, st>>>(a);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

// ---- kernel-level operators ---------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) k_gram_raw(const T* A, int64_t lda, int64_t sa, int m, int w, T* G,
                                                   int64_t ldg, int64_t sg) {
    const T* Ap = A + (size_t)blockIdx.x * sa;
    T* Gp = G + (size_t)blockIdx.x * sg;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
        const int ra = e % w, cb = e / w;
        if (ra > cb) continue;
        T acc = zero<T>();
        for (int r = 0; r < m; ++r) acc = cmac(acc, Ap[r + (size_t)ra * lda], Ap[r + (size_t)cb * lda]);
        if (ra == cb) {
            if constexpr (tr<T>::cplx) acc.im = 0;
            Gp[ra + (size_t)ra * ldg] = acc;
        } else {
            Gp[ra + (size_t)cb * ldg] = acc;
            Gp[cb + (size_t)ra * ldg] = conjT(acc);
        }
    }
}

template <class T>
__global__ void __launch_bounds__(256) k_fused_raw(T* B, int64_t ldb, int64_t sb, int m, int w, const T* J,
                                                    int64_t ldj, int64_t sj, int delta) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int RT = 32;
    T* Tl = reinterpret_cast<T*>(smem);
    T* Bp = B + (size_t)blockIdx.x * sb;
    const T* Jp = J + (size_t)blockIdx.x * sj;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int r0 = 0; r0 < m; r0 += RT) {
        const int rt = min(RT, m - r0);
        for (int e = tid; e < rt * w; e += nt) {
            const int rr = e % rt, x = e / rt;
            Tl[rr + x * RT] = Bp[r0 + rr + (size_t)x * ldb];
        }
        __syncthreads();
        for (int e = tid; e < rt * w; e += nt) {
            const int rr = e % rt, q = e / rt;
            T z = zero<T>();
            for (int k = 0; k < w; ++k) z = mac(z, Tl[rr + k * RT], Jp[k + (size_t)q * ldj]);
            Bp[r0 + rr + (size_t)q * ldb] = delta ? addT(Tl[rr + q * RT], z) : z;
        }
        __syncthreads();
    }
}

template <class T>
int launch_gram_raw(const T* A, int64_t lda, int64_t sa, int m, int wi, int wj, int batch, T* G, int64_t ldg,
                    int64_t sg, cudaStream_t st) {
    k_gram_raw<T><<<batch, 256, 0, st>>>(A, lda, sa, m, wi + wj, G, ldg, sg);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

template <class T>
int launch_fused_raw(T* B, int64_t ldb, int64_t sb, int m, int w, int batch, const T* J, int64_t ldj, int64_t sj,
                     int delta, cudaStream_t st) {
    const size_t smem = (size_t)32 * w * sizeof(T);
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(k_fused_raw<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return BSVD_ERR_CUDA;
    }
    k_fused_raw<T><<<batch, 256, smem, st>>>(B, ldb, sb, m, w, J, ldj, sj, delta);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

#define BSVD_INST_RAW(T)                                                                                    \
    template int launch_gram_raw<T>(const T*, int64_t, int64_t, int, int, int, int, T*, int64_t, int64_t,   \
                                    cudaStream_t);                                                          \
    template int launch_fused_raw<T>(T*, int64_t, int64_t, int, int, int, const T*, int64_t, int64_t, int,  \
                                     cudaStream_t);
BSVD_INST_RAW(float)
BSVD_INST_RAW(double)
BSVD_INST_RAW(cx<float>)
BSVD_INST_RAW(cx<double>)

template int launch_blocked_general<float>(SolveArgs<float>, const Plan&, cudaStream_t);
template int launch_blocked_general<double>(SolveArgs<double>, const Plan&, cudaStream_t);
template int launch_blocked_general<cx<float>>(SolveArgs<cx<float>>, const Plan&, cudaStream_t);
template int launch_blocked_general<cx<double>>(SolveArgs<cx<double>>, const Plan&, cudaStream_t);

}  // namespace bsvd
