// heevj.cu -- batched Hermitian eigensolver by cyclic Jacobi rotations:
// jacobi_hermitian_eig (src/eig.py:90-148) driving eig_sweeps in its
// non-delta form (src/_kernels_numba.py:17-82), one CTA per problem.
//
// Per problem: d = real(diag(G)); the working copy is exactly Hermitian from
// the upper triangle (src/eig.py:139-141) with a zero diagonal; M is the
// identity or the caller's starting matrix (rotations accumulated in place).
// A sweep runs the n-1 round-robin iterations (src/ordering.py:32-75); the
// floor(n/2) disjoint pairs of an iteration get their rotations in parallel
// (guard |g_ij| >= k u sqrt(|d_i| |d_j|), the reference formulas with c - 1
// carried separately), then every 2x2 block (p < q) of G takes rotation p on
// its rows and rotation q on its columns (the reference's order for p < q)
// with the conjugate mirror written exactly, the pivots are zeroed, d is
// updated (d_i += t|g|, d_j -= t|g|) and M's columns rotate.  A sweep without
// rotations ends the problem; it counts in sweeps_run, like the reference.
// G and M live in shared memory when they fit, else in the workspace (L2).
#include "kernel_args.cuh"
#include "launch.h"

namespace bsvd {
namespace heev {

template <class T>
BSVD_DEV double realpart(T x) {
    if constexpr (tr<T>::cplx) return (double)x.re;
    else return (double)x;
}

BSVD_DEV double addW(double a, double b) { return a + b; }
BSVD_DEV cx<double> addW(cx<double> a, cx<double> b) { return {a.re + b.re, a.im + b.im}; }
BSVD_DEV double subW(double a, double b) { return a - b; }
BSVD_DEV cx<double> subW(cx<double> a, cx<double> b) { return {a.re - b.re, a.im - b.im}; }
template <class W>
BSVD_DEV W fromD(double x) {
    if constexpr (sizeof(W) == sizeof(double)) return x;
    else return W{x, 0.0};
}

template <class T>
struct Rot {
    typename tr<T>::W ws, wsc;
    double cm1;
    int i, j;  // j < 0: unpaired (odd n)
    int rot;
};

template <class T>
// mode bits: 1 M starts from the caller's M (else I), 2 delta form (M accumulates P - I: the implicit
// identity columns' contribution, src/_kernels_numba.py:75-80), 4 d from the caller's D (else real diag G),
// 8 write G's rotated off-diagonal back (eig_sweeps mutates g in place)
__global__ void __launch_bounds__(256) k_heevj(int n, T* G, int64_t ldg, int64_t sG,
                                               typename tr<T>::R* D, int64_t sD, T* M, int64_t ldm, int64_t sM,
                                               int mode, double tol, int max_sweeps, bsvd_info* info, T* work,
                                               int in_smem) {
    using R = typename tr<T>::R;
    using Wt = typename tr<T>::W;
    extern __shared__ __align__(16) unsigned char smem[];
    const int prob = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int S = n + (n & 1), hw = S / 2, nit = S - 1;
    T* Gw;
    T* Mw;
    size_t off;
    if (in_smem) {
        Gw = reinterpret_cast<T*>(smem);
        Mw = Gw + (size_t)n * n;
        off = 2 * (size_t)n * n * sizeof(T);
    } else {
        Gw = work + (size_t)prob * 2 * n * n;
        Mw = Gw + (size_t)n * n;
        off = 0;
    }
    off = (off + 15) & ~size_t(15);
    R* d = reinterpret_cast<R*>(smem + off);
    off += ((size_t)n * sizeof(R) + 15) & ~size_t(15);
    Rot<T>* prm = reinterpret_cast<Rot<T>*>(smem + off);
    off += (size_t)hw * sizeof(Rot<T>);
    int* cnt = reinterpret_cast<int*>(smem + ((off + 15) & ~size_t(15)));
    T* Gp = G + (size_t)prob * sG;
    T* Mp = M + (size_t)prob * sM;
    const R* Dp_in = D + (size_t)prob * sD;
    const bool delta = (mode & 2) != 0;
    for (int e = tid; e < n * n; e += nt) {
        const int r = e % n, c = e / n;
        T x = zero<T>();
        if (r < c) x = Gp[r + (size_t)c * ldg];
        else if (r > c) x = conjT(Gp[c + (size_t)r * ldg]);
        else d[r] = (mode & 4) ? Dp_in[r] : (R)realpart(Gp[r + (size_t)r * ldg]);
        Gw[e] = x;
        Mw[e] = (mode & 1) ? Mp[r + (size_t)c * ldm] : ((r == c) ? one<T>() : zero<T>());
    }
    if (tid < 2) cnt[tid] = 0;
    __syncthreads();
    int sweeps = 0;
    long long rotations = 0;
    bool converged = n < 2;
    if (n < 2) sweeps = 1;
    while (!converged && sweeps < max_sweeps) {
        ++sweeps;
        for (int tw = 0; tw < nit; ++tw) {
            for (int p = tid; p < hw; p += nt) {
                int i, j;
                const bool v = rr_pair(tw, p, S, n, i, j);
                Rot<T> pr;
                pr.i = i;
                pr.j = v ? j : -1;
                pr.rot = 0;
                pr.cm1 = 0.0;
                pr.ws = Wt{};
                pr.wsc = Wt{};
                if (v) {
                    const T gij = Gw[i + (size_t)j * n];
                    const R absg = absT(gij);
                    const R sq = sqrt((R)(fabs(d[i]) * fabs(d[j])));
                    if (!(absg <= (R)0) && !((double)absg < tol * (double)sq)) {
                        const T wph = divR(gij, absg);
                        const RotParams q = rot_params((double)(d[i] - d[j]), 2.0 * (double)absg);
                        pr.rot = 1;
                        pr.cm1 = q.cm1;
                        pr.ws = scaleW(q.s, wide(wph));
                        pr.wsc = scaleW(q.s, wide(conjT(wph)));
                        const double td = q.t * (double)absg;
                        d[i] = (R)((double)d[i] + td);
                        d[j] = (R)((double)d[j] - td);
                        atomicAdd(&cnt[sweeps & 1], 1);
                    }
                }
                prm[p] = pr;
            }
            __syncthreads();
            // G <- J^H G J over 2x2 blocks (p < q); pivots zeroed
            for (int e = tid; e < hw * hw; e += nt) {
                const int p = e / hw, q = e % hw;
                const Rot<T> P = prm[p];
                if (p == q) {
                    if (P.rot) {
                        Gw[P.i + (size_t)P.j * n] = zero<T>();
                        Gw[P.j + (size_t)P.i * n] = zero<T>();
                    }
                    continue;
                }
                if (p > q) continue;
                const Rot<T> Q = prm[q];
                if (!P.rot && !Q.rot) continue;
                const int np = P.j >= 0 ? 2 : 1, nq = Q.j >= 0 ? 2 : 1;
                const int ip[2] = {P.i, P.j}, iq[2] = {Q.i, Q.j};
                Wt x[2][2];
                for (int u = 0; u < np; ++u)
                    for (int v2 = 0; v2 < nq; ++v2) x[u][v2] = wide(Gw[ip[u] + (size_t)iq[v2] * n]);
                if (P.rot)  // rows: g_iq + (cm1 g_iq + ws g_jq), g_jq + (cm1 g_jq - wsc g_iq)
                    for (int v2 = 0; v2 < nq; ++v2) rot_pair(x[0][v2], x[1][v2], P.cm1, P.wsc, P.ws);
                if (Q.rot)  // columns (the conjugate mirror of the rows update)
                    for (int u = 0; u < np; ++u) rot_pair(x[u][0], x[u][1], Q.cm1, Q.ws, Q.wsc);
                for (int u = 0; u < np; ++u)
                    for (int v2 = 0; v2 < nq; ++v2) {
                        store(&Gw[ip[u] + (size_t)iq[v2] * n], x[u][v2]);
                        store(&Gw[iq[v2] + (size_t)ip[u] * n], conjW(x[u][v2]));
                    }
            }
            // eigenvector columns: m_i + (cm1 m_i + wsc m_j), m_j + (cm1 m_j - ws m_i)
            for (int e = tid; e < n * hw; e += nt) {
                const int r = e % n, p = e / n;
                const Rot<T> P = prm[p];
                if (!P.rot) continue;
                Wt xi = wide(Mw[r + (size_t)P.i * n]), xj = wide(Mw[r + (size_t)P.j * n]);
                rot_pair(xi, xj, P.cm1, P.ws, P.wsc);
                if (delta) {  // + J - I: m_ii += cm1, m_ji += wsc, m_ij -= ws, m_jj += cm1
                    if (r == P.i) {
                        xi = addW(xi, fromD<Wt>(P.cm1));
                        xj = subW(xj, P.ws);
                    } else if (r == P.j) {
                        xi = addW(xi, P.wsc);
                        xj = addW(xj, fromD<Wt>(P.cm1));
                    }
                }
                store(&Mw[r + (size_t)P.i * n], xi);
                store(&Mw[r + (size_t)P.j * n], xj);
            }
            __syncthreads();
        }
        const int rot = cnt[sweeps & 1];  // sweep parity: the next sweep counts in the other slot
        if (tid == 0) cnt[(sweeps + 1) & 1] = 0;
        __syncthreads();
        rotations += rot;
        if (rot == 0) converged = true;
    }
    R* Dp = D + (size_t)prob * sD;
    for (int r = tid; r < n; r += nt) Dp[r] = d[r];
    for (int e = tid; e < n * n; e += nt) Mp[(e % n) + (size_t)(e / n) * ldm] = Mw[e];
    if (mode & 8)  // rotated off-diagonal back into g (its diagonal is never touched by eig_sweeps)
        for (int e = tid; e < n * n; e += nt)
            if ((e % n) != (e / n)) Gp[(e % n) + (size_t)(e / n) * ldg] = Gw[e];
    if (tid == 0 && info) {
        bsvd_info inf;
        inf.converged = converged ? 1 : 0;
        inf.outer_sweeps = sweeps;  // EigInfo.sweeps_run (the quiet sweep included)
        inf.rotations = rotations;
        inf.gram_calls = 0;
        inf.update_calls = 0;
        inf.last_rotations = 0;
        inf.path = 3;
        inf.status = 0;
        inf.kernel = KV_HEEVJ;
        info[prob] = inf;
    }
}

template <class T>
size_t smem_bytes(int n, bool in_smem) {
    const int hw = (n + (n & 1)) / 2;
    size_t off = in_smem ? 2 * (size_t)n * n * sizeof(T) : 0;
    off = (off + 15) & ~size_t(15);
    off += ((size_t)n * sizeof(typename tr<T>::R) + 15) & ~size_t(15);
    off += (size_t)hw * sizeof(Rot<T>);
    return ((off + 15) & ~size_t(15)) + 16;  // + the two sweep counters
}

template <class T>
int launch(int n, int batch, const void* G, int64_t ldg, int64_t sG, void* D, int64_t sD, void* M, int64_t ldm,
           int64_t sM, int mode, double k, int max_sweeps, bsvd_info* info, void* work, size_t work_bytes,
           size_t smem_limit, cudaStream_t st) {
    const bool in_smem = smem_bytes<T>(n, true) <= smem_limit;
    const size_t need = in_smem ? 0 : 2 * (size_t)n * n * sizeof(T) * (size_t)batch;
    if (need > work_bytes || (need && !work)) return BSVD_ERR_WORKSPACE;
    const size_t smem = smem_bytes<T>(n, in_smem);
    auto kern = k_heevj<T>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                                cudaSuccess)
        return BSVD_ERR_CUDA;
    // mode bit 16: k is already the absolute tolerance (eig_sweeps(tol)), else k * u
    const double tol = (mode & 16) ? k : k * tr<T>::u;
    kern<<<batch, 256, smem, st>>>(n, const_cast<T*>(static_cast<const T*>(G)), ldg, sG,
                                   static_cast<typename tr<T>::R*>(D), sD, static_cast<T*>(M), ldm, sM, mode & 15,
                                   tol, max_sweeps, info, static_cast<T*>(work), in_smem ? 1 : 0);
    return cudaPeekAtLastError() == cudaSuccess ? BSVD_OK : BSVD_ERR_CUDA;
}

}  // namespace heev

size_t heevj_workspace(int dtype, int n, int batch, size_t smem_limit) {
    const size_t es = dtype == BSVD_S ? 4 : (dtype == BSVD_Z ? 16 : 8);
    const bool fits = dtype == BSVD_S   ? heev::smem_bytes<float>(n, true) <= smem_limit
                      : dtype == BSVD_D ? heev::smem_bytes<double>(n, true) <= smem_limit
                      : dtype == BSVD_C ? heev::smem_bytes<cx<float>>(n, true) <= smem_limit
                                        : heev::smem_bytes<cx<double>>(n, true) <= smem_limit;
    return fits ? 0 : 2 * (size_t)n * n * es * (size_t)batch;
}

int launch_heevj(int dtype, int n, int batch, const void* G, int64_t ldg, int64_t sG, void* D, int64_t sD, void* M,
                 int64_t ldm, int64_t sM, int m_init, double k, int max_sweeps, bsvd_info* info, void* work,
                 size_t work_bytes, size_t smem_limit, cudaStream_t st) {
    switch (dtype) {
        case BSVD_S:
            return heev::launch<float>(n, batch, G, ldg, sG, D, sD, M, ldm, sM, m_init, k, max_sweeps, info, work,
                                       work_bytes, smem_limit, st);
        case BSVD_D:
            return heev::launch<double>(n, batch, G, ldg, sG, D, sD, M, ldm, sM, m_init, k, max_sweeps, info, work,
                                        work_bytes, smem_limit, st);
        case BSVD_C:
            return heev::launch<cx<float>>(n, batch, G, ldg, sG, D, sD, M, ldm, sM, m_init, k, max_sweeps, info,
                                           work, work_bytes, smem_limit, st);
        case BSVD_Z:
            return heev::launch<cx<double>>(n, batch, G, ldg, sG, D, sD, M, ldm, sM, m_init, k, max_sweeps, info,
                                            work, work_bytes, smem_limit, st);
    }
    return BSVD_ERR_ARG;
}

}  // namespace bsvd
