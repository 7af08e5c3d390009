// Stage latencies of the register kernel's W iteration for one warp per SMSP
// (development aid): builds unblocked_reg32b.cu with R32_PROBE_ON and reports
// clock cycles per iteration between the stage probes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -I include -I paper_2601_17979_b200/csrc tools/microbench/wchain.cu \
//        paper_2601_17979_b200/csrc/finalize.cu -o gpurun_out/wchain
#define R32_PROBE_ON
#include "unblocked_reg32b.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
    using namespace bsvd;
    const int B = 8;  // one CTA of 4 warps, two problems each
    std::vector<double> hA(B * 1024);
    srand(1);
    for (auto& v : hA) v = rand() / (double)RAND_MAX;
    double *A, *U, *S, *V, *W;
    bsvd_info* info;
    cudaMalloc(&A, hA.size() * 8);
    cudaMalloc(&U, hA.size() * 8);
    cudaMalloc(&S, B * 32 * 8);
    cudaMalloc(&V, hA.size() * 8);
    cudaMalloc(&W, (size_t)B * (2048 + r32b::LOG_ELEMS) * 8);
    cudaMalloc(&info, B * sizeof(bsvd_info));
    cudaMemcpy(A, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
    SolveArgs<double> a{};
    a.A = A; a.lda = 32; a.strideA = 1024; a.m = a.n = a.bm = a.bn = 32;
    a.U = U; a.ldu = 32; a.strideU = 1024; a.S = S; a.strideS = 32; a.V = V; a.ldv = 32; a.strideV = 1024;
    a.want_v = a.need_v = argc > 1 ? atoi(argv[1]) : 0;
    a.tol = 30 * 0x1p-53; a.max_sweeps = 30; a.batch = B; a.work = W; a.work_stride = 2048 + r32b::LOG_ELEMS;
    a.info = info;
    const size_t smem = 4 * sizeof(r32b::WarpSmem) + r32b::NIT * r32b::H * 4;
    auto k = r32b::k_reg32b<4, 2, 2, 2, 8, true>;  // the default (scaled rotations)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(r32b::g_r32_probe, z, sizeof(z));
        k<<<1, 128, smem>>>(a);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long p[16];
        cudaMemcpyFromSymbol(p, r32b::g_r32_probe, sizeof(p));
        const double n = (double)p[0];
        printf("want_v=%d iters %.0f | partials %.0f | sync+first LDS %.0f | reduce %.0f | params %.0f | "
               "publish %.0f | update %.0f  (cycles/iter)\n",
               a.want_v, n, p[4] / n, p[5] / n, p[1] / n, p[2] / n, p[6] / n, p[3] / n);
        if (a.want_v) printf("   V replay per iteration: wait+stage %.0f | update %.0f | tail+shift %.0f\n",
                             p[8] / n, p[9] / n, p[7] / n);
    }
    return 0;
}
