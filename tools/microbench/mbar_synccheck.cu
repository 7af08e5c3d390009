// Does compute-sanitizer synccheck model mbarrier.init + __syncthreads + try_wait.parity?
// (development aid for the reg32e report)  nvcc -gencode arch=compute_100a,code=sm_100a mbar_synccheck.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int* out) {
    __shared__ uint64_t bar;
    __shared__ int val;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(32) : "memory");
    __syncthreads();
    if (threadIdx.x < 32) {  // producer warp
        if (threadIdx.x == 0) val = 42;
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(sa(&bar)) : "memory");
    } else {  // consumer warp
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                     ::"r"(sa(&bar)), "r"(0) : "memory");
        if (threadIdx.x == 32) out[0] = val;
    }
}
int main() {
    int* d; cudaMalloc(&d, 4);
    k<<<1, 64>>>(d);
    int h = 0; cudaError_t e = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("val %d (%s)\n", h, cudaGetErrorString(e));
    return 0;
}
