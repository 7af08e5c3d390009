// Does compute-sanitizer synccheck model reg32e's mbarrier protocol?  (development aid)
//   case 0: init / __syncthreads / one arrive / one try_wait.parity
//   case 3: case 1 after the warp that initialised the barriers has exited
//   case 2: case 1 with the ring in dynamic shared memory behind a large buffer (reg32e's layout)
//   case 1: a RING = 4 slot ring, producer warp (waits `empty` from the 5th slot on, arrives `full`)
//           and consumer warp (waits `full`, arrives `empty`), 64 hand-overs -- reg32e's W / V protocol
// nvcc -gencode arch=compute_100a,code=sm_100a mbar_synccheck.cu && compute-sanitizer --tool synccheck ./a.out
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                 ::"r"(sa(b)), "r"(par) : "memory");
}
constexpr int RING = 4;
struct Ring {
    double pad[1100];  // reg32e-like layout: barriers behind a large buffer
    int slot[RING];
    uint64_t full[RING], empty[RING];
};
__global__ void k(int mode, int* out) {
    extern __shared__ __align__(16) unsigned char raw[];  // case 2: dynamic shared memory, 4 rings
    __shared__ uint64_t sfull[RING], sempty[RING];
    __shared__ int sslot[RING];
    Ring& R = reinterpret_cast<Ring*>(raw)[mode == 2 ? 2 : 0];
    uint64_t* full = mode == 2 ? R.full : sfull;
    uint64_t* empty = mode == 2 ? R.empty : sempty;
    int* slot = mode == 2 ? R.slot : sslot;
    if (threadIdx.x < RING) {
        init(&full[threadIdx.x], 32);
        init(&empty[threadIdx.x], 32);
    }
    __syncthreads();
    const int n = mode == 0 ? 1 : 64;
    int t = threadIdx.x;
    if (mode == 3) {  // case 3: the initialising warp exits; warps 1 / 2 run the ring
        if (t < 32) return;
        t -= 32;
    }
    if (t >= 32) {  // producer
        for (uint32_t g = 0; g < (uint32_t)n; ++g) {
            const uint32_t s = g % RING;
            if (g >= RING) wait(&empty[s], ((g / RING) - 1) & 1);
            if (t == 32) slot[s] = (int)g;
            __syncwarp();
            arrive(&full[s]);
        }
    } else {  // consumer
        int sum = 0;
        for (uint32_t g = 0; g < (uint32_t)n; ++g) {
            const uint32_t s = g % RING;
            wait(&full[s], (g / RING) & 1);
            sum += slot[s];
            __syncwarp();
            arrive(&empty[s]);
        }
        if (t == 0) out[0] = sum;
    }
}
int main() {
    int* d;
    cudaMalloc(&d, 4);
    for (int mode = 0; mode < 4; ++mode) {
        k<<<1, mode == 3 ? 96 : 64, 4 * sizeof(Ring)>>>(mode, d);
        int h = 0;
        cudaError_t e = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
        printf("mode %d sum %d (%s)\n", mode, h, cudaGetErrorString(e));
    }
    return 0;
}
