// tma.cuh -- bulk asynchronous copies (the TMA engine's non-tensor mode, cp.async.bulk -> UBLKCP)
// and the mbarrier transaction-count protocol they complete on.
//
// Kernel (1) of the north star, the loader: a problem's column-major columns are contiguous runs of
// m elements (src/core.py:54-60 keeps every problem column-major), so each column is one bulk copy
// global -> shared, issued by one lane, with no address arithmetic per element and no registers
// held while the bytes are in flight; the copy engine signals an mbarrier when all bytes landed.
#pragma once

#include <cstdint>

namespace bsvd {
namespace tma {

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
// make the initialised barrier visible to the async proxy (the copy engine)
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// order this thread's earlier generic-proxy shared-memory accesses before later async-proxy ones
// (a bulk copy into a buffer that was just read with ordinary loads)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// one arrival that also announces `bytes` of incoming transactions for the current phase
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar))
        : "memory");
}
// spin until the phase with parity `phase` has completed
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TMA_WAIT_%=;\n}" ::"r"(saddr(bar)),
        "r"(phase)
        : "memory");
}

}  // namespace tma
}  // namespace bsvd
