// tma.cuh -- TMA (cp.async.bulk.tensor) and mbarrier helpers shared by the
// column passes that stage their tiles through the tensor-memory accelerator
// (ntt_fast32.cu: the C3 2^16 column passes; gold_cols.cu: the Goldilocks
// column pass of C4).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.h"

namespace mm {

// One elected thread moves a whole tile with one 3-D box copy (coordinates
// beyond the tensor zero-filled) and arms an mbarrier with its byte count;
// every thread waits on the barrier's phase parity.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile("{\n\t.reg .pred P1;\n"
                 "LAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra DONE;\n\t"
                 "bra LAB_WAIT;\n"
                 "DONE:\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// issued by one thread: generic-proxy reads of dst must be ordered before the async write
__device__ __forceinline__ void tma_load_tile(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar,
                                              unsigned bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"((const void*)tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// arm the barrier for `bytes` of box copies issued after it (several boxes, one phase)
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// one 2-D box copy completing on a barrier armed by mbar_arrive_tx
__device__ __forceinline__ void tma_load_box2(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"((const void*)tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// one 3-D box copy completing on a barrier armed by mbar_arrive_tx
__device__ __forceinline__ void tma_load_box3(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"((const void*)tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)p;
    }();
    return fn;
}

}  // namespace mm
