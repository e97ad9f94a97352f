// tma.cuh -- the Blackwell tile-movement primitives the sweeps use: mbarriers in shared
// memory and cp.async.bulk.tensor (TMA) loads described by a CUtensorMap, plus the host
// side that encodes a tensor map of a padded state buffer (driver entry point resolved
// through the runtime, so libmfc.so does not link libcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mfc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

// make the initialised barriers visible to the async proxy (TMA complete_tx)
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// order this thread's earlier generic-proxy shared-memory accesses (as published by the
// barrier before it) before subsequent async-proxy (TMA) writes to the same memory
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// wait for the phase with the given parity to complete (HW-suspending try_wait loop)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// 4D tile load global -> shared, completion counted on bar (bytes of the whole box,
// out-of-range elements are zero-filled and counted too)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
}

// Host: a 4D tensor map (x, y, z, equation) of a padded state buffer with x pitch X,
// Y and Z padded planes and E equations, boxes of box_x cells along x (one row, all E
// equations).  Returns cudaSuccess or the error of the driver call.
cudaError_t encode_state_map(CUtensorMap* out, const double* base, int64_t X, int64_t Y,
                             int64_t Z, int E, int box_x);

}  // namespace mfc
