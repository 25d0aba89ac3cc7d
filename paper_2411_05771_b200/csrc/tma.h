// tma.h — TMA bulk copies and mbarriers (sm_90+ async proxy) as inline PTX, shared by the
// forward projector and the backprojector.
#pragma once
#include <cstdint>

#include "internal.h"

namespace skei {

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    // cp.async.bulk: 16-byte aligned addresses, size a non-zero multiple of 16
    SKEI_DCHECK(((smem_u32(dst) | (unsigned)(uintptr_t)src | bytes) & 15u) == 0u && bytes != 0u,
                "bulk copy alignment");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// cp.async.bulk.tensor (4-D tiled box of a tensor map in param / const / global space) -> shared
__device__ __forceinline__ void tma_load_4d(void *dst, const void *tmap, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    SKEI_DCHECK((smem_u32(dst) & 127u) == 0u, "tensor copy alignment");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::
            "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
#ifdef SKEI_CHECKS
    // checked build: a phase that never completes (a lost or mis-sized copy, a missing
    // arrive) traps after ~4 s instead of hanging the GPU
    const long long t0 = clock64();
    for (;;) {
        unsigned ok;
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
        if (ok) return;
        SKEI_DCHECK(clock64() - t0 < 8000000000LL, "mbarrier wait timed out");
    }
#else
    // try_wait with a suspend-time hint: a waiting warp sleeps in hardware until the phase
    // completes (or the hint expires) instead of spinning on issue slots other warps need
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
#endif
}

}  // namespace skei
