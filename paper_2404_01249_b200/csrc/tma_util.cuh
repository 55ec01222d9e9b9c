// tma_util.cuh — the sm_100a TMA / mbarrier primitives used by the
// plane-streaming stencil kernels (kernels_tma.cu), written as inline PTX.
//   cp.async.bulk.tensor.4d ... mbarrier::complete_tx   (SASS: UTMALDG)
//   mbarrier.init / arrive.expect_tx / try_wait.parity   (SASS: SYNCS.*)
#pragma once

#include <cuda.h>
#include <cstdint>

namespace dfm {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

#ifndef DFM_MBAR_SUSPEND_NS
#define DFM_MBAR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if DFM_MBAR_SUSPEND_NS > 0
    // suspend-time hint: a waiting warp sleeps until the phase completes (or
    // the hint expires) instead of re-polling
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(DFM_MBAR_SUSPEND_NS)
        : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// 4-D tiled TMA load (x, y, z, component) into shared memory, completion
// signalled on `bar` by transaction bytes; out-of-bounds elements are zero.
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
        "r"(c3)
        : "memory");
}

// per-thread asynchronous gathers (cp.async, SASS LDGSTS): the data lands in
// shared memory and is waited for with cp.async.wait_all where it is consumed,
// so a gather in flight across a loop iteration occupies no register
// scoreboard (ptxas drains shared scoreboards at loop heads)
template <int B>
__device__ __forceinline__ void cp_async(void* s, const void* g) {
    static_assert(B == 4 || B == 8 || B == 16, "cp.async size");
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(s)), "l"(g), "n"(B)
                 : "memory");
}
template <int B>
__device__ __forceinline__ void cp_async_u32(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(saddr), "l"(g), "n"(B)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace dfm
