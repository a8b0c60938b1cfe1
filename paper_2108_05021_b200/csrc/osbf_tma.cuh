// TMA (cp.async.bulk.tensor) + mbarrier helpers for sm_100a, and host-side
// tensor-map encoding through the driver entry point (no -lcuda needed).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace osbf_gpu {
namespace tma {

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 3-D tiled load {c0 = x, c1 = y, c2 = plane}; out-of-bounds elements are zero.
__device__ __forceinline__ void load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                        uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// 4-D tiled load {c0 = x % V, c1 = x / V, c2 = y, c3 = plane} (see encode_4d).
__device__ __forceinline__ void load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                        int c3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
#endif

// Host: encode a 4-D tiled map that views every row of `width` elements as
// width / vec groups of `vec` elements: dims {vec, width/vec, height, planes},
// box {vec, box_groups, box_h, 1}.  A box then lands in shared memory as
// box_h dense rows of vec * box_groups elements, so one TMA load can stage a
// strip wider than the 256-element box limit of a plain 2-D/3-D map.  The
// strip's x start must be a multiple of vec.  Returns false when width % vec
// != 0 or the layout violates TMA constraints.
bool encode_rows_4d(CUtensorMap* map, CUtensorMapDataType dtype, size_t elem_bytes,
                    const void* base, uint64_t width, uint64_t height, uint64_t planes,
                    uint64_t pitch_bytes, uint64_t plane_bytes, uint32_t vec, uint32_t box_groups,
                    uint32_t box_h);

// Host: encode a 3-D tiled map over `planes` planes of `height` rows, row
// pitch `pitch_bytes`, plane stride `plane_bytes`; box {box_w, box_h, 1}.
// Returns false when the layout violates TMA constraints (caller falls back).
bool encode_3d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, uint64_t width,
               uint64_t height, uint64_t planes, uint64_t pitch_bytes, uint64_t plane_bytes,
               uint32_t box_w, uint32_t box_h);

}  // namespace tma
}  // namespace osbf_gpu
