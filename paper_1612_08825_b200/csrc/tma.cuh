// TMA (cp.async.bulk.tensor) + mbarrier helpers for sm_100a, and the host
// side tensor-map encoder (driver entry point fetched through cudart, so the
// library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ct {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// Optional suspend-time hint (CT_MBAR_SUSPEND_NS > 0): the hardware may park a
// waiting warp that long before try_wait returns false.  The moments kernels
// retry ~15 times per frame pair without it; removing those retries changed
// nothing measurable, so the plain form stays.
#ifndef CT_MBAR_SUSPEND_NS
#define CT_MBAR_SUSPEND_NS 0  // measured with 20000: no change (cfg2 fp64 1.814 vs 1.812 ms, 1080p fp32 0.956 vs 0.956 ms)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if CT_MBAR_SUSPEND_NS > 0
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"((uint32_t)CT_MBAR_SUSPEND_NS)
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

// Order this thread's prior generic-proxy shared-memory accesses before
// subsequent async-proxy (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
      : "memory");
}

// Rank-4 tiled map over [d3][d2][d1][d0] elements with a box0 x box1 x 1 x 1 box.
bool encode_tmap_4d(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                    uint32_t box0, uint32_t box1);

// Rank-3 tiled map over [d2][d1][d0] elements (d0 contiguous) with a box of
// box0 x box1 x 1; out-of-range reads are zero-filled.
bool encode_tmap_3d(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, uint64_t d2,
                    uint32_t box0, uint32_t box1);

// Encode a rank-2 tiled tensor map over a row-major [rows][cols] array of
// `esz`-byte elements with a box of box_cols x box_rows; out-of-range reads
// are zero-filled.  Returns false if the layout is not TMA-compatible
// (16-byte aligned base and row pitch) or the driver entry point is missing.
bool encode_tmap_2d(CUtensorMap* map, const void* base, int esz, uint64_t cols, uint64_t rows,
                    uint32_t box_cols, uint32_t box_rows);

}  // namespace ct
