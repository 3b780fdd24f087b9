// TMA (cp.async.bulk.tensor) staging of pixel-grid tiles for the persistent
// split-Bregman kernel.
//
// Every array a tile needs is row data of the image, [H][W][K] doubles
// (K = d for iterates, S for stencil weights / coefficients, S*d for the
// 8-neighbour b_old owner rows, 1 for diag / inv diag).  A tile's halo box
// (TW + 2R) x (TH + 2R) or interior box TW x TH is one TMA copy: one elected
// thread issues it, the hardware fills positions outside the image with
// zeros (exactly the zero fill of the cp.async path) and signals the
// buffer's mbarrier with the byte count.  This replaces the per-element
// address arithmetic of the cp.async staging loops, which the profiles show
// as ~30 % of the issued instructions of the tiled stencil phases.
//
// Requirements (checked on the host; otherwise the cp.async path runs):
// K * 8 and W * 8 multiples of 16 bytes (even d, even image width).
#pragma once

#include <cuda.h>

#include <cstdint>

namespace pfe_dev {

// Tensor maps of one persistent launch (encoded on the host per launch).
struct TileMaps {
  CUtensorMap y[2];      // Y buffers, halo box [HH][HW][D]
  CUtensorMap p[2];      // search directions, halo box
  CUtensorMap r_halo;    // residual, halo box
  CUtensorMap r_int;     // residual as the rhs of inner iterations >= 2, interior box [TH][TW][D]
  CUtensorMap rhs0_int;  // rhs of the first inner iteration, interior box
  CUtensorMap rq_int;    // (r/2) sqrt(D)(P - B), interior box
  CUtensorMap iv_halo;   // 1 / A_vv, halo box [HH][HW]
  CUtensorMap iv_int;    // 1 / A_vv, interior box [TH][TW]
  CUtensorMap dg_int;    // A_vv, interior box
  CUtensorMap cf_halo;   // off-diagonal coefficients [HH][HW][S]
  CUtensorMap wf_halo;   // edge weights [HH][HW][S]
  CUtensorMap bo[2];     // split_b ping-pong as owner rows [TH+R][HW][S*D] (8-neighbour grids)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
// Orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Box of rows of width K at image position (x, y) (may be negative / past the
// edge: zero filled) into dst.
template <int K>
__device__ __forceinline__ void tma_rows(double* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
  if constexpr (K == 1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(0), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
  }
}

// One contiguous global -> shared copy (16-byte aligned, size a multiple of
// 16) completing on an mbarrier.
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

}  // namespace pfe_dev
