// rqa_band.cuh -- TMA / mbarrier helpers of the band kernels.
//
// Column windows of the series are staged into shared memory with 1-D bulk
// copies (cp.async.bulk) completing on an mbarrier; the kernels double-buffer
// them so the copy for iteration x+1 overlaps iteration x.
#pragma once
#include "rqa_device.cuh"

namespace rqa {

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx_arrive(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
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

// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Stage s[i0+k_x+q] (q in [0, CW-1)) into a column buffer; returns the
// element offset introduced by aligning the source down to 16 bytes.
template <typename T>
__device__ __forceinline__ int col_window_src(const T* s, int64_t start, const T** src) {
  const uintptr_t a = (uintptr_t)(s + start);
  const int off = (int)((a & 15u) / sizeof(T));
  *src = s + start - off;
  return off;
}

}  // namespace rqa
