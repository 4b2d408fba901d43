// dts_rank.cuh — helpers of the in-tile stable order repair path (k_scatter,
// k_scatter_wc, k_local_sort).  The ranking itself lives in the kernels:
// per-warp SMEM atomic counters give stable in-tile ranks when a warp
// instruction's same-address atomics are served in lane order; every kernel
// verifies the resulting order and repairs it if it ever is not.
#pragma once
#include "dts_common.cuh"

namespace dts {

// Test hook: 1 forces the general in-step re-sort paths on every tile (the
// fast path relies on a verified-but-unpromised atomic order).
#ifndef DTS_FORCE_FIXUP
#define DTS_FORCE_FIXUP 0
#endif

// Insertion sort of w[0..c) ascending (stable tile order restored by the
// slot index held in the low bits).
__device__ __forceinline__ void small_isort(uint32_t* w, uint32_t c) {
  for (uint32_t i = 1; i < c; ++i) {
    const uint32_t x = w[i];
    uint32_t j = i;
    while (j > 0 && w[j - 1] > x) {
      w[j] = w[j - 1];
      --j;
    }
    w[j] = x;
  }
}

}  // namespace dts
