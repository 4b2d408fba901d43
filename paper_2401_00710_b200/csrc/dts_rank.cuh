// dts_rank.cuh — stable in-tile ranking primitives shared by k_scatter and
// k_local_sort.
//
// Fast path ("slot + fix-up"): every record takes a slot inside its bucket's
// range of the tile with one SMEM atomic; the (rare) buckets holding 2..FIXMAX
// records of the tile are then put back into input order by a per-bucket
// insertion sort on the record's tile index, and the few buckets holding
// more than FIXMAX records ("large": heavy keys) get exact stable slots from a
// packed block-wide prefix of per-thread counts.  Per record this is a
// couple of SMEM atomics and moves, several times cheaper than LSD radix-rank
// passes; tiles with more than NLARGE large buckets fall back to
// block_rank_packed passes.
#pragma once
#include "dts_common.cuh"

namespace dts {

// Test hook: 1 forces the general in-step re-sort paths on every tile (the
// fast path relies on a verified-but-unpromised atomic order).
#ifndef DTS_FORCE_FIXUP
#define DTS_FORCE_FIXUP 0
#endif

constexpr int FIXMAX = 64;  // small-bucket insertion-sort limit
constexpr int NLARGE = 8;   // large buckets per tile with exact packed-prefix slots

__device__ __forceinline__ uint32_t u4_get(const uint4& v, uint32_t j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ void u4_add(uint4& v, uint32_t j, uint32_t a) {
  if (j == 0) v.x += a;
  else if (j == 1) v.y += a;
  else if (j == 2) v.z += a;
  else v.w += a;
}

// Block-wide exclusive scan of a uint4 per thread (componentwise, u32
// wrap-free as long as totals fit).  tmp: (NT/32 + 1) uint4.
template <int NT>
__device__ __forceinline__ uint4 block_exscan_u4(uint4 v, uint4* tmp) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint4 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t a = __shfl_up_sync(FULL, x.x, o), b = __shfl_up_sync(FULL, x.y, o);
    const uint32_t c = __shfl_up_sync(FULL, x.z, o), d = __shfl_up_sync(FULL, x.w, o);
    if (lane >= o) {
      x.x += a; x.y += b; x.z += c; x.w += d;
    }
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint4 w = lane < NW ? tmp[lane] : make_uint4(0, 0, 0, 0);
    uint4 incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t a = __shfl_up_sync(FULL, incl.x, o), b = __shfl_up_sync(FULL, incl.y, o);
      const uint32_t c = __shfl_up_sync(FULL, incl.z, o), d = __shfl_up_sync(FULL, incl.w, o);
      if (lane >= o) {
        incl.x += a; incl.y += b; incl.z += c; incl.w += d;
      }
    }
    if (lane < NW) tmp[lane] = make_uint4(incl.x - w.x, incl.y - w.y, incl.z - w.z, incl.w - w.w);
  }
  __syncthreads();
  const uint4 base = tmp[warp];
  const uint4 r = make_uint4(base.x + x.x - v.x, base.y + x.y - v.y, base.z + x.z - v.z,
                             base.w + x.w - v.w);
  __syncthreads();
  return r;
}

// Exact stable slots for items of up to NLARGE large buckets.  `li[i]` is the
// item's large-bucket index (0xFF: not large).  Counts are packed 16-bit
// fields (2 large buckets per u32 word); returns each large item's offset
// within its bucket in rel[i].
template <int NT, int IPT>
__device__ __forceinline__ void large_ranks(const uint32_t (&li)[IPT], uint32_t (&rel)[IPT],
                                            uint4* tmp) {
  uint4 c = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if (li[i] != 0xFFu) {
      const uint32_t wj = li[i] >> 1, sh = (li[i] & 1u) << 4;
      rel[i] = (u4_get(c, wj) >> sh) & 0xffffu;
      u4_add(c, wj, 1u << sh);
    }
  }
  const uint4 pre = block_exscan_u4<NT>(c, tmp);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    if (li[i] != 0xFFu) {
      const uint32_t wj = li[i] >> 1, sh = (li[i] & 1u) << 4;
      rel[i] += (u4_get(pre, wj) >> sh) & 0xffffu;
    }
  }
}

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
