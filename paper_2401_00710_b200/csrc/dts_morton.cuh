// dts_morton.cuh — Morton (z-order) keys, the paper's second application
// ("a z-value is calculated by
// interleaving the binary representations of each coordinate", then the
// z-values are sorted).  One HBM-bound elementwise pass: coordinates in,
// 64-bit z-values (and the point index as the payload) out; the sort is
// dts_sort.  Bit order: coordinate 0 takes the lowest bit of every group
// (z bit d*i + c = bit i of coordinate c).
#pragma once
#include "dts_common.cuh"

namespace dts {

// spread the low 32 bits of x to the even bit positions of a 64-bit word
__host__ __device__ inline uint64_t morton_spread2(uint64_t x) {
  x &= 0xFFFFFFFFull;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

// spread the low 21 bits of x to every third bit position (0, 3, ..., 60)
__host__ __device__ inline uint64_t morton_spread3(uint64_t x) {
  x &= 0x1FFFFFull;
  x = (x | (x << 32)) & 0x001F00000000FFFFull;
  x = (x | (x << 16)) & 0x001F0000FF0000FFull;
  x = (x | (x << 8)) & 0x100F00F00F00F00Full;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

// keys[i] = z-value of point i; vals (optional) = first_index + i.
// flags[0] |= 1 when a coordinate has bits at or above `bits`.
template <int D>
__global__ void k_morton(const uint32_t* __restrict__ x, const uint32_t* __restrict__ y,
                         const uint32_t* __restrict__ z, uint64_t n, uint32_t bits, uint64_t* __restrict__ keys,
                         uint64_t* __restrict__ vals, uint64_t first_index, uint32_t* __restrict__ flags) {
  const uint32_t lim = bits >= 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
  bool bad = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = x[i], b = y[i];
    uint64_t k;
    if constexpr (D == 2) {
      bad |= (a > lim) | (b > lim);
      k = morton_spread2(a) | (morton_spread2(b) << 1);
    } else {
      const uint32_t c = z[i];
      bad |= (a > lim) | (b > lim) | (c > lim);
      k = morton_spread3(a) | (morton_spread3(b) << 1) | (morton_spread3(c) << 2);
    }
    keys[i] = k;
    if (vals) vals[i] = first_index + i;
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

}  // namespace dts
