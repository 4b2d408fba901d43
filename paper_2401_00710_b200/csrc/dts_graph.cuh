// dts_graph.cuh — the steps either side of the graph-transpose sort (C5,
// SURVEY.md §8(d)/(f) row 4): a seeded R-MAT edge generator and the CSR
// row offsets of destination-sorted edges (the reference's transpose demo,
// bench.py:338-351: np.bincount(dst) + cumsum).  Both are HBM-bound
// elementwise passes; neither touches the sort itself.
#pragma once
#include "dts_common.cuh"

namespace dts {

// Counter-based draw for (seed, edge, level): splitmix64 of a golden-ratio
// combination, high 32 bits.  The numpy twin is gen.rmat_edges_host.
__host__ __device__ inline uint64_t rmat_mix(uint64_t seed, uint64_t edge, uint32_t level) {
  uint64_t x = seed * 0x9E3779B97F4A7C15ull + edge * 0xD1B54A32D192ED03ull + (uint64_t)level * 0x8CB92BA72F3D8DD7ull;
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Edge i (global index base + i) descends `scale` levels of the adjacency
// matrix; at level l, draw u (32 bits) and pick quadrant a (u < t0), b
// (< t1), c (< t2) or d: src bit = quadrant in {c, d}, dst bit = quadrant
// in {b, d}, most significant bit first.
__global__ void k_gen_rmat(uint32_t* __restrict__ dst, uint32_t* __restrict__ src, uint64_t n, uint64_t base,
                           uint64_t seed, uint32_t scale, uint32_t t0, uint32_t t1, uint32_t t2) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s = 0, d = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      const uint32_t u = (uint32_t)(rmat_mix(seed, base + i, l) >> 32);
      const uint32_t bit = 1u << (scale - 1 - l);
      if (u >= t0) {
        if (u < t1) {
          d |= bit;
        } else if (u < t2) {
          s |= bit;
        } else {
          s |= bit;
          d |= bit;
        }
      }
    }
    dst[i] = d;
    src[i] = s;
  }
}

// CSR offsets of ascending keys < nverts: row_ptr[v] = #keys < v for
// v in [0, nverts].  Each index i in [0, n] owns the vertices v in
// (key[i-1], key[i]] (key[-1] = -1, key[n] = nverts) and writes
// row_ptr[v] = i; gaps longer than LONG are queued and filled by a block
// each.  A key >= nverts or a descent sets *bad.
constexpr uint32_t CSR_LONG = 256;
template <typename K>
__global__ void k_csr_offsets(const K* __restrict__ keys, uint64_t n, uint64_t nverts, uint64_t* __restrict__ row_ptr,
                              uint64_t* __restrict__ gaps, uint32_t* __restrict__ ngaps, uint32_t gap_cap,
                              uint32_t* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t lo = i == 0 ? 0 : (uint64_t)keys[i - 1] + 1;  // first owned vertex
    const uint64_t hi = i == n ? nverts : (uint64_t)keys[i];     // last owned vertex
    if (i < n && ((uint64_t)keys[i] >= nverts || (i > 0 && keys[i] < keys[i - 1]))) {
      *bad = 1u;
      continue;
    }
    if (lo > hi) continue;
    if (hi - lo + 1 <= CSR_LONG) {
      for (uint64_t v = lo; v <= hi; ++v) row_ptr[v] = i;
    } else {
      const uint32_t g = atomicAdd(ngaps, 1u);
      if (g < gap_cap) {
        gaps[3 * g] = lo;
        gaps[3 * g + 1] = hi;
        gaps[3 * g + 2] = i;
      } else {
        *bad = 2u;  // gap list full (host retries with a larger list)
      }
    }
  }
}

__global__ void k_csr_fill_gaps(const uint64_t* __restrict__ gaps, const uint32_t* __restrict__ ngaps,
                                uint64_t* __restrict__ row_ptr) {
  const uint32_t g = blockIdx.x;
  if (g >= *ngaps) return;
  const uint64_t lo = gaps[3 * g], hi = gaps[3 * g + 1], i = gaps[3 * g + 2];
  for (uint64_t v = lo + threadIdx.x; v <= hi; v += blockDim.x) row_ptr[v] = i;
}

}  // namespace dts
