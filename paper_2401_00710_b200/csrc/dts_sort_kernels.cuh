// dts_sort_kernels.cuh — k_histogram, the per-block bucket counts of a
// distribution pass (counting.py:123-137).  The scatters are in
// dts_scatter.cuh / dts_scatter_wc.cuh, the base case in dts_local.cuh.
#pragma once
#include "dts_kernels.cuh"

namespace dts {

// ---------------------------------------------------------------------------
// k_histogram: persistent CTAs pull blocks; per block, count records per
// bucket with shared-memory atomics (B200 SMEM atomics sustain >1.4 Tkeys/s
// chip-wide, well above the 4-byte-key HBM stream) and store the row into
// the [bucket][row] count matrix.
// ---------------------------------------------------------------------------
// KEEP: waves with heavy keys — the bucket ids of heavy segments' records are
// written to `bid` for the scatter (its own instantiation: the plain path's
// code, at the copy peak on C2, stays as it is)
template <typename K, int NT, bool SPLIT, bool KEEP = false>
__global__ void __launch_bounds__(NT) k_histogram(const SegPlan* __restrict__ plans,
                                                  const Blk* __restrict__ blks, uint32_t nblk,
                                                  uint32_t* __restrict__ ctr,
                                                  const K* __restrict__ keys,
                                                  uint32_t* __restrict__ counts,
                                                  const K* __restrict__ heavy_pool,
                                                  const uint32_t* __restrict__ hz_pool,
                                                  const uint64_t* __restrict__ split_idx,
                                                  uint64_t global_base, Caps caps,
                                                  uint16_t* __restrict__ bid = nullptr) {
  constexpr int VEC = 16 / sizeof(K);
  constexpr int U = 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const HistLayout L = hist_layout(sizeof(K), caps, SPLIT);
  K* hk = reinterpret_cast<K*>(smem_raw + L.hk);
  uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + L.si);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw + L.hist);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + L.hz);
  __shared__ uint32_t s_blk;
  const int tid = threadIdx.x;

  for (;;) {
    if (tid == 0) s_blk = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t bi = s_blk;
    if (bi >= nblk) break;
    const Blk B = blks[bi];
    const SegPlan P = plans[B.seg];
    for (uint32_t i = tid; i < P.nbmax; i += NT) hist[i] = 0;
    load_tables<K>(P, heavy_pool, hz_pool, split_idx, hk, si, hz);
    __syncthreads();
    const Router<K> R = make_router<K>(P, hz, hk);
    SplitRouter<K> SR;
    SR.sk = hk; SR.si = si; SR.ns = P.nheavy;
    SR.tab = (SPLIT && P.nheavy <= 15) ? reinterpret_cast<const uint8_t*>(hz) : nullptr;
    const K* p = keys + B.begin;
    const uint64_t n = B.end - B.begin;
    // (no warp aggregation needed: the increments compile to
    // ATOMS.POPC.INC, which combines a warp instruction's same-address lanes;
    // a per-thread register count of the sampler's hot bucket was measured
    // slower on Zipf 1.5 — the branch costs more than it saves)
    // segments with heavy keys: the bucket ids (zone word, then the zone's
    // heavy key: two dependent SMEM loads per record) are kept, 2 bytes per
    // record, for the scatter of the same wave — it ranks from them instead
    // of routing every record again
    const bool keep = KEEP && !SPLIT && bid != nullptr && (P.flags & PF_HEAVY);
    uint16_t* bq = keep ? bid + B.begin : nullptr;
    auto count_one = [&](K key, uint64_t e) -> uint32_t {
      const uint32_t b = SPLIT ? SR(key, global_base + B.begin + e) : R(key);
      atomicAdd(&hist[b], 1u);
      return b;
    };
    // partition (<= 8 destinations): 8-bit counters packed in one u64
    // register per thread (a thread counts < 256 keys of a block), reduced
    // over the warp at the end of the block
    const bool packed = SPLIT && P.nb <= 8;
    unsigned long long pc = 0ull;
    auto count_split = [&](K key, uint64_t e) {
      const uint32_t b = SR(key, global_base + B.begin + e);
      if (packed) pc += 1ull << (8 * b);
      else atomicAdd(&hist[b], 1u);
    };
    const uint64_t addr = reinterpret_cast<uint64_t>(p);
    uint64_t head = ((16 - (addr & 15)) & 15) / sizeof(K);
    if (head > n) head = n;
    const uint64_t nvec = (n - head) / VEC;
    const uint64_t tail0 = head + nvec * VEC;
    if ((uint64_t)tid < head) {
      if (SPLIT) {
        count_split(p[tid], tid);
      } else {
        const uint32_t b = count_one(p[tid], tid);
        if (KEEP && keep) bq[tid] = (uint16_t)b;
      }
    }
    if ((uint64_t)tid < n - tail0) {
      if (SPLIT) {
        count_split(p[tail0 + tid], tail0 + tid);
      } else {
        const uint32_t b = count_one(p[tail0 + tid], tail0 + tid);
        if (KEEP && keep) bq[tail0 + tid] = (uint16_t)b;
      }
    }
    // (the ids of a 16-byte key vector leave as one 8- or 4-byte store when
    // the id array is aligned like the keys)
    const bool bvec = keep && ((reinterpret_cast<uint64_t>(bq + head) & (2 * VEC - 1)) == 0);
    const uint4* pv = reinterpret_cast<const uint4*>(p + head);
    for (uint64_t vb = 0; vb < nvec; vb += (uint64_t)NT * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t vi = vb + (uint64_t)u * NT + tid;
        if (vi < nvec) v[u] = ld_stream(pv + vi);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t vi = vb + (uint64_t)u * NT + tid;
        if (SPLIT) {
          if (vi < nvec) {
            const K* kk = reinterpret_cast<const K*>(&v[u]);
#pragma unroll
            for (int e = 0; e < VEC; ++e) count_split(kk[e], head + vi * VEC + e);
          }
        } else if (vi < nvec) {
          const K* kk = reinterpret_cast<const K*>(&v[u]);
          uint32_t bb[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) bb[e] = count_one(kk[e], head + vi * VEC + e);
          if (KEEP && keep) {
            uint16_t* q = bq + head + vi * VEC;
            if (bvec) {
              if constexpr (VEC == 4)
                *reinterpret_cast<uint2*>(q) = make_uint2(bb[0] | (bb[1] << 16), bb[2] | (bb[3] << 16));
              else
                *reinterpret_cast<uint32_t*>(q) = bb[0] | (bb[1] << 16);
            } else {
#pragma unroll
              for (int e = 0; e < VEC; ++e) q[e] = (uint16_t)bb[e];
            }
          }
        }
      }
    }
    if (SPLIT && packed) {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        uint32_t c = (uint32_t)(pc >> (8 * b)) & 0xffu;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&hist[b], c);
      }
    }
    __syncthreads();
    uint32_t* row = counts + P.cnt_base + B.row;
    for (uint32_t b = tid; b < P.nbmax; b += NT) row[(uint64_t)b * P.nrows] = hist[b];
    __syncthreads();
  }
}

}  // namespace dts
