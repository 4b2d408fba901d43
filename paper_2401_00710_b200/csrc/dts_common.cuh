// dts_common.cuh — shared host/device descriptors and warp primitives for the
// B200 DovetailSort hot path.  See DESIGN.md for the data layout.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dts {

constexpr unsigned FULL = 0xffffffffu;

// Plan flags (SegPlan::flags)
enum : uint32_t {
  PF_HEAVY = 1u,     // segment has heavy keys (sampler.py:177-189)
  PF_OVF = 2u,       // overflow bucket for keys >= ovf_thr (sampler.py:192-207)
  PF_SAMPLE = 4u,    // sample this segment on device before routing
  PF_ROOTSKIP = 8u,  // root: skip leading zero bits seen in the sample max
  PF_SPLIT = 16u,    // partition mode: route by (key, index) splitters
  PF_UNIQ = 32u,     // the segment's sample held no repeated key (set by the sampler)
};

// Bucket kinds written for the host planner (sampler.py:103-118 descriptors)
enum : uint8_t { KIND_LIGHT = 0, KIND_HEAVY = 1, KIND_OVF = 2, KIND_PAD = 3 };

// One distribution subproblem of an MSD level (the `_sort_rec` range
// [lo, hi) of dtsort.py:150-209 together with its BucketPlan,
// sampler.py:49-118).  Host-written; the sample kernel rewrites the routing
// fields of sampled segments.
struct SegPlan {
  uint64_t offset;    // first record (index into both buffers)
  uint64_t len;       // records
  uint64_t scanbase;  // sum of len of earlier segments of this level
  uint64_t ovf_thr;   // keys >= ovf_thr go to the overflow bucket (PF_OVF)
  uint64_t cnt_base;  // first count entry ([bucket][row] layout)
  uint32_t shift;     // low bit of the digit
  uint32_t gamma;     // digit width (zones = 2^gamma)
  uint32_t nb;        // buckets in use: 2^gamma + 2*nheavy (+1 overflow)
  uint32_t nbmax;     // column capacity reserved by the host
  uint32_t nheavy;    // heavy keys (ascending) at heavy_pool[heavy_base..]
  uint32_t heavy_base;
  uint32_t hz_base;   // zone table at hz_pool[hz_base .. +2^gamma]
  uint32_t flags;
  uint32_t sample_gs; // sampled segments: |S| = 2^sample_gs * stride
  uint32_t nrows;     // block rows of this segment
  uint32_t consumed;  // top bits known equal across the segment
  uint32_t bs_base;   // bucket-bounds / kinds base index (nbmax+1 entries)
};
static_assert(sizeof(SegPlan) == 88, "SegPlan layout");

// One count-matrix row: a contiguous chunk of one segment
// (counting.py:116-118 block bounds).
struct Blk {
  uint32_t seg, row;
  uint64_t begin, end;  // absolute record indices
};

// A base-case span: adjacent buckets sorted together by full key
// (dtsort.py:263-281 span batching, _base_sort :127-147).
struct Span {
  uint64_t offset;
  uint32_t len;
  // bit 0: records are in A (caller buffer, 0) or T (temporary, 1);
  // bits 8-15: the keys agree above this bit (SPAN_NOBOUND: unknown)
  uint32_t src;
};
constexpr uint32_t SPAN_NOBOUND = 255u;
constexpr uint32_t LOCAL_NB = 12u;  // the base case's one-pass counting takes spans differing in <= LOCAL_NB bits

// A finished range that must be copied T -> A (dtsort.py:111-124).
struct CopyR {
  uint64_t offset;
  uint32_t len;
  uint32_t pad;
};

// Per-launch shared-memory table capacities (host and device agree).
struct Caps {
  uint32_t nbc;  // bucket columns (>= max nb of any segment in the launch)
  uint32_t hzc;  // zone-table entries
  uint32_t hkc;  // heavy keys / splitters
  uint32_t pad;
};

template <int VB> struct ValOf { using T = uint32_t; };
template <> struct ValOf<8> { using T = uint64_t; };

__host__ __device__ inline uint32_t ceil_log2_u64(uint64_t x) {
  // smallest k with 2^k >= x (0 for x <= 1)
  if (x <= 1) return 0;
#ifdef __CUDA_ARCH__
  return 64 - __clzll((long long)(x - 1));
#else
  return 64 - __builtin_clzll(x - 1);
#endif
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes of the warp whose bucket equals this lane's (warp-level multisplit
// peer set).  `nbits` ballots, one per bucket-id bit; deterministic cost and
// no dependence on how many distinct ids the warp holds.
// ---------------------------------------------------------------------------
// Streaming loads / L2-sticky stores.  DTS_HINTS: 0 plain, 1 evict-first
// loads, 2 evict-first loads + evict-last stores (keeps partially written
// output lines in L2 until the next tile completes them).
// ---------------------------------------------------------------------------
#ifndef DTS_HINTS
#define DTS_HINTS 0
#endif
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
#if DTS_HINTS >= 1
  return __ldcs(p);
#else
  return *p;
#endif
}
// ---------------------------------------------------------------------------
// TMA 1-D bulk copies (cp.async.bulk) completed on an mbarrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Route one key to its bucket id: overflow > heavy (exact match) > light
// zone, with heavy keys splitting their zone's light bucket so every bucket
// id is monotone in the key (sampler.py:76-100 precedence; the id layout is
// the fused-dovetail layout of DESIGN.md §4).
//
// The SMEM zone table is packed: hzp[z] = base(z) | (heavy keys in zone z)
// << 16, base(z) = z + 2 * #heavy keys below zone z (hz_pool holds the
// plain prefix counts; `pack_zone_table` converts).  A key of a zone with at
// most one heavy key is routed without a branch (the zone's first heavy key
// is loaded unconditionally and compared); only zones holding several heavy
// keys search the rest.  (A divergent binary search on every zone that holds
// a heavy key made every warp instruction of a Zipf input take the slow
// path: 1.6 warp instructions per record in k_histogram, 5x C2's.)
template <typename K>
struct Router {
  K ovf_thr;
  uint32_t shift, mask, flags, nb;
  const uint32_t* hz;  // packed zone table
  const K* hk;

  __device__ __forceinline__ uint32_t operator()(K key) const {
    const uint32_t z = (uint32_t)(key >> shift) & mask;
    uint32_t b = z;
    if (flags & PF_HEAVY) {
      const uint32_t e = hz[z];
      const uint32_t c = e >> 16;
      b = e & 0xffffu;
      const uint32_t h0 = (b - z) >> 1;
      const K x = hk[c ? h0 : 0u];
      b += (c != 0u && x <= key) ? (x == key ? 1u : 2u) : 0u;
      if (c > 1u && x < key) {  // several heavy keys in the zone (rare)
        uint32_t lo = h0 + 1, hi = h0 + c;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (hk[mid] < key) lo = mid + 1; else hi = mid;
        }
        b = (e & 0xffffu) + 2u * (lo - h0) + ((lo < h0 + c && hk[lo] == key) ? 1u : 0u);
      }
    }
    return ((flags & PF_OVF) && key >= ovf_thr) ? nb - 1 : b;
  }
};

// SMEM packed zone table from the prefix counts (nz = 2^gamma zones).
__device__ __forceinline__ void pack_zone_table(const uint32_t* __restrict__ hzc, uint32_t nz,
                                                uint32_t* hzp) {
  for (uint32_t z = threadIdx.x; z < nz; z += blockDim.x) {
    const uint32_t h0 = hzc[z], h1 = hzc[z + 1];
    hzp[z] = (z + 2u * h0) | ((h1 - h0) << 16);
  }
}

// Partition router: destination = number of (key, index) splitters strictly
// below the record (SURVEY.md §8e composite splitters).
// Lanes of the warp holding the same small id b (< 2^nbits) as this lane,
// from nbits ballots (`valid` lanes only).
__device__ __forceinline__ uint32_t warp_peers(uint32_t b, bool valid, int nbits) {
  uint32_t m = __ballot_sync(FULL, valid);
  for (int i = 0; i < nbits; ++i) {
    const bool bit = (b >> i) & 1u;
    const uint32_t bb = __ballot_sync(FULL, bit);
    m &= bit ? bb : ~bb;
  }
  return m;
}

// Destination rank of a record: the number of (key, global index) splitters
// strictly below it.  With <= 15 splitters a 1024-entry prefix table (top 10
// key bits -> first splitter of the prefix | splitters in it << 4) answers
// most keys with one SMEM load; keys sharing a prefix with a splitter compare
// against those few.
constexpr int SPLIT_TB = 10;
template <typename K>
struct SplitRouter {
  const K* sk;
  const uint64_t* si;
  uint32_t ns;
  const uint8_t* tab;  // nullptr: binary search
  __device__ __forceinline__ uint32_t operator()(K key, uint64_t gidx) const {
    uint32_t lo, hi;
    if (tab) {
      const uint32_t e = tab[(uint32_t)(key >> (sizeof(K) * 8 - SPLIT_TB))];
      lo = e & 15u;
      const uint32_t c = e >> 4;
      if (c == 0) return lo;
      hi = lo + c;
    } else {
      lo = 0;
      hi = ns;
    }
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const bool less = sk[mid] < key || (sk[mid] == key && si[mid] < gidx);
      if (less) lo = mid + 1; else hi = mid;
    }
    return lo;
  }
};

// Block-wide exclusive scan of a[0..n) in shared memory (in place); returns
// the total.  All threads of the block must call it.  `tmp` holds NT/32
// entries.
template <int NT, typename T>
__device__ __forceinline__ uint32_t block_exscan(T* a, int n, uint32_t* tmp) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + NT - 1) / NT;
  const int s0 = min(n, tid * per), e0 = min(n, s0 + per);
  uint32_t sum = 0;
  for (int i = s0; i < e0; ++i) sum += (uint32_t)a[i];
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < NW ? tmp[lane] : 0u;
    uint32_t incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane < NW) tmp[lane] = incl - w;
    if (lane == NW - 1) tmp[NW] = incl;  // block total
  }
  __syncthreads();
  uint32_t run = tmp[warp] + x - sum;
  for (int i = s0; i < e0; ++i) {
    const uint32_t t = (uint32_t)a[i];
    a[i] = (T)run;
    run += t;
  }
  const uint32_t total = tmp[NW];
  __syncthreads();
  return total;
}

}  // namespace dts
