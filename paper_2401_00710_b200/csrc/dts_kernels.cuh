// dts_kernels.cuh — sm_100a kernels of the DovetailSort hot path.
//
//   k_sample_plan  : per-segment sample, sort, heavy detection, root skip
//                    (sampler.py:121-252, dtsort.py:212-241)
//   k_histogram    : per-block bucket counts (counting.py:123-137)
//   k_scan_*       : flat exclusive scan of the [bucket][row] count matrix
//                    = column-major offsets (counting.py:58-79)
//   k_bucket_bounds: bucket boundaries + kinds for the planner (counting.py:153)
//   k_scatter      : stable tile-ranked scatter (counting.py:141-151,
//                    _kernels.py:12-25)
//   k_local_sort   : SMEM stable LSD sort of base-case spans (dtsort.py:127-147)
//   k_copy_ranges  : T -> A copies of finished ranges (dtsort.py:111-124)
//   k_merge_*      : dovetail merge pieces (dtmerge.py:58-238)
#pragma once
#include <type_traits>
#include "dts_common.cuh"

namespace dts {

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// ---------------------------------------------------------------------------
// Shared-memory layouts (host and device compute the same offsets)
// ---------------------------------------------------------------------------
struct HistLayout {
  size_t hk, si, hist, hz, total;
};
__host__ __device__ inline HistLayout hist_layout(int kb, Caps c, bool split) {
  HistLayout L;
  size_t o = 0;
  L.hk = o; o = align16(o + (size_t)c.hkc * kb);
  L.si = o; o = align16(o + (split ? (size_t)c.hkc * 8 : 0));
  L.hist = o; o = align16(o + (size_t)c.nbc * 4);
  L.hz = o; o = align16(o + (size_t)(split ? (c.hzc > 256 ? c.hzc : 256) : c.hzc) * 4);  // split: prefix table
  L.total = o;
  return L;
}


// Load a segment's routing tables into shared memory.
template <typename K>
__device__ __forceinline__ void load_tables(const SegPlan& P, const K* __restrict__ heavy_pool,
                                            const uint32_t* __restrict__ hz_pool,
                                            const uint64_t* __restrict__ split_idx, K* hk,
                                            uint64_t* si, uint32_t* hz) {
  if (P.flags & PF_SPLIT) {
    for (uint32_t i = threadIdx.x; i < P.nheavy; i += blockDim.x) {
      hk[i] = heavy_pool[P.heavy_base + i];
      si[i] = split_idx[P.heavy_base + i];
    }
    if (P.nheavy <= 15) {  // prefix table (SplitRouter), in the hz area
      __syncthreads();       // (block-uniform call) splitter keys are in hk
      uint8_t* tab = reinterpret_cast<uint8_t*>(hz);
      constexpr int W = sizeof(K) * 8;
      for (uint32_t pfx = threadIdx.x; pfx < (1u << SPLIT_TB); pfx += blockDim.x) {
        uint32_t below = 0, in = 0;
        for (uint32_t j = 0; j < P.nheavy; ++j) {
          const uint32_t sp = (uint32_t)(hk[j] >> (W - SPLIT_TB));
          below += sp < pfx;
          in += sp == pfx;
        }
        tab[pfx] = (uint8_t)(below | (in << 4));
      }
    }
  } else if (P.flags & PF_HEAVY) {
    pack_zone_table(hz_pool + P.hz_base, 1u << P.gamma, hz);
    for (uint32_t i = threadIdx.x; i < P.nheavy; i += blockDim.x)
      hk[i] = heavy_pool[P.heavy_base + i];
  }
}

template <typename K>
__device__ __forceinline__ Router<K> make_router(const SegPlan& P, const uint32_t* hz,
                                                 const K* hk) {
  Router<K> R;
  R.ovf_thr = (K)P.ovf_thr;
  R.shift = P.shift;
  R.mask = (P.gamma >= 32) ? 0xffffffffu : ((1u << P.gamma) - 1u);
  R.flags = P.flags;
  R.nb = P.nb;
  R.hz = hz;
  R.hk = hk;
  return R;
}

// ---------------------------------------------------------------------------
// k_sample_plan: one CTA per sampled segment.  Draws |S| keys uniformly with
// replacement (counter-based hash instead of numpy Philox — only the heavy
// set can differ, never the output), sorts them in SMEM (bitonic), applies
// the root leading-bit skip and the strided-repeat heavy rule, and writes the
// zone table.  sampler.py:121-252, dtsort.py:212-241.
// ---------------------------------------------------------------------------
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_sample_plan(SegPlan* __restrict__ plans,
                                                    const uint32_t* __restrict__ seg_ids,
                                                    const K* __restrict__ keys,
                                                    K* __restrict__ heavy_pool,
                                                    uint32_t* __restrict__ hz_pool, uint64_t seed,
                                                    uint32_t level, uint32_t stride,
                                                    uint32_t gs_max, uint32_t smax, uint32_t wc_cols) {
  constexpr int W = sizeof(K) * 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sm = reinterpret_cast<K*>(smem_raw);
  __shared__ uint32_t s_tmp[NT / 32 + 1];
  __shared__ uint32_t s_m;

  const uint32_t s = seg_ids[blockIdx.x];
  SegPlan P = plans[s];
  const uint32_t gs = min(P.sample_gs, gs_max);
  uint64_t S = (uint64_t(1) << gs) * stride;
  if (S > P.len) S = P.len;
  if (S > smax) S = smax;
  uint32_t P2 = 1;
  while (P2 < S) P2 <<= 1;
  const uint64_t stream = splitmix64(seed ^ splitmix64((uint64_t(level) << 56) ^ P.offset));
  for (uint32_t i = threadIdx.x; i < P2; i += NT) {
    if (i < S) {
      const uint64_t r = splitmix64(stream + i);
      const uint64_t idx = __umul64hi(r, P.len);
      sm[i] = keys[P.offset + idx];
    } else {
      sm[i] = (K)~(K)0;
    }
  }
  __syncthreads();
  // bitonic sort of sm[0..P2).  Stages with compare distance j <= 128 stay
  // inside aligned 256-element blocks: warp w owns blocks w, w + NW, ... (its
  // lanes take the block's 128 pairs), so those stages need only __syncwarp;
  // a block barrier is needed only around the j >= 256 stages (8192 keys:
  // 20 block barriers instead of 91).
  {
    constexpr uint32_t NWS = NT / 32;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nblk = (P2 + 255) / 256;
    auto cswap = [&](uint32_t a, uint32_t j, uint32_t k) {
      const uint32_t b = a + j;
      const bool up = (a & k) == 0;
      const K x = sm[a], y = sm[b];
      if ((x > y) == up) {
        sm[a] = y;
        sm[b] = x;
      }
    };
    for (uint32_t k = 2; k <= P2; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        if (j >= 256) {
          for (uint32_t i = threadIdx.x; i < P2 / 2; i += NT) cswap(2 * i - (i & (j - 1)), j, k);
          __syncthreads();
        } else {
          const uint32_t np = P2 < 256 ? P2 / 2 : 128u;  // pairs per block
          for (uint32_t bl = warp; bl < nblk; bl += NWS)
            for (uint32_t r = lane; r < np; r += 32) cswap(256 * bl + 2 * r - (r & (j - 1)), j, k);
          __syncwarp();
        }
      }
      if (k >= 256) __syncthreads();  // (the next k starts with a block-wide stage)
    }
    __syncthreads();
  }
  uint32_t gamma = P.gamma, shift = P.shift;
  uint32_t flags = P.flags & ~(PF_HEAVY | PF_OVF | PF_UNIQ);
  uint64_t thr = 0;
  if (flags & PF_ROOTSKIP) {
    // plan_overflow (sampler.py:192-207) at bit granularity: skip the
    // sample max's leading zeros, keep >= 1 bit, keys above go to overflow.
    const K mx = sm[S - 1];
    int bl = 0;
    if (sizeof(K) == 8) bl = mx ? 64 - __clzll((long long)mx) : 0;
    else bl = mx ? 32 - __clz((int)(uint32_t)mx) : 0;
    int skip = W - bl;
    if (skip > W - 1) skip = W - 1;
    if (skip > 0) {
      flags |= PF_OVF;
      thr = uint64_t(1) << (W - skip);
      const uint32_t rem = (uint32_t)(W - skip);
      if (gamma > rem) gamma = rem;
      shift = rem - gamma;
    }
  }
  // no key repeats anywhere in the sorted sample (birthday test): the
  // children of this segment skip their own samples (dts_api.cu)
  {
    if (threadIdx.x == 0) s_m = 0;
    __syncthreads();
    bool dup = false;
    for (uint32_t i = threadIdx.x; i + 1 < S; i += NT) dup |= sm[i] == sm[i + 1];
    if (__any_sync(FULL, dup) && (threadIdx.x & 31) == 0) s_m = 1;
    __syncthreads();
    if (s_m == 0) flags |= PF_UNIQ;
    __syncthreads();
  }
  // detect_heavy (sampler.py:177-189): keys repeating in S[::stride].
  const uint32_t nsub = (uint32_t)((S + stride - 1) / stride);
  // compaction in chunks of NT subsample points
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  K* hk_out = heavy_pool + P.heavy_base;
  for (uint32_t base = 0; base < nsub; base += NT) {
    const uint32_t j = base + threadIdx.x;
    bool f = false;
    K v = 0;
    if (j + 1 < nsub) {
      v = sm[(uint64_t)j * stride];
      f = (v == sm[(uint64_t)(j + 1) * stride]) && (j == 0 || sm[(uint64_t)(j - 1) * stride] != v);
    }
    const uint32_t bal = __ballot_sync(FULL, f);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_tmp[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = s_m;
      for (int w = 0; w < NT / 32; ++w) {
        const uint32_t t = s_tmp[w];
        s_tmp[w] = acc;
        acc += t;
      }
      s_m = acc;
    }
    __syncthreads();
    if (f) hk_out[s_tmp[warp] + __popc(bal & lanemask_lt())] = v;
    __syncthreads();
  }
  // The host reserved nbmax = 2^gamma + 2^gs + 1 columns: keep 2m within
  // it.  When more keys qualify than the write-combining scatter's columns
  // hold (wc_cols: 2^gamma light zones, 2 per heavy key, the overflow
  // bucket) and the keys beyond that count hold <= 1/20 of the subsample,
  // only the heaviest keys that fit stay — the segment then takes the
  // faster write-combining scatter, and the few records of the dropped keys
  // stay in their light buckets (any heavy set gives the same stable
  // output).  Kept keys are the ones with the most subsample hits, in key
  // order.  (Zipf 1.0: 8 qualify at the root, the 5 lightest hold ~3.6 %:
  // WC; Zipf 1.5 / 1.2: the keys beyond 3 hold 11-15 %: all kept.)
  // (wc_cols = the write-combining scatter's columns | its wide variant's
  // columns << 16: the wide variant is the second choice)
  const uint32_t m_all = (P.nbmax - (1u << gamma) - 1u) / 2u;
  const uint32_t ovf1 = (flags & PF_OVF) ? 1u : 0u;
  const uint32_t wc1 = wc_cols & 0xffffu, wc2 = wc_cols >> 16;
  const uint32_t m_wc = wc1 > (1u << gamma) + ovf1 ? (wc1 - (1u << gamma) - ovf1) / 2u : 0u;
  const uint32_t m_wc2 = wc2 > (1u << gamma) + ovf1 ? (wc2 - (1u << gamma) - ovf1) / 2u : 0u;
  __syncthreads();
  uint32_t m = min(s_m, m_all);
  if (s_m > m_wc) {
    constexpr uint32_t HC = 512;  // candidates <= nsub / 2 <= 2^gs_max / 2
    __shared__ uint32_t s_hc[HC];
    __shared__ K s_keep[HC];
    const uint32_t nc = min(s_m, HC);
    for (uint32_t c = threadIdx.x; c < nc; c += NT) {
      const K v = hk_out[c];
      uint32_t lo = 0, hi = nsub;  // first subsample point >= v
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sm[(uint64_t)mid * stride] < v) lo = mid + 1; else hi = mid;
      }
      uint32_t lo2 = lo, hi2 = nsub;  // first subsample point > v
      while (lo2 < hi2) {
        const uint32_t mid = (lo2 + hi2) >> 1;
        if (sm[(uint64_t)mid * stride] <= v) lo2 = mid + 1; else hi2 = mid;
      }
      s_hc[c] = lo2 - lo;
    }
    __shared__ uint32_t s_drop, s_drop2;
    if (threadIdx.x == 0) {
      s_m = 0;
      s_drop = 0;
      s_drop2 = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // rank by (hits desc, key asc); hits of the keys ranked >= m_wc
    uint32_t rk = 0xFFFFFFFFu;
    if (threadIdx.x < nc) {
      const uint32_t c = threadIdx.x, mc = s_hc[c];
      rk = 0;
      for (uint32_t c2 = 0; c2 < nc; ++c2) {
        const uint32_t x = s_hc[c2];
        rk += (x > mc) || (x == mc && c2 < c);
      }
      if (rk >= m_wc) atomicAdd(&s_drop, mc);
      if (rk >= m_wc2) atomicAdd(&s_drop2, mc);
    }
    __syncthreads();
    const uint32_t keep_n = 20u * s_drop <= nsub ? m_wc : (20u * s_drop2 <= nsub ? max(m_wc, m_wc2) : m_all);
    for (uint32_t base = 0; base < nc; base += NT) {
      const uint32_t c = base + threadIdx.x;
      bool keep = false;
      K v = 0;
      if (c < nc) {
        keep = rk < keep_n;
        v = hk_out[c];
      }
      const uint32_t bal = __ballot_sync(FULL, keep);
      if (lane == 0) s_tmp[warp] = __popc(bal);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t acc = s_m;
        for (int w = 0; w < NT / 32; ++w) {
          const uint32_t t = s_tmp[w];
          s_tmp[w] = acc;
          acc += t;
        }
        s_m = acc;
      }
      __syncthreads();
      if (keep) s_keep[s_tmp[warp] + __popc(bal & lanemask_lt())] = v;
      __syncthreads();
    }
    m = min(s_m, m_all);
    for (uint32_t i = threadIdx.x; i < m; i += NT) hk_out[i] = s_keep[i];
    __syncthreads();
  }
  // copy heavy keys back into SMEM (sm is free now) for the zone table
  for (uint32_t i = threadIdx.x; i < m; i += NT) sm[i] = hk_out[i];
  __syncthreads();
  if (m > 0) {
    flags |= PF_HEAVY;
    const uint32_t nz = 1u << gamma;
    const uint32_t mask = nz - 1u;
    for (uint32_t z = threadIdx.x; z <= nz; z += NT) {
      // hz[z] = #heavy keys whose zone < z (zones are non-decreasing)
      uint32_t lo = 0, hi = m;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t hzm = (uint32_t)(sm[mid] >> shift) & mask;
        if (hzm < z) lo = mid + 1; else hi = mid;
      }
      hz_pool[P.hz_base + z] = lo;
    }
  }
  if (threadIdx.x == 0) {
    P.gamma = gamma;
    P.shift = shift;
    P.flags = flags;
    P.ovf_thr = thr;
    P.nheavy = m;
    P.nb = (1u << gamma) + 2u * m + ((flags & PF_OVF) ? 1u : 0u);
    plans[s] = P;
  }
}

// ---------------------------------------------------------------------------
// Flat exclusive scan u32 -> u64 (reduce / spine / downsweep).
// ---------------------------------------------------------------------------
constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_CHUNK = SCAN_NT * SCAN_IPT;

__global__ void __launch_bounds__(SCAN_NT) k_scan_reduce(const uint32_t* __restrict__ in,
                                                         uint64_t n,
                                                         uint64_t* __restrict__ partial) {
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_CHUNK;
  uint64_t s = 0;
  for (int i = 0; i < SCAN_IPT; ++i) {
    const uint64_t idx = base + (uint64_t)i * SCAN_NT + threadIdx.x;
    if (idx < n) s += in[idx];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  __shared__ uint64_t ws[SCAN_NT / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < SCAN_NT / 32; ++w) t += ws[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_spine(uint64_t* __restrict__ partial,
                                                     uint32_t nchunks) {
  __shared__ uint64_t ws[33];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t base = 0; base < nchunks; base += 1024) {
    const uint32_t i = base + threadIdx.x;
    const uint64_t v = i < nchunks ? partial[i] : 0;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      const uint64_t w = ws[lane];
      uint64_t incl = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      ws[lane] = incl - w;
      if (lane == 31) ws[32] = incl;
    }
    __syncthreads();
    if (i < nchunks) partial[i] = carry + ws[warp] + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += ws[32];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SCAN_NT) k_scan_down(const uint32_t* __restrict__ in, uint64_t n,
                                                       const uint64_t* __restrict__ partial,
                                                       uint64_t* __restrict__ out) {
  // thread t owns entries [base + t*IPT, base + (t+1)*IPT) (blocked layout,
  // staged through SMEM for coalescing)
  __shared__ uint32_t sv[SCAN_CHUNK];
  __shared__ uint64_t ws[SCAN_NT / 32 + 1];
  const uint64_t base = (uint64_t)blockIdx.x * SCAN_CHUNK;
  for (int i = 0; i < SCAN_IPT; ++i) {
    const uint64_t idx = base + (uint64_t)i * SCAN_NT + threadIdx.x;
    sv[i * SCAN_NT + threadIdx.x] = idx < n ? in[idx] : 0u;
  }
  __syncthreads();
  uint64_t local[SCAN_IPT];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    local[i] = s;
    s += sv[threadIdx.x * SCAN_IPT + i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int w = 0; w < SCAN_NT / 32; ++w) {
      const uint64_t t = ws[w];
      ws[w] = acc;
      acc += t;
    }
  }
  __syncthreads();
  const uint64_t off = partial[blockIdx.x] + ws[warp] + x - s;
  __syncthreads();
  // write back through SMEM as u64 pairs would need 2x space; write directly
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    const uint64_t idx = base + (uint64_t)threadIdx.x * SCAN_IPT + i;
    if (idx < n) out[idx] = off + local[i];
  }
}

// ---------------------------------------------------------------------------
// k_bucket_bounds: per segment, bucket starts (relative to the segment) and
// bucket kinds for the host planner.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bucket_bounds(const SegPlan* __restrict__ plans,
                                                       const uint64_t* __restrict__ scan,
                                                       const uint32_t* __restrict__ hz_pool,
                                                       uint64_t* __restrict__ bstart,
                                                       uint8_t* __restrict__ kinds,
                                                       uint16_t* __restrict__ zones) {
  const SegPlan P = plans[blockIdx.x];
  for (uint32_t b = threadIdx.x; b <= P.nbmax; b += blockDim.x) {
    uint64_t v = P.len;
    uint8_t kind = KIND_PAD;
    uint32_t zone = b;  // the bucket's digit value (k_classify: key bound of merged spans)
    if (b < P.nb) {
      v = scan[P.cnt_base + (uint64_t)b * P.nrows] - P.scanbase;
      if ((P.flags & PF_OVF) && b == P.nb - 1) {
        kind = KIND_OVF;
      } else if (P.flags & PF_HEAVY) {
        // zone z with base(z) = z + 2*hz[z] <= b (largest such z)
        const uint32_t* hz = hz_pool + P.hz_base;
        uint32_t lo = 0, hi = 1u << P.gamma;  // find last z with base(z) <= b
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (mid + 2u * hz[mid] <= b) lo = mid; else hi = mid;
        }
        const uint32_t off = b - (lo + 2u * hz[lo]);
        kind = (off & 1u) ? KIND_HEAVY : KIND_LIGHT;
        zone = lo;
      } else {
        kind = KIND_LIGHT;
      }
    }
    bstart[P.bs_base + b] = v;
    kinds[P.bs_base + b] = kind;
    if (zones) zones[P.bs_base + b] = (uint16_t)zone;
  }
}

// ---------------------------------------------------------------------------
// k_copy_ranges: finished ranges T -> A (heavy runs, exhausted-digit runs);
// persistent CTAs over a device-resident list (count in *ncopy).
// ---------------------------------------------------------------------------
template <typename K, int VB>
__global__ void __launch_bounds__(256) k_copy_ranges(const CopyR* __restrict__ rs,
                                                     const uint32_t* __restrict__ ncopy,
                                                     K* __restrict__ Ak,
                                                     typename ValOf<VB>::T* __restrict__ Av,
                                                     const K* __restrict__ Tk,
                                                     const typename ValOf<VB>::T* __restrict__ Tv) {
  const uint32_t nc = *ncopy;
  // one column: 16-byte vectors for the aligned body, elements at the ends
  auto col = [&](auto* dst, const auto* src, uint64_t off, uint32_t len) {
    using E = typename std::remove_const<typename std::remove_pointer<decltype(src)>::type>::type;
    constexpr uint32_t VEC = 16 / sizeof(E);
    // (the caller's column may start anywhere: vectors only when both ends
    // share their 16-byte phase, head taken from the destination address)
    const uintptr_t da = reinterpret_cast<uintptr_t>(dst + off), sa = reinterpret_cast<uintptr_t>(src + off);
    const bool vec_ok = ((da ^ sa) & 15u) == 0;
    const uint32_t h0 = (uint32_t)(((16u - (da & 15u)) & 15u) / sizeof(E));
    const uint32_t head = !vec_ok ? len : (h0 < len ? h0 : len);
    const uint32_t nv = (len - head) / VEC;
    for (uint32_t i = threadIdx.x; i < head; i += blockDim.x) dst[off + i] = src[off + i];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + off + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + off + head);
    constexpr uint32_t U = 4;  // 4 vectors in flight per thread
    uint32_t i = threadIdx.x;
    for (; i + (U - 1) * blockDim.x < nv; i += U * blockDim.x) {
      uint4 t[U];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) t[u] = ld_stream(s4 + i + u * blockDim.x);
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) d4[i + u * blockDim.x] = t[u];
    }
    for (; i < nv; i += blockDim.x) d4[i] = ld_stream(s4 + i);
    for (uint32_t i = head + nv * VEC + threadIdx.x; i < len; i += blockDim.x) dst[off + i] = src[off + i];
  };
  for (uint32_t c = blockIdx.x; c < nc; c += gridDim.x) {
    const CopyR r = rs[c];
    col(Ak, Tk, r.offset, r.len);
    if (VB) col(Av, Tv, r.offset, r.len);
  }
}

// ---------------------------------------------------------------------------
// k_classify: the reference's per-child decisions (dtsort.py:244-318
// _children_step) on the device, one thread per segment over its buckets:
//   * exhausted buckets (heavy keys, or no digit bits left) are finished —
//     if they sit in T they are copied (or, when small, sorted-as-copied by a
//     base-case span);
//   * light buckets <= thr join the current base-case span (adjacent
//     buckets of one source are batched up to thr records, dtsort.py:262-286);
//   * larger light buckets become next-level segments.
// Spans / copies / next segments are appended with one atomic per segment;
// the level's counters go to ctr[4..8) (InstrumentReport fields).
// ---------------------------------------------------------------------------
struct NextSeg {
  uint64_t offset, len;
  uint32_t consumed, pad;  // pad: bit 0 root (host only), bit 1 parent had heavy keys, bit 2 parent sample unique
};

constexpr int CLS_NT = 256;
constexpr int CLS_MAXB = 1032;  // buckets per segment handled in SMEM (nbmax + 1)

__global__ void __launch_bounds__(CLS_NT) k_classify(const SegPlan* __restrict__ plans,
                                                     const uint64_t* __restrict__ bs,
                                                     const uint8_t* __restrict__ kinds, uint32_t W,
                                                     uint32_t out_src, uint64_t thr, uint32_t copy_chunk,
                                                     Span* __restrict__ spans, CopyR* __restrict__ copies,
                                                     NextSeg* __restrict__ next,
                                                     unsigned long long* __restrict__ ctr,
                                                     const uint16_t* __restrict__ zones, uint32_t rules) {
  enum : uint32_t { T_EMPTY = 0, T_CAND = 1, T_FLUSH = 2, T_COPY = 3, T_NEXT = 4 };
  __shared__ uint64_t s_bs[CLS_MAXB];
  __shared__ uint32_t s_ty[CLS_MAXB];
  __shared__ Span s_sp[CLS_MAXB];
  __shared__ uint32_t s_n[4];  // spans, copies, next, base slots
  __shared__ unsigned long long s_acc[4];
  __shared__ uint32_t s_base[3];
  __shared__ uint32_t s_slow;
  const SegPlan P = plans[blockIdx.x];
  const uint32_t nb = P.nb;
  if (threadIdx.x < 4) {
    s_n[threadIdx.x] = 0;
    s_acc[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) s_slow = 0u;
  for (uint32_t b = threadIdx.x; b <= nb; b += CLS_NT) s_bs[b] = bs[P.bs_base + b];
  __syncthreads();
  // ---- per bucket: decision (parallel) ----
  unsigned long long light = 0, heavy = 0, copyrec = 0;
  for (uint32_t b = threadIdx.x; b < nb; b += CLS_NT) {
    const uint64_t lo = s_bs[b], sz = s_bs[b + 1] - lo;
    uint32_t ty = T_EMPTY;
    if (sz) {
      const uint8_t kind = kinds[P.bs_base + b];
      const uint32_t rem = kind == KIND_OVF ? W : (kind == KIND_HEAVY ? 0u : P.shift);
      if (rem == 0) {
        if (kind == KIND_HEAVY) heavy += sz;
        ty = out_src == 1 ? (sz <= thr ? T_CAND : T_COPY) : T_FLUSH;
      } else {
        light += sz;
        ty = sz <= thr ? T_CAND : T_NEXT;
      }
      if (ty == T_COPY) copyrec += sz;
    }
    s_ty[b] = ty;
  }
  if (light) atomicAdd(&s_acc[0], light);
  if (heavy) atomicAdd(&s_acc[1], heavy);
  if (copyrec) atomicAdd(&s_acc[2], copyrec);
  __syncthreads();
  // ---- spans: greedy packing of adjacent candidates.  When no two
  // neighbouring candidates fit one span together (and no bucket is empty)
  // every candidate is its own span: emitted in parallel; otherwise one
  // thread walks the buckets. ----
  for (uint32_t b = threadIdx.x; b < nb; b += CLS_NT) {
    const uint32_t ty = s_ty[b];
    if (ty == T_EMPTY) s_slow = 1u;
    if (ty == T_CAND && b + 1 < nb && s_ty[b + 1] == T_CAND &&
        (s_bs[b + 2] - s_bs[b]) <= thr)
      s_slow = 1u;
  }
  __syncthreads();
  if (!s_slow) {
    unsigned long long rec = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += CLS_NT) {
      if (s_ty[b] == T_CAND) {
        const uint32_t sz = (uint32_t)(s_bs[b + 1] - s_bs[b]);
        // one light bucket: its keys agree on every bit from the digit up
        const uint32_t bound = kinds[P.bs_base + b] == KIND_LIGHT ? P.shift : SPAN_NOBOUND;
        s_sp[atomicAdd(&s_n[0], 1u)] = Span{P.offset + s_bs[b], sz, out_src | (bound << 8)};
        rec += sz;
      }
    }
    if (rec) atomicAdd(&s_acc[3], rec);
  } else if (threadIdx.x == 0) {
    // Merge rules (`rules` bits, DTS_CLS_RULES): (1) a bucket of equal keys
    // (heavy run, exhausted bucket) stays alone — the base case only copies
    // it, while merged into a neighbour it is a huge equal-key group of a
    // wide span (C4 exp 1e-5: local sort 2.3 -> 1.7 ms).  (2) light buckets
    // that fit the base case's one-pass counting (<= LOCAL_NB differing
    // bits) merge only while the span still does — measured slower (Zipf 1.2
    // local sort 2.8 -> 5.3 ms: the extra small spans cost more than the LSD
    // passes they avoid), off by default.
    uint32_t nsp = 0, first_z = 0;
    bool have = false, cur_equal = false;
    Span cur{0, 0, 0};
    unsigned long long spanrec = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      const uint32_t ty = s_ty[b];
      if (ty == T_EMPTY) continue;
      if (ty == T_CAND) {
        const uint64_t lo = P.offset + s_bs[b];
        const uint32_t sz = (uint32_t)(s_bs[b + 1] - s_bs[b]);
        spanrec += sz;
        const uint8_t kind = kinds[P.bs_base + b];
        const bool equal = (rules & 1u) && (kind == KIND_HEAVY || (kind == KIND_LIGHT && P.shift == 0));
        const uint32_t bound = kind == KIND_LIGHT ? P.shift : SPAN_NOBOUND;
        bool merge = have && !equal && !cur_equal && cur.offset + cur.len == lo && cur.len + sz <= thr;
        uint32_t nbd = SPAN_NOBOUND;
        if (merge) {
          const uint32_t cb = (cur.src >> 8) & 255u;
          if (cb != SPAN_NOBOUND && bound != SPAN_NOBOUND) {
            // several light buckets: the keys agree above the highest bit in
            // which their digits differ (sub-buckets of one zone, split at
            // its heavy keys: above the digit)
            const uint32_t z = zones[P.bs_base + b];
            nbd = P.shift + (32u - (uint32_t)__clz((int)(first_z ^ z)));
            if ((rules & 2u) && P.shift <= LOCAL_NB && nbd > LOCAL_NB) merge = false;
          }
        }
        if (merge) {
          cur.len += sz;
          cur.src = (cur.src & 255u) | (nbd << 8);
        } else {
          if (have) s_sp[nsp++] = cur;
          cur = Span{lo, sz, out_src | (bound << 8)};
          have = true;
          cur_equal = equal;
          first_z = zones[P.bs_base + b];
        }
      } else {
        if (have) s_sp[nsp++] = cur;
        have = false;
      }
    }
    if (have) s_sp[nsp++] = cur;
    s_n[0] = nsp;
    s_acc[3] = spanrec;
  }
  // ---- copies (chunked) and next segments: counted per bucket ----
  for (uint32_t b = threadIdx.x; b < nb; b += CLS_NT) {
    const uint32_t ty = s_ty[b];
    if (ty == T_COPY) {
      const uint64_t sz = s_bs[b + 1] - s_bs[b];
      atomicAdd(&s_n[1], (uint32_t)((sz + copy_chunk - 1) / copy_chunk));
    } else if (ty == T_NEXT) {
      atomicAdd(&s_n[2], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s_base[0] = s_n[0] ? atomicAdd(reinterpret_cast<unsigned int*>(&ctr[0]), s_n[0]) : 0u;
    s_base[1] = s_n[1] ? atomicAdd(reinterpret_cast<unsigned int*>(&ctr[1]), s_n[1]) : 0u;
    s_base[2] = s_n[2] ? atomicAdd(reinterpret_cast<unsigned int*>(&ctr[2]), s_n[2]) : 0u;
    if (s_acc[0]) atomicAdd(&ctr[4], s_acc[0]);
    if (s_acc[1]) atomicAdd(&ctr[5], s_acc[1]);
    if (s_acc[3]) atomicAdd(&ctr[6], s_acc[3]);
    if (s_acc[2]) atomicAdd(&ctr[7], s_acc[2]);
    s_n[1] = 0;
    s_n[2] = 0;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < s_n[0]; i += CLS_NT) spans[s_base[0] + i] = s_sp[i];
  for (uint32_t b = threadIdx.x; b < nb; b += CLS_NT) {
    const uint32_t ty = s_ty[b];
    if (ty == T_COPY) {
      const uint64_t lo = P.offset + s_bs[b], sz = s_bs[b + 1] - s_bs[b];
      const uint32_t nc = (uint32_t)((sz + copy_chunk - 1) / copy_chunk);
      const uint32_t at = s_base[1] + atomicAdd(&s_n[1], nc);
      for (uint32_t c = 0; c < nc; ++c) {
        CopyR r;
        r.offset = lo + (uint64_t)c * copy_chunk;
        r.len = (uint32_t)(sz - (uint64_t)c * copy_chunk < copy_chunk ? sz - (uint64_t)c * copy_chunk : copy_chunk);
        r.pad = 0;
        copies[at + c] = r;
      }
    } else if (ty == T_NEXT) {
      const uint64_t lo = P.offset + s_bs[b], sz = s_bs[b + 1] - s_bs[b];
      const uint8_t kind = kinds[P.bs_base + b];
      const uint32_t rem = kind == KIND_OVF ? W : P.shift;
      // pad bit 1: the parent segment had heavy keys (its children are
      // sampled even when small, dts_api.cu SAMPLE_MIN); bit 2: the parent's
      // sample held no repeated key (its light children are not sampled)
      const uint32_t fl = (P.nheavy ? 2u : 0u) | ((P.flags & PF_UNIQ) && kind != KIND_OVF ? 4u : 0u);
      next[s_base[2] + atomicAdd(&s_n[2], 1u)] = NextSeg{lo, sz, W - rem, fl};
    }
  }
}

// ---------------------------------------------------------------------------
// Dovetail merge (dtmerge.py): insertion points, validation, and the
// out-of-place permutation of the whole zone.
// ---------------------------------------------------------------------------
template <typename K>
__global__ void k_merge_layout(const K* __restrict__ light, uint64_t light_len,
                               const K* __restrict__ hkeys, uint64_t m,
                               uint64_t* __restrict__ ins) {
  // compute_layout: insert point of every heavy key (searchsorted left),
  // dtmerge.py:58-78.
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const K key = hkeys[i];
  uint64_t lo = 0, hi = light_len;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (light[mid] < key) lo = mid + 1; else hi = mid;
  }
  ins[i] = lo;
}

template <typename K>
__global__ void k_merge_validate(const K* __restrict__ zone, uint64_t light_len, uint64_t total,
                                 const K* __restrict__ hkeys, const uint64_t* __restrict__ hprefix,
                                 uint64_t m, const uint64_t* __restrict__ ins,
                                 uint32_t* __restrict__ err) {
  // _validate (dtmerge.py:108-129): bit0 light unsorted, bit1 heavy key in
  // light run, bit2 foreign key inside a heavy run.
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    if (i + 1 < light_len && zone[i + 1] < zone[i]) atomicOr(err, 1u);
    if (i < m) {
      const uint64_t p = ins[i];
      if (p < light_len && zone[p] == hkeys[i]) atomicOr(err, 2u);
    }
    if (i >= light_len) {
      const uint64_t h = i - light_len;
      uint64_t lo = 0, hi = m;  // run r with hprefix[r] <= h < hprefix[r+1]
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (hprefix[mid] <= h) lo = mid; else hi = mid;
      }
      if (m > 0 && zone[i] != hkeys[lo]) atomicOr(err, 4u);
    }
  }
}

// Layout-driven out-of-place merge permutation (dtmerge.py:58-78 layout, the
// result of :132-238): light record j lands at j + (heavy records whose key
// is below it) = j + hprefix[#{i : ins[i] <= j}]; heavy record r of run i at
// ins[i] + hprefix[i] + r.  One pass over the zone into the workspace copy.
template <typename K, int VB>
__global__ void k_merge_permute(const K* __restrict__ zk, const typename ValOf<VB>::T* __restrict__ zv,
                                uint64_t light_len, uint64_t total, const uint64_t* __restrict__ ins,
                                const uint64_t* __restrict__ hprefix, uint64_t m, K* __restrict__ ok,
                                typename ValOf<VB>::T* __restrict__ ov) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < total; s += stride) {
    uint64_t d;
    if (s < light_len) {
      uint64_t lo = 0, hi = m;  // #{i : ins[i] <= s}
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (ins[mid] <= s) lo = mid + 1; else hi = mid;
      }
      d = s + hprefix[lo];
    } else {
      const uint64_t h = s - light_len;
      uint64_t lo = 0, hi = m;  // run i: hprefix[i] <= h < hprefix[i + 1]
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (hprefix[mid] <= h) lo = mid; else hi = mid;
      }
      d = ins[lo] + h;
    }
    ok[d] = zk[s];
    if (VB && zv) ov[d] = zv[s];
  }
}

template <typename K, int VB>
__global__ void k_copy_back(K* __restrict__ dk, typename ValOf<VB>::T* __restrict__ dv,
                            const K* __restrict__ sk, const typename ValOf<VB>::T* __restrict__ sv,
                            uint64_t len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    dk[i] = sk[i];
    if (VB && dv) dv[i] = sv[i];
  }
}

}  // namespace dts
