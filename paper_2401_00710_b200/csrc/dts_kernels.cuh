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
  L.hz = o; o = align16(o + (size_t)c.hzc * 4);
  L.total = o;
  return L;
}

struct ScatterLayout {
  size_t run, sk, sv, hk, si, tst, hz, wh, sb, total;
};
__host__ __device__ inline ScatterLayout scatter_layout(int T, int NW, int kb, int vb,
                                                        Caps c, bool split) {
  ScatterLayout L;
  size_t o = 0;
  L.run = o; o = align16(o + (size_t)c.nbc * 8);
  L.sk = o; o = align16(o + (size_t)T * kb);
  L.sv = o; o = align16(o + (size_t)T * vb);
  L.hk = o; o = align16(o + (size_t)c.hkc * kb);
  L.si = o; o = align16(o + (split ? (size_t)c.hkc * 8 : 0));
  L.tst = o; o = align16(o + ((size_t)c.nbc + 1) * 4);
  L.hz = o; o = align16(o + (size_t)c.hzc * 4);
  L.wh = o; o = align16(o + (size_t)NW * c.nbc * 2);
  L.sb = o; o = align16(o + (size_t)T * 2);
  L.total = o;
  return L;
}

struct LocalLayout {
  size_t sk, sv, si, wh, total;
};
__host__ __device__ inline LocalLayout local_layout(int CAP, int NW, int kb, int vb) {
  LocalLayout L;
  size_t o = 0;
  L.sk = o; o = align16(o + (size_t)CAP * kb);
  L.sv = o; o = align16(o + (size_t)CAP * vb);
  L.si = o; o = align16(o + (size_t)CAP * 2);
  L.wh = o; o = align16(o + (size_t)256 * NW * 2);
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
  } else if (P.flags & PF_HEAVY) {
    const uint32_t nz = (1u << P.gamma) + 1u;
    for (uint32_t i = threadIdx.x; i < nz; i += blockDim.x) hz[i] = hz_pool[P.hz_base + i];
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
                                                    uint32_t gs_max, uint32_t smax) {
  constexpr int W = sizeof(K) * 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sm = reinterpret_cast<K*>(smem_raw);
  __shared__ uint32_t s_tmp[NT / 32 + 1];
  __shared__ uint32_t s_m;

  const uint32_t s = seg_ids[blockIdx.x];
  SegPlan P = plans[s];
  const uint32_t gs = min(P.gamma, gs_max);
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
  // bitonic sort of sm[0..P2)
  for (uint32_t k = 2; k <= P2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P2 / 2; i += NT) {
        const uint32_t a = 2 * i - (i & (j - 1));
        const uint32_t b = a + j;
        const bool up = (a & k) == 0;
        const K x = sm[a], y = sm[b];
        if ((x > y) == up) {
          sm[a] = y;
          sm[b] = x;
        }
      }
      __syncthreads();
    }
  }
  uint32_t gamma = P.gamma, shift = P.shift;
  uint32_t flags = P.flags & ~(PF_HEAVY | PF_OVF);
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
  const uint32_t m = s_m;
  __syncthreads();
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
// k_histogram: persistent CTAs pull blocks; per block, count records per
// bucket in SMEM with warp-aggregated atomics (one atomic per distinct
// bucket per warp step) and store the row into the [bucket][row] matrix.
// counting.py:123-137.
// ---------------------------------------------------------------------------
template <typename K, int NT, bool SPLIT>
__global__ void __launch_bounds__(NT) k_histogram(const SegPlan* __restrict__ plans,
                                                  const Blk* __restrict__ blks, uint32_t nblk,
                                                  uint32_t* __restrict__ ctr,
                                                  const K* __restrict__ keys,
                                                  uint32_t* __restrict__ counts,
                                                  const K* __restrict__ heavy_pool,
                                                  const uint32_t* __restrict__ hz_pool,
                                                  const uint64_t* __restrict__ split_idx,
                                                  uint64_t global_base, Caps caps) {
  constexpr int VEC = 16 / sizeof(K);
  constexpr int U = 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const HistLayout L = hist_layout(sizeof(K), caps, SPLIT);
  K* hk = reinterpret_cast<K*>(smem_raw + L.hk);
  uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + L.si);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem_raw + L.hist);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + L.hz);
  __shared__ uint32_t s_blk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

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
    const int nbits = max(1, (int)ceil_log2_u64(P.nb));

    auto count_one = [&](K key, bool valid, uint64_t gidx) {
      uint32_t b = 0;
      if (valid) b = SPLIT ? SR(key, gidx) : R(key);
      const uint32_t vm = __ballot_sync(FULL, valid);
      if (vm == 0) return;
      const uint32_t peers = peer_mask(b, vm, nbits);
      if (valid && (peers & lanemask_lt()) == 0) atomicAdd(&hist[b], (uint32_t)__popc(peers));
    };

    const K* p = keys + B.begin;
    const uint64_t n = B.end - B.begin;
    const uint64_t addr = reinterpret_cast<uint64_t>(p);
    uint64_t head = ((16 - (addr & 15)) & 15) / sizeof(K);
    if (head > n) head = n;
    const uint64_t nvec = (n - head) / VEC;
    const uint64_t tail0 = head + nvec * VEC;
    if (warp == 0) {
      const uint64_t ntail = n - tail0;
      uint64_t e = lane < head ? (uint64_t)lane : tail0 + (lane - head);
      const bool valid = (uint64_t)lane < head + ntail;
      count_one(valid ? p[e] : (K)0, valid, global_base + B.begin + e);
    }
    const uint4* pv = reinterpret_cast<const uint4*>(p + head);
    for (uint64_t vb = 0; vb < nvec; vb += (uint64_t)NT * U) {
      uint4 v[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t vi = vb + (uint64_t)u * NT + tid;
        ok[u] = vi < nvec;
        if (ok[u]) v[u] = __ldg(pv + vi);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t e0 = head + (vb + (uint64_t)u * NT + tid) * VEC;
        const K* kk = reinterpret_cast<const K*>(&v[u]);
#pragma unroll
        for (int e = 0; e < VEC; ++e) count_one(ok[u] ? kk[e] : (K)0, ok[u], global_base + B.begin + e0 + e);
      }
    }
    __syncthreads();
    uint32_t* row = counts + P.cnt_base + B.row;
    for (uint32_t b = tid; b < P.nbmax; b += NT) row[(uint64_t)b * P.nrows] = hist[b];
    __syncthreads();
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
                                                       uint8_t* __restrict__ kinds) {
  const SegPlan P = plans[blockIdx.x];
  for (uint32_t b = threadIdx.x; b <= P.nbmax; b += blockDim.x) {
    uint64_t v = P.len;
    uint8_t kind = KIND_PAD;
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
      } else {
        kind = KIND_LIGHT;
      }
    }
    bstart[P.bs_base + b] = v;
    kinds[P.bs_base + b] = kind;
  }
}

// ---------------------------------------------------------------------------
// k_scatter: persistent CTAs pull blocks; each block walks its tiles in
// order.  Per tile: records go to registers (warp-contiguous, lane-striped,
// i.e. input order), get a stable in-tile rank from warp-private counters and
// ballot peer sets, are regrouped by bucket in SMEM, and are written out as
// contiguous runs at run[b] (the block's running offset row — the GPU twin of
// scatter_block's `run`, _kernels.py:19-25).  Stable for every block count.
// ---------------------------------------------------------------------------
template <typename K, int VB, int NT, int IPT, bool SPLIT>
__global__ void __launch_bounds__(NT) k_scatter(const SegPlan* __restrict__ plans,
                                                const Blk* __restrict__ blks, uint32_t nblk,
                                                uint32_t* __restrict__ ctr,
                                                const K* __restrict__ kin,
                                                const typename ValOf<VB>::T* __restrict__ vin,
                                                K* __restrict__ kout,
                                                typename ValOf<VB>::T* __restrict__ vout,
                                                const uint64_t* __restrict__ scan,
                                                const K* __restrict__ heavy_pool,
                                                const uint32_t* __restrict__ hz_pool,
                                                const uint64_t* __restrict__ split_idx,
                                                uint64_t global_base, Caps caps) {
  using V = typename ValOf<VB>::T;
  constexpr int NW = NT / 32;
  constexpr int T = NT * IPT;
  constexpr int IPW = 32 * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const ScatterLayout L = scatter_layout(T, NW, sizeof(K), VB, caps, SPLIT);
  uint64_t* run = reinterpret_cast<uint64_t*>(smem_raw + L.run);
  K* sk = reinterpret_cast<K*>(smem_raw + L.sk);
  V* sv = reinterpret_cast<V*>(smem_raw + L.sv);
  K* hk = reinterpret_cast<K*>(smem_raw + L.hk);
  uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + L.si);
  uint32_t* tst = reinterpret_cast<uint32_t*>(smem_raw + L.tst);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + L.hz);
  uint16_t* wh = reinterpret_cast<uint16_t*>(smem_raw + L.wh);
  uint16_t* sb = reinterpret_cast<uint16_t*>(smem_raw + L.sb);
  __shared__ uint32_t s_blk;
  __shared__ uint32_t s_tmp[NW + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nbc = caps.nbc;
  uint16_t* mywh = wh + warp * nbc;

  for (;;) {
    if (tid == 0) s_blk = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t bi = s_blk;
    if (bi >= nblk) break;
    const Blk B = blks[bi];
    const SegPlan P = plans[B.seg];
    const uint32_t nb = P.nb;
    load_tables<K>(P, heavy_pool, hz_pool, split_idx, hk, si, hz);
    {
      const uint64_t* col = scan + P.cnt_base + B.row;
      const uint64_t rb = P.offset - P.scanbase;
      for (uint32_t b = tid; b < nb; b += NT) run[b] = rb + col[(uint64_t)b * P.nrows];
      uint32_t* wh32 = reinterpret_cast<uint32_t*>(wh);
      for (uint32_t i = tid; i < NW * nbc / 2; i += NT) wh32[i] = 0u;
    }
    __syncthreads();
    const Router<K> R = make_router<K>(P, hz, hk);
    SplitRouter<K> SR;
    SR.sk = hk; SR.si = si; SR.ns = P.nheavy;
    const int nbits = max(1, (int)ceil_log2_u64(nb));

    for (uint64_t tile = B.begin; tile < B.end; tile += T) {
      const uint64_t rem_ = B.end - tile;
      const uint32_t tn = rem_ < (uint64_t)T ? (uint32_t)rem_ : (uint32_t)T;
      K k[IPT];
      V v[IPT];
      uint32_t br[IPT];
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const uint32_t loc = warp * IPW + j * 32 + lane;
        if (loc < tn) {
          k[j] = kin[tile + loc];
          if (VB) v[j] = vin[tile + loc];
        }
      }
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const uint32_t loc = warp * IPW + j * 32 + lane;
        const bool valid = loc < tn;
        const uint32_t vm = __ballot_sync(FULL, valid);
        br[j] = 0;
        if (vm) {
          uint32_t b = 0;
          if (valid) b = SPLIT ? SR(k[j], global_base + tile + loc) : R(k[j]);
          const uint32_t peers = peer_mask(b, vm, nbits);
          const uint32_t before = __popc(peers & lanemask_lt());
          uint32_t old = 0;
          if (valid) old = mywh[b];
          __syncwarp();
          if (valid && before == 0) mywh[b] = (uint16_t)(old + __popc(peers));
          __syncwarp();
          br[j] = (b << 16) | (old + before);
        }
      }
      __syncthreads();
      // per bucket: exclusive prefix over warps (in place) and tile count
      for (uint32_t b = tid; b < nb; b += NT) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint32_t t = wh[w * nbc + b];
          wh[w * nbc + b] = (uint16_t)s;
          s += t;
        }
        tst[b] = s;
      }
      __syncthreads();
      block_exscan<NT>(tst, (int)nb, s_tmp);
      if (tid == 0) tst[nb] = tn;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const uint32_t loc = warp * IPW + j * 32 + lane;
        if (loc < tn) {
          const uint32_t b = br[j] >> 16;
          const uint32_t pos = tst[b] + mywh[b] + (br[j] & 0xffffu);
          sk[pos] = k[j];
          if (VB) sv[pos] = v[j];
          sb[pos] = (uint16_t)b;
        }
      }
      __syncthreads();
      for (uint32_t p = tid; p < tn; p += NT) {
        const uint32_t b = sb[p];
        const uint64_t d = run[b] + (p - tst[b]);
        kout[d] = sk[p];
        if (VB) vout[d] = sv[p];
      }
      __syncthreads();
      for (uint32_t b = tid; b < nb; b += NT) run[b] += tst[b + 1] - tst[b];
      {
        uint32_t* wh32 = reinterpret_cast<uint32_t*>(wh);
        for (uint32_t i = tid; i < NW * nbc / 2; i += NT) wh32[i] = 0u;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// k_local_sort: one CTA per base-case span (<= CAP records).  Loads the span
// into SMEM, finds the bits that differ inside it, and runs stable LSD passes
// of <= 8 bits on (key, slot) pairs; payloads are gathered once at the end.
// Output always lands in A.  dtsort.py:127-147 (stable sort by full key of a
// span of adjacent buckets, valid per :128-131).
// ---------------------------------------------------------------------------
template <typename K, int VB, int NT, int CAP>
__global__ void __launch_bounds__(NT) k_local_sort(const Span* __restrict__ spans,
                                                   K* __restrict__ Ak,
                                                   typename ValOf<VB>::T* __restrict__ Av,
                                                   const K* __restrict__ Tk,
                                                   const typename ValOf<VB>::T* __restrict__ Tv) {
  using V = typename ValOf<VB>::T;
  constexpr int W = sizeof(K) * 8;
  constexpr int NW = NT / 32;
  constexpr int IPT = CAP / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const LocalLayout L = local_layout(CAP, NW, sizeof(K), VB);
  K* sk = reinterpret_cast<K*>(smem_raw + L.sk);
  V* sv = reinterpret_cast<V*>(smem_raw + L.sv);
  uint16_t* si = reinterpret_cast<uint16_t*>(smem_raw + L.si);
  uint16_t* wh = reinterpret_cast<uint16_t*>(smem_raw + L.wh);  // [digit][warp]
  __shared__ uint32_t s_tmp[NW + 1];
  __shared__ K s_diff[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const Span S = spans[blockIdx.x];
  const uint32_t n = S.len;
  const K* srck = S.src ? Tk : Ak;
  const V* srcv = S.src ? Tv : Av;
  const K* gk = srck + S.offset;
  const K k0 = gk[0];
  K diff = 0;
  for (uint32_t i = tid; i < n; i += NT) {
    const K x = gk[i];
    sk[i] = x;
    diff |= x ^ k0;
    if (VB) sv[i] = srcv[S.offset + i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) diff |= __shfl_xor_sync(FULL, diff, o);
  if (lane == 0) s_diff[warp] = diff;
  __syncthreads();
  diff = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) diff |= s_diff[w];
  int bits = 0;
  if (diff) bits = (sizeof(K) == 8) ? 64 - __clzll((long long)diff) : 32 - __clz((int)(uint32_t)diff);

  if (bits > 0) {
    const int passes = (bits + 7) / 8;
    const int R = (bits + passes - 1) / passes;
    const uint32_t nd = 1u << R;
    const uint32_t dmask = nd - 1u;
    for (uint32_t i = tid; i < n; i += NT) si[i] = (uint16_t)i;
    const uint32_t per = (((n + NW - 1) / NW) + 31u) & ~31u;  // items per warp
    const uint32_t w0 = warp * per;
    const uint32_t w1 = min(n, w0 + per);
    for (int pass = 0; pass < passes; ++pass) {
      const int shift = pass * R;
      for (uint32_t i = tid; i < nd * NW; i += NT) wh[i] = 0;
      __syncthreads();
      K k[IPT];
      uint32_t ix[IPT];
      uint32_t br[IPT];
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const uint32_t loc = w0 + j * 32 + lane;
        const bool valid = loc < w1;
        br[j] = 0;
        if ((uint32_t)(j * 32) >= per) continue;  // warp-uniform
        if (valid) {
          k[j] = sk[loc];
          ix[j] = si[loc];
        }
        const uint32_t vm = __ballot_sync(FULL, valid);
        if (!vm) continue;
        const uint32_t d = valid ? (uint32_t)(k[j] >> shift) & dmask : 0u;
        const uint32_t peers = peer_mask(d, vm, R);
        const uint32_t before = __popc(peers & lanemask_lt());
        uint32_t old = 0;
        if (valid) old = wh[d * NW + warp];
        __syncwarp();
        if (valid && before == 0) wh[d * NW + warp] = (uint16_t)(old + __popc(peers));
        __syncwarp();
        br[j] = (d << 16) | (old + before);
      }
      __syncthreads();
      block_exscan<NT>(wh, (int)(nd * NW), s_tmp);
#pragma unroll
      for (int j = 0; j < IPT; ++j) {
        const uint32_t loc = w0 + j * 32 + lane;
        if ((uint32_t)(j * 32) < per && loc < w1) {
          const uint32_t d = br[j] >> 16;
          const uint32_t pos = wh[d * NW + warp] + (br[j] & 0xffffu);
          sk[pos] = k[j];
          si[pos] = (uint16_t)ix[j];
        }
      }
      __syncthreads();
    }
    K* ok = Ak + S.offset;
    for (uint32_t i = tid; i < n; i += NT) {
      ok[i] = sk[i];
      if (VB) Av[S.offset + i] = sv[si[i]];
    }
  } else if (S.src) {
    K* ok = Ak + S.offset;
    for (uint32_t i = tid; i < n; i += NT) {
      ok[i] = sk[i];
      if (VB) Av[S.offset + i] = sv[i];
    }
  }
}

// ---------------------------------------------------------------------------
// k_copy_ranges: finished ranges T -> A (heavy runs, exhausted-digit runs).
// ---------------------------------------------------------------------------
template <typename K, int VB>
__global__ void __launch_bounds__(256) k_copy_ranges(const CopyR* __restrict__ rs,
                                                     K* __restrict__ Ak,
                                                     typename ValOf<VB>::T* __restrict__ Av,
                                                     const K* __restrict__ Tk,
                                                     const typename ValOf<VB>::T* __restrict__ Tv) {
  const CopyR r = rs[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < r.len; i += blockDim.x) {
    Ak[r.offset + i] = Tk[r.offset + i];
    if (VB) Av[r.offset + i] = Tv[r.offset + i];
  }
}

// ---------------------------------------------------------------------------
// Dovetail-merge pieces (dtmerge.py).  The host runs the reference's piece
// loop and launches these grid-parallel moves.
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

template <typename K, int VB>
__global__ void k_move(K* __restrict__ dk, typename ValOf<VB>::T* __restrict__ dv,
                       const K* __restrict__ sk, const typename ValOf<VB>::T* __restrict__ sv,
                       uint64_t len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    dk[i] = sk[i];
    if (VB) dv[i] = sv[i];
  }
}

template <typename K, int VB>
__global__ void k_reverse(K* __restrict__ k, typename ValOf<VB>::T* __restrict__ v, uint64_t lo,
                          uint64_t hi) {
  // reverse_range (_kernels.py:28-38): pairs (lo+i, hi-1-i) swap independently.
  const uint64_t half = (hi - lo) / 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < half; i += stride) {
    const uint64_t a = lo + i, b = hi - 1 - i;
    const K t = k[a];
    k[a] = k[b];
    k[b] = t;
    if (VB) {
      const typename ValOf<VB>::T u = v[a];
      v[a] = v[b];
      v[b] = u;
    }
  }
}

}  // namespace dts
