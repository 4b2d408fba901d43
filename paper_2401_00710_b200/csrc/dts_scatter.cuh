// dts_scatter.cuh — k_scatter, the stable distribution pass
// (counting.py:141-151 scatter phase, _kernels.py:12-25 scatter_block).
#pragma once
#include "dts_rank.cuh"
#include "dts_sort_kernels.cuh"

namespace dts {

// Per-(key, value) width tiling of the scatter.
template <typename K, int VB> struct ScatterTile {
  static constexpr int NT = 512;
  static constexpr int NW = NT / 32;
  static constexpr int IPT = (sizeof(K) == 4 && VB <= 4) ? 9 : 5;
  static constexpr int WS = 32 * IPT;  // records per warp sub-tile
  static constexpr int T = NT * IPT;
  static constexpr int NBC = 1024;     // bucket capacity (ids < 2^10)
  static constexpr int LB = 8;         // tiles per hist block (look-back depth < LB)
  static constexpr int HKC = 1024;     // heavy keys / splitters capacity
  static constexpr int HZC = 520;      // zone table capacity (2^9 + 1, padded)
};

// Look-back status: one u32 per (tile, bucket pair) = the tile's packed
// counts of buckets 2j (bits 0-12) and 2j+1 (bits 16-28) | ST_VALID (bit 15).
// Tile counts are <= T < 2^13 and a tile sums <= LB-1 predecessors, so the
// packed sums never carry into bit 15 or bit 31.
constexpr uint32_t ST_VALID = 0x8000u;
constexpr uint32_t ST_MASK = 0x7fff7fffu;

__host__ __device__ constexpr size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

// Compile-time SMEM layout (immediate-offset addressing in the kernel).
template <typename K, int VB, bool SPLIT> struct ScatterSmem {
  using TL = ScatterTile<K, VB>;
  static constexpr size_t sk = 0;
  static constexpr size_t sv = a16(sk + (size_t)(TL::T + 8) * sizeof(K));
  static constexpr size_t pk = a16(sv + (size_t)(TL::T + 8) * VB);
  static constexpr size_t wh = a16(pk + (size_t)(TL::T + 1) * 4);  // + sentinel
  static constexpr size_t tst = a16(wh + (size_t)TL::NW * (TL::NBC / 2) * 4);
  static constexpr size_t db = a16(tst + (size_t)(TL::NBC + 1) * 4);
  static constexpr size_t hk = a16(db + (size_t)TL::NBC * 4);
  static constexpr size_t si = a16(hk + (size_t)(SPLIT ? TL::HKC : 256) * sizeof(K));
  static constexpr size_t hz = a16(si + (SPLIT ? (size_t)TL::HKC * 8 : 0));
  static constexpr size_t geo = a16(hz + (SPLIT ? ((size_t)1 << SPLIT_TB) : (size_t)TL::HZC * 4));
  static constexpr size_t plan = a16(geo + 2 * 32);
  static constexpr size_t bar = a16(plan + 2 * sizeof(SegPlan));
  static constexpr size_t total = a16(bar + 16);
};

// Split [g0, g0+tn) of a T-typed column into head / 16-byte aligned body /
// tail by absolute address (the caller's column may start anywhere); returns
// the body bytes (moved by cp.async.bulk).
template <typename T>
__device__ __forceinline__ uint32_t tile_body(const T* col, uint64_t g0, uint32_t tn, uint32_t& off,
                                              uint32_t& head, uint32_t& nbody) {
  constexpr uint32_t VEC = 16 / sizeof(T);
  off = (uint32_t)((reinterpret_cast<uintptr_t>(col + g0) & 15u) / sizeof(T));
  const uint32_t h0 = (VEC - off) % VEC;
  head = h0 < tn ? h0 : tn;
  nbody = ((tn - head) / VEC) * VEC;
  return nbody * (uint32_t)sizeof(T);
}

// 16-byte aligned superset [floor16(g0), ceil16(g0+tn)) of a column's tile
// (whole 16-byte chunks never cross a page, so the few extra bytes read at
// either end are always mapped); `off` = elements before g0 in SMEM.
template <typename T>
__device__ __forceinline__ uint32_t tile_span(const T* col, uint64_t g0, uint32_t tn,
                                              const char*& src, uint32_t& off) {
  const uint64_t b0 = reinterpret_cast<uint64_t>(col + g0);
  const uint64_t a0 = b0 & ~uint64_t(15);
  const uint64_t a1 = (reinterpret_cast<uint64_t>(col + g0 + tn) + 15) & ~uint64_t(15);
  src = reinterpret_cast<const char*>(a0);
  off = (uint32_t)(b0 - a0) / (uint32_t)sizeof(T);
  return (uint32_t)(a1 - a0);
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_global(uint32_t* p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ void st_global(unsigned long long* p, unsigned long long v) {
  asm volatile("st.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}
__device__ __forceinline__ void st_global(unsigned long* p, unsigned long v) {
  asm volatile("st.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}
// two adjacent elements (8- or 16-byte aligned) in one store
__device__ __forceinline__ void st_global2(uint32_t* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b));
}
__device__ __forceinline__ void st_global2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b));
}
__device__ __forceinline__ void st_global2(unsigned long* p, unsigned long a, unsigned long b) {
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b));
}
template <typename T>
__device__ __forceinline__ T* opaque_ptr(T* p) {
  asm volatile("mov.b64 %0, %0;" : "+l"(p));
  return p;
}

// DTS_PHASE_PROF=1 (tools build only): thread 0 of every CTA accumulates
// clock64() cycles per tile phase; read back with dts_debug_phases().
#ifndef DTS_PHASE_PROF
#define DTS_PHASE_PROF 0
#endif
#if DTS_PHASE_PROF
__device__ unsigned long long g_phase[16];
// each kernel sets `ph_on` (DTS_PHASE_PROF == 1: scatter kernels, 2: local sort)
#define PH_INIT unsigned long long ph_acc[11] = {0}; long long ph_t = clock64();
#define PH(k)                                         \
  if (ph_on && tid == 0) {                            \
    const long long now_ = clock64();                 \
    ph_acc[k] += (unsigned long long)(now_ - ph_t);   \
    ph_t = now_;                                      \
  }
#define PH_SPIN if (ph_on && tid < 512) atomicAdd(&g_phase[15], 1ull);
#define PH_DONE                                                          \
  if (ph_on && tid == 0) {                                               \
    for (int k_ = 0; k_ < 11; ++k_) atomicAdd(&g_phase[k_], ph_acc[k_]); \
    atomicAdd(&g_phase[14], 1ull);                                       \
  }
#else
#define PH_INIT
#define PH(k)
#define PH_SPIN
#define PH_DONE
#endif

struct TileGeo {  // one scatter tile: hist block bi, tile kt in it, records [g0, g0+tn)
  uint64_t g0;
  uint32_t tn, kt, bi, seg, row, t;
};

// ---------------------------------------------------------------------------
// k_scatter: persistent CTAs (2 per SM) take tiles round-robin in input
// order (onesweep-style).  Per tile:
//   * keys/values arrive in SMEM by one TMA bulk copy each (cp.async.bulk on
//     an mbarrier); warp 1 meanwhile resolves the CTA's next tile and
//     prefetches it into L2;
//   * stable in-tile rank with per-warp bucket counters: warp w owns the
//     contiguous sub-tile [w*WS, (w+1)*WS) in lane-striped order and takes
//     its records' ranks from SMEM atomics on its own packed u16 counters;
//     an exclusive prefix over warps orders the warps; the in-step lane
//     order (served by the hardware, verified here) orders the rest;
//   * the tile's bucket bases = its hist block's offsets (count matrix scan,
//     counting.py:58-79, loaded early) + the counts of the earlier tiles of
//     the block (< LB of them, read in parallel from per-tile status words
//     published right after ranking: decoupled look-back);
//   * the tile is regrouped by bucket in SMEM and each bucket run is stored
//     contiguously.  Tiles in flight are consecutive in input order, so the
//     partial 32-byte sectors at run ends are completed by neighbouring
//     tiles within microseconds and merge in L2.
// Stable for every block and tile count (counting.py:1-10 invariant;
// scatter_block, _kernels.py:12-25, keeps the same per-bucket `run` order).
// Segment-relative positions are u32 (segments < 2^32 records).
// ---------------------------------------------------------------------------
template <typename K, int VB, bool SPLIT>
__global__ void __launch_bounds__(ScatterTile<K, VB>::NT, 2)
    k_scatter(const SegPlan* __restrict__ plans, const Blk* __restrict__ blks,
              const uint32_t* __restrict__ tile_blk, const uint32_t* __restrict__ blk_tile0,
              uint32_t ntile, uint32_t nbs, const K* __restrict__ kin,
              const typename ValOf<VB>::T* __restrict__ vin, K* __restrict__ kout,
              typename ValOf<VB>::T* __restrict__ vout, const uint64_t* __restrict__ scan,
              uint32_t* __restrict__ status, const K* __restrict__ heavy_pool,
              const uint32_t* __restrict__ hz_pool, const uint64_t* __restrict__ split_idx,
              uint64_t global_base) {
  using V = typename ValOf<VB>::T;
  using TL = ScatterTile<K, VB>;
  using SL = ScatterSmem<K, VB, SPLIT>;
  constexpr int NT = TL::NT, NW = TL::NW, IPT = TL::IPT, WS = TL::WS, T = TL::T, LB = TL::LB;
  constexpr uint32_t HW = TL::NBC / 2;  // packed counter words per warp = bucket pairs
  static_assert(HW <= (uint32_t)NT, "one bucket pair per thread");
  static_assert((LB - 1) * T < 32768 && T < 8192, "packed look-back sums must not carry");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* skb = reinterpret_cast<K*>(smem_raw + SL::sk);
  V* svb = reinterpret_cast<V*>(smem_raw + SL::sv);
  uint32_t* pk = reinterpret_cast<uint32_t*>(smem_raw + SL::pk);
  uint32_t* wh = reinterpret_cast<uint32_t*>(smem_raw + SL::wh);
  uint32_t* tst = reinterpret_cast<uint32_t*>(smem_raw + SL::tst);
  uint32_t* db = reinterpret_cast<uint32_t*>(smem_raw + SL::db);
  K* hk = reinterpret_cast<K*>(smem_raw + SL::hk);
  uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + SL::si);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + SL::hz);
  TileGeo* sgeo = reinterpret_cast<TileGeo*>(smem_raw + SL::geo);
  SegPlan* splan = reinterpret_cast<SegPlan*>(smem_raw + SL::plan);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + SL::bar);
  __shared__ uint32_t s_fix, s_seg;
  __shared__ uint32_t s_wt[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* mywh = wh + warp * HW;

  // resolve tile t's geometry and plan into slot `slot` (one warp)
  auto resolve = [&](uint32_t t, int slot) {
    if (lane == 0) {
      const uint32_t bi = tile_blk[t];
      const Blk B = blks[bi];
      TileGeo g;
      g.kt = t - blk_tile0[bi];
      g.g0 = B.begin + (uint64_t)g.kt * T;
      g.tn = (uint32_t)min((uint64_t)T, B.end - g.g0);
      g.bi = bi;
      g.seg = B.seg;
      g.row = B.row;
      g.t = t;
      sgeo[slot] = g;
    }
    __syncwarp();
    const uint32_t seg = sgeo[slot].seg;
    constexpr int PW = sizeof(SegPlan) / 4;
    if (lane < PW)
      reinterpret_cast<uint32_t*>(&splan[slot])[lane] =
          reinterpret_cast<const uint32_t*>(&plans[seg])[lane];
  };

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    fence_mbar_init();
    s_fix = 0u;
    s_seg = 0xFFFFFFFFu;
    pk[T] = 0xFFFFFFFFu;  // write-out sentinel of full tiles
  }
  for (uint32_t i = tid; i < NW * HW; i += NT) wh[i] = 0u;
  if (warp == 0 && blockIdx.x < ntile) resolve(blockIdx.x, 0);
  __syncthreads();
  uint32_t phase = 0u;
  int cur = 0;
  [[maybe_unused]] constexpr bool ph_on = DTS_PHASE_PROF == 1;
  PH_INIT

  for (uint32_t t = blockIdx.x; t < ntile; t += gridDim.x, cur ^= 1) {
    PH(0)
    const TileGeo G = sgeo[cur];
    const SegPlan& P = splan[cur];
    const uint32_t nb = P.nb, tn = G.tn, kt = G.kt;
    const uint32_t npair = (nb + 1) >> 1;
    const uint64_t g0 = G.g0;
    const bool full = tn == (uint32_t)T;
    // ---- issue the tile loads (one bulk copy per column) ----
    uint32_t ko, vo = 0;
    {
      const char* ksrc;
      const uint32_t kbytes = tile_span<K>(kin, g0, tn, ksrc, ko);
      const char* vsrc = nullptr;
      uint32_t vbytes = 0;
      if (VB) vbytes = tile_span<V>(vin, g0, tn, vsrc, vo);
      if (tid == 0) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bar[0], kbytes + vbytes);
        tma_load_1d(skb, ksrc, kbytes, &bar[0]);
        if (VB) tma_load_1d(svb, vsrc, vbytes, &bar[0]);
        if (!full) pk[tn] = 0xFFFFFFFFu;  // sentinel
      }
    }
    // hist-block offsets of this thread's bucket pair (needed much later)
    // (raw u64 values: nothing waits on these loads before the look-back)
    uint64_t bo0 = 0, bo1 = 0;
    if ((uint32_t)tid < npair) {
      const uint64_t* col = scan + P.cnt_base + G.row;
      const uint64_t nr = P.nrows;
      bo0 = col[(uint64_t)(2 * tid) * nr];
      if ((uint32_t)(2 * tid + 1) < nb) bo1 = col[(uint64_t)(2 * tid + 1) * nr];
    }
    if (G.seg != s_seg) {  // block-uniform
      load_tables<K>(P, heavy_pool, hz_pool, split_idx, hk, si, hz);
    }
    __syncthreads();
    PH(1)
    if (tid == 0) s_seg = G.seg;
    mbar_wait(&bar[0], phase);
    phase ^= 1u;
    PH(2)
    const K* sk = skb + ko;
    const V* sv = svb + vo;

    // ---- route + per-warp rank (lane-striped within the warp sub-tile) ----
    uint32_t bk[IPT], lr[IPT];
    auto rank_one = [&](int i, uint32_t b) {
      const uint32_t sh = (b & 1u) << 4;
      const uint32_t old = atomicAdd(&mywh[b >> 1], 1u << sh);
      bk[i] = b;
      lr[i] = (old >> sh) & 0xffffu;
    };
    if (!SPLIT && full && !(P.flags & PF_HEAVY)) {
      // light digit, overflow bucket by select (sampler.py:76-100 bucket ids;
      // without an overflow bucket the all-ones key maps to its own digit)
      const uint32_t shift = P.shift, mask = (1u << P.gamma) - 1u;
      const bool ovf = (P.flags & PF_OVF) != 0;
      const K thr = ovf ? P.ovf_thr : ~K(0);
      const uint32_t ovfb = ovf ? nb - 1 : ((uint32_t)(~K(0) >> shift) & mask);
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const K key = sk[warp * WS + i * 32 + lane];
        rank_one(i, key >= thr ? ovfb : ((uint32_t)(key >> shift) & mask));
        __syncwarp();
      }
    } else if (SPLIT) {
      // very few destinations (G <= 4 ranks): ranks from ballot peer masks;
      // the first lane of each group bumps the warp's u16 counter (no
      // atomics: 8-16 lanes per address would serialise)
      SplitRouter<K> SR;
      SR.sk = hk; SR.si = si; SR.ns = P.nheavy;
      SR.tab = P.nheavy <= 15 ? reinterpret_cast<const uint8_t*>(hz) : nullptr;
      if (nb <= 4) {
      uint16_t* myc16 = reinterpret_cast<uint16_t*>(mywh);
      const int nbits = nb > 1 ? 32 - __clz((int)(nb - 1)) : 0;
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        const bool valid = e < tn;
        const uint32_t b = valid ? SR(sk[e], global_base + g0 + e) : 0u;
        const uint32_t peers = warp_peers(b, valid, nbits);
        const uint32_t before = __popc(peers & lanemask_lt());
        uint32_t base = 0;
        if (valid) base = myc16[b];
        __syncwarp();
        bk[i] = valid ? b : 0xFFFFu;
        lr[i] = base + before;
        if (valid && before == 0) myc16[b] = (uint16_t)(base + __popc(peers));
        __syncwarp();
      }
      } else {
        // more destinations: the rank atomics of any digit — G destinations
        // put ~32 / G lanes of a warp instruction on one counter, which the
        // B200 serves at full rate up to ~5 lanes per address
        // (tools/mb_atoms.cu), while the ballot peer masks cost 1.3 warp
        // instructions per record (10^9 records, G = 8: 9.7 -> 8.2 ms, G = 64:
        // 19.6 -> 16.7; G = 2: 7.8 -> 9.1, hence the ballots above)
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t e = warp * WS + i * 32 + lane;
          bk[i] = 0xFFFFu;
          if (e < tn) rank_one(i, SR(sk[e], global_base + g0 + e));
          __syncwarp();
        }
      }
    } else {
      const Router<K> R = make_router<K>(P, hz, hk);
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        bk[i] = 0xFFFFu;
        if (e < tn) rank_one(i, R(sk[e]));
        __syncwarp();
      }
    }
    __syncthreads();
    PH(3)

    // ---- bucket pair j = tid: prefix over warps, tile counts (published
    // for the later tiles of the block), exclusive scan over the tile ----
    uint32_t s = 0;
    if ((uint32_t)tid < npair) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t x = wh[w * HW + tid];
        wh[w * HW + tid] = s;
        s += x;
      }
      if (kt + 1 < LB) st_volatile(status + (uint64_t)t * nbs + tid, s | ST_VALID);
    }
    const uint32_t ptot = (s & 0xffffu) + (s >> 16);
    uint32_t incl = ptot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wt[warp] = incl;
    __syncthreads();
    PH(4)
    {
      uint32_t wp = lane < NW ? s_wt[lane] : 0u;
#pragma unroll
      for (int o = 1; o < NW; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, wp, o);
        if (lane >= o) wp += y;
      }
      const uint32_t wex = __shfl_sync(FULL, wp, (warp + 31) & 31);
      const uint32_t ex = (warp ? wex : 0u) + incl - ptot;
      if ((uint32_t)tid < npair) {
        tst[2 * tid] = ex;
        tst[2 * tid + 1] = ex + (s & 0xffffu);
      }
    }
    __syncthreads();
    PH(5)

    // ---- placement (regroup by bucket in SMEM) ----
    if (full) {
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t b = bk[i];
        const uint32_t pre = (mywh[b >> 1] >> ((b & 1u) << 4)) & 0xffffu;
        pk[tst[b] + pre + lr[i]] = (b << 16) | (warp * WS + i * 32 + lane);
      }
    } else {
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        if (bk[i] != 0xFFFFu) {
          const uint32_t b = bk[i];
          const uint32_t pre = (mywh[b >> 1] >> ((b & 1u) << 4)) & 0xffffu;
          pk[tst[b] + pre + lr[i]] = (b << 16) | (warp * WS + i * 32 + lane);
        }
      }
    }
    // each warp read only its own counters above: reset them for the next tile
    __syncwarp();
    for (uint32_t i = lane; i < HW; i += 32) mywh[i] = 0u;
    PH(6)
    // next tile: geometry + plan into the other slot, data into L2
    if (warp == 1 && t + gridDim.x < ntile) {
      resolve(t + gridDim.x, cur ^ 1);
      if (lane == 0) {
        const TileGeo& N = sgeo[cur ^ 1];
        uint32_t o2, h2, b2;
        const uint32_t kb2 = tile_body<K>(kin, N.g0, N.tn, o2, h2, b2);
        if (kb2) prefetch_l2(kin + N.g0 + h2, kb2);
        if (VB) {
          const uint32_t vb2 = tile_body<V>(vin, N.g0, N.tn, o2, h2, b2);
          if (vb2) prefetch_l2(vin + N.g0 + h2, vb2);
        }
      }
    }

    // ---- bucket bases of pair j: block offsets + earlier tiles of the
    // block (look-back over <= LB-1 status words, read in parallel) ----
    if ((uint32_t)tid < npair) {
      const uint32_t* st0 = status + (uint64_t)(t - kt) * nbs + tid;
      uint32_t v[LB - 1];
#pragma unroll
      for (int j = 0; j < LB - 1; ++j)
        if ((uint32_t)j < kt) v[j] = ld_volatile(st0 + (uint64_t)j * nbs);
      uint32_t ex = 0;
#pragma unroll
      for (int j = 0; j < LB - 1; ++j) {
        if ((uint32_t)j < kt) {
          while (!(v[j] & ST_VALID)) {
            PH_SPIN
            __nanosleep(64);
            v[j] = ld_volatile(st0 + (uint64_t)j * nbs);
          }
          ex += v[j] & ST_MASK;
        }
      }
      const uint32_t sb = (uint32_t)P.scanbase;
      db[2 * tid] = (uint32_t)bo0 - sb + (ex & 0xffffu) - tst[2 * tid];
      db[2 * tid + 1] = (uint32_t)bo1 - sb + (ex >> 16) - tst[2 * tid + 1];
    }
    PH(7)
    __syncthreads();
    PH(8)

    // ---- write the bucket runs; the stable order check is fused: within a
    // bucket, adjacent records must ascend in tile position.  If a pair does
    // not, the bucket runs are re-sorted and the tile is written again (same
    // addresses, corrected values). ----
    // segment base pointers kept opaque so each store address is one
    // IMAD.WIDE.U32 of the u32 position (no 64-bit re-association); st_global
    // keeps the stores in the global space
    K* ko_seg = opaque_ptr(kout + P.offset);
    V* vo_seg = VB ? opaque_ptr(vout + P.offset) : nullptr;
    bool bad = false;
    if (full) {
#pragma unroll
      for (int it = 0; it < IPT; ++it) {
        const uint32_t p = it * NT + tid;
        const uint32_t wd = pk[p], nx = pk[p + 1];
        bad |= ((wd ^ nx) < 65536u) & (nx < wd);
        const uint32_t e = wd & 0xffffu;
        const uint32_t d = db[wd >> 16] + p;
        st_global(ko_seg + d, sk[e]);
        if (VB) st_global(vo_seg + d, sv[e]);
      }
    } else {
#pragma unroll
      for (int it = 0; it < IPT; ++it) {
        const uint32_t p = it * NT + tid;
        if (p < tn) {
          const uint32_t wd = pk[p], nx = pk[p + 1];
          bad |= ((wd ^ nx) < 65536u) & (nx < wd);
          const uint32_t e = wd & 0xffffu;
          const uint32_t d = db[wd >> 16] + p;
          st_global(ko_seg + d, sk[e]);
          if (VB) st_global(vo_seg + d, sv[e]);
        }
      }
    }
    if (__any_sync(FULL, bad) && lane == 0) s_fix = 1u;
    __syncthreads();
    PH(9)
    if (s_fix || DTS_FORCE_FIXUP) {
#if DTS_PHASE_PROF
      if (tid == 0 && s_fix) atomicAdd(&g_phase[12], 1ull);
#endif
      for (uint32_t p = tid; p < tn; p += NT) {
        const uint32_t x = pk[p];
        const bool leader = p == 0 || ((pk[p - 1] ^ x) >= 65536u);
        if (leader && p + 1 < tn && ((pk[p + 1] ^ x) < 65536u)) {
          uint32_t c = 2;
          while (p + c < tn && ((pk[p + c] ^ x) < 65536u)) ++c;
          small_isort(pk + p, c);
        }
      }
      __syncthreads();
      for (uint32_t p = tid; p < tn; p += NT) {
        const uint32_t wd = pk[p];
        const uint32_t bb = wd >> 16, e = wd & 0xffffu;
        const uint32_t d = db[bb] + p;
        ko_seg[d] = sk[e];
        if (VB) vo_seg[d] = sv[e];
      }
      __syncthreads();
      if (tid == 0) s_fix = 0u;
    }
  }
  PH_DONE
}

}  // namespace dts
