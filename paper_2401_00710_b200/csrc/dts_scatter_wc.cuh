// dts_scatter_wc.cuh — k_scatter_wc, the write-combining stable distribution
// pass (counting.py:141-151 scatter phase, _kernels.py:12-25 scatter_block).
//
// Why: on B200 the cost of a scattered store is set by the number of L2
// write requests and by partially written 32-byte sectors (those force a
// DRAM read-modify-write).  tools/mb_mem.cu measured, for 16 B/record of
// traffic: runs of ~9 records written in place 1.2 TB/s, whole 32-byte
// sectors 2.4 TB/s, whole 64-byte chunks 4.1-4.4 TB/s, 128-byte lines
// 4.6-5.3 TB/s.  So every bucket's output is assembled in SMEM and leaves the
// SM only as whole, aligned C-record chunks (64 or 128 bytes).
//
// Structure: one CTA per SM walks whole stripes (= count-matrix rows, many
// tiles) in input order, so a bucket's records of consecutive tiles are
// contiguous in its output region and the CTA can carry each bucket's
// unfinished chunk (< C records) from tile to tile in SMEM.  Only the first
// and last chunk of each (stripe, bucket) region may be partial.  No
// look-back, no per-tile status.
#pragma once
#include "dts_scatter.cuh"

namespace dts {

// (key, value) pair of one staging slot when both have the same width: one
// 8/16-byte SMEM access per record instead of two (AoS staging)
template <typename K> struct StPair;
template <> struct StPair<uint32_t> {
  using T = uint2;
  __device__ static T make(uint32_t k, uint32_t v) { return make_uint2(k, v); }
};
template <> struct StPair<unsigned long> {
  using T = ulonglong2;
  __device__ static T make(unsigned long k, unsigned long v) { return make_ulonglong2(k, v); }
};
template <> struct StPair<unsigned long long> {
  using T = ulonglong2;
  __device__ static T make(unsigned long long k, unsigned long long v) { return make_ulonglong2(k, v); }
};

// WIDE = 1: the variant for waves with heavy keys (2^9 zones + up to 43
// heavy keys + overflow = 600 bucket columns: the carries and per-warp
// counters grow by 80 columns): it ranks heavy segments from the bucket ids
// k_histogram kept and writes long runs' chunk descriptors with the whole CTA
template <typename K, int VB, int WIDE = 0> struct WcTile {
  // 512 threads: 768 (16.4 ms) and 1024 measured slower on C2 — the
  // per-bucket phases lengthen with the warp count
  static constexpr int NT = 512;
  static constexpr int NW = NT / 32;
  static constexpr int PT = 1;  // threads per bucket pair in the pair phases
  static constexpr bool PAIR8 = sizeof(K) == 8 && VB == 8;
#ifndef DTS_WC_IPT4
#define DTS_WC_IPT4 18
#endif
#ifndef DTS_WC_IPT8
#define DTS_WC_IPT8 10
#endif
  // records per thread: the tile is as large as the registers allow (the
  // records wait in registers from their loads to the placement); SMEM holds
  // one staging buffer, so the wide variant keeps the same tile
  static constexpr int IPT = (sizeof(K) == 4 && VB <= 4) ? DTS_WC_IPT4 : DTS_WC_IPT8;
  static constexpr int WS = 32 * IPT;
  static constexpr int T = NT * IPT;
  static constexpr int NBW = WIDE ? 600 : 520;  // bucket capacity (2^9 light + 2 per heavy key + overflow)
  static constexpr int C = (sizeof(K) == 8 || VB == 8) ? 8 : 16;  // chunk records (64 B)
  static constexpr int CP = C;  // carry stride (unpadded: the two half-warp runs of a carry step conflict at most 2-way)
  static constexpr int MAXCH = (T + (C - 1) * NBW) / C + 2;       // chunks per tile bound
  static constexpr int HKC = 256;
  static constexpr int HZC = 520;
};

template <typename K, int VB, int WIDE = 0> struct WcSmem {
  using TL = WcTile<K, VB, WIDE>;
  static constexpr size_t kb = a16((size_t)TL::T * sizeof(K));
  static constexpr size_t vb = a16((size_t)TL::T * VB);
  static constexpr size_t buf = 0;                                   // staging (keys | vals)
  static constexpr size_t pk = a16(buf + kb + vb);                   // staging: tile position (u16)
  static constexpr size_t be = a16(pk + (size_t)(TL::T + 2) * 2);    // staging: bucket-run end bits
  static constexpr size_t ck = a16(be + (size_t)(TL::T / 32 + 2) * 4);  // carry keys
  static constexpr size_t cv = a16(ck + (size_t)TL::NBW * TL::CP * sizeof(K));
  static constexpr size_t wh = a16(cv + (size_t)TL::NBW * TL::CP * VB);  // per-warp counters
  // per chunk of the tile: {dest of slot 0, staging index of slot 0,
  // carry slots | hole << 8, bucket}
  static constexpr size_t cd = a16(wh + (size_t)TL::NW * (TL::NBW / 2) * 4);
  static constexpr size_t nf = a16(cd + (size_t)TL::MAXCH * 8);        // carry copy descriptors
  static constexpr size_t cst = a16(nf + (size_t)TL::NBW * 4);         // carry state
  static constexpr size_t hk = a16(cst + (size_t)(TL::NBW + 1) * 8);
  static constexpr size_t hz = a16(hk + (size_t)TL::HKC * sizeof(K));
  static constexpr size_t plan = a16(hz + (size_t)TL::HZC * 4);
  static constexpr size_t total = a16(plan + sizeof(SegPlan));
};

// ---------------------------------------------------------------------------
// k_scatter_wc: persistent, one CTA per SM, stripes taken from an atomic
// counter in input order.  A tile's records come in by coalesced streaming
// loads straight into registers, issued right after the previous tile's
// placement (a TMA bulk prefetch pulls the tile into L2 one tile earlier);
// the one SMEM tile buffer is the staging area.  The kernel is bound by the
// SM's load/store pipe (SMEM wavefronts + the 32 B/clk store port,
// tools/mb_store.cu, tools/mb_mio.cu).  Per tile:
//   * ranks: route each key and take per-warp packed u16 counters (SMEM
//     atomicAdd-with-return, k_scatter's scheme; the lane order of one
//     instruction's same-address atomics is verified below — never seen
//     violated with one atomic per __syncwarp);
//   * per bucket pair: prefix over warps, tile counts, and one packed block
//     scan giving both the tile offsets (tst) and the chunk offsets (sfc) of
//     carry + run; the owner writes its chunks into the chunk -> bucket map;
//   * placement into the staging area in bucket order; the stable order is
//     checked over the whole staging (every adjacent pair of one bucket must
//     ascend in tile position) and repaired if ever needed;
//   * write-out of every complete chunk (carry slots first, then staging)
//     as aligned C-record chunks (64 bytes);
//   * each bucket's unfinished chunk moves to its carry slots.
// At the end of a stripe the carries are flushed.
// ---------------------------------------------------------------------------
template <typename K, int VB, int WIDE>
__global__ void __launch_bounds__(WcTile<K, VB, WIDE>::NT, 1)
    k_scatter_wc(const SegPlan* __restrict__ plans, const Blk* __restrict__ blks, uint32_t nblk,
                 uint32_t* __restrict__ ctr, const K* __restrict__ kin,
                 const typename ValOf<VB>::T* __restrict__ vin, K* __restrict__ kout,
                 typename ValOf<VB>::T* __restrict__ vout, const uint64_t* __restrict__ scan,
                 const K* __restrict__ heavy_pool, const uint32_t* __restrict__ hz_pool,
                 const uint16_t* __restrict__ bid) {
  using V = typename ValOf<VB>::T;
  using TL = WcTile<K, VB, WIDE>;
  using SL = WcSmem<K, VB, WIDE>;
  constexpr int NT = TL::NT, NW = TL::NW, IPT = TL::IPT, WS = TL::WS, T = TL::T, C = TL::C,
                CP = TL::CP;
  constexpr uint32_t HW = TL::NBW / 2;
  constexpr int PT = TL::PT, WPT = NW / PT;  // threads per bucket pair, warps per thread
  static_assert(HW * PT <= (uint32_t)NT, "PT threads per bucket pair");
  static_assert(T < 65536, "packed u16 counts");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint16_t* pk = reinterpret_cast<uint16_t*>(smem_raw + SL::pk);
  uint32_t* bend = reinterpret_cast<uint32_t*>(smem_raw + SL::be);  // bit p: slot p ends a bucket run
  K* ck = reinterpret_cast<K*>(smem_raw + SL::ck);
  V* cv = reinterpret_cast<V*>(smem_raw + SL::cv);
  uint32_t* wh = reinterpret_cast<uint32_t*>(smem_raw + SL::wh);
  // chunk descriptor: {dest of slot 0, staging index of slot 0 + 16 (14 bits)
  // | carry slots << 14 | hole << 18 | bucket << 22}
  uint2* cdesc = reinterpret_cast<uint2*>(smem_raw + SL::cd);
  static_assert(TL::T + 2 * C + 16 < (1 << 14) && TL::NBW <= 1024 && C <= 16, "packed chunk descriptors");
  uint32_t* bnf = reinterpret_cast<uint32_t*>(smem_raw + SL::nf);  // copy: src | dst<<16 | cnt<<24
  uint2* cst = reinterpret_cast<uint2*>(smem_raw + SL::cst);      // {fill | hole << 16, chunk base}
  K* hk = reinterpret_cast<K*>(smem_raw + SL::hk);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + SL::hz);
  SegPlan* splan = reinterpret_cast<SegPlan*>(smem_raw + SL::plan);
  K* const xk = reinterpret_cast<K*>(smem_raw + SL::buf);            // staging keys (or AoS pairs)
  V* const xv = reinterpret_cast<V*>(smem_raw + SL::buf + SL::kb);   // staging values
  __shared__ uint32_t s_blk, s_fix, s_seg;
  __shared__ uint32_t s_wt[NW];
  __shared__ Blk s_B;
  // WIDE (waves with heavy keys): a bucket with many complete chunks in a
  // tile — a heavy key's — has its descriptors written by the whole CTA (one
  // thread per chunk) after the pair phase, not by the pair's owner in a
  // serial loop (Zipf 1.5: scatter 11.1 -> 10.3 ms).  Not in the plain
  // variant: the extra code cost C2 2 %.
  constexpr bool COOP = WIDE != 0;
  constexpr uint32_t COOP_MIN = 16, COOP_CAP = COOP ? T / ((COOP_MIN - 1) * C) + 2 : 1;  // (> COOP_MIN chunks hold > (COOP_MIN - 1) * C records)
  __shared__ uint32_t s_nlong;
  __shared__ uint32_t s_long[COOP_CAP][5];  // {first chunk, chunks, dest, staging index | bucket, first-chunk bits}
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* mywh = wh + warp * HW;
  // key and value of the same width: staging slots and carry slots are
  // (key, value) pairs (AoS), one SMEM access per record
  constexpr bool AOS = VB == (int)sizeof(K);
  using PairT = typename StPair<K>::T;

  if (tid == 0) {
    s_fix = 0u;
    s_seg = 0xFFFFFFFFu;
    s_nlong = 0u;
  }
  for (uint32_t i = tid; i < NW * HW; i += NT) wh[i] = 0u;
  [[maybe_unused]] constexpr bool ph_on = DTS_PHASE_PROF == 1;
  PH_INIT

  for (;;) {
    __syncthreads();
    PH(7)
    if (tid == 0) s_blk = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t bi = s_blk;
    if (bi >= nblk) break;
    if (tid == 0) s_B = blks[bi];
    if (warp == 1) {
      const uint32_t seg = blks[bi].seg;
      constexpr int PW = sizeof(SegPlan) / 4;
      if (lane < PW)
        reinterpret_cast<uint32_t*>(splan)[lane] = reinterpret_cast<const uint32_t*>(&plans[seg])[lane];
    }
    __syncthreads();
    const Blk B = s_B;
    const SegPlan& P = *splan;
    const uint32_t nb = P.nb, npair = (nb + 1) >> 1;
    if (B.seg != s_seg && (P.flags & PF_HEAVY)) {
      // zone table and heavy keys of the segment (sampler.py:76-100)
      pack_zone_table(hz_pool + P.hz_base, 1u << P.gamma, hz);
      for (uint32_t i = tid; i < P.nheavy && i < (uint32_t)TL::HKC; i += NT) hk[i] = heavy_pool[P.heavy_base + i];
    }
    // per bucket: block offset -> chunk base, hole = fill (carry state kept
    // in cst = {fill | hole << 16, chunk base}: read by each bucket pair's
    // owner in the pair phase, rewritten by it after the next barrier)
    // chunks are aligned to the key array's absolute 64-byte boundaries (a
    // segment may start anywhere): offsets count from the aligned base
    // kout + offset - al, whose first `al` slots the hole logic never writes
    const uint32_t al = (uint32_t)((reinterpret_cast<uintptr_t>(kout + P.offset) / sizeof(K)) & (C - 1));
    for (uint32_t b = tid; b < nb; b += NT) {
      const uint32_t o = (uint32_t)(scan[P.cnt_base + (uint64_t)b * P.nrows + B.row] - P.scanbase) + al;
      const uint32_t h = o & (uint32_t)(C - 1);
      cst[b] = make_uint2(h | (h << 16), o & ~(uint32_t)(C - 1));
    }
    K* ko_seg = opaque_ptr(kout + P.offset - al);
    V* vo_seg = VB ? opaque_ptr(vout + P.offset - al) : nullptr;
    const uint64_t len = B.end - B.begin;
    const uint32_t ntl = (uint32_t)((len + T - 1) / T);
    auto tile_n = [&](uint32_t kt) {
      const uint64_t r = len - (uint64_t)kt * T;
      return (uint32_t)(r < (uint64_t)T ? r : (uint64_t)T);
    };
    // ---- records of a tile: global -> registers by coalesced streaming
    // loads (warp instruction i of warp w covers tile positions
    // w*WS + i*32 + lane), issued one phase ahead — right after the previous
    // tile's placement, so they land behind its write-out and carries; a
    // TMA bulk prefetch pulls the tile into L2 one tile earlier.  The tile
    // never passes through SMEM on its way in (the load/store pipe is the
    // bound: no TMA write + LDS per record), and the one SMEM tile buffer is
    // the staging area.
    K key[IPT];
    V val[IPT];
    // WIDE (waves with heavy keys): the bucket ids k_histogram kept for a
    // heavy segment come in with the records — no routing in the rank phase
    // (the router's two dependent SMEM loads per record made it 4x C2's)
    [[maybe_unused]] uint32_t pb[WIDE ? IPT : 1];
    const bool use_bid = WIDE != 0 && bid != nullptr && (P.flags & PF_HEAVY) != 0;
    auto load_tile = [&](uint32_t kt) {
      const uint32_t tn = tile_n(kt);
      const K* gk = kin + B.begin + (uint64_t)kt * T + warp * WS + lane;
      const V* gv = VB ? vin + B.begin + (uint64_t)kt * T + warp * WS + lane : nullptr;
      if (tn == (uint32_t)T) {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          key[i] = __ldcs(gk + i * 32);
          if (VB) val[i] = __ldcs(gv + i * 32);
        }
      } else {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          if ((uint32_t)(warp * WS + i * 32 + lane) < tn) {
            key[i] = __ldcs(gk + i * 32);
            if (VB) val[i] = __ldcs(gv + i * 32);
          }
        }
      }
      if constexpr (WIDE != 0) {
        if (use_bid) {
          const uint16_t* gb = bid + B.begin + (uint64_t)kt * T + warp * WS + lane;
#pragma unroll
          for (int i = 0; i < IPT; ++i)
            if ((uint32_t)(warp * WS + i * 32 + lane) < tn) pb[i] = __ldcs(gb + i * 32);
        }
      }
    };
    auto prefetch_tile = [&](uint32_t kt) {  // (one thread)
      const char* src;
      uint32_t off;
      const uint64_t g0 = B.begin + (uint64_t)kt * T;
      const uint32_t kbytes = tile_span<K>(kin, g0, tile_n(kt), src, off);
      prefetch_l2(src, kbytes);
      if (VB) {
        const uint32_t vbytes = tile_span<V>(vin, g0, tile_n(kt), src, off);
        prefetch_l2(src, vbytes);
      }
    };
    PH(9)
    if (ntl) load_tile(0);
    if (tid == 0 && ntl > 1) prefetch_tile(1);
    __syncthreads();
    if (tid == 0) s_seg = B.seg;

    for (uint32_t kt = 0; kt < ntl; ++kt) {
      PH(0)
      const uint32_t tn = tile_n(kt);
      const bool full = tn == (uint32_t)T;
      if (tid == 0 && kt + 2 < ntl) prefetch_tile(kt + 2);
      // staging slot accessors (AoS pairs when key and value widths match;
      // the pair array spans this tile's key+value buffer)
      auto st_put = [&](uint32_t p, K k, V v) {
        if constexpr (AOS) {
          reinterpret_cast<typename StPair<K>::T*>(xk)[p] = StPair<K>::make(k, (K)v);
        } else {
          xk[p] = k;
          if (VB) xv[p] = v;
        }
      };
      auto st_get = [&](uint32_t p, K& k, V& v) {
        if constexpr (AOS) {
          const auto q = reinterpret_cast<const typename StPair<K>::T*>(xk)[p];
          k = q.x;
          v = (V)q.y;
        } else {
          k = xk[p];
          if (VB) v = xv[p];
        }
      };

      // (run-end bits of this tile: set in the pair phase below; the last
      // reads of the previous tile's were before its write-out barrier)
      for (uint32_t i = tid; i < (uint32_t)(T / 32 + 2); i += NT) bend[i] = 0u;
      // ---- route + per-warp rank ----
      // 2 * bucket << 16 | rank within the warp's bucket run (the high half is
      // the byte offset of the bucket's u16 counter in the warp's row)
      uint32_t bk[IPT];
      auto rank_one = [&](int i, uint32_t b) {
        const uint32_t sh = (b & 1u) << 4;
        const uint32_t old = atomicAdd(&mywh[b >> 1], 1u << sh);
        bk[i] = (b << 17) | ((old >> sh) & 0xffffu);
      };
      if (full && !(P.flags & PF_HEAVY)) {
        const uint32_t shift = P.shift, mask = (1u << P.gamma) - 1u;
        const bool ovf = (P.flags & PF_OVF) != 0;
        const K thr = ovf ? P.ovf_thr : ~K(0);
        const uint32_t ovfb = ovf ? nb - 1 : ((uint32_t)(~K(0) >> shift) & mask);
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          rank_one(i, key[i] >= thr ? ovfb : ((uint32_t)(key[i] >> shift) & mask));
          __syncwarp();
        }
      } else {
        const Router<K> R = make_router<K>(P, hz, hk);
        if (WIDE != 0 && use_bid) {
#pragma unroll
          for (int i = 0; i < IPT; ++i) {
            const uint32_t e = warp * WS + i * 32 + lane;
            bk[i] = 0xFFFFFFFFu;
            if (e < tn) rank_one(i, pb[WIDE ? i : 0]);
            __syncwarp();
          }
        } else {
#pragma unroll
          for (int i = 0; i < IPT; ++i) {
            const uint32_t e = warp * WS + i * 32 + lane;
            bk[i] = 0xFFFFFFFFu;
            if (e < tn) rank_one(i, R(key[i]));
            __syncwarp();
          }
        }
      }
      __syncthreads();
      PH(2)

      // ---- bucket pair j = tid: prefix over warps; packed scan of
      // (tile count | complete chunks of carry + run) ----
      uint32_t s = 0, n0 = 0, n1 = 0, f0 = 0, f1 = 0;
      uint2 I0 = make_uint2(0, 0), I1 = make_uint2(0, 0);
      const uint2* cin = cst;
      const uint32_t pj = tid / PT, pq = tid % PT;  // bucket pair, part of it
      const bool own = pj < npair;
      if (own) {
        I0 = cin[2 * pj];
        if (2 * pj + 1 < nb) I1 = cin[2 * pj + 1];
#pragma unroll
        for (int w = pq * WPT; w < (int)(pq + 1) * WPT; ++w) {
          const uint32_t x = wh[w * HW + pj];
          wh[w * HW + pj] = s;
          s += x;
        }
      }
      // combine the PT parts of a pair (adjacent lanes)
      uint32_t pex = s, tot = s;
      if (PT > 1) {
#pragma unroll
        for (int o = 1; o < PT; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, pex, o);
          if ((int)pq >= o) pex += y;
        }
        tot = __shfl_sync(FULL, pex, (lane | (PT - 1)));
        pex -= s;  // exclusive over the parts
      } else {
        pex = 0u;
      }
      if (own) {
        n0 = tot & 0xffffu;
        n1 = tot >> 16;
        f0 = ((I0.x & 0xffffu) + n0) / C;
        f1 = ((I1.x & 0xffffu) + n1) / C;
      }
      const uint32_t pv = (own && pq == PT - 1) ? ((n0 + n1) | ((f0 + f1) << 16)) : 0u;
      uint32_t incl = pv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wt[warp] = incl;
      __syncthreads();
      PH(3)
      uint32_t nch;
      {
        uint32_t wp = lane < NW ? s_wt[lane] : 0u;
#pragma unroll
        for (int o = 1; o < NW; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, wp, o);
          if (lane >= o) wp += y;
        }
        const uint32_t wex = __shfl_sync(FULL, wp, (warp + 31) & 31);
        nch = __shfl_sync(FULL, wp, NW - 1) >> 16;  // chunks of the whole tile
        const uint32_t ex = (warp ? wex : 0u) + incl - pv;
        if (own) {
          const uint32_t t0 = ex & 0xffffu, c0 = ex >> 16;
          // next carry state and the copy that produces it
          uint2* cout = cst;
          auto next = [&](uint32_t b, uint2 I, uint32_t n, uint32_t f, uint32_t t) {
            const uint32_t cc = I.x & 0xffffu;
            if (f == 0) {
              bnf[b] = t | (cc << 16) | (n << 24);
              cout[b] = make_uint2(I.x + n, I.y);
            } else {
              const uint32_t cnt = cc + n - f * C;
              bnf[b] = (t + f * C - cc) | (cnt << 24);
              cout[b] = make_uint2(cnt, I.y + f * C);
            }
          };
          // descriptors of this pair's complete chunks
          auto chunks = [&](uint32_t b, uint2 I, uint32_t f, uint32_t t, uint32_t g0) {
            const uint32_t cc = I.x & 0xffffu, ch = I.x >> 16;
            if (COOP && f > COOP_MIN) {
              const uint32_t at = atomicAdd(&s_nlong, 1u);
              s_long[at][0] = g0;
              s_long[at][1] = f;
              s_long[at][2] = I.y;
              s_long[at][3] = (t - cc + 16u) | (b << 22);
              s_long[at][4] = (cc << 14) | (ch << 18);
              return;
            }
            for (uint32_t k = 0; k < f; ++k)
              cdesc[g0 + k] = make_uint2(I.y + k * C, (t - cc + k * C + 16u) | (k ? 0u : ((cc << 14) | (ch << 18))) | (b << 22));
          };
          // the last staging slot of a bucket run (order check, repair)
          auto mark_end = [&](uint32_t e) { atomicOr(&bend[e >> 5], 1u << (e & 31)); };
          if (pq == 0) {
            next(2 * pj, I0, n0, f0, t0);
            chunks(2 * pj, I0, f0, t0, c0);
            if (n0) mark_end(t0 + n0 - 1);
          }
          if (pq == PT - 1 && 2 * pj + 1 < nb) {
            next(2 * pj + 1, I1, n1, f1, t0 + n0);
            chunks(2 * pj + 1, I1, f1, t0 + n0, c0 + f0);
            if (n1) mark_end(t0 + n0 + n1 - 1);
          }
          // fold the tile offsets (and the earlier parts' counts) into this
          // part's per-warp prefixes
          const uint32_t add = (t0 | ((t0 + n0) << 16)) + pex;
          uint32_t hv[WPT];
#pragma unroll
          for (int w = 0; w < WPT; ++w) hv[w] = wh[(pq * WPT + w) * HW + pj];
#pragma unroll
          for (int w = 0; w < WPT; ++w) wh[(pq * WPT + w) * HW + pj] = hv[w] + add;
        }
      }
      __syncthreads();
      PH(4)
      if constexpr (COOP) {
        const uint32_t nl = s_nlong;
        for (uint32_t e = 0; e < nl; ++e) {
          const uint32_t g0 = s_long[e][0], f = s_long[e][1], dst = s_long[e][2], sb = s_long[e][3],
                         fb = s_long[e][4];
          for (uint32_t k = tid; k < f; k += NT)
            cdesc[g0 + k] = make_uint2(dst + k * C, (sb + k * C) | (k ? 0u : fb));
        }
      }

      // ---- placement into the staging area (this tile's buffer) ----
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        if (full || bk[i] != 0xFFFFFFFFu) {
          // (the packed pair words read as a u16 array: bucket b's prefix is
          // element b — one LDS.U16 at the byte offset kept in bk)
          const uint32_t p = (uint32_t)*reinterpret_cast<const uint16_t*>(
                                 reinterpret_cast<const unsigned char*>(mywh) + (bk[i] >> 16)) +
                             (bk[i] & 0xffffu);
          st_put(p, key[i], VB ? val[i] : V(0));
          pk[p] = (uint16_t)(warp * WS + i * 32 + lane);
        }
      }
      __syncwarp();
      for (uint32_t i = lane; i < HW; i += 32) mywh[i] = 0u;
      __syncthreads();
      PH(5)
      if (COOP && tid == 0) s_nlong = 0u;
      // the records sit in the staging area: the next tile's loads start now
      if (kt + 1 < ntl) load_tile(kt + 1);

      // ---- stable order check (within a bucket, tile positions ascend) and
      // write-out of every complete chunk: slot r of bucket b's current chunk
      // run (carry slots [0, cc) first, then the staging run) ----
      auto write_chunks = [&]() {
        const uint32_t nslot = nch * C;
        const uint32_t stoff = (uint32_t)SL::buf;  // staging pairs
        if constexpr (AOS) {
          // (the SM's load/store pipe is the kernel's bound — SMEM wavefronts
          // plus the 32 B/clk store port, tools/mb_store.cu, tools/mb_mio.cu —
          // so conflict-free reads beat the fewer instructions of two adjacent
          // slots per thread, whose LDS.64 pairs are 4-way conflicted)
          // one slot per lane, two independent slots (q, q + 32) per thread:
          // a warp's LDS.64 covers 32 consecutive pairs (no bank conflicts),
          // keys and values leave as two 128-byte rows each
          for (uint32_t q0 = 64 * (tid >> 5) + (tid & 31); q0 < nslot; q0 += 2 * NT) {
            uint2 D[2];
            uint32_t off[2], d[2];
            bool on[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t q = q0 + 32 * u;
              D[u] = cdesc[(q < nslot ? q : q0) / C];
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const uint32_t q = q0 + 32 * u;
              const uint32_t r = q % C;
              const uint32_t hole = (D[u].y >> 18) & 15u, cc = (D[u].y >> 14) & 15u;
              on[u] = q < nslot && r >= hole;
              const uint32_t cbase = (uint32_t)SL::ck + (D[u].y >> 22) * CP * (uint32_t)sizeof(PairT);
              const uint32_t sbase = stoff + ((D[u].y & 0x3FFFu) - 16u) * (uint32_t)sizeof(PairT);
              off[u] = (r < cc ? cbase : sbase) + r * (uint32_t)sizeof(PairT);
              d[u] = D[u].x + r;
            }
            PairT pr[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) pr[u] = *reinterpret_cast<const PairT*>(smem_raw + off[u]);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (on[u]) {
                st_global(ko_seg + d[u], (K)pr[u].x);
                st_global(vo_seg + d[u], (V)pr[u].y);
              }
            }
          }
          return;
        }
        for (uint32_t q = tid; q < nslot; q += NT) {
          const uint2 D = cdesc[q / C];
          const uint32_t r = q % C;
          if (r < ((D.y >> 18) & 15u)) continue;  // hole: the previous stripe's records
          K kk;
          V vv = V(0);
          if constexpr (AOS) {
            // carry slot or staging slot: both are (key, value) pairs — one
            // select of the SMEM offset, one load, no divergent branch
            const uint32_t off = r < ((D.y >> 14) & 15u)
                                     ? (uint32_t)SL::ck + ((D.y >> 22) * CP + r) * (uint32_t)sizeof(PairT)
                                     : stoff + ((D.y & 0x3FFFu) - 16u + r) * (uint32_t)sizeof(PairT);
            const PairT pr = *reinterpret_cast<const PairT*>(smem_raw + off);
            kk = pr.x;
            vv = (V)pr.y;
          } else if (r < ((D.y >> 14) & 15u)) {
            const uint32_t b = D.y >> 22;
            kk = ck[b * CP + r];
            if (VB) vv = cv[b * CP + r];
          } else {
            st_get((D.y & 0x3FFFu) - 16u + r, kk, vv);
          }
          const uint32_t d = D.x + r;
          st_global(ko_seg + d, kk);
          if (VB) st_global(vo_seg + d, vv);
        }
      };
      {
        // 8 staging slots per thread: one 16-byte load of their tile
        // positions, packed u16 compares of every adjacent pair, masked by
        // the run-end bits (a pair across two bucket runs is not checked)
        uint32_t bad = 0u;
        const uint4* pk4 = reinterpret_cast<const uint4*>(pk);
        for (uint32_t q = tid; 8 * q + 1 < tn; q += NT) {
          const uint4 X = pk4[q];
          const uint32_t x8 = pk[8 * q + 8];  // (pk has T + 2 entries)
          const uint32_t S0 = __byte_perm(X.x, X.y, 0x5432), S1 = __byte_perm(X.y, X.z, 0x5432);
          const uint32_t S2 = __byte_perm(X.z, X.w, 0x5432), S3 = __byte_perm(X.w, x8, 0x5432);
          // byte j = 0xff when pair (8q+j, 8q+j+1) descends
          const uint32_t lo = __byte_perm(__vcmpltu2(S0, X.x), __vcmpltu2(S1, X.y), 0x6420);
          const uint32_t hi = __byte_perm(__vcmpltu2(S2, X.z), __vcmpltu2(S3, X.w), 0x6420);
          // pairs inside one run and inside the tile: bit j of `in`
          const uint32_t p0 = 8 * q;
          const uint32_t lim = tn - 1 - p0;  // pairs j < lim are inside the tile
          uint32_t in = ~(bend[p0 >> 5] >> (p0 & 31)) & (lim >= 8 ? 0xffu : ((1u << lim) - 1u));
          const uint32_t inlo = ((in & 15u) * 0x00204081u) & 0x01010101u;
          const uint32_t inhi = (((in >> 4) & 15u) * 0x00204081u) & 0x01010101u;
          bad |= (lo & inlo) | (hi & inhi);
        }
        if (__any_sync(FULL, bad != 0u) && lane == 0) s_fix = 1u;
      }
      write_chunks();
      __syncthreads();
      PH(6)
      if (s_fix || DTS_FORCE_FIXUP) {
#if DTS_PHASE_PROF
        if (tid == 0 && s_fix) atomicAdd(&g_phase[13], 1ull);
#endif
        // re-sort each bucket run by tile position (insertion sort), then
        // write the chunks again (same addresses, corrected values)
        auto run_end = [&](uint32_t q) { return ((bend[q >> 5] >> (q & 31)) & 1u) != 0u; };
        for (uint32_t p = tid; p < tn; p += NT) {
          const bool leader = p == 0 || run_end(p - 1);
          if (leader && p + 1 < tn && !run_end(p)) {
            uint32_t c = 2;
            while (p + c < tn && !run_end(p + c - 1)) ++c;
            for (uint32_t a = 1; a < c; ++a) {
              const uint16_t xw = pk[p + a];
              K xk2;
              V xv2 = V(0);
              st_get(p + a, xk2, xv2);
              uint32_t b2 = a;
              while (b2 > 0 && pk[p + b2 - 1] > xw) {
                pk[p + b2] = pk[p + b2 - 1];
                K tk2;
                V tv2 = V(0);
                st_get(p + b2 - 1, tk2, tv2);
                st_put(p + b2, tk2, tv2);
                --b2;
              }
              pk[p + b2] = xw;
              st_put(p + b2, xk2, xv2);
            }
          }
        }
        __syncthreads();
        write_chunks();
        __syncthreads();
        if (tid == 0) s_fix = 0u;
      }

      // ---- unfinished chunks become the carries: C lanes per bucket, one
      // record each (32 / C buckets per warp step, 4 steps in flight) ----
      {
        constexpr uint32_t BPW = 32 / C;
        constexpr uint32_t U = 4;
        const uint32_t sub = lane / C, i = lane % C;
        for (uint32_t b0 = warp * BPW; b0 < nb; b0 += NW * BPW * U) {
          uint32_t dw[U];
#pragma unroll
          for (uint32_t u = 0; u < U; ++u) {
            const uint32_t b = b0 + u * NW * BPW + sub;
            dw[u] = b < nb ? bnf[b] : 0u;
          }
          if constexpr (AOS) {
            const PairT* sp = reinterpret_cast<const PairT*>(xk);
            PairT* cpr = reinterpret_cast<PairT*>(smem_raw + SL::ck);
            PairT tp[U];
#pragma unroll
            for (uint32_t u = 0; u < U; ++u)
              if (i < (dw[u] >> 24)) tp[u] = sp[(dw[u] & 0xffffu) + i];
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
              if (i < (dw[u] >> 24)) {
                const uint32_t b = b0 + u * NW * BPW + sub;
                cpr[b * CP + ((dw[u] >> 16) & 0xffu) + i] = tp[u];
              }
            }
          } else {
            K tk[U];
            V tv[U];
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
              if (i < (dw[u] >> 24)) {
                const uint32_t src = (dw[u] & 0xffffu) + i;
                st_get(src, tk[u], tv[u]);
              }
            }
#pragma unroll
            for (uint32_t u = 0; u < U; ++u) {
              if (i < (dw[u] >> 24)) {
                const uint32_t b = b0 + u * NW * BPW + sub;
                const uint32_t dst = b * CP + ((dw[u] >> 16) & 0xffu) + i;
                ck[dst] = tk[u];
                if (VB) cv[dst] = tv[u];
              }
            }
          }
        }
      }
      PH(8)
    }
    // ---- stripe end: flush the unfinished chunks (partial sectors) ----
    // (C lanes per bucket, one slot each: a warp store covers 32 / C
    // buckets' runs instead of 32 scattered records)
    __syncthreads();
    {
      constexpr uint32_t BPW = 32 / C;
      const uint32_t sub = lane / C, r = lane % C;
      for (uint32_t b0 = warp * BPW; b0 < nb; b0 += NW * BPW) {
        const uint32_t b = b0 + sub;
        if (b < nb) {
          const uint2 I = cst[b];
          if (r >= (I.x >> 16) && r < (I.x & 0xffffu)) {
            if constexpr (AOS) {
              const PairT pr = reinterpret_cast<const PairT*>(smem_raw + SL::ck)[b * CP + r];
              st_global(ko_seg + I.y + r, (K)pr.x);
              st_global(vo_seg + I.y + r, (V)pr.y);
            } else {
              st_global(ko_seg + I.y + r, ck[b * CP + r]);
              if (VB) st_global(vo_seg + I.y + r, cv[b * CP + r]);
            }
          }
        }
      }
    }
  }
  PH_DONE
}

}  // namespace dts
