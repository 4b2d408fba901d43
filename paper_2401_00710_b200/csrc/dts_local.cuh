// dts_local.cuh — k_local_sort, the base case (dtsort.py:127-147 _base_sort:
// stable sort by full key of a span of adjacent buckets, valid per :128-131).
#pragma once
#include "dts_scatter.cuh"

namespace dts {

#ifndef DTS_LOCAL_REGATOM
#define DTS_LOCAL_REGATOM 1  // register-sourced rank atomics (order verified on the output)
#endif

#ifndef DTS_OVN_LSD
#define DTS_OVN_LSD (1 << 30)  // wrapped 4-bit fields in one warp that send a span to LSD, not the retry
                               // (the retry's 16-bit fields cannot carry: every carrying span is queued)
#endif

template <int FB> struct FieldBits {
  static constexpr uint32_t value = FB;
};

template <typename K, int VB> struct LocalTile {
  // 8 warps: one 4-bit per-warp field per bin in a 32-bit bin word (the
  // stable counting path below); 2 CTAs per SM
  static constexpr int NT = 256;
  static constexpr int NW = NT / 32;
#ifndef DTS_LOCAL_IPT8
#define DTS_LOCAL_IPT8 18
#endif
  // 8-byte columns: ONE span buffer (the next span streams in once this one
  // has left; the SM's other CTA covers the wait), so a span holds as many
  // records as with 4-byte columns — with two buffers the capacity was 2560
  // records and every 64-bit config of BASELINE.json needed a third
  // distribution pass for buckets of ~3800 records
  static constexpr bool SINGLE = !(sizeof(K) == 4 && VB <= 4);
  static constexpr int IPT = SINGLE ? DTS_LOCAL_IPT8 : 18;
  static constexpr int WS = 32 * IPT;  // records per warp sub-tile
  static constexpr int CAP = NT * IPT; // records per span
  static constexpr int RB = 8;         // LSD radix bits per pass (fallback path)
  static constexpr int NB = 12;        // nibble counting path: spans differing in <= NB bits
  static constexpr int CB = 13;        // packed counting path: top CB differing bits
  static constexpr int FIXMAX = 64;    // packed counting path: largest equal-key group
  static_assert(NB == (int)LOCAL_NB, "k_classify's merge rule follows the counting path's width");
};

// Compile-time SMEM layout: two span buffers (TMA double buffering), the
// per-record index array, and the counter area (8192 packed u16 bins for the
// counting path; per-warp digit counters + digit totals for the LSD path).
template <typename K, int VB> struct LocalSmem {
  using TL = LocalTile<K, VB>;
  static constexpr size_t kcap = (size_t)(TL::CAP + 8) * sizeof(K);
  static constexpr size_t vcap = (size_t)(TL::CAP + 8) * VB;
  static constexpr size_t k0 = 0;
  static constexpr size_t v0 = a16(k0 + kcap);
  static constexpr size_t k1 = TL::SINGLE ? k0 : a16(v0 + vcap);
  static constexpr size_t v1 = TL::SINGLE ? v0 : a16(k1 + kcap);
  static constexpr size_t si = a16(v1 + vcap);
  static constexpr size_t cnt = a16(si + (size_t)TL::CAP * 4);
  static constexpr size_t cnt_bytes = ((size_t)1 << TL::CB) * 2;
  static constexpr size_t wc_bytes = (size_t)TL::NW * ((size_t)1 << (TL::RB - 1)) * 4;
  static_assert(wc_bytes + (((size_t)1 << TL::RB) + 1) * 4 <= cnt_bytes, "LSD counters alias cnt");
  static constexpr size_t bar = a16(cnt + cnt_bytes);
  static constexpr size_t total = a16(bar + 16);
};

struct SpanSlot {  // a span staged in one buffer
  uint64_t offset;
  uint32_t len, src, ko, vo;
};

// ---------------------------------------------------------------------------
// k_local_sort: persistent CTAs (2 per SM) take spans round-robin; while one
// span is sorted the next one is already streaming into the other SMEM
// buffer (one cp.async.bulk per column on its mbarrier).  Per span:
//   * the bits in which its keys differ (keys agree above `bits`);
//   * bits <= CB (the common case: last-level buckets): ONE counting pass on
//     the differing bits — those bits are the whole key order — SMEM-atomic
//     histogram, scan, atomic slots, then each equal-key group (<= FIXMAX
//     records, else the LSD path) is put back in input order (insertion sort
//     of record indices): stable without relying on any atomic ordering;
//   * otherwise stable LSD passes of <= RB bits with per-warp packed counters
//     (the k_scatter ranking; in-step order verified and repaired if needed).
// Output always lands in A.
// ---------------------------------------------------------------------------
template <typename K, int VB, bool RETRY = false>
__global__ void __launch_bounds__(LocalTile<K, VB>::NT, 2)
    k_local_sort(const Span* __restrict__ spans, const uint32_t* __restrict__ nspan_p, K* __restrict__ Ak,
                 typename ValOf<VB>::T* __restrict__ Av, const K* __restrict__ Tk,
                 const typename ValOf<VB>::T* __restrict__ Tv, Span* __restrict__ rq = nullptr,
                 uint32_t* __restrict__ rq_n = nullptr) {
  using V = typename ValOf<VB>::T;
  using TL = LocalTile<K, VB>;
  using SL = LocalSmem<K, VB>;
  constexpr int NT = TL::NT, NW = TL::NW, IPT = TL::IPT, WS = TL::WS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* si = reinterpret_cast<uint32_t*>(smem_raw + SL::si);
  uint16_t* si16 = reinterpret_cast<uint16_t*>(smem_raw + SL::si);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + SL::cnt);
  uint32_t* wc = cnt;
  uint32_t* dt = reinterpret_cast<uint32_t*>(smem_raw + SL::cnt + SL::wc_bytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + SL::bar);
  __shared__ SpanSlot s_slot[2];
  __shared__ uint32_t s_wt[NW + 1];
  __shared__ K s_diff[NW];
  __shared__ uint32_t s_fix, s_big, s_ovn;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // issue span `s` into buffer `b` (thread 0; the descriptor is in hand)
  auto issue = [&](const Span& S, int b) {
    const K* kc = (S.src & 1u) ? Tk : Ak;
    const V* vc = (S.src & 1u) ? Tv : Av;
    SpanSlot sl;
    sl.offset = S.offset;
    sl.len = S.len;
    sl.src = S.src;
    const char* ks;
    const uint32_t kbytes = S.len ? tile_span<K>(kc, S.offset, S.len, ks, sl.ko) : 0u;
    const char* vs = nullptr;
    uint32_t vbytes = 0;
    sl.vo = 0;
    if (VB && S.len) vbytes = tile_span<V>(vc, S.offset, S.len, vs, sl.vo);
    s_slot[b] = sl;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bar[b], kbytes + vbytes);
    if (kbytes) tma_load_1d(smem_raw + (b ? SL::k1 : SL::k0), ks, kbytes, &bar[b]);
    if (vbytes) tma_load_1d(smem_raw + (b ? SL::v1 : SL::v0), vs, vbytes, &bar[b]);
  };

  const uint32_t G = gridDim.x;
  const uint32_t nspan = *nspan_p;  // device-resident count (k_classify)
  // (one thread's) descriptor of the span after the one in flight: in SMEM —
  // a register copy costs every thread 4 registers of a kernel at its cap
  __shared__ __align__(16) Span s_next;
  // (fetched by cp.async: a plain load + store would stall the fetching warp
  // on the global latency in front of its rank atomics, and the block's next
  // barrier behind it)
  auto fetch_next = [&](const Span* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;" ::"r"(smem_u32(&s_next)), "l"(src) : "memory");
  };
  auto next_ready = [&]() { asm volatile("cp.async.wait_group 0;" ::: "memory"); };
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    s_fix = 0u;
    s_big = 0u;
    s_ovn = 0u;
  }
  __syncthreads();
  if (tid == NT - 1) {
    if (blockIdx.x < nspan) issue(spans[blockIdx.x], 0);
    if (blockIdx.x + G < nspan) fetch_next(spans + blockIdx.x + G);
  }
  for (uint32_t i = tid; i < (uint32_t)(SL::cnt_bytes / 4); i += NT) cnt[i] = 0u;
  __syncthreads();
  uint32_t ph0 = 0u, ph1 = 0u;
  int cur = 0;
  [[maybe_unused]] constexpr bool ph_on = DTS_PHASE_PROF == 2;
  PH_INIT
  for (uint32_t sidx = blockIdx.x; sidx < nspan; sidx += G, cur ^= 1) {
    PH(9)
    if (TL::SINGLE && sidx != blockIdx.x && tid == NT - 1) {
      // one buffer: every thread is past the previous span's last read (its
      // final barrier), the span's descriptor was fetched an iteration ago
      next_ready();
      issue(s_next, cur);
      if (sidx + G < nspan) fetch_next(spans + sidx + G);
    }
    if (cur == 0) {
      mbar_wait(&bar[0], ph0);
      ph0 ^= 1u;
    } else {
      mbar_wait(&bar[1], ph1);
      ph1 ^= 1u;
    }
    PH(0)
    const SpanSlot S = s_slot[cur];
    const uint32_t n = S.len;
    K* sk = reinterpret_cast<K*>(smem_raw + (cur ? SL::k1 : SL::k0)) + S.ko;
    V* sv = reinterpret_cast<V*>(smem_raw + (cur ? SL::v1 : SL::v0)) + S.vo;
    K* ok = Ak + S.offset;
    V* ov = VB ? Av + S.offset : nullptr;

    // ---- keys into registers (lane-striped warp sub-tiles), differing bits ----
    // (a span of one light bucket comes with its bound: the keys agree above
    // it, so the counting path starts without a reduction or a barrier;
    // otherwise the differing bits are reduced over the span)
    const K k0 = sk[0];
    K key[IPT];
    K diff = 0;
    const uint32_t bound = (S.src >> 8) & 255u;
    const bool known = bound <= (uint32_t)TL::NB;
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t e = warp * WS + i * 32 + lane;
      key[i] = e < n ? sk[e] : k0;
      diff |= key[i] ^ k0;
    }
    int bits = (int)bound;
    if (!known) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) diff |= __shfl_xor_sync(FULL, diff, o);
      if (lane == 0) s_diff[warp] = diff;
      __syncthreads();
    }
    PH(1)
    // stream the next span into the other buffer (freed by the previous
    // iteration's final barrier); fetch the descriptor after it
    if (TL::SINGLE && tid == NT - 1 && sidx + G < nspan) {
      // one buffer: the next span cannot stream into SMEM yet, but a TMA
      // bulk prefetch pulls it into L2 while this span is sorted
      next_ready();
      const Span N = s_next;
      if (N.len) {
        const char* src;
        uint32_t off;
        const uint32_t kbytes = tile_span<K>((N.src & 1u) ? Tk : Ak, N.offset, N.len, src, off);
        prefetch_l2(src, kbytes);
        if (VB) {
          const uint32_t vbytes = tile_span<V>((N.src & 1u) ? Tv : Av, N.offset, N.len, src, off);
          prefetch_l2(src, vbytes);
        }
      }
    }
    if (!TL::SINGLE && tid == NT - 1) {
      if (sidx + G < nspan) {
        next_ready();
        issue(s_next, cur ^ 1);
      }
      if (sidx + 2 * G < nspan) fetch_next(spans + sidx + 2 * G);
    }
    if (!known) {
      diff = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) diff |= s_diff[w];
      bits = 0;
      if (diff) bits = (sizeof(K) == 8) ? 64 - __clzll((long long)diff) : 32 - __clz((int)(uint32_t)diff);
    }

    if (bits == 0) {
#if DTS_PHASE_PROF == 2
      if (tid == 0) atomicAdd(&g_phase[15], 1ull);
#endif
      if (S.src & 1u) {
        for (uint32_t i = tid; i < n; i += NT) {
          ok[i] = sk[i];
          if (VB) ov[i] = sv[i];
        }
      }
      __syncthreads();
      continue;
    }

    bool lsd = false;
    // exclusive scan over packed u16 bin pairs cnt[0..nwd) (uint4 quads, a
    // contiguous range per thread); sets s_big when a bin exceeds FIXMAX
    auto scan_bins = [&](uint32_t nwd) {
      const uint32_t nq = (nwd + 3) >> 2, qpt = (nq + NT - 1) / NT;
      const uint32_t q0 = min(nq, tid * qpt), q1 = min(nq, q0 + qpt);
      uint4* cq = reinterpret_cast<uint4*>(cnt);
      uint32_t sum = 0, mx = 0;
      for (uint32_t q = q0; q < q1; ++q) {
        const uint4 x = cq[q];
        sum += (x.x & 0xffffu) + (x.x >> 16) + (x.y & 0xffffu) + (x.y >> 16) + (x.z & 0xffffu) +
               (x.z >> 16) + (x.w & 0xffffu) + (x.w >> 16);
        const uint32_t m2 = __vmaxu2(__vmaxu2(x.x, x.y), __vmaxu2(x.z, x.w));
        mx = max(mx, max(m2 & 0xffffu, m2 >> 16));
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
      if (lane == 31) s_wt[warp] = incl;
      if (lane == 0 && mx > (uint32_t)TL::FIXMAX) s_big = 1u;
      __syncthreads();
      PH(4)
      uint32_t wp = lane < NW ? s_wt[lane] : 0u;
#pragma unroll
      for (int o = 1; o < NW; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, wp, o);
        if (lane >= o) wp += y;
      }
      const uint32_t wex = __shfl_sync(FULL, wp, (warp + 31) & 31);
      uint32_t base = (warp ? wex : 0u) + incl - sum;
      auto ex = [&](uint32_t x) {
        const uint32_t lo = x & 0xffffu, r = base | ((base + lo) << 16);
        base += lo + (x >> 16);
        return r;
      };
      for (uint32_t q = q0; q < q1; ++q) {
        uint4 x = cq[q];
        x.x = ex(x.x);
        x.y = ex(x.y);
        x.z = ex(x.z);
        x.w = ex(x.w);
        cq[q] = x;
      }
      __syncthreads();
    };
    auto zero_bins = [&](uint32_t nwd) {
      const uint32_t nq = (nwd + 3) >> 2;
      for (uint32_t q = tid; q < nq; q += NT) reinterpret_cast<uint4*>(cnt)[q] = make_uint4(0u, 0u, 0u, 0u);
    };
    if (bits <= TL::NB) {
      // ================= field counting path: the differing bits are the
      // whole key order, so ONE stable counting pass sorts the span.  Bin
      // word d holds one FB-bit count per rank group — FB = 4: 8 groups, one
      // per warp; FB = 8 (the retry launch): 4 groups, one per warp pair
      // whose atomics run in two phases (even warps, then odd), so each
      // group's counts still follow record order.  A record's stable slot =
      // start(d) + records of d in earlier groups (from the final word) + its
      // own group's earlier records of d (the atomic's return; the
      // lane/instruction order of one warp's atomics is verified on the
      // output).  Slot words hold (bin << 16 | position): the key is rebuilt
      // from the bin, only the value is gathered.
      const uint32_t nbin = 1u << bits, mask = nbin - 1u, nq = (nbin + 3) >> 2;
      uint16_t* st16 = reinterpret_cast<uint16_t*>(smem_raw + (cur ? SL::k1 : SL::k0));  // bin starts
      auto counting = [&](auto fbc) -> bool {
        constexpr uint32_t FB = decltype(fbc)::value;
        constexpr uint32_t FM = (1u << FB) - 1u;
        constexpr int RPW = 32 / (int)FB;  // ranks per register word
        auto fsum = [](uint32_t x) -> uint32_t {  // sum of the word's fields
          if constexpr (FB == 4) {
            x = (x & 0x0F0F0F0Fu) + ((x >> 4) & 0x0F0F0F0Fu);
            return (x * 0x01010101u) >> 24;
          } else if constexpr (FB == 8) {
            return __dp4a(x, 0x01010101u, 0u);
          } else {
            return (x & 0xFFFFu) + (x >> 16);
          }
        };
        const uint32_t nib = FB == 4 ? 4u * (uint32_t)warp
                                     : (FB == 8 ? 8u * ((uint32_t)warp >> 1) : 16u * ((uint32_t)warp >> 2));
        uint32_t rkp[(IPT + RPW - 1) / RPW];  // own-group ranks, FB bits each
#pragma unroll
        for (int j = 0; j < (IPT + RPW - 1) / RPW; ++j) rkp[j] = 0u;
        bool ovf = false;
        // (the bins are zero here: zeroed at start and after every span)
        PH(2)
        auto atomics = [&]() {
#pragma unroll
          for (int i = 0; i < IPT; ++i) {
            const uint32_t e = warp * WS + i * 32 + lane;
            if (e < n) {
#if DTS_LOCAL_REGATOM
              const uint32_t d = (uint32_t)key[i] & mask;
#else
              const uint32_t d = (uint32_t)sk[e] & mask;  // key read right before its atomic
#endif
              const uint32_t r = (atomicAdd(&cnt[d], 1u << nib) >> nib) & FM;
              ovf |= r == FM;
              rkp[i / RPW] |= r << ((i % RPW) * FB);
            }
#if !DTS_LOCAL_REGATOM
            __syncwarp();
#endif
          }
        };
        if constexpr (FB == 4) {
          atomics();
        } else if constexpr (FB == 8) {
          if (!(warp & 1)) atomics();
          __syncthreads();
          if (warp & 1) atomics();
        } else {
          // 16-bit fields, 2 groups of 4 warps whose atomics run in 4 phases
          // (warp order inside a group): no field can carry (spans hold
          // < 2^16 records), so a span never needs the LSD passes
#pragma unroll 1
          for (int ph = 0; ph < 4; ++ph) {
            if ((warp & 3) == ph) atomics();
            if (ph < 3) __syncthreads();
          }
        }
        if (ovf) s_big = 1u;  // a field would carry
        __syncthreads();
        PH(3)
        if (s_big) {
          if constexpr (FB == 4) {
            // fields that wrapped in this warp (ranks of 15): many mean a
            // key too frequent for 8-bit fields as well -> LSD directly
            uint32_t ev = 0;
#pragma unroll
            for (int j = 0; j < (IPT + RPW - 1) / RPW; ++j) {
              const uint32_t x = rkp[j];
              ev += __popc(x & (x >> 1) & (x >> 2) & (x >> 3) & 0x11111111u);
            }
            ev = __reduce_add_sync(FULL, ev);
            if (lane == 0) atomicMax(&s_ovn, ev);
          }
          return false;
        }
        // exclusive scan of the bin totals (sum of the fields) -> st16
        {
          // (<= 2^NB bins: at most QPT quads of 4 bin words per thread, kept
          // in registers across the barrier)
          constexpr uint32_t QPT = ((1u << TL::NB) / 4 + NT - 1) / NT;
          const uint32_t qpt = (nq + NT - 1) / NT;
          const uint32_t q0 = min(nq, tid * qpt), q1 = min(nq, q0 + qpt);
          const uint4* cq = reinterpret_cast<const uint4*>(cnt);
          uint4 xq[QPT];
#pragma unroll
          for (uint32_t j = 0; j < QPT; ++j) xq[j] = q0 + j < q1 ? cq[q0 + j] : make_uint4(0u, 0u, 0u, 0u);
          uint32_t sum = 0;
#pragma unroll
          for (uint32_t j = 0; j < QPT; ++j) {
            xq[j] = make_uint4(fsum(xq[j].x), fsum(xq[j].y), fsum(xq[j].z), fsum(xq[j].w));
            sum += xq[j].x + xq[j].y + xq[j].z + xq[j].w;
          }
          uint32_t incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane == 31) s_wt[warp] = incl;
          __syncthreads();
          PH(4)
          uint32_t wp = lane < NW ? s_wt[lane] : 0u;
#pragma unroll
          for (int o = 1; o < NW; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, wp, o);
            if (lane >= o) wp += y;
          }
          const uint32_t wex = __shfl_sync(FULL, wp, (warp + 31) & 31);
          uint32_t base = (warp ? wex : 0u) + incl - sum;
#pragma unroll
          for (uint32_t j = 0; j < QPT; ++j) {
            const uint32_t a0 = base, a1 = a0 + xq[j].x, a2 = a1 + xq[j].y, a3 = a2 + xq[j].z;
            base = a3 + xq[j].w;
            if (q0 + j < q1) reinterpret_cast<uint2*>(st16)[q0 + j] = make_uint2(a0 | (a1 << 16), a2 | (a3 << 16));
          }
        }
        __syncthreads();
        PH(5)
        // slots
        const uint32_t lowm = (1u << nib) - 1u;  // fields of earlier groups
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t e = warp * WS + i * 32 + lane;
          if (e < n) {
            const uint32_t d = (uint32_t)key[i] & mask;
            const uint32_t pre = fsum(cnt[d] & lowm);
            const uint32_t p = (uint32_t)st16[d] + pre + ((rkp[i / RPW] >> ((i % RPW) * FB)) & FM);
            si[p] = (d << 16) | e;
          }
        }
        __syncthreads();
        PH(6)
        // write-out in slot order (coalesced), checking that positions ascend
        // inside every bin; a violation re-sorts the bin runs and rewrites
        const K hi = k0 & ~(K)mask;
        bool bad = false;
        for (uint32_t p = tid; p < n; p += NT) {
          const uint32_t w = si[p];
          if (p + 1 < n) {
            const uint32_t nx = si[p + 1];
            bad |= ((w ^ nx) < 65536u) & (nx < w);
          }
          ok[p] = hi | (K)(w >> 16);
          if (VB) ov[p] = sv[w & 0xffffu];
        }
        // bins ready for the next span before E's barrier (the next span may
        // start its atomics without a barrier of its own)
        for (uint32_t q = tid; q < nq; q += NT) reinterpret_cast<uint4*>(cnt)[q] = make_uint4(0u, 0u, 0u, 0u);
        if (__syncthreads_or(bad) || DTS_FORCE_FIXUP) {
#if DTS_PHASE_PROF == 2
          if (tid == 0) atomicAdd(&g_phase[12], 1ull);
#endif
          for (uint32_t p = tid; p + 1 < n; p += NT) {
            const uint32_t x = si[p], y = si[p + 1];
            const bool lead = (p == 0 || (si[p - 1] >> 16) != (x >> 16)) && (y >> 16) == (x >> 16);
            if (lead) {
              const uint32_t b = x >> 16;
              uint32_t c = 2;
              while (p + c < n && (si[p + c] >> 16) == b) ++c;
              for (uint32_t a = 1; a < c; ++a) {
                const uint32_t w = si[p + a];
                uint32_t j = a;
                while (j > 0 && si[p + j - 1] > w) {
                  si[p + j] = si[p + j - 1];
                  --j;
                }
                si[p + j] = w;
              }
            }
          }
          __syncthreads();
          for (uint32_t p = tid; p < n; p += NT) {
            const uint32_t w = si[p];
            ok[p] = hi | (K)(w >> 16);
            if (VB) ov[p] = sv[w & 0xffffu];
          }
          __syncthreads();  // (the next span may reuse this buffer right away)
        }
        PH(7)
        PH(8)
        return true;
      };
#if DTS_PHASE_PROF == 2
      if (tid == 0) atomicAdd(&g_phase[11], 1ull);
#endif
      if constexpr (RETRY) {
        if (counting(FieldBits<8>{})) continue;
        // a byte field would carry (a key with hundreds of copies per warp
        // pair): bins back to zero, then 16-bit fields — never LSD
        for (uint32_t q = tid; q < nq; q += NT) reinterpret_cast<uint4*>(cnt)[q] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        if (tid == 0) s_big = 0u;
        __syncthreads();
        if (counting(FieldBits<16>{})) continue;
      } else {
        if (counting(FieldBits<4>{})) continue;
        if (rq != nullptr) {
          // a 4-bit field would have carried: hand the span to the retry
          // launch (8-bit fields) untouched; bins back to zero for the next
          // span (every thread has read s_big before the reset)
          for (uint32_t q = tid; q < nq; q += NT) reinterpret_cast<uint4*>(cnt)[q] = make_uint4(0u, 0u, 0u, 0u);
          __syncthreads();
          const uint32_t ovn = s_ovn;
          __syncthreads();
          const bool queue = ovn < (uint32_t)DTS_OVN_LSD;
          if (tid == 0) {
            s_ovn = 0u;
            if (queue) {
              s_big = 0u;
              const uint32_t qi = atomicAdd(rq_n, 1u);
              Span R;
              R.offset = S.offset;
              R.len = S.len;
              R.src = S.src;
              rq[qi] = R;
            }
          }
          if (queue) {
            __syncthreads();
            continue;
          }
        }
      }
      lsd = true;
    } else {
      // ================= counting path on the top CB of more differing bits;
      // records sharing those bits are ranked by (key, position) ======
      constexpr int dbits = TL::CB;
      const int dsh = bits - dbits;
      const uint32_t nbin = 1u << dbits, mask = nbin - 1u, nwd = (nbin + 1) >> 1;
      PH(2)
#if DTS_PHASE_PROF == 2
      if (tid == 0) atomicAdd(&g_phase[10], 1ull);
#endif
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        if (e < n) {
          const uint32_t d = (uint32_t)(key[i] >> dsh) & mask;
          atomicAdd(&cnt[d >> 1], 1u << ((d & 1u) << 4));
        }
      }
      __syncthreads();
      PH(3)
      scan_bins(nwd);
      PH(5)
      lsd = s_big != 0u;
      if (!lsd) {
        // atomic slots (arbitrary order inside a group)
        uint16_t* fidx = si16 + TL::CAP;  // final order (second half of si)
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t e = warp * WS + i * 32 + lane;
          if (e < n) {
            const uint32_t d = (uint32_t)(key[i] >> dsh) & mask;
            const uint32_t sh = (d & 1u) << 4;
            const uint32_t old = atomicAdd(&cnt[d >> 1], 1u << sh);
            si16[(old >> sh) & 0xffffu] = (uint16_t)e;
          }
        }
        __syncthreads();
        PH(6)
        // stable position = group start + number of group members that
        // precede the record by (key, position) (groups hold <= FIXMAX records)
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t e = warp * WS + i * 32 + lane;
          if (e < n) {
            const uint32_t d = (uint32_t)(key[i] >> dsh) & mask;
            const uint32_t end = (cnt[d >> 1] >> ((d & 1u) << 4)) & 0xffffu;
            const uint32_t dp = d - 1u;
            const uint32_t start = d ? (cnt[dp >> 1] >> ((dp & 1u) << 4)) & 0xffffu : 0u;
            uint32_t r = 0;
            const K me = key[i];
            for (uint32_t q = start; q < end; ++q) {
              const uint32_t x = si16[q];
              const K kx = sk[x];
              r += (kx < me) || (kx == me && x < e);
            }
            fidx[start + r] = (uint16_t)e;
          }
        }
        __syncthreads();
        PH(7)
        for (uint32_t p = tid; p < n; p += NT) {
          const uint32_t e = si16[TL::CAP + p];
          ok[p] = sk[e];
          if (VB) ov[p] = sv[e];
        }
        zero_bins(nwd);
        __syncthreads();
        PH(8)
        continue;
      }
    }

    // ================= LSD path: stable passes of <= RB bits ==================
#if DTS_PHASE_PROF == 2
      if (tid == 0) atomicAdd(&g_phase[13], 1ull);
#endif
    if (known) {
      // the span's bound is only an upper bound: the LSD passes follow the
      // bits its keys really differ in (duplicate-heavy spans: often few)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) diff |= __shfl_xor_sync(FULL, diff, o);
      if (lane == 0) s_diff[warp] = diff;
      __syncthreads();
      diff = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) diff |= s_diff[w];
      bits = 0;
      if (diff) bits = (sizeof(K) == 8) ? 64 - __clzll((long long)diff) : 32 - __clz((int)(uint32_t)diff);
      if (bits == 0) {  // all keys equal: in place already, or one copy from T
        if (S.src & 1u) {
          for (uint32_t i = tid; i < n; i += NT) {
            ok[i] = sk[i];
            if (VB) ov[i] = sv[i];
          }
        }
        for (uint32_t i = tid; i < (uint32_t)(SL::cnt_bytes / 4); i += NT) cnt[i] = 0u;
        if (tid == 0) s_big = 0u;
        __syncthreads();
        continue;
      }
    }
    uint32_t idx[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) idx[i] = warp * WS + i * 32 + lane;
    const int npass = (bits + TL::RB - 1) / TL::RB;
    const int pb = (bits + npass - 1) / npass;
    uint32_t* mywc = wc + warp * (1u << (TL::RB - 1));
    for (int pass = 0; pass < npass; ++pass) {
      const int sh = pass * pb;
      const int pbits = min(pb, bits - sh);
      const uint32_t D = 1u << pbits;
      const uint32_t DW = (D + 1) / 2;  // packed counter words per warp
      for (uint32_t i = tid; i < NW * (1u << (TL::RB - 1)); i += NT) wc[i] = 0u;
      __syncthreads();
      uint32_t dg[IPT], lr[IPT];
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        if (e < n) {
          const uint32_t d = (uint32_t)(key[i] >> sh) & (D - 1);
          const uint32_t s2 = (d & 1u) << 4;
          const uint32_t old = atomicAdd(&mywc[d >> 1], 1u << s2);
          dg[i] = d;
          lr[i] = (old >> s2) & 0xffffu;
        }
        __syncwarp();
      }
      __syncthreads();
      for (uint32_t j = tid; j < DW; j += NT) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint32_t x = wc[w * (1u << (TL::RB - 1)) + j];
          wc[w * (1u << (TL::RB - 1)) + j] = s;
          s += x;
        }
        dt[2 * j] = s & 0xffffu;
        dt[2 * j + 1] = s >> 16;
      }
      __syncthreads();
      block_exscan<NT>(dt, (int)D, s_wt);
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        if (e < n) {
          const uint32_t d = dg[i];
          const uint32_t pos = dt[d] + ((mywc[d >> 1] >> ((d & 1u) << 4)) & 0xffffu) + lr[i];
          sk[pos] = key[i];
          si[pos] = (e << 16) | idx[i];
        }
      }
      __syncthreads();
      // stable order check: within one digit, pass-input positions must
      // ascend; a violation is repaired by re-sorting the digit runs
      bool bad = false;
      for (uint32_t p = tid; p + 1 < n; p += NT) {
        const uint32_t a = si[p], b = si[p + 1];
        const bool same = (((uint32_t)(sk[p] >> sh) ^ (uint32_t)(sk[p + 1] >> sh)) & (D - 1)) == 0u;
        bad |= same && (b >> 16) < (a >> 16);
      }
      if (__any_sync(FULL, bad) && lane == 0) s_fix = 1u;
      __syncthreads();
      if (s_fix || DTS_FORCE_FIXUP) {
        for (uint32_t p = tid; p < n; p += NT) {
          const uint32_t dx = (uint32_t)(sk[p] >> sh) & (D - 1);
          auto same = [&](uint32_t q) { return ((uint32_t)(sk[q] >> sh) & (D - 1)) == dx; };
          const bool leader = p == 0 || !same(p - 1);
          if (leader && p + 1 < n && same(p + 1)) {
            uint32_t c = 2;
            while (p + c < n && same(p + c)) ++c;
            for (uint32_t a2 = 1; a2 < c; ++a2) {
              const uint32_t xs = si[p + a2];
              const K xk = sk[p + a2];
              uint32_t b2 = a2;
              while (b2 > 0 && si[p + b2 - 1] > xs) {
                si[p + b2] = si[p + b2 - 1];
                sk[p + b2] = sk[p + b2 - 1];
                --b2;
              }
              si[p + b2] = xs;
              sk[p + b2] = xk;
            }
          }
        }
        __syncthreads();
        if (tid == 0) s_fix = 0u;
      }
      if (pass + 1 < npass) {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t e = warp * WS + i * 32 + lane;
          if (e < n) {
            key[i] = sk[e];
            idx[i] = si[e] & 0xffffu;
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t p = tid; p < n; p += NT) {
      ok[p] = sk[p];
      if (VB) ov[p] = sv[si[p] & 0xffffu];
    }
    for (uint32_t i = tid; i < (uint32_t)(SL::cnt_bytes / 4); i += NT) cnt[i] = 0u;
    if (tid == 0) s_big = 0u;  // (only the LSD path is entered with it set)
    __syncthreads();
  }
  PH_DONE
}

}  // namespace dts
