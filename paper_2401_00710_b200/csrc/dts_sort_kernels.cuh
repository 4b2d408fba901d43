// dts_sort_kernels.cuh — the distribution and base-case kernels:
//   k_histogram  : per-block bucket counts            (counting.py:123-137)
//   k_scatter    : stable tile-ranked scatter          (counting.py:141-151,
//                                                       _kernels.py:12-25)
//   k_local_sort : SMEM stable LSD sort of spans       (dtsort.py:127-147)
#pragma once
#include "dts_kernels.cuh"

namespace dts {

// ---------------------------------------------------------------------------
// k_histogram: persistent CTAs pull blocks; per block, count records per
// bucket with shared-memory atomics (B200 SMEM atomics sustain >1.4 Tkeys/s
// chip-wide, well above the 4-byte-key HBM stream) and store the row into
// the [bucket][row] count matrix.
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
    const K* p = keys + B.begin;
    const uint64_t n = B.end - B.begin;
    auto count_one = [&](K key, uint64_t e) {
      const uint32_t b = SPLIT ? SR(key, global_base + B.begin + e) : R(key);
      atomicAdd(&hist[b], 1u);
    };
    const uint64_t addr = reinterpret_cast<uint64_t>(p);
    uint64_t head = ((16 - (addr & 15)) & 15) / sizeof(K);
    if (head > n) head = n;
    const uint64_t nvec = (n - head) / VEC;
    const uint64_t tail0 = head + nvec * VEC;
    if ((uint64_t)tid < head) count_one(p[tid], tid);
    if ((uint64_t)tid < n - tail0) count_one(p[tail0 + tid], tail0 + tid);
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
        if (vi < nvec) {
          const K* kk = reinterpret_cast<const K*>(&v[u]);
#pragma unroll
          for (int e = 0; e < VEC; ++e) count_one(kk[e], head + vi * VEC + e);
        }
      }
    }
    __syncthreads();
    uint32_t* row = counts + P.cnt_base + B.row;
    for (uint32_t b = tid; b < P.nbmax; b += NT) row[(uint64_t)b * P.nrows] = hist[b];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Tile staging: copy [g0, g0+tn) of a global column into SMEM so that element
// e lands at buf[off + e] with off = g0 % (16/sizeof(T)); the 16-byte aligned
// body moves as uint4 (LDG.128/STS.128), head/tail elementwise.
// ---------------------------------------------------------------------------
template <typename T, int NT>
__device__ __forceinline__ uint32_t stage_tile(T* buf, const T* __restrict__ src, uint64_t g0,
                                               uint32_t tn) {
  constexpr int VEC = 16 / sizeof(T);
  const uint32_t off = (uint32_t)(g0 % VEC);
  T* dst = buf + off;
  const T* s = src + g0;
  // elements before the first aligned one
  const uint32_t head0 = (VEC - off) % VEC;
  const uint32_t head = head0 < tn ? head0 : tn;
  const uint32_t nvec = (tn - head) / VEC;
  const uint32_t tail0 = head + nvec * VEC;
  const int tid = threadIdx.x;
  if ((uint32_t)tid < head) dst[tid] = ld_stream(s + tid);
  if ((uint32_t)tid < tn - tail0) dst[tail0 + tid] = ld_stream(s + tail0 + tid);
  const uint4* sv = reinterpret_cast<const uint4*>(s + head);
  uint4* dv = reinterpret_cast<uint4*>(dst + head);
  constexpr int U = 8;
  for (uint32_t b = 0; b < nvec; b += NT * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = b + u * NT + tid;
      if (i < nvec) r[u] = ld_stream(sv + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = b + u * NT + tid;
      if (i < nvec) dv[i] = r[u];
    }
  }
  return off;
}

// Per-(key, value) width tiling of the scatter.
template <typename K, int VB> struct ScatterTile {
  static constexpr int NT = 512;
  static constexpr int IPT = (sizeof(K) == 4 && VB <= 4) ? 9 : 5;  // odd: conflict-free
  static constexpr int T = NT * IPT;
  static constexpr int AK = 32 / (int)sizeof(K);
  static constexpr int AV = VB ? 32 / VB : AK;
  static constexpr int A = AK > AV ? AK : AV;  // flush granularity (records): whole sectors
  static constexpr int NBC = 1024;             // bucket capacity (ids < 2^10)
};

struct ScatterLayout {
  size_t run, sk, sv, lk, lv, hk, si, pk, cnt, tst, fl, loc, hz, bar, total;
};
__host__ __device__ inline ScatterLayout scatter_layout(int T, int NT, int A, int kb, int vb,
                                                        Caps c, bool split) {
  ScatterLayout L;
  size_t o = 0;
  const size_t nb = c.nbc;
  L.run = o; o = align16(o + nb * 8);
  L.sk = o; o = align16(o + 2 * (size_t)(T + 8) * kb);
  L.sv = o; o = align16(o + 2 * (size_t)(T + 8) * vb);
  L.lk = o; o = align16(o + nb * A * kb);
  L.lv = o; o = align16(o + nb * A * vb);
  L.hk = o; o = align16(o + (size_t)c.hkc * kb);
  L.si = o; o = align16(o + (split ? (size_t)c.hkc * 8 : 0));
  L.pk = o; o = align16(o + (size_t)T * 4);
  L.cnt = o; o = align16(o + (size_t)32 * NT * 2);
  L.tst = o; o = align16(o + (nb + 1) * 4);
  L.fl = o; o = align16(o + nb * 4);
  L.loc = o; o = align16(o + nb);
  L.hz = o; o = align16(o + (size_t)c.hzc * 4);
  L.bar = o; o = align16(o + 16);
  L.total = o;
  return L;
}

// Issue the TMA copy of tile [g0, g0+tn) of one column into `buf` (element e
// at buf[off + e], off = g0 % VEC): the 16-byte aligned body goes through
// cp.async.bulk on `bar`; returns the body bytes.  Head/tail elements (< VEC
// each) are loaded by the caller.
template <typename T>
__device__ __forceinline__ uint32_t tile_body(uint64_t g0, uint32_t tn, uint32_t& off,
                                              uint32_t& head, uint32_t& nbody) {
  constexpr uint32_t VEC = 16 / sizeof(T);
  off = (uint32_t)(g0 % VEC);
  const uint32_t h0 = (VEC - off) % VEC;
  head = h0 < tn ? h0 : tn;
  nbody = ((tn - head) / VEC) * VEC;
  return nbody * (uint32_t)sizeof(T);
}

// ---------------------------------------------------------------------------
// k_scatter: one persistent CTA per SM pulls blocks; each block walks its
// tiles in input order.  Per tile:
//   * the tile's keys/values arrive in SMEM by TMA bulk copy (the next tile
//     is prefetched into the other buffer while this one is processed);
//   * every record is routed to its bucket (tile histogram by SMEM atomics);
//   * the tile's (bucket, slot) words are stably sorted by bucket with
//     per-thread-counter block radix rank passes (<= 5 bits each);
//   * bucket runs are written at run[b] — the block's running offset row,
//     the GPU twin of scatter_block's `run` (_kernels.py:19-25) — through a
//     per-bucket SMEM write-combining buffer so global stores only ever
//     complete whole 32-byte sectors (no L2 partial-sector evictions).
// Stable for every block count (counting.py:1-10 invariant).
// ---------------------------------------------------------------------------
template <typename K, int VB, bool SPLIT>
__global__ void __launch_bounds__(ScatterTile<K, VB>::NT, 1)
    k_scatter(const SegPlan* __restrict__ plans, const Blk* __restrict__ blks, uint32_t nblk,
              uint32_t* __restrict__ ctr, const K* __restrict__ kin,
              const typename ValOf<VB>::T* __restrict__ vin, K* __restrict__ kout,
              typename ValOf<VB>::T* __restrict__ vout, const uint64_t* __restrict__ scan,
              const K* __restrict__ heavy_pool, const uint32_t* __restrict__ hz_pool,
              const uint64_t* __restrict__ split_idx, uint64_t global_base, Caps caps) {
  using V = typename ValOf<VB>::T;
  using TL = ScatterTile<K, VB>;
  constexpr int NT = TL::NT, IPT = TL::IPT, T = TL::T, A = TL::A;
  constexpr uint64_t AM = A - 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const ScatterLayout L = scatter_layout(T, NT, A, sizeof(K), VB, caps, SPLIT);
  uint64_t* run = reinterpret_cast<uint64_t*>(smem_raw + L.run);
  K* skb = reinterpret_cast<K*>(smem_raw + L.sk);
  V* svb = reinterpret_cast<V*>(smem_raw + L.sv);
  K* lk = reinterpret_cast<K*>(smem_raw + L.lk);
  V* lv = reinterpret_cast<V*>(smem_raw + L.lv);
  K* hk = reinterpret_cast<K*>(smem_raw + L.hk);
  uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + L.si);
  uint32_t* pk = reinterpret_cast<uint32_t*>(smem_raw + L.pk);
  uint16_t* cnt = reinterpret_cast<uint16_t*>(smem_raw + L.cnt);
  uint32_t* tst = reinterpret_cast<uint32_t*>(smem_raw + L.tst);
  int32_t* fl = reinterpret_cast<int32_t*>(smem_raw + L.fl);
  uint8_t* loc = reinterpret_cast<uint8_t*>(smem_raw + L.loc);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + L.hz);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  __shared__ uint32_t s_blk;
  __shared__ uint32_t s_tmp[NT / 32 + 1];
  const int tid = threadIdx.x;
  constexpr uint32_t SKB = T + 8;  // per-buffer stride (elements)

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase[2] = {0u, 0u};

  // issue the loads of tile [g0, g0+tn) into buffer `bf`: TMA for the body,
  // plain loads (returned in registers) for the head/tail elements
  auto issue = [&](int bf, uint64_t g0, uint32_t tn, K& hkv, V& hvv, int& hpos) {
    uint32_t ko, khead, kbody, vo = 0, vhead = 0, vbody = 0;
    const uint32_t kbytes = tile_body<K>(g0, tn, ko, khead, kbody);
    uint32_t vbytes = 0;
    if (VB) vbytes = tile_body<V>(g0, tn, vo, vhead, vbody);
    if (tid == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bar[bf], kbytes + vbytes);
      if (kbytes) tma_load_1d(skb + bf * SKB + ko + khead, kin + g0 + khead, kbytes, &bar[bf]);
      if (vbytes) tma_load_1d(svb + bf * SKB + vo + vhead, vin + g0 + vhead, vbytes, &bar[bf]);
    }
    // head/tail: element positions not covered by the bulk copies
    hpos = -1;
    const uint32_t ktail = tn - khead - kbody;
    const uint32_t nk = khead + ktail;
    const uint32_t nv = VB ? vhead + (tn - vhead - vbody) : 0;
    if ((uint32_t)tid < nk) {
      const uint32_t e = (uint32_t)tid < khead ? (uint32_t)tid : khead + kbody + (tid - khead);
      hkv = kin[g0 + e];
      hpos = (int)e;
    }
    if (VB && (uint32_t)tid >= 64 && (uint32_t)tid < 64 + nv) {
      const uint32_t t2 = tid - 64;
      const uint32_t e = t2 < vhead ? t2 : vhead + vbody + (t2 - vhead);
      hvv = vin[g0 + e];
      hpos = (int)e;
    }
  };
  auto commit_ht = [&](int bf, uint64_t g0, K hkv, V hvv, int hpos) {
    if (hpos < 0) return;
    if ((uint32_t)tid < 64) {
      skb[bf * SKB + (uint32_t)(g0 % (16 / sizeof(K))) + hpos] = hkv;
    } else if (VB) {
      svb[bf * SKB + (uint32_t)(g0 % (16 / (VB ? VB : 4))) + hpos] = hvv;
    }
  };

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
      for (uint32_t b = tid; b < nb; b += NT) {
        run[b] = rb + col[(uint64_t)b * P.nrows];
        tst[b] = 0;
        loc[b] = 0;
      }
    }
    const Router<K> R = make_router<K>(P, hz, hk);
    SplitRouter<K> SR;
    SR.sk = hk; SR.si = si; SR.ns = P.nheavy;
    const int nbits = max(1, (int)ceil_log2_u64(nb));
    const int npass = (nbits + 4) / 5;
    const int pbits = (nbits + npass - 1) / npass;

    const uint64_t ntile = (B.end - B.begin + T - 1) / T;
    K hkv = 0;
    V hvv = 0;
    int hpos = -1;
    {
      const uint64_t g0 = B.begin;
      const uint32_t tn = (uint32_t)min((uint64_t)T, B.end - g0);
      issue(0, g0, tn, hkv, hvv, hpos);
      commit_ht(0, g0, hkv, hvv, hpos);
    }
    __syncthreads();
    for (uint64_t ti = 0; ti < ntile; ++ti) {
      const int cb = (int)(ti & 1);
      const uint64_t tile = B.begin + ti * T;
      const uint32_t tn = (uint32_t)min((uint64_t)T, B.end - tile);
      // prefetch the next tile of this block into the other buffer
      const bool has_next = ti + 1 < ntile;
      uint64_t ng0 = tile + T;
      if (has_next) {
        const uint32_t ntn = (uint32_t)min((uint64_t)T, B.end - ng0);
        issue(cb ^ 1, ng0, ntn, hkv, hvv, hpos);
      }
      mbar_wait(&bar[cb], phase[cb]);
      phase[cb] ^= 1u;
      const uint32_t ko = (uint32_t)(tile % (16 / sizeof(K)));
      const uint32_t vo = VB ? (uint32_t)(tile % (16 / (VB ? VB : 4))) : 0u;
      const K* sk = skb + cb * SKB + ko;
      const V* sv = svb + cb * SKB + vo;
      // route (blocked order) + tile histogram
      uint32_t w[IPT];
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = tid * IPT + i;
        if (e < tn) {
          const K key = sk[e];
          const uint32_t b = SPLIT ? SR(key, global_base + tile + e) : R(key);
          atomicAdd(&tst[b], 1u);
          w[i] = (b << 16) | e;
        } else {
          w[i] = 0xFFFF0000u | e;
        }
      }
      // stable sort of the (bucket, slot) words by bucket: LSD passes
      for (int pass = 0; pass < npass; ++pass) {
        const int sh = 16 + pass * pbits;
        const int bits = min(pbits, nbits - pass * pbits);
        const int D = 1 << bits;
        uint32_t dig[IPT], rk[IPT];
#pragma unroll
        for (int i = 0; i < IPT; ++i) dig[i] = (w[i] >> sh) & (uint32_t)(D - 1);
        block_rank<NT, IPT>(dig, D, rk, cnt, s_tmp);
#pragma unroll
        for (int i = 0; i < IPT; ++i) pk[rk[i]] = w[i];
        __syncthreads();
        if (pass + 1 < npass) {
#pragma unroll
          for (int i = 0; i < IPT; ++i) w[i] = pk[tid * IPT + i];
        }
      }
      block_exscan<NT>(tst, (int)nb, s_tmp);
      if (tid == 0) tst[nb] = tn;
      __syncthreads();
      // W1: per bucket, flush limit F (whole sectors) and old leftovers
      for (uint32_t b = tid; b < nb; b += NT) {
        const uint32_t c = tst[b + 1] - tst[b];
        const uint64_t r = run[b];
        const uint32_t lc = loc[b];
        const uint64_t end = r + c;
        uint64_t F = end & ~AM;
        if (lc == 0 && (r & AM) && end <= ((r + AM) & ~AM)) F = end;  // block's head sector
        fl[b] = (int32_t)((int64_t)F - (int64_t)r);
        const uint64_t lo0 = r - lc;
        for (uint32_t s = 0; s < lc; ++s) {
          const uint64_t d = lo0 + s;
          if (d < F) {
            kout[d] = lk[b * A + s];
            if (VB) vout[d] = lv[b * A + s];
          } else {
            lk[b * A + (d - F)] = lk[b * A + s];
            if (VB) lv[b * A + (d - F)] = lv[b * A + s];
          }
        }
        loc[b] = (uint8_t)(end - F);
        run[b] = end;
      }
      __syncthreads();
      // W2: tile records -> global (flushable) or leftover buffer
      for (uint32_t p = tid; p < tn; p += NT) {
        const uint32_t wd = pk[p];
        const uint32_t b = wd >> 16, e = wd & 0xffffu;
        const int32_t dr = (int32_t)(p - tst[b]);
        const int32_t f = fl[b];
        if (dr < f) {
          const uint64_t d = run[b] - (tst[b + 1] - tst[b]) + (uint32_t)dr;
          kout[d] = sk[e];
          if (VB) vout[d] = sv[e];
        } else {
          const uint32_t s = (uint32_t)(dr - f);
          lk[b * A + s] = sk[e];
          if (VB) lv[b * A + s] = sv[e];
        }
      }
      if (has_next) commit_ht(cb ^ 1, ng0, hkv, hvv, hpos);
      __syncthreads();
      for (uint32_t b = tid; b < nb; b += NT) tst[b] = 0;
      // (the next tile's route phase follows a barrier inside mbar/route)
      __syncthreads();
    }
    // block end: flush the remaining partial sectors
    for (uint32_t b = tid; b < nb; b += NT) {
      const uint32_t lc = loc[b];
      const uint64_t lo0 = run[b] - lc;
      for (uint32_t s = 0; s < lc; ++s) {
        kout[lo0 + s] = lk[b * A + s];
        if (VB) vout[lo0 + s] = lv[b * A + s];
      }
    }
    __syncthreads();
  }
}

struct LocalLayout {
  size_t sk, sv, si, cnt, total;
};
__host__ __device__ inline LocalLayout local_layout(int CAP, int NT, int kb, int vb, int RB) {
  LocalLayout L;
  size_t o = 0;
  L.sk = o; o = align16(o + (size_t)(CAP + 4) * kb);
  L.sv = o; o = align16(o + (size_t)(CAP + 4) * vb);
  L.si = o; o = align16(o + (size_t)CAP * 2);
  L.cnt = o; o = align16(o + ((size_t)NT << RB) * 2);
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------
// k_local_sort: one CTA per base-case span (<= CAP records).  Loads the span
// into SMEM, finds the bits that differ inside it, and runs stable LSD passes
// of <= 6 bits (block radix rank) on (key, slot) pairs; payloads are
// gathered once at the end.  Output always lands in A.  dtsort.py:127-147
// (stable sort by full key of a span of adjacent buckets, valid per :128-131).
// ---------------------------------------------------------------------------
template <typename K, int VB, int NT, int IPT, int RB>
__global__ void __launch_bounds__(NT, 3) k_local_sort(const Span* __restrict__ spans,
                                                   K* __restrict__ Ak,
                                                   typename ValOf<VB>::T* __restrict__ Av,
                                                   const K* __restrict__ Tk,
                                                   const typename ValOf<VB>::T* __restrict__ Tv) {
  using V = typename ValOf<VB>::T;
  constexpr int NW = NT / 32;
  constexpr int CAP = NT * IPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const LocalLayout L = local_layout(CAP, NT, sizeof(K), VB, RB);
  K* skb = reinterpret_cast<K*>(smem_raw + L.sk);
  V* svb = reinterpret_cast<V*>(smem_raw + L.sv);
  uint16_t* si = reinterpret_cast<uint16_t*>(smem_raw + L.si);
  uint16_t* cnt = reinterpret_cast<uint16_t*>(smem_raw + L.cnt);
  __shared__ uint32_t s_tmp[NW + 1];
  __shared__ K s_diff[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const Span S = spans[blockIdx.x];
  const uint32_t n = S.len;
  const K* srck = S.src ? Tk : Ak;
  const V* srcv = S.src ? Tv : Av;
  const uint32_t ko = stage_tile<K, NT>(skb, srck, S.offset, n);
  uint32_t vo = 0;
  if (VB) vo = stage_tile<V, NT>(svb, srcv, S.offset, n);
  K* sk = skb + ko;
  __syncthreads();
  const K k0 = sk[0];
  K key[IPT];
  K diff = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t e = tid * IPT + i;
    key[i] = e < n ? sk[e] : k0;
    diff |= key[i] ^ k0;
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

  K* ok = Ak + S.offset;
  if (bits > 0) {
    const int npass = (bits + RB - 1) / RB;
    const int pbits = (bits + npass - 1) / npass;
    uint32_t ix[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) ix[i] = tid * IPT + i;
    for (int pass = 0; pass < npass; ++pass) {
      const int sh = pass * pbits;
      const int pb = min(pbits, bits - sh);
      const int D = 1 << pb;
      uint32_t dig[IPT], rk[IPT];
#pragma unroll
      for (int i = 0; i < IPT; ++i)
        dig[i] = ix[i] < n ? (uint32_t)(key[i] >> sh) & (uint32_t)(D - 1) : (uint32_t)(D - 1);
      block_rank<NT, IPT>(dig, D, rk, cnt, s_tmp);
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        sk[rk[i]] = key[i];
        si[rk[i]] = (uint16_t)ix[i];
      }
      __syncthreads();
      if (pass + 1 < npass) {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          key[i] = sk[tid * IPT + i];
          ix[i] = si[tid * IPT + i];
        }
      }
    }
    for (uint32_t i = tid; i < n; i += NT) {
      ok[i] = sk[i];
      if (VB) Av[S.offset + i] = svb[vo + si[i]];
    }
  } else if (S.src) {
    for (uint32_t i = tid; i < n; i += NT) {
      ok[i] = sk[i];
      if (VB) Av[S.offset + i] = svb[vo + i];
    }
  }
}

}  // namespace dts
