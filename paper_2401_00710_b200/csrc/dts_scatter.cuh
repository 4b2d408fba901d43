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
  static constexpr int AK = 32 / (int)sizeof(K);
  static constexpr int AV = VB ? 32 / VB : AK;
  static constexpr int A = AK > AV ? AK : AV;  // flush granularity (records): whole sectors
  // bucket capacity (SMEM budget: write-combining buffers + per-warp counters)
  static constexpr int NBC = (sizeof(K) == 4 && VB == 8) ? 512 : 1024;
};

struct ScatterLayout {
  size_t run, dbase, sk, sv, lk, lv, hk, si, pk, wh, tst, fl, loc, hz, bar, total;
};
__host__ __device__ inline ScatterLayout scatter_layout(int T, int NT, int A, int kb, int vb,
                                                        Caps c, bool split) {
  ScatterLayout L;
  size_t o = 0;
  const size_t nb = c.nbc;
  L.run = o; o = align16(o + nb * 8);
  L.dbase = o; o = align16(o + nb * 8);
  L.sk = o; o = align16(o + 2 * (size_t)(T + 8) * kb);
  L.sv = o; o = align16(o + 2 * (size_t)(T + 8) * vb);
  L.lk = o; o = align16(o + nb * A * kb);
  L.lv = o; o = align16(o + nb * A * vb);
  L.hk = o; o = align16(o + (size_t)c.hkc * kb);
  L.si = o; o = align16(o + (split ? (size_t)c.hkc * 8 : 0));
  L.pk = o; o = align16(o + (size_t)T * 4);
  L.wh = o; o = align16(o + (size_t)(NT / 32) * ((nb + 1) / 2) * 4);
  L.tst = o; o = align16(o + (nb + 1) * 4);
  L.fl = o; o = align16(o + nb * 4);
  L.loc = o; o = align16(o + nb);
  L.hz = o; o = align16(o + (size_t)c.hzc * 4);
  L.bar = o; o = align16(o + 16);
  L.total = o;
  return L;
}

// Split [g0, g0+tn) of a T-typed column into head / 16-byte aligned body /
// tail; returns the body bytes (moved by cp.async.bulk).
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
//   * keys/values arrive in SMEM by TMA bulk copy (cp.async.bulk on an
//     mbarrier; the next tile is prefetched into the other buffer while this
//     one is processed);
//   * stable in-tile rank with per-warp bucket counters: warp w owns the
//     contiguous sub-tile [w*WS, (w+1)*WS) in lane-striped order and takes
//     its records' ranks from SMEM atomics on its own packed u16 counters
//     (ordered across the warp's steps); an exclusive prefix over warps per
//     bucket orders the warps; the only freedom left — lanes of one warp
//     step hitting the same bucket — is removed by a tiny per-group sort on
//     the record index (groups are contiguous and <= 32 long);
//   * bucket runs go to run[b] — the block's running offset row, the GPU
//     twin of scatter_block's `run` (_kernels.py:19-25) — through a
//     per-bucket SMEM write-combining buffer so global stores only complete
//     whole 32-byte sectors (no L2 partial-sector evictions).
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
  constexpr int NT = TL::NT, NW = TL::NW, IPT = TL::IPT, WS = TL::WS, T = TL::T, A = TL::A;
  constexpr uint64_t AM = A - 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const ScatterLayout L = scatter_layout(T, NT, A, sizeof(K), VB, caps, SPLIT);
  uint64_t* run = reinterpret_cast<uint64_t*>(smem_raw + L.run);
  uint64_t* dbase = reinterpret_cast<uint64_t*>(smem_raw + L.dbase);
  K* skb = reinterpret_cast<K*>(smem_raw + L.sk);
  V* svb = reinterpret_cast<V*>(smem_raw + L.sv);
  K* lk = reinterpret_cast<K*>(smem_raw + L.lk);
  V* lv = reinterpret_cast<V*>(smem_raw + L.lv);
  K* hk = reinterpret_cast<K*>(smem_raw + L.hk);
  uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + L.si);
  uint32_t* pk = reinterpret_cast<uint32_t*>(smem_raw + L.pk);
  uint32_t* wh = reinterpret_cast<uint32_t*>(smem_raw + L.wh);
  uint32_t* tst = reinterpret_cast<uint32_t*>(smem_raw + L.tst);
  int32_t* fl = reinterpret_cast<int32_t*>(smem_raw + L.fl);
  uint8_t* loc = reinterpret_cast<uint8_t*>(smem_raw + L.loc);
  uint32_t* hz = reinterpret_cast<uint32_t*>(smem_raw + L.hz);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + L.bar);
  __shared__ uint32_t s_blk, s_fix;
  __shared__ uint32_t s_tmp[NW + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t SKB = T + 8;  // per-buffer stride (elements)
  const uint32_t HW = (caps.nbc + 1) / 2;  // packed counter words per warp
  uint32_t* mywh = wh + warp * HW;

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    s_fix = 0u;
  }
  for (uint32_t i = tid; i < NW * HW; i += NT) wh[i] = 0u;
  __syncthreads();
  uint32_t phase[2] = {0u, 0u};

  // issue tile [g0, g0+tn) into buffer bf: TMA for the aligned bodies, plain
  // loads into registers for the (< 16 B) heads / tails, committed later
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
    hpos = -1;
    const uint32_t nk = tn - kbody;
    const uint32_t nv = VB ? tn - vbody : 0;
    if ((uint32_t)tid < nk) {
      const uint32_t e = (uint32_t)tid < khead ? (uint32_t)tid : kbody + (uint32_t)tid;
      hkv = kin[g0 + e];
      hpos = (int)e;
    }
    if (VB && (uint32_t)tid >= 64 && (uint32_t)tid < 64 + nv) {
      const uint32_t t2 = tid - 64;
      const uint32_t e = t2 < vhead ? t2 : vbody + t2;
      hvv = vin[g0 + e];
      hpos = (int)e;
    }
  };
  auto commit_ht = [&](int bf, uint64_t g0, K hkv, V hvv, int hpos) {
    if (hpos < 0) return;
    if ((uint32_t)tid < 64) {
      skb[bf * SKB + (uint32_t)(g0 % (16 / sizeof(K))) + hpos] = hkv;
    } else if (VB) {
      svb[bf * SKB + (uint32_t)(g0 % (16 / sizeof(V))) + hpos] = hvv;
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
    const uint32_t nw2 = (nb + 1) / 2;
    load_tables<K>(P, heavy_pool, hz_pool, split_idx, hk, si, hz);
    {
      const uint64_t* col = scan + P.cnt_base + B.row;
      const uint64_t rb = P.offset - P.scanbase;
      for (uint32_t b = tid; b < nb; b += NT) {
        run[b] = rb + col[(uint64_t)b * P.nrows];
        loc[b] = 0;
      }
    }
    const Router<K> R = make_router<K>(P, hz, hk);
    SplitRouter<K> SR;
    SR.sk = hk; SR.si = si; SR.ns = P.nheavy;

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
      const bool has_next = ti + 1 < ntile;
      const uint64_t ng0 = tile + T;
      if (has_next) issue(cb ^ 1, ng0, (uint32_t)min((uint64_t)T, B.end - ng0), hkv, hvv, hpos);
      mbar_wait(&bar[cb], phase[cb]);
      phase[cb] ^= 1u;
      const K* sk = skb + cb * SKB + (uint32_t)(tile % (16 / sizeof(K)));
      const V* sv = svb + cb * SKB + (uint32_t)(tile % (16 / sizeof(V)));
      // ---- route + per-warp rank (lane-striped within the warp sub-tile) ----
      uint32_t bk[IPT], lr[IPT];
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        bk[i] = 0xFFFFu;
        if (e < tn) {
          const K key = sk[e];
          const uint32_t b = SPLIT ? SR(key, global_base + tile + e) : R(key);
          const uint32_t sh = (b & 1u) << 4;
          const uint32_t old = atomicAdd(&mywh[b >> 1], 1u << sh);
          bk[i] = b;
          lr[i] = (old >> sh) & 0xffffu;
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- per bucket pair: exclusive prefix over warps, tile totals ----
      for (uint32_t j = tid; j < nw2; j += NT) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint32_t x = wh[w * HW + j];
          wh[w * HW + j] = s;
          s += x;
        }
        tst[2 * j] = s & 0xffffu;
        tst[2 * j + 1] = s >> 16;
      }
      __syncthreads();
      block_exscan<NT>(tst, (int)nb, s_tmp);
      if (tid == 0) tst[nb] = tn;
      __syncthreads();
      // ---- placement ----
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        if (bk[i] != 0xFFFFu) {
          const uint32_t b = bk[i];
          const uint32_t pre = (mywh[b >> 1] >> ((b & 1u) << 4)) & 0xffffu;
          const uint32_t e = warp * WS + i * 32 + lane;
          pk[tst[b] + pre + lr[i]] = (b << 16) | e;
        }
      }
      __syncthreads();
      // ---- verify the in-step order.  Lanes of one warp step that hit the
      // same bucket form a group (b, e >> 5) of contiguous records; the
      // SMEM atomics gave them increasing ranks in lane order on every B200
      // probed (tools/atomic_order.cu: 0 of 5e9 colliding pairs out of
      // order), which the PTX model does not promise — so check each
      // adjacent pair and re-sort groups only if one is out of order.
      // The check runs in the same phase as W1 (no extra barrier). ----
      for (uint32_t i = tid; i < NW * HW; i += NT) wh[i] = 0u;
      {
        bool bad = false;
        for (uint32_t p = tid; p + 1 < tn; p += NT) {
          const uint32_t x = pk[p], y = pk[p + 1];
          bad |= ((x ^ y) < 32u) && (y < x);  // same bucket & step, descending
        }
        if (__any_sync(FULL, bad) && lane == 0) s_fix = 1u;
      }
      // ---- W1: per bucket, flush limit F (whole sectors), old leftovers ----
      for (uint32_t b = tid; b < nb; b += NT) {
        const uint32_t ts = tst[b];
        const uint32_t c = tst[b + 1] - ts;
        const uint64_t r = run[b];
        const uint32_t lc = loc[b];
        const uint64_t end = r + c;
        uint64_t F = end & ~AM;
        if (lc == 0 && (r & AM) && end <= ((r + AM) & ~AM)) F = end;  // block's head sector
        dbase[b] = r - ts;
        fl[b] = (int32_t)ts + (int32_t)((int64_t)F - (int64_t)r);
        const uint64_t lo0 = r - lc;
        for (uint32_t s2 = 0; s2 < lc; ++s2) {
          const uint64_t d = lo0 + s2;
          if (d < F) {
            kout[d] = lk[b * A + s2];
            if (VB) vout[d] = lv[b * A + s2];
          } else {
            lk[b * A + (d - F)] = lk[b * A + s2];
            if (VB) lv[b * A + (d - F)] = lv[b * A + s2];
          }
        }
        loc[b] = (uint8_t)(end - F);
        run[b] = end;
      }
      __syncthreads();
      if (s_fix || DTS_FORCE_FIXUP) {
        // general path: sort every group (b, e >> 5) of >= 2 records by e
        for (uint32_t p = tid; p < tn; p += NT) {
          const uint32_t x = pk[p];
          const bool leader = p == 0 || ((pk[p - 1] ^ x) >= 32u);
          if (leader && p + 1 < tn && ((pk[p + 1] ^ x) < 32u)) {
            uint32_t c = 2;
            while (p + c < tn && ((pk[p + c] ^ x) < 32u)) ++c;
            small_isort(pk + p, c);
          }
        }
        __syncthreads();
        if (tid == 0) s_fix = 0u;
      }
      // ---- W2: tile records -> global (flushable) or leftover buffer ----
#pragma unroll
      for (int it = 0; it < IPT; ++it) {
        const uint32_t p = it * NT + tid;
        if (p < tn) {
          const uint32_t wd = pk[p];
          const uint32_t b = wd >> 16, e = wd & 0xffffu;
          const int32_t lim = fl[b];
          const K kv = sk[e];
          V vv = 0;
          if (VB) vv = sv[e];
          if ((int32_t)p < lim) {
            const uint64_t d = dbase[b] + p;
            kout[d] = kv;
            if (VB) vout[d] = vv;
          } else {
            const uint32_t s = (uint32_t)((int32_t)p - lim);
            lk[b * A + s] = kv;
            if (VB) lv[b * A + s] = vv;
          }
        }
      }
      if (has_next) commit_ht(cb ^ 1, ng0, hkv, hvv, hpos);
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

}  // namespace dts
