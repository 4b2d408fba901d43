// dts_local.cuh — k_local_sort, the base case (dtsort.py:127-147 _base_sort:
// stable sort by full key of a span of adjacent buckets, valid per :128-131).
#pragma once
#include "dts_rank.cuh"
#include "dts_sort_kernels.cuh"

namespace dts {

template <typename K, int VB> struct LocalTile {
  static constexpr int NT = 256;
  static constexpr int NW = NT / 32;
  static constexpr int IPT = 17;
  static constexpr int WS = 32 * IPT;  // records per warp sub-tile
  static constexpr int CAP = NT * IPT;
  static constexpr int RB = 8;         // radix bits per pass (<= 2^8 digit values)
};

struct LocalLayout {
  size_t sk, sv, si, wc, dt, total;
};
__host__ __device__ inline LocalLayout local_layout(int CAP, int NT, int kb, int vb, int RB) {
  LocalLayout L;
  size_t o = 0;
  L.sk = o; o = align16(o + (size_t)(CAP + 8) * kb);
  L.sv = o; o = align16(o + (size_t)(CAP + 8) * vb);
  L.si = o; o = align16(o + (size_t)CAP * 4);
  L.wc = o; o = align16(o + (size_t)(NT / 32) * ((size_t)1 << (RB - 1)) * 4);
  L.dt = o; o = align16(o + (((size_t)1 << RB) + 1) * 4);
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------
// k_local_sort: one CTA per span (<= CAP records).  Loads the span into SMEM,
// finds the bits that differ inside it (keys agree above bit `bits`), and
// runs stable LSD passes of <= RB bits.  Each pass ranks records with the
// per-warp counter scheme of k_scatter (warp w owns a contiguous sub-tile in
// lane-striped order; SMEM atomics on its packed u16 digit counters; an
// exclusive prefix over (digit, warp)); in-step order is verified and
// repaired if ever needed.  Records move as (key, position|slot) pairs;
// payloads are gathered once at the end.  Output always lands in A.
// ---------------------------------------------------------------------------
template <typename K, int VB>
__global__ void __launch_bounds__(LocalTile<K, VB>::NT, 3)
    k_local_sort(const Span* __restrict__ spans, K* __restrict__ Ak,
                 typename ValOf<VB>::T* __restrict__ Av, const K* __restrict__ Tk,
                 const typename ValOf<VB>::T* __restrict__ Tv) {
  using V = typename ValOf<VB>::T;
  using TL = LocalTile<K, VB>;
  constexpr int NT = TL::NT, NW = TL::NW, IPT = TL::IPT, WS = TL::WS, CAP = TL::CAP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const LocalLayout L = local_layout(CAP, NT, sizeof(K), VB, TL::RB);
  K* skb = reinterpret_cast<K*>(smem_raw + L.sk);
  V* svb = reinterpret_cast<V*>(smem_raw + L.sv);
  uint32_t* si = reinterpret_cast<uint32_t*>(smem_raw + L.si);
  uint32_t* wc = reinterpret_cast<uint32_t*>(smem_raw + L.wc);
  uint32_t* dt = reinterpret_cast<uint32_t*>(smem_raw + L.dt);
  __shared__ uint32_t s_tmp[NW + 1];
  __shared__ K s_diff[NW];
  __shared__ uint32_t s_fix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const Span S = spans[blockIdx.x];
  const uint32_t n = S.len;
  const K* srck = S.src ? Tk : Ak;
  const V* srcv = S.src ? Tv : Av;
  const uint32_t ko = stage_tile<K, NT>(skb, srck, S.offset, n);
  uint32_t vo = 0;
  if (VB) vo = stage_tile<V, NT>(svb, srcv, S.offset, n);
  K* sk = skb + ko;
  const V* sv = svb + vo;
  if (tid == 0) s_fix = 0u;
  __syncthreads();
  const K k0 = sk[0];
  K key[IPT];
  uint32_t idx[IPT];
  K diff = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t e = warp * WS + i * 32 + lane;
    key[i] = e < n ? sk[e] : k0;
    idx[i] = e;
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
  if (bits == 0) {
    if (S.src) {
      for (uint32_t i = tid; i < n; i += NT) {
        ok[i] = sk[i];
        if (VB) Av[S.offset + i] = sv[i];
      }
    }
    return;
  }

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
    // ---- per-warp rank: lane-striped steps, atomics on own counters ----
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
    // ---- exclusive prefix over warps per digit, digit totals ----
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
    block_exscan<NT>(dt, (int)D, s_tmp);
    // ---- placement (all records are in registers) ----
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
    // ---- next pass input (lane-striped) or the output; the in-step order
    // check is fused: within one (digit, warp step) group positions must
    // ascend.  A violation triggers the repair below and a redo. ----
    auto group_fix = [&]() {
      for (uint32_t p = tid; p < n; p += NT) {
        const uint32_t x = si[p];
        const uint32_t dx = (uint32_t)(sk[p] >> sh) & (D - 1);
        auto same = [&](uint32_t q) {
          return ((uint32_t)(sk[q] >> sh) & (D - 1)) == dx && (si[q] >> 21) == (x >> 21);
        };
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
    };
    auto pair_bad = [&](K ka, uint32_t sa, K kb, uint32_t sb) {
      return (((uint32_t)(ka >> sh) ^ (uint32_t)(kb >> sh)) & (D - 1)) == 0u &&
             (sa >> 21) == (sb >> 21) && sb < sa;
    };
    if (pass + 1 < npass) {
      bool bad = false;
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = warp * WS + i * 32 + lane;
        K kk = k0;
        uint32_t ss = 0xFFFFFFFFu;
        if (e < n) {
          kk = sk[e];
          ss = si[e];
          key[i] = kk;
          idx[i] = ss & 0xffffu;
        }
        K kn = __shfl_down_sync(FULL, kk, 1);
        uint32_t sn = __shfl_down_sync(FULL, ss, 1);
        if (lane == 31 && e + 1 < n) {
          kn = sk[e + 1];
          sn = si[e + 1];
        }
        if (e + 1 < n) bad |= pair_bad(kk, ss, kn, sn);
      }
      if (__any_sync(FULL, bad) && lane == 0) s_fix = 1u;
      __syncthreads();
      if (s_fix || DTS_FORCE_FIXUP) {
        group_fix();
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
          const uint32_t e = warp * WS + i * 32 + lane;
          if (e < n) {
            key[i] = sk[e];
            idx[i] = si[e] & 0xffffu;
          }
        }
        __syncthreads();
        if (tid == 0) s_fix = 0u;
      }
    } else {
      bool bad = false;
      for (uint32_t p0 = 0; p0 < n; p0 += NT) {
        const uint32_t p = p0 + tid;
        K kk = k0;
        uint32_t ss = 0xFFFFFFFFu;
        if (p < n) {
          kk = sk[p];
          ss = si[p];
          ok[p] = kk;
          if (VB) Av[S.offset + p] = sv[ss & 0xffffu];
        }
        K kn = __shfl_down_sync(FULL, kk, 1);
        uint32_t sn = __shfl_down_sync(FULL, ss, 1);
        if (lane == 31 && p + 1 < n) {
          kn = sk[p + 1];
          sn = si[p + 1];
        }
        if (p + 1 < n) bad |= pair_bad(kk, ss, kn, sn);
      }
      if (__any_sync(FULL, bad) && lane == 0) s_fix = 1u;
      __syncthreads();
      if (s_fix || DTS_FORCE_FIXUP) {
        group_fix();
        for (uint32_t p = tid; p < n; p += NT) {
          ok[p] = sk[p];
          if (VB) Av[S.offset + p] = sv[si[p] & 0xffffu];
        }
        if (tid == 0) s_fix = 0u;
      }
    }
  }
}

}  // namespace dts
