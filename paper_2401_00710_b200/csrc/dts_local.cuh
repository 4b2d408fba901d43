// dts_local.cuh — k_local_sort, the base case (dtsort.py:127-147 _base_sort:
// stable sort by full key of a span of adjacent buckets, valid per :128-131).
#pragma once
#include "dts_rank.cuh"
#include "dts_sort_kernels.cuh"

namespace dts {

template <typename K, int VB> struct LocalTile {
  static constexpr int NT = 256;
  static constexpr int IPT = 17;  // odd: conflict-free blocked SMEM reads
  static constexpr int CAP = NT * IPT;
  static constexpr int FAST_BITS = 13;  // counting-slot path up to 2^13 digit values
  static constexpr int RB = 5;          // fallback LSD radix bits per pass
};

struct LocalLayout {
  size_t sk, sv, si, cnt, u4, total;
};
__host__ __device__ inline LocalLayout local_layout(int CAP, int NT, int kb, int vb, int fast_bits) {
  LocalLayout L;
  size_t o = 0;
  L.sk = o; o = align16(o + (size_t)(CAP + 8) * kb);
  L.sv = o; o = align16(o + (size_t)(CAP + 8) * vb);
  L.si = o; o = align16(o + (size_t)CAP * 4);
  L.cnt = o; o = align16(o + ((size_t)1 << fast_bits) * 4);
  L.u4 = o; o = align16(o + (size_t)(NT / 32 + 1) * 16);
  L.total = o;
  return L;
}

// ---------------------------------------------------------------------------
// k_local_sort: one CTA per span (<= CAP records).  Loads the span into SMEM
// and finds the bits that differ inside it (keys agree above bit `bits`).
//  * bits <= FAST_BITS: one counting pass over the differing bits — SMEM
//    atomic histogram, block scan, atomic slot per record, then equal keys
//    are put back into input order (per-digit insertion sort; digits with
//    more than FIXMAX records get exact packed-prefix slots);
//  * otherwise (or with > NLARGE large digits): stable LSD passes of <= RB
//    bits with block_rank_packed on (key, slot) pairs.
// Payloads are gathered once at the end.  Output always lands in A.
// ---------------------------------------------------------------------------
template <typename K, int VB>
__global__ void __launch_bounds__(LocalTile<K, VB>::NT, 2)
    k_local_sort(const Span* __restrict__ spans, K* __restrict__ Ak,
                 typename ValOf<VB>::T* __restrict__ Av, const K* __restrict__ Tk,
                 const typename ValOf<VB>::T* __restrict__ Tv) {
  using V = typename ValOf<VB>::T;
  using TL = LocalTile<K, VB>;
  constexpr int NT = TL::NT, IPT = TL::IPT, CAP = TL::CAP, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const LocalLayout L = local_layout(CAP, NT, sizeof(K), VB, TL::FAST_BITS);
  K* skb = reinterpret_cast<K*>(smem_raw + L.sk);
  V* svb = reinterpret_cast<V*>(smem_raw + L.sv);
  uint32_t* si = reinterpret_cast<uint32_t*>(smem_raw + L.si);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw + L.cnt);
  uint4* u4tmp = reinterpret_cast<uint4*>(smem_raw + L.u4);
  __shared__ uint32_t s_tmp[NW + 1];
  __shared__ K s_diff[NW];
  __shared__ uint32_t s_nlarge;
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
  if (tid == 0) s_nlarge = 0;
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
  if (bits == 0) {
    if (S.src) {
      for (uint32_t i = tid; i < n; i += NT) {
        ok[i] = sk[i];
        if (VB) Av[S.offset + i] = sv[i];
      }
    }
    return;
  }

  bool done = false;
  if (bits <= TL::FAST_BITS) {
    const uint32_t D = 1u << bits;
    for (uint32_t d = tid; d < D; d += NT) cnt[d] = 0;
    __syncthreads();
    uint32_t dig[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      dig[i] = (uint32_t)key[i] & (D - 1);
      if (tid * IPT + i < n) atomicAdd(&cnt[dig[i]], 1u);
    }
    __syncthreads();
    // exclusive scan of the D digit counts (per-thread contiguous chunks)
    const uint32_t per = (D + NT - 1) / NT;
    const uint32_t d0 = min(D, tid * per), d1 = min(D, d0 + per);
    uint32_t sum = 0;
    for (uint32_t d = d0; d < d1; ++d) {
      const uint32_t c = cnt[d];
      sum += c;
      if (c > (uint32_t)FIXMAX) atomicAdd(&s_nlarge, 1u);
    }
    uint32_t total;
    uint32_t runv = block_exscan_val<NT>(sum, s_tmp, &total);
    for (uint32_t d = d0; d < d1; ++d) {
      const uint32_t c = cnt[d];
      cnt[d] = runv;
      runv += c;
    }
    __syncthreads();
    const uint32_t nlarge = s_nlarge;
    if (nlarge <= (uint32_t)NLARGE) {
      // large digits: exact slots; the large index = rank among large digits
      uint32_t li[IPT], rel[IPT];
      __shared__ uint32_t s_ldig[NLARGE], s_lcnt[NLARGE];
      if (nlarge) {
        if (tid == 0) {
          uint32_t k = 0;
          for (uint32_t d = 0; d < D && k < nlarge; ++d) {
            const uint32_t e = d + 1 < D ? cnt[d + 1] : n;
            if (e - cnt[d] > (uint32_t)FIXMAX) {
              s_ldig[k] = d;
              s_lcnt[k++] = e - cnt[d];
            }
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        li[i] = 0xFFu;
        for (uint32_t k = 0; k < nlarge; ++k)
          if (dig[i] == s_ldig[k]) li[i] = k;
        if (tid * IPT + i >= n) li[i] = 0xFFu;
      }
      if (nlarge) {
        // starts of the large digits must be read before atomics move cnt
        large_ranks<NT, IPT>(li, rel, u4tmp);
#pragma unroll
        for (int i = 0; i < IPT; ++i)
          if (li[i] != 0xFFu) rel[i] += cnt[dig[i]];
        __syncthreads();
      }
      // all keys are in registers: reuse sk / si for the sorted order
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const uint32_t e = tid * IPT + i;
        if (e < n) {
          const uint32_t slot = li[i] != 0xFFu ? rel[i] : atomicAdd(&cnt[dig[i]], 1u);
          sk[slot] = key[i];
          si[slot] = e;
        }
      }
      __syncthreads();
      // large digits took exact slots: move their cursor to the digit end
      if ((uint32_t)tid < nlarge) cnt[s_ldig[tid]] += s_lcnt[tid];
      __syncthreads();
      // equal keys back into input order: cnt[d] now holds the end of digit
      // d, its start is the end of digit d-1 (large digits advanced nothing:
      // skip them, their slots are exact)
      for (uint32_t d = tid; d < D; d += NT) {
        const uint32_t e = cnt[d];
        const uint32_t s = d ? cnt[d - 1] : 0u;
        if (e > s + 1 && e - s <= (uint32_t)FIXMAX) small_isort(si + s, e - s);
      }
      __syncthreads();
      done = true;
    }
  }
  if (!done) {
    // stable LSD passes of <= RB bits on (key, slot) pairs
    const int npass = (bits + TL::RB - 1) / TL::RB;
    const int pbits = (bits + npass - 1) / npass;
    uint32_t ix[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) ix[i] = tid * IPT + i;
    for (int pass = 0; pass < npass; ++pass) {
      const int sh = pass * pbits;
      const int pb = min(pbits, bits - sh);
      const uint32_t D = 1u << pb;
      uint32_t dig[IPT], rk[IPT];
#pragma unroll
      for (int i = 0; i < IPT; ++i)
        dig[i] = ix[i] < n ? (uint32_t)(key[i] >> sh) & (D - 1) : D - 1;
      block_rank_packed<NT, IPT>(dig, pb - 1, rk, cnt, s_tmp);
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        sk[rk[i]] = key[i];
        si[rk[i]] = ix[i];
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
  }
  for (uint32_t i = tid; i < n; i += NT) {
    ok[i] = sk[i];
    if (VB) Av[S.offset + i] = sv[si[i]];
  }
}

}  // namespace dts
