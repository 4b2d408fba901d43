// ORACLE — TEST INFRASTRUCTURE ONLY.  Never shipped, never on the product path.
//
// A CPU restatement (C++17 + OpenMP) of the reference DovetailSort package
// (/root/reference/pkg/src/dovetail, arXiv 2401.00710).  Only tests/,
// __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl
// reference arm) may load it, and only as the checker / the CPU baseline.
//
// Every function cites the reference file:line it follows.  The sampler
// reproduces numpy's Philox4x64-10 stream and Generator.integers bounded
// draws (Lemire, numpy/random/src/distributions) so the sample draws, the
// heavy-key sets and therefore the InstrumentReport counters equal the
// reference's — pinned by tests/golden (generated from the reference here).
//
// Payloads may be 0, 4 or 8 bytes (the reference takes u64 only; widening
// u32 payloads is lossless).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {
typedef struct ora_config {
  uint64_t seed;
  int32_t gamma_lo, gamma_hi;
  uint64_t base_case_threshold;
  int32_t theory_mode, base_case_exponent;
  int32_t mode;  // 0 dt_sort, 1 plain_msd_sort
  int32_t threads;
  uint64_t parallel_grain;
} ora_config;

typedef struct ora_report {
  uint64_t moves, merge_out_copies, merge_in_array_moves, base_case_records;
  int32_t levels, skipped_bits;
  uint64_t level_mass[64];
  uint64_t heavy_records_removed[64];
  int32_t level_mass_len, heavy_len;
  uint64_t records_distributed;  // D: records through counting_sort
} ora_report;
}

namespace {

// ---------------------------------------------------------------------------
// numpy Philox4x64-10 (numpy/random/src/philox/philox.h) and bounded ints
// ---------------------------------------------------------------------------
struct Philox {
  uint64_t ctr[4] = {0, 0, 0, 0};
  uint64_t key[2];
  uint64_t buf[4];
  int pos = 4;
  int has32 = 0;
  uint32_t u32 = 0;
  Philox(uint64_t k0, uint64_t k1) { key[0] = k0; key[1] = k1; }
  static inline uint64_t mulhilo(uint64_t a, uint64_t b, uint64_t* hi) {
    const unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    return (uint64_t)p;
  }
  void block() {
    uint64_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint64_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
      if (r) {
        k[0] += 0x9E3779B97F4A7C15ull;
        k[1] += 0xBB67AE8584CAA73Bull;
      }
      uint64_t hi0, hi1;
      const uint64_t lo0 = mulhilo(0xD2E7470EE14C6C93ull, c[0], &hi0);
      const uint64_t lo1 = mulhilo(0xCA5A826395121157ull, c[2], &hi1);
      const uint64_t n0 = hi1 ^ c[1] ^ k[0], n2 = hi0 ^ c[3] ^ k[1];
      c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
    for (int i = 0; i < 4; ++i) buf[i] = c[i];
  }
  uint64_t next64() {
    if (pos < 4) return buf[pos++];
    if (++ctr[0] == 0)
      if (++ctr[1] == 0)
        if (++ctr[2] == 0) ++ctr[3];
    block();
    pos = 1;
    return buf[0];
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = (uint32_t)(v >> 32);
    return (uint32_t)(v & 0xffffffffu);
  }
  // Generator.integers(0, high, dtype=uint64): rng = high - 1
  uint64_t bounded(uint64_t rng) {
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFull) {
      if (rng == 0xFFFFFFFFull) return next32();
      const uint32_t excl = (uint32_t)rng + 1u;
      uint64_t m = (uint64_t)next32() * excl;
      uint32_t left = (uint32_t)m;
      if (left < excl) {
        const uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % excl;
        while (left < thr) {
          m = (uint64_t)next32() * excl;
          left = (uint32_t)m;
        }
      }
      return m >> 32;
    }
    if (rng == ~0ull) return next64();
    const uint64_t excl = rng + 1;
    unsigned __int128 m = (unsigned __int128)next64() * excl;
    uint64_t left = (uint64_t)m;
    if (left < excl) {
      const uint64_t thr = (~0ull - rng) % excl;
      while (left < thr) {
        m = (unsigned __int128)next64() * excl;
        left = (uint64_t)m;
      }
    }
    return (uint64_t)(m >> 64);
  }
};

// ---------------------------------------------------------------------------
// core.py helpers
// ---------------------------------------------------------------------------
inline int bitlen(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

// ceil_log2 (core.py:98-103)
inline uint32_t ceil_log2(uint64_t n) { return n <= 2 ? 1 : (uint32_t)bitlen(n - 1); }

struct Cfg {
  ora_config c;
  // gamma_for (core.py:154-164)
  uint32_t gamma_for(uint64_t n, int remaining) const {
    const int raw = (bitlen(std::max<uint64_t>(n, 1)) - 1) / 3;
    const int clamped = std::min(c.gamma_hi, std::max(c.gamma_lo, raw));
    return (uint32_t)std::max(1, std::min(remaining, clamped));
  }
  // SortConfig.effective_theta (core.py:148-151)
  uint64_t theta(uint32_t g) const {
    if (c.theory_mode) {
      const uint64_t e = (uint64_t)c.base_case_exponent * g;
      return e >= 64 ? ~0ull : (1ull << e);
    }
    return c.base_case_threshold;
  }
};

struct Report {
  uint64_t moves = 0, out_copies = 0, in_moves = 0, base = 0, distributed = 0;
  int levels = 0, skipped = 0;
  std::vector<uint64_t> mass, heavy;
  void add_mass(size_t d, uint64_t c) {
    if (mass.size() <= d) mass.resize(d + 1, 0);
    mass[d] += c;
  }
  void add_heavy(size_t d, uint64_t c) {
    if (heavy.size() <= d) heavy.resize(d + 1, 0);
    heavy[d] += c;
  }
  void merge(const Report& o) {  // InstrumentReport.merge_from (core.py:198-210)
    moves += o.moves; out_copies += o.out_copies; in_moves += o.in_moves;
    levels = std::max(levels, o.levels); base += o.base; distributed += o.distributed;
    skipped = std::max(skipped, o.skipped);
    for (size_t d = 0; d < o.mass.size(); ++d) add_mass(d, o.mass[d]);
    for (size_t d = 0; d < o.heavy.size(); ++d) add_heavy(d, o.heavy[d]);
  }
};

// Stable sort of [0,n) of (k, p) by key: bottom-up merge, ties keep the
// left run first (bench.py:60-92 _merge_pass; equivalent to
// np.argsort(kind="stable") + gathers used by _base_sort, dtsort.py:127-147).
template <typename K, typename P>
void stable_sort(K* k, P* p, uint64_t n, bool has_pay) {
  if (n < 2) return;
  if (n <= 32) {  // insertion sort (stable)
    for (uint64_t i = 1; i < n; ++i) {
      const K x = k[i];
      const P y = has_pay ? p[i] : P();
      uint64_t j = i;
      while (j > 0 && k[j - 1] > x) {
        k[j] = k[j - 1];
        if (has_pay) p[j] = p[j - 1];
        --j;
      }
      k[j] = x;
      if (has_pay) p[j] = y;
    }
    return;
  }
  std::vector<K> tk(n);
  std::vector<P> tp(has_pay ? n : 0);
  K* ak = k; P* ap = p; K* bk = tk.data(); P* bp = tp.data();
  for (uint64_t width = 1; width < n; width *= 2) {
    for (uint64_t lo = 0; lo < n; lo += 2 * width) {
      const uint64_t mid = std::min(lo + width, n), hi = std::min(lo + 2 * width, n);
      uint64_t i = lo, j = mid, o = lo;
      while (i < mid && j < hi) {
        if (ak[j] < ak[i]) { bk[o] = ak[j]; if (has_pay) bp[o] = ap[j]; ++j; }
        else { bk[o] = ak[i]; if (has_pay) bp[o] = ap[i]; ++i; }
        ++o;
      }
      while (i < mid) { bk[o] = ak[i]; if (has_pay) bp[o] = ap[i]; ++i; ++o; }
      while (j < hi) { bk[o] = ak[j]; if (has_pay) bp[o] = ap[j]; ++j; ++o; }
    }
    std::swap(ak, bk);
    std::swap(ap, bp);
  }
  if (ak != k) {
    std::memcpy(k, ak, n * sizeof(K));
    if (has_pay) std::memcpy(p, ap, n * sizeof(P));
  }
}

// ---------------------------------------------------------------------------
// BucketPlan (sampler.py:49-118, plan_buckets :210-252)
// ---------------------------------------------------------------------------
template <typename K>
struct Plan {
  uint32_t gamma = 0, shift = 0, key_width = 0;
  std::vector<int32_t> light_ids;
  std::vector<K> heavy_keys;
  std::vector<int32_t> heavy_ids;
  std::vector<int64_t> zone_off;
  uint64_t nbuckets = 0;
  int64_t overflow_id = -1;
  uint64_t overflow_thr = 0;

  // bucket_ids / get_bucket_id (sampler.py:76-100): overflow > heavy > light
  inline int32_t bucket(K key) const {
    if (overflow_id >= 0 && (uint64_t)key >= overflow_thr) return (int32_t)overflow_id;
    const size_t m = heavy_keys.size();
    if (m) {
      const size_t pos = std::lower_bound(heavy_keys.begin(), heavy_keys.end(), key) - heavy_keys.begin();
      if (pos < m && heavy_keys[pos] == key) return heavy_ids[pos];
    }
    const uint64_t mask = (gamma >= 64) ? ~0ull : ((1ull << gamma) - 1);
    return light_ids[(size_t)(((uint64_t)key >> shift) & mask)];
  }
};

template <typename K>
Plan<K> plan_buckets(const std::vector<K>& heavy, uint32_t gamma, uint32_t shift, uint32_t w,
                     bool has_thr, uint64_t thr) {
  Plan<K> P;
  P.gamma = gamma; P.shift = shift; P.key_width = w;
  const uint64_t nz = 1ull << gamma;
  const size_t m = heavy.size();
  std::vector<int64_t> hz(m);
  std::vector<int64_t> per(nz, 0);
  for (size_t i = 0; i < m; ++i) {
    hz[i] = (int64_t)(((uint64_t)heavy[i] >> shift) & (nz - 1));
    per[hz[i]]++;
  }
  P.zone_off.assign(nz + 1, 0);
  for (uint64_t z = 0; z < nz; ++z) P.zone_off[z + 1] = P.zone_off[z] + per[z];
  P.light_ids.resize(nz);
  for (uint64_t z = 0; z < nz; ++z) P.light_ids[z] = (int32_t)(z + P.zone_off[z]);
  P.heavy_ids.resize(m);
  for (size_t i = 0; i < m; ++i)
    P.heavy_ids[i] = (int32_t)(P.light_ids[hz[i]] + 1 + ((int64_t)i - P.zone_off[hz[i]]));
  P.heavy_keys = heavy;
  P.nbuckets = nz + m;
  if (has_thr) {
    P.overflow_id = (int64_t)P.nbuckets;
    P.nbuckets += 1;
    P.overflow_thr = thr;
  }
  return P;
}

// ---------------------------------------------------------------------------
// counting_sort (counting.py:82-156): stable blocked counting sort
// ---------------------------------------------------------------------------
inline uint64_t default_block_count(uint64_t n, uint64_t nb, uint64_t workers) {
  // counting.py:49-55
  if (n < 2 * nb) return 1;
  const uint64_t per = std::max<uint64_t>(nb, 1024);
  return std::max<uint64_t>(1, std::min<uint64_t>((n + per - 1) / per, 8 * workers));
}

template <typename K, typename P, typename BucketOf>
void counting_sort(const K* keys, const P* pays, bool has_pay, uint64_t n, uint64_t nb,
                   K* out_k, P* out_p, uint64_t workers, bool par, BucketOf bucket_of,
                   std::vector<int64_t>& offsets_out) {
  offsets_out.assign(nb + 1, 0);
  if (n == 0) return;
  const uint64_t l = default_block_count(n, nb, workers);
  std::vector<uint64_t> bounds(l + 1);
  for (uint64_t j = 0; j <= l; ++j) bounds[j] = (uint64_t)((unsigned __int128)n * j / l);
  std::vector<int32_t> bids(n);
  std::vector<int64_t> counts(l * nb, 0);
  // phase 1: count (counting.py:123-137)
#pragma omp parallel for schedule(dynamic, 1) if (par && l > 1)
  for (uint64_t j = 0; j < l; ++j) {
    int64_t* row = counts.data() + j * nb;
    for (uint64_t i = bounds[j]; i < bounds[j + 1]; ++i) {
      const int32_t b = bucket_of(keys[i]);
      bids[i] = b;
      row[b]++;
    }
  }
  // phase 2: column-major exclusive offsets (counting.py:58-79)
  std::vector<int64_t> totals(nb, 0), starts(nb, 0);
  for (uint64_t j = 0; j < l; ++j)
    for (uint64_t b = 0; b < nb; ++b) totals[b] += counts[j * nb + b];
  for (uint64_t b = 1; b < nb; ++b) starts[b] = starts[b - 1] + totals[b - 1];
  std::vector<int64_t> offs(l * nb);
  for (uint64_t b = 0; b < nb; ++b) {
    int64_t run = starts[b];
    for (uint64_t j = 0; j < l; ++j) {
      offs[j * nb + b] = run;
      run += counts[j * nb + b];
    }
  }
  // phase 3: scatter_block per block (_kernels.py:12-25)
#pragma omp parallel for schedule(dynamic, 1) if (par && l > 1)
  for (uint64_t j = 0; j < l; ++j) {
    int64_t* run = offs.data() + j * nb;
    for (uint64_t i = bounds[j]; i < bounds[j + 1]; ++i) {
      const int64_t d = run[bids[i]]++;
      out_k[d] = keys[i];
      if (has_pay) out_p[d] = pays[i];
    }
  }
  for (uint64_t b = 0; b < nb; ++b) offsets_out[b + 1] = offsets_out[b] + totals[b];
}

// ---------------------------------------------------------------------------
// dt_merge (dtmerge.py:58-238)
// ---------------------------------------------------------------------------
template <typename K, typename P>
void reverse_range(K* k, P* p, bool hp, uint64_t lo, uint64_t hi) {  // _kernels.py:28-38
  if (hi <= lo) return;
  uint64_t i = lo, j = hi - 1;
  while (i < j) {
    std::swap(k[i], k[j]);
    if (hp) std::swap(p[i], p[j]);
    ++i; --j;
  }
}

template <typename K, typename P>
uint64_t shift_block(K* k, P* p, bool hp, uint64_t src, uint64_t len, uint64_t dest) {
  // dtmerge.py:81-105
  if (len == 0 || dest == src) return 0;
  reverse_range(k, p, hp, src, src + len);
  if (dest < src) reverse_range(k, p, hp, dest, src + len);
  else reverse_range(k, p, hp, src, dest + len);
  return 2 * len;
}

// returns 0 ok, else an error code (1 tile, 2 nonneg, 3 increasing, 4 sorted,
// 5 light run, 6 foreign, 7 scratch) — dtmerge.py:108-165
template <typename K, typename P>
int dt_merge(K* zk, P* zp, bool hp, uint64_t total, uint64_t light, const K* hk,
             const int64_t* hl, uint64_t m, K* sk, P* sp, uint64_t scratch_len, bool validate,
             uint64_t stats[3]) {
  stats[0] = stats[1] = stats[2] = 0;
  int64_t ht = 0;
  for (uint64_t i = 0; i < m; ++i) ht += hl[i];
  const uint64_t small = (uint64_t)std::min<int64_t>((int64_t)light, ht);
  if (scratch_len < small) return 7;
  if (validate) {
    if ((int64_t)light + ht != (int64_t)total) return 1;
    for (uint64_t i = 0; i < m; ++i) if (hl[i] < 0) return 2;
    for (uint64_t i = 1; i < m; ++i) if (!(hk[i] > hk[i - 1])) return 3;
    for (uint64_t i = 1; i < light; ++i) if (zk[i] < zk[i - 1]) return 4;
    if (m && light) {
      for (uint64_t i = 0; i < m; ++i) {
        uint64_t pos = std::lower_bound(zk, zk + light, hk[i]) - zk;
        pos = std::min<uint64_t>(pos, light - 1);
        if (zk[pos] == hk[i]) return 5;
      }
    }
    uint64_t off = light;
    for (uint64_t i = 0; i < m; ++i) {
      for (int64_t t = 0; t < hl[i]; ++t) if (zk[off + t] != hk[i]) return 6;
      off += (uint64_t)hl[i];
    }
  }
  if (m == 0 || total == 0) return 0;
  // compute_layout (dtmerge.py:58-78)
  std::vector<uint64_t> prefix(m + 1, 0), p(m), bounds(m + 2);
  for (uint64_t i = 0; i < m; ++i) prefix[i + 1] = prefix[i] + (uint64_t)hl[i];
  for (uint64_t i = 0; i < m; ++i) p[i] = std::lower_bound(zk, zk + light, hk[i]) - zk;
  bounds[0] = 0;
  for (uint64_t i = 0; i < m; ++i) bounds[i + 1] = p[i];
  bounds[m + 1] = light;
  uint64_t out = 0, in = 0, res = 0;
  auto copy = [&](K* dk, P* dp, const K* s_k, const P* s_p, uint64_t len) {
    std::memmove(dk, s_k, len * sizeof(K));
    if (hp) std::memmove(dp, s_p, len * sizeof(P));
  };
  if ((uint64_t)ht >= light) {  // dtmerge.py:178-207
    copy(sk, sp, zk, zp, light);
    out += light;
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t ln = (uint64_t)hl[i], src = light + prefix[i], dst = p[i] + prefix[i];
      if (ln == 0 || dst == src) continue;
      if (dst + ln <= src) {
        copy(zk + dst, hp ? zp + dst : nullptr, zk + src, hp ? zp + src : nullptr, ln);
        in += ln;
      } else {
        in += shift_block(zk, zp, hp, src, ln, dst);
      }
    }
    for (uint64_t i = 0; i <= m; ++i) {
      const uint64_t f0 = bounds[i], f1 = bounds[i + 1], fl = f1 - f0, dst = f0 + prefix[i];
      if (fl == 0 || dst == f0) continue;
      copy(zk + dst, hp ? zp + dst : nullptr, sk + f0, hp ? sp + f0 : nullptr, fl);
      res += fl;
    }
  } else {  // dtmerge.py:208-237
    copy(sk, sp, zk + light, hp ? zp + light : nullptr, (uint64_t)ht);
    out += (uint64_t)ht;
    for (uint64_t i = m; i >= 1; --i) {
      const uint64_t f0 = bounds[i], f1 = bounds[i + 1], fl = f1 - f0, dst = f0 + prefix[i];
      if (fl == 0 || dst == f0) continue;
      if (f0 + fl <= dst) {
        copy(zk + dst, hp ? zp + dst : nullptr, zk + f0, hp ? zp + f0 : nullptr, fl);
        in += fl;
      } else {
        in += shift_block(zk, zp, hp, f0, fl, dst);
      }
    }
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t ln = (uint64_t)hl[i];
      if (!ln) continue;
      copy(zk + p[i] + prefix[i], hp ? zp + p[i] + prefix[i] : nullptr, sk + prefix[i],
           hp ? sp + prefix[i] : nullptr, ln);
      res += ln;
    }
  }
  stats[0] = out; stats[1] = in; stats[2] = res;
  return 0;
}

// ---------------------------------------------------------------------------
// The sorter (dtsort.py)
// ---------------------------------------------------------------------------
constexpr uint64_t SAMPLE_CHUNK = 8192;   // sampler.py:37
constexpr uint64_t SAMPLE_TAG = 1ull << 60;  // sampler.py:38
constexpr uint64_t INLINE_CHILD_CUTOFF = 1ull << 18;  // dtsort.py:50

template <typename K, typename P>
struct Ctx {
  Cfg cfg;
  int mode;  // 0 dt, 1 plain
  uint32_t w;
  uint64_t n_total;
  K* keys[2];
  P* pays[2];
  bool hp;
  uint64_t workers;
};

template <typename K, typename P>
void base_sort(Ctx<K, P>& c, int buf, uint64_t lo, uint64_t hi, Report* r) {
  // _base_sort (dtsort.py:127-147)
  const uint64_t n = hi - lo;
  if (n == 0) return;
  if (r) r->base += n;
  if (n == 1) return;
  stable_sort(c.keys[buf] + lo, c.hp ? c.pays[buf] + lo : (P*)nullptr, n, c.hp);
  if (r) r->moves += n;
}

template <typename K, typename P>
void copy_between(Ctx<K, P>& c, int src, int dst, uint64_t lo, uint64_t hi) {
  // _copy_between (dtsort.py:111-124)
  std::memcpy(c.keys[dst] + lo, c.keys[src] + lo, (hi - lo) * sizeof(K));
  if (c.hp) std::memcpy(c.pays[dst] + lo, c.pays[src] + lo, (hi - lo) * sizeof(P));
}

// draw_samples (sampler.py:139-174)
template <typename K>
std::vector<K> draw_samples(const K* keys, uint64_t n_prime, uint32_t gamma, uint64_t n_total,
                            uint64_t seed, uint32_t depth, uint64_t base_index) {
  uint64_t count = std::min<uint64_t>(n_prime, (1ull << gamma) * ceil_log2(n_total));
  count = std::min(count, n_prime);
  std::vector<K> out(count);
  for (uint64_t c = 0, off = 0; off < count; ++c, off += SAMPLE_CHUNK) {
    const uint64_t cnt = std::min(SAMPLE_CHUNK, count - off);
    const uint64_t sid = SAMPLE_TAG | (((uint64_t)depth & 0xFF) << 48) |
                         ((base_index & 0xFFFFFFFFFFull) << 8) | (c & 0xFF);
    Philox g(seed, sid);
    for (uint64_t i = 0; i < cnt; ++i) out[off + i] = keys[g.bounded(n_prime - 1)];
  }
  std::sort(out.begin(), out.end());
  return out;
}

// detect_heavy (sampler.py:177-189)
template <typename K>
std::vector<K> detect_heavy(const std::vector<K>& s, uint64_t n_total) {
  std::vector<K> h;
  if (s.empty()) return h;
  const uint64_t st = ceil_log2(n_total);
  std::vector<K> sub;
  for (uint64_t i = 0; i < s.size(); i += st) sub.push_back(s[i]);
  for (size_t i = 0; i < sub.size();) {
    size_t j = i;
    while (j < sub.size() && sub[j] == sub[i]) ++j;
    if (j - i >= 2) h.push_back(sub[i]);
    i = j;
  }
  return h;
}

template <typename K, typename P>
int sort_rec(Ctx<K, P>& c, uint64_t lo, uint64_t hi, uint32_t consumed, uint32_t depth, int src,
             bool par, Report* rep);

template <typename K, typename P>
int sort_rec(Ctx<K, P>& c, uint64_t lo, uint64_t hi, uint32_t consumed, uint32_t depth, int src,
             bool par, Report* rep) {
  // _sort_rec (dtsort.py:150-209)
  const Cfg& cfg = c.cfg;
  const uint64_t n_sub = hi - lo;
  if (rep) rep->add_mass(depth, n_sub);
  if (n_sub == 0) return src;
  const int remaining = (int)c.w - (int)consumed;
  if (remaining <= 0) return src;
  uint32_t gamma = cfg.gamma_for(n_sub, remaining);
  if (n_sub < cfg.theta(gamma)) {
    base_sort(c, src, lo, hi, rep);
    return src;
  }
  // Step 1: _plan_step (dtsort.py:212-241)
  uint32_t shift = c.w - consumed - gamma;
  Plan<K> plan;
  bool planned = false;
  if (c.mode == 0) {
    const uint64_t sc = std::min<uint64_t>(n_sub, (1ull << gamma) * ceil_log2(c.n_total));
    if (!(n_sub < 2 * sc)) {
      std::vector<K> S = draw_samples(c.keys[src] + lo, n_sub, gamma, c.n_total, cfg.c.seed,
                                      depth, lo);
      bool has_thr = false;
      uint64_t thr = 0;
      if (depth == 0 && consumed == 0) {
        // plan_overflow (sampler.py:192-207)
        const uint64_t mx = S.empty() ? 0 : (uint64_t)S.back();
        const int clz = (int)c.w - bitlen(mx);
        int skip = (clz / (int)gamma) * (int)gamma;
        skip = std::min(skip, (((int)c.w - 1) / (int)gamma) * (int)gamma);
        if (skip > 0) {
          has_thr = true;
          thr = 1ull << (c.w - skip);
          consumed = (uint32_t)skip;
          gamma = std::min<uint32_t>(gamma, c.w - consumed);
          shift = c.w - consumed - gamma;
        }
      }
      std::vector<K> heavy = detect_heavy(S, c.n_total);
      plan = plan_buckets<K>(heavy, gamma, shift, c.w, has_thr, thr);
      planned = true;
    }
  }
  if (!planned) plan = plan_buckets<K>(std::vector<K>(), gamma, shift, c.w, false, 0);
  if (rep && depth == 0 && consumed > 0) rep->skipped = (int)consumed;

  // Step 2: distribute into the opposite buffer (dtsort.py:174-186)
  const int o = 1 - src;
  std::vector<int64_t> offs;
  counting_sort<K, P>(c.keys[src] + lo, c.hp ? c.pays[src] + lo : nullptr, c.hp, n_sub,
                      plan.nbuckets, c.keys[o] + lo, c.hp ? c.pays[o] + lo : nullptr, c.workers,
                      par, [&plan](K k) { return plan.bucket(k); }, offs);
  if (rep) {
    rep->moves += n_sub;
    rep->distributed += n_sub;
    rep->levels = std::max(rep->levels, (int)depth + 1);
    rep->add_mass(depth + 1, 0);
    uint64_t ovf = 0, light_total = 0;
    if (plan.overflow_id >= 0) ovf = offs[plan.overflow_id + 1] - offs[plan.overflow_id];
    for (auto b : plan.light_ids) light_total += offs[b + 1] - offs[b];
    rep->add_heavy(depth, n_sub - light_total - ovf);
  }

  // Step 3: _children_step (dtsort.py:244-318)
  const int remaining_after = (int)c.w - (int)consumed - (int)gamma;
  const bool children_done = remaining_after <= 0;
  struct Job { int kind; uint64_t a, b; };  // 0 span, 1 child, 2 overflow
  std::vector<Job> jobs;
  int64_t span_start = -1, span_end = -1;
  auto flush = [&]() {
    if (span_start >= 0 && span_end > span_start) jobs.push_back({0, (uint64_t)span_start, (uint64_t)span_end});
    span_start = span_end = -1;
  };
  if (!children_done) {
    const uint64_t nz = 1ull << plan.gamma;
    for (uint64_t z = 0; z < nz; ++z) {
      const int32_t b = plan.light_ids[z];
      const uint64_t clo = lo + offs[b], chi = lo + offs[b + 1];
      const uint64_t size = chi - clo;
      const int64_t h0 = plan.zone_off[z], h1 = plan.zone_off[z + 1];
      if (size > 0) {
        const uint32_t cg = cfg.gamma_for(size, remaining_after);
        if (size < cfg.theta(cg)) {
          if (span_start < 0) span_start = (int64_t)clo;
          span_end = (int64_t)chi;
        } else {
          flush();
          jobs.push_back({1, clo, chi});
        }
      }
      if (h1 > h0) flush();
    }
    flush();
  }
  if (plan.overflow_id >= 0) {
    const uint64_t alo = lo + offs[plan.overflow_id], ahi = lo + offs[plan.overflow_id + 1];
    if (ahi > alo) jobs.push_back({2, alo, ahi});
  }
  std::vector<Report> child_reps(rep ? jobs.size() : 0);
  auto run_job = [&](size_t ji, bool inline_par) {
    const Job& J = jobs[ji];
    Report* r = rep ? &child_reps[ji] : nullptr;
    if (J.kind == 0) {
      if (r) r->add_mass(depth + 1, J.b - J.a);
      base_sort(c, o, J.a, J.b, r);
    } else if (J.kind == 2) {
      base_sort(c, o, J.a, J.b, r);
    } else {
      const int buf = sort_rec(c, J.a, J.b, consumed + gamma, depth + 1, o, inline_par, r);
      if (buf != o) {
        copy_between(c, buf, o, J.a, J.b);
        if (r) r->moves += J.b - J.a;
      }
    }
  };
  if (par && jobs.size() > 1) {
    // pooled jobs in parallel; large children inline with their own
    // internal parallelism (parallel.py:63-81, dtsort.py:298-317)
    std::vector<size_t> pooled, inl;
    for (size_t i = 0; i < jobs.size(); ++i) {
      if (jobs[i].kind == 1 && jobs[i].b - jobs[i].a >= INLINE_CHILD_CUTOFF) inl.push_back(i);
      else pooled.push_back(i);
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (size_t t = 0; t < pooled.size(); ++t) run_job(pooled[t], false);
    for (size_t i : inl) run_job(i, true);
  } else {
    for (size_t i = 0; i < jobs.size(); ++i) run_job(i, par);
  }

  // Step 4: _merge_step (dtsort.py:321-354)
  uint64_t mo = 0, mi = 0, mr = 0;
  if (c.mode == 0 && !plan.heavy_keys.empty()) {
    const uint64_t nz = 1ull << plan.gamma;
    std::vector<uint64_t> zs;
    for (uint64_t z = 0; z < nz; ++z)
      if (plan.zone_off[z + 1] > plan.zone_off[z]) zs.push_back(z);
    std::vector<uint64_t> st(zs.size() * 3, 0);
#pragma omp parallel for schedule(dynamic, 1) if (par && zs.size() > 1)
    for (size_t t = 0; t < zs.size(); ++t) {
      const uint64_t z = zs[t];
      const int64_t h0 = plan.zone_off[z], h1 = plan.zone_off[z + 1];
      const int32_t b = plan.light_ids[z];
      const uint64_t cnt = (uint64_t)(h1 - h0);
      const uint64_t zlo = lo + offs[b], zhi = lo + offs[b + cnt + 1];
      if (zhi == zlo) continue;
      const uint64_t light = offs[b + 1] - offs[b];
      std::vector<int64_t> hl(cnt);
      for (uint64_t i = 0; i < cnt; ++i) hl[i] = offs[b + 2 + i] - offs[b + 1 + i];
      dt_merge<K, P>(c.keys[o] + zlo, c.hp ? c.pays[o] + zlo : nullptr, c.hp, zhi - zlo, light,
                     plan.heavy_keys.data() + h0, hl.data(), cnt, c.keys[src] + zlo,
                     c.hp ? c.pays[src] + zlo : nullptr, zhi - zlo, false, &st[3 * t]);
    }
    for (size_t t = 0; t < zs.size(); ++t) {
      mo += st[3 * t]; mi += st[3 * t + 1]; mr += st[3 * t + 2];
    }
  }
  if (rep) {
    for (auto& r : child_reps) rep->merge(r);
    rep->out_copies += mo;
    rep->in_moves += mi;
    rep->moves += mo + mi + mr;
  }
  return o;
}

template <typename K, typename P>
void run_sort(void* keys, void* pays, uint64_t n, const ora_config* cc, ora_report* out) {
  // _run (dtsort.py:81-108)
  Report rep;
  Report* r = out ? &rep : nullptr;
  if (n == 0) {
    if (r) r->add_mass(0, 0);
  } else {
    Ctx<K, P> c;
    c.cfg.c = *cc;
    c.mode = cc->mode;
    c.w = sizeof(K) * 8;
    c.n_total = n;
    c.hp = pays != nullptr;
    std::vector<K> tk(n);
    std::vector<P> tp(c.hp ? n : 0);
    c.keys[0] = (K*)keys; c.keys[1] = tk.data();
    c.pays[0] = (P*)pays; c.pays[1] = c.hp ? tp.data() : nullptr;
    int threads = 1;
#ifdef _OPENMP
    threads = cc->threads > 0 ? cc->threads : omp_get_max_threads();
    omp_set_num_threads(threads);
    omp_set_max_active_levels(1);
#endif
    c.workers = (uint64_t)threads;
    const bool par = threads > 1 && n >= cc->parallel_grain;
    const int buf = sort_rec(c, 0, n, 0, 0, 0, par, r);
    if (buf == 1) {
      copy_between(c, 1, 0, 0, n);
      if (r) r->moves += n;
    }
  }
  if (out) {
    std::memset(out, 0, sizeof(*out));
    out->moves = rep.moves;
    out->merge_out_copies = rep.out_copies;
    out->merge_in_array_moves = rep.in_moves;
    out->base_case_records = rep.base;
    out->levels = rep.levels;
    out->skipped_bits = rep.skipped;
    out->level_mass_len = (int)std::min<size_t>(64, rep.mass.size());
    for (int d = 0; d < out->level_mass_len; ++d) out->level_mass[d] = rep.mass[d];
    out->heavy_len = (int)std::min<size_t>(64, rep.heavy.size());
    for (int d = 0; d < out->heavy_len; ++d) out->heavy_records_removed[d] = rep.heavy[d];
    out->records_distributed = rep.distributed;
  }
}

}  // namespace

extern "C" {

// Stable in-place sort (dt_sort / plain_msd_sort, dtsort.py:64-108).
int ora_sort(void* keys, void* pays, uint64_t n, int kb, int pb, const ora_config* cfg,
             ora_report* rep) {
  if (kb == 4) {
    if (pb == 0) run_sort<uint32_t, uint64_t>(keys, nullptr, n, cfg, rep);
    else if (pb == 4) run_sort<uint32_t, uint32_t>(keys, pays, n, cfg, rep);
    else if (pb == 8) run_sort<uint32_t, uint64_t>(keys, pays, n, cfg, rep);
    else return -1;
  } else if (kb == 8) {
    if (pb == 0) run_sort<uint64_t, uint64_t>(keys, nullptr, n, cfg, rep);
    else if (pb == 4) run_sort<uint64_t, uint32_t>(keys, pays, n, cfg, rep);
    else if (pb == 8) run_sort<uint64_t, uint64_t>(keys, pays, n, cfg, rep);
    else return -1;
  } else {
    return -1;
  }
  return 0;
}

// dt_merge (dtmerge.py:132-238); returns 0 or the error code listed above.
int ora_dt_merge(void* zk, void* zp, uint64_t total, uint64_t light, const void* hk,
                 const int64_t* hl, uint64_t m, void* sk, void* sp, uint64_t scratch_len, int kb,
                 int pb, int validate, uint64_t stats[3]) {
  if (kb == 4) {
    if (pb == 4)
      return dt_merge<uint32_t, uint32_t>((uint32_t*)zk, (uint32_t*)zp, zp != nullptr, total, light, (const uint32_t*)hk, hl, m, (uint32_t*)sk, (uint32_t*)sp, scratch_len, validate, stats);
    return dt_merge<uint32_t, uint64_t>((uint32_t*)zk, (uint64_t*)zp, zp != nullptr, total, light, (const uint32_t*)hk, hl, m, (uint32_t*)sk, (uint64_t*)sp, scratch_len, validate, stats);
  }
  if (pb == 4)
    return dt_merge<uint64_t, uint32_t>((uint64_t*)zk, (uint32_t*)zp, zp != nullptr, total, light, (const uint64_t*)hk, hl, m, (uint64_t*)sk, (uint32_t*)sp, scratch_len, validate, stats);
  return dt_merge<uint64_t, uint64_t>((uint64_t*)zk, (uint64_t*)zp, zp != nullptr, total, light, (const uint64_t*)hk, hl, m, (uint64_t*)sk, (uint64_t*)sp, scratch_len, validate, stats);
}

// counting_sort with caller-supplied bucket ids (counting.py:82-156).
int ora_counting_sort(const void* keys, const void* pays, uint64_t n, int kb, int pb,
                      const int32_t* bids, uint64_t nb, void* out_k, void* out_p,
                      int64_t* offsets_out) {
  std::vector<int64_t> offs;
  // bucket ids are given per position: run the blocked sort sequentially
  // so position i maps to bids[i] (l = 1 block; output is block-count
  // invariant, test_counting.py:54-65).
  if (kb == 4 && pb == 8) {
    const uint32_t* k = (const uint32_t*)keys;
    uint64_t pos = 0;
    counting_sort<uint32_t, uint64_t>(k, (const uint64_t*)pays, pays != nullptr, n, nb,
                                      (uint32_t*)out_k, (uint64_t*)out_p, 1, false,
                                      [&](uint32_t) { return bids[pos++]; }, offs);
  } else if (kb == 4 && pb == 4) {
    uint64_t pos = 0;
    counting_sort<uint32_t, uint32_t>((const uint32_t*)keys, (const uint32_t*)pays, pays != nullptr, n, nb,
                                      (uint32_t*)out_k, (uint32_t*)out_p, 1, false,
                                      [&](uint32_t) { return bids[pos++]; }, offs);
  } else if (kb == 8 && pb == 8) {
    uint64_t pos = 0;
    counting_sort<uint64_t, uint64_t>((const uint64_t*)keys, (const uint64_t*)pays, pays != nullptr, n, nb,
                                      (uint64_t*)out_k, (uint64_t*)out_p, 1, false,
                                      [&](uint64_t) { return bids[pos++]; }, offs);
  } else {
    return -1;
  }
  for (uint64_t b = 0; b <= nb; ++b) offsets_out[b] = offs[b];
  return 0;
}

// reference_sort (bench.py:95-109): independent bottom-up stable mergesort.
int ora_reference_sort(void* keys, void* pays, uint64_t n, int kb, int pb) {
  if (kb == 4 && pb == 4) stable_sort((uint32_t*)keys, (uint32_t*)pays, n, pays != nullptr);
  else if (kb == 4) stable_sort((uint32_t*)keys, (uint64_t*)pays, n, pays != nullptr);
  else if (pb == 4) stable_sort((uint64_t*)keys, (uint32_t*)pays, n, pays != nullptr);
  else stable_sort((uint64_t*)keys, (uint64_t*)pays, n, pays != nullptr);
  return 0;
}

// numpy Philox check: first `cnt` bounded draws of Generator(Philox(key)).integers(0, high)
void ora_philox_integers(uint64_t k0, uint64_t k1, uint64_t high, uint64_t cnt, uint64_t* out) {
  Philox g(k0, k1);
  for (uint64_t i = 0; i < cnt; ++i) out[i] = g.bounded(high - 1);
}

int ora_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
