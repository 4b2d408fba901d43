// dts_api.cu — C ABI (include/dts.h) and the level-synchronous MSD scheduler.
//
// The scheduler replaces the reference's recursive driver
// (dtsort.py:81-209, `_run` / `_sort_rec` / `_children_step`): instead of one
// recursive call per subproblem it processes all subproblems of one MSD
// depth together — one sample / histogram / scan / scatter launch per level
// over every segment, one k_local_sort launch over every base-case span —
// and reads the level's bucket boundaries back to the host once per level to
// plan the next one.  Output is the unique stable sort, identical to the
// reference's.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dts.h"
#include "dts_local.cuh"
#include "dts_scatter.cuh"
#include "dts_scatter_wc.cuh"
#include "dts_graph.cuh"
#include "dts_morton.cuh"

using namespace dts;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(DTS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));      \
  } while (0)

#define DTS_TRY(expr)        \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != 0) return rc_; \
  } while (0)

// ---------------------------------------------------------------------------
// Tunables (B200-sized)
// ---------------------------------------------------------------------------
constexpr int HIST_NT = 512;
constexpr int SAMPLE_NT = 1024;
// scatter tile size per record width (ScatterTile<K, VB>::T) and the hist
// block = LB consecutive tiles (one count-matrix row, look-back depth < LB)
inline uint64_t scatter_T(int kb, int vb) { return (kb == 4 && vb <= 4) ? 512 * 9 : 512 * 5; }
inline uint64_t block_records(int kb, int vb) { return scatter_T(kb, vb) * 8; }
// write-combining scatter: stripe (= count-matrix row) of WC_LBS tiles
constexpr uint64_t WC_LBS = 44;  // ~315 K records (u32/u32 tiles of 7168): boundary cost vs last-wave imbalance
constexpr uint32_t COPY_CHUNK = 1u << 16;
constexpr size_t CLS_SIDE_MAX = 1024;  // waves of <= this many segments classify on the side stream
// sample iff n' >= SAMPLE_FACTOR x |S|.  The reference samples from 2|S|
// (dtsort.py:225); here small segments skip it: heavy keys found there save
// little, and each sampled segment costs a sample sort (output unaffected).
constexpr uint64_t SAMPLE_FACTOR = 32;
// ... and, below the root, small segments (< SAMPLE_MIN records) only when
// their parent had heavy keys or the level has <= SAMPLE_MANY segments: a
// heavy key of a small segment saves at most one small pass, while every
// sampled segment costs a sample sort, a plan read-back and host planning
// (C4 level 2: 0.6-1.3 x 10^5 segments of ~6-16 K records); skewed inputs
// (Zipf) keep finding heavy keys level after level in fewer segments
constexpr uint64_t SAMPLE_MIN = 1u << 17;
constexpr size_t SAMPLE_MANY = 8192;

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// DTS_TRACE=1: one stderr line per wave (host planning / wait / classify µs)
inline double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
inline bool trace_on() {
  static const int t = env_int("DTS_TRACE", 0);
  return t != 0;
}

// Local-sort capacity per record width (SMEM ~ CAP*(kb+vb+2) bytes).

// ---------------------------------------------------------------------------
// Pinned host staging (grown on demand at sync points)
// ---------------------------------------------------------------------------
struct Pinned {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 1 << 20);
    want = want + want / 2;
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess)
      return fail(DTS_ECUDA, "cudaHostAlloc failed for pinned staging");
    cap = want;
    return 0;
  }
};
thread_local Pinned g_pin_plan, g_pin_back, g_pin_span;

// Mapped pinned host memory (zero-copy): k_classify writes the next level's
// segment list straight into it, so the host has the whole list when the
// classifier's event fires — whatever its length, without a copy that
// would queue behind the scatter.
struct Mapped {
  void* p = nullptr;
  void* d = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFreeHost(p);
    p = d = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 1 << 20);
    want = want + want / 2;
    if (cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return fail(DTS_ECUDA, "cudaHostAlloc (mapped) failed for the next-segment list");
    if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess)
      return fail(DTS_ECUDA, "cudaHostGetDevicePointer failed for the next-segment list");
    cap = want;
    return 0;
  }
};
thread_local Mapped g_map_next;

// Per-thread, per-device side stream (high priority, non-blocking) for the
// classifier and the sorter's two fork / join events; created once and kept
// (creating them per call costs host microseconds at the start of a sort).
cudaStream_t side_stream(cudaEvent_t* ev_cls, cudaEvent_t* ev_fork) {
  struct Side {
    cudaStream_t st = nullptr;
    cudaEvent_t cls = nullptr, fork = nullptr;
  };
  static thread_local Side sides[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  Side& s = sides[dev];
  if (!s.st) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&s.st, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.cls, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess) {
      s.st = nullptr;
      return nullptr;
    }
  }
  *ev_cls = s.cls;
  *ev_fork = s.fork;
  return s.st;
}

int device_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// ---------------------------------------------------------------------------
// Launch bookkeeping: counts launches, optionally times each class with
// CUDA events on the launching stream.
// ---------------------------------------------------------------------------
struct Timer {
  cudaStream_t st;
  bool profile;
  dts_report* rep;
  uint64_t launches = 0;
  struct Ev {
    cudaEvent_t a, b;
    int cls;
  };
  std::vector<Ev> pending;
  std::vector<cudaEvent_t> pool;

  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void begin(int cls, Ev& ev) {
    ev.cls = cls;
    ev.a = ev.b = nullptr;
    if (!profile) return;
    ev.a = get();
    ev.b = get();
    cudaEventRecord(ev.a, st);
  }
  void end(Ev& ev, uint64_t records) {
    ++launches;
    if (rep) {
      rep->kernel_launches[ev.cls] += 1;
      rep->kernel_records[ev.cls] += records;
    }
    if (!profile) return;
    cudaEventRecord(ev.b, st);
    pending.push_back(ev);
  }
  void harvest() {  // call after a stream sync
    // DTS_TIMELINE=1 (profiled runs): every timed launch as start/end in ms
    // from the first one — the gaps between launches are host round trips
    static const int tl = env_int("DTS_TIMELINE", 0);
    if (tl && !pending.empty()) {
      static const char* names[] = {"sample", "hist", "scan", "scatter", "local", "copy", "bounds", "merge"};
      for (auto& e : pending) {
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, pending[0].a, e.a);
        cudaEventElapsedTime(&b, pending[0].a, e.b);
        std::fprintf(stderr, "[dts-timeline] %-8s %9.3f %9.3f ms\n", names[e.cls], a, b);
      }
    }
    for (auto& e : pending) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e.a, e.b);
      if (rep) rep->kernel_ms[e.cls] += ms;
      pool.push_back(e.a);
      pool.push_back(e.b);
    }
    pending.clear();
  }
  ~Timer() {
    for (auto& e : pending) {
      pool.push_back(e.a);
      pool.push_back(e.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

// Kernel attributes and occupancies are set / queried once per (thread,
// device, kernel, size) and cached: each driver call costs microseconds of
// host time that the GPU spends idle at the start of a level.
struct AttrKey {
  const void* fn;
  int dev, nt;
  size_t bytes;
  bool operator==(const AttrKey& o) const { return fn == o.fn && dev == o.dev && nt == o.nt && bytes == o.bytes; }
};
struct AttrHash {
  size_t operator()(const AttrKey& k) const {
    return std::hash<const void*>()(k.fn) ^ (std::hash<size_t>()(k.bytes) * 31u) ^ (size_t)(k.dev * 131 + k.nt);
  }
};
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

template <typename F>
int set_smem(F* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    static thread_local std::unordered_map<AttrKey, int, AttrHash> done;
    const AttrKey key{(const void*)fn, current_device(), 0, bytes};
    if (done.count(key)) return 0;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess)
      return fail(DTS_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    done.emplace(key, 1);
  }
  return 0;
}

template <typename F>
int persistent_grid(F* fn, int nt, size_t smem, uint32_t nblk) {
  static thread_local std::unordered_map<AttrKey, int, AttrHash> occ;
  const AttrKey key{(const void*)fn, current_device(), nt, smem};
  auto it = occ.find(key);
  int per = 0;
  if (it != occ.end()) {
    per = it->second;
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, nt, smem);
    if (per < 1) per = 1;
    occ.emplace(key, per);
  }
  const uint64_t g = (uint64_t)per * device_sms();
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(g, nblk));
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DTS_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

// ---------------------------------------------------------------------------
// Meta-region bump allocator over the caller's workspace.
// ---------------------------------------------------------------------------
struct Bump {
  char* base;
  size_t cap, off = 0;
  void* take(size_t bytes) {
    size_t o = align256(off);
    if (o + bytes > cap) return nullptr;
    off = o + bytes;
    return base + o;
  }
};

// Level metadata bound: count matrix / scan / bounds (~n/4 B) plus the
// scatter's look-back status (one u32 per tile per bucket column; tiles hold
// >= 2560 records, columns <= 1024) — about 1.9 B per record at most.
size_t meta_bytes(uint64_t n) {
  // (independent of the widths: 4/4 has the smallest blocks and 8/8 the
  // smallest tiles, both bounds are used)
  // count matrix (u32) + scan (u64) per block row and bucket column, plus the
  // look-back status (u32 per tile and column); columns <= 1024
  const uint64_t rows = n / block_records(4, 4) + 2;
  const uint64_t tiles = n / 2560 + 2 * rows + 2;
  return (size_t(64) << 20) + (size_t)(rows * 1024 * 12) + (size_t)(tiles * 1024 * 4);
}

struct HostSeg {  // same layout as the device's NextSeg (bulk-copied)
  uint64_t offset, len;
  uint32_t consumed;
  uint32_t root;
};
static_assert(sizeof(HostSeg) == sizeof(NextSeg), "HostSeg mirrors NextSeg");

// Flat exclusive scan of `e` u32 counts into u64 offsets.
int flat_scan(const uint32_t* cnt, uint64_t e, uint64_t* out, uint64_t* partial, Timer& tm) {
  if (e == 0) return 0;
  const uint64_t nch = (e + SCAN_CHUNK - 1) / SCAN_CHUNK;
  Timer::Ev ev;
  tm.begin(DTS_K_SCAN, ev);
  k_scan_reduce<<<(unsigned)nch, SCAN_NT, 0, tm.st>>>(cnt, e, partial);
  k_scan_spine<<<1, 1024, 0, tm.st>>>(partial, (uint32_t)nch);
  k_scan_down<<<(unsigned)nch, SCAN_NT, 0, tm.st>>>(cnt, e, partial, out);
  tm.end(ev, e);
  tm.launches += 2;
  return check_launch("k_scan");
}

// ---------------------------------------------------------------------------
// The sort
// ---------------------------------------------------------------------------
template <typename K, int VB>
struct Sorter {
  using V = typename ValOf<VB>::T;
  static constexpr int W = sizeof(K) * 8;

  K* Ak;
  V* Av;
  K* Tk;
  V* Tv;
  uint16_t* bid = nullptr;  // bucket ids of heavy segments' records (k_histogram -> k_scatter_wc)
  uint64_t n;
  Bump meta;
  dts_config cfg;
  dts_report* rep;
  Timer& tm;
  cudaStream_t st;
  cudaEvent_t ev_cls = nullptr;  // after k_classify's read-back of a wave
  cudaEvent_t ev_fork = nullptr;  // bucket bounds ready (side stream may classify)
  cudaStream_t side = nullptr;    // k_classify + its read-back, beside the scatter

  int cap;        // local-sort capacity (records)
  uint64_t thr;   // base-case threshold (records <= thr -> k_local_sort)
  uint32_t gcap, glo;
  uint32_t gcap_hw;  // log2 of the scatter's bucket capacity
  uint32_t stride;  // ceil_log2(n) (sampler.py:121-127)
  uint32_t gs_max, smax;
  bool no_uniq_skip = false;  // DTS_UNIQ_SKIP=0: sample children of unique-sample parents too

  // span / copy batches (host), flushed per level
  std::vector<Span> spans;
  std::vector<CopyR> copies;
  Span cur{0, 0, 0};
  bool have_cur = false;

  Sorter(Timer& t) : tm(t) {}

  // Digit width of a segment: just enough buckets for children of ~thr/2
  // records (the reference's γ_lo floor, core.py:156-164, is not applied:
  // small segments split into few, large buckets — fewer, longer runs;
  // the output does not depend on γ).
  uint32_t choose_gamma(uint64_t len, uint32_t remaining) const {
    const uint64_t target = std::max<uint64_t>(1, thr / 2);
    uint32_t need = ceil_log2_u64((len + target - 1) / target);
    // (a segment just above the base case is usually rich in duplicates —
    // near-unique keys would have fitted: a 2-bit digit per level leaves
    // skewed inputs a tail of levels that are all launch latency, Zipf 1.0:
    // levels 3-7 hold 5 % of the records; at least gamma_min bits at once)
    static const uint32_t gamma_min = (uint32_t)env_int("DTS_GAMMA_MIN", 6);
    need = std::max(need, gamma_min);
    uint32_t g = std::min(need, gcap);
    g = std::min(g, remaining);
    return std::max<uint32_t>(g, 1);
  }

  // dt_sort sampling decision (dtsort.py:225-228: sample only when the
  // segment holds at least SAMPLE_FACTOR x the sample).  Adjusts g (<= 9)
  // and returns the subsample exponent gs (|S| = 2^gs * stride).
  // Below the root the strided subsample has <= 2^7 entries (heavy keys of
  // >= 1/128 of a segment): each sampled segment sorts its sample in one CTA.
  bool sampled_plan(uint64_t len, uint32_t remaining, uint32_t& g, uint32_t& gs, bool root,
                    bool small_ok, bool parent_unique = false) const {
    // (a parent whose own sample held no repeated key — near-unique keys
    // such as C2 — has no key frequent enough to be heavy in a child, up to
    // the birthday test's resolution: its children skip the sample)
    const uint32_t g9 = std::min<uint32_t>(g, gcap_hw > 1 ? gcap_hw - 1 : 1);
    if (!root && parent_unique && !no_uniq_skip) {
      g = std::min(g9, remaining);  // (the digit a sampled plan would get: the WC scatter's)
      return false;
    }
    gs = std::min<uint32_t>(g9 > 1 ? g9 - 1 : 1, root ? gs_max : std::min<uint32_t>(gs_max, 7));
    uint64_t S = std::min<uint64_t>(len, (uint64_t(1) << gs) * stride);
    S = std::min<uint64_t>(S, smax);
    if (len < SAMPLE_FACTOR * S || (!root && !small_ok && len < SAMPLE_MIN)) return false;
    g = std::min(g9, remaining);
    gs = std::min<uint32_t>(gs, g > 1 ? g - 1 : 1);
    return true;
  }

  // The base case over a span list (count device-resident): k_local_sort,
  // then the 8-bit-field retry (k_local_sort<.., true>) of the spans whose
  // 4-bit counting pass would carry — duplicate-rich spans, queued on the
  // device by the first launch — so the common path's code stays as it is.
  int local_sort_launch(const Span* dsp, const uint32_t* dn, uint64_t cap, uint32_t grid_hint, uint64_t recs) {
    static const int retry = env_int("DTS_LOCAL_RETRY", 1);
    constexpr int NT = LocalTile<K, VB>::NT;
    const size_t sm = LocalSmem<K, VB>::total;
    Span* rq = nullptr;
    uint32_t* rqn = nullptr;
    if (retry) {
      rq = (Span*)meta.take(std::max<uint64_t>(1, cap) * sizeof(Span));
      rqn = (uint32_t*)meta.take(16);
      if (!rq || !rqn) return fail(DTS_ENOMEM, "workspace too small for the local-sort retry queue");
      CUDA_TRY(cudaMemsetAsync(rqn, 0, 4, st));
    }
    {
      Timer::Ev ev;
      tm.begin(DTS_K_LOCAL, ev);
      auto fn = k_local_sort<K, VB, false>;
      DTS_TRY(set_smem(fn, sm));
      const int grid = persistent_grid(fn, NT, sm, grid_hint);
      fn<<<grid, NT, sm, st>>>(dsp, dn, Ak, Av, Tk, Tv, rq, rqn);
      tm.end(ev, recs);
      DTS_TRY(check_launch("k_local_sort"));
    }
    if (retry) {
      Timer::Ev ev;
      tm.begin(DTS_K_LOCAL, ev);
      auto fr = k_local_sort<K, VB, true>;
      DTS_TRY(set_smem(fr, sm));
      const int grid = persistent_grid(fr, NT, sm, grid_hint);
      fr<<<grid, NT, sm, st>>>(rq, rqn, Ak, Av, Tk, Tv, nullptr, nullptr);
      tm.end(ev, 0);
      DTS_TRY(check_launch("k_local_sort (retry)"));
    }
    return 0;
  }

  void flush_span() {
    if (have_cur && cur.len) {
      cur.src |= SPAN_NOBOUND << 8;  // (host spans: key bound unknown)
      spans.push_back(cur);
    }
    have_cur = false;
  }
  void add_span(uint64_t lo, uint64_t sz, uint32_t src) {
    if (have_cur && cur.src == src && cur.offset + cur.len == lo && cur.len + sz <= thr) {
      cur.len += (uint32_t)sz;
      return;
    }
    flush_span();
    cur = Span{lo, (uint32_t)sz, src};
    have_cur = true;
  }
  void add_copy(uint64_t lo, uint64_t sz) {
    for (uint64_t o = 0; o < sz; o += COPY_CHUNK) {
      CopyR r;
      r.offset = lo + o;
      r.len = (uint32_t)std::min<uint64_t>(COPY_CHUNK, sz - o);
      r.pad = 0;
      copies.push_back(r);
    }
  }

  // Host-built spans/copies (the whole-input base case): copy the lists and
  // their counts to the device and launch.
  int launch_spans_and_copies() {
    flush_span();
    if (spans.empty() && copies.empty()) return 0;
    const size_t sb = spans.size() * sizeof(Span), cb = copies.size() * sizeof(CopyR);
    DTS_TRY(g_pin_span.ensure(512 + align256(sb) + cb + 512));
    char* hp = (char*)g_pin_span.p;
    uint32_t* hcnt = (uint32_t*)hp;
    hcnt[0] = (uint32_t)spans.size();
    hcnt[1] = (uint32_t)copies.size();
    std::memcpy(hp + 512, spans.data(), sb);
    std::memcpy(hp + 512 + align256(sb), copies.data(), cb);
    size_t save = meta.off;
    uint32_t* dcnt = (uint32_t*)meta.take(16);
    Span* dsp = (Span*)meta.take(std::max<size_t>(1, spans.size()) * sizeof(Span));
    CopyR* dcp = (CopyR*)meta.take(std::max<size_t>(1, copies.size()) * sizeof(CopyR));
    if (!dcnt || !dsp || !dcp) return fail(DTS_ENOMEM, "workspace too small for span descriptors");
    CUDA_TRY(cudaMemcpyAsync(dcnt, hp, 8, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dsp, hp + 512, sb, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dcp, hp + 512 + align256(sb), cb, cudaMemcpyHostToDevice, st));
    uint64_t recs = 0;
    for (const Span& x : spans) recs += x.len;
    if (!spans.empty()) {
      DTS_TRY(local_sort_launch(dsp, dcnt, spans.size(), (uint32_t)spans.size(), recs));
      if (rep) {
        rep->base_case_records += recs;
        rep->moves += recs;
      }
    }
    if (!copies.empty()) {
      uint64_t crecs = 0;
      for (const CopyR& x : copies) crecs += x.len;
      Timer::Ev ev;
      tm.begin(DTS_K_COPY, ev);
      k_copy_ranges<K, VB><<<(unsigned)std::min<size_t>(copies.size(), device_sms() * 4), 256, 0, st>>>(
          dcp, dcnt + 1, Ak, Av, Tk, Tv);
      tm.end(ev, crecs);
      DTS_TRY(check_launch("k_copy_ranges"));
      if (rep) rep->moves += crecs;
    }
    // the pinned staging is reused: make sure the copies above have landed
    CUDA_TRY(cudaStreamSynchronize(st));
    meta.off = save;
    spans.clear();
    copies.clear();
    return 0;
  }

  // One wave: a subset of one level's segments processed by one set of launches.
  int run_wave(const std::vector<HostSeg>& segs, size_t s0, size_t s1, int level, bool in_T,
               std::vector<HostSeg>& next) {
    const size_t ns = s1 - s0;
    const bool dt = cfg.mode == DTS_MODE_DT;
    const double t_plan0 = trace_on() ? now_us() : 0.0;
    const K* ink = in_T ? Tk : Ak;
    const V* inv = in_T ? Tv : Av;
    K* outk = in_T ? Ak : Tk;
    V* outv = in_T ? Av : Tv;
    // ---- host plans (digit, sampling decision, table pools) ----
    std::vector<SegPlan> plans(ns);
    std::vector<uint32_t> sampled;
    uint64_t heavy_total = 0, hz_total = 0, scanbase = 0, wave_recs = 0;
    uint32_t hzc = 0, hkc = 0;
    for (size_t i = 0; i < ns; ++i) {
      const HostSeg& hs = segs[s0 + i];
      SegPlan& P = plans[i];
      std::memset(&P, 0, sizeof(P));
      const uint32_t remaining = W - hs.consumed;
      uint32_t g = choose_gamma(hs.len, remaining);
      P.offset = hs.offset;
      P.len = hs.len;
      P.scanbase = scanbase;
      scanbase += hs.len;
      wave_recs += hs.len;
      P.gamma = g;
      P.shift = remaining - g;
      P.consumed = hs.consumed;
      P.nb = 1u << g;
      P.nbmax = P.nb;
      uint32_t gs = 0;
      if (dt && sampled_plan(hs.len, remaining, g, gs, (hs.root & 1u) && hs.consumed == 0,
                             (hs.root & 2u) != 0 || segs.size() <= SAMPLE_MANY, (hs.root & 4u) != 0)) {
        // sampled segments may gain heavy / overflow buckets; the digit is
        // capped so bucket ids stay below the scatter's 2^10 capacity
        P.gamma = g;
        P.shift = remaining - g;
        P.flags |= PF_SAMPLE;
        P.sample_gs = gs;
        if ((hs.root & 1u) && hs.consumed == 0) P.flags |= PF_ROOTSKIP;
        P.nb = 1u << g;
        P.nbmax = (1u << g) + (1u << gs) + 1u;
        P.heavy_base = (uint32_t)heavy_total;
        heavy_total += (1u << gs);
        P.hz_base = (uint32_t)hz_total;
        hz_total += (1u << g) + 1u;
        sampled.push_back((uint32_t)i);
        hzc = std::max(hzc, (1u << g) + 1u);
        hkc = std::max(hkc, 1u << gs);
      } else if (g != P.gamma) {  // (not sampled, digit capped for the WC scatter)
        P.gamma = g;
        P.shift = remaining - g;
        P.nb = P.nbmax = 1u << g;
      }
    }
    const size_t save = meta.off;
    const double t_p1 = trace_on() ? now_us() : 0.0;
    const size_t pb = ns * sizeof(SegPlan), sb = sampled.size() * 4;
    SegPlan* dplans = (SegPlan*)meta.take(pb);
    uint32_t* dsampled = (uint32_t*)meta.take(std::max<size_t>(1, sampled.size()) * 4);
    K* dheavy = (K*)meta.take(std::max<uint64_t>(1, heavy_total) * sizeof(K));
    uint32_t* dhz = (uint32_t*)meta.take(std::max<uint64_t>(1, hz_total) * 4);
    uint32_t* dctr = (uint32_t*)meta.take(16);
    if (!dplans || !dsampled || !dheavy || !dhz || !dctr)
      return fail(DTS_ENOMEM, "workspace too small for level metadata");

    // ---- sample + plan (sampler.py:121-252); the resolved plans come back
    // so the scatter variant and the count-matrix shape fit the real bucket
    // counts ----
    static const int wc_env = env_int("DTS_WC", 1);
    static const int wide_env = env_int("DTS_WC_WIDE", 1);
    // sampler: the columns of the write-combining scatter | its wide variant's << 16
    const uint32_t wc_cols =
        (uint32_t)WcTile<K, VB>::NBW | (wide_env ? (uint32_t)WcTile<K, VB, 1>::NBW << 16 : 0u);
    if (!sampled.empty()) {
      DTS_TRY(g_pin_plan.ensure(align256(pb) + sb + 512));
      char* hp = (char*)g_pin_plan.p;
      std::memcpy(hp, plans.data(), pb);
      std::memcpy(hp + align256(pb), sampled.data(), sb);
      CUDA_TRY(cudaMemcpyAsync(dplans, hp, pb, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(dsampled, hp + align256(pb), sb, cudaMemcpyHostToDevice, st));
      Timer::Ev ev;
      tm.begin(DTS_K_SAMPLE, ev);
      auto fn = k_sample_plan<K, SAMPLE_NT>;
      const size_t sm = (size_t)smax * sizeof(K);
      DTS_TRY(set_smem(fn, sm));
      fn<<<(unsigned)sampled.size(), SAMPLE_NT, sm, st>>>(dplans, dsampled, ink, dheavy, dhz,
                                                           cfg.seed, (uint32_t)level, stride,
                                                           gs_max, smax, wc_cols);
      tm.end(ev, sampled.size());
      DTS_TRY(check_launch("k_sample_plan"));
      if (wc_env) {
        DTS_TRY(g_pin_back.ensure(pb + 256));
        CUDA_TRY(cudaMemcpyAsync(g_pin_back.p, dplans, pb, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        std::memcpy(plans.data(), g_pin_back.p, pb);
      } else {
        // (DTS_WC=0, a debugging path: the pinned plan staging is rewritten
        // below — the copies above must have left it)
        CUDA_TRY(cudaStreamSynchronize(st));
      }
    }
    // the write-combining scatter takes waves whose bucket columns fit its
    // SMEM carries; its count-matrix rows are whole stripes
    uint32_t nbc = 2;
    for (size_t i = 0; i < ns; ++i) {
      const bool known = !(plans[i].flags & PF_SAMPLE) || wc_env;
      nbc = std::max(nbc, known ? plans[i].nb : plans[i].nbmax);
    }
    nbc = (nbc + 1) & ~1u;
    // (the wide variant takes heavy-key-rich waves of up to 600 columns)
    const bool wc = wc_env != 0 && nbc <= (wide_env ? (uint32_t)WcTile<K, VB, 1>::NBW : (uint32_t)WcTile<K, VB>::NBW);
    // (and every wave with heavy keys: the variant writes the many chunk
    // descriptors of a heavy bucket cooperatively)
    bool any_heavy = false;
    for (size_t i = 0; i < ns && !any_heavy; ++i) any_heavy = (plans[i].flags & PF_HEAVY) != 0;
    const bool wide = wc && wide_env && (nbc > (uint32_t)WcTile<K, VB>::NBW || any_heavy);
    const uint64_t WT = wide ? (uint64_t)WcTile<K, VB, 1>::T : (uint64_t)WcTile<K, VB>::T;
    static const int wc_lbs_env = env_int("DTS_WC_LBS", 0);
    const uint64_t wc_lbs = wc_lbs_env > 0 ? (uint64_t)wc_lbs_env : WC_LBS;
    const uint64_t BR = wc ? WT * wc_lbs : block_records(sizeof(K), VB);
    const uint64_t TT = wc ? WT : (uint64_t)ScatterTile<K, VB>::T;
    const double t_p2 = trace_on() ? now_us() : 0.0;
    // ---- count-matrix shape and hist blocks ----
    // Stripes (WC) go to one persistent CTA per SM in order: the wave gets
    // a multiple of the CTA count of about WC_LBS tiles each, shared out
    // over its segments in proportion to their length (largest remainders),
    // so the last round of stripes keeps every SM busy (C2 level 0: 44-tile
    // stripes gave 3171 = 21 x 148 + 63 — 85 SMs idle for the last stripe).
    std::vector<uint64_t> seg_rows(ns);
    if (wc && wc_lbs_env <= 0) {
      const uint64_t G = (uint64_t)device_sms();
      uint64_t total_tiles = 0;
      for (size_t i = 0; i < ns; ++i) total_tiles += (plans[i].len + TT - 1) / TT;
      const uint64_t k = std::max<uint64_t>(1, (total_tiles + G * WC_LBS / 2) / (G * WC_LBS));
      const uint64_t R = std::max<uint64_t>(G * k, 1);
      std::vector<std::pair<double, size_t>> frac;
      uint64_t given = 0;
      for (size_t i = 0; i < ns; ++i) {
        const double want = (double)plans[i].len * (double)R / (double)std::max<uint64_t>(wave_recs, 1);
        const uint64_t tiles = std::max<uint64_t>(1, (plans[i].len + TT - 1) / TT);
        seg_rows[i] = std::min<uint64_t>(tiles, std::max<uint64_t>(1, (uint64_t)want));
        given += seg_rows[i];
        if (seg_rows[i] < tiles) frac.emplace_back(want - std::floor(want), i);
      }
      if (given < R) {
        const size_t extra = std::min<size_t>(frac.size(), (size_t)(R - given));
        std::partial_sort(frac.begin(), frac.begin() + extra, frac.end(),
                          [](const std::pair<double, size_t>& x, const std::pair<double, size_t>& y) {
                            return x.first > y.first;
                          });
        for (size_t j = 0; j < extra; ++j) ++seg_rows[frac[j].second];
      }
    } else {
      for (size_t i = 0; i < ns; ++i) seg_rows[i] = std::max<uint64_t>(1, (plans[i].len + BR - 1) / BR);
    }
    std::vector<Blk> blks;
    blks.reserve(ns + wave_recs / BR + 1);
    uint64_t cnt_total = 0, bs_total = 0;
    for (size_t i = 0; i < ns; ++i) {
      SegPlan& P = plans[i];
      const uint64_t len = P.len;
      // whole tiles per block, no empty blocks
      const uint64_t per0 = ((len + seg_rows[i] - 1) / seg_rows[i] + TT - 1) / TT * TT;
      const uint64_t rows = std::max<uint64_t>(1, (len + per0 - 1) / per0);
      if (wc_env && (P.flags & PF_SAMPLE)) P.nbmax = P.nb;  // resolved
      P.nrows = (uint32_t)rows;
      P.cnt_base = cnt_total;
      cnt_total += (uint64_t)P.nbmax * rows;
      P.bs_base = (uint32_t)bs_total;
      bs_total += P.nbmax + 1;
      const uint64_t per = per0;
      for (uint64_t r = 0; r < rows; ++r) {
        Blk b;
        b.seg = (uint32_t)i;
        b.row = (uint32_t)r;
        b.begin = P.offset + std::min(len, r * per);
        b.end = P.offset + std::min(len, (r + 1) * per);
        blks.push_back(b);
      }
    }
    Caps caps{nbc, hzc, hkc, 0};
    // look-back scatter: tiles in input order (each hist block split into tiles)
    constexpr uint32_t ST_T = ScatterTile<K, VB>::T;
    std::vector<uint32_t> blk_tile0;
    std::vector<uint32_t> tile_blk;
    uint64_t ntile = 0;
    if (!wc) {
      blk_tile0.resize(blks.size());
      for (size_t bi = 0; bi < blks.size(); ++bi) {
        blk_tile0[bi] = (uint32_t)ntile;
        ntile += (blks[bi].end - blks[bi].begin + ST_T - 1) / ST_T;
      }
      tile_blk.resize(ntile);
      for (size_t bi = 0; bi < blks.size(); ++bi) {
        const uint32_t e = bi + 1 < blks.size() ? blk_tile0[bi + 1] : (uint32_t)ntile;
        for (uint32_t t = blk_tile0[bi]; t < e; ++t) tile_blk[t] = (uint32_t)bi;
      }
    }

    const double t_p3 = trace_on() ? now_us() : 0.0;
    // ---- device meta ----
    Blk* dblks = (Blk*)meta.take(blks.size() * sizeof(Blk));
    uint32_t* dcnt = (uint32_t*)meta.take(cnt_total * 4);
    uint64_t* dscan = (uint64_t*)meta.take(cnt_total * 8);
    const uint64_t nch = (cnt_total + SCAN_CHUNK - 1) / SCAN_CHUNK;
    uint64_t* dpart = (uint64_t*)meta.take(std::max<uint64_t>(1, nch) * 8);
    uint64_t* dbs = (uint64_t*)meta.take(bs_total * 8);
    uint8_t* dkinds = (uint8_t*)meta.take(bs_total);
    uint16_t* dzones = (uint16_t*)meta.take(bs_total * 2);
    uint32_t* dtile_blk = (uint32_t*)meta.take(std::max<uint64_t>(1, ntile) * 4);
    uint32_t* dblk_tile0 = (uint32_t*)meta.take(std::max<size_t>(1, blk_tile0.size()) * 4);
    uint32_t* dstatus = (uint32_t*)meta.take(std::max<uint64_t>(1, ntile) * (nbc / 2) * 4);
    if (!dblks || !dcnt || !dscan || !dpart || !dbs || !dkinds || !dzones || !dtile_blk || !dblk_tile0 ||
        !dstatus)
      return fail(DTS_ENOMEM, "workspace too small for level metadata");

    // ---- H2D ----
    const size_t bb = blks.size() * sizeof(Blk);
    const size_t tb = ntile * 4, b0b = blk_tile0.size() * 4;
    DTS_TRY(g_pin_plan.ensure(align256(pb) + align256(bb) + align256(sb) + align256(tb) + b0b + 512));
    char* hp = (char*)g_pin_plan.p;
    std::memcpy(hp, plans.data(), pb);
    std::memcpy(hp + align256(pb), blks.data(), bb);
    if (sb) std::memcpy(hp + align256(pb) + align256(bb), sampled.data(), sb);
    char* htl = hp + align256(pb) + align256(bb) + align256(sb);
    if (!wc) {
      std::memcpy(htl, tile_blk.data(), tb);
      std::memcpy(htl + align256(tb), blk_tile0.data(), b0b);
      CUDA_TRY(cudaMemcpyAsync(dtile_blk, htl, tb, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(dblk_tile0, htl + align256(tb), b0b, cudaMemcpyHostToDevice, st));
    }
    const bool sample_later = !sampled.empty() && !wc_env;
    CUDA_TRY(cudaMemcpyAsync(dplans, hp, pb, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dblks, hp + align256(pb), bb, cudaMemcpyHostToDevice, st));
    if (sample_later) {
      // DTS_WC=0: plans (with the count-matrix shape) go up before sampling
      Timer::Ev ev;
      tm.begin(DTS_K_SAMPLE, ev);
      auto fn = k_sample_plan<K, SAMPLE_NT>;
      const size_t sm = (size_t)smax * sizeof(K);
      DTS_TRY(set_smem(fn, sm));
      CUDA_TRY(cudaMemcpyAsync(dsampled, hp + align256(pb) + align256(bb), sb,
                               cudaMemcpyHostToDevice, st));
      fn<<<(unsigned)sampled.size(), SAMPLE_NT, sm, st>>>(dplans, dsampled, ink, dheavy, dhz,
                                                           cfg.seed, (uint32_t)level, stride,
                                                           gs_max, smax, wc_cols);
      tm.end(ev, sampled.size());
      DTS_TRY(check_launch("k_sample_plan"));
    }
    const double t_p4 = trace_on() ? now_us() : 0.0;
    // ---- histogram ----
    {
      CUDA_TRY(cudaMemsetAsync(dctr, 0, 16, st));
      Timer::Ev ev;
      tm.begin(DTS_K_HIST, ev);
      auto fn = wide ? k_histogram<K, HIST_NT, false, true> : k_histogram<K, HIST_NT, false, false>;
      const size_t sm = hist_layout(sizeof(K), caps, false).total;
      DTS_TRY(set_smem(fn, sm));
      const int grid = persistent_grid(fn, HIST_NT, sm, (uint32_t)blks.size());
      fn<<<grid, HIST_NT, sm, st>>>(dplans, dblks, (uint32_t)blks.size(), dctr, ink, dcnt, dheavy,
                                    dhz, nullptr, 0, caps, wide ? bid : nullptr);
      tm.end(ev, wave_recs);
      DTS_TRY(check_launch("k_histogram"));
    }
    DTS_TRY(flat_scan(dcnt, cnt_total, dscan, dpart, tm));
    {
      Timer::Ev ev;
      tm.begin(DTS_K_BOUNDS, ev);
      k_bucket_bounds<<<(unsigned)ns, 256, 0, st>>>(dplans, dscan, dhz, dbs, dkinds, dzones);
      tm.end(ev, bs_total);
      DTS_TRY(check_launch("k_bucket_bounds"));
    }
    // ---- classify buckets on the device (dtsort.py:244-318 _children_step)
    // from the bucket bounds; the scatter, the base case and the copies
    // follow; only the counters, the (few) next-level segments and the plans
    // come back ----
    const uint32_t out_src = in_T ? 0u : 1u;  // where the scatter wrote
    const uint64_t cap_copy = bs_total + wave_recs / COPY_CHUNK + 1;
    Span* dspan = (Span*)meta.take(std::max<uint64_t>(1, bs_total) * sizeof(Span));
    CopyR* dcopy = (CopyR*)meta.take(cap_copy * sizeof(CopyR));
    DTS_TRY(g_map_next.ensure(std::max<uint64_t>(1, bs_total) * sizeof(NextSeg)));
    NextSeg* dnext = (NextSeg*)g_map_next.d;  // (mapped host memory)
    unsigned long long* dcc = (unsigned long long*)meta.take(8 * sizeof(unsigned long long));
    if (!dspan || !dcopy || !dcc) return fail(DTS_ENOMEM, "workspace too small for level metadata");
    // (on the side stream: the classifier's few CTAs and the read-back run
    // beside the scatter, which only needs the scan; the base case waits)
    // Only before the write-combining scatter (stripes taken in any order):
    // the look-back scatter's tiles wait on their predecessors, and a tile
    // whose CTA starts late behind the classifier stalls its successors
    // (measured: Zipf 1.2 -3.5 %); and only for waves of few segments
    cudaStream_t cs = (wc && ns <= CLS_SIDE_MAX) ? side : st;
    if (cs != st) {
      CUDA_TRY(cudaEventRecord(ev_fork, st));
      CUDA_TRY(cudaStreamWaitEvent(side, ev_fork, 0));
    }
    static const uint32_t cls_rules = (uint32_t)env_int("DTS_CLS_RULES", 1);
    CUDA_TRY(cudaMemsetAsync(dcc, 0, 8 * sizeof(unsigned long long), cs));
    k_classify<<<(unsigned)ns, CLS_NT, 0, cs>>>(dplans, dbs, dkinds, (uint32_t)W, out_src, thr, COPY_CHUNK,
                                             dspan, dcopy, dnext, dcc, dzones, cls_rules);
    tm.launches += 1;
    DTS_TRY(check_launch("k_classify"));
    DTS_TRY(g_pin_back.ensure(256 + align256(pb) + 256));
    char* bp = (char*)g_pin_back.p;
    CUDA_TRY(cudaMemcpyAsync(bp, dcc, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaMemcpyAsync(bp + 256, dplans, pb, cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(cudaEventRecord(ev_cls, cs));
    // ---- scatter (after the classifier: it only needs the bucket bounds,
    // so the host receives the next level while the scatter runs) ----
    if (wc) {
      CUDA_TRY(cudaMemsetAsync(dctr + 1, 0, 4, st));
      Timer::Ev ev;
      tm.begin(DTS_K_SCATTER, ev);
      auto fn = wide ? k_scatter_wc<K, VB, 1> : k_scatter_wc<K, VB, 0>;
      const size_t sm = wide ? WcSmem<K, VB, 1>::total : WcSmem<K, VB, 0>::total;
      DTS_TRY(set_smem(fn, sm));
      const int grid = persistent_grid(fn, WcTile<K, VB>::NT, sm, (uint32_t)blks.size());
      fn<<<grid, WcTile<K, VB>::NT, sm, st>>>(dplans, dblks, (uint32_t)blks.size(), dctr + 1, ink, inv,
                                              outk, outv, dscan, dheavy, dhz, wide ? bid : nullptr);
      tm.end(ev, wave_recs);
      DTS_TRY(check_launch("k_scatter_wc"));
    } else {
      CUDA_TRY(cudaMemsetAsync(dctr + 1, 0, 4, st));
      CUDA_TRY(cudaMemsetAsync(dstatus, 0, ntile * (nbc / 2) * 4, st));
      Timer::Ev ev;
      tm.begin(DTS_K_SCATTER, ev);
      using TL = ScatterTile<K, VB>;
      auto fn = k_scatter<K, VB, false>;
      const size_t sm = ScatterSmem<K, VB, false>::total;
      DTS_TRY(set_smem(fn, sm));
      const int grid = persistent_grid(fn, TL::NT, sm, (uint32_t)ntile);
      fn<<<grid, TL::NT, sm, st>>>(dplans, dblks, dtile_blk, dblk_tile0, (uint32_t)ntile, nbc / 2,
                                    ink, inv, outk, outv, dscan, dstatus, dheavy, dhz, nullptr, 0);
      tm.end(ev, wave_recs);
      DTS_TRY(check_launch("k_scatter"));
    }
    if (cs != st) CUDA_TRY(cudaStreamWaitEvent(st, ev_cls, 0));  // spans / copies from the classifier
    DTS_TRY(local_sort_launch(dspan, reinterpret_cast<const uint32_t*>(dcc), bs_total, 1u << 30, 0));
    if (out_src == 1) {
      Timer::Ev ev;
      tm.begin(DTS_K_COPY, ev);
      k_copy_ranges<K, VB><<<(unsigned)(device_sms() * 4), 256, 0, st>>>(
          dcopy, reinterpret_cast<const uint32_t*>(dcc + 1), Ak, Av, Tk, Tv);
      tm.end(ev, 0);
      DTS_TRY(check_launch("k_copy_ranges"));
    }
    const double t_launch = trace_on() ? now_us() : 0.0;
    CUDA_TRY(cudaEventSynchronize(ev_cls));  // the base case keeps the GPU busy meanwhile
    const double t_sync = trace_on() ? now_us() : 0.0;
    const unsigned long long* hc = (const unsigned long long*)bp;
    const SegPlan* rp = (const SegPlan*)(bp + 256);
    const uint64_t nsp = hc[0] & 0xffffffffull, ncp = hc[1] & 0xffffffffull, nnx = hc[2] & 0xffffffffull;
    // (next-level order only shapes the waves; results do not depend on it;
    // NextSeg.pad = 0 reads as root = false)
    const size_t nx0 = next.size();
    next.resize(nx0 + nnx);
    if (nnx) std::memcpy(next.data() + nx0, g_map_next.p, nnx * sizeof(NextSeg));
    if (rep) {
      rep->moves += wave_recs + hc[6] + hc[7];
      rep->records_distributed += wave_recs;
      rep->levels = std::max(rep->levels, level + 1);
      if (level + 1 < 64) rep->level_mass[level + 1] += hc[4];
      if (level < 64) rep->heavy_records_removed[level] += hc[5];
      rep->base_case_records += hc[6];
      rep->kernel_records[DTS_K_LOCAL] += hc[6];
      rep->kernel_records[DTS_K_COPY] += hc[7];
      if (level == 0)
        for (size_t i = 0; i < ns; ++i)
          if (rp[i].flags & PF_OVF) rep->skipped_bits = (int32_t)(W - (rp[i].shift + rp[i].gamma));
    }
    meta.off = save;
    if (trace_on()) {
      std::fprintf(stderr,
                   "[dts] level %d segs %zu recs %llu blks %zu tiles %llu sampled %zu wc %d nbc %u | plan+launch %.0f us, "
                   "wait %.0f us, spans %llu copies %llu next %llu, host %.0f us\n",
                   level, ns, (unsigned long long)wave_recs, blks.size(), (unsigned long long)ntile,
                   sampled.size(), (int)wc, nbc, t_launch - t_plan0, t_sync - t_launch,
                   (unsigned long long)nsp, (unsigned long long)ncp, (unsigned long long)nnx,
                   now_us() - t_sync);
      std::fprintf(stderr, "[dts]   host: segment plans %.0f us, sample + read-back %.0f us, blocks / tile lists %.0f us, "
                   "meta + H2D %.0f us\n", t_p1 - t_plan0, t_p2 - t_p1, t_p3 - t_p2, t_p4 - t_p3);
    }
    return 0;
  }

  size_t wave_meta_bytes(const HostSeg& s, size_t level_segs) const {
    const uint64_t BR = block_records(sizeof(K), VB);
    const uint64_t rows = std::max<uint64_t>(1, (s.len + BR - 1) / BR);
    // (the digit and bucket capacity run_wave will choose)
    uint32_t g = choose_gamma(s.len, W - s.consumed), gs = 0;
    uint64_t nbmax;
    if (cfg.mode == DTS_MODE_DT &&
        sampled_plan(s.len, W - s.consumed, g, gs, (s.root & 1u) && s.consumed == 0,
                     (s.root & 2u) != 0 || level_segs <= SAMPLE_MANY, (s.root & 4u) != 0))
      nbmax = (1u << g) + (1u << gs) + 1u;
    else
      nbmax = 1u << g;
    const uint64_t tiles = s.len / 2560 + rows + 1;
    return 88 + rows * 28 + nbmax * rows * 12 + (nbmax + 1) * 11 + (1u << g) * 12 + 4096 +
           tiles * (4 + ((nbmax + 1) & ~1ull) * 4);
  }

  int run() {
    if (n <= 1) return 0;
    if (n <= thr) {
      add_span(0, n, 0);
      return launch_spans_and_copies();
    }
    std::vector<HostSeg> segs{HostSeg{0, n, 0, 1u}};
    if (rep) rep->level_mass[0] = n;
    int level = 0;
    bool in_T = false;
    // the span/copy descriptor area must stay available after a wave
    const size_t budget = meta.cap > (size_t(24) << 20) ? meta.cap - (size_t(16) << 20) : meta.cap / 2;
    while (!segs.empty()) {
      std::vector<HostSeg> next;
      size_t s0 = 0;
      // (waves of at most wave_segs segments: the host plans wave k + 1
      // while the GPU runs wave k — a level of 10^5 small segments, C4's
      // third, costs milliseconds of host planning)
      static const size_t wave_segs = (size_t)std::max(1, env_int("DTS_WAVE_SEGS", 1 << 30));
      while (s0 < segs.size()) {
        size_t s1 = s0, need = 1 << 16;
        while (s1 < segs.size()) {
          const size_t b = wave_meta_bytes(segs[s1], segs.size());
          if (s1 > s0 && (need + b > budget || s1 - s0 >= wave_segs)) break;
          need += b;
          ++s1;
        }
        DTS_TRY(run_wave(segs, s0, s1, level, in_T, next));
        s0 = s1;
      }
      segs.swap(next);
      in_T = !in_T;
      ++level;
      if (level > 200) return fail(DTS_ECUDA, "MSD recursion did not terminate");
    }
    return 0;
  }
};

template <typename K, int VB>
int sort_impl(void* keys, void* vals, uint64_t n, void* ws, size_t wsb, const dts_config* cfg,
              dts_report* rep, cudaStream_t st) {
  using V = typename ValOf<VB>::T;
  Timer tm;
  tm.st = st;
  tm.profile = cfg->profile != 0;
  tm.rep = rep;
  Sorter<K, VB> S(tm);
  S.Ak = (K*)keys;
  S.Av = (V*)vals;
  char* w = (char*)ws;
  const size_t kbytes = align256(n * sizeof(K)), vbytes = align256(n * (size_t)VB);
  S.Tk = (K*)w;
  S.Tv = VB ? (V*)(w + kbytes) : nullptr;
  const size_t bbytes = align256(n * 2);
  S.bid = (uint16_t*)(w + kbytes + vbytes);
  S.meta.base = w + kbytes + vbytes + bbytes;
  S.meta.cap = wsb - kbytes - vbytes - bbytes;
  S.n = n;
  S.cfg = *cfg;
  S.rep = rep;
  S.st = st;
  S.cap = LocalTile<K, VB>::CAP;
  // theta: SortConfig.effective_theta (core.py:148-151), capped by SMEM.
  uint64_t theta = cfg->base_case_threshold;
  const uint32_t gcap_hw = ceil_log2_u64(ScatterTile<K, VB>::NBC);
  uint32_t gcap = std::min<uint32_t>((uint32_t)std::max(1, cfg->gamma_hi),
                                     (uint32_t)env_int("DTS_GMAX", (int)gcap_hw));
  gcap = std::min(gcap, gcap_hw);
  gcap = std::max<uint32_t>(1, std::min<uint32_t>(gcap, 12));
  if (cfg->theory_mode) {
    const uint64_t e = (uint64_t)std::max(1, cfg->base_case_exponent) * gcap;
    theta = e >= 63 ? ~0ull : (1ull << e);
  }
  // reference: n_sub < theta -> base case, i.e. base case holds <= theta-1
  uint64_t thr = theta > 0 ? theta - 1 : 0;
  thr = std::min<uint64_t>(thr, (uint64_t)S.cap);
  if (thr < 1) thr = 1;
  S.thr = thr;
  S.gcap = gcap;
  S.gcap_hw = gcap_hw;
  S.glo = (uint32_t)std::max(1, cfg->gamma_lo);
  S.stride = n <= 2 ? 1 : ceil_log2_u64(n);
  S.gs_max = sizeof(K) == 4 ? 10 : 9;
  S.no_uniq_skip = env_int("DTS_UNIQ_SKIP", 1) == 0;
  S.smax = sizeof(K) == 4 ? 32768 : 16384;
  S.side = side_stream(&S.ev_cls, &S.ev_fork);
  if (!S.side) return fail(DTS_ECUDA, "cudaStreamCreate / cudaEventCreate failed for the classifier stream");
  int rc = S.run();
  // (stream-ordered calls return with the last level's base case still in
  // flight: a GPU step is not charged for the host's return path; the
  // per-kernel timers need the stream drained)
  if (rc == 0 && (!cfg->stream_ordered || tm.profile)) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(DTS_ECUDA, std::string("sort: ") + cudaGetErrorString(e));
  }
  if (rc == 0 && cfg->stream_ordered) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = fail(DTS_ECUDA, std::string("sort: ") + cudaGetErrorString(e));
  }
  tm.harvest();
  if (rc != 0) cudaStreamSynchronize(S.side);  // (nothing of this call left in flight)
  if (rep) rep->gpu_launches += tm.launches;
  return rc;
}

// ---------------------------------------------------------------------------
// Partition (multi-GPU key-range exchange)
// ---------------------------------------------------------------------------
template <typename K, int VB>
int partition_impl(const void* keys, const void* vals, uint64_t n, uint64_t gbase,
                   const void* split_keys, const uint64_t* split_idx, int nsplit, void* okeys,
                   void* ovals, uint64_t* counts, void* ws, size_t wsb, cudaStream_t st) {
  using V = typename ValOf<VB>::T;
  const uint32_t G = (uint32_t)nsplit + 1;
  if (n == 0) {
    for (uint32_t g = 0; g < G; ++g) counts[g] = 0;
    return 0;
  }
  Timer tm;
  tm.st = st;
  tm.profile = false;
  tm.rep = nullptr;
  Bump meta{(char*)ws, wsb, 0};
  const uint64_t BR = block_records(sizeof(K), VB);
  const uint64_t rows = std::max<uint64_t>(1, (n + BR - 1) / BR);
  SegPlan P;
  std::memset(&P, 0, sizeof(P));
  P.offset = 0;
  P.len = n;
  P.nb = G;
  P.nbmax = G;
  P.flags = PF_SPLIT;
  P.nheavy = (uint32_t)nsplit;
  P.nrows = (uint32_t)rows;
  std::vector<Blk> blks;
  constexpr uint64_t TT = ScatterTile<K, VB>::T;
  const uint64_t per = ((n + rows - 1) / rows + TT - 1) / TT * TT;
  for (uint64_t r = 0; r < rows; ++r)
    blks.push_back(Blk{0, (uint32_t)r, std::min(n, r * per), std::min(n, (r + 1) * per)});
  const uint64_t cnt_total = (uint64_t)G * rows;
  SegPlan* dplan = (SegPlan*)meta.take(sizeof(SegPlan));
  Blk* dblks = (Blk*)meta.take(blks.size() * sizeof(Blk));
  uint32_t* dcnt = (uint32_t*)meta.take(cnt_total * 4);
  uint64_t* dscan = (uint64_t*)meta.take(cnt_total * 8);
  uint64_t* dpart = (uint64_t*)meta.take(((cnt_total + SCAN_CHUNK - 1) / SCAN_CHUNK + 1) * 8);
  uint64_t* dbs = (uint64_t*)meta.take((G + 1) * 8);
  uint8_t* dkinds = (uint8_t*)meta.take(G + 1);
  K* dsk = (K*)meta.take(std::max(1, nsplit) * sizeof(K));
  uint64_t* dsi = (uint64_t*)meta.take(std::max(1, nsplit) * 8);
  uint32_t* dctr = (uint32_t*)meta.take(16);
  constexpr uint32_t ST_T = ScatterTile<K, VB>::T;
  std::vector<uint32_t> blk_tile0(blks.size());
  uint64_t ntile = 0;
  for (size_t bi = 0; bi < blks.size(); ++bi) {
    blk_tile0[bi] = (uint32_t)ntile;
    ntile += (blks[bi].end - blks[bi].begin + ST_T - 1) / ST_T;
  }
  std::vector<uint32_t> tile_blk(ntile);
  for (size_t bi = 0; bi < blks.size(); ++bi) {
    const uint32_t e = bi + 1 < blks.size() ? blk_tile0[bi + 1] : (uint32_t)ntile;
    for (uint32_t t = blk_tile0[bi]; t < e; ++t) tile_blk[t] = (uint32_t)bi;
  }
  const uint32_t nbc = (G + 1) & ~1u;
  uint32_t* dtile_blk = (uint32_t*)meta.take(std::max<uint64_t>(1, ntile) * 4);
  uint32_t* dblk_tile0 = (uint32_t*)meta.take(std::max<size_t>(1, blks.size()) * 4);
  uint32_t* dstatus = (uint32_t*)meta.take(std::max<uint64_t>(1, ntile) * (nbc / 2) * 4);
  if (!dplan || !dblks || !dcnt || !dscan || !dpart || !dbs || !dkinds || !dsk || !dsi || !dctr ||
      !dtile_blk || !dblk_tile0 || !dstatus)
    return fail(DTS_ENOMEM, "workspace too small for partition metadata");
  const size_t bb = blks.size() * sizeof(Blk);
  const size_t tb = ntile * 4, b0b = blks.size() * 4;
  DTS_TRY(g_pin_plan.ensure(512 + align256(bb) + 16 * (size_t)(nsplit + 1) + align256(tb) + b0b + 512));
  char* hp = (char*)g_pin_plan.p;
  std::memcpy(hp, &P, sizeof(P));
  std::memcpy(hp + 256, blks.data(), bb);
  char* htl = hp + 256 + align256(bb);
  std::memcpy(htl, tile_blk.data(), tb);
  std::memcpy(htl + align256(tb), blk_tile0.data(), b0b);
  CUDA_TRY(cudaMemcpyAsync(dtile_blk, htl, tb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dblk_tile0, htl + align256(tb), b0b, cudaMemcpyHostToDevice, st));
  char* hs = htl + align256(tb) + align256(b0b);
  if (nsplit) {
    std::memcpy(hs, split_keys, nsplit * sizeof(K));
    std::memcpy(hs + align256(nsplit * sizeof(K)), split_idx, nsplit * 8);
  }
  CUDA_TRY(cudaMemcpyAsync(dplan, hp, sizeof(P), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dblks, hp + 256, bb, cudaMemcpyHostToDevice, st));
  if (nsplit) {
    CUDA_TRY(cudaMemcpyAsync(dsk, hs, nsplit * sizeof(K), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dsi, hs + align256(nsplit * sizeof(K)), nsplit * 8,
                             cudaMemcpyHostToDevice, st));
  }
  Caps caps{(G + 1) & ~1u, 0, (uint32_t)std::max(2, nsplit + (nsplit & 1)), 0};
  CUDA_TRY(cudaMemsetAsync(dctr, 0, 16, st));
  {
    auto fn = k_histogram<K, HIST_NT, true>;
    const size_t sm = hist_layout(sizeof(K), caps, true).total;
    DTS_TRY(set_smem(fn, sm));
    const int grid = persistent_grid(fn, HIST_NT, sm, (uint32_t)blks.size());
    fn<<<grid, HIST_NT, sm, st>>>(dplan, dblks, (uint32_t)blks.size(), dctr, (const K*)keys, dcnt,
                                  dsk, nullptr, dsi, gbase, caps, nullptr);
    DTS_TRY(check_launch("k_histogram(split)"));
  }
  DTS_TRY(flat_scan(dcnt, cnt_total, dscan, dpart, tm));
  k_bucket_bounds<<<1, 256, 0, st>>>(dplan, dscan, nullptr, dbs, dkinds, nullptr);
  DTS_TRY(check_launch("k_bucket_bounds(split)"));
  {
    using TL = ScatterTile<K, VB>;
    auto fn = k_scatter<K, VB, true>;
    const size_t sm = ScatterSmem<K, VB, true>::total;
    DTS_TRY(set_smem(fn, sm));
    CUDA_TRY(cudaMemsetAsync(dstatus, 0, ntile * (nbc / 2) * 4, st));
    const int grid = persistent_grid(fn, TL::NT, sm, (uint32_t)ntile);
    fn<<<grid, TL::NT, sm, st>>>(dplan, dblks, dtile_blk, dblk_tile0, (uint32_t)ntile, nbc / 2,
                                  (const K*)keys, (const V*)vals, (K*)okeys, (V*)ovals, dscan,
                                  dstatus, dsk, nullptr, dsi, gbase);
    DTS_TRY(check_launch("k_scatter(split)"));
  }
  DTS_TRY(g_pin_back.ensure((G + 1) * 8 + 256));
  CUDA_TRY(cudaMemcpyAsync(g_pin_back.p, dbs, (G + 1) * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const uint64_t* bs = (const uint64_t*)g_pin_back.p;
  for (uint32_t g = 0; g < G; ++g) counts[g] = bs[g + 1] - bs[g];
  return 0;
}

// ---------------------------------------------------------------------------
// Dovetail merge (dtmerge.py:132-238) as a layout-driven permutation: the
// insertion points (compute_layout, :58-78) and the reference's _validate
// checks (:108-129) on the GPU, then one out-of-place pass of the zone into
// the caller's workspace and one copy back — 3-4 launches and one read-back
// of the insertion points, whatever the number of heavy runs.  MergeStats
// are the reference's piece-loop counts, computed on the host from the
// insertion points and run lengths (merge_stats below).
// ---------------------------------------------------------------------------

// The reference's write counts for a zone (dtmerge.py:166-238: out_copies of
// the smaller side, in-array moves — a direct move of len, or a two-flip
// block shift of 2 len (shift_block, :81-105) when source and destination
// overlap — and restore copies from scratch).
void merge_stats(uint64_t light, const int64_t* hlens, uint64_t m, const uint64_t* ins,
                 const uint64_t* prefix, uint64_t heavy_total, uint64_t stats[3]) {
  uint64_t out_copies = 0, in_moves = 0, restores = 0;
  auto bound = [&](uint64_t i) -> uint64_t { return i == 0 ? 0 : (i <= m ? ins[i - 1] : light); };
  if (heavy_total >= light) {
    out_copies = light;
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t ln = (uint64_t)hlens[i], src = light + prefix[i], dst = ins[i] + prefix[i];
      if (ln == 0 || dst == src) continue;
      in_moves += dst + ln <= src ? ln : 2 * ln;
    }
    for (uint64_t i = 0; i <= m; ++i) {
      const uint64_t f0 = bound(i), flen = bound(i + 1) - f0;
      if (flen == 0 || f0 + prefix[i] == f0) continue;
      restores += flen;
    }
  } else {
    out_copies = heavy_total;
    for (uint64_t i = m; i >= 1; --i) {
      const uint64_t f0 = bound(i), flen = bound(i + 1) - f0, dst = f0 + prefix[i];
      if (flen == 0 || dst == f0) continue;
      in_moves += f0 + flen <= dst ? flen : 2 * flen;
    }
    for (uint64_t i = 0; i < m; ++i) restores += (uint64_t)hlens[i];
  }
  stats[0] = out_copies;
  stats[1] = in_moves;
  stats[2] = restores;
}

struct MergeWs {  // the caller's merge workspace, carved
  size_t keys, vals, hk, pre, ins, err, total;
};
MergeWs merge_ws_layout(uint64_t zone_len, uint64_t m, int kb, int vb) {
  MergeWs w;
  w.keys = 0;
  w.vals = align256(zone_len * (size_t)kb);
  w.hk = w.vals + align256(zone_len * (size_t)vb);
  w.pre = w.hk + align256(std::max<uint64_t>(1, m) * (size_t)kb);
  w.ins = w.pre + align256((m + 1) * 8);
  w.err = w.ins + align256(std::max<uint64_t>(1, m) * 8);
  w.total = w.err + 256;
  return w;
}

template <typename K, int VB>
int merge_impl(void* zk_, void* zv_, uint64_t total, uint64_t light, const void* hkeys_,
               const int64_t* hlens, uint64_t m, uint64_t scratch_len, bool scratch_vals, int validate,
               void* ws_, size_t wsb, uint64_t stats[3], cudaStream_t st) {
  using V = typename ValOf<VB>::T;
  K* zk = (K*)zk_;
  V* zv = VB ? (V*)zv_ : nullptr;
  const K* hkeys = (const K*)hkeys_;
  stats[0] = stats[1] = stats[2] = 0;
  int64_t heavy_total_s = 0;
  for (uint64_t i = 0; i < m; ++i) heavy_total_s += hlens[i];
  const uint64_t heavy_total = heavy_total_s < 0 ? 0 : (uint64_t)heavy_total_s;
  const uint64_t small = std::min<uint64_t>(light, heavy_total);
  if (scratch_len < small)
    return fail(DTS_EINVAL, "scratch holds " + std::to_string(scratch_len) + " records, need " +
                                std::to_string(small));
  if (VB && zv && !scratch_vals && small > 0) return fail(DTS_EINVAL, "scratch payloads too small");
  if (validate) {
    if ((int64_t)light + heavy_total_s != (int64_t)total)
      return fail(DTS_EINVAL, "light_len plus heavy run lengths must tile the zone");
    for (uint64_t i = 0; i < m; ++i)
      if (hlens[i] < 0) return fail(DTS_EINVAL, "heavy run lengths must be nonnegative");
    for (uint64_t i = 1; i < m; ++i)
      if (!(hkeys[i] > hkeys[i - 1]))
        return fail(DTS_EINVAL, "heavy keys must be strictly increasing");
  } else {
    for (uint64_t i = 0; i < m; ++i)
      if (hlens[i] < 0) return fail(DTS_EINVAL, "heavy run lengths must be nonnegative");
    if (light + heavy_total != total)
      return fail(DTS_EINVAL, "light_len plus heavy run lengths must tile the zone");
  }
  const bool check_light = validate && light > 1;
  if ((m == 0 || total == 0) && !check_light) return 0;
  const MergeWs L = merge_ws_layout(total, m, sizeof(K), VB);
  if (!ws_ || wsb < L.total)
    return fail(DTS_ENOMEM, "merge workspace holds " + std::to_string(wsb) + " bytes, need " +
                                std::to_string(L.total) + " (dts_merge_workspace_bytes)");
  char* ws = (char*)ws_;
  K* ok = (K*)(ws + L.keys);
  V* ov = VB ? (V*)(ws + L.vals) : nullptr;
  K* dh = (K*)(ws + L.hk);
  uint64_t* dpre = (uint64_t*)(ws + L.pre);
  uint64_t* dins = (uint64_t*)(ws + L.ins);
  uint32_t* derr = (uint32_t*)(ws + L.err);
  // heavy keys + run prefix sums up, through the pinned staging
  std::vector<uint64_t> prefix(m + 1, 0);
  for (uint64_t i = 0; i < m; ++i) prefix[i + 1] = prefix[i] + (uint64_t)hlens[i];
  const size_t hb = align256(m * sizeof(K)), pb = (m + 1) * 8;
  DTS_TRY(g_pin_plan.ensure(hb + pb + 256));
  char* hp = (char*)g_pin_plan.p;
  if (m) std::memcpy(hp, hkeys, m * sizeof(K));
  std::memcpy(hp + hb, prefix.data(), pb);
  if (m) CUDA_TRY(cudaMemcpyAsync(dh, hp, m * sizeof(K), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dpre, hp + hb, pb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(derr, 0, 4, st));
  if (m) {
    k_merge_layout<K><<<(unsigned)((m + 255) / 256), 256, 0, st>>>(zk, light, dh, m, dins);
    DTS_TRY(check_launch("k_merge_layout"));
  }
  if (validate) {
    const uint64_t work = std::max<uint64_t>(total, m);
    const unsigned grid = (unsigned)std::min<uint64_t>(8 * device_sms(), (work + 255) / 256 + 1);
    k_merge_validate<K><<<grid, 256, 0, st>>>(zk, light, total, dh, dpre, m, dins, derr);
    DTS_TRY(check_launch("k_merge_validate"));
  }
  const bool permute = m > 0 && total > 0;
  if (permute) {
    const unsigned grid = (unsigned)std::min<uint64_t>(8 * device_sms(), (total + 255) / 256);
    k_merge_permute<K, VB><<<grid, 256, 0, st>>>(zk, zv, light, total, dins, dpre, m, ok, ov);
    DTS_TRY(check_launch("k_merge_permute"));
  }
  // one read-back: the error flags and the insertion points (MergeStats)
  DTS_TRY(g_pin_back.ensure(256 + m * 8 + 256));
  char* bp = (char*)g_pin_back.p;
  CUDA_TRY(cudaMemcpyAsync(bp, derr, 4, cudaMemcpyDeviceToHost, st));
  if (m) CUDA_TRY(cudaMemcpyAsync(bp + 256, dins, m * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  const uint32_t err = *(const uint32_t*)bp;
  if (err) {  // the zone is untouched: the permutation went to the workspace
    if (err & 1u) return fail(DTS_EINVAL, "light run must be sorted");
    if (err & 2u) return fail(DTS_EINVAL, "a heavy key also appears in the light run");
    return fail(DTS_EINVAL, "heavy run contains a foreign key");
  }
  if (!permute) return 0;
  {
    const unsigned grid = (unsigned)std::min<uint64_t>(8 * device_sms(), (total + 255) / 256);
    k_copy_back<K, VB><<<grid, 256, 0, st>>>(zk, zv, ok, ov, total);
    DTS_TRY(check_launch("k_copy_back"));
  }
  merge_stats(light, hlens, m, (const uint64_t*)(bp + 256), prefix.data(), heavy_total, stats);
  return 0;
}

bool valid_widths(int kb, int vb) { return (kb == 4 || kb == 8) && (vb == 0 || vb == 4 || vb == 8); }

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

// Tools-only: per-phase cycle sums of k_scatter (DTS_PHASE_PROF builds);
// returns the number of entries written (0 in product builds).
int dts_debug_phases(unsigned long long* out, int n, int reset) {
#if DTS_PHASE_PROF
  unsigned long long h[16];
  if (cudaMemcpyFromSymbol(h, g_phase, sizeof(h)) != cudaSuccess) return -1;
  const int m = n < 16 ? n : 16;
  for (int i = 0; i < m; ++i) out[i] = h[i];
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  }
  return m;
#else
  (void)out; (void)n; (void)reset;
  return 0;
#endif
}


size_t dts_workspace_bytes(uint64_t n, int key_bytes, int val_bytes) {
  if (!valid_widths(key_bytes, val_bytes)) return 0;
  // twin T (keys, values), 2 bytes per record of bucket ids, metadata
  return align256(n * (size_t)key_bytes) + align256(n * (size_t)val_bytes) + align256(n * 2) + meta_bytes(n);
}

int dts_sort(void* keys, void* vals, uint64_t n, int kb, int vb, void* ws, size_t wsb,
             const dts_config* cfg, dts_report* rep, void* stream) {
  if (!valid_widths(kb, vb)) return fail(DTS_EINVAL, "key_bytes must be 4|8 and val_bytes 0|4|8");
  if (!cfg) return fail(DTS_EINVAL, "cfg must not be NULL");
  if (n && !keys) return fail(DTS_EINVAL, "keys must not be NULL");
  if (n && vb && !vals) return fail(DTS_EINVAL, "vals must not be NULL when val_bytes > 0");
  if (cfg->gamma_lo < 1 || cfg->gamma_lo > cfg->gamma_hi || cfg->gamma_hi > 16)
    return fail(DTS_EINVAL, "need 1 <= gamma_lo <= gamma_hi <= 16");
  if (rep) std::memset(rep, 0, sizeof(*rep));
  if (n == 0) return 0;
  if (n >= (uint64_t(1) << 32))
    return fail(DTS_EINVAL, "n must be < 2^32 per call (segment positions are 32-bit); shard larger "
                            "inputs with distributed.dist_sort");
  if (wsb < dts_workspace_bytes(n, kb, vb))
    return fail(DTS_ENOMEM, "workspace holds " + std::to_string(wsb) + " bytes, need " +
                                std::to_string(dts_workspace_bytes(n, kb, vb)));
  cudaStream_t st = (cudaStream_t)stream;
  if (kb == 4) {
    if (vb == 0) return sort_impl<uint32_t, 0>(keys, vals, n, ws, wsb, cfg, rep, st);
    if (vb == 4) return sort_impl<uint32_t, 4>(keys, vals, n, ws, wsb, cfg, rep, st);
    return sort_impl<uint32_t, 8>(keys, vals, n, ws, wsb, cfg, rep, st);
  }
  if (vb == 0) return sort_impl<uint64_t, 0>(keys, vals, n, ws, wsb, cfg, rep, st);
  if (vb == 4) return sort_impl<uint64_t, 4>(keys, vals, n, ws, wsb, cfg, rep, st);
  return sort_impl<uint64_t, 8>(keys, vals, n, ws, wsb, cfg, rep, st);
}

size_t dts_merge_workspace_bytes(uint64_t zone_len, uint64_t m, int kb, int vb) {
  if (!valid_widths(kb, vb)) return 0;
  return merge_ws_layout(zone_len, m, kb, vb).total;
}

int dts_merge(void* zk, void* zv, uint64_t zone_len, uint64_t light_len, const void* hkeys,
              const int64_t* hlens, uint64_t m, void* sk, void* sv, uint64_t scratch_len, int kb,
              int vb, int validate, void* ws, size_t wsb, uint64_t stats_out[3], void* stream) {
  (void)sk;  // scratch keys: validated by size only (the permutation uses the workspace)
  if (!valid_widths(kb, vb)) return fail(DTS_EINVAL, "key_bytes must be 4|8 and val_bytes 0|4|8");
  if (!stats_out) return fail(DTS_EINVAL, "stats_out must not be NULL");
  if (m && (!hkeys || !hlens)) return fail(DTS_EINVAL, "heavy_keys and heavy_lens must have equal length");
  cudaStream_t st = (cudaStream_t)stream;
#define DTS_MERGE_CALL(K, VB) \
  merge_impl<K, VB>(zk, zv, zone_len, light_len, hkeys, hlens, m, scratch_len, sv != nullptr, validate, ws, wsb, \
                    stats_out, st)
  if (kb == 4) {
    if (vb == 0) return DTS_MERGE_CALL(uint32_t, 0);
    if (vb == 4) return DTS_MERGE_CALL(uint32_t, 4);
    return DTS_MERGE_CALL(uint32_t, 8);
  }
  if (vb == 0) return DTS_MERGE_CALL(uint64_t, 0);
  if (vb == 4) return DTS_MERGE_CALL(uint64_t, 4);
  return DTS_MERGE_CALL(uint64_t, 8);
#undef DTS_MERGE_CALL
}

int dts_partition(const void* keys, const void* vals, uint64_t n, uint64_t gbase,
                  const void* split_keys, const uint64_t* split_idx, int nsplit, void* okeys,
                  void* ovals, uint64_t* counts, int kb, int vb, void* ws, size_t wsb,
                  void* stream) {
  if (!valid_widths(kb, vb)) return fail(DTS_EINVAL, "key_bytes must be 4|8 and val_bytes 0|4|8");
  if (nsplit < 0 || nsplit >= ScatterTile<uint32_t, 4>::HKC)
    return fail(DTS_EINVAL, "nsplit must be in [0, 1023]");  // SMEM splitter / bucket tables (ScatterTile HKC, NBC)
  if (!counts) return fail(DTS_EINVAL, "send_counts must not be NULL");
  if (nsplit && (!split_keys || !split_idx)) return fail(DTS_EINVAL, "splitters must not be NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (kb == 4) {
    if (vb == 0) return partition_impl<uint32_t, 0>(keys, vals, n, gbase, split_keys, split_idx, nsplit, okeys, ovals, counts, ws, wsb, st);
    if (vb == 4) return partition_impl<uint32_t, 4>(keys, vals, n, gbase, split_keys, split_idx, nsplit, okeys, ovals, counts, ws, wsb, st);
    return partition_impl<uint32_t, 8>(keys, vals, n, gbase, split_keys, split_idx, nsplit, okeys, ovals, counts, ws, wsb, st);
  }
  if (vb == 0) return partition_impl<uint64_t, 0>(keys, vals, n, gbase, split_keys, split_idx, nsplit, okeys, ovals, counts, ws, wsb, st);
  if (vb == 4) return partition_impl<uint64_t, 4>(keys, vals, n, gbase, split_keys, split_idx, nsplit, okeys, ovals, counts, ws, wsb, st);
  return partition_impl<uint64_t, 8>(keys, vals, n, gbase, split_keys, split_idx, nsplit, okeys, ovals, counts, ws, wsb, st);
}

int dts_gen_rmat(uint32_t* dst, uint32_t* src, uint64_t n, uint64_t edge_base, uint64_t seed, int scale,
                 uint32_t t0, uint32_t t1, uint32_t t2, void* stream) {
  if (scale < 1 || scale > 32) return fail(DTS_EINVAL, "scale must be in [1, 32]");
  if (!(t0 <= t1 && t1 <= t2)) return fail(DTS_EINVAL, "quadrant thresholds must be non-decreasing");
  if (n == 0) return 0;
  if (!dst || !src) return fail(DTS_EINVAL, "dst and src must not be NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 64);
  k_gen_rmat<<<(unsigned)blocks, 256, 0, st>>>(dst, src, n, edge_base, seed, (uint32_t)scale, t0, t1, t2);
  return check_launch("k_gen_rmat");
}

size_t dts_csr_workspace_bytes(uint64_t nverts) { return 256 + 24 * (size_t)(nverts / CSR_LONG + 2); }

int dts_csr_offsets(const void* keys, uint64_t n, int kb, uint64_t nverts, uint64_t* row_ptr, void* ws, size_t wsb,
                    void* stream) {
  if (kb != 4 && kb != 8) return fail(DTS_EINVAL, "key_bytes must be 4|8");
  if (!row_ptr) return fail(DTS_EINVAL, "row_ptr must not be NULL");
  if (n && !keys) return fail(DTS_EINVAL, "keys must not be NULL");
  if (wsb < dts_csr_workspace_bytes(nverts) || !ws) return fail(DTS_ENOMEM, "workspace too small for dts_csr_offsets");
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* flags = (uint32_t*)ws;  // [0] gap count, [1] bad
  uint64_t* gaps = (uint64_t*)((char*)ws + 256);
  const uint32_t cap = (uint32_t)std::min<uint64_t>((wsb - 256) / 24, 0xFFFFFFFFull);
  CUDA_TRY(cudaMemsetAsync(flags, 0, 8, st));
  const uint64_t blocks = std::min<uint64_t>((n + 1 + 255) / 256, 148ull * 64);
  if (kb == 4)
    k_csr_offsets<uint32_t><<<(unsigned)blocks, 256, 0, st>>>((const uint32_t*)keys, n, nverts, row_ptr, gaps, flags, cap, flags + 1);
  else
    k_csr_offsets<uint64_t><<<(unsigned)blocks, 256, 0, st>>>((const uint64_t*)keys, n, nverts, row_ptr, gaps, flags, cap, flags + 1);
  DTS_TRY(check_launch("k_csr_offsets"));
  uint32_t h[2];
  CUDA_TRY(cudaMemcpyAsync(h, flags, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (h[1] == 1u) return fail(DTS_EINVAL, "keys must be ascending and below nverts");
  if (h[1] == 2u) return fail(DTS_ENOMEM, "workspace too small for the CSR gap list");
  if (h[0]) {
    k_csr_fill_gaps<<<h[0], 256, 0, st>>>(gaps, flags, row_ptr);
    DTS_TRY(check_launch("k_csr_fill_gaps"));
  }
  return 0;
}

int dts_morton_keys(const uint32_t* x, const uint32_t* y, const uint32_t* z, uint64_t n, int dims, int bits,
                    uint64_t* keys, uint64_t* vals, uint64_t first_index, void* ws, size_t wsb, void* stream) {
  if (dims != 2 && dims != 3) return fail(DTS_EINVAL, "dims must be 2 or 3");
  if (bits < 1 || bits > (dims == 2 ? 32 : 21))
    return fail(DTS_EINVAL, "bits per coordinate must be in [1, 32] (2-D) or [1, 21] (3-D)");
  if (!ws || wsb < 16) return fail(DTS_ENOMEM, "workspace too small for dts_morton_keys (16 bytes)");
  if (n == 0) return 0;
  if (!x || !y || (dims == 3 && !z) || !keys) return fail(DTS_EINVAL, "coordinate and key arrays must not be NULL");
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* flags = (uint32_t*)ws;
  CUDA_TRY(cudaMemsetAsync(flags, 0, 4, st));
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)device_sms() * 16);
  if (dims == 2)
    k_morton<2><<<(unsigned)blocks, 256, 0, st>>>(x, y, nullptr, n, (uint32_t)bits, keys, vals, first_index, flags);
  else
    k_morton<3><<<(unsigned)blocks, 256, 0, st>>>(x, y, z, n, (uint32_t)bits, keys, vals, first_index, flags);
  DTS_TRY(check_launch("k_morton"));
  uint32_t h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, flags, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (h) return fail(DTS_EINVAL, "a coordinate does not fit in `bits` bits");
  return 0;
}

const char* dts_last_error(void) { return g_err.c_str(); }

int dts_abi_version(void) { return DTS_ABI_VERSION; }

int dts_build_arch(void) { return 100; }

}  // extern "C"
