/*
 * dts.h — C ABI of libdts.so, the B200 (sm_100a) DovetailSort hot path.
 *
 * This is the drop-in boundary for the reference package `dovetail`
 * (arXiv 2401.00710, /root/reference/pkg/src/dovetail).  Every entry point
 * below replaces one reference interface; the reference location is cited
 * on each declaration.  All pointers named *keys / *vals / workspace /
 * scratch are DEVICE pointers owned by the caller; small descriptor arrays
 * (heavy_keys, heavy_lens, splitters, counts) are HOST pointers.  Every call
 * is ordered on the CUDA stream passed in and returns after the result is
 * complete on that stream (the sort reads a few per-level counters back to
 * the host, so it synchronises the stream once per MSD level) — except
 * dts_sort with dts_config.stream_ordered, which returns as soon as its last
 * kernels are enqueued.
 *
 * Status codes: 0 ok, DTS_EINVAL (-1) invalid argument (Python: ValueError),
 * DTS_ENOMEM (-2) workspace too small (MemoryError), DTS_ECUDA (-3) CUDA
 * error (RuntimeError).  dts_last_error() returns a thread-local message for
 * the last nonzero status.  No entry point ever falls back to the CPU.
 */
#ifndef DTS_H_
#define DTS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DTS_ABI_VERSION 2

#define DTS_OK 0
#define DTS_EINVAL (-1)
#define DTS_ENOMEM (-2)
#define DTS_ECUDA (-3)

#define DTS_MODE_DT 0    /* dt_sort: sampling + heavy buckets (dtsort.py:64-71)   */
#define DTS_MODE_PLAIN 1 /* plain_msd_sort: no sampling/heavy/overflow (:74-78)   */

/* Kernel classes timed in dts_report.kernel_ms when dts_config.profile != 0. */
#define DTS_K_SAMPLE 0    /* k_sample_plan   — sampler.py:139-252                 */
#define DTS_K_HIST 1      /* k_histogram     — counting.py:123-137 (count phase)  */
#define DTS_K_SCAN 2      /* k_scan_*        — counting.py:58-79 (offsets)        */
#define DTS_K_SCATTER 3   /* k_scatter       — counting.py:141-151, _kernels.py:12*/
#define DTS_K_LOCAL 4     /* k_local_sort    — dtsort.py:127-147 (_base_sort)     */
#define DTS_K_COPY 5      /* k_copy_ranges   — dtsort.py:111-124 (_copy_between)  */
#define DTS_K_BOUNDS 6    /* k_bucket_bounds — counting.py:153 (bucket offsets)   */
#define DTS_K_MERGE 7     /* dt_merge kernels — dtmerge.py:132-238                */
#define DTS_NKCLASS 8

/* Mirrors SortConfig (core.py:106-151).  sample_rule / block_policy are
 * Python callables and cannot cross this ABI (the Python layer rejects them
 * with NotImplementedError). */
typedef struct dts_config {
  uint64_t seed;                /* SortConfig.seed                              */
  int32_t gamma_lo, gamma_hi;   /* SortConfig.gamma_lo / gamma_hi (digit clamp) */
  uint64_t base_case_threshold; /* SortConfig.base_case_threshold (theta)       */
  int32_t theory_mode;          /* SortConfig.theory_mode                       */
  int32_t base_case_exponent;   /* SortConfig.base_case_exponent                */
  int32_t mode;                 /* DTS_MODE_DT | DTS_MODE_PLAIN                 */
  int32_t instrument;           /* fill dts_report counters                     */
  int32_t profile;              /* time every kernel with CUDA events           */
  int32_t stream_ordered;       /* nonzero: dts_sort returns once its last kernels
                                   are enqueued (no final stream synchronisation;
                                   the result is complete in stream order) —
                                   the device-resident API (dtsort.sort_device) */
  int32_t reserved[6];
} dts_config;

/* Mirrors InstrumentReport (core.py:167-227) plus B200 timing fields. */
typedef struct dts_report {
  uint64_t moves;                 /* record writes (scatter+base+copies)          */
  uint64_t merge_out_copies;      /* 0: heavy runs are placed by the scatter      */
  uint64_t merge_in_array_moves;  /* 0: (fused dovetail)           */
  uint64_t base_case_records;     /* records finished by k_local_sort             */
  int32_t levels;                 /* MSD levels that ran a distribution pass      */
  int32_t skipped_bits;           /* root leading-bit skip (overflow bucket)      */
  uint64_t level_mass[64];
  uint64_t heavy_records_removed[64];
  uint64_t records_distributed;   /* D: records through a distribution pass       */
  uint64_t gpu_launches;          /* kernels launched by this call                */
  double kernel_ms[DTS_NKCLASS];  /* profile only: summed CUDA-event time         */
  uint64_t kernel_launches[DTS_NKCLASS];
  uint64_t kernel_records[DTS_NKCLASS]; /* records processed per class            */
} dts_report;

/* Device workspace needed by dts_sort / dts_partition for n records of the
 * given widths (key_bytes 4|8, val_bytes 0|4|8).  Holds the temporary
 * buffer twin (dtsort.py:92-99 `np.empty_like`), 2 bytes per record of bucket
 * ids (heavy-key segments: the histogram's routing result, reused by the
 * scatter) and per-level metadata. */
size_t dts_workspace_bytes(uint64_t n, int key_bytes, int val_bytes);

/* Stable ascending sort in place — replaces dt_sort / plain_msd_sort / _run
 * (dtsort.py:64-108).  keys: n keys (u32 or u64); vals: NULL (keys only) or n
 * payloads of val_bytes each; both arrays receive the sorted result.
 * report may be NULL.  stream is a cudaStream_t (NULL = legacy default). */
int dts_sort(void* keys, void* vals, uint64_t n, int key_bytes, int val_bytes,
             void* workspace, size_t workspace_bytes, const dts_config* cfg,
             dts_report* report, void* stream);

/* Dovetail merge of one zone in place — replaces dt_merge (dtmerge.py:132-238).
 * zone = [sorted light run of light_len | heavy run 0 | heavy run 1 | ...].
 * heavy_keys (host, m keys, strictly increasing) / heavy_lens (host, m int64).
 * scratch_len must be at least min(light_len, sum(heavy_lens)) records (the
 * reference's contract, checked with its messages); the GPU permutes the zone
 * out of place through `workspace` (caller-owned device memory of at least
 * dts_merge_workspace_bytes(zone_len, m, ...) bytes), so scratch is not
 * written.  stats_out[3] = {out_copies, in_array_moves, restore_copies}: the
 * reference's MergeStats for this zone.  validate != 0 runs the reference's
 * _validate checks (dtmerge.py:108-129); on a validation error the zone is
 * left unchanged.  Blocks once (reads the insertion points back). */
size_t dts_merge_workspace_bytes(uint64_t zone_len, uint64_t m, int key_bytes,
                                 int val_bytes);
int dts_merge(void* zone_keys, void* zone_vals, uint64_t zone_len,
              uint64_t light_len, const void* heavy_keys,
              const int64_t* heavy_lens, uint64_t m, void* scratch_keys,
              void* scratch_vals, uint64_t scratch_len, int key_bytes,
              int val_bytes, int validate, void* workspace,
              size_t workspace_bytes, uint64_t stats_out[3], void* stream);

/* Stable G-way partition by (key, global index) against nsplit = G-1 sorted
 * splitters (host arrays split_keys / split_idx).  Record i (global index
 * global_base + i) goes to destination g = #{s : (split_key[s], split_idx[s])
 * < (key, global index)}.  Writes the records grouped by g (input order kept
 * within each group) to out_keys/out_vals and the group sizes to
 * send_counts[G] (host).  0 <= nsplit <= 1023 (G <= 1024: the splitter and
 * bucket tables live in shared memory); larger nsplit returns DTS_EINVAL.
 * No reference counterpart (multi-GPU extension); built from
 * the counting_sort machinery (counting.py:82-156). */
int dts_partition(const void* keys, const void* vals, uint64_t n,
                  uint64_t global_base, const void* split_keys,
                  const uint64_t* split_idx, int nsplit, void* out_keys,
                  void* out_vals, uint64_t* send_counts, int key_bytes,
                  int val_bytes, void* workspace, size_t workspace_bytes,
                  void* stream);

/* Seeded R-MAT edge generator (C5 workload; the reference's edge generator is
 * generate_edges, gen.py:194-214, Zipf-skewed instead).  Edge i (global index
 * edge_base + i) descends `scale` levels; at level l a 32-bit draw
 * u = hi32(splitmix64 mix of (seed, edge, l)) picks quadrant a (u < t0),
 * b (< t1), c (< t2) or d; src bit = {c,d}, dst bit = {b,d}, MSB first.
 * dst/src: device arrays of n uint32. */
int dts_gen_rmat(uint32_t* dst, uint32_t* src, uint64_t n, uint64_t edge_base,
                 uint64_t seed, int scale, uint32_t t0, uint32_t t1, uint32_t t2,
                 void* stream);

/* CSR row offsets of ascending keys below nverts (graph transpose after the
 * sort; reference bench.py:348-349: bincount + cumsum): row_ptr[v] = number
 * of keys < v for v in [0, nverts] (nverts + 1 device uint64).  EINVAL if the
 * keys descend or reach nverts.  Blocks on the stream (one flag read). */
size_t dts_csr_workspace_bytes(uint64_t nverts);
int dts_csr_offsets(const void* keys, uint64_t n, int key_bytes, uint64_t nverts,
                    uint64_t* row_ptr, void* workspace, size_t workspace_bytes,
                    void* stream);

/* Message for the last nonzero status on this thread. */
const char* dts_last_error(void);

/* Morton (z-order) keys of n points — the paper's Morton-sort application
 * (PAPER.md:1149-1165): keys[i] interleaves the low `bits` bits of the
 * point's coordinates (x, y[, z]: device arrays of uint32; dims 2 or 3; bits
 * <= 32 for 2-D, <= 21 for 3-D), coordinate 0 in the lowest bit of each
 * group: bit dims*i + c of the key = bit i of coordinate c.  vals (may be
 * NULL) receives first_index + i, the payload that makes dts_sort(keys,
 * vals) a Morton sort returning the point permutation.  workspace: >= 16
 * device bytes.  DTS_EINVAL (and keys written) when a coordinate has a bit
 * at or above `bits`.  Blocks once (the range check). */
int dts_morton_keys(const uint32_t* x, const uint32_t* y, const uint32_t* z,
                    uint64_t n, int dims, int bits, uint64_t* keys,
                    uint64_t* vals, uint64_t first_index, void* workspace,
                    size_t workspace_bytes, void* stream);

/* DTS_ABI_VERSION and the SM architecture the library was built for (100). */
int dts_abi_version(void);
int dts_build_arch(void);

#ifdef __cplusplus
}
#endif
#endif /* DTS_H_ */
