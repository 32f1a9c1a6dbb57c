/*
 * ipls.h — C ABI of the B200 (sm_100a) IPLS distribution-step library, libipls.so.
 *
 * Paper: "In-Place Parallel Learned Sort" (IPLS), arXiv 2208.06902; the reference text is
 * PAPER.md, cited here as P:<line>.  Readings of the paper where it is silent or ambiguous
 * are numbered R<n> and listed in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *  - d_* arguments are CUDA device pointers, h_* arguments host pointers.  Keys are 64-bit
 *    words: IEEE binary64 (IPLS_KEY_F64) or unsigned 64-bit integers (IPLS_KEY_U64),
 *    8-byte aligned, contiguous.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is
 *    stream-ordered; every call synchronises `stream` once before returning so it can
 *    return a status (timing with events must bracket the call).
 *  - No exceptions cross the ABI; errors are returned as ipls_status.  On any error other
 *    than IPLS_ERR_CUDA the caller's key array is left unmodified.
 *  - Thread safety: concurrent calls on different streams are safe; the library keeps one
 *    internal workspace per stream (guarded by a mutex) unless the caller passes its own.
 *  - Ordering: keys are sorted by the ordering key of P:576 (the float -> integer map):
 *    numeric order for doubles with -0.0 before +0.0; NaN is rejected (R0).
 */
#ifndef IPLS_H
#define IPLS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IPLS_OK = 0,
  IPLS_ERR_INVALID_ARGUMENT = 1, /* null pointer with n > 0, k < 3 or k > IPLS_MAX_K, ... */
  IPLS_ERR_NAN_KEY = 2,          /* a float64 key is NaN; the array is left unmodified  */
  IPLS_ERR_DEGENERATE_SAMPLE = 3,/* ipls_fit_fmcd only: Listing 1 gave no usable model */
  IPLS_ERR_OUT_OF_MEMORY = 4,    /* device allocation or caller workspace too small     */
  IPLS_ERR_CUDA = 5,             /* a CUDA runtime error (see ipls_last_cuda_error)      */
  IPLS_ERR_NOT_IMPLEMENTED = 6
} ipls_status;

typedef enum { IPLS_KEY_F64 = 0, IPLS_KEY_U64 = 1 } ipls_key_type;

/* Partition model kinds.  LINEAR: F(x) = clamp(floor(a*x + b), 0, k-1) with
 * (a, b) from FMCD (Listing 1).  EQ3: equality split into <pivot, ==pivot,
 * >pivot by ordering key (IPS4o equality buckets; used for degenerate samples, R5). */
typedef enum { IPLS_MODEL_LINEAR = 0, IPLS_MODEL_EQ3 = 1, IPLS_MODEL_TREE = 2 } ipls_model_kind;

/* ipls_config.flags.  IPLS_FLAG_TREE_MODEL: classify with IPS4o's splitter tree (
 * SURVEY §8(f) NEXT #2; R22-R24) instead of the FMCD linear model: the k-1
 * splitters are the equidistant order statistics of the same sorted sample, and every key
 * descends j <- 2j + (x > a_j) (ties left).  k must be a power of two.  Degenerate cases
 * and the no-progress guard are the same (EQ3).  Trace records carry kind IPLS_MODEL_TREE. */
#define IPLS_FLAG_TREE_MODEL 1u
/* IPLS_FLAG_TREE_EQUAL_BUCKETS (only with IPLS_FLAG_TREE_MODEL; k a power of two >= 8):
 * IPS4o's equality buckets ("a bucket B_i just for the elements x = s_i"; DESIGN.md
 * R24).  The tree has k / 2 leaves (k / 2 - 1 splitters s_0 <= s_1 <= ...); a key in leaf i
 * goes to bucket 2i + 1 if it equals s_i and to bucket 2i otherwise, so the k buckets stay
 * range-ordered and every odd bucket holds one value (final after the partition). */
#define IPLS_FLAG_TREE_EQUAL_BUCKETS 2u

#define IPLS_MAX_K 1024u          /* fan-out limit of the sm_100a kernels (smem-resident) */
#define IPLS_MAX_BASE_CASE 4096u  /* base-case limit (n <= 2^12)                    */
#define IPLS_DEFAULT_SEED 0x49504C53ull

typedef struct {
  uint32_t k;         /* buckets per level, 3..IPLS_MAX_K (P:473 uses 256)                 */
  uint32_t base_case; /* segments of <= base_case keys go to the base case, 1..4096 */
  uint64_t seed;      /* sampling seed (R18)                                               */
  uint32_t flags;     /* 0, IPLS_FLAG_TREE_MODEL (k a power of two), or that with
                         IPLS_FLAG_TREE_EQUAL_BUCKETS; other bits or combinations: invalid  */
} ipls_config;

typedef struct {
  double a, b;        /* LINEAR: slope A and intercept B of Listing 1 (0 for EQ3)          */
  uint32_t k;         /* bucket count the model was fitted for (k_eff = 3 for EQ3)         */
  uint32_t D;         /* FMCD conflict degree (0 for EQ3)                                   */
  uint32_t kind;      /* ipls_model_kind                                                    */
  uint32_t capped;    /* 1 if Listing 1 stopped at D*3 > N (R4)                             */
  uint64_t pivot_ok;  /* EQ3: ordering key of the pivot (0 for LINEAR)                      */
} ipls_model;

/* Default configuration: k = 256, base_case = 4096, seed = IPLS_DEFAULT_SEED. */
ipls_config ipls_default_config(void);

/* Sort n keys in place on the device (P:114-121 recursion, P:469-475 IPLS parameters).
 * d_keys: device array of n keys, caller-owned.  Uses an internal workspace (8n bytes of
 * scratch plus metadata, see ipls_workspace_bytes) cached per stream.
 * n == 0 or 1: IPLS_OK without touching memory.  Errors: INVALID_ARGUMENT (d_keys NULL
 * with n > 0, n > 2^32-1), NAN_KEY (array unmodified), OUT_OF_MEMORY, CUDA. */
ipls_status ipls_sort_f64(double* d_keys, size_t n, void* stream);
ipls_status ipls_sort_u64(uint64_t* d_keys, size_t n, void* stream);

/* As above with an explicit key type and configuration.  d_workspace may be NULL (internal
 * cache) or a device buffer of at least ipls_workspace_bytes(n, t, cfg) bytes, which the
 * call owns for its duration.  cfg NULL = ipls_default_config(). */
ipls_status ipls_sort_ex(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                         void* d_workspace, size_t ws_bytes, void* stream);

/* Device workspace ipls_sort_ex needs: one n-key scratch buffer (8n bytes; the ping-pong
 * target that replaces IPS4o's in-place block permutation) plus per-level
 * metadata bounded by n, k and base_case. */
size_t ipls_workspace_bytes(size_t n, ipls_key_type t, const ipls_config* cfg);

/* End-to-end variant: h_keys is a HOST array (ideally pinned); the call copies it to the
 * device, sorts, and copies the result back, all on `stream`. */
ipls_status ipls_sort_host(void* h_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                           void* stream);

/* Sort `count` HOST arrays (P:637's sorting rate for data that starts and ends in host
 * memory): array j is copied from h_in[j] to the device, sorted as ipls_sort_ex sorts it, and
 * copied back to h_out[j] (which may equal h_in[j]).  The copies are pipelined over three
 * internal streams, each with its own device buffer: array j+1's host-to-device copy is issued
 * before array j is sorted, so it overlaps that sort and the earlier arrays' device-to-host
 * copies (the PCIe link carries both directions at once).  The batch starts after the work queued on `stream`; the call returns
 * when every output is written.  h_in[j], h_out[j]: host (pinned for overlap), n[j] keys each;
 * distinct outputs must not overlap each other or another array's input.  Device memory:
 * three io buffers and three workspaces (one per internal stream), cached.  Errors: INVALID_ARGUMENT
 * (NULL arrays, a NULL buffer with n[j] > 0, bad key type or config), the first sort's error
 * (e.g. NAN_KEY: arrays from that one on are left unspecified), OUT_OF_MEMORY, CUDA. */
ipls_status ipls_sort_host_batch(const void* const* h_in, void* const* h_out, const size_t* n,
                                 uint32_t count, ipls_key_type t, const ipls_config* cfg,
                                 void* stream);

/* FMCD fit (Listing 1, binary64, R3/R4) of one already-sorted sample.
 * d_sorted_sample: S keys of type t sorted by ordering key (device).  S >= 4, 3 <= k <=
 * IPLS_MAX_K, S <= 8192 (the fit kernel's smem sample).  Writes *h_out.  Returns IPLS_ERR_DEGENERATE_SAMPLE (with
 * h_out->kind = EQ3 and pivot_ok = ordering key of s[S/2]) when !(u_d > 0) or A, B are not
 * finite (R5). */
ipls_status ipls_fit_fmcd(const void* d_sorted_sample, size_t S, ipls_key_type t, uint32_t k,
                          ipls_model* h_out, void* stream);

/* As ipls_fit_fmcd for an UNSORTED sample: the fit kernel sorts the S keys by ordering key
 * in shared memory first (the same CTA sort the sort's own fits use), then fits.
 * Used by the multi-GPU top level (one launch instead of a sort call plus a fit call). */
ipls_status ipls_fit_sample(const void* d_sample, size_t S, ipls_key_type t, uint32_t k,
                            ipls_model* h_out, void* stream);

/* One distribution step of a single segment with a caller-supplied model: classify every
 * key (evaluated as RN(RN(a*x) + b), no FMA, R7), histogram, prefix-sum and
 * stable scatter into contiguous buckets (R11).
 * d_in, d_out: n keys each (device, must not overlap).  d_offsets: k_eff+1 uint64 bucket
 * boundaries (device).  d_bucket_ids: nullable; n uint16 per-key buckets in input order. */
ipls_status ipls_partition_level(const void* d_in, void* d_out, size_t n, ipls_key_type t,
                                 const ipls_model* h_model, uint64_t* d_offsets,
                                 uint16_t* d_bucket_ids, void* stream);

/* ---- distributed top level (P:144-153 parallel sample sort) ----
 * A global array is the concatenation, in rank order, of G ranks' device shards.  The
 * exchange (paper_2208_06902_b200/distributed.py) is: (1) every rank writes the strata of
 * the global level-0 sample it holds (ipls_sample_strata) and a SUM all-reduce assembles the
 * whole sample; (2) every rank sorts it (ipls_sort_ex) and fits the same model
 * (ipls_fit_fmcd); (3) every rank partitions its shard by that model (ipls_partition_level);
 * (4) the per-rank bucket counts are all-gathered and ipls_assign_cuts gives rank r the
 * global positions [cuts[r], cuts[r+1]) of the bucket-major order (bucket boundaries, or
 * inside EQ3's one-valued ==pivot bucket); (5) one all-to-all moves the keys, every rank puts
 * its G runs into bucket-major order (ipls_regroup_runs) and resumes the recursion at level 1
 * (ipls_sort_segments).  Rank r then holds the r-th key range. */

/* The exchange fused into the partition (DESIGN.md §7 "fused exchange"; every
 * thread -- here every GPU -- moves its keys straight into the buckets' final places).
 * Instead of steps (3) and (5)'s partition + all-to-all + regroup, a rank (3') counts its
 * buckets (ipls_partition_count), the counts are all-gathered and the plan of step (4) gives,
 * for every bucket b, the address in the owning rank's receive buffer where this rank's keys
 * of b belong (bucket-major, then source rank: base of b in the owner's buffer + the counts of
 * b on lower ranks), and (5') ipls_partition_scatter_to writes them there directly (peer
 * memory over NVLink; plain 8-byte stores in runs of consecutive keys).  After a barrier the
 * owner's buffer is what ipls_regroup_runs would have produced.
 *
 * ipls_partition_count: the classify half of ipls_partition_level.  d_in: n keys (device);
 * d_offsets: k_eff+1 uint64 bucket boundaries of the stable partition (device).
 * ipls_partition_scatter_to: classifies again (the per-chunk prefixes are not kept between
 * calls: 8 B/key of reads buy a stateless interface) and scatters stably: this array's keys
 * of bucket b, in input order, go to the consecutive 64-bit words starting at the ADDRESS
 * d_bucket_dst[b] (device array of k_eff addresses, each 8-byte aligned, of memory the
 * device can store to: its own or a peer's mapped allocation); the destinations of different
 * buckets must not overlap each other or d_in.  Entries of empty buckets are ignored.
 * Both: models LINEAR or EQ3, n <= 2^32-1, synchronise `stream`; errors as
 * ipls_partition_level. */
ipls_status ipls_partition_count(const void* d_in, size_t n, ipls_key_type t,
                                 const ipls_model* h_model, uint64_t* d_offsets, void* stream);
ipls_status ipls_partition_scatter_to(const void* d_in, size_t n, ipls_key_type t,
                                      const ipls_model* h_model, const uint64_t* d_bucket_dst,
                                      void* stream);

/* Sort n keys that form nseg consecutive range-ordered segments -- every key of segment i
 * precedes (ordering key) every key of segment i+1 -- by resuming the recursion
 * at `level`: each segment of more than base_case keys is partitioned as a
 * level-`level` segment (its sample drawn with that level's hash, R2/R18, as if an earlier
 * level had produced it), each smaller one goes to the base case.  This is the local
 * sort of the multi-GPU top level: with level = 1, the top level's buckets, in
 * global order, as the segments and global_begin = the position of d_keys[0] in the global
 * bucket-major order, every model and layout below the top level equals the one-GPU sort's.
 * global_begin only enters the sampling hash (R18 hashes a segment's begin; here begin =
 * global_begin + the segment's offset in d_keys); addressing stays local.  d_keys: device, n
 * keys sorted in place.  h_seg_sizes: host, nseg sizes summing to n (zeros allowed).  Uses
 * the stream's internal workspace.  Errors: as
 * ipls_sort_ex (NaN: the array is left unmodified), INVALID_ARGUMENT if the sizes do not sum
 * to n.  The segments are trusted to be range-ordered (not checked); if they are not, the
 * output is not sorted. */
ipls_status ipls_sort_segments(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                               const uint64_t* h_seg_sizes, uint32_t nseg, uint32_t level,
                               uint64_t global_begin, void* stream);

/* Multi-GPU exchange: the receiving rank holds G runs back to back, run g
 * (from source rank g, in rank order) holding that source's keys of buckets b0 .. b0+nb-1,
 * bucket-major (a stable partition's output).  Moves them into bucket-major order: for each
 * bucket, run 0's keys, then run 1's, ... -- the stable partition of the concatenated global
 * array restricted to these buckets.  d_src, d_dst: device, distinct, sum(h_counts) keys
 * each.  h_counts: host, G x nb (row g = run g's bucket counts).  Synchronises `stream`.
 * Errors: INVALID_ARGUMENT (NULL), OUT_OF_MEMORY, CUDA. */
ipls_status ipls_regroup_runs(const void* d_src, void* d_dst, const uint64_t* h_counts,
                              uint32_t G, uint32_t nb, void* stream);

/* S(m) = min(max(ceil(ceil(log2 m)/5) k - 1, 4), floor(m/2)) (R1, R19).  Host only. */
uint32_t ipls_sample_size(uint64_t m, uint32_t k);

/* Level-0 stratified sample (R2, R18: stratum j of [0, global_m) at level 0, begin 0,
 * position lo_j + umulhi(h_j, hi_j - lo_j)) of the global array, restricted to this rank's
 * positions [global_begin, global_begin + n_local).  d_keys: the rank's n_local keys
 * (device).  d_sample: S uint64 slots (device, caller-owned); slot j receives the key's bits
 * if this rank holds stratum j's position and is left untouched otherwise, so zero-filled
 * buffers summed over ranks give exactly the sample a one-GPU ipls_sort of the concatenated
 * array draws at level 0 (same seed).  S == 0: no-op.  Errors: INVALID_ARGUMENT (NULL
 * pointers, S > global_m, S > 8192 (the largest sample the fit kernels take), the rank's range
 * outside [0, global_m), global_m >= 2^48), CUDA. */
ipls_status ipls_sample_strata(const void* d_keys, size_t n_local, uint64_t global_begin,
                               uint64_t global_m, uint32_t S, uint64_t seed, uint64_t* d_sample,
                               void* stream);

/* Contiguous bucket ranges for G ranks balanced by count.  Host only.
 * h_counts: k global bucket counts.  h_bounds: G+1 entries out; bounds[0] = 0, bounds[G] = k,
 * nondecreasing; bounds[r] is the boundary b >= bounds[r-1] whose prefix count
 * sum(counts[0..b)) is closest to r/G of the total (ties: the lower b).  Rank r receives
 * buckets [bounds[r], bounds[r+1]).  Errors: INVALID_ARGUMENT (NULL, k == 0, G == 0). */
ipls_status ipls_assign_ranges(const uint64_t* h_counts, uint32_t k, uint32_t G,
                               uint32_t* h_bounds);

/* Global cut positions for G ranks when some buckets may be split between ranks (SURVEY
 * §8(e) step 4; a bucket known to hold one key value, e.g. EQ3's ==pivot bucket (R5), can go
 * to several ranks without changing the sorted result).  Host only.  h_counts: k global bucket
 * counts; h_splittable: k flags (NULL = none).  h_cuts: G+1 positions out in the bucket-major
 * global order; cuts[0] = 0, cuts[G] = total, nondecreasing; cuts[r] is the candidate >=
 * cuts[r-1] closest to r/G of the total (ties: the lower), the candidates being the bucket
 * boundaries and every position strictly inside a splittable bucket.  Rank r receives
 * positions [cuts[r], cuts[r+1]).  With no splittable bucket cuts[r] is the prefix count at
 * ipls_assign_ranges' bounds[r].  Errors: INVALID_ARGUMENT (NULL counts/cuts, k == 0,
 * G == 0, total >= 2^64). */
ipls_status ipls_assign_cuts(const uint64_t* h_counts, uint32_t k, uint32_t G,
                             const uint8_t* h_splittable, uint64_t* h_cuts);

/* ---- trace (tests and diagnostics) ---- */
typedef struct {
  uint32_t level, kind;     /* level of the recursion; ipls_model_kind                      */
  uint64_t begin, m, S;     /* segment [begin, begin+m) and its sample size                  */
  double a, b;              /* model (0 for EQ3)                                             */
  uint32_t D, capped;       /* FMCD outputs (0 for EQ3)                                      */
  uint64_t pivot_ok;        /* EQ3 pivot (0 for LINEAR)                                      */
  uint32_t k_eff, requeued; /* children count; 1 if re-queued by the no-progress guard (R10) */
} ipls_segment_record;

typedef struct {
  ipls_segment_record* records; size_t records_cap; size_t records_len; /* host, out       */
  uint64_t* counts; size_t counts_cap; size_t counts_len;  /* host: k_eff per record, out  */
  uint64_t* samples; size_t samples_cap; size_t samples_len; /* host: sorted sample bits  */
  void* d_snapshots;        /* device, nullable: snapshot_levels * n keys, array after level L */
  uint32_t snapshot_levels;
  uint32_t levels;          /* out: number of partition levels run                           */
} ipls_trace;

/* ipls_sort_ex plus a per-segment trace, records ordered by (level, begin).  Arrays that
 * are too small are filled up to their capacity and *_len reports the full size. */
ipls_status ipls_sort_trace(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                            ipls_trace* trace, void* stream);
/* ipls_sort_segments with the per-segment trace of ipls_sort_trace (records carry the hash
 * level, starting at `level`; snapshots by iteration).  Same arguments and errors. */
ipls_status ipls_sort_segments_trace(void* d_keys, size_t n, ipls_key_type t,
                                     const ipls_config* cfg, const uint64_t* h_seg_sizes,
                                     uint32_t nseg, uint32_t level, uint64_t global_begin,
                                     ipls_trace* trace, void* stream);

const char* ipls_status_string(ipls_status s);
const char* ipls_last_cuda_error(void);
/* Test hook: set the level counter whose low 16 bits tag the lookback status words (the
 * regression test for stale words that look valid, tests/test_gpu_parity.py). */
void ipls_debug_set_epoch(uint32_t e);
/* Test hook: on != 0 makes every CTA of the stable scatter rank keys with match.any peer
 * masks (stable by construction), the path it otherwise takes only if its probe finds that
 * same-address lanes of a shared-memory atomic are not served in lane order (DESIGN.md §5,
 * K3).  Applies to the current device; 0 restores the default. */
void ipls_debug_force_match_rank(int on);
/* Test hook: how a level's terminal segments (every child <= base case) are processed.
 * 0 (default): the child scatter fused with the warp base case (k_term_fused) when the
 * level's segments average >= 32 Ki keys, else the child scatter and the base-case kernels
 * separately; 1: always fused; 2: never fused; 3: the terminal segment sort -- windows of
 * whole children of <= 16 Ki keys, a window scatter for segments of several windows, one CTA
 * sorting each window into the user array (k_tss_scatter, k_win_sort; measured slower,
 * DESIGN.md §5).  All four give identical records and final arrays.  Process-wide. */
void ipls_debug_term_mode(int mode);
/* Number of kernels the library enqueued since load (diagnostics / bench launch count). */
uint64_t ipls_kernel_launch_count(void);

/* ---- per-kernel timing (bench.py roofline) ----
 * When enabled, every kernel launch is bracketed by CUDA events recorded on the launching
 * stream; durations are collected when the call synchronises.  `bytes` is the launch's
 * ALGORITHMIC traffic: 8 B/key read for classify, 16 B/key for scatter and
 * base case, 8 B/key for fills; 0 for metadata kernels. */
typedef struct {
  char name[32];
  uint64_t launches;
  double total_ms;
  double bytes;
} ipls_profile_entry;
void ipls_profile_enable(int on);
void ipls_profile_reset(void);
/* Copies up to cap entries into out; returns the number of distinct kernels. */
size_t ipls_profile_read(ipls_profile_entry* out, size_t cap);

#ifdef __cplusplus
}
#endif
#endif
