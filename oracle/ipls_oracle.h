/*
 * ipls_oracle.h — plain, slow, single-threaded CPU oracle for the IPLS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2208_06902_b200 + libipls.so) never links, imports or calls it, and the
 * two share no code: no headers, helpers, tables or constants.
 *
 * Paper: "In-Place Parallel Learned Sort" (arXiv 2208.06902), reference file
 * /root/reference/PAPER.md, cited as P:<line>.  Readings of the paper where it is
 * silent or ambiguous are listed in DESIGN.md §3 ("R<n>").
 *
 * Every floating-point step is one IEEE binary64 round-to-nearest operation in the
 * order written (compile with -ffp-contract=off, SSE2; no fast-math).
 */
#ifndef IPLS_ORACLE_H
#define IPLS_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_KEY_F64 = 0, ORACLE_KEY_U64 = 1 };
enum { ORACLE_MODEL_LINEAR = 0, ORACLE_MODEL_EQ3 = 1, ORACLE_MODEL_TREE = 2,
       ORACLE_MODEL_TREE_EQ = 3 /* a sort option: its records carry kind ORACLE_MODEL_TREE */ };

/* Order-preserving key ("extractor ... maps double to integers"). */
uint64_t oracle_ordering_key(uint64_t bits, int key_type);

/* SplitMix64 output function (R18). */
uint64_t oracle_splitmix64(uint64_t z);

/* Sample size S(m) = min(max(ceil(ceil(log2 m)/5)*k - 1, 4), floor(m/2)) (R1, R19). */
uint64_t oracle_sample_size(uint64_t m, uint32_t k);

/* Stratified sample positions of a segment (R2, R18); writes S absolute indices. */
void oracle_sample_positions(uint64_t seed, uint32_t level, uint64_t begin, uint64_t m,
                             uint64_t S, uint64_t* idx_out);

/* FMCD, Listing 1 in binary64 (R3, R4).  s: S sorted model values.
 * Returns 0 for a usable linear model, 1 when degenerate (R5: !(u>0) or A/B
 * non-finite).  A, B, D, capped are always written. */
int oracle_fit_fmcd(const double* s, size_t S, uint32_t k, double* A, double* B,
                    uint32_t* D, uint32_t* capped);

/* Bucket of one key (R7).  kind LINEAR uses (A,B,k); EQ3 uses pivot_ok. */
uint32_t oracle_bucket(uint64_t bits, int key_type, int kind, double A, double B, uint32_t k,
                       uint64_t pivot_ok);

/* Stable counting partition of n keys (R11).  offsets: k_eff+1 entries
 * (k_eff = k for LINEAR, 3 for EQ3).  ids (nullable): per-key bucket, input order. */
void oracle_partition(const uint64_t* in, uint64_t* out, size_t n, int key_type, int kind,
                      double A, double B, uint32_t k, uint64_t pivot_ok, uint64_t* offsets,
                      uint16_t* ids);

/* Splitter-tree model (IPS4o's decision tree; DESIGN.md
 * R22-R24): the k-1 splitters are the equidistant order statistics s[floor(i S / k)],
 * i = 1..k-1, of the sorted sample (k a power of two), as ordering keys.  spl_ok: k-1
 * entries, nondecreasing. */
void oracle_tree_splitters(const uint64_t* sorted_bits, size_t S, uint32_t k, int key_type,
                           uint64_t* spl_ok);
/* Bucket of one key under the tree: the branchless descent j <- 2j + (x > a_j) over the
 * implicit tree of the splitters ends at leaf #{i : spl_i < ok(x)} (ties go left, R23),
 * which is what this returns (the plain definition, by binary search). */
uint32_t oracle_tree_bucket(uint64_t bits, int key_type, const uint64_t* spl_ok, uint32_t k);
/* IPS4o's equality buckets ("a bucket B_i just for the elements x = s_i"; DESIGN.md
 * R24): a tree of `leaves` leaves (leaves-1 splitters spl_ok) feeds 2*leaves buckets; a key in
 * leaf i goes to bucket 2i+1 if it equals splitter s_i (i < leaves-1), else to bucket 2i.
 * Every odd bucket holds one value, so it is final after the partition. */
uint32_t oracle_tree_eq_bucket(uint64_t bits, int key_type, const uint64_t* spl_ok,
                               uint32_t leaves);

/* One record per partitioned segment, in level order then increasing begin. */
typedef struct {
  uint32_t level, kind;
  uint64_t begin, m, S;
  double A, B;
  uint32_t D, capped;
  uint64_t pivot_ok;
  uint32_t k_eff;      /* number of children (k or 3) */
  uint32_t requeued;   /* 1 when the no-progress guard re-queued this segment (R10) */
} oracle_record;

typedef struct oracle_trace oracle_trace;
oracle_trace* oracle_trace_new(int keep_snapshots);
void oracle_trace_free(oracle_trace* t);
size_t oracle_trace_num_records(const oracle_trace* t);
void oracle_trace_record(const oracle_trace* t, size_t i, oracle_record* out);
/* Sorted sample of record i, as raw key bits (S entries). */
const uint64_t* oracle_trace_sample(const oracle_trace* t, size_t i);
/* Child counts of record i (k_eff entries). */
const uint64_t* oracle_trace_counts(const oracle_trace* t, size_t i);
uint32_t oracle_trace_num_levels(const oracle_trace* t);
/* Array image after level L's partition (n keys), when snapshots were kept. */
const uint64_t* oracle_trace_snapshot(const oracle_trace* t, uint32_t level);

/* Whole sort, level-batched.  keys: n raw 64-bit words,
 * sorted in place by ordering key.  Returns 0, or 2 if a NaN key was found (array
 * unmodified), or 1 on invalid arguments. */
int oracle_sort(uint64_t* keys, size_t n, int key_type, uint32_t k, uint32_t base_case,
                uint64_t seed, oracle_trace* trace);
/* Same with the model chosen: ORACLE_MODEL_LINEAR (FMCD, the paper's IPLS) or
 * ORACLE_MODEL_TREE (splitter tree, IPS4o's classifier; k must be a power of two >= 4) or
 * ORACLE_MODEL_TREE_EQ (the tree with equality buckets, R24: k/2 leaves, k buckets; k a
 * power of two >= 8). */
int oracle_sort_model(uint64_t* keys, size_t n, int key_type, uint32_t k, uint32_t base_case,
                      uint64_t seed, int model, oracle_trace* trace);

#ifdef __cplusplus
}
#endif
#endif
