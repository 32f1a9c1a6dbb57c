/*
 * ipls_oracle.cpp — plain, slow, single-threaded CPU oracle for the IPLS hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see ipls_oracle.h).  Written from the paper, step by
 * step, in the paper's order; no blocking, fusion or reordering.  Compiled with
 * g++ -O2 -ffp-contract=off (no FMA contraction, SSE2 binary64).
 *
 * Parity pins (tests/test_oracle_*.py): the worked example P:477-561, Listing 1's
 * declarative characterisation (brute force), closed forms for s_i = i, exact
 * rationals for the bucket function, std::sort / numpy sort of the whole array,
 * the SplitMix64 published test vector, brute-force partitions for n <= 64.
 * Parity unpinned against the paper: the sampling positions (the paper says only
 * "random elements") — pinned by structure tests only.
 */
#include "ipls_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace {

/* ---- order-preserving map from the key's bits to an unsigned integer. ---- */
uint64_t ok_of(uint64_t bits, int key_type) {
  if (key_type == ORACLE_KEY_U64) return bits;
  /* negative doubles: invert every bit; non-negative: set the sign bit. */
  if (bits >> 63) return ~bits;
  return bits | (1ull << 63);
}

/* Model domain: the double itself (f64) or the u64 converted with RN-even (R17). */
double value_of(uint64_t bits, int key_type) {
  if (key_type == ORACLE_KEY_U64) return (double)bits;
  double x;
  std::memcpy(&x, &bits, 8);
  return x;
}

bool is_nan_bits(uint64_t bits) {
  return ((bits >> 52) & 0x7ff) == 0x7ff && (bits & 0xfffffffffffffull) != 0;
}

uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t bit_length(uint64_t x) {
  uint64_t r = 0;
  while (x) { ++r; x >>= 1; }
  return r;
}

/* floor(h * r / 2^64) — plain 128-bit product. */
uint64_t mulhi(uint64_t h, uint64_t r) {
  return (uint64_t)(((unsigned __int128)h * (unsigned __int128)r) >> 64);
}

struct Model {
  int kind;
  double A, B;
  uint32_t k;
  uint32_t D, capped;
  uint64_t pivot_ok;
  const uint64_t* spl = nullptr;  /* TREE: leaves-1 sorted splitters (ordering keys) */
  uint32_t leaves = 0;            /* TREE: k, or k/2 with equality buckets (R24) */
};

/* R23: leaf of the descent j <- 2j + (x > a_j) = number of splitters strictly below x. */
uint32_t tree_bucket_of(uint64_t o, const uint64_t* spl, uint32_t k) {
  return (uint32_t)(std::lower_bound(spl, spl + (k - 1), o) - spl);
}

/* R24: leaf i of a tree of L leaves as above; the keys equal to splitter s_i take the
 * equality bucket 2i+1, the keys strictly between s_{i-1} and s_i the bucket 2i. */
uint32_t tree_eq_bucket_of(uint64_t o, const uint64_t* spl, uint32_t L) {
  const uint32_t i = tree_bucket_of(o, spl, L);
  const bool eq = i < L - 1 && spl[i] == o;
  return 2 * i + (eq ? 1u : 0u);
}

/* P:394-402 with R7: y = RN(RN(A*v) + B); 0 if !(y >= 0); k-1 if y >= k; else floor(y). */
uint32_t bucket_of(uint64_t bits, int key_type, const Model& md) {
  if (md.kind == ORACLE_MODEL_TREE)
    return md.leaves == md.k ? tree_bucket_of(ok_of(bits, key_type), md.spl, md.k)
                             : tree_eq_bucket_of(ok_of(bits, key_type), md.spl, md.leaves);
  if (md.kind == ORACLE_MODEL_EQ3) {
    uint64_t o = ok_of(bits, key_type);
    if (o < md.pivot_ok) return 0;
    if (o == md.pivot_ok) return 1;
    return 2;
  }
  double v = value_of(bits, key_type);
  volatile double t = md.A * v; /* volatile: one rounding for the product, then one for the sum */
  double y = t + md.B;
  if (!(y >= 0.0)) return 0;
  if (y >= (double)md.k) return md.k - 1;
  return (uint32_t)y; /* 0 <= y < k: truncation == floor */
}

struct Seg {
  uint64_t begin, m;
  int force_eq3;
};

}  // namespace

struct oracle_trace {
  int keep_snapshots;
  std::vector<oracle_record> recs;
  std::vector<std::vector<uint64_t>> samples;
  std::vector<std::vector<uint64_t>> counts;
  std::vector<std::vector<uint64_t>> snaps;
  uint32_t levels = 0;
};

extern "C" {

uint64_t oracle_ordering_key(uint64_t bits, int key_type) { return ok_of(bits, key_type); }
uint64_t oracle_splitmix64(uint64_t z) { return sm64(z); }

uint64_t oracle_sample_size(uint64_t m, uint32_t k) {
  /* "alpha k - 1 random elements ... alpha = 0.2 log N", read as
   * alpha = ceil(ceil(log2 m) / 5) (R1); at least 4 so Listing 1 has s[D], s[N-1-D]
   * (R19); at most floor(m/2). */
  uint64_t lg = (m > 0) ? bit_length(m - 1) : 0; /* ceil(log2 m) */
  uint64_t alpha = (lg + 4) / 5;
  uint64_t S = alpha * (uint64_t)k;
  S = (S >= 1) ? S - 1 : 0;
  if (S < 4) S = 4;
  if (S > m / 2) S = m / 2;
  return S;
}

void oracle_sample_positions(uint64_t seed, uint32_t level, uint64_t begin, uint64_t m,
                             uint64_t S, uint64_t* idx_out) {
  /* One position per stratum j: [floor(j m / S), floor((j+1) m / S)) (R2, R18). */
  uint64_t t = sm64(sm64(sm64(seed) ^ (uint64_t)level) ^ begin);
  for (uint64_t j = 0; j < S; ++j) {
    uint64_t lo = (uint64_t)(((unsigned __int128)j * m) / S);
    uint64_t hi = (uint64_t)(((unsigned __int128)(j + 1) * m) / S);
    uint64_t h = sm64(t ^ j);
    idx_out[j] = begin + lo + mulhi(h, hi - lo);
  }
}

int oracle_fit_fmcd(const double* s, size_t S, uint32_t k, double* A_out, double* B_out,
                    uint32_t* D_out, uint32_t* capped_out) {
  /* Listing 1, literally, in binary64 (R3).  N = S, K = k. */
  const size_t N = S;
  size_t i = 0;
  size_t D = 1;
  const double km2 = (double)(k - 2);
  double u_d = (s[N - 1 - D] - s[D]) / km2;
  int capped = 0;
  while (i <= N - 1 - D) {
    while (i + D < N && (s[i + D] - s[i]) >= u_d) {
      i++;
    }
    if (i + D >= N) break;
    D += 1;
    if (D * 3 > N) { capped = 1; break; } /* R4: u_d stays u_d(D-1) */
    u_d = (s[N - 1 - D] - s[D]) / km2;
  }
  double A = 1.0 / u_d;
  double sum = s[N - 1 - D] + s[D];
  double prod = A * sum;
  double B = ((double)k - prod) / 2.0;
  *A_out = A;
  *B_out = B;
  *D_out = (uint32_t)D;
  *capped_out = (uint32_t)capped;
  /* R5: degenerate sample -> the caller uses the equality split instead. */
  if (!(u_d > 0.0) || !std::isfinite(A) || !std::isfinite(B) || !(A > 0.0)) return 1;
  return 0;
}

uint32_t oracle_bucket(uint64_t bits, int key_type, int kind, double A, double B, uint32_t k,
                       uint64_t pivot_ok) {
  Model md{kind, A, B, k, 0, 0, pivot_ok};
  return bucket_of(bits, key_type, md);
}

void oracle_tree_splitters(const uint64_t* sorted_bits, size_t S, uint32_t k, int key_type,
                           uint64_t* spl_ok) {
  /* R22: equidistant order statistics of the sorted sample. */
  for (uint32_t i = 1; i < k; ++i)
    spl_ok[i - 1] = ok_of(sorted_bits[(size_t)(((unsigned __int128)i * S) / k)], key_type);
}

uint32_t oracle_tree_bucket(uint64_t bits, int key_type, const uint64_t* spl_ok, uint32_t k) {
  return tree_bucket_of(ok_of(bits, key_type), spl_ok, k);
}

uint32_t oracle_tree_eq_bucket(uint64_t bits, int key_type, const uint64_t* spl_ok,
                               uint32_t leaves) {
  return tree_eq_bucket_of(ok_of(bits, key_type), spl_ok, leaves);
}

namespace {
void partition_model(const uint64_t* in, uint64_t* out, size_t n, int key_type, const Model& md,
                     uint64_t* offsets, uint16_t* ids);
}

void oracle_partition(const uint64_t* in, uint64_t* out, size_t n, int key_type, int kind,
                      double A, double B, uint32_t k, uint64_t pivot_ok, uint64_t* offsets,
                      uint16_t* ids) {
  Model md{kind, A, B, k, 0, 0, pivot_ok};
  partition_model(in, out, n, key_type, md, offsets, ids);
}

namespace {
void partition_model(const uint64_t* in, uint64_t* out, size_t n, int key_type, const Model& md,
                     uint64_t* offsets, uint16_t* ids) {
  /* Counting sort by bucket, stable (R11). */
  const int kind = md.kind;
  const uint32_t k = md.k;
  uint32_t ke = (kind == ORACLE_MODEL_EQ3) ? 3 : k;
  std::vector<uint32_t> b(n);
  std::vector<uint64_t> cnt(ke, 0);
  for (size_t i = 0; i < n; ++i) {
    b[i] = bucket_of(in[i], key_type, md);
    cnt[b[i]]++;
    if (ids) ids[i] = (uint16_t)b[i];
  }
  std::vector<uint64_t> pos(ke + 1, 0);
  for (uint32_t j = 0; j < ke; ++j) pos[j + 1] = pos[j] + cnt[j];
  if (offsets)
    for (uint32_t j = 0; j <= ke; ++j) offsets[j] = pos[j];
  for (size_t i = 0; i < n; ++i) out[pos[b[i]]++] = in[i];
}
}  // namespace

oracle_trace* oracle_trace_new(int keep_snapshots) {
  oracle_trace* t = new oracle_trace();
  t->keep_snapshots = keep_snapshots;
  return t;
}
void oracle_trace_free(oracle_trace* t) { delete t; }
size_t oracle_trace_num_records(const oracle_trace* t) { return t->recs.size(); }
void oracle_trace_record(const oracle_trace* t, size_t i, oracle_record* out) { *out = t->recs[i]; }
const uint64_t* oracle_trace_sample(const oracle_trace* t, size_t i) { return t->samples[i].data(); }
const uint64_t* oracle_trace_counts(const oracle_trace* t, size_t i) { return t->counts[i].data(); }
uint32_t oracle_trace_num_levels(const oracle_trace* t) { return t->levels; }
const uint64_t* oracle_trace_snapshot(const oracle_trace* t, uint32_t level) {
  return level < t->snaps.size() ? t->snaps[level].data() : nullptr;
}

int oracle_sort(uint64_t* keys, size_t n, int key_type, uint32_t k, uint32_t base_case,
                uint64_t seed, oracle_trace* trace) {
  return oracle_sort_model(keys, n, key_type, k, base_case, seed, ORACLE_MODEL_LINEAR, trace);
}

int oracle_sort_model(uint64_t* keys, size_t n, int key_type, uint32_t k, uint32_t base_case,
                      uint64_t seed, int model, oracle_trace* trace) {
  if (k < 3 || k > 65535) return 1;
  if (model != ORACLE_MODEL_LINEAR && model != ORACLE_MODEL_TREE && model != ORACLE_MODEL_TREE_EQ)
    return 1;
  if (model == ORACLE_MODEL_TREE && (k < 4 || (k & (k - 1)) != 0)) return 1;
  if (model == ORACLE_MODEL_TREE_EQ && (k < 8 || (k & (k - 1)) != 0)) return 1;
  if (key_type != ORACLE_KEY_F64 && key_type != ORACLE_KEY_U64) return 1;
  if (n > 0 && keys == nullptr) return 1;
  /* Ingest: reject NaN before any write (R0). */
  if (key_type == ORACLE_KEY_F64)
    for (size_t i = 0; i < n; ++i)
      if (is_nan_bits(keys[i])) return 2;
  if (n <= 1) return 0;

  std::vector<uint64_t> tmp(n);
  std::vector<Seg> work, base;
  /* Root: partition unless n <= B (P:475 base case "n <= 2^12"; R13). */
  if (n <= base_case) base.push_back(Seg{0, n, 0});
  else work.push_back(Seg{0, n, 0});

  uint32_t level = 0;
  while (!work.empty()) {
    std::vector<Seg> next;
    for (const Seg& sg : work) {
      const uint64_t m = sg.m;
      uint64_t* a = keys + sg.begin;
      /* Phase 1: sample. */
      uint64_t S = oracle_sample_size(m, k);
      std::vector<uint64_t> idx(S);
      oracle_sample_positions(seed, level, sg.begin, m, S, idx.data());
      std::vector<uint64_t> smp(S);
      for (uint64_t j = 0; j < S; ++j) smp[j] = keys[idx[j]];
      /* Phase 2: sort the sample, by ordering key. */
      std::sort(smp.begin(), smp.end(), [&](uint64_t x, uint64_t y) {
        return ok_of(x, key_type) < ok_of(y, key_type);
      });
      /* Phase 3: train (Listing 1) or fall back to the equality split (R5, R10, R19);
       * with the tree model, pick the splitters (R22). */
      Model md{ORACLE_MODEL_LINEAR, 0.0, 0.0, k, 0, 0, 0};
      std::vector<uint64_t> spl;
      bool eq3 = sg.force_eq3 || S < 4;
      if (!eq3 && (model == ORACLE_MODEL_TREE || model == ORACLE_MODEL_TREE_EQ)) {
        /* R24: with equality buckets the k buckets are k/2 leaves x {between, equal}. */
        const uint32_t leaves = model == ORACLE_MODEL_TREE_EQ ? k / 2 : k;
        spl.resize(leaves - 1);
        oracle_tree_splitters(smp.data(), S, leaves, key_type, spl.data());
        md.kind = ORACLE_MODEL_TREE;
        md.spl = spl.data();
        md.leaves = leaves;
      } else if (!eq3) {
        std::vector<double> sv(S);
        for (uint64_t j = 0; j < S; ++j) sv[j] = value_of(smp[j], key_type);
        int deg = oracle_fit_fmcd(sv.data(), S, k, &md.A, &md.B, &md.D, &md.capped);
        if (deg) eq3 = true;
      }
      if (eq3) {
        md.kind = ORACLE_MODEL_EQ3;
        md.A = 0.0; md.B = 0.0; md.D = 0; md.capped = 0;
        md.pivot_ok = ok_of(smp[S / 2], key_type);
      }
      const uint32_t ke = eq3 ? 3 : k;
      /* Phase 4: predict every key, then move keys into contiguous buckets (stable). */
      std::vector<uint64_t> off(ke + 1);
      partition_model(a, tmp.data(), m, key_type, md, off.data(), nullptr);
      std::memcpy(a, tmp.data(), m * 8);

      if (trace) {
        oracle_record r{};
        r.level = level; r.kind = (uint32_t)md.kind; r.begin = sg.begin; r.m = m; r.S = S;
        r.A = md.A; r.B = md.B; r.D = md.D; r.capped = md.capped; r.pivot_ok = md.pivot_ok;
        r.k_eff = ke;
        std::vector<uint64_t> c(ke);
        for (uint32_t j = 0; j < ke; ++j) c[j] = off[j + 1] - off[j];
        r.requeued = 0;
        for (uint32_t j = 0; j < ke; ++j)
          if (md.kind != ORACLE_MODEL_EQ3 && c[j] == m) r.requeued = 1;
        trace->recs.push_back(r);
        trace->samples.push_back(smp);
        trace->counts.push_back(c);
      }
      /* No-progress guard (R10, R24): a linear or tree model that kept every key in one
       * bucket. */
      bool stuck = false;
      if (md.kind != ORACLE_MODEL_EQ3)
        for (uint32_t j = 0; j < ke; ++j)
          if (off[j + 1] - off[j] == m) stuck = true;
      if (stuck) {
        next.push_back(Seg{sg.begin, m, 1});
        continue;
      }
      /* Children (P:120-121 recursion; R9 homogeneity; R20 precedence). */
      for (uint32_t j = 0; j < ke; ++j) {
        uint64_t cb = off[j], cm = off[j + 1] - off[j];
        if (cm == 0) continue;
        uint64_t mn = ~0ull, mx = 0;
        for (uint64_t q = 0; q < cm; ++q) {
          uint64_t o = ok_of(a[cb + q], key_type);
          mn = std::min(mn, o);
          mx = std::max(mx, o);
        }
        bool homog = (md.kind == ORACLE_MODEL_EQ3 && j == 1) || mn == mx;
        if (homog) continue;                       /* final: never touched again */
        if (cm <= base_case) base.push_back(Seg{sg.begin + cb, cm, 0});
        else next.push_back(Seg{sg.begin + cb, cm, 0});
      }
    }
    if (trace && trace->keep_snapshots) trace->snaps.emplace_back(keys, keys + n);
    ++level;
    work.swap(next);
  }
  if (trace) trace->levels = level;
  /* Base case: any exact sort of each small bucket, by ordering key. */
  for (const Seg& sg : base) {
    std::sort(keys + sg.begin, keys + sg.begin + sg.m, [&](uint64_t x, uint64_t y) {
      return ok_of(x, key_type) < ok_of(y, key_type);
    });
  }
  return 0;
}

}  // extern "C"
