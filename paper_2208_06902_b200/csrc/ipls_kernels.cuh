// ipls_kernels.cuh — sm_100a kernels of one IPLS distribution level and the base case.
//
// Per level (the four phases of P:265-287):
//   k_fit_small /     phases 1-3: stratified sample of every segment (R2, R18),
//   k_gather_fit      exact sort of the sample, FMCD fit (Listing 1)
//   k_classify_scan   phase 4a: model evaluation + smem histogram per chunk, NaN
//                     flag (level 0), decoupled-lookback prefix of the (chunk x bucket) counts;
//                     the last chunk of a segment writes the bucket bases (segment_bases)
//   k_scatter         phase 4b: stable in-tile rank (per-warp atomic counters), or unstable
//                     placement inside terminal segments; smem staging by bucket, run-contiguous
//                     writes (R11); homogeneity (R9); the last
//                     chunk of a segment classes the children (R20) and emits the next level's
//                     work, the base-case windows and the fills (segment_emit)
// After the level: k_base_warp / k_base_sort (base case) and k_fill.
#pragma once
#include <type_traits>

#include "ipls_device.cuh"

namespace ipls {

#ifdef IPLS_SCATTER_TIMING  // dev builds only (tools/phase_scatter.py)
__device__ unsigned long long g_sc_phase[32];
#define FIT_TICK(N) do { if (threadIdx.x == 0) { const long long t_ = clock64(); atomicAdd(&g_sc_phase[N], (unsigned long long)(t_ - ft_prev_)); ft_prev_ = t_; } } while (0)
#else
#define FIT_TICK(N)
#endif

constexpr int kCThreads = 512;                 // classify
constexpr int kCItems = 8;
constexpr int kCTile = kCThreads * kCItems;    // 4096
constexpr int kFitThreads = 1024;
constexpr int kFitMaxS = 8192;
constexpr uint32_t kMaxK = 1024;
// big-window base case (k_base_sort)
constexpr int kBCThreads = 512;
constexpr int kBCItems = 8;
constexpr int kBigCap = kBCThreads * kBCItems;  // 4096 = the largest base child
// keys + fine-bin words (4 pad words per 32: each thread's 8 bins are 2 conflict-free uint4)
constexpr size_t kBCSmem = (size_t)kBigCap * 8 + (size_t)(kBigCap + kBigCap / 8) * 4;

// small-window base case (k_base_warp)
constexpr int kWBCap = 256;                      // keys per warp window
#ifndef IPLS_WB_BPK
#define IPLS_WB_BPK 2
#endif
#ifndef IPLS_WB_WARPS
#define IPLS_WB_WARPS 32
#endif
constexpr int kWBBinsPerKey = IPLS_WB_BPK;
constexpr int kWBBins = kWBBinsPerKey * kWBCap;  // fine bins per warp
constexpr int kWBWarps = IPLS_WB_WARPS;          // warps per CTA, one CTA per SM
constexpr int kWBStride = kWBCap + 4;            // keys per prefetch buffer (+ alignment slack)
constexpr int kWBItems = kWBCap / 32;            // keys per lane (held in registers)
constexpr int kWBBpl = kWBBins / 32;             // bins per lane in the scan (16)
constexpr int kWBBinWords = kWBBins + kWBBins / 8;  // bins with 4 pad words per 32
constexpr size_t kWBSmemPerWarp = (size_t)2 * kWBStride * 8 + (size_t)kWBBinWords * 4;
__device__ __forceinline__ uint32_t wb_phys(uint32_t f) { return f + ((f >> 5) << 2); }
constexpr uint32_t kFineOverflow = 32;          // fine-bin load that triggers the bitonic fallback

// Terminal segment sort (k_tss_scatter + k_win_sort, ipls_tss.cuh): a terminal segment is cut
// into windows of whole children of <= kTW keys; a window of W' = kTW - (largest child)
// positions starts at the first child starting in [g W', (g+1) W'), so every window holds
// <= kTW keys and child c lies in window floor(start(c) / W').
#ifndef IPLS_TW
#define IPLS_TW 16384
#endif
constexpr uint32_t kTW = IPLS_TW;
static_assert(kTW >= 8192 && kTW <= 32768, "W' and the window sort's u16 bin starts fit 16 bits");
constexpr uint32_t kTWMaxWin = (uint32_t)(((uint64_t)1024 * 4096 + (kTW - 4096) - 1) / (kTW - 4096)) + 2;

// ------------------------------------------------------------------------------------
// Block-wide exact sort of n <= cap ordering keys in smem (used for samples and base-case
// windows).  A 256-way coarse histogram of (ok - min) >> shift allots each coarse bin as
// many fine bins as it holds keys; a fine counting sort leaves runs of ~1 key that an
// insertion sort finishes.  Inputs whose fine bins overflow take a bitonic sort instead.
// Any exact sort yields the identical bytes, so the method is free (R13).
struct SortSmem {
  uint32_t ccnt[256];
  uint32_t coff[256];
  uint32_t ccnt2[256];  // k_fit_small: coarse counts in the other key space
  uint32_t cmax[2];
  uint64_t red[64];
  uint32_t warp[40];
};

template <int NT>
__device__ void bitonic_sort_smem(uint64_t* a, uint32_t n) {
  uint32_t NP = 1;
  while (NP < n) NP <<= 1;
  for (uint32_t i = n + threadIdx.x; i < NP; i += NT) a[i] = ~0ull;
  __syncthreads();
  for (uint32_t size = 2; size <= NP; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = threadIdx.x; i < NP / 2; i += NT) {
        uint32_t lo = 2 * i - (i & (stride - 1));
        uint32_t hi = lo + stride;
        bool asc = (lo & size) == 0;
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == asc) { a[lo] = y; a[hi] = x; }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ uint32_t fine_bin(uint64_t v, uint64_t mn, int sh, const uint32_t* coff,
                                             const uint32_t* ccnt) {
  uint64_t d = v - mn;
  uint32_t c = (uint32_t)(d >> sh);
  uint32_t f = coff[c];
  if (sh > 0) f += (uint32_t)__umul64hi((d - ((uint64_t)c << sh)) << (64 - sh), ccnt[c]);
  return f;
}

// Sorts a[0..n) (a must hold the next power of two >= n for the fallback).  tmp: n u64,
// fh: n u32 scratch.  Ends with a barrier.
template <int NT>
__device__ void block_sort_ok(uint64_t* a, uint64_t* tmp, uint32_t* fh, uint32_t n, SortSmem& ss) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint64_t mn = ~0ull, mx = 0ull;
  for (uint32_t i = threadIdx.x; i < n; i += NT) {
    uint64_t v = a[i];
    mn = min(mn, v);
    mx = max(mx, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) { ss.red[wp] = mn; ss.red[32 + wp] = mx; }
  for (uint32_t c = threadIdx.x; c < 256; c += NT) ss.ccnt[c] = 0;
  for (uint32_t i = threadIdx.x; i < n; i += NT) fh[i] = 0;
  __syncthreads();
  mn = ss.red[0]; mx = ss.red[32];
  for (int w = 1; w < NW; ++w) { mn = min(mn, ss.red[w]); mx = max(mx, ss.red[32 + w]); }
  if (mn == mx || n < 2) { __syncthreads(); return; }
  const uint64_t range = mx - mn;
  const int bl = 64 - __clzll((long long)range);
  const int sh = bl > 8 ? bl - 8 : 0;
  for (uint32_t i = threadIdx.x; i < n; i += NT) atomicAdd(&ss.ccnt[(uint32_t)((a[i] - mn) >> sh)], 1u);
  __syncthreads();
  {
    uint32_t c = (threadIdx.x < 256) ? ss.ccnt[threadIdx.x] : 0u;
    uint32_t ex = block_exclusive_scan<NT>(c, ss.warp, nullptr);
    if (threadIdx.x < 256) ss.coff[threadIdx.x] = ex;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += NT)
    atomicAdd(&fh[fine_bin(a[i], mn, sh, ss.coff, ss.ccnt)], 1u);
  __syncthreads();
  // exclusive scan of fh[0..n): thread t owns the contiguous run [t*E, t*E+E)
  const uint32_t E = (n + NT - 1) / NT;
  uint32_t mxc = 0, sum = 0;
  const uint32_t b0 = threadIdx.x * E;
  for (uint32_t j = 0; j < E; ++j) {
    uint32_t i = b0 + j;
    uint32_t c = (i < n) ? fh[i] : 0u;
    sum += c;
    mxc = max(mxc, c);
  }
  uint32_t run = block_exclusive_scan<NT>(sum, ss.warp, nullptr);
  for (uint32_t j = 0; j < E; ++j) {
    uint32_t i = b0 + j;
    if (i < n) {
      uint32_t c = fh[i];
      fh[i] = run;
      run += c;
    }
  }
  // sh == 0: every coarse bin is one value, so the counting pass is already an exact sort
  // (duplicate-heavy samples, e.g. root-dups).  Otherwise bins are finished by insertion
  // sort, unless one holds more than kFineOverflow keys (then a bitonic sort).
  if (__syncthreads_or(sh > 0 && mxc > kFineOverflow)) {  // also orders the scan writes
    bitonic_sort_smem<NT>(a, n);
    return;
  }
  for (uint32_t i = threadIdx.x; i < n; i += NT) {
    uint64_t v = a[i];
    uint32_t pos = atomicAdd(&fh[fine_bin(v, mn, sh, ss.coff, ss.ccnt)], 1u);
    tmp[pos] = v;
  }
  __syncthreads();
  if (sh > 0) {
    for (uint32_t f = threadIdx.x; f < n; f += NT) {
      uint32_t beg = f ? fh[f - 1] : 0u, end = fh[f];
      for (uint32_t i = beg + 1; i < end; ++i) {
        uint64_t x = tmp[i];
        uint32_t j = i;
        while (j > beg && tmp[j - 1] > x) { tmp[j] = tmp[j - 1]; --j; }
        tmp[j] = x;
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += NT) a[i] = tmp[i];
  __syncthreads();
}

// ------------------------------------------------------------------------------------
// Root work item (level 0): one segment covering [0, n), chunked.
__global__ void k_init_root(SegDesc* segs, ChunkDesc* chunks, uint64_t n, uint32_t S,
                            uint32_t chunk_keys, uint32_t flags) {
  uint32_t nch = (uint32_t)((n + chunk_keys - 1) / chunk_keys);
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    SegDesc sg{};
    sg.begin = 0; sg.m = (uint32_t)n; sg.S = S; sg.sample_off = 0;
    sg.chunk_first = 0; sg.nchunks = nch; sg.flags = flags;
    segs[0] = sg;
  }
  for (uint32_t c = i; c < nch; c += gridDim.x * blockDim.x) {
    ChunkDesc cd;
    cd.start = (uint64_t)c * chunk_keys;
    cd.len = (uint32_t)min((uint64_t)chunk_keys, n - cd.start);
    cd.seg = 0;
    chunks[c] = cd;
  }
}

// ------------------------------------------------------------------------------------
// Phases 1-3 for one segment per CTA.
// Sample: one position per stratum [floor(j m/S), floor((j+1) m/S)) (R2), SplitMix64 keyed by
// (seed, level, begin, j) (R18).  Sort by ordering key.  FMCD: Listing 1 returns the least
// D >= 1 whose every window satisfies s[i+D]-s[i] >= u(D), u(D) = (s[N-1-D]-s[D])/(k-2); if
// no D <= floor(N/3) qualifies it stops with D = floor(N/3)+1 and the stale u(floor(N/3))
// (R4).  The predicate is monotone in D in binary64 (RN is monotone), so the CTA finds that
// D by galloping + bisection, testing each candidate with all threads (K1).
// Every arithmetic step is one RN operation in Listing 1's order.
__device__ __forceinline__ double fmcd_u(const double* s, uint32_t N, uint32_t D, double km2) {
  return __ddiv_rn(__dsub_rn(s[N - 1 - D], s[D]), km2);
}

template <int NT>
__device__ bool fmcd_pred(const double* s, uint32_t N, uint32_t D, double u) {
  int fail = 0;
  for (uint32_t i = threadIdx.x; i + D < N; i += NT) {
    if (!(__dsub_rn(s[i + D], s[i]) >= u)) { fail = 1; break; }
  }
  return __syncthreads_or(fail) == 0;
}

// Splitter tree (R22): node j (1..k-1, heap order) of the perfect tree of
// depth log2 k holds the splitter of in-order rank i = (2 p + 1) 2^(L-1-d) (d = depth of j,
// p = j - 2^d), and splitter i is the order statistic s[floor(i S / k)] of the sorted sample
// `so` (ordering keys).  One thread per node.
template <int NT>
__device__ __forceinline__ void write_tree(const uint64_t* so, uint32_t S, uint32_t k,
                                           uint64_t* heap) {
  const int L = 31 - __clz(k);
  for (uint32_t j = threadIdx.x + 1; j < k; j += NT) {
    const int d = 31 - __clz(j);
    const uint32_t i = (2 * (j - (1u << d)) + 1) << (L - 1 - d);
    heap[j] = so[(uint32_t)(((uint64_t)i * S) >> L)];
  }
}

template <bool F64>
__global__ __launch_bounds__(kFitThreads) void k_gather_fit(
    const uint64_t* __restrict__ src, const SegDesc* __restrict__ segs, uint64_t seed,
    uint64_t hbase, uint32_t level, uint32_t k, uint32_t cap, uint64_t* __restrict__ samples_out,
    ModelDev* __restrict__ models, const uint64_t* __restrict__ presorted_ok,
    const uint32_t* __restrict__ redo, uint64_t* __restrict__ tree, int sort_given = 0,
    const uint32_t* __restrict__ redo_cnt = nullptr, uint32_t tree_leaves = 0) {
  // With redo_cnt: the CTAs walk the list redo[0, *redo_cnt) of segments k_fit_small left over
  // (usually none: a launch of a few idle CTAs).  Without: CTA s fits segment s.
  const uint32_t nitems = redo_cnt ? *((volatile const uint32_t*)redo_cnt) : 1u;
  for (uint32_t item = redo_cnt ? blockIdx.x : 0u; item < nitems; item += gridDim.x) {
  const uint32_t sgi = redo_cnt ? redo[item] : blockIdx.x;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* a = reinterpret_cast<uint64_t*>(smraw);   // cap
  uint64_t* tmp = a + cap;                             // cap
  uint32_t* fh = reinterpret_cast<uint32_t*>(tmp + cap);  // cap
  __shared__ SortSmem ss;
  __shared__ uint64_t s_pivot;
  __syncthreads();  // smem of the previous item
  const SegDesc sg = segs[sgi];
  const uint32_t S = sg.S;
#ifdef IPLS_SCATTER_TIMING
  long long ft_prev_ = clock64();
#endif
  if (presorted_ok) {
    for (uint32_t j = threadIdx.x; j < S; j += kFitThreads) a[j] = presorted_ok[j];
    __syncthreads();
    if (sort_given) block_sort_ok<kFitThreads>(a, tmp, fh, S, ss);  // ipls_fit_sample
  } else {
    // hbase: position of this array in the one whose recursion is resumed (ipls_sort_segments)
    const uint64_t t = sm64(sm64(sm64(seed) ^ (uint64_t)level) ^ (sg.begin + hbase));
    StrataWalk sw(threadIdx.x, kFitThreads, sg.m, S);
    // batches of 8 loads in flight per thread (S <= cap <= 8 kFitThreads)
    for (uint32_t j0 = threadIdx.x; j0 < S; j0 += 8 * kFitThreads) {
      uint64_t x[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint32_t j = j0 + r * kFitThreads;
        const uint64_t lo = sw.lo(), hi = sw.hi();
        const uint64_t idx = sg.begin + lo + __umul64hi(sm64(t ^ (uint64_t)j), hi - lo);
        x[r] = __ldg(src + (j < S ? idx : sg.begin));
        sw.next();
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint32_t j = j0 + r * kFitThreads;
        if (j < S) a[j] = ok_of<F64>(x[r]);
      }
    }
    __syncthreads();
    FIT_TICK(8);
    block_sort_ok<kFitThreads>(a, tmp, fh, S, ss);
    FIT_TICK(9);
  }
  if (samples_out)
    for (uint32_t j = threadIdx.x; j < S; j += kFitThreads) samples_out[sg.sample_off + j] = a[j];
  if (threadIdx.x == 0) s_pivot = a[S / 2];
  __syncthreads();
  ModelDev md{};
  md.k_eff = k;
  bool eq3 = (sg.flags & kSegForceEq3) || S < 4;
  if (!eq3 && tree) {  // splitter-tree model instead of FMCD
    uint64_t* hp = tree + (size_t)sgi * kMaxK;
    const uint32_t leaves = tree_leaves ? tree_leaves : k;  // k / 2 with equality buckets (R24)
    write_tree<kFitThreads>(a, S, leaves, hp);
    md.kind = kModelTree; md.heap = hp; md.leaves = leaves;
  } else if (!eq3) {
    double* s = reinterpret_cast<double*>(tmp);
    for (uint32_t i = threadIdx.x; i < S; i += kFitThreads) s[i] = value_of<F64>(bits_of_ok<F64>(a[i]));
    __syncthreads();
    const uint32_t N = S;
    const uint32_t Dcap = N / 3;  // >= 1 since N >= 4
    const double km2 = (double)(k - 2);
    uint32_t lo = 0, hi = 0;      // pred(lo) false (0 = sentinel), pred(hi) true
    uint32_t D = 1;
    bool found = false;
    while (true) {
      if (D > Dcap) D = Dcap;
      if (fmcd_pred<kFitThreads>(s, N, D, fmcd_u(s, N, D, km2))) { hi = D; found = true; break; }
      lo = D;
      if (D == Dcap) break;
      D <<= 1;
    }
    uint32_t Dres;
    double ures;
    if (!found) {
      Dres = Dcap + 1;
      ures = fmcd_u(s, N, Dcap, km2);
      md.capped = 1;
    } else {
      while (hi - lo > 1) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (fmcd_pred<kFitThreads>(s, N, mid, fmcd_u(s, N, mid, km2))) hi = mid; else lo = mid;
      }
      Dres = hi;
      ures = fmcd_u(s, N, hi, km2);
      md.capped = 0;
    }
    double A = __ddiv_rn(1.0, ures);
    double sum = __dadd_rn(s[N - 1 - Dres], s[Dres]);
    double prod = __dmul_rn(A, sum);
    double B = __ddiv_rn(__dsub_rn((double)k, prod), 2.0);
    bool degenerate = !(ures > 0.0) || !isfinite(A) || !isfinite(B) || !(A > 0.0);
    if (!degenerate) {
      md.kind = kModelLinear; md.A = A; md.B = B; md.D = Dres; md.pivot_ok = 0;
    } else {
      eq3 = true;
    }
  }
  if (eq3) {
    md.kind = kModelEq3; md.A = 0.0; md.B = 0.0; md.D = 0; md.capped = 0;
    md.pivot_ok = s_pivot; md.k_eff = 3;
  }
  FIT_TICK(10);
  if (threadIdx.x == 0) models[sgi] = md;
  }
}


// Phases 1-3 for segments with S <= kFSMax samples: 256 threads, samples held in registers,
// 3 CTAs per SM (the 1024-thread k_gather_fit below takes S > kFSMax, i.e. level 0 at 1e8
// keys, and any segment whose sample overflows a fine bin; they are listed in redo[]).
// Same result as k_gather_fit: same sample, exact sort, Listing 1 by galloping + bisection.
constexpr int kFSThreads = 256;
constexpr int kFSItems = 20;                     // samples per thread
constexpr int kFSMax = kFSThreads * kFSItems;    // 5120 (S(m) for m <= 2^25 at k = 1024)
constexpr size_t kFSSmem = (size_t)kFSMax * 12;
// 16 samples per thread for samples of <= 4096 keys (S(m) for m <= 2^20 at k = 1024): fewer
// registers than the 20-sample variant (no spills), same 3 CTAs per SM
constexpr int kFMItems = 16;
constexpr int kFMMax = kFSThreads * kFMItems;
constexpr size_t kFMSmem = (size_t)kFMMax * 12;
// Large-sample variant (one CTA of 1024 threads, 8 samples each: every S(m) <= 7k - 1 < 8192),
// used for the levels whose largest sample exceeds kFSMax (level 0 at >= 2^25 keys).
constexpr int kFLThreads = 1024;
constexpr int kFLItems = 8;
constexpr int kFLMax = kFLThreads * kFLItems;    // 8192
constexpr size_t kFLSmem = (size_t)kFLMax * 12;

template <bool F64, int NT, int IT>
__global__ __launch_bounds__(NT, NT == 256 ? 3 : 1) void k_fit_small(
    const uint64_t* __restrict__ src, const SegDesc* __restrict__ segs, uint64_t seed,
    uint64_t hbase, uint32_t level, uint32_t k, uint64_t* __restrict__ samples_out,
    ModelDev* __restrict__ models,
    uint32_t* __restrict__ redo, uint64_t* __restrict__ tree, uint32_t* __restrict__ redo_cnt,
    uint32_t tree_leaves) {
  constexpr int NW = NT / 32, SMAX = NT * IT;
  static_assert(NT >= 256 && IT % 4 == 0, "256 coarse bins, uint4 fine-bin scan");
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* B = reinterpret_cast<uint64_t*>(smraw);      // SMAX
  uint32_t* fh = reinterpret_cast<uint32_t*>(B + SMAX);  // SMAX
  __shared__ SortSmem ss;
  __shared__ uint64_t s_pivot;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const SegDesc sg = segs[blockIdx.x];
  const uint32_t S = sg.S;
  if (S > (uint32_t)SMAX) {
    if (threadIdx.x == 0) redo[atomicAdd(redo_cnt, 1u)] = blockIdx.x;
    return;
  }
  // ---- stratified sample (R2, R18), as ordering keys in registers ----
#ifdef IPLS_SCATTER_TIMING
  long long ft_prev_ = clock64();
#define FITL_TICK(N) do { if (NT == 1024) { if ((N) < 22) FIT_TICK(N); } else FIT_TICK((N) < 22 ? (N) + 3 : (N)); } while (0)
#else
#define FITL_TICK(N)
#endif
  // hbase: position of this array in the one whose recursion is resumed (ipls_sort_segments)
    const uint64_t t = sm64(sm64(sm64(seed) ^ (uint64_t)level) ^ (sg.begin + hbase));
  StrataWalk sw(threadIdx.x, NT, sg.m, S);
  uint64_t v[IT];
  uint64_t mn = ~0ull, mx = 0ull;
  // all IT loads are issued before any is used (one DRAM latency per thread, not IT)
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const uint32_t j = r * NT + threadIdx.x;
    const uint64_t lo = sw.lo(), hi = sw.hi();
    const uint64_t idx = sg.begin + lo + __umul64hi(sm64(t ^ (uint64_t)j), hi - lo);
    v[r] = __ldg(src + (j < S ? idx : sg.begin));
    sw.next();
  }
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    if (r * NT + threadIdx.x < S) {
      v[r] = ok_of<F64>(v[r]);
      mn = min(mn, v[r]);
      mx = max(mx, v[r]);
    } else {
      v[r] = 0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  FITL_TICK(16);
  if (lane == 0) { ss.red[wp] = mn; ss.red[32 + wp] = mx; }
  for (uint32_t c = threadIdx.x; c < 256; c += NT) ss.ccnt[c] = 0u;
  {
    uint4* f4 = reinterpret_cast<uint4*>(fh) + threadIdx.x * (IT / 4);
#pragma unroll
    for (int q = 0; q < IT / 4; ++q) f4[q] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
    FITL_TICK(22);
  mn = ss.red[0]; mx = ss.red[32];
#pragma unroll
  for (int w = 1; w < NW; ++w) { mn = min(mn, ss.red[w]); mx = max(mx, ss.red[32 + w]); }
  // ---- exact sort: coarse + fine interpolation bins, counting placement, in-bin insertion ----
  if (mn == mx) {
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      const uint32_t j = r * NT + threadIdx.x;
      if (j < S) B[j] = v[r];
    }
  } else {
    const int bl = 64 - __clzll((long long)(mx - mn));
    const int sh = bl > 8 ? bl - 8 : 0;
    // f64: bins in key-value space (linear in the key) whenever the range allows it.
    // Ordering-key space is linear only inside a binade, so a sample spanning many binades
    // (a Normal around 0 at level 0) piles into a few coarse bins and long insertion runs.
    // Heavy-tailed samples (a LogNormal) are the opposite case, so both coarse histograms
    // are built and the space with the smaller largest coarse bin is used.
    bool lin = false;
    double vmn = 0.0, vsc = 0.0;
    if constexpr (F64) {
      vmn = __longlong_as_double((long long)bits_of_ok<true>(mn));
      const double rg = __longlong_as_double((long long)bits_of_ok<true>(mx)) - vmn;
      vsc = 256.0 / rg;
      lin = rg > 0.0 && isfinite(rg) && isfinite(vsc);
    }
    auto vpos = [&](uint64_t o) -> double {  // (x - min) * 256 / range, monotone in x
      return __dmul_rn(__dsub_rn(__longlong_as_double((long long)bits_of_ok<true>(o)), vmn), vsc);
    };
    if (F64 && lin) {
      for (uint32_t c = threadIdx.x; c < 256; c += NT) ss.ccnt2[c] = 0u;
      if (threadIdx.x < 2) ss.cmax[threadIdx.x] = 0u;
      __syncthreads();
#pragma unroll
      for (int r = 0; r < IT; ++r)
        if (r * NT + threadIdx.x < S) {
          atomicAdd(&ss.ccnt[(uint32_t)((v[r] - mn) >> sh)], 1u);
          atomicAdd(&ss.ccnt2[min(__double2uint_rz(vpos(v[r])), 255u)], 1u);
        }
      __syncthreads();
      if (threadIdx.x < 256) {
        atomicMax(&ss.cmax[0], ss.ccnt[threadIdx.x]);
        atomicMax(&ss.cmax[1], ss.ccnt2[threadIdx.x]);
      }
      __syncthreads();
      lin = ss.cmax[1] < ss.cmax[0];
      if (lin && threadIdx.x < 256) ss.ccnt[threadIdx.x] = ss.ccnt2[threadIdx.x];
    } else {
#pragma unroll
      for (int r = 0; r < IT; ++r)
        if (r * NT + threadIdx.x < S) atomicAdd(&ss.ccnt[(uint32_t)((v[r] - mn) >> sh)], 1u);
    }
    const bool exact = !lin && sh == 0;  // every coarse bin is one value: counting is exact
    auto fine_of = [&](uint64_t o) -> uint32_t {
      if (F64 && lin) {
        const double y = vpos(o);
        const uint32_t c = min(__double2uint_rz(y), 255u), n = ss.ccnt[c];
        return ss.coff[c] + min(__double2uint_rz(__dmul_rn(__dsub_rn(y, (double)c), (double)n)), n - 1);
      }
      return fine_bin(o, mn, sh, ss.coff, ss.ccnt);
    };
    __syncthreads();
    FITL_TICK(23);
    {
      const uint32_t cc = threadIdx.x < 256 ? ss.ccnt[threadIdx.x] : 0u;  // 256 coarse bins
      const uint32_t ex = block_exclusive_scan<NT>(cc, ss.warp, nullptr);
      if (threadIdx.x < 256) ss.coff[threadIdx.x] = ex;
    }
    __syncthreads();
    FITL_TICK(24);
    uint32_t f[IT];
#pragma unroll
    for (int r = 0; r < IT; ++r) {
      f[r] = 0;
      if (r * NT + threadIdx.x < S) {
        f[r] = fine_of(v[r]);
        atomicAdd(&fh[f[r]], 1u);
      }
    }
    __syncthreads();
    FITL_TICK(25);
    uint32_t mxc = 0;
    {
      uint4* f4 = reinterpret_cast<uint4*>(fh) + threadIdx.x * (IT / 4);
      uint32_t sum = 0;
#pragma unroll
      for (int q = 0; q < IT / 4; ++q) {
        const uint4 c = f4[q];
        sum += c.x + c.y + c.z + c.w;
        mxc = max(mxc, max(max(c.x, c.y), max(c.z, c.w)));
      }
      uint32_t run = block_exclusive_scan<NT>(sum, ss.warp, nullptr);
#pragma unroll
      for (int q = 0; q < IT / 4; ++q) {
        const uint4 c = f4[q];
        uint4 o;
        o.x = run; run += c.x;
        o.y = run; run += c.y;
        o.z = run; run += c.z;
        o.w = run; run += c.w;
        f4[q] = o;
      }
    }
    const bool ovf = __syncthreads_or(!exact && mxc > kFineOverflow) != 0;
    if (ovf) {
      // A fine bin above kFineOverflow keys that holds one value (duplicate-heavy samples)
      // needs no sorting: every key of a big bin is compared with one of them, stored at the
      // bin's first slot.  Bins of different keys go to the 1024-thread kernel (bitonic).
      auto big_start = [&](uint32_t fb) -> uint32_t {
        const uint32_t st = fh[fb], en = fb + 1 < (uint32_t)SMAX ? fh[fb + 1] : S;
        return en - st > kFineOverflow ? st : ~0u;
      };
#pragma unroll
      for (int r = 0; r < IT; ++r)
        if (r * NT + threadIdx.x < S) {
          const uint32_t st = big_start(f[r]);
          if (st != ~0u) B[st] = v[r];
        }
      __syncthreads();
      bool mixed = false;
#pragma unroll
      for (int r = 0; r < IT; ++r)
        if (r * NT + threadIdx.x < S) {
          const uint32_t st = big_start(f[r]);
          if (st != ~0u && B[st] != v[r]) mixed = true;
        }
      if (__syncthreads_or(mixed)) {
        if (threadIdx.x == 0) redo[atomicAdd(redo_cnt, 1u)] = blockIdx.x;  // the 1024-thread kernel sorts it
        return;
      }
    }
#pragma unroll
    for (int r = 0; r < IT; ++r)
      if (r * NT + threadIdx.x < S) B[atomicAdd(&fh[f[r]], 1u)] = v[r];
    __syncthreads();
    FITL_TICK(26);
    if (!exact) {
      // every thread insertion-sorts the range of its fine bins [IT t, IT t + IT) (keys of
      // different bins are already ordered); with big bins (duplicates only) the range is
      // sorted one bin at a time and the big bins are skipped
      const uint32_t f0 = threadIdx.x * IT;
      const uint32_t beg = f0 ? fh[f0 - 1] : 0u, end = fh[f0 + IT - 1];
      auto insertion = [&](uint32_t b0, uint32_t b1) {
        for (uint32_t i = b0 + 1; i < b1; ++i) {
          const uint64_t x = B[i];
          uint64_t y = B[i - 1];
          if (y <= x) continue;
          uint32_t j = i;
          do { B[j] = y; --j; } while (j > b0 && (y = B[j - 1]) > x);
          B[j] = x;
        }
      };
      if (!ovf) {
        insertion(beg, end);
      } else {
        uint32_t b0 = beg;
        for (int qb = 0; qb < IT; ++qb) {
          const uint32_t b1 = fh[f0 + qb];
          if (b1 - b0 <= kFineOverflow) insertion(b0, b1);
          b0 = b1;
        }
      }
    }
  }
  __syncthreads();
  FITL_TICK(17);
  if (samples_out)
    for (uint32_t j = threadIdx.x; j < S; j += NT) samples_out[sg.sample_off + j] = B[j];
  if (threadIdx.x == 0) s_pivot = B[S / 2];
  __syncthreads();
  // ---- FMCD (Listing 1) on the sorted model values ----
  ModelDev md{};
  md.k_eff = k;
  bool eq3 = (sg.flags & kSegForceEq3) || S < 4;
  if (!eq3 && tree) {  // splitter-tree model instead of FMCD
    uint64_t* hp = tree + (size_t)blockIdx.x * kMaxK;
    const uint32_t leaves = tree_leaves ? tree_leaves : k;  // k / 2 with equality buckets (R24)
    write_tree<NT>(B, S, leaves, hp);
    md.kind = kModelTree; md.heap = hp; md.leaves = leaves;
  } else if (!eq3) {
    double* s = reinterpret_cast<double*>(B);
    for (uint32_t i = threadIdx.x; i < S; i += NT) s[i] = value_of<F64>(bits_of_ok<F64>(B[i]));
    __syncthreads();
    const uint32_t N = S;
    const uint32_t Dcap = N / 3;
    const double km2 = (double)(k - 2);
    uint32_t lo = 0, hi = 0;
    uint32_t D = 1;
    bool found = false;
    while (true) {
      if (D > Dcap) D = Dcap;
      if (fmcd_pred<NT>(s, N, D, fmcd_u(s, N, D, km2))) { hi = D; found = true; break; }
      lo = D;
      if (D == Dcap) break;
      D <<= 1;
    }
    uint32_t Dres;
    double ures;
    if (!found) {
      Dres = Dcap + 1;
      ures = fmcd_u(s, N, Dcap, km2);
      md.capped = 1;
    } else {
      while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (fmcd_pred<NT>(s, N, mid, fmcd_u(s, N, mid, km2))) hi = mid; else lo = mid;
      }
      Dres = hi;
      ures = fmcd_u(s, N, hi, km2);
      md.capped = 0;
    }
    const double A = __ddiv_rn(1.0, ures);
    const double sum = __dadd_rn(s[N - 1 - Dres], s[Dres]);
    const double prod = __dmul_rn(A, sum);
    const double Bm = __ddiv_rn(__dsub_rn((double)k, prod), 2.0);
    const bool degenerate = !(ures > 0.0) || !isfinite(A) || !isfinite(Bm) || !(A > 0.0);
    if (!degenerate) {
      md.kind = kModelLinear; md.A = A; md.B = Bm; md.D = Dres; md.pivot_ok = 0;
    } else {
      eq3 = true;
    }
  }
  if (eq3) {
    md.kind = kModelEq3; md.A = 0.0; md.B = 0.0; md.D = 0; md.capped = 0;
    md.pivot_ok = s_pivot; md.k_eff = 3;
  }
  FITL_TICK(18);
  if (threadIdx.x == 0) models[blockIdx.x] = md;
}

// ------------------------------------------------------------------------------------
// Phase 4a.  One CTA per chunk, chunks taken in ticket order so that every predecessor of a
// chunk has started (no deadlock in the lookback).
struct LevelArgs {
  const uint64_t* src;
  const SegDesc* segs;
  const ChunkDesc* chunks;
  const ModelDev* models;
  uint32_t k, base_case, level, chunk_keys;
  uint64_t nkeys;        // length of the arrays (src and both destinations)
  uint32_t dstbuf;       // buffer the level scatters into: 1 = scratch, 0 = user array
  uint32_t fused_term;   // terminal segments go through k_term_fused (else k_scatter_term)
  uint32_t* ticket;
  uint64_t* status;      // [chunk][k]: epoch<<48 | state<<46 | count
  uint32_t* chunk_pre;   // [chunk][k] exclusive prefix within the segment
  uint64_t* seg_dst;     // [seg][k]   encoded destination base of every child
  uint32_t* seg_tot;     // [seg][k]   child counts
  uint8_t* cflag;        // [chunk][k] scatter homogeneity flag: 0 empty, 1 one value, 2 several
  uint64_t* cref;        // [chunk][k] the chunk's value of a one-value bucket
  uint32_t* seg_term;    // [seg]      1: every child <= base case (terminal segment)
  uint32_t* seg_done;    // [seg]      chunks of the segment scattered (k_term_fused)
  uint32_t tss;          // terminal segments: window scatter + window sort (k_tss_scatter, k_win_sort)
  uint2* seg_tw;         // [seg]      {first terminal window, W'} (W' = 0: the segment is one window)
  Window* twins;         // terminal windows of the level (k_win_sort)
  uint32_t* twcur;       // [window]   k_tss_scatter's fill cursor
  uint32_t cap_twin;
  uint32_t epoch;
  uint32_t* err;
  int check_nan;
  uint16_t* ids;         // partition_level only: per-key buckets
  uint64_t* single_offsets;  // partition_level only: k_eff+1 bucket boundaries
  const uint64_t* bucket_dst;  // partition_scatter_to only (PEER kernels): bucket b's keys of this
                               // array go to the words from address bucket_dst[b] on (any
                               // device-accessible memory, e.g. a peer GPU's over NVLink)
  SegDesc* nsegs;
  ChunkDesc* nchunks;
  LevelCounters* nctr;
  uint32_t cap_segs, cap_chunks, cap_samples;
  Window* wins;        // small windows (<= kWBCap keys): k_base_warp
  uint32_t cap_wins;
  Window* wins_big;    // single base children above kWBCap: k_base_sort
  uint32_t cap_wbig;
  Fill* fills;
  uint32_t cap_fills;
};

constexpr uint32_t kStAgg = 1, kStInc = 2;
constexpr int kCBpt = kMaxK / kCThreads;  // buckets per thread in the scans (2)

__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint32_t st, uint32_t inh,
                                                uint32_t cnt) {
  return ((uint64_t)(epoch & 0xffff) << 48) | ((uint64_t)st << 46) | ((uint64_t)inh << 45) |
         (uint64_t)cnt;
}


// Adds every thread's v into *dst with one atomic per warp (the level's key counters only feed
// the per-kernel byte counts; one atomic per item would serialise every CTA of the level on
// one L2 address).
__device__ __forceinline__ void warp_add_u64(unsigned long long* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// Chunks of a segment at levels >= 1: round(m / chunk_keys) chunks of equal length (at least
// one), i.e. 2/3 to 3/2 of chunk_keys each -- no small remainder chunk that would pay a CTA's
// whole per-chunk setup for a few keys (a 97k-key segment used to become 96k + 1k).
__host__ __device__ __forceinline__ uint32_t chunks_of(uint32_t m, uint32_t ck) {
  const uint32_t n = (uint32_t)(((uint64_t)m + ck / 2) / ck);
  return n ? n : 1u;
}

__device__ void emit_segment(const LevelArgs& a, uint64_t begin, uint32_t m, uint32_t flags,
                             uint32_t seg_idx, uint32_t samp_off, uint32_t ch_off) {
  SegDesc sd{};
  sd.begin = begin; sd.m = m; sd.S = sample_size(m, a.k); sd.sample_off = samp_off;
  const uint32_t nch = chunks_of(m, a.chunk_keys);
  const uint32_t per = (m + nch - 1) / nch;
  sd.chunk_first = ch_off; sd.nchunks = nch; sd.flags = flags;
  a.nsegs[seg_idx] = sd;
  atomicMax(&a.nctr->max_S, sd.S);
  for (uint32_t j = 0; j < nch; ++j) {
    ChunkDesc cd;
    cd.start = begin + (uint64_t)j * per;
    cd.len = min(per, m - j * per);
    cd.seg = seg_idx;
    a.nchunks[ch_off + j] = cd;
  }
}

// Per segment (run by the CTA that finished its last chunk): bucket bases (exclusive scan over
// k), child classes with the precedence of R20 (homogeneous > base > partition; small
// homogeneous children go with the base case, which leaves them unchanged), the no-progress
// guard (R10), next-level work, base-case windows and fills.  Thread t owns buckets
// 2t, 2t+1.
struct OffSmem {
  uint32_t warp[40];
  uint32_t res[8];
};
// Window-formation scratch (aliases the classify CTA's dynamic smem at the segment's end).
constexpr uint32_t kWinArrays = 8;  // start, end, brk_incl, sm_incl, small_idx, jump, J, mark
__host__ __device__ constexpr size_t win_scratch_bytes(uint32_t k) {
  return (size_t)kWinArrays * (k + 1) * 4;
}

// Greedy left-to-right packing of the children selected by `sel` into windows of <= cap keys
// (a window is a contiguous run of selected and empty children; any other non-empty child
// breaks it).  jump(c) = last child reachable from selected child c without a breaker and
// within cap keys (binary search); J(c) = first selected child after jump(c); the window
// starts are the orbit of the first selected child under J, marked by pointer doubling
// (log2 k rounds).  Appends the windows to `out` (global counter `cnt`, keys to `keys`).
template <int NT>
__device__ void pack_windows(const LevelArgs& a, const SegDesc& sg, uint32_t k,
                             const uint32_t (&bb)[kMaxK / NT], const uint32_t (&base)[kMaxK / NT],
                             const uint32_t (&tot)[kMaxK / NT], const bool (&sel)[kMaxK / NT], uint32_t cap,
                             uint32_t dstbuf, OffSmem& os, uint32_t* wsm, Window* out,
                             uint32_t out_cap, uint32_t* cnt, uint64_t* keys) {
  constexpr int BPT = kMaxK / NT;
  const uint32_t K1 = k + 1;
  uint32_t* w_start = wsm;
  uint32_t* w_end = wsm + K1;
  uint32_t* w_brk = wsm + 2 * K1;
  uint32_t* w_sm = wsm + 3 * K1;
  uint32_t* w_idx = wsm + 4 * K1;
  uint32_t* w_jump = wsm + 5 * K1;
  uint32_t* w_J = wsm + 6 * K1;
  uint32_t* w_mark = wsm + 7 * K1;
  uint32_t nbrk = 0, nsel = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    nbrk += (bb[q] < k && tot[q] && !sel[q]) ? 1u : 0u;
    nsel += sel[q] ? 1u : 0u;
  }
  uint32_t t_sel;
  uint32_t brk_run = block_exclusive_scan<NT>(nbrk, os.warp, nullptr);
  uint32_t sel_run = block_exclusive_scan<NT>(nsel, os.warp, &t_sel);
  if (t_sel == 0) return;  // block-uniform
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    if (bb[q] < k) {
      brk_run += (tot[q] && !sel[q]) ? 1u : 0u;
      if (sel[q]) w_idx[sel_run] = bb[q];
      sel_run += sel[q] ? 1u : 0u;
      w_start[bb[q]] = base[q];
      w_end[bb[q]] = base[q] + tot[q];
      w_brk[bb[q]] = brk_run;
      w_sm[bb[q]] = sel_run;
      w_mark[bb[q]] = 0u;
    }
  }
  if (threadIdx.x == 0) { w_J[k] = k; w_mark[k] = 0u; }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    if (sel[q]) {
      const uint32_t c = bb[q], st0 = base[q], bk0 = w_brk[c];
      uint32_t lo = c, hi = k;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (w_brk[mid] == bk0 && w_end[mid] - st0 <= cap) lo = mid; else hi = mid;
      }
      w_jump[c] = lo;
      const uint32_t m = w_sm[lo];
      w_J[c] = (m < t_sel) ? w_idx[m] : k;
    } else if (bb[q] < k) {
      w_J[bb[q]] = k;
    }
  }
  if (threadIdx.x == 0) w_mark[w_idx[0]] = 1u;
  __syncthreads();
  for (uint32_t span = 1; span < t_sel; span <<= 1) {
    uint32_t mk[BPT], jj[BPT], j2[BPT];
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      mk[q] = 0; jj[q] = k; j2[q] = k;
      if (bb[q] < k) {
        mk[q] = w_mark[bb[q]];
        jj[q] = w_J[bb[q]];
        j2[q] = w_J[jj[q]];
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      if (mk[q] && jj[q] < k) w_mark[jj[q]] = 1u;
      if (bb[q] < k) w_J[bb[q]] = j2[q];
    }
    __syncthreads();
  }
  uint32_t nw = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) nw += (sel[q] && w_mark[bb[q]]) ? 1u : 0u;
  uint32_t t_w;
  uint32_t w_off = block_exclusive_scan<NT>(nw, os.warp, &t_w);
  if (threadIdx.x == 0) os.res[4] = atomicAdd(cnt, t_w);
  __syncthreads();
  unsigned long long wkeys = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    if (sel[q] && w_mark[bb[q]]) {
      const uint32_t gi = os.res[4] + w_off++;
      if (gi < out_cap) {
        Window wv;
        wv.begin = sg.begin + base[q];
        wv.len = w_end[w_jump[bb[q]]] - base[q];
        wv.buf = dstbuf;
        out[gi] = wv;
        wkeys += wv.len;
      } else {
        atomicOr(a.err, kErrOverflow);
      }
    }
  }
  warp_add_u64((unsigned long long*)keys, wkeys);
  __syncthreads();  // scratch is reused by the next packing
}

// Per segment, at the end of phase 4a (run by the CTA that finished the segment's last
// chunk): bucket bases (exclusive scan over k) and child counts.  Thread t owns buckets
// 2t, 2t+1.
__device__ void segment_bases(const LevelArgs& a, uint32_t s, const SegDesc& sg,
                              const ModelDev& md, const uint32_t (&tot)[kCBpt], OffSmem& os) {
  const uint32_t k = a.k;
  uint32_t x = 0;
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) x += tot[q];
  uint32_t ex = block_exclusive_scan<kCThreads>(x, os.warp, nullptr);
  const uint32_t dstbuf = a.dstbuf;  // 1 = scratch, 0 = user array
  uint32_t cst[kCBpt];               // child starts inside the segment
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    const uint32_t b = threadIdx.x * kCBpt + q;
    cst[q] = ex;
    if (b < k) {
      const uint64_t enc = a.single_offsets ? (uint64_t)ex
                                            : ((dstbuf == 0 ? kDstUserBit : 0ull) | (sg.begin + ex));
      a.seg_dst[(size_t)s * k + b] = enc;
      a.seg_tot[(size_t)s * k + b] = tot[q];
      if (a.single_offsets && b < md.k_eff) a.single_offsets[b] = ex;
    }
    ex += tot[q];
  }
  if (a.single_offsets && threadIdx.x == 0) a.single_offsets[md.k_eff] = sg.m;
  // Terminal segment: every child goes to the base case, so the order inside a child before
  // the base case is unobservable (R13) and the scatter may place it unstably.
  int big = 0;
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) big |= tot[q] > a.base_case;
  const int any_big = __syncthreads_or(big);
  if (threadIdx.x == 0) a.seg_term[s] = (!a.single_offsets && !any_big) ? 1u : 0u;
  if (!a.tss || a.single_offsets || any_big) return;  // block-uniform
  // ---- terminal segment sort: windows of whole children (kTW, above) ----
  __shared__ uint32_t s_bnd[kTWMaxWin];
  __shared__ uint32_t s_mc, s_last, s_first;
  uint32_t mc = 0, last = 0;  // largest child, start of the last non-empty child
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    mc = max(mc, tot[q]);
    if (tot[q]) last = max(last, cst[q]);
  }
  if (threadIdx.x == 0) { s_mc = 0; s_last = 0; }
  __syncthreads();
  if (mc) atomicMax(&s_mc, mc);
  if (last) atomicMax(&s_last, last);
  __syncthreads();
  const uint32_t m = sg.m;
  const uint32_t Wp = (m <= kTW) ? 0u : kTW - s_mc;   // s_mc <= base case <= 4096 < kTW / 2
  // window g holds the children starting in [g W', (g+1) W'): none of these intervals is
  // empty up to the one holding the last child's start (no child is longer than W')
  const uint32_t G = Wp ? s_last / Wp + 1 : 1u;
  for (uint32_t g = threadIdx.x; g < G; g += kCThreads) s_bnd[g] = ~0u;
  __syncthreads();
  if (Wp) {
#pragma unroll
    for (int q = 0; q < kCBpt; ++q)
      if (tot[q]) atomicMin(&s_bnd[cst[q] / Wp], cst[q]);
  } else if (threadIdx.x == 0) {
    s_bnd[0] = 0;
  }
  if (threadIdx.x == 0) {
    s_first = atomicAdd(&a.nctr->n_twin, G);
    atomicAdd((unsigned long long*)&a.nctr->twin_keys, (unsigned long long)m);
    if (Wp) {
      atomicAdd(&a.nctr->n_twin_split, G);
      atomicAdd((unsigned long long*)&a.nctr->tsplit_keys, (unsigned long long)m);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.seg_tw[s] = make_uint2(s_first, Wp | (G << 16));
  for (uint32_t g = threadIdx.x; g < G; g += kCThreads) {
    const uint32_t gi = s_first + g;
    if (gi < a.cap_twin) {
      Window wv;
      wv.begin = sg.begin + s_bnd[g];
      wv.len = (g + 1 < G ? s_bnd[g + 1] : m) - s_bnd[g];
      wv.buf = Wp ? dstbuf : 1u - dstbuf;  // a one-window segment is sorted where it lies
      a.twins[gi] = wv;
      a.twcur[gi] = 0;
    } else {
      atomicOr(a.err, kErrOverflow);
    }
  }
}

// Per segment, after its last chunk has been scattered (run by that CTA): child classes with
// the precedence of R20 (homogeneous > base > partition; small homogeneous children go with
// the base case, which leaves them unchanged), the no-progress guard (R10), next-level work,
// base-case windows and fills.  Homogeneity of a child (R9) is merged here from
// the per-(chunk, bucket) flags the scatter recorded: a child is homogeneous iff every chunk
// that holds keys of it saw one value and all those values agree.  Only children above the
// base case can be classed homogeneous-final, so only they are merged.
template <int NT>
__device__ void segment_emit(const LevelArgs& a, uint32_t s, const SegDesc& sg, const ModelDev& md,
                             OffSmem& os, uint32_t* wsm) {
  constexpr int BPT = kMaxK / NT;
  const uint32_t k = a.k;
  uint32_t bb[BPT], base[BPT], tot[BPT], inh[BPT];
  uint64_t rep[BPT];
  uint32_t x = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    bb[q] = threadIdx.x * BPT + q;
    tot[q] = (bb[q] < k) ? a.seg_tot[(size_t)s * k + bb[q]] : 0u;
    x += tot[q];
    inh[q] = 1;
    rep[q] = 0;
    if (bb[q] < k && tot[q] > a.base_case) {
      bool have = false;
      uint64_t ref = 0;
      inh[q] = 0;
      for (uint32_t j = sg.chunk_first; j < sg.chunk_first + sg.nchunks; ++j) {
        const size_t jx = (size_t)j * k + bb[q];
        const uint8_t f = a.cflag[jx];
        if (f == 0) continue;
        if (f == 2) { inh[q] = 1; break; }
        const uint64_t r = a.cref[jx];
        if (have && r != ref) { inh[q] = 1; break; }
        ref = r;
        have = true;
      }
      rep[q] = ref;
    }
  }
  uint32_t ex = block_exclusive_scan<NT>(x, os.warp, nullptr);
#pragma unroll
  for (int q = 0; q < BPT; ++q) { base[q] = ex; ex += tot[q]; }
  int st = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q)
    if (md.kind != kModelEq3 && bb[q] < k && tot[q] == sg.m) st = 1;  // R10, R24
  const bool stuck = __syncthreads_or(st) != 0;
  const uint32_t dstbuf = a.dstbuf;  // 1 = scratch, 0 = user array
  uint32_t cls[BPT];
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    cls[q] = 0;  // 0 empty, 1 base (or small homogeneous), 2 partition, 3 big homogeneous
    if (!stuck && bb[q] < k && tot[q] > 0) {
      const bool homog = (md.kind == kModelEq3 && bb[q] == 1) || !inh[q];
      if (tot[q] <= a.base_case) cls[q] = 1;
      else if (homog) cls[q] = 3;
      else cls[q] = 2;
    }
  }
  // ---- next-level segments ----
  uint32_t w_seg = 0, w_samp = 0, w_ch = 0;
  uint32_t cm[BPT];
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    cm[q] = 0;
    if (stuck) { if (threadIdx.x == 0 && q == 0) cm[q] = sg.m; }
    else if (cls[q] == 2) cm[q] = tot[q];
    if (cm[q]) {
      w_seg += 1;
      w_samp += sample_size(cm[q], k);
      w_ch += chunks_of(cm[q], a.chunk_keys);
    }
  }
  uint32_t t_seg, t_samp, t_ch;
  uint32_t o_seg = block_exclusive_scan<NT>(w_seg, os.warp, &t_seg);
  uint32_t o_samp = block_exclusive_scan<NT>(w_samp, os.warp, &t_samp);
  uint32_t o_ch = block_exclusive_scan<NT>(w_ch, os.warp, &t_ch);
  if (threadIdx.x == 0 && t_seg) {
    os.res[0] = atomicAdd(&a.nctr->n_segs, t_seg);
    os.res[1] = atomicAdd(&a.nctr->n_samples, t_samp);
    os.res[2] = atomicAdd(&a.nctr->n_chunks, t_ch);
  }
  __syncthreads();
  if (t_seg) {
    bool ok = os.res[0] + t_seg <= a.cap_segs && os.res[1] + t_samp <= a.cap_samples &&
              os.res[2] + t_ch <= a.cap_chunks;
    if (!ok) {
      if (threadIdx.x == 0) atomicOr(a.err, kErrOverflow);
    } else {
      uint32_t i_seg = os.res[0] + o_seg, i_samp = os.res[1] + o_samp, i_ch = os.res[2] + o_ch;
      unsigned long long nkeys = 0;
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        if (cm[q]) {
          uint64_t cb = stuck ? sg.begin : sg.begin + base[q];
          emit_segment(a, cb, cm[q], stuck ? kSegForceEq3 : 0u, i_seg, i_samp, i_ch);
          nkeys += cm[q];
          i_seg += 1;
          i_samp += sample_size(cm[q], k);
          i_ch += chunks_of(cm[q], a.chunk_keys);
        }
      }
      warp_add_u64((unsigned long long*)&a.nctr->keys, nkeys);
    }
  }
  if (stuck) return;  // block-uniform
  // ---- base-case windows ----
  // Base children of <= kWBCap keys ("small") are packed into windows of <= kWBCap keys
  // (sorted by k_base_warp); base children above kWBCap ("big") into windows of <= kBigCap
  // keys (k_base_sort).  Every other child breaks a window.
  {
    bool small[BPT], bigb[BPT];
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      small[q] = bb[q] < k && cls[q] == 1 && tot[q] <= (uint32_t)kWBCap;
      bigb[q] = bb[q] < k && cls[q] == 1 && tot[q] > (uint32_t)kWBCap;
    }
    pack_windows<NT>(a, sg, k, bb, base, tot, small, (uint32_t)kWBCap, dstbuf, os, wsm, a.wins,
                 a.cap_wins, &a.nctr->n_windows, &a.nctr->win_keys);
    pack_windows<NT>(a, sg, k, bb, base, tot, bigb, (uint32_t)kBigCap, dstbuf, os, wsm, a.wins_big,
                 a.cap_wbig, &a.nctr->n_wbig, &a.nctr->wbig_keys);
  }
  // ---- homogeneous children that land in scratch must be filled into the user array ----
  uint32_t nf = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) nf += (cls[q] == 3 && dstbuf == 1) ? 1u : 0u;
  uint32_t t_fill;
  uint32_t o_fill = block_exclusive_scan<NT>(nf, os.warp, &t_fill);
  if (threadIdx.x == 0 && t_fill) os.res[5] = atomicAdd(&a.nctr->n_fills, t_fill);
  __syncthreads();
  unsigned long long fkeys = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    if (cls[q] == 3 && dstbuf == 1) {
      uint32_t gi = os.res[5] + o_fill++;
      if (gi < a.cap_fills) {
        Fill f;
        f.begin = sg.begin + base[q]; f.len = tot[q]; f.value = rep[q]; f.pad = 0;
        a.fills[gi] = f;
        fkeys += tot[q];
      } else {
        atomicOr(a.err, kErrOverflow);
      }
    }
  }
  warp_add_u64((unsigned long long*)&a.nctr->fill_keys, fkeys);
}

// Tile loop of phase 4a with the model kind and the optional outputs fixed at compile time.
// Per key: model evaluation (2 RN ops + saturating convert) and one smem atomicAdd into the
// chunk histogram (+ the NaN test at level 0).  The next tile is loaded while this one is
// classified.
template <bool F64, int MODE, bool NANCHK, bool IDS>
__device__ void classify_tiles(const LevelArgs& a, const ChunkDesc& ch, const ModelDev& md,
                               uint32_t* hist, int& nan_seen) {
  const Bucketer<F64, MODE> bucket(md, a.k);
  const uint64_t* p = a.src + ch.start;
  uint64_t cur[kCItems], nxt[kCItems];
#pragma unroll
  for (int r = 0; r < kCItems; ++r) {
    const uint32_t i = r * kCThreads + threadIdx.x;
    cur[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
  }
  bool nan = false;
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kCTile) {
    const uint32_t tl = min((uint32_t)kCTile, ch.len - t0);
    const uint32_t t1 = t0 + kCTile;
#pragma unroll
    for (int r = 0; r < kCItems; ++r) {
      const uint32_t i = t1 + r * kCThreads + threadIdx.x;
      nxt[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
    }
#pragma unroll
    for (int r = 0; r < kCItems; ++r) {
      const uint32_t i = r * kCThreads + threadIdx.x;
      if (i < tl) {
        if (NANCHK) nan |= isnan(__longlong_as_double((long long)cur[r]));
        const uint32_t b = bucket(cur[r]);
        atomicAdd(&hist[b], 1u);
        if (IDS) a.ids[ch.start + t0 + i] = (uint16_t)b;
      }
    }
#pragma unroll
    for (int r = 0; r < kCItems; ++r) cur[r] = nxt[r];
  }
  nan_seen = nan ? 1 : 0;
}

template <bool F64, int MODE>
__device__ __forceinline__ void classify_dispatch(const LevelArgs& a, const ChunkDesc& ch,
                                                  const ModelDev& md, uint32_t* hist,
                                                  int& nan_seen) {
  if (a.ids)
    classify_tiles<F64, MODE, false, true>(a, ch, md, hist, nan_seen);
  else if (F64 && a.check_nan)
    classify_tiles<F64, MODE, F64, false>(a, ch, md, hist, nan_seen);
  else
    classify_tiles<F64, MODE, false, false>(a, ch, md, hist, nan_seen);
}

// TREE selects the kernel instantiation of the splitter-tree model (IPLS_FLAG_TREE_MODEL):
// its segments are TREE or EQ3, the default instantiation's LINEAR or EQ3, so each kernel
// carries two bucket functions only.
template <bool F64, bool TREE>
__global__ __launch_bounds__(kCThreads) void k_classify_scan(LevelArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const uint32_t k = a.k;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smraw);  // k
  __shared__ uint32_t s_c;
  __shared__ OffSmem os;
  if (threadIdx.x == 0) s_c = atomicAdd(a.ticket, 1u);
  for (uint32_t b = threadIdx.x; b < k; b += kCThreads) hist[b] = 0;
  __syncthreads();
  const uint32_t c = s_c;
  const ChunkDesc ch = a.chunks[c];
  const SegDesc sg = a.segs[ch.seg];
  ModelDev md = a.models[ch.seg];
  if constexpr (TREE) {  // top 8 levels of the splitter heap into smem
    __shared__ uint64_t s_top[256];
    if (md.kind == kModelTree)
      for (uint32_t j = threadIdx.x; j < min(k, 256u); j += kCThreads) s_top[j] = md.heap[j];
    md.top = s_top;
    __syncthreads();
  }
  int nan_seen = 0;
  if (md.kind == kModelEq3) {
    classify_dispatch<F64, kModelEq3>(a, ch, md, hist, nan_seen);
  } else if constexpr (TREE) {
    if (md.leaves != k) classify_dispatch<F64, kModelTreeEq>(a, ch, md, hist, nan_seen);
    else classify_dispatch<F64, kModelTree>(a, ch, md, hist, nan_seen);
  } else {
    classify_dispatch<F64, kModelLinear>(a, ch, md, hist, nan_seen);
  }
  if (a.check_nan) {
    if (__syncthreads_or(nan_seen) && threadIdx.x == 0) atomicOr(a.err, kErrNan);
  } else {
    __syncthreads();
  }
  // ---- decoupled lookback over the chunks of this segment, bucket by bucket ----
  // One 64-bit status word per (chunk, bucket): AGG (own count) or INC (inclusive prefix),
  // tagged with the level's epoch; the host clears the status region before every level (a
  // stale word of another array could otherwise carry the current tag).
  const bool first = (c == sg.chunk_first);
  const bool last = (c == sg.chunk_first + sg.nchunks - 1);
  uint32_t tot[kCBpt];
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    const uint32_t b = threadIdx.x * kCBpt + q;
    tot[q] = (b < k) ? hist[b] : 0u;
    if (b < k && sg.nchunks > 1 && !last)
      *((volatile uint64_t*)&a.status[(size_t)c * k + b]) =
          pack_status(a.epoch, first ? kStInc : kStAgg, 0u, tot[q]);
  }
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    const uint32_t b = threadIdx.x * kCBpt + q;
    if (b >= k) continue;
    uint32_t ex_cnt = 0;
    if (!first) {
      uint32_t j = c - 1;
      while (true) {
        const uint64_t st = *((volatile const uint64_t*)&a.status[(size_t)j * k + b]);
        const uint32_t state = (uint32_t)(st >> 46) & 3u;
        if ((uint32_t)(st >> 48) != (a.epoch & 0xffff) || state == 0) continue;  // not yet
        ex_cnt += (uint32_t)st;
        if (state == kStInc) break;
        --j;
      }
      if (!last)
        *((volatile uint64_t*)&a.status[(size_t)c * k + b]) =
            pack_status(a.epoch, kStInc, 0u, ex_cnt + tot[q]);
    }
    a.chunk_pre[(size_t)c * k + b] = ex_cnt;
    tot[q] += ex_cnt;
  }
  if (last) segment_bases(a, ch.seg, sg, md, tot, os);
}

// ------------------------------------------------------------------------------------
// Phase 4b: scatter of one chunk into its segment's children (R11).
//
// Two kernels of 512 threads with tiles of kSTile = 8192 keys (16 per thread, in registers;
// warp w owns keys [512 w, 512 w + 512) of the tile and item r of lane l is key
// 512 w + 32 r + l, so every load is one coalesced 256-byte warp access):
//   k_scatter_stable  chunks of segments with a child above the base case: those children are
//                     sampled by position at the next level, so the layout is the stable one
//                     (R11); 1 CTA per SM.
//   k_scatter_term    chunks of terminal segments (every child <= base case): the children go
//                     to the base case, an exact sort, so their interior order is free;
//                     2 CTAs per SM.
// Each kernel returns at once for the other kind of chunk; a segment's chunks are all of one
// kind.  The CTA that completes a segment's last chunk runs segment_emit.
//
// Per tile: (A) ranks, (B) per-bucket offsets, (C) placement into a bucket-sorted smem stage,
// (D) write-out of the stage.  Staged key q of bucket b goes to adjo[b] + q, adjo[b] = the
// absolute position of bucket b's next key minus the run's start in the stage: a warp's 32
// consecutive staged keys cover a few runs, so the stores coalesce per run.  Stores carry an
// L2 evict_last policy so that lines of runs still open survive until the next tile completes
// them.
//
// Cost model.  Both kernels are bound by the shared-memory (LSU) pipe, ~1 wavefront per clock
// per SM, and its latency, not by instruction issue (ncu, profiles/r02_*).  So the write-out
// recomputes a staged key's bucket (two FP64 ops) instead of staging it (a random 4-byte
// store and a load), and a key's staged predecessor comes from the neighbouring lane by
// shuffle instead of a second load.
//
// Stable rank (k_scatter_stable).  Every key does one shared-memory atomicAdd with return on
// its warp's 16-bit counter for its bucket (two warps share a 32-bit word); the per-bucket
// prefix over the warps (B) completes it.  The returned value is the key's rank among the
// warp's earlier keys of its bucket if same-address lanes of one atomic are served in lane
// order.  B200 does that (tools/micro/atom_order.cu: 0 violations in 2.2e9 lane pairs), but
// the PTX model does not promise it, so every CTA first probes it on a few lane patterns
// (atomic_lane_order_ok) and ranks with match.any peer masks if the probe fails: the leader of
// each group of same-bucket lanes does one atomic for the group and the others add their
// popcount rank -- stable by construction.  That path is the fallback, not the default,
// because match.any serialises per distinct value: tools/micro/rank.cu measures 2.2 T keys/s
// for the atomic rank, 0.26 T for a 10-ballot peer mask and 0.15 T for match.any, against
// ~0.4 T keys/s for one pass at HBM speed.  ipls_debug_force_match_rank forces the fallback
// (the tests run both).
//
// Homogeneity (R9, stable kernel only): a staged key that differs from its staged predecessor
// of the same bucket marks the bucket "several values"; the first key of every bucket run in
// a tile is compared with the chunk's first key of that bucket.  The chunk's flags (0 empty,
// 1 one value, 2 several) and values go to global memory for segment_emit.
constexpr int kSThreads = 512;
constexpr int kSWarps = kSThreads / 32;      // 16
constexpr int kSItems = 16;                  // keys per thread per tile
constexpr int kSTile = kSThreads * kSItems;  // 8192
constexpr int kSPairs = kSWarps / 2;         // counter words per bucket (two warps per word)
constexpr int kSBpt = kMaxK / kSThreads;     // buckets per thread (t and t + 512)
static_assert(kSBpt == 2, "bucket ownership t, t + kSThreads");

__host__ __device__ constexpr size_t scatter_stable_smem_bytes(uint32_t k) {
  return (size_t)kSTile * 8 + (size_t)kSTile * 2 + (size_t)2 * kSPairs * k * 4 + (size_t)k * 8 +
         (size_t)k * 4 * 2 + (size_t)k * 2 + 64;
}
// PEER variant: plus the k per-bucket destination bases
__host__ __device__ constexpr size_t scatter_peer_smem_bytes(uint32_t k) {
  return scatter_stable_smem_bytes(k) + (size_t)k * 8 + 8;
}

#ifdef IPLS_SCATTER_TIMING
#define SC_TICK(N) do { if (threadIdx.x == 0) { const long long t_ = clock64(); atomicAdd(&g_sc_phase[N], (unsigned long long)(t_ - t_prev_)); t_prev_ = t_; } } while (0)
#else
#define SC_TICK(N)
#endif

__device__ int g_force_match_rank;  // ipls_debug_force_match_rank: every CTA ranks by match.any

// L2 evict_last policy for the run stores (created once per thread)
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp 0: are same-address lanes of one shared-memory atomicAdd served in lane order?  Four
// lane patterns (all lanes on one word; two interleaved groups; blocks of 8; a scrambled
// 4-group pattern), each compared with the rank popc(lanes below on the same word).
__device__ bool atomic_lane_order_ok(uint32_t* scratch /* 4 words */) {
  const uint32_t lane = threadIdx.x & 31;
  bool ok = true;
#pragma unroll
  for (int pat = 0; pat < 4; ++pat) {
    auto addr = [&](uint32_t l) -> uint32_t {
      return pat == 0 ? 0u : pat == 1 ? (l & 1u) : pat == 2 ? (l >> 3) : ((l * 13u + 5u) >> 2) & 3u;
    };
    if (lane < 4) scratch[lane] = 0u;
    __syncwarp();
    const uint32_t my = addr(lane);
    const uint32_t got = atomicAdd(&scratch[my], 1u);
    uint32_t want = 0;
    for (uint32_t l = 0; l < lane; ++l) want += addr(l) == my ? 1u : 0u;
    ok &= got == want;
    __syncwarp();
  }
  return __all_sync(0xffffffffu, ok);
}

// Destination of a chunk's bucket runs: the buffer and every run's absolute start (u32; the
// ABI limits n to 2^32 - 1 keys).
template <int NT>
__device__ __forceinline__ uint64_t* chunk_runs(const LevelArgs& a, uint64_t* dst_user,
                                                uint64_t* dst_scr, uint32_t c, uint32_t seg,
                                                uint32_t* runo) {
  const uint32_t k = a.k;
  for (uint32_t b = threadIdx.x; b < k; b += NT) {
    const uint64_t d = a.seg_dst[(size_t)seg * k + b] + a.chunk_pre[(size_t)c * k + b];
    runo[b] = (uint32_t)(d & ~kDstUserBit);
  }
  return (a.seg_dst[(size_t)seg * k] & kDstUserBit) ? dst_user : dst_scr;
}

// Exclusive scan of one u32 per thread over the CTA with one barrier (the warp totals are
// read by every thread; `sw` must not be reused before the caller's next barrier).
template <int NT>
__device__ __forceinline__ uint32_t scan_excl_1bar(uint32_t x, uint32_t* sw, uint32_t& total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sw[w] = inc;
  __syncthreads();
  // every warp scans the NW warp totals itself (one load per lane, shuffles): no second
  // barrier, and no NW broadcast loads per thread
  const uint32_t wt = (lane < NW) ? sw[lane] : 0u;
  uint32_t wi = wt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
    if (lane >= o) wi += y;
  }
  const uint32_t before = __shfl_sync(0xffffffffu, wi - wt, w);
  total = __shfl_sync(0xffffffffu, wi, NW - 1);
  return before + inc - x;
}

// Rank modes of phase A in the stable kernel.
constexpr int kRankAtomic = 0, kRankDense = 1, kRankMatch = 2;

// PEER (the multi-GPU exchange fused into the scatter): every bucket has its own
// destination base address (a.bucket_dst, copied to smem), so a run is written straight into
// the buffer of the rank that owns the bucket; the run offsets are the chunk prefixes alone.
template <bool F64, int MODE, bool PEER = false>
__device__ void scatter_stable_chunk(const LevelArgs& a, uint64_t* __restrict__ dst_user,
                                     uint64_t* __restrict__ dst_scr, uint32_t c,
                                     const ChunkDesc& ch, const ModelDev& md,
                                     unsigned char* smraw) {
  constexpr int NT = kSThreads;
  constexpr bool kStageBucket =  // a tree descent costs more than a load
      MODE == (int)kModelTree || MODE == (int)kModelTreeEq;
  const uint32_t k = a.k;
  uint64_t* stage = reinterpret_cast<uint64_t*>(smraw);              // kSTile keys
  uint16_t* sbk = reinterpret_cast<uint16_t*>(stage + kSTile);        // kSTile (tree only)
  uint32_t* tab0 = reinterpret_cast<uint32_t*>(sbk + kSTile);         // 2 x kSPairs x k counters
  uint64_t* ref = reinterpret_cast<uint64_t*>(tab0 + 2 * kSPairs * k);  // k: chunk's first key
  uint32_t* runo = reinterpret_cast<uint32_t*>(ref + k);              // k: next write position
  uint32_t* adjo = runo + k;                                          // k: runo - run start
  uint8_t* seen = reinterpret_cast<uint8_t*>(adjo + k);               // k: bucket seen in chunk
  uint8_t* multi = seen + k;                                          // k: several values seen
  __shared__ uint32_t s_warp[2][kSWarps];
  __shared__ uint32_t s_probe[4];
  __shared__ int s_match;
  const Bucketer<F64, MODE> bucket(md, k);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const uint32_t t = threadIdx.x;
  const uint32_t lt = lanemask_lt();
  uint64_t* dst = nullptr;
  uint64_t** pdst = nullptr;  // PEER: per-bucket destination bases
  if constexpr (PEER) {
    pdst = reinterpret_cast<uint64_t**>((reinterpret_cast<uintptr_t>(multi + k) + 7) & ~(uintptr_t)7);
    for (uint32_t b = t; b < k; b += NT) {
      runo[b] = a.chunk_pre[(size_t)c * k + b];
      pdst[b] = reinterpret_cast<uint64_t*>(a.bucket_dst[b]);
    }
  } else {
    dst = chunk_runs<NT>(a, dst_user, dst_scr, c, ch.seg, runo);
  }
  for (uint32_t b = t; b < k; b += NT) { seen[b] = 0; multi[b] = 0; }
  {  // both counter tables start cleared
    uint4* z = reinterpret_cast<uint4*>(tab0);
    for (uint32_t i = t; i < 2 * kSPairs * k / 4; i += NT) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (wp == 0) {
    const bool ok = atomic_lane_order_ok(s_probe);
    if (lane == 0) s_match = (!ok || *((volatile int*)&g_force_match_rank)) ? 1 : 0;
  }
  const uint64_t pol = policy_evict_last();
  const uint32_t winc = 1u << (16 * (wp & 1));
  const int wsh = 16 * (wp & 1);
  const uint64_t* p = a.src + ch.start;
  uint64_t key[kSItems];
#pragma unroll
  for (int r = 0; r < kSItems; ++r) {
    const uint32_t i = wp * (kSItems * 32) + r * 32 + lane;
    key[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
  }
  __syncthreads();
  const bool use_match = s_match != 0;  // block-uniform
#ifdef IPLS_SCATTER_TIMING
  long long t_prev_ = clock64();
#endif
  bool dense = false;  // block-uniform
  int it = 0;
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kSTile, ++it) {
    const uint32_t tl = min((uint32_t)kSTile, ch.len - t0);
    const bool full = tl == (uint32_t)kSTile;  // block-uniform: no bounds checks
    uint32_t* tab = tab0 + (it & 1) * (kSPairs * k);
    uint32_t* tabn = tab0 + ((it & 1) ^ 1) * (kSPairs * k);
    uint32_t* tw = tab + (wp >> 1) * k;
    // ---- (A) ranks: bucket | in-warp rank << 16 ----
    uint32_t bl[kSItems];
    if (full && !dense && !use_match) {
      // all buckets, then all atomics back to back, then the ranks: the atomics' latency
      // overlaps instead of stalling every item
#pragma unroll
      for (int r = 0; r < kSItems; ++r) bl[r] = bucket(key[r]);
      uint32_t old[kSItems];
#pragma unroll
      for (int r = 0; r < kSItems; ++r) old[r] = atomicAdd(&tw[bl[r]], winc);
#pragma unroll
      for (int r = 0; r < kSItems; ++r) bl[r] |= ((old[r] >> wsh) & 0xffffu) << 16;
    } else {
      auto rank_items = [&](auto mode_tag) {
        constexpr int RM = decltype(mode_tag)::value;
#pragma unroll
        for (int r = 0; r < kSItems; ++r) {
          const uint32_t i = wp * (kSItems * 32) + r * 32 + lane;
          const bool valid = i < tl;
          const uint32_t b = valid ? bucket(key[r]) : 0u;
          uint32_t loc = 0;
          if constexpr (RM == kRankMatch) {
            const uint32_t peers = __match_any_sync(0xffffffffu, valid ? b : 0xffffffffu);
            const int leader = __ffs(peers) - 1;
            uint32_t old = 0;
            if (valid && lane == leader) old = atomicAdd(&tw[b], __popc(peers) * winc);
            old = __shfl_sync(0xffffffffu, old, leader);
            loc = ((old >> wsh) & 0xffffu) + __popc(peers & lt);
          } else if constexpr (RM == kRankDense) {
            // few buckets per tile (presorted, clustered or EQ3 input): a warp whose keys
            // share one bucket takes one atomic instead of 32 serialised same-address lanes
            const uint32_t b0 = __shfl_sync(0xffffffffu, b, 0);
            if (__all_sync(0xffffffffu, !valid || b == b0)) {
              const uint32_t nv = __popc(__ballot_sync(0xffffffffu, valid));
              uint32_t base = 0;
              if (lane == 0 && nv) base = atomicAdd(&tw[b0], nv * winc);
              loc = ((__shfl_sync(0xffffffffu, base, 0) >> wsh) & 0xffffu) + lane;
            } else if (valid) {
              loc = (atomicAdd(&tw[b], winc) >> wsh) & 0xffffu;
            }
          } else {
            if (valid) loc = (atomicAdd(&tw[b], winc) >> wsh) & 0xffffu;
          }
          bl[r] = b | (loc << 16);
        }
      };
      if (use_match) rank_items(std::integral_constant<int, kRankMatch>{});
      else if (dense) rank_items(std::integral_constant<int, kRankDense>{});
      else rank_items(std::integral_constant<int, kRankAtomic>{});
    }
    __syncthreads();
    SC_TICK(0);
#ifdef IPLS_SCATTER_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_sc_phase[28], 1ull);
#endif
    // ---- (B) warp prefixes and run starts per bucket ----
    uint32_t cnt[kSBpt], wv[kSBpt][kSPairs];
#pragma unroll
    for (int q = 0; q < kSBpt; ++q) {
      const uint32_t b = t + q * NT;
      uint32_t s = 0;
#pragma unroll
      for (int pp = 0; pp < kSPairs; ++pp) {
        wv[q][pp] = (b < k) ? tab[pp * k + b] : 0u;
        s += wv[q][pp];
      }
      cnt[q] = (s & 0xffffu) + (s >> 16);  // no carry: a tile holds <= 8192 keys
    }
    {  // clear the other table for the next tile
      uint4* z = reinterpret_cast<uint4*>(tabn);
#pragma unroll
      for (int j = 0; j < kSPairs * kMaxK / 4 / NT; ++j) {
        const uint32_t i = t + j * NT;
        if (i < kSPairs * k / 4) z[i] = make_uint4(0, 0, 0, 0);
      }
    }
    uint32_t tot;
    const uint32_t ex = scan_excl_1bar<NT>(cnt[0] | (cnt[1] << 16), s_warp[it & 1], tot);
    const uint32_t off[kSBpt] = {ex & 0xffffu, (tot & 0xffffu) + (ex >> 16)};
#pragma unroll
    for (int q = 0; q < kSBpt; ++q) {
      const uint32_t b = t + q * NT;
      if (b < k) {
        const uint32_t ro = runo[b];
        adjo[b] = ro - off[q];
        runo[b] = ro + cnt[q];
        uint32_t run = off[q];
#pragma unroll
        for (int pp = 0; pp < kSPairs; ++pp) {
          const uint32_t w = wv[q][pp], lo = w & 0xffffu;
          tab[pp * k + b] = run | ((run + lo) << 16);
          run += lo + (w >> 16);
        }
      }
    }
    // next tile's path: dense when this tile averages >= 32 keys per non-empty bucket
    // (__syncthreads_count counts threads: bucket t + 512 is assumed as full as bucket t)
    dense = (uint32_t)__syncthreads_count(cnt[0] != 0) * (k > NT ? 2u : 1u) * 32u <= tl;
    SC_TICK(1);
    // ---- (C) placement into the stage; loads of the next tile ----
    if (full) {
      uint32_t pos[kSItems];
#pragma unroll
      for (int r = 0; r < kSItems; ++r) pos[r] = tw[bl[r] & 0xffffu];
#pragma unroll
      for (int r = 0; r < kSItems; ++r) {
        const uint32_t q = ((pos[r] >> wsh) & 0xffffu) + (bl[r] >> 16);
        stage[q] = key[r];
        if constexpr (kStageBucket) sbk[q] = (uint16_t)(bl[r] & 0xffffu);
      }
    } else {
#pragma unroll
      for (int r = 0; r < kSItems; ++r) {
        const uint32_t i = wp * (kSItems * 32) + r * 32 + lane;
        if (i < tl) {
          const uint32_t b = bl[r] & 0xffffu;
          const uint32_t q = ((tw[b] >> wsh) & 0xffffu) + (bl[r] >> 16);
          stage[q] = key[r];
          if constexpr (kStageBucket) sbk[q] = (uint16_t)b;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kSItems; ++r) {
      const uint32_t i = t0 + kSTile + wp * (kSItems * 32) + r * 32 + lane;
      key[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
    }
    {  // and the tile after it into the L2, one 128-byte line per thread
      const uint32_t i = t0 + 2 * kSTile + t * 16;
      if (i < ch.len) asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(p + i));
    }
    __syncthreads();
    SC_TICK(2);
    // ---- (D) write-out: warp w writes staged slots [512 w, 512 w + 512), 8 at a time ----
    {
      const uint32_t q0 = wp * (kSItems * 32);
      // the staged predecessor of slot q comes from lane - 1 (a rotate by one lane); lane 0
      // takes lane 31's from the previous batch item
      uint64_t cv = 0;
      uint32_t cb = 0xffffffffu;  // no predecessor
      if (q0 > 0 && q0 - 1 < tl) {
        cv = stage[q0 - 1];
        if constexpr (kStageBucket) cb = sbk[q0 - 1]; else cb = bucket(cv);
      }
      const int src_lane = (lane + 31) & 31;
#pragma unroll
      for (int h = 0; h < kSItems / 8; ++h) {
        uint64_t v[8];
        uint32_t b[8], ao[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t q = q0 + (h * 8 + j) * 32 + lane;
          v[j] = (full || q < tl) ? stage[q] : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t q = q0 + (h * 8 + j) * 32 + lane;
          if constexpr (kStageBucket) b[j] = (full || q < tl) ? sbk[q] : 0xfffffffeu;
          else b[j] = (full || q < tl) ? bucket(v[j]) : 0xfffffffeu;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) ao[j] = adjo[min(b[j], k - 1)];  // invalid slots: any bucket
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t q = q0 + (h * 8 + j) * 32 + lane;
          const uint64_t rv = __shfl_sync(0xffffffffu, v[j], src_lane);
          const uint32_t rb = __shfl_sync(0xffffffffu, b[j], src_lane);
          const uint64_t vp = lane ? rv : cv;
          const uint32_t bp = lane ? rb : cb;
          cv = rv;
          cb = rb;
          if (full || q < tl) {
            if (b[j] == bp) {
              if (v[j] != vp) multi[b[j]] = 1;
            } else {  // first key of bucket b's run in this tile
              if (!seen[b[j]]) { ref[b[j]] = v[j]; seen[b[j]] = 1; }
              else if (ref[b[j]] != v[j]) multi[b[j]] = 1;
            }
            if constexpr (PEER) pdst[b[j]][(uint32_t)(ao[j] + q)] = v[j];
            else st_hint(dst + (uint32_t)(ao[j] + q), v[j], pol);
          }
        }
      }
    }
    SC_TICK(3);
  }
  __syncthreads();
  for (uint32_t b = t; b < k; b += NT) {
    const uint8_t cf = seen[b] ? (multi[b] ? 2 : 1) : 0;
    a.cflag[(size_t)c * k + b] = cf;
    if (cf == 1) a.cref[(size_t)c * k + b] = ref[b];
  }
}

// Terminal chunks (k_scatter_term): 1024 threads (32 warps, 1 CTA per SM), tiles of 8192 keys
// streamed through a ring of kTRing smem slots by TMA bulk copies issued two tiles ahead, so
// no load latency is exposed inside a chunk and keys never wait in prefetch registers.  A
// slot doubles as its tile's stage: (A) keys to registers + count per bucket, (B) run starts,
// (C) placement by an atomic cursor per bucket into the same slot, (D) write-out with the
// bucket recomputed from the staged key.  No warp counters, no homogeneity (terminal
// segments have no child above the base case).
constexpr int kTThreads = 1024;
constexpr int kTItems = 8;
constexpr int kTTile = kTThreads * kTItems;   // 8192
constexpr int kTRing = 3;
constexpr int kTSlot = kTTile + 4;            // keys per slot (+ parity shift, 32-byte multiple)

__host__ __device__ constexpr size_t scatter_term_smem_bytes(uint32_t k) {
  return (size_t)kTRing * kTSlot * 8 + (size_t)k * 4 * 4 + 64;
}

// Tile [t0, t0 + tl) of a chunk starting at p (h = parity of its start): the keys land at
// slot[h + i].  One TMA bulk copy completing on `bar` moves the 16-byte-aligned span around
// them (a key before and after the tile are read along and ignored); only at the very end of
// the array, where no key follows an odd span, the last key is loaded by the issuing thread
// itself (synchronously: once per level).  Thread 0 only.  room = keys from p + t0 to the end
// of the array.
__device__ __forceinline__ void tile_issue(uint64_t* slot, const uint64_t* p, uint32_t h,
                                           uint32_t t0, uint32_t tl, uint64_t room, uint64_t* bar) {
  uint32_t n = h + tl;               // keys from p + t0 - h (16-byte aligned)
  if ((n & 1u) && (uint64_t)tl < room) ++n;
  const uint32_t body = n & ~1u;
  if (n & 1u) slot[n - 1] = __ldcs(p + t0 + tl - 1);
  if (body) {
    mbar_arrive_tx(bar, body * 8u);
    bulk_g2s(slot, p + t0 - h, body * 8u, bar);
  } else {
    mbar_arrive(bar);
  }
}

template <bool F64, int MODE>
__device__ void scatter_term_chunk(const LevelArgs& a, uint64_t* __restrict__ dst_user,
                                   uint64_t* __restrict__ dst_scr, uint32_t c,
                                   const ChunkDesc& ch, const ModelDev& md, unsigned char* smraw,
                                   uint32_t* next_ticket = nullptr) {
  constexpr int NT = kTThreads;
  const uint32_t k = a.k;
  uint64_t* slots = reinterpret_cast<uint64_t*>(smraw);            // kTRing x kTSlot
  uint32_t* cnt = reinterpret_cast<uint32_t*>(slots + kTRing * kTSlot);  // k
  uint32_t* cur = cnt + k;                                          // k: placement cursor
  uint32_t* runo = cur + k;                                         // k
  uint32_t* adjo = runo + k;                                        // k
  __shared__ uint32_t s_warp[2][32];
  __shared__ __align__(8) uint64_t s_bar[kTRing];
  const Bucketer<F64, MODE> bucket(md, k);
  const int lane = threadIdx.x & 31;
  const uint32_t t = threadIdx.x;
  uint64_t* dst = chunk_runs<NT>(a, dst_user, dst_scr, c, ch.seg, runo);
  for (uint32_t b = t; b < k; b += NT) cnt[b] = 0;
  const uint64_t* p = a.src + ch.start;
  const uint32_t h = (uint32_t)(reinterpret_cast<uintptr_t>(p) >> 3) & 1u;
  const uint32_t ntile = (ch.len + kTTile - 1) / kTTile;
  const uint64_t room = a.nkeys - ch.start;
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < kTRing; ++s) mbar_init(&s_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t j = 0; j < min(ntile, (uint32_t)kTRing - 1); ++j)
      tile_issue(slots + j * kTSlot, p, h, j * kTTile, min((uint32_t)kTTile, ch.len - j * kTTile),
                 room - j * kTTile, &s_bar[j]);
    // k_term_fused: the next chunk's ticket, while the first tiles load
    if (next_ticket) *next_ticket = atomicAdd(&a.nctr->sticket, 1u);
  }
  const uint64_t pol = policy_evict_last();
  __syncthreads();
#ifdef IPLS_SCATTER_TIMING
  long long t_prev_ = clock64();
#endif
  bool dense = false;  // block-uniform
  for (uint32_t it = 0; it < ntile; ++it) {
    const uint32_t t0 = it * kTTile;
    const uint32_t tl = min((uint32_t)kTTile, ch.len - t0);
    const uint32_t s = it % kTRing;
    uint64_t* slot = slots + s * kTSlot;
    mbar_wait(&s_bar[s], (it / kTRing) & 1u);
    // ---- (A) keys to registers, counts ----
    uint64_t v[kTItems];
    uint32_t bk[kTItems];
#pragma unroll
    for (int r = 0; r < kTItems; ++r) {
      const uint32_t i = r * NT + t;
      v[r] = (i < tl) ? slot[h + i] : 0ull;
      bk[r] = (i < tl) ? bucket(v[r]) : 0xffffffffu;
    }
    // The count's return value is the key's rank among the tile's keys of its bucket (the
    // order inside a terminal child is free, R11): bk = bucket | rank << 16.
    if (!dense) {
#pragma unroll
      for (int r = 0; r < kTItems; ++r)
        if (bk[r] != 0xffffffffu) bk[r] |= atomicAdd(&cnt[bk[r]], 1u) << 16;
    } else {
#pragma unroll
      for (int r = 0; r < kTItems; ++r) {
        const uint32_t b0 = __shfl_sync(0xffffffffu, bk[r], 0);
        if (__all_sync(0xffffffffu, bk[r] == b0 || bk[r] == 0xffffffffu)) {
          // valid lanes are a prefix of the warp (the tile's tail is its last keys)
          const uint32_t nv = __popc(__ballot_sync(0xffffffffu, bk[r] != 0xffffffffu));
          uint32_t base = 0;
          if (lane == 0 && nv) base = atomicAdd(&cnt[b0], nv);
          base = __shfl_sync(0xffffffffu, base, 0);
          if (bk[r] != 0xffffffffu) bk[r] |= (base + (uint32_t)lane) << 16;
        } else if (bk[r] != 0xffffffffu) {
          bk[r] |= atomicAdd(&cnt[bk[r]], 1u) << 16;
        }
      }
    }
    __syncthreads();
    SC_TICK(4);
#ifdef IPLS_SCATTER_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_sc_phase[29], 1ull);
#endif
    // every thread is past D(it - 1): its slot takes tile it + kTRing - 1
    if (t == 0 && it + kTRing - 1 < ntile) {
      const uint32_t jn = it + kTRing - 1, sn = jn % kTRing;
      tile_issue(slots + sn * kTSlot, p, h, jn * kTTile, min((uint32_t)kTTile, ch.len - jn * kTTile),
                 room - jn * kTTile, &s_bar[sn]);
    }
    // ---- (B) run starts (scan over buckets, thread t owns bucket t) ----
    uint32_t cc = 0;
    if (t < k) { cc = cnt[t]; cnt[t] = 0; }
    uint32_t tot;
    const uint32_t off = scan_excl_1bar<NT>(cc, s_warp[it & 1], tot);
    if (t < k) {
      cur[t] = off;
      const uint32_t ro = runo[t];
      adjo[t] = ro - off;
      runo[t] = ro + cc;
    }
    dense = (uint32_t)__syncthreads_count(cc != 0) * 32u <= tl;
    SC_TICK(5);
    // ---- (C) placement into the slot (every thread holds its keys in registers) ----
#pragma unroll
    for (int r = 0; r < kTItems; ++r)
      if (r * NT + t < tl) slot[cur[bk[r] & 0xffffu] + (bk[r] >> 16)] = v[r];
    __syncthreads();
    SC_TICK(6);
    // ---- (D) write-out ----
#pragma unroll
    for (int r = 0; r < kTItems; ++r) {
      const uint32_t q = r * NT + t;
      v[r] = (q < tl) ? slot[q] : 0ull;
    }
#pragma unroll
    for (int r = 0; r < kTItems; ++r) bk[r] = adjo[bucket(v[r])];
#pragma unroll
    for (int r = 0; r < kTItems; ++r) {
      const uint32_t q = r * NT + t;
      if (q < tl) st_hint(dst + (uint32_t)(bk[r] + q), v[r], pol);
    }
    SC_TICK(7);
  }
}

// After both scatter kernels: one CTA per segment classes its children (R20), applies the
// no-progress guard (R10) and emits the next level's work, the base-case windows and the fills
// (segment_emit).  A kernel of its own, so that the level's ~k-wide per-segment bookkeeping runs
// on all SMs at once instead of as a serial tail inside the scatter CTA that finished last.
constexpr int kEThreads = 512;
__global__ __launch_bounds__(kEThreads) void k_emit(LevelArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ OffSmem os;
  if (*((volatile const uint32_t*)a.err) & kErrNan) return;
  const uint32_t s = blockIdx.x;
  if ((a.fused_term || a.tss) && a.seg_term[s]) return;  // k_term_fused / the window sort own them
  const SegDesc sg = a.segs[s];
  const ModelDev md = a.models[s];
  segment_emit<kEThreads>(a, s, sg, md, os, reinterpret_cast<uint32_t*>(smraw));
}

template <bool TREE, int NT>
__device__ __forceinline__ void tree_top_to_smem(ModelDev& md, uint32_t k) {
  if constexpr (TREE) {  // top 8 levels of the splitter heap into smem
    __shared__ uint64_t s_top[256];
    if (md.kind == kModelTree)
      for (uint32_t j = threadIdx.x; j < min(k, 256u); j += NT) s_top[j] = md.heap[j];
    md.top = s_top;
    __syncthreads();
  }
}

template <bool F64, bool TREE>
__global__ __launch_bounds__(kSThreads, 1) void k_scatter_stable(LevelArgs a, uint64_t* __restrict__ dst_user,
                                                                 uint64_t* __restrict__ dst_scr) {
  const uint32_t c = blockIdx.x;
  const ChunkDesc ch = a.chunks[c];
  if (!a.single_offsets && a.seg_term[ch.seg]) return;  // k_scatter_term's chunk
  if (*((volatile const uint32_t*)a.err) & kErrNan) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  ModelDev md = a.models[ch.seg];
  tree_top_to_smem<TREE, kSThreads>(md, a.k);
  constexpr int kMain = TREE ? (int)kModelTree : (int)kModelLinear;
  if (md.kind == kModelEq3)
    scatter_stable_chunk<F64, kModelEq3>(a, dst_user, dst_scr, c, ch, md, smraw);
  else if (TREE && md.leaves != a.k)
    scatter_stable_chunk<F64, TREE ? (int)kModelTreeEq : kMain>(a, dst_user, dst_scr, c, ch, md, smraw);
  else
    scatter_stable_chunk<F64, kMain>(a, dst_user, dst_scr, c, ch, md, smraw);
}

// The stable scatter with per-bucket destinations (ipls_partition_scatter_to): one segment,
// every chunk stable, linear or EQ3 model.
template <bool F64>
__global__ __launch_bounds__(kSThreads, 1) void k_scatter_peer(LevelArgs a) {
  const uint32_t c = blockIdx.x;
  const ChunkDesc ch = a.chunks[c];
  extern __shared__ __align__(128) unsigned char smraw[];
  const ModelDev md = a.models[ch.seg];
  if (md.kind == kModelEq3)
    scatter_stable_chunk<F64, kModelEq3, true>(a, nullptr, nullptr, c, ch, md, smraw);
  else
    scatter_stable_chunk<F64, kModelLinear, true>(a, nullptr, nullptr, c, ch, md, smraw);
}

template <bool F64, bool TREE>
__global__ __launch_bounds__(kTThreads, 1) void k_scatter_term(LevelArgs a, uint64_t* __restrict__ dst_user,
                                                               uint64_t* __restrict__ dst_scr) {
  const uint32_t c = blockIdx.x;
  const ChunkDesc ch = a.chunks[c];
  if (a.single_offsets || !a.seg_term[ch.seg]) return;  // k_scatter_stable's chunk
  if (*((volatile const uint32_t*)a.err) & kErrNan) return;
  extern __shared__ __align__(128) unsigned char smraw[];
  ModelDev md = a.models[ch.seg];
  tree_top_to_smem<TREE, kTThreads>(md, a.k);
  constexpr int kMain = TREE ? (int)kModelTree : (int)kModelLinear;
  if (md.kind == kModelEq3)
    scatter_term_chunk<F64, kModelEq3>(a, dst_user, dst_scr, c, ch, md, smraw);
  else if (TREE && md.leaves != a.k)
    scatter_term_chunk<F64, TREE ? (int)kModelTreeEq : kMain>(a, dst_user, dst_scr, c, ch, md, smraw);
  else
    scatter_term_chunk<F64, kMain>(a, dst_user, dst_scr, c, ch, md, smraw);
}

// ------------------------------------------------------------------------------------
// Base case: sort windows of whole final segments (<= 4096 keys) by ordering key and
// write them to the user array.  Buckets are range-ordered (the model is monotone, R7), so
// sorting a window of consecutive final segments sorts each of them; any exact sort gives the
// identical bytes (R13).
//
// Two kernels: k_base_sort (windows of base children above kWBCap keys, one window per
// 512-thread CTA, keys in registers) and k_base_warp (windows of <= kWBCap keys, one per warp,
// below).
//
// Sort = interpolation sort in ordering-key space: a 256-bin coarse histogram of
// (ok - min) >> sh gives each coarse bin as many fine bins as it holds keys; the fine bin of
// a key is its coarse bin's first fine bin plus its fractional position inside the coarse bin
// times the coarse count (32-bit fraction, one IMAD.HI).  A counting pass places the keys bin
// by bin; every thread then insertion-sorts the contiguous range of its 8 fine bins (keys of
// different bins are already ordered, so only in-bin inversions move).  Windows whose fine
// bins overflow (> kFineOverflow keys: adversarial clusters) take a bitonic sort.

struct BaseSmem {
  uint32_t cinfo[256];   // coarse bin: first fine bin | count << 16
  uint64_t red[64];      // per-warp min, then per-warp max (<= 32 warps)
  uint32_t warp[40];
};

__device__ __forceinline__ uint32_t base_fine_bin(uint64_t d, int sh, const uint32_t* cinfo) {
  const uint32_t ci = cinfo[(uint32_t)(d >> sh)];
  uint32_t f = ci & 0xffffu;
  if (sh > 0) f += __umulhi((uint32_t)((d << (64 - sh)) >> 32), ci >> 16);
  return f;
}

// Window geometry for the bulk copy: keys [head, head + body) are 16-byte aligned in global
// memory and land at smem buf[2 ...]; the 0-1 keys before and after (head, tail) are loaded
// by thread 0 and stored around the body, so key i of the window sits at buf[2 - head + i].
struct WinGeom {
  uint32_t head, body, tail;
};
__device__ __forceinline__ WinGeom win_geom(const uint64_t* g, uint32_t len) {
  WinGeom w;
  w.head = ((reinterpret_cast<uintptr_t>(g) & 15u) != 0 && len > 0) ? 1u : 0u;
  w.body = (len - w.head) & ~1u;
  w.tail = len - w.head - w.body;
  return w;
}

// Sort the keys v[] (ordering keys; slots j*NT+tid < len valid) of one window.  On return
// the sorted (ok - min) values are in B[0, len) and `mn` holds min.  B: NT*ITEMS u64 smem;
// fh: NT*ITEMS u32 smem.  Ends with a barrier.
#ifdef IPLS_BASE_TIMING  // dev harness only: per-phase clock accumulation by thread 0
__device__ unsigned long long g_base_phase[16];
#define BASE_TICK(N)                                                         \
  do {                                                                       \
    if (threadIdx.x == 0) {                                                  \
      const long long t_ = clock64();                                        \
      atomicAdd(&g_base_phase[N], (unsigned long long)(t_ - t_prev_));       \
      t_prev_ = t_;                                                          \
    }                                                                        \
  } while (0)
#else
#define BASE_TICK(N)
#endif
template <int NT, int ITEMS>
__device__ uint64_t* sort_regs_to_smem(uint64_t (&v)[ITEMS], uint32_t len, uint64_t* B,
                                       uint32_t* fh, BaseSmem& ss, uint64_t& mn_out,
                                       long long& t_prev_) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint64_t mn = ~0ull, mx = 0ull;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (j * NT + threadIdx.x < len) { mn = min(mn, v[j]); mx = max(mx, v[j]); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) { ss.red[wp] = mn; ss.red[NW + wp] = mx; }
  for (uint32_t c = threadIdx.x; c < 256; c += NT) ss.cinfo[c] = 0u;
  {
    uint4* f4 = reinterpret_cast<uint4*>(fh + wb_phys(threadIdx.x * ITEMS));
#pragma unroll
    for (int q = 0; q < ITEMS / 4; ++q) f4[q] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  {
    uint64_t a = ss.red[lane & (NW - 1)], b = ss.red[NW + (lane & (NW - 1))];
#pragma unroll
    for (int o = NW / 2; o > 0; o >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    mn = a; mx = b;
  }
  BASE_TICK(2);
  mn_out = mn;
  if (mn == mx) {  // constant window: every key is mn
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (j * NT + threadIdx.x < len) B[j * NT + threadIdx.x] = 0;
    __syncthreads();
    return B;
  }
  const int bl = 64 - __clzll((long long)(mx - mn));
  const int sh = bl > 8 ? bl - 8 : 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    v[j] -= mn;  // v now holds ok - min
    if (j * NT + threadIdx.x < len) atomicAdd(&ss.cinfo[(uint32_t)(v[j] >> sh)], 1u);
  }
  __syncthreads();
  BASE_TICK(3);
  {
    uint32_t cc = 0;
    if (threadIdx.x < 256) cc = ss.cinfo[threadIdx.x];
    const uint32_t ex = block_exclusive_scan<NT>(cc, ss.warp, nullptr);
    if (threadIdx.x < 256) ss.cinfo[threadIdx.x] = ex | (cc << 16);
  }
  __syncthreads();
  BASE_TICK(4);
  // fine bin f's count is fh[wb_phys(f)]; the atomic returns the key's arrival rank in its
  // bin, so the placement needs no second atomic
  uint32_t fs[ITEMS];  // fine bin | rank << 16
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    fs[j] = 0;
    if (j * NT + threadIdx.x < len) {
      const uint32_t f = base_fine_bin(v[j], sh, ss.cinfo);
      fs[j] = f | (atomicAdd(&fh[wb_phys(f)], 1u) << 16);
    }
  }
  __syncthreads();
  BASE_TICK(5);
  // exclusive scan of the NT*ITEMS fine-bin counts: thread t owns bins [ITEMS t, ITEMS t + ITEMS)
  uint32_t mxc = 0, lo, hi;  // this thread's fine bins hold B[lo, hi) after placement
  {
    uint4* f4 = reinterpret_cast<uint4*>(fh + wb_phys(threadIdx.x * ITEMS));
    uint32_t sum = 0;
#pragma unroll
    for (int q = 0; q < ITEMS / 4; ++q) {
      const uint4 c = f4[q];
      sum += c.x + c.y + c.z + c.w;
      mxc = max(mxc, max(max(c.x, c.y), max(c.z, c.w)));
    }
    uint32_t run = block_exclusive_scan<NT>(sum, ss.warp, nullptr);
    lo = run;
    hi = run + sum;
#pragma unroll
    for (int q = 0; q < ITEMS / 4; ++q) {
      const uint4 c = f4[q];
      uint4 o;
      o.x = run; run += c.x;
      o.y = run; run += c.y;
      o.z = run; run += c.z;
      o.w = run; run += c.w;
      f4[q] = o;
    }
  }
  const bool overflow = __syncthreads_or(mxc > kFineOverflow) != 0;
  BASE_TICK(6);
  if (overflow) {
    // An overflowing fine bin that holds one value (duplicates) needs no sorting: every key
    // of a big bin is compared with one of them, stored at the bin's first slot.  Only bins
    // of different keys send the window to the bitonic fallback.
    constexpr uint32_t NB = NT * ITEMS;
    auto big_start = [&](uint32_t f) -> uint32_t {  // start of bin f if it is big, else ~0
      const uint32_t st = fh[wb_phys(f)], en = f + 1 < NB ? fh[wb_phys(f + 1)] : len;
      return en - st > kFineOverflow ? st : ~0u;
    };
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (j * NT + threadIdx.x < len) {
        const uint32_t st = big_start(fs[j] & 0xffffu);
        if (st != ~0u) B[st] = v[j];
      }
    __syncthreads();
    bool mixed = false;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (j * NT + threadIdx.x < len) {
        const uint32_t st = big_start(fs[j] & 0xffffu);
        if (st != ~0u && B[st] != v[j]) mixed = true;
      }
    if (__syncthreads_or(mixed)) {
#pragma unroll
      for (int j = 0; j < ITEMS; ++j)
        if (j * NT + threadIdx.x < len) B[j * NT + threadIdx.x] = v[j];
      bitonic_sort_smem<NT>(B, len);
      return B;
    }
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (j * NT + threadIdx.x < len) {
      B[fh[wb_phys(fs[j] & 0xffffu)] + (fs[j] >> 16)] = v[j];
    }
  }
  __syncthreads();
  BASE_TICK(7);
  // fine bin f occupies B[fh[wb_phys(f)], fh[wb_phys(f + 1)]) (the last one ends at len).
  constexpr uint32_t NBF = NT * ITEMS;
  auto bin_end = [&](uint32_t f) -> uint32_t { return f + 1 < NBF ? fh[wb_phys(f + 1)] : len; };
  uint32_t big = 0;  // this thread's fine bins above kFineOverflow keys (one value each)
  if (overflow) {
    uint32_t e0 = lo;
    for (int q = 0; q < ITEMS; ++q) {
      const uint32_t e1 = bin_end(threadIdx.x * ITEMS + q);
      big |= (e1 - e0 > kFineOverflow ? 1u : 0u) << q;
      e0 = e1;
    }
  }
  // B is ordered across fine bins: every thread insertion-sorts its range B[lo, hi) (only
  // in-bin inversions move; each key moves at most its bin's load - 1 places), cut around
  // its duplicate-only big bins.  The last two keys of the sorted prefix stay in registers
  // (pp <= prev): a key that moves by at most one place costs no branch; only a key below
  // both walks the prefix.
  uint32_t s0 = lo, msk = big;
  while (true) {
    uint32_t s1 = hi, nxt = 0;
    if (msk) {
      const uint32_t f = threadIdx.x * ITEMS + (__ffs(msk) - 1);
      s1 = fh[wb_phys(f)];
      nxt = bin_end(f);
    }
    if (s0 + 1 < s1) {
      uint64_t* q = B + s0;  // q[1] is the key being inserted
      uint64_t prev = q[0], pp = 0ull, nx = q[1];
#pragma unroll 2
      for (uint32_t i = s0 + 1; i < s1; ++i, ++q) {
        const uint64_t x = nx;
        nx = q[2];  // never written while x is inserted (may read past the piece: B has
                    // room, fh follows it)
        const bool lt = x < prev;
        const uint64_t m = max(pp, x);
        if (lt) {
          q[1] = prev;
          q[0] = m;
        }
        if (lt && x < pp) {  // rare: x belongs below pp (q[0] = pp already)
          uint64_t* r = q - 1;
          while (r > B + s0 && r[-1] > x) { r[0] = r[-1]; --r; }
          r[0] = x;
        }
        pp = lt ? m : prev;
        prev = lt ? prev : x;
      }
    }
    if (!msk) break;
    msk &= msk - 1;
    s0 = nxt;
  }
  __syncthreads();
  BASE_TICK(8);
  return B;
}

// One window of big base children (<= kBigCap keys) per CTA: 512 threads, 8 keys per thread
// in registers, 3 CTAs per SM (48 KB smem each), so one CTA's barriers and load latency
// overlap the others' work.

template <bool F64, bool NANCHK>
#ifndef IPLS_BS_OCC
#define IPLS_BS_OCC 3
#endif
__global__ __launch_bounds__(kBCThreads, IPLS_BS_OCC) void k_base_sort(
    const Window* __restrict__ wins, uint64_t* __restrict__ user, const uint64_t* __restrict__ scr,
    uint32_t* __restrict__ err) {
  constexpr int NT = kBCThreads, ITEMS = kBCItems;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* A = reinterpret_cast<uint64_t*>(smraw);           // kBigCap: placement array
  uint32_t* fh = reinterpret_cast<uint32_t*>(A + kBigCap);     // kBigCap
  __shared__ BaseSmem ss;
  long long t_prev_ = 0;
  const Window wv = wins[blockIdx.x];
  const uint32_t len = wv.len;
  if (len == 0) return;
  const uint64_t* g = (wv.buf ? scr : user) + wv.begin;
  uint64_t* dst = user + wv.begin;
  uint64_t v[ITEMS];
  bool nan_seen = false;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t i = j * NT + threadIdx.x;
    const uint64_t bits = (i < len) ? __ldcs(g + i) : 0ull;
    if (F64 && NANCHK) nan_seen |= isnan(__longlong_as_double((long long)bits));
    v[j] = ok_of<F64>(bits);
  }
  if (NANCHK) {
    if (__syncthreads_or(nan_seen)) {
      if (threadIdx.x == 0) atomicOr(err, kErrNan);
      return;  // the array is left untouched
    }
  }
  uint64_t mn;
  const uint64_t* out = sort_regs_to_smem<NT, ITEMS>(v, len, A, fh, ss, mn, t_prev_);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t i = j * NT + threadIdx.x;
    if (i < len) __stcs(dst + i, bits_of_ok<F64>(out[i] + mn));
  }
}

// ------------------------------------------------------------------------------------
// Base case for small windows (<= kWBCap keys): persistent warps, one window per warp at a
// time, no CTA barriers.  Each warp streams its next window into a second smem buffer with a
// TMA bulk copy (mbarrier completion) while it sorts the current one, so every SM keeps
// ~kWBWarps x 4 KB of loads in flight independently of the sorting work.  Windows are dealt
// round-robin to the warps of the grid (a contended global ticket per window would
// serialise at the L2).  Each lane holds kWBItems keys of the window in registers.
//
// Sort = interpolation sort on the raw keys.  Bin of a key = trunc((x - min) * nb / (max -
// min)) evaluated in binary64 (f64 keys directly, u64 keys through the exact difference
// x - min converted to double): every step is monotone, so bins are ordered.  Counting pass
// into smem, placement; the window is then ordered across bins and every lane insertion-sorts
// the contiguous range of its own bins.  Inside a window that does not reach zero all keys
// have one sign, so raw bits ^ (negative ? 0x7ff..f : 0) compared as u64 is the key order
// (applied at placement, undone at the write-out).  Windows that
// reach zero (they may mix -0.0 and +0.0), whose range is not finite (infinities, overflow)
// or whose bins overflow (> kFineOverflow keys: extreme skew) take an exact warp bitonic sort
// on ordering keys.

// exact warp bitonic sort of B[0, len) by ordering key (B has room for the next power of 2)
template <bool F64>
__device__ void warp_bitonic_ok(uint64_t* B, uint32_t len, int lane) {
  uint32_t NP = 32;
  while (NP < len) NP <<= 1;
  for (uint32_t i = len + lane; i < NP; i += 32) B[i] = ~0ull;  // ordering-key sentinel
  for (uint32_t i = lane; i < len; i += 32) B[i] = ok_of<F64>(B[i]);
  __syncwarp();
  for (uint32_t size = 2; size <= NP; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = lane; i < NP / 2; i += 32) {
        const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const uint64_t x = B[lo], y = B[hi];
        if ((x > y) == asc) { B[lo] = y; B[hi] = x; }
      }
      __syncwarp();
    }
  }
  for (uint32_t i = lane; i < len; i += 32) B[i] = bits_of_ok<F64>(B[i]);
  __syncwarp();
}

// One warp sorts the windows first, first + stride, ... < nwin of `wins` (its smem region:
// IN, bins; its two mbarriers, initialised by the caller; it_base: the number of windows the
// warp has taken through these mbarriers so far, which fixes their phase).
template <bool F64, bool WSMEM>
__device__ void base_warp_windows(const Window* __restrict__ wins, uint32_t first, uint32_t nwin,
                                  uint32_t stride, uint64_t* __restrict__ user,
                                  const uint64_t* __restrict__ scr, uint64_t* IN, uint32_t* bins,
                                  uint64_t* mbar, Window* dring, uint32_t& it_base) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = first, gstride = stride;
  // lane 0: start the copies of window wv into IN[b]: its 16-byte-aligned body by a TMA bulk
  // copy (mbar[b]), the 0-1 keys before and after it (head, tail) by 8-byte cp.async into the
  // slots around the body (lane 0's cp.async group of this iteration, complete by the next)
  auto issue = [&](const Window& wv, int b) {
    const uint64_t* g = (wv.buf ? scr : user) + wv.begin;
    const WinGeom gm = win_geom(g, wv.len);
    uint64_t* K = IN + (size_t)b * kWBStride + 2 - gm.head;
    if (gm.head) cp_async8(K, g);
    if (gm.tail) cp_async8(K + wv.len - 1, g + wv.len - 1);
    if (gm.body) {
      mbar_arrive_tx(&mbar[b], gm.body * 8u);
      bulk_g2s(IN + (size_t)b * kWBStride + 2, g + gm.head, gm.body * 8u, &mbar[b]);
    } else {
      mbar_arrive(&mbar[b]);
    }
  };
#ifdef IPLS_BASE_TIMING
  long long t_prev_ = clock64();
  unsigned long long acc_[10] = {0};
#define WB_TICK(N) do { const long long t_ = clock64(); acc_[N] += (unsigned long long)(t_ - t_prev_); t_prev_ = t_; } while (0)
#else
#define WB_TICK(N)
#endif
  // Descriptors: WSMEM (k_term_fused's window list in shared memory) are read in place;
  // global ones go through a per-warp ring of 4 smem slots, fetched by cp.async two windows
  // ahead (slot it & 3: the current window, it + 1: the one being issued, it + 2: in flight),
  // so no lane holds descriptors in registers.
  uint32_t it = it_base;
  if (lane == 0 && gw < nwin) {
    Window w0;
    if constexpr (WSMEM) {
      w0 = wins[gw];
    } else {
      w0 = wins[gw];
      dring[it & 3] = w0;
      if (gw + gstride < nwin) cp_async16(&dring[(it + 1) & 3], &wins[gw + gstride]);
    }
    issue(w0, it & 1);
    cp_async_commit();
  }
  for (uint32_t cur = gw; cur < nwin; ++it, cur += gstride) {
    const int b = it & 1;
    if (lane == 0) {
      cp_async_wait_all();  // head/tail of window cur, descriptor of cur + stride
      if (cur + gstride < nwin) {
        if constexpr (WSMEM) {
          issue(wins[cur + gstride], b ^ 1);
        } else {
          issue(dring[(it + 1) & 3], b ^ 1);
          if (cur + 2 * gstride < nwin) cp_async16(&dring[(it + 2) & 3], &wins[cur + 2 * gstride]);
        }
      }
      cp_async_commit();
    }
    __syncwarp();
    Window wv;
    if constexpr (WSMEM) wv = wins[cur];
    else wv = dring[it & 3];
    WB_TICK(0);
    const uint32_t len = wv.len;
    const uint64_t* src = (wv.buf ? scr : user) + wv.begin;
    uint64_t* dst = user + wv.begin;
    const WinGeom gm = win_geom(src, len);
    uint64_t* INb = IN + (size_t)b * kWBStride;
    uint64_t* K = INb + 2 - gm.head;  // key i of the window
    uint64_t* B = INb;                // placement array once the keys are in registers
    mbar_wait(&mbar[b], (it >> 1) & 1);
    __syncwarp();
    // Slots past the end hold a copy of key 0 so that the bounds need no predicate.
    uint64_t v[kWBItems];
    {
      const uint64_t k0 = K[0];
#pragma unroll
      for (int j = 0; j < kWBItems; ++j) {
        const uint32_t i = j * 32 + lane;
        v[j] = (i < len) ? K[i] : k0;
      }
    }
    WB_TICK(1);
    // ---- bounds (no NaN reaches the base case: R0) ----
    double mn = 0.0, range;
    uint64_t umn = v[0], umx = v[0];
    uint64_t flip = 0;  // ordering of raw bits inside a one-signed window: (bits ^ flip) as u64
    if constexpr (F64) {
      double mx = __longlong_as_double((long long)v[0]);
      mn = mx;
#pragma unroll
      for (int j = 1; j < kWBItems; ++j) {
        const double x = __longlong_as_double((long long)v[j]);
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
      }
      range = mx - mn;
      // a window reaching zero (it may mix -0.0 and +0.0) takes the exact path below
      if (mn <= 0.0 && mx >= 0.0) range = 0.0;
      flip = mx < 0.0 ? 0x7fffffffffffffffull : 0ull;
    } else {
#pragma unroll
      for (int j = 1; j < kWBItems; ++j) {
        umn = min(umn, v[j]);
        umx = max(umx, v[j]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        umn = min(umn, __shfl_xor_sync(0xffffffffu, umn, o));
        umx = max(umx, __shfl_xor_sync(0xffffffffu, umx, o));
      }
      range = (double)(umx - umn);
    }
    const uint64_t* OUT = K;  // constant windows (one bit pattern) are already sorted
    uint64_t oflip = 0;       // OUT holds bits ^ oflip
    WB_TICK(2);
    bool constant = !F64 && umn == umx;
    if (F64 && range == 0.0) {  // one value, but it may mix -0.0 and +0.0: compare the bits
      const uint64_t v00 = __shfl_sync(0xffffffffu, v[0], 0);  // every lane (not short-circuited)
      bool same = true;
#pragma unroll
      for (int j = 0; j < kWBItems; ++j) same &= v[j] == v00;
      constant = __all_sync(0xffffffffu, same);
    }
    if (constant) {
      // nothing to sort
    } else if (!(range > 0.0) || !(range < 1.79e308)) {  // zero inside, infinities, overflow
      __syncwarp();  // every lane holds its keys: B may overwrite K
#pragma unroll
      for (int j = 0; j < kWBItems; ++j)
        if (j * 32 + lane < len) B[j * 32 + lane] = v[j];
      __syncwarp();
      warp_bitonic_ok<F64>(B, len, lane);
      OUT = B;
    } else {
      const uint32_t nb = kWBBinsPerKey * len;
      const double scale = (double)nb / range;
      // Bin f lives at bins[f + 4 (f / 32)]: lane l's 16 bins are one 16-byte-aligned run, and
      // the 8 lanes of a quarter-warp start on distinct 16-byte bank groups (conflict-free
      // LDS.128 / STS.128 in the scan).
      {
        uint4* b4 = reinterpret_cast<uint4*>(bins);
        for (uint32_t q = lane; q < (uint32_t)kWBBinWords / 4; q += 32) b4[q] = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      // histogram; the atomic's return is the key's arrival rank in its bin
      uint32_t fr[kWBItems];  // bin | rank << 16
#pragma unroll
      for (int j = 0; j < kWBItems; ++j) {
        fr[j] = 0;
        if (j * 32 + lane < len) {
          double y;
          if constexpr (F64) y = __longlong_as_double((long long)v[j]) - mn;
          else y = (double)(v[j] - umn);
          const uint32_t fb = min(__double2uint_rz(y * scale), nb - 1);
          const uint32_t r = atomicAdd(&bins[wb_phys(fb)], 1u);
          fr[j] = fb | (r << 16);
        }
      }
      __syncwarp();
      // exclusive scan: lane l owns bins [16 l, 16 l + 16); counts -> starts in place
      uint32_t mxc = 0, multi = 0;  // largest count; bins of this lane with 2..kFineOverflow keys
      {
        uint4* lb = reinterpret_cast<uint4*>(bins + wb_phys(lane * kWBBpl));
        uint4 c[kWBBpl / 4];
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < kWBBpl / 4; ++q) {
          c[q] = lb[q];
          const uint32_t cs[4] = {c[q].x, c[q].y, c[q].z, c[q].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            sum += cs[e];
            mxc = max(mxc, cs[e]);
            multi |= (cs[e] >= 2u && cs[e] <= kFineOverflow ? 1u : 0u) << (4 * q + e);
          }
        }
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        uint32_t run = inc - sum;
#pragma unroll
        for (int q = 0; q < kWBBpl / 4; ++q) {
          uint4 o;
          o.x = run; run += c[q].x;
          o.y = run; run += c[q].y;
          o.z = run; run += c[q].z;
          o.w = run; run += c[q].w;
          lb[q] = o;
        }
      }
      const bool overflow = __any_sync(0xffffffffu, mxc > kFineOverflow);
      __syncwarp();
      // placement: bin start + arrival rank, in u64 key order (bits ^ flip)
#pragma unroll
      for (int j = 0; j < kWBItems; ++j)
        if (j * 32 + lane < len) B[bins[wb_phys(fr[j] & 0xffffu)] + (fr[j] >> 16)] = v[j] ^ flip;
      __syncwarp();
      // A bin above kFineOverflow keys that holds one value (duplicates) needs no sorting;
      // bins of different keys above it send the window to the bitonic sort.
      bool mixed = false;
      if (overflow) {
#pragma unroll
        for (int j = 0; j < kWBItems; ++j) {
          if (j * 32 + lane < len) {
            const uint32_t f = fr[j] & 0xffffu;
            const uint32_t b0 = bins[wb_phys(f)], b1 = f + 1 < nb ? bins[wb_phys(f + 1)] : len;
            if (b1 - b0 > kFineOverflow && (v[j] ^ flip) != B[b0]) mixed = true;
          }
        }
        mixed = __any_sync(0xffffffffu, mixed);
      }
      if (mixed) {
        for (uint32_t i = lane; i < len; i += 32) B[i] ^= flip;
        __syncwarp();
        warp_bitonic_ok<F64>(B, len, lane);
        OUT = B;
      } else {
        // B is ordered across bins; inside a bin the order is the atomics' arrival order.
        // Every lane insertion-sorts its own bins of 2..kFineOverflow keys (~1.4 per lane at
        // 2 bins per key), reading each bin's start back from the scan.
        while (multi) {
          const int jb = __ffs(multi) - 1;
          multi &= multi - 1;
          const uint32_t f = lane * kWBBpl + jb;
          const uint32_t s = bins[wb_phys(f)];
          const uint32_t e = f + 1 < nb ? bins[wb_phys(f + 1)] : len;
          uint64_t* q = B + s;
          if (e - s == 2) {  // ~70 % of the multi-key bins at 2 bins per key
            const uint64_t x0 = q[0], x1 = q[1];
            if (x0 > x1) { q[0] = x1; q[1] = x0; }
          } else {
            for (uint32_t i = 1; i < e - s; ++i) {
              const uint64_t x = q[i];
              uint32_t m = i;
              while (m > 0 && q[m - 1] > x) { q[m] = q[m - 1]; --m; }
              q[m] = x;
            }
          }
        }
        oflip = flip;
        OUT = B;
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kWBItems; ++j) v[j] = OUT[j * 32 + lane] ^ oflip;
#pragma unroll
    for (int j = 0; j < kWBItems; ++j)
      if (j * 32 + lane < len) __stcs(dst + j * 32 + lane, v[j]);
    WB_TICK(8);
    fence_proxy_async_smem();  // generic accesses to IN[b] before the bulk copy that reuses it
    __syncwarp();
  }
  it_base = it;
#ifdef IPLS_BASE_TIMING
  if (lane == 0)
    for (int q = 0; q < 10; ++q) atomicAdd(&g_base_phase[q], acc_[q]);
#endif
}

template <bool F64>
__global__ __launch_bounds__(kWBWarps * 32, 1) void k_base_warp(
    const Window* __restrict__ wins, uint32_t nwin, uint64_t* __restrict__ user,
    const uint64_t* __restrict__ scr) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint64_t s_mbar[kWBWarps][2];
  __shared__ __align__(16) Window s_dring[kWBWarps][4];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint64_t* IN = reinterpret_cast<uint64_t*>(smraw + wp * kWBSmemPerWarp);  // 2 x kWBStride
  uint32_t* bins = reinterpret_cast<uint32_t*>(IN + 2 * kWBStride);          // kWBBinWords
  uint64_t* mbar = s_mbar[wp];
  if (lane == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t it = 0;
  base_warp_windows<F64, false>(wins, blockIdx.x * kWBWarps + wp, nwin, gridDim.x * kWBWarps, user,
                                scr, IN, bins, mbar, s_dring[wp], it);
}

// ------------------------------------------------------------------------------------
// Last partition level fused with the base case (P:136-142, P:708,
// P:725).  Persistent CTAs (one per SM, 1024 threads) take the level's terminal chunks by
// ticket and scatter each one (scatter_term_chunk).  The CTA that completes a segment's last
// chunk then base-sorts that segment's children itself, right away, while they are still in
// the L2 (the level's data in flight at any time is ~148 chunks): it packs the children of
// <= kWBCap keys into windows (pack_windows, into shared memory) and its 32 warps sort them
// (base_warp_windows, the k_base_warp code); children above kWBCap become windows of
// k_base_sort, launched after the level.  Terminal segments get no segment_emit (k_emit skips
// them) and no k_base_warp windows.  Shared memory: the scatter's tile ring, then the base
// warps' regions plus the segment's window list.
constexpr size_t kFusedListOff = kWBSmemPerWarp * kWBWarps;  // window list after the warps
constexpr size_t fused_smem_bytes(uint32_t k) {
  return (kFusedListOff + (size_t)kMaxK * sizeof(Window)) > scatter_term_smem_bytes(k)
             ? kFusedListOff + (size_t)kMaxK * sizeof(Window)
             : scatter_term_smem_bytes(k);
}
static_assert(kWBWarps * 32 == kTThreads, "the fused kernel's warps are the base warps");
constexpr uint32_t kFusedMaxM = 262144;  // larger segments: windows to k_base_warp

template <bool F64, bool TREE>
__global__ __launch_bounds__(kTThreads, 1) void k_term_fused(LevelArgs a, uint64_t* __restrict__ dst_user,
                                                             uint64_t* __restrict__ dst_scr,
                                                             uint32_t nchunk) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint64_t s_mbar[kWBWarps][2];
  __shared__ OffSmem os;
  __shared__ uint32_t s_ticket[2], s_last, s_nw;
  __shared__ uint64_t s_keys;
  const uint32_t t = threadIdx.x;
  const int lane = t & 31, wp = t >> 5;
  uint64_t* IN = reinterpret_cast<uint64_t*>(smraw + wp * kWBSmemPerWarp);
  uint32_t* bins = reinterpret_cast<uint32_t*>(IN + 2 * kWBStride);
  Window* list = reinterpret_cast<Window*>(smraw + kFusedListOff);
  if (lane == 0) {
    mbar_init(&s_mbar[wp][0], 1);
    mbar_init(&s_mbar[wp][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t it_base = 0;  // windows this warp has sorted (mbarrier phase)
  const uint32_t k = a.k;
  if (*((volatile const uint32_t*)a.err) & kErrNan) return;
  // Chunk tickets are taken one chunk ahead (s_ticket[ip & 1] is this chunk's, thread 0 fills
  // the other slot early in the chunk), so the ticket's L2 round trip overlaps the chunk's
  // first tile load instead of stalling the whole CTA between chunks.
  if (t == 0) s_ticket[0] = atomicAdd(&a.nctr->sticket, 1u);
  for (uint32_t ip = 0;; ++ip) {
    __syncthreads();
    const uint32_t c = s_ticket[ip & 1];
    if (c >= nchunk) break;
    uint32_t* next_ticket = &s_ticket[(ip + 1) & 1];
    const ChunkDesc ch = a.chunks[c];
    if (!a.seg_term[ch.seg]) {  // k_scatter_stable's chunk
      if (t == 0) *next_ticket = atomicAdd(&a.nctr->sticket, 1u);
      continue;
    }
    ModelDev md = a.models[ch.seg];
    tree_top_to_smem<TREE, kTThreads>(md, k);
    constexpr int kMain = TREE ? (int)kModelTree : (int)kModelLinear;
    if (md.kind == kModelEq3)
      scatter_term_chunk<F64, kModelEq3>(a, dst_user, dst_scr, c, ch, md, smraw, next_ticket);
    else if (TREE && md.leaves != k)
      scatter_term_chunk<F64, TREE ? (int)kModelTreeEq : kMain>(a, dst_user, dst_scr, c, ch, md, smraw,
                                                                next_ticket);
    else
      scatter_term_chunk<F64, kMain>(a, dst_user, dst_scr, c, ch, md, smraw, next_ticket);
    // this chunk's stores are visible before it counts; the last one reads them all
    __threadfence();
    __syncthreads();
    const SegDesc sg = a.segs[ch.seg];
    if (sg.nchunks > 1) {  // block-uniform; a one-chunk segment is complete here
      if (t == 0) s_last = (atomicAdd(&a.seg_done[ch.seg], 1u) == sg.nchunks - 1) ? 1u : 0u;
      __syncthreads();
      if (!s_last) continue;
      __threadfence();
    }
    // ---- the segment's windows (thread t owns child t) ----
    const uint32_t b = t;
    const uint32_t tot = (b < k) ? a.seg_tot[(size_t)ch.seg * k + b] : 0u;
    const uint32_t base = (b < k) ? (uint32_t)((a.seg_dst[(size_t)ch.seg * k + b] & ~kDstUserBit) - sg.begin) : 0u;
    const uint32_t dstbuf = a.dstbuf;
    if (t == 0) { s_nw = 0; s_keys = 0; }
    __syncthreads();
    // Once the chunk tickets have run out, the remaining segments complete at the very end
    // of the kernel; sorting them here would leave most SMs idle behind a few CTAs, so their
    // windows go to the level's k_base_warp launch instead (all SMs).
    // Likewise a segment above kFusedMaxM keys: one CTA would hold it long after the others.
    if (t == 0) s_last = *((volatile const uint32_t*)&a.nctr->sticket) >= nchunk || sg.m > kFusedMaxM;
    __syncthreads();
    const bool tail = s_last != 0;  // block-uniform
    {
      const uint32_t bb[1] = {b < k ? b : k}, bs[1] = {base}, tt[1] = {tot};
      const bool small[1] = {b < k && tot > 0 && tot <= (uint32_t)kWBCap};
      const bool big[1] = {b < k && tot > (uint32_t)kWBCap};
      if (tail)
        pack_windows<kTThreads>(a, sg, k, bb, bs, tt, small, (uint32_t)kWBCap, dstbuf, os,
                                reinterpret_cast<uint32_t*>(smraw), a.wins, a.cap_wins,
                                &a.nctr->n_windows, &a.nctr->win_keys);
      else
        pack_windows<kTThreads>(a, sg, k, bb, bs, tt, small, (uint32_t)kWBCap, dstbuf, os,
                                reinterpret_cast<uint32_t*>(smraw), list, kMaxK, &s_nw, &s_keys);
      // children above kWBCap: windows of <= kBigCap keys for k_base_sort, after the level
      pack_windows<kTThreads>(a, sg, k, bb, bs, tt, big, (uint32_t)kBigCap, dstbuf, os,
                              reinterpret_cast<uint32_t*>(smraw), a.wins_big, a.cap_wbig,
                              &a.nctr->n_wbig, &a.nctr->wbig_keys);
    }
    if (tail) continue;
    fence_proxy_async_smem();  // generic accesses (stage, scratch) before the warps' bulk loads
    __syncthreads();
    if (t == 0) atomicAdd((unsigned long long*)&a.nctr->term_keys, (unsigned long long)s_keys);
    base_warp_windows<F64, true>(list, wp, s_nw, kWBWarps, dst_user, dst_scr, IN, bins, s_mbar[wp],
                                 nullptr, it_base);
    fence_proxy_async_smem();  // and before the next chunk's tile ring
  }
}

__global__ void k_fill(const Fill* __restrict__ fills, uint64_t* __restrict__ user) {
  const Fill f = fills[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < f.len; i += blockDim.x) user[f.begin + i] = f.value;
}

// Trace only: snapshot of the array image after a level (segments of this level copied
// from the buffer they were scattered into).
__global__ void k_snapshot(const SegDesc* __restrict__ segs, const uint64_t* __restrict__ user,
                           const uint64_t* __restrict__ scr, uint32_t dstbuf,
                           uint64_t* __restrict__ snap) {
  const SegDesc sg = segs[blockIdx.x];
  const uint64_t* s = (dstbuf ? scr : user) + sg.begin;
  for (uint32_t i = threadIdx.x; i < sg.m; i += blockDim.x) snap[sg.begin + i] = s[i];
}

// Trace only: a terminal segment's image after its level is its sorted keys (k_win_sort's
// output in the user array): every child holds its multiset there.
__global__ void k_snapshot_term(const SegDesc* __restrict__ segs, const uint32_t* __restrict__ seg_term,
                                const uint64_t* __restrict__ user, uint64_t* __restrict__ snap) {
  if (!seg_term[blockIdx.x]) return;
  const SegDesc sg = segs[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < sg.m; i += blockDim.x) snap[sg.begin + i] = user[sg.begin + i];
}

// ipls_regroup_runs: move pieces (src offset, dst offset, length) of keys, one warp per piece,
// coalesced (the multi-GPU exchange's G received runs into bucket-major order).
struct Piece {
  uint64_t src, dst;
  uint64_t len;
};
__global__ void k_move_pieces(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                              const Piece* __restrict__ pieces, uint32_t npieces) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < npieces;
       w += (gridDim.x * blockDim.x) >> 5) {
    const Piece pc = pieces[w];
    for (uint64_t i = lane; i < pc.len; i += 32) dst[pc.dst + i] = __ldcs(src + pc.src + i);
  }
}

// ipls_sort_segments (f64): any NaN rejects the input before anything is written (R0).
__global__ void k_nan_scan(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ err) {
  int nan = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    nan |= isnan(__longlong_as_double((long long)__ldcs(keys + i)));
  if (__syncthreads_or(nan) && threadIdx.x == 0) atomicOr(err, kErrNan);
}

__global__ void k_keys_to_ok(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                             uint32_t n, int f64) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = f64 ? ok_of_f64(in[i]) : in[i];
}

// Distributed top level: the level-0 stratified sample
// (R2, R18) of a global array of m keys of which this rank holds positions
// [gbegin, gbegin + n).  Thread j computes stratum j's position exactly as the fit kernels do
// for the root segment (level 0, begin 0) and copies the key if this rank holds it, so the
// ranks' outputs, summed, are the sample a one-GPU sort of the concatenation draws.
__global__ void k_sample_strata(const uint64_t* __restrict__ keys, uint64_t n, uint64_t gbegin,
                                uint64_t m, uint32_t S, uint64_t seed,
                                uint64_t* __restrict__ out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S) return;
  const uint64_t t = sm64(sm64(sm64(seed) ^ 0ull) ^ 0ull);
  const uint64_t lo = (uint64_t)j * m / S, hi = (uint64_t)(j + 1) * m / S;
  const uint64_t idx = lo + __umul64hi(sm64(t ^ (uint64_t)j), hi - lo);
  if (idx >= gbegin && idx - gbegin < n) out[j] = keys[idx - gbegin];
}

}  // namespace ipls
