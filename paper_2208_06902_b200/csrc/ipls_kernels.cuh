// ipls_kernels.cuh — sm_100a kernels of one IPLS distribution level and the base case.
//
// Per level (the four phases of P:265-287), three launches:
//   k_gather_fit      phase 1-3: stratified sample of every segment (R2, R18),
//                     smem sort of the sample, FMCD fit (Listing 1)
//   k_classify_scan   phase 4a: model eval + smem histogram per chunk, NaN flag,
//                     homogeneity (R9), decoupled-lookback prefix of the
//                     (chunk x bucket) counts; the last chunk of each segment computes the
//                     bucket bases, child classes (R20), next-level work, base-case windows
//   k_scatter         phase 4b: stable in-tile rank (smem bitmap multisplit), smem staging by
//                     bucket, run-contiguous writes (R11)
// After the level: k_base_sort (base case) and k_fill.
#pragma once
#include "ipls_device.cuh"

namespace ipls {

constexpr int kCThreads = 512;                 // classify
constexpr int kCItems = 8;
constexpr int kCTile = kCThreads * kCItems;    // 4096
constexpr int kSThreads = 256;                 // scatter
constexpr int kSWarps = kSThreads / 32;        // 8
constexpr int kSRounds = 16;  // keys per thread per tile
constexpr int kSTile = kSThreads * kSRounds;   // 4096
constexpr int kFitThreads = 1024;
constexpr int kFitMaxS = 8192;
constexpr int kBaseThreads = 512;
constexpr int kBaseMax = 8192;                 // keys per base-case window (W + B)
constexpr uint32_t kWindowNominal = 4096;
constexpr uint32_t kMaxK = 1024;
constexpr uint32_t kFineOverflow = 32;          // fine-bin load that triggers the bitonic fallback

// ------------------------------------------------------------------------------------
// Block-wide exact sort of n <= cap ordering keys in smem (used for samples and base-case
// windows).  A 256-way coarse histogram of (ok - min) >> shift allots each coarse bin as
// many fine bins as it holds keys; a fine counting sort leaves runs of ~1 key that an
// insertion sort finishes.  Inputs whose fine bins overflow take a bitonic sort instead.
// Any exact sort yields the identical bytes, so the method is free (R13).
struct SortSmem {
  uint32_t ccnt[256];
  uint32_t coff[256];
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
  if (__syncthreads_or(mxc > kFineOverflow)) {
    bitonic_sort_smem<NT>(a, n);
    return;
  }
  for (uint32_t i = threadIdx.x; i < n; i += NT) {
    uint64_t v = a[i];
    uint32_t pos = atomicAdd(&fh[fine_bin(v, mn, sh, ss.coff, ss.ccnt)], 1u);
    tmp[pos] = v;
  }
  __syncthreads();
  for (uint32_t f = threadIdx.x; f < n; f += NT) {
    uint32_t beg = f ? fh[f - 1] : 0u, end = fh[f];
    for (uint32_t i = beg + 1; i < end; ++i) {
      uint64_t x = tmp[i];
      uint32_t j = i;
      while (j > beg && tmp[j - 1] > x) { tmp[j] = tmp[j - 1]; --j; }
      tmp[j] = x;
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

template <bool F64>
__global__ __launch_bounds__(kFitThreads) void k_gather_fit(
    const uint64_t* __restrict__ src, const SegDesc* __restrict__ segs, uint64_t seed,
    uint32_t level, uint32_t k, uint32_t cap, uint64_t* __restrict__ samples_out,
    ModelDev* __restrict__ models, const uint64_t* __restrict__ presorted_ok) {
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* a = reinterpret_cast<uint64_t*>(smraw);   // cap
  uint64_t* tmp = a + cap;                             // cap
  uint32_t* fh = reinterpret_cast<uint32_t*>(tmp + cap);  // cap
  __shared__ SortSmem ss;
  __shared__ uint64_t s_pivot;
  const SegDesc sg = segs[blockIdx.x];
  const uint32_t S = sg.S;
  if (presorted_ok) {
    for (uint32_t j = threadIdx.x; j < S; j += kFitThreads) a[j] = presorted_ok[j];
    __syncthreads();
  } else {
    const uint64_t t = sm64(sm64(sm64(seed) ^ (uint64_t)level) ^ sg.begin);
    const uint64_t m = sg.m;
    for (uint32_t j = threadIdx.x; j < S; j += kFitThreads) {
      uint64_t lo = ((uint64_t)j * m) / S;
      uint64_t hi = ((uint64_t)(j + 1) * m) / S;
      uint64_t h = sm64(t ^ (uint64_t)j);
      uint64_t idx = sg.begin + lo + __umul64hi(h, hi - lo);
      a[j] = ok_of<F64>(__ldg(src + idx));
    }
    __syncthreads();
    block_sort_ok<kFitThreads>(a, tmp, fh, S, ss);
  }
  if (samples_out)
    for (uint32_t j = threadIdx.x; j < S; j += kFitThreads) samples_out[sg.sample_off + j] = a[j];
  if (threadIdx.x == 0) s_pivot = a[S / 2];
  __syncthreads();
  ModelDev md{};
  md.k_eff = k;
  bool eq3 = (sg.flags & kSegForceEq3) || S < 4;
  if (!eq3) {
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
  uint32_t* ticket;
  uint64_t* status;      // [chunk][k]: epoch<<48 | state<<46 | inh<<45 | count
  uint32_t* cnt_agg;     // [chunk][k]: own count | inh<<31
  uint64_t* rep_agg;     // [chunk][k]: own representative key
  uint32_t* chunk_pre;   // [chunk][k] exclusive prefix within the segment
  uint64_t* seg_dst;     // [seg][k]   encoded destination base of every child
  uint32_t* seg_tot;     // [seg][k]   child counts (trace)
  uint32_t epoch;
  uint32_t* err;
  int check_nan;
  uint16_t* ids;         // partition_level only: per-key buckets
  uint64_t* single_offsets;  // partition_level only: k_eff+1 bucket boundaries
  SegDesc* nsegs;
  ChunkDesc* nchunks;
  LevelCounters* nctr;
  uint32_t cap_segs, cap_chunks, cap_samples;
  Window* wins;
  uint32_t cap_wins;
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


__device__ void emit_segment(const LevelArgs& a, uint64_t begin, uint32_t m, uint32_t flags,
                             uint32_t seg_idx, uint32_t samp_off, uint32_t ch_off) {
  SegDesc sd{};
  sd.begin = begin; sd.m = m; sd.S = sample_size(m, a.k); sd.sample_off = samp_off;
  uint32_t nch = (m + a.chunk_keys - 1) / a.chunk_keys;
  sd.chunk_first = ch_off; sd.nchunks = nch; sd.flags = flags;
  a.nsegs[seg_idx] = sd;
  atomicMax(&a.nctr->max_S, sd.S);
  for (uint32_t j = 0; j < nch; ++j) {
    ChunkDesc cd;
    cd.start = begin + (uint64_t)j * a.chunk_keys;
    cd.len = min(a.chunk_keys, m - j * a.chunk_keys);
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
  uint32_t basey[kMaxK];
  uint32_t wid[kMaxK];
  uint32_t wbeg[kMaxK];
  uint32_t wend[kMaxK];
};

__device__ void segment_offsets(const LevelArgs& a, uint32_t s, const SegDesc& sg,
                                const ModelDev& md, const uint32_t (&tot)[kCBpt],
                                const uint32_t (&inh)[kCBpt], const uint64_t (&rep)[kCBpt],
                                OffSmem& os) {
  const uint32_t k = a.k;
  uint32_t bb[kCBpt], base[kCBpt];
  uint32_t x = 0;
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) { bb[q] = threadIdx.x * kCBpt + q; x += tot[q]; }
  uint32_t ex = block_exclusive_scan<kCThreads>(x, os.warp, nullptr);
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) { base[q] = ex; ex += tot[q]; }
  int st = 0;
#pragma unroll
  for (int q = 0; q < kCBpt; ++q)
    if (md.kind == kModelLinear && bb[q] < k && tot[q] == sg.m) st = 1;
  const bool stuck = __syncthreads_or(st) != 0;
  const uint32_t dstbuf = (a.level + 1) & 1;  // 1 = scratch, 0 = user array
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    if (bb[q] < k) {
      uint64_t enc = a.single_offsets ? (uint64_t)base[q]
                                      : ((dstbuf == 0 ? kDstUserBit : 0ull) | (sg.begin + base[q]));
      a.seg_dst[(size_t)s * k + bb[q]] = enc;
      if (a.seg_tot) a.seg_tot[(size_t)s * k + bb[q]] = tot[q];
    }
  }
  if (a.single_offsets) {
#pragma unroll
    for (int q = 0; q < kCBpt; ++q)
      if (bb[q] < md.k_eff) a.single_offsets[bb[q]] = base[q];
    if (threadIdx.x == 0) a.single_offsets[md.k_eff] = sg.m;
    return;
  }
  uint32_t cls[kCBpt];
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    cls[q] = 0;  // 0 empty, 1 base (or small homogeneous), 2 partition, 3 big homogeneous
    if (!stuck && bb[q] < k && tot[q] > 0) {
      bool homog = (md.kind == kModelEq3 && bb[q] == 1) || !inh[q];
      if (tot[q] <= a.base_case) cls[q] = 1;
      else if (homog) cls[q] = 3;
      else cls[q] = 2;
    }
  }
  // ---- next-level segments ----
  uint32_t w_seg = 0, w_samp = 0, w_ch = 0;
  uint32_t cm[kCBpt];
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    cm[q] = 0;
    if (stuck) { if (threadIdx.x == 0 && q == 0) cm[q] = sg.m; }
    else if (cls[q] == 2) cm[q] = tot[q];
    if (cm[q]) {
      w_seg += 1;
      w_samp += sample_size(cm[q], k);
      w_ch += (cm[q] + a.chunk_keys - 1) / a.chunk_keys;
    }
  }
  uint32_t t_seg, t_samp, t_ch;
  uint32_t o_seg = block_exclusive_scan<kCThreads>(w_seg, os.warp, &t_seg);
  uint32_t o_samp = block_exclusive_scan<kCThreads>(w_samp, os.warp, &t_samp);
  uint32_t o_ch = block_exclusive_scan<kCThreads>(w_ch, os.warp, &t_ch);
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
#pragma unroll
      for (int q = 0; q < kCBpt; ++q) {
        if (cm[q]) {
          uint64_t cb = stuck ? sg.begin : sg.begin + base[q];
          emit_segment(a, cb, cm[q], stuck ? kSegForceEq3 : 0u, i_seg, i_samp, i_ch);
          atomicAdd((unsigned long long*)&a.nctr->keys, (unsigned long long)cm[q]);
          i_seg += 1;
          i_samp += sample_size(cm[q], k);
          i_ch += (cm[q] + a.chunk_keys - 1) / a.chunk_keys;
        }
      }
    }
  }
  if (stuck) return;  // block-uniform
  // ---- base-case windows: maximal runs of base/empty children within one W-window ----
  bool basey[kCBpt];
  uint32_t wid[kCBpt];
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    basey[q] = (bb[q] < k) && (cls[q] <= 1);
    wid[q] = base[q] / kWindowNominal;
    if (bb[q] < k) { os.basey[bb[q]] = basey[q]; os.wid[bb[q]] = wid[q]; }
  }
  __syncthreads();
  uint32_t start[kCBpt], nst = 0;
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    start[q] = 0;
    if (basey[q])
      start[q] = (bb[q] == 0) || !os.basey[bb[q] - 1] || os.wid[bb[q] - 1] != wid[q];
    nst += start[q];
  }
  uint32_t t_win;
  uint32_t o_win = block_exclusive_scan<kCThreads>(nst, os.warp, &t_win);
  uint32_t widx[kCBpt];
  {
    uint32_t run = o_win;
#pragma unroll
    for (int q = 0; q < kCBpt; ++q) {
      run += start[q];
      widx[q] = run - 1;
      if (start[q]) { os.wbeg[widx[q]] = base[q]; os.wend[widx[q]] = base[q]; }
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kCBpt; ++q)
    if (basey[q] && tot[q]) atomicMax(&os.wend[widx[q]], base[q] + tot[q]);
  if (threadIdx.x == 0 && t_win) os.res[4] = atomicAdd(&a.nctr->n_windows, t_win);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    if (start[q]) {
      uint32_t gi = os.res[4] + widx[q];
      if (gi < a.cap_wins) {
        Window wv;
        wv.begin = sg.begin + os.wbeg[widx[q]];
        wv.len = os.wend[widx[q]] - os.wbeg[widx[q]];
        wv.buf = dstbuf;
        a.wins[gi] = wv;
        if (wv.len) atomicAdd((unsigned long long*)&a.nctr->win_keys, (unsigned long long)wv.len);
      } else {
        atomicOr(a.err, kErrOverflow);
      }
    }
  }
  // ---- homogeneous children that land in scratch must be filled into the user array ----
  uint32_t nf = 0;
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) nf += (cls[q] == 3 && dstbuf == 1) ? 1u : 0u;
  uint32_t t_fill;
  uint32_t o_fill = block_exclusive_scan<kCThreads>(nf, os.warp, &t_fill);
  if (threadIdx.x == 0 && t_fill) os.res[5] = atomicAdd(&a.nctr->n_fills, t_fill);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    if (cls[q] == 3 && dstbuf == 1) {
      uint32_t gi = os.res[5] + o_fill++;
      if (gi < a.cap_fills) {
        Fill f;
        f.begin = sg.begin + base[q]; f.len = tot[q]; f.value = rep[q]; f.pad = 0;
        a.fills[gi] = f;
        atomicAdd((unsigned long long*)&a.nctr->fill_keys, (unsigned long long)tot[q]);
      } else {
        atomicOr(a.err, kErrOverflow);
      }
    }
  }
}

// Tile loop of phase 4a with the model kind and the optional outputs fixed at compile time.
// Per key: model evaluation (2 RN ops + saturating convert), one smem atomicAdd into the
// chunk histogram, and the homogeneity representative (racy store; after a barrier every
// key compares against it).  The next tile is loaded while this one is classified.
template <bool F64, bool EQ3, bool NANCHK, bool IDS>
__device__ void classify_tiles(const LevelArgs& a, const ChunkDesc& ch, const ModelDev& md,
                               uint32_t* hist, uint64_t* rep, uint32_t* has, uint32_t* inhs,
                               int& nan_seen) {
  const Bucketer<F64, EQ3> bucket(md, a.k);
  const uint64_t* p = a.src + ch.start;
  uint64_t cur[kCItems], nxt[kCItems];
#pragma unroll
  for (int r = 0; r < kCItems; ++r) {
    const uint32_t i = r * kCThreads + threadIdx.x;
    cur[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
  }
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kCTile) {
    const uint32_t tl = min((uint32_t)kCTile, ch.len - t0);
    const uint32_t t1 = t0 + kCTile;
#pragma unroll
    for (int r = 0; r < kCItems; ++r) {
      const uint32_t i = t1 + r * kCThreads + threadIdx.x;
      nxt[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
    }
    uint32_t bk[kCItems];
#pragma unroll
    for (int r = 0; r < kCItems; ++r) {
      const uint32_t i = r * kCThreads + threadIdx.x;
      if (i < tl) {
        if (NANCHK && is_nan_bits(cur[r])) nan_seen = 1;
        bk[r] = bucket(cur[r]);
        atomicAdd(&hist[bk[r]], 1u);
        if (!has[bk[r]]) rep[bk[r]] = cur[r];
        if (IDS) a.ids[ch.start + t0 + i] = (uint16_t)bk[r];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kCItems; ++r) {
      const uint32_t i = r * kCThreads + threadIdx.x;
      if (i < tl) {
        has[bk[r]] = 1;
        if (rep[bk[r]] != cur[r]) inhs[bk[r]] = 1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kCItems; ++r) cur[r] = nxt[r];
  }
}

template <bool F64, bool EQ3>
__device__ __forceinline__ void classify_dispatch(const LevelArgs& a, const ChunkDesc& ch,
                                                  const ModelDev& md, uint32_t* hist,
                                                  uint64_t* rep, uint32_t* has, uint32_t* inhs,
                                                  int& nan_seen) {
  if (a.ids)
    classify_tiles<F64, EQ3, false, true>(a, ch, md, hist, rep, has, inhs, nan_seen);
  else if (F64 && a.check_nan)
    classify_tiles<F64, EQ3, F64, false>(a, ch, md, hist, rep, has, inhs, nan_seen);
  else
    classify_tiles<F64, EQ3, false, false>(a, ch, md, hist, rep, has, inhs, nan_seen);
}

template <bool F64>
__global__ __launch_bounds__(kCThreads) void k_classify_scan(LevelArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const uint32_t k = a.k;
  uint64_t* rep = reinterpret_cast<uint64_t*>(smraw);  // k
  uint32_t* hist = reinterpret_cast<uint32_t*>(rep + k);
  uint32_t* has = hist + k;
  uint32_t* inhs = has + k;
  __shared__ uint32_t s_c;
  __shared__ OffSmem os;
  if (threadIdx.x == 0) s_c = atomicAdd(a.ticket, 1u);
  for (uint32_t b = threadIdx.x; b < k; b += kCThreads) { hist[b] = 0; has[b] = 0; inhs[b] = 0; }
  __syncthreads();
  const uint32_t c = s_c;
  const ChunkDesc ch = a.chunks[c];
  const SegDesc sg = a.segs[ch.seg];
  const ModelDev md = a.models[ch.seg];
  int nan_seen = 0;
  if (md.kind == kModelEq3)
    classify_dispatch<F64, true>(a, ch, md, hist, rep, has, inhs, nan_seen);
  else
    classify_dispatch<F64, false>(a, ch, md, hist, rep, has, inhs, nan_seen);
  if (a.check_nan) {
    if (__syncthreads_or(nan_seen) && threadIdx.x == 0) atomicOr(a.err, kErrNan);
  }
  // ---- decoupled lookback over the chunks of this segment, bucket by bucket ----
  // Every chunk first records its own count and representative (read only by the last
  // chunk's homogeneity check), fences once, then publishes one 64-bit status word per
  // bucket: AGG (own count) or INC (inclusive prefix), tagged with the level's epoch.
  const bool first = (c == sg.chunk_first);
  const bool last = (c == sg.chunk_first + sg.nchunks - 1);
  uint32_t tot[kCBpt], inh[kCBpt];
  uint64_t rp[kCBpt];
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    const uint32_t b = threadIdx.x * kCBpt + q;
    tot[q] = hist[b < k ? b : 0]; inh[q] = inhs[b < k ? b : 0]; rp[q] = rep[b < k ? b : 0];
    if (b < k && sg.nchunks > 1) {
      const size_t ix = (size_t)c * k + b;
      a.cnt_agg[ix] = tot[q] | (inh[q] << 31);
      a.rep_agg[ix] = rp[q];
    }
  }
  if (sg.nchunks > 1) {
    __threadfence();
#pragma unroll
    for (int q = 0; q < kCBpt; ++q) {
      const uint32_t b = threadIdx.x * kCBpt + q;
      if (b < k && !last)
        *((volatile uint64_t*)&a.status[(size_t)c * k + b]) =
            pack_status(a.epoch, first ? kStInc : kStAgg, inh[q], tot[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < kCBpt; ++q) {
    const uint32_t b = threadIdx.x * kCBpt + q;
    if (b >= k) continue;
    uint32_t ex_cnt = 0, ex_inh = 0;
    if (!first) {
      uint32_t j = c - 1;
      while (true) {
        const uint64_t st = *((volatile const uint64_t*)&a.status[(size_t)j * k + b]);
        const uint32_t state = (uint32_t)(st >> 46) & 3u;
        if ((uint32_t)(st >> 48) != (a.epoch & 0xffff) || state == 0) continue;  // not yet
        ex_cnt += (uint32_t)st;
        ex_inh |= (uint32_t)(st >> 45) & 1u;
        if (state == kStInc) break;
        --j;
      }
      if (!last)
        *((volatile uint64_t*)&a.status[(size_t)c * k + b]) =
            pack_status(a.epoch, kStInc, inh[q] | ex_inh, ex_cnt + tot[q]);
    }
    a.chunk_pre[(size_t)c * k + b] = ex_cnt;
    tot[q] += ex_cnt;
    inh[q] |= ex_inh;
  }
  if (last && sg.nchunks > 1) {
    // Homogeneity across chunks (R9): a child stays homogeneous only if every chunk that
    // holds keys of it saw one value and all those values agree.  Only children that could
    // be partitioned (> base case) matter (R20), so only they are checked.
    __threadfence();
#pragma unroll
    for (int q = 0; q < kCBpt; ++q) {
      const uint32_t b = threadIdx.x * kCBpt + q;
      if (b >= k || inh[q] || tot[q] <= a.base_case) continue;
      bool have = false;
      uint64_t ref = 0;
      for (uint32_t j = sg.chunk_first; j < c && !inh[q]; ++j) {
        const size_t jx = (size_t)j * k + b;
        const uint32_t cw = *((volatile const uint32_t*)&a.cnt_agg[jx]);
        if ((cw & ~kInhBit) == 0) continue;
        const uint64_t r = *((volatile const uint64_t*)&a.rep_agg[jx]);
        if (cw & kInhBit) inh[q] = 1;
        if (have && r != ref) inh[q] = 1;
        if (!have) { ref = r; have = true; }
      }
      if (hist[b]) {
        if (have && rep[b] != ref) inh[q] = 1;
        if (!have) ref = rep[b];
      }
      rp[q] = ref;
    }
  }
  if (last) segment_offsets(a, ch.seg, sg, md, tot, inh, rp, os);
}

// ------------------------------------------------------------------------------------
// Phase 4b: stable scatter of one chunk (R11).
//
// Tile = 4096 keys; warp w owns keys [512w, 512w+512) in 16 rounds of 32.
// Rank: every key does one smem atomicAdd on its warp's counter for its bucket (u16 halves
// of packed u32 words, two warps per word).  Same-address lanes of one atomic instruction
// are served in lane order on B200 (tools/micro/atom_order.cu: 0 violations in 2.2e9 lane
// pairs), so the returned values are the stable in-warp ranks; a cross-warp scan and a scan
// over buckets place every key in a bucket-sorted smem tile.  Stability is VERIFIED on the
// staged tile (tile index must increase inside every bucket run) while it is written out,
// and any offending run is rewritten in index order afterwards, so the layout is stable by
// construction whatever the hardware does.
// Write-out: per bucket, a byte-address base and a flush limit are precomputed once per
// tile, so a key costs one load of its (bucket, index) word, two smem loads and one store.
// Only whole 32-byte sectors are written while a chunk is in flight: the 0-3 trailing keys
// of a bucket that do not complete a sector wait in smem for the next tile (flushed at the
// chunk's end).  Partial-sector writes cost an ECC read-modify-write fill in HBM (ncu:
// lts__d_sectors_fill_device), which this avoids except at chunk boundaries.
constexpr uint32_t kPendSlots = 3;

template <bool F64, bool EQ3>
__device__ void scatter_tiles(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst_user,
                              uint64_t* __restrict__ dst_scr, const ChunkDesc& ch,
                              const ModelDev& md, uint32_t k, const uint32_t* __restrict__ chunk_pre,
                              const uint64_t* __restrict__ seg_dst, unsigned char* smraw) {
  uint64_t* stage = reinterpret_cast<uint64_t*>(smraw);                  // kSTile
  uint64_t* abase = stage + kSTile;                                      // k: byte address state
  uint64_t* pend = abase + k;                                            // k * kPendSlots
  uint32_t* sbi = reinterpret_cast<uint32_t*>(pend + (size_t)k * kPendSlots);  // kSTile
  uint32_t* wc = sbi + kSTile;                                           // (kSWarps/2) * k
  uint32_t* toff = wc + (kSWarps / 2) * k;                               // k + 1
  int32_t* qlim = reinterpret_cast<int32_t*>(toff + k + 1);              // k
  int32_t* pbase = qlim + k;                                             // k
  uint8_t* plen = reinterpret_cast<uint8_t*>(pbase + k);                 // k
  __shared__ uint32_t s_warp[40];

  const Bucketer<F64, EQ3> bucket(md, k);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // abase holds the byte address of the bucket's next destination between tiles
  for (uint32_t b = threadIdx.x; b < k; b += kSThreads) {
    const uint64_t d = seg_dst[(size_t)ch.seg * k + b] + chunk_pre[(size_t)blockIdx.x * k + b];
    uint64_t* buf = (d & kDstUserBit) ? dst_user : dst_scr;
    abase[b] = reinterpret_cast<uint64_t>(buf + (d & ~kDstUserBit));
    plen[b] = 0;
  }
  uint32_t* wcw = wc + (wp >> 1) * k;
  const uint32_t winc = 1u << (16 * (wp & 1));
  const int wsh = 16 * (wp & 1);
  const uint64_t* p = src + ch.start;
  uint64_t key[kSRounds];
#pragma unroll
  for (int r = 0; r < kSRounds; ++r) {
    const uint32_t i = wp * (kSRounds * 32) + r * 32 + lane;
    key[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
  }
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kSTile) {
    const uint32_t tl = min((uint32_t)kSTile, ch.len - t0);
    const bool last_tile = t0 + kSTile >= ch.len;
    for (uint32_t i = threadIdx.x; i < (kSWarps / 2) * k; i += kSThreads) wc[i] = 0u;
    __syncthreads();
    uint32_t bk[kSRounds], loc[kSRounds];
#pragma unroll
    for (int r = 0; r < kSRounds; ++r) {
      const uint32_t i = wp * (kSRounds * 32) + r * 32 + lane;
      bk[r] = (i < tl) ? bucket(key[r]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < kSRounds; ++r) {
      const uint32_t i = wp * (kSRounds * 32) + r * 32 + lane;
      loc[r] = (i < tl) ? ((atomicAdd(&wcw[bk[r]], winc) >> wsh) & 0xffffu) : 0u;
    }
    __syncthreads();
    // cross-warp exclusive scan per bucket (warp order = key order); tile totals into toff
    for (uint32_t b = threadIdx.x; b < k; b += kSThreads) {
      uint32_t run = 0;
#pragma unroll
      for (int w2 = 0; w2 < kSWarps / 2; ++w2) {
        const uint32_t wv = wc[w2 * k + b];
        const uint32_t lo = wv & 0xffffu, hi = wv >> 16;
        wc[w2 * k + b] = run | ((run + lo) << 16);
        run += lo + hi;
      }
      toff[b] = run;
    }
    __syncthreads();
    {
      uint32_t c4[4], s4 = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t b = threadIdx.x * 4 + q;
        c4[q] = (b < k) ? toff[b] : 0u;
        s4 += c4[q];
      }
      uint32_t tot;
      uint32_t ex = block_exclusive_scan<kSThreads>(s4, s_warp, &tot);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t b = threadIdx.x * 4 + q;
        if (b < k) toff[b] = ex;
        ex += c4[q];
      }
      if (threadIdx.x == 0) toff[k] = tot;
    }
    __syncthreads();
    // Per bucket: E = end address of this tile's keys, F = flush bound (last whole sector,
    // or E at the chunk's end), P = first pending address.  If F > P every old pending key
    // lies below F and is written now; keys at or above F (all keys when F <= P) wait in
    // slots relative to max(F, P).  Positions q of the staged tile map to addresses
    // abase + 8q.
    for (uint32_t b = threadIdx.x; b < k; b += kSThreads) {
      const uint64_t cur = abase[b];
      const uint32_t pl = plen[b];
      const uint32_t t_off = toff[b], n = toff[b + 1] - t_off;
      const uint64_t e = cur + 8ull * n;
      const uint64_t f = last_tile ? e : (e & ~31ull);
      const uint64_t pb = cur - 8ull * pl;
      uint64_t s0 = pb;
      if (f > pb) {
        for (uint32_t j = 0; j < pl; ++j)
          __stcs(reinterpret_cast<uint64_t*>(pb) + j, pend[b * kPendSlots + j]);
        s0 = f;
      }
      qlim[b] = (int32_t)t_off + (int32_t)((int64_t)(f - cur) / 8);
      pbase[b] = (int32_t)t_off + (int32_t)((int64_t)(s0 - cur) / 8);
      plen[b] = (uint8_t)((e - s0) / 8);
      abase[b] = cur - 8ull * t_off;
    }
#pragma unroll
    for (int r = 0; r < kSRounds; ++r) {
      const uint32_t i = wp * (kSRounds * 32) + r * 32 + lane;
      if (i < tl) {
        const uint32_t pos = toff[bk[r]] + ((wcw[bk[r]] >> wsh) & 0xffffu) + loc[r];
        stage[pos] = key[r];
        sbi[pos] = (bk[r] << 16) | i;
      }
    }
    {  // prefetch the next tile while this one drains
      const uint32_t t1 = t0 + kSTile;
#pragma unroll
      for (int r = 0; r < kSRounds; ++r) {
        const uint32_t i = t1 + wp * (kSRounds * 32) + r * 32 + lane;
        key[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
      }
    }
    __syncthreads();
    int bad = 0;
    for (uint32_t q = threadIdx.x; q < tl; q += kSThreads) {
      const uint32_t x = sbi[q];
      const uint32_t b = x >> 16;
      if (q > 0) {
        const uint32_t y = sbi[q - 1];
        if ((y >> 16) == b && (y & 0xffffu) > (x & 0xffffu)) bad = 1;
      }
      const uint64_t v = stage[q];
      if ((int32_t)q < qlim[b]) __stcs(reinterpret_cast<uint64_t*>(abase[b]) + q, v);
      else pend[b * kPendSlots + (uint32_t)((int32_t)q - pbase[b])] = v;
    }
    if (__syncthreads_or(bad)) {
      // Repair (never observed on B200): rewrite every bucket run in tile-index order.
      for (uint32_t b = threadIdx.x; b < k; b += kSThreads) {
        const uint32_t beg = toff[b], end = toff[b + 1];
        for (uint32_t i = beg + 1; i < end; ++i) {
          const uint32_t xi = sbi[i];
          const uint64_t xv = stage[i];
          uint32_t j = i;
          while (j > beg && (sbi[j - 1] & 0xffffu) > (xi & 0xffffu)) {
            sbi[j] = sbi[j - 1];
            stage[j] = stage[j - 1];
            --j;
          }
          sbi[j] = xi;
          stage[j] = xv;
        }
        for (uint32_t q = beg; q < end; ++q) {
          if ((int32_t)q < qlim[b]) reinterpret_cast<uint64_t*>(abase[b])[q] = stage[q];
          else pend[b * kPendSlots + (uint32_t)((int32_t)q - pbase[b])] = stage[q];
        }
      }
      __syncthreads();
    }
    for (uint32_t b = threadIdx.x; b < k; b += kSThreads) abase[b] += 8ull * toff[b + 1];
  }
}

template <bool F64>
__global__ __launch_bounds__(kSThreads, 2) void k_scatter(
    const uint64_t* __restrict__ src, uint64_t* __restrict__ dst_user,
    uint64_t* __restrict__ dst_scr, const ChunkDesc* __restrict__ chunks,
    const ModelDev* __restrict__ models, uint32_t k, const uint32_t* __restrict__ chunk_pre,
    const uint64_t* __restrict__ seg_dst, const uint32_t* __restrict__ err) {
  if (*((volatile const uint32_t*)err) & kErrNan) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  const ChunkDesc ch = chunks[blockIdx.x];
  const ModelDev md = models[ch.seg];
  if (md.kind == kModelEq3)
    scatter_tiles<F64, true>(src, dst_user, dst_scr, ch, md, k, chunk_pre, seg_dst, smraw);
  else
    scatter_tiles<F64, false>(src, dst_user, dst_scr, ch, md, k, chunk_pre, seg_dst, smraw);
}

// ------------------------------------------------------------------------------------
// Base case: sort one window of whole final segments (<= 8192 keys) by ordering key
// and write it to the user array.  Buckets are range-ordered (the model is monotone, R7),
// so sorting a window of consecutive final segments sorts each of them; any exact sort
// gives the identical bytes (R13).
// Keys stay in registers (16 per thread).  Fine bin of a key = its position on a linear
// map of [min, max] in ordering-key space onto len bins (windows at the last level span a
// narrow, locally smooth range), through a 256-bin coarse histogram only when the window
// spans more than two binades.  One counting pass places the keys into smem; bins hold ~1
// key and are finished by insertion sort; windows whose bins overflow take a bitonic sort.
constexpr int kBaseItems = kBaseMax / kBaseThreads;  // 16

template <bool F64>
__global__ __launch_bounds__(kBaseThreads, 2) void k_base_sort(
    const Window* __restrict__ wins, uint64_t* __restrict__ user, const uint64_t* __restrict__ scr,
    uint32_t* __restrict__ err, int check_nan) {
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* tmp = reinterpret_cast<uint64_t*>(smraw);             // kBaseMax
  uint32_t* fh = reinterpret_cast<uint32_t*>(tmp + kBaseMax);      // kBaseMax
  __shared__ SortSmem ss;
  const Window wv = wins[blockIdx.x];
  const uint32_t len = wv.len;
  if (len == 0) return;
  const uint64_t* srcp = (wv.buf ? scr : user) + wv.begin;
  uint64_t* dst = user + wv.begin;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  uint64_t v[kBaseItems];
  uint64_t mn = ~0ull, mx = 0ull;
  int nan_seen = 0;
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    const uint32_t i = j * kBaseThreads + threadIdx.x;
    v[j] = 0;
    if (i < len) {
      const uint64_t bits = __ldcs(srcp + i);
      if (F64 && check_nan && is_nan_bits(bits)) nan_seen = 1;
      v[j] = ok_of<F64>(bits);
      mn = min(mn, v[j]);
      mx = max(mx, v[j]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) { ss.red[wp] = mn; ss.red[32 + wp] = mx; }
  for (uint32_t i = threadIdx.x; i < len; i += kBaseThreads) fh[i] = 0u;
  for (uint32_t c = threadIdx.x; c < 256; c += kBaseThreads) ss.ccnt[c] = 0u;
  if (check_nan) {
    if (__syncthreads_or(nan_seen)) {
      if (threadIdx.x == 0) atomicOr(err, kErrNan);
      return;
    }
  } else {
    __syncthreads();
  }
  mn = ss.red[0]; mx = ss.red[32];
#pragma unroll
  for (int w = 1; w < kBaseThreads / 32; ++w) { mn = min(mn, ss.red[w]); mx = max(mx, ss.red[32 + w]); }
  if (mn == mx) {  // constant window: already sorted
    if (wv.buf) {
#pragma unroll
      for (int j = 0; j < kBaseItems; ++j) {
        const uint32_t i = j * kBaseThreads + threadIdx.x;
        if (i < len) __stcs(dst + i, bits_of_ok<F64>(v[j]));
      }
    }
    return;
  }
  const uint64_t range = mx - mn;
  const int bl = 64 - __clzll((long long)range);
  const bool coarse = bl > 54;  // more than two binades of doubles
  uint32_t f[kBaseItems];
  int sh = 0;
  if (coarse) {
    sh = bl - 8;
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) {
      const uint32_t i = j * kBaseThreads + threadIdx.x;
      if (i < len) atomicAdd(&ss.ccnt[(uint32_t)((v[j] - mn) >> sh)], 1u);
    }
    __syncthreads();
    uint32_t cc = (threadIdx.x < 256) ? ss.ccnt[threadIdx.x] : 0u;
    uint32_t ex = block_exclusive_scan<kBaseThreads>(cc, ss.warp, nullptr);
    if (threadIdx.x < 256) ss.coff[threadIdx.x] = ex;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) {
      const uint32_t i = j * kBaseThreads + threadIdx.x;
      f[j] = (i < len) ? fine_bin(v[j], mn, sh, ss.coff, ss.ccnt) : 0u;
    }
  } else {
    const int up = 64 - bl;  // (ok - mn) << up is the fraction of the range in [0, 1)
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) f[j] = (uint32_t)__umul64hi((v[j] - mn) << up, len);
  }
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    const uint32_t i = j * kBaseThreads + threadIdx.x;
    if (i < len) atomicAdd(&fh[f[j]], 1u);
  }
  __syncthreads();
  // exclusive scan of fh[0..len): thread t owns bins [t*16, t*16+16)
  uint32_t mxc = 0;
  {
    const uint32_t b0 = threadIdx.x * kBaseItems;
    uint32_t c[kBaseItems], sum = 0;
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) {
      c[j] = (b0 + j < len) ? fh[b0 + j] : 0u;
      sum += c[j];
      mxc = max(mxc, c[j]);
    }
    uint32_t run = block_exclusive_scan<kBaseThreads>(sum, ss.warp, nullptr);
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) {
      if (b0 + j < len) fh[b0 + j] = run;
      run += c[j];
    }
  }
  const bool overflow = __syncthreads_or(mxc > kFineOverflow) != 0;
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    const uint32_t i = j * kBaseThreads + threadIdx.x;
    if (i < len) tmp[atomicAdd(&fh[f[j]], 1u)] = v[j];
  }
  __syncthreads();
  if (!overflow) {
    for (uint32_t b = threadIdx.x; b < len; b += kBaseThreads) {
      const uint32_t beg = b ? fh[b - 1] : 0u, end = fh[b];
      for (uint32_t i = beg + 1; i < end; ++i) {
        const uint64_t x = tmp[i];
        uint32_t j = i;
        while (j > beg && tmp[j - 1] > x) { tmp[j] = tmp[j - 1]; --j; }
        tmp[j] = x;
      }
    }
    __syncthreads();
  } else {
    bitonic_sort_smem<kBaseThreads>(tmp, len);
  }
  for (uint32_t i = threadIdx.x; i < len; i += kBaseThreads) __stcs(dst + i, bits_of_ok<F64>(tmp[i]));
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

__global__ void k_keys_to_ok(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                             uint32_t n, int f64) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = f64 ? ok_of_f64(in[i]) : in[i];
}

}  // namespace ipls
