// ipls_kernels.cuh — sm_100a kernels of one IPLS distribution level and the base case.
//
// Per level (the four phases of P:265-287):
//   k_sample_gather   phase 1: stratified sample of every segment (R2, R18)
//   k_fit             phase 2+3: sort the sample in smem, FMCD fit (Listing 1)
//   k_classify_hist   phase 4a: model eval + smem histogram per chunk, NaN flag,
//                     per-chunk homogeneity representative (R9)
//   k_unit_reduce / k_seg_scan / k_chunk_prefix
//                     column scan of the (chunk x bucket) histogram -> per-chunk offsets
//   k_seg_offsets     per segment: bucket bases, child classes (R20), next-level work,
//                     base-case windows, fills of homogeneous children
//   k_scatter         phase 4b: stable in-tile rank (ballot multisplit), smem staging by
//                     bucket, run-contiguous writes (R11)
// After the level: k_base_sort (base case) and k_fill.
#pragma once
#include "ipls_device.cuh"

namespace ipls {

constexpr int kTileThreads = 512;
constexpr int kTileItems = 8;
constexpr int kTile = kTileThreads * kTileItems;  // 4096 keys per tile
constexpr int kTileWarps = kTileThreads / 32;     // 16
constexpr int kUnitChunks = 32;
constexpr int kFitThreads = 1024;
constexpr int kFitMaxS = 8192;
constexpr int kBaseThreads = 512;
constexpr int kBaseItems = 16;
constexpr int kBaseMax = kBaseThreads * kBaseItems;  // 8192 keys per window
constexpr uint32_t kWindowNominal = 4096;
constexpr int kOffThreads = 1024;
constexpr uint32_t kMaxK = 1024;

// ------------------------------------------------------------------------------------
// Root work item (level 0): one segment covering [0, n), chunked, grouped in units.
__global__ void k_init_root(SegDesc* segs, ChunkDesc* chunks, UnitDesc* units, uint64_t n,
                            uint32_t S, uint32_t chunk_keys, uint32_t flags) {
  uint32_t nch = (uint32_t)((n + chunk_keys - 1) / chunk_keys);
  uint32_t nu = (nch + kUnitChunks - 1) / kUnitChunks;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    SegDesc sg{};
    sg.begin = 0; sg.m = (uint32_t)n; sg.S = S; sg.sample_off = 0;
    sg.chunk_first = 0; sg.nchunks = nch; sg.unit_first = 0; sg.nunits = nu; sg.flags = flags;
    segs[0] = sg;
  }
  for (uint32_t c = i; c < nch; c += gridDim.x * blockDim.x) {
    ChunkDesc cd;
    cd.start = (uint64_t)c * chunk_keys;
    cd.len = (uint32_t)min((uint64_t)chunk_keys, n - cd.start);
    cd.seg = 0;
    chunks[c] = cd;
  }
  for (uint32_t u = i; u < nu; u += gridDim.x * blockDim.x) {
    UnitDesc ud;
    ud.seg = 0; ud.chunk_first = u * kUnitChunks;
    ud.nch = min((uint32_t)kUnitChunks, nch - u * kUnitChunks); ud.pad = 0;
    units[u] = ud;
  }
}

// ------------------------------------------------------------------------------------
// Phase 1: one position per stratum [floor(j m/S), floor((j+1) m/S)) (R2), SplitMix64 keyed
// by (seed, level, begin, j) (R18).  Stores ordering keys.
template <bool F64>
__global__ void k_sample_gather(const uint64_t* __restrict__ src, const SegDesc* __restrict__ segs,
                                uint64_t seed, uint32_t level, uint64_t* __restrict__ samples) {
  const SegDesc sg = segs[blockIdx.x];
  const uint64_t t = sm64(sm64(sm64(seed) ^ (uint64_t)level) ^ sg.begin);
  const uint64_t m = sg.m, S = sg.S;
  for (uint32_t j = threadIdx.x; j < sg.S; j += blockDim.x) {
    uint64_t lo = ((uint64_t)j * m) / S;
    uint64_t hi = ((uint64_t)(j + 1) * m) / S;
    uint64_t h = sm64(t ^ (uint64_t)j);
    uint64_t idx = sg.begin + lo + __umul64hi(h, hi - lo);
    samples[sg.sample_off + j] = ok_of<F64>(__ldg(src + idx));
  }
}

// ------------------------------------------------------------------------------------
// Phase 2+3: sort the sample (bitonic, smem), then FMCD.
//
// Listing 1 returns the least D >= 1 whose every window satisfies s[i+D]-s[i] >= u(D),
// u(D) = (s[N-1-D]-s[D])/(k-2); if no D <= floor(N/3) qualifies it stops with
// D = floor(N/3)+1 and the stale u(floor(N/3)) (R4).  The predicate is monotone in D in
// binary64 (RN is monotone), so the CTA finds that D by galloping + bisection, testing each
// candidate with all threads (K2).  Every arithmetic step is one RN op.
__device__ __forceinline__ double fmcd_u(const double* s, uint32_t N, uint32_t D, double km2) {
  return __ddiv_rn(__dsub_rn(s[N - 1 - D], s[D]), km2);
}

__device__ bool fmcd_pred(const double* s, uint32_t N, uint32_t D, double u) {
  int fail = 0;
  for (uint32_t i = threadIdx.x; i + D < N; i += blockDim.x) {
    if (!(__dsub_rn(s[i + D], s[i]) >= u)) { fail = 1; break; }
  }
  return __syncthreads_or(fail) == 0;
}

template <bool F64>
__global__ __launch_bounds__(kFitThreads) void k_fit(const SegDesc* __restrict__ segs,
                                                     uint64_t* __restrict__ samples, uint32_t k,
                                                     ModelDev* __restrict__ models,
                                                     int presorted) {
  extern __shared__ __align__(16) uint64_t sk[];
  __shared__ uint64_t s_pivot;
  const SegDesc sg = segs[blockIdx.x];
  const uint32_t S = sg.S;
  uint32_t NP = 1;
  while (NP < S) NP <<= 1;
  for (uint32_t i = threadIdx.x; i < NP; i += blockDim.x)
    sk[i] = (i < S) ? samples[sg.sample_off + i] : ~0ull;
  __syncthreads();
  if (!presorted) {
    for (uint32_t size = 2; size <= NP; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = threadIdx.x; i < NP / 2; i += blockDim.x) {
          uint32_t lo = 2 * i - (i & (stride - 1));
          uint32_t hi = lo + stride;
          bool asc = (lo & size) == 0;
          uint64_t a = sk[lo], b = sk[hi];
          if ((a > b) == asc) { sk[lo] = b; sk[hi] = a; }
        }
        __syncthreads();
      }
    }
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) samples[sg.sample_off + i] = sk[i];
  }
  if (threadIdx.x == 0) s_pivot = sk[S / 2];
  __syncthreads();
  ModelDev md{};
  md.k_eff = k;
  bool eq3 = (sg.flags & kSegForceEq3) || S < 4;
  if (!eq3) {
    // model values of the sorted sample, in place
    double* s = reinterpret_cast<double*>(sk);
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x)
      s[i] = value_of<F64>(bits_of_ok<F64>(sk[i]));
    __syncthreads();
    const uint32_t N = S;
    const uint32_t Dcap = N / 3;  // >= 1 since N >= 4
    const double km2 = (double)(k - 2);
    // gallop: D = 1, 2, 4, ... (all tested D < found are false)
    uint32_t lo = 0, hi = 0;  // pred(lo) false (lo = 0 sentinel), pred(hi) true
    uint32_t D = 1;
    bool found = false;
    while (true) {
      if (D > Dcap) D = Dcap;
      double u = fmcd_u(s, N, D, km2);
      if (fmcd_pred(s, N, D, u)) { hi = D; found = true; break; }
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
        double u = fmcd_u(s, N, mid, km2);
        if (fmcd_pred(s, N, mid, u)) hi = mid; else lo = mid;
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
// Phase 4a: classify + histogram of one chunk.  Histogram by smem atomics (measured
// 2.2 T updates/s on B200, tools/micro).  Homogeneity (R9): per bucket, a racy store picks
// one representative key per tile; every key then compares against it; any mismatch marks
// the bucket inhomogeneous (plain idempotent stores, two barriers per tile).
template <bool F64>
__global__ __launch_bounds__(kTileThreads) void k_classify_hist(
    const uint64_t* __restrict__ src, const ChunkDesc* __restrict__ chunks,
    const SegDesc* __restrict__ segs, const ModelDev* __restrict__ models, uint32_t k,
    uint32_t* __restrict__ chunk_hist, uint64_t* __restrict__ chunk_rep,
    uint32_t* __restrict__ err, int check_nan, uint16_t* __restrict__ ids,
    uint64_t ids_origin) {
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* rep = reinterpret_cast<uint64_t*>(smraw);
  uint32_t* hist = reinterpret_cast<uint32_t*>(rep + k);
  uint32_t* has = hist + k;
  uint32_t* inh = has + k;
  const ChunkDesc ch = chunks[blockIdx.x];
  const ModelDev md = models[ch.seg];
  const double kd = (double)k;
  const uint32_t km1 = k - 1;
  for (uint32_t b = threadIdx.x; b < k; b += blockDim.x) { hist[b] = 0; has[b] = 0; inh[b] = 0; }
  __syncthreads();
  int nan_seen = 0;
  const uint64_t* p = src + ch.start;
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kTile) {
    const uint32_t tl = min((uint32_t)kTile, ch.len - t0);
    uint64_t key[kTileItems];
    uint32_t bk[kTileItems];
#pragma unroll
    for (int r = 0; r < kTileItems; ++r) {
      uint32_t i = r * kTileThreads + threadIdx.x;
      key[r] = (i < tl) ? __ldcs(p + t0 + i) : 0ull;
    }
#pragma unroll
    for (int r = 0; r < kTileItems; ++r) {
      uint32_t i = r * kTileThreads + threadIdx.x;
      if (i < tl) {
        if (F64 && check_nan && is_nan_bits(key[r])) nan_seen = 1;
        bk[r] = bucket_of<F64>(key[r], md, kd, km1);
        atomicAdd(&hist[bk[r]], 1u);
        if (!has[bk[r]]) rep[bk[r]] = key[r];
        if (ids) ids[ch.start + t0 + i - ids_origin] = (uint16_t)bk[r];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kTileItems; ++r) {
      uint32_t i = r * kTileThreads + threadIdx.x;
      if (i < tl) {
        has[bk[r]] = 1;
        if (rep[bk[r]] != key[r]) inh[bk[r]] = 1;
      }
    }
    __syncthreads();
  }
  if (check_nan) {
    if (__syncthreads_or(nan_seen) && threadIdx.x == 0) atomicOr(err, kErrNan);
  }
  uint32_t* hout = chunk_hist + (size_t)blockIdx.x * k;
  uint64_t* rout = chunk_rep + (size_t)blockIdx.x * k;
  for (uint32_t b = threadIdx.x; b < k; b += blockDim.x) {
    hout[b] = hist[b] | (inh[b] ? kInhBit : 0u);
    rout[b] = rep[b];
  }
}

// ------------------------------------------------------------------------------------
// Column scan of the (chunk x bucket) counts, three light passes (warp per (unit, 32
// buckets)): unit aggregates -> per-segment exclusive prefix over units + totals ->
// per-chunk exclusive prefix.  Homogeneity is folded in: a child is homogeneous iff no
// chunk saw two different keys in it and all chunks' representatives agree.
__global__ void k_unit_reduce(const UnitDesc* __restrict__ units, uint32_t nunits, uint32_t k,
                              const uint32_t* __restrict__ chunk_hist,
                              const uint64_t* __restrict__ chunk_rep,
                              uint32_t* __restrict__ unit_cnt, uint64_t* __restrict__ unit_rep) {
  const uint32_t nsl = (k + 31) / 32;
  const uint32_t gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t u = gw / nsl;
  if (u >= nunits) return;
  const uint32_t b = (gw % nsl) * 32 + (threadIdx.x & 31);
  if (b >= k) return;
  const UnitDesc ud = units[u];
  uint32_t cnt = 0, bad = 0, have = 0;
  uint64_t ref = 0;
  for (uint32_t c = ud.chunk_first; c < ud.chunk_first + ud.nch; ++c) {
    uint32_t h = chunk_hist[(size_t)c * k + b];
    uint32_t cn = h & ~kInhBit;
    if (cn) {
      uint64_t r = chunk_rep[(size_t)c * k + b];
      bad |= h >> 31;
      if (have && r != ref) bad = 1;
      if (!have) { ref = r; have = 1; }
      cnt += cn;
    }
  }
  unit_cnt[(size_t)u * k + b] = cnt | (bad ? kInhBit : 0u);
  unit_rep[(size_t)u * k + b] = ref;
}

__global__ void k_seg_scan(const SegDesc* __restrict__ segs, uint32_t nsegs, uint32_t k,
                           uint32_t* __restrict__ unit_cnt, const uint64_t* __restrict__ unit_rep,
                           uint32_t* __restrict__ seg_tot, uint64_t* __restrict__ seg_rep) {
  const uint32_t nsl = (k + 31) / 32;
  const uint32_t gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t s = gw / nsl;
  if (s >= nsegs) return;
  const uint32_t b = (gw % nsl) * 32 + (threadIdx.x & 31);
  if (b >= k) return;
  const SegDesc sg = segs[s];
  uint32_t run = 0, bad = 0, have = 0;
  uint64_t ref = 0;
  for (uint32_t u = sg.unit_first; u < sg.unit_first + sg.nunits; ++u) {
    uint32_t w = unit_cnt[(size_t)u * k + b];
    uint32_t cn = w & ~kInhBit;
    unit_cnt[(size_t)u * k + b] = run;  // exclusive prefix of the unit
    if (cn) {
      uint64_t r = unit_rep[(size_t)u * k + b];
      bad |= w >> 31;
      if (have && r != ref) bad = 1;
      if (!have) { ref = r; have = 1; }
      run += cn;
    }
  }
  seg_tot[(size_t)s * k + b] = run | (bad ? kInhBit : 0u);
  seg_rep[(size_t)s * k + b] = ref;
}

__global__ void k_chunk_prefix(const UnitDesc* __restrict__ units, uint32_t nunits, uint32_t k,
                               const uint32_t* __restrict__ unit_pre,
                               uint32_t* __restrict__ chunk_hist) {
  const uint32_t nsl = (k + 31) / 32;
  const uint32_t gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const uint32_t u = gw / nsl;
  if (u >= nunits) return;
  const uint32_t b = (gw % nsl) * 32 + (threadIdx.x & 31);
  if (b >= k) return;
  const UnitDesc ud = units[u];
  uint32_t run = unit_pre[(size_t)u * k + b];
  for (uint32_t c = ud.chunk_first; c < ud.chunk_first + ud.nch; ++c) {
    uint32_t h = chunk_hist[(size_t)c * k + b] & ~kInhBit;
    chunk_hist[(size_t)c * k + b] = run;
    run += h;
  }
}

// ------------------------------------------------------------------------------------
// Per segment: bucket bases (exclusive scan over k), child classes with the precedence of
// R20 (homogeneous > base > partition; small homogeneous children go with the base case,
// which leaves them unchanged), the no-progress guard (R10), and next-level work.
struct OffsetsArgs {
  const SegDesc* segs;
  const ModelDev* models;
  const uint32_t* seg_tot;
  const uint64_t* seg_rep;
  uint64_t* seg_dst;
  uint32_t k, base_case, level, chunk_keys;
  SegDesc* nsegs;
  ChunkDesc* nchunks;
  UnitDesc* nunits;
  LevelCounters* nctr;
  uint32_t cap_segs, cap_chunks, cap_units, cap_samples;
  Window* wins;
  uint32_t cap_wins;
  Fill* fills;
  uint32_t cap_fills;
  uint32_t* err;
};

__device__ void emit_segment(const OffsetsArgs& a, uint64_t begin, uint32_t m, uint32_t flags,
                             uint32_t seg_idx, uint32_t samp_off, uint32_t ch_off,
                             uint32_t un_off) {
  SegDesc sd{};
  sd.begin = begin; sd.m = m; sd.S = sample_size(m, a.k); sd.sample_off = samp_off;
  uint32_t nch = (m + a.chunk_keys - 1) / a.chunk_keys;
  uint32_t nu = (nch + kUnitChunks - 1) / kUnitChunks;
  sd.chunk_first = ch_off; sd.nchunks = nch; sd.unit_first = un_off; sd.nunits = nu;
  sd.flags = flags;
  a.nsegs[seg_idx] = sd;
  for (uint32_t j = 0; j < nch; ++j) {
    ChunkDesc cd;
    cd.start = begin + (uint64_t)j * a.chunk_keys;
    cd.len = min(a.chunk_keys, m - j * a.chunk_keys);
    cd.seg = seg_idx;
    a.nchunks[ch_off + j] = cd;
  }
  for (uint32_t u = 0; u < nu; ++u) {
    UnitDesc ud;
    ud.seg = seg_idx; ud.chunk_first = ch_off + u * kUnitChunks;
    ud.nch = min((uint32_t)kUnitChunks, nch - u * kUnitChunks); ud.pad = 0;
    a.nunits[un_off + u] = ud;
  }
}

__global__ __launch_bounds__(kOffThreads) void k_seg_offsets(OffsetsArgs a) {
  __shared__ uint32_t s_warp[40];
  __shared__ uint32_t s_res[8];
  __shared__ uint32_t s_basey[kMaxK];
  __shared__ uint32_t s_wid[kMaxK];
  __shared__ uint32_t s_wbeg[kMaxK];
  __shared__ uint32_t s_wend[kMaxK];
  const uint32_t s = blockIdx.x;
  const uint32_t b = threadIdx.x;
  const SegDesc sg = a.segs[s];
  const ModelDev md = a.models[s];
  const uint32_t k = a.k;
  const uint32_t w = (b < k) ? a.seg_tot[(size_t)s * k + b] : 0u;
  const uint32_t tot = w & ~kInhBit;
  const bool inh = (w & kInhBit) != 0;
  const uint32_t base = block_exclusive_scan<kOffThreads>(tot, s_warp, nullptr);
  const bool stuck =
      __syncthreads_or(md.kind == kModelLinear && b < k && tot == sg.m) != 0;
  const uint32_t dstbuf = (a.level + 1) & 1;  // 1 = scratch, 0 = user array
  const uint64_t enc = (dstbuf == 0 ? kDstUserBit : 0ull) | (sg.begin + base);
  if (b < k) a.seg_dst[(size_t)s * k + b] = enc;

  // class: 0 empty, 1 base (or small homogeneous), 2 partition, 3 big homogeneous (final)
  uint32_t cls = 0;
  if (!stuck && b < k && tot > 0) {
    bool homog = (md.kind == kModelEq3 && b == 1) || !inh;
    if (tot <= a.base_case) cls = 1;
    else if (homog) cls = 3;
    else cls = 2;
  }
  // ---- next-level segments (partition children, or the whole segment when stuck) ----
  uint32_t want_seg = 0, want_samp = 0, want_ch = 0, want_un = 0, cm = 0;
  if (stuck) {
    if (b == 0) cm = sg.m;
  } else if (cls == 2) {
    cm = tot;
  }
  if (cm) {
    want_seg = 1;
    want_samp = sample_size(cm, k);
    want_ch = (cm + a.chunk_keys - 1) / a.chunk_keys;
    want_un = (want_ch + kUnitChunks - 1) / kUnitChunks;
  }
  uint32_t t_seg, t_samp, t_ch, t_un;
  uint32_t o_seg = block_exclusive_scan<kOffThreads>(want_seg, s_warp, &t_seg);
  uint32_t o_samp = block_exclusive_scan<kOffThreads>(want_samp, s_warp, &t_samp);
  uint32_t o_ch = block_exclusive_scan<kOffThreads>(want_ch, s_warp, &t_ch);
  uint32_t o_un = block_exclusive_scan<kOffThreads>(want_un, s_warp, &t_un);
  if (threadIdx.x == 0 && t_seg) {
    s_res[0] = atomicAdd(&a.nctr->n_segs, t_seg);
    s_res[1] = atomicAdd(&a.nctr->n_samples, t_samp);
    s_res[2] = atomicAdd(&a.nctr->n_chunks, t_ch);
    s_res[3] = atomicAdd(&a.nctr->n_units, t_un);
  }
  __syncthreads();
  if (t_seg) {
    bool ok = s_res[0] + t_seg <= a.cap_segs && s_res[1] + t_samp <= a.cap_samples &&
              s_res[2] + t_ch <= a.cap_chunks && s_res[3] + t_un <= a.cap_units;
    if (!ok) {
      if (threadIdx.x == 0) atomicOr(a.err, kErrOverflow);
    } else if (cm) {
      uint64_t cb = stuck ? sg.begin : sg.begin + base;
      emit_segment(a, cb, cm, stuck ? kSegForceEq3 : 0u, s_res[0] + o_seg, s_res[1] + o_samp,
                   s_res[2] + o_ch, s_res[3] + o_un);
      atomicAdd((unsigned long long*)&a.nctr->keys, (unsigned long long)cm);
    }
  }
  if (stuck) return;  // block-uniform

  // ---- base-case windows: maximal runs of base/empty children within one W-window ----
  const bool basey = (b < k) && (cls <= 1);
  const uint32_t wid = base / kWindowNominal;
  if (b < k) { s_basey[b] = basey; s_wid[b] = wid; }
  __syncthreads();
  uint32_t start = 0;
  if (basey) start = (b == 0) || !s_basey[b - 1] || s_wid[b - 1] != wid;
  uint32_t t_win;
  uint32_t o_win = block_exclusive_scan<kOffThreads>(start, s_warp, &t_win);
  // window index of a basey child = (inclusive count of starts up to it) - 1
  const uint32_t widx = o_win + start - 1;
  if (start) { s_wbeg[widx] = base; s_wend[widx] = base; }
  __syncthreads();
  if (basey) atomicMax(&s_wend[widx], base + tot);
  if (threadIdx.x == 0 && t_win) s_res[4] = atomicAdd(&a.nctr->n_windows, t_win);
  __syncthreads();
  if (start) {
    uint32_t gi = s_res[4] + widx;
    if (gi < a.cap_wins) {
      Window wv;
      wv.begin = sg.begin + s_wbeg[widx];
      wv.len = s_wend[widx] - s_wbeg[widx];
      wv.buf = dstbuf;
      a.wins[gi] = wv;
      atomicAdd((unsigned long long*)&a.nctr->win_keys, (unsigned long long)wv.len);
    } else {
      atomicOr(a.err, kErrOverflow);
    }
  }
  // ---- homogeneous children that land in scratch must be filled into the user array ----
  const uint32_t want_fill = (cls == 3 && dstbuf == 1) ? 1u : 0u;
  uint32_t t_fill;
  uint32_t o_fill = block_exclusive_scan<kOffThreads>(want_fill, s_warp, &t_fill);
  if (threadIdx.x == 0 && t_fill) s_res[5] = atomicAdd(&a.nctr->n_fills, t_fill);
  __syncthreads();
  if (want_fill) {
    uint32_t gi = s_res[5] + o_fill;
    if (gi < a.cap_fills) {
      Fill f;
      f.begin = sg.begin + base; f.len = tot; f.value = a.seg_rep[(size_t)s * k + b]; f.pad = 0;
      a.fills[gi] = f;
      atomicAdd((unsigned long long*)&a.nctr->fill_keys, (unsigned long long)tot);
    } else {
      atomicOr(a.err, kErrOverflow);
    }
  }
}

// Offsets of a single segment for ipls_partition_level: bases -> seg_dst and k_eff+1 offsets.
__global__ __launch_bounds__(kOffThreads) void k_single_offsets(const uint32_t* __restrict__ seg_tot,
                                                                uint32_t k, uint32_t k_eff,
                                                                uint64_t* __restrict__ seg_dst,
                                                                uint64_t* __restrict__ offsets) {
  __shared__ uint32_t s_warp[40];
  const uint32_t b = threadIdx.x;
  const uint32_t tot = (b < k) ? (seg_tot[b] & ~kInhBit) : 0u;
  uint32_t total;
  const uint32_t base = block_exclusive_scan<kOffThreads>(tot, s_warp, &total);
  if (b < k) seg_dst[b] = base;  // buffer bit 0 -> "scratch" pointer = caller's d_out
  if (b < k_eff) offsets[b] = base;
  if (b == 0) offsets[k_eff] = total;
}

// ------------------------------------------------------------------------------------
// Phase 4b: stable scatter of one chunk.  Per tile of 4096 keys: every warp owns 256
// consecutive keys and ranks them in 8 rounds of 32 with a ballot multisplit (LOG2K
// ballots give each lane the mask of lanes with the same bucket; __match_any_sync measured
// 16x slower on B200, tools/micro); per-warp u16 counters, a cross-warp scan and a scan
// over buckets give each key its position in the bucket-sorted smem tile; the tile is then
// written bucket-run by bucket-run to running per-bucket cursors (contiguous runs).
template <bool F64, int LOG2K>
__global__ __launch_bounds__(kTileThreads, 2) void k_scatter(
    const uint64_t* __restrict__ src, uint64_t* __restrict__ dst_user,
    uint64_t* __restrict__ dst_scr, const ChunkDesc* __restrict__ chunks,
    const ModelDev* __restrict__ models, uint32_t k, const uint32_t* __restrict__ chunk_pre,
    const uint64_t* __restrict__ seg_dst, const uint32_t* __restrict__ err) {
  if (*((volatile const uint32_t*)err) & kErrNan) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* stage = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* cursor = stage + kTile;
  uint32_t* toff = reinterpret_cast<uint32_t*>(cursor + k);
  uint32_t* tcnt = toff + k;
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(tcnt + k);
  uint16_t* sb = wcnt + kTileWarps * k;
  __shared__ uint32_t s_warp[40];

  const ChunkDesc ch = chunks[blockIdx.x];
  const ModelDev md = models[ch.seg];
  const double kd = (double)k;
  const uint32_t km1 = k - 1;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t b = threadIdx.x; b < k; b += blockDim.x)
    cursor[b] = seg_dst[(size_t)ch.seg * k + b] + chunk_pre[(size_t)blockIdx.x * k + b];
  const uint64_t* p = src + ch.start;
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kTile) {
    const uint32_t tl = min((uint32_t)kTile, ch.len - t0);
    uint32_t* wz = reinterpret_cast<uint32_t*>(wcnt);
    for (uint32_t i = threadIdx.x; i < (kTileWarps * k) / 2; i += blockDim.x) wz[i] = 0u;
    __syncthreads();
    uint64_t key[kTileItems];
    uint32_t bk[kTileItems], loc[kTileItems];
#pragma unroll
    for (int r = 0; r < kTileItems; ++r) {
      uint32_t i = wp * 256 + r * 32 + lane;
      key[r] = (i < tl) ? __ldcs(p + t0 + i) : 0ull;
    }
    uint16_t* mycnt = wcnt + wp * k;
#pragma unroll
    for (int r = 0; r < kTileItems; ++r) {
      uint32_t i = wp * 256 + r * 32 + lane;
      bool v = i < tl;
      bk[r] = v ? bucket_of<F64>(key[r], md, kd, km1) : 0u;
      uint32_t peers = __ballot_sync(0xffffffffu, v);
#pragma unroll
      for (int bit = 0; bit < LOG2K; ++bit) {
        uint32_t x = (bk[r] >> bit) & 1u;
        uint32_t mb = __ballot_sync(0xffffffffu, x);
        peers &= x ? mb : ~mb;
      }
      uint32_t below = peers & lt;
      uint32_t before = v ? (uint32_t)mycnt[bk[r]] : 0u;
      __syncwarp();
      if (v && below == 0) mycnt[bk[r]] = (uint16_t)(before + __popc(peers));
      __syncwarp();
      loc[r] = before + __popc(below);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < k; b += blockDim.x) {
      uint32_t run = 0;
#pragma unroll
      for (int w2 = 0; w2 < kTileWarps; ++w2) {
        uint32_t c = wcnt[w2 * k + b];
        wcnt[w2 * k + b] = (uint16_t)run;
        run += c;
      }
      tcnt[b] = run;
    }
    __syncthreads();
    {
      // k <= 1024: two consecutive buckets per thread
      uint32_t b0 = 2 * threadIdx.x, b1 = b0 + 1;
      uint32_t c0 = (b0 < k) ? tcnt[b0] : 0u, c1 = (b1 < k) ? tcnt[b1] : 0u;
      uint32_t ex = block_exclusive_scan<kTileThreads>(c0 + c1, s_warp, nullptr);
      if (b0 < k) toff[b0] = ex;
      if (b1 < k) toff[b1] = ex + c0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kTileItems; ++r) {
      uint32_t i = wp * 256 + r * 32 + lane;
      if (i < tl) {
        uint32_t pos = toff[bk[r]] + mycnt[bk[r]] + loc[r];
        stage[pos] = key[r];
        sb[pos] = (uint16_t)bk[r];
      }
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < tl; q += blockDim.x) {
      uint32_t b = sb[q];
      uint64_t d = cursor[b] + (q - toff[b]);
      uint64_t* out = (d & kDstUserBit) ? dst_user : dst_scr;
      out[d & ~kDstUserBit] = stage[q];
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < k; b += blockDim.x) cursor[b] += tcnt[b];
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// Base case: sort one window of whole final segments (<= 8192 keys) by ordering
// key and write it to the user array.  Buckets are range-ordered (the model is monotone,
// R7), so sorting a window of consecutive final segments sorts each of them.
// Method: ordering keys in smem; a 256-way coarse histogram (shift of ok - min) allots
// each coarse bin as many fine bins as it has keys; a fine counting sort then leaves runs
// of ~1 key, finished by insertion sort.  Windows whose fine bins overflow fall back to
// a bitonic sort.  Any exact sort gives the identical bytes (R13).
template <bool F64>
__global__ __launch_bounds__(kBaseThreads, 2) void k_base_sort(
    const Window* __restrict__ wins, uint64_t* __restrict__ user, const uint64_t* __restrict__ scr,
    uint32_t* __restrict__ err, int check_nan) {
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* stage = reinterpret_cast<uint64_t*>(smraw);          // kBaseMax
  uint32_t* fh = reinterpret_cast<uint32_t*>(stage + kBaseMax);  // kBaseMax
  __shared__ uint32_t ccnt[256], coff[256];
  __shared__ uint64_t s_mn[32], s_mx[32];
  __shared__ uint32_t s_warp[40];
  __shared__ uint32_t s_flag;
  const Window wv = wins[blockIdx.x];
  const uint32_t len = wv.len;
  if (len == 0) return;
  const uint64_t* srcp = (wv.buf ? scr : user) + wv.begin;
  uint64_t okv[kBaseItems];
  uint64_t mn = ~0ull, mx = 0ull;
  int nan_seen = 0;
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    uint32_t i = j * kBaseThreads + threadIdx.x;
    if (i < len) {
      uint64_t bits = srcp[i];
      if (F64 && check_nan && is_nan_bits(bits)) nan_seen = 1;
      okv[j] = ok_of<F64>(bits);
      mn = min(mn, okv[j]);
      mx = max(mx, okv[j]);
    }
  }
  if (check_nan) {
    if (__syncthreads_or(nan_seen)) {
      if (threadIdx.x == 0) atomicOr(err, kErrNan);
      return;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  if (lane == 0) { s_mn[wp] = mn; s_mx[wp] = mx; }
  for (uint32_t c = threadIdx.x; c < 256; c += blockDim.x) ccnt[c] = 0;
  __syncthreads();
  mn = s_mn[0]; mx = s_mx[0];
  for (int w = 1; w < kBaseThreads / 32; ++w) { mn = min(mn, s_mn[w]); mx = max(mx, s_mx[w]); }
  uint64_t* dst = user + wv.begin;
  if (mn == mx) {  // constant window: already sorted
    if (wv.buf) {
      for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) dst[i] = srcp[i];
    }
    return;
  }
  const uint64_t range = mx - mn;
  const int bl = 64 - __clzll((long long)range);
  const int sh = bl > 8 ? bl - 8 : 0;
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    uint32_t i = j * kBaseThreads + threadIdx.x;
    if (i < len) atomicAdd(&ccnt[(uint32_t)((okv[j] - mn) >> sh)], 1u);
  }
  for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) fh[i] = 0;
  __syncthreads();
  {
    uint32_t c = (threadIdx.x < 256) ? ccnt[threadIdx.x] : 0u;
    uint32_t ex = block_exclusive_scan<kBaseThreads>(c, s_warp, nullptr);
    if (threadIdx.x < 256) coff[threadIdx.x] = ex;
  }
  __syncthreads();
  uint32_t fb[kBaseItems];
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    uint32_t i = j * kBaseThreads + threadIdx.x;
    if (i < len) {
      uint64_t d = okv[j] - mn;
      uint32_t c = (uint32_t)(d >> sh);
      uint32_t f = coff[c];
      if (sh > 0) f += (uint32_t)__umul64hi((d - ((uint64_t)c << sh)) << (64 - sh), ccnt[c]);
      fb[j] = f;
      atomicAdd(&fh[f], 1u);
    }
  }
  __syncthreads();
  // exclusive scan of fh over [0, len): each thread owns kBaseItems consecutive bins
  uint32_t mxc = 0;
  {
    uint32_t base_i = threadIdx.x * kBaseItems;
    uint32_t loc[kBaseItems];
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) {
      uint32_t i = base_i + j;
      uint32_t c = (i < len) ? fh[i] : 0u;
      loc[j] = sum;
      sum += c;
      mxc = max(mxc, c);
    }
    uint32_t ex = block_exclusive_scan<kBaseThreads>(sum, s_warp, nullptr);
#pragma unroll
    for (int j = 0; j < kBaseItems; ++j) {
      uint32_t i = base_i + j;
      if (i < len) fh[i] = ex + loc[j];
    }
  }
  const bool overflow = __syncthreads_or(mxc > 24) != 0;
#pragma unroll
  for (int j = 0; j < kBaseItems; ++j) {
    uint32_t i = j * kBaseThreads + threadIdx.x;
    if (i < len) {
      uint32_t pos = atomicAdd(&fh[fb[j]], 1u);
      stage[pos] = okv[j];
    }
  }
  __syncthreads();
  if (!overflow) {
    for (uint32_t f = threadIdx.x; f < len; f += blockDim.x) {
      uint32_t beg = f ? fh[f - 1] : 0u, end = fh[f];
      for (uint32_t i = beg + 1; i < end; ++i) {
        uint64_t x = stage[i];
        uint32_t j = i;
        while (j > beg && stage[j - 1] > x) { stage[j] = stage[j - 1]; --j; }
        stage[j] = x;
      }
    }
  } else {
    uint32_t NP = 1;
    while (NP < len) NP <<= 1;
    for (uint32_t i = len + threadIdx.x; i < NP; i += blockDim.x) stage[i] = ~0ull;
    __syncthreads();
    for (uint32_t size = 2; size <= NP; size <<= 1) {
      for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
        for (uint32_t i = threadIdx.x; i < NP / 2; i += blockDim.x) {
          uint32_t lo = 2 * i - (i & (stride - 1));
          uint32_t hi = lo + stride;
          bool asc = (lo & size) == 0;
          uint64_t x = stage[lo], y = stage[hi];
          if ((x > y) == asc) { stage[lo] = y; stage[hi] = x; }
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) dst[i] = bits_of_ok<F64>(stage[i]);
  (void)s_flag;
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

__global__ void k_keys_to_ok_f64(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                 uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = ok_of_f64(in[i]);
}

}  // namespace ipls
