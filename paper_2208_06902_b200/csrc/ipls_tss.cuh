// ipls_tss.cuh — terminal segment sort: the last partition level fused with the base case
// (P:136-142).
//
// A terminal segment (every child <= base case) ends as its keys in ascending order: the
// base case sorts every child exactly (R13) and the children are range-ordered (the model is
// monotone, R7), so the level's output for the segment is the sorted segment, whatever order
// the children's keys had in between (R11).  Its level record (model, counts) comes from the
// fit and k_classify_scan as for every segment.  Instead of scattering the keys into k
// children and sorting every child again (two placements of every key through shared memory,
// windows of <= 256 keys per warp), the segment is cut into windows of whole children of
// <= kTW keys (segment_bases, from the child counts) and
//   k_tss_scatter  moves each key of a segment with several windows into its window (a
//                  handful of windows per segment: warp ranks from ballots, one smem
//                  placement, long coalesced runs; unstable, R11);
//   k_win_sort     sorts one window per CTA: an interpolation counting sort on the key value
//                  (two bins per key), then every position p of the placed window computes its
//                  key's rank inside its bin and stores the key to its final place -- a warp's
//                  32 positions land in a permutation of ~32 consecutive places, so the output
//                  is written coalesced straight from the fix-up.  Bins above kWSBig keys are
//                  sorted by a warp (a bitonic network); duplicate-only bins are copied.
// A segment of <= kTW keys is one window and is sorted where it lies: no scatter at all.
#pragma once

namespace ipls {

// ------------------------------------------------------------------------------------
// k_tss_scatter: one CTA per chunk of a terminal segment with >= 2 windows, 2 CTAs per SM.
// The chunk's share of window g starts at the window's begin plus the keys of the window's
// children in the segment's earlier chunks (k_classify_scan's per-(chunk, child) prefixes),
// so tiles advance a cursor per window in shared memory (no global atomics).
constexpr int kXThreads = 512;
constexpr int kXItems = 8;
constexpr int kXTile = kXThreads * kXItems;  // 4096

__host__ __device__ constexpr size_t tss_scatter_smem_bytes() {
  return (size_t)kXTile * 8 + (size_t)kXTile * 2 + (size_t)kMaxK * 2 + (size_t)kTWMaxWin * 4 * 4 + 64;
}

template <bool F64, int MODE>
__device__ void tss_scatter_chunk(const LevelArgs& a, uint64_t* __restrict__ dst_user,
                                  uint64_t* __restrict__ dst_scr, uint32_t c, const ChunkDesc& ch,
                                  const ModelDev& md, uint2 tw, unsigned char* smraw) {
  constexpr int NT = kXThreads;
  uint64_t* stage = reinterpret_cast<uint64_t*>(smraw);              // kXTile keys
  uint16_t* stg = reinterpret_cast<uint16_t*>(stage + kXTile);        // kXTile window ids
  uint16_t* gtab = stg + kXTile;                                      // kMaxK: child -> window
  uint32_t* cnt = reinterpret_cast<uint32_t*>(gtab + kMaxK);          // kTWMaxWin
  uint32_t* rs = cnt + kTWMaxWin;                                     // run start in the stage
  uint32_t* cur = rs + kTWMaxWin;                                     // next dst index (absolute)
  uint32_t* adj = cur + kTWMaxWin;                                    // dst index - stage index
  const uint32_t t = threadIdx.x, lane = t & 31;
  const uint32_t k = a.k;
  const SegDesc sg = a.segs[ch.seg];
  const uint32_t first = tw.x, Wp = tw.y & 0xffffu, G = tw.y >> 16;  // G >= 2
  uint64_t* dst = a.dstbuf ? dst_scr : dst_user;
  const Bucketer<F64, MODE> bucket(md, k);
  for (uint32_t g = t; g < G; g += NT) {
    cnt[g] = 0;
    cur[g] = (uint32_t)a.twins[first + g].begin;
  }
  __syncthreads();
  for (uint32_t b = t; b < k; b += NT) {
    const uint32_t g = ((uint32_t)(a.seg_dst[(size_t)ch.seg * k + b] & ~kDstUserBit) -
                        (uint32_t)sg.begin) / Wp;
    gtab[b] = (uint16_t)g;
    const uint32_t pre = a.chunk_pre[(size_t)c * k + b];  // child b's keys in earlier chunks
    if (pre) atomicAdd(&cur[g], pre);
  }
  const uint64_t* p = a.src + ch.start;
  uint64_t v[kXItems], vn[kXItems];
#pragma unroll
  for (int r = 0; r < kXItems; ++r) {
    const uint32_t i = r * NT + t;
    vn[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
  }
  __syncthreads();
  for (uint32_t t0 = 0; t0 < ch.len; t0 += kXTile) {
    const uint32_t tl = min((uint32_t)kXTile, ch.len - t0);
#pragma unroll
    for (int r = 0; r < kXItems; ++r) v[r] = vn[r];
    if (t0 + kXTile < ch.len) {
#pragma unroll
      for (int r = 0; r < kXItems; ++r) {
        const uint32_t i = t0 + kXTile + r * NT + t;
        vn[r] = (i < ch.len) ? __ldcs(p + i) : 0ull;
      }
    }
    // ---- (A) window of every key; its rank among the tile's keys of that window (the
    // order inside a window is free, R11: one shared-memory atomic per key, same-window
    // lanes of a warp served one after another) ----
    uint32_t rk[kXItems];  // window << 16 | rank
#pragma unroll
    for (int r = 0; r < kXItems; ++r) {
      if (r * NT + t < tl) {
        const uint32_t g = gtab[bucket(v[r])];
        rk[r] = (g << 16) | atomicAdd(&cnt[g], 1u);
      }
    }
    __syncthreads();
    // ---- (B) runs: stage starts, dst index - stage index per window ----
    if (t < 32) {
      uint32_t carry = 0;
      for (uint32_t g0 = 0; g0 < G; g0 += 32) {
        const uint32_t g = g0 + lane;
        const uint32_t cg = (g < G) ? cnt[g] : 0u;
        uint32_t inc = cg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= (uint32_t)o) inc += y;
        }
        if (g < G) {
          const uint32_t st = carry + inc - cg;
          rs[g] = st;
          adj[g] = cur[g] - st;
          cur[g] += cg;
          cnt[g] = 0;
        }
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    // ---- (C) placement into the stage, window-major ----
#pragma unroll
    for (int r = 0; r < kXItems; ++r) {
      if (r * NT + t < tl) {
        const uint32_t g = rk[r] >> 16;
        const uint32_t q = rs[g] + (rk[r] & 0xffffu);
        stage[q] = v[r];
        stg[q] = (uint16_t)g;
      }
    }
    __syncthreads();
    // ---- (D) write-out: runs of ~tile / G keys per window ----
#pragma unroll
    for (int r = 0; r < kXItems; ++r) {
      const uint32_t q = r * NT + t;
      if (q < tl) dst[adj[stg[q]] + q] = stage[q];
    }
  }
}

template <bool F64, bool TREE>
__global__ __launch_bounds__(kXThreads, 2) void k_tss_scatter(LevelArgs a, uint64_t* __restrict__ dst_user,
                                                             uint64_t* __restrict__ dst_scr) {
  const ChunkDesc ch = a.chunks[blockIdx.x];
  if (a.single_offsets || !a.seg_term[ch.seg]) return;  // k_scatter_stable's chunk
  if (*((volatile const uint32_t*)a.err) & kErrNan) return;
  const uint2 tw = a.seg_tw[ch.seg];
  if ((tw.y & 0xffffu) == 0) return;  // a one-window segment: k_win_sort reads it in place
  extern __shared__ __align__(128) unsigned char smraw[];
  ModelDev md = a.models[ch.seg];
  tree_top_to_smem<TREE, kXThreads>(md, a.k);
  constexpr int kMain = TREE ? (int)kModelTree : (int)kModelLinear;
  if (md.kind == kModelEq3)
    tss_scatter_chunk<F64, kModelEq3>(a, dst_user, dst_scr, blockIdx.x, ch, md, tw, smraw);
  else if (TREE && md.leaves != a.k)
    tss_scatter_chunk<F64, TREE ? (int)kModelTreeEq : kMain>(a, dst_user, dst_scr, blockIdx.x, ch, md, tw,
                                                            smraw);
  else
    tss_scatter_chunk<F64, kMain>(a, dst_user, dst_scr, blockIdx.x, ch, md, tw, smraw);
}

// ------------------------------------------------------------------------------------
// k_win_sort: one CTA sorts one window of <= kTW keys into the user array.
#ifndef IPLS_WS_THREADS
#define IPLS_WS_THREADS (kTW / 16)
#endif
constexpr int kWSThreads = IPLS_WS_THREADS;  // 1024 threads, 16 keys each at kTW = 16 Ki
constexpr int kWSItems = kTW / kWSThreads;
#ifndef IPLS_WS_OCC
#define IPLS_WS_OCC (kTW <= 8192 && kWSThreads <= 512 ? 2 : 1)
#endif
constexpr int kWSOcc = IPLS_WS_OCC;  // CTAs per SM (shared memory: ~12 B per key)
constexpr bool kWSReload = kWSItems > 8;  // keys reloaded at the placement instead of kept
constexpr uint32_t kWSBig = 32;                            // largest bin its keys rank themselves in
constexpr uint32_t kWSMaxBig = kTW / (kWSBig + 1) + 1;     // bins above kWSBig per window
static_assert(kWSItems % 4 == 0, "the scan reads its words as uint4");

__host__ __device__ constexpr size_t win_sort_smem_bytes() {
  return (size_t)kTW * 8 + (size_t)kTW * 4 + (size_t)kWSMaxBig * 8;
}

// Ascending sort of a[0, n) by one warp: bitonic network in the all-ascending form (each
// merge first compares i with its mirror in the block, then half-cleaners), so the virtual
// +inf padding up to the next power of two never moves and its comparators are skipped.
__device__ void warp_sort_range(uint64_t* a, uint32_t n, uint32_t lane) {
  uint32_t P = 1;
  while (P < n) P <<= 1;
  for (uint32_t size = 2; size <= P; size <<= 1) {
    const uint32_t half = size >> 1;
    for (uint32_t q = lane; q < P / 2; q += 32) {
      const uint32_t j = q & (half - 1);
      const uint32_t lo = (q - j) * 2 + j, hi = (q - j) * 2 + size - 1 - j;
      if (hi < n) {
        const uint64_t x = a[lo], y = a[hi];
        if (x > y) { a[lo] = y; a[hi] = x; }
      }
    }
    __syncwarp();
    for (uint32_t stride = half >> 1; stride > 0; stride >>= 1) {
      for (uint32_t q = lane; q < P / 2; q += 32) {
        const uint32_t lo = 2 * q - (q & (stride - 1)), hi = lo + stride;
        if (hi < n) {
          const uint64_t x = a[lo], y = a[hi];
          if (x > y) { a[lo] = y; a[hi] = x; }
        }
      }
      __syncwarp();
    }
  }
}

// Interpolation bin of a key: trunc((h x - h min) * scale) clamped to [0, nb), evaluated in
// binary64 with separately rounded operations (every step is monotone, so bins are ordered).
// f64: x the key (finite min/max of the window; +-inf land in the end bins; h = 1/2 if
// max - min overflows); u64: x = key - min converted (exact difference, RN).
struct WinBin {
  double mnh, h, scale;
  uint64_t umn;
  uint32_t nbm1;
  template <bool F64>
  __device__ __forceinline__ uint32_t of(uint64_t bits) const {
    double y;
    if constexpr (F64) y = __dadd_rn(__dmul_rn(__longlong_as_double((long long)bits), h), -mnh);
    else y = __ull2double_rn(bits - umn);
    return min(__double2uint_rz(__dmul_rn(y, scale)), nbm1);
  }
};

template <bool F64>
__global__ __launch_bounds__(kWSThreads, kWSOcc) void k_win_sort(const Window* __restrict__ wins,
                                                          uint64_t* __restrict__ user,
                                                          const uint64_t* __restrict__ scr,
                                                          const uint32_t* __restrict__ err) {
  constexpr int NT = kWSThreads, ITEMS = kWSItems, NW = NT / 32;
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* Bk = reinterpret_cast<uint64_t*>(smraw);          // kTW ordering keys, bin-major
  uint32_t* bins = reinterpret_cast<uint32_t*>(Bk + kTW);      // kTW words: two u16 bins each
  uint2* big = reinterpret_cast<uint2*>(bins + kTW);           // bins above kWSBig
  __shared__ uint64_t s_lo[NW], s_hi[NW];
  __shared__ uint32_t s_warp[40];
  __shared__ uint32_t s_nbig;
  if (*((volatile const uint32_t*)err) & kErrNan) return;
  const Window wv = wins[blockIdx.x];
  const uint32_t len = wv.len;
  const uint64_t* src = (wv.buf ? scr : user) + wv.begin;
  uint64_t* dst = user + wv.begin;
  const uint32_t t = threadIdx.x, lane = t & 31, wp = t >> 5;
  uint64_t v[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t i = j * NT + t;
    v[j] = (i < len) ? (kWSReload ? __ldg(src + i) : __ldcs(src + i)) : 0ull;  // __ldg: kept in the L2 for the reload
  }
  const uint32_t nb = 2 * len;          // bins; words [0, len)
  const uint32_t nwz = (len + ITEMS - 1) / ITEMS * ITEMS;
  {
    uint4* b4 = reinterpret_cast<uint4*>(bins);
    for (uint32_t q = t; q < nwz / 4; q += NT) b4[q] = make_uint4(0, 0, 0, 0);
  }
  if (t == 0) s_nbig = 0;
  // ---- window bounds ----
  WinBin wb;
  wb.nbm1 = nb - 1;
  if constexpr (F64) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    double mn = inf, mx = -inf;  // finite keys only
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const double x = __longlong_as_double((long long)v[j]);
      const double xf = (j * NT + t < len && fabs(x) < inf) ? x : __longlong_as_double(0x7ff8000000000000ll);
      mn = xf < mn ? xf : mn;  // the NaN of excluded slots compares false
      mx = xf > mx ? xf : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
      mn = a < mn ? a : mn;
      mx = b > mx ? b : mx;
    }
    if (lane == 0) { s_lo[wp] = (uint64_t)__double_as_longlong(mn); s_hi[wp] = (uint64_t)__double_as_longlong(mx); }
    __syncthreads();
    mn = __longlong_as_double((long long)s_lo[lane % NW]);
    mx = __longlong_as_double((long long)s_hi[lane % NW]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
      mn = a < mn ? a : mn;
      mx = b > mx ? b : mx;
    }
    if (!(mn <= mx)) { mn = 0.0; mx = 0.0; }  // no finite key
    double h = 1.0, range = __dadd_rn(mx, -mn);
    if (!(range < inf)) {
      h = 0.5;
      range = __dadd_rn(__dmul_rn(mx, 0.5), -__dmul_rn(mn, 0.5));
    }
    wb.h = h;
    wb.mnh = __dmul_rn(mn, h);
    wb.scale = range > 0.0 ? __ddiv_rn((double)nb, range) : 1.0;
    wb.umn = 0;
  } else {
    uint64_t umn = ~0ull, umx = 0;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j)
      if (j * NT + t < len) { umn = min(umn, v[j]); umx = max(umx, v[j]); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      umn = min(umn, __shfl_xor_sync(0xffffffffu, umn, o));
      umx = max(umx, __shfl_xor_sync(0xffffffffu, umx, o));
    }
    if (lane == 0) { s_lo[wp] = umn; s_hi[wp] = umx; }
    __syncthreads();
    umn = s_lo[lane % NW];
    umx = s_hi[lane % NW];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      umn = min(umn, __shfl_xor_sync(0xffffffffu, umn, o));
      umx = max(umx, __shfl_xor_sync(0xffffffffu, umx, o));
    }
    const double range = __ull2double_rn(umx - umn);
    wb.h = 1.0; wb.mnh = 0.0;
    wb.umn = umn;
    wb.scale = range > 0.0 ? __ddiv_rn((double)nb, range) : 1.0;
  }
  // ---- histogram: the atomic returns the key's arrival rank in its bin ----
  uint32_t fr[ITEMS];  // bin | rank << 16
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    fr[j] = 0;
    if (j * NT + t < len) {
      const uint32_t f = wb.of<F64>(v[j]);
      const uint32_t sh = (f & 1u) << 4;
      const uint32_t old = atomicAdd(&bins[f >> 1], 1u << sh);
      fr[j] = f | (((old >> sh) & 0xffffu) << 16);
    }
  }
  __syncthreads();
  // ---- exclusive scan of the bin counts: thread t owns words [ITEMS t, ITEMS t + ITEMS) ----
  uint32_t mxc = 0;  // this thread's largest bin
  {
    uint32_t sum = 0;
    const bool mine = t * ITEMS < nwz;
    uint4* b4 = reinterpret_cast<uint4*>(bins) + t * (ITEMS / 4);
    if (mine) {
#pragma unroll
      for (int q = 0; q < ITEMS / 4; ++q) {
        const uint4 c = b4[q];
        const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t lo = w[e] & 0xffffu, hi = w[e] >> 16;
          sum += lo + hi;
          mxc = max(mxc, max(lo, hi));
        }
      }
    }
    uint32_t run = block_exclusive_scan<NT>(sum, s_warp, nullptr);
    if (mine) {
#pragma unroll
      for (int q = 0; q < ITEMS / 4; ++q) {
        const uint4 c = b4[q];
        uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t lo = w[e] & 0xffffu, hi = w[e] >> 16;
          w[e] = run | ((run + lo) << 16);
          run += lo + hi;
        }
        b4[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  // bins above kWSBig are rare: the fix-up lists them (a second barrier below only if any)
  const bool any_big = __syncthreads_or(mxc > kWSBig) != 0;
  // ---- placement: bin start + arrival rank.  A key alone in its bin is at its final
  // place.  Keys of bins of 2..kWSBig keys (two bins per key: ~40 % of the keys in bins of
  // ~2.5) are listed and ranked inside their bin after the write-out, one list entry per
  // lane (no lane idles behind a neighbour's bin); bins above kWSBig go to a warp each ----
  auto start_of = [&](uint32_t f) -> uint32_t { return (bins[f >> 1] >> ((f & 1u) << 4)) & 0xffffu; };
  uint32_t multi = 0;  // items in bins of 2..kWSBig keys; fr[j] becomes start | rank << 15 | c << 20
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    if (j * NT + t < len) {
      const uint32_t f = fr[j] & 0xffffu, r = fr[j] >> 16;
      const uint32_t s0 = start_of(f);
      const uint32_t c = ((f < wb.nbm1) ? start_of(f + 1) : len) - s0;
      // the key is reloaded (an L2 hit) rather than kept in registers since the histogram
      Bk[s0 + r] = ok_of<F64>(kWSReload ? __ldcs(src + j * NT + t) : v[j]);
      if (c >= 2) {
        if (c <= kWSBig) {
          multi |= 1u << j;
          fr[j] = s0 | (r << 15) | (c << 20);
        } else if (r == 0) {
          big[atomicAdd(&s_nbig, 1u)] = make_uint2(s0, s0 + c);
        }
      }
    }
  }
  if (t == 0) s_warp[39] = 0;
  __syncthreads();
  // ---- list of the multi-key bins' keys (in the bins' words, free now) ----
  uint32_t* list = bins;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const bool m = (multi >> j) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, m);
    uint32_t base = 0;
    if (lane == 0 && bal) base = atomicAdd(&s_warp[39], (uint32_t)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (m) list[base + __popc(bal & lanemask_lt())] = fr[j];
  }
  if (any_big) {
    __syncthreads();
    // ---- bins above kWSBig: one warp each (duplicate-only bins stay as they are) ----
    const uint32_t nbig = s_nbig;
    for (uint32_t i = wp; i < nbig; i += NW) {
      const uint2 se = big[i];
      uint64_t* a = Bk + se.x;
      const uint32_t n = se.y - se.x;
      const uint64_t o0 = a[0];
      bool same = true;
      for (uint32_t q = lane; q < n; q += 32) same &= a[q] == o0;
      if (!__all_sync(0xffffffffu, same)) warp_sort_range(a, n, lane);
    }
  }
  __syncthreads();
  // ---- write-out, coalesced (the listed keys' slots are rewritten below) ----
#pragma unroll 4
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t p = j * NT + t;
    if (p < len) __stcs(dst + p, bits_of_ok<F64>(Bk[p]));
  }
  const uint32_t nmulti = s_warp[39];
  __syncthreads();  // the stores above precede the ones below (same addresses)
  // ---- listed keys: rank among the bin's keys (smaller keys, equal keys placed before) ----
  for (uint32_t i = t; i < nmulti; i += NT) {
    const uint32_t e = list[i];
    const uint32_t s0 = e & 0x7fffu, r = (e >> 15) & 31u, c = e >> 20;
    const uint64_t x = Bk[s0 + r];
    uint32_t rr = 0;
    for (uint32_t q = 0; q < c; ++q) {
      const uint64_t y = Bk[s0 + q];
      rr += (y < x || (y == x && q < r)) ? 1u : 0u;
    }
    __stcs(dst + s0 + rr, bits_of_ok<F64>(x));
  }
}

}  // namespace ipls
