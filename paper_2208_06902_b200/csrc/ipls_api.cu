// ipls_api.cu — C ABI (include/ipls.h) and the host-side level scheduler.
//
// The host owns only control: workspace carve-up, the level loop (one batched launch per
// kernel per level, P:120-121 recursion batched by level), and one small device->host read of
// the next level's counters per level.  Every step of the path runs in the kernels of
// ipls_kernels.cuh; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/ipls.h"
#include "ipls_kernels.cuh"
#include "ipls_tss.cuh"

using namespace ipls;

namespace {

std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_term_mode{0};  // ipls_debug_term_mode: 0 auto, 1 k_term_fused, 2 separate, 3 window sort
thread_local std::string g_last_cuda_error;

struct CudaFail {
  cudaError_t e;
};

inline void ck(cudaError_t e) {
  if (e != cudaSuccess) throw CudaFail{e};
}
inline void ck_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  ck(cudaGetLastError());
}

// Optional per-kernel CUDA-event timing (ipls_profile_*): events bracket each launch on its
// stream; durations are folded in when the call synchronises (prof_collect).
struct ProfAcc {
  uint64_t launches = 0;
  double ms = 0.0, bytes = 0.0;
};
struct ProfPending {
  const char* name;
  double bytes;
  cudaEvent_t e0, e1;
};
std::atomic<int> g_prof_on{0};
std::mutex g_prof_mu;
std::map<std::string, ProfAcc> g_prof;
thread_local std::vector<ProfPending> t_pending;
thread_local std::vector<cudaEvent_t> t_event_pool;

cudaEvent_t prof_event() {
  if (!t_event_pool.empty()) {
    cudaEvent_t e = t_event_pool.back();
    t_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  ck(cudaEventCreate(&e));
  return e;
}

struct ProfScope {
  bool on;
  ProfPending p;
  cudaStream_t st;
  ProfScope(const char* name, double bytes, cudaStream_t s) : on(g_prof_on.load() != 0), st(s) {
    if (on) {
      p.name = name; p.bytes = bytes; p.e0 = prof_event(); p.e1 = prof_event();
      ck(cudaEventRecord(p.e0, st));
    }
  }
  ~ProfScope() {
    if (on) {
      cudaEventRecord(p.e1, st);
      t_pending.push_back(p);
    }
  }
};

void prof_collect() {
  if (t_pending.empty()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& p : t_pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.e1) == cudaSuccess && cudaEventElapsedTime(&ms, p.e0, p.e1) == cudaSuccess) {
      ProfAcc& a = g_prof[p.name];
      a.launches += 1;
      a.ms += ms;
      a.bytes += p.bytes;
    }
    t_event_pool.push_back(p.e0);
    t_event_pool.push_back(p.e1);
  }
  t_pending.clear();
}
// algorithmic bytes known only after a level (the base case inside k_term_fused)
void prof_add_bytes(const char* name, double bytes) {
  if (!g_prof_on.load() || bytes == 0.0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof[name].bytes += bytes;
}
#define IPLS_CAT2(a, b) a##b
#define IPLS_CAT(a, b) IPLS_CAT2(a, b)
#define IPLS_PROF(name, bytes) ProfScope IPLS_CAT(_prof_scope_, __LINE__)(name, (double)(bytes), st)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Params {
  uint64_t n;
  uint32_t k, B, chunk_keys;
  uint32_t cap_segs, cap_chunks, cap_samples, cap_wins, cap_wbig, cap_fills, cap_twin;
  bool tree;  // IPLS_FLAG_TREE_MODEL: splitter-tree model instead of FMCD
  uint32_t tree_leaves;  // tree: k, or k / 2 with IPLS_FLAG_TREE_EQUAL_BUCKETS (R24)
};

#ifndef IPLS_CHUNK_CAP
#define IPLS_CHUNK_CAP 114688  // 112 Ki: C5 -0.6 % against 96 Ki (interleaved A/B; C2-C4 unchanged)
#endif
uint32_t pick_chunk_keys(uint64_t n) {
  // ~8 chunks per SM at level 0 (148 SMs), 4096..IPLS_CHUNK_CAP keys; from 16384 keys up a multiple of
  // the terminal scatter's 16384-key tile.  Larger chunks amortise each chunk's k-wide
  // lookback, histogram and run setup (98304 keys: C2 -1.2 %, C5 -1.2 % against 65536).
  uint64_t c = n / (148 * 8);
  if (c >= 16384) c = (c + 16383) / 16384 * 16384;
  else c = (c + kCTile - 1) / kCTile * kCTile;
  if (c < (uint64_t)kCTile) c = kCTile;
  if (c > IPLS_CHUNK_CAP) c = IPLS_CHUNK_CAP;
  return (uint32_t)c;
}

Params make_params(uint64_t n, uint32_t k, uint32_t B, bool tree = false, bool tree_eq = false) {
  Params p{};
  p.n = n; p.k = k; p.B = B; p.tree = tree;
  p.tree_leaves = tree ? (tree_eq ? k / 2 : k) : 0;
  p.chunk_keys = pick_chunk_keys(n);
  const uint64_t segs = n / ((uint64_t)B + 1) + 2;
  const uint64_t chunks = n / p.chunk_keys + segs + 1;
  const uint64_t smax = sample_size(n, k);
  uint64_t samples = std::min<uint64_t>(n / 2 + 8, segs * smax + 8);
  // small windows: greedy packing makes consecutive windows of a run exceed kWBCap keys
  // together, runs are cut by breakers (<= n / (kWBCap + 1) big base children and <= segs
  // partition/homogeneous children per level) and by segment ends
  uint64_t wins = std::min<uint64_t>(n + 1, 2 * n / kWBCap + 2 * (n / (kWBCap + 1)) + 4 * segs) + 64;
  uint64_t wbig = std::min<uint64_t>(n / (kWBCap + 1), 2 * n / kBigCap + 2 * (n / (kWBCap + 1)) + 4 * segs) + 64;
  uint64_t fills = n / ((uint64_t)B + 1) + 16;
  p.cap_segs = (uint32_t)segs;
  p.cap_chunks = (uint32_t)chunks;
  p.cap_samples = (uint32_t)samples;
  p.cap_wins = (uint32_t)wins;
  p.cap_wbig = (uint32_t)wbig;
  p.cap_fills = (uint32_t)fills;
  // terminal windows: a segment of m keys has <= ceil(m / (kTW - 4096)) of them
  p.cap_twin = (uint32_t)std::min<uint64_t>(n / (kTW - 4096) + segs + 64, 0xffffffffull);
  return p;
}

// Fixed part of the workspace: scratch keys + descriptors of two levels + windows/fills of
// two levels + counters.  The k-scaled per-level metadata is carved after it.
struct FixedLayout {
  size_t scratch, segs[2], chunks[2], wins[2], wbig[2], fills[2], ctr[2], twins, twcur, err, tickets,
      total;
};

FixedLayout fixed_layout(const Params& p) {
  FixedLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.scratch = take(p.n * 8);
  for (int i = 0; i < 2; ++i) {
    L.segs[i] = take((size_t)p.cap_segs * sizeof(SegDesc));
    L.chunks[i] = take((size_t)p.cap_chunks * sizeof(ChunkDesc));
    L.wins[i] = take((size_t)p.cap_wins * sizeof(Window));
    L.wbig[i] = take((size_t)p.cap_wbig * sizeof(Window));
    L.fills[i] = take((size_t)p.cap_fills * sizeof(Fill));
    L.ctr[i] = take(sizeof(LevelCounters));
  }
  L.twins = take((size_t)p.cap_twin * sizeof(Window));
  L.twcur = take((size_t)p.cap_twin * 4);
  L.err = take(16);
  L.tickets = take(64);
  L.total = o;
  return L;
}

// Per-level metadata (sized by the level's actual counts).  `status` comes first so a fresh
// allocation can be cleared cheaply.
struct MetaLayout {
  size_t status, cflag, cref, chunk_pre, models, samples, seg_dst, seg_tot, seg_term, seg_done,
      seg_tw, tree, total;
};

MetaLayout meta_layout(uint64_t segs, uint64_t chunks, uint64_t samples, uint32_t k,
                       bool tree = false) {
  MetaLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.status = take(chunks * k * 8);
  L.cflag = take(chunks * k);
  L.cref = take(chunks * k * 8);
  L.chunk_pre = take(chunks * k * 4);
  L.models = take(segs * sizeof(ModelDev));
  L.samples = take(samples * 8 + 64);
  L.seg_dst = take(segs * k * 8);
  L.seg_tot = take(segs * k * 4);
  L.seg_term = take(segs * 4);
  L.seg_done = take(segs * 4);
  L.seg_tw = take(segs * 8);
  L.tree = take(tree ? segs * kMaxK * 8 : 0);  // splitter heaps (8 KB per segment)
  L.total = o;
  return L;
}

// The caller-workspace path never traces, and the level's sorted samples are kept only for
// the trace (the fit kernels keep them on chip), so the worst case reserves no sample space.
size_t worst_meta_bytes(const Params& p) {
  return meta_layout(p.cap_segs, p.cap_chunks, 0, p.k, p.tree).total;
}

// Device buffers for one call: either the caller's workspace or the per-stream cache.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  bool fresh = false;  // set when (re)allocated: lookback status words must be cleared
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  void ensure(size_t want) {
    if (bytes >= want) return;
    release();
    ck(cudaMalloc(&ptr, want));
    bytes = want;
    fresh = true;
  }
};

struct StreamCache {
  DevBuf fixed, meta, io;          // io: device copy for ipls_sort_host
  LevelCounters* h_ctr = nullptr;  // pinned
  StreamCache() { ck(cudaMallocHost((void**)&h_ctr, 2 * sizeof(LevelCounters) + 64)); }
  ~StreamCache() {
    fixed.release(); meta.release(); io.release();
    if (h_ctr) cudaFreeHost(h_ctr);
  }
};

std::mutex g_mu;
std::map<std::pair<int, void*>, std::unique_ptr<StreamCache>> g_cache;
std::atomic<uint32_t> g_epoch{0};

StreamCache& cache_for(void* stream) {
  int dev = 0;
  ck(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, stream);
  auto it = g_cache.find(key);
  if (it == g_cache.end()) it = g_cache.emplace(key, std::make_unique<StreamCache>()).first;
  return *it->second;
}

template <typename T>
T* at(void* base, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

// ---------------------------------------------------------------------------------------
struct TraceSink {
  ipls_trace* tr;
  uint32_t k;
  bool f64;
  std::vector<ipls_segment_record> recs;
  std::vector<std::vector<uint64_t>> counts, samples;
};

size_t scatter_stable_smem(uint32_t k) { return scatter_stable_smem_bytes(k); }
size_t scatter_term_smem(uint32_t k) { return scatter_term_smem_bytes(k); }

uint32_t num_sms();
// Both scatter kernels over the level's chunks: each one takes its own kind of chunk (stable
// or terminal, known on the device after K2) and returns at once for the other.
template <bool F64>
void launch_scatter(uint32_t nchunk, cudaStream_t st, const LevelArgs& la, uint64_t* user,
                    uint64_t* scr, bool tree = false, bool stable_only = false) {
  {
  IPLS_PROF("scatter_stable", 0);
  if (tree)
    k_scatter_stable<F64, true><<<nchunk, kSThreads, scatter_stable_smem(la.k), st>>>(la, user, scr);
  else
    k_scatter_stable<F64, false><<<nchunk, kSThreads, scatter_stable_smem(la.k), st>>>(la, user, scr);
  ck_launch();
  }
  if (stable_only) return;
  if (la.tss) {
    // terminal segments of several windows: keys into their windows (k_win_sort after the level)
    IPLS_PROF("tss_scatter", 0);
    if (tree)
      k_tss_scatter<F64, true><<<nchunk, kXThreads, tss_scatter_smem_bytes(), st>>>(la, user, scr);
    else
      k_tss_scatter<F64, false><<<nchunk, kXThreads, tss_scatter_smem_bytes(), st>>>(la, user, scr);
    ck_launch();
    return;
  }
  if (la.fused_term) {
    // terminal chunks, each terminal segment base-sorted by the CTA that completes it
    IPLS_PROF("term_fused", 0);
    const uint32_t grid = std::min(nchunk, num_sms());
    if (tree)
      k_term_fused<F64, true><<<grid, kTThreads, fused_smem_bytes(la.k), st>>>(la, user, scr, nchunk);
    else
      k_term_fused<F64, false><<<grid, kTThreads, fused_smem_bytes(la.k), st>>>(la, user, scr, nchunk);
    ck_launch();
    return;
  }
  IPLS_PROF("scatter_term", 0);
  if (tree)
    k_scatter_term<F64, true><<<nchunk, kTThreads, scatter_term_smem(la.k), st>>>(la, user, scr);
  else
    k_scatter_term<F64, false><<<nchunk, kTThreads, scatter_term_smem(la.k), st>>>(la, user, scr);
  ck_launch();
}
template <bool F64>
void launch_classify(uint32_t nchunk, cudaStream_t st, const LevelArgs& la, bool tree = false);
size_t classify_smem(uint32_t k) { return (size_t)k * 4; }
template <bool F64>
void launch_classify(uint32_t nchunk, cudaStream_t st, const LevelArgs& la, bool tree) {
  if (tree)
    k_classify_scan<F64, true><<<nchunk, kCThreads, classify_smem(la.k), st>>>(la);
  else
    k_classify_scan<F64, false><<<nchunk, kCThreads, classify_smem(la.k), st>>>(la);
  ck_launch();
}
size_t warp_base_smem() { return kWBSmemPerWarp * kWBWarps; }
size_t base_smem() { return kBCSmem; }
uint32_t num_sms() {
  int dev = 0, n = 0;
  ck(cudaGetDevice(&dev));
  ck(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return (uint32_t)n;
}
uint32_t fit_cap(uint32_t maxS) {
  uint32_t c = 64;
  while (c < maxS) c <<= 1;
  return c;
}
size_t fit_smem(uint32_t cap) { return (size_t)cap * 20; }

// The dynamic-smem limits are per (device context, kernel): set once per device, under a
// lock (first calls may race from several threads).
template <bool F64>
void set_attrs() {
  int dev = 0;
  ck(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return;
  ck(cudaFuncSetAttribute(k_gather_fit<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)fit_smem(kFitMaxS)));
  ck(cudaFuncSetAttribute(k_fit_small<F64, kFSThreads, kFSItems>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFSSmem));
  ck(cudaFuncSetAttribute(k_fit_small<F64, kFSThreads, kFMItems>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFMSmem));
  ck(cudaFuncSetAttribute(k_fit_small<F64, kFLThreads, kFLItems>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFLSmem));
  ck(cudaFuncSetAttribute(k_base_sort<F64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)base_smem()));
  ck(cudaFuncSetAttribute(k_base_sort<F64, F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)base_smem()));
  ck(cudaFuncSetAttribute(k_base_warp<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)warp_base_smem()));
  ck(cudaFuncSetAttribute(k_scatter_peer<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)scatter_peer_smem_bytes(kMaxK)));
  for (int tr = 0; tr < 2; ++tr) {
    ck(cudaFuncSetAttribute(tr ? k_classify_scan<F64, true> : k_classify_scan<F64, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)classify_smem(kMaxK)));
    ck(cudaFuncSetAttribute(tr ? k_scatter_stable<F64, true> : k_scatter_stable<F64, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)scatter_stable_smem(kMaxK)));
    ck(cudaFuncSetAttribute(tr ? k_scatter_term<F64, true> : k_scatter_term<F64, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)scatter_term_smem(kMaxK)));
    ck(cudaFuncSetAttribute(tr ? k_term_fused<F64, true> : k_term_fused<F64, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)fused_smem_bytes(kMaxK)));
    ck(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)win_scratch_bytes(kMaxK)));
    ck(cudaFuncSetAttribute(tr ? k_tss_scatter<F64, true> : k_tss_scatter<F64, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)tss_scatter_smem_bytes()));
  }
  ck(cudaFuncSetAttribute(k_win_sort<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)win_sort_smem_bytes()));
  done.insert(dev);
}

uint32_t next_epoch(bool* wrapped) {
  uint32_t e = g_epoch.fetch_add(1) + 1;
  *wrapped = (e & 0xffff) == 0;
  if (*wrapped) e = g_epoch.fetch_add(1) + 1;
  return e & 0xffff;
}

// ipls_sort_segments: the array is nseg consecutive range-ordered segments; the recursion
// resumes at `level` (the hash level of R18) with them as its segments.
struct InitSegs {
  const uint64_t* sizes;  // host, nseg entries summing to n
  uint32_t nseg;
  uint32_t level;
  uint64_t hash_base;     // position of the array in the one whose recursion is resumed
};

// Greedy left-to-right packing of the base-case segments of an initial segment list into
// windows (small: <= kWBCap keys each, packed to <= kWBCap; big: packed to <= kBigCap); a
// segment of the other classes breaks a window (as pack_windows does on the device).
void pack_initial(const InitSegs& in, uint32_t B, std::vector<Window>& small,
                  std::vector<Window>& big, uint64_t& small_keys, uint64_t& big_keys) {
  Window cs{0, 0, 0}, cb{0, 0, 0};
  auto flush = [](Window& w, std::vector<Window>& out, uint64_t& keys) {
    if (w.len) { out.push_back(w); keys += w.len; }
    w.len = 0;
  };
  uint64_t pos = 0;
  for (uint32_t i = 0; i < in.nseg; ++i) {
    const uint64_t m = in.sizes[i];
    const bool is_small = m > 0 && m <= (uint64_t)kWBCap;
    const bool is_big = m > (uint64_t)kWBCap && m <= B;
    if (m > 0 && !is_small) flush(cs, small, small_keys);
    if (m > 0 && !is_big) flush(cb, big, big_keys);
    if (is_small) {
      if (cs.len && cs.len + m > (uint64_t)kWBCap) flush(cs, small, small_keys);
      if (!cs.len) cs.begin = pos;
      cs.len += (uint32_t)m;
    } else if (is_big) {
      if (cb.len && cb.len + m > (uint64_t)kBigCap) flush(cb, big, big_keys);
      if (!cb.len) cb.begin = pos;
      cb.len += (uint32_t)m;
    }
    pos += m;
  }
  flush(cs, small, small_keys);
  flush(cb, big, big_keys);
}

// Run the whole level-batched sort.  keys: device array (user buffer).  init: nullptr for a
// whole sort (root segment at level 0), else the segments to resume from.
template <bool F64>
ipls_status run_sort(uint64_t* keys, const Params& p, void* fixed, void* d_meta_in,
                     size_t meta_bytes_in, DevBuf* meta_cache, LevelCounters* h_ctr,
                     cudaStream_t st, uint64_t seed, TraceSink* trace,
                     const InitSegs* init = nullptr) {
  set_attrs<F64>();
  const FixedLayout FL = fixed_layout(p);
  uint64_t* scr = at<uint64_t>(fixed, FL.scratch);
  uint32_t* d_err = at<uint32_t>(fixed, FL.err);
  ck(cudaMemsetAsync(d_err, 0, 16, st));
  const uint64_t n = p.n;
  const uint32_t k = p.k;

  const uint32_t level0 = init ? init->level : 0u;
  const uint64_t hbase = init ? init->hash_base : 0u;  // sampling hash: segment begin + hbase
  if (!init && n <= p.B) {
    // The root is a base-case segment: one window in place.
    Window w{0, (uint32_t)n, 0};
    Window* dw = at<Window>(fixed, FL.wins[0]);
    ck(cudaMemcpyAsync(dw, &w, sizeof(Window), cudaMemcpyHostToDevice, st));
    {
      IPLS_PROF("base_sort", 16.0 * n);
      k_base_sort<F64, F64><<<1, kBCThreads, base_smem(), st>>>(dw, keys, scr, d_err);
      ck_launch();
    }
    ck(cudaMemcpyAsync(&h_ctr[1].err, d_err, 4, cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    if (h_ctr[1].err & kErrNan) return IPLS_ERR_NAN_KEY;
    return IPLS_OK;
  }

  uint32_t nseg = 1, nchunk = 0, nsample = 0, max_S = 0;
  uint64_t level_keys = n;
  LevelCounters init_ctr{};  // the initial segments' base-case windows (counted as level 0's)
  ck(cudaMemsetAsync(at<LevelCounters>(fixed, FL.ctr[0]), 0, sizeof(LevelCounters), st));
  if (!init) {
    // level-0 work: the root segment
    nchunk = (uint32_t)((n + p.chunk_keys - 1) / p.chunk_keys);
    nsample = sample_size(n, k);
    max_S = nsample;
    k_init_root<<<std::max<uint32_t>(1, (nchunk + 255) / 256), 256, 0, st>>>(
        at<SegDesc>(fixed, FL.segs[0]), at<ChunkDesc>(fixed, FL.chunks[0]), n, nsample,
        p.chunk_keys, 0u);
    ck_launch();
  } else {
    if (F64) {  // NaN anywhere: rejected before any write (R0)
      k_nan_scan<<<num_sms() * 4, 256, 0, st>>>(keys, n, d_err);
      ck_launch();
      ck(cudaMemcpyAsync(&h_ctr[1].err, d_err, 4, cudaMemcpyDeviceToHost, st));
      ck(cudaStreamSynchronize(st));
      if (h_ctr[1].err & kErrNan) return IPLS_ERR_NAN_KEY;
    }
    std::vector<SegDesc> hs;
    std::vector<ChunkDesc> hc;
    std::vector<Window> hw, hwb;
    uint64_t wk = 0, wbk = 0, pos = 0;
    nsample = 0;
    level_keys = 0;
    for (uint32_t i = 0; i < init->nseg; ++i) {
      const uint64_t m = init->sizes[i];
      if (m > p.B) {
        SegDesc sd{};
        sd.begin = pos; sd.m = (uint32_t)m; sd.S = sample_size(m, k); sd.sample_off = nsample;
        const uint32_t nch = chunks_of((uint32_t)m, p.chunk_keys), per = (uint32_t)((m + nch - 1) / nch);
        sd.chunk_first = (uint32_t)hc.size(); sd.nchunks = nch; sd.flags = 0;
        for (uint32_t j = 0; j < nch; ++j)
          hc.push_back(ChunkDesc{pos + (uint64_t)j * per,
                                 (uint32_t)std::min<uint64_t>(per, m - (uint64_t)j * per),
                                 (uint32_t)hs.size()});
        hs.push_back(sd);
        nsample += sd.S;
        max_S = std::max(max_S, sd.S);
        level_keys += m;
      }
      pos += m;
    }
    pack_initial(*init, p.B, hw, hwb, wk, wbk);
    if (hs.size() > p.cap_segs || hc.size() > p.cap_chunks || hw.size() > p.cap_wins ||
        hwb.size() > p.cap_wbig)
      return IPLS_ERR_OUT_OF_MEMORY;
    if (!hs.empty()) {
      ck(cudaMemcpy(at<SegDesc>(fixed, FL.segs[0]), hs.data(), hs.size() * sizeof(SegDesc),
                    cudaMemcpyHostToDevice));
      ck(cudaMemcpy(at<ChunkDesc>(fixed, FL.chunks[0]), hc.data(), hc.size() * sizeof(ChunkDesc),
                    cudaMemcpyHostToDevice));
    }
    if (!hw.empty())
      ck(cudaMemcpy(at<Window>(fixed, FL.wins[0]), hw.data(), hw.size() * sizeof(Window),
                    cudaMemcpyHostToDevice));
    if (!hwb.empty())
      ck(cudaMemcpy(at<Window>(fixed, FL.wbig[0]), hwb.data(), hwb.size() * sizeof(Window),
                    cudaMemcpyHostToDevice));
    init_ctr.n_windows = (uint32_t)hw.size(); init_ctr.win_keys = wk;
    init_ctr.n_wbig = (uint32_t)hwb.size(); init_ctr.wbig_keys = wbk;
    nseg = (uint32_t)hs.size();
    nchunk = (uint32_t)hc.size();
    if (nseg == 0) {  // every segment goes to the base case
      if (hw.size()) {
        IPLS_PROF("base_warp", 16.0 * wk);
        k_base_warp<F64><<<std::min<uint32_t>(((uint32_t)hw.size() + kWBWarps - 1) / kWBWarps, num_sms()),
                           kWBWarps * 32, warp_base_smem(), st>>>(at<Window>(fixed, FL.wins[0]),
                                                                  (uint32_t)hw.size(), keys, scr);
        ck_launch();
      }
      if (hwb.size()) {
        IPLS_PROF("base_sort", 16.0 * wbk);
        k_base_sort<F64, false><<<(uint32_t)hwb.size(), kBCThreads, base_smem(), st>>>(
            at<Window>(fixed, FL.wbig[0]), keys, scr, d_err);
        ck_launch();
      }
      ck(cudaStreamSynchronize(st));
      return IPLS_OK;
    }
  }

  for (uint32_t iter = 0; nseg > 0; ++iter) {
    const uint32_t level = level0 + iter;  // the sampling hash's level (R18)
    const int cur = iter & 1, nxt = cur ^ 1;
    const uint64_t* src = (cur == 0) ? keys : scr;
    SegDesc* segs = at<SegDesc>(fixed, FL.segs[cur]);
    ChunkDesc* chunks = at<ChunkDesc>(fixed, FL.chunks[cur]);
    LevelCounters* cctr = at<LevelCounters>(fixed, FL.ctr[cur]);
    LevelCounters* nctr = at<LevelCounters>(fixed, FL.ctr[nxt]);
    Window* wins = at<Window>(fixed, FL.wins[cur]);
    Window* wbig = at<Window>(fixed, FL.wbig[cur]);
    Fill* fills = at<Fill>(fixed, FL.fills[cur]);

    // per-level metadata, sized by this level's actual counts
    const MetaLayout ML = meta_layout(nseg, nchunk, trace ? nsample : 0, k, p.tree);
    void* meta = d_meta_in;
    if (meta_cache) {
      meta_cache->ensure(ML.total);
      meta = meta_cache->ptr;
      if (meta_cache->fresh) {
        ck(cudaMemsetAsync(meta, 0, meta_cache->bytes, st));
        meta_cache->fresh = false;
      }
    } else {
      if (ML.total > meta_bytes_in) return IPLS_ERR_OUT_OF_MEMORY;
    }
    bool wrapped = false;
    const uint32_t epoch = next_epoch(&wrapped);
    // The status region is cleared at EVERY level: the layout is sized per level, so this
    // level's status words overlap what earlier levels (and calls) stored there — cref keys,
    // prefixes — and a stale 64-bit word whose top 16 bits happen to equal the epoch tag would
    // pass the lookback's validity test (an f64 key near 1.0 carries 0x3ff0 there).  ~2 us
    // per level; the epoch tag still orders the words written within the level.
    (void)wrapped;
    ck(cudaMemsetAsync(at<uint64_t>(meta, ML.status), 0, (size_t)nchunk * k * 8, st));
    ck(cudaMemsetAsync(at<uint32_t>(meta, ML.seg_done), 0, (size_t)nseg * 4, st));
    ModelDev* models = at<ModelDev>(meta, ML.models);
    uint64_t* samples = at<uint64_t>(meta, ML.samples);
    uint64_t* seg_dst = at<uint64_t>(meta, ML.seg_dst);
    uint32_t* seg_tot = at<uint32_t>(meta, ML.seg_tot);
    uint32_t* chunk_pre = at<uint32_t>(meta, ML.chunk_pre);
    uint64_t* tree = p.tree ? at<uint64_t>(meta, ML.tree) : nullptr;

    if (iter == 0 && init)  // the initial segments' windows are this level's first windows
      ck(cudaMemcpyAsync(nctr, &init_ctr, sizeof(LevelCounters), cudaMemcpyHostToDevice, st));
    else
      ck(cudaMemsetAsync(nctr, 0, sizeof(LevelCounters), st));
    {
      IPLS_PROF("gather_fit", 0);
      const uint32_t cap = fit_cap(max_S);
      uint32_t* redo = at<uint32_t>(meta, ML.seg_term);  // scratch until K2 writes seg_term
      uint32_t* redo_cnt = &cctr->n_redo;                 // zero: cleared with the counters
      if (max_S <= (uint32_t)kFMMax)
        k_fit_small<F64, kFSThreads, kFMItems><<<nseg, kFSThreads, kFMSmem, st>>>(
            src, segs, seed, hbase, level, k, trace ? samples : nullptr, models, redo, tree, redo_cnt,
            p.tree_leaves);
      else if (max_S <= (uint32_t)kFSMax)
        k_fit_small<F64, kFSThreads, kFSItems><<<nseg, kFSThreads, kFSSmem, st>>>(
            src, segs, seed, hbase, level, k, trace ? samples : nullptr, models, redo, tree, redo_cnt,
            p.tree_leaves);
      else
        k_fit_small<F64, kFLThreads, kFLItems><<<nseg, kFLThreads, kFLSmem, st>>>(
            src, segs, seed, hbase, level, k, trace ? samples : nullptr, models, redo, tree, redo_cnt,
            p.tree_leaves);
      ck_launch();
      k_gather_fit<F64><<<std::min(nseg, num_sms()), kFitThreads, fit_smem(cap), st>>>(
          src, segs, seed, hbase, level, k, cap, trace ? samples : nullptr, models, nullptr, redo, tree, 0,
          redo_cnt, p.tree_leaves);
      ck_launch();
    }
    LevelArgs la{};
    la.src = src; la.segs = segs; la.chunks = chunks; la.models = models;
    la.k = k; la.base_case = p.B; la.level = level; la.chunk_keys = p.chunk_keys; la.nkeys = n;
    la.dstbuf = (iter + 1) & 1;
    // Fusing the last level with the base case pays when a terminal segment is worth a CTA's
    // base-case pass (its packing runs inside the completing CTA): levels whose segments
    // average >= 32 Ki keys (C2-C5 level 1); small segments (level 2 of C3/C5) keep the
    // separate kernels, whose emit runs 4 CTAs per SM.
    // and whose segments are all <= 2^20 keys (the level's largest sample is S(2^20)): with
    // larger segments (skewed inputs: C3, C5, the paper's mixture and Zipf) the fused kernel's
    // per-CTA base-case phases balance worse than the separate launches (C3 -1.2 %, C5 -1.4 %,
    // mixture -2.7 %, Zipf -2.8 % separate; C2 -2.1 % fused)
    // The splitter tree keeps the separate kernels too (C2 / C3 / C5 -1.5 to -2 % separate).
    la.fused_term = (level_keys / std::max<uint32_t>(nseg, 1) >= 32768u &&
                     max_S <= sample_size(1ull << 20, k) && !p.tree) ? 1u : 0u;
    if (g_term_mode.load() == 1) la.fused_term = 1;
    if (g_term_mode.load() == 2) la.fused_term = 0;
    // Terminal segments sorted by windows (ipls_tss.cuh) unless a test hook asks for the
    // child scatter + base case (modes 1, 2).
    // The terminal segment sort (ipls_tss.cuh) is a test-hook alternative: measured slower
    // than the child scatter + warp base case on C1-C5 (rejected round 2).
    la.tss = (g_term_mode.load() == 3) ? 1u : 0u;
    if (la.tss) la.fused_term = 0;
    la.seg_tw = at<uint2>(meta, ML.seg_tw);
    la.twins = at<Window>(fixed, FL.twins);
    la.twcur = at<uint32_t>(fixed, FL.twcur);
    la.cap_twin = p.cap_twin;
    la.ticket = &cctr->ticket;
    la.status = at<uint64_t>(meta, ML.status);
    la.cflag = at<uint8_t>(meta, ML.cflag);
    la.cref = at<uint64_t>(meta, ML.cref);
    la.seg_term = at<uint32_t>(meta, ML.seg_term);
    la.seg_done = at<uint32_t>(meta, ML.seg_done);
    la.chunk_pre = chunk_pre;
    la.seg_dst = seg_dst;
    la.seg_tot = seg_tot;
    la.epoch = epoch;
    la.err = d_err;
    la.check_nan = (F64 && iter == 0 && !init) ? 1 : 0;
    la.ids = nullptr;
    la.single_offsets = nullptr;
    la.nsegs = at<SegDesc>(fixed, FL.segs[nxt]);
    la.nchunks = at<ChunkDesc>(fixed, FL.chunks[nxt]);
    la.nctr = nctr;
    la.cap_segs = p.cap_segs; la.cap_chunks = p.cap_chunks; la.cap_samples = p.cap_samples;
    la.wins = wins; la.cap_wins = p.cap_wins; la.fills = fills; la.cap_fills = p.cap_fills;
    la.wins_big = wbig; la.cap_wbig = p.cap_wbig;
    {
      IPLS_PROF("classify_scan", 8.0 * level_keys);
      launch_classify<F64>(nchunk, st, la, p.tree);
    }
    {
      IPLS_PROF("scatter", 16.0 * level_keys);
      // A segment of more than k * B keys has a child above B, so it is not terminal: the
      // root level of a large sort skips the (empty) terminal launch.
      const bool no_terminal = iter == 0 && !init && n > (uint64_t)k * p.B;
      launch_scatter<F64>(nchunk, st, la, keys, scr, p.tree, no_terminal);
    }
    {
      IPLS_PROF("emit", 0);
      k_emit<<<nseg, kEThreads, win_scratch_bytes(k), st>>>(la);
      ck_launch();
    }

    if (trace) {
      std::vector<SegDesc> hs(nseg);
      std::vector<ModelDev> hm(nseg);
      std::vector<uint32_t> ht((size_t)nseg * k);
      std::vector<uint64_t> hsmp(nsample);
      ck(cudaMemcpyAsync(hs.data(), segs, nseg * sizeof(SegDesc), cudaMemcpyDeviceToHost, st));
      ck(cudaMemcpyAsync(hm.data(), models, nseg * sizeof(ModelDev), cudaMemcpyDeviceToHost, st));
      ck(cudaMemcpyAsync(ht.data(), seg_tot, ht.size() * 4, cudaMemcpyDeviceToHost, st));
      ck(cudaMemcpyAsync(hsmp.data(), samples, (size_t)nsample * 8, cudaMemcpyDeviceToHost, st));
      if (trace->tr->d_snapshots && iter < trace->tr->snapshot_levels) {
        uint64_t* snap = static_cast<uint64_t*>(trace->tr->d_snapshots) + (size_t)iter * n;
        if (iter > 0)
          ck(cudaMemcpyAsync(snap, snap - n, n * 8, cudaMemcpyDeviceToDevice, st));
        k_snapshot<<<nseg, 256, 0, st>>>(segs, keys, scr, (iter + 1) & 1, snap);
        ck_launch();
      }
      ck(cudaStreamSynchronize(st));
      for (uint32_t s = 0; s < nseg; ++s) {
        ipls_segment_record r{};
        r.level = level; r.kind = hm[s].kind; r.begin = hs[s].begin; r.m = hs[s].m;
        r.S = hs[s].S; r.a = hm[s].A; r.b = hm[s].B; r.D = hm[s].D; r.capped = hm[s].capped;
        r.pivot_ok = hm[s].pivot_ok; r.k_eff = (hm[s].kind == kModelEq3) ? 3 : k;
        std::vector<uint64_t> c(r.k_eff);
        r.requeued = 0;
        for (uint32_t b = 0; b < r.k_eff; ++b) {
          c[b] = ht[(size_t)s * k + b];
          if (hm[s].kind != kModelEq3 && c[b] == hs[s].m) r.requeued = 1;
        }
        std::vector<uint64_t> smp(hsmp.begin() + hs[s].sample_off,
                                  hsmp.begin() + hs[s].sample_off + hs[s].S);
        for (auto& v : smp) v = F64 ? ((v >> 63) ? (v & ~(1ull << 63)) : ~v) : v;
        trace->recs.push_back(r);
        trace->counts.push_back(std::move(c));
        trace->samples.push_back(std::move(smp));
      }
    }

    ck(cudaMemcpyAsync(&h_ctr[0], nctr, sizeof(LevelCounters), cudaMemcpyDeviceToHost, st));
    ck(cudaMemcpyAsync(&h_ctr[1].err, d_err, 4, cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    const LevelCounters c = h_ctr[0];
    const uint32_t herr = h_ctr[1].err;
    prof_add_bytes("scatter", 16.0 * c.term_keys);  // the base case done inside k_term_fused
    prof_add_bytes("tss_scatter", 16.0 * c.tsplit_keys);
    if (herr & kErrNan) return IPLS_ERR_NAN_KEY;
    if (herr & kErrOverflow) return IPLS_ERR_OUT_OF_MEMORY;

    // terminal segments: one CTA sorts each window into the user array
    if (c.n_twin) {
      IPLS_PROF("win_sort", 16.0 * c.twin_keys);
      k_win_sort<F64><<<c.n_twin, kWSThreads, win_sort_smem_bytes(), st>>>(
          at<Window>(fixed, FL.twins), keys, scr, d_err);
      ck_launch();
      if (trace && trace->tr->d_snapshots && iter < trace->tr->snapshot_levels) {
        // the level's image of a terminal segment: its sorted keys (each child's multiset)
        uint64_t* snap = static_cast<uint64_t*>(trace->tr->d_snapshots) + (size_t)iter * n;
        k_snapshot_term<<<nseg, 256, 0, st>>>(segs, la.seg_term, keys, snap);
        ck_launch();
      }
    }
    // base case of this level's base children, fills of its homogeneous children
    if (c.n_windows) {
      IPLS_PROF("base_warp", 16.0 * c.win_keys);
      k_base_warp<F64><<<std::min((c.n_windows + kWBWarps - 1) / kWBWarps, num_sms()),
                         kWBWarps * 32, warp_base_smem(), st>>>(wins, c.n_windows, keys, scr);
      ck_launch();
    }
    if (c.n_wbig) {
      IPLS_PROF("base_sort", 16.0 * c.wbig_keys);
      k_base_sort<F64, false><<<c.n_wbig, kBCThreads, base_smem(), st>>>(wbig, keys, scr, d_err);
      ck_launch();
    }
    if (c.n_fills) {
      IPLS_PROF("fill", 8.0 * c.fill_keys);
      k_fill<<<c.n_fills, 256, 0, st>>>(fills, keys);
      ck_launch();
    }
    if (trace) trace->tr->levels = iter + 1;
    nseg = c.n_segs;
    level_keys = c.keys;
    nchunk = c.n_chunks;
    nsample = c.n_samples;
    max_S = c.max_S;
  }
  ck(cudaStreamSynchronize(st));
  return IPLS_OK;
}

ipls_status check_cfg(const ipls_config* cfg, ipls_config* out) {
  ipls_config c = cfg ? *cfg : ipls_default_config();
  if (c.k < 3 || c.k > IPLS_MAX_K) return IPLS_ERR_INVALID_ARGUMENT;
  if (c.base_case < 1 || c.base_case > IPLS_MAX_BASE_CASE) return IPLS_ERR_INVALID_ARGUMENT;
  if (c.flags & ~(IPLS_FLAG_TREE_MODEL | IPLS_FLAG_TREE_EQUAL_BUCKETS)) return IPLS_ERR_INVALID_ARGUMENT;
  if ((c.flags & IPLS_FLAG_TREE_MODEL) && (c.k < 4 || (c.k & (c.k - 1)) != 0))
    return IPLS_ERR_INVALID_ARGUMENT;  // the splitter tree is a perfect binary tree
  if (c.flags & IPLS_FLAG_TREE_EQUAL_BUCKETS)  // k / 2 leaves, each with its equality bucket
    if (!(c.flags & IPLS_FLAG_TREE_MODEL) || c.k < 8) return IPLS_ERR_INVALID_ARGUMENT;
  *out = c;
  return IPLS_OK;
}

ipls_status sort_impl(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg_in,
                      void* d_ws, size_t ws_bytes, void* stream, ipls_trace* tr,
                      const InitSegs* init = nullptr) {
  ipls_config cfg;
  ipls_status s = check_cfg(cfg_in, &cfg);
  if (s != IPLS_OK) return s;
  if (t != IPLS_KEY_F64 && t != IPLS_KEY_U64) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0 && !d_keys) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0xFFFFFFFFull) return IPLS_ERR_INVALID_ARGUMENT;
  if (tr) { tr->records_len = 0; tr->counts_len = 0; tr->samples_len = 0; tr->levels = 0; }
  if (n <= 1) return IPLS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    const Params p = make_params(n, cfg.k, cfg.base_case, (cfg.flags & IPLS_FLAG_TREE_MODEL) != 0,
                                  (cfg.flags & IPLS_FLAG_TREE_EQUAL_BUCKETS) != 0);
    const FixedLayout FL = fixed_layout(p);
    StreamCache& sc = cache_for(stream);
    void* fixed;
    void* meta_in = nullptr;
    size_t meta_bytes = 0;
    DevBuf* meta_cache = nullptr;
    if (d_ws) {
      if (ws_bytes < FL.total + worst_meta_bytes(p)) return IPLS_ERR_OUT_OF_MEMORY;
      fixed = d_ws;
      meta_in = static_cast<char*>(d_ws) + FL.total;
      meta_bytes = ws_bytes - FL.total;
    } else {
      sc.fixed.ensure(FL.total);
      fixed = sc.fixed.ptr;
      meta_cache = &sc.meta;
    }
    TraceSink sink{tr, cfg.k, t == IPLS_KEY_F64, {}, {}, {}};
    ipls_status r =
        (t == IPLS_KEY_F64)
            ? run_sort<true>(static_cast<uint64_t*>(d_keys), p, fixed, meta_in, meta_bytes,
                             meta_cache, sc.h_ctr, st, cfg.seed, tr ? &sink : nullptr, init)
            : run_sort<false>(static_cast<uint64_t*>(d_keys), p, fixed, meta_in, meta_bytes,
                              meta_cache, sc.h_ctr, st, cfg.seed, tr ? &sink : nullptr, init);
    prof_collect();
    if (tr) {
      // order records by (level, begin)
      std::vector<size_t> idx(sink.recs.size());
      for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
      std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
        if (sink.recs[a].level != sink.recs[b].level) return sink.recs[a].level < sink.recs[b].level;
        return sink.recs[a].begin < sink.recs[b].begin;
      });
      size_t nc = 0, ns = 0;
      for (size_t j = 0; j < idx.size(); ++j) {
        size_t i = idx[j];
        if (j < tr->records_cap && tr->records) tr->records[j] = sink.recs[i];
        for (uint64_t v : sink.counts[i]) {
          if (nc < tr->counts_cap && tr->counts) tr->counts[nc] = v;
          ++nc;
        }
        for (uint64_t v : sink.samples[i]) {
          if (ns < tr->samples_cap && tr->samples) tr->samples[ns] = v;
          ++ns;
        }
      }
      tr->records_len = idx.size();
      tr->counts_len = nc;
      tr->samples_len = ns;
    }
    return r;
  } catch (const CudaFail& f) {
    prof_collect();
    g_last_cuda_error = cudaGetErrorString(f.e);
    return f.e == cudaErrorMemoryAllocation ? IPLS_ERR_OUT_OF_MEMORY : IPLS_ERR_CUDA;
  }
}

}  // namespace

extern "C" {

ipls_config ipls_default_config(void) {
  ipls_config c;
  c.k = 256;
  c.base_case = 4096;
  c.seed = IPLS_DEFAULT_SEED;
  c.flags = 0;
  return c;
}

ipls_status ipls_sort_f64(double* d_keys, size_t n, void* stream) {
  return sort_impl(d_keys, n, IPLS_KEY_F64, nullptr, nullptr, 0, stream, nullptr);
}

ipls_status ipls_sort_u64(uint64_t* d_keys, size_t n, void* stream) {
  return sort_impl(d_keys, n, IPLS_KEY_U64, nullptr, nullptr, 0, stream, nullptr);
}

ipls_status ipls_sort_ex(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                         void* d_workspace, size_t ws_bytes, void* stream) {
  return sort_impl(d_keys, n, t, cfg, d_workspace, ws_bytes, stream, nullptr);
}

ipls_status ipls_sort_trace(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                            ipls_trace* trace, void* stream) {
  if (!trace) return IPLS_ERR_INVALID_ARGUMENT;
  return sort_impl(d_keys, n, t, cfg, nullptr, 0, stream, trace);
}

static ipls_status sort_segments_impl(void* d_keys, size_t n, ipls_key_type t,
                                      const ipls_config* cfg, const uint64_t* h_seg_sizes,
                                      uint32_t nseg, uint32_t level, uint64_t global_begin,
                                      ipls_trace* tr, void* stream) {
  if (nseg == 0 || !h_seg_sizes) return n == 0 ? IPLS_OK : IPLS_ERR_INVALID_ARGUMENT;
  unsigned __int128 tot = 0;
  for (uint32_t i = 0; i < nseg; ++i) tot += h_seg_sizes[i];
  if (tot != n) return IPLS_ERR_INVALID_ARGUMENT;
  if (n <= 1) return sort_impl(d_keys, n, t, cfg, nullptr, 0, stream, tr);
  const InitSegs init{h_seg_sizes, nseg, level, global_begin};
  return sort_impl(d_keys, n, t, cfg, nullptr, 0, stream, tr, &init);
}

ipls_status ipls_sort_segments(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                               const uint64_t* h_seg_sizes, uint32_t nseg, uint32_t level,
                               uint64_t global_begin, void* stream) {
  return sort_segments_impl(d_keys, n, t, cfg, h_seg_sizes, nseg, level, global_begin, nullptr,
                            stream);
}

ipls_status ipls_sort_segments_trace(void* d_keys, size_t n, ipls_key_type t,
                                     const ipls_config* cfg, const uint64_t* h_seg_sizes,
                                     uint32_t nseg, uint32_t level, uint64_t global_begin,
                                     ipls_trace* trace, void* stream) {
  if (!trace) return IPLS_ERR_INVALID_ARGUMENT;
  return sort_segments_impl(d_keys, n, t, cfg, h_seg_sizes, nseg, level, global_begin, trace,
                            stream);
}

ipls_status ipls_regroup_runs(const void* d_src, void* d_dst, const uint64_t* h_counts,
                              uint32_t G, uint32_t nb, void* stream) {
  if (G == 0 || nb == 0) return IPLS_OK;
  if (!h_counts || !d_src || !d_dst) return IPLS_ERR_INVALID_ARGUMENT;
  // run g starts after runs 0..g-1; bucket b of the output after buckets < b (all runs) and
  // after runs < g's keys of bucket b
  std::vector<uint64_t> run_start(G + 1, 0), bucket_tot(nb, 0), dst_start(nb + 1, 0);
  for (uint32_t g = 0; g < G; ++g) {
    uint64_t t = 0;
    for (uint32_t b = 0; b < nb; ++b) { t += h_counts[(size_t)g * nb + b]; bucket_tot[b] += h_counts[(size_t)g * nb + b]; }
    run_start[g + 1] = run_start[g] + t;
  }
  for (uint32_t b = 0; b < nb; ++b) dst_start[b + 1] = dst_start[b] + bucket_tot[b];
  std::vector<Piece> pcs;
  std::vector<uint64_t> fill(nb, 0);
  for (uint32_t g = 0; g < G; ++g) {
    uint64_t so = run_start[g];
    for (uint32_t b = 0; b < nb; ++b) {
      const uint64_t c = h_counts[(size_t)g * nb + b];
      if (c) pcs.push_back(Piece{so, dst_start[b] + fill[b], c});
      so += c;
      fill[b] += c;
    }
  }
  if (pcs.empty()) return IPLS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    Piece* dp = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&dp), pcs.size() * sizeof(Piece), st));
    ck(cudaMemcpyAsync(dp, pcs.data(), pcs.size() * sizeof(Piece), cudaMemcpyHostToDevice, st));
    const uint32_t np = (uint32_t)pcs.size();
    k_move_pieces<<<std::min<uint32_t>((np + 7) / 8, num_sms() * 8), 256, 0, st>>>(
        static_cast<const uint64_t*>(d_src), static_cast<uint64_t*>(d_dst), dp, np);
    ck_launch();
    ck(cudaFreeAsync(dp, st));
    ck(cudaStreamSynchronize(st));
    return IPLS_OK;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return f.e == cudaErrorMemoryAllocation ? IPLS_ERR_OUT_OF_MEMORY : IPLS_ERR_CUDA;
  }
}

size_t ipls_workspace_bytes(size_t n, ipls_key_type t, const ipls_config* cfg) {
  ipls_config c;
  if (check_cfg(cfg, &c) != IPLS_OK || (t != IPLS_KEY_F64 && t != IPLS_KEY_U64)) return 0;
  if (n <= 1) return 0;
  const Params p = make_params(n, c.k, c.base_case, (c.flags & IPLS_FLAG_TREE_MODEL) != 0,
                                (c.flags & IPLS_FLAG_TREE_EQUAL_BUCKETS) != 0);
  return fixed_layout(p).total + worst_meta_bytes(p);
}

ipls_status ipls_sort_host(void* h_keys, size_t n, ipls_key_type t, const ipls_config* cfg,
                           void* stream) {
  if (n > 0 && !h_keys) return IPLS_ERR_INVALID_ARGUMENT;
  if (n <= 1) return IPLS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    StreamCache& sc = cache_for(stream);
    sc.io.ensure(n * 8);
    ck(cudaMemcpyAsync(sc.io.ptr, h_keys, n * 8, cudaMemcpyHostToDevice, st));
    ipls_status s = sort_impl(sc.io.ptr, n, t, cfg, nullptr, 0, stream, nullptr);
    if (s != IPLS_OK) return s;
    ck(cudaMemcpyAsync(h_keys, sc.io.ptr, n * 8, cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    return IPLS_OK;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return f.e == cudaErrorMemoryAllocation ? IPLS_ERR_OUT_OF_MEMORY : IPLS_ERR_CUDA;
  }
}

// Internal streams per device for ipls_sort_host_batch (created once, kept).  Array j uses
// stream j % kPipe and its device buffer: with three, array j+1's upload waits only for array
// j-2's download, so the uploads run back to back.
constexpr int kPipe = 3;
struct PipeStreams {
  cudaStream_t s[kPipe];
  cudaEvent_t ev;
};
PipeStreams& pipe_streams() {
  static std::map<int, PipeStreams> m;
  int dev = 0;
  ck(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = m.find(dev);
  if (it == m.end()) {
    PipeStreams p;
    for (int i = 0; i < kPipe; ++i) ck(cudaStreamCreateWithFlags(&p.s[i], cudaStreamNonBlocking));
    ck(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
    it = m.emplace(dev, p).first;
  }
  return it->second;
}

ipls_status ipls_sort_host_batch(const void* const* h_in, void* const* h_out, const size_t* n,
                                 uint32_t count, ipls_key_type t, const ipls_config* cfg,
                                 void* stream) {
  if (count == 0) return IPLS_OK;
  if (!h_in || !h_out || !n) return IPLS_ERR_INVALID_ARGUMENT;
  for (uint32_t j = 0; j < count; ++j)
    if (n[j] > 0 && (!h_in[j] || !h_out[j])) return IPLS_ERR_INVALID_ARGUMENT;
  if (t != IPLS_KEY_F64 && t != IPLS_KEY_U64) return IPLS_ERR_INVALID_ARGUMENT;
  {
    ipls_config c;
    const ipls_status s = check_cfg(cfg, &c);
    if (s != IPLS_OK) return s;
  }
  try {
    PipeStreams& ps = pipe_streams();
    // the batch starts after the work already queued on the caller's stream
    ck(cudaEventRecord(ps.ev, static_cast<cudaStream_t>(stream)));
    for (int i = 0; i < kPipe; ++i) ck(cudaStreamWaitEvent(ps.s[i], ps.ev, 0));
    auto upload = [&](uint32_t j) {  // array j into its stream's device buffer
      if (n[j] <= 1) return;
      cudaStream_t s = ps.s[j % kPipe];
      StreamCache& sc = cache_for(s);
      sc.io.ensure(n[j] * 8);  // stream-ordered after this buffer's previous download
      ck(cudaMemcpyAsync(sc.io.ptr, h_in[j], n[j] * 8, cudaMemcpyHostToDevice, s));
    };
    ipls_status st = IPLS_OK;
    upload(0);
    for (uint32_t j = 0; j < count && st == IPLS_OK; ++j) {
      if (j + 1 < count) upload(j + 1);  // overlaps this sort and the previous download
      if (n[j] == 0) continue;
      if (n[j] == 1) {
        std::memmove(h_out[j], h_in[j], 8);
        continue;
      }
      cudaStream_t s = ps.s[j % kPipe];
      StreamCache& sc = cache_for(s);
      st = sort_impl(sc.io.ptr, n[j], t, cfg, nullptr, 0, s, nullptr);
      if (st == IPLS_OK)
        ck(cudaMemcpyAsync(h_out[j], sc.io.ptr, n[j] * 8, cudaMemcpyDeviceToHost, s));
    }
    for (int i = 0; i < kPipe; ++i) ck(cudaStreamSynchronize(ps.s[i]));
    return st;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return f.e == cudaErrorMemoryAllocation ? IPLS_ERR_OUT_OF_MEMORY : IPLS_ERR_CUDA;
  }
}

static ipls_status fit_given(const void* d_sorted_sample, size_t S, ipls_key_type t, uint32_t k,
                             ipls_model* h_out, void* stream, int sort_given);

ipls_status ipls_fit_fmcd(const void* d_sorted_sample, size_t S, ipls_key_type t, uint32_t k,
                          ipls_model* h_out, void* stream) {
  return fit_given(d_sorted_sample, S, t, k, h_out, stream, 0);
}

ipls_status ipls_fit_sample(const void* d_sample, size_t S, ipls_key_type t, uint32_t k,
                            ipls_model* h_out, void* stream) {
  return fit_given(d_sample, S, t, k, h_out, stream, 1);
}

static ipls_status fit_given(const void* d_sorted_sample, size_t S, ipls_key_type t, uint32_t k,
                             ipls_model* h_out, void* stream, int sort_given) {
  if (!d_sorted_sample || !h_out) return IPLS_ERR_INVALID_ARGUMENT;
  if (S < 4 || S > (size_t)kFitMaxS || k < 3 || k > IPLS_MAX_K) return IPLS_ERR_INVALID_ARGUMENT;
  if (t != IPLS_KEY_F64 && t != IPLS_KEY_U64) return IPLS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    StreamCache& sc = cache_for(stream);
    const size_t need = align_up(S * 8, 256) + 256 + 256;
    sc.meta.ensure(need);
    sc.meta.fresh = true;  // the lookback region is clobbered; clear it before the next sort
    uint64_t* smp = static_cast<uint64_t*>(sc.meta.ptr);
    SegDesc* dseg = at<SegDesc>(sc.meta.ptr, align_up(S * 8, 256));
    ModelDev* dmod = at<ModelDev>(sc.meta.ptr, align_up(S * 8, 256) + 256);
    k_keys_to_ok<<<(uint32_t)((S + 255) / 256), 256, 0, st>>>(
        static_cast<const uint64_t*>(d_sorted_sample), smp, (uint32_t)S, t == IPLS_KEY_F64);
    ck_launch();
    SegDesc sd{};
    sd.S = (uint32_t)S;
    ck(cudaMemcpyAsync(dseg, &sd, sizeof(sd), cudaMemcpyHostToDevice, st));
    const uint32_t cap = fit_cap((uint32_t)S);
    if (t == IPLS_KEY_F64) {
      set_attrs<true>();
      k_gather_fit<true><<<1, kFitThreads, fit_smem(cap), st>>>(nullptr, dseg, 0, 0, 0, k, cap,
                                                                nullptr, dmod, smp, nullptr,
                                                                nullptr, sort_given);
    } else {
      set_attrs<false>();
      k_gather_fit<false><<<1, kFitThreads, fit_smem(cap), st>>>(nullptr, dseg, 0, 0, 0, k, cap,
                                                                 nullptr, dmod, smp, nullptr,
                                                                 nullptr, sort_given);
    }
    ck_launch();
    ModelDev hm;
    ck(cudaMemcpyAsync(&hm, dmod, sizeof(hm), cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    h_out->a = hm.A; h_out->b = hm.B; h_out->k = hm.kind == kModelEq3 ? 3 : k; h_out->D = hm.D;
    h_out->kind = hm.kind; h_out->capped = hm.capped; h_out->pivot_ok = hm.pivot_ok;
    return hm.kind == kModelEq3 ? IPLS_ERR_DEGENERATE_SAMPLE : IPLS_OK;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return IPLS_ERR_CUDA;
  }
}

uint32_t ipls_sample_size(uint64_t m, uint32_t k) { return sample_size(m, k); }

ipls_status ipls_sample_strata(const void* d_keys, size_t n_local, uint64_t global_begin,
                               uint64_t global_m, uint32_t S, uint64_t seed, uint64_t* d_sample,
                               void* stream) {
  if (S == 0) return IPLS_OK;
  if (!d_sample || (n_local > 0 && !d_keys)) return IPLS_ERR_INVALID_ARGUMENT;
  // S is a level-0 sample size (<= kFitMaxS): j * m below stays inside 64 bits
  if (S > (uint32_t)kFitMaxS) return IPLS_ERR_INVALID_ARGUMENT;
  if (global_m >= (1ull << 48) || S > global_m || global_begin > global_m ||
      n_local > global_m - global_begin)
    return IPLS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    k_sample_strata<<<(S + 255) / 256, 256, 0, st>>>(static_cast<const uint64_t*>(d_keys),
                                                     n_local, global_begin, global_m, S, seed,
                                                     d_sample);
    ck_launch();
    ck(cudaStreamSynchronize(st));
    return IPLS_OK;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return IPLS_ERR_CUDA;
  }
}

ipls_status ipls_assign_ranges(const uint64_t* h_counts, uint32_t k, uint32_t G,
                               uint32_t* h_bounds) {
  if (!h_counts || !h_bounds || k == 0 || G == 0) return IPLS_ERR_INVALID_ARGUMENT;
  unsigned __int128 total = 0;
  for (uint32_t b = 0; b < k; ++b) total += h_counts[b];
  h_bounds[0] = 0;
  uint32_t b = 0;
  unsigned __int128 pre = 0;  // keys in buckets [0, b)
  for (uint32_t r = 1; r < G; ++r) {
    // the boundary b >= bounds[r-1] whose prefix is closest to r/G of the keys (ties: lower)
    const unsigned __int128 target = total * r;
    auto dist = [&](unsigned __int128 p) {
      const unsigned __int128 x = p * G;
      return x > target ? x - target : target - x;
    };
    uint32_t best = b;
    unsigned __int128 bestd = dist(pre), p = pre;
    for (uint32_t c = b; c < k && p * G <= target; ++c) {  // past the target dist only grows
      p += h_counts[c];
      if (dist(p) < bestd) { bestd = dist(p); best = c + 1; }
    }
    while (b < best) pre += h_counts[b++];
    h_bounds[r] = b;
  }
  h_bounds[G] = k;
  return IPLS_OK;
}

ipls_status ipls_assign_cuts(const uint64_t* h_counts, uint32_t k, uint32_t G,
                             const uint8_t* h_splittable, uint64_t* h_cuts) {
  if (!h_counts || !h_cuts || k == 0 || G == 0) return IPLS_ERR_INVALID_ARGUMENT;
  unsigned __int128 total = 0;
  for (uint32_t b = 0; b < k; ++b) total += h_counts[b];
  if (total > UINT64_MAX - 1) return IPLS_ERR_INVALID_ARGUMENT;
  h_cuts[0] = 0;
  uint32_t b = 0;                  // bucket whose start boundary `pre` is <= the last cut
  unsigned __int128 pre = 0, prev = 0;
  for (uint32_t r = 1; r < G; ++r) {
    const unsigned __int128 target = total * r;
    auto dist = [&](unsigned __int128 p) {
      const unsigned __int128 x = p * G;
      return x > target ? x - target : target - x;
    };
    unsigned __int128 best = prev, bestd = dist(prev), p = pre;
    for (uint32_t c = b;; ++c) {   // boundary c at position p, then the inside of bucket c
      if (p >= prev && dist(p) < bestd) { bestd = dist(p); best = p; }
      if (p * G > target || c == k) break;  // past the target distances only grow
      const unsigned __int128 e = p + h_counts[c];
      if (h_splittable && h_splittable[c]) {
        const unsigned __int128 q = target / G;  // floor and ceil of the ideal position
        for (unsigned __int128 x = q; x <= q + 1; ++x)
          if (x > p && x < e && x >= prev && dist(x) < bestd) { bestd = dist(x); best = x; }
      }
      p = e;
    }
    while (b < k && pre + h_counts[b] <= best) pre += h_counts[b++];
    h_cuts[r] = (uint64_t)best;
    prev = best;
  }
  h_cuts[G] = (uint64_t)total;
  return IPLS_OK;
}

}  // extern "C"

namespace {
// ipls_partition_level and its two halves for the fused multi-GPU exchange: kPartCount
// classifies only (offsets), kPartScatterTo classifies and scatters every bucket to its own
// destination address (k_scatter_peer).
enum PartMode { kPartFull, kPartCount, kPartScatterTo };

ipls_status partition_impl(PartMode mode, const void* d_in, void* d_out, size_t n, ipls_key_type t,
                           const ipls_model* h_model, uint64_t* d_offsets,
                           uint16_t* d_bucket_ids, const uint64_t* d_bucket_dst, void* stream) {
  if (!h_model) return IPLS_ERR_INVALID_ARGUMENT;
  if (mode != kPartScatterTo && !d_offsets) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0 && !d_in) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0 && mode == kPartFull && !d_out) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0 && mode == kPartScatterTo && !d_bucket_dst) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0xFFFFFFFFull) return IPLS_ERR_INVALID_ARGUMENT;
  if (t != IPLS_KEY_F64 && t != IPLS_KEY_U64) return IPLS_ERR_INVALID_ARGUMENT;
  const bool eq3 = h_model->kind == IPLS_MODEL_EQ3;
  if (!eq3 && h_model->kind != IPLS_MODEL_LINEAR) return IPLS_ERR_INVALID_ARGUMENT;
  const uint32_t k = eq3 ? 3u : h_model->k;
  if (k < 3 || k > IPLS_MAX_K) return IPLS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    if (n == 0) {
      if (d_offsets) {
        std::vector<uint64_t> z(k + 1, 0);
        ck(cudaMemcpyAsync(d_offsets, z.data(), z.size() * 8, cudaMemcpyHostToDevice, st));
        ck(cudaStreamSynchronize(st));
      }
      return IPLS_OK;
    }
    StreamCache& sc = cache_for(stream);
    const uint32_t ck_keys = pick_chunk_keys(n);
    const uint32_t nchunk = (uint32_t)((n + ck_keys - 1) / ck_keys);
    const MetaLayout ML = meta_layout(1, nchunk, 0, k);
    size_t o = align_up(ML.total, 256);
    const size_t off_own = o; o = align_up(o + (size_t)(k + 1) * 8, 256);  // offsets nobody asked for
    const size_t off_seg = o; o += 256;
    const size_t off_ch = o; o = align_up(o + nchunk * sizeof(ChunkDesc), 256);
    const size_t off_err = o; o += 256;
    const size_t off_ctr = o; o += 256;
    sc.meta.ensure(o);
    sc.meta.fresh = true;
    void* meta = sc.meta.ptr;
    SegDesc* dseg = at<SegDesc>(meta, off_seg);
    ChunkDesc* dch = at<ChunkDesc>(meta, off_ch);
    uint32_t* derr = at<uint32_t>(meta, off_err);
    LevelCounters* dctr = at<LevelCounters>(meta, off_ctr);
    ModelDev hm{};
    hm.A = h_model->a; hm.B = h_model->b; hm.pivot_ok = h_model->pivot_ok;
    hm.kind = h_model->kind; hm.D = h_model->D; hm.capped = h_model->capped; hm.k_eff = k;
    ModelDev* dmod = at<ModelDev>(meta, ML.models);
    ck(cudaMemcpyAsync(dmod, &hm, sizeof(hm), cudaMemcpyHostToDevice, st));
    ck(cudaMemsetAsync(derr, 0, 16, st));
    ck(cudaMemsetAsync(dctr, 0, sizeof(LevelCounters), st));
    ck(cudaMemsetAsync(at<uint64_t>(meta, ML.status), 0, (size_t)nchunk * k * 8, st));
    k_init_root<<<std::max<uint32_t>(1, (nchunk + 255) / 256), 256, 0, st>>>(dseg, dch, n, 0,
                                                                          ck_keys, 0u);
    ck_launch();
    LevelArgs la{};
    la.src = static_cast<const uint64_t*>(d_in); la.segs = dseg; la.chunks = dch;
    la.models = dmod; la.k = k; la.base_case = 0; la.level = 0; la.chunk_keys = ck_keys; la.nkeys = n;
    la.dstbuf = 1;
    la.ticket = &dctr->ticket;
    la.status = at<uint64_t>(meta, ML.status);
    la.cflag = at<uint8_t>(meta, ML.cflag);
    la.cref = at<uint64_t>(meta, ML.cref);
    la.seg_term = at<uint32_t>(meta, ML.seg_term);
    la.chunk_pre = at<uint32_t>(meta, ML.chunk_pre);
    la.seg_dst = at<uint64_t>(meta, ML.seg_dst);
    la.seg_tot = at<uint32_t>(meta, ML.seg_tot);
    bool wrapped = false;
    la.epoch = next_epoch(&wrapped);
    la.err = derr;
    la.check_nan = 0;
    la.ids = d_bucket_ids;
    la.single_offsets = d_offsets ? d_offsets : at<uint64_t>(meta, off_own);
    la.bucket_dst = d_bucket_dst;
    uint64_t* out = static_cast<uint64_t*>(d_out);
    auto body = [&](auto f64tag) {
      constexpr bool F64 = decltype(f64tag)::value;
      set_attrs<F64>();
      launch_classify<F64>(nchunk, st, la);
      if (mode == kPartFull) {
        launch_scatter<F64>(nchunk, st, la, out, out, false, true);
      } else if (mode == kPartScatterTo) {
        IPLS_PROF("scatter_peer", 16.0 * n);
        k_scatter_peer<F64><<<nchunk, kSThreads, scatter_peer_smem_bytes(k), st>>>(la);
        ck_launch();
      }
    };
    if (t == IPLS_KEY_F64) body(std::true_type{}); else body(std::false_type{});
    ck(cudaStreamSynchronize(st));
    return IPLS_OK;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return IPLS_ERR_CUDA;
  }
}
}  // namespace

extern "C" {

ipls_status ipls_partition_level(const void* d_in, void* d_out, size_t n, ipls_key_type t,
                                 const ipls_model* h_model, uint64_t* d_offsets,
                                 uint16_t* d_bucket_ids, void* stream) {
  return partition_impl(kPartFull, d_in, d_out, n, t, h_model, d_offsets, d_bucket_ids, nullptr,
                        stream);
}

ipls_status ipls_partition_count(const void* d_in, size_t n, ipls_key_type t,
                                 const ipls_model* h_model, uint64_t* d_offsets, void* stream) {
  return partition_impl(kPartCount, d_in, nullptr, n, t, h_model, d_offsets, nullptr, nullptr,
                        stream);
}

ipls_status ipls_partition_scatter_to(const void* d_in, size_t n, ipls_key_type t,
                                      const ipls_model* h_model, const uint64_t* d_bucket_dst,
                                      void* stream) {
  return partition_impl(kPartScatterTo, d_in, nullptr, n, t, h_model, nullptr, nullptr,
                        d_bucket_dst, stream);
}

const char* ipls_status_string(ipls_status s) {
  switch (s) {
    case IPLS_OK: return "ok";
    case IPLS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case IPLS_ERR_NAN_KEY: return "NaN key";
    case IPLS_ERR_DEGENERATE_SAMPLE: return "degenerate sample";
    case IPLS_ERR_OUT_OF_MEMORY: return "out of memory";
    case IPLS_ERR_CUDA: return "CUDA error";
    case IPLS_ERR_NOT_IMPLEMENTED: return "not implemented";
  }
  return "unknown status";
}

const char* ipls_last_cuda_error(void) { return g_last_cuda_error.c_str(); }

uint64_t ipls_kernel_launch_count(void) { return g_launches.load(); }

void ipls_debug_set_epoch(uint32_t e) { g_epoch.store(e); }

void ipls_debug_term_mode(int mode) { g_term_mode.store(mode); }

void ipls_debug_force_match_rank(int on) {
  const int v = on ? 1 : 0;
  cudaMemcpyToSymbol(g_force_match_rank, &v, sizeof(v));
}

#ifdef IPLS_SCATTER_TIMING
// dev builds only (tools/phase_scatter.py): per-phase cycle sums of thread 0 of every CTA
void ipls_debug_scatter_phases(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_sc_phase, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_sc_phase, z, sizeof(z));
  }
}
#endif

void ipls_profile_enable(int on) { g_prof_on.store(on ? 1 : 0); }

void ipls_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.clear();
}

size_t ipls_profile_read(ipls_profile_entry* out, size_t cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  size_t i = 0;
  for (auto& kv : g_prof) {
    if (out && i < cap) {
      ipls_profile_entry& e = out[i];
      std::memset(&e, 0, sizeof(e));
      std::strncpy(e.name, kv.first.c_str(), sizeof(e.name) - 1);
      e.launches = kv.second.launches;
      e.total_ms = kv.second.ms;
      e.bytes = kv.second.bytes;
    }
    ++i;
  }
  return i;
}

}  // extern "C"
