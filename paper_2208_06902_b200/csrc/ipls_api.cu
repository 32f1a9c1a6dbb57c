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
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ipls.h"
#include "ipls_kernels.cuh"

using namespace ipls;

namespace {

std::atomic<uint64_t> g_launches{0};
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
#define IPLS_CAT2(a, b) a##b
#define IPLS_CAT(a, b) IPLS_CAT2(a, b)
#define IPLS_PROF(name, bytes) ProfScope IPLS_CAT(_prof_scope_, __LINE__)(name, (double)(bytes), st)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Params {
  uint64_t n;
  uint32_t k, B, chunk_keys, log2k;
  uint32_t cap_segs, cap_chunks, cap_units, cap_samples, cap_wins, cap_fills;
};

uint32_t pick_chunk_keys(uint64_t n) {
  // ~4 waves of 2 CTAs per SM over 148 SMs at level 0, whole tiles, 4096..65536 keys.
  uint64_t c = n / (148 * 8);
  c = (c + kTile - 1) / kTile * kTile;
  if (c < (uint64_t)kTile) c = kTile;
  if (c > 65536) c = 65536;
  return (uint32_t)c;
}

Params make_params(uint64_t n, uint32_t k, uint32_t B) {
  Params p{};
  p.n = n; p.k = k; p.B = B;
  p.chunk_keys = pick_chunk_keys(n);
  p.log2k = 0;
  while ((1u << p.log2k) < k) ++p.log2k;
  const uint64_t segs = n / ((uint64_t)B + 1) + 2;
  const uint64_t chunks = n / p.chunk_keys + segs + 1;
  const uint64_t units = chunks / kUnitChunks + segs + 1;
  const uint64_t smax = sample_size(n, k);
  uint64_t samples = std::min<uint64_t>(n / 2 + 8, segs * smax + 8);
  uint64_t wins = std::min<uint64_t>(n + 1, n / ((uint64_t)B + 1) + n / kWindowNominal + 2 * segs) + 16;
  uint64_t fills = n / ((uint64_t)B + 1) + 16;
  p.cap_segs = (uint32_t)segs;
  p.cap_chunks = (uint32_t)chunks;
  p.cap_units = (uint32_t)units;
  p.cap_samples = (uint32_t)samples;
  p.cap_wins = (uint32_t)wins;
  p.cap_fills = (uint32_t)fills;
  return p;
}

// Fixed part of the workspace: scratch keys + descriptors of two levels + windows/fills of
// two levels + counters.  The k-scaled per-level metadata is carved after it.
struct FixedLayout {
  size_t scratch, segs[2], chunks[2], units[2], wins[2], fills[2], ctr[2], err, total;
};

FixedLayout fixed_layout(const Params& p) {
  FixedLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.scratch = take(p.n * 8);
  for (int i = 0; i < 2; ++i) {
    L.segs[i] = take((size_t)p.cap_segs * sizeof(SegDesc));
    L.chunks[i] = take((size_t)p.cap_chunks * sizeof(ChunkDesc));
    L.units[i] = take((size_t)p.cap_units * sizeof(UnitDesc));
    L.wins[i] = take((size_t)p.cap_wins * sizeof(Window));
    L.fills[i] = take((size_t)p.cap_fills * sizeof(Fill));
    L.ctr[i] = take(sizeof(LevelCounters));
  }
  L.err = take(16);
  L.total = o;
  return L;
}

struct MetaLayout {
  size_t models, samples, chunk_hist, chunk_rep, unit_cnt, unit_rep, seg_tot, seg_rep, seg_dst,
      total;
};

MetaLayout meta_layout(uint64_t segs, uint64_t chunks, uint64_t units, uint64_t samples,
                       uint32_t k) {
  MetaLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.models = take(segs * sizeof(ModelDev));
  L.samples = take(samples * 8 + 64);
  L.chunk_hist = take(chunks * k * 4);
  L.chunk_rep = take(chunks * k * 8);
  L.unit_cnt = take(units * k * 4);
  L.unit_rep = take(units * k * 8);
  L.seg_tot = take(segs * k * 4);
  L.seg_rep = take(segs * k * 8);
  L.seg_dst = take(segs * k * 8);
  L.total = o;
  return L;
}

size_t worst_meta_bytes(const Params& p) {
  return meta_layout(p.cap_segs, p.cap_chunks, p.cap_units, p.cap_samples, p.k).total;
}

// Device buffers for one call: either the caller's workspace or the per-stream cache.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
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
  }
};

struct StreamCache {
  DevBuf fixed, meta, io;  // io: device copy for ipls_sort_host
  LevelCounters* h_ctr = nullptr;  // pinned
  StreamCache() { ck(cudaMallocHost((void**)&h_ctr, 2 * sizeof(LevelCounters) + 64)); }
  ~StreamCache() {
    fixed.release(); meta.release(); io.release();
    if (h_ctr) cudaFreeHost(h_ctr);
  }
};

std::mutex g_mu;
std::map<std::pair<int, void*>, std::unique_ptr<StreamCache>> g_cache;

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

template <bool F64>
void launch_scatter(uint32_t log2k, dim3 grid, size_t smem, cudaStream_t st,
                    const uint64_t* src, uint64_t* user, uint64_t* scr, const ChunkDesc* chunks,
                    const ModelDev* models, uint32_t k, const uint32_t* chunk_pre,
                    const uint64_t* seg_dst, const uint32_t* err) {
#define IPLS_SC(L)                                                                          \
  case L:                                                                                   \
    ck(cudaFuncSetAttribute(k_scatter<F64, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                            (int)smem));                                                    \
    k_scatter<F64, L><<<grid, kTileThreads, smem, st>>>(src, user, scr, chunks, models, k,  \
                                                       chunk_pre, seg_dst, err);            \
    break;
  switch (log2k) {
    IPLS_SC(2) IPLS_SC(3) IPLS_SC(4) IPLS_SC(5) IPLS_SC(6) IPLS_SC(7) IPLS_SC(8) IPLS_SC(9)
    IPLS_SC(10)
    default: throw CudaFail{cudaErrorInvalidValue};
  }
#undef IPLS_SC
  ck_launch();
}

size_t scatter_smem(uint32_t k) {
  return (size_t)kTile * 8 + (size_t)k * 8 + (size_t)k * 8 + (size_t)kTileWarps * k * 2 +
         (size_t)kTile * 2;
}
size_t classify_smem(uint32_t k) { return (size_t)k * 8 + (size_t)k * 12; }
size_t base_smem() { return (size_t)kBaseMax * 12; }
size_t fit_smem() { return (size_t)kFitMaxS * 8; }

template <bool F64>
void set_attrs() {
  static bool done = false;
  if (done) return;
  ck(cudaFuncSetAttribute(k_fit<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fit_smem()));
  ck(cudaFuncSetAttribute(k_base_sort<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)base_smem()));
  ck(cudaFuncSetAttribute(k_classify_hist<F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)classify_smem(kMaxK)));
  done = true;
}

uint32_t col_blocks(uint64_t items, uint32_t k) {
  uint64_t warps = items * ((k + 31) / 32);
  return (uint32_t)std::max<uint64_t>(1, (warps + 7) / 8);
}

// Run the whole level-batched sort.  keys: device array (user buffer).
template <bool F64>
ipls_status run_sort(uint64_t* keys, const Params& p, void* fixed, void* d_meta_in,
                     size_t meta_bytes_in, DevBuf* meta_cache, LevelCounters* h_ctr,
                     cudaStream_t st, uint64_t seed, TraceSink* trace) {
  set_attrs<F64>();
  const FixedLayout FL = fixed_layout(p);
  uint64_t* scr = at<uint64_t>(fixed, FL.scratch);
  uint32_t* d_err = at<uint32_t>(fixed, FL.err);
  ck(cudaMemsetAsync(d_err, 0, 16, st));
  const uint64_t n = p.n;
  const uint32_t k = p.k;

  if (n <= p.B) {
    // The root is a base-case segment: one window in place.
    Window w{0, (uint32_t)n, 0};
    Window* dw = at<Window>(fixed, FL.wins[0]);
    ck(cudaMemcpyAsync(dw, &w, sizeof(Window), cudaMemcpyHostToDevice, st));
    {
      IPLS_PROF("base_sort", 16.0 * n);
      k_base_sort<F64><<<1, kBaseThreads, base_smem(), st>>>(dw, keys, scr, d_err, F64 ? 1 : 0);
      ck_launch();
    }
    uint32_t herr = 0;
    ck(cudaMemcpyAsync(&h_ctr[1].err, d_err, 4, cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    herr = h_ctr[1].err;
    if (herr & kErrNan) return IPLS_ERR_NAN_KEY;
    return IPLS_OK;
  }

  // level-0 work: the root segment
  uint32_t nseg = 1;
  uint32_t nchunk = (uint32_t)((n + p.chunk_keys - 1) / p.chunk_keys);
  uint32_t nunit = (nchunk + kUnitChunks - 1) / kUnitChunks;
  uint32_t nsample = sample_size(n, k);
  uint64_t level_keys = n;
  k_init_root<<<std::max<uint32_t>(1, (nchunk + 255) / 256), 256, 0, st>>>(
      at<SegDesc>(fixed, FL.segs[0]), at<ChunkDesc>(fixed, FL.chunks[0]),
      at<UnitDesc>(fixed, FL.units[0]), n, nsample, p.chunk_keys, 0u);
  ck_launch();

  for (uint32_t level = 0; nseg > 0; ++level) {
    const int cur = level & 1, nxt = cur ^ 1;
    const uint64_t* src = (cur == 0) ? keys : scr;
    SegDesc* segs = at<SegDesc>(fixed, FL.segs[cur]);
    ChunkDesc* chunks = at<ChunkDesc>(fixed, FL.chunks[cur]);
    UnitDesc* units = at<UnitDesc>(fixed, FL.units[cur]);
    LevelCounters* nctr = at<LevelCounters>(fixed, FL.ctr[nxt]);
    Window* wins = at<Window>(fixed, FL.wins[cur]);
    Fill* fills = at<Fill>(fixed, FL.fills[cur]);

    // per-level metadata, sized by this level's actual counts
    MetaLayout ML = meta_layout(nseg, nchunk, nunit, nsample, k);
    void* meta = d_meta_in;
    if (meta_cache) {
      meta_cache->ensure(ML.total);
      meta = meta_cache->ptr;
    } else if (ML.total > meta_bytes_in) {
      return IPLS_ERR_OUT_OF_MEMORY;
    }
    ModelDev* models = at<ModelDev>(meta, ML.models);
    uint64_t* samples = at<uint64_t>(meta, ML.samples);
    uint32_t* chunk_hist = at<uint32_t>(meta, ML.chunk_hist);
    uint64_t* chunk_rep = at<uint64_t>(meta, ML.chunk_rep);
    uint32_t* unit_cnt = at<uint32_t>(meta, ML.unit_cnt);
    uint64_t* unit_rep = at<uint64_t>(meta, ML.unit_rep);
    uint32_t* seg_tot = at<uint32_t>(meta, ML.seg_tot);
    uint64_t* seg_rep = at<uint64_t>(meta, ML.seg_rep);
    uint64_t* seg_dst = at<uint64_t>(meta, ML.seg_dst);

    ck(cudaMemsetAsync(nctr, 0, sizeof(LevelCounters), st));
    {
      IPLS_PROF("sample_gather", 0);
      k_sample_gather<F64><<<nseg, 256, 0, st>>>(src, segs, seed, level, samples);
      ck_launch();
    }
    {
      IPLS_PROF("fit", 0);
      k_fit<F64><<<nseg, kFitThreads, fit_smem(), st>>>(segs, samples, k, models, 0);
      ck_launch();
    }
    {
      IPLS_PROF("classify_hist", 8.0 * level_keys);
      k_classify_hist<F64><<<nchunk, kTileThreads, classify_smem(k), st>>>(
          src, chunks, segs, models, k, chunk_hist, chunk_rep, d_err,
          (F64 && level == 0) ? 1 : 0, nullptr, 0);
      ck_launch();
    }
    {
      IPLS_PROF("unit_reduce", 0);
      k_unit_reduce<<<col_blocks(nunit, k), 256, 0, st>>>(units, nunit, k, chunk_hist,
                                                           chunk_rep, unit_cnt, unit_rep);
      ck_launch();
    }
    {
      IPLS_PROF("seg_scan", 0);
      k_seg_scan<<<col_blocks(nseg, k), 256, 0, st>>>(segs, nseg, k, unit_cnt, unit_rep,
                                                       seg_tot, seg_rep);
      ck_launch();
    }
    OffsetsArgs oa;
    oa.segs = segs; oa.models = models; oa.seg_tot = seg_tot; oa.seg_rep = seg_rep;
    oa.seg_dst = seg_dst; oa.k = k; oa.base_case = p.B; oa.level = level;
    oa.chunk_keys = p.chunk_keys;
    oa.nsegs = at<SegDesc>(fixed, FL.segs[nxt]);
    oa.nchunks = at<ChunkDesc>(fixed, FL.chunks[nxt]);
    oa.nunits = at<UnitDesc>(fixed, FL.units[nxt]);
    oa.nctr = nctr;
    oa.cap_segs = p.cap_segs; oa.cap_chunks = p.cap_chunks; oa.cap_units = p.cap_units;
    oa.cap_samples = p.cap_samples;
    oa.wins = wins; oa.cap_wins = p.cap_wins; oa.fills = fills; oa.cap_fills = p.cap_fills;
    oa.err = d_err;
    {
      IPLS_PROF("seg_offsets", 0);
      k_seg_offsets<<<nseg, kOffThreads, 0, st>>>(oa);
      ck_launch();
    }
    {
      IPLS_PROF("chunk_prefix", 0);
      k_chunk_prefix<<<col_blocks(nunit, k), 256, 0, st>>>(units, nunit, k, unit_cnt,
                                                            chunk_hist);
      ck_launch();
    }
    {
      IPLS_PROF("scatter", 16.0 * level_keys);
      launch_scatter<F64>(p.log2k, dim3(nchunk), scatter_smem(k), st, src, keys, scr, chunks,
                          models, k, chunk_hist, seg_dst, d_err);
    }

    if (trace) {
      std::vector<SegDesc> hs(nseg);
      std::vector<ModelDev> hm(nseg);
      std::vector<uint32_t> ht((size_t)nseg * k);
      std::vector<uint64_t> hsmp(nsample);
      ck(cudaMemcpyAsync(hs.data(), segs, nseg * sizeof(SegDesc), cudaMemcpyDeviceToHost, st));
      ck(cudaMemcpyAsync(hm.data(), models, nseg * sizeof(ModelDev), cudaMemcpyDeviceToHost, st));
      ck(cudaMemcpyAsync(ht.data(), seg_tot, ht.size() * 4, cudaMemcpyDeviceToHost, st));
      ck(cudaMemcpyAsync(hsmp.data(), samples, nsample * 8, cudaMemcpyDeviceToHost, st));
      if (trace->tr->d_snapshots && level < trace->tr->snapshot_levels) {
        uint64_t* snap = static_cast<uint64_t*>(trace->tr->d_snapshots) + (size_t)level * n;
        if (level > 0)
          ck(cudaMemcpyAsync(snap, snap - n, n * 8, cudaMemcpyDeviceToDevice, st));
        k_snapshot<<<nseg, 256, 0, st>>>(segs, keys, scr, (level + 1) & 1, snap);
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
          c[b] = ht[(size_t)s * k + b] & ~kInhBit;
          if (hm[s].kind == kModelLinear && c[b] == hs[s].m) r.requeued = 1;
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
    if (herr & kErrNan) return IPLS_ERR_NAN_KEY;
    if (herr & kErrOverflow) return IPLS_ERR_OUT_OF_MEMORY;

    // base case of this level's base children, fills of its homogeneous children
    if (c.n_windows) {
      IPLS_PROF("base_sort", 16.0 * c.win_keys);
      k_base_sort<F64><<<c.n_windows, kBaseThreads, base_smem(), st>>>(wins, keys, scr, d_err, 0);
      ck_launch();
    }
    if (c.n_fills) {
      IPLS_PROF("fill", 8.0 * c.fill_keys);
      k_fill<<<c.n_fills, 256, 0, st>>>(fills, keys);
      ck_launch();
    }
    if (trace) trace->tr->levels = level + 1;
    nseg = c.n_segs;
    level_keys = c.keys;
    nchunk = c.n_chunks;
    nunit = c.n_units;
    nsample = c.n_samples;
  }
  ck(cudaStreamSynchronize(st));
  prof_collect();
  return IPLS_OK;
}

ipls_status check_cfg(const ipls_config* cfg, ipls_config* out) {
  ipls_config c = cfg ? *cfg : ipls_default_config();
  if (c.k < 3 || c.k > IPLS_MAX_K) return IPLS_ERR_INVALID_ARGUMENT;
  if (c.base_case < 1 || c.base_case > IPLS_MAX_BASE_CASE) return IPLS_ERR_INVALID_ARGUMENT;
  if (c.flags != 0) return IPLS_ERR_INVALID_ARGUMENT;
  *out = c;
  return IPLS_OK;
}

ipls_status sort_impl(void* d_keys, size_t n, ipls_key_type t, const ipls_config* cfg_in,
                      void* d_ws, size_t ws_bytes, void* stream, ipls_trace* tr) {
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
    const Params p = make_params(n, cfg.k, cfg.base_case);
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
                             meta_cache, sc.h_ctr, st, cfg.seed, tr ? &sink : nullptr)
            : run_sort<false>(static_cast<uint64_t*>(d_keys), p, fixed, meta_in, meta_bytes,
                              meta_cache, sc.h_ctr, st, cfg.seed, tr ? &sink : nullptr);
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

size_t ipls_workspace_bytes(size_t n, ipls_key_type t, const ipls_config* cfg) {
  ipls_config c;
  if (check_cfg(cfg, &c) != IPLS_OK || (t != IPLS_KEY_F64 && t != IPLS_KEY_U64)) return 0;
  if (n <= 1) return 0;
  const Params p = make_params(n, c.k, c.base_case);
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

ipls_status ipls_fit_fmcd(const void* d_sorted_sample, size_t S, ipls_key_type t, uint32_t k,
                          ipls_model* h_out, void* stream) {
  if (!d_sorted_sample || !h_out) return IPLS_ERR_INVALID_ARGUMENT;
  if (S < 4 || S > (size_t)kFitMaxS || k < 3 || k > IPLS_MAX_K) return IPLS_ERR_INVALID_ARGUMENT;
  if (t != IPLS_KEY_F64 && t != IPLS_KEY_U64) return IPLS_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    StreamCache& sc = cache_for(stream);
    const size_t need = align_up(S * 8, 256) + 256 + 256;
    sc.meta.ensure(need);
    uint64_t* smp = static_cast<uint64_t*>(sc.meta.ptr);
    SegDesc* dseg = at<SegDesc>(sc.meta.ptr, align_up(S * 8, 256));
    ModelDev* dmod = at<ModelDev>(sc.meta.ptr, align_up(S * 8, 256) + 256);
    if (t == IPLS_KEY_F64) {
      set_attrs<true>();
      k_keys_to_ok_f64<<<(uint32_t)((S + 255) / 256), 256, 0, st>>>(
          static_cast<const uint64_t*>(d_sorted_sample), smp, (uint32_t)S);
      ck_launch();
    } else {
      set_attrs<false>();
      ck(cudaMemcpyAsync(smp, d_sorted_sample, S * 8, cudaMemcpyDeviceToDevice, st));
    }
    SegDesc sd{};
    sd.S = (uint32_t)S;
    ck(cudaMemcpyAsync(dseg, &sd, sizeof(sd), cudaMemcpyHostToDevice, st));
    if (t == IPLS_KEY_F64)
      k_fit<true><<<1, kFitThreads, fit_smem(), st>>>(dseg, smp, k, dmod, 1);
    else
      k_fit<false><<<1, kFitThreads, fit_smem(), st>>>(dseg, smp, k, dmod, 1);
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

ipls_status ipls_partition_level(const void* d_in, void* d_out, size_t n, ipls_key_type t,
                                 const ipls_model* h_model, uint64_t* d_offsets,
                                 uint16_t* d_bucket_ids, void* stream) {
  if (!h_model || !d_offsets) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0 && (!d_in || !d_out)) return IPLS_ERR_INVALID_ARGUMENT;
  if (n > 0xFFFFFFFFull) return IPLS_ERR_INVALID_ARGUMENT;
  if (t != IPLS_KEY_F64 && t != IPLS_KEY_U64) return IPLS_ERR_INVALID_ARGUMENT;
  const bool eq3 = h_model->kind == IPLS_MODEL_EQ3;
  if (!eq3 && h_model->kind != IPLS_MODEL_LINEAR) return IPLS_ERR_INVALID_ARGUMENT;
  const uint32_t k = eq3 ? 3u : h_model->k;
  if (k < 3 || k > IPLS_MAX_K) return IPLS_ERR_INVALID_ARGUMENT;
  const uint32_t k_eff = k;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  try {
    if (n == 0) {
      std::vector<uint64_t> z(k_eff + 1, 0);
      ck(cudaMemcpyAsync(d_offsets, z.data(), z.size() * 8, cudaMemcpyHostToDevice, st));
      ck(cudaStreamSynchronize(st));
      return IPLS_OK;
    }
    StreamCache& sc = cache_for(stream);
    const uint32_t ck_keys = pick_chunk_keys(n);
    const uint32_t nchunk = (uint32_t)((n + ck_keys - 1) / ck_keys);
    const uint32_t nunit = (nchunk + kUnitChunks - 1) / kUnitChunks;
    MetaLayout ML = meta_layout(1, nchunk, nunit, 0, k);
    size_t o = align_up(ML.total, 256);
    const size_t off_seg = o; o += 256;
    const size_t off_ch = o; o = align_up(o + nchunk * sizeof(ChunkDesc), 256);
    const size_t off_un = o; o = align_up(o + nunit * sizeof(UnitDesc), 256);
    const size_t off_err = o; o += 256;
    sc.meta.ensure(o);
    void* meta = sc.meta.ptr;
    SegDesc* dseg = at<SegDesc>(meta, off_seg);
    ChunkDesc* dch = at<ChunkDesc>(meta, off_ch);
    UnitDesc* dun = at<UnitDesc>(meta, off_un);
    uint32_t* derr = at<uint32_t>(meta, off_err);
    ModelDev hm{};
    hm.A = h_model->a; hm.B = h_model->b; hm.pivot_ok = h_model->pivot_ok;
    hm.kind = h_model->kind; hm.D = h_model->D; hm.capped = h_model->capped; hm.k_eff = k_eff;
    ModelDev* dmod = at<ModelDev>(meta, ML.models);
    ck(cudaMemcpyAsync(dmod, &hm, sizeof(hm), cudaMemcpyHostToDevice, st));
    ck(cudaMemsetAsync(derr, 0, 16, st));
    k_init_root<<<std::max<uint32_t>(1, (nchunk + 255) / 256), 256, 0, st>>>(dseg, dch, dun, n, 0,
                                                                          ck_keys, 0u);
    ck_launch();
    uint32_t* chunk_hist = at<uint32_t>(meta, ML.chunk_hist);
    uint64_t* chunk_rep = at<uint64_t>(meta, ML.chunk_rep);
    uint32_t* unit_cnt = at<uint32_t>(meta, ML.unit_cnt);
    uint64_t* unit_rep = at<uint64_t>(meta, ML.unit_rep);
    uint32_t* seg_tot = at<uint32_t>(meta, ML.seg_tot);
    uint64_t* seg_rep = at<uint64_t>(meta, ML.seg_rep);
    uint64_t* seg_dst = at<uint64_t>(meta, ML.seg_dst);
    const uint64_t* in = static_cast<const uint64_t*>(d_in);
    uint64_t* out = static_cast<uint64_t*>(d_out);
    uint32_t log2k = 0;
    while ((1u << log2k) < k) ++log2k;
    if (log2k < 2) log2k = 2;
    auto body = [&](auto f64tag) {
      constexpr bool F64 = decltype(f64tag)::value;
      set_attrs<F64>();
      k_classify_hist<F64><<<nchunk, kTileThreads, classify_smem(k), st>>>(
          in, dch, dseg, dmod, k, chunk_hist, chunk_rep, derr, 0, d_bucket_ids, 0);
      ck_launch();
      k_unit_reduce<<<col_blocks(nunit, k), 256, 0, st>>>(dun, nunit, k, chunk_hist, chunk_rep,
                                                           unit_cnt, unit_rep);
      ck_launch();
      k_seg_scan<<<col_blocks(1, k), 256, 0, st>>>(dseg, 1, k, unit_cnt, unit_rep, seg_tot,
                                                    seg_rep);
      ck_launch();
      k_single_offsets<<<1, kOffThreads, 0, st>>>(seg_tot, k, k_eff, seg_dst, d_offsets);
      ck_launch();
      k_chunk_prefix<<<col_blocks(nunit, k), 256, 0, st>>>(dun, nunit, k, unit_cnt, chunk_hist);
      ck_launch();
      launch_scatter<F64>(log2k, dim3(nchunk), scatter_smem(k), st, in, out, out, dch, dmod, k,
                          chunk_hist, seg_dst, derr);
    };
    if (t == IPLS_KEY_F64) body(std::true_type{}); else body(std::false_type{});
    ck(cudaStreamSynchronize(st));
    return IPLS_OK;
  } catch (const CudaFail& f) {
    g_last_cuda_error = cudaGetErrorString(f.e);
    return IPLS_ERR_CUDA;
  }
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
