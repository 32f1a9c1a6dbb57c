// ipls_device.cuh — device primitives of the sm_100a IPLS path.
//
// Key domains (R0, R17): a key is a raw 64-bit word.  Its ordering key `ok` is the
// order-preserving unsigned image (doubles: flip all bits of negatives, set the sign bit of
// non-negatives; u64: identity) and its model value `v` is the double itself or the u64
// converted round-to-nearest.  The partition model is evaluated as two separately
// rounded operations, y = RN(RN(a*v) + b), written with __dmul_rn/__dadd_rn so that no FMA
// contraction can change a bucket (R7).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ipls {

constexpr uint32_t kModelLinear = 0;
constexpr uint32_t kModelEq3 = 1;
constexpr uint32_t kModelTree = 2;   // splitter tree (IPS4o's classifier)
// Bucketer MODE only (ModelDev.kind stays kModelTree; leaves != k selects it per chunk): the
// tree with equality buckets (R24).  Its own instantiation, so that the plain tree's loops keep
// their code (a run-time flag inside one instantiation cost the plain tree 4.5 % on C2).
constexpr uint32_t kModelTreeEq = 3;
constexpr uint32_t kSegForceEq3 = 1u;
constexpr uint64_t kDstUserBit = 1ull << 63;  // seg_dst encoding: buffer select
constexpr uint32_t kInhBit = 1u << 31;        // count word: child not homogeneous

struct SegDesc {            // one partition work item of a level (segment of the array)
  uint64_t begin;           // absolute position of the segment
  uint32_t m;               // keys in the segment (> base case, or requeued)
  uint32_t S;               // sample size S(m) (R1, R19)
  uint64_t sample_off;      // offset of its sample in the level's sample buffer
  uint32_t chunk_first, nchunks;
  uint32_t flags;           // kSegForceEq3
  uint32_t pad;
};

struct ModelDev {           // fitted model of one segment (Listing 1 outputs, EQ3 or a tree)
  double A, B;
  uint64_t pivot_ok;
  uint32_t kind, D, capped, k_eff;
  uint32_t leaves, pad_;    // tree: leaves of the splitter tree (k, or k / 2 with equality buckets)
  const uint64_t* heap;     // tree: splitters (ordering keys) in heap order, heap[1..leaves-1]
  const uint64_t* top;      // tree, set per CTA: smem copy of heap[0..256) (the top 8 levels)
};

struct ChunkDesc {          // a run of <= CHUNK keys of one segment, processed by one CTA
  uint64_t start;
  uint32_t len, seg;
};

struct Window {             // contiguous run of whole final segments for the base case
  uint64_t begin;
  uint32_t len, buf;        // buf: 0 = user array, 1 = scratch
};

struct Fill {               // homogeneous child that must be written into the user array
  uint64_t begin;
  uint64_t value;
  uint32_t len, pad;
};

struct LevelCounters {      // device-side counters of the level being built
  uint32_t n_segs, n_chunks, max_S, n_samples;
  uint32_t n_windows, n_fills, err, ticket;  // ticket: chunk order of this level's classify
  uint64_t keys;            // keys in next-level segments
  uint32_t n_wbig, pad;     // single-child base windows above the warp-window cap
  uint64_t win_keys;        // keys in this level's small base-case windows
  uint64_t wbig_keys;       // keys in this level's big base-case windows
  uint64_t fill_keys;       // keys in this level's fills
  uint32_t n_redo;          // this level's segments k_fit_small left to k_gather_fit
  uint32_t sticket;         // chunk tickets of k_term_fused (next level's struct, zeroed)
  uint64_t term_keys;       // keys base-sorted inside k_term_fused
  uint32_t n_twin, n_twin_split;  // terminal windows (k_win_sort); those of split segments
  uint64_t twin_keys;       // keys in terminal windows
  uint64_t tsplit_keys;     // keys of terminal segments scattered into windows (k_tss_scatter)
};

constexpr uint32_t kErrNan = 1u;
constexpr uint32_t kErrOverflow = 2u;

__device__ __forceinline__ uint64_t ok_of_f64(uint64_t bits) {
  return (bits >> 63) ? ~bits : (bits | (1ull << 63));
}
template <bool F64>
__device__ __forceinline__ uint64_t ok_of(uint64_t bits) {
  if constexpr (F64) return ok_of_f64(bits); else return bits;
}
template <bool F64>
__device__ __forceinline__ uint64_t bits_of_ok(uint64_t ok) {
  if constexpr (F64) return (ok >> 63) ? (ok & ~(1ull << 63)) : ~ok; else return ok;
}
template <bool F64>
__device__ __forceinline__ double value_of(uint64_t bits) {
  if constexpr (F64) return __longlong_as_double((long long)bits);
  else return __ull2double_rn(bits);
}

// P:394-402 with R7: 0 if !(y >= 0); k-1 if y >= k; floor(y) otherwise, y = RN(RN(A*v) + B).
// cvt.rzi.u32.f64 (__double2uint_rz) truncates toward zero and saturates: y < 0 (also -inf,
// -0.0 and (-1, 0)) gives 0, NaN gives 0, y >= 2^32 gives 2^32-1; min(., k-1) then clamps
// the top.  That is exactly the three-way rule above, in two instructions.
__device__ __forceinline__ uint32_t linear_bucket(double v, double A, double B, uint32_t km1) {
  const double y = __dadd_rn(__dmul_rn(A, v), B);
  return min(__double2uint_rz(y), km1);
}

// Bucket function with the model kind (MODE = kModelLinear / kModelEq3 / kModelTree) fixed
// at compile time (the kind is uniform per chunk).  Tree: the branchless descent
// j <- 2j + (x > a_j) of P:377-379 over the implicit tree of the k-1 splitters (k a power of
// two); the top 8 levels come from the CTA's smem copy, deeper levels through the L1; ties go
// left (R23).  Equality buckets (R24: a tree of k / 2 leaves): the splitter of the node
// where the descent last went left is the least splitter >= x, i.e. the leaf's own splitter
// s_i; a key equal to it takes bucket 2i + 1, any other key of leaf i bucket 2i.
template <bool F64, int MODE>
struct Bucketer {
  double A, B;
  uint64_t piv;
  uint32_t km1;
  const uint64_t* heap;
  const uint64_t* top;
  int depth;
  uint32_t leaves;
  __device__ __forceinline__ explicit Bucketer(const ModelDev& md, uint32_t k)
      : A(md.A), B(md.B), piv(md.pivot_ok), km1(k - 1), heap(md.heap), top(md.top), depth(0),
        leaves(k) {
    if constexpr (MODE == (int)kModelTree || MODE == (int)kModelTreeEq) {
      leaves = md.leaves;
      while ((2u << depth) <= leaves) ++depth;  // log2 leaves (a power of two)
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint64_t bits) const {
    if constexpr (MODE == (int)kModelEq3) {
      const uint64_t o = ok_of<F64>(bits);
      return (o < piv) ? 0u : ((o == piv) ? 1u : 2u);
    } else if constexpr (MODE == (int)kModelTree) {
      const uint64_t o = ok_of<F64>(bits);
      uint32_t j = 1;
      const int dt = depth < 8 ? depth : 8;
      for (int d = 0; d < dt; ++d) j = 2 * j + (o > top[j] ? 1u : 0u);
      for (int d = dt; d < depth; ++d) j = 2 * j + (o > __ldg(heap + j) ? 1u : 0u);
      return j - leaves;
    } else if constexpr (MODE == (int)kModelTreeEq) {
      const uint64_t o = ok_of<F64>(bits);
      uint32_t j = 1;
      const int dt = depth < 8 ? depth : 8;
      uint64_t last = ~o;  // splitter of the last left turn; != o while there was none
      for (int d = 0; d < dt; ++d) {
        const uint64_t s = top[j];
        const bool right = o > s;
        last = right ? last : s;
        j = 2 * j + (right ? 1u : 0u);
      }
      for (int d = dt; d < depth; ++d) {
        const uint64_t s = __ldg(heap + j);
        const bool right = o > s;
        last = right ? last : s;
        j = 2 * j + (right ? 1u : 0u);
      }
      return 2 * (j - leaves) + (o == last ? 1u : 0u);
    } else {
      return linear_bucket(value_of<F64>(bits), A, B, km1);
    }
  }
};

// ---- async bulk copies (TMA 1-D, cp.async.bulk) and mbarriers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared, completion counted on `bar` (bytes and both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// global store that asks the L2 to keep the line (partially written bucket runs stay
// resident until the next tile completes them)
__device__ __forceinline__ void st_evict_last(uint64_t* p, uint64_t v) {
  asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
               " st.global.L2::cache_hint.b64 [%0], %1, pol;\n}" ::"l"(p), "l"(v) : "memory");
}
// 8- / 16-byte global -> shared copies completed by the issuing thread's cp.async groups
// (the window descriptors and the unaligned head/tail keys of the base case, fetched one
// window ahead so that their latency is not exposed)
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// SplitMix64 output function (R18).
__device__ __forceinline__ uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// S(m) = min(max(ceil(ceil(log2 m)/5) k - 1, 4), floor(m/2))   (R1, R19)
__host__ __device__ __forceinline__ uint32_t sample_size(uint64_t m, uint32_t k) {
  uint32_t lg = 0;
  for (uint64_t x = (m > 0 ? m - 1 : 0); x; x >>= 1) ++lg;
  uint64_t S = (uint64_t)((lg + 4) / 5) * k;
  S = S ? S - 1 : 0;
  if (S < 4) S = 4;
  if (S > m / 2) S = m / 2;
  return (uint32_t)S;
}

// Stratum bounds lo_j = floor(j m / S), hi_j = floor((j+1) m / S) (R2) for j = j0, j0 + step,
// j0 + 2 step, ... with three divisions per thread instead of two 64-bit divisions per
// sample: exact recurrences on (quotient, remainder) of j m / S.
struct StrataWalk {
  uint64_t q, r;    // floor(j m / S), j m mod S
  uint64_t sq, sr;  // floor(step m / S), step m mod S
  uint64_t mq, mr;  // floor(m / S), m mod S: lo_{j+1} = lo_j + mq + (r + mr >= S)
  uint64_t S;
  __device__ __forceinline__ StrataWalk(uint32_t j0, uint32_t step, uint64_t m, uint32_t S_)
      : S(S_) {
    const uint64_t a = (uint64_t)j0 * m, b = (uint64_t)step * m;
    q = a / S; r = a - q * S;
    sq = b / S; sr = b - sq * S;
    mq = m / S; mr = m - mq * S;
  }
  __device__ __forceinline__ uint64_t lo() const { return q; }
  __device__ __forceinline__ uint64_t hi() const { return q + mq + (r + mr >= S ? 1u : 0u); }
  __device__ __forceinline__ void next() {
    q += sq;
    r += sr;
    if (r >= S) { r -= S; ++q; }
  }
};

// ---- block-wide exclusive scan of one uint32 per thread (blockDim multiple of 32) ----
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t* s_warp,
                                                          uint32_t* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    uint32_t t = (lane < NW) ? s_warp[lane] : 0u;
    uint32_t ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < NW) s_warp[lane] = ti - t;
    if (lane == NW - 1) s_warp[NW] = ti;
  }
  __syncthreads();
  uint32_t res = s_warp[w] + inc - x;
  if (total) *total = s_warp[NW];
  __syncthreads();
  return res;
}

}  // namespace ipls
