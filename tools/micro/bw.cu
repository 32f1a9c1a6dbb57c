// Bandwidth microbenchmarks that decide the pass structure of the sort (dev tool):
// DRAM vs L2-resident streaming reads/copies, and gathers/scatters of runs of R 8-byte keys
// at random 8-byte-aligned offsets (the access pattern of a level that reads or writes
// bucket runs).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__global__ void rd(const int4* __restrict__ a, size_t n, int passes, int* sink) {
  int acc = 0;
  for (int p = 0; p < passes; ++p)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      int4 v = __ldcg(a + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678) *sink = acc;
}
__global__ void cp(const int4* __restrict__ a, int4* __restrict__ b, size_t n, int passes) {
  for (int p = 0; p < passes; ++p)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      __stcg(b + i, __ldcg(a + i));
}
// each warp handles runs: run r starts at a random 8B offset, R keys, lanes stride over keys
__global__ void gather_runs(const uint64_t* __restrict__ a, size_t n, uint64_t* __restrict__ out,
                            uint32_t nruns, int R) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = w; r < nruns; r += nw) {
    size_t off = ((size_t)hsh(r) * 2654435761ull) % (n - R);
    for (int j = lane; j < R; j += 32) out[(size_t)r * R + j] = __ldcs(a + off + j);
  }
}
__global__ void scatter_runs(const uint64_t* __restrict__ in, size_t n, uint64_t* __restrict__ a,
                             uint32_t nruns, int R) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = w; r < nruns; r += nw) {
    // disjoint destinations: run r -> slot perm(r) (bijective on nruns since multiplier is odd)
    size_t slot = ((size_t)r * 2654435761ull) % nruns;
    for (int j = lane; j < R; j += 32) __stcs(a + slot * R + j, in[(size_t)r * R + j]);
  }
}

int main() {
  const size_t N = 1ull << 27;  // 1 GiB of u64
  uint64_t *a, *b;
  int* sink;
  CK(cudaMalloc(&a, N * 8)); CK(cudaMalloc(&b, N * 8)); CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(a, 1, N * 8)); CK(cudaMemset(b, 2, N * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto T = [&](auto f) { f(); cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); return ms; };
  const int G = 148 * 8, TB = 256;
  ms = T([&] { rd<<<G, TB>>>((const int4*)a, N / 2, 1, sink); });
  printf("dram read      %.0f GB/s\n", N * 8 / ms / 1e6);
  ms = T([&] { cp<<<G, TB>>>((const int4*)a, (int4*)b, N / 2, 1); });
  printf("dram copy      %.0f GB/s (r+w)\n", 2.0 * N * 8 / ms / 1e6);
  for (size_t mb : {8, 16, 32, 48, 64, 96}) {
    size_t n16 = mb * (1 << 20) / 16; int passes = (int)(4096 / mb);
    ms = T([&] { rd<<<G, TB>>>((const int4*)a, n16, passes, sink); });
    printf("L2 read %3zu MB  %.0f GB/s\n", mb, (double)passes * n16 * 16 / ms / 1e6);
    ms = T([&] { cp<<<G, TB>>>((const int4*)a, (int4*)b, n16 / 2, passes); });
    printf("L2 copy %3zu MB  %.0f GB/s (r+w)\n", mb, 2.0 * passes * (n16 / 2) * 16 / ms / 1e6);
  }
  for (int R : {4, 8, 16, 32, 64, 128}) {
    uint32_t nruns = (uint32_t)(N / 2 / R);
    ms = T([&] { gather_runs<<<G, TB>>>(a, N, b, nruns, R); });
    printf("gather runs R=%3d  %.0f GB/s (r+w)\n", R, 2.0 * nruns * R * 8 / ms / 1e6);
    ms = T([&] { scatter_runs<<<G, TB>>>(b, N, a, nruns, R); });
    printf("scatter runs R=%3d %.0f GB/s (r+w)\n", R, 2.0 * nruns * R * 8 / ms / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
