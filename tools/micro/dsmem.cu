// DSMEM throughput on B200 (dev tool): random 8-byte stores from every thread of a thread-block
// cluster into the shared memory of random CTAs of the same cluster, vs local random stores.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}
constexpr int BUF = 16384;  // u64 per CTA (128 KB)
template <bool REMOTE>
__global__ void k(int iters, uint64_t* out) {
  extern __shared__ uint64_t buf[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned nb = cl.num_blocks();
  for (int i = threadIdx.x; i < BUF; i += blockDim.x) buf[i] = 0;
  cl.sync();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hsh(s * 977u + it);
    const unsigned r = REMOTE ? (h >> 20) % nb : cl.block_rank();
    uint64_t* dst = cl.map_shared_rank(buf, r);
    dst[h & (BUF - 1)] = (uint64_t)h * it;
  }
  cl.sync();
  uint64_t acc = 0;
  for (int i = threadIdx.x; i < BUF; i += blockDim.x) acc ^= buf[i];
  if (acc == 0x123) out[0] = acc;
}
// coalesced remote reads: each warp reads 32 consecutive u64 (256 B) of a random CTA
__global__ void kr(int iters, uint64_t* out) {
  extern __shared__ uint64_t buf[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned nb = cl.num_blocks();
  for (int i = threadIdx.x; i < BUF; i += blockDim.x) buf[i] = i;
  cl.sync();
  const int lane = threadIdx.x & 31;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hsh((s >> 5) * 977u + it);
    const unsigned r = (h >> 20) % nb;
    const uint64_t* src = cl.map_shared_rank(buf, r);
    acc += src[((h & (BUF / 32 - 1)) << 5) + lane];
  }
  cl.sync();
  if (acc == 0x123) out[0] = acc;
}
void runr(int csize, int threads) {
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = BUF * 8;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cfg.gridDim = dim3(csize * (148 / csize));
  cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, BUF * 8);
  cudaFuncSetAttribute(kr, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, (void*)kr, &cfg);
  cfg.gridDim = dim3(csize * ncl);
  uint64_t* out; cudaMalloc(&out, 8);
  const int iters = 2048;
  cudaLaunchKernelEx(&cfg, kr, iters, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kr, iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)cfg.gridDim.x * threads * iters * 8;
  printf("coalesced remote reads cluster=%2d SMs=%3d: %.0f GB/s total, %.1f B/clk/SM\n", csize, csize * ncl,
         bytes / ms / 1e6, bytes / ms / 1e3 / 1.9e6 / (csize * ncl));
  cudaFree(out);
}
template <bool REMOTE>
void run(int csize, int threads) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize * (148 / csize));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = BUF * 8;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<REMOTE>, cudaFuncAttributeMaxDynamicSharedMemorySize, BUF * 8);
  cudaFuncSetAttribute(k<REMOTE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int ncl = 0;
  cudaOccupancyMaxActiveClusters(&ncl, (void*)k<REMOTE>, &cfg);
  cfg.gridDim = dim3(csize * ncl);
  uint64_t* out; cudaMalloc(&out, 8);
  const int iters = 2048;
  cudaLaunchKernelEx(&cfg, k<REMOTE>, iters, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k<REMOTE>, iters, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  const double stores = (double)cfg.gridDim.x * threads * iters;
  printf("%s cluster=%2d clusters=%3d SMs=%3d threads=%d: %.1f G stores/s (%.2f per SM-clk @1.9GHz) %s\n",
         REMOTE ? "remote" : "local ", csize, ncl, csize * ncl, threads, stores / ms / 1e6,
         stores / ms / 1e3 / 1.9e6 / (csize * ncl), cudaGetErrorString(e));
  cudaFree(out);
}
int main() {
  for (int cs : {2, 4, 8, 16}) { run<true>(cs, 1024); run<false>(cs, 1024); runr(cs, 1024); }
  return 0;
}
