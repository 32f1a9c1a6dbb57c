// In-warp stable rank of a 10-bit bucket id (dev tool): match.any vs 10 ballots vs an smem
// atomic with return.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/rank tools/micro/rank.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m;
}
template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t kmask) {
  extern __shared__ uint32_t h[];  // 32 warps x 1024 counters
  for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
  const uint32_t lt = lanemask_lt();
  for (int it = 0; it < iters; ++it) {
    const uint32_t b = hsh(s + it * 0x9E3779B9u) & kmask;
    if (MODE == 0) {  // match.any: peers, rank, the leader updates the warp's counter
      const uint32_t peers = __match_any_sync(0xffffffffu, b);
      const uint32_t r = __popc(peers & lt);
      const uint32_t c = h[w * 1024 + b];
      __syncwarp();
      if (r == 0) h[w * 1024 + b] = c + __popc(peers);
      acc += c + r;
    } else if (MODE == 1) {  // ballots on the 10 bits
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < 10; ++i) {
        const bool bit = (b >> i) & 1u;
        const uint32_t v = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? v : ~v;
      }
      const uint32_t r = __popc(peers & lt);
      const uint32_t c = h[w * 1024 + b];
      __syncwarp();
      if (r == 0) h[w * 1024 + b] = c + __popc(peers);
      acc += c + r;
    } else if (MODE == 2) {  // atomic with return (lane order of same-address lanes)
      acc += atomicAdd(&h[w * 1024 + b], 1u);
    } else if (MODE == 3) {  // match only
      acc += __match_any_sync(0xffffffffu, b);
    } else {  // hash only (loop overhead)
      acc += b;
    }
  }
  __syncthreads();
  atomicAdd(&out[threadIdx.x], acc + h[threadIdx.x]);
}
template <int MODE> void run(const char* name, uint32_t* out, uint32_t kmask) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, G = 148, T = 1024;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024 * 4);
  k<MODE><<<G, T, 32 * 1024 * 4>>>(out, iters, kmask);
  cudaEventRecord(e0); k<MODE><<<G, T, 32 * 1024 * 4>>>(out, iters, kmask); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)G * T * iters;  // thread-ops (keys)
  printf("%-22s kmask=%4u  %.3f ms  %.1f G keys/s  %.2f clk per warp-op per SMSP\n", name, kmask, ms,
         ops / ms / 1e6, (ms * 1e-3 * 1.965e9) / ((double)T / 32 / 4 * iters));
}
int main() {
  uint32_t* out; cudaMalloc(&out, 1 << 20);
  for (uint32_t km : {1023u, 15u}) {
    run<4>("hash only", out, km);
    run<3>("match only", out, km);
    run<0>("match rank", out, km);
    run<1>("ballot rank", out, km);
    run<2>("atomic rank", out, km);
  }
  cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
