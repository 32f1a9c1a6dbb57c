// smem atomic throughput on B200 (dev tool): random bins, with and without the return value.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}
template <int MODE, int K>
__global__ void k(uint32_t* out, int iters) {
  __shared__ uint32_t h[K];
  __shared__ uint64_t st[K];
  for (int i = threadIdx.x; i < K; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t b = hsh(s + it * 0x9E3779B9u) & (K - 1);
    if (MODE == 0) atomicAdd(&h[b], 1u);
    if (MODE == 1) acc += atomicAdd(&h[b], 1u);
    if (MODE == 2) { uint32_t p = atomicAdd(&h[b], 1u); st[p & (K - 1)] = s; }
    if (MODE == 3) atomicAdd(&h[b], it | 1u);  // non-constant increment
    if (MODE == 4) st[b] = (uint64_t)s * it;   // plain random 8-byte stores
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += blockDim.x) atomicAdd(&out[i], h[i] + (uint32_t)st[i] + acc);
}
template <int MODE, int K> void run(const char* name, uint32_t* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, G = 148 * 4, T = 512;
  k<MODE, K><<<G, T>>>(out, iters);
  cudaEventRecord(e0); k<MODE, K><<<G, T>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)G * T * iters;
  printf("%-28s K=%5d  %.2f T ops/s  %.2f ops/clk/SM (1.9GHz)\n", name, K, ops / ms / 1e9, ops / ms / 1e3 / 1.9e6 / 148);
}
int main() {
  uint32_t* out; cudaMalloc(&out, 1 << 20);
  run<0, 1024>("atomicAdd no-ret", out);
  run<1, 1024>("atomicAdd ret", out);
  run<2, 1024>("atomicAdd ret + STS", out);
  run<3, 1024>("atomicAdd var-inc no-ret", out);
  run<4, 1024>("STS.64 random", out);
  run<0, 8192>("atomicAdd no-ret", out);
  run<1, 8192>("atomicAdd ret", out);
  cudaDeviceSynchronize();
  return 0;
}
