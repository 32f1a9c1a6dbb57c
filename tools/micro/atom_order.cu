// Does a shared-memory atomicAdd from one warp instruction return values in lane order for
// lanes that hit the same address?  (Decides whether the stable-rank fix-up ever triggers.)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}
__global__ void k(unsigned long long* bad, unsigned long long* total, int iters, int nb) {
  extern __shared__ uint32_t c[];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* cw = c + w * 1024;
  for (int i = lane; i < 1024; i += 32) cw[i] = 0;
  __syncwarp();
  unsigned long long nbad = 0, ntot = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t b = hsh(blockIdx.x * 7919u + threadIdx.x * 31u + it * 0x9E3779B9u) % nb;
    uint32_t old = atomicAdd(&cw[b], 1u);
    // lanes with the same b: check order
    for (int src = 0; src < 32; ++src) {
      uint32_t bs = __shfl_sync(~0u, b, src), os = __shfl_sync(~0u, old, src);
      if (src < lane && bs == b) { ntot++; if (os > old) nbad++; }
    }
  }
  atomicAdd(bad, nbad); atomicAdd(total, ntot);
}
int main() {
  unsigned long long *d; cudaMalloc(&d, 16);
  for (int nb : {1, 4, 32, 1024}) {
    for (int bs : {256, 512, 1024}) {
      cudaMemset(d, 0, 16);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
      k<<<296, bs, (bs / 32) * 4096>>>(d, d + 1, 256, nb);
      unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("nb=%4d bs=%4d: same-address lane pairs %llu, out of lane order %llu (%s)\n", nb, bs, h[1], h[0], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
