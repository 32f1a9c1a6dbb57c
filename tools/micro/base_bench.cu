// Base-case kernel harness (dev tool): times k_base_sort on synthetic windows shaped like the
// last level's output (each window = W keys drawn uniformly from a narrow value range, in
// random order), and checks the result is sorted.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
//          -I paper_2208_06902_b200/csrc -o tools/micro/base_bench tools/micro/base_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "ipls_kernels.cuh"
using namespace ipls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void gen(double* a, uint64_t n, uint32_t W) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    double u = (z >> 11) * (1.0 / 9007199254740992.0);
    a[i] = 1.0 + (double)(i / W) * 1e-3 + u * 1e-3;  // window w spans [1+w e-3, 1+(w+1)e-3)
  }
}
__global__ void chk(const double* a, uint64_t n, uint32_t* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] > a[i + 1]) atomicAdd(bad, 1u);
}

int main(int argc, char** argv) {
  const uint64_t n = 100000000ull;
  for (uint32_t W : {256u, 1024u, 2048u, 4096u}) {
    double *a, *b;
    uint32_t* err;
    CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8)); CK(cudaMalloc(&err, 16));
    gen<<<1184, 256>>>(a, n, W);
    const uint32_t nw = (uint32_t)((n + W - 1) / W);
    std::vector<Window> hw(nw);
    for (uint32_t w = 0; w < nw; ++w) { hw[w].begin = (uint64_t)w * W; hw[w].len = (uint32_t)std::min<uint64_t>(W, n - hw[w].begin); hw[w].buf = 1; }
    Window* dw; CK(cudaMalloc(&dw, nw * sizeof(Window)));
    CK(cudaMemcpy(dw, hw.data(), nw * sizeof(Window), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_base_sort<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBCSmem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaMemset(err, 0, 16));
      cudaEventRecord(e0);
      if (W <= kWBCap) {
        const size_t ws = kWBSmemPerWarp * kWBWarps;
        cudaFuncSetAttribute(k_base_warp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws);
        k_base_warp<true><<<148, kWBWarps * 32, ws>>>(dw, nw, (uint64_t*)b, (const uint64_t*)a);
      } else {
        k_base_sort<true, false><<<nw, kBCThreads, kBCSmem>>>(dw, (uint64_t*)b, (const uint64_t*)a, err + 1);
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    CK(cudaMemset(err, 0, 16)); chk<<<1184, 256>>>(b, n, err + 2);
    uint32_t he[3]; CK(cudaMemcpy(he, err, 12, cudaMemcpyDeviceToHost));
#ifdef IPLS_BASE_TIMING
    { unsigned long long ph[16]; cudaMemcpyFromSymbol(ph, g_base_phase, sizeof(ph)); unsigned long long z[16] = {0};
      cudaMemcpyToSymbol(g_base_phase, z, sizeof(z)); double tot = 0; for (int q = 0; q < 11; ++q) tot += ph[q];
      printf("  phases (cycles/window, thread 0 / lane 0):"); for (int q = 0; q < 11; ++q) printf(" %d:%.0f", q, ph[q] / 6.0 / nw); printf(" (cycles per window per warp)"); printf("\n"); }
#endif
    printf("W=%5u windows=%u  %.3f ms  %.0f GB/s (16 B/key)  unsorted=%u\n", W, nw, best, 16.0 * n / best / 1e6, he[2]);
    cudaFree(a); cudaFree(b); cudaFree(err); cudaFree(dw);
  }
  return 0;
}
