// Microbenchmarks that decide the B200 design of the classify/scatter kernels:
// smem histogram update strategies at k=1024, match.any cost, and copy bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352d;x^=x>>15;x*=0x846ca68b;x^=x>>16;return x;}

template<int K>
__global__ void hist_atomic(uint32_t* out, int iters){
  __shared__ uint32_t h[K];
  for(int i=threadIdx.x;i<K;i+=blockDim.x) h[i]=0;
  __syncthreads();
  uint32_t s = blockIdx.x*blockDim.x+threadIdx.x;
  for(int it=0; it<iters; ++it){
    uint32_t b = hsh(s + it*0x9E3779B9u) & (K-1);
    atomicAdd(&h[b],1u);
  }
  __syncthreads();
  for(int i=threadIdx.x;i<K;i+=blockDim.x) atomicAdd(&out[i],h[i]);
}
template<int K>
__global__ void hist_match(uint32_t* out, int iters){
  extern __shared__ uint32_t hw[]; // [warps][K]
  int w=threadIdx.x>>5, lane=threadIdx.x&31; int nw=blockDim.x>>5;
  for(int i=threadIdx.x;i<K*nw;i+=blockDim.x) hw[i]=0;
  __syncthreads();
  uint32_t* h=hw+w*K;
  uint32_t s = blockIdx.x*blockDim.x+threadIdx.x;
  for(int it=0; it<iters; ++it){
    uint32_t b = hsh(s + it*0x9E3779B9u) & (K-1);
    uint32_t peers=__match_any_sync(0xffffffffu,b);
    int leader=__ffs(peers)-1;
    if(lane==leader) h[b]+=__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for(int i=threadIdx.x;i<K;i+=blockDim.x){uint32_t t=0; for(int j=0;j<nw;++j) t+=hw[j*K+i]; atomicAdd(&out[i],t);}
}
template<int K>
__global__ void minmax_atomic(unsigned long long* out, int iters){
  __shared__ unsigned long long mn[K], mx[K];
  for(int i=threadIdx.x;i<K;i+=blockDim.x){mn[i]=~0ull;mx[i]=0;}
  __syncthreads();
  uint32_t s = blockIdx.x*blockDim.x+threadIdx.x;
  for(int it=0; it<iters; ++it){
    uint32_t r=hsh(s + it*0x9E3779B9u); uint32_t b = r & (K-1);
    unsigned long long v=((unsigned long long)r<<20)|it;
    atomicMin(&mn[b],v); atomicMax(&mx[b],v);
  }
  __syncthreads();
  for(int i=threadIdx.x;i<K;i+=blockDim.x){atomicMin(&out[i],mn[i]);atomicMax(&out[K+i],mx[i]);}
}
__global__ void copy128(const int4* __restrict__ a, int4* __restrict__ b, size_t n){
  size_t st=(size_t)gridDim.x*blockDim.x;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=st) b[i]=a[i];
}
__global__ void read128(const int4* __restrict__ a, size_t n, int* sink){
  size_t st=(size_t)gridDim.x*blockDim.x; int acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=st){int4 v=a[i]; acc^=v.x^v.w;}
  if(acc==0x12345) *sink=acc;
}
// unrolled copy: each thread 4 x 16B in flight
__global__ void copy128u(const int4* __restrict__ a, int4* __restrict__ b, size_t n){
  size_t base=(blockIdx.x*(size_t)blockDim.x)*4+threadIdx.x; size_t st=(size_t)gridDim.x*blockDim.x*4;
  for(size_t i=base;i<n;i+=st){int4 v[4];
#pragma unroll
    for(int u=0;u<4;++u){size_t j=i+u*blockDim.x; if(j<n) v[u]=a[j];}
#pragma unroll
    for(int u=0;u<4;++u){size_t j=i+u*blockDim.x; if(j<n) b[j]=v[u];}}
}
int main(){
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  printf("SMs %d\n",sms);
  uint32_t* out; CK(cudaMalloc(&out,1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int iters=2048;
  for(int bs: {256,512,1024}){
    int grid=sms*(2048/bs);
    long long keys=(long long)grid*bs*iters;
    hist_atomic<1024><<<grid,bs>>>(out,iters); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); hist_atomic<1024><<<grid,bs>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("hist_atomic k=1024 bs=%d: %.1f Gkeys/s\n",bs,keys/ms/1e6);
    hist_atomic<256><<<grid,bs>>>(out,iters); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); hist_atomic<256><<<grid,bs>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("hist_atomic k=256 bs=%d: %.1f Gkeys/s\n",bs,keys/ms/1e6);
    size_t sm=(size_t)1024*(bs/32)*4;
    if(sm<=200*1024){
      cudaFuncSetAttribute(hist_match<1024>,cudaFuncAttributeMaxDynamicSharedMemorySize,200*1024);
      int g2=sms*std::max(1,(int)(200*1024/sm)); if(g2*bs>sms*2048) g2=sms*(2048/bs);
      long long k2=(long long)g2*bs*iters;
      hist_match<1024><<<g2,bs,sm>>>(out,iters); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); hist_match<1024><<<g2,bs,sm>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms,e0,e1); printf("hist_match k=1024 bs=%d grid=%d: %.1f Gkeys/s\n",bs,g2,k2/ms/1e6);
    }
    minmax_atomic<1024><<<grid,bs>>>((unsigned long long*)out,iters/4); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); minmax_atomic<1024><<<grid,bs>>>((unsigned long long*)out,iters/4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("minmax_atomic k=1024 bs=%d: %.1f Gkeys/s\n",bs,keys/4/ms/1e6);
  }
  size_t bytes=(size_t)1<<31; int4 *a,*b; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&b,bytes)); cudaMemset(a,1,bytes);
  size_t n=bytes/16; int* sink; cudaMalloc(&sink,4);
  for(int rep=0;rep<2;++rep){
  for(int g: {sms*4, sms*8, sms*16}){
    copy128<<<g,512>>>(a,b,n); cudaEventRecord(e0); copy128<<<g,512>>>(a,b,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("copy128 grid=%d: %.0f GB/s (r+w)\n",g,2.0*bytes/ms/1e6);
    copy128u<<<g,512>>>(a,b,n); cudaEventRecord(e0); copy128u<<<g,512>>>(a,b,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("copy128u grid=%d: %.0f GB/s (r+w)\n",g,2.0*bytes/ms/1e6);
    read128<<<g,512>>>(a,n,sink); cudaEventRecord(e0); read128<<<g,512>>>(a,n,sink); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("read128 grid=%d: %.0f GB/s\n",g,1.0*bytes/ms/1e6);
  }}
  return 0;
}
