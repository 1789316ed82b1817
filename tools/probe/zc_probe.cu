// Host-link probe: copy-engine H2D vs SM-driven zero-copy reads of pinned host memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  #pragma unroll 4
  for (; i < n; i += stride) dst[i] = src[i];
}
__global__ void zc_copy_unroll(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  // each thread issues 8 independent loads before storing
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 7*stride < n; i += 8*stride) {
    uint4 v[8];
    #pragma unroll
    for (int j=0;j<8;j++) v[j] = __ldg(src + i + j*stride);
    #pragma unroll
    for (int j=0;j<8;j++) dst[i + j*stride] = v[j];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

int main() {
  int dev=0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d pciBus %d asyncEngines %d\n", p.name, p.multiProcessorCount, p.pciBusID, p.asyncEngineCount);
  size_t bytes = 352321536ull;  // one 8x7B expert
  void* h; CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped|cudaHostAllocPortable));
  memset(h, 1, bytes);
  void* d; CK(cudaMalloc(&d, bytes));
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best=1e9, ms;
  for (int it=0; it<10; it++) { cudaEventRecord(a,s); cudaMemcpyAsync(d,h,bytes,cudaMemcpyHostToDevice,s); cudaEventRecord(b,s); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
  printf("copy-engine H2D 352MB: best %.3f ms = %.2f GB/s\n", best, bytes/best/1e6);
  // chunked copies 4 MB in 2 streams
  cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  best=1e9;
  for (int it=0; it<5; it++) { cudaEventRecord(a,s); size_t ch=8<<20; for(size_t o=0;o<bytes;o+=ch){size_t n=bytes-o<ch?bytes-o:ch; cudaMemcpyAsync((char*)d+o,(char*)h+o,n,cudaMemcpyHostToDevice,s);} cudaEventRecord(b,s); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
  printf("copy-engine H2D 8MB chunks: best %.3f ms = %.2f GB/s\n", best, bytes/best/1e6);
  size_t n = bytes/16;
  for (int blocks : {148, 296, 592, 1184, 2368}) for (int threads : {256, 512, 1024}) {
    best=1e9;
    for (int it=0; it<5; it++) { cudaEventRecord(a,s); zc_copy_unroll<<<blocks,threads,0,s>>>((const uint4*)hd,(uint4*)d,n); cudaEventRecord(b,s); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
    printf("zero-copy SM read unroll8 grid %d x %d: best %.3f ms = %.2f GB/s\n", blocks, threads, best, bytes/best/1e6);
  }
  for (int blocks : {296, 1184}) {
    best=1e9;
    for (int it=0; it<5; it++) { cudaEventRecord(a,s); zc_copy<<<blocks,512,0,s>>>((const uint4*)hd,(uint4*)d,n); cudaEventRecord(b,s); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
    printf("zero-copy SM read simple grid %d x 512: best %.3f ms = %.2f GB/s\n", blocks, best, bytes/best/1e6);
  }
  // concurrent: copy engine + zero-copy on different halves
  best=1e9;
  for (int it=0; it<5; it++) { cudaEventRecord(a,s); cudaMemcpyAsync(d,h,bytes/2,cudaMemcpyHostToDevice,s2); zc_copy_unroll<<<1184,512,0,s>>>((const uint4*)hd + n/2,(uint4*)d + n/2,n/2); cudaEventRecord(b,s); cudaStreamSynchronize(s2); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
  printf("CE half + ZC half concurrently: %.3f ms = %.2f GB/s (approx)\n", best, bytes/best/1e6);
  // 1 GiB
  size_t gb = 1ull<<30; void* h2; CK(cudaHostAlloc(&h2, gb, 0)); memset(h2,2,gb); void* d2; CK(cudaMalloc(&d2, gb));
  best=1e9;
  for (int it=0; it<10; it++) { cudaEventRecord(a,s); cudaMemcpyAsync(d2,h2,gb,cudaMemcpyHostToDevice,s); cudaEventRecord(b,s); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
  printf("copy-engine H2D 1GiB: best %.3f ms = %.2f GB/s\n", best, gb/best/1e6);
  best=1e9;
  for (int it=0; it<10; it++) { cudaEventRecord(a,s); cudaMemcpyAsync(h2,d2,gb,cudaMemcpyDeviceToHost,s); cudaEventRecord(b,s); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms; }
  printf("copy-engine D2H 1GiB: best %.3f ms = %.2f GB/s\n", best, gb/best/1e6);
  return 0;
}
