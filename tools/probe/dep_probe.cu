// Does a kernel spinning on mapped host memory block copy-engine work on another stream?
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <chrono>
#include <vector>
#include <cuda_runtime.h>

__global__ void spin(volatile unsigned* flag, unsigned target, int* timed_out) {
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag < target) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > 2000000000ull) { *timed_out = 1; return; }
    __nanosleep(500);
  }
}

int run(const char* name, int prio_copy, int dummies, int create_copy_first, size_t bytes) {
  std::vector<cudaStream_t> dummy(dummies);
  cudaStream_t comp, copy;
  int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (create_copy_first) cudaStreamCreateWithPriority(&copy, cudaStreamNonBlocking, prio_copy ? hi : lo);
  for (auto& d : dummy) cudaStreamCreateWithFlags(&d, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
  if (!create_copy_first) cudaStreamCreateWithPriority(&copy, cudaStreamNonBlocking, prio_copy ? hi : lo);
  unsigned* flag; cudaHostAlloc(&flag, 4, cudaHostAllocMapped); *flag = 0;
  unsigned* flag_d; cudaHostGetDevicePointer((void**)&flag_d, flag, 0);
  int* to; cudaHostAlloc(&to, 4, cudaHostAllocMapped); *to = 0; int* to_d; cudaHostGetDevicePointer((void**)&to_d, to, 0);
  void* h; cudaHostAlloc(&h, bytes, 0); void* d; cudaMalloc(&d, bytes);
  int stuck = 0;
  for (int it = 1; it <= 4; ++it) {
    spin<<<1, 32, 0, comp>>>(flag_d, it, to_d);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, copy);
    cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); cudaEventRecord(e, copy);
    auto t0 = std::chrono::steady_clock::now();
    while (cudaEventQuery(e) == cudaErrorNotReady) {}
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *flag = it;
    cudaStreamSynchronize(comp);
    if (*to) { stuck++; *to = 0; }
    printf("%-28s iter %d copy-wait %.2f ms %s\n", name, it, ms, ms > 1000 ? "BLOCKED" : "");
    cudaEventDestroy(e);
  }
  for (auto& x : dummy) cudaStreamDestroy(x);
  cudaStreamDestroy(comp); cudaStreamDestroy(copy);
  cudaFreeHost(flag); cudaFreeHost(to); cudaFreeHost(h); cudaFree(d);
  return stuck;
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  run("plain", 0, 0, 0, 512 << 10);
  run("plain-copyfirst", 0, 0, 1, 512 << 10);
  run("32dummies", 0, 32, 0, 512 << 10);
  run("32dummies-copyfirst", 0, 32, 1, 512 << 10);
  run("hiprio", 1, 0, 0, 512 << 10);
  run("hiprio-32dummies", 1, 32, 0, 512 << 10);
  run("plain-32MB", 0, 0, 0, 32 << 20);
  return 0;
}
