// Faithful replica of the engine's signalling: compute thread enqueues [gate -> spin -> work]*N;
// a worker thread polls the gate's mapped mail, issues memcpy+event on its own stream,
// polls the event and releases the spin through a mapped flag.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <thread>
#include <chrono>
#include <vector>
#include <cuda_runtime.h>

struct Ctl { volatile unsigned ready; volatile unsigned mail; volatile unsigned timeouts; };

__global__ void gate(Ctl* c, unsigned seq) {
  if (threadIdx.x == 0) { __threadfence_system(); c->mail = seq + 1; __threadfence_system(); }
}
__global__ void spin(Ctl* c, unsigned target) {
  if (threadIdx.x) return;
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while ((int)(c->ready - target) < 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > 1000000000ull) { atomicAdd((unsigned*)&c->timeouts, 1u); return; }
    __nanosleep(256);
  }
}
__global__ void work(float* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] * 0.5f + 1.f;
}

int main(int argc, char** argv) {
  const int steps = 8;
  const int follow = argc > 1 ? atoi(argv[1]) : 4;
  const int use_legacy = argc > 2 ? atoi(argv[2]) : 0;
  cudaSetDevice(0);
  Ctl* c; cudaHostAlloc(&c, sizeof(Ctl), cudaHostAllocMapped); memset(c, 0, sizeof(Ctl));
  Ctl* cd; cudaHostGetDevicePointer((void**)&cd, c, 0);
  size_t bytes = 512 << 10;
  char* h; cudaHostAlloc(&h, bytes * steps, cudaHostAllocPortable);
  char* d; cudaMalloc(&d, bytes * steps);
  float* x; cudaMalloc(&x, 1 << 20);
  cudaStream_t comp = 0, copy;
  if (!use_legacy) cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking);
  const int precreate = argc > 3 ? atoi(argv[3]) : 0;
  std::vector<cudaEvent_t> pool;
  if (precreate) {
    for (int i = 0; i < 64; ++i) { cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming); pool.push_back(e); }
    cudaMemcpyAsync(d, h, 4096, cudaMemcpyHostToDevice, copy);
    cudaEventRecord(pool[0], copy);
    cudaStreamSynchronize(copy);
  }
  std::atomic<bool> stop{false};
  std::thread worker([&] {
    cudaSetDevice(0);
    unsigned next = 0;
    std::vector<std::pair<unsigned, cudaEvent_t>> pend;
    while (!stop) {
      if (!pend.empty() && cudaEventQuery(pend.front().second) == cudaSuccess) {
        c->ready = pend.front().first + 1;
        if (precreate) pool.push_back(pend.front().second); else cudaEventDestroy(pend.front().second);
        pend.erase(pend.begin());
        continue;
      }
      if (c->mail >= next + 1) {
        cudaMemcpyAsync(d + next * bytes, h + next * bytes, bytes, cudaMemcpyHostToDevice, copy);
        cudaEvent_t e;
        if (precreate) { e = pool.back(); pool.pop_back(); } else cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        cudaEventRecord(e, copy);
        pend.push_back({next, e});
        ++next;
      }
    }
  });
  auto t0 = std::chrono::steady_clock::now();
  for (int s = 0; s < steps; ++s) {
    gate<<<1, 32, 0, comp>>>(cd, s);
    spin<<<1, 32, 0, comp>>>(cd, s + 1);
    for (int k = 0; k < follow; ++k) work<<<256, 256, 0, comp>>>(x, 1 << 18);
  }
  cudaStreamSynchronize(comp);
  double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  stop = true; worker.join();
  printf("precreate=%d follow=%d legacy=%d: %d steps in %.2f ms, timeouts=%u\n", precreate, follow, use_legacy, steps, ms, c->timeouts);
  (void)0;
  return 0;
}
