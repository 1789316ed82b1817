// Host DRAM read bandwidth of the box (the resource N replicas share: each replica's copy
// engine reads its coded experts from the node-shared host store at ~55 GB/s).
// gcc -O3 -march=native -pthread tools/probe/host_bw.c -o /tmp/host_bw && /tmp/host_bw [GiB]
// Prints read GB/s for 1, 2, 4, ... all threads (best of 3, each thread sums its slice with
// 512-bit loads), plus a multi-threaded memcpy (read + write) figure.
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static uint8_t* buf;
static uint8_t* dst;
static size_t total;

typedef struct {
  size_t off, len;
  int copy;
  uint64_t sink;
} job_t;

static void* worker(void* p) {
  job_t* j = (job_t*)p;
  if (j->copy) {
    memcpy(dst + j->off, buf + j->off, j->len);
    return NULL;
  }
  const __m512i* s = (const __m512i*)(buf + j->off);
  size_t n = j->len / 64;
  __m512i a0 = _mm512_setzero_si512(), a1 = a0, a2 = a0, a3 = a0;
  for (size_t i = 0; i + 4 <= n; i += 4) {
    a0 = _mm512_xor_si512(a0, _mm512_load_si512(s + i));
    a1 = _mm512_xor_si512(a1, _mm512_load_si512(s + i + 1));
    a2 = _mm512_xor_si512(a2, _mm512_load_si512(s + i + 2));
    a3 = _mm512_xor_si512(a3, _mm512_load_si512(s + i + 3));
  }
  a0 = _mm512_xor_si512(_mm512_xor_si512(a0, a1), _mm512_xor_si512(a2, a3));
  j->sink = (uint64_t)_mm512_reduce_add_epi64(a0);
  return NULL;
}

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

static double run(int threads, int copy) {
  pthread_t th[256];
  job_t jobs[256];
  size_t per = total / threads / 4096 * 4096;
  double best = 0;
  for (int r = 0; r < 3; ++r) {
    double t0 = now();
    for (int i = 0; i < threads; ++i) {
      jobs[i] = (job_t){(size_t)i * per, per, copy, 0};
      pthread_create(&th[i], NULL, worker, &jobs[i]);
    }
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    double gbs = (double)per * threads * (copy ? 2 : 1) / (now() - t0) / 1e9;
    if (gbs > best) best = gbs;
  }
  return best;
}

int main(int argc, char** argv) {
  double gib = argc > 1 ? atof(argv[1]) : 8.0;
  total = (size_t)(gib * (1ull << 30));
  int ncpu = (int)sysconf(_SC_NPROCESSORS_ONLN);
  buf = aligned_alloc(4096, total);
  dst = aligned_alloc(4096, total);
  memset(buf, 1, total);
  memset(dst, 0, total);
  printf("{\"buffer_GiB\": %.1f, \"cpus\": %d, \"read_GBps\": {", gib, ncpu);
  int first = 1;
  for (int t = 1; t <= ncpu; t *= 2) {
    printf("%s\"%d\": %.1f", first ? "" : ", ", t, run(t, 0));
    first = 0;
    if (t * 2 > ncpu && t != ncpu) t = ncpu / 2;
  }
  printf("}, \"memcpy_rw_GBps_all_threads\": %.1f}\n", run(ncpu, 1));
  return 0;
}
