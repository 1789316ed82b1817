/*
 * ORACLE -- test infrastructure only.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this; the product never does.
 *
 * Plain-C restatement of moesim's whole-layer policy replay
 * (/root/reference/pkg/src/moesim/kernels.py:60-147), one scalar loop per step:
 *   OPT next-use table, backward scan ......................... kernels.py:79-88
 *   lfu-aged decay when t > 0 and t % period == 0 ............. kernels.py:92-94
 *   resident_before snapshot .................................. kernels.py:98-99
 *   misses counted per activation entry ....................... kernels.py:101-104
 *   `need` victims, ascending-e scans with strict comparisons . kernels.py:106-134
 *   load: resident, freq += 1.0, last_touch = t ............... kernels.py:136-142
 * Pinned against the reference's own outputs in tests/golden (see tests/test_oracle.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

enum { O_LRU = 0, O_LFU = 1, O_LFU_AGED = 2, O_OPT = 3 };

int oracle_replay_policy(const int64_t* acts, int64_t T, int32_t K, int32_t E, int32_t C,
                         int32_t policy, double decay_factor, int64_t decay_period,
                         uint8_t* resident_before, uint8_t* evicted) {
  uint8_t* resident = calloc((size_t)E, 1);
  uint8_t* in_act = calloc((size_t)E, 1);
  double* freq = calloc((size_t)E, sizeof(double));
  int64_t* last_touch = malloc(sizeof(int64_t) * (size_t)E);
  int64_t* next_use = NULL;
  int status = 0;
  for (int e = 0; e < E; ++e) last_touch[e] = -1;
  memset(resident_before, 0, (size_t)(T * E));
  memset(evicted, 0, (size_t)(T * E));
  if (policy == O_OPT && T > 0) {
    next_use = malloc(sizeof(int64_t) * (size_t)(T * E));
    int64_t* upcoming = malloc(sizeof(int64_t) * (size_t)E);
    for (int e = 0; e < E; ++e) upcoming[e] = T;
    for (int64_t t = T - 1; t >= 0; --t) {
      for (int e = 0; e < E; ++e) next_use[t * E + e] = upcoming[e];
      for (int j = 0; j < K; ++j) upcoming[acts[t * K + j]] = t;
    }
    free(upcoming);
  }
  int64_t n_res = 0;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t* row = acts + t * K;
    if (policy == O_LFU_AGED && t > 0 && t % decay_period == 0)
      for (int e = 0; e < E; ++e) freq[e] *= decay_factor;
    for (int j = 0; j < K; ++j) in_act[row[j]] = 1;
    for (int e = 0; e < E; ++e) resident_before[t * E + e] = resident[e];
    int64_t n_miss = 0;
    for (int j = 0; j < K; ++j) n_miss += resident[row[j]] == 0;
    int64_t need = n_res + n_miss - C;
    for (int64_t r = 0; r < need; ++r) {
      int victim = -1;
      if (policy == O_LRU) {
        int64_t best = (int64_t)1 << 62;
        for (int e = 0; e < E; ++e)
          if (resident[e] && !in_act[e] && last_touch[e] < best) { best = last_touch[e]; victim = e; }
      } else if (policy == O_OPT) {
        int64_t best = -1;
        for (int e = 0; e < E; ++e)
          if (resident[e] && !in_act[e] && next_use[t * E + e] > best) { best = next_use[t * E + e]; victim = e; }
      } else {
        double bf = INFINITY;
        int64_t bt = (int64_t)1 << 62;
        for (int e = 0; e < E; ++e)
          if (resident[e] && !in_act[e] && (freq[e] < bf || (freq[e] == bf && last_touch[e] < bt))) {
            bf = freq[e]; bt = last_touch[e]; victim = e;
          }
      }
      if (victim < 0) { status = 1; break; }  /* K > C: the reference indexes [-1] here */
      evicted[t * E + victim] = 1;
      resident[victim] = 0;
      --n_res;
    }
    for (int j = 0; j < K; ++j) {
      const int64_t e = row[j];
      if (!resident[e]) { resident[e] = 1; ++n_res; }
      freq[e] += 1.0;
      last_touch[e] = t;
    }
    for (int j = 0; j < K; ++j) in_act[row[j]] = 0;
  }
  free(resident); free(in_act); free(freq); free(last_touch); free(next_use);
  return status;
}
