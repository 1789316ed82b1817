/*
 * ORACLE -- test infrastructure only (see oracle/__init__.py).
 *
 * C restatement of the engine's synthetic-weight definition (DESIGN.md "Synthetic
 * weights"), written from the spec, not shared with paper_2511_05814_b200/csrc:
 *   key = sm(seed ^ sm(tensor_id))   (sm = splitmix64 finaliser)
 *   a = sm(key + 2i), b = sm(key + 2i + 1)
 *   s = t(a >> 40) + t(a >> 16) + t(b >> 40) + t(b >> 16),  t(x) = (x mod 2^24) - 2^23
 *   v = (float)s * (float)(sqrt(3) * std / 2^24)   (int -> float and the multiply round RNE)
 *   bf16 = round-to-nearest-even(v)
 * Compile with -ffp-contract=off (a single multiply, but keep the rule explicit).
 * Multi-threaded fills let the CPU baseline materialise Mixtral-sized experts quickly.
 */
#include <stdint.h>
#include <string.h>
#include <pthread.h>

static uint64_t sm(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static float scale_of(float std) { return (float)(1.7320508075688772 * (double)std / 16777216.0); }

static inline int32_t t24(uint64_t x) { return (int32_t)(x & 0xFFFFFFu) - (1 << 23); }

static inline float value_at(uint64_t key, uint64_t i, float c) {
  const uint64_t a = sm(key + 2 * i), b = sm(key + 2 * i + 1);
  const int32_t s = t24(a >> 40) + t24(a >> 16) + t24(b >> 40) + t24(b >> 16);
  return (float)s * c;
}

static inline uint16_t to_bf16(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

typedef struct { uint64_t key; float c; int64_t lo, hi; void* out; int kind; } job_t;

static void* run(void* p) {
  job_t* j = (job_t*)p;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    float v = value_at(j->key, (uint64_t)i, j->c);
    if (j->kind == 0) ((uint16_t*)j->out)[i] = to_bf16(v);
    else if (j->kind == 1) ((float*)j->out)[i] = v;
    else {  /* bf16-rounded, widened: the oracle's "identical inputs" (2: f64, 3: f32) */
      uint32_t u = (uint32_t)to_bf16(v) << 16;
      float f;
      memcpy(&f, &u, 4);
      if (j->kind == 2) ((double*)j->out)[i] = (double)f;
      else ((float*)j->out)[i] = f;
    }
  }
  return NULL;
}

/* kind 0: bf16 bits, 1: f32, 2: bf16 widened to f64, 3: bf16 widened to f32 */
void oracle_hash_fill(uint64_t seed, uint64_t tensor_id, float std, int64_t n, int kind,
                      void* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  pthread_t th[64];
  job_t jobs[64];
  const uint64_t key = sm(seed ^ sm(tensor_id));
  const float c = scale_of(std);
  const int64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    int64_t lo = t * per, hi = lo + per < n ? lo + per : n;
    if (lo > hi) lo = hi;
    jobs[t] = (job_t){key, c, lo, hi, out, kind};
    pthread_create(&th[t], NULL, run, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}

/* The transpose of the logical (rows, cols) tensor: out[c * rows + r] = value(r * cols + c),
 * widened bf16 -> f64 (kind 2) or f32 (kind 1).  Lets the CPU baseline hold every matrix in
 * the reference's (d_in, d_out) layout without a separate transpose pass. */
typedef struct { uint64_t key; float c; int64_t rows, cols, c0, c1; void* out; int kind; } tjob_t;

static void* run_t(void* p) {
  tjob_t* j = (tjob_t*)p;
  for (int64_t cc = j->c0; cc < j->c1; ++cc)
    for (int64_t r = 0; r < j->rows; ++r) {
      float v = value_at(j->key, (uint64_t)(r * j->cols + cc), j->c);
      if (j->kind == 1) {
        ((float*)j->out)[cc * j->rows + r] = v;
      } else {
        uint32_t u = (uint32_t)to_bf16(v) << 16;
        float f;
        memcpy(&f, &u, 4);
        if (j->kind == 2) ((double*)j->out)[cc * j->rows + r] = (double)f;
        else ((float*)j->out)[cc * j->rows + r] = f;  /* kind 3: bf16 widened to f32 */
      }
    }
  return NULL;
}

void oracle_hash_fill_t(uint64_t seed, uint64_t tensor_id, float std, int64_t rows, int64_t cols,
                        int kind, void* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  pthread_t th[64];
  tjob_t jobs[64];
  const uint64_t key = sm(seed ^ sm(tensor_id));
  const float c = scale_of(std);
  const int64_t per = (cols + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    int64_t c0 = t * per, c1 = c0 + per < cols ? c0 + per : cols;
    if (c0 > c1) c0 = c1;
    jobs[t] = (tjob_t){key, c, rows, cols, c0, c1, out, kind};
    pthread_create(&th[t], NULL, run_t, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
}
