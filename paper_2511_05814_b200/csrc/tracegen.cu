// Synthetic routing workloads on the GPU: the reference's Zipf and Markov
// activation samplers, driven by host-generated uniforms so traces are bit-identical to
// moesim.tracegen.gen_zipf / gen_markov.
//
//   moe_sample_zipf    <- kernels.sample_zipf_layer    kernels.py:150-184  (one thread per (t, l))
//   moe_sample_markov  <- kernels.sample_markov_layer  kernels.py:187-232  (one thread per layer:
//                                                       token t depends on token t-1)
// Arithmetic follows the reference exactly: fp64 running totals summed in ascending expert
// order, x = u * total, first e with x < acc wins, the last available expert if rounding left
// x == total; rows sorted ascending (_sort_row, kernels.py:235-244).
#include "common.cuh"

namespace moe {
namespace {

constexpr int kMaxTraceE = 64;

__device__ __forceinline__ int draw(const double* w, int E, const uint64_t avail, double u) {
  double total = 0.0;
  for (int e = 0; e < E; ++e)
    if ((avail >> e) & 1ull) total = __dadd_rn(total, w[e]);
  const double x = __dmul_rn(u, total);
  double acc = 0.0;
  for (int e = 0; e < E; ++e)
    if ((avail >> e) & 1ull) {
      acc = __dadd_rn(acc, w[e]);
      if (x < acc) return e;
    }
  for (int e = E - 1; e >= 0; --e)
    if ((avail >> e) & 1ull) return e;
  return -1;
}

__device__ __forceinline__ void sort_row(int64_t* v, int k) {
  for (int i = 1; i < k; ++i) {
    const int64_t key = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > key) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = key;
  }
}

__global__ void zipf_kernel(const double* __restrict__ weights, int L, int E, long long T, int K,
                            const double* __restrict__ uniforms, int64_t* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= T * L) return;
  const long long t = i / L;
  const int l = static_cast<int>(i % L);
  const double* w = weights + static_cast<size_t>(l) * E;
  const double* u = uniforms + (static_cast<size_t>(l) * T + t) * K;
  int64_t* row = out + (static_cast<size_t>(t) * L + l) * K;
  uint64_t avail = E >= 64 ? ~0ull : ((1ull << E) - 1ull);
  for (int j = 0; j < K; ++j) {
    const int e = draw(w, E, avail, u[j]);
    row[j] = e;
    avail &= ~(1ull << e);
  }
  sort_row(row, K);
}

__global__ void markov_kernel(const double* __restrict__ weights, int L, int E, long long T, int K,
                              double repeat_prob, const double* __restrict__ u_retain,
                              const double* __restrict__ u_draw, int64_t* __restrict__ out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const double* w = weights + static_cast<size_t>(l) * E;
  const uint64_t all = E >= 64 ? ~0ull : ((1ull << E) - 1ull);
  for (long long t = 0; t < T; ++t) {
    int64_t* row = out + (static_cast<size_t>(t) * L + l) * K;
    const double* ur = u_retain + (static_cast<size_t>(l) * T + t) * K;
    const double* ud = u_draw + (static_cast<size_t>(l) * T + t) * K;
    uint64_t avail = all;
    int filled = 0;
    if (t > 0) {
      const int64_t* prev = out + (static_cast<size_t>(t - 1) * L + l) * K;
      for (int j = 0; j < K; ++j)
        if (ur[j] < repeat_prob) {
          row[filled++] = prev[j];
          avail &= ~(1ull << prev[j]);
        }
    }
    int draws = 0;
    while (filled < K) {
      const int e = draw(w, E, avail, ud[draws]);
      row[filled++] = e;
      avail &= ~(1ull << e);
      ++draws;
    }
    sort_row(row, K);
  }
}

}  // namespace
}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_sample_zipf(const double* weights_dev, int32_t L, int32_t E, int64_t T, int32_t K,
                           const double* uniforms_dev, int64_t* out_dev, void* stream) {
  MOE_REQUIRE(L >= 1 && E >= 1 && E <= kMaxTraceE && K >= 1 && K <= E && T >= 0,
              "bad trace shape L=%d E=%d K=%d (E <= %d, 1 <= K <= E)", L, E, K, kMaxTraceE);
  if (T == 0) return MOE_OK;
  MOE_REQUIRE(weights_dev && uniforms_dev && out_dev, "null argument");
  const long long n = T * L;
  zipf_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      weights_dev, L, E, T, K, uniforms_dev, out_dev);
  MOE_LAUNCHED();
  return MOE_OK;
}

moe_status moe_sample_markov(const double* weights_dev, int32_t L, int32_t E, int64_t T, int32_t K,
                             double repeat_prob, const double* u_retain_dev,
                             const double* u_draw_dev, int64_t* out_dev, void* stream) {
  MOE_REQUIRE(L >= 1 && E >= 1 && E <= kMaxTraceE && K >= 1 && K <= E && T >= 0,
              "bad trace shape L=%d E=%d K=%d (E <= %d, 1 <= K <= E)", L, E, K, kMaxTraceE);
  MOE_REQUIRE(repeat_prob >= 0.0 && repeat_prob <= 1.0, "repeat_prob must be in [0, 1]");
  if (T == 0) return MOE_OK;
  MOE_REQUIRE(weights_dev && u_retain_dev && u_draw_dev && out_dev, "null argument");
  markov_kernel<<<(L + 31) / 32, 32, 0, as_stream(stream)>>>(weights_dev, L, E, T, K, repeat_prob,
                                                             u_retain_dev, u_draw_dev, out_dev);
  MOE_LAUNCHED();
  return MOE_OK;
}

}  // extern "C"
