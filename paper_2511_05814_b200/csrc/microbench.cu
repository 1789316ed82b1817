// Isolated timing of the decode GEMV kernels on synthetic resident weights: the tuning aid
// behind DESIGN.md's kernel table (bench.py measures the same kernels live in the decode).
#include "stream_gemv.cuh"

#include <algorithm>

namespace moe {
moe_status launch_hash_bf16(uint64_t seed, uint64_t tid, float std, long long n, uint16_t* out,
                            cudaStream_t s);
}
using namespace moe;

extern "C" moe_status moe_microbench_gemv(int32_t kernel, int32_t d, int32_t f, int32_t experts,
                                          int32_t stage_kb, int32_t max_stages, int32_t grid,
                                          int32_t rpb, int32_t iters, float* ms_per_iter,
                                          int64_t* bytes_per_iter) {
  MOE_REQUIRE(kernel >= 0 && kernel <= 8, "kernel must be 0..8");
  const bool stream_only = kernel >= 6;  // 6/7/8: stream kernels with the compute skipped
  if (stream_only) kernel -= 6;
  MOE_REQUIRE(experts >= 1 && experts <= 2 && d % 256 == 0 && f % 256 == 0, "bad shape");
  const bool mix = kernel == 0 || kernel == 3;
  const int mode = kernel % 3;
  const long long expert_bytes = 3ll * f * d * 2;
  const int nsets = 4;  // rotate weight sets so consecutive iterations miss in L2
  const long long set_bytes = mix ? 2ll * d * d * 2 : expert_bytes * experts;
  char* pool = nullptr;
  MOE_CUDA(cudaMalloc(&pool, set_bytes * nsets * (mix ? 4 : 1)));
  const long long total = set_bytes * nsets * (mix ? 4 : 1);

  for (long long off = 0; off < total; off += (1ll << 28)) {
    const long long n = std::min<long long>(1ll << 28, total - off) / 2;
    moe_status st = launch_hash_bf16(7, 99 + off, 0.02f, n, reinterpret_cast<uint16_t*>(pool + off), 0);
    if (st != MOE_OK) return st;
  }
  LayerState* state = nullptr;
  StepRecord* rec = nullptr;
  float *x = nullptr, *act = nullptr, *y = nullptr, *h_mid = nullptr, *h_in = nullptr;
  MOE_CUDA(cudaMalloc(&state, sizeof(LayerState) * nsets));
  MOE_CUDA(cudaMalloc(&rec, sizeof(StepRecord)));
  MOE_CUDA(cudaMalloc(&x, sizeof(float) * d));
  MOE_CUDA(cudaMalloc(&act, sizeof(float) * 2 * f));
  MOE_CUDA(cudaMalloc(&y, sizeof(float) * 2 * d));
  MOE_CUDA(cudaMalloc(&h_mid, sizeof(float) * d));
  MOE_CUDA(cudaMalloc(&h_in, sizeof(float) * d));
  MOE_CUDA(cudaMemset(x, 0, sizeof(float) * d));
  MOE_CUDA(cudaMemset(act, 0, sizeof(float) * 2 * f));
  MOE_CUDA(cudaMemset(y, 0, sizeof(float) * 2 * d));
  // every set: experts 0..experts-1 resident in buffers 0..experts-1, all hits (phase 0)
  LayerState hs{};
  for (int e = 0; e < kMaxE; ++e) hs.buf_of[e] = e < experts ? e : -1;
  StepRecord hr{};
  for (int j = 0; j < kMaxK; ++j) hr.sel[j] = hr.acts[j] = -1;
  for (int j = 0; j < experts; ++j) {
    hr.sel[j] = j;
    hr.prob[j] = 0.5f;
    hr.acts[j] = j;
  }
  hr.rb = (1u << experts) - 1u;
  for (int i = 0; i < nsets; ++i)
    MOE_CUDA(cudaMemcpy(state + i, &hs, sizeof(hs), cudaMemcpyHostToDevice));
  MOE_CUDA(cudaMemcpy(rec, &hr, sizeof(hr), cudaMemcpyHostToDevice));

  const StreamGeom gg = stream_geometry(mode, d, f, stage_kb * 1024, max_stages, rpb);
  MOE_REQUIRE(kernel >= 3 || gg.ncb > 0, "no stream geometry for stage_kb=%d rpb=%d", stage_kb, rpb);
  if (kernel >= 3) {
    cudaFuncSetAttribute(mix_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(swiglu_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(down_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  const int G = grid > 0 ? grid : stream_grid(mix ? 1 : 2);
  auto launch = [&](int it) {
    const int set = it % nsets;
    const char* base = pool + set * set_bytes * (mix ? 4 : 1);
    if (kernel < 3) {
      StreamParams sp{};
      sp.d = d;
      sp.f = f;
      sp.K = 2;
      sp.x = x;
      sp.M = reinterpret_cast<const uint16_t*>(base);
      sp.alpha = 0.01f;
      sp.h_in = h_in;
      sp.h_mid = h_mid;
      sp.xin = x;
      sp.rec = rec;
      sp.state = state + set;
      sp.pool = base;
      sp.expert_bytes = expert_bytes;
      sp.phase = 0;
      sp.only = -1;
      sp.act = act;
      sp.yout = y;
      sp.stream_only = stream_only ? 1 : 0;
      if (mode == kModeMix)
        launch_stream<kModeMix>(gg, G, sp, 0);
      else if (mode == kModeUp)
        launch_stream<kModeUp>(gg, G, sp, 0);
      else
        launch_stream<kModeDown>(gg, G, sp, 0);
    } else if (mode == kModeMix) {
      MixParams mp{x, nullptr, nullptr, nullptr, base, 0.01f, d, 2, h_in, h_mid};
      mix_kernel<true><<<std::min(d / 8, 296), 256, static_cast<size_t>(d) * 8>>>(mp);
    } else {
      FfnParams fp{x, rec, state + set, base, expert_bytes, d, f, 2, 0, act, y};
      if (mode == kModeUp)
        swiglu_up_kernel<<<dim3(std::min(f / 8, 296), 2), 256, static_cast<size_t>(d) * 4>>>(fp);
      else
        down_kernel<true><<<dim3(std::min(d / 8, 148), 2), 256, static_cast<size_t>(f) * 4>>>(fp);
    }
  };
  for (int it = 0; it < 3; ++it) launch(it);
  MOE_CUDA(cudaGetLastError());
  MOE_CUDA(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < iters; ++it) launch(it);
  cudaEventRecord(b);
  MOE_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *ms_per_iter = ms / iters;
  const long long per_expert = mode == kModeUp ? 2ll * f * d * 2 : (mode == kModeDown ? 1ll * f * d * 2 : 0);
  *bytes_per_iter = mix ? 2ll * d * d : per_expert * experts;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(pool);
  cudaFree(state);
  cudaFree(rec);
  cudaFree(x);
  cudaFree(act);
  cudaFree(y);
  cudaFree(h_mid);
  cudaFree(h_in);
  return MOE_OK;
}
