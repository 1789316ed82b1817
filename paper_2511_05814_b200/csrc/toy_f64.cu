// fp64 device implementations of the reference's per-call model API:
//   _gate_topk / gate_select / speculate_next   (toymoe.py:99-126, 149-156)
//   _forward / forward_token                    (toymoe.py:129-146)
// These serve the drop-in object API on arbitrary (possibly tiny) user gates; the decode
// engine uses the fused fp32/bf16 kernels in engine.cu instead.
#include "common.cuh"

namespace moe {

// y[j] = sum_i x[i] * A[i * n + j]   (reference `x @ A` with A (m, n) row-major).
// Threads own output columns, so every warp reads contiguous rows of A.
__global__ void rowvec_matmul_f64(const double* __restrict__ x, const double* __restrict__ A,
                                  int m, int n, double* __restrict__ y) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int i = 0; i < m; ++i) acc = fma(x[i], A[static_cast<long long>(i) * n + j], acc);
  y[j] = acc;
}

// Gate epilogue on one thread: logits (+bias), finiteness, top-k (z desc, id asc),
// softmax with max subtraction (toymoe.py:93-96).  E is small; a single thread keeps the
// reference's exact selection order trivially.
__global__ void gate_select_f64(const double* __restrict__ z_in, const double* __restrict__ bias,
                                int E, int k, int64_t* __restrict__ order,
                                double* __restrict__ probs, int* __restrict__ nonfinite) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool finite = true;
  double m = -INFINITY;
  for (int e = 0; e < E; ++e) {
    const double z = z_in[e] + (bias ? bias[e] : 0.0);
    probs[e] = z;  // stash logits
    finite = finite && isfinite(z);
    m = fmax(m, z);
  }
  if (!finite) {
    *nonfinite = 1;
    return;
  }
  // selection: k rounds of argmax with ties to the lower id (lexsort((arange, -z)))
  for (int r = 0; r < k; ++r) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      bool taken = false;
      for (int q = 0; q < r; ++q) taken = taken || (order[q] == e);
      if (taken) continue;
      if (best < 0 || probs[e] > probs[best]) best = e;
    }
    order[r] = best;
  }
  double s = 0.0;
  for (int e = 0; e < E; ++e) {
    const double v = exp(probs[e] - m);
    probs[e] = v;
    s += v;
  }
  for (int e = 0; e < E; ++e) probs[e] /= s;
}

// h = x + alpha * mixed
__global__ void axpy_f64(const double* __restrict__ x, const double* __restrict__ mixed,
                         double alpha, int n, double* __restrict__ h) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) h[j] = __dadd_rn(x[j], __dmul_rn(alpha, mixed[j]));
}

// inner = tanh(h @ W1[e]) for the expert selected at position `slot`.
__global__ void toy_expert_up_f64(const double* __restrict__ h, const double* __restrict__ w1,
                                  const int64_t* __restrict__ sel, int slot, int d,
                                  double* __restrict__ inner) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const double* W = w1 + sel[slot] * static_cast<long long>(d) * d;
  double acc = 0.0;
  for (int i = 0; i < d; ++i) acc = fma(h[i], W[static_cast<long long>(i) * d + j], acc);
  inner[j] = tanh(acc);
}

// out += p_e * (inner @ W2[e])  (toymoe.py:145; applied in selection order)
__global__ void toy_expert_down_f64(const double* __restrict__ inner,
                                    const double* __restrict__ w2,
                                    const int64_t* __restrict__ sel,
                                    const double* __restrict__ probs, int slot, int d,
                                    double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const int e = static_cast<int>(sel[slot]);
  const double* W = w2 + e * static_cast<long long>(d) * d;
  double acc = 0.0;
  for (int i = 0; i < d; ++i) acc = fma(inner[i], W[static_cast<long long>(i) * d + j], acc);
  out[j] = __dadd_rn(out[j], __dmul_rn(probs[e], acc));
}

static int* nonfinite_flag() {
  static int* p = nullptr;
  if (!p) {
    if (cudaMalloc(&p, sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, sizeof(int));
  }
  return p;
}

static moe_status finish_gate(cudaStream_t s) {
  int* flag = nonfinite_flag();
  int h = 0;
  MOE_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  MOE_CUDA(cudaStreamSynchronize(s));
  if (h) {
    MOE_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    MOE_CUDA(cudaStreamSynchronize(s));
    set_error("gate logits are not finite");
    return MOE_NONFINITE;
  }
  return MOE_OK;
}

}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_gate_topk_f64(const double* h_dev, const double* w_dev, const double* bias_dev,
                             int32_t d, int32_t E, int32_t k, int64_t* order_dev,
                             double* probs_dev, void* stream) {
  MOE_REQUIRE(d >= 1 && E >= 1, "bad gate shape (%d, %d)", d, E);
  MOE_REQUIRE(k >= 1 && k <= E, "top_k must be in [1, %d], got %d", E, k);
  cudaStream_t s = as_stream(stream);
  int* flag = nonfinite_flag();
  MOE_REQUIRE(flag != nullptr, "cannot allocate the device flag");
  double* z = nullptr;
  MOE_CUDA(cudaMallocAsync(&z, sizeof(double) * E, s));
  rowvec_matmul_f64<<<(E + 127) / 128, 128, 0, s>>>(h_dev, w_dev, d, E, z);
  MOE_LAUNCHED();
  gate_select_f64<<<1, 32, 0, s>>>(z, bias_dev, E, k, order_dev, probs_dev, flag);
  MOE_LAUNCHED();
  MOE_CUDA(cudaFreeAsync(z, s));
  return finish_gate(s);
}

moe_status moe_toy_forward_f64(const double* x_dev, const double* mixing_dev,
                               const double* gate_w_dev, const double* gate_b_dev,
                               const double* w1_dev, const double* w2_dev, int32_t d, int32_t E,
                               int32_t k, double alpha, double* out_dev, int64_t* selected_dev,
                               double* probs_dev, void* stream) {
  MOE_REQUIRE(d >= 1 && E >= 1, "bad model shape (d=%d, E=%d)", d, E);
  MOE_REQUIRE(k >= 1 && k <= E, "top_k must be in [1, %d], got %d", E, k);
  cudaStream_t s = as_stream(stream);
  int* flag = nonfinite_flag();
  MOE_REQUIRE(flag != nullptr, "cannot allocate the device flag");
  double *mixed = nullptr, *z = nullptr, *inner = nullptr;
  MOE_CUDA(cudaMallocAsync(&mixed, sizeof(double) * d, s));
  MOE_CUDA(cudaMallocAsync(&z, sizeof(double) * E, s));
  MOE_CUDA(cudaMallocAsync(&inner, sizeof(double) * d, s));
  const int tb = 128, gb = (d + tb - 1) / tb;
  rowvec_matmul_f64<<<gb, tb, 0, s>>>(x_dev, mixing_dev, d, d, mixed);
  MOE_LAUNCHED();
  axpy_f64<<<gb, tb, 0, s>>>(x_dev, mixed, alpha, d, out_dev);  // out = h (mixed stream)
  MOE_LAUNCHED();
  rowvec_matmul_f64<<<(E + 127) / 128, 128, 0, s>>>(out_dev, gate_w_dev, d, E, z);
  MOE_LAUNCHED();
  gate_select_f64<<<1, 32, 0, s>>>(z, gate_b_dev, E, k, selected_dev, probs_dev, flag);
  MOE_LAUNCHED();
  moe_status st = finish_gate(s);
  if (st != MOE_OK) {
    cudaFreeAsync(mixed, s);
    cudaFreeAsync(z, s);
    cudaFreeAsync(inner, s);
    return st;
  }
  // h lives in out_dev; experts read h, so stage it before accumulating
  double* h = mixed;
  MOE_CUDA(cudaMemcpyAsync(h, out_dev, sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
  for (int slot = 0; slot < k; ++slot) {
    toy_expert_up_f64<<<gb, tb, 0, s>>>(h, w1_dev, selected_dev, slot, d, inner);
    MOE_LAUNCHED();
    toy_expert_down_f64<<<gb, tb, 0, s>>>(inner, w2_dev, selected_dev, probs_dev, slot, d,
                                          out_dev);
    MOE_LAUNCHED();
  }
  MOE_CUDA(cudaFreeAsync(mixed, s));
  MOE_CUDA(cudaFreeAsync(z, s));
  MOE_CUDA(cudaFreeAsync(inner, s));
  MOE_CUDA(cudaStreamSynchronize(s));
  return MOE_OK;
}

}  // extern "C"
