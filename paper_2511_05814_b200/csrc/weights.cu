// Synthetic weight generation on the device (counter hash, see hash.cuh).
#include "common.cuh"
#include "hash.cuh"

namespace moe {

__global__ void hash_bf16_kernel(uint64_t key, float c, long long n, uint16_t* __restrict__ out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x * 8;
  for (long long base = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
       base < n; base += stride) {
    if (base + 8 <= n) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float a = hash_value(key, base + 2 * q, c);
        const float b = hash_value(key, base + 2 * q + 1, c);
        w[q] = static_cast<uint32_t>(f32_to_bf16_rne(a)) |
               (static_cast<uint32_t>(f32_to_bf16_rne(b)) << 16);
      }
      *reinterpret_cast<uint4*>(out + base) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (long long i = base; i < n; ++i)
        out[i] = f32_to_bf16_rne(hash_value(key, i, c));
    }
  }
}

__global__ void hash_f32_kernel(uint64_t key, float c, long long n, float* __restrict__ out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    out[i] = hash_value(key, i, c);
}

moe_status launch_hash_bf16(uint64_t seed, uint64_t tid, float std, long long n, uint16_t* out,
                            cudaStream_t s) {
  if (n <= 0) return MOE_OK;
  MOE_REQUIRE((reinterpret_cast<uintptr_t>(out) & 15) == 0, "output must be 16-byte aligned");
  const long long groups = (n + 7) / 8;
  const int threads = 256;
  const long long want = (groups + threads - 1) / threads;
  const int blocks = static_cast<int>(want < 148 * 16 ? want : 148 * 16);
  hash_bf16_kernel<<<blocks, threads, 0, s>>>(tensor_key(seed, tid), hash_scale(std), n, out);
  MOE_LAUNCHED();
  return MOE_OK;
}

moe_status launch_hash_f32(uint64_t seed, uint64_t tid, float std, long long n, float* out,
                           cudaStream_t s) {
  if (n <= 0) return MOE_OK;
  const int threads = 256;
  const long long want = (n + threads - 1) / threads;
  const int blocks = static_cast<int>(want < 148 * 16 ? want : 148 * 16);
  hash_f32_kernel<<<blocks, threads, 0, s>>>(tensor_key(seed, tid), hash_scale(std), n, out);
  MOE_LAUNCHED();
  return MOE_OK;
}

}  // namespace moe

extern "C" {

moe_status moe_hash_weights_bf16(uint64_t seed, uint64_t tensor_id, float std, int64_t n,
                                 uint16_t* out_dev, void* stream) {
  return moe::launch_hash_bf16(seed, tensor_id, std, n, out_dev, moe::as_stream(stream));
}

moe_status moe_hash_weights_f32(uint64_t seed, uint64_t tensor_id, float std, int64_t n,
                                float* out_dev, void* stream) {
  return moe::launch_hash_f32(seed, tensor_id, std, n, out_dev, moe::as_stream(stream));
}

}  // extern "C"
