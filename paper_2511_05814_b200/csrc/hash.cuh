// Counter-based synthetic weights.
//   h   = mix64(mix64(seed ^ mix64(tensor_id)) + index)          (splitmix64 finaliser)
//   s24 = (int32)(h >> 40) - 2^23                                 in [-2^23, 2^23)
//   v   = (float)s24 * c,  c = (float)(sqrt(3) * std / 2^23)     one fp32 rounding
//   w   = bf16_rne(v)  (or v itself for f32 tensors)
// Uniform with variance std^2; integer-only up to one multiply, so the CUDA kernel, the
// oracle's C restatement (oracle/weights.c) and numpy produce identical bits.
#pragma once
#include <cstdint>

namespace moe {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t tensor_key(uint64_t seed, uint64_t tensor_id) {
  return mix64(seed ^ mix64(tensor_id));
}

__host__ __device__ __forceinline__ int32_t hash_s24(uint64_t key, uint64_t index) {
  return static_cast<int32_t>(mix64(key + index) >> 40) - (1 << 23);
}

inline float hash_scale(float std) {
  return static_cast<float>(1.7320508075688772 * static_cast<double>(std) / 8388608.0);
}

__host__ __device__ __forceinline__ uint16_t f32_to_bf16_rne(float v) {
  uint32_t u;
#ifdef __CUDA_ARCH__
  u = __float_as_uint(v);
#else
  __builtin_memcpy(&u, &v, 4);
#endif
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Tensor ids: kind << 40 | layer << 16 | expert << 4 | matrix
enum : uint64_t { kTMixing = 1, kTGateW = 2, kTGateB = 3, kTExpert = 4, kTInput = 5 };
enum : uint64_t { kMatW1 = 1, kMatW3 = 2, kMatW2 = 3 };
__host__ __device__ __forceinline__ uint64_t tensor_id(uint64_t kind, uint64_t layer,
                                                       uint64_t expert, uint64_t matrix) {
  return (kind << 40) | (layer << 16) | (expert << 4) | matrix;
}

}  // namespace moe
