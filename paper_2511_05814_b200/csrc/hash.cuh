// Counter-based synthetic weights, approximately N(0, std^2):
//   key = mix64(seed ^ mix64(tensor_id))                          (splitmix64 finaliser)
//   a   = mix64(key + 2 i),  b = mix64(key + 2 i + 1)
//   s   = u(a >> 40) + u(a >> 16) + u(b >> 40) + u(b >> 16),  u(x) = (x & 0xFFFFFF) - 2^23
//         (an Irwin-Hall sum of four uniform 24-bit integers: variance 2^48 / 3)
//   v   = (float)s * c,  c = (float)(sqrt(3) * std / 2^24)       two RNE roundings
//   w   = bf16_rne(v)  (or v itself for f32 tensors)
// Integer-only up to one conversion and one multiply, so the CUDA kernel, the oracle's C
// restatement (oracle/weights.c) and numpy produce identical bits.  The bell shape matters for
// the exponent statistics that expert compression sees (a uniform draw would flatter it).
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

__host__ __device__ __forceinline__ int32_t hash_u24(uint64_t x) {
  return static_cast<int32_t>(x & 0xFFFFFFull) - (1 << 23);
}

__host__ __device__ __forceinline__ int32_t hash_sum4(uint64_t key, uint64_t index) {
  const uint64_t a = mix64(key + 2 * index), b = mix64(key + 2 * index + 1);
  return hash_u24(a >> 40) + hash_u24(a >> 16) + hash_u24(b >> 40) + hash_u24(b >> 16);
}

__host__ __device__ __forceinline__ float hash_value(uint64_t key, uint64_t index, float c) {
#ifdef __CUDA_ARCH__
  return __fmul_rn(__int2float_rn(hash_sum4(key, index)), c);
#else
  return static_cast<float>(hash_sum4(key, index)) * c;
#endif
}

inline float hash_scale(float std) {
  return static_cast<float>(1.7320508075688772 * static_cast<double>(std) / 16777216.0);
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
