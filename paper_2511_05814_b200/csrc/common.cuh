// Shared plumbing for libmoeb200: status/error reporting, launch accounting, warp helpers.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <string>
#include <atomic>

#include "../../include/moeb200.h"

namespace moe {

// thread-local last error (moe_last_error)
void set_error(const char* fmt, ...);
std::atomic<uint64_t>& launch_counter();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Kernel attributes (cudaFuncSetAttribute) are per device: run `f` once per device per call
// site.  Concurrent first calls may both run it, which is harmless.
template <class F>
inline void once_per_device(std::atomic<uint64_t>& done, F f) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(done.load(std::memory_order_acquire) & bit)) {
    f();
    done.fetch_or(bit, std::memory_order_release);
  }
}

#define MOE_CUDA(expr)                                                            \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::moe::set_error("%s failed at %s:%d: %s", #expr, __FILE__, __LINE__,       \
                       cudaGetErrorString(_e));                                   \
      return _e == cudaErrorMemoryAllocation ? MOE_OOM : MOE_CUDA_ERROR;          \
    }                                                                             \
  } while (0)

// Run the rest of the scope on `dev` and give the calling thread its own current device back
// on exit: an ABI call on an engine never leaves the caller's device switched.
struct DeviceGuard {
  int prev = -1;
  cudaError_t status = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) status = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
#define MOE_ON_DEVICE(dev)                 \
  ::moe::DeviceGuard moe_device_guard_(dev); \
  MOE_CUDA(moe_device_guard_.status)

// Check the launch that just happened and count it.
#define MOE_LAUNCHED()                                                            \
  do {                                                                            \
    ::moe::launch_counter().fetch_add(1, std::memory_order_relaxed);              \
    MOE_CUDA(cudaGetLastError());                                                 \
  } while (0)

#define MOE_REQUIRE(cond, ...)                                                    \
  do {                                                                            \
    if (!(cond)) {                                                                \
      ::moe::set_error(__VA_ARGS__);                                              \
      return MOE_INVALID_CONFIG;                                                  \
    }                                                                             \
  } while (0)

constexpr unsigned FULL = 0xffffffffu;

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its predecessor runs; it
// must pdl_wait() before reading the predecessor's outputs.  Predecessors pdl_trigger() early
// so the dependent's launch and prologue overlap their tail.  Both are no-ops otherwise.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
// 64-bit warp min / max as two 32-bit redux.sync steps: the extreme high word, then the
// extreme low word among the lanes holding it (exactly the 64-bit extreme; 2 instructions in
// place of a 5-level shuffle tree -- these sit on the gate's and the replay's serial path)
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
  const uint32_t hi = static_cast<uint32_t>(v >> 32);
  const uint32_t mh = __reduce_min_sync(FULL, hi);
  const uint32_t ml = __reduce_min_sync(FULL, hi == mh ? static_cast<uint32_t>(v) : 0xFFFFFFFFu);
  return (static_cast<uint64_t>(mh) << 32) | ml;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const uint32_t hi = static_cast<uint32_t>(v >> 32);
  const uint32_t mh = __reduce_max_sync(FULL, hi);
  const uint32_t ml = __reduce_max_sync(FULL, hi == mh ? static_cast<uint32_t>(v) : 0u);
  return (static_cast<uint64_t>(mh) << 32) | ml;
}

// Order-preserving map of a finite float/double onto unsigned integers, with -0 == +0
// (numpy's comparison semantics, which lexsort relies on in toymoe.py:114).
__device__ __forceinline__ uint32_t ordered_bits(float f) {
  if (f == 0.0f) f = 0.0f;
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// inverse of ordered_bits(float) (-0 comes back as +0)
__device__ __forceinline__ float key_float(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ uint64_t ordered_bits(double f) {
  if (f == 0.0) f = 0.0;
  uint64_t u = static_cast<uint64_t>(__double_as_longlong(f));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

}  // namespace moe
