// K7: offline whole-layer policy replay on the GPU (kernels.replay_policy, kernels.py:60-147)
// and the per-step object API (policies.policy_step, policies.py:140-228).
//
// One warp per layer replays its T steps in order (the recurrence is sequential in t);
// layers are independent (simulate.py:167-174) and run as separate warps.
#include "policy.cuh"

#include <mutex>

namespace moe {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
std::atomic<uint64_t>& launch_counter() { return g_launches; }

// OPT needs next_use[t][e]: first step > t activating e (T = never), kernels.py:79-88.
// Each lane fills the column of its own experts with a backward scan.
template <int EPL>
__device__ void fill_next_use(const int64_t* acts, long long T, int K, int E, int32_t* nu) {
  const int lane = threadIdx.x & 31;
  int32_t upcoming[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) upcoming[i] = static_cast<int32_t>(T);
  for (long long t = T - 1; t >= 0; --t) {
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = i * 32 + lane;
      if (e < E) nu[t * E + e] = upcoming[i];
    }
    const int64_t* row = acts + t * K;
    for (int j = 0; j < K; ++j) {
      const int e = static_cast<int>(row[j]);
      if ((e & 31) == lane) {
#pragma unroll
        for (int i = 0; i < EPL; ++i)
          if (i == (e >> 5)) upcoming[i] = static_cast<int32_t>(t);
      }
    }
  }
}

template <int EPL>
__global__ void __launch_bounds__(128) replay_kernel(const int64_t* __restrict__ acts, int L,
                                                     long long T, int K, int E, int C, int policy,
                                                     double df, long long dp,
                                                     uint8_t* __restrict__ rb_out,
                                                     uint8_t* __restrict__ ev_out,
                                                     int32_t* __restrict__ nu_scratch,
                                                     int* __restrict__ err) {
  const int layer = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (layer >= L) return;
  const int lane = threadIdx.x & 31;
  const int64_t* a = acts + static_cast<long long>(layer) * T * K;
  uint8_t* rb = rb_out + static_cast<long long>(layer) * T * E;
  uint8_t* ev = ev_out + static_cast<long long>(layer) * T * E;
  int32_t* nu = nu_scratch ? nu_scratch + static_cast<long long>(layer) * T * E : nullptr;
  if (policy == MOE_P_OPT) {
    fill_next_use<EPL>(a, T, K, E, nu);
    __syncwarp();
  }
  WarpCacheState<EPL> st;
  st.resident = 0;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    st.freq[i] = 0.0;
    st.last_touch[i] = -1;
  }
  bool ok = true;
  for (long long t = 0; t < T; ++t) {
    const int64_t* row = a + t * K;
    uint32_t rbb, evb;
    const bool step_ok = warp_policy_step<EPL>(
        st, E, C, policy, df, dp, t, [&](int j) { return row[j]; }, K,
        [&](int i) { return static_cast<long long>(nu[t * E + i * 32 + lane]); }, rbb, evb);
    ok = ok && step_ok;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = i * 32 + lane;
      if (e < E) {
        rb[t * E + e] = static_cast<uint8_t>((rbb >> i) & 1u);
        ev[t * E + e] = static_cast<uint8_t>((evb >> i) & 1u);
      }
    }
  }
  if (!ok && lane == 0) atomicExch(err, 1);
}

// Same replay with the activation rows staged 32 steps at a time (lane i loads row t0 + i in
// one coalesced read, each step broadcasts its row by shuffle): the step chain no longer waits
// on a global load every few steps.  K is a template constant (ids stay in registers).
template <int EPL, int KK>
__global__ void __launch_bounds__(128) replay_kernel_staged(const int64_t* __restrict__ acts, int L,
                                                            long long T, int E, int C, int policy,
                                                            double df, long long dp,
                                                            uint8_t* __restrict__ rb_out,
                                                            uint8_t* __restrict__ ev_out,
                                                            int32_t* __restrict__ nu_scratch,
                                                            int* __restrict__ err) {
  const int layer = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (layer >= L) return;
  const int lane = threadIdx.x & 31;
  const int64_t* a = acts + static_cast<long long>(layer) * T * KK;
  uint8_t* rb = rb_out + static_cast<long long>(layer) * T * E;
  uint8_t* ev = ev_out + static_cast<long long>(layer) * T * E;
  int32_t* nu = nu_scratch ? nu_scratch + static_cast<long long>(layer) * T * E : nullptr;
  if (policy == MOE_P_OPT) {
    fill_next_use<EPL>(a, T, KK, E, nu);
    __syncwarp();
  }
  WarpCacheState<EPL> st;
  st.resident = 0;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    st.freq[i] = 0.0;
    st.last_touch[i] = -1;
  }
  bool ok = true;
  int64_t mine[KK];
  auto load = [&](long long t0) {
#pragma unroll
    for (int j = 0; j < KK; ++j) mine[j] = t0 + lane < T ? a[(t0 + lane) * KK + j] : 0;
  };
  load(0);
  for (long long t0 = 0; t0 < T; t0 += 32) {
    int64_t cur[KK];
#pragma unroll
    for (int j = 0; j < KK; ++j) cur[j] = mine[j];
    if (t0 + 32 < T) load(t0 + 32);  // next chunk in flight while this one is replayed
    const int n = T - t0 < 32 ? static_cast<int>(T - t0) : 32;
    for (int u = 0; u < n; ++u) {
      const long long t = t0 + u;
      int64_t row[KK];
#pragma unroll
      for (int j = 0; j < KK; ++j) row[j] = __shfl_sync(FULL, cur[j], u);
      uint32_t rbb, evb;
      const bool step_ok = warp_policy_step<EPL>(
          st, E, C, policy, df, dp, t, [&](int j) { return row[j]; }, KK,
          [&](int i) { return static_cast<long long>(nu[t * E + i * 32 + lane]); }, rbb, evb);
      ok = ok && step_ok;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int e = i * 32 + lane;
        if (e < E) {
          rb[t * E + e] = static_cast<uint8_t>((rbb >> i) & 1u);
          ev[t * E + e] = static_cast<uint8_t>((evb >> i) & 1u);
        }
      }
    }
  }
  if (!ok && lane == 0) atomicExch(err, 1);
}

template <int EPL>
__global__ void policy_step_kernel(uint8_t* resident, int64_t* last_touch, double* freq,
                                   long long step, int E, int C, int policy, double df,
                                   long long dp, const int64_t* act, int n_act,
                                   const int64_t* fut_ids, const int64_t* fut_off,
                                   long long n_future, uint8_t* rb_out, uint8_t* ev_out,
                                   int* err) {
  const int lane = threadIdx.x & 31;
  WarpCacheState<EPL> st;
  st.resident = 0;
  long long nu[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const int e = i * 32 + lane;
    st.freq[i] = 0.0;
    st.last_touch[i] = -kTouchBias;
    nu[i] = kNeverUsed - 1;
    if (e < E) {
      if (resident[e]) st.resident |= 1u << i;
      st.freq[i] = freq[e];
      st.last_touch[i] = last_touch[e];
    }
  }
  if (policy == MOE_P_OPT) {
    // distance to the first future set containing e (policies.py:222-228); never -> inf
    for (long long s = n_future - 1; s >= 0; --s) {
      for (long long q = fut_off[s]; q < fut_off[s + 1]; ++q) {
        const int e = static_cast<int>(fut_ids[q]);
        if ((e & 31) == lane) {
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (i == (e >> 5)) nu[i] = step + 1 + s;
        }
      }
    }
  }
  uint32_t rbb, evb;
  const bool ok = warp_policy_step<EPL>(
      st, E, C, policy, df, dp, step, [&](int j) { return act[j]; }, n_act,
      [&](int i) {
        long long v = 0;
#pragma unroll
        for (int q = 0; q < EPL; ++q)
          if (q == i) v = nu[q];
        return v;
      },
      rbb, evb);
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const int e = i * 32 + lane;
    if (e < E) {
      resident[e] = static_cast<uint8_t>((st.resident >> i) & 1u);
      freq[e] = st.freq[i];
      last_touch[e] = st.last_touch[i];
      rb_out[e] = static_cast<uint8_t>((rbb >> i) & 1u);
      ev_out[e] = static_cast<uint8_t>((evb >> i) & 1u);
    }
  }
  if (!ok && lane == 0) atomicExch(err, 1);
}

// Error flag shared by the replay entry points (K > C never reaches the kernel: callers
// validate, as simulate.py:148-151 does; the flag guards direct C-ABI misuse).
static int* device_err_flag() {
  static int* p = nullptr;
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  if (!p) {
    if (cudaMalloc(&p, sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, sizeof(int));
  }
  return p;
}

static moe_status check_err_flag(cudaStream_t s) {
  int* flag = device_err_flag();
  int h = 0;
  MOE_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  MOE_CUDA(cudaStreamSynchronize(s));
  if (h) {
    MOE_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    set_error("eviction found no candidate: activation set larger than the cache capacity");
    return MOE_INVALID_CONFIG;
  }
  return MOE_OK;
}

#define MOE_EPL_DISPATCH(E, FN)              \
  if ((E) <= 32) { FN(1); }                  \
  else if ((E) <= 64) { FN(2); }             \
  else if ((E) <= 128) { FN(4); }            \
  else { FN(8); }

}  // namespace moe

using namespace moe;

extern "C" {

const char* moe_last_error(void) { return g_last_error.c_str(); }
int32_t moe_abi_version(void) { return MOE_ABI_VERSION; }
uint64_t moe_kernel_launches(void) { return g_launches.load(); }

moe_status moe_replay_policy_layers(const int64_t* acts_dev, int32_t L, int64_t T, int32_t K,
                                    int32_t E, int32_t C, int32_t policy, double decay_factor,
                                    int64_t decay_period, uint8_t* resident_before_dev,
                                    uint8_t* evicted_dev, void* stream) {
  MOE_REQUIRE(E >= 1 && E <= 256, "num_experts must be in [1, 256], got %d", E);
  MOE_REQUIRE(K >= 1 && K <= E, "top_k must be in [1, %d], got %d", E, K);
  MOE_REQUIRE(C >= K, "top_k=%d experts per step cannot fit in cache_size=%d", K, C);
  MOE_REQUIRE(policy >= MOE_P_LRU && policy <= MOE_P_OPT, "unknown policy code %d", policy);
  MOE_REQUIRE(policy != MOE_P_LFU_AGED || decay_period >= 1, "decay_period must be >= 1");
  MOE_REQUIRE(L >= 0 && T >= 0, "negative shape");
  MOE_REQUIRE(T < (1ll << 31), "T must be < 2^31");
  if (L == 0 || T == 0) return MOE_OK;
  cudaStream_t s = as_stream(stream);
  int* err = device_err_flag();
  MOE_REQUIRE(err != nullptr, "cannot allocate the device error flag");
  int32_t* nu = nullptr;
  if (policy == MOE_P_OPT)
    MOE_CUDA(cudaMallocAsync(&nu, sizeof(int32_t) * static_cast<size_t>(L) * T * E, s));
  const int threads = 128;
  const int blocks = (L * 32 + threads - 1) / threads;
#define STAGED(EPL_, KK_)                                                                        \
  replay_kernel_staged<EPL_, KK_><<<blocks, threads, 0, s>>>(acts_dev, L, T, E, C, policy,         \
                                                             decay_factor, decay_period,           \
                                                             resident_before_dev, evicted_dev, nu, err)
#define LAUNCH(EPL_)                                                                      \
  do {                                                                                    \
    if (K == 1) STAGED(EPL_, 1);                                                          \
    else if (K == 2) STAGED(EPL_, 2);                                                     \
    else if (K == 4) STAGED(EPL_, 4);                                                     \
    else                                                                                  \
      replay_kernel<EPL_><<<blocks, threads, 0, s>>>(acts_dev, L, T, K, E, C, policy,     \
                                                     decay_factor, decay_period,          \
                                                     resident_before_dev, evicted_dev, nu, err); \
  } while (0)
  MOE_EPL_DISPATCH(E, LAUNCH);
#undef LAUNCH
#undef STAGED
  MOE_LAUNCHED();
  if (nu) MOE_CUDA(cudaFreeAsync(nu, s));
  return check_err_flag(s);
}

moe_status moe_replay_policy(const int64_t* acts_dev, int64_t T, int32_t K, int32_t E,
                             int32_t C, int32_t policy, double decay_factor,
                             int64_t decay_period, uint8_t* resident_before_dev,
                             uint8_t* evicted_dev, void* stream) {
  return moe_replay_policy_layers(acts_dev, 1, T, K, E, C, policy, decay_factor, decay_period,
                                  resident_before_dev, evicted_dev, stream);
}

moe_status moe_policy_step(uint8_t* resident_dev, int64_t* last_touch_dev, double* freq_dev,
                           int64_t step, int32_t E, int32_t C, int32_t policy,
                           double decay_factor, int64_t decay_period, const int64_t* act_dev,
                           int32_t n_act, const int64_t* future_ids_dev,
                           const int64_t* future_offsets_dev, int64_t n_future,
                           uint8_t* resident_before_dev, uint8_t* evicted_dev, void* stream) {
  MOE_REQUIRE(E >= 1 && E <= 256, "num_experts must be in [1, 256], got %d", E);
  MOE_REQUIRE(C >= 1, "cache capacity must be >= 1, got %d", C);
  MOE_REQUIRE(n_act <= C, "activated set of size %d cannot fit in capacity %d", n_act, C);
  MOE_REQUIRE(policy >= MOE_P_LRU && policy <= MOE_P_OPT, "unknown policy code %d", policy);
  MOE_REQUIRE(policy != MOE_P_OPT || future_offsets_dev != nullptr,
              "opt policy requires the remaining activation stream");
  MOE_REQUIRE(policy != MOE_P_LFU_AGED || decay_period >= 1, "decay_period must be >= 1");
  cudaStream_t s = as_stream(stream);
  int* err = device_err_flag();
  MOE_REQUIRE(err != nullptr, "cannot allocate the device error flag");
#define LAUNCH(EPL_)                                                                      \
  policy_step_kernel<EPL_><<<1, 32, 0, s>>>(resident_dev, last_touch_dev, freq_dev, step, E, \
                                            C, policy, decay_factor, decay_period, act_dev,  \
                                            n_act, future_ids_dev, future_offsets_dev,       \
                                            n_future, resident_before_dev, evicted_dev, err)
  MOE_EPL_DISPATCH(E, LAUNCH);
#undef LAUNCH
  MOE_LAUNCHED();
  return check_err_flag(s);
}

}  // extern "C"
