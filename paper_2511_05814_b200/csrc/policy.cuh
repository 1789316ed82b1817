// Warp-level cache-policy step shared by the offline replay (K7), the per-step object API
// and the live engine's gate+cache kernel (K2).
//
// One warp owns one layer's cache. Expert e lives on lane e % 32, register slot e / 32
// (EPL = experts per lane).  Semantics follow kernels.replay_policy (kernels.py:60-147):
//   decay (lfu-aged, t > 0 and t % period == 0; kernels.py:92-94)
//   -> resident_before snapshot (:98-99)
//   -> misses counted per activation entry (:101-104)
//   -> need = n_res + n_miss - C evictions, each the argmin over resident & not-activated
//      with the lowest id winning ties (strict '<' scans in ascending e, :106-131):
//        LRU      key (last_touch, e)
//        LFU/aged key (freq, last_touch, e)
//        OPT      key (-next_use, e)
//   -> load: resident = 1, freq += 1.0, last_touch = t per activation entry (:136-142).
#pragma once
#include "common.cuh"

namespace moe {

constexpr long long kTouchBias = 1ll << 40;  // last_touch may be as low as -2^40
constexpr long long kNeverUsed = 1ll << 52;  // next_use upper bound for OPT keys

template <int EPL>
struct WarpCacheState {
  uint32_t resident;            // bit i: expert i*32+lane resident
  double freq[EPL];
  long long last_touch[EPL];
};

__device__ __forceinline__ uint64_t lru_key(long long last_touch, int e) {
  return (static_cast<uint64_t>(last_touch + kTouchBias) << 10) | static_cast<uint64_t>(e);
}

// One policy step. `act` points at K activation ids (identical for all lanes).
// `next_use(i)` returns the next-use step of the lane's expert i*32+lane (OPT only).
// Returns false if an eviction found no candidate (K > C: the reference's latent
// out-of-range write, kernels.py:132); the caller reports it.
template <int EPL, class Act, class NextUse>
__device__ __forceinline__ bool warp_policy_step(WarpCacheState<EPL>& st, int E, int C,
                                                 int policy, double decay_factor,
                                                 long long decay_period, long long t,
                                                 Act act, int K, NextUse next_use,
                                                 uint32_t& rb_bits, uint32_t& ev_bits) {
  const int lane = threadIdx.x & 31;
  if (policy == MOE_P_LFU_AGED && t > 0 && (t % decay_period) == 0) {
#pragma unroll
    for (int i = 0; i < EPL; ++i) st.freq[i] *= decay_factor;
  }
  // activation membership + multiplicity (malformed rows with repeats behave as in the
  // reference: each entry counts and increments separately)
  uint32_t in_act = 0;
  int my_miss = 0;
  for (int j = 0; j < K; ++j) {
    const int e = static_cast<int>(act(j));
    if ((e & 31) == lane) {
      const int i = e >> 5;
      in_act |= 1u << i;
      if (!((st.resident >> i) & 1u)) ++my_miss;
    }
  }
  rb_bits = st.resident;
  ev_bits = 0;
  const int n_miss = __reduce_add_sync(FULL, my_miss);
  const int n_res = __reduce_add_sync(FULL, __popc(st.resident));
  const int need = n_res + n_miss - C;
  bool ok = true;
  for (int r = 0; r < need; ++r) {
    uint64_t best = ~0ull;
    if (policy == MOE_P_LFU || policy == MOE_P_LFU_AGED) {
      // two-level argmin: freq first (non-negative doubles order as their bit patterns),
      // then (last_touch, e) among the lanes holding the minimum frequency.
      uint64_t fbest = ~0ull;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const bool cand = ((st.resident >> i) & 1u) && !((in_act >> i) & 1u);
        const uint64_t fb = static_cast<uint64_t>(__double_as_longlong(st.freq[i]));
        if (cand && fb < fbest) fbest = fb;
      }
      fbest = warp_min_u64(fbest);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const bool cand = ((st.resident >> i) & 1u) && !((in_act >> i) & 1u);
        const uint64_t fb = static_cast<uint64_t>(__double_as_longlong(st.freq[i]));
        if (cand && fb == fbest) {
          const uint64_t k = lru_key(st.last_touch[i], i * 32 + lane);
          best = k < best ? k : best;
        }
      }
    } else if (policy == MOE_P_OPT) {
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const bool cand = ((st.resident >> i) & 1u) && !((in_act >> i) & 1u);
        if (cand) {
          const long long nu = next_use(i);
          const uint64_t k = (static_cast<uint64_t>(kNeverUsed - nu) << 10) |
                             static_cast<uint64_t>(i * 32 + lane);
          best = k < best ? k : best;
        }
      }
    } else {  // LRU
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const bool cand = ((st.resident >> i) & 1u) && !((in_act >> i) & 1u);
        if (cand) {
          const uint64_t k = lru_key(st.last_touch[i], i * 32 + lane);
          best = k < best ? k : best;
        }
      }
    }
    best = warp_min_u64(best);
    if (best == ~0ull) {
      ok = false;
      break;
    }
    const int victim = static_cast<int>(best & 1023u);
    if ((victim & 31) == lane) {
      st.resident &= ~(1u << (victim >> 5));
      ev_bits |= 1u << (victim >> 5);
    }
  }
  for (int j = 0; j < K; ++j) {
    const int e = static_cast<int>(act(j));
    if ((e & 31) == lane) {
      const int i = e >> 5;
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        if (q == i) {
          st.freq[q] += 1.0;
          st.last_touch[q] = t;
        }
      }
      st.resident |= 1u << i;
    }
  }
  (void)E;
  return ok;
}

// Single-thread form of warp_policy_step for E <= EM experts held in registers (fully
// unrolled): the same decisions, bit for bit (same keys, same tie-breaks, same fp64 freq
// arithmetic), without the warp reductions -- for long sequential replays where one step's
// shuffle latency would dominate (the prefill replays T steps per layer).  LRU / LFU /
// LFU-aged (OPT needs the future and stays on the warp path).
template <int EM>
struct ScalarCacheState {
  uint32_t resident;
  double freq[EM];
  long long last_touch[EM];
};

template <int EM>
__device__ __forceinline__ bool scalar_policy_step(ScalarCacheState<EM>& st, int E, int C,
                                                   int policy, double decay_factor,
                                                   long long decay_period, long long t,
                                                   const uint8_t* act, int K, uint32_t& rb,
                                                   uint32_t& ev) {
  if (policy == MOE_P_LFU_AGED && t > 0 && (t % decay_period) == 0) {
#pragma unroll
    for (int e = 0; e < EM; ++e) st.freq[e] *= decay_factor;
  }
  uint32_t in_act = 0;
  int n_miss = 0;
  for (int j = 0; j < K; ++j) {
    const int e = act[j];
    in_act |= 1u << e;
    if (!((st.resident >> e) & 1u)) ++n_miss;
  }
  rb = st.resident;
  ev = 0;
  const int need = __popc(st.resident) + n_miss - C;
  bool ok = true;
  for (int r = 0; r < need; ++r) {
    const uint32_t cand = st.resident & ~in_act;
    if (!cand) {
      ok = false;
      break;
    }
    int best = -1;
    uint64_t bf = ~0ull, bl = ~0ull;
#pragma unroll
    for (int e = 0; e < EM; ++e) {
      if (e >= E || !((cand >> e) & 1u)) continue;
      const uint64_t lk = static_cast<uint64_t>(st.last_touch[e] + kTouchBias);
      const uint64_t fk = (policy == MOE_P_LFU || policy == MOE_P_LFU_AGED)
                              ? static_cast<uint64_t>(__double_as_longlong(st.freq[e]))
                              : 0ull;
      // strict '<' in ascending e: the lowest id wins ties (kernels.py:109-131)
      if (fk < bf || (fk == bf && lk < bl)) {
        bf = fk;
        bl = lk;
        best = e;
      }
    }
    st.resident &= ~(1u << best);
    ev |= 1u << best;
  }
  for (int j = 0; j < K; ++j) {
    const int e = act[j];
#pragma unroll
    for (int q = 0; q < EM; ++q)
      if (q == e) {
        st.freq[q] += 1.0;
        st.last_touch[q] = t;
      }
    st.resident |= 1u << e;
  }
  return ok;
}

// The same step with the top-k a compile-time constant and the activation ids in registers
// (the prefill replay software-pipelines the next step's ids behind the current step).
template <int EM, int KK>
__device__ __forceinline__ bool scalar_policy_step_k(ScalarCacheState<EM>& st, int E, int C,
                                                     int policy, double decay_factor,
                                                     long long decay_period, long long t,
                                                     const uint32_t (&act)[KK], uint32_t& rb,
                                                     uint32_t& ev) {
  if (policy == MOE_P_LFU_AGED && t > 0 && (t % decay_period) == 0) {
#pragma unroll
    for (int e = 0; e < EM; ++e) st.freq[e] *= decay_factor;
  }
  uint32_t in_act = 0;
  int n_miss = 0;
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    in_act |= 1u << act[j];
    n_miss += !((st.resident >> act[j]) & 1u);
  }
  rb = st.resident;
  ev = 0;
  const int need = __popc(st.resident) + n_miss - C;
  bool ok = true;
  for (int r = 0; r < need; ++r) {
    const uint32_t cand = st.resident & ~in_act;
    if (!cand) {
      ok = false;
      break;
    }
    int best = -1;
    uint64_t bf = ~0ull, bl = ~0ull;
#pragma unroll
    for (int e = 0; e < EM; ++e) {
      if (e >= E || !((cand >> e) & 1u)) continue;
      const uint64_t lk = static_cast<uint64_t>(st.last_touch[e] + kTouchBias);
      const uint64_t fk = (policy == MOE_P_LFU || policy == MOE_P_LFU_AGED)
                              ? static_cast<uint64_t>(__double_as_longlong(st.freq[e]))
                              : 0ull;
      if (fk < bf || (fk == bf && lk < bl)) {
        bf = fk;
        bl = lk;
        best = e;
      }
    }
    st.resident &= ~(1u << best);
    ev |= 1u << best;
  }
#pragma unroll
  for (int e = 0; e < EM; ++e)
    if ((in_act >> e) & 1u) {
      st.freq[e] += 1.0;
      st.last_touch[e] = t;
    }
  st.resident |= in_act;
  return ok;
}

}  // namespace moe
