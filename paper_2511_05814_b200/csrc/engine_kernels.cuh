// Device side of the offload decode engine: per-layer mix (K0), fused gate + top-k +
// cache policy + slot assignment (K1+K2), expert FFN GEMVs (K3) and the token finaliser.
#pragma once
#include "common.cuh"
#include "policy.cuh"

namespace moe {

constexpr int kMaxK = 8;      // top-k supported by the live engine
constexpr int kMaxE = 32;     // experts per layer supported by the live engine (one per lane)
constexpr int kMaxBuf = 64;   // HBM expert buffers per layer (policy slots + staging)
constexpr int kMailRing = 256;

// Per-layer cache state, device resident (policies.CacheState, policies.py:104-117, in the
// array form kernels.replay_policy keeps, kernels.py:70-75) plus the HBM buffer table.
struct LayerState {
  uint32_t resident;                 // bit e: expert e is policy-resident
  int32_t pad0;
  long long step;                    // tokens this layer has processed (CacheState.step)
  double freq[kMaxE];
  long long last_touch[kMaxE];
  int32_t buf_of[kMaxE];             // buffer holding resident expert e, -1 otherwise
  int32_t buf_expert[kMaxBuf];       // expert whose bytes occupy (or are landing in) buffer b
  int32_t buf_policy[kMaxBuf];       // 1: buffer holds a policy-resident expert
  long long buf_stage_seq[kMaxBuf];  // prefetch tag: staged for step `seq`, -1 none
};

// One (token, layer) step record, written by the gate kernel into the device ring.
struct StepRecord {
  int32_t sel[kMaxK];    // selected ids in selection order (prob desc, ties -> lower id)
  float prob[kMaxK];     // routing weight applied to each selected expert
  int32_t acts[kMaxK];   // selected ids ascending (ActivationTrace row, toymoe.py:182-184)
  int32_t guess[kMaxK];  // reference-definition guess, ascending (toymoe.py:178-180)
  uint32_t rb, ev;       // resident_before / evicted masks (kernels.py:98-99, 132-134)
  uint32_t flags;        // bit0 non-finite logits, bit1 policy failure
  uint32_t pad;
};

// Mailbox entry the gate kernel hands to the host transfer thread (mapped pinned memory).
// The device decides everything (which experts, which buffers); the host only forwards
// the copies to the copy engine.
struct MailRecord {
  long long seq;
  int32_t layer, n_demand, n_cancel, n_prefetch, need_ack, pad;
  int32_t demand_expert[kMaxK], demand_buf[kMaxK], demand_adopt[kMaxK];
  int32_t cancel_buf[kMaxK];
  int32_t prefetch_expert[kMaxK], prefetch_buf[kMaxK];
  volatile long long ready;  // seq + 1 once the fields above are visible
};

struct DeviceStats {
  unsigned long long hits, misses;
};

// Mapped pinned control block shared by the device and the host forwarder.
struct HostControl {
  volatile long long consumed;      // host -> device: mails fully processed (back-pressure)
  volatile unsigned int gate_done;  // device -> host: last gate seq + 1 (diagnostics)
  volatile unsigned int pad;
};

// ---------------------------------------------------------------------------------------
// Vector staging: x (n floats) is kept in shared memory as two float4 planes so that a lane
// reading the 8 activations matching one 16-byte weight vector hits consecutive banks.
__device__ __forceinline__ void stage_planes(const float* __restrict__ x, int n, float4* pa,
                                             float4* pb) {
  for (int i = threadIdx.x; i < n / 8; i += blockDim.x) {
    const float4* src = reinterpret_cast<const float4*>(x) + 2 * i;
    pa[i] = src[0];
    pb[i] = src[1];
  }
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ float dot8_bf16(uint4 w, float4 a, float4 b, float acc) {
  acc = fmaf(bf_lo(w.x), a.x, acc);
  acc = fmaf(bf_hi(w.x), a.y, acc);
  acc = fmaf(bf_lo(w.y), a.z, acc);
  acc = fmaf(bf_hi(w.y), a.w, acc);
  acc = fmaf(bf_lo(w.z), b.x, acc);
  acc = fmaf(bf_hi(w.z), b.y, acc);
  acc = fmaf(bf_lo(w.w), b.z, acc);
  acc = fmaf(bf_hi(w.w), b.w, acc);
  return acc;
}

// Per-lane partial dot of one bf16 row (n % 8 == 0) with the staged vector.
template <int UNROLL>
__device__ __forceinline__ float lane_dot_bf16(const uint16_t* __restrict__ row, int n,
                                               const float4* pa, const float4* pb) {
  const int lane = threadIdx.x & 31;
  const uint4* r = reinterpret_cast<const uint4*>(row);
  const int n8 = n >> 3;
  float acc = 0.f;
  int i = lane;
  for (; i + 32 * (UNROLL - 1) < n8; i += 32 * UNROLL) {
    uint4 w[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) w[u] = ld_stream(r + i + 32 * u);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc = dot8_bf16(w[u], pa[i + 32 * u], pb[i + 32 * u], acc);
  }
  for (; i < n8; i += 32) acc = dot8_bf16(ld_stream(r + i), pa[i], pb[i], acc);
  return acc;
}

// Per-lane partial dot of one f32 row (n % 8 == 0) with the staged vector.
__device__ __forceinline__ float lane_dot_f32(const float* __restrict__ row, int n,
                                              const float4* pa, const float4* pb) {
  const int lane = threadIdx.x & 31;
  const float4* r = reinterpret_cast<const float4*>(row);
  float acc = 0.f;
  for (int i = lane; i < (n >> 3); i += 32) {
    const float4 w0 = __ldg(r + 2 * i), w1 = __ldg(r + 2 * i + 1);
    const float4 a = pa[i], b = pb[i];
    acc = fmaf(w0.x, a.x, acc);
    acc = fmaf(w0.y, a.y, acc);
    acc = fmaf(w0.z, a.z, acc);
    acc = fmaf(w0.w, a.w, acc);
    acc = fmaf(w1.x, b.x, acc);
    acc = fmaf(w1.y, b.y, acc);
    acc = fmaf(w1.z, b.z, acc);
    acc = fmaf(w1.w, b.w, acc);
  }
  return acc;
}

template <bool kBF16>
__device__ __forceinline__ float lane_dot(const void* row, int n, const float4* pa,
                                          const float4* pb) {
  if constexpr (kBF16)
    return lane_dot_bf16<8>(static_cast<const uint16_t*>(row), n, pa, pb);
  else
    return lane_dot_f32(static_cast<const float*>(row), n, pa, pb);
}

// h = h_mid + sum_j prob[j] * y[j] in selection order (toymoe.py:142-145), element i.
__device__ __forceinline__ float combine_elem(const float* h_mid, const float* y,
                                              const StepRecord* rec, int K, int d, int i) {
  float v = h_mid[i];
  for (int j = 0; j < K; ++j) v = __fadd_rn(v, __fmul_rn(rec->prob[j], y[j * d + i]));
  return v;
}

// ---- K0: mixing GEMV, h' = h + alpha * (h @ M) (toymoe.py:140) ---------------------------
struct MixParams {
  const float* x;          // layer 0 input row (token input), else nullptr
  const float* prev_mid;   // previous layer's h' (layer > 0)
  const float* y;          // previous layer's expert outputs [K][d]
  const StepRecord* prev;  // previous layer's record (selection + probs)
  const void* M;           // [d_out][d_in] device layout (= reference M transposed)
  float alpha;
  int d, K;
  float* h_in;             // written by CTA 0: the layer input (for the speculation gate)
  float* h_mid;            // output h'
};

template <bool kBF16>
__global__ void __launch_bounds__(256) mix_kernel(MixParams p) {
  extern __shared__ float4 smem4[];
  float4* pa = smem4;
  float4* pb = smem4 + p.d / 8;
  float* hs = reinterpret_cast<float*>(smem4 + p.d / 4);
  // layer input: fresh token or the combined output of the previous layer
  for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
    const float v = p.x ? p.x[i] : combine_elem(p.prev_mid, p.y, p.prev, p.K, p.d, i);
    hs[i] = v;
    if (blockIdx.x == 0) p.h_in[i] = v;
  }
  __syncthreads();
  stage_planes(hs, p.d, pa, pb);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const size_t esz = kBF16 ? 2 : 4;
  for (int r = blockIdx.x * nwarps + warp; r < p.d; r += gridDim.x * nwarps) {
    const char* row = static_cast<const char*>(p.M) + static_cast<size_t>(r) * p.d * esz;
    const float s = warp_sum(lane_dot<kBF16>(row, p.d, pa, pb));
    if (lane == 0) p.h_mid[r] = __fadd_rn(hs[r], __fmul_rn(p.alpha, s));
  }
}

// ---- K1 + K2: gate, softmax, top-k, speculation, cache policy, buffer table, mailbox ----
struct GateParams {
  const float* h_mid;      // h' of this layer
  const float* h_in;       // layer input (reference guess point for this layer)
  const float* gate_w;     // [L][E][d]
  const float* gate_b;     // [L][E]
  int layer, L, E, K, d, C, NB, policy;
  double decay_factor;
  long long decay_period;
  int record_spec, prefetch, renorm;
  long long seq;           // token_abs * L + layer
  LayerState* states;      // [L]
  StepRecord* rec;         // this step's record
  MailRecord* mail;        // ring base (device view of mapped pinned memory)
  HostControl* ctl;        // device view of the mapped control block
  int* err;
  DeviceStats* stats;
};

// top-k over lanes (value z on lane e < E), selection order: z desc, ties -> lower id.
__device__ __forceinline__ void warp_topk(float z, bool valid, int K, int* out) {
  const int lane = threadIdx.x & 31;
  bool taken = false;
  for (int j = 0; j < K; ++j) {
    uint64_t key = 0;
    if (valid && !taken)
      key = (static_cast<uint64_t>(ordered_bits(z)) << 32) | (0xffffffffu - lane) | 0;
    // ordered_bits of any finite float is > 0, so key 0 means "no candidate"
    key = warp_max_u64(key);
    const int e = static_cast<int>(0xffffffffu - static_cast<uint32_t>(key & 0xffffffffu));
    out[j] = e;
    if (lane == e) taken = true;
  }
}

__device__ __forceinline__ void sort_small(int* v, int n) {
  for (int i = 1; i < n; ++i) {
    const int key = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > key) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = key;
  }
}

__global__ void __launch_bounds__(256) gate_cache_kernel(GateParams p) {
  __shared__ float z[3][kMaxE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const bool do_guess = p.record_spec && p.layer >= 1;
  const bool do_prefetch = p.prefetch == MOE_PREFETCH_EARLY && p.layer + 1 < p.L;
  // logits: job q = (which, expert); which 0 = route(h'), 1 = guess(h_in), 2 = early(h' , l+1)
  const int njobs = 3 * p.E;
  for (int q = warp; q < njobs; q += nwarps) {
    const int which = q / p.E, e = q % p.E;
    if ((which == 1 && !do_guess) || (which == 2 && !do_prefetch)) continue;
    const int gl = which == 2 ? p.layer + 1 : p.layer;
    const float* w = p.gate_w + (static_cast<size_t>(gl) * p.E + e) * p.d;
    const float* v = which == 1 ? p.h_in : p.h_mid;
    float acc = 0.f;
    for (int i = lane; i < p.d / 4; i += 32) {
      const float4 a = reinterpret_cast<const float4*>(w)[i];
      const float4 b = reinterpret_cast<const float4*>(v)[i];
      acc = fmaf(a.x, b.x, acc);
      acc = fmaf(a.y, b.y, acc);
      acc = fmaf(a.z, b.z, acc);
      acc = fmaf(a.w, b.w, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) z[which][e] = acc + p.gate_b[gl * p.E + e];
  }
  __syncthreads();
  if (warp != 0) return;

  const bool valid = lane < p.E;
  LayerState& S = p.states[p.layer];
  StepRecord* rec = p.rec;
  // -- route: finiteness (toymoe.py:109-110), softmax over all E (toymoe.py:93-96) --
  const float zr = valid ? z[0][lane] : 0.f;
  bool finite = __all_sync(FULL, !valid || isfinite(zr));
  float zg = 0.f;
  if (do_guess) {
    zg = valid ? z[1][lane] : 0.f;
    finite = finite && __all_sync(FULL, !valid || isfinite(zg));
  }
  int sel[kMaxK], acts[kMaxK], gs[kMaxK];
  uint32_t flags = finite ? 0u : 1u;
  const float m = warp_max(valid ? zr : -INFINITY);
  const float ez = valid ? expf(zr - m) : 0.f;
  const float sum = warp_sum(ez);
  const float prob = ez / sum;
  warp_topk(zr, valid && finite, p.K, sel);
  float psel[kMaxK];
  float ssel = 0.f;
  for (int j = 0; j < p.K; ++j) {
    psel[j] = __shfl_sync(FULL, prob, sel[j] & 31);
    ssel += psel[j];
  }
  if (p.renorm)
    for (int j = 0; j < p.K; ++j) psel[j] = psel[j] / ssel;
  for (int j = 0; j < p.K; ++j) acts[j] = sel[j];
  sort_small(acts, p.K);

  // -- cache policy step (kernels.py:89-145), state held one expert per lane --
  WarpCacheState<1> st;
  st.resident = valid ? ((S.resident >> lane) & 1u) : 0u;
  st.freq[0] = valid ? S.freq[lane] : 0.0;
  st.last_touch[0] = valid ? S.last_touch[lane] : -1;
  const long long t = S.step;
  uint32_t rbb = 0, evb = 0;
  bool ok = true;
  if (finite) {
    ok = warp_policy_step<1>(st, p.E, p.C, p.policy, p.decay_factor, p.decay_period, t,
                             [&](int j) { return static_cast<long long>(acts[j]); }, p.K,
                             [&](int) { return 0ll; }, rbb, evb);
  }
  if (!ok) flags |= 2u;
  const uint32_t emask = p.E >= 32 ? 0xffffffffu : ((1u << p.E) - 1u);
  const uint32_t rb = __ballot_sync(FULL, rbb & 1u) & emask;
  const uint32_t ev = __ballot_sync(FULL, evb & 1u) & emask;
  const uint32_t res_after = __ballot_sync(FULL, st.resident & 1u) & emask;
  if (valid && finite) {
    S.freq[lane] = st.freq[0];
    S.last_touch[lane] = st.last_touch[0];
  }
  // speculation guesses
  if (do_guess) {
    warp_topk(zg, valid && finite, p.K, gs);
    sort_small(gs, p.K);
  }
  int pf[kMaxK];
  if (do_prefetch) {
    const float ze = valid ? z[2][lane] : 0.f;
    const bool fe = __all_sync(FULL, !valid || isfinite(ze));
    warp_topk(ze, valid && fe, p.K, pf);
    sort_small(pf, p.K);
  }
  if (lane != 0) return;

  // -- record --
  for (int j = 0; j < p.K; ++j) {
    rec->sel[j] = sel[j];
    rec->prob[j] = psel[j];
    rec->acts[j] = acts[j];
    rec->guess[j] = do_guess ? gs[j] : -1;
  }
  rec->rb = rb;
  rec->ev = ev;
  rec->flags = flags;
  if (flags) atomicOr(p.err, static_cast<int>(flags));

  MailRecord* mr = p.mail + (p.seq % kMailRing);
  int nd = 0, nc = 0, np = 0;
  if (finite && ok) {
    S.resident = res_after;
    S.step = t + 1;
    int hits = 0;
    for (int j = 0; j < p.K; ++j) hits += (rb >> acts[j]) & 1u;
    atomicAdd(&p.stats->hits, static_cast<unsigned long long>(hits));
    atomicAdd(&p.stats->misses, static_cast<unsigned long long>(p.K - hits));
    // release buffers of evicted experts (their bytes stay until overwritten)
    for (int e = 0; e < p.E; ++e)
      if ((ev >> e) & 1u) {
        const int b = S.buf_of[e];
        if (b >= 0) S.buf_policy[b] = 0;
        S.buf_of[e] = -1;
      }
    // misses whose expert was prefetched for exactly this step adopt the staging buffer
    for (int j = 0; j < p.K; ++j) {
      const int e = acts[j];
      if ((rb >> e) & 1u) continue;
      for (int b = 0; b < p.NB; ++b)
        if (S.buf_stage_seq[b] == p.seq && S.buf_expert[b] == e && !S.buf_policy[b]) {
          S.buf_policy[b] = 1;
          S.buf_of[e] = b;
          S.buf_stage_seq[b] = -1;
          mr->demand_expert[nd] = e;
          mr->demand_buf[nd] = b;
          mr->demand_adopt[nd] = 1;
          ++nd;
          break;
        }
    }
    // the remaining staged buffers of this step were wrong guesses: cancel them
    for (int b = 0; b < p.NB; ++b)
      if (S.buf_stage_seq[b] == p.seq) {
        S.buf_stage_seq[b] = -1;
        mr->cancel_buf[nc++] = b;
      }
    // fresh demand misses take the lowest free buffer
    for (int j = 0; j < p.K; ++j) {
      const int e = acts[j];
      if (((rb >> e) & 1u) || S.buf_of[e] >= 0) continue;
      int pick = -1;
      for (int b = 0; b < p.NB && pick < 0; ++b)
        if (!S.buf_policy[b]) pick = b;
      S.buf_policy[pick] = 1;
      S.buf_expert[pick] = e;
      S.buf_of[e] = pick;
      mr->demand_expert[nd] = e;
      mr->demand_buf[nd] = pick;
      mr->demand_adopt[nd] = 0;
      ++nd;
    }
    // speculative prefetch of layer l+1's guesses that are not resident there
    if (do_prefetch) {
      LayerState& S1 = p.states[p.layer + 1];
      for (int j = 0; j < p.K; ++j) {
        const int g = pf[j];
        if (g < 0 || g >= p.E || S1.buf_of[g] >= 0) continue;
        int pick = -1;
        for (int b = 0; b < p.NB && pick < 0; ++b)
          if (!S1.buf_policy[b] && S1.buf_stage_seq[b] != p.seq + 1) pick = b;
        if (pick < 0) continue;
        S1.buf_stage_seq[pick] = p.seq + 1;
        S1.buf_expert[pick] = g;
        mr->prefetch_expert[np] = g;
        mr->prefetch_buf[np] = pick;
        ++np;
      }
    }
  }
  // ring back-pressure: if the host is far behind, make it acknowledge this step
  const long long consumed = p.ctl->consumed;
  const int need_ack = (p.seq - consumed) >= (kMailRing / 2) ? 1 : 0;
  mr->seq = p.seq;
  mr->layer = p.layer;
  mr->n_demand = nd;
  mr->n_cancel = nc;
  mr->n_prefetch = np;
  mr->need_ack = need_ack;
  __threadfence_system();
  mr->ready = p.seq + 1;
  p.ctl->gate_done = static_cast<unsigned int>(p.seq + 1);
}



// ---- K3: expert FFN over the selected slots ---------------------------------------------
struct FfnParams {
  const float* h_mid;        // x of this layer
  const StepRecord* rec;
  const LayerState* state;   // buf_of for this layer
  const char* pool;          // this layer's buffers: pool + b * expert_bytes
  long long expert_bytes;
  int d, f, K;
  int phase;                 // 0: experts that hit (resident before), 1: misses
  float* act;                // [K][f]
  float* y;                  // [K][d]
};

__device__ __forceinline__ bool ffn_phase_match(const FfnParams& p, int j, int* e_out) {
  const int e = p.rec->sel[j];
  *e_out = e;
  if (e < 0 || e >= kMaxE || p.rec->flags) return false;  // failed gate: nothing to run
  if (p.state->buf_of[e] < 0) return false;
  const bool hit = (p.rec->rb >> e) & 1u;
  return (p.phase == 0) == hit;
}

// SwiGLU up projection: act[j][r] = silu(w1[r] . x) * (w3[r] . x)
__global__ void __launch_bounds__(256) swiglu_up_kernel(FfnParams p) {
  const int j = blockIdx.y;
  int e;
  if (!ffn_phase_match(p, j, &e)) return;
  extern __shared__ float4 smem4[];
  float4* pa = smem4;
  float4* pb = smem4 + p.d / 8;
  stage_planes(p.h_mid, p.d, pa, pb);
  __syncthreads();
  const int b = p.state->buf_of[e];
  const uint16_t* w1 = reinterpret_cast<const uint16_t*>(p.pool + b * p.expert_bytes);
  const uint16_t* w3 = w1 + static_cast<size_t>(p.f) * p.d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int r = blockIdx.x * nwarps + warp; r < p.f; r += gridDim.x * nwarps) {
    const float a1 = warp_sum(lane_dot_bf16<8>(w1 + static_cast<size_t>(r) * p.d, p.d, pa, pb));
    const float a3 = warp_sum(lane_dot_bf16<8>(w3 + static_cast<size_t>(r) * p.d, p.d, pa, pb));
    if (lane == 0) p.act[j * p.f + r] = a1 / (1.f + expf(-a1)) * a3;
  }
}

// Toy up projection: act[j][r] = tanh(W1t[r] . x)   (toymoe.py:144)
__global__ void __launch_bounds__(256) toy_up_kernel(FfnParams p) {
  const int j = blockIdx.y;
  int e;
  if (!ffn_phase_match(p, j, &e)) return;
  extern __shared__ float4 smem4[];
  float4* pa = smem4;
  float4* pb = smem4 + p.d / 8;
  stage_planes(p.h_mid, p.d, pa, pb);
  __syncthreads();
  const int b = p.state->buf_of[e];
  const float* w1 = reinterpret_cast<const float*>(p.pool + b * p.expert_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int r = blockIdx.x * nwarps + warp; r < p.d; r += gridDim.x * nwarps) {
    const float s = warp_sum(lane_dot_f32(w1 + static_cast<size_t>(r) * p.d, p.d, pa, pb));
    if (lane == 0) p.act[j * p.f + r] = tanhf(s);
  }
}

// Down projection: y[j][c] = W[c] . act[j]; W = w2 (SwiGLU, [d][f]) or W2t (toy, [d][d]).
template <bool kBF16>
__global__ void __launch_bounds__(256) down_kernel(FfnParams p) {
  const int j = blockIdx.y;
  int e;
  if (!ffn_phase_match(p, j, &e)) return;
  extern __shared__ float4 smem4[];
  float4* pa = smem4;
  float4* pb = smem4 + p.f / 8;
  stage_planes(p.act + static_cast<size_t>(j) * p.f, p.f, pa, pb);
  __syncthreads();
  const int b = p.state->buf_of[e];
  const char* blk = p.pool + b * p.expert_bytes;
  const size_t esz = kBF16 ? 2 : 4;
  // SwiGLU block: [w1 f*d | w3 f*d | w2 d*f]; toy block: [W1t d*d | W2t d*d]
  const char* W = kBF16 ? blk + 2 * static_cast<size_t>(p.f) * p.d * esz
                        : blk + static_cast<size_t>(p.d) * p.d * esz;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int c = blockIdx.x * nwarps + warp; c < p.d; c += gridDim.x * nwarps) {
    const float s = warp_sum(lane_dot<kBF16>(W + static_cast<size_t>(c) * p.f * esz, p.f, pa, pb));
    if (lane == 0) p.y[j * p.d + c] = s;
  }
}

// Final layer: h_out = h' + sum_j p_j y_j
__global__ void finalize_kernel(const float* h_mid, const float* y, const StepRecord* rec, int K,
                                int d, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) out[i] = combine_elem(h_mid, y, rec, K, d, i);
}

__global__ void reset_states_kernel(LayerState* s, int L, int NB) {
  const int l = blockIdx.x;
  if (l >= L) return;
  LayerState& S = s[l];
  for (int e = threadIdx.x; e < kMaxE; e += blockDim.x) {
    S.freq[e] = 0.0;
    S.last_touch[e] = -1;
    S.buf_of[e] = -1;
  }
  for (int b = threadIdx.x; b < kMaxBuf; b += blockDim.x) {
    S.buf_expert[b] = -1;
    S.buf_policy[b] = 0;
    S.buf_stage_seq[b] = -1;
  }
  if (threadIdx.x == 0) {
    S.resident = 0;
    S.step = 0;
  }
  (void)NB;
}

}  // namespace moe
