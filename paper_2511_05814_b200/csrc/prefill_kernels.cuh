// Device side of the batched prefill (moe_engine_prefill): per layer, for T independent
// tokens at once,
//   pf_combine_kernel  layer input x = h'_{l-1} + sum_j p_j y_j (selection order), bf16 copy
//                      for the mixing GEMM                                  (toymoe.py:142-145)
//   [tcgen05 GEMM]     h' = x + alpha * M x                                   (toymoe.py:140)
//   pf_gate_kernel     per token: RMS scale, route logits, softmax, top-k, reference guess
//                                                          (toymoe.py:99-115, 178-180)
//   pf_plan_kernel     the layer's cache policy replayed over the T steps in token order
//                      (kernels.py:89-145, the same warp step as decode), then the HBM
//                      buffer plan, the token -> expert grouping and the GEMM tile tables
//   pf_gather_kernel   bf16 rows of the normalised h' in expert-grouped order
//   [tcgen05 GEMMs]    SwiGLU up (fused silu * gate), down (scatter to (token, slot) rows)
// The device decides every expert / buffer / copy; the host reads the plan from a mapped
// mailbox and forwards the copies, as in decode.
#pragma once
#include "engine_kernels.cuh"
#include "tc_gemm.cuh"

namespace moe {

struct __align__(16) PrefillMail {
  long long seq;
  int32_t layer, n_loads, n_moves, n_res_groups;
  int32_t res_rows;                 // token rows of the experts already resident (list 0)
  int32_t pad[3];
  int32_t load_expert[kMaxE];       // copy order == GEMM list order 1 + i
  int32_t load_dst[kMaxE];          // >= 0: pool buffer of this layer; < 0: scratch slot -1-dst
  int32_t load_rows[kMaxE];         // token rows routed to that expert
  int32_t move_expert[kMaxE];       // after the layer's GEMMs: scratch[e] -> pool buffer
  int32_t move_buf[kMaxE];
  volatile long long ready;         // seq + 1 once the fields above are visible
  long long pad2;
};

__device__ __forceinline__ StepRecord* pf_rec(StepRecord* ring, long long tok, int max_tokens,
                                              int L, int l) {
  return ring + (tok % max_tokens) * L + l;
}

// x[t] = layer input; a[t] = bf16(x[t]).  Layer 0 copies the token input; otherwise the
// previous layer's h' plus the weighted expert outputs in selection order (the decode path's
// arithmetic), each expert output the sum of its split-K planes in split order.
__global__ void __launch_bounds__(256) pf_combine_kernel(const float* __restrict__ in,
                                                         const float* __restrict__ hm,
                                                         const float* __restrict__ y,
                                                         int splits, long long split_stride,
                                                         const StepRecord* ring, long long tok0,
                                                         int max_tokens, int L, int prev_layer,
                                                         int d, int K, float* __restrict__ x,
                                                         uint16_t* __restrict__ a) {
  const int t = blockIdx.y;
  const int i4 = blockIdx.x * blockDim.x + threadIdx.x;  // float4 index
  if (i4 * 4 >= d) return;
  float4 v;
  if (in) {
    v = reinterpret_cast<const float4*>(in + static_cast<size_t>(t) * d)[i4];
  } else {
    const StepRecord* rec = pf_rec(const_cast<StepRecord*>(ring), tok0 + t, max_tokens, L, prev_layer);
    v = reinterpret_cast<const float4*>(hm + static_cast<size_t>(t) * d)[i4];
    for (int j = 0; j < K; ++j) {
      const float* yj = y + (static_cast<size_t>(t) * K + j) * d;
      float4 s = reinterpret_cast<const float4*>(yj)[i4];
      for (int q = 1; q < splits; ++q) {
        const float4 u = reinterpret_cast<const float4*>(yj + q * split_stride)[i4];
        s.x = __fadd_rn(s.x, u.x);
        s.y = __fadd_rn(s.y, u.y);
        s.z = __fadd_rn(s.z, u.z);
        s.w = __fadd_rn(s.w, u.w);
      }
      const float pj = rec->prob[j];
      v.x = __fadd_rn(v.x, __fmul_rn(pj, s.x));
      v.y = __fadd_rn(v.y, __fmul_rn(pj, s.y));
      v.z = __fadd_rn(v.z, __fmul_rn(pj, s.z));
      v.w = __fadd_rn(v.w, __fmul_rn(pj, s.w));
    }
  }
  reinterpret_cast<float4*>(x + static_cast<size_t>(t) * d)[i4] = v;
  if (a) {
    uint2 o;
    o.x = tc::pack_bf16(v.x, v.y);
    o.y = tc::pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(a + static_cast<size_t>(t) * d)[i4] = o;
  }
}

struct PfGateParams {
  const float* x;       // [T][d] layer input (reference guess point)
  const float* hm;      // [T][d] h'
  const float* gate_w;  // [E][d] this layer
  const float* gate_b;  // [E]
  StepRecord* ring;
  long long tok0;
  int max_tokens, L, layer, T, d, E, K;
  int record_spec, renorm, rms_norm;
  float rms_eps;
  float* inv;           // [T] 1/rms(h') (1 without RMSNorm)
  int* err;
  const int32_t* forced;  // trace-driven routing: (T, L, K) ids, or nullptr
};

// One CTA per token: every thread owns a fixed slice of the row (all its loads in flight
// together), per-warp partial logits reduced in a fixed order; warp 0 then applies the
// gate of toymoe._gate_topk with the decode path's routing rules.
template <int EM>
__global__ void __launch_bounds__(256) pf_gate_kernel(PfGateParams p) {
  __shared__ float part[2 * EM + 2][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x;
  const bool do_guess = p.record_spec && p.layer >= 1;
  const float* hm = p.hm + static_cast<size_t>(t) * p.d;
  const float* x = p.x + static_cast<size_t>(t) * p.d;
  float az[EM], ag[EM];
#pragma unroll
  for (int e = 0; e < EM; ++e) az[e] = ag[e] = 0.f;
  float sm = 0.f, si = 0.f;
  for (int i = threadIdx.x; i < p.d / 4; i += blockDim.x) {
    const float4 h = reinterpret_cast<const float4*>(hm)[i];
    const float4 xi = do_guess ? reinterpret_cast<const float4*>(x)[i] : h;
    sm = fmaf(h.x, h.x, fmaf(h.y, h.y, fmaf(h.z, h.z, fmaf(h.w, h.w, sm))));
    si = fmaf(xi.x, xi.x, fmaf(xi.y, xi.y, fmaf(xi.z, xi.z, fmaf(xi.w, xi.w, si))));
#pragma unroll
    for (int e = 0; e < EM; ++e) {
      if (e >= p.E) break;
      const float4 w = reinterpret_cast<const float4*>(p.gate_w + static_cast<size_t>(e) * p.d)[i];
      az[e] = fmaf(w.x, h.x, fmaf(w.y, h.y, fmaf(w.z, h.z, fmaf(w.w, h.w, az[e]))));
      if (do_guess) ag[e] = fmaf(w.x, xi.x, fmaf(w.y, xi.y, fmaf(w.z, xi.z, fmaf(w.w, xi.w, ag[e]))));
    }
  }
  {
    const float a = warp_sum(sm), b = warp_sum(si);
    if (lane == 0) {
      part[2 * EM][warp] = a;
      part[2 * EM + 1][warp] = b;
    }
  }
#pragma unroll
  for (int e = 0; e < EM; ++e) {
    if (e >= p.E) break;
    const float a = warp_sum(az[e]);
    const float b = do_guess ? warp_sum(ag[e]) : 0.f;
    if (lane == 0) {
      part[e][warp] = a;
      part[EM + e][warp] = b;
    }
  }
  __syncthreads();
  if (warp != 0) return;
  const int nw = blockDim.x >> 5;
  float smt = 0.f, sit = 0.f;
  for (int w = 0; w < nw; ++w) {
    smt += part[2 * EM][w];
    sit += part[2 * EM + 1][w];
  }
  const float inv_mid = p.rms_norm ? rsqrtf(smt / p.d + p.rms_eps) : 1.f;
  const float inv_in = p.rms_norm ? rsqrtf(sit / p.d + p.rms_eps) : 1.f;
  const bool valid = lane < p.E;
  float zr = 0.f, zg = 0.f;
  if (valid) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < nw; ++w) {
      a += part[lane][w];
      b += part[EM + lane][w];
    }
    zr = a * inv_mid + p.gate_b[lane];
    zg = b * inv_in + p.gate_b[lane];
  }
  bool finite = __all_sync(FULL, !valid || isfinite(zr));
  if (do_guess) finite = finite && __all_sync(FULL, !valid || isfinite(zg));
  const float m = warp_max(valid ? zr : -INFINITY);
  const float ez = valid ? expf(zr - m) : 0.f;
  const float prob = ez / warp_sum(ez);
  int sel[kMaxK], acts[kMaxK], gs[kMaxK];
  bool routed_ok = true;
  if (p.forced)
    routed_ok = load_forced(p.forced + (static_cast<size_t>(t) * p.L + p.layer) * p.K, p.K, p.E, sel);
  else
    warp_topk(zr, valid && finite, p.K, sel);
  const float gap = p.forced ? NAN : topk_gap(zr, valid, sel, p.K);
  const float zs_r = warp_max(valid ? fabsf(zr) : 0.f);
  const float zs_g = do_guess ? warp_max(valid ? fabsf(zg) : 0.f) : 0.f;
  float psel[kMaxK], ssel = 0.f;
  for (int j = 0; j < p.K; ++j) {
    psel[j] = __shfl_sync(FULL, prob, sel[j] & 31);
    ssel += psel[j];
  }
  if (p.renorm)
    for (int j = 0; j < p.K; ++j) psel[j] = psel[j] / ssel;
  for (int j = 0; j < p.K; ++j) acts[j] = sel[j];
  sort_small(acts, p.K);
  float ggap = NAN;
  if (do_guess) {
    warp_topk(zg, valid && finite, p.K, gs);
    ggap = topk_gap(zg, valid, gs, p.K);
    sort_small(gs, p.K);
  }
  if (lane == 0) {
    StepRecord* rec = pf_rec(p.ring, p.tok0 + t, p.max_tokens, p.L, p.layer);
    for (int j = 0; j < p.K; ++j) {
      rec->sel[j] = sel[j];
      rec->prob[j] = psel[j];
      rec->acts[j] = acts[j];
      rec->guess[j] = do_guess ? gs[j] : -1;
      rec->early[j] = -1;
    }
    rec->rb = 0;
    rec->ev = 0;
    const uint32_t fl = (finite ? 0u : 1u) | (routed_ok ? 0u : 4u);
    rec->flags = fl;
    rec->gap = gap;
    rec->guess_gap = ggap;
    rec->zscale[0] = zs_r;
    rec->zscale[1] = zs_g;
    if (fl) atomicOr(p.err, static_cast<int>(fl));
    p.inv[t] = inv_mid;
  }
}

struct PfPlanParams {
  StepRecord* ring;
  long long tok0;
  int max_tokens, L, layer, T, E, K, C, NB, policy;
  int pool_nb;         // buffers allocated per layer (the pool's layer stride) >= NB in use
  double decay_factor;
  long long decay_period;
  LayerState* state;
  DeviceStats* stats;
  int* err;
  int d, f;
  long long rows_per_buf_d, rows_per_buf_f;  // expert block in rows of d / f bf16 elements
  int* row_map;        // [T*K] grouped position -> t*K + j
  int* pos_of;         // [T*K] t*K + j -> grouped position (-1: token failed its gate)
  tc::Group* grp_up;   // [E] in list order
  tc::Group* grp_dn;
  tc::Tile* tiles_up;  // [1 + E][max_up]
  tc::Tile* tiles_dn;  // [1 + E][max_dn]
  int* cnt_up;         // [1 + E]
  int* cnt_dn;
  int max_up, max_dn;
  long long seq;
  PrefillMail* mail;   // device view of the mapped mailbox
};

// Replays the T steps of this layer in token order with the decode path's warp_policy_step
// (warp 0, lanes = experts), so the records and the final state equal T decode steps; the
// records are staged in shared memory first (the replay is sequential in t, its inputs need
// not be).  Then the HBM buffer plan (lane 0), the token -> expert grouping (one warp per
// expert, ballot scans in token order) and the tile lists (all threads).
// Dynamic shared memory: pf_plan_smem(T, K) bytes.
__host__ __device__ inline size_t pf_plan_smem(int T, int K) {
  return static_cast<size_t>(T) * (2 * sizeof(uint32_t) + 1 + 2 * K);
}

template <int EM>
__device__ __noinline__ void pf_replay(const PfPlanParams& p, LayerState& S, uint32_t R0,
                                       uint32_t emask, uint8_t* s_flags, const uint8_t* s_acts,
                                       uint32_t* s_rb, uint32_t* s_ev, int* cnt, uint32_t& RT,
                                       uint32_t& needed) {
  const int T = p.T, K = p.K;
  {
      ScalarCacheState<EM> st;
      st.resident = R0;
#pragma unroll
      for (int e = 0; e < EM; ++e) {
        st.freq[e] = e < p.E ? S.freq[e] : 0.0;
        st.last_touch[e] = e < p.E ? S.last_touch[e] : -1;
      }
      long long step = S.step;
      unsigned long long hits = 0, done = 0;
      for (int t = 0; t < T; ++t) {
        if (s_flags[t]) {
          s_rb[t] = s_ev[t] = 0;
          continue;
        }
        const uint8_t* acts = s_acts + t * K;
        uint32_t amask = 0;
        for (int j = 0; j < K; ++j) amask |= 1u << acts[j];
        const uint32_t res_save = st.resident;
        uint32_t rb = 0, ev = 0;
        const bool ok = scalar_policy_step<EM>(st, p.E, p.C, p.policy, p.decay_factor,
                                                  p.decay_period, step, acts, K, rb, ev);
        s_rb[t] = rb & emask;
        s_ev[t] = ev & emask;
        if (!ok) {
          s_flags[t] |= 2u;
          atomicOr(p.err, 2);
          st.resident = res_save;
          continue;
        }
        ++step;
        ++done;
        for (int j = 0; j < K; ++j) hits += (rb >> acts[j]) & 1u;
        needed |= amask;
      }
      RT = st.resident & emask;
#pragma unroll
      for (int e = 0; e < EM; ++e)
        if (e < p.E) {
          S.freq[e] = st.freq[e];
          S.last_touch[e] = st.last_touch[e];
        }
      S.step = step;
      atomicAdd(&p.stats->hits, hits);
      atomicAdd(&p.stats->misses, done * K - hits);
    }
}

// pf_replay for a compile-time top-k: the next step's ids and flag are loaded while the current
// step is decided (a single thread's replay is a dependency chain; shared-memory loads off it).
template <int EM, int KK>
__device__ __noinline__ void pf_replay_k(const PfPlanParams& p, LayerState& S, uint32_t R0,
                                         uint32_t emask, uint8_t* s_flags, const uint8_t* s_acts,
                                         uint32_t* s_rb, uint32_t* s_ev, uint32_t& RT,
                                         uint32_t& needed) {
  const int T = p.T;
  ScalarCacheState<EM> st;
  st.resident = R0;
#pragma unroll
  for (int e = 0; e < EM; ++e) {
    st.freq[e] = e < p.E ? S.freq[e] : 0.0;
    st.last_touch[e] = e < p.E ? S.last_touch[e] : -1;
  }
  long long step = S.step;
  unsigned long long hits = 0, done = 0;
  uint32_t cur[KK], nxt[KK];
  uint32_t fcur = T > 0 ? s_flags[0] : 0, fnxt = 0;
#pragma unroll
  for (int j = 0; j < KK; ++j) cur[j] = T > 0 ? s_acts[j] : 0;
  for (int t = 0; t < T; ++t) {
    if (t + 1 < T) {
      fnxt = s_flags[t + 1];
#pragma unroll
      for (int j = 0; j < KK; ++j) nxt[j] = s_acts[(t + 1) * KK + j];
    }
    if (fcur) {
      s_rb[t] = s_ev[t] = 0;
    } else {
      const uint32_t res_save = st.resident;
      uint32_t rb = 0, ev = 0;
      const bool ok = scalar_policy_step_k<EM, KK>(st, p.E, p.C, p.policy, p.decay_factor,
                                                   p.decay_period, step, cur, rb, ev);
      s_rb[t] = rb & emask;
      s_ev[t] = ev & emask;
      if (!ok) {
        s_flags[t] |= 2u;
        atomicOr(p.err, 2);
        st.resident = res_save;
      } else {
        ++step;
        ++done;
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          hits += (rb >> cur[j]) & 1u;
          needed |= 1u << cur[j];
        }
      }
    }
    fcur = fnxt;
#pragma unroll
    for (int j = 0; j < KK; ++j) cur[j] = nxt[j];
  }
  RT = st.resident & emask;
#pragma unroll
  for (int e = 0; e < EM; ++e)
    if (e < p.E) {
      S.freq[e] = st.freq[e];
      S.last_touch[e] = st.last_touch[e];
    }
  S.step = step;
  atomicAdd(&p.stats->hits, hits);
  atomicAdd(&p.stats->misses, done * KK - hits);
}

__global__ void __launch_bounds__(256) pf_plan_kernel(PfPlanParams p) {
  __shared__ __align__(16) LayerState S;
  __shared__ __align__(16) PrefillMail M;
  __shared__ int cnt[kMaxE], off[kMaxE], order[kMaxE], buf_before[kMaxE];
  __shared__ int s_n_res, s_n_groups;
  __shared__ uint32_t s_needed;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int T = p.T, K = p.K;
  uint32_t* s_rb = reinterpret_cast<uint32_t*>(dsm);
  uint32_t* s_ev = s_rb + T;
  uint8_t* s_flags = reinterpret_cast<uint8_t*>(s_ev + T);
  uint8_t* s_acts = s_flags + T;
  uint8_t* s_sel = s_acts + static_cast<size_t>(T) * K;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  copy16(&S, p.state, sizeof(LayerState), tid, blockDim.x);
  if (tid < kMaxE) cnt[tid] = 0;
  for (int t = tid; t < T; t += blockDim.x) {
    const StepRecord* rec = pf_rec(p.ring, p.tok0 + t, p.max_tokens, p.L, p.layer);
    s_flags[t] = static_cast<uint8_t>(rec->flags);
    for (int j = 0; j < K; ++j) {
      s_acts[t * K + j] = static_cast<uint8_t>(rec->acts[j]);
      s_sel[t * K + j] = static_cast<uint8_t>(rec->sel[j]);
    }
  }
  __syncthreads();
  const uint32_t emask = p.E >= 32 ? 0xffffffffu : ((1u << p.E) - 1u);
  const uint32_t R0 = S.resident & emask;
  __shared__ uint32_t s_RT;
  // sequential replay by one thread, experts in registers (scalar_policy_step == the warp
  // step decode uses, without its shuffle latency)
  if (tid == 0) {
    uint32_t RT = 0, needed = 0;
    if (p.E <= 8 && K == 2)
      pf_replay_k<8, 2>(p, S, R0, emask, s_flags, s_acts, s_rb, s_ev, RT, needed);
    else if (p.E <= 8)
      pf_replay<8>(p, S, R0, emask, s_flags, s_acts, s_rb, s_ev, cnt, RT, needed);
    else
      pf_replay<kMaxE>(p, S, R0, emask, s_flags, s_acts, s_rb, s_ev, cnt, RT, needed);
    s_RT = RT;
    s_needed = needed;
  }
  __syncthreads();
  // token rows per expert (tokens whose gate and policy step succeeded), one warp per expert
  for (int e = warp; e < p.E; e += nwarps) {
    int n = 0;
    for (int t0 = 0; t0 < T; t0 += 32) {
      const int t = t0 + lane;
      bool hit = false;
      if (t < T && !s_flags[t])
        for (int j = 0; j < K; ++j) hit |= s_acts[t * K + j] == e;
      n += __popc(__ballot_sync(FULL, hit));
    }
    if (lane == 0) cnt[e] = n;
  }
  __syncthreads();
  if (warp == 0) {
    const bool valid = lane < p.E;
    const uint32_t RT = s_RT, needed = s_needed;
    if (valid) buf_before[lane] = S.buf_of[lane];
    __syncwarp();
    if (lane == 0) {
      S.resident = RT;
      // group (list) order: experts already resident first, then the loads in ascending id
      int ng = 0, rows = 0;
      for (int e = 0; e < p.E; ++e)
        if (((needed & R0) >> e) & 1u) order[ng++] = e;
      const int nres = ng;
      for (int e = 0; e < p.E; ++e)
        if (((needed & ~R0) >> e) & 1u) order[ng++] = e;
      for (int i = 0; i < ng; ++i) {
        off[order[i]] = rows;
        rows += cnt[order[i]];
      }
      s_n_res = nres;
      s_n_groups = ng;
      // HBM buffers: loads that stay resident go straight into a free buffer when one is
      // free now; the rest land in their scratch slot (moved after the GEMMs if they stay)
      int nl = 0, nm = 0;
      int pending[kMaxE], np = 0;
      for (int i = nres; i < ng; ++i) {
        const int e = order[i];
        int dst = -1 - e;
        if ((RT >> e) & 1u) {
          int pick = -1;
          for (int b = 0; b < p.NB && pick < 0; ++b)
            if (!S.buf_policy[b]) pick = b;
          if (pick >= 0) {
            S.buf_policy[pick] = 1;
            S.buf_expert[pick] = e;
            S.buf_of[e] = pick;
            dst = pick;
          } else {
            pending[np++] = e;
          }
        }
        M.load_expert[nl] = e;
        M.load_dst[nl] = dst;
        M.load_rows[nl] = cnt[e];
        ++nl;
      }
      for (int e = 0; e < p.E; ++e)
        if (((R0 & ~RT) >> e) & 1u) {
          const int b = S.buf_of[e];
          if (b >= 0) S.buf_policy[b] = 0;
          S.buf_of[e] = -1;
        }
      for (int i = 0; i < np; ++i) {
        const int e = pending[i];
        int pick = -1;
        for (int b = 0; b < p.NB && pick < 0; ++b)
          if (!S.buf_policy[b]) pick = b;
        S.buf_policy[pick] = 1;
        S.buf_expert[pick] = e;
        S.buf_of[e] = pick;
        M.move_expert[nm] = e;
        M.move_buf[nm] = pick;
        ++nm;
      }
      for (int b = 0; b < kMaxBuf; ++b) S.buf_stage_seq[b] = -1;
      int res_rows = 0;
      for (int i = 0; i < nres; ++i) res_rows += cnt[order[i]];
      M.seq = p.seq;
      M.layer = p.layer;
      M.n_loads = nl;
      M.n_moves = nm;
      M.n_res_groups = nres;
      M.res_rows = res_rows;
    }
  }
  __syncthreads();
  // records: resident_before / evicted masks (and policy failures)
  for (int t = tid; t < T; t += blockDim.x) {
    StepRecord* rec = pf_rec(p.ring, p.tok0 + t, p.max_tokens, p.L, p.layer);
    rec->rb = s_rb[t];
    rec->ev = s_ev[t];
    rec->flags = s_flags[t];
    if (s_flags[t])
      for (int j = 0; j < K; ++j) p.pos_of[t * K + j] = -1;
  }
  // token -> grouped position, in token order: warp w scans for experts w, w + nwarps, ...
  const uint32_t needed = s_needed;
  for (int e = warp; e < p.E; e += nwarps) {
    if (!((needed >> e) & 1u)) continue;
    int cur = off[e];
    for (int t0 = 0; t0 < T; t0 += 32) {
      const int t = t0 + lane;
      int j_hit = -1;
      if (t < T && !s_flags[t])
        for (int j = 0; j < K; ++j)
          if (s_sel[t * K + j] == e) j_hit = j;
      const uint32_t bal = __ballot_sync(FULL, j_hit >= 0);
      if (j_hit >= 0) {
        const int pos = cur + __popc(bal & ((1u << lane) - 1u));
        p.row_map[pos] = t * K + j_hit;
        p.pos_of[t * K + j_hit] = pos;
      }
      cur += __popc(bal);
    }
  }
  // groups and tile lists: list 0 = resident experts, list 1 + i = i-th load
  const int ng = s_n_groups, nres = s_n_res;
  if (tid < ng) {
    const int e = order[tid];
    int b_map = 0;
    long long buf_index;
    if (tid < nres) {
      buf_index = static_cast<long long>(p.layer) * p.pool_nb + buf_before[e];
    } else {
      const int dst = M.load_dst[tid - nres];
      if (dst >= 0) {
        buf_index = static_cast<long long>(p.layer) * p.pool_nb + dst;
      } else {
        b_map = 1;
        buf_index = e;
      }
    }
    tc::Group gu, gd;
    gu.a_row0 = gd.a_row0 = off[e];
    gu.m = gd.m = cnt[e];
    gu.b_map = gd.b_map = b_map;
    gu.b_row0 = static_cast<int>(buf_index * p.rows_per_buf_d);
    gu.b_row1 = gu.b_row0 + p.f;
    gd.b_row0 = static_cast<int>(buf_index * p.rows_per_buf_f + 2ll * p.d);
    gd.b_row1 = 0;
    p.grp_up[tid] = gu;
    p.grp_dn[tid] = gd;
  }
  const int nlists = 1 + (ng - nres);
  for (int list = 0; list < nlists; ++list) {
    const int g0 = list == 0 ? 0 : nres + list - 1;
    const int g1 = list == 0 ? nres : g0 + 1;
    int nu = 0, nd = 0;
    for (int gi = g0; gi < g1; ++gi) {
      const int m = cnt[order[gi]];
      const int mt = (m + tc::BM - 1) / tc::BM;
      const int ntu = (p.f / (tc::BN / 2)) * mt, ntd = (p.d / tc::BN) * mt;
      for (int i = tid; i < ntu; i += blockDim.x)
        p.tiles_up[list * p.max_up + nu + i] = tc::Tile{gi, (i % mt) * tc::BM, (i / mt) * (tc::BN / 2)};
      for (int i = tid; i < ntd; i += blockDim.x)
        p.tiles_dn[list * p.max_dn + nd + i] = tc::Tile{gi, (i % mt) * tc::BM, (i / mt) * tc::BN};
      nu += ntu;
      nd += ntd;
    }
    if (tid == 0) {
      p.cnt_up[list] = nu;
      p.cnt_dn[list] = nd;
    }
  }
  __syncthreads();
  if (warp == 0) {
    copy16(p.state, &S, sizeof(LayerState), lane, 32);
    PrefillMail* dst = p.mail;
    copy16(dst, &M, offsetof(PrefillMail, ready), lane, 32);
    __threadfence_system();
    __syncwarp();
    if (lane == 0) dst->ready = p.seq + 1;
  }
}

// an[pos] = bf16(h'[t] * inv[t]) for every routed (t, j); rows of tokens whose gate failed get
// zero expert outputs.  One warp per (t, j).
__global__ void __launch_bounds__(256) pf_gather_kernel(const float* __restrict__ hm,
                                                        const float* __restrict__ inv,
                                                        const int* __restrict__ pos_of, int TK,
                                                        int K, int d, uint16_t* __restrict__ an,
                                                        float* __restrict__ y, int splits,
                                                        long long split_stride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * (blockDim.x >> 5) + warp;
  if (q >= TK) return;
  const int t = q / K;
  const int pos = pos_of[q];
  if (pos < 0) {
    for (int sp = 0; sp < splits; ++sp) {
      float4* dst = reinterpret_cast<float4*>(y + sp * split_stride + static_cast<size_t>(q) * d);
      for (int i = lane; i < d / 4; i += 32) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return;
  }
  const float s = inv[t];
  const float4* src = reinterpret_cast<const float4*>(hm + static_cast<size_t>(t) * d);
  uint2* dst = reinterpret_cast<uint2*>(an + static_cast<size_t>(pos) * d);
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = src[i];
    uint2 o;
    o.x = tc::pack_bf16(v.x * s, v.y * s);
    o.y = tc::pack_bf16(v.z * s, v.w * s);
    dst[i] = o;
  }
}

}  // namespace moe
