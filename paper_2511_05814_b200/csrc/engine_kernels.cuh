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
struct __align__(16) LayerState {
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
  float gap;             // route logit of the K-th selection minus the best unselected one
                         // (near-tie margin; +inf when K == E, NaN under forced routing)
  int32_t early[kMaxK];  // early guess for layer l+1 (gate_{l+1} on h'_l, ascending) that
                         // drove this step's speculative prefetch; -1 when prefetch is off
  float guess_gap;       // the same margin for the reference-definition guess (NaN: none)
  float zscale[2];       // max |logit| of the route / guess (relative near-tie tests)
  uint32_t pad2;
};
static_assert(sizeof(StepRecord) % 16 == 0, "records are copied with 16-byte stores");

// Mailbox entry the gate kernel hands to the host transfer thread (mapped pinned memory).
// The device decides everything (which experts, which buffers); the host only forwards
// the copies to the copy engine.
struct __align__(16) MailRecord {
  long long seq;
  int32_t layer, n_demand, n_cancel, n_prefetch, need_ack, pad;
  int32_t demand_expert[kMaxK], demand_buf[kMaxK], demand_adopt[kMaxK];
  int32_t cancel_buf[kMaxK];
  int32_t prefetch_expert[kMaxK], prefetch_buf[kMaxK];
  volatile long long ready;  // seq + 1 once the fields above are visible
  long long pad2;
};
static_assert(sizeof(MailRecord) % 16 == 0 && offsetof(MailRecord, ready) % 16 == 0,
              "mail records are copied with 16-byte stores");
static_assert(sizeof(LayerState) % 16 == 0, "layer state is copied with 16-byte stores");

struct DeviceStats {
  unsigned long long hits, misses;
  unsigned long long fetched_bytes;  // SM transfer mode: bytes read from the host store
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

// Same, with an explicit participating thread count (warp-specialised kernels).
__device__ __forceinline__ void stage_planes_n(const float* __restrict__ x, int n, float4* pa,
                                               float4* pb, int nthreads) {
#pragma unroll 4
  for (int i = threadIdx.x; i < n / 8; i += nthreads) {
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

// Vectorised combine of 4 consecutive elements (float4 index i4): same arithmetic order.
__device__ __forceinline__ float4 combine4(const float* h_mid, const float* y,
                                           const StepRecord* rec, int K, int d, int i4) {
  float4 v = reinterpret_cast<const float4*>(h_mid)[i4];
  for (int j = 0; j < K; ++j) {
    const float p = rec->prob[j];
    const float4 yj = reinterpret_cast<const float4*>(y + static_cast<size_t>(j) * d)[i4];
    v.x = __fadd_rn(v.x, __fmul_rn(p, yj.x));
    v.y = __fadd_rn(v.y, __fmul_rn(p, yj.y));
    v.z = __fadd_rn(v.z, __fmul_rn(p, yj.z));
    v.w = __fadd_rn(v.w, __fmul_rn(p, yj.w));
  }
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
  pdl_trigger();  // the gate may launch and stage its cache state meanwhile
  pdl_wait();     // (SM-transfer graphs launch this programmatically after the down pass)
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
constexpr int kMaxParts = 152;   // mixing-GEMV CTAs whose gate partials the gate sums (>= 148)
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
  int rms_norm;            // 1: RMSNorm (no learned scale) before gate and experts
  float rms_eps;
  float* h_norm;           // out: expert input (h' / rms(h') when rms_norm)
  unsigned long long* phase_ns;  // optional diagnostics: accumulated ns per kernel phase [8]
  // fused path (bf16 engine): the mixing GEMV's CTAs already reduced their rows into
  // part[c][job] (jobs: 3E logits + sum h'^2 + sum h_in^2); the gate sums them in CTA order
  const float* part;
  int nparts;
  float* norm_scale;       // out: 1/rms(h') (or 1) for the up projection's input staging
  const int32_t* forced;   // trace-driven routing: this step's K ids, or nullptr (gate top-k)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

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

// Near-tie margin of a top-k selection: z of the K-th selected lane minus the largest z
// among the unselected valid lanes (toymoe.py:114's order; +inf when every lane is taken).
__device__ __forceinline__ float topk_gap(float z, bool valid, const int* sel, int K) {
  const int lane = threadIdx.x & 31;
  bool taken = false;
  for (int j = 0; j < K; ++j) taken = taken || sel[j] == lane;
  const float zk = __shfl_sync(FULL, z, sel[K - 1] & 31);
  const float next = warp_max(valid && !taken ? z : -INFINITY);
  return zk - next;
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

// Register forms of warp_topk / topk_gap / load_forced: `out` / `sel` are indexed by unrolled
// constants only, so the K-long id lists stay in registers.
__device__ __forceinline__ void warp_topk_k(float z, bool valid, int K, int (&out)[kMaxK]) {
  const int lane = threadIdx.x & 31;
  bool taken = false;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) {
    if (j >= K) break;
    uint64_t key = 0;
    if (valid && !taken) key = (static_cast<uint64_t>(ordered_bits(z)) << 32) | (0xffffffffu - lane);
    key = warp_max_u64(key);   // key 0: no candidate left (-1)
    const int e = static_cast<int>(0xffffffffu - static_cast<uint32_t>(key & 0xffffffffu));
    out[j] = e;
    if (lane == e) taken = true;
  }
}
__device__ __forceinline__ float topk_gap_k(float z, bool valid, const int (&sel)[kMaxK], int K) {
  const int lane = threadIdx.x & 31;
  bool taken = false;
  int last = 0;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j)
    if (j < K) {
      taken = taken || sel[j] == lane;
      last = sel[j] & 31;
    }
  const float zk = __shfl_sync(FULL, z, last);
  const float next = key_float(__reduce_max_sync(FULL, valid && !taken ? ordered_bits(z)
                                                                         : ordered_bits(-INFINITY)));
  return zk - next;
}
__device__ __forceinline__ bool load_forced_k(const int32_t* forced, int K, int E, int (&sel)[kMaxK]) {
  uint32_t seen = 0;
  bool ok = true;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j)
    if (j < K) {
      const int e = forced[j];
      const bool in = e >= 0 && e < E && e < 32;
      ok = ok && in && !((seen >> (in ? e : 0)) & 1u);
      if (in) seen |= 1u << e;
      sel[j] = in ? e : 0;
    }
  return ok;
}
// ascending sort of the first n (<= kMaxK) entries, fully unrolled (registers, no stack)
__device__ __forceinline__ void sort_k(int (&v)[kMaxK], int n) {
#pragma unroll
  for (int i = 0; i < kMaxK - 1; ++i)
#pragma unroll
    for (int j = 0; j < kMaxK - 1 - i; ++j)
      if (j + 1 < n && v[j] > v[j + 1]) {
        const int x = v[j];
        v[j] = v[j + 1];
        v[j + 1] = x;
      }
}

// The same from global to shared memory without a register round trip (cp.async, 16 bytes
// per copy); the caller cp_async_wait_all()s before the barrier that publishes it.
__device__ __forceinline__ void copy16_async(void* dst, const void* src, int n, int tid, int nthreads) {
  const char* s = static_cast<const char*>(src);
  for (int i = tid; i < n / 16; i += nthreads)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(static_cast<char*>(dst) + 16 * i))),
                 "l"(s + 16 * i)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Copy `n` bytes (multiple of 16) with the calling threads (tid in [0, nthreads)).
__device__ __forceinline__ void copy16(void* dst, const void* src, int n, int tid, int nthreads) {
  int4* d = static_cast<int4*>(dst);
  const int4* s = static_cast<const int4*>(src);
  for (int i = tid; i < n / 16; i += nthreads) d[i] = s[i];
}

// Trace-driven routing: the step's K expert ids come from a caller-supplied activation trace
// (ActivationTrace row, ascending) instead of the gate's top-k; the gate's softmax still
// weights them.  Returns false for ids out of range or repeated (the step is then flagged).
__device__ __forceinline__ bool load_forced(const int32_t* forced, int K, int E, int* sel) {
  uint32_t seen = 0;
  bool ok = true;
  for (int j = 0; j < K; ++j) {
    const int e = forced[j];
    const bool in = e >= 0 && e < E && e < 32;
    ok = ok && in && !((seen >> (in ? e : 0)) & 1u);
    if (in) seen |= 1u << e;
    sel[j] = in ? e : 0;
  }
  return ok;
}

constexpr int kGateThreads = 512;  // d=4096: two float4 columns per thread, loads all in flight

// Working set of the gate / cache step in shared memory.
struct GateSmem {
  float z[3][kMaxE];
  float red[2][kGateThreads / 32];
  __align__(16) LayerState sS;    // working copies of this / next layer's state
  __align__(16) LayerState sS1;
  __align__(16) MailRecord sM;
};

// The gate + cache step run by `nthreads` threads (tid in [0, nthreads), a multiple of 32):
// as its own single-CTA kernel (gate_cache_kernel) or by the last CTA of the fused mixing
// GEMV (stream_gemv_kernel<kModeMix>, fuse_gate).  sync() is a barrier over those threads.
template <class Sync>
__device__ __forceinline__ void gate_cache_body(const GateParams& p, GateSmem& gsm, int tid,
                                                int nthreads, Sync sync, bool wait_pdl) {
  float (&z)[3][kMaxE] = gsm.z;
  float (&red)[2][kGateThreads / 32] = gsm.red;
  LayerState& sS = gsm.sS;
  LayerState& sS1 = gsm.sS1;
  MailRecord& sM = gsm.sM;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthreads >> 5;
  const bool do_guess = p.record_spec && p.layer >= 1;
  const bool do_prefetch = p.prefetch == MOE_PREFETCH_EARLY && p.layer + 1 < p.L;
  const unsigned long long t0 = p.phase_ns ? gtimer() : 0;
  // stage the cache state in shared memory asynchronously (cp.async: its latency overlaps the
  // partial sums / logits below; waited for before the barrier that ends them)
  copy16_async(&sS, &p.states[p.layer], sizeof(LayerState), tid, nthreads);
  if (do_prefetch) copy16_async(&sS1, &p.states[p.layer + 1], sizeof(LayerState), tid, nthreads);
  // the host's acknowledgement counter lives in mapped host memory: a PCIe round trip, so
  // thread 0 (lane 0 of warp 0, which writes the mail) issues the load now and uses it last
  const long long consumed0 = (tid == 0 && p.mail) ? p.ctl->consumed : 0;
  // launched programmatically after the mixing kernel: its outputs are read from here on
  if (wait_pdl) pdl_wait();
  // RMSNorm scales of h' (route, early guess, experts) and of h_in (reference guess)
  float inv_mid = 1.f, inv_in = 1.f;
  const int njob = 3 * p.E + 2;
  if (p.part) {
    // fused: sum the per-CTA partials, one warp per job, lanes over CTAs, then a fixed
    // shuffle tree (the same order every call: deterministic)
    // Eight threads per job, each summing every 8th CTA's partial in CTA order with its loads
    // all in flight (one L2 round trip instead of one per job), then a fixed xor tree over
    // the eight: the same order every call (deterministic).
    for (int q0 = 0; q0 < njob; q0 += nthreads / 8) {
      const int q = q0 + tid / 8, sub = tid & 7;
      float acc = 0.f;
      if (q < njob) {
        float v[kMaxParts / 8];
#pragma unroll
        for (int i = 0; i < kMaxParts / 8; ++i) {
          const int c = sub + 8 * i;
          v[i] = c < p.nparts ? p.part[c * njob + q] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < kMaxParts / 8; ++i) acc += v[i];
      }
      acc += __shfl_xor_sync(FULL, acc, 4);
      acc += __shfl_xor_sync(FULL, acc, 2);
      acc += __shfl_xor_sync(FULL, acc, 1);
      if (q < njob && sub == 0) {
        if (q < 3 * p.E) z[q / p.E][q % p.E] = acc;
        else red[q - 3 * p.E][0] = acc;
      }
    }
    sync();
    if (p.rms_norm) {
      inv_mid = rsqrtf(red[0][0] / p.d + p.rms_eps);
      inv_in = rsqrtf(red[1][0] / p.d + p.rms_eps);
    }
    if (tid < 3 * p.E) {
      const int which = tid / p.E, e = tid % p.E;
      const int gl = which == 2 ? p.layer + 1 : p.layer;
      if ((which == 1 && do_guess) || (which == 2 && do_prefetch) || which == 0)
        z[which][e] = z[which][e] * (which == 1 ? inv_in : inv_mid) + p.gate_b[gl * p.E + e];
    }
    if (tid == 0 && p.norm_scale) *p.norm_scale = inv_mid;
  } else {
    if (p.rms_norm) {
      float sm = 0.f, si = 0.f;
      for (int i = tid; i < p.d; i += nthreads) {
        const float a = p.h_mid[i];
        sm = fmaf(a, a, sm);
        if (do_guess) {
          const float b = p.h_in[i];
          si = fmaf(b, b, si);
        }
      }
      sm = warp_sum(sm);
      si = warp_sum(si);
      if (lane == 0) {
        red[0][warp] = sm;
        red[1][warp] = si;
      }
      sync();
      float tm = 0.f, ti = 0.f;
      for (int w = 0; w < nwarps; ++w) {
        tm += red[0][w];
        ti += red[1][w];
      }
      inv_mid = rsqrtf(tm / p.d + p.rms_eps);
      inv_in = rsqrtf(ti / p.d + p.rms_eps);
      for (int i = tid; i < p.d; i += nthreads) p.h_norm[i] = p.h_mid[i] * inv_mid;
    }
    if (tid == 0 && p.norm_scale) *p.norm_scale = 1.f;
  }
  const unsigned long long t1 = p.phase_ns ? gtimer() : 0;
  if (!p.part) {
  // logits: job q = (which, expert); which 0 = route(h'), 1 = guess(h_in), 2 = early(h', l+1).
  // One warp per job (16 warps, 3E jobs): coalesced row loads, one shuffle reduction per job
  // -- the latency of a handful of dependent steps instead of 3E sequential reductions.
  const int nv = p.d / 4;  // float4 columns
  for (int q = warp; q < 3 * p.E; q += nwarps) {
    const int which = q / p.E, e = q % p.E;
    if ((which == 1 && !do_guess) || (which == 2 && !do_prefetch)) continue;
    const int gl = which == 2 ? p.layer + 1 : p.layer;
    const float4* w = reinterpret_cast<const float4*>(p.gate_w + (static_cast<size_t>(gl) * p.E + e) * p.d);
    const float4* v = reinterpret_cast<const float4*>(which == 1 ? p.h_in : p.h_mid);
    float acc = 0.f;
    for (int i = lane; i < nv; i += 32) {
      const float4 a4 = w[i], b4 = v[i];
      acc = fmaf(a4.x, b4.x, acc);
      acc = fmaf(a4.y, b4.y, acc);
      acc = fmaf(a4.z, b4.z, acc);
      acc = fmaf(a4.w, b4.w, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) z[which][e] = acc * (which == 1 ? inv_in : inv_mid) + p.gate_b[gl * p.E + e];
  }
  }
  cp_async_wait_all();
  sync();
  if (warp != 0) return;
  const unsigned long long t2 = p.phase_ns ? gtimer() : 0;

  const bool valid = lane < p.E;
  LayerState& S = sS;
  StepRecord* rec = p.rec;
  const long long t = S.step;
  const uint32_t emask = p.E >= 32 ? 0xffffffffu : ((1u << p.E) - 1u);
  int sel[kMaxK], acts[kMaxK], gs[kMaxK], pf[kMaxK];
  float psel[kMaxK];
  uint32_t flags = 0u, rb = 0u, ev = 0u, res_after = S.resident & emask;
  float gap = NAN, ggap = NAN, zs_r = 0.f, zs_g = 0.f;
  bool go = false, ok = true;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) sel[j] = acts[j] = gs[j] = pf[j] = -1, psel[j] = 0.f;
  // One expert per lane, everything in registers (the K-long id lists are indexed by unrolled
  // constants only), extremes by redux.sync on order-preserving keys: the decision is a short
  // chain of warp reductions -- this tail runs on one SM while the others wait for it.
  // -- route: finiteness (toymoe.py:109-110), softmax over all E (toymoe.py:93-96) --
  const float zr = valid ? z[0][lane] : 0.f;
  const float zg = valid && do_guess ? z[1][lane] : 0.f;
  const float ze = valid && do_prefetch ? z[2][lane] : 0.f;
  bool finite = __all_sync(FULL, !valid || isfinite(zr));
  if (do_guess) finite = finite && __all_sync(FULL, !valid || isfinite(zg));
  flags = finite ? 0u : 1u;
  // max over the valid lanes (-inf elsewhere): the ordered-key maximum is fmaxf's result for
  // finite values (non-finite rows are flagged and their numbers unused)
  const float m = key_float(__reduce_max_sync(FULL, valid ? ordered_bits(zr) : ordered_bits(-INFINITY)));
  const float ez = valid ? expf(zr - m) : 0.f;
  const float sum = warp_sum(ez);   // butterfly order, as before
  const float prob = ez / sum;
  bool routed_ok = true;
  if (p.forced) {
    routed_ok = load_forced_k(p.forced, p.K, p.E, sel);
    if (!routed_ok) flags |= 4u;
  } else {
    warp_topk_k(zr, valid && finite, p.K, sel);
    gap = topk_gap_k(zr, valid, sel, p.K);
  }
  zs_r = __uint_as_float(__reduce_max_sync(FULL, valid ? __float_as_uint(fabsf(zr)) : 0u));
  zs_g = do_guess ? __uint_as_float(__reduce_max_sync(FULL, valid ? __float_as_uint(fabsf(zg)) : 0u)) : 0.f;
  go = finite && routed_ok;
  float ssel = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j)
    if (j < p.K) {
      psel[j] = __shfl_sync(FULL, prob, sel[j] & 31);
      ssel += psel[j];
    }
  if (p.renorm) {
#pragma unroll
    for (int j = 0; j < kMaxK; ++j)
      if (j < p.K) psel[j] = psel[j] / ssel;
  }
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) acts[j] = sel[j];
  sort_k(acts, p.K);
  // -- cache policy step (kernels.py:89-145), state held one expert per lane --
  if (go) {
    uint32_t in_act = 0;   // the K activated ids are distinct (top-k, or checked forced ids)
#pragma unroll
    for (int j = 0; j < kMaxK; ++j)
      if (j < p.K) in_act |= 1u << acts[j];
    const uint32_t res0 = S.resident & emask;
    double fq = valid ? S.freq[lane] : 0.0;
    long long lt = valid ? S.last_touch[lane] : -1;
    if (p.policy == MOE_P_LFU_AGED && t > 0 && (t % p.decay_period) == 0) fq *= p.decay_factor;
    uint32_t res = res0;
    rb = res0;
    const bool lfu = p.policy == MOE_P_LFU || p.policy == MOE_P_LFU_AGED;
    const int need = __popc(res0) + __popc(in_act & ~res0) - p.C;
    for (int r = 0; r < need; ++r) {
      // argmin over resident & not activated: LRU (last_touch, id), LFU (freq, last_touch, id)
      const bool cand = ((res >> lane) & 1u) && !((in_act >> lane) & 1u);
      uint64_t best = ~0ull;
      if (lfu) {
        const uint64_t fb = cand ? static_cast<uint64_t>(__double_as_longlong(fq)) : ~0ull;
        const uint64_t fmin = warp_min_u64(fb);
        if (cand && fb == fmin) best = lru_key(lt, lane);
      } else if (cand) {
        best = lru_key(lt, lane);
      }
      best = warp_min_u64(best);
      if (best == ~0ull) {   // K > C: the reference's latent out-of-range eviction
        ok = false;
        break;
      }
      const int victim = static_cast<int>(best & 1023u);
      res &= ~(1u << victim);
      ev |= 1u << victim;
    }
    if ((in_act >> lane) & 1u) {
      fq += 1.0;
      lt = t;
    }
    res_after = (res | in_act) & emask;
    if (valid) {
      S.freq[lane] = fq;
      S.last_touch[lane] = lt;
    }
  }
  if (!ok) flags |= 2u;
  // speculation guesses
  if (do_guess) {
    warp_topk_k(zg, valid && finite, p.K, gs);
    ggap = topk_gap_k(zg, valid, gs, p.K);
    sort_k(gs, p.K);
  }
  if (do_prefetch) {
    const bool fe = __all_sync(FULL, !valid || isfinite(ze));
    warp_topk_k(ze, valid && fe, p.K, pf);
    sort_k(pf, p.K);
  }
  MailRecord& mr = sM;
  const unsigned long long t3 = p.phase_ns ? gtimer() : 0;
  // every lane has read S.resident / S.step above; lane 0 rewrites them below (racecheck:
  // warp-level WAR without this barrier)
  __syncwarp();
  if (lane == 0) {
    // -- record --
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j >= p.K) break;
      rec->sel[j] = sel[j];
      rec->prob[j] = psel[j];
      rec->acts[j] = acts[j];
      rec->guess[j] = do_guess ? gs[j] : -1;
      rec->early[j] = do_prefetch ? pf[j] : -1;
    }
    rec->rb = rb;
    rec->ev = ev;
    rec->flags = flags;
    rec->gap = gap;
    rec->guess_gap = ggap;
    rec->zscale[0] = zs_r;
    rec->zscale[1] = zs_g;
    if (flags) atomicOr(p.err, static_cast<int>(flags));
    int nd = 0, nc = 0, np = 0;
    if (go && ok) {
      S.resident = res_after;
      S.step = t + 1;
      int hits = 0;
#pragma unroll
      for (int j = 0; j < kMaxK; ++j)
        if (j < p.K) hits += (rb >> acts[j]) & 1u;
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
#pragma unroll
      for (int j = 0; j < kMaxK; ++j) {
        if (j >= p.K) break;
        const int e = acts[j];
        if ((rb >> e) & 1u) continue;
        for (int b = 0; b < p.NB; ++b)
          if (S.buf_stage_seq[b] == p.seq && S.buf_expert[b] == e && !S.buf_policy[b]) {
            S.buf_policy[b] = 1;
            S.buf_of[e] = b;
            S.buf_stage_seq[b] = -1;
            mr.demand_expert[nd] = e;
            mr.demand_buf[nd] = b;
            mr.demand_adopt[nd] = 1;
            ++nd;
            break;
          }
      }
      // the remaining staged buffers of this step were wrong guesses: cancel them
      for (int b = 0; b < p.NB; ++b)
        if (S.buf_stage_seq[b] == p.seq) {
          S.buf_stage_seq[b] = -1;
          mr.cancel_buf[nc++] = b;
        }
      // fresh demand misses take the lowest free buffer
#pragma unroll
      for (int j = 0; j < kMaxK; ++j) {
        if (j >= p.K) break;
        const int e = acts[j];
        if (((rb >> e) & 1u) || S.buf_of[e] >= 0) continue;
        int pick = -1;
        for (int b = 0; b < p.NB && pick < 0; ++b)
          if (!S.buf_policy[b]) pick = b;
        S.buf_policy[pick] = 1;
        S.buf_expert[pick] = e;
        S.buf_of[e] = pick;
        mr.demand_expert[nd] = e;
        mr.demand_buf[nd] = pick;
        mr.demand_adopt[nd] = 0;
        ++nd;
      }
      // speculative prefetch of layer l+1's guesses that are not resident there
      if (do_prefetch) {
        LayerState& S1 = sS1;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
          if (j >= p.K) break;
          const int g = pf[j];
          if (g < 0 || g >= p.E || S1.buf_of[g] >= 0) continue;
          int pick = -1;
          for (int b = 0; b < p.NB && pick < 0; ++b)
            if (!S1.buf_policy[b] && S1.buf_stage_seq[b] != p.seq + 1) pick = b;
          if (pick < 0) continue;
          S1.buf_stage_seq[pick] = p.seq + 1;
          S1.buf_expert[pick] = g;
          mr.prefetch_expert[np] = g;
          mr.prefetch_buf[np] = pick;
          ++np;
        }
      }
    }
    // ring back-pressure: if the host is far behind, make it acknowledge this step
    mr.seq = p.seq;
    mr.layer = p.layer;
    mr.n_demand = nd;
    mr.n_cancel = nc;
    mr.n_prefetch = np;
    mr.need_ack = (p.seq - consumed0) >= (kMailRing / 2) ? 1 : 0;
  }
  __syncwarp();
  const unsigned long long t4 = p.phase_ns ? gtimer() : 0;
  // write back the state and post the mail (all lanes, 16-byte stores)
  copy16(&p.states[p.layer], &sS, sizeof(LayerState), lane, 32);
  if (do_prefetch) copy16(&p.states[p.layer + 1], &sS1, sizeof(LayerState), lane, 32);
  // copy-engine transfer: post the decision to the host forwarder (SM transfer: no host)
  MailRecord* dst = p.mail ? p.mail + (p.seq % kMailRing) : nullptr;
  if (dst) {
    copy16(dst, &sM, offsetof(MailRecord, ready), lane, 32);
    __threadfence_system();
  }
  __syncwarp();
  if (lane == 0) {
    if (dst) {
      dst->ready = p.seq + 1;
      p.ctl->gate_done = static_cast<unsigned int>(p.seq + 1);
    }
    if (p.phase_ns) {
      const unsigned long long t5 = gtimer();
      atomicAdd(&p.phase_ns[0], t1 - t0);
      atomicAdd(&p.phase_ns[1], t2 - t1);
      atomicAdd(&p.phase_ns[2], t3 - t2);
      atomicAdd(&p.phase_ns[3], t4 - t3);
      atomicAdd(&p.phase_ns[4], t5 - t4);
      atomicAdd(&p.phase_ns[5], 1ull);
      // fused: first mixing CTA start -> gate start (the GEMV stream, partials, ticket)
      const unsigned long long mix0 = p.phase_ns[7];
      if (mix0) {
        const unsigned long long st0 = ~0ull - mix0;
        atomicAdd(&p.phase_ns[6], t0 - st0);
        // milestones of the slowest CTA (slots 8-10: last start, staging, main loop; 15:
        // partials), relative to the first CTA's start
        atomicAdd(&p.phase_ns[11], p.phase_ns[8] - st0);
        atomicAdd(&p.phase_ns[12], p.phase_ns[9] - st0);
        atomicAdd(&p.phase_ns[13], p.phase_ns[10] - st0);
        atomicAdd(&p.phase_ns[14], p.phase_ns[15] - st0);
        p.phase_ns[7] = p.phase_ns[8] = p.phase_ns[9] = p.phase_ns[10] = p.phase_ns[15] = 0ull;
      }
    }
  }
}

// (internal linkage: this header is included by several translation units)
static __global__ void __launch_bounds__(kGateThreads) gate_cache_kernel(GateParams p) {
  pdl_trigger();  // the FFN pass may launch and wait for the decision meanwhile
  __shared__ GateSmem gsm;
  gate_cache_body(p, gsm, threadIdx.x, blockDim.x, [] { __syncthreads(); }, true);
}

// ---- K3: expert FFN over the selected slots ---------------------------------------------
struct FfnParams {
  const float* h_mid;        // x of this layer
  const StepRecord* rec;
  const LayerState* state;   // buf_of for this layer
  const char* pool;          // this layer's buffers: pool + b * expert_bytes
  long long expert_bytes;
  int d, f, K;
  int phase;                 // 0: experts that hit (resident before), 1: misses, 2: all
  float* act;                // [K][f]
  float* y;                  // [K][d]
  // fused SM fetch (toy experts, SM transfer): a missed expert's rows are read from the mapped
  // host store and written through to its HBM buffer while they are used
  const char* store;         // this layer's host experts (device view), or nullptr
  DeviceStats* stats;
};

__device__ __forceinline__ bool ffn_phase_match(const FfnParams& p, int j, int* e_out) {
  const int e = p.rec->sel[j];
  *e_out = e;
  if (e < 0 || e >= kMaxE || p.rec->flags) return false;  // failed gate: nothing to run
  if (p.state->buf_of[e] < 0) return false;
  const bool hit = (p.rec->rb >> e) & 1u;
  return p.phase == 2 || (p.phase == 0) == hit;
}

// ---- SM transfer: missed experts copied from the mapped pinned store by the SMs ----------
// (device-driven: no host round trip per layer; for small experts, where latency dominates)
struct FetchParams {
  const StepRecord* rec;
  const LayerState* state;   // buf_of after this step's policy decision
  const char* store;         // device view of this layer's host experts [E][expert_bytes]
  char* pool;                // this layer's HBM buffers
  long long expert_bytes;    // multiple of 16
  int K;
  DeviceStats* stats;
};

static __global__ void __launch_bounds__(512) fetch_kernel(FetchParams p) {
  pdl_trigger();
  pdl_wait();
  if (p.rec->flags) return;
  // the step's missed experts as one flat range of 16-byte words, so every PCIe read of the
  // step is in flight together (8 per thread before its stores)
  const char* src[kMaxK];
  char* dst[kMaxK];
  int misses = 0;
  for (int j = 0; j < p.K; ++j) {
    const int e = p.rec->acts[j];
    if (e < 0 || e >= kMaxE || ((p.rec->rb >> e) & 1u)) continue;
    const int b = p.state->buf_of[e];
    if (b < 0) continue;
    src[misses] = p.store + e * p.expert_bytes;
    dst[misses] = p.pool + b * p.expert_bytes;
    ++misses;
  }
  if (!misses) return;
  const long long per = p.expert_bytes / 16, n16 = per * misses;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long k = i + u * stride, m = k / per;
      v[u] = ld_stream(reinterpret_cast<const uint4*>(src[m]) + (k - m * per));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long k = i + u * stride, m = k / per;
      reinterpret_cast<uint4*>(dst[m])[k - m * per] = v[u];
    }
  }
  for (; i < n16; i += stride) {
    const long long m = i / per;
    reinterpret_cast<uint4*>(dst[m])[i - m * per] = ld_stream(reinterpret_cast<const uint4*>(src[m]) + (i - m * per));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&p.stats->fetched_bytes, static_cast<unsigned long long>(misses) * p.expert_bytes);
}

// SwiGLU up projection: act[j][r] = silu(w1[r] . x) * (w3[r] . x)
static __global__ void __launch_bounds__(256) swiglu_up_kernel(FfnParams p) {
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
// Per-lane partial dot of one f32 row read from `src` (e.g. mapped host memory) that also
// stores the row to `dst` (the expert's HBM buffer): fetch and use in one pass.
__device__ __forceinline__ float lane_dot_f32_copy(const float* __restrict__ src, float* __restrict__ dst,
                                                   int n, const float4* pa, const float4* pb) {
  const int lane = threadIdx.x & 31;
  const float4* r = reinterpret_cast<const float4*>(src);
  float4* w = reinterpret_cast<float4*>(dst);
  float acc = 0.f;
  for (int i = lane; i < (n >> 3); i += 32) {
    const float4 w0 = r[2 * i], w1 = r[2 * i + 1];
    w[2 * i] = w0;
    w[2 * i + 1] = w1;
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

static __global__ void __launch_bounds__(256) toy_up_kernel(FfnParams p) {
  pdl_trigger();
  pdl_wait();  // before any early exit: a dependent's wait must cover the whole chain
  const int j = blockIdx.y;
  int e;
  if (!ffn_phase_match(p, j, &e)) return;
  extern __shared__ float4 smem4[];
  float4* pa = smem4;
  float4* pb = smem4 + p.d / 8;
  stage_planes(p.h_mid, p.d, pa, pb);
  __syncthreads();
  const int b = p.state->buf_of[e];
  float* w1 = reinterpret_cast<float*>(const_cast<char*>(p.pool) + b * p.expert_bytes);
  const bool fetch = p.store && !((p.rec->rb >> e) & 1u);
  const float* src = fetch ? reinterpret_cast<const float*>(p.store + e * p.expert_bytes) : w1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // a missed expert's W2t row r travels with its W1t row r (both reads in flight together),
  // so the down projection finds the whole expert in HBM
  const size_t half = static_cast<size_t>(p.d) * p.d;  // floats per matrix
  for (int r = blockIdx.x * nwarps + warp; r < p.d; r += gridDim.x * nwarps) {
    const size_t o = static_cast<size_t>(r) * p.d;
    float4 c2[4];
    const int n4 = p.d / 4;
    if (fetch)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = lane + 32 * u;
        if (i < n4) c2[u] = reinterpret_cast<const float4*>(src + half + o)[i];
      }
    const float s = warp_sum(fetch ? lane_dot_f32_copy(src + o, w1 + o, p.d, pa, pb)
                                   : lane_dot_f32(src + o, p.d, pa, pb));
    if (fetch) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = lane + 32 * u;
        if (i < n4) reinterpret_cast<float4*>(w1 + half + o)[i] = c2[u];
      }
      for (int i = lane + 128; i < n4; i += 32)  // rows wider than 512 floats
        reinterpret_cast<float4*>(w1 + half + o)[i] = reinterpret_cast<const float4*>(src + half + o)[i];
    }
    if (lane == 0) p.act[j * p.f + r] = tanhf(s);
  }
  if (fetch && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&p.stats->fetched_bytes, static_cast<unsigned long long>(p.expert_bytes));
}

// Down projection: y[j][c] = W[c] . act[j]; W = w2 (SwiGLU, [d][f]) or W2t (toy, [d][d]).
template <bool kBF16>
__global__ void __launch_bounds__(256) down_kernel(FfnParams p) {
  pdl_trigger();
  pdl_wait();
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
  const bool fetch = !kBF16 && p.store && !((p.rec->rb >> e) & 1u);
  const char* src = fetch ? p.store + e * p.expert_bytes + static_cast<size_t>(p.d) * p.d * esz : W;
  for (int c = blockIdx.x * nwarps + warp; c < p.d; c += gridDim.x * nwarps) {
    float part;
    if constexpr (!kBF16) {
      const size_t o = static_cast<size_t>(c) * p.f;
      part = fetch ? lane_dot_f32_copy(reinterpret_cast<const float*>(src) + o,
                                       reinterpret_cast<float*>(const_cast<char*>(W)) + o, p.f, pa, pb)
                   : lane_dot_f32(reinterpret_cast<const float*>(W) + o, p.f, pa, pb);
    } else {
      part = lane_dot<kBF16>(W + static_cast<size_t>(c) * p.f * esz, p.f, pa, pb);
    }
    const float s = warp_sum(part);
    if (lane == 0) p.y[j * p.d + c] = s;
  }
  if (fetch && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(&p.stats->fetched_bytes, static_cast<unsigned long long>(p.expert_bytes / 2));
}

// Final layer: h_out = h' + sum_j p_j y_j
static __global__ void finalize_kernel(const float* h_mid, const float* y, const StepRecord* rec, int K,
                                int d, float* out) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) out[i] = combine_elem(h_mid, y, rec, K, d, i);
}

// ---- token graph plumbing: move the token in flight between the rings and the fixed buffers
static __global__ void set_cursor_kernel(long long* cursor, long long v) { *cursor = v; }

static __global__ void token_begin_kernel(const long long* cursor, const float* x_stage, int cap,
                                          int D, float* x_cur) {
  pdl_trigger();
  pdl_wait();
  const float* src = x_stage + (*cursor % cap) * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) x_cur[i] = src[i];
}

static __global__ void token_end_kernel(long long* cursor, const StepRecord* cur_rec,
                                        StepRecord* ring, const float* out_cur, float* out_stage,
                                        int cap, int L, int D) {
  pdl_wait();
  const long long row = *cursor % cap;
  copy16(ring + row * L, cur_rec, static_cast<int>(sizeof(StepRecord)) * L, threadIdx.x, blockDim.x);
  for (int i = threadIdx.x; i < D; i += blockDim.x) out_stage[row * D + i] = out_cur[i];
  __syncthreads();
  if (threadIdx.x == 0) *cursor += 1;
}

static __global__ void reset_states_kernel(LayerState* s, int L, int NB) {
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
