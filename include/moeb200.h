/*
 * moeb200.h -- C ABI of libmoeb200.so, the B200-native MoE-offloading decode engine.
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes (no torch or
 * CUDA runtime types in the signatures: streams are passed as `void*` holding a
 * cudaStream_t, 0 = the legacy default stream) and returns a moe_status.
 * On failure, moe_last_error() returns a thread-local message.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/moesim):
 *   moe_replay_policy          <- kernels.replay_policy            kernels.py:60-147
 *   moe_replay_policy_layers   <- simulate.simulate's layer loop   simulate.py:167-174
 *   moe_policy_step            <- policies.policy_step             policies.py:140-228
 *   moe_gate_topk_f64          <- toymoe._gate_topk / gate_select  toymoe.py:99-126
 *   moe_toy_forward_f64        <- toymoe._forward / forward_token  toymoe.py:129-146
 *   moe_engine_*               <- toymoe.run_model decode loop     toymoe.py:159-190
 *                                 + per-layer cache (simulate.py:140-184) live on device
 * Status codes map onto the reference exception taxonomy (errors.py:8-31):
 *   MOE_INVALID_CONFIG -> ConfigError, MOE_NONFINITE -> FloatingPointError
 *   (toymoe.py:109-110).
 */
#ifndef MOEB200_H
#define MOEB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_ABI_VERSION 4

typedef int32_t moe_status;
enum {
  MOE_OK = 0,
  MOE_INVALID_CONFIG = 1, /* ConfigError */
  MOE_NONFINITE = 2,      /* FloatingPointError("gate logits are not finite") */
  MOE_CUDA_ERROR = 3,
  MOE_OOM = 4,
};

/* Policy codes shared with the reference (kernels.py:53-57, simulate.py:23). */
enum { MOE_P_LRU = 0, MOE_P_LFU = 1, MOE_P_LFU_AGED = 2, MOE_P_OPT = 3 };

/* Expert bodies. TOY_TANH is the reference's expert (toymoe.py:143-145),
 * SWIGLU the Mixtral-shaped north-star expert (w2 . (silu(w1 h) * w3 h)). */
enum { MOE_EXPERT_TOY_TANH_F32 = 0, MOE_EXPERT_SWIGLU_BF16 = 1 };

/* Transfer engines.  COPY_ENGINE: the device posts its decision to a mapped
 * mailbox and the host forwards cudaMemcpyAsync on a copy stream (peak link bandwidth, one host
 * round trip per layer).  SM: a fetch kernel reads the missed experts from the mapped pinned
 * store itself (no host in the loop; ~15 % below the copy engine's bandwidth).  AUTO: SM for
 * experts <= 16 MiB (latency-bound), the copy engine otherwise; prefetch needs the copy engine. */
enum { MOE_TRANSFER_AUTO = 0, MOE_TRANSFER_COPY_ENGINE = 1, MOE_TRANSFER_SM = 2 };

/* Speculative prefetch issue point. */
enum {
  MOE_PREFETCH_OFF = 0,
  MOE_PREFETCH_EARLY = 1 /* gate_{l+1}(h'_l): post-mixing state of layer l */
};

const char* moe_last_error(void);
int32_t moe_abi_version(void);
/* Number of CUDA kernels this library has launched in this process (all entry points). */
uint64_t moe_kernel_launches(void);

/* ---- cache policy: offline replay (K7) ------------------------------------------- */

/* Replay one layer's activation stream through a policy, on the GPU.
 * acts_dev: (T, K) int64, C-contiguous, rows ascending distinct ids in [0, E).
 * resident_before_dev / evicted_dev: (T, E) uint8 outputs (device).
 * decay_factor / decay_period are only read for MOE_P_LFU_AGED (pass 1.0 / 1 otherwise).
 * Bit-exact with kernels.replay_policy (kernels.py:60-147). E <= 256, K <= C. */
moe_status moe_replay_policy(const int64_t* acts_dev, int64_t T, int32_t K, int32_t E,
                             int32_t C, int32_t policy, double decay_factor,
                             int64_t decay_period, uint8_t* resident_before_dev,
                             uint8_t* evicted_dev, void* stream);

/* L independent layers in one launch: acts (L, T, K), outputs (L, T, E). */
moe_status moe_replay_policy_layers(const int64_t* acts_dev, int32_t L, int64_t T, int32_t K,
                                    int32_t E, int32_t C, int32_t policy, double decay_factor,
                                    int64_t decay_period, uint8_t* resident_before_dev,
                                    uint8_t* evicted_dev, void* stream);

/* ---- cache policy: one step with explicit state (policies.policy_step) ------------ */

/* State arrays (device, length E, updated in place):
 *   resident u8, last_touch i64 (larger = more recent; ties break to the lower id),
 *   freq f64.  *step is the step counter (host value, used for lfu-aged decay).
 * act_dev: n_act int64 ids.  For MOE_P_OPT, future_ids_dev / future_offsets_dev describe
 * the remaining stream as a ragged array (n_future sets; offsets has n_future+1 entries).
 * Outputs (device, length E): resident_before u8, evicted u8.
 * The caller validates n_act <= C (policies.py:153-156). */
moe_status moe_policy_step(uint8_t* resident_dev, int64_t* last_touch_dev, double* freq_dev,
                           int64_t step, int32_t E, int32_t C, int32_t policy,
                           double decay_factor, int64_t decay_period, const int64_t* act_dev,
                           int32_t n_act, const int64_t* future_ids_dev,
                           const int64_t* future_offsets_dev, int64_t n_future,
                           uint8_t* resident_before_dev, uint8_t* evicted_dev, void* stream);

/* ---- gate (K1) on arbitrary gates, fp64 (toymoe.gate_select / speculate_next) ------ */

/* h_dev (d,), w_dev (d, E) in the reference layout (toymoe.py:50), bias_dev (E,) or NULL.
 * Outputs: order_dev (k,) int64 prob-desc with ties to the lower id, probs_dev (E,) f64.
 * Returns MOE_NONFINITE if any logit is non-finite. */
moe_status moe_gate_topk_f64(const double* h_dev, const double* w_dev, const double* bias_dev,
                             int32_t d, int32_t E, int32_t k, int64_t* order_dev,
                             double* probs_dev, void* stream);

/* One toy layer step, fp64 (toymoe._forward, toymoe.py:138-146):
 * h = x + alpha * (x @ M); gate; out = h + sum_{e in sel, prob-desc} p_e * tanh(h @ W1_e) @ W2_e.
 * mixing (d, d), gate_w (d, E), gate_b (E,) or NULL, w1/w2 (E, d, d), all reference layout. */
moe_status moe_toy_forward_f64(const double* x_dev, const double* mixing_dev,
                               const double* gate_w_dev, const double* gate_b_dev,
                               const double* w1_dev, const double* w2_dev, int32_t d, int32_t E,
                               int32_t k, double alpha, double* out_dev, int64_t* selected_dev,
                               double* probs_dev, void* stream);

/* ---- the offload decode engine ------------------------------------------------------ */

typedef struct moe_engine moe_engine;

typedef struct {
  int32_t num_layers;     /* L */
  int32_t num_experts;    /* E (<= 32 for the live engine) */
  int32_t top_k;          /* K */
  int32_t hidden_dim;     /* d */
  int32_t ffn_dim;        /* f (SwiGLU); ignored for the toy expert (f = d) */
  int32_t expert_kind;    /* MOE_EXPERT_* */
  int32_t cache_size;     /* C policy slots per layer (simulate.SimConfig.cache_size) */
  int32_t policy;         /* MOE_P_LRU / MOE_P_LFU / MOE_P_LFU_AGED (OPT is offline-only) */
  double decay_factor;    /* lfu-aged only */
  int64_t decay_period;   /* lfu-aged only */
  float mixing_scale;     /* alpha (toymoe.py:140) */
  int32_t prefetch;       /* MOE_PREFETCH_* */
  int32_t renormalize;    /* 0: reference routing (softmax over E, no renorm, toymoe.py:122-123)
                             1: Mixtral routing (renormalise the top-k probabilities) */
  int32_t record_speculation; /* record the reference-definition guess (toymoe.py:178-180) */
  int32_t max_tokens;     /* capacity of the device step-record ring */
  int64_t chunk_bytes;    /* transfer chunk size (prefetch cancellation granularity) */
  int32_t prefetch_depth; /* max prefetch chunks in flight on the copy stream */
  int32_t device;
  int32_t rms_norm;       /* 1: RMSNorm (unit scale) of h' before gate and experts, as in
                             Mixtral; keeps the SwiGLU residual stream finite.  0: reference
                             toy semantics (no norm, toymoe.py:138-146). */
  float rms_eps;          /* RMSNorm epsilon (Mixtral: 1e-5) */
  int32_t transfer;       /* MOE_TRANSFER_*: how missed experts reach HBM */
  int32_t store_layers;   /* host expert store depth: 0 = num_layers.  S < num_layers aliases
                             layer l's experts to store layer l % S (synthetic models deeper
                             than host RAM holds, e.g. Mixtral-8x22B's 271 GB on a 196 GB
                             host); HBM caches, routing and transfers stay per layer. */
  int32_t prefetch_buffers; /* staging buffers per layer with prefetch on: 0 = top_k; fewer
                               fit deeper models in HBM (prefetch then covers the best guesses) */
  int32_t compress;       /* 1: demand and prefill copies move the experts exponent-coded
                             (expcodec.cuh, lossless, ~0.65x the bytes) and decode them in HBM;
                             SwiGLU engines, copy engine.  2: the same with no raw store kept
                             (coded store only: deeper models fit the host; private stores) */
} moe_engine_config;

typedef struct {
  int64_t tokens;           /* decode tokens processed */
  int64_t steps;            /* (token, layer) steps */
  int64_t hits, misses;     /* policy hits / misses */
  int64_t h2d_bytes;        /* bytes copied host->device for experts (demand + prefetch) */
  int64_t demand_bytes;     /* expert bytes delivered to demand misses (== misses * expert_bytes
                               without prefetch; raw bf16 equivalent when compressed) */
  int64_t prefetch_bytes;   /* of which speculative prefetch chunks issued */
  int64_t prefetch_issued;  /* experts prefetched (guess not resident) */
  int64_t prefetch_used;    /* prefetched experts adopted by a demand miss */
  int64_t prefetch_wasted_bytes; /* bytes of prefetch chunks for guesses that were wrong */
  int64_t expert_bytes;     /* bytes of one expert block */
  double copy_busy_ms;      /* copy-stream busy time for demand transfers (events) */
  int64_t prefill_tokens;   /* tokens processed by moe_engine_prefill */
  int64_t prefill_bytes;    /* bytes copied host->device by prefill (one load per needed expert
                               per layer; included in h2d_bytes) */
  int64_t demand_link_bytes;   /* bytes the demand copies put on the link (== demand_bytes
                                  uncompressed; h2d_bytes = demand_link + prefetch + prefill) */
  int64_t compressed_store_bytes; /* host bytes of the exponent-coded expert store (0: off) */
  int64_t peer_bytes;             /* expert bytes copied from the peer-HBM tier (ABI 4; not in
                                     h2d_bytes, which counts the PCIe link only) */
} moe_stats;

moe_status moe_engine_create(const moe_engine_config* cfg, moe_engine** out);
/* Same, with a caller-owned host expert store ([L][E][expert] bytes, e.g. a POSIX shared-memory
 * segment shared by the replicas of one node); the engine page-locks it with cudaHostRegister
 * and never frees it.  store == NULL allocates a private pinned store. */
moe_status moe_engine_create_ex(const moe_engine_config* cfg, void* store, int64_t store_bytes,
                                moe_engine** out);
moe_status moe_engine_destroy(moe_engine* eng);

/* Dense per-layer weights from host memory, reference layout (toymoe.py:74-83):
 * mixing (d, d) as `x @ M`, gate_w (d, E), gate_b (E,). dtype: f32. */
moe_status moe_engine_set_dense_f32(moe_engine* eng, int32_t layer, const float* mixing,
                                    const float* gate_w, const float* gate_b);
/* One toy expert from host memory, reference layout: w1, w2 (d, d) f32 (toymoe.py:82-83). */
moe_status moe_engine_set_toy_expert_f32(moe_engine* eng, int32_t layer, int32_t expert,
                                         const float* w1, const float* w2);
/* Synthetic Mixtral-shaped weights from the counter-hash generator (moe_hash_weights).
 * gate_bias_std is the reference's expert-imbalance knob (toymoe `skew`, toymoe.py:75);
 * see DESIGN.md for the value the bench uses.  init_experts = 0 writes only the device-resident
 * dense weights (a replica attached to a store its owner already filled). */
moe_status moe_engine_init_random(moe_engine* eng, uint64_t seed, float gate_bias_std,
                                  int32_t init_experts);
/* Host view of one expert block in the pinned store ([w1 | w3 | w2] bf16 or [W1t | W2t] f32). */
moe_status moe_engine_expert_host_ptr(moe_engine* eng, int32_t layer, int32_t expert,
                                      void** ptr, int64_t* bytes);
/* Node-shared coded store (compress = 1 with a caller-owned raw store): the raw experts must be
 * written first.  coded_size returns the bytes of the coded segment (layout planned from the
 * raw store); attach_coded with build = 1 encodes into `seg` (the segment's owner), build = 0
 * reads an already built segment (the other replicas).  The segment is page-locked. */
moe_status moe_engine_coded_size(moe_engine* eng, int64_t* bytes);
moe_status moe_engine_attach_coded(moe_engine* eng, void* seg, int64_t seg_bytes, int32_t build);
/* Copy back the device-layout dense weights (for the oracle): mixing (d,d) in the device
 * dtype's bytes, gate_w (E,d) f32, gate_b (E,) f32; host destinations. */
moe_status moe_engine_dense_host(moe_engine* eng, int32_t layer, void* mixing, float* gate_w,
                                 float* gate_b);

/* Reset every per-layer cache to the cold state (policies.warm_state, policies.py:133-137). */
moe_status moe_engine_reset(moe_engine* eng);

/* Switch policy / cache size / prefetch mode and reset to cold caches.  cache_size may not
 * exceed the capacity given at creation; prefetch needs the engine to have been created
 * with prefetch != OFF (staging buffers are allocated then). */
moe_status moe_engine_set_mode(moe_engine* eng, int32_t policy, double decay_factor,
                               int64_t decay_period, int32_t cache_size, int32_t prefetch);

/* Per-launch CUDA-event timing of the engine's kernels (recorded on the compute stream). */
typedef struct {
  double mix_ms, gate_ms, ffn_ms, finalize_ms; /* summed device time per kernel class */
  int64_t mix_launches, gate_launches, ffn_launches, finalize_launches;
  int64_t ffn_expert_runs; /* expert FFN executions (K per step) covered by ffn_ms */
  double ffn_active_ms;     /* device time of the FFN launches that processed >= 1 expert */
  int64_t ffn_active_bytes; /* weight bytes those launches streamed (device-counted) */
  int64_t ffn_active_launches;
  /* prefill: tcgen05 grouped GEMM launches (mix, SwiGLU up, down) */
  double gemm_ms;           /* summed CUDA-event time of the GEMM launches */
  int64_t gemm_launches;
  double gemm_flops;        /* algorithmic FLOPs of those launches (2*m*n*k per group) */
  int64_t gemm_bytes;       /* algorithmic bytes: weights + activations read + outputs written */
  double prefill_ms;        /* whole-prefill device time (first kernel to last, per call, summed) */
  double ffn_kernel_ms;     /* in-kernel span (globaltimer, first CTA start -> last CTA end) of
                               the FFN launches that processed >= 1 expert: excludes launch
                               latency and the host-side gaps the events see */
  double gemm_kernel_ms;    /* the same in-kernel span summed over the prefill GEMM launches */
  /* decode: exponent-decode launches of coded demand / adopted experts (ABI 3) */
  double xdec_ms;           /* summed CUDA-event time */
  double xdec_kernel_ms;    /* summed in-kernel span (globaltimer) */
  int64_t xdec_bytes;       /* algorithmic bytes: coded part read + bf16 weights written */
  int64_t xdec_launches;
} moe_kernel_times;
moe_status moe_engine_profile(moe_engine* eng, int32_t enable);
/* Resolves outstanding events (synchronises) and returns the running totals. */
moe_status moe_engine_kernel_times(moe_engine* eng, moe_kernel_times* out);

/* Decode T tokens: h_in_dev (T, d) f32 device, h_out_dev (T, d) f32 device.
 * Token t's step records go to ring position (tokens_done + t) % max_tokens. */
moe_status moe_engine_decode(moe_engine* eng, const float* h_in_dev, int64_t T,
                             float* h_out_dev, void* stream);

/* Prefill T tokens as one batch (layer-major): for each layer, the mixing map for all T rows
 * on the tensor cores, the gate for every token, the cache policy replayed over the T steps in
 * token order (so step records, hit/miss/evict traces and the final cache state equal those of
 * T decode steps), one H2D load of every needed expert that is not resident, and the SwiGLU
 * experts as tcgen05 grouped GEMMs over the token groups.  Activations enter the GEMMs in bf16
 * (the decode path keeps them f32), so outputs agree with decode within the bf16 tolerance.
 * SwiGLU engines only; T <= max_tokens; hidden_dim % 256 == 0, ffn_dim % 128 == 0.
 * h_in_dev / h_out_dev as for moe_engine_decode.  Replaces run_model's token loop
 * (toymoe.py:175-185) for a batch of independent tokens. */
moe_status moe_engine_prefill(moe_engine* eng, const float* h_in_dev, int64_t T,
                              float* h_out_dev, void* stream);

/* Trace-driven routing: as moe_engine_decode / moe_engine_prefill, but step
 * (t, l) activates the K experts routing_dev[(t * L + l) * K + 0..K) (int32, device; e.g. an
 * ActivationTrace from gen_zipf / gen_markov or a recorded trace) instead of the gate's top-k.
 * The gate's softmax still weights them; caches, transfers and the FFN run as usual, so the
 * event log equals the reference's simulate() of that trace.  Ids out of range or repeated in
 * a step flag the step (moe_engine_sync -> MOE_INVALID_CONFIG). */
moe_status moe_engine_decode_routed(moe_engine* eng, const float* h_in_dev, int64_t T,
                                    float* h_out_dev, const int32_t* routing_dev, void* stream);
moe_status moe_engine_prefill_routed(moe_engine* eng, const float* h_in_dev, int64_t T,
                                     float* h_out_dev, const int32_t* routing_dev, void* stream);

/* Block until the engine's outstanding work is complete; reports MOE_NONFINITE if any
 * gate produced non-finite logits since the last call. */
moe_status moe_engine_sync(moe_engine* eng);

/* Read the step records of tokens [t0, t0+T) (absolute token indices; must still be in
 * the ring). Host outputs, any may be NULL:
 *   acts (T, L, K) int64 sorted ascending; guessed (T, L-1, K) int64 sorted;
 *   resident_before / evicted (T, L, E) uint8; probs (T, L, K) f32 in selection order. */
moe_status moe_engine_records(moe_engine* eng, int64_t t0, int64_t T, int64_t* acts,
                              int64_t* guessed, uint8_t* resident_before, uint8_t* evicted,
                              float* probs);

/* Per-step margins and early guesses of the same steps (ABI 4); either output may be NULL.
 *   gaps (T, L) f32: the route logit of the K-th selected expert minus the largest unselected
 *     logit (toymoe.py:99-115 ranks by logit desc, ties to the lower id; a margin below the fp
 *     tolerance marks a selection the fp64 reference could order differently).  +inf when
 *     K == E, NaN for trace-driven steps.
 *   guess_gaps (T, L-1) f32: the same margin of the reference-definition guess for layer l
 *     (gate_l on the output of l-1, toymoe.py:178-180); NaN without speculation records.
 *   zscales (T, L, 2) f32: the largest |logit| of the route and of the guess at each step,
 *     for margins relative to the logit scale (fp32 logit error grows with it).
 *   early (T, L-1, K) int64: the early guess for layer l+1 made at step (t, l) (gate_{l+1} on
 *     h'_l, ascending) that drove its speculative prefetch; -1 with prefetch off or in a
 *     prefill. */
moe_status moe_engine_record_gaps(moe_engine* eng, int64_t t0, int64_t T, float* gaps,
                                  float* guess_gaps, float* zscales, int64_t* early);

moe_status moe_engine_stats(moe_engine* eng, moe_stats* out);

/* NVLink peer-HBM miss tier (ABI 4), off until attached.  ptrs[l * E + e] is the
 * device address of the raw expert block (layer l, expert e) -- on a peer GPU of the node
 * (opened with cudaIpcOpenMemHandle, peer access enabled) or on this GPU -- or NULL for
 * experts the tier does not hold.  Demand misses and speculative prefetches of held experts
 * are copied from there by the copy engine (device to device, NVLink for a peer) instead of
 * from the pinned host store over PCIe; only the transfer source changes: selections, cache
 * decisions and buffers are the device's as before, so traces and outputs are identical.
 * The reference models the transfer source as a constant bandwidth (costmodel.py:90-111).
 * Copy-engine transfer mode only.  n = L * E; ptrs == NULL (n = 0) detaches.  The caller keeps
 * the blocks alive and unchanged while attached. */
moe_status moe_engine_attach_peer_tier(moe_engine* eng, const void* const* ptrs, int64_t n);

/* ---- kernel microbenchmark (tuning aid) --------------------------------------------- */

/* Times one decode GEMV kernel in isolation on synthetic resident weights (4 rotating
 * weight sets, so consecutive iterations miss in L2).  kernel: 0 stream mix, 1 stream up,
 * 2 stream down (bulk-copy pipelines), 3/4/5 the same ops as plain LDG kernels.
 * stage_kb / max_stages / grid / rpb (rows per block: 8, 4, 2) tune the stream kernels;
 * 0 selects the engine's default for each. */
moe_status moe_microbench_gemv(int32_t kernel, int32_t d, int32_t f, int32_t experts,
                               int32_t stage_kb, int32_t max_stages, int32_t grid, int32_t rpb,
                               int32_t iters, float* ms_per_iter, int64_t* bytes_per_iter);

/* ---- K4: tcgen05 grouped GEMM (prefill), test / microbenchmark entry points ----------- */

/* Grouped C = A . B^T on the tensor cores (tcgen05.mma 128x256x16, TMA, TMEM accumulators).
 * A (sum(group_m), K) bf16 row-major, groups stacked in order; B (G*N, K) bf16 row-major,
 * group g's matrix at rows [g*N, (g+1)*N) (nn.Linear layout); C (sum(group_m), N) f32.
 * group_m: host array of G row counts (0 allowed).  K % 64 == 0, N % 256 == 0.
 * splits > 1: split-K; C then holds `splits` planes (splits, sum(group_m), N) whose sum is the
 * product (each plane one contiguous k-range; 1 <= splits <= K/64).
 * Runs `iters` times; ms_per_iter (may be NULL) gets the CUDA-event time per launch. */
moe_status moe_tc_grouped_gemm_bf16(const uint16_t* A, const uint16_t* B, float* C, int32_t G,
                                    const int32_t* group_m, int32_t N, int32_t K, int32_t splits,
                                    int32_t iters, float* ms_per_iter, void* stream);
/* Grouped SwiGLU up projection, the prefill expert's first half:
 * act = bf16(silu(X . w1^T) * (X . w3^T)); X (sum(group_m), d) bf16; W13 (G, 2f, d) bf16 with
 * w1 rows [0, f) and w3 rows [f, 2f) per group; act (sum(group_m), f) bf16.
 * d % 64 == 0, f % 128 == 0. */
moe_status moe_tc_grouped_swiglu_bf16(const uint16_t* X, const uint16_t* W13, uint16_t* act,
                                      int32_t G, const int32_t* group_m, int32_t f, int32_t d,
                                      int32_t iters, float* ms_per_iter, void* stream);

/* ---- synthetic routing workloads (tracegen) ---------------------------------------------- */

/* kernels.sample_zipf_layer for all L layers at once (kernels.py:150-184): weights (L, E) f64,
 * uniforms (L, T, K) f64 (the reference's per-layer rng.random((T, K)) draws, tracegen.py:86),
 * out (T, L, K) int64 rows ascending.  Device pointers; E <= 64. */
moe_status moe_sample_zipf(const double* weights_dev, int32_t L, int32_t E, int64_t T, int32_t K,
                           const double* uniforms_dev, int64_t* out_dev, void* stream);
/* kernels.sample_markov_layer for all L layers (kernels.py:187-232): u_retain / u_draw
 * (L, T, K) f64 (tracegen.py:104-105), out (T, L, K) int64. */
moe_status moe_sample_markov(const double* weights_dev, int32_t L, int32_t E, int64_t T, int32_t K,
                             double repeat_prob, const double* u_retain_dev,
                             const double* u_draw_dev, int64_t* out_dev, void* stream);

/* ---- lossless bf16 exponent coding of expert parts (expcodec.cuh) --------------------- */

/* Encode n bf16 words (host) into one part: out == NULL returns the size only.  kbits 0 picks
 * 3 or 4 bits per exponent code (smaller output).  Multi-threaded. */
moe_status moe_xc_encode(const uint16_t* in, uint64_t n, int32_t kbits, void* out, uint64_t cap,
                         uint64_t* size);
/* Decode a part already in device memory; header_host = a host copy of its first 64 bytes. */
moe_status moe_xc_decode(const void* part_dev, const void* header_host, uint16_t* out_dev,
                         void* stream);

/* ---- trace / event-log JSONL (host only, no CUDA) ------------------------------------ */

/* A formatted document owned by the library (moe_text_free). */
typedef struct moe_text moe_text;
const char* moe_text_data(const moe_text* doc);
int64_t moe_text_size(const moe_text* doc);
void moe_text_free(moe_text* doc);

/* traces.write_trace (traces.py:267-312), byte for byte.  kind 0: ActivationTrace, grid_a
 * (T, L, K) int64 sorted rows; kind 1: SpeculationTrace, grid_g = guessed and grid_a = actual,
 * both (T, L-1, K).  Formatted on all host threads for long traces. */
moe_status moe_format_trace(int32_t kind, int32_t num_layers, int32_t num_experts, int32_t top_k,
                            int64_t T, const int64_t* grid_a, const int64_t* grid_g,
                            moe_text** doc);
/* simulate.write_event_log (simulate.py:187-226) of a columnar CacheEventLog: layers[n_layers]
 * (log.layers), activated (n_layers, T, K) int64, resident_before / evicted (n_layers, T, E)
 * uint8; policy is str(PolicyKind) (e.g. "lru", "lfu-aged:0.5:16"). */
moe_status moe_format_event_log(const char* policy, int32_t cache_size, int32_t num_layers,
                                int32_t num_experts, int32_t top_k, int64_t warmup_tokens,
                                int32_t n_layers, const int32_t* layers, int64_t T,
                                const int64_t* activated, const uint8_t* resident_before,
                                const uint8_t* evicted, moe_text** doc);

/* ---- synthetic weights (counter hash), shared with oracle/weights.c ---------------- */

/* bf16 bits of element `index` of tensor `tensor_id` for seed `seed`, scaled to unit
 * variance * std (uniform on [-sqrt(3), sqrt(3)) * std).  See DESIGN.md "Synthetic weights". */
moe_status moe_hash_weights_bf16(uint64_t seed, uint64_t tensor_id, float std, int64_t n,
                                 uint16_t* out_dev, void* stream);
moe_status moe_hash_weights_f32(uint64_t seed, uint64_t tensor_id, float std, int64_t n,
                                float* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOEB200_H */
