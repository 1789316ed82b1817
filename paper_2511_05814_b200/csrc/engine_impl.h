// Host-side state of one offload engine (engine.cu: decode; prefill.cu: batched prefill).
#pragma once
#include "engine_kernels.cuh"
#include "expcodec.cuh"

#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace moe {

moe_status launch_hash_bf16(uint64_t seed, uint64_t tid, float std, long long n, uint16_t* out,
                            cudaStream_t s);
moe_status launch_hash_f32(uint64_t seed, uint64_t tid, float std, long long n, float* out,
                           cudaStream_t s);

// ---- pinned host store ------------------------------------------------------------------
// Default: cudaHostAlloc (portable).  MOE_PIN_MODE=register: anonymous mapping with
// transparent huge pages, first-touched by all host threads in parallel, then
// cudaHostRegister (faster to set up for the 90 GB Mixtral-8x7B store).
struct PinnedStore {
  char* base = nullptr;
  size_t bytes = 0;
  bool registered = false;
  bool via_alloc = false;
  bool external = false;  // caller-owned memory (e.g. a shared-memory store), only registered
  double setup_ms = 0;

  moe_status attach(void* p, size_t n) {
    base = static_cast<char*>(p);
    bytes = n;
    external = true;
    const cudaError_t e = cudaHostRegister(base, n, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {  // another engine of this process did
      cudaGetLastError();
      return MOE_OK;
    }
    MOE_CUDA(e);
    registered = true;
    return MOE_OK;
  }

  moe_status allocate(size_t n) {
    const auto t0 = std::chrono::steady_clock::now();
    bytes = n;
    const char* mode = getenv("MOE_PIN_MODE");
    if (!(mode && strcmp(mode, "register") == 0)) {
      via_alloc = true;
      MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&base), n,
                             cudaHostAllocPortable | cudaHostAllocMapped));
    } else {
      void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
      if (p == MAP_FAILED) {
        set_error("mmap of %zu bytes for the expert store failed", n);
        return MOE_OOM;
      }
      base = static_cast<char*>(p);
      madvise(base, n, MADV_HUGEPAGE);
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      const size_t per = ((n + hw - 1) / hw + 4095) & ~size_t(4095);
      std::vector<std::thread> th;
      for (unsigned i = 0; i < hw; ++i)
        th.emplace_back([this, i, per] {
          const size_t lo = i * per, hi = std::min(bytes, lo + per);
          for (size_t o = lo; o < hi; o += 4096) base[o] = 0;
        });
      for (auto& x : th) x.join();
      MOE_CUDA(cudaHostRegister(base, n, cudaHostRegisterPortable | cudaHostRegisterMapped));
      registered = true;
    }
    setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return MOE_OK;
  }
  void release() {
    if (!base) return;
    if (external) {
      if (registered) cudaHostUnregister(base);
      base = nullptr;
      return;
    }
    if (via_alloc) {
      cudaFreeHost(base);
    } else {
      if (registered) cudaHostUnregister(base);
      munmap(base, bytes);
    }
    base = nullptr;
  }
};

struct PrefillState;
void prefill_release(PrefillState* pf);

struct PrefetchJob {
  int layer, buf, expert;
  long long next_chunk, n_chunks;
  bool cancelled, adopted;
  int zone = -1;        // compressed: landing zone of the exponent-coded expert (-1: raw copy
                        // straight into the staging buffer)
  long long bytes = 0;  // bytes this job moves (expert_bytes raw, or the coded size)
  bool peer = false;    // raw copy from the peer-HBM tier (not over PCIe)
};

}  // namespace moe

using namespace moe;

struct moe_engine {
  moe_engine_config cfg{};
  int d = 0, dpad = 0, f = 0, NB = 0, S = 0;
  int SL = 0;  // layers held by the host store (layer l uses store layer l % SL)
  bool bf16 = false;
  long long expert_bytes = 0;
  int device = 0;

  // device memory
  char* pool = nullptr;          // [L][NB][expert_bytes]
  void* mixing = nullptr;        // [L][dpad][dpad] (bf16 or f32), device layout
  float* gate_w = nullptr;       // [L][E][dpad]
  float* gate_b = nullptr;       // [L][E]
  LayerState* states = nullptr;  // [L]
  StepRecord* ring = nullptr;    // [max_tokens][L]
  float *h_in = nullptr, *h_mid = nullptr, *h_norm = nullptr, *y = nullptr, *act = nullptr;
  float* gate_part = nullptr;   // [148][3E + 2] partial gate logits from the mixing GEMV
  unsigned int* mix_ctr = nullptr;  // fused mix + gate: CTAs done (zero between launches)
  float* norm_scale = nullptr;  // 1 / rms(h') of the current layer
  float *x_pad = nullptr, *out_pad = nullptr;  // padded token staging when d % 8 != 0
  int* err = nullptr;
  DeviceStats* dstats = nullptr;

  // mapped pinned memory shared with the device
  MailRecord* mail_h = nullptr;
  MailRecord* mail_d = nullptr;
  HostControl* ctl_h = nullptr;
  HostControl* ctl_d = nullptr;

  PinnedStore store;
  // exponent-coded copy of the store (compress = 1): parts A (w1|w3) and B (w2) per expert
  struct CPart {
    uint64_t off, size;
    moe::xc::PartHeader hdr;
  };
  // coded expert = part 0 (w1|w3) + kCodedBParts row pieces of w2, contiguous in the store, so
  // the last piece of a transfer is small and its decode (the step's tail) short
  static constexpr int kCodedBParts = 4;
  static constexpr int kCodedParts = 1 + kCodedBParts;
  const CPart* coded_parts(int layer, int expert) const {
    return &ctab[(static_cast<size_t>(layer % SL) * cfg.num_experts + expert) * kCodedParts];
  }
  // w2 row pieces: the first kCodedBParts - 1 equal, the last short (~1/8 of w2), since only
  // the last is decoded and reduced after a step's final byte lands
  int coded_head_rows() const { return dpad * 7 / 24 / 32 * 32; }
  int coded_piece_row0(int p) const { return (p - 1) * coded_head_rows(); }  // p = 1..kCodedBParts
  int coded_piece_rows(int p) const {
    return p < kCodedBParts ? coded_head_rows() : dpad - (kCodedBParts - 1) * coded_head_rows();
  }
  // decoded bytes of part p and its offset in the expert block
  long long coded_part_out_off(int p) const {
    const long long a = 2ll * f * dpad * 2;
    return p == 0 ? 0 : a + 1ll * coded_piece_row0(p) * f * 2;
  }
  char* cstore = nullptr;                 // pinned host (private) or a registered shared segment
  bool cstore_external = false;
  bool coded_only = false;                // compress = 2: no raw store after encoding
  bool cstore_registered = false;
  uint64_t coded_total = 0;
  std::vector<CPart> ctab;                // [(SL * E + e) * 2 + part]
  char* cstage = nullptr;                 // HBM landing slots: [K][expert_bytes]
  std::vector<cudaEvent_t> cstage_free;   // per slot: decoded (slot may be overwritten)
  char* pzone = nullptr;                  // prefetch landing zones [NZ][pzone_bytes]
  long long pzone_bytes = 0;
  std::vector<cudaEvent_t> pzone_free;    // per zone: decoded
  int pzone_next = 0;
  const char* store_dev = nullptr;  // device view of the store (SM transfer)
  bool sm_transfer = false;
  // token graph (SM transfer): one token captured once, replayed per token
  bool no_graph = getenv("MOE_NO_GRAPH") != nullptr;
  bool no_pdl = getenv("MOE_NO_PDL") != nullptr;
  bool no_l2_prefetch = getenv("MOE_NO_L2_PREFETCH") != nullptr;   // A/B: mixing-matrix prefetch off
  bool no_split_down = getenv("MOE_NO_SPLIT_DOWN") != nullptr;     // A/B: last miss's down in one launch
  bool no_fused_gate = getenv("MOE_NO_FUSED_GATE") != nullptr;  // A/B: separate gate launch
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_kernels = 0;
  cudaStream_t cap_stream = nullptr;
  long long* cursor = nullptr;        // absolute index of the token the graph processes next
  StepRecord* cur_rec = nullptr;      // [L] records of the token in flight
  float *x_cur = nullptr, *out_cur = nullptr;       // [D]
  float *x_stage = nullptr, *out_stage = nullptr;   // [max_tokens][D] rings
  cudaStream_t copy_stream = nullptr;

  // forwarder state (driven by the thread calling decode)
  long long next_mail = 0;    // first mail seq not yet forwarded
  long long tokens_done = 0;  // absolute tokens enqueued
  std::deque<PrefetchJob> jobs;
  std::deque<cudaEvent_t> prefetch_inflight;  // one event per prefetch chunk in flight
  std::vector<cudaEvent_t> sync_events;       // free list (timing disabled)
  std::vector<cudaEvent_t> order_events;      // ring of events ordering phase 1 after copies
  size_t order_next = 0;
  std::mutex stats_mu;
  moe_stats st{};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> busy_events;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> free_events;
  bool debug = getenv("MOE_DEBUG") != nullptr;
  unsigned long long* gate_phase_ns = nullptr;  // MOE_GATE_TIMING: per-phase gate kernel time
  // MOE_TIMELINE=<csv>: per copy-engine step, copy-stream and compute-stream events plus host
  // times, written at destroy (diagnostics: where the link idles between steps)
  struct TimelineRec {
    long long seq;
    int layer, n_demand;
    cudaEvent_t copy0, copy1, gate, done;
    long long host_mail_ns, host_issued_ns;
  };
  const char* timeline_path = getenv("MOE_TIMELINE");
  std::vector<TimelineRec> timeline;
  cudaEvent_t timeline_base = nullptr;
  int cap_C = 0;  // policy slots allocated per layer (set_mode may use fewer)
  void* ext_store = nullptr;  // caller-provided expert store (shared between replicas)
  int64_t ext_store_bytes = 0;

  // kernel profiling (moe_engine_profile): per-layer event sextets, resolved lazily
  bool profiling = false;
  std::vector<cudaEvent_t> prof_free;
  std::vector<std::array<cudaEvent_t, 3>> prof_pending;  // before mix, after mix, after gate
  std::vector<std::array<cudaEvent_t, 2>> prof_ffn;      // around each expert-FFN launch group
  long long* prof_bytes_dev = nullptr;                    // per FFN launch: bytes streamed
  std::vector<std::array<cudaEvent_t, 2>> prof_dec;      // around each exponent-decode launch
  std::vector<long long> prof_dec_bytes;                 // its algorithmic bytes
  long long* prof_dec_dev = nullptr;                     // its in-kernel span slots [2]
  static constexpr int kProfSlots = 1 << 16;
  std::vector<std::array<cudaEvent_t, 2>> prof_final;
  std::vector<int> prof_pending_k;
  moe_kernel_times ktimes{};

  // batched prefill (prefill.cu), allocated on first use
  moe::PrefillState* pf = nullptr;

  // NVLink peer-HBM tier (moe_engine_attach_peer_tier): raw expert blocks by [l * E + e]
  std::vector<const char*> peer;
  const char* peer_block(int layer, int expert) const {
    return peer.empty() ? nullptr : peer[static_cast<size_t>(layer) * cfg.num_experts + expert];
  }

  // host block of expert e of layer l (store layers alias modulo SL)
  char* store_block(int layer, int expert) const {
    return store.base + (static_cast<long long>(layer % SL) * cfg.num_experts + expert) * expert_bytes;
  }
  const char* store_block_dev(int layer, int expert) const {
    return store_dev + (static_cast<long long>(layer % SL) * cfg.num_experts + expert) * expert_bytes;
  }
};

