// Host runtime of the offload decode engine: weights in pinned host DRAM, a fixed-size
// per-layer expert cache in HBM, and a forwarder that hands the device's load decisions to
// the copy engine.
//
// Per (token t, layer l), on the caller's compute stream:
//   mix_kernel        h_in -> h' = h_in + alpha * M h_in                 (toymoe.py:140)
//   gate_cache_kernel gate, softmax, top-k, guess, policy step, buffers  (toymoe.py:99-115,
//                     178-180; kernels.py:89-145) -> step record + mailbox entry
//   up/down (phase 0) experts that hit: run while the misses are in flight
//   [cudaStreamWaitEvent on the copy stream's event, only if the step has demand copies]
//   up/down (phase 1) experts that missed
// The calling thread runs in lockstep one layer behind the GPU: it polls the mailbox
// (mapped pinned memory) for the gate's decision, issues cudaMemcpyAsync of the missed
// expert blocks on the copy stream, and orders phase 1 after them with an event.  The
// host never chooses anything: the device picked the experts and the HBM buffers.
// (Cross-stream waits on memory flags -- cuStreamWaitValue or a spinning kernel -- were
// measured to stall copies queued behind them on this driver; every dependency here is
// CUDA-visible.)  While it waits for the next decision
// the thread trickles speculative-prefetch chunks onto the copy stream.
#include "hash.cuh"
#include "stream_gemv.cuh"

#include "engine_impl.h"

namespace {

#define TRY(x)                     \
  do {                             \
    moe_status _s = (x);           \
    if (_s != MOE_OK) return _s;   \
  } while (0)

moe_status create_resources(moe_engine* g);

// Raw bytes [off, off + n) of (layer, expert) into buffer `buf`: from the peer-HBM tier when it
// holds the expert (device to device), else from the pinned host store (PCIe).
moe_status issue_copy(moe_engine* g, int layer, int buf, int expert, long long off, long long n) {
  char* dst = g->pool + (static_cast<long long>(layer) * g->NB + buf) * g->expert_bytes + off;
  if (const char* pb = g->peer_block(layer, expert)) {
    MOE_CUDA(cudaMemcpyAsync(dst, pb + off, n, cudaMemcpyDefault, g->copy_stream));
    return MOE_OK;
  }
  const char* src = g->store_block(layer, expert) + off;
  MOE_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, g->copy_stream));
  return MOE_OK;
}

std::pair<cudaEvent_t, cudaEvent_t> take_timing_events(moe_engine* g) {
  std::lock_guard<std::mutex> lk(g->stats_mu);
  if (!g->free_events.empty()) {
    auto e = g->free_events.back();
    g->free_events.pop_back();
    return e;
  }
  cudaEvent_t a = nullptr, b = nullptr;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  return {a, b};
}

cudaEvent_t take_sync_event(moe_engine* g) {
  if (!g->sync_events.empty()) {
    cudaEvent_t e = g->sync_events.back();
    g->sync_events.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

// Demand copy order and events of one step: misses in ascending expert id, each copied as
// part A (w1|w3 or the toy W1t) then part B (w2 / W2t), each part followed by an event the
// compute stream waits on before that expert's up / down kernel.
struct DemandPlan {
  int n = 0;
  cudaEvent_t ev_a[kMaxK], ev_b[kMaxK];
  // compressed transfer of miss k: decode the landing slot into the expert's buffer
  bool comp[kMaxK] = {};
  cudaEvent_t ev_part[kMaxK][moe_engine::kCodedParts] = {};  // coded: after part p landed
  const char* land[kMaxK] = {};      // where the coded parts landed (contiguous, in order)
  cudaEvent_t free_ev[kMaxK] = {};   // recorded once decoded: the landing area may be reused
  char* dst[kMaxK] = {};
  const moe_engine::CPart* part[kMaxK] = {};  // the expert's first coded part
};

cudaEvent_t next_order_event(moe_engine* g);

// Copy the coded bytes [from, total) of (layer, expert) to `land` on the copy stream with an
// event after each part boundary (ev[p] fires once part p has fully landed).
moe_status copy_coded(moe_engine* g, int layer, int expert, char* land, long long from,
                      cudaEvent_t* ev, long long* link) {
  const moe_engine::CPart* cp = g->coded_parts(layer, expert);
  long long end = 0;
  for (int p = 0; p < moe_engine::kCodedParts; ++p) {
    const long long a = end;
    end += static_cast<long long>(cp[p].size);
    const long long lo = std::max(from, a);
    if (lo < end) {
      MOE_CUDA(cudaMemcpyAsync(land + lo, g->cstore + cp[0].off + lo, end - lo, cudaMemcpyHostToDevice,
                               g->copy_stream));
      *link += end - lo;
    }
    ev[p] = next_order_event(g);
    MOE_CUDA(cudaEventRecord(ev[p], g->copy_stream));
  }
  return MOE_OK;
}

long long coded_total(const moe_engine* g, int layer, int expert) {
  const moe_engine::CPart* cp = g->coded_parts(layer, expert);
  long long t = 0;
  for (int p = 0; p < moe_engine::kCodedParts; ++p) t += static_cast<long long>(cp[p].size);
  return t;
}

long long part_a_bytes(const moe_engine* g) {
  return g->bf16 ? 2ll * g->f * g->dpad * 2 : static_cast<long long>(g->dpad) * g->dpad * 4;
}

cudaEvent_t next_order_event(moe_engine* g) {
  return g->order_events[g->order_next++ % g->order_events.size()];
}

// Forward one mailbox entry: cancels, demand copies, new prefetch jobs.
moe_status handle_mail(moe_engine* g, const MailRecord& m, DemandPlan* plan) {
  const long long chunk = g->cfg.chunk_bytes;
  const long long nchunks = (g->expert_bytes + chunk - 1) / chunk;
  const long long split = part_a_bytes(g);
  // cancelled staging buffers of this step's layer: stop issuing their remaining chunks
  for (int i = 0; i < m.n_cancel; ++i)
    for (auto& j : g->jobs)
      if (!j.cancelled && !j.adopted && j.layer == m.layer && j.buf == m.cancel_buf[i]) {
        j.cancelled = true;
        std::lock_guard<std::mutex> lk(g->stats_mu);
        g->st.prefetch_wasted_bytes += std::min(j.next_chunk * chunk, j.bytes);
      }
  // demand entries in ascending expert id (the order the phase-1 kernels enumerate misses)
  int order[kMaxK];
  for (int i = 0; i < m.n_demand; ++i) order[i] = i;
  std::sort(order, order + m.n_demand,
            [&](int x, int y) { return m.demand_expert[x] < m.demand_expert[y]; });
  long long demand = 0, link = 0, peer = 0;
  std::pair<cudaEvent_t, cudaEvent_t> tev{nullptr, nullptr};
  if (m.n_demand > 0) {
    tev = take_timing_events(g);
    MOE_CUDA(cudaEventRecord(tev.first, g->copy_stream));
  }
  plan->n = m.n_demand;
  for (int k = 0; k < m.n_demand; ++k) {
    const int i = order[k];
    const int e = m.demand_expert[i], b = m.demand_buf[i];
    long long from = 0;
    int zone = -1;
    if (m.demand_adopt[i]) {
      for (auto& j : g->jobs)
        if (!j.cancelled && !j.adopted && j.layer == m.layer && j.buf == b && j.expert == e) {
          j.adopted = true;
          from = std::min(j.next_chunk * chunk, j.bytes);
          zone = j.zone;
          break;
        }
      std::lock_guard<std::mutex> lk(g->stats_mu);
      g->st.prefetch_used += 1;
    }
    plan->comp[k] = false;
    const bool via_peer = g->peer_block(m.layer, e) != nullptr;
    if (zone >= 0 || (g->cstore && from == 0 && !via_peer)) {
      // exponent-coded: an adopted prefetch finishes the coded bytes in its zone, a fresh miss
      // lands in slot k (after that slot's previous decode); the compute stream decodes each
      // part into the expert's buffer as it lands
      char* land;
      if (zone >= 0) {
        land = g->pzone + static_cast<long long>(zone) * g->pzone_bytes;
        plan->free_ev[k] = g->pzone_free[zone];
      } else {
        land = g->cstage + static_cast<long long>(k) * g->expert_bytes;
        plan->free_ev[k] = g->cstage_free[k];
        MOE_CUDA(cudaStreamWaitEvent(g->copy_stream, g->cstage_free[k], 0));
      }
      const long long tot = coded_total(g, m.layer, e);
      TRY(copy_coded(g, m.layer, e, land, from, plan->ev_part[k], &link));
      plan->ev_a[k] = plan->ev_part[k][0];
      plan->ev_b[k] = plan->ev_part[k][moe_engine::kCodedParts - 1];
      plan->comp[k] = true;
      plan->land[k] = land;
      plan->dst[k] = g->pool + (static_cast<long long>(m.layer) * g->NB + b) * g->expert_bytes;
      plan->part[k] = g->coded_parts(m.layer, e);
      demand += g->expert_bytes - static_cast<long long>(static_cast<double>(from) / tot * g->expert_bytes);
      continue;
    }
    // part A: [from, split), then event; part B: [max(from, split), end), then event
    long long& over = via_peer ? peer : link;   // bytes over NVLink / over PCIe
    if (from < split) {
      TRY(issue_copy(g, m.layer, b, e, from, split - from));
      demand += split - from;
      over += split - from;
    }
    plan->ev_a[k] = next_order_event(g);
    MOE_CUDA(cudaEventRecord(plan->ev_a[k], g->copy_stream));
    const long long fb = std::max(from, split);
    if (fb < g->expert_bytes) {
      TRY(issue_copy(g, m.layer, b, e, fb, g->expert_bytes - fb));
      demand += g->expert_bytes - fb;
      over += g->expert_bytes - fb;
    }
    plan->ev_b[k] = next_order_event(g);
    MOE_CUDA(cudaEventRecord(plan->ev_b[k], g->copy_stream));
  }
  if (m.n_demand > 0) MOE_CUDA(cudaEventRecord(tev.second, g->copy_stream));
  for (int i = 0; i < m.n_prefetch; ++i) {
    PrefetchJob j{m.layer + 1, m.prefetch_buf[i], m.prefetch_expert[i], 0, nchunks, false, false};
    j.bytes = g->expert_bytes;
    j.peer = g->peer_block(j.layer, j.expert) != nullptr;
    if (g->pzone && !j.peer) {
      j.zone = g->pzone_next;
      g->pzone_next = (g->pzone_next + 1) % static_cast<int>(g->pzone_free.size());
      j.bytes = coded_total(g, m.layer + 1, j.expert);
      j.n_chunks = (j.bytes + chunk - 1) / chunk;
    }
    g->jobs.push_back(j);
  }
  std::lock_guard<std::mutex> lk(g->stats_mu);
  g->st.demand_bytes += demand;
  g->st.demand_link_bytes += link;
  g->st.h2d_bytes += link;
  g->st.peer_bytes += peer;
  g->st.prefetch_issued += m.n_prefetch;
  if (m.n_demand > 0) g->busy_events.push_back(tev);
  return MOE_OK;
}

// Fold completed demand-copy timing pairs into copy_busy_ms and recycle them.
void recycle_busy_events(moe_engine* g) {
  std::lock_guard<std::mutex> lk(g->stats_mu);
  size_t keep = 0;
  for (size_t i = 0; i < g->busy_events.size(); ++i) {
    auto e = g->busy_events[i];
    float ms = 0.f;
    if (keep == 0 && cudaEventQuery(e.second) == cudaSuccess &&
        cudaEventElapsedTime(&ms, e.first, e.second) == cudaSuccess) {
      g->st.copy_busy_ms += ms;
      g->free_events.push_back(e);
    } else {
      g->busy_events[keep++] = e;
    }
  }
  g->busy_events.resize(keep);
}

// Issue one chunk of the oldest live prefetch job if the in-flight budget allows.
moe_status pump_prefetch(moe_engine* g, bool* did) {
  *did = false;
  if (g->busy_events.size() > 16) recycle_busy_events(g);
  while (!g->prefetch_inflight.empty() &&
         cudaEventQuery(g->prefetch_inflight.front()) == cudaSuccess) {
    g->sync_events.push_back(g->prefetch_inflight.front());
    g->prefetch_inflight.pop_front();
  }
  while (!g->jobs.empty() &&
         (g->jobs.front().cancelled || g->jobs.front().adopted ||
          g->jobs.front().next_chunk >= g->jobs.front().n_chunks))
    g->jobs.pop_front();
  if (g->jobs.empty()) return MOE_OK;
  if (g->prefetch_inflight.size() >= static_cast<size_t>(g->cfg.prefetch_depth)) return MOE_OK;
  PrefetchJob& j = g->jobs.front();
  const long long chunk = g->cfg.chunk_bytes;
  const long long off = j.next_chunk * chunk, n = std::min(chunk, j.bytes - off);
  if (j.zone >= 0) {
    // coded bytes into the job's landing zone (after the zone's previous decode)
    if (j.next_chunk == 0) MOE_CUDA(cudaStreamWaitEvent(g->copy_stream, g->pzone_free[j.zone], 0));
    MOE_CUDA(cudaMemcpyAsync(g->pzone + static_cast<long long>(j.zone) * g->pzone_bytes + off,
                             g->cstore + g->coded_parts(j.layer, j.expert)[0].off + off, n,
                             cudaMemcpyHostToDevice, g->copy_stream));
  } else {
    moe_status s = issue_copy(g, j.layer, j.buf, j.expert, off, n);
    if (s != MOE_OK) return s;
  }
  j.next_chunk += 1;
  cudaEvent_t ev = take_sync_event(g);
  MOE_CUDA(cudaEventRecord(ev, g->copy_stream));
  g->prefetch_inflight.push_back(ev);
  std::lock_guard<std::mutex> lk(g->stats_mu);
  g->st.prefetch_bytes += n;
  (j.peer ? g->st.peer_bytes : g->st.h2d_bytes) += n;
  *did = true;
  return MOE_OK;
}

// Wait for the gate's mail of step `seq` (the GPU is at most one step ahead), pumping
// prefetch chunks meanwhile.  A stream that finished or failed without posting it is an
// error, never a hang.
moe_status await_mail(moe_engine* g, long long seq, cudaStream_t compute, MailRecord* out) {
  MailRecord& m = g->mail_h[seq % kMailRing];
  long long spins = 0;
  const auto t0 = std::chrono::steady_clock::now();
  while (m.ready != seq + 1) {
    bool did = false;
    TRY(pump_prefetch(g, &did));
    if (did) continue;
    if ((++spins & 1023) == 0) {
      const cudaError_t q = cudaStreamQuery(compute);
      if (q != cudaSuccess && q != cudaErrorNotReady) {
        set_error("compute stream failed while waiting for step %lld: %s", seq, cudaGetErrorString(q));
        return MOE_CUDA_ERROR;
      }
      if (q == cudaSuccess && m.ready != seq + 1) {
        std::atomic_thread_fence(std::memory_order_acquire);
        if (m.ready != seq + 1) {
          set_error("gate of step %lld finished without posting its decision", seq);
          return MOE_CUDA_ERROR;
        }
      }
      const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (waited > 120.0) {
        set_error("no gate decision for step %lld after %.0f s", seq, waited);
        return MOE_CUDA_ERROR;
      }
      if (spins > (1 << 16)) std::this_thread::yield();
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  memcpy(out, const_cast<MailRecord*>(&m), sizeof(MailRecord));
  return MOE_OK;
}

cudaEvent_t timeline_event(cudaStream_t s) {
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  cudaEventRecord(e, s);
  return e;
}

long long host_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

void write_timeline(moe_engine* g) {
  if (!g->timeline_path || g->timeline.empty()) return;
  cudaDeviceSynchronize();
  FILE* f = fopen(g->timeline_path, "w");
  if (f) {
    fprintf(f, "seq,layer,n_demand,copy_start_ms,copy_end_ms,gate_end_ms,layer_done_ms,host_issue_us\n");
    auto at = [&](cudaEvent_t e) {
      float ms = -1.f;
      if (e) cudaEventElapsedTime(&ms, g->timeline_base, e);
      return ms;
    };
    for (const auto& r : g->timeline)
      fprintf(f, "%lld,%d,%d,%.4f,%.4f,%.4f,%.4f,%.2f\n", r.seq, r.layer, r.n_demand, at(r.copy0),
              at(r.copy1), at(r.gate), at(r.done), (r.host_issued_ns - r.host_mail_ns) / 1e3);
    fclose(f);
  }
  for (auto& r : g->timeline)
    for (cudaEvent_t e : {r.copy0, r.copy1, r.gate, r.done})
      if (e) cudaEventDestroy(e);
  g->timeline.clear();
}

cudaEvent_t take_prof_event(moe_engine* g) {
  if (!g->prof_free.empty()) {
    cudaEvent_t e = g->prof_free.back();
    g->prof_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Fold every recorded event group into the running totals (caller synchronised).
void resolve_profile(moe_engine* g) {
  moe_kernel_times& k = g->ktimes;
  for (size_t i = 0; i < g->prof_pending.size(); ++i) {
    auto& e = g->prof_pending[i];
    k.mix_ms += elapsed(e[0], e[1]);
    k.gate_ms += elapsed(e[1], e[2]);
    k.mix_launches += 1;
    k.gate_launches += 1;
    k.ffn_expert_runs += g->prof_pending_k[i];
    for (int q = 0; q < 3; ++q) g->prof_free.push_back(e[q]);
  }
  std::vector<long long> slots(4 * g->prof_ffn.size(), 0);
  if (g->bf16 && g->prof_bytes_dev && !slots.empty()) {
    cudaMemcpy(slots.data(), g->prof_bytes_dev, sizeof(long long) * slots.size(),
               cudaMemcpyDeviceToHost);
    cudaMemset(g->prof_bytes_dev, 0, sizeof(long long) * slots.size());
  }
  std::vector<long long> bytes(g->prof_ffn.size(), 0);
  for (size_t i = 0; i < bytes.size(); ++i) bytes[i] = slots[4 * i];
  static const bool dump = getenv("MOE_PROF_DUMP") != nullptr;
  for (size_t i = 0; i < g->prof_ffn.size(); ++i) {
    auto& e = g->prof_ffn[i];
    const float ms = elapsed(e[0], e[1]);
    if (dump)
      fprintf(stderr, "[moe-prof] ffn %zu %.4f ms %lld B kernel %.4f ms\n", i, ms, (long long)bytes[i],
              slots.empty() ? 0.0 : (slots[4 * i + 2] - (0x7fffffffffffffffll - slots[4 * i + 1])) / 1e6);
    k.ffn_ms += ms;
    k.ffn_launches += 1;
    if (!g->bf16 || bytes[i] > 0) {
      k.ffn_active_ms += ms;
      k.ffn_active_bytes += bytes[i];
      k.ffn_active_launches += 1;
      const long long t0 = 0x7fffffffffffffffll - slots[4 * i + 1], t1 = slots[4 * i + 2];
      if (g->bf16 && slots[4 * i + 1] > 0 && t1 > t0) k.ffn_kernel_ms += (t1 - t0) / 1e6;
    }
    g->prof_free.push_back(e[0]);
    g->prof_free.push_back(e[1]);
  }
  g->prof_ffn.clear();
  if (!g->prof_dec.empty()) {
    std::vector<long long> ds(2 * g->prof_dec.size(), 0);
    if (g->prof_dec_dev) {
      cudaMemcpy(ds.data(), g->prof_dec_dev, sizeof(long long) * ds.size(), cudaMemcpyDeviceToHost);
      cudaMemset(g->prof_dec_dev, 0, sizeof(long long) * ds.size());
    }
    for (size_t i = 0; i < g->prof_dec.size(); ++i) {
      auto& e = g->prof_dec[i];
      k.xdec_ms += elapsed(e[0], e[1]);
      k.xdec_bytes += g->prof_dec_bytes[i];
      k.xdec_launches += 1;
      const long long t0 = 0x7fffffffffffffffll - ds[2 * i], t1 = ds[2 * i + 1];
      if (ds[2 * i] > 0 && t1 > t0) k.xdec_kernel_ms += (t1 - t0) / 1e6;
      g->prof_free.push_back(e[0]);
      g->prof_free.push_back(e[1]);
    }
    g->prof_dec.clear();
    g->prof_dec_bytes.clear();
  }
  for (auto& e : g->prof_final) {
    k.finalize_ms += elapsed(e[0], e[1]);
    k.finalize_launches += 1;
    g->prof_free.push_back(e[0]);
    g->prof_free.push_back(e[1]);
  }
  g->prof_pending.clear();
  g->prof_pending_k.clear();
  g->prof_final.clear();
}

moe_status alloc_device(void** p, size_t n) {
  MOE_CUDA(cudaMalloc(p, n));
  MOE_CUDA(cudaMemset(*p, 0, n));
  return MOE_OK;
}

int round8(int x) { return (x + 7) / 8 * 8; }

}  // namespace

namespace {
// The exponent-coded store (compress = 1): a table of parts [(SL * E + e) * 2 + part] and the
// parts themselves, either in a private pinned buffer or in a caller's (node-shared) segment:
//   CodedSegHeader | CodedEntry[n] | parts (16-byte aligned)
struct CodedSegHeader {
  uint64_t magic, n_entries, data_off, total;
};
struct CodedEntry {
  uint64_t off, size;  // relative to the segment base
  xc::PartHeader hdr;
};
constexpr uint64_t kCodedMagic = 0x4d4f45584332ull;  // "MOEXC2"

// Sizes of every part from the raw store (the layout of a coded segment).  Parts of an expert:
// w1|w3, then kCodedBParts row pieces of w2 (the last short), contiguous.
void part_span(const moe_engine* g, int part, long long* first, long long* n) {
  const long long na = 2ll * g->f * g->dpad;
  *first = part == 0 ? 0 : na + 1ll * g->coded_piece_row0(part) * g->f;
  *n = part == 0 ? na : 1ll * g->coded_piece_rows(part) * g->f;
}

// Raw bf16 words of expert e of a layer whose blocks start at `raw_layer` ([E][expert]).
inline const uint16_t* raw_words(const moe_engine* g, const char* raw_layer, int e) {
  return reinterpret_cast<const uint16_t*>(raw_layer + static_cast<long long>(e) * g->expert_bytes);
}

// Sizes of one layer's parts (offsets assigned in order from *off).
void plan_layer(moe_engine* g, int l, const char* raw_layer, uint64_t* off) {
  const int E = g->cfg.num_experts, NP = moe_engine::kCodedParts;
  for (int e = 0; e < E; ++e)
    for (int part = 0; part < NP; ++part) {
      long long first, cnt;
      part_span(g, part, &first, &cnt);
      auto& c = g->ctab[(static_cast<size_t>(l) * E + e) * NP + part];
      c.off = *off;
      c.size = xc::encoded_size(raw_words(g, raw_layer, e) + first, cnt, 0);
      *off += c.size;
    }
}

void encode_layer(moe_engine* g, int l, const char* raw_layer, char* seg) {
  const int E = g->cfg.num_experts, NP = moe_engine::kCodedParts;
  for (int e = 0; e < E; ++e)
    for (int part = 0; part < NP; ++part) {
      long long first, cnt;
      part_span(g, part, &first, &cnt);
      auto& c = g->ctab[(static_cast<size_t>(l) * E + e) * NP + part];
      xc::encode(raw_words(g, raw_layer, e) + first, cnt, 0, reinterpret_cast<uint8_t*>(seg + c.off));
      memcpy(&c.hdr, seg + c.off, sizeof(c.hdr));
    }
}

void write_seg_table(moe_engine* g, char* seg) {
  CodedSegHeader h{kCodedMagic, g->ctab.size(), 0, g->coded_total};
  h.data_off = xc::align16(sizeof(CodedSegHeader) + sizeof(CodedEntry) * g->ctab.size());
  memcpy(seg, &h, sizeof(h));
  CodedEntry* ent = reinterpret_cast<CodedEntry*>(seg + sizeof(CodedSegHeader));
  for (size_t i = 0; i < g->ctab.size(); ++i) ent[i] = CodedEntry{g->ctab[i].off, g->ctab[i].size, g->ctab[i].hdr};
}

moe_status plan_coded(moe_engine* g) {
  MOE_REQUIRE(g->coded_head_rows() >= 32 && g->coded_piece_rows(moe_engine::kCodedBParts) >= 32,
              "compressed transfers need hidden_dim >= 256");
  MOE_REQUIRE(!g->coded_only, "a coded-only engine has no raw store to plan from");
  const int E = g->cfg.num_experts, NP = moe_engine::kCodedParts;
  const size_t n = static_cast<size_t>(g->SL) * E * NP;
  g->ctab.assign(n, moe_engine::CPart{});
  uint64_t off = xc::align16(sizeof(CodedSegHeader) + sizeof(CodedEntry) * n);
  for (int l = 0; l < g->SL; ++l) plan_layer(g, l, g->store_block(l, 0), &off);
  g->coded_total = off;
  return MOE_OK;
}

// Encode the planned parts into `seg` (host) and write its table.
void encode_coded(moe_engine* g, char* seg) {
  for (int l = 0; l < g->SL; ++l) encode_layer(g, l, g->store_block(l, 0), seg);
  write_seg_table(g, seg);
}

// HBM landing slots for demand misses (K) and prefetch zones (2K when prefetch is on).
moe_status alloc_landing(moe_engine* g) {
  if (!g->cstage) {
    const int slots = std::max(g->cfg.top_k, 1);
    MOE_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->cstage), static_cast<size_t>(slots) * g->expert_bytes));
    for (int i = 0; i < slots; ++i) {
      cudaEvent_t ev = nullptr;
      MOE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      g->cstage_free.push_back(ev);
    }
  }
  if (g->S > 0 && !g->pzone) {
    uint64_t mx = 0;
    for (size_t i = 0; i < g->ctab.size(); i += moe_engine::kCodedParts) {
      uint64_t t = 0;
      for (int q = 0; q < moe_engine::kCodedParts; ++q) t += g->ctab[i + q].size;
      mx = std::max<uint64_t>(mx, t);
    }
    g->pzone_bytes = static_cast<long long>(xc::align16(mx));
    const int zones = 2 * g->cfg.top_k;
    MOE_CUDA(cudaMalloc(reinterpret_cast<void**>(&g->pzone), static_cast<size_t>(zones) * g->pzone_bytes));
    for (int i = 0; i < zones; ++i) {
      cudaEvent_t ev = nullptr;
      MOE_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      g->pzone_free.push_back(ev);
    }
  }
  return MOE_OK;
}

// Private coded store: plan, pinned allocation, encode, landing buffers.
moe_status build_compressed_store(moe_engine* g) {
  if (g->cstore && !g->cstore_external) cudaFreeHost(g->cstore);
  g->cstore = nullptr;
  TRY(plan_coded(g));
  MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->cstore), g->coded_total, cudaHostAllocPortable));
  g->cstore_external = false;
  encode_coded(g, g->cstore);
  TRY(alloc_landing(g));
  g->st.compressed_store_bytes = static_cast<int64_t>(g->coded_total);
  return MOE_OK;
}
}  // namespace

namespace {
// <<<grid, block, smem, s>>> with programmatic stream serialization when `pdl` (the kernel may
// launch while its predecessor runs; every kernel of such a chain pdl_wait()s first)
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...);
}
}  // namespace

extern "C" {

moe_status moe_engine_create(const moe_engine_config* cfg_in, moe_engine** out) {
  return moe_engine_create_ex(cfg_in, nullptr, 0, out);
}

moe_status moe_engine_create_ex(const moe_engine_config* cfg_in, void* store, int64_t store_bytes,
                                moe_engine** out) {
  MOE_REQUIRE(cfg_in && out, "null argument");
  const moe_engine_config& c = *cfg_in;
  MOE_REQUIRE(c.num_layers >= 1, "num_layers must be >= 1, got %d", c.num_layers);
  MOE_REQUIRE(c.num_experts >= 1 && c.num_experts <= kMaxE,
              "the live engine supports 1..%d experts per layer, got %d", kMaxE, c.num_experts);
  MOE_REQUIRE(c.top_k >= 1 && c.top_k <= c.num_experts && c.top_k <= kMaxK,
              "top_k must be in [1, min(E, %d)], got %d", kMaxK, c.top_k);
  MOE_REQUIRE(c.cache_size >= c.top_k,
              "top_k=%d experts per step cannot fit in cache_size=%d", c.top_k, c.cache_size);
  MOE_REQUIRE(c.hidden_dim >= 1, "hidden_dim must be >= 1, got %d", c.hidden_dim);
  MOE_REQUIRE(c.expert_kind == MOE_EXPERT_TOY_TANH_F32 || c.expert_kind == MOE_EXPERT_SWIGLU_BF16,
              "unknown expert kind %d", c.expert_kind);
  MOE_REQUIRE(c.policy == MOE_P_LRU || c.policy == MOE_P_LFU || c.policy == MOE_P_LFU_AGED,
              "the live engine runs lru/lfu/lfu-aged; opt needs the future and is offline-only");
  MOE_REQUIRE(c.policy != MOE_P_LFU_AGED || (c.decay_period >= 1 && c.decay_factor > 0.0 &&
                                              c.decay_factor <= 1.0),
              "bad lfu-aged parameters");
  MOE_REQUIRE(c.mixing_scale >= 0.f, "mixing_scale must be >= 0");
  MOE_REQUIRE(c.prefetch == MOE_PREFETCH_OFF || c.prefetch == MOE_PREFETCH_EARLY,
              "unknown prefetch mode %d", c.prefetch);
  MOE_REQUIRE(c.max_tokens >= 1, "max_tokens must be >= 1");
  MOE_REQUIRE(c.rms_norm == 0 || (c.rms_norm == 1 && c.rms_eps > 0.f), "bad rms_norm settings");
  MOE_REQUIRE(c.expert_kind != MOE_EXPERT_SWIGLU_BF16 ||
                  (c.hidden_dim % 8 == 0 && c.ffn_dim >= 8 && c.ffn_dim % 8 == 0),
              "SwiGLU experts need hidden_dim and ffn_dim multiples of 8");
  MOE_REQUIRE(c.store_layers >= 0, "store_layers must be >= 0");
  MOE_REQUIRE(c.transfer >= MOE_TRANSFER_AUTO && c.transfer <= MOE_TRANSFER_SM,
              "unknown transfer mode %d", c.transfer);
  MOE_REQUIRE(!(c.transfer == MOE_TRANSFER_SM && c.prefetch),
              "speculative prefetch runs on the copy engine (transfer=SM has no staging path)");
  MOE_REQUIRE(c.prefetch_buffers >= 0, "prefetch_buffers must be >= 0");
  MOE_REQUIRE(c.compress >= 0 && c.compress <= 2, "compress must be 0, 1 or 2");
  MOE_REQUIRE(c.compress != 2 || !store, "a coded-only engine owns its store (no shared raw store)");
  MOE_REQUIRE(!c.compress || c.expert_kind == MOE_EXPERT_SWIGLU_BF16,
              "compressed transfers code bf16 experts (SwiGLU engines)");
  MOE_REQUIRE(!c.compress || c.transfer != MOE_TRANSFER_SM,
              "compressed transfers run on the copy engine (transfer=SM reads the raw store)");
  MOE_REQUIRE(c.cache_size + (c.prefetch ? c.top_k : 0) <= kMaxBuf,
              "cache_size + staging buffers must be <= %d", kMaxBuf);

  auto* g = new moe_engine();
  g->cfg = c;
  if (g->cfg.chunk_bytes <= 0) g->cfg.chunk_bytes = 4ll << 20;
  if (g->cfg.prefetch_depth <= 0) g->cfg.prefetch_depth = 2;
  g->device = c.device;
  g->d = c.hidden_dim;
  g->bf16 = c.expert_kind == MOE_EXPERT_SWIGLU_BF16;
  if (g->bf16) {
    g->dpad = c.hidden_dim;
    g->f = c.ffn_dim;
    g->expert_bytes = 3ll * g->f * g->dpad * 2;
  } else {
    g->dpad = round8(c.hidden_dim);
    g->f = g->dpad;
    g->expert_bytes = 2ll * g->dpad * g->dpad * 4;
  }
  g->coded_only = c.compress == 2;
  g->sm_transfer = c.transfer == MOE_TRANSFER_SM ||
                   (c.transfer == MOE_TRANSFER_AUTO && !c.prefetch && !c.compress &&
                    g->expert_bytes <= (16ll << 20));
  g->S = c.prefetch ? (c.prefetch_buffers > 0 ? std::min(c.prefetch_buffers, c.top_k) : c.top_k) : 0;
  g->SL = c.store_layers > 0 ? std::min(c.store_layers, c.num_layers) : c.num_layers;
  g->NB = c.cache_size + g->S;
  g->cap_C = c.cache_size;
  g->ext_store = store;
  g->ext_store_bytes = store_bytes;
  const moe_status st = create_resources(g);
  if (st != MOE_OK) {
    const std::string msg = moe_last_error();
    moe_engine_destroy(g);
    set_error("%s", msg.c_str());
    return st;
  }
  *out = g;
  return MOE_OK;
}

}  // extern "C"

namespace {
moe_status create_resources(moe_engine* g) {
  const moe_engine_config& c = g->cfg;
  const int L = c.num_layers, E = c.num_experts, K = c.top_k, D = g->dpad;
  MOE_ON_DEVICE(g->device);
  const size_t msz = g->bf16 ? 2 : 4;
  TRY(alloc_device(reinterpret_cast<void**>(&g->pool), static_cast<size_t>(L) * g->NB * g->expert_bytes));
  TRY(alloc_device(&g->mixing, static_cast<size_t>(L) * D * D * msz));
  TRY(alloc_device(reinterpret_cast<void**>(&g->gate_w), sizeof(float) * L * E * D));
  TRY(alloc_device(reinterpret_cast<void**>(&g->gate_b), sizeof(float) * L * E));
  TRY(alloc_device(reinterpret_cast<void**>(&g->states), sizeof(LayerState) * L));
  TRY(alloc_device(reinterpret_cast<void**>(&g->ring), sizeof(StepRecord) * L * static_cast<size_t>(c.max_tokens)));
  TRY(alloc_device(reinterpret_cast<void**>(&g->h_in), sizeof(float) * D));
  TRY(alloc_device(reinterpret_cast<void**>(&g->h_mid), sizeof(float) * 2 * D));
  TRY(alloc_device(reinterpret_cast<void**>(&g->h_norm), sizeof(float) * D));
  TRY(alloc_device(reinterpret_cast<void**>(&g->gate_part), sizeof(float) * 148 * (3 * kMaxE + 2)));
  TRY(alloc_device(reinterpret_cast<void**>(&g->norm_scale), sizeof(float)));
  TRY(alloc_device(reinterpret_cast<void**>(&g->mix_ctr), sizeof(unsigned int)));
  MOE_CUDA(cudaMemset(g->mix_ctr, 0, sizeof(unsigned int)));
  TRY(alloc_device(reinterpret_cast<void**>(&g->y), sizeof(float) * K * D));
  TRY(alloc_device(reinterpret_cast<void**>(&g->act), sizeof(float) * K * g->f));
  TRY(alloc_device(reinterpret_cast<void**>(&g->err), sizeof(int)));
  TRY(alloc_device(reinterpret_cast<void**>(&g->dstats), sizeof(DeviceStats)));
  if (D != g->d) {
    TRY(alloc_device(reinterpret_cast<void**>(&g->x_pad), sizeof(float) * D));
    TRY(alloc_device(reinterpret_cast<void**>(&g->out_pad), sizeof(float) * D));
  }
  MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->mail_h), sizeof(MailRecord) * kMailRing,
                         cudaHostAllocMapped | cudaHostAllocPortable));
  memset(g->mail_h, 0, sizeof(MailRecord) * kMailRing);
  MOE_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->mail_d), g->mail_h, 0));
  MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->ctl_h), sizeof(HostControl),
                         cudaHostAllocMapped | cudaHostAllocPortable));
  memset(g->ctl_h, 0, sizeof(HostControl));
  MOE_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g->ctl_d), g->ctl_h, 0));
  MOE_CUDA(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));

  // every event the forwarder will need, created up front (no allocation on the hot path)
  for (int i = 0; i < 64; ++i) {
    cudaEvent_t e = nullptr;
    MOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g->sync_events.push_back(e);
  }
  for (int i = 0; i < 4 * kMaxK; ++i) {
    cudaEvent_t e = nullptr;
    MOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g->order_events.push_back(e);
  }
  for (int i = 0; i < 4 * c.num_layers; ++i) {
    cudaEvent_t a = nullptr, b = nullptr;
    MOE_CUDA(cudaEventCreate(&a));
    MOE_CUDA(cudaEventCreate(&b));
    g->free_events.push_back({a, b});
  }
  if (getenv("MOE_GATE_TIMING"))
    TRY(alloc_device(reinterpret_cast<void**>(&g->gate_phase_ns), 16 * sizeof(unsigned long long)));
  // coded-only engines keep one raw layer as the encoder's staging buffer
  const size_t store_bytes = static_cast<size_t>(g->coded_only ? 1 : g->SL) * E * g->expert_bytes;
  if (g->ext_store) {
    MOE_REQUIRE(static_cast<size_t>(g->ext_store_bytes) >= store_bytes,
                "external expert store holds %lld bytes, the model needs %zu",
                (long long)g->ext_store_bytes, store_bytes);
    TRY(g->store.attach(g->ext_store, store_bytes));
  } else {
    TRY(g->store.allocate(store_bytes));
  }
  {
    void* dp = nullptr;
    MOE_CUDA(cudaHostGetDevicePointer(&dp, g->store.base, 0));
    g->store_dev = static_cast<const char*>(dp);
  }
  reset_states_kernel<<<L, 64>>>(g->states, L, g->NB);
  MOE_LAUNCHED();
  MOE_CUDA(cudaDeviceSynchronize());
  g->st.expert_bytes = g->expert_bytes;
  return MOE_OK;
}
}  // namespace

extern "C" {

moe_status moe_engine_destroy(moe_engine* g) {
  if (!g) return MOE_OK;
  ::moe::DeviceGuard moe_device_guard_(g->device);
  cudaDeviceSynchronize();
  write_timeline(g);
  if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);
  for (auto& e : g->busy_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto& e : g->free_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto e : g->sync_events) cudaEventDestroy(e);
  for (auto e : g->prefetch_inflight) cudaEventDestroy(e);
  for (auto e : g->order_events) cudaEventDestroy(e);
  for (auto e : g->prof_free) cudaEventDestroy(e);
  for (auto& a : g->prof_pending)
    for (auto e : a) cudaEventDestroy(e);
  for (auto& a : g->prof_final)
    for (auto e : a) cudaEventDestroy(e);
  for (auto& a : g->prof_ffn)
    for (auto e : a) cudaEventDestroy(e);
  if (g->prof_bytes_dev) cudaFree(g->prof_bytes_dev);
  for (auto& a : g->prof_dec)
    for (auto e : a) cudaEventDestroy(e);
  if (g->prof_dec_dev) cudaFree(g->prof_dec_dev);
  if (g->pf) prefill_release(g->pf);
  if (g->cstore && !g->cstore_external) cudaFreeHost(g->cstore);
  if (g->cstore && g->cstore_external && g->cstore_registered) cudaHostUnregister(g->cstore);
  if (g->cstage) cudaFree(g->cstage);
  if (g->pzone) cudaFree(g->pzone);
  for (auto e : g->pzone_free) cudaEventDestroy(e);
  for (auto e : g->cstage_free) cudaEventDestroy(e);
  if (g->graph_exec) cudaGraphExecDestroy(g->graph_exec);
  if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
  for (void* p : {static_cast<void*>(g->cursor), static_cast<void*>(g->cur_rec), static_cast<void*>(g->x_cur),
                  static_cast<void*>(g->out_cur), static_cast<void*>(g->x_stage), static_cast<void*>(g->out_stage)})
    if (p) cudaFree(p);
  if (g->gate_phase_ns) {
    unsigned long long h[16] = {};
    cudaMemcpy(h, g->gate_phase_ns, sizeof(h), cudaMemcpyDeviceToHost);
    if (h[5] && h[6])
      fprintf(stderr, "[moe] fused mixing kernel (avg ns from its first CTA start): last CTA start "
              "%llu, last staging done %llu, last main loop done %llu, last partials done %llu\n",
              h[11] / h[5], h[12] / h[5], h[13] / h[5], h[14] / h[5]);
    if (h[5])
      fprintf(stderr, "[moe] gate kernel phases (avg ns over %llu): mix stream+partials (fused: "
              "first CTA start -> gate start) %llu, state+rms %llu, logits %llu, route+policy %llu, "
              "bookkeeping %llu, writeback+mail %llu\n", h[5], h[6] / h[5], h[0] / h[5],
              h[1] / h[5], h[2] / h[5], h[3] / h[5], h[4] / h[5]);
    cudaFree(g->gate_phase_ns);
  }
  void* dev[] = {g->pool, g->mixing, g->gate_w, g->gate_b, g->states, g->ring, g->h_in,
                 g->h_mid, g->h_norm, g->gate_part, g->norm_scale, g->y, g->act, g->err, g->dstats, g->x_pad, g->out_pad,
                 g->mix_ctr};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (g->mail_h) cudaFreeHost(g->mail_h);
  if (g->ctl_h) cudaFreeHost(g->ctl_h);
  if (g->copy_stream) cudaStreamDestroy(g->copy_stream);

  g->store.release();
  delete g;
  return MOE_OK;
}

moe_status moe_engine_set_dense_f32(moe_engine* g, int32_t layer, const float* mixing,
                                    const float* gate_w, const float* gate_b) {
  MOE_REQUIRE(g && layer >= 0 && layer < g->cfg.num_layers, "layer %d out of range", layer);
  MOE_REQUIRE(!g->bf16, "set_dense_f32 is for the f32 (toy) engine");
  MOE_ON_DEVICE(g->device);
  const int d = g->d, D = g->dpad, E = g->cfg.num_experts;
  // device layout: M_dev[j][i] = M_ref[i][j]; W_dev[e][i] = W_ref[i][e]; zero padding
  std::vector<float> mt(static_cast<size_t>(D) * D, 0.f), gw(static_cast<size_t>(E) * D, 0.f);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) mt[static_cast<size_t>(j) * D + i] = mixing[static_cast<size_t>(i) * d + j];
  for (int i = 0; i < d; ++i)
    for (int e = 0; e < E; ++e) gw[static_cast<size_t>(e) * D + i] = gate_w[static_cast<size_t>(i) * E + e];
  MOE_CUDA(cudaMemcpy(static_cast<float*>(g->mixing) + static_cast<size_t>(layer) * D * D, mt.data(),
                      sizeof(float) * mt.size(), cudaMemcpyHostToDevice));
  MOE_CUDA(cudaMemcpy(g->gate_w + static_cast<size_t>(layer) * E * D, gw.data(),
                      sizeof(float) * gw.size(), cudaMemcpyHostToDevice));
  std::vector<float> gb(E, 0.f);
  if (gate_b)
    for (int e = 0; e < E; ++e) gb[e] = gate_b[e];
  MOE_CUDA(cudaMemcpy(g->gate_b + static_cast<size_t>(layer) * E, gb.data(), sizeof(float) * E,
                      cudaMemcpyHostToDevice));
  return MOE_OK;
}

moe_status moe_engine_set_toy_expert_f32(moe_engine* g, int32_t layer, int32_t expert,
                                         const float* w1, const float* w2) {
  MOE_REQUIRE(g && layer >= 0 && layer < g->cfg.num_layers, "layer %d out of range", layer);
  MOE_REQUIRE(expert >= 0 && expert < g->cfg.num_experts, "expert %d out of range", expert);
  MOE_REQUIRE(!g->bf16, "set_toy_expert_f32 is for the toy engine");
  const int d = g->d, D = g->dpad;
  float* blk = reinterpret_cast<float*>(
      g->store_block(layer, expert));
  memset(blk, 0, g->expert_bytes);
  float* w1t = blk;
  float* w2t = blk + static_cast<size_t>(D) * D;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      w1t[static_cast<size_t>(j) * D + i] = w1[static_cast<size_t>(i) * d + j];
      w2t[static_cast<size_t>(j) * D + i] = w2[static_cast<size_t>(i) * d + j];
    }
  return MOE_OK;
}

moe_status moe_engine_init_random(moe_engine* g, uint64_t seed, float gate_bias_std,
                                  int32_t init_experts) {
  MOE_REQUIRE(g, "null engine");
  MOE_REQUIRE(g->bf16, "init_random synthesises Mixtral-shaped (SwiGLU bf16) weights");
  MOE_ON_DEVICE(g->device);
  const int L = g->cfg.num_layers, E = g->cfg.num_experts, d = g->d, f = g->f;
  cudaStream_t s = g->copy_stream;
  // std = float(1 / sqrt(n)) rounded once from double (the oracle uses the same rule)
  const float sd = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  const float sf = static_cast<float>(1.0 / std::sqrt(static_cast<double>(f)));
  for (int l = 0; l < L; ++l) {
    uint16_t* M = static_cast<uint16_t*>(g->mixing) + static_cast<size_t>(l) * d * d;
    TRY(launch_hash_bf16(seed, tensor_id(kTMixing, l, 0, 0), 1.f, 1ll * d * d, M, s));
    TRY(launch_hash_f32(seed, tensor_id(kTGateW, l, 0, 0), sd, 1ll * E * d,
                        g->gate_w + static_cast<size_t>(l) * E * d, s));
    TRY(launch_hash_f32(seed, tensor_id(kTGateB, l, 0, 0), gate_bias_std, E,
                        g->gate_b + static_cast<size_t>(l) * E, s));
  }
  // experts: generate into a free HBM buffer, then copy down into the pinned store (a
  // replica attached to a shared store leaves this to the store's owner)
  uint16_t* scratch = reinterpret_cast<uint16_t*>(g->pool);
  const long long fd = 1ll * f * d;
  if (g->coded_only && init_experts) {
    // no raw store: each layer is generated into a one-layer host staging buffer and coded;
    // two passes (sizes, then bytes) so the coded store is one exact pinned allocation
    auto gen_layer = [&](int l) -> moe_status {
      for (int e = 0; e < E; ++e) {
        TRY(launch_hash_bf16(seed, tensor_id(kTExpert, l, e, kMatW1), sd, fd, scratch, s));
        TRY(launch_hash_bf16(seed, tensor_id(kTExpert, l, e, kMatW3), sd, fd, scratch + fd, s));
        TRY(launch_hash_bf16(seed, tensor_id(kTExpert, l, e, kMatW2), sf, fd, scratch + 2 * fd, s));
        MOE_CUDA(cudaMemcpyAsync(g->store.base + static_cast<long long>(e) * g->expert_bytes, scratch,
                                 g->expert_bytes, cudaMemcpyDeviceToHost, s));
      }
      MOE_CUDA(cudaStreamSynchronize(s));
      return MOE_OK;
    };
    const int NP = moe_engine::kCodedParts;
    g->ctab.assign(static_cast<size_t>(g->SL) * E * NP, moe_engine::CPart{});
    uint64_t off = xc::align16(sizeof(CodedSegHeader) + sizeof(CodedEntry) * g->ctab.size());
    for (int l = 0; l < g->SL; ++l) {
      TRY(gen_layer(l));
      plan_layer(g, l, g->store.base, &off);
    }
    g->coded_total = off;
    if (g->cstore) cudaFreeHost(g->cstore);
    g->cstore = nullptr;
    MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g->cstore), g->coded_total, cudaHostAllocPortable));
    g->cstore_external = false;
    for (int l = 0; l < g->SL; ++l) {
      TRY(gen_layer(l));
      encode_layer(g, l, g->store.base, g->cstore);
    }
    write_seg_table(g, g->cstore);
    TRY(alloc_landing(g));
    g->st.compressed_store_bytes = static_cast<int64_t>(g->coded_total);
    return MOE_OK;
  }
  for (int l = 0; l < (init_experts ? g->SL : 0); ++l)
    for (int e = 0; e < E; ++e) {
      TRY(launch_hash_bf16(seed, tensor_id(kTExpert, l, e, kMatW1), sd, fd, scratch, s));
      TRY(launch_hash_bf16(seed, tensor_id(kTExpert, l, e, kMatW3), sd, fd, scratch + fd, s));
      TRY(launch_hash_bf16(seed, tensor_id(kTExpert, l, e, kMatW2), sf, fd, scratch + 2 * fd, s));
      MOE_CUDA(cudaMemcpyAsync(g->store_block(l, e),
                               scratch, g->expert_bytes, cudaMemcpyDeviceToHost, s));
    }
  MOE_CUDA(cudaStreamSynchronize(s));
  // a private store is coded here; replicas of a node-shared store attach a shared coded
  // segment instead (moe_engine_coded_size / moe_engine_attach_coded)
  if (g->cfg.compress && init_experts && !g->ext_store) TRY(build_compressed_store(g));
  return MOE_OK;
}

moe_status moe_engine_coded_size(moe_engine* g, int64_t* bytes) {
  MOE_REQUIRE(g && bytes, "null argument");
  MOE_REQUIRE(g->cfg.compress, "the engine was created with compress = 0");
  TRY(plan_coded(g));
  *bytes = static_cast<int64_t>(g->coded_total);
  return MOE_OK;
}

moe_status moe_engine_attach_coded(moe_engine* g, void* seg, int64_t seg_bytes, int32_t build) {
  MOE_REQUIRE(g && seg, "null argument");
  MOE_REQUIRE(g->cfg.compress, "the engine was created with compress = 0");
  MOE_ON_DEVICE(g->device);
  char* base = static_cast<char*>(seg);
  if (build) {
    if (g->ctab.empty()) TRY(plan_coded(g));
    MOE_REQUIRE(static_cast<uint64_t>(seg_bytes) >= g->coded_total, "coded segment holds %lld bytes, needs %llu",
                (long long)seg_bytes, (unsigned long long)g->coded_total);
    encode_coded(g, base);
  } else {
    CodedSegHeader h;
    memcpy(&h, base, sizeof(h));
    MOE_REQUIRE(h.magic == kCodedMagic &&
                    h.n_entries == static_cast<uint64_t>(g->SL) * g->cfg.num_experts * moe_engine::kCodedParts &&
                    h.total <= static_cast<uint64_t>(seg_bytes),
                "not a coded expert segment of this model");
    const CodedEntry* ent = reinterpret_cast<const CodedEntry*>(base + sizeof(CodedSegHeader));
    g->ctab.assign(h.n_entries, moe_engine::CPart{});
    for (size_t i = 0; i < h.n_entries; ++i) g->ctab[i] = moe_engine::CPart{ent[i].off, ent[i].size, ent[i].hdr};
    g->coded_total = h.total;
  }
  if (g->cstore && !g->cstore_external) cudaFreeHost(g->cstore);
  const cudaError_t re = cudaHostRegister(base, g->coded_total, cudaHostRegisterPortable);
  if (re == cudaErrorHostMemoryAlreadyRegistered) cudaGetLastError();  // another engine did
  else MOE_CUDA(re);
  g->cstore_registered = re == cudaSuccess;
  g->cstore = base;
  g->cstore_external = true;
  TRY(alloc_landing(g));
  g->st.compressed_store_bytes = static_cast<int64_t>(g->coded_total);
  return MOE_OK;
}

moe_status moe_engine_expert_host_ptr(moe_engine* g, int32_t layer, int32_t expert, void** ptr,
                                      int64_t* bytes) {
  MOE_REQUIRE(g && layer >= 0 && layer < g->cfg.num_layers && expert >= 0 &&
                  expert < g->cfg.num_experts,
              "expert (%d, %d) out of range", layer, expert);
  MOE_REQUIRE(!g->coded_only, "a coded-only engine keeps no raw expert blocks");
  *ptr = g->store_block(layer, expert);
  *bytes = g->expert_bytes;
  return MOE_OK;
}

moe_status moe_engine_dense_host(moe_engine* g, int32_t layer, void* mixing, float* gate_w,
                                 float* gate_b) {
  MOE_REQUIRE(g && layer >= 0 && layer < g->cfg.num_layers, "layer %d out of range", layer);
  MOE_ON_DEVICE(g->device);
  const int D = g->dpad, E = g->cfg.num_experts;
  const size_t msz = g->bf16 ? 2 : 4;
  if (mixing)
    MOE_CUDA(cudaMemcpy(mixing, static_cast<char*>(g->mixing) + static_cast<size_t>(layer) * D * D * msz,
                        static_cast<size_t>(D) * D * msz, cudaMemcpyDeviceToHost));
  if (gate_w)
    MOE_CUDA(cudaMemcpy(gate_w, g->gate_w + static_cast<size_t>(layer) * E * D,
                        sizeof(float) * E * D, cudaMemcpyDeviceToHost));
  if (gate_b)
    MOE_CUDA(cudaMemcpy(gate_b, g->gate_b + static_cast<size_t>(layer) * E, sizeof(float) * E,
                        cudaMemcpyDeviceToHost));
  return MOE_OK;
}

moe_status moe_engine_reset(moe_engine* g) {
  MOE_REQUIRE(g, "null engine");
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());
  MOE_CUDA(cudaStreamSynchronize(g->copy_stream));
  g->jobs.clear();
  reset_states_kernel<<<g->cfg.num_layers, 64>>>(g->states, g->cfg.num_layers, g->NB);
  MOE_LAUNCHED();
  MOE_CUDA(cudaMemset(g->err, 0, sizeof(int)));
  MOE_CUDA(cudaDeviceSynchronize());
  return MOE_OK;
}

moe_status moe_engine_decode(moe_engine* g, const float* h_in_dev, int64_t T, float* h_out_dev,
                             void* stream) {
  return moe_engine_decode_routed(g, h_in_dev, T, h_out_dev, nullptr, stream);
}

moe_status moe_engine_decode_routed(moe_engine* g, const float* h_in_dev, int64_t T,
                                    float* h_out_dev, const int32_t* routing_dev, void* stream) {
  MOE_REQUIRE(g, "null engine");
  MOE_REQUIRE(T >= 0, "negative token count");
  MOE_ON_DEVICE(g->device);
  cudaStream_t s = as_stream(stream);
  const moe_engine_config& c = g->cfg;
  const int L = c.num_layers, K = c.top_k, D = g->dpad, d = g->d;
  const size_t msz = g->bf16 ? 2 : 4;
  const int mix_grid = std::max(1, std::min(D / 8, 148 * 2));
  const size_t mix_smem = static_cast<size_t>(D) * 8;
  const int up_rows = g->bf16 ? g->f : D;
  const int up_grid = std::max(1, std::min(up_rows / 8, 148 * 2));
  const int down_grid = std::max(1, std::min(D / 8, 148));
  const size_t up_smem = static_cast<size_t>(D) * 4;
  const size_t down_smem = static_cast<size_t>(g->f) * 4;
  static std::atomic<uint64_t> attrs{0};
  once_per_device(attrs, [] {
    cudaFuncSetAttribute(mix_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(mix_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(swiglu_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(toy_up_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(down_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(down_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // one shared-memory carveout for every kernel of the step: switching the L1/shared split
    // between consecutive kernels drains the SMs (seen as ~20 us gaps around the FFN launches)
    if (!getenv("MOE_NO_CARVEOUT")) {
      const int mx = cudaSharedmemCarveoutMaxShared;
      cudaFuncSetAttribute(gate_cache_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(fetch_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(token_begin_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(token_end_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(set_cursor_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(mix_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(mix_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(swiglu_up_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(toy_up_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(down_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      cudaFuncSetAttribute(down_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, mx);
      set_stream_carveout(mx);
    }
  });
  MOE_REQUIRE(mix_smem <= 200 * 1024 && down_smem <= 200 * 1024, "hidden/ffn dims too large");
  // bf16 path: bulk-copy streaming GEMVs (stream_gemv.cuh)
  StreamGeom gmix{}, gup{}, gdown{};
  if (g->bf16) {
    // MIX rows per block: MOE_MIX_RPB (A/B; 0 = the default geometry)
    static const int mix_rpb = getenv("MOE_MIX_RPB") ? atoi(getenv("MOE_MIX_RPB")) : 0;
    static const int mix_kb = getenv("MOE_MIX_STAGE_KB") ? atoi(getenv("MOE_MIX_STAGE_KB")) : 0;
    gmix = stream_geometry(kModeMix, D, g->f, mix_kb * 1024, 6, mix_rpb);
    if (gmix.ncb == 0) gmix = stream_geometry(kModeMix, D, g->f);
    gup = stream_geometry(kModeUp, D, g->f);
    gdown = stream_geometry(kModeDown, D, g->f);
    MOE_REQUIRE(gmix.ncb && gup.ncb && gdown.ncb,
                "bf16 engine needs hidden_dim and ffn_dim multiples of 256");
  }
  const int grid_mix = stream_grid(1), grid_ffn = stream_grid(K);
  static_assert(148 <= kMaxParts, "the gate sums one partial per mixing CTA");
  // SM transfer runs a token as one kernel chain (no copy-event waits): launch it programmatically
  const bool pdl = g->sm_transfer && !g->no_pdl;
  // bf16 engines take the gate / cache step in the mixing GEMV's last CTA (one launch)
  const bool fused_gate = g->bf16 && !g->no_fused_gate;
  // copy-engine decode: the stream GEMVs launch programmatically (each overlaps its launch and
  // prologue with its predecessor's tail; MIX also streams its weights meanwhile)
  const bool pdl_stream = !g->sm_transfer && !g->no_pdl && fused_gate;
  // one expert-FFN launch group: phase 0 = hits, 1 = misses; only = -1 all, i = i-th miss
  if (g->profiling && !g->prof_bytes_dev)
    MOE_CUDA(cudaMalloc(&g->prof_bytes_dev, 4 * sizeof(long long) * moe_engine::kProfSlots));
  if (g->profiling && g->prof_ffn.empty())
    MOE_CUDA(cudaMemsetAsync(g->prof_bytes_dev, 0, 4 * sizeof(long long) * moe_engine::kProfSlots, s));
  auto prof_slot = [&]() -> long long* {
    if (!g->profiling || g->prof_ffn.size() >= static_cast<size_t>(moe_engine::kProfSlots)) return nullptr;
    return g->prof_bytes_dev + 4 * g->prof_ffn.size();
  };
  auto prof_begin = [&](std::array<cudaEvent_t, 2>& ev) -> moe_status {
    if (g->profiling) {
      if (g->prof_ffn.size() >= static_cast<size_t>(moe_engine::kProfSlots)) {
        MOE_CUDA(cudaStreamSynchronize(s));
        resolve_profile(g);
      }
      ev = {take_prof_event(g), take_prof_event(g)};
      MOE_CUDA(cudaEventRecord(ev[0], s));
    }
    return MOE_OK;
  };
  auto prof_end = [&](std::array<cudaEvent_t, 2>& ev) -> moe_status {
    if (g->profiling) {
      MOE_CUDA(cudaEventRecord(ev[1], s));
      g->prof_ffn.push_back(ev);
    }
    return MOE_OK;
  };
  // exponent decode of n coded parts in one launch, with an event pair and an in-kernel span
  // when profiling
  auto xdecode_n = [&](const char* const* src, const xc::PartHeader* h, char* const* dst, int n) -> moe_status {
    long long* slot = nullptr;
    std::array<cudaEvent_t, 2> ev{};
    if (g->profiling && g->prof_dec.size() < static_cast<size_t>(moe_engine::kProfSlots)) {
      if (!g->prof_dec_dev) {
        MOE_CUDA(cudaMalloc(&g->prof_dec_dev, 2 * sizeof(long long) * moe_engine::kProfSlots));
        MOE_CUDA(cudaMemset(g->prof_dec_dev, 0, 2 * sizeof(long long) * moe_engine::kProfSlots));
      }
      slot = g->prof_dec_dev + 2 * g->prof_dec.size();
      ev = {take_prof_event(g), take_prof_event(g)};
      MOE_CUDA(cudaEventRecord(ev[0], s));
    }
    const void* ps[xc::kMaxBatch];
    uint16_t* os[xc::kMaxBatch];
    long long bytes = 0;
    for (int i = 0; i < n; ++i) {
      ps[i] = src[i];
      os[i] = reinterpret_cast<uint16_t*>(dst[i]);
      bytes += static_cast<long long>(h[i].total) + static_cast<long long>(h[i].n) * 2;
    }
    TRY(xc::decode_batch(ps, h, os, n, s, slot));
    if (slot) {
      MOE_CUDA(cudaEventRecord(ev[1], s));
      g->prof_dec.push_back(ev);
      g->prof_dec_bytes.push_back(bytes);
    }
    return MOE_OK;
  };
  auto xdecode = [&](const char* src, const xc::PartHeader& h, char* dst) -> moe_status {
    return xdecode_n(&src, &h, &dst, 1);
  };
  auto launch_ffn = [&](FfnParams fp, int only) -> moe_status {
    if (g->bf16) {
      StreamParams sp{};
      sp.d = D;
      sp.f = g->f;
      sp.K = K;
      sp.xin = fp.h_mid;
      sp.xscale = c.rms_norm ? g->norm_scale : nullptr;
      sp.rec = fp.rec;
      sp.state = fp.state;
      sp.pool = fp.pool;
      sp.expert_bytes = fp.expert_bytes;
      sp.phase = fp.phase;
      sp.only = only;
      sp.act = fp.act;
      sp.yout = fp.y;
      sp.prof_bytes = prof_slot();
      const int grid = only >= 0 ? stream_grid(1) : grid_ffn;
      MOE_CUDA(launch_stream<kModeUp>(gup, grid, sp, s, pdl_stream));
      MOE_LAUNCHED();
      return MOE_OK;
    }
    MOE_CUDA(launch_k(pdl, toy_up_kernel, dim3(up_grid, K), dim3(256), up_smem, s, fp));
    MOE_LAUNCHED();
    return MOE_OK;
  };
  auto launch_down = [&](FfnParams fp, int only, int row_lo = 0, int row_hi = 0) -> moe_status {
    if (g->bf16) {
      StreamParams sp{};
      sp.row_lo = row_lo;
      sp.row_hi = row_hi;
      sp.d = D;
      sp.f = g->f;
      sp.K = K;
      sp.rec = fp.rec;
      sp.state = fp.state;
      sp.pool = fp.pool;
      sp.expert_bytes = fp.expert_bytes;
      sp.phase = fp.phase;
      sp.only = only;
      sp.act = fp.act;
      sp.yout = fp.y;
      sp.prof_bytes = prof_slot();
      const int grid = only >= 0 ? stream_grid(1) : grid_ffn;
      MOE_CUDA(launch_stream<kModeDown>(gdown, grid, sp, s, pdl_stream));
      MOE_LAUNCHED();
      return MOE_OK;
    }
    MOE_CUDA(launch_k(pdl, down_kernel<false>, dim3(down_grid, K), dim3(256), down_smem, s, fp));
    MOE_LAUNCHED();
    return MOE_OK;
  };
  // One token through all layers.  Graph mode (fixed = true): token-invariant pointers --
  // the input in x_cur, records in cur_rec, the output in out_cur -- so the sequence can be
  // captured once and replayed (token_begin / token_end move them to / from the rings).
  auto run_token = [&](long long tok, int64_t t, bool fixed) -> moe_status {
    StepRecord* trec = fixed ? g->cur_rec : g->ring + (tok % c.max_tokens) * L;
    const float* x = fixed ? g->x_cur : h_in_dev + t * d;
    if (!fixed && D != d) {
      MOE_CUDA(cudaMemcpyAsync(g->x_pad, x, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
      x = g->x_pad;
    }
    for (int l = 0; l < L; ++l) {
      const long long seq = tok * L + l;
      float* hm = g->h_mid + (l & 1) * D;
      const float* hm_prev = g->h_mid + ((l + 1) & 1) * D;
      MixParams mp{l == 0 ? x : nullptr, hm_prev, g->y, l == 0 ? nullptr : trec + (l - 1),
                   static_cast<char*>(g->mixing) + static_cast<size_t>(l) * D * D * msz,
                   c.mixing_scale, D, K, g->h_in, hm};
      GateParams gp{hm, g->h_in, g->gate_w, g->gate_b, l, L, c.num_experts, K, D, c.cache_size,
                    c.cache_size + (c.prefetch ? g->S : 0), c.policy, c.decay_factor, c.decay_period, c.record_speculation,
                    c.prefetch, c.renormalize, seq, g->states, trec + l,
                    g->sm_transfer ? nullptr : g->mail_d,
                    g->ctl_d, g->err, g->dstats, c.rms_norm, c.rms_eps, g->h_norm,
                    g->gate_phase_ns, g->bf16 ? g->gate_part : nullptr, grid_mix, g->norm_scale,
                    routing_dev ? routing_dev + (static_cast<size_t>(t) * L + l) * K : nullptr};
      std::array<cudaEvent_t, 3> pe{};
      if (g->profiling) {
        for (auto& e : pe) e = take_prof_event(g);
        MOE_CUDA(cudaEventRecord(pe[0], s));
      }
      if (g->bf16) {
        StreamParams sp{};
        sp.d = D;
        sp.f = g->f;
        sp.K = K;
        sp.x = mp.x;
        sp.prev_mid = mp.prev_mid;
        sp.y = mp.y;
        sp.prev = mp.prev;
        sp.M = static_cast<const uint16_t*>(mp.M);
        if (!g->no_l2_prefetch)   // layer l+1 (after the last layer: the next token's layer 0)
          sp.M_next = reinterpret_cast<const uint16_t*>(static_cast<char*>(g->mixing) +
                                                        static_cast<size_t>((l + 1) % L) * D * D * msz);
        sp.alpha = mp.alpha;
        sp.h_in = mp.h_in;
        sp.h_mid = mp.h_mid;
        sp.gate_w = g->gate_w + static_cast<size_t>(l) * c.num_experts * D;
        sp.gate_w_next = (c.prefetch == MOE_PREFETCH_EARLY && l + 1 < L)
                             ? g->gate_w + static_cast<size_t>(l + 1) * c.num_experts * D
                             : nullptr;
        sp.E = c.num_experts;
        sp.do_guess = c.record_speculation && l >= 1;
        sp.part = g->gate_part;
        sp.fuse_gate = fused_gate ? 1 : 0;
        sp.done_ctr = g->mix_ctr;
        sp.gate = gp;
        MOE_CUDA(launch_stream<kModeMix>(gmix, grid_mix, sp, s, pdl_stream));
      } else {
        MOE_CUDA(launch_k(pdl, mix_kernel<false>, dim3(mix_grid), dim3(256), mix_smem, s, mp));
      }
      MOE_LAUNCHED();
      if (g->profiling) MOE_CUDA(cudaEventRecord(pe[1], s));
      if (!fused_gate) {
        // programmatic launch: the gate's launch and state staging overlap the mixing tail
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(1);
        lc.blockDim = dim3(kGateThreads);
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = g->no_pdl ? 0 : 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        MOE_CUDA(cudaLaunchKernelEx(&lc, gate_cache_kernel, gp));
        MOE_LAUNCHED();
      }
      if (g->profiling) MOE_CUDA(cudaEventRecord(pe[2], s));
      const bool tl = g->timeline_path && !g->sm_transfer && !fixed;
      moe_engine::TimelineRec trc{};
      if (tl) {
        if (!g->timeline_base) g->timeline_base = timeline_event(s);
        trc.gate = timeline_event(s);
      }
      FfnParams fp{(c.rms_norm && !g->bf16) ? g->h_norm : hm, trec + l, g->states + l,
                   g->pool + static_cast<long long>(l) * g->NB * g->expert_bytes, g->expert_bytes,
                   D, g->f, K, 0, g->act, g->y, nullptr, nullptr};
      std::array<cudaEvent_t, 2> fev{};
      if (g->sm_transfer) {
        // device-driven: the SMs fetch the missed experts, then one FFN pass over all K.
        // Toy (f32) experts fuse the fetch into the FFN: a missed expert's rows are read from
        // the mapped store and written through to its buffer as they are used.
        if (!g->bf16) {
          fp.store = g->store_block_dev(l, 0);
          fp.stats = g->dstats;
        } else {
          FetchParams fp2{trec + l, g->states + l, g->store_block_dev(l, 0),
                          g->pool + static_cast<long long>(l) * g->NB * g->expert_bytes, g->expert_bytes,
                          K, g->dstats};
          const long long n16 = g->expert_bytes / 16;
          const int fgrid = static_cast<int>(std::max(1ll, std::min<long long>(296, (K * n16 + 4095) / 4096)));
          MOE_CUDA(launch_k(pdl, fetch_kernel, dim3(fgrid), dim3(512), 0, s, fp2));
          MOE_LAUNCHED();
        }
        fp.phase = 2;
        TRY(prof_begin(fev));
        TRY(launch_ffn(fp, -1));
        TRY(prof_end(fev));
        fp.store = nullptr;  // the up pass already brought both matrices of a missed toy expert
        TRY(prof_begin(fev));
        TRY(launch_down(fp, -1));
        TRY(prof_end(fev));
        if (g->profiling) {
          g->prof_pending.push_back(pe);
          g->prof_pending_k.push_back(K);
        }
        continue;
      }
      if (fixed) {
        set_error("graph capture of a copy-engine step");
        return MOE_INVALID_CONFIG;
      }
      // phase 0: experts that hit run while the misses are fetched
      TRY(prof_begin(fev));
      TRY(launch_ffn(fp, -1));
      TRY(prof_end(fev));
      TRY(prof_begin(fev));
      TRY(launch_down(fp, -1));
      TRY(prof_end(fev));
      // forward the device's decision for this step (lockstep, one step behind the GPU)
      MailRecord m;
      TRY(await_mail(g, seq, s, &m));
      if (tl) {
        trc.host_mail_ns = host_ns();
        trc.copy0 = timeline_event(g->copy_stream);
      }
      if (g->debug)
        fprintf(stderr, "[moe] seq=%lld layer=%d demand=%d cancel=%d prefetch=%d\n", m.seq,
                m.layer, m.n_demand, m.n_cancel, m.n_prefetch);
      DemandPlan plan;
      TRY(handle_mail(g, m, &plan));
      if (tl) {
        trc.host_issued_ns = host_ns();
        trc.copy1 = timeline_event(g->copy_stream);
        trc.seq = seq;
        trc.layer = l;
        trc.n_demand = m.n_demand;
      }
      g->next_mail = seq + 1;
      g->ctl_h->consumed = seq + 1;
      // phase 1: each missed expert's up runs once its w1|w3 landed (overlapping its w2
      // copy), its down once w2 landed (overlapping the next expert's copy)
      fp.phase = 1;
      if (g->bf16) {
        for (int i = 0; i < plan.n; ++i) {
          MOE_CUDA(cudaStreamWaitEvent(s, plan.ev_a[i], 0));
          long long coff = 0;
          if (plan.comp[i]) {
            TRY(xdecode(plan.land[i], plan.part[i][0].hdr, plan.dst[i]));
            coff = static_cast<long long>(plan.part[i][0].size);
          }
          TRY(prof_begin(fev));
          TRY(launch_ffn(fp, i));
          TRY(prof_end(fev));
          if (plan.comp[i]) {
            // w2 pieces 1..3 decode in one launch once the third has landed (overlapping the
            // last piece's copy), the last piece on its own after it lands
            const int NP = moe_engine::kCodedParts;
            const char* src[xc::kMaxBatch];
            char* dst[xc::kMaxBatch];
            xc::PartHeader hh[xc::kMaxBatch];
            int nb = 0;
            // the step's last miss reduces the rows of pieces 1..3 before the last piece
            // lands, so only the short piece's decode + rows trail the step's last byte
            const bool split = i == plan.n - 1 && !g->no_split_down;
            const int head = g->coded_piece_row0(NP - 1);
            for (int q = 1; q < NP; ++q) {
              MOE_CUDA(cudaStreamWaitEvent(s, plan.ev_part[i][q], 0));
              src[nb] = plan.land[i] + coff;
              dst[nb] = plan.dst[i] + g->coded_part_out_off(q);
              hh[nb] = plan.part[i][q].hdr;
              ++nb;
              coff += static_cast<long long>(plan.part[i][q].size);
              if (q == NP - 2 || q == NP - 1) {
                TRY(xdecode_n(src, hh, dst, nb));
                nb = 0;
              }
              if (split && q == NP - 2) {
                TRY(prof_begin(fev));
                TRY(launch_down(fp, i, 0, head));
                TRY(prof_end(fev));
              }
            }
            MOE_CUDA(cudaEventRecord(plan.free_ev[i], s));
            TRY(prof_begin(fev));
            if (split)
              TRY(launch_down(fp, i, head, D));
            else
              TRY(launch_down(fp, i));
            TRY(prof_end(fev));
            continue;
          }
          MOE_CUDA(cudaStreamWaitEvent(s, plan.ev_b[i], 0));
          TRY(prof_begin(fev));
          TRY(launch_down(fp, i));
          TRY(prof_end(fev));
        }
      } else if (plan.n > 0) {
        MOE_CUDA(cudaStreamWaitEvent(s, plan.ev_b[plan.n - 1], 0));
        TRY(prof_begin(fev));
        TRY(launch_ffn(fp, -1));
        TRY(prof_end(fev));
        TRY(prof_begin(fev));
        TRY(launch_down(fp, -1));
        TRY(prof_end(fev));
      }
      if (g->profiling) {
        g->prof_pending.push_back(pe);
        g->prof_pending_k.push_back(K);
      }
      if (tl) {
        trc.done = timeline_event(s);
        g->timeline.push_back(trc);
      }
    }
    float* out = fixed ? g->out_cur : h_out_dev + t * d;
    float* dst = (!fixed && D != d) ? g->out_pad : out;
    std::array<cudaEvent_t, 2> fe{};
    if (g->profiling) {
      fe = {take_prof_event(g), take_prof_event(g)};
      MOE_CUDA(cudaEventRecord(fe[0], s));
    }
    MOE_CUDA(launch_k(pdl, finalize_kernel, dim3((D + 255) / 256), dim3(256), 0, s,
                      static_cast<const float*>(g->h_mid + ((L - 1) & 1) * D),
                      static_cast<const float*>(g->y), static_cast<const StepRecord*>(trec + (L - 1)),
                      K, D, dst));
    MOE_LAUNCHED();
    if (g->profiling) {
      MOE_CUDA(cudaEventRecord(fe[1], s));
      g->prof_final.push_back(fe);
    }
    if (!fixed && D != d)
      MOE_CUDA(cudaMemcpyAsync(out, g->out_pad, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    return MOE_OK;
  };

  const bool graph = g->sm_transfer && !g->profiling && !routing_dev && !g->no_graph && T >= 1;
  if (graph && !g->cursor) {
    const size_t rows = static_cast<size_t>(c.max_tokens) * D;
    TRY(alloc_device(reinterpret_cast<void**>(&g->cursor), sizeof(long long)));
    TRY(alloc_device(reinterpret_cast<void**>(&g->cur_rec), sizeof(StepRecord) * L));
    TRY(alloc_device(reinterpret_cast<void**>(&g->x_cur), sizeof(float) * D));
    TRY(alloc_device(reinterpret_cast<void**>(&g->out_cur), sizeof(float) * D));
    TRY(alloc_device(reinterpret_cast<void**>(&g->x_stage), sizeof(float) * rows));
    TRY(alloc_device(reinterpret_cast<void**>(&g->out_stage), sizeof(float) * rows));
    MOE_CUDA(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
  }
  if (!graph) {
    for (int64_t t = 0; t < T; ++t) TRY(run_token(g->tokens_done + t, t, false));
  } else {
    if (!g->graph_exec) {
      // capture one token on a private stream; kernels counted per replay below
      const uint64_t n0 = launch_counter().load();
      cudaStream_t user = s;
      s = g->cap_stream;
      MOE_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      token_begin_kernel<<<1, 256, 0, s>>>(g->cursor, g->x_stage, c.max_tokens, D, g->x_cur);
      MOE_LAUNCHED();
      const moe_status st = run_token(0, 0, true);
      MOE_CUDA(launch_k(pdl, token_end_kernel, dim3(1), dim3(256), 0, s, g->cursor,
                        static_cast<const StepRecord*>(g->cur_rec), g->ring,
                        static_cast<const float*>(g->out_cur), g->out_stage, static_cast<int>(c.max_tokens), L, D));
      MOE_LAUNCHED();
      cudaGraph_t graph_obj = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(s, &graph_obj);
      s = user;
      if (st != MOE_OK) {
        if (graph_obj) cudaGraphDestroy(graph_obj);
        return st;
      }
      MOE_CUDA(ce);
      MOE_CUDA(cudaGraphInstantiate(&g->graph_exec, graph_obj, 0));
      cudaGraphDestroy(graph_obj);
      g->graph_kernels = launch_counter().load() - n0;
      launch_counter().fetch_sub(g->graph_kernels);
    }
    // per chunk of <= max_tokens tokens: stage the inputs into the ring rows, replay the token
    // graph once per token, collect the outputs from the ring rows
    const long long cap = c.max_tokens, t0 = g->tokens_done;
    set_cursor_kernel<<<1, 1, 0, s>>>(g->cursor, t0);
    MOE_LAUNCHED();
    for (long long done = 0; done < T;) {
      const long long chunk = std::min<long long>(T - done, cap);
      for (long long k = 0; k < chunk;) {
        const long long pos = (t0 + done + k) % cap, n = std::min<long long>(chunk - k, cap - pos);
        MOE_CUDA(cudaMemcpy2DAsync(g->x_stage + pos * D, sizeof(float) * D, h_in_dev + (done + k) * d,
                                   sizeof(float) * d, sizeof(float) * d, n, cudaMemcpyDeviceToDevice, s));
        k += n;
      }
      for (long long i = 0; i < chunk; ++i) MOE_CUDA(cudaGraphLaunch(g->graph_exec, s));
      launch_counter().fetch_add(g->graph_kernels * chunk);
      for (long long k = 0; k < chunk;) {
        const long long pos = (t0 + done + k) % cap, n = std::min<long long>(chunk - k, cap - pos);
        MOE_CUDA(cudaMemcpy2DAsync(h_out_dev + (done + k) * d, sizeof(float) * d, g->out_stage + pos * D,
                                   sizeof(float) * D, sizeof(float) * d, n, cudaMemcpyDeviceToDevice, s));
        k += n;
      }
      done += chunk;
    }
  }
  g->tokens_done += T;
  return MOE_OK;
}

moe_status moe_engine_sync(moe_engine* g) {
  MOE_REQUIRE(g, "null engine");
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());
  int h = 0;
  MOE_CUDA(cudaMemcpy(&h, g->err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) {
    MOE_CUDA(cudaMemset(g->err, 0, sizeof(int)));
    if (h & 1) {
      set_error("gate logits are not finite");
      return MOE_NONFINITE;
    }
    if (h & 4) {
      set_error("routed activations out of range or repeated within a step");
      return MOE_INVALID_CONFIG;
    }
    set_error("cache policy found no eviction candidate");
    return MOE_INVALID_CONFIG;
  }
  return MOE_OK;
}

moe_status moe_engine_records(moe_engine* g, int64_t t0, int64_t T, int64_t* acts,
                              int64_t* guessed, uint8_t* resident_before, uint8_t* evicted,
                              float* probs) {
  MOE_REQUIRE(g, "null engine");
  const moe_engine_config& c = g->cfg;
  MOE_REQUIRE(t0 >= 0 && T >= 0 && t0 + T <= g->tokens_done, "tokens [%lld, %lld) not decoded",
              (long long)t0, (long long)(t0 + T));
  MOE_REQUIRE(g->tokens_done - t0 <= c.max_tokens, "tokens [%lld, ...) left the record ring",
              (long long)t0);
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());
  const int L = c.num_layers, K = c.top_k, E = c.num_experts;
  std::vector<StepRecord> buf(static_cast<size_t>(L));
  for (int64_t t = 0; t < T; ++t) {
    const long long tok = t0 + t;
    MOE_CUDA(cudaMemcpy(buf.data(), g->ring + (tok % c.max_tokens) * L, sizeof(StepRecord) * L,
                        cudaMemcpyDeviceToHost));
    for (int l = 0; l < L; ++l) {
      const StepRecord& r = buf[l];
      for (int j = 0; j < K; ++j) {
        if (acts) acts[(t * L + l) * K + j] = r.acts[j];
        if (probs) probs[(t * L + l) * K + j] = r.prob[j];
        if (guessed && l >= 1) guessed[(t * (L - 1) + (l - 1)) * K + j] = r.guess[j];
      }
      for (int e = 0; e < E; ++e) {
        if (resident_before) resident_before[(t * L + l) * E + e] = (r.rb >> e) & 1u;
        if (evicted) evicted[(t * L + l) * E + e] = (r.ev >> e) & 1u;
      }
    }
  }
  return MOE_OK;
}

moe_status moe_engine_record_gaps(moe_engine* g, int64_t t0, int64_t T, float* gaps,
                                  float* guess_gaps, float* zscales, int64_t* early) {
  MOE_REQUIRE(g, "null engine");
  const moe_engine_config& c = g->cfg;
  MOE_REQUIRE(t0 >= 0 && T >= 0 && t0 + T <= g->tokens_done, "tokens [%lld, %lld) not decoded",
              (long long)t0, (long long)(t0 + T));
  MOE_REQUIRE(g->tokens_done - t0 <= c.max_tokens, "tokens [%lld, ...) left the record ring",
              (long long)t0);
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());
  const int L = c.num_layers;
  std::vector<StepRecord> buf(static_cast<size_t>(L));
  for (int64_t t = 0; t < T; ++t) {
    const long long tok = t0 + t;
    MOE_CUDA(cudaMemcpy(buf.data(), g->ring + (tok % c.max_tokens) * L, sizeof(StepRecord) * L,
                        cudaMemcpyDeviceToHost));
    for (int l = 0; l < L; ++l) {
      if (gaps) gaps[t * L + l] = buf[l].gap;
      if (guess_gaps && l >= 1) guess_gaps[t * (L - 1) + (l - 1)] = buf[l].guess_gap;
      if (zscales) {
        zscales[(t * L + l) * 2] = buf[l].zscale[0];
        zscales[(t * L + l) * 2 + 1] = buf[l].zscale[1];
      }
      if (early && l + 1 < L)
        for (int j = 0; j < c.top_k; ++j)
          early[(t * (L - 1) + l) * c.top_k + j] = buf[l].early[j];
    }
  }
  return MOE_OK;
}

moe_status moe_engine_set_mode(moe_engine* g, int32_t policy, double decay_factor,
                               int64_t decay_period, int32_t cache_size, int32_t prefetch) {
  MOE_REQUIRE(g, "null engine");
  MOE_REQUIRE(policy == MOE_P_LRU || policy == MOE_P_LFU || policy == MOE_P_LFU_AGED,
              "the live engine runs lru/lfu/lfu-aged; opt needs the future and is offline-only");
  MOE_REQUIRE(policy != MOE_P_LFU_AGED || (decay_period >= 1 && decay_factor > 0.0 &&
                                            decay_factor <= 1.0),
              "bad lfu-aged parameters");
  MOE_REQUIRE(cache_size >= g->cfg.top_k && cache_size <= g->cap_C,
              "cache_size must be in [top_k=%d, allocated %d], got %d", g->cfg.top_k, g->cap_C,
              cache_size);
  MOE_REQUIRE(prefetch == MOE_PREFETCH_OFF || (prefetch == MOE_PREFETCH_EARLY && g->S > 0),
              "prefetch needs staging buffers: create the engine with prefetch enabled");
  TRY(moe_engine_reset(g));
  if (g->graph_exec) {  // kernel parameters (policy, cache size) are baked into the graph
    cudaGraphExecDestroy(g->graph_exec);
    g->graph_exec = nullptr;
  }
  g->cfg.policy = policy;
  g->cfg.decay_factor = decay_factor;
  g->cfg.decay_period = decay_period;
  g->cfg.cache_size = cache_size;
  g->cfg.prefetch = prefetch;
  return MOE_OK;
}

moe_status moe_engine_profile(moe_engine* g, int32_t enable) {
  MOE_REQUIRE(g, "null engine");
  g->profiling = enable != 0;
  return MOE_OK;
}

moe_status moe_engine_kernel_times(moe_engine* g, moe_kernel_times* out) {
  MOE_REQUIRE(g && out, "null argument");
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());
  resolve_profile(g);
  *out = g->ktimes;
  return MOE_OK;
}

moe_status moe_engine_attach_peer_tier(moe_engine* g, const void* const* ptrs, int64_t n) {
  MOE_REQUIRE(g, "null engine");
  const moe_engine_config& c = g->cfg;
  if (!ptrs) {
    g->peer.clear();
    return MOE_OK;
  }
  MOE_REQUIRE(n == static_cast<int64_t>(c.num_layers) * c.num_experts,
              "peer tier table needs L * E = %d entries, got %lld", c.num_layers * c.num_experts,
              (long long)n);
  MOE_REQUIRE(!g->sm_transfer, "the peer tier serves the copy-engine transfer mode");
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());   // no copy of the previous source is in flight
  std::vector<const char*> t(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    t[i] = static_cast<const char*>(ptrs[i]);
    if (!t[i]) continue;
    cudaPointerAttributes a{};
    MOE_CUDA(cudaPointerGetAttributes(&a, t[i]));
    MOE_REQUIRE(a.type == cudaMemoryTypeDevice, "peer tier entry %lld is not device memory",
                (long long)i);
    if (a.device != g->device) {
      int ok = 0;
      MOE_CUDA(cudaDeviceCanAccessPeer(&ok, g->device, a.device));
      MOE_REQUIRE(ok, "GPU %d cannot access peer GPU %d", g->device, a.device);
      const cudaError_t e = cudaDeviceEnablePeerAccess(a.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else MOE_CUDA(e);
    }
  }
  g->peer.swap(t);
  return MOE_OK;
}

moe_status moe_engine_stats(moe_engine* g, moe_stats* out) {
  MOE_REQUIRE(g && out, "null argument");
  MOE_ON_DEVICE(g->device);
  MOE_CUDA(cudaDeviceSynchronize());
  MOE_CUDA(cudaStreamSynchronize(g->copy_stream));
  DeviceStats ds{};
  MOE_CUDA(cudaMemcpy(&ds, g->dstats, sizeof(ds), cudaMemcpyDeviceToHost));
  recycle_busy_events(g);
  std::lock_guard<std::mutex> lk(g->stats_mu);
  *out = g->st;
  out->hits = static_cast<int64_t>(ds.hits);
  out->misses = static_cast<int64_t>(ds.misses);
  out->demand_bytes += static_cast<int64_t>(ds.fetched_bytes);
  out->demand_link_bytes += static_cast<int64_t>(ds.fetched_bytes);
  out->h2d_bytes += static_cast<int64_t>(ds.fetched_bytes);
  out->tokens = g->tokens_done;
  out->steps = g->tokens_done * g->cfg.num_layers;
  out->expert_bytes = g->expert_bytes;
  return MOE_OK;
}

}  // extern "C"
