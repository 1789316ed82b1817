// Batched prefill (moe_engine_prefill): T independent tokens through every layer at once,
// the expert FFN and the mixing map on the tensor cores (tcgen05 grouped GEMM, tc_gemm.cuh).
//
// Per layer, on the caller's stream:
//   mix GEMM (T x d x d) -> gate (one warp per token) -> plan (policy replayed over the T steps
//   in token order, HBM buffer plan, grouping, tile tables, mailbox) -> gather (bf16 rows per
//   expert group) -> [host forwards one H2D copy per needed expert that is not resident] ->
//   up/down GEMMs of the resident experts, then per loaded expert after its copy events ->
//   scratch -> cache-buffer moves -> combine (next layer's input).
// Semantics equal T decode steps: the same step records, cache traces and final
// cache state; only the GEMM operand precision differs (bf16 activations).
#include "engine_impl.h"
#include "prefill_kernels.cuh"
#include "tc_gemm.h"

namespace moe {

struct PrefillState {
  int cap_T = 0;
  int max_up = 0, max_dn = 0;
  int splits = 1;              // split-K of the down projection (fills the SMs per expert)
  long long split_stride = 0;  // floats per split plane of y
  // activations
  float *x = nullptr, *hm = nullptr, *y = nullptr, *inv = nullptr;
  uint16_t *a_mix = nullptr, *an = nullptr, *act = nullptr;
  int *row_map = nullptr, *pos_of = nullptr;
  // plan outputs
  tc::Group *grp_up = nullptr, *grp_dn = nullptr, *grp_mix = nullptr;
  tc::Tile *tiles_up = nullptr, *tiles_dn = nullptr, *tiles_mix = nullptr;
  int *cnt_up = nullptr, *cnt_dn = nullptr, *cnt_mix = nullptr;
  int mix_T = -1;  // T the mix tile table was built for
  int mix_tiles_per_layer = 0;
  std::vector<tc::Tile> h_tiles_mix;
  std::vector<tc::Group> h_grp_mix;
  std::vector<int> h_cnt_mix;
  // scratch expert slots (one per expert id) for experts that are not (or not yet) cached
  char* scratch = nullptr;
  // mapped mailbox
  PrefillMail* mail_h = nullptr;
  PrefillMail* mail_d = nullptr;
  std::vector<cudaEvent_t> ev;  // copy-order events
  std::vector<void*> allocs;
};

void prefill_release(PrefillState* pf) {
  if (!pf) return;
  for (void* p : pf->allocs) cudaFree(p);
  if (pf->scratch) cudaFree(pf->scratch);
  if (pf->mail_h) cudaFreeHost(pf->mail_h);
  for (auto e : pf->ev) cudaEventDestroy(e);
  delete pf;
}

namespace {

#define TRY(x)                   \
  do {                           \
    moe_status _s = (x);         \
    if (_s != MOE_OK) return _s; \
  } while (0)

template <class T>
moe_status pf_alloc(PrefillState* pf, T** p, size_t n) {
  void* q = nullptr;
  MOE_CUDA(cudaMalloc(&q, std::max<size_t>(n, 16)));
  MOE_CUDA(cudaMemset(q, 0, std::max<size_t>(n, 16)));
  pf->allocs.push_back(q);
  *p = static_cast<T*>(q);
  return MOE_OK;
}

moe_status ensure_state(moe_engine* g, int T) {
  const int L = g->cfg.num_layers, E = g->cfg.num_experts, K = g->cfg.top_k, d = g->d, f = g->f;
  if (!g->pf) {
    g->pf = new PrefillState();
    PrefillState* pf = g->pf;
    MOE_CUDA(cudaMalloc(reinterpret_cast<void**>(&pf->scratch), static_cast<size_t>(E) * g->expert_bytes));
    MOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pf->mail_h), sizeof(PrefillMail),
                           cudaHostAllocMapped | cudaHostAllocPortable));
    memset(pf->mail_h, 0, sizeof(PrefillMail));
    MOE_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&pf->mail_d), pf->mail_h, 0));
    for (int i = 0; i < moe_engine::kCodedParts * kMaxE; ++i) {
      cudaEvent_t e = nullptr;
      MOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      pf->ev.push_back(e);
    }
  }
  PrefillState* pf = g->pf;
  if (pf->cap_T >= T) return MOE_OK;
  for (void* p : pf->allocs) cudaFree(p);
  pf->allocs.clear();
  pf->mix_T = -1;
  const size_t TK = static_cast<size_t>(T) * K;
  const int mt = static_cast<int>((TK + tc::BM - 1) / tc::BM) + E;  // m-tiles over all groups
  pf->max_up = (f / (tc::BN / 2)) * mt;
  pf->max_dn = (d / tc::BN) * mt;
  // down projection per expert: (d / 256) n-tiles x ceil(rows / 128) m-tiles, typically far
  // fewer than the SMs; split K so one expert's launch covers about one wave
  const int rows_per_expert = static_cast<int>((TK + E - 1) / E);
  const int base_tiles = (d / tc::BN) * std::max(1, (rows_per_expert + tc::BM - 1) / tc::BM);
  pf->splits = std::max(1, std::min({tc::sm_count() / base_tiles, 16, f / tc::BK / 8}));
  pf->split_stride = static_cast<long long>(TK) * d;
  TRY(pf_alloc(pf, &pf->x, sizeof(float) * T * d));
  TRY(pf_alloc(pf, &pf->hm, sizeof(float) * T * d));
  TRY(pf_alloc(pf, &pf->y, sizeof(float) * TK * d * pf->splits));
  TRY(pf_alloc(pf, &pf->inv, sizeof(float) * T));
  TRY(pf_alloc(pf, &pf->a_mix, sizeof(uint16_t) * T * d));
  TRY(pf_alloc(pf, &pf->an, sizeof(uint16_t) * TK * d));
  TRY(pf_alloc(pf, &pf->act, sizeof(uint16_t) * TK * f));
  TRY(pf_alloc(pf, &pf->row_map, sizeof(int) * TK));
  TRY(pf_alloc(pf, &pf->pos_of, sizeof(int) * TK));
  TRY(pf_alloc(pf, &pf->grp_up, sizeof(tc::Group) * kMaxE));
  TRY(pf_alloc(pf, &pf->grp_dn, sizeof(tc::Group) * kMaxE));
  TRY(pf_alloc(pf, &pf->grp_mix, sizeof(tc::Group) * L));
  TRY(pf_alloc(pf, &pf->tiles_up, sizeof(tc::Tile) * (1 + E) * pf->max_up));
  TRY(pf_alloc(pf, &pf->tiles_dn, sizeof(tc::Tile) * (1 + E) * pf->max_dn));
  const int mix_tiles = (d / tc::BN) * ((T + tc::BM - 1) / tc::BM);
  TRY(pf_alloc(pf, &pf->tiles_mix, sizeof(tc::Tile) * L * mix_tiles));
  TRY(pf_alloc(pf, &pf->cnt_up, sizeof(int) * (1 + E)));
  TRY(pf_alloc(pf, &pf->cnt_dn, sizeof(int) * (1 + E)));
  TRY(pf_alloc(pf, &pf->cnt_mix, sizeof(int) * L));
  pf->cap_T = T;
  return MOE_OK;
}

// Mixing GEMM tiles depend only on T (one group per layer: rows [0, T), M_l at rows l*d).
moe_status ensure_mix_tiles(moe_engine* g, int T, cudaStream_t s) {
  PrefillState* pf = g->pf;
  if (pf->mix_T == T) return MOE_OK;
  const int L = g->cfg.num_layers, d = g->d;
  const int mt = (T + tc::BM - 1) / tc::BM, per = (d / tc::BN) * mt;
  pf->h_grp_mix.assign(L, tc::Group{});
  pf->h_tiles_mix.assign(static_cast<size_t>(L) * per, tc::Tile{});
  pf->h_cnt_mix.assign(L, per);
  for (int l = 0; l < L; ++l) {
    pf->h_grp_mix[l] = tc::Group{0, T, l * d, 0, 0};
    for (int i = 0; i < per; ++i)
      pf->h_tiles_mix[static_cast<size_t>(l) * per + i] = tc::Tile{l, (i % mt) * tc::BM, (i / mt) * tc::BN};
  }
  MOE_CUDA(cudaMemcpyAsync(pf->grp_mix, pf->h_grp_mix.data(), sizeof(tc::Group) * L, cudaMemcpyHostToDevice, s));
  MOE_CUDA(cudaMemcpyAsync(pf->tiles_mix, pf->h_tiles_mix.data(), sizeof(tc::Tile) * pf->h_tiles_mix.size(),
                           cudaMemcpyHostToDevice, s));
  MOE_CUDA(cudaMemcpyAsync(pf->cnt_mix, pf->h_cnt_mix.data(), sizeof(int) * L, cudaMemcpyHostToDevice, s));
  MOE_CUDA(cudaStreamSynchronize(s));  // host vectors may be rebuilt on the next call
  pf->mix_T = T;
  pf->mix_tiles_per_layer = per;
  return MOE_OK;
}

moe_status await_prefill_mail(moe_engine* g, long long seq, cudaStream_t compute, PrefillMail* out) {
  PrefillMail& m = *g->pf->mail_h;
  long long spins = 0;
  const auto t0 = std::chrono::steady_clock::now();
  while (m.ready != seq + 1) {
    if ((++spins & 1023) == 0) {
      const cudaError_t q = cudaStreamQuery(compute);
      if (q != cudaSuccess && q != cudaErrorNotReady) {
        set_error("compute stream failed during prefill (seq %lld): %s", seq, cudaGetErrorString(q));
        return MOE_CUDA_ERROR;
      }
      if (q == cudaSuccess) {
        std::atomic_thread_fence(std::memory_order_acquire);
        if (m.ready != seq + 1) {
          set_error("prefill plan of seq %lld finished without posting its decision", seq);
          return MOE_CUDA_ERROR;
        }
      }
      const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (waited > 120.0) {
        set_error("no prefill plan for seq %lld after %.0f s", seq, waited);
        return MOE_CUDA_ERROR;
      }
      if (spins > (1 << 16)) std::this_thread::yield();
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  memcpy(out, const_cast<PrefillMail*>(&m), sizeof(PrefillMail));
  return MOE_OK;
}

}  // namespace
}  // namespace moe

using namespace moe;

extern "C" moe_status moe_engine_prefill(moe_engine* g, const float* h_in_dev, int64_t T64,
                                         float* h_out_dev, void* stream) {
  return moe_engine_prefill_routed(g, h_in_dev, T64, h_out_dev, nullptr, stream);
}

extern "C" moe_status moe_engine_prefill_routed(moe_engine* g, const float* h_in_dev, int64_t T64,
                                                float* h_out_dev, const int32_t* routing_dev,
                                                void* stream) {
  MOE_REQUIRE(g, "null engine");
  MOE_REQUIRE(g->bf16, "prefill runs the SwiGLU (bf16) engine; the toy engine decodes token by token");
  const moe_engine_config& c = g->cfg;
  MOE_REQUIRE(T64 >= 0 && T64 <= c.max_tokens, "prefill of %lld tokens needs max_tokens >= T (%d)",
              (long long)T64, c.max_tokens);
  if (T64 == 0) return MOE_OK;
  MOE_REQUIRE(g->d % tc::BN == 0 && g->f % (tc::BN / 2) == 0,
              "prefill needs hidden_dim %% 256 == 0 and ffn_dim %% 128 == 0 (got %d, %d)", g->d, g->f);
  MOE_ON_DEVICE(g->device);
  MOE_REQUIRE(pf_plan_smem(static_cast<int>(T64), c.top_k) <= 160 * 1024,
              "prefill of %lld tokens exceeds the plan kernel's staging (split the batch)", (long long)T64);
  static std::atomic<uint64_t> plan_attr{0};
  once_per_device(plan_attr, [] {
    cudaFuncSetAttribute(pf_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  });
  const int T = static_cast<int>(T64);
  const int L = c.num_layers, E = c.num_experts, K = c.top_k, d = g->d, f = g->f;
  cudaStream_t s = as_stream(stream);
  TRY(ensure_state(g, T));
  TRY(ensure_mix_tiles(g, T, s));
  PrefillState* pf = g->pf;

  // outstanding speculative prefetch jobs are abandoned (the plan clears the staging tags)
  for (auto& j : g->jobs)
    if (!j.cancelled && !j.adopted) {
      j.cancelled = true;
      std::lock_guard<std::mutex> lk(g->stats_mu);
      g->st.prefetch_wasted_bytes += std::min(j.next_chunk * c.chunk_bytes, g->expert_bytes);
    }

  // tensor maps: A operands, the mixing stack, and the pool / scratch in d- and f-row views
  const size_t pool_bytes = static_cast<size_t>(L) * g->NB * g->expert_bytes;
  const size_t scratch_bytes = static_cast<size_t>(E) * g->expert_bytes;
  CUtensorMap m_amix, m_mix, m_an, m_act, m_pool_d, m_pool_f, m_scr_d, m_scr_f;
  TRY(tc::make_tmap_bf16(&m_amix, pf->a_mix, T, d));
  TRY(tc::make_tmap_bf16(&m_mix, g->mixing, static_cast<long long>(L) * d, d));
  TRY(tc::make_tmap_bf16(&m_an, pf->an, static_cast<long long>(T) * K, d));
  TRY(tc::make_tmap_bf16(&m_act, pf->act, static_cast<long long>(T) * K, f));
  TRY(tc::make_tmap_bf16(&m_pool_d, g->pool, pool_bytes / (2 * d), d));
  TRY(tc::make_tmap_bf16(&m_pool_f, g->pool, pool_bytes / (2 * f), f));
  TRY(tc::make_tmap_bf16(&m_scr_d, pf->scratch, scratch_bytes / (2 * d), d));
  TRY(tc::make_tmap_bf16(&m_scr_f, pf->scratch, scratch_bytes / (2 * f), f));

  const int grid = tc::sm_count();
  const long long tok0 = g->tokens_done;
  const long long split = 2ll * f * d * 2;  // w1|w3 bytes; w2 follows
  long long loaded = 0;
  // profiling: events around every GEMM launch with its algorithmic flops / bytes
  struct GemmEv {
    cudaEvent_t a, b;
    double flops;
    long long bytes;
    int slot;  // in-kernel span slot (prof buffer), -1 none
  };
  long long* gprof = nullptr;  // [launches][2] in-kernel spans (profiling only)
  constexpr int kMaxGemmProf = 4096;
  if (g->profiling) {
    MOE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&gprof), sizeof(long long) * 2 * kMaxGemmProf, s));
    MOE_CUDA(cudaMemsetAsync(gprof, 0, sizeof(long long) * 2 * kMaxGemmProf, s));
  }
  std::vector<GemmEv> gev;
  cudaEvent_t pf_begin = nullptr, pf_end = nullptr;
  auto gemm = [&](const CUtensorMap& ma, const CUtensorMap& mb0, const CUtensorMap& mb1,
                  const tc::Params& p, double flops, long long bytes) -> moe_status {
    GemmEv e{nullptr, nullptr, flops, bytes, -1};
    tc::Params pp = p;
    if (g->profiling && gev.size() < static_cast<size_t>(kMaxGemmProf)) {
      e.slot = static_cast<int>(gev.size());
      pp.prof = gprof + 2 * e.slot;
    }
    if (g->profiling) {
      MOE_CUDA(cudaEventCreate(&e.a));
      MOE_CUDA(cudaEventCreate(&e.b));
      MOE_CUDA(cudaEventRecord(e.a, s));
    }
    TRY(tc::launch_grouped(ma, mb0, mb1, pp, grid, s));
    if (g->profiling) {
      MOE_CUDA(cudaEventRecord(e.b, s));
      gev.push_back(e);
    }
    return MOE_OK;
  };
  if (g->profiling) {
    MOE_CUDA(cudaEventCreate(&pf_begin));
    MOE_CUDA(cudaEventCreate(&pf_end));
    MOE_CUDA(cudaEventRecord(pf_begin, s));
  }

  const int cgrid = (d / 4 + 255) / 256;
  pf_combine_kernel<<<dim3(cgrid, T), 256, 0, s>>>(h_in_dev, nullptr, nullptr, 1, 0, g->ring, tok0,
                                                    c.max_tokens, L, 0, d, K, pf->x, pf->a_mix);
  MOE_LAUNCHED();
  for (int l = 0; l < L; ++l) {
    const long long seq = (tok0 + T - 1) * L + l;
    // ---- mixing map on the tensor cores: h' = x + alpha * M x ----
    tc::Params pm{};
    pm.tiles = pf->tiles_mix + static_cast<size_t>(l) * pf->mix_tiles_per_layer;
    pm.n_tiles = pf->cnt_mix + l;
    pm.groups = pf->grp_mix;
    pm.K = d;
    pm.N = d;
    pm.epi = tc::kEpiMix;
    pm.x = pf->x;
    pm.h_mid = pf->hm;
    pm.alpha = c.mixing_scale;
    TRY(gemm(m_amix, m_mix, m_mix, pm, 2.0 * T * d * d, 2ll * d * d + 2ll * T * d + 8ll * T * d));
    // ---- gate, one warp per token ----
    PfGateParams gp{pf->x, pf->hm, g->gate_w + static_cast<size_t>(l) * E * d,
                    g->gate_b + static_cast<size_t>(l) * E, g->ring, tok0, c.max_tokens, L, l, T, d,
                    E, K, c.record_speculation, c.renormalize, c.rms_norm, c.rms_eps, pf->inv, g->err,
                    routing_dev};
    if (E <= 8)
      pf_gate_kernel<8><<<T, 256, 0, s>>>(gp);
    else
      pf_gate_kernel<kMaxE><<<T, 256, 0, s>>>(gp);
    MOE_LAUNCHED();
    // ---- policy replay over the T steps + buffer plan + grouping + tiles + mailbox ----
    PfPlanParams pp{};
    pp.ring = g->ring;
    pp.tok0 = tok0;
    pp.max_tokens = c.max_tokens;
    pp.L = L;
    pp.layer = l;
    pp.T = T;
    pp.E = E;
    pp.K = K;
    pp.C = c.cache_size;
    pp.NB = c.cache_size + (c.prefetch ? g->S : 0);
    pp.pool_nb = g->NB;  // set_mode may run fewer buffers than allocated
    pp.policy = c.policy;
    pp.decay_factor = c.decay_factor;
    pp.decay_period = c.decay_period;
    pp.state = g->states + l;
    pp.stats = g->dstats;
    pp.err = g->err;
    pp.d = d;
    pp.f = f;
    pp.rows_per_buf_d = g->expert_bytes / (2 * d);
    pp.rows_per_buf_f = g->expert_bytes / (2 * f);
    pp.row_map = pf->row_map;
    pp.pos_of = pf->pos_of;
    pp.grp_up = pf->grp_up;
    pp.grp_dn = pf->grp_dn;
    pp.tiles_up = pf->tiles_up;
    pp.tiles_dn = pf->tiles_dn;
    pp.cnt_up = pf->cnt_up;
    pp.cnt_dn = pf->cnt_dn;
    pp.max_up = pf->max_up;
    pp.max_dn = pf->max_dn;
    pp.seq = seq;
    pp.mail = pf->mail_d;
    pf_plan_kernel<<<1, 256, pf_plan_smem(T, K), s>>>(pp);
    MOE_LAUNCHED();
    pf_gather_kernel<<<(T * K + 7) / 8, 256, 0, s>>>(pf->hm, pf->inv, pf->pos_of, T * K, K, d, pf->an, pf->y,
                                                     pf->splits, pf->split_stride);
    MOE_LAUNCHED();
    // ---- forward the device's plan: one H2D load per needed, uncached expert ----
    PrefillMail m;
    TRY(await_prefill_mail(g, seq, s, &m));
    if (g->debug)
      fprintf(stderr, "[moe] prefill layer=%d loads=%d moves=%d resident_groups=%d\n", l, m.n_loads,
              m.n_moves, m.n_res_groups);
    std::pair<cudaEvent_t, cudaEvent_t> tev{nullptr, nullptr};
    if (m.n_loads > 0) {
      {
        std::lock_guard<std::mutex> lk(g->stats_mu);
        if (!g->free_events.empty()) {
          tev = g->free_events.back();
          g->free_events.pop_back();
        }
      }
      if (!tev.first) {
        MOE_CUDA(cudaEventCreate(&tev.first));
        MOE_CUDA(cudaEventCreate(&tev.second));
      }
      MOE_CUDA(cudaEventRecord(tev.first, g->copy_stream));
    }
    std::vector<char*> dest(m.n_loads);
    const int nslots = g->cstore ? static_cast<int>(g->cstage_free.size()) : 0;
    // exponent-coded load i lands in slot i % nslots once that slot's previous part is decoded:
    // issued here for the first nslots loads, later right after the decode that frees the slot
    // (a stream wait captures the event's latest record at the time of the call)
    auto issue_coded = [&](int i) -> moe_status {
      const int e = m.load_expert[i], slot = i % nslots;
      const moe_engine::CPart* cp = g->coded_parts(l, e);
      char* land = g->cstage + static_cast<long long>(slot) * g->expert_bytes;
      MOE_CUDA(cudaStreamWaitEvent(g->copy_stream, g->cstage_free[slot], 0));
      long long off = 0;
      for (int q = 0; q < moe_engine::kCodedParts; ++q) {
        MOE_CUDA(cudaMemcpyAsync(land + off, g->cstore + cp[q].off, cp[q].size, cudaMemcpyHostToDevice,
                                 g->copy_stream));
        off += static_cast<long long>(cp[q].size);
        // events: part 0 (w1|w3) lets the up GEMM go; the w2 pieces are decoded as they land
        MOE_CUDA(cudaEventRecord(pf->ev[i * moe_engine::kCodedParts + q], g->copy_stream));
      }
      loaded += off;
      return MOE_OK;
    };
    for (int i = 0; i < m.n_loads; ++i) {
      const int e = m.load_expert[i], dst = m.load_dst[i];
      char* to = dst >= 0 ? g->pool + (static_cast<long long>(l) * g->NB + dst) * g->expert_bytes
                          : pf->scratch + static_cast<long long>(-1 - dst) * g->expert_bytes;
      dest[i] = to;
      if (g->cstore) {
        if (i < nslots) TRY(issue_coded(i));
        continue;
      }
      const char* from = g->store_block(l, e);
      MOE_CUDA(cudaMemcpyAsync(to, from, split, cudaMemcpyHostToDevice, g->copy_stream));
      MOE_CUDA(cudaEventRecord(pf->ev[2 * i], g->copy_stream));
      MOE_CUDA(cudaMemcpyAsync(to + split, from + split, g->expert_bytes - split, cudaMemcpyHostToDevice,
                               g->copy_stream));
      MOE_CUDA(cudaEventRecord(pf->ev[2 * i + 1], g->copy_stream));
      loaded += g->expert_bytes;
    }
    g->ctl_h->consumed = seq + 1;
    // ---- expert FFN: resident experts now, each loaded expert after its copies ----
    tc::Params pu{};
    pu.groups = pf->grp_up;
    pu.K = d;
    pu.N = f;
    pu.epi = tc::kEpiSwiGLU;
    pu.act = pf->act;
    tc::Params pd{};
    pd.groups = pf->grp_dn;
    pd.K = f;
    pd.N = d;
    pd.epi = tc::kEpiScatter;
    pd.row_map = pf->row_map;
    pd.y = pf->y;
    pd.splits = pf->splits;
    pd.split_stride = pf->split_stride;
    auto ffn = [&](int list, int rows, int ngroups) -> moe_status {
      pu.tiles = pf->tiles_up + static_cast<size_t>(list) * pf->max_up;
      pu.n_tiles = pf->cnt_up + list;
      const double fu = 2.0 * rows * 2.0 * f * d;
      TRY(gemm(m_an, m_pool_d, m_scr_d, pu, fu,
               4ll * f * d * ngroups + 2ll * rows * d + 2ll * rows * f));
      return MOE_OK;
    };
    auto ffn_down = [&](int list, int rows, int ngroups) -> moe_status {
      pd.tiles = pf->tiles_dn + static_cast<size_t>(list) * pf->max_dn;
      pd.n_tiles = pf->cnt_dn + list;
      const double fd = 2.0 * rows * static_cast<double>(f) * d;
      TRY(gemm(m_act, m_pool_f, m_scr_f, pd, fd,
               2ll * f * d * ngroups + 2ll * rows * f + 4ll * rows * d * pf->splits));
      return MOE_OK;
    };
    if (m.n_res_groups > 0) {
      TRY(ffn(0, m.res_rows, m.n_res_groups));
      TRY(ffn_down(0, m.res_rows, m.n_res_groups));
    }
    for (int i = 0; i < m.n_loads; ++i) {
      if (g->cstore) {
        const int slot = i % nslots, NP = moe_engine::kCodedParts;
        const char* land = g->cstage + static_cast<long long>(slot) * g->expert_bytes;
        const moe_engine::CPart* cp = g->coded_parts(l, m.load_expert[i]);
        MOE_CUDA(cudaStreamWaitEvent(s, pf->ev[i * NP], 0));
        TRY(xc::decode(land, cp[0].hdr, reinterpret_cast<uint16_t*>(dest[i]), s));
        TRY(ffn(1 + i, m.load_rows[i], 1));
        long long coff = static_cast<long long>(cp[0].size);
        // w2 pieces 1..3 in one launch once the third has landed, the last on its own
        const void* src[xc::kMaxBatch];
        uint16_t* dst[xc::kMaxBatch];
        xc::PartHeader hh[xc::kMaxBatch];
        int nb = 0;
        for (int q = 1; q < NP; ++q) {
          MOE_CUDA(cudaStreamWaitEvent(s, pf->ev[i * NP + q], 0));
          src[nb] = land + coff;
          dst[nb] = reinterpret_cast<uint16_t*>(dest[i] + g->coded_part_out_off(q));
          hh[nb] = cp[q].hdr;
          ++nb;
          coff += static_cast<long long>(cp[q].size);
          if (q == NP - 2 || q == NP - 1) {
            TRY(xc::decode_batch(src, hh, dst, nb, s));
            nb = 0;
          }
        }
        MOE_CUDA(cudaEventRecord(g->cstage_free[slot], s));
        if (i + nslots < m.n_loads) TRY(issue_coded(i + nslots));
      } else {
        MOE_CUDA(cudaStreamWaitEvent(s, pf->ev[2 * i], 0));
        TRY(ffn(1 + i, m.load_rows[i], 1));
        MOE_CUDA(cudaStreamWaitEvent(s, pf->ev[2 * i + 1], 0));
      }
      TRY(ffn_down(1 + i, m.load_rows[i], 1));
    }
    if (m.n_loads > 0) {
      MOE_CUDA(cudaEventRecord(tev.second, g->copy_stream));
      std::lock_guard<std::mutex> lk(g->stats_mu);
      g->busy_events.push_back(tev);
    }
    // experts that stay cached but were loaded into scratch move into their cache buffer
    for (int i = 0; i < m.n_moves; ++i) {
      const int e = m.move_expert[i], b = m.move_buf[i];
      MOE_CUDA(cudaMemcpyAsync(g->pool + (static_cast<long long>(l) * g->NB + b) * g->expert_bytes,
                               pf->scratch + static_cast<long long>(e) * g->expert_bytes, g->expert_bytes,
                               cudaMemcpyDeviceToDevice, s));
    }
    // ---- next layer's input (or the output) ----
    const bool last = l + 1 == L;
    pf_combine_kernel<<<dim3(cgrid, T), 256, 0, s>>>(nullptr, pf->hm, pf->y, pf->splits, pf->split_stride,
                                                      g->ring, tok0, c.max_tokens,
                                                      L, l, d, K, last ? h_out_dev : pf->x,
                                                      last ? nullptr : pf->a_mix);
    MOE_LAUNCHED();
  }
  if (g->profiling) {
    MOE_CUDA(cudaEventRecord(pf_end, s));
    MOE_CUDA(cudaEventSynchronize(pf_end));
    moe_kernel_times& k = g->ktimes;
    std::vector<long long> spans(2 * kMaxGemmProf, 0);
    MOE_CUDA(cudaMemcpy(spans.data(), gprof, sizeof(long long) * spans.size(), cudaMemcpyDeviceToHost));
    cudaFree(gprof);
    for (auto& e : gev) {
      if (e.slot >= 0) {
        const long long t0 = 0x7fffffffffffffffll - spans[2 * e.slot], t1 = spans[2 * e.slot + 1];
        if (spans[2 * e.slot] > 0 && t1 > t0) k.gemm_kernel_ms += (t1 - t0) / 1e6;
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e.a, e.b);
      k.gemm_ms += ms;
      k.gemm_launches += 1;
      k.gemm_flops += e.flops;
      k.gemm_bytes += e.bytes;
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pf_begin, pf_end);
    k.prefill_ms += ms;
    cudaEventDestroy(pf_begin);
    cudaEventDestroy(pf_end);
  }
  {
    std::lock_guard<std::mutex> lk(g->stats_mu);
    g->st.prefill_tokens += T;
    g->st.prefill_bytes += loaded;
    g->st.h2d_bytes += loaded;
  }
  g->tokens_done += T;
  return MOE_OK;
}
