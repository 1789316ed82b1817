// Bulk-copy (TMA engine) streaming GEMV for the bf16 decode path: mixing map (K0),
// SwiGLU up projection and down projection (K3).
//
// Batch-1 decode reads every weight byte exactly once, so these kernels are HBM-bound.
// Each CTA owns a contiguous band of 8-row blocks of one matrix.  A producer thread streams
// the band through a ring of shared-memory stages with cp.async.bulk (one bulk copy per
// row slice, completion counted on an mbarrier, L2 evict-first since nothing re-reads the
// weights), while 8 consumer warps each reduce one row of the stage against the activation
// vector kept in shared memory.  Bytes in flight per SM are the ring size (~130-160 KB),
// independent of register pressure; the grid is sized so every CTA gets the same number of
// row blocks (HBM, not the SM count, is the bound).
#pragma once
#include "engine_kernels.cuh"
#include "sm100.cuh"

namespace moe {

constexpr int kStreamWarps = 8;                       // consumer warps = rows per block
constexpr int kStreamThreads = (kStreamWarps + 1) * 32; // + one producer warp
constexpr int kStreamStageBytes = 32 * 1024;
constexpr int kStreamSmemBudget = 200 * 1024;
constexpr int kMixBandRows = 64;   // MIX: gate partials from registers / smem up to this band

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kStreamWarps * 32) : "memory");
}

enum StreamMode { kModeMix = 0, kModeUp = 1, kModeDown = 2 };

struct StreamParams {
  // geometry
  int d, f, K, cb, ncb, stages;
  // MIX
  const float* x;          // layer-0 token input, else nullptr (then combine prev layer)
  const float* prev_mid;
  const float* y;          // previous layer's expert outputs [K][d] (MIX) / output (DOWN)
  const StepRecord* prev;
  const uint16_t* M;       // mixing [d][d]
  const uint16_t* M_next;  // the next layer's mixing matrix: each CTA prefetches its band into
                           // L2 once its own copies are issued (read by the next MIX launch,
                           // same grid, same bands), or nullptr
  float alpha;
  float* h_in;
  float* h_mid;
  // UP / DOWN
  const float* xin;        // UP: h_norm [d]
  const StepRecord* rec;
  const LayerState* state;
  const char* pool;        // this layer's buffers
  long long expert_bytes;
  int phase;
  int only;                // -1: every expert of the phase; i: just the i-th (ascending id)
  float* act;              // [K][f]
  float* yout;             // [K][d]
  int row_lo, row_hi;      // DOWN: only output rows [row_lo, row_hi) (multiples of the row
                           // block), e.g. the w2 pieces already decoded; row_hi = 0: all rows
  long long* prof_bytes;   // optional profiling slot [4]: weight bytes this launch streams,
                           // max(LLONG_MAX - CTA start ns), max(consumer end ns) (globaltimer)
  // MIX: per-CTA partial gate logits over the CTA's rows (see GateParams::part)
  const float* gate_w;     // this layer's gate [E][d]
  const float* gate_w_next;  // next layer's gate (early speculative guess) or nullptr
  int E, do_guess;
  float* part;             // [gridDim.x][3E + 2]
  // UP: scale applied to xin while staging (1/rms(h') from the gate), or nullptr
  const float* xscale;
  int stream_only;         // microbenchmark: consumers release stages without computing
  // MIX with fuse_gate: the last CTA to finish (done_ctr, zero between launches) runs the
  // gate / cache step on the summed partials -- no separate gate launch on the critical path
  int fuse_gate;
  unsigned int* done_ctr;
  GateParams gate;
};

// Which experts this launch covers: (selection slot j, weight block), in ascending expert
// id.  phase 0 = experts that hit, 1 = experts that missed; `only` >= 0 keeps just the
// only-th of those (the host orders per-expert launches after that expert's copies).
__device__ __forceinline__ int stream_active(const StreamParams& p, int* slot, const char** blk) {
  int n = 0, seen = 0;
  if (p.rec->flags) return 0;
  for (int k = 0; k < p.K; ++k) {
    const int e = p.rec->acts[k];
    if (e < 0 || e >= kMaxE) continue;
    const bool hit = (p.rec->rb >> e) & 1u;
    if (p.phase != 2 && (p.phase == 0) != hit) continue;
    const int idx = seen++;
    if (p.only >= 0 && idx != p.only) continue;
    const int b = p.state->buf_of[e];
    if (b < 0) continue;
    int j = 0;
    while (j < p.K && p.rec->sel[j] != e) ++j;
    slot[n] = j;
    blk[n] = p.pool + b * p.expert_bytes;
    ++n;
  }
  return n;
}

// RPB rows per block, WPR = 8 / RPB warps per row (each reduces a column slice of the row;
// pairs/quads combine through shared memory in a fixed order).
template <int MODE, int RPB>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_gemv_kernel(StreamParams p) {
  // Programmatic launch (copy-engine decode): MIX lets the next kernel launch at once and only
  // its consumers wait for the previous layer (its producer streams M meanwhile); UP / DOWN
  // read the gate's record and their predecessor's outputs, so every thread waits first.
  if constexpr (MODE == kModeMix) {
    pdl_trigger();
    if (p.gate.phase_ns && threadIdx.x == 0) {   // diagnostics: this launch's first CTA start
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(&p.gate.phase_ns[7], ~0ull - t);
      atomicMax(&p.gate.phase_ns[8], t);
    }
  } else {
    pdl_wait();
    pdl_trigger();
  }
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NM = MODE == kModeUp ? 2 : 1;  // matrices streamed per row block
  constexpr int WPR = kStreamWarps / RPB;
  static_assert(RPB * WPR == kStreamWarps, "RPB must divide the consumer warp count");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = MODE == kModeDown ? p.f : p.d;  // row length
  const int R = MODE == kModeUp ? p.f : p.d;    // rows per matrix
  const bool ranged = MODE == kModeDown && p.row_hi > p.row_lo;
  const int RS = ranged ? p.row_hi - p.row_lo : R;   // rows this launch covers
  const int rbase = ranged ? p.row_lo / RPB : 0;
  const int cb = p.cb, ncb = p.ncb, S = p.stages;
  const uint32_t slice = static_cast<uint32_t>(cb) * 2;   // bytes per row slice
  const uint32_t stage_bytes = slice * RPB * NM;

  // ---- which matrix (expert) and which row blocks this CTA owns ----
  int slot[kMaxK];
  const char* blk[kMaxK];
  int n_active = 1;
  if (MODE != kModeMix) n_active = stream_active(p, slot, blk);
  if (p.prof_bytes && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&p.prof_bytes[1], 0x7fffffffffffffffll - static_cast<long long>(t));
    if (blockIdx.x == 0) p.prof_bytes[0] = static_cast<long long>(n_active) * NM * RS * C * 2;
    if (n_active == 0) atomicMax(&p.prof_bytes[2], static_cast<long long>(t));
  }
  if (n_active == 0) return;
  const int a = static_cast<int>((static_cast<long long>(blockIdx.x) * n_active) / gridDim.x);
  const int c0 = static_cast<int>((static_cast<long long>(a) * gridDim.x + n_active - 1) / n_active);
  const int c1 = static_cast<int>((static_cast<long long>(a + 1) * gridDim.x + n_active - 1) / n_active);
  const int nrb = RS / RPB;
  const int my = blockIdx.x - c0, ncta = c1 - c0;
  const int rb0 = rbase + static_cast<int>((static_cast<long long>(my) * nrb) / ncta);
  const int rb1 = rbase + static_cast<int>((static_cast<long long>(my + 1) * nrb) / ncta);
  const int n_work = (rb1 - rb0) * ncb;

  // MIX: this thread's gate-weight operands for the epilogue's partial logits, loaded now so
  // their latency hides behind the stream (job q = tid / 8 of the first 32, rows sub + 8k of
  // the band, sub = tid % 8; they do not depend on the previous kernel)
  float wpre[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) wpre[k] = 0.f;
  if constexpr (MODE == kModeMix) {
    const int r0 = rb0 * RPB, nr = (rb1 - rb0) * RPB;
    const int q = threadIdx.x >> 3, sub = threadIdx.x & 7;
    if (p.part && nr <= kMixBandRows && threadIdx.x < kStreamWarps * 32 && q < 3 * p.E) {
      const int which = q / p.E, e = q % p.E;
      const float* w = which == 2 ? p.gate_w_next : (which == 1 && !p.do_guess ? nullptr : p.gate_w);
      if (w) {
        w += static_cast<size_t>(e) * p.d + r0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (sub + 8 * k < nr) wpre[k] = w[sub + 8 * k];
      }
    }
  }

  const uint16_t* W[NM];
  if constexpr (MODE == kModeMix) {
    W[0] = p.M;
  } else if constexpr (MODE == kModeUp) {
    W[0] = reinterpret_cast<const uint16_t*>(blk[a]);                 // w1 [f][d]
    W[1] = W[0] + static_cast<size_t>(p.f) * p.d;                      // w3 [f][d]
  } else {
    W[0] = reinterpret_cast<const uint16_t*>(blk[a]) + 2 * static_cast<size_t>(p.f) * p.d;  // w2 [d][f]
  }

  uint8_t* stage_base = smem;
  float4* pa = reinterpret_cast<float4*>(smem + static_cast<size_t>(S) * stage_bytes);
  float4* pb = pa + C / 8;
  float* hs = reinterpret_cast<float*>(pb + C / 8);                 // MIX: layer input
  float* xch = hs + (MODE == kModeMix ? p.d : 0);                   // [RPB][WPR][NM] partials
  float* hb = xch + 64;                                              // MIX: this CTA's h' rows
  uint64_t* full = reinterpret_cast<uint64_t*>(xch + (MODE == kModeMix ? 64 + kMixBandRows : 64));
  uint64_t* empty = full + S;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kStreamWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kStreamWarps) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      for (int it = 0; it < n_work; ++it) {
        const int s = it % S;
        if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
        const int rb = rb0 + it / ncb, c = it % ncb;
        uint8_t* dst = stage_base + static_cast<size_t>(s) * stage_bytes;
        mbar_expect_tx(&full[s], stage_bytes);
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          if (ncb == 1) {  // the block's full rows are contiguous: one copy
            bulk_g2s(dst + m * RPB * slice, W[m] + static_cast<size_t>(rb) * RPB * C,
                     RPB * slice, &full[s], pol);
            continue;
          }
#pragma unroll
          for (int r = 0; r < RPB; ++r) {
            const uint16_t* src = W[m] + static_cast<size_t>(rb * RPB + r) * C +
                                  static_cast<size_t>(c) * cb;
            bulk_g2s(dst + (m * RPB + r) * slice, src, slice, &full[s], pol);
          }
        }
      }
      if constexpr (MODE == kModeMix) {
        // the next layer's band of M into L2 while this layer's experts stream (their weights
        // are evict-first, so the prefetched band survives until the next mixing launch)
        if (p.M_next) {
          const char* b0 = reinterpret_cast<const char*>(p.M_next + static_cast<size_t>(rb0) * RPB * C);
          const long long nb = static_cast<long long>(rb1 - rb0) * RPB * C * 2;
          for (long long o = 0; o < nb; o += 32768)
            bulk_prefetch_l2(b0 + o, static_cast<uint32_t>(nb - o < 32768 ? nb - o : 32768));
        }
      }
    }
    return;
  }

  // ---------------- consumers: stage the activation vector ----------------
  if constexpr (MODE == kModeMix) {
    pdl_wait();   // the previous layer's outputs (a no-op unless launched programmatically)
    constexpr int kI4 = 8;   // float4s per thread staged with every load in flight (d <= 8192)
    if (!p.x && p.K <= 2 && p.d <= kI4 * 4 * kStreamWarps * 32) {
      // h_in = h'_{l-1} + p_0 y_0 + p_1 y_1 (selection order, as combine4): all of this
      // thread's loads issued before the first use -- one L2 round trip, not one per expert
      const int K = p.K;
      const float p0 = p.prev->prob[0], p1 = K > 1 ? p.prev->prob[1] : 0.f;
      const float4* hm = reinterpret_cast<const float4*>(p.prev_mid);
      const float4* y0 = reinterpret_cast<const float4*>(p.y);
      const float4* y1 = reinterpret_cast<const float4*>(p.y + p.d);
      float4 a[kI4], b[kI4], c[kI4];
#pragma unroll
      for (int u = 0; u < kI4; ++u) {
        const int i4 = threadIdx.x + u * kStreamWarps * 32;
        if (i4 < p.d / 4) {
          a[u] = hm[i4];
          b[u] = y0[i4];
          if (K > 1) c[u] = y1[i4];
        }
      }
#pragma unroll
      for (int u = 0; u < kI4; ++u) {
        const int i4 = threadIdx.x + u * kStreamWarps * 32;
        if (i4 < p.d / 4) {
          float4 v = a[u];
          v.x = __fadd_rn(v.x, __fmul_rn(p0, b[u].x));
          v.y = __fadd_rn(v.y, __fmul_rn(p0, b[u].y));
          v.z = __fadd_rn(v.z, __fmul_rn(p0, b[u].z));
          v.w = __fadd_rn(v.w, __fmul_rn(p0, b[u].w));
          if (K > 1) {
            v.x = __fadd_rn(v.x, __fmul_rn(p1, c[u].x));
            v.y = __fadd_rn(v.y, __fmul_rn(p1, c[u].y));
            v.z = __fadd_rn(v.z, __fmul_rn(p1, c[u].z));
            v.w = __fadd_rn(v.w, __fmul_rn(p1, c[u].w));
          }
          reinterpret_cast<float4*>(hs)[i4] = v;
          if (blockIdx.x == 0) reinterpret_cast<float4*>(p.h_in)[i4] = v;
        }
      }
    } else {
#pragma unroll 4
      for (int i4 = threadIdx.x; i4 < p.d / 4; i4 += kStreamWarps * 32) {
        const float4 v = p.x ? reinterpret_cast<const float4*>(p.x)[i4]
                             : combine4(p.prev_mid, p.y, p.prev, p.K, p.d, i4);
        reinterpret_cast<float4*>(hs)[i4] = v;
        if (blockIdx.x == 0) reinterpret_cast<float4*>(p.h_in)[i4] = v;
      }
    }
    consumers_sync();
    stage_planes_n(hs, p.d, pa, pb, kStreamWarps * 32);
    if (p.gate.phase_ns && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(&p.gate.phase_ns[9], t);
    }
  } else if constexpr (MODE == kModeUp) {
    stage_planes_n(p.xin, p.d, pa, pb, kStreamWarps * 32);
    if (p.xscale) {  // RMSNorm applied on the fly: x = h' * (1 / rms(h'))
      consumers_sync();
      const float sc = *p.xscale;
      for (int i = threadIdx.x; i < p.d / 8; i += kStreamWarps * 32) {
        float4 u = pa[i], v = pb[i];
        u.x *= sc; u.y *= sc; u.z *= sc; u.w *= sc;
        v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
        pa[i] = u;
        pb[i] = v;
      }
    }
  } else {
    stage_planes_n(p.act + static_cast<size_t>(slot[a]) * p.f, p.f, pa, pb, kStreamWarps * 32);
  }
  consumers_sync();

  const int row_in_block = warp / WPR, part_id = warp % WPR;
  const int span = cb / WPR;                  // columns this warp reduces per stage
  const int per_lane = span / 8 / 32;         // uint4 per lane (span multiple of 256)
  float acc[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) acc[m] = 0.f;
  for (int it = 0; it < n_work; ++it) {
    const int s = it % S;
    const int c = it % ncb;
    mbar_wait(&full[s], (it / S) & 1);
    const uint8_t* st = stage_base + static_cast<size_t>(s) * stage_bytes;
    const int col8 = (c * cb + part_id * span) / 8;
    if (!p.stream_only) {
      const uint4* row0 = reinterpret_cast<const uint4*>(st + row_in_block * slice) + part_id * (span / 8);
      const uint4* row1 = reinterpret_cast<const uint4*>(st + ((NM - 1) * RPB + row_in_block) * slice) +
                          part_id * (span / 8);
      float part0 = 0.f, part1 = 0.f;
#pragma unroll 4
      for (int q = 0; q < per_lane; ++q) {
        const int i = lane + 32 * q;
        const float4 xa = pa[col8 + i], xb = pb[col8 + i];  // shared by both matrices
        part0 = dot8_bf16(row0[i], xa, xb, part0);
        if constexpr (NM == 2) part1 = dot8_bf16(row1[i], xa, xb, part1);
      }
      acc[0] += part0;
      if constexpr (NM == 2) acc[NM - 1] += part1;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (c == ncb - 1) {
      const int r = (rb0 + it / ncb) * RPB + row_in_block;
      float v[NM];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        v[m] = warp_sum(acc[m]);
        acc[m] = 0.f;
      }
      if constexpr (WPR > 1) {
        // fixed-order combine of the row's column slices (deterministic)
        if (lane == 0)
#pragma unroll
          for (int m = 0; m < NM; ++m) xch[(row_in_block * WPR + part_id) * NM + m] = v[m];
        asm volatile("bar.sync %0, %1;" ::"r"(2 + row_in_block), "n"(WPR * 32) : "memory");
        if (part_id == 0 && lane == 0)
#pragma unroll
          for (int m = 0; m < NM; ++m) {
            float t = xch[(row_in_block * WPR) * NM + m];
            for (int q = 1; q < WPR; ++q) t += xch[(row_in_block * WPR + q) * NM + m];
            v[m] = t;
          }
        asm volatile("bar.sync %0, %1;" ::"r"(2 + row_in_block), "n"(WPR * 32) : "memory");
      }
      if (part_id == 0 && lane == 0) {
        if constexpr (MODE == kModeMix) {
          const float hm = __fadd_rn(hs[r], __fmul_rn(p.alpha, v[0]));
          p.h_mid[r] = hm;
          if (r - rb0 * RPB < kMixBandRows) hb[r - rb0 * RPB] = hm;
        } else if constexpr (MODE == kModeUp) {
          p.act[static_cast<size_t>(slot[a]) * p.f + r] = v[0] / (1.f + expf(-v[0])) * v[NM - 1];
        } else {
          p.yout[static_cast<size_t>(slot[a]) * p.d + r] = v[0];
        }
      }
    }
  }
  if constexpr (MODE == kModeMix) {
    if (p.part) {
      // gate logits fused into the mixing epilogue: this CTA's rows [r0, r1) of
      //   route  W_l h',  guess  W_l h_in,  early  W_{l+1} h',  and sum h'^2, sum h_in^2
      consumers_sync();
      if (p.gate.phase_ns && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(&p.gate.phase_ns[10], t);
      }
      const int r0 = rb0 * RPB, r1 = rb1 * RPB, E = p.E, njob = 3 * E + 2;
      if (r1 - r0 <= kMixBandRows) {
        // eight threads per job, each over every 8th row of the band with its operands in
        // registers (weights) and shared memory (h', h_in), then a fixed xor tree: no global
        // round trip on this serial path
        const int nr = r1 - r0, sub = threadIdx.x & 7;
        for (int q0 = 0; q0 < njob; q0 += kStreamWarps * 4) {
          const int q = q0 + (threadIdx.x >> 3);
          float acc = 0.f;
          if (q < njob) {
            const int which = q < 3 * E ? q / E : 3, e = q < 3 * E ? q % E : q - 3 * E;
            const bool on = !(which == 1 && !p.do_guess) && !(which == 2 && !p.gate_w_next);
            const float* wg = which == 2 ? p.gate_w_next : p.gate_w;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int r = sub + 8 * k;
              if (r < nr && on) {
                const float vh = which == 1 || (which == 3 && e == 1) ? hs[r0 + r] : hb[r];
                const float w = which == 3 ? vh : (q0 == 0 ? wpre[k] : wg[static_cast<size_t>(e) * p.d + r0 + r]);
                acc = fmaf(w, vh, acc);
              }
            }
          }
          acc += __shfl_xor_sync(FULL, acc, 4);
          acc += __shfl_xor_sync(FULL, acc, 2);
          acc += __shfl_xor_sync(FULL, acc, 1);
          if (q < njob && sub == 0) p.part[static_cast<size_t>(blockIdx.x) * njob + q] = acc;
        }
      } else
      for (int q = warp; q < njob; q += kStreamWarps) {
        const int which = q < 3 * E ? q / E : 3, e = q < 3 * E ? q % E : q - 3 * E;
        float acc = 0.f;
        if (which == 3) {
          const float* v = e == 0 ? p.h_mid : hs;
          for (int r = r0 + lane; r < r1; r += 32) acc = fmaf(v[r], v[r], acc);
        } else if (!(which == 1 && !p.do_guess) && !(which == 2 && !p.gate_w_next)) {
          const float* w = (which == 2 ? p.gate_w_next : p.gate_w) + static_cast<size_t>(e) * p.d;
          const float* v = which == 1 ? hs : p.h_mid;
          for (int r = r0 + lane; r < r1; r += 32) acc = fmaf(w[r], v[r], acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) p.part[static_cast<size_t>(blockIdx.x) * njob + q] = acc;
      }
      if (p.fuse_gate) {
        // last-CTA-done: the CTA whose ticket completes the grid sums every CTA's partials
        // (fence: they are visible once their ticket is) and takes the gate / cache step
        // the flag lives in the dynamic region (xch[63]; the partial exchange uses <= 16):
        // a static __shared__ would push static + 227 KB dynamic past the per-CTA limit
        volatile int* s_last = reinterpret_cast<volatile int*>(xch + 63);
        consumers_sync();
        if (p.gate.phase_ns && threadIdx.x == 0) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          atomicMax(&p.gate.phase_ns[15], t);
        }
        if (threadIdx.x == 0) {
          __threadfence();
          *s_last = atomicAdd(p.done_ctr, 1u) == gridDim.x - 1;
        }
        consumers_sync();
        if (*s_last) {
          __threadfence();
          // the stage ring is idle (every stage consumed): it holds the gate's working set
          GateSmem& gsm = *reinterpret_cast<GateSmem*>(stage_base);
          if (threadIdx.x == 0) *p.done_ctr = 0u;   // ready for the next launch (stream order)
          gate_cache_body(p.gate, gsm, threadIdx.x, kStreamWarps * 32, [] { consumers_sync(); }, false);
        }
      }
    }
  }
  if (p.prof_bytes && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&p.prof_bytes[2], static_cast<long long>(t));
  }
}

// Shared-memory bytes and stage geometry for one stream launch.
struct StreamGeom {
  int rpb, cb, ncb, stages;
  size_t smem;
};

// Rows per block / column block / ring depth for one mode.  Tuned on B200 with
// tools/tune_gemv.py: 4 KB+ row slices, 150-200 KB of ring per SM.
inline StreamGeom stream_geometry_rpb(int mode, int d, int f, int stage_budget, int max_stages,
                                      int rpb);

inline StreamGeom stream_geometry(int mode, int d, int f, int stage_budget = 0, int max_stages = 6,
                                  int rpb = 0) {
  // preferred rows-per-block first, then the always-valid 8 (one warp per row)
  const int pref = rpb ? rpb : (mode == kModeUp ? 8 : 4);
  StreamGeom g = stream_geometry_rpb(mode, d, f, stage_budget, max_stages, pref);
  if (g.ncb == 0 && rpb == 0 && pref != 8) g = stream_geometry_rpb(mode, d, f, stage_budget, max_stages, 8);
  return g;
}

inline StreamGeom stream_geometry_rpb(int mode, int d, int f, int stage_budget, int max_stages,
                                      int rpb) {
  const int NM = mode == kModeUp ? 2 : 1;
  const int C = mode == kModeDown ? f : d;
  if (stage_budget == 0) stage_budget = mode == kModeUp ? 64 * 1024 : 32 * 1024;
  const int wpr = kStreamWarps / rpb;
  StreamGeom g{};
  g.rpb = rpb;
  // widest column block whose stage fits the budget; each warp's share a multiple of 256
  g.ncb = 0;
  for (int n = 1; n <= C / 256; ++n) {
    if (C % n) continue;
    const int cb = C / n;
    if (cb % (256 * wpr)) continue;
    if (static_cast<long long>(cb) * 2 * rpb * NM <= stage_budget) {
      g.ncb = n;
      g.cb = cb;
      break;
    }
  }
  if (g.ncb == 0) return g;
  const size_t stage = static_cast<size_t>(g.cb) * 2 * rpb * NM;
  const size_t fixed = static_cast<size_t>(C) * 4 +
                       (mode == kModeMix ? static_cast<size_t>(d) * 4 + kMixBandRows * 4 : 0) + 64 * 4;
  if (fixed + 2 * stage + 256 > 227 * 1024) {
    g.ncb = 0;
    return g;
  }
  int S = static_cast<int>((224 * 1024 - fixed - 256) / stage);
  S = S < 2 ? 2 : (S > max_stages ? max_stages : S);
  g.stages = S;
  g.smem = S * stage + fixed + 2 * S * sizeof(uint64_t);
  return g;
}

// Grid: one CTA per SM -- per-SM bulk-copy throughput, not the HBM, limits a partial grid
// (tools/tune_gemv.py: 74 / 96 / 128 / 148 CTAs -> 3.0 / 3.9 / 5.2 / 5.7 TB/s); a multiple of
// the expert count so each active expert gets an equal band of CTAs.
inline int stream_grid(int experts, int sms = 148) { return sms / experts * experts; }

// Preferred L1/shared carveout of every stream GEMV instantiation (engine.cu keeps all kernels
// of a decode step on the same split).
inline void set_stream_carveout(int carveout) {
  cudaFuncSetAttribute(stream_gemv_kernel<kModeMix, 8>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeMix, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeMix, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeUp, 8>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeUp, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeUp, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeDown, 8>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeDown, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  cudaFuncSetAttribute(stream_gemv_kernel<kModeDown, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
}

// Launch one stream GEMV with the template instantiation matching the geometry.
template <int MODE>
inline cudaError_t launch_stream(const StreamGeom& g, int grid, const StreamParams& sp,
                                 cudaStream_t s, bool pdl = false) {
  static std::atomic<uint64_t> attrs{0};
  cudaError_t set = cudaSuccess;
  once_per_device(attrs, [&set] {
    // the opt-in limit covers static + dynamic shared memory (227 KB per CTA)
    auto opt_in = [&set](auto* fn) {
      cudaFuncAttributes fa{};
      cudaError_t e = cudaFuncGetAttributes(&fa, fn);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 227 * 1024 - static_cast<int>(fa.sharedSizeBytes));
      if (e != cudaSuccess && set == cudaSuccess) set = e;
    };
    opt_in(stream_gemv_kernel<MODE, 8>);
    opt_in(stream_gemv_kernel<MODE, 4>);
    opt_in(stream_gemv_kernel<MODE, 2>);
  });
  if (set != cudaSuccess) return set;
  StreamParams p = sp;
  p.cb = g.cb;
  p.ncb = g.ncb;
  p.stages = g.stages;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(kStreamThreads);
  lc.dynamicSmemBytes = g.smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (g.rpb == 8) return cudaLaunchKernelEx(&lc, stream_gemv_kernel<MODE, 8>, p);
  if (g.rpb == 4) return cudaLaunchKernelEx(&lc, stream_gemv_kernel<MODE, 4>, p);
  return cudaLaunchKernelEx(&lc, stream_gemv_kernel<MODE, 2>, p);
}

}  // namespace moe
