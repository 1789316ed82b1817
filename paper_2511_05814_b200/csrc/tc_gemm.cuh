// K4: grouped bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA) for the
// prefill path, where token batches make the expert FFN a real contraction.
//
//   for every group g (an expert, or the single mixing map):
//     acc[m][n] = sum_k A[a_row0(g) + m][k] * B[b_row(g, n)][k]        (A, B bf16, K-major)
//   followed by a fused epilogue (mixing residual, SwiGLU, or the down projection's scatter
//   into the per-(token, slot) outputs).
//
// One persistent CTA per SM walks a device-resident tile table (group, m0, n0), so the host
// never learns how many tokens each expert received.  Warp roles:
//   warp 0      TMA producer: A box 128x64 + two B boxes 128x64 per k-step into a 4-stage ring
//   warp 1      MMA issuer: one thread issues tcgen05.mma 128x256x16 into TMEM
//   warp 2      TMEM allocator (512 columns = two 128x256 f32 accumulators)
//   warps 4..7  epilogue: tcgen05.ld (each thread owns one accumulator row) -> fused math ->
//               global stores; the second accumulator lets the next tile's MMAs overlap it.
// Tiles: BM = 128 rows (UMMA M), BN = 256 columns (UMMA N), BK = 64 (one 128-byte swizzle row).
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

namespace moe {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;                    // 16 KB
constexpr int B_STAGE = BN * BK * 2;                    // 32 KB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024; // + alignment slack
constexpr int THREADS = 256;
constexpr int TMEM_COLS = 512;

enum Epilogue {
  kEpiStoreF32 = 0,  // c[out_row0 + m][n] = acc                         (tests, generic)
  kEpiMix = 1,       // h_mid[m][n] = x[m][n] + alpha * acc               (toymoe.py:140)
  kEpiSwiGLU = 2,    // act[a_row0 + m][n0/2 + c] = bf16(silu(acc_w1) * acc_w3)
  kEpiScatter = 3,   // y[row_map[a_row0 + m]][n] = acc                   (per (token, slot))
};

struct Group {
  int a_row0;  // first A row of the group (rows of a group are contiguous)
  int m;       // rows in the group
  int b_row0;  // first B row (N index 0); SwiGLU: first w1 row
  int b_row1;  // SwiGLU: first w3 row; otherwise unused
  int b_map;   // which B tensor map holds the group's matrix (0 or 1)
};

struct Tile {
  int group, m0, n0;  // n0: output column of the tile (SwiGLU: first act column)
};

struct Params {
  const Tile* tiles;
  const int* n_tiles;  // device count (prepared on the device)
  const Group* groups;
  int K;               // reduction length, multiple of 64
  int N;               // output row length (SwiGLU: f = act row length)
  int epi;
  // epilogue operands
  float* c;            // kEpiStoreF32: [rows][N]
  const float* x;      // kEpiMix: residual input [rows][N]
  float* h_mid;        // kEpiMix: output [rows][N]
  float alpha;
  uint16_t* act;       // kEpiSwiGLU: [rows][N] bf16
  const int* row_map;  // kEpiScatter: A row -> output row
  float* y;            // kEpiScatter: [out rows][N]
  // split-K (kEpiStoreF32 / kEpiScatter): tile list walked `splits` times, split s reducing
  // k-blocks [s*nk/splits, (s+1)*nk/splits) into its own output plane c/y + s*split_stride;
  // the consumer sums the planes in split order (deterministic, no atomics)
  int splits;
  long long split_stride;
  // optional profiling slot [2]: max(LLONG_MAX - CTA start ns), max(CTA end ns) (globaltimer)
  long long* prof;
};

__device__ __forceinline__ float silu_mul(float a1, float a3) {
  return a1 / (1.f + expf(-a1)) * a3;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

#ifdef MOE_TC_GEMM_KERNEL  // defined by tc_gemm.cu only: the one TU that owns the kernel
__global__ void __launch_bounds__(THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b0,
                        const __grid_constant__ CUtensorMap tmap_b1, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                        // [STAGES][A_STAGE]
  uint8_t* sb = smem + STAGES * A_STAGE;     // [STAGES][B_STAGE]
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&p.prof[0], 0x7fffffffffffffffll - static_cast<long long>(t));
  }
  const int nbase = *p.n_tiles;
  const int splits = p.splits > 1 ? p.splits : 1;
  const int ntiles = nbase * splits;
  const int nk = p.K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    mbar_fence_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b0);
    tma_prefetch_desc(&tmap_b1);
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol_a = evict_last_policy();   // activations: re-read by every N tile
      const uint64_t pol_b = evict_first_policy();  // weights: streamed
      int it = 0;
      for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const Tile t = p.tiles[ti % nbase];
        const int sp = ti / nbase;
        const int kb0 = sp * nk / splits, kb1 = (sp + 1) * nk / splits;
        const Group g = p.groups[t.group];
        const int arow = g.a_row0 + t.m0;
        const void* tmap_b = g.b_map ? static_cast<const void*>(&tmap_b1) : static_cast<const void*>(&tmap_b0);
        int brow0, brow1;
        if (p.epi == kEpiSwiGLU) {
          brow0 = g.b_row0 + t.n0;
          brow1 = g.b_row1 + t.n0;
        } else {
          brow0 = g.b_row0 + t.n0;
          brow1 = brow0 + BN / 2;
        }
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(sa + s * A_STAGE, &tmap_a, &full[s], kb * BK, arow, pol_a);
          tma_load_2d(sb + s * B_STAGE, tmap_b, &full[s], kb * BK, brow0, pol_b);
          tma_load_2d(sb + s * B_STAGE + B_STAGE / 2, tmap_b, &full[s], kb * BK, brow1, pol_b);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int it = 0, lt = 0;
      for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++lt) {
        const int acc = lt & 1;
        mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int sp = ti / nbase;
        const int kb0 = sp * nk / splits, kb1 = (sp + 1) * nk / splits;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sa + s * A_STAGE), b0 = smem_u32(sb + s * B_STAGE);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
        }
        umma_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;       // accumulator row owned by this thread
    int lt = 0;
    for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const Tile t = p.tiles[ti % nbase];
      const long long plane = static_cast<long long>(ti / nbase) * p.split_stride;
      const Group g = p.groups[t.group];
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + acc * BN + (static_cast<uint32_t>(q * 32) << 16);
      const bool valid = t.m0 + r < g.m;
      const int arow = g.a_row0 + t.m0 + r;
      if (p.epi == kEpiSwiGLU) {
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t v1[32], v3[32];
          tmem_ld32(tbase + c, v1);
          tmem_ld32(tbase + BN / 2 + c, v3);
          tmem_ld_wait();
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(p.act + static_cast<size_t>(arow) * p.N + t.n0 + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint4 o;
              o.x = pack_bf16(silu_mul(__uint_as_float(v1[8 * i + 0]), __uint_as_float(v3[8 * i + 0])),
                              silu_mul(__uint_as_float(v1[8 * i + 1]), __uint_as_float(v3[8 * i + 1])));
              o.y = pack_bf16(silu_mul(__uint_as_float(v1[8 * i + 2]), __uint_as_float(v3[8 * i + 2])),
                              silu_mul(__uint_as_float(v1[8 * i + 3]), __uint_as_float(v3[8 * i + 3])));
              o.z = pack_bf16(silu_mul(__uint_as_float(v1[8 * i + 4]), __uint_as_float(v3[8 * i + 4])),
                              silu_mul(__uint_as_float(v1[8 * i + 5]), __uint_as_float(v3[8 * i + 5])));
              o.w = pack_bf16(silu_mul(__uint_as_float(v1[8 * i + 6]), __uint_as_float(v3[8 * i + 6])),
                              silu_mul(__uint_as_float(v1[8 * i + 7]), __uint_as_float(v3[8 * i + 7])));
              dst[i] = o;
            }
          }
        }
      } else {
        float* out = nullptr;
        const float* res = nullptr;
        if (valid) {
          if (p.epi == kEpiStoreF32) {
            out = p.c + plane + static_cast<size_t>(arow) * p.N + t.n0;
          } else if (p.epi == kEpiMix) {
            out = p.h_mid + static_cast<size_t>(arow) * p.N + t.n0;
            res = p.x + static_cast<size_t>(arow) * p.N + t.n0;
          } else {
            out = p.y + plane + static_cast<size_t>(p.row_map[arow]) * p.N + t.n0;
          }
        }
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c, v);
          tmem_ld_wait();
          if (valid) {
            float4* dst = reinterpret_cast<float4*>(out + c);
            if (res) {
              const float4* src = reinterpret_cast<const float4*>(res + c);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 xr = src[i];
                float4 o;
                o.x = __fadd_rn(xr.x, __fmul_rn(p.alpha, __uint_as_float(v[4 * i + 0])));
                o.y = __fadd_rn(xr.y, __fmul_rn(p.alpha, __uint_as_float(v[4 * i + 1])));
                o.z = __fadd_rn(xr.z, __fmul_rn(p.alpha, __uint_as_float(v[4 * i + 2])));
                o.w = __fadd_rn(xr.w, __fmul_rn(p.alpha, __uint_as_float(v[4 * i + 3])));
                dst[i] = o;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                dst[i] = make_float4(__uint_as_float(v[4 * i + 0]), __uint_as_float(v[4 * i + 1]),
                                     __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<TMEM_COLS>(tmem_base);
  if (p.prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&p.prof[1], static_cast<long long>(t));
  }
}
#endif  // MOE_TC_GEMM_KERNEL

}  // namespace tc
}  // namespace moe
