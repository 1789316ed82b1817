// Exponent codec for expert transfers (expcodec.cuh): multi-threaded host encoder, GPU decoder.
#include "common.cuh"
#include "expcodec.cuh"
#include "sm100.cuh"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace moe {
namespace xc {

namespace {

inline int expo(uint16_t w) { return (w >> 7) & 0xFF; }

struct ChunkStats {
  uint8_t base, win;
  uint32_t e3, e4, l2, l3;  // escapes of mode 3 / 4; mode 23 level-2 codes and byte escapes
};

struct Plan {
  int mode;
  uint32_t nch;
  std::vector<ChunkStats> st;
  std::vector<uint32_t> esc_off, l2_off;
  uint64_t low_off, code_off, l2_off_b, esc_off_b, total;
};

template <class F>
void parallel_chunks(uint32_t nch, F f) {
  unsigned nth = std::max(1u, std::min(std::thread::hardware_concurrency(), 64u));
  if (nch < 64) nth = 1;
  std::vector<std::thread> th;
  for (unsigned i = 0; i < nth; ++i)
    th.emplace_back([&, i] {
      for (uint32_t c = nch * static_cast<uint64_t>(i) / nth; c < nch * static_cast<uint64_t>(i + 1) / nth; ++c) f(c);
    });
  for (auto& t : th) t.join();
}

Plan make_plan(const uint16_t* in, uint64_t n, int mode_req) {
  Plan p{};
  p.nch = static_cast<uint32_t>((n + kChunk - 1) / kChunk);
  p.st.assign(p.nch, ChunkStats{});
  parallel_chunks(p.nch, [&](uint32_t c) {
    const uint64_t a = static_cast<uint64_t>(c) * kChunk, b = std::min<uint64_t>(n, a + kChunk);
    int mx = 0;
    for (uint64_t i = a; i < b; ++i) mx = std::max(mx, expo(in[i]));
    uint32_t hist[256] = {};
    for (uint64_t i = a; i < b; ++i) ++hist[mx - expo(in[i])];
    ChunkStats s{static_cast<uint8_t>(mx), 0, 0, 0, 0, 0};
    for (int dl = 0; dl < 256; ++dl) {
      s.e3 += dl >= 7 ? hist[dl] : 0;
      s.e4 += dl >= 15 ? hist[dl] : 0;
    }
    // mode 23 window: level 1 covers dl in [w, w + 3), level 2 the 7 ranks r from w2 =
    // max(0, w - 2) (r = dl below the window, dl - 3 above it); the rest are escape bytes
    uint64_t best = ~0ull;
    const uint32_t cnt = static_cast<uint32_t>(b - a);
    for (int w = 0; w <= mx; ++w) {
      const int w2 = w > 2 ? w - 2 : 0;
      uint32_t in1 = 0, in2 = 0;
      for (int dl = w; dl < w + 3 && dl < 256; ++dl) in1 += hist[dl];
      for (int r = w2; r < w2 + 7; ++r) {
        const int dl = r < w ? r : r + 3;
        if (dl < 256) in2 += hist[dl];
      }
      const uint32_t l2 = cnt - in1, l3 = l2 - in2;
      const uint64_t cost = 3ull * l2 + 8ull * l3;
      if (cost < best) best = cost, s.win = static_cast<uint8_t>(w), s.l2 = l2, s.l3 = l3;
    }
    p.st[c] = s;
  });
  uint64_t t3 = 0, t4 = 0, tl2 = 0, tl3 = 0;
  for (const auto& s : p.st) {
    t3 += s.e3;
    t4 += s.e4;
    tl2 += s.l2;
    tl3 += s.l3;
  }
  const uint64_t head = align16(sizeof(PartHeader)) + align16(sizeof(ChunkEntry) * p.nch) + align16(n);
  const uint64_t s3 = head + align16((n * 3 + 7) / 8) + align16(t3);
  const uint64_t s4 = head + align16((n * 4 + 7) / 8) + align16(t4);
  const uint64_t s23 = head + align16((n * 2 + 7) / 8) + align16(tl2 * 3 / 8 + 16) + align16(tl3);
  if (mode_req == 3 || mode_req == 4 || mode_req == kMode23) {
    p.mode = mode_req;
  } else {
    p.mode = s23 <= s3 && s23 <= s4 ? kMode23 : (s3 <= s4 ? 3 : 4);
  }
  p.esc_off.assign(p.nch, 0);
  p.l2_off.assign(p.nch, 0);
  uint32_t run = 0, run2 = 0;
  for (uint32_t c = 0; c < p.nch; ++c) {
    const auto& s = p.st[c];
    p.esc_off[c] = run;
    p.l2_off[c] = run2;
    run += p.mode == 3 ? s.e3 : p.mode == 4 ? s.e4 : s.l3;
    run2 += p.mode == kMode23 ? s.l2 : 0;
  }
  p.low_off = align16(sizeof(PartHeader)) + align16(sizeof(ChunkEntry) * p.nch);
  p.code_off = p.low_off + align16(n);
  const int k1 = p.mode == kMode23 ? 2 : p.mode;
  p.l2_off_b = p.code_off + align16((n * k1 + 7) / 8);
  p.esc_off_b = p.l2_off_b + (p.mode == kMode23 ? align16(static_cast<uint64_t>(run2) * 3 / 8 + 16) : 0);
  p.total = p.esc_off_b + align16(run);
  return p;
}

// bit-stream writer: `k`-bit value at bit position `bit` (little-endian within bytes)
inline void put_bits(uint8_t* plane, uint64_t bit, uint32_t v, int k) {
  uint8_t* q = plane + (bit >> 3);
  const uint32_t sh = bit & 7;
  const uint32_t x = v << sh;
  q[0] |= static_cast<uint8_t>(x);
  if (sh + k > 8) q[1] |= static_cast<uint8_t>(x >> 8);
}

}  // namespace

uint64_t encoded_size(const uint16_t* in, uint64_t n, int mode) { return make_plan(in, n, mode).total; }

uint64_t encode(const uint16_t* in, uint64_t n, int mode_req, uint8_t* out) {
  const Plan p = make_plan(in, n, mode_req);
  memset(out, 0, p.total);
  PartHeader h{};
  h.magic = kMagic;
  h.kbits = static_cast<uint32_t>(p.mode);
  h.n = n;
  h.nch = p.nch;
  h.low_off = p.low_off;
  h.code_off = p.code_off;
  h.l2_off = p.l2_off_b;
  h.esc_off = p.esc_off_b;
  h.total = p.total;
  memcpy(out, &h, sizeof(h));
  ChunkEntry* ce = reinterpret_cast<ChunkEntry*>(out + align16(sizeof(PartHeader)));
  uint8_t* low = out + p.low_off;
  uint8_t* codes = out + p.code_off;
  uint8_t* l2 = out + p.l2_off_b;
  uint8_t* escb = out + p.esc_off_b;
  parallel_chunks(p.nch, [&](uint32_t c) {
    ChunkEntry e{};
    e.esc_off = p.esc_off[c];
    e.l2_off = p.l2_off[c];
    e.base = p.st[c].base;
    e.win = p.mode == kMode23 ? p.st[c].win : 0;
    ce[c] = e;
    const uint64_t a = static_cast<uint64_t>(c) * kChunk, b = std::min<uint64_t>(n, a + kChunk);
    uint32_t ei = p.esc_off[c];
    uint64_t l2i = p.l2_off[c];
    const int base = p.st[c].base, win = e.win;
    // chunks start on whole bytes of the low and level-1 planes (kChunk * k bits); mode 23's
    // level-2 codes run on across chunks, each warp's start recorded in the chunk entry
    for (uint64_t i = a; i < b; ++i) {
      const uint16_t w = in[i];
      if (p.mode == kMode23 && i > a && (i - a) % kWarpWeights == 0) {
        const int wq = static_cast<int>((i - a) / kWarpWeights) - 1;
        ce[c].l2_rel[wq] = static_cast<uint16_t>(l2i - p.l2_off[c]);
        ce[c].esc_rel[wq] = static_cast<uint16_t>(ei - p.esc_off[c]);
      }
      low[i] = static_cast<uint8_t>(((w >> 8) & 0x80) | (w & 0x7F));
      const int dl = base - expo(w);
      if (p.mode == kMode23) {
        const uint32_t c1 = dl >= win && dl < win + 3 ? static_cast<uint32_t>(dl - win + 1) : 0u;
        put_bits(codes, i * 2, c1, 2);
        if (!c1) {
          const int r = dl < win ? dl : dl - 3, w2 = win > 2 ? win - 2 : 0;
          const uint32_t c2 = r >= w2 && r < w2 + 7 ? static_cast<uint32_t>(r - w2 + 1) : 0u;
          put_bits(l2, l2i * 3, c2, 3);
          ++l2i;
          if (!c2) escb[ei++] = static_cast<uint8_t>(expo(w));
        }
      } else {
        const int lim = (1 << p.mode) - 1;
        const uint32_t code = dl < lim ? static_cast<uint32_t>(dl + 1) : 0u;
        put_bits(codes, i * p.mode, code, p.mode);
        if (!code) escb[ei++] = static_cast<uint8_t>(expo(w));
      }
    }
  });
  return p.total;
}

// CTA-wide exclusive scan of one int per thread (element order = thread order).
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int before = incl - v;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  __syncthreads();  // warp_tot may be reused by a second scan
  return before;
}

__device__ __forceinline__ void store_out(uint16_t* out, uint64_t first, int cnt, const uint32_t (&o)[16]) {
  if (cnt == 32) {
    uint4* op = reinterpret_cast<uint4*>(out + first);
    op[0] = make_uint4(o[0], o[1], o[2], o[3]);
    op[1] = make_uint4(o[4], o[5], o[6], o[7]);
    op[2] = make_uint4(o[8], o[9], o[10], o[11]);
    op[3] = make_uint4(o[12], o[13], o[14], o[15]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < cnt) out[first + j] = static_cast<uint16_t>(o[j >> 1] >> (16 * (j & 1)));
  }
}

__device__ __forceinline__ uint32_t bf16_word(uint32_t b8, uint32_t ex) {
  return ((b8 & 0x80u) << 8) | ((ex & 0xFFu) << 7) | (b8 & 0x7Fu);
}

// bf16 words of 4 weights from their sign+mantissa bytes B and exponent bytes X, packed in
// 32-bit words, as two 32-bit output words (weights 0,1 and 2,3): per byte, the high half
// is sign | ex >> 1, the low half ex & 1 | mantissa; byte permutes interleave them.
__device__ __forceinline__ void bf16x4(uint32_t B, uint32_t X, uint32_t& o01, uint32_t& o23) {
  const uint32_t H = (B & 0x80808080u) | ((X >> 1) & 0x7F7F7F7Fu);
  const uint32_t L = (B & 0x7F7F7F7Fu) | ((X << 7) & 0x80808080u);
  o01 = __byte_perm(L, H, 0x5140);
  o23 = __byte_perm(L, H, 0x7362);
}

// four 2-bit codes (one code byte) spread to the low bits of four bytes
__device__ __forceinline__ uint32_t spread2(uint32_t cb) {
  uint32_t s = (cb | (cb << 12)) & 0x000F000Fu;
  return (s | (s << 6)) & 0x03030303u;
}

// Modes 3 / 4: one CTA per chunk, 32 consecutive weights per thread; escapes ranked by a
// block scan.
template <int K>
__global__ void __launch_bounds__(kThreads) decode_kernel(const PartBatch pb,
                                                          long long* __restrict__ prof) {
  __shared__ int warp_tot[kThreads / 32];
  // which part of the batch this CTA decodes (parts laid out back to back in the grid);
  // constant-indexed parameter reads only (no local copy of the batch)
  const uint8_t* part = pb.part[0];
  uint16_t* out = pb.out[0];
  uint32_t pstart = 0;
#pragma unroll
  for (int q = 1; q < kMaxBatch; ++q)
    if (q < pb.n && blockIdx.x >= pb.start[q]) {
      part = pb.part[q];
      out = pb.out[q];
      pstart = pb.start[q];
    }
  if (prof && threadIdx.x == 0) {  // in-kernel span: max(LLONG_MAX - CTA start), max(end)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[0], 0x7fffffffffffffffll - static_cast<long long>(t));
  }
  const PartHeader& h = *reinterpret_cast<const PartHeader*>(part);
  const uint32_t c = blockIdx.x - pstart;
  const ChunkEntry ce = reinterpret_cast<const ChunkEntry*>(part + align16(sizeof(PartHeader)))[c];
  const uint64_t first = static_cast<uint64_t>(c) * kChunk + threadIdx.x * 32ull;
  const bool active = first < h.n;
  const int cnt = active ? static_cast<int>(h.n - first < 32 ? h.n - first : 32) : 0;
  uint32_t lo[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t c0 = 0, c1 = 0;  // K-bit codes 0..15 / 16..31
  uint32_t escm = 0;        // bit j = weight j escapes to a byte
  if (active) {
    const uint4* lp = reinterpret_cast<const uint4*>(part + h.low_off + first);
    const uint4 l0 = lp[0], l1 = lp[1];
    lo[0] = l0.x; lo[1] = l0.y; lo[2] = l0.z; lo[3] = l0.w;
    lo[4] = l1.x; lo[5] = l1.y; lo[6] = l1.z; lo[7] = l1.w;
    if constexpr (K == 4) {
      const uint4 q = *reinterpret_cast<const uint4*>(part + h.code_off + first / 2);
      c0 = (static_cast<uint64_t>(q.y) << 32) | q.x;
      c1 = (static_cast<uint64_t>(q.w) << 32) | q.z;
    } else {
      const uint32_t* q = reinterpret_cast<const uint32_t*>(part + h.code_off + first * 3 / 8);
      const uint32_t w0 = q[0], w1 = q[1], w2 = q[2];
      c0 = (static_cast<uint64_t>(w1) << 32) | w0;                    // stream bits 0..63
      c1 = (static_cast<uint64_t>(w2) << 16) | (w1 >> 16);            // stream bits 48..95
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint32_t code = static_cast<uint32_t>((j < 16 ? c0 >> (K * j) : c1 >> (K * (j - 16))) & ((1u << K) - 1));
      if (j < cnt && !code) escm |= 1u << j;
    }
  }
  const int before1 = block_exclusive_scan(__popc(escm), warp_tot);
  if (!active) return;
  uint32_t o[16];
  const uint8_t* esc = part + h.esc_off + ce.esc_off + before1;
  int e = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint32_t b8 = (lo[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t code = static_cast<uint32_t>((j < 16 ? c0 >> (K * j) : c1 >> (K * (j - 16))) & ((1u << K) - 1));
    uint32_t ex = static_cast<uint32_t>(ce.base) + 1u - code;
    if ((escm >> j) & 1u) {  // rare: exponent from the side list
      ex = esc[e];
      ++e;
    }
    const uint32_t w = bf16_word(b8, ex);
    if (j & 1) o[j >> 1] |= w << 16;
    else o[j >> 1] = w;
  }
  store_out(out, first, cnt, o);
  if (prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[1], static_cast<long long>(t));
  }
}

// ---- mode 23: warp-independent, table-driven -------------------------------------------
// Expansion selectors for one group of four weights, indexed by its code byte (four 2-bit
// level-1 codes, weight i at bits 2i): nibble i selects byte `rank` of the group's level-2
// value word (operand a of the byte permute) for a zero code, byte 4 + c of the level-1
// table word (operand b: byte c = exponent of code c) otherwise; bits 16.. hold 8 x the
// number of zero codes (how far the value stream advances past the group).
struct ExpandTable {
  uint32_t v[256];
  constexpr ExpandTable() : v() {
    for (int i = 0; i < 256; ++i) {
      uint32_t sel = 0, rank = 0;
      for (int k = 0; k < 4; ++k) {
        const uint32_t code = (static_cast<uint32_t>(i) >> (2 * k)) & 3u;
        sel |= (code ? 4u + code : rank++) << (4 * k);
      }
      v[i] = sel | ((8u * rank) << 16);
    }
  }
};
__device__ constexpr ExpandTable kExpand{};

// twelve bits = four 3-bit codes -> the low bits of four nibbles (a byte-permute selector)
__device__ __forceinline__ uint32_t nib3(uint32_t x) {
  const uint32_t a = (x & 0x3Fu) | ((x << 2) & 0x3F00u);      // codes 0,1 | codes 2,3
  return (a & 0x0707u) | ((a << 1) & 0x7070u);
}

__device__ __forceinline__ int warp_exclusive_sum(int v, int lane) {
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  return incl - v;
}

// per-byte rotate right by one: exponent byte e -> (e >> 1) | (e & 1) << 7, the two halves
// of its bf16 word in place (bits 0..6 -> the high byte, bit 7 -> the low byte)
__device__ __forceinline__ uint32_t ror8x4(uint32_t x) {
  return ((x >> 1) & 0x7F7F7F7Fu) | ((x << 7) & 0x80808080u);
}

// One CTA per 4096-weight chunk, four independent warps of 1024 weights, 32 per lane.
// Per lane: (1) its level-1 escapes (zero 2-bit codes) ranked by a warp scan; (2) their
// level-2 codes read as one bit run and turned into exponent bytes by byte permutes through
// an 8-entry table (zero level-2 codes take the next escape byte); (3) each group of four
// weights resolved by one byte permute -- level-1 exponents from a 3-entry table, level-2
// values from the head of the lane's value stream -- with the selector from kExpand;
// (4) bf16 words from the exponent and sign|mantissa bytes: every table holds its exponents
// rotated (ror8x4), so each half-word is one 3-input logic op, then two byte permutes.
// The part descriptors come from the host copy of the headers (kernel parameters), so the
// chunk's loads issue at once.
__global__ void __launch_bounds__(kThreads) decode23_kernel(const __grid_constant__ Batch23 pb,
                                                            long long* __restrict__ prof) {
  __shared__ uint32_t stab[256];
  __shared__ uint32_t vsm[kThreads * 8];   // escape-byte patching: [warp][word][lane]
  stab[threadIdx.x] = kExpand.v[threadIdx.x];
  stab[threadIdx.x + kThreads] = kExpand.v[threadIdx.x + kThreads];
  const uint32_t bx = blockIdx.x;
  const int pi = (bx >= pb.start[1]) + (bx >= pb.start[2]) + (bx >= pb.start[3]);
  const Part23& P = pb.p[pi];
  const uint8_t* part = P.part;
  if (prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[0], 0x7fffffffffffffffll - static_cast<long long>(t));
  }
  const uint32_t c = bx - pb.start[pi];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 32-bit weight and code indices (decode_batch: n < 2^30)
  const uint32_t n = static_cast<uint32_t>(P.n);
  const uint32_t first = c * kChunk + threadIdx.x * 32u;
  const bool active = first < n;
  const int cnt = active ? static_cast<int>(min(n - first, 32u)) : 0;
  // the chunk entry as three 8-byte words (ChunkEntry: esc_off, l2_off | base, win,
  // l2_rel[0] | l2_rel[1..2] | esc_rel[0..1] | esc_rel[2], pad); this warp's offsets picked
  // by shifts (no indexed local copy)
  const uint2* ep = reinterpret_cast<const uint2*>(part + align16(sizeof(PartHeader))) + 3 * c;
  const uint2 e0 = ep[0], e1 = ep[1], e2 = ep[2];
  uint32_t lo[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint2 cw = make_uint2(0u, 0u);   // the lane's 32 level-1 codes, weight j at bits 2j
  if (active) {
    const uint4* lp = reinterpret_cast<const uint4*>(part + P.low_off + first);
    const uint4 l0 = lp[0], l1 = lp[1];
    lo[0] = l0.x; lo[1] = l0.y; lo[2] = l0.z; lo[3] = l0.w;
    lo[4] = l1.x; lo[5] = l1.y; lo[6] = l1.z; lo[7] = l1.w;
    cw = *reinterpret_cast<const uint2*>(part + P.code_off + first / 4);
  }
  const uint64_t c0 = (static_cast<uint64_t>(cw.y) << 32) | cw.x;
  uint64_t zm = ~(c0 | (c0 >> 1)) & 0x5555555555555555ull;   // bit 2j: weight j escapes
  if (cnt < 32) zm &= (1ull << (2 * cnt)) - 1ull;               // (cnt = 0: no escapes)
  const int nh0 = __popc(static_cast<uint32_t>(zm)), n1 = nh0 + __popc(static_cast<uint32_t>(zm >> 32));
  const int before1 = warp_exclusive_sum(n1, lane);
  const uint32_t l2_rel = warp == 0 ? 0u : warp == 1 ? e1.x >> 16 : warp == 2 ? e1.y & 0xFFFFu : e1.y >> 16;
  // chunk tables: level 1 (byte c = exponent of 2-bit code c = base - (win + c - 1)) and
  // level 2 (byte c = exponent of 3-bit code c: r = w2 + c - 1, dl = r < win ? r : r + 3).
  // Bytes of codes a chunk cannot hold (dl > base) may borrow from higher bytes, which are
  // unused codes too; byte 0 (the escape code) is never read.
  const uint32_t base = e1.x & 0xFFu, win = (e1.x >> 8) & 0xFFu, w2 = win > 2u ? win - 2u : 0u, d = win - w2;
  const uint32_t lut1 = ror8x4((base - win) * 0x01010100u - 0x02010000u);
  const uint32_t b4 = base * 0x01010101u;
  const uint32_t lut2lo = ror8x4(b4 - (w2 * 0x01010100u + 0x02010000u + (d == 0 ? 0x03030300u : d == 1 ? 0x03030000u : 0x03000000u)));
  const uint32_t lut2hi = ror8x4(b4 - (w2 * 0x01010101u + 0x06050403u + 0x03030303u));
  // level-2 values of each half (16 weights: at most 16 escapes), as a byte stream in 4 words
  const uint32_t* l2w = reinterpret_cast<const uint32_t*>(part + P.l2_off);
  const uint32_t l2base = e0.y + l2_rel + before1;
  uint32_t v[2][4];
  uint64_t zt[2];   // zero level-2 codes of each half: bit 3k = code k
  int n2 = 0;
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    const int nh = hf ? n1 - nh0 : nh0;
    uint64_t x = 0;
    if (nh) {
      const uint32_t bit = (l2base + (hf ? nh0 : 0)) * 3u;
      const uint32_t* wp = l2w + (bit >> 5);
      const uint32_t s = bit & 31u;
      const uint32_t w0 = wp[0], w1 = wp[1], w2w = wp[2];
      x = (static_cast<uint64_t>(__funnelshift_r(w1, w2w, s)) << 32) | __funnelshift_r(w0, w1, s);
    }
    zt[hf] = ~(x | (x >> 1) | (x >> 2)) & 0x0000249249249249ull & ((1ull << (3 * nh)) - 1ull);
    n2 += __popcll(zt[hf]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[hf][q] = 0;
      // quartets 2, 3 only when some lane of the warp needs them (past 8 escapes)
      if (q < 2 || __any_sync(0xffffffffu, nh > 4 * q))
        v[hf][q] = __byte_perm(lut2lo, lut2hi, nib3(static_cast<uint32_t>(x >> (12 * q)) & 0xFFFu));
    }
  }
  // zero level-2 codes (~3 per warp on bell-shaped weights) take the next escape bytes, in
  // weight order across the warp
  if (__any_sync(0xffffffffu, n2)) {
    const uint32_t esc_rel = warp == 0 ? 0u : warp == 1 ? e2.x & 0xFFFFu : warp == 2 ? e2.x >> 16 : e2.y & 0xFFFFu;
    int before2;
    if (__all_sync(0xffffffffu, n2 <= 1)) {
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      before2 = __popc(__ballot_sync(0xffffffffu, n2) & lt);
    } else {
      before2 = warp_exclusive_sum(n2, lane);
    }
    const uint8_t* esc = part + P.esc_off + e0.x + esc_rel + before2;
    // patch in shared memory: the lane's 8 value words out ([word][lane], conflict-free),
    // each escape byte stored at its stream position, the words back
    uint32_t* vw = vsm + warp * 256 + lane;
#pragma unroll
    for (int k = 0; k < 8; ++k) vw[32 * k] = v[k >> 2][k & 3];
    uint8_t* vb = reinterpret_cast<uint8_t*>(vsm + warp * 256);
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
      for (uint64_t t = zt[hf]; t; t &= t - 1ull) {
        const uint32_t k = ((__ffsll(static_cast<long long>(t)) - 1) * 43u) >> 7;   // bit 3k -> k
        const uint32_t b = *esc++;
        vb[((4 * hf + (k >> 2)) * 32 + lane) * 4 + (k & 3u)] = static_cast<uint8_t>((b >> 1) | (b << 7));
      }
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k >> 2][k & 3] = vw[32 * k];
  }
  __syncthreads();   // stab
  if (!active) return;
  uint32_t o[16];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    uint32_t v0 = v[hf][0], v1 = v[hf][1], v2 = v[hf][2], v3 = v[hf][3];
    const uint32_t cwh = hf ? cw.y : cw.x;
#pragma unroll
    for (int gq = 0; gq < 4; ++gq) {
      const int g = 4 * hf + gq;
      const uint32_t e = stab[__byte_perm(cwh, 0u, 0x4440u | gq)];
      const uint32_t R = __byte_perm(v0, lut1, e);   // rotated exponent bytes of the group
      if (gq < 3) {   // advance the value stream past this group's escapes
        const uint32_t sh = e >> 16;
        v0 = __funnelshift_rc(v0, v1, sh);
        v1 = __funnelshift_rc(v1, v2, sh);
        v2 = __funnelshift_rc(v2, v3, sh);
        v3 = __funnelshift_rc(v3, 0u, sh);
      }
      // high bytes sign | e >> 1, low bytes e & 1 | mantissa, interleaved into bf16 words
      const uint32_t H = (lo[g] & 0x80808080u) | (R & 0x7F7F7F7Fu);
      const uint32_t L = (lo[g] & 0x7F7F7F7Fu) | (R & 0x80808080u);
      o[2 * g] = __byte_perm(L, H, 0x5140);
      o[2 * g + 1] = __byte_perm(L, H, 0x7362);
    }
  }
  store_out(P.out, first, cnt, o);
  if (prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[1], static_cast<long long>(t));
  }
}

// ---- mode 23, persistent and bulk-copy fed ---------------------------------------------
// The decode of a chunk needs its sign|mantissa bytes, level-1 codes, level-2 codes and escape
// bytes; issued as dependent global loads (entry -> codes -> warp scan -> level-2 words ->
// escape bytes) they leave the kernel latency-bound.  Here a producer warp per CTA streams
// each chunk's four byte ranges into a ring of shared-memory stages with cp.async.bulk (the
// TMA engine; completion on an mbarrier, the entry words alongside), several chunks ahead,
// while four consumer warps decode the previous stages from shared memory and release them.
// CTAs are persistent: CTA b takes chunks b, b + G, b + 2G, ... of the launch.
#ifndef XC_STAGES
#define XC_STAGES 3
#endif
#ifndef XC_LO_GLOBAL
#define XC_LO_GLOBAL 0
#endif
#ifndef XC_MINB
#define XC_MINB 8
#endif
constexpr int kStages23 = XC_STAGES;
constexpr int kL2Win = 1600;   // level-2 window: 4096 codes * 3 bits + alignment and read slack
constexpr int kEscWin = 64;    // escape-byte window (larger runs are read from global memory)
// Per-chunk metadata the producer derives from the chunk entry (lane-uniform work done once):
enum : int {
  kMLut1 = 0, kMLut2lo, kMLut2hi,   // rotated exponent tables (levels 1 and 2)
  kMRem,                            // weights of the chunk (4096 but for a part's last chunk)
  kML2Bit,                          // [4]: each warp's first level-2 code, as a bit of the window
  kMEsc = kML2Bit + 4,              // [4]: each warp's first escape byte (index in the part)
  kMEscWin = kMEsc + 4,             // escape window's first index (0xFFFFFFFF: global memory)
  kMPart,                           // part of the launch
  kMeta = 16
};
struct __align__(16) Stage23 {
#if !XC_LO_GLOBAL
  uint8_t lo[kChunk];
#endif
  uint8_t codes[kChunk / 4];
  uint8_t l2[kL2Win];
  uint8_t esc[kEscWin];
  uint32_t meta[kMeta];
};
constexpr int kThreads23 = kThreads + 32;   // four consumer warps + the producer warp

__device__ __forceinline__ int part_of(const Batch23& pb, uint32_t k) {
  return (k >= pb.start[1]) + (k >= pb.start[2]) + (k >= pb.start[3]);
}

// (a & m) | (b & ~m) as one 3-input logic op
__device__ __forceinline__ uint32_t bitsel(uint32_t m, uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(m), "r"(a), "r"(b));   // m ? a : b (0xF0 ? 0xCC : 0xAA)
  return d;
}

__global__ void __launch_bounds__(kThreads23, XC_MINB) decode23p_kernel(const __grid_constant__ Batch23 pb,
                                                               long long* __restrict__ prof) {
  __shared__ Stage23 stages[kStages23];
  __shared__ uint64_t full[kStages23], empty[kStages23];
  __shared__ uint32_t stab[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256; i += kThreads23) stab[i] = kExpand.v[i];
  if (threadIdx.x == 0) {
    for (int q = 0; q < kStages23; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kThreads / 32);
    }
    mbar_fence_init();
  }
  if (prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[0], 0x7fffffffffffffffll - static_cast<long long>(t));
  }
  __syncthreads();
  const uint32_t G = gridDim.x;
  if (warp == kThreads / 32) {
    // ---------------- producer warp ----------------
    const uint64_t pol = evict_first_policy();   // coded bytes are read once
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};    // lane j: entry words + next chunk's offsets
    int i = 0;
    for (uint32_t k = blockIdx.x; k < pb.chunks; k += G, ++i) {
      if ((i & 31) == 0) {   // the entries of the next 32 chunks, one per lane
        const uint32_t kj = k + lane * G;
        if (kj < pb.chunks) {
          const int pj = part_of(pb, kj);
          const Part23& P = pb.p[pj];
          const uint32_t c = kj - pb.start[pj];
          const uint2* ep = reinterpret_cast<const uint2*>(P.part + align16(sizeof(PartHeader))) + 3 * c;
          const uint2 a = ep[0], b = ep[1], d = ep[2];
          m[0] = a.x; m[1] = a.y; m[2] = b.x; m[3] = b.y; m[4] = d.x; m[5] = d.y;
          if (c + 1 < P.nch) {
            const uint2 f = ep[3];
            m[6] = f.x;   // next chunk's first escape byte
            m[7] = f.y;   // next chunk's first level-2 code
          } else {
            m[6] = m[7] = 0xFFFFFFFFu;   // last chunk: its runs end with their sections
          }
        }
      }
      uint32_t e[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) e[q] = __shfl_sync(0xffffffffu, m[q], i & 31);
      if (lane == 0) {
        const int s = i % kStages23;
        // the producer mostly waits here (the consumers set the pace): back off instead of
        // spinning, so the wait takes no issue slots from the consumer warps
        if (i >= kStages23)
          while (!mbar_try_wait(&empty[s], ((i / kStages23) - 1) & 1)) __nanosleep(64);
        Stage23& st = stages[s];
        const int pi = part_of(pb, k);
        const Part23& P = pb.p[pi];
        const uint32_t c = k - pb.start[pi];
        const uint32_t rem = min(static_cast<uint32_t>(P.n) - c * kChunk, static_cast<uint32_t>(kChunk));
        const uint32_t lo_b = (rem + 15u) & ~15u;
        const uint32_t cd_b = ((rem + 3u) / 4u + 15u) & ~15u;
        // level-2 window [wb, we): whole 16-byte units around the chunk's codes + 16 bytes of
        // read slack, within the section (esc_off - l2_off bytes, a multiple of 16)
        const uint32_t l2sec = static_cast<uint32_t>(P.esc_off - P.l2_off);
        const uint32_t wb = ((3u * e[1]) >> 3) & ~15u;
        uint32_t we = e[7] == 0xFFFFFFFFu ? l2sec : ((((3u * e[7]) + 7u) >> 3) + 15u & ~15u) + 16u;
        if (we > l2sec) we = l2sec;
        // escape window: the chunk's escape bytes if they fit kEscWin from a 16-byte boundary
        const uint32_t escsec = static_cast<uint32_t>(P.total - P.esc_off);
        const uint32_t eb = e[0] & ~15u;
        const uint32_t eend = e[6] == 0xFFFFFFFFu ? escsec : e[6];
        uint32_t esc_b = 0, escw = 0xFFFFFFFFu;
        if (eend <= e[0]) {
          escw = eb;   // no escapes: nothing to read
        } else if (eend - eb <= kEscWin) {
          esc_b = (eend - eb + 15u) & ~15u;
          if (eb + esc_b > escsec) esc_b = escsec - eb;
          escw = eb;
        }
        // tables (chunk-uniform): level 1 byte c = exponent of code c = base - (win + c - 1);
        // level 2 byte c: r = w2 + c - 1, dl = r < win ? r : r + 3.  Bytes of codes a chunk
        // cannot hold (dl > base) may borrow from higher bytes, unused codes too; byte 0 (the
        // escape code) is never read.  Stored rotated (ror8x4).
        const uint32_t base = e[2] & 0xFFu, win = (e[2] >> 8) & 0xFFu, w2 = win > 2u ? win - 2u : 0u, dd = win - w2;
        const uint32_t b4 = base * 0x01010101u;
        uint32_t* mt = st.meta;
        mt[kMLut1] = ror8x4((base - win) * 0x01010100u - 0x02010000u);
        mt[kMLut2lo] = ror8x4(b4 - (w2 * 0x01010100u + 0x02010000u + (dd == 0 ? 0x03030300u : dd == 1 ? 0x03030000u : 0x03000000u)));
        mt[kMLut2hi] = ror8x4(b4 - (w2 * 0x01010101u + 0x06050403u + 0x03030303u));
        mt[kMRem] = rem;
        const uint32_t l2rel[4] = {0u, e[2] >> 16, e[3] & 0xFFFFu, e[3] >> 16};
        const uint32_t escrel[4] = {0u, e[4] & 0xFFFFu, e[4] >> 16, e[5] & 0xFFFFu};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          mt[kML2Bit + w] = 3u * (e[1] + l2rel[w]) - 8u * wb;
          mt[kMEsc + w] = e[0] + escrel[w];
        }
        mt[kMEscWin] = escw;
        mt[kMPart] = static_cast<uint32_t>(pi);
        const uint32_t l2_b = we > wb ? we - wb : 0u;
#if XC_LO_GLOBAL
        mbar_expect_tx(&full[s], cd_b + l2_b + esc_b);
        (void)lo_b;
#else
        mbar_expect_tx(&full[s], lo_b + cd_b + l2_b + esc_b);
        bulk_g2s(st.lo, P.part + P.low_off + static_cast<uint64_t>(c) * kChunk, lo_b, &full[s], pol);
#endif
        bulk_g2s(st.codes, P.part + P.code_off + static_cast<uint64_t>(c) * (kChunk / 4), cd_b, &full[s], pol);
        if (l2_b) bulk_g2s(st.l2, P.part + P.l2_off + wb, l2_b, &full[s], pol);
        if (esc_b) bulk_g2s(st.esc, P.part + P.esc_off + eb, esc_b, &full[s], pol);
      }
      __syncwarp();
    }
    return;
  }
  // ---------------- consumer warps ----------------
  int i = 0;
  for (uint32_t k = blockIdx.x; k < pb.chunks; k += G, ++i) {
    const int s = i % kStages23;
#if XC_LO_GLOBAL
    // sign|mantissa bytes straight from global memory, issued before the stage wait
    uint4 lg0 = make_uint4(0, 0, 0, 0), lg1 = lg0;
    {
      const int pk = part_of(pb, k);
      const Part23& P = pb.p[pk];
      const uint32_t lf = (k - pb.start[pk]) * kChunk + threadIdx.x * 32u;
      if (lf < static_cast<uint32_t>(P.n)) {
        const uint4* lp = reinterpret_cast<const uint4*>(P.part + P.low_off + lf);
        lg0 = __ldcs(lp);
        lg1 = __ldcs(lp + 1);
      }
    }
#endif
    mbar_wait(&full[s], (i / kStages23) & 1);
    const Stage23& st = stages[s];
    const uint4 mq = *reinterpret_cast<const uint4*>(st.meta);   // luts, rem
    const uint32_t lut1 = mq.x, lut2lo = mq.y, lut2hi = mq.z, rem = mq.w;
    const uint32_t l2bit = st.meta[kML2Bit + warp];
    const uint32_t lfirst = threadIdx.x * 32u;   // the lane's first weight in the chunk
    const int cnt = lfirst < rem ? static_cast<int>(min(rem - lfirst, 32u)) : 0;
    uint32_t lo[8];
    {
#if XC_LO_GLOBAL
      const uint4 l0 = lg0, l1 = lg1;
#else
      const uint4* lp = reinterpret_cast<const uint4*>(st.lo + lfirst);
      const uint4 l0 = lp[0], l1 = lp[1];   // (stale bytes past rem: never stored)
#endif
      lo[0] = l0.x; lo[1] = l0.y; lo[2] = l0.z; lo[3] = l0.w;
      lo[4] = l1.x; lo[5] = l1.y; lo[6] = l1.z; lo[7] = l1.w;
    }
    const uint2 cw = *reinterpret_cast<const uint2*>(st.codes + threadIdx.x * 8);
    const uint64_t c0 = (static_cast<uint64_t>(cw.y) << 32) | cw.x;
    uint64_t zm = ~(c0 | (c0 >> 1)) & 0x5555555555555555ull;   // bit 2j: weight j escapes
    if (cnt < 32) zm &= (1ull << (2 * cnt)) - 1ull;
    const int nh0 = __popc(static_cast<uint32_t>(zm)), n1 = nh0 + __popc(static_cast<uint32_t>(zm >> 32));
    const int before1 = warp_exclusive_sum(n1, lane);
    const uint32_t* l2w = reinterpret_cast<const uint32_t*>(st.l2);
    uint32_t v[2][4];
    uint64_t zt[2];   // zero level-2 codes of each half: bit 3k = code k
    int n2 = 0;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int nh = hf ? n1 - nh0 : nh0;
      uint64_t x = 0;
      if (nh) {
        const uint32_t bit = l2bit + 3u * static_cast<uint32_t>(before1 + (hf ? nh0 : 0));
        const uint32_t* wp = l2w + (bit >> 5);
        const uint32_t sft = bit & 31u;
        const uint32_t w0 = wp[0], w1 = wp[1], w2w = wp[2];
        x = (static_cast<uint64_t>(__funnelshift_r(w1, w2w, sft)) << 32) | __funnelshift_r(w0, w1, sft);
      }
      zt[hf] = ~(x | (x >> 1) | (x >> 2)) & 0x0000249249249249ull & ((1ull << (3 * nh)) - 1ull);
      n2 += __popcll(zt[hf]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[hf][q] = 0;
        if (q < 2 || __any_sync(0xffffffffu, nh > 4 * q))
          v[hf][q] = __byte_perm(lut2lo, lut2hi, nib3(static_cast<uint32_t>(x >> (12 * q)) & 0xFFFu));
      }
    }
    // zero level-2 codes (~3 per warp on bell-shaped weights) take the next escape bytes, in
    // weight order across the warp
    if (__any_sync(0xffffffffu, n2)) {
      int before2;
      if (__all_sync(0xffffffffu, n2 <= 1)) {
        unsigned lt;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
        before2 = __popc(__ballot_sync(0xffffffffu, n2) & lt);
      } else {
        before2 = warp_exclusive_sum(n2, lane);
      }
      const uint32_t escw = st.meta[kMEscWin];
      const uint32_t ei = st.meta[kMEsc + warp] + before2;   // the lane's first escape byte
      const uint8_t* esc;
      if (escw != 0xFFFFFFFFu) {
        esc = st.esc + (ei - escw);
      } else {
        const Part23& P = pb.p[st.meta[kMPart]];
        esc = P.part + P.esc_off + ei;
      }
      // patched in registers: each escape byte is merged into the one value word (of the
      // half's four) that holds its stream position, by a masked select per word
#pragma unroll
      for (int hf = 0; hf < 2; ++hf)
        for (uint64_t t = zt[hf]; t; t &= t - 1ull) {
          const uint32_t kk = ((__ffsll(static_cast<long long>(t)) - 1) * 43u) >> 7;   // bit 3k -> k
          const uint32_t b = *esc++;
          const uint32_t sh = 8u * (kk & 3u), wq = kk >> 2;
          const uint32_t m = 0xFFu << sh, val = (((b >> 1) | (b << 7)) & 0xFFu) << sh;
#pragma unroll
          for (int q = 0; q < 4; ++q) v[hf][q] = bitsel(wq == static_cast<uint32_t>(q) ? m : 0u, val, v[hf][q]);
        }
    }
    const int pi = static_cast<int>(st.meta[kMPart]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with the stage
    if (cnt > 0) {
      uint32_t o[16];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t v0 = v[hf][0], v1 = v[hf][1], v2 = v[hf][2], v3 = v[hf][3];
        const uint32_t cwh = hf ? cw.y : cw.x;
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) {
          const int g = 4 * hf + gq;
          const uint32_t e = stab[__byte_perm(cwh, 0u, 0x4440u | gq)];
          const uint32_t R = __byte_perm(v0, lut1, e);   // rotated exponent bytes of the group
          if (gq < 3) {   // advance the value stream past this group's escapes
            const uint32_t sh = e >> 16;
            v0 = __funnelshift_rc(v0, v1, sh);
            v1 = __funnelshift_rc(v1, v2, sh);
            v2 = __funnelshift_rc(v2, v3, sh);
            v3 = __funnelshift_rc(v3, 0u, sh);
          }
          // high bytes sign | e >> 1, low bytes e & 1 | mantissa, interleaved into bf16 words
          const uint32_t H = bitsel(0x80808080u, lo[g], R);
          const uint32_t L = bitsel(0x80808080u, R, lo[g]);
          o[2 * g] = __byte_perm(L, H, 0x5140);
          o[2 * g + 1] = __byte_perm(L, H, 0x7362);
        }
      }
      const Part23& P = pb.p[pi];
      store_out(P.out, static_cast<uint64_t>(k - pb.start[pi]) * kChunk + lfirst, cnt, o);
    }
  }
  if (prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[1], static_cast<long long>(t));
  }
}

moe_status decode_batch(const void* const* parts_dev, const PartHeader* hs, uint16_t* const* outs_dev,
                        int n, cudaStream_t s, long long* prof) {
  MOE_REQUIRE(n >= 1 && n <= kMaxBatch, "1..%d parts per decode launch, got %d", kMaxBatch, n);
  PartBatch pb{};
  uint32_t grid = 0;
  int kb = 0, m = 0;
  for (int i = 0; i < n; ++i) {
    const PartHeader& h = hs[i];
    MOE_REQUIRE(h.magic == kMagic && (h.kbits == 3 || h.kbits == 4 || h.kbits == kMode23),
                "not an exponent-coded part");
    if (h.n == 0) continue;
    MOE_REQUIRE(kb == 0 || static_cast<int>(h.kbits) == kb, "parts of one launch share a code mode");
    kb = static_cast<int>(h.kbits);
    pb.part[m] = static_cast<const uint8_t*>(parts_dev[i]);
    pb.out[m] = outs_dev[i];
    pb.start[m] = grid;
    grid += h.nch;
    ++m;
  }
  if (m == 0) return MOE_OK;
  pb.n = m;
  if (kb == kMode23) {
    // mode 23 takes each part's section offsets as parameters (from the host header copy)
    Batch23 b{};
    for (int q = 0; q < kMaxBatch; ++q) b.start[q] = 0xFFFFFFFFu;
    for (int i = 0, j = 0; i < n; ++i) {
      if (hs[i].n == 0) continue;
      MOE_REQUIRE(hs[i].n < (1ull << 30), "a mode-23 part holds < 2^30 weights, got %llu",
                  (unsigned long long)hs[i].n);
      b.p[j] = Part23{pb.part[j], pb.out[j], hs[i].n, hs[i].low_off, hs[i].code_off, hs[i].l2_off,
                      hs[i].esc_off, hs[i].total, hs[i].nch};
      b.start[j] = pb.start[j];
      ++j;
    }
    b.chunks = grid;
    static const bool simple = getenv("MOE_XC_SIMPLE") != nullptr;   // A/B: one CTA per chunk
    if (simple) {
      decode23_kernel<<<grid, kThreads, 0, s>>>(b, prof);
    } else {
      // persistent: every CTA slot of the device, capped by the chunk count
      static std::atomic<uint64_t> occ_done{0};
      static int occ[64] = {};
      int dev = 0;
      MOE_CUDA(cudaGetDevice(&dev));
      once_per_device(occ_done, [&] {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode23p_kernel, kThreads23, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        occ[dev & 63] = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
      });
      const uint32_t g = std::min<uint32_t>(grid, static_cast<uint32_t>(occ[dev & 63]));
      decode23p_kernel<<<g, kThreads23, 0, s>>>(b, prof);
    }
    MOE_LAUNCHED();
    return MOE_OK;
  }
  if (kb == 3)
    decode_kernel<3><<<grid, kThreads, 0, s>>>(pb, prof);
  else
    decode_kernel<4><<<grid, kThreads, 0, s>>>(pb, prof);
  MOE_LAUNCHED();
  return MOE_OK;
}

moe_status decode(const void* part_dev, const PartHeader& h, uint16_t* out_dev, cudaStream_t s,
                  long long* prof) {
  return decode_batch(&part_dev, &h, &out_dev, 1, s, prof);
}

}  // namespace xc
}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_xc_encode(const uint16_t* in, uint64_t n, int32_t kbits, void* out, uint64_t cap,
                         uint64_t* size) {
  MOE_REQUIRE(size && (in || n == 0), "null argument");
  MOE_REQUIRE(kbits == 0 || kbits == 3 || kbits == 4 || kbits == xc::kMode23,
              "mode must be 0 (auto), 3, 4 or 23");
  if (!out) {
    *size = xc::encoded_size(in, n, kbits);
    return MOE_OK;
  }
  const uint64_t need = xc::encoded_size(in, n, kbits);
  MOE_REQUIRE(cap >= need, "output holds %llu bytes, the part needs %llu",
              (unsigned long long)cap, (unsigned long long)need);
  *size = xc::encode(in, n, kbits, static_cast<uint8_t*>(out));
  return MOE_OK;
}

moe_status moe_xc_decode(const void* part_dev, const void* header_host, uint16_t* out_dev,
                         void* stream) {
  MOE_REQUIRE(part_dev && header_host && out_dev, "null argument");
  xc::PartHeader h;
  memcpy(&h, header_host, sizeof(h));
  return xc::decode(part_dev, h, out_dev, as_stream(stream));
}

}  // extern "C"
