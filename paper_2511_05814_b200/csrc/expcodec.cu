// Exponent codec for expert transfers (expcodec.cuh): multi-threaded host encoder, GPU decoder.
#include "common.cuh"
#include "expcodec.cuh"

#include <algorithm>
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

// One CTA per 4096-weight chunk, four independent warps of 1024 weights, 32 per lane.
// Per lane: (1) its level-1 escapes (zero 2-bit codes) ranked by a warp scan; (2) their
// level-2 codes read as one bit run and turned into exponent bytes by byte permutes through
// an 8-entry table (the rare zero level-2 codes take an escape byte); (3) each group of four
// weights resolved by one byte permute -- level-1 exponents from a 3-entry table, level-2
// values from the head of the lane's value stream -- with the selector from kExpand;
// (4) bf16 words from the exponent and sign|mantissa bytes by byte permutes.
__global__ void __launch_bounds__(kThreads) decode23_kernel(const PartBatch pb,
                                                            long long* __restrict__ prof) {
  __shared__ uint32_t stab[256];
  stab[threadIdx.x] = kExpand.v[threadIdx.x];
  stab[threadIdx.x + kThreads] = kExpand.v[threadIdx.x + kThreads];
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
  if (prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&prof[0], 0x7fffffffffffffffll - static_cast<long long>(t));
  }
  const PartHeader& h = *reinterpret_cast<const PartHeader*>(part);
  const uint32_t c = blockIdx.x - pstart;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the chunk entry as three 8-byte words (ChunkEntry: esc_off, l2_off | base, win,
  // l2_rel[0] | l2_rel[1..2] | esc_rel[0..1] | esc_rel[2], pad); this warp's offsets picked
  // by shifts (no indexed local copy)
  const uint2* ep = reinterpret_cast<const uint2*>(part + align16(sizeof(PartHeader))) + 3 * c;
  const uint2 e0 = ep[0], e1 = ep[1], e2 = ep[2];
  const uint32_t l2_rel = warp == 0 ? 0u : warp == 1 ? e1.x >> 16 : warp == 2 ? e1.y & 0xFFFFu : e1.y >> 16;
  const uint32_t esc_rel = warp == 0 ? 0u : warp == 1 ? e2.x & 0xFFFFu : warp == 2 ? e2.x >> 16 : e2.y & 0xFFFFu;
  const uint64_t first = static_cast<uint64_t>(c) * kChunk + threadIdx.x * 32ull;
  const bool active = first < h.n;
  const int cnt = active ? static_cast<int>(h.n - first < 32 ? h.n - first : 32) : 0;
  uint32_t lo[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t c0 = 0;   // the lane's 32 level-1 codes, weight j at bits 2j
  if (active) {
    const uint4* lp = reinterpret_cast<const uint4*>(part + h.low_off + first);
    const uint4 l0 = lp[0], l1 = lp[1];
    lo[0] = l0.x; lo[1] = l0.y; lo[2] = l0.z; lo[3] = l0.w;
    lo[4] = l1.x; lo[5] = l1.y; lo[6] = l1.z; lo[7] = l1.w;
    const uint2 q = *reinterpret_cast<const uint2*>(part + h.code_off + first / 4);
    c0 = (static_cast<uint64_t>(q.y) << 32) | q.x;
  }
  uint64_t zm = ~(c0 | (c0 >> 1)) & 0x5555555555555555ull;   // bit 2j: weight j escapes
  if (cnt < 32) zm &= (1ull << (2 * cnt)) - 1ull;               // (cnt = 0: no escapes)
  const int nh0 = __popc(static_cast<uint32_t>(zm)), n1 = nh0 + __popc(static_cast<uint32_t>(zm >> 32));
  const int before1 = warp_exclusive_sum(n1, lane);
  // chunk tables: level 1 (byte c = exponent of 2-bit code c = base - (win + c - 1)) and
  // level 2 (byte c = exponent of 3-bit code c: r = w2 + c - 1, dl = r < win ? r : r + 3).
  // Bytes of codes a chunk cannot hold (dl > base) may borrow from higher bytes, which are
  // unused codes too; byte 0 (the escape code) is never read.
  const uint32_t base = e1.x & 0xFFu, win = (e1.x >> 8) & 0xFFu, w2 = win > 2u ? win - 2u : 0u, d = win - w2;
  const uint32_t lut1 = (base - win) * 0x01010100u - 0x02010000u;
  const uint32_t b4 = base * 0x01010101u;
  const uint32_t lut2lo = b4 - (w2 * 0x01010100u + 0x02010000u + (d == 0 ? 0x03030300u : d == 1 ? 0x03030000u : 0x03000000u));
  const uint32_t lut2hi = b4 - (w2 * 0x01010101u + 0x06050403u + 0x03030303u);
  // level-2 values of each half (16 weights: at most 16 escapes), as a byte stream in 4 words
  const uint32_t* l2w = reinterpret_cast<const uint32_t*>(part + h.l2_off);
  const uint64_t l2base = static_cast<uint64_t>(e0.y) + l2_rel + before1;
  uint32_t v[2][4];
  uint32_t zq[2][4];   // zero level-2 codes: bit 4i of quartet q = code 4q + i of the half
  int n2 = 0;
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    const int nh = hf ? n1 - nh0 : nh0;
    uint64_t x = 0;
    if (nh) {
      const uint64_t bit = (l2base + (hf ? nh0 : 0)) * 3ull;
      const uint32_t* wp = l2w + (bit >> 5);
      const uint32_t s = static_cast<uint32_t>(bit & 31);
      const uint32_t w0 = wp[0], w1 = wp[1], w2w = wp[2];
      x = (static_cast<uint64_t>(__funnelshift_r(w1, w2w, s)) << 32) | __funnelshift_r(w0, w1, s);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[hf][q] = 0;
      zq[hf][q] = 0;
      // quartets 2, 3 only when some lane of the warp needs them (rare past 8 escapes)
      if (q < 2 || __any_sync(0xffffffffu, nh > 4 * q)) {
        const uint32_t sel = nib3(static_cast<uint32_t>(x >> (12 * q)) & 0xFFFu);
        v[hf][q] = __byte_perm(lut2lo, lut2hi, sel);
        uint32_t z = ~(sel | (sel >> 1) | (sel >> 2)) & 0x1111u;
        const int valid = nh - 4 * q;   // codes of this quartet that belong to the lane
        z &= valid >= 4 ? 0x1111u : valid <= 0 ? 0u : (0x1111u >> (4 * (4 - valid)));
        zq[hf][q] = z;
        n2 += __popc(z);
      }
    }
  }
  // rare: zero level-2 codes take the next escape bytes (weight order across the warp)
  if (__any_sync(0xffffffffu, n2)) {
    const int before2 = warp_exclusive_sum(n2, lane);
    const uint8_t* esc = part + h.esc_off + e0.x + esc_rel + before2;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        for (uint32_t z = zq[hf][q]; z; z &= z - 1u) {
          const int i = (__ffs(z) - 1) >> 2;
          const uint32_t sh = 8u * i;
          v[hf][q] = (v[hf][q] & ~(0xFFu << sh)) | (static_cast<uint32_t>(*esc++) << sh);
        }
  }
  __syncthreads();   // stab
  if (!active) return;
  uint32_t o[16];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    uint32_t v0 = v[hf][0], v1 = v[hf][1], v2 = v[hf][2], v3 = v[hf][3];
#pragma unroll
    for (int gq = 0; gq < 4; ++gq) {
      const int g = 4 * hf + gq;
      const uint32_t e = stab[static_cast<uint32_t>(c0 >> (8 * g)) & 0xFFu];
      const uint32_t X = __byte_perm(v0, lut1, e);
      if (gq < 3) {   // advance the value stream past this group's escapes
        const uint32_t sh = e >> 16;
        v0 = __funnelshift_rc(v0, v1, sh);
        v1 = __funnelshift_rc(v1, v2, sh);
        v2 = __funnelshift_rc(v2, v3, sh);
        v3 = __funnelshift_rc(v3, 0u, sh);
      }
      bf16x4(lo[g], X, o[2 * g], o[2 * g + 1]);
    }
  }
  store_out(out, first, cnt, o);
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
  if (kb == 3)
    decode_kernel<3><<<grid, kThreads, 0, s>>>(pb, prof);
  else if (kb == 4)
    decode_kernel<4><<<grid, kThreads, 0, s>>>(pb, prof);
  else
    decode23_kernel<<<grid, kThreads, 0, s>>>(pb, prof);
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
