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

struct Plan {
  int kbits;
  uint32_t nch;
  std::vector<uint8_t> base;
  std::vector<uint32_t> esc_off;
  std::vector<uint16_t> n_esc;
  uint64_t low_off, code_off, esc_off_bytes, total, total_esc;
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

Plan make_plan(const uint16_t* in, uint64_t n, int kbits_req) {
  Plan p{};
  p.nch = static_cast<uint32_t>((n + kChunk - 1) / kChunk);
  p.base.assign(p.nch, 0);
  std::vector<uint32_t> esc3(p.nch, 0), esc4(p.nch, 0);
  parallel_chunks(p.nch, [&](uint32_t c) {
    const uint64_t a = static_cast<uint64_t>(c) * kChunk, b = std::min<uint64_t>(n, a + kChunk);
    int mx = 0;
    for (uint64_t i = a; i < b; ++i) mx = std::max(mx, expo(in[i]));
    uint32_t e3 = 0, e4 = 0;
    for (uint64_t i = a; i < b; ++i) {
      const int dlt = mx - expo(in[i]);
      e3 += dlt >= 7;
      e4 += dlt >= 15;
    }
    p.base[c] = static_cast<uint8_t>(mx);
    esc3[c] = e3;
    esc4[c] = e4;
  });
  auto size_for = [&](int k, const std::vector<uint32_t>& esc, uint64_t* tot_esc) {
    uint64_t t = 0;
    for (auto e : esc) t += e;
    *tot_esc = t;
    return align16(sizeof(PartHeader)) + align16(sizeof(ChunkEntry) * p.nch) + align16(n) +
           align16((n * k + 7) / 8) + align16(t);
  };
  uint64_t t3 = 0, t4 = 0;
  const uint64_t s3 = size_for(3, esc3, &t3), s4 = size_for(4, esc4, &t4);
  p.kbits = kbits_req == 3 || kbits_req == 4 ? kbits_req : (s3 <= s4 ? 3 : 4);
  const std::vector<uint32_t>& esc = p.kbits == 3 ? esc3 : esc4;
  p.total_esc = p.kbits == 3 ? t3 : t4;
  p.esc_off.assign(p.nch, 0);
  p.n_esc.assign(p.nch, 0);
  uint32_t run = 0;
  for (uint32_t c = 0; c < p.nch; ++c) {
    p.esc_off[c] = run;
    p.n_esc[c] = static_cast<uint16_t>(esc[c]);
    run += esc[c];
  }
  p.low_off = align16(sizeof(PartHeader)) + align16(sizeof(ChunkEntry) * p.nch);
  p.code_off = p.low_off + align16(n);
  p.esc_off_bytes = p.code_off + align16((n * p.kbits + 7) / 8);
  p.total = p.esc_off_bytes + align16(p.total_esc);
  return p;
}

}  // namespace

uint64_t encoded_size(const uint16_t* in, uint64_t n, int kbits) { return make_plan(in, n, kbits).total; }

uint64_t encode(const uint16_t* in, uint64_t n, int kbits_req, uint8_t* out) {
  const Plan p = make_plan(in, n, kbits_req);
  memset(out, 0, p.total);
  PartHeader h{};
  h.magic = kMagic;
  h.kbits = static_cast<uint32_t>(p.kbits);
  h.n = n;
  h.nch = p.nch;
  h.low_off = p.low_off;
  h.code_off = p.code_off;
  h.esc_off = p.esc_off_bytes;
  h.total = p.total;
  memcpy(out, &h, sizeof(h));
  ChunkEntry* ce = reinterpret_cast<ChunkEntry*>(out + align16(sizeof(PartHeader)));
  uint8_t* low = out + p.low_off;
  uint8_t* codes = out + p.code_off;
  uint8_t* escb = out + p.esc_off_bytes;
  const int k = p.kbits, lim = (1 << k) - 1;
  parallel_chunks(p.nch, [&](uint32_t c) {
    ce[c] = ChunkEntry{p.esc_off[c], p.base[c], 0, p.n_esc[c]};
    const uint64_t a = static_cast<uint64_t>(c) * kChunk, b = std::min<uint64_t>(n, a + kChunk);
    uint32_t e = p.esc_off[c];
    // chunks start on whole bytes of the code plane (kChunk * k is a multiple of 8)
    for (uint64_t i = a; i < b; ++i) {
      const uint16_t w = in[i];
      low[i] = static_cast<uint8_t>(((w >> 8) & 0x80) | (w & 0x7F));
      const int dlt = p.base[c] - expo(w);
      const uint32_t code = dlt < lim ? static_cast<uint32_t>(dlt + 1) : 0u;
      if (!code) escb[e++] = static_cast<uint8_t>(expo(w));
      const uint64_t bit = i * k;
      uint32_t v = code << (bit & 7);
      uint8_t* q = codes + (bit >> 3);
      q[0] |= static_cast<uint8_t>(v);
      if ((bit & 7) + k > 8) q[1] |= static_cast<uint8_t>(v >> 8);
    }
  });
  return p.total;
}

// One CTA per chunk, 32 consecutive weights per thread; escapes ranked by a block scan.
template <int K>
__global__ void __launch_bounds__(kThreads) decode_kernel(const uint8_t* __restrict__ part,
                                                          uint16_t* __restrict__ out) {
  const PartHeader& h = *reinterpret_cast<const PartHeader*>(part);
  const uint32_t c = blockIdx.x;
  const ChunkEntry ce = reinterpret_cast<const ChunkEntry*>(part + align16(sizeof(PartHeader)))[c];
  const uint64_t first = static_cast<uint64_t>(c) * kChunk + threadIdx.x * 32ull;
  const bool active = first < h.n;
  const int cnt = active ? static_cast<int>(h.n - first < 32 ? h.n - first : 32) : 0;
  uint32_t lo[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // the thread's 32 codes as two 64-bit words: codes 0..15 in c0, 16..31 in c1
  uint64_t c0 = 0, c1 = 0;
  int esc_mask_n = 0;
  uint32_t escm = 0;
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
    esc_mask_n = __popc(escm);
  }
  // exclusive scan of escape counts across the CTA (element order)
  __shared__ int warp_tot[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = esc_mask_n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int before = incl - esc_mask_n;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  if (!active) return;
  const uint8_t* esc = part + h.esc_off + ce.esc_off + before;
  uint32_t o[16];
  int e = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint32_t b8 = (lo[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    const uint32_t code = static_cast<uint32_t>((j < 16 ? c0 >> (K * j) : c1 >> (K * (j - 16))) & ((1u << K) - 1));
    uint32_t ex = (static_cast<uint32_t>(ce.base) + 1u - code) & 0xFFu;
    if ((escm >> j) & 1u) {  // rare (~1 % of weights at k = 3): exponent from the side list
      ex = esc[e];
      ++e;
    }
    const uint32_t w = ((b8 & 0x80u) << 8) | (ex << 7) | (b8 & 0x7Fu);
    if (j & 1) o[j >> 1] |= w << 16;
    else o[j >> 1] = w;
  }
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

moe_status decode(const void* part_dev, const PartHeader& h, uint16_t* out_dev, cudaStream_t s) {
  MOE_REQUIRE(h.magic == kMagic && (h.kbits == 3 || h.kbits == 4), "not an exponent-coded part");
  if (h.n == 0) return MOE_OK;
  if (h.kbits == 3)
    decode_kernel<3><<<h.nch, kThreads, 0, s>>>(static_cast<const uint8_t*>(part_dev), out_dev);
  else
    decode_kernel<4><<<h.nch, kThreads, 0, s>>>(static_cast<const uint8_t*>(part_dev), out_dev);
  MOE_LAUNCHED();
  return MOE_OK;
}

}  // namespace xc
}  // namespace moe

using namespace moe;

extern "C" {

moe_status moe_xc_encode(const uint16_t* in, uint64_t n, int32_t kbits, void* out, uint64_t cap,
                         uint64_t* size) {
  MOE_REQUIRE(size && (in || n == 0), "null argument");
  MOE_REQUIRE(kbits == 0 || kbits == 3 || kbits == 4, "kbits must be 0 (auto), 3 or 4");
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
