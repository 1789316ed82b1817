// Lossless bf16 expert compression for the PCIe path ("exponent coding", in the spirit of
// ZipNN / DFloat11): a bf16 word is sign(1) | exponent(8) | mantissa(7).  Weights concentrate
// their exponents in a few values just below each block's maximum (entropy ~2.1 bits on the
// synthetic Mixtral weights), so a part is stored as a sign+mantissa byte per weight plus an
// exponent code relative to the largest exponent of its 4096-weight chunk (dl = base - exp):
//   mode 3 / 4   k-bit code c = dl + 1 in [1, 2^k - 1]; c = 0 escapes to an exponent byte
//   mode 23      2-bit code c1 = dl - w + 1 for dl in the chunk's window [w, w + 3); c1 = 0
//                escapes to a 3-bit second-level code over the next 7 values, c2 = r - w2 + 1
//                for r = (dl < w ? dl : dl - 3) in [w2, w2 + 7), w2 = max(0, w - 2), whose 0
//                escapes to an exponent byte.  The encoder picks the cheapest w per chunk
//                (0 for a uniform draw, 1 for a bell-shaped one, deeper under an outlier)
// The encoder picks the smallest mode per part: on the synthetic (bell-shaped) weights 1.35
// bytes / weight with mode 23 (1.41 with mode 3, 1.50 with 4; raw 2; the exponent entropy
// bounds it at 1.32).  Decoding is exact, so everything downstream is bit-identical.
//
// Part layout (every section 16-byte aligned):
//   PartHeader | ChunkEntry[nch] | low[n] | codes (k * n bits, or 2 * n bits in mode 23)
//   | level-2 codes (mode 23: 3 bits each, contiguous over the part) | escape bytes
// Mode 23 decodes warp by warp (1024 weights, 32 per lane) with no block-level scan: each
// chunk entry stores where its warps 1..3 start in the level-2 and escape-byte streams.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace moe {
namespace xc {

constexpr int kChunk = 4096;        // weights per chunk
constexpr int kThreads = 128;       // decoder CTA: 32 weights per thread
constexpr uint32_t kMagic = 0x58503332u;  // "XP32"
constexpr int kMode23 = 23;

struct __align__(16) PartHeader {
  uint32_t magic, kbits;  // kbits: 3, 4 or kMode23
  uint64_t n;             // weights
  uint32_t nch;           // chunks
  uint32_t pad;
  uint64_t low_off, code_off, l2_off, esc_off, total;  // byte offsets from the header; size
};

struct ChunkEntry {      // 24 bytes
  uint32_t esc_off;     // index of the chunk's first escape byte
  uint32_t l2_off;      // mode 23: index of the chunk's first level-2 code
  uint8_t base;         // largest exponent in the chunk
  uint8_t win;          // mode 23: first dl of the level-1 window (w)
  uint16_t l2_rel[3];   // mode 23: first level-2 code of warps 1..3, relative to l2_off
  uint16_t esc_rel[3];  // mode 23: first escape byte of warps 1..3, relative to esc_off
  uint16_t pad;
};
static_assert(sizeof(ChunkEntry) == 24, "chunk entries are read as three 8-byte words");
constexpr int kWarpWeights = 1024;  // mode 23: weights per decoding warp

inline __host__ __device__ uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// host: size of / encode n bf16 words into one part (mode 0 = smallest of 3, 4, 23);
// multi-threaded over chunks
uint64_t encoded_size(const uint16_t* in, uint64_t n, int mode);
uint64_t encode(const uint16_t* in, uint64_t n, int mode, uint8_t* out);
// device: decode a part (already in HBM) into n bf16 words, on stream s; `prof` (optional,
// 2 zeroed int64) receives the launch's in-kernel span (LLONG_MAX - first CTA start, last end)
moe_status decode(const void* part_dev, const PartHeader& h, uint16_t* out_dev, cudaStream_t s,
                  long long* prof = nullptr);
// up to kMaxBatch parts of one code mode in a single launch (their chunks back to back)
constexpr int kMaxBatch = 4;
struct PartBatch {
  const uint8_t* part[kMaxBatch];
  uint16_t* out[kMaxBatch];
  uint32_t start[kMaxBatch];  // first CTA of each part
  int n;
};
struct Part23 {   // mode-23 part descriptor (the header's fields the decoder needs)
  const uint8_t* part;
  uint16_t* out;
  uint64_t n, low_off, code_off, l2_off, esc_off, total;
  uint32_t nch;
};
struct Batch23 {
  Part23 p[kMaxBatch];
  uint32_t start[kMaxBatch];  // first chunk of each part in the launch (unused: 0xFFFFFFFF)
  uint32_t chunks;            // chunks of all parts
};
moe_status decode_batch(const void* const* parts_dev, const PartHeader* hs, uint16_t* const* outs_dev,
                        int n, cudaStream_t s, long long* prof = nullptr);

}  // namespace xc
}  // namespace moe
