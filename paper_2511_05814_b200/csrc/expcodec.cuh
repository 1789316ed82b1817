// Lossless bf16 expert compression for the PCIe path ("exponent coding", in the spirit of
// ZipNN / DFloat11): a bf16 word is sign(1) | exponent(8) | mantissa(7).  Weights concentrate
// their exponents in a few values just below each block's maximum (entropy ~2.1 bits on the
// synthetic Mixtral weights), so a part is stored as
//   low plane   1 byte / weight   sign << 7 | mantissa
//   code plane  k bits / weight   c = base - exponent + 1 in [1, 2^k - 1], 0 = escape
//   escapes     1 byte / escape   the exponent, in element order within the chunk
// with base = the chunk's largest exponent, per 4096-weight chunk.  k = 3 or 4, chosen per part
// (smaller output wins).  1.38 bytes / weight at k = 3 on the synthetic weights (-31 % PCIe
// bytes); decoding is exact, so everything downstream is bit-identical.
//
// Part layout (every section 16-byte aligned):
//   PartHeader | ChunkEntry[nch] | low[n] | codes[n * k / 8] | escapes[total]
#pragma once
#include <cstdint>

#include "common.cuh"

namespace moe {
namespace xc {

constexpr int kChunk = 4096;        // weights per chunk
constexpr int kThreads = 128;       // decoder CTA: 32 weights per thread
constexpr uint32_t kMagic = 0x58503331u;  // "XP31"

struct __align__(16) PartHeader {
  uint32_t magic, kbits;
  uint64_t n;           // weights
  uint32_t nch;         // chunks
  uint32_t pad;
  uint64_t low_off, code_off, esc_off, total;  // byte offsets from the header; total size
};

struct ChunkEntry {
  uint32_t esc_off;     // index of the chunk's first escape byte
  uint8_t base;         // largest exponent in the chunk
  uint8_t pad;
  uint16_t n_esc;
};

inline __host__ __device__ uint64_t align16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// host: size of / encode n bf16 words into one part (kbits 0 = pick 3 or 4); multi-threaded
uint64_t encoded_size(const uint16_t* in, uint64_t n, int kbits);
uint64_t encode(const uint16_t* in, uint64_t n, int kbits, uint8_t* out);
// device: decode a part (already in HBM) into n bf16 words, on stream s
moe_status decode(const void* part_dev, const PartHeader& h, uint16_t* out_dev, cudaStream_t s);

}  // namespace xc
}  // namespace moe
