// codec.cuh — lossless packing of bf16 expert weights for the host link
// ("exp4" below, and the entropy-coded "exph" further down).
//
// The offloaded executor is host-link-bound (C3/C5 stream every
// expert over PCIe each pass), so the bytes per expert ARE the step time.  A
// bf16 weight is sign | 8-bit exponent | 7-bit mantissa; the mantissa and sign
// are near-incompressible, but the exponents of a weight matrix cluster just
// below its largest one (entropy ~2 bits for the bench's weights).  exp4
// stores, per block of 32768 values, the largest exponent (the base), and per
// value one byte (sign << 7 | mantissa) plus a 4-bit code base - exponent;
// code 15 escapes to an exception list (uint16 index in the block | exponent
// << 16) for exponents more than 14 below the base (zeros, subnormals, rare
// small values).  12 bits per value + exceptions: ~25% fewer bytes over the
// link, decoded on the GPU into the bf16 slot (HBM-bound, ~25 us per matrix),
// bit for bit.
//
// Pack layout for n values (n % 16 == 0), all offsets from the pack start:
//   [0, n)                 sign/mantissa bytes
//   [n, n + n/2)           codes, two per byte (even value in the low nibble)
//   [off_base, +nblocks)   per-block base exponent
//   [off_exc_off, ...)     uint32 exception offsets per block [nblocks + 1]
//   [off_exc, ...)         uint32 exceptions (index in block | exponent << 16)
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace infmoe {
namespace codec {

constexpr int kExp4Block = 32768;

struct Exp4Layout {
  uint64_t n = 0, nblocks = 0;
  uint64_t off_base = 0, off_exc_off = 0, off_exc = 0;
};

inline uint64_t align16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

inline Exp4Layout exp4_layout(uint64_t n) {
  Exp4Layout L;
  L.n = n;
  L.nblocks = (n + kExp4Block - 1) / kExp4Block;
  L.off_base = n + n / 2;
  L.off_exc_off = align16(L.off_base + L.nblocks);
  L.off_exc = align16(L.off_exc_off + 4 * (L.nblocks + 1));
  return L;
}

// host: per-block bases and exception counts of one matrix (parallel over blocks)
struct Exp4Plan {
  Exp4Layout L;
  std::vector<uint8_t> base;
  std::vector<uint32_t> exc_off;  // [nblocks + 1], prefix sum
  uint64_t bytes = 0;             // total pack bytes (16-aligned)
};
Exp4Plan exp4_plan(const uint16_t* in, uint64_t n);
// host: write the pack described by plan into out (plan.bytes bytes)
void exp4_fill(const uint16_t* in, const Exp4Plan& plan, uint8_t* out);
// host reference decoder (tests)
void exp4_unpack_host(const uint8_t* pack, uint64_t n, uint16_t* out);

// device: decode one pack (16-byte aligned) into n bf16 values
void launch_exp4_unpack(const uint8_t* pack, uint64_t n, uint16_t* out, cudaStream_t s);

// ------------------------------------------------------------------ exph --
// Entropy-coded exponents ("exph"): per value a canonical Huffman code (<= 12
// bits, one code table per matrix) of the symbol (dist, m2): dist =
// min(base - exponent, 31) against the per-block base (the encoder may give
// every block the matrix's base when that codes shorter), m2 the top two
// mantissa bits -- a Gaussian weight's mantissa is not uniform inside its
// binade, so coding them jointly with the exponent saves ~0.07 bits per value;
// dist 31 escapes: the raw 8-bit exponent follows the code.  The sign and the
// low five mantissa bits (6 bits) are stored raw, two values per 12-bit field.  Codes are concatenated
// MSB-first per 256-value chunk; a chunk's starting bit is a uint32 per group
// of 8 chunks plus a uint16 offset inside the group (0.078 bits per value), so
// one GPU thread decodes one chunk through a 4096-entry lookup table in shared
// memory.  ~10.6 bits per value for Gaussian bf16 weights (entropy 10.46).
//
// Layout: [0, 3n/4) raw residuals (exph_res_offset; per 32 values 16 pair
// fields of 12 bits = s1 << 11 | m5_1 << 6 | s0 << 5 | m5_0, little-endian) |
// [off_bits) bitstream (uint32 words, + 32 B slack) | [off_group) uint32 start
// bit per group | [off_chunk) uint16 offset per chunk | [off_base) base per
// block | [off_lut) uint2 LUT[4096]: .x = len0 | sym0 << 4 | (len0 + len1) << 11 |
// two << 16, .y = off0 | off1 << 16 with off = (m2 << 5) - (dist << 7) + 4096, so
// (base << 7) - 4096 + off is a value's exponent and top mantissa bits (positive
// 16-bit halves: one 32-bit add decodes a pair); "two" when both
// codes fit in the 12-bit window and neither escapes (one packed add then
// yields both values)
constexpr int kExphChunk = 256;
constexpr int kExphWarpChunks = 32;  // chunks decoded together by one warp (one per lane)
constexpr int kExphSyms = 128;       // (dist, m2)
constexpr int kExphRec = 24;         // residual record of 32 values: 16 pair fields of 12 bits

// byte offset of the residual record of chunk c's 32-value group q: the chunks
// of a warp group are interleaved per record, so one warp-wide load of group q
// reads contiguous memory
__host__ __device__ inline uint64_t exph_res_offset(uint64_t c, uint32_t q, uint64_t nchunks) {
  const uint64_t g = c / kExphWarpChunks, lane = c % kExphWarpChunks;
  const uint64_t first = g * kExphWarpChunks;
  const uint64_t nch = (nchunks - first) < uint64_t(kExphWarpChunks) ? (nchunks - first)
                                                                      : uint64_t(kExphWarpChunks);
  return first * (kExphChunk / 32) * kExphRec + uint64_t(q) * nch * kExphRec + lane * kExphRec;
}
constexpr int kExphGroup = 8;  // chunks per group (8 x 256 x 20 bits < 2^16: uint16 offsets)
constexpr int kExphMaxLen = 12;
constexpr int kExphEsc = 31;   // dist of the escape symbols (sym >> 2 == 31)
constexpr uint32_t kExphOffBias = 4096;  // keeps the table's exponent offsets positive

struct ExphLayout {
  uint64_t n = 0, nblocks = 0, nchunks = 0, ngroups = 0;
  uint64_t off_bits = 0, off_group = 0, off_chunk = 0, off_base = 0, off_lut = 0, bytes = 0;
};
struct ExphPlan {
  ExphLayout L;
  std::vector<uint8_t> base;
  uint8_t len[kExphSyms] = {};
  uint32_t code[kExphSyms] = {};
  std::vector<uint32_t> chunk_bit;  // [nchunks + 1]
};
ExphPlan exph_plan(const uint16_t* in, uint64_t n);
void exph_fill(const uint16_t* in, const ExphPlan& plan, uint8_t* out);
void exph_unpack_host(const uint8_t* pack, const ExphLayout& L, uint16_t* out);
void launch_exph_unpack(const uint8_t* pack, const ExphLayout& L, uint16_t* out, cudaStream_t s);

}  // namespace codec
}  // namespace infmoe
