// codec.cu — lossless bf16 weight packing for the host link (exp4: 4-bit
// exponent codes; exph: canonical-Huffman exponent codes): host packers
// (threads over blocks / chunks), host reference decoders (tests), and the
// device decoders the offload executor runs between an expert's H2D copy and
// its FFN.  Formats: codec.cuh.
#include "codec.cuh"

#include <algorithm>
#include <cstring>
#include <atomic>
#include <iterator>
#include <queue>
#include <thread>

#include "common.cuh"

namespace infmoe {
namespace codec {
namespace {

template <class F>
void parallel_blocks(uint64_t nblocks, F&& f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t T = std::min<uint64_t>(hw, std::max<uint64_t>(1, nblocks / 4));
  std::vector<std::thread> th;
  for (uint64_t t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (uint64_t b = t; b < nblocks; b += T) f(b);
    });
  for (auto& x : th) x.join();
}

// one 32768-value block: 256 threads x 8 steps of 16 values (16 B of
// sign/mantissa + 8 B of codes in, 32 B of bf16 out), then the block's
// exceptions patch their exponents in place
__global__ void __launch_bounds__(256) exp4_unpack_kernel(const uint8_t* __restrict__ pack,
                                                          Exp4Layout L, uint16_t* out) {
  const uint64_t b = blockIdx.x;
  const uint64_t v0 = b * kExp4Block;
  const uint64_t nv = min(uint64_t(kExp4Block), L.n - v0);
  const uint32_t base = pack[L.off_base + b];
  const uint8_t* sm = pack + v0;
  const uint8_t* code = pack + L.n + v0 / 2;
  uint16_t* o = out + v0;
  for (uint64_t i = uint64_t(threadIdx.x) * 16; i < nv; i += 256 * 16) {
    const uint4 s = __ldg(reinterpret_cast<const uint4*>(sm + i));
    const uint2 c = __ldg(reinterpret_cast<const uint2*>(code + i / 2));
    const uint32_t sw[4] = {s.x, s.y, s.z, s.w};
    const uint32_t cw[2] = {c.x, c.y};
    uint32_t r[8];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t smb = (sw[j / 4] >> (8 * (j % 4))) & 0xFFu;
      const uint32_t cd = (cw[j / 8] >> (4 * (j % 8))) & 0xFu;
      const uint32_t e = (base - cd) & 0xFFu;
      const uint32_t v = ((smb & 0x80u) << 8) | (e << 7) | (smb & 0x7Fu);
      if (j % 2 == 0) r[j / 2] = v;
      else r[j / 2] |= v << 16;
    }
    uint4* d = reinterpret_cast<uint4*>(o + i);
    d[0] = make_uint4(r[0], r[1], r[2], r[3]);
    d[1] = make_uint4(r[4], r[5], r[6], r[7]);
  }
  __syncthreads();  // the block's plain stores land before the exception patches
  const uint32_t* exc_off = reinterpret_cast<const uint32_t*>(pack + L.off_exc_off);
  const uint32_t* exc = reinterpret_cast<const uint32_t*>(pack + L.off_exc);
  for (uint32_t q = exc_off[b] + threadIdx.x; q < exc_off[b + 1]; q += 256) {
    const uint32_t x = exc[q];
    uint16_t& t = o[x & 0xFFFFu];
    t = uint16_t((t & 0x807Fu) | (((x >> 16) & 0xFFu) << 7));
  }
}

}  // namespace

Exp4Plan exp4_plan(const uint16_t* in, uint64_t n) {
  require(n > 0 && n % 16 == 0, "exp4: value count must be a positive multiple of 16");
  Exp4Plan p;
  p.L = exp4_layout(n);
  const uint64_t nb = p.L.nblocks;
  p.base.assign(nb, 0);
  std::vector<uint32_t> cnt(nb, 0);
  parallel_blocks(nb, [&](uint64_t b) {
    const uint64_t v0 = b * kExp4Block, v1 = std::min(n, v0 + kExp4Block);
    uint32_t mx = 0;
    for (uint64_t i = v0; i < v1; ++i) mx = std::max<uint32_t>(mx, (in[i] >> 7) & 0xFFu);
    uint32_t c = 0;
    for (uint64_t i = v0; i < v1; ++i) c += (mx - ((in[i] >> 7) & 0xFFu)) > 14;
    p.base[b] = uint8_t(mx);
    cnt[b] = c;
  });
  p.exc_off.assign(nb + 1, 0);
  for (uint64_t b = 0; b < nb; ++b) p.exc_off[b + 1] = p.exc_off[b] + cnt[b];
  p.bytes = align16(p.L.off_exc + 4 * uint64_t(p.exc_off[nb]));
  return p;
}

void exp4_fill(const uint16_t* in, const Exp4Plan& p, uint8_t* out) {
  const uint64_t n = p.L.n;
  uint8_t* code = out + n;
  auto* exc = reinterpret_cast<uint32_t*>(out + p.L.off_exc);
  parallel_blocks(p.L.nblocks, [&](uint64_t b) {
    const uint64_t v0 = b * kExp4Block, v1 = std::min(n, v0 + kExp4Block);
    const uint32_t mx = p.base[b];
    uint32_t q = p.exc_off[b];
    for (uint64_t i = v0; i < v1; i += 2) {
      uint32_t nib[2];
      for (int h = 0; h < 2; ++h) {
        const uint16_t v = in[i + h];
        const uint32_t e = (v >> 7) & 0xFFu;
        out[i + h] = uint8_t(((v >> 8) & 0x80u) | (v & 0x7Fu));
        const uint32_t cd = mx - e;
        if (cd > 14) {
          nib[h] = 15;
          exc[q++] = uint32_t(i + h - v0) | (e << 16);
        } else {
          nib[h] = cd;
        }
      }
      code[i / 2] = uint8_t(nib[0] | (nib[1] << 4));
    }
  });
  std::copy(p.base.begin(), p.base.end(), out + p.L.off_base);
  std::copy(p.exc_off.begin(), p.exc_off.end(), reinterpret_cast<uint32_t*>(out + p.L.off_exc_off));
  // zero the alignment padding so identical inputs give identical packs
  for (uint64_t i = p.L.off_base + p.L.nblocks; i < p.L.off_exc_off; ++i) out[i] = 0;
  for (uint64_t i = p.L.off_exc_off + 4 * (p.L.nblocks + 1); i < p.L.off_exc; ++i) out[i] = 0;
  for (uint64_t i = p.L.off_exc + 4 * uint64_t(p.exc_off[p.L.nblocks]); i < p.bytes; ++i) out[i] = 0;
}

void exp4_unpack_host(const uint8_t* pack, uint64_t n, uint16_t* out) {
  const Exp4Layout L = exp4_layout(n);
  const auto* exc_off = reinterpret_cast<const uint32_t*>(pack + L.off_exc_off);
  const auto* exc = reinterpret_cast<const uint32_t*>(pack + L.off_exc);
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t base = pack[L.off_base + i / kExp4Block];
    const uint32_t smb = pack[i];
    const uint32_t cd = (pack[n + i / 2] >> (4 * (i % 2))) & 0xFu;
    out[i] = uint16_t(((smb & 0x80u) << 8) | (((base - cd) & 0xFFu) << 7) | (smb & 0x7Fu));
  }
  for (uint64_t b = 0; b < L.nblocks; ++b)
    for (uint32_t q = exc_off[b]; q < exc_off[b + 1]; ++q) {
      uint16_t& t = out[b * kExp4Block + (exc[q] & 0xFFFFu)];
      t = uint16_t((t & 0x807Fu) | (((exc[q] >> 16) & 0xFFu) << 7));
    }
}

void launch_exp4_unpack(const uint8_t* pack, uint64_t n, uint16_t* out, cudaStream_t s) {
  const Exp4Layout L = exp4_layout(n);
  exp4_unpack_kernel<<<unsigned(L.nblocks), 256, 0, s>>>(pack, L, out);
  INFMOE_LAUNCH_CHECK();
}

// ------------------------------------------------------------------ exph --
namespace {

// (dist, m2) symbol of a bf16 value against its base
inline uint32_t exph_sym(uint16_t v, uint32_t base) {
  const uint32_t d = base - ((v >> 7) & 0xFFu);
  return ((d >= uint32_t(kExphEsc) ? uint32_t(kExphEsc) : d) << 2) | ((v >> 5) & 3u);
}
inline bool exph_is_esc(uint32_t sym) { return (sym >> 2) == uint32_t(kExphEsc); }

// Optimal code lengths for kExphSyms symbols under the kExphMaxLen-bit limit
// (package-merge: the L-1 rounds of pairing the cheapest entries; a symbol's
// length is the number of chosen entries that contain it).  Canonical codes
// are then assigned by (length, symbol).
void huffman_lengths(const uint64_t* freq, uint8_t* len) {
  constexpr int S = kExphSyms;
  struct Entry {
    uint64_t w;
    std::vector<uint16_t> syms;  // symbols (with multiplicity) inside this entry
  };
  std::vector<Entry> items;
  for (int i = 0; i < S; ++i) {
    len[i] = 0;
    if (freq[i]) items.push_back({freq[i], {uint16_t(i)}});
  }
  const size_t n = items.size();
  if (n == 0) return;
  if (n == 1) { len[items[0].syms[0]] = 1; return; }
  // ascending weight, ties by the lowest symbol inside (deterministic)
  auto less = [](const Entry& x, const Entry& y) {
    return x.w != y.w ? x.w < y.w : x.syms.front() < y.syms.front();
  };
  std::stable_sort(items.begin(), items.end(), less);
  std::vector<Entry> list = items;
  for (int round = 1; round < kExphMaxLen; ++round) {
    std::vector<Entry> merged;
    for (size_t j = 0; j + 1 < list.size(); j += 2) {
      Entry e{list[j].w + list[j + 1].w, list[j].syms};
      e.syms.insert(e.syms.end(), list[j + 1].syms.begin(), list[j + 1].syms.end());
      merged.push_back(std::move(e));
    }
    std::vector<Entry> next;
    next.reserve(items.size() + merged.size());
    std::merge(items.begin(), items.end(), merged.begin(), merged.end(),
               std::back_inserter(next), less);
    list = std::move(next);
  }
  for (size_t j = 0; j < 2 * n - 2; ++j)
    for (uint16_t sym : list[j].syms) ++len[sym];
}

void canonical_codes(const uint8_t* len, uint32_t* code) {
  uint32_t c = 0;
  int prev = 0;
  for (int l = 1; l <= kExphMaxLen; ++l) {
    for (int s = 0; s < kExphSyms; ++s)
      if (len[s] == l) {
        c <<= (l - prev);
        prev = l;
        code[s] = c++;
      }
  }
}

// bits [bit, bit + 12) of the 192-bit little-endian residual record (A, B, C)
__device__ __forceinline__ uint32_t rec12(uint64_t A, uint64_t B, uint64_t C, int bit) {
  if (bit + 12 <= 64) return uint32_t(A >> bit) & 0xFFFu;
  if (bit < 64) return uint32_t((A >> bit) | (B << (64 - bit))) & 0xFFFu;
  if (bit + 12 <= 128) return uint32_t(B >> (bit - 64)) & 0xFFFu;
  if (bit < 128) return uint32_t((B >> (bit - 64)) | (C << (128 - bit))) & 0xFFFu;
  return uint32_t(C >> (bit - 128)) & 0xFFFu;
}

// a pair field s1 | m5_1 | s0 | m5_0 spread onto two bf16 values' sign and low
// mantissa bits
__device__ __forceinline__ uint32_t pair_resid(uint32_t f) {
  return (f & 0x1Fu) | ((f << 10) & 0x1F8000u) | ((f << 20) & 0x80000000u);
}

// One warp decodes 32 consecutive chunks, one per lane (Huffman codes are
// sequential within a chunk).  The residuals are stored as 24-byte records per
// 32 values, lane-interleaved (exph_res_offset), so each record load is one
// contiguous 768-byte warp access.  A table lookup yields, for two short codes,
// both values' exponent and top mantissa bits as 16-bit offsets from the
// block base (one packed add); a 12-bit pair field then supplies both values'
// signs and low mantissa bits.  Each group's 64 output bytes per lane are
// staged in shared memory (16-byte slots XOR-swizzled by row) and written
// back row by row as whole 32-byte sectors.  Only the bitstream refills stay
// per lane (one word ahead).
constexpr int kExphWarps = 8;
__global__ void __launch_bounds__(kExphWarps * 32) exph_unpack_kernel(const uint8_t* __restrict__ pack,
                                                                      ExphLayout L,
                                                                      uint16_t* __restrict__ out) {
  __shared__ uint2 lut[1 << kExphMaxLen];
  extern __shared__ uint4 stage[];  // [kExphWarps][kExphWarpChunks * 4]: 2 KB per warp
  const auto* glut = reinterpret_cast<const uint4*>(pack + L.off_lut);
  for (int i = threadIdx.x; i < (1 << kExphMaxLen) / 2; i += blockDim.x)
    reinterpret_cast<uint4*>(lut)[i] = __ldg(glut + i);
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint4* st = stage + warp * (kExphWarpChunks * 4);
  const auto* bw = reinterpret_cast<const uint32_t*>(pack + L.off_bits);
  const auto* gbit = reinterpret_cast<const uint32_t*>(pack + L.off_group);
  const auto* cbit = reinterpret_cast<const uint16_t*>(pack + L.off_chunk);
  const uint64_t ngroups = (L.nchunks + kExphWarpChunks - 1) / kExphWarpChunks;
  for (uint64_t g = uint64_t(blockIdx.x) * kExphWarps + warp; g < ngroups;
       g += uint64_t(gridDim.x) * kExphWarps) {
    const uint64_t c0 = g * kExphWarpChunks;
    const int nch = int(min(uint64_t(kExphWarpChunks), L.nchunks - c0));
    const unsigned active = nch == 32 ? 0xffffffffu : ((1u << nch) - 1u);
    if (lane < nch) {
      const uint64_t c = c0 + lane;
      const uint64_t v0 = c * kExphChunk;
      // table offsets carry a +4096 bias (positive halves: no carry between them)
      const uint32_t base7 = uint32_t(pack[L.off_base + v0 / kExp4Block]) << 7;
      const uint32_t base7b = base7 - kExphOffBias;  // mod 2^32
      const uint32_t base7x2b = (base7 | (base7 << 16)) - (kExphOffBias | (kExphOffBias << 16));
      const uint32_t p = __ldg(gbit + c / kExphGroup) + __ldg(cbit + c);
      const uint32_t* wp = bw + (p >> 5);
      uint64_t buf = ((uint64_t(__ldg(wp)) << 32) | __ldg(wp + 1)) << (p & 31);
      int nbits = 64 - int(p & 31);
      wp += 2;
      uint32_t nw = __ldg(wp);
      auto refill = [&]() {
        if (nbits < 32) {
          buf |= uint64_t(nw) << (32 - nbits);
          nbits += 32;
          nw = __ldg(++wp);
        }
      };
      // exponent << 7 | m2 << 5 of one value (escape: the raw exponent follows)
      auto one = [&](uint2 ent) -> uint32_t {
        const uint32_t sym = (ent.x >> 4) & 127u, ln = ent.x & 15u;
        buf <<= ln;
        nbits -= int(ln);
        if ((sym >> 2) == uint32_t(kExphEsc)) {
          const uint32_t e = uint32_t(buf >> 56);
          buf <<= 8;
          nbits -= 8;
          return (e << 7) | ((sym & 3u) << 5);
        }
        return (base7b + (ent.y & 0xFFFFu)) & 0xFFFFu;
      };
      const uint64_t* rec = reinterpret_cast<const uint64_t*>(
          pack + c0 * (kExphChunk / 32) * kExphRec + uint64_t(lane) * kExphRec);
      const uint64_t qstride = uint64_t(nch) * kExphRec / 8;  // in uint64
      uint64_t nA = __ldg(rec), nB = __ldg(rec + 1), nC = __ldg(rec + 2);
#pragma unroll 1
      for (int q = 0; q < kExphChunk / 32; ++q) {
        const uint64_t A = nA, B = nB, C = nC;
        if (q + 1 < kExphChunk / 32) {
          const uint64_t* r2 = rec + uint64_t(q + 1) * qstride;
          nA = __ldg(r2);
          nB = __ldg(r2 + 1);
          nC = __ldg(r2 + 2);
        }
        uint32_t r[16];
#pragma unroll
        for (int jp = 0; jp < 16; ++jp) {  // values in pairs: one table lookup per pair
          refill();
          const uint2 ent = lut[uint32_t(buf >> (64 - kExphMaxLen))];
          uint32_t hp;  // both values' exponent and top mantissa bits
          if (ent.x & (1u << 16)) {
            const uint32_t ln = (ent.x >> 11) & 31u;
            buf <<= ln;
            nbits -= int(ln);
            hp = base7x2b + ent.y;  // each half ends in [0, 2^15): exact per half
          } else {  // a long code or an escape: the two values one at a time
            const uint32_t h0 = one(ent);
            refill();
            hp = h0 | (one(lut[uint32_t(buf >> (64 - kExphMaxLen))]) << 16);
          }
          r[jp] = hp | pair_resid(rec12(A, B, C, 12 * jp));
        }
        // row = lane (this group's 64 output bytes: 4 16-byte slots), swizzled;
        // the warp then stores every row's 64 bytes (two full 32-byte sectors)
#pragma unroll
        for (int t = 0; t < 4; ++t)
          st[lane * 4 + (t ^ (lane & 3))] =
              make_uint4(r[4 * t], r[4 * t + 1], r[4 * t + 2], r[4 * t + 3]);
        __syncwarp(active);
        uint4* dst = reinterpret_cast<uint4*>(out + c0 * kExphChunk);
        for (int u = lane; u < nch * 4; u += nch) {
          const int row = u / 4, slot = u % 4;
          dst[row * (kExphChunk / 8) + q * 4 + slot] = st[row * 4 + (slot ^ (row & 3))];
        }
        __syncwarp(active);
      }
    }
    __syncwarp();  // every lane is done with st before the next group reuses it
  }
}

}  // namespace

ExphPlan exph_plan(const uint16_t* in, uint64_t n) {
  require(n > 0 && n % kExphChunk == 0, "exph: value count must be a positive multiple of 256");
  constexpr int S = kExphSyms;
  ExphPlan p;
  ExphLayout& L = p.L;
  L.n = n;
  L.nblocks = (n + kExp4Block - 1) / kExp4Block;
  L.nchunks = n / kExphChunk;
  L.ngroups = (L.nchunks + kExphGroup - 1) / kExphGroup;
  p.base.assign(L.nblocks, 0);
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  auto run = [&](auto&& body) {  // body(thread, block) over all blocks
    std::vector<std::thread> th;
    for (unsigned t = 0; t < hw; ++t)
      th.emplace_back([&, t] {
        for (uint64_t b = t; b < L.nblocks; b += hw) body(t, b);
      });
    for (auto& x : th) x.join();
  };
  // exponent bases: each block's largest exponent, and the matrix's largest
  run([&](unsigned, uint64_t b) {
    const uint64_t v0 = b * kExp4Block, v1 = std::min(n, v0 + kExp4Block);
    uint32_t mx = 0;
    for (uint64_t i = v0; i < v1; ++i) mx = std::max<uint32_t>(mx, (in[i] >> 7) & 0xFFu);
    p.base[b] = uint8_t(mx);
  });
  const uint32_t gmax = *std::max_element(p.base.begin(), p.base.end());
  // histograms of the symbols against both choices of base
  std::vector<std::vector<uint64_t>> hb(hw, std::vector<uint64_t>(S, 0)), hg = hb;
  run([&](unsigned t, uint64_t b) {
    const uint64_t v0 = b * kExp4Block, v1 = std::min(n, v0 + kExp4Block);
    for (uint64_t i = v0; i < v1; ++i) {
      ++hb[t][exph_sym(in[i], p.base[b])];
      ++hg[t][exph_sym(in[i], gmax)];
    }
  });
  // One base for the whole matrix codes the distance with the exponent's own
  // entropy (i.i.d. weights), block bases add the spread of the block maxima;
  // blocks help when the magnitude drifts along the matrix.  The encoder keeps
  // whichever costs fewer bits; the pack format (a base per block) and the
  // decoder are the same either way.
  uint64_t fb[S] = {}, fg[S] = {};
  for (unsigned t = 0; t < hw; ++t)
    for (int i = 0; i < S; ++i) {
      fb[i] += hb[t][size_t(i)];
      fg[i] += hg[t][size_t(i)];
    }
  uint8_t lb[S], lg[S];
  huffman_lengths(fb, lb);
  huffman_lengths(fg, lg);
  auto cost = [](const uint64_t* f, const uint8_t* l) {
    uint64_t bits = 0;
    for (int i = 0; i < S; ++i) bits += f[i] * (l[i] + (exph_is_esc(uint32_t(i)) ? 8u : 0u));
    return bits;
  };
  if (cost(fg, lg) < cost(fb, lb)) {
    std::fill(p.base.begin(), p.base.end(), uint8_t(gmax));
    std::copy(lg, lg + S, p.len);
  } else {
    std::copy(lb, lb + S, p.len);
  }
  canonical_codes(p.len, p.code);
  std::vector<uint32_t> cb(L.nchunks, 0);
  parallel_blocks(L.nchunks, [&](uint64_t c) {
    uint32_t bits = 0;
    const uint32_t base = p.base[c * kExphChunk / kExp4Block];
    for (uint64_t i = c * kExphChunk; i < (c + 1) * kExphChunk; ++i) {
      const uint32_t sym = exph_sym(in[i], base);
      bits += p.len[sym] + (exph_is_esc(sym) ? 8u : 0u);
    }
    cb[c] = bits;
  });
  p.chunk_bit.assign(L.nchunks + 1, 0);
  uint64_t total = 0;
  for (uint64_t c = 0; c < L.nchunks; ++c) {
    p.chunk_bit[c] = uint32_t(total);
    total += cb[c];
  }
  require(total < (uint64_t(1) << 32) - 64, "exph: bitstream exceeds 2^32 bits");
  p.chunk_bit[L.nchunks] = uint32_t(total);
  L.off_bits = align16(n / 32 * kExphRec);
  L.off_group = align16(L.off_bits + (total + 31) / 32 * 4 + 32);  // reader runs 32 B ahead
  L.off_chunk = align16(L.off_group + 4 * L.ngroups);
  L.off_base = align16(L.off_chunk + 2 * L.nchunks);
  L.off_lut = align16(L.off_base + L.nblocks);
  L.bytes = align16(L.off_lut + 8 * (1 << kExphMaxLen));
  return p;
}

void exph_fill(const uint16_t* in, const ExphPlan& p, uint8_t* out) {
  const ExphLayout& L = p.L;
  std::fill(out, out + L.bytes, uint8_t(0));
  auto* words = reinterpret_cast<uint32_t*>(out + L.off_bits);
  parallel_blocks(L.nchunks, [&](uint64_t c) {
    // the chunk's bits go to a local buffer (<= 256 x 20 bits); only its first
    // and last words can be shared with the neighbouring chunks
    const uint32_t base = p.base[c * kExphChunk / kExp4Block];
    const uint64_t start = p.chunk_bit[c];
    uint32_t loc[kExphChunk * 20 / 32 + 2] = {};
    uint64_t pos = start & 31;  // bit position inside loc
    auto put = [&](uint32_t val, uint32_t nb) {  // MSB-first, may straddle words
      while (nb) {
        const uint32_t w = uint32_t(pos >> 5), off = uint32_t(pos & 31);
        const uint32_t take = std::min(nb, 32 - off);
        const uint32_t bits = (val >> (nb - take)) & ((take == 32) ? 0xFFFFFFFFu : ((1u << take) - 1));
        loc[w] |= bits << (32 - off - take);
        pos += take;
        nb -= take;
      }
    };
    for (uint32_t q = 0; q < kExphChunk / 32; ++q) {
      // residual record: 16 pair fields s1 | m5_1 | s0 | m5_0 of 12 bits, little-endian
      uint64_t rec[3] = {0, 0, 0};
      for (uint32_t j = 0; j < 32; ++j) {
        const uint16_t v = in[c * kExphChunk + q * 32 + j];
        const uint64_t six = ((v >> 10) & 0x20u) | (v & 31u);  // sign << 5 | m5
        const uint32_t bit = 12 * (j / 2) + 6 * (j % 2);
        rec[bit / 64] |= six << (bit % 64);
        if (bit % 64 > 58) rec[bit / 64 + 1] |= six >> (64 - bit % 64);
        const uint32_t sym = exph_sym(v, base);
        put(p.code[sym], p.len[sym]);
        if (exph_is_esc(sym)) put((v >> 7) & 0xFFu, 8);
      }
      std::memcpy(out + exph_res_offset(c, q, L.nchunks), rec, kExphRec);
    }
    if (pos == (start & 31)) return;  // empty chunk (cannot happen: lengths >= 1)
    const uint64_t w0 = start >> 5;
    const uint32_t nw = uint32_t((pos + 31) >> 5);
    for (uint32_t k = 0; k < nw; ++k) {
      if (k == 0 || k + 1 == nw)
        std::atomic_ref<uint32_t>(words[w0 + k]).fetch_or(loc[k], std::memory_order_relaxed);
      else
        words[w0 + k] = loc[k];
    }
  });
  auto* gb = reinterpret_cast<uint32_t*>(out + L.off_group);
  auto* cb = reinterpret_cast<uint16_t*>(out + L.off_chunk);
  for (uint64_t c = 0; c < L.nchunks; ++c) {
    if (c % kExphGroup == 0) gb[c / kExphGroup] = p.chunk_bit[c];
    cb[c] = uint16_t(p.chunk_bit[c] - p.chunk_bit[c - c % kExphGroup]);
  }
  std::copy(p.base.begin(), p.base.end(), out + L.off_base);
  // LUT entry per 12-bit window (uint2): .x = len0 | sym0 << 4 | (len0 + len1) << 11 |
  // two << 16, .y = off(sym0) | off(sym1) << 16, off = (m2 << 5) - (dist << 7) + 4096;
  // "two" when a second code also fits inside the window and neither escapes
  std::vector<uint32_t> one(1u << kExphMaxLen, 0);
  for (int sym = 0; sym < kExphSyms; ++sym) {
    const uint32_t l = p.len[sym];
    if (!l) continue;
    const uint32_t first = p.code[sym] << (kExphMaxLen - l);
    for (uint32_t s = 0; s < (1u << (kExphMaxLen - l)); ++s) one[first | s] = (uint32_t(sym) << 4) | l;
  }
  auto off = [](uint32_t sym) {  // biased: >= 256 for every non-escape symbol
    return (((sym & 3u) << 5) - ((sym >> 2) << 7) + uint32_t(kExphOffBias)) & 0xFFFFu;
  };
  auto* lut = reinterpret_cast<uint32_t*>(out + L.off_lut);
  const uint32_t mask = (1u << kExphMaxLen) - 1;
  for (uint32_t w = 0; w <= mask; ++w) {
    const uint32_t e0 = one[w];
    const uint32_t l0 = e0 & 15u, s0 = (e0 >> 4) & 127u;
    uint32_t x = e0, y = l0 ? off(s0) : 0u;
    if (l0 && l0 < uint32_t(kExphMaxLen) && !exph_is_esc(s0)) {
      const uint32_t e1 = one[(w << l0) & mask];
      const uint32_t l1 = e1 & 15u, s1 = (e1 >> 4) & 127u;
      if (l1 && l0 + l1 <= uint32_t(kExphMaxLen) && !exph_is_esc(s1)) {
        x |= ((l0 + l1) << 11) | (1u << 16);
        y |= off(s1) << 16;
      }
    }
    lut[2 * w] = x;
    lut[2 * w + 1] = y;
  }
}

void exph_unpack_host(const uint8_t* pack, const ExphLayout& L, uint16_t* out) {
  const auto* words = reinterpret_cast<const uint32_t*>(pack + L.off_bits);
  const auto* gbit = reinterpret_cast<const uint32_t*>(pack + L.off_group);
  const auto* cbit = reinterpret_cast<const uint16_t*>(pack + L.off_chunk);
  const auto* lut = reinterpret_cast<const uint32_t*>(pack + L.off_lut);
  auto bit = [&](uint64_t q) { return (words[q >> 5] >> (31 - (q & 31))) & 1u; };
  for (uint64_t c = 0; c < L.nchunks; ++c) {
    uint64_t q = uint64_t(gbit[c / kExphGroup]) + cbit[c];
    const uint32_t base = pack[L.off_base + c * kExphChunk / kExp4Block];
    for (uint32_t g = 0; g < kExphChunk / 32; ++g) {
      uint64_t rec[3];
      std::memcpy(rec, pack + exph_res_offset(c, g, L.nchunks), kExphRec);
      for (uint32_t j = 0; j < 32; ++j) {
        uint32_t peek = 0;
        for (int k = 0; k < kExphMaxLen; ++k) peek = (peek << 1) | bit(q + k);
        const uint32_t sym = (lut[2 * peek] >> 4) & 127u, ln = lut[2 * peek] & 15u;
        q += ln;
        uint32_t e = (base - (sym >> 2)) & 0xFFu;
        if (exph_is_esc(sym)) {
          e = 0;
          for (int k = 0; k < 8; ++k) e = (e << 1) | bit(q + k);
          q += 8;
        }
        const uint32_t b = 12 * (j / 2) + 6 * (j % 2);
        uint64_t six = rec[b / 64] >> (b % 64);
        if (b % 64 > 58) six |= rec[b / 64 + 1] << (64 - b % 64);
        out[c * kExphChunk + g * 32 + j] = uint16_t(((six & 0x20u) << 10) | (e << 7) |
                                                    ((sym & 3u) << 5) | uint32_t(six & 31u));
      }
    }
  }
}

void launch_exph_unpack(const uint8_t* pack, const ExphLayout& L, uint16_t* out, cudaStream_t s) {
  const uint64_t groups = (L.nchunks + kExphWarpChunks - 1) / kExphWarpChunks;
  const uint64_t want = (groups + kExphWarps - 1) / kExphWarps;
  const uint64_t cap = uint64_t(device_sm_count()) * 4;  // 4 CTAs (32 KB LUT + 16 KB staging) per SM
  constexpr int kStage = kExphWarps * kExphWarpChunks * 4 * 16;
  ensure_dyn_smem(reinterpret_cast<const void*>(exph_unpack_kernel), size_t(kStage));
  exph_unpack_kernel<<<unsigned(std::max<uint64_t>(std::min(want, cap), 1)), kExphWarps * 32,
                       kStage, s>>>(pack, L, out);
  INFMOE_LAUNCH_CHECK();
}

}  // namespace codec
}  // namespace infmoe
