// codec.cu — exp4 lossless bf16 packing: host packer (threads over blocks) and
// the device decoder the offload executor runs between an expert's H2D copy
// and its FFN.  Format: codec.cuh.
#include "codec.cuh"

#include <algorithm>
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

}  // namespace codec
}  // namespace infmoe
