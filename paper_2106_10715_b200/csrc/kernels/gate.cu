// gate.cu — N1a softmax/top-k gate and N1b LSH gate (warp-level kernels).
//
// Both gates assign one lane per (token, expert-or-hash-bit) and accumulate
// the dot product as ONE sequential chain over d (ascending), so the routing
// decision is reproducible bit for bit on the CPU (oracle.c or_gate_softmax /
// or_gate_lsh) with no dependence on a reduction tree:
//   softmax gate: acc = fmaf(x[c], wg[e][c], acc)            (fp32)
//   LSH gate    : dot = dot + x[c] * P[j][c], two roundings   (fp64,
//                 gating.hpp:70-80; the reference build does not contract)
// x and the gate weights are staged through shared memory in d-chunks so the
// weight matrix is read once per CTA of tokens, not once per token.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace infmoe {
namespace {

struct Cand {
  float v;
  int i;  // -1 = no candidate
};

// max non-NaN value, ties and the all-NaN case -> lower expert index
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.i < 0) return false;
  if (b.i < 0) return true;
  const bool an = isnan(a.v), bn = isnan(b.v);
  if (an != bn) return bn;
  if (!an && a.v != b.v) return a.v > b.v;
  return a.i < b.i;
}

// Multi-stage cp.async ring shared by both gates: column chunks of the token
// rows (raw dtype) and of the gate matrix are staged kGateStages-1 chunks ahead
// of the math, so global latency (~1 us) is covered by ~2 us of in-flight work.
constexpr int kGateStages = 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- N1a ----
// Softmax / top-k gate.  The logit reduction order is defined by the warp
// (the reference leaves this gate unspecified; oracle.c
// or_gate_softmax restates the same order): d is walked in 256-column chunks,
// lane l owns columns 8l..8l+7 of every chunk and keeps one fmaf chain per
// (token, expert) over them; the 32 lane partials are combined by a butterfly
// (p += shfl_xor(p, off), off = 16..1), then the bias is added.  So a warp
// streams 16-byte slices of x and W_g with no dependent chain longer than d/32
// steps.  A CTA owns TT tokens and all experts: warp w holds experts
// [w*EB, w*EB+EB) for the TT tokens (TT*EB = 64 accumulators per lane), the
// x tile of a chunk is staged once per CTA through the cp.async ring, and the
// gate weights (E x d fp32, L1/L2-resident) are read straight from global.
// Selection (top-k, softmax) then runs one warp per token from the logits
// tile in shared memory.
constexpr int kSoftChunk = 256;

template <typename T, int EB>
struct SoftCfg {
  static constexpr int TT = 64 / EB;                    // tokens per CTA
  static constexpr int V = 16 / int(sizeof(T));         // x elements per 16 B
  static constexpr int XROW = kSoftChunk + V;           // +16 B per row
  static constexpr size_t STAGE = size_t(TT) * XROW * sizeof(T);
  // warps per CTA (E <= MAXW*EB): 16 while the 64 accumulators + 4 weight
  // slices fit 128 registers (EB <= 4), else 8
  static constexpr int MAXW = EB <= 4 ? 16 : 8;
  static size_t smem(int E) {
    return kGateStages * STAGE + size_t(TT) * (E + 1) * sizeof(float);
  }
};

// Selection from the logits tile lg_s [TT][E+1] (one warp per token): top-k by
// logit (ties and NaN -> lower index), softmax weights (renormalised over the
// picks for k > 1), per-CTA histogram merged into counts.
__device__ __forceinline__ void softmax_select(const float* lg_s, int TT, int64_t tok0,
                                               int64_t N, int E, int k, int warp, int nwarps,
                                               int lane, int* hist, int32_t* __restrict__ topk_idx,
                                               float* __restrict__ topk_w,
                                               int32_t* __restrict__ counts) {
  const int NT = nwarps * 32;
  constexpr int SQ = 4;  // logits per lane during selection (E <= 128)
  for (int row = warp; row < TT; row += nwarps) {
    const int64_t tok = tok0 + row;
    if (tok >= N) break;
    float lg[SQ];
    bool live[SQ];
#pragma unroll
    for (int q = 0; q < SQ; ++q) {
      const int e = lane + 32 * q;
      live[q] = e < E;
      lg[q] = live[q] ? lg_s[row * (E + 1) + e] : 0.0f;
    }
    // softmax denominator over all experts (fp32; weights are tolerance-checked)
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < SQ; ++q)
      if (live[q] && !isnan(lg[q])) mx = fmaxf(mx, lg[q]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.0f;
#pragma unroll
    for (int q = 0; q < SQ; ++q)
      if (live[q]) se += expf(lg[q] - mx);
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);

    float psum = 0.0f;
    float pk_mine = 0.0f;
    int ik_mine = 0;
    for (int j = 0; j < k; ++j) {
      Cand best{0.0f, -1};
#pragma unroll
      for (int q = 0; q < SQ; ++q) {
        Cand c{lg[q], live[q] ? lane + 32 * q : -1};
        if (better(c, best)) best = c;
      }
      for (int o = 16; o; o >>= 1) {
        Cand other{__shfl_xor_sync(0xffffffffu, best.v, o),
                   __shfl_xor_sync(0xffffffffu, best.i, o)};
        if (better(other, best)) best = other;
      }
      const float pj = expf(best.v - mx) / se;
      psum += pj;
      if (lane == j) { pk_mine = pj; ik_mine = best.i; }  // lane j keeps pick j
#pragma unroll
      for (int q = 0; q < SQ; ++q)
        if (lane + 32 * q == best.i) live[q] = false;  // exclude from the next pick
    }
    if (lane < k) {
      topk_idx[tok * k + lane] = ik_mine;
      topk_w[tok * k + lane] = k > 1 ? pk_mine / psum : pk_mine;
      atomicAdd(&hist[ik_mine], 1);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += NT)
    if (hist[e]) atomicAdd(&counts[e], hist[e]);
}

template <typename T, int EB>
__global__ void __launch_bounds__(SoftCfg<T, EB>::MAXW * 32) gate_softmax_kernel(
    const T* __restrict__ x, int64_t N, int d, const float* __restrict__ wg,
    const float* __restrict__ bias, int E, int k, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_w, int32_t* __restrict__ counts) {
  using C = SoftCfg<T, EB>;
  constexpr int TT = C::TT, V = C::V, CH = kSoftChunk;
  extern __shared__ __align__(16) uint8_t soft_smem[];
  __shared__ int hist[128];
  const int NT = blockDim.x, nwarps = NT / 32;
  float* lg_s = reinterpret_cast<float*>(soft_smem + kGateStages * C::STAGE);  // [TT][E+1]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t tok0 = int64_t(blockIdx.x) * TT;
  for (int i = threadIdx.x; i < E; i += NT) hist[i] = 0;

  auto xs = [&](int st) { return reinterpret_cast<T*>(soft_smem + st * C::STAGE); };
  const int nch = (d + CH - 1) / CH;
  auto issue = [&](int ch) {
    if (ch < nch) {
      const int c0 = ch * CH;
      T* xd = xs(ch % kGateStages);
      for (int i = threadIdx.x; i < TT * (CH / V); i += NT) {
        const int t = i / (CH / V), c = (i % (CH / V)) * V;
        const bool ok = tok0 + t < N && c0 + c < d;
        cp_async16(xd + t * C::XROW + c, ok ? x + size_t(tok0 + t) * d + c0 + c : x, ok);
      }
    }
    cp_async_commit();  // empty groups keep the wait count uniform
  };

  float acc[TT][EB];
#pragma unroll
  for (int t = 0; t < TT; ++t)
#pragma unroll
    for (int e = 0; e < EB; ++e) acc[t][e] = 0.0f;
  const int e0 = warp * EB;

  for (int ch = 0; ch < kGateStages - 1; ++ch) issue(ch);
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait<kGateStages - 2>();  // chunk ch has landed (for this thread)
    __syncthreads();                   // ... for every thread; slot ch-1 is free
    issue(ch + kGateStages - 1);
    const int c = ch * CH + lane * 8;  // this lane's 8 columns (zero past d)
    const T* xb = xs(ch % kGateStages) + lane * 8;
    constexpr int EG = EB < 4 ? EB : 4;  // experts whose weight slices sit in registers
#pragma unroll
    for (int g = 0; g < EB; g += EG) {
    float wv[EG][8];
#pragma unroll
    for (int e = 0; e < EG; ++e) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (e0 + g + e < E && c < d) {
        const float4* wp = reinterpret_cast<const float4*>(wg + size_t(e0 + g + e) * d + c);
        a = __ldg(wp);
        b = __ldg(wp + 1);
      }
      wv[e][0] = a.x; wv[e][1] = a.y; wv[e][2] = a.z; wv[e][3] = a.w;
      wv[e][4] = b.x; wv[e][5] = b.y; wv[e][6] = b.z; wv[e][7] = b.w;
    }
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      float xv[8];
      if constexpr (sizeof(T) == 2) {
        const uint4 raw = *reinterpret_cast<const uint4*>(xb + t * C::XROW);
        xv[0] = __uint_as_float(raw.x << 16); xv[1] = __uint_as_float(raw.x & 0xffff0000u);
        xv[2] = __uint_as_float(raw.y << 16); xv[3] = __uint_as_float(raw.y & 0xffff0000u);
        xv[4] = __uint_as_float(raw.z << 16); xv[5] = __uint_as_float(raw.z & 0xffff0000u);
        xv[6] = __uint_as_float(raw.w << 16); xv[7] = __uint_as_float(raw.w & 0xffff0000u);
      } else {
        const float4 r0 = *reinterpret_cast<const float4*>(xb + t * C::XROW);
        const float4 r1 = *reinterpret_cast<const float4*>(xb + t * C::XROW + 4);
        xv[0] = r0.x; xv[1] = r0.y; xv[2] = r0.z; xv[3] = r0.w;
        xv[4] = r1.x; xv[5] = r1.y; xv[6] = r1.z; xv[7] = r1.w;
      }
#pragma unroll
      for (int e = 0; e < EG; ++e)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[t][g + e] = fmaf(xv[i], wv[e][i], acc[t][g + e]);
    }
    }
  }
  cp_async_wait<0>();
  // butterfly over the 32 lane partials (every lane ends with the sum)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int t = 0; t < TT; ++t)
#pragma unroll
      for (int e = 0; e < EB; ++e) acc[t][e] += __shfl_xor_sync(0xffffffffu, acc[t][e], off);
  // logits (+ bias, one fp32 add) into shared memory: lane t writes token t
#pragma unroll
  for (int t = 0; t < TT; ++t)
    if (lane == (t & 31))
#pragma unroll
      for (int e = 0; e < EB; ++e)
        if (e0 + e < E)
          lg_s[t * (E + 1) + e0 + e] = bias ? __fadd_rn(acc[t][e], bias[e0 + e]) : acc[t][e];
  __syncthreads();

  softmax_select(lg_s, TT, tok0, N, E, k, warp, nwarps, lane, hist, topk_idx, topk_w, counts);
}

// ---------------------------------------------------------------- N1b ----
// LSH: lane = (token sub-slot, hash bit); tokens per warp G = 32 / bits.  Each
// lane owns one sequential fp64 chain over d (gating.hpp:70-80: separate
// multiply and add roundings), so the kernel is bound by the 8-cycle dadd
// dependency chain.  x rows (raw dtype) and the hyperplane rows are staged
// through the cp.async ring; each hyperplane row is read as 16-byte pairs
// (rows padded onto distinct bank groups, broadcast across a token's lanes).
constexpr int kLshWarps = 4;
constexpr int kLshChunk = 128;

template <typename T>
__global__ void __launch_bounds__(kLshWarps * 32) gate_lsh_kernel(
    const T* __restrict__ x, int64_t N, int d, const double* __restrict__ proj, int bits, int E,
    uint32_t* __restrict__ codes, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
    int32_t* __restrict__ counts) {
  constexpr int NT = kLshWarps * 32;
  constexpr int V = 16 / sizeof(T);
  constexpr int XROW = kLshChunk + V;  // elements (+16 B)
  constexpr int PROW = kLshChunk + 2;  // doubles (+16 B)
  extern __shared__ __align__(16) uint8_t lsh_smem[];
  const int G = 32 / bits;
  const int TB = kLshWarps * G;
  const size_t xbytes = size_t(TB) * XROW * sizeof(T);
  const size_t stage = xbytes + size_t(bits) * PROW * sizeof(double);
  auto xs = [&](int st) { return reinterpret_cast<T*>(lsh_smem + st * stage); };
  auto ps = [&](int st) { return reinterpret_cast<double*>(lsh_smem + st * stage + xbytes); };
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int sub = lane / bits, j = lane % bits;
  const int local = warp * G + (sub < G ? sub : 0);
  const int64_t tok0 = int64_t(blockIdx.x) * TB;
  const int64_t tok = tok0 + local;
  const bool active = sub < G && tok < N;
  const int nch = (d + kLshChunk - 1) / kLshChunk;

  auto issue = [&](int ch) {
    if (ch < nch) {
      const int c0 = ch * kLshChunk;
      T* xd = xs(ch % kGateStages);
      double* pd = ps(ch % kGateStages);
      for (int i = threadIdx.x; i < TB * (kLshChunk / V); i += NT) {
        const int t = i / (kLshChunk / V), c = (i % (kLshChunk / V)) * V;
        const bool ok = tok0 + t < N && c0 + c < d;
        cp_async16(xd + t * XROW + c, ok ? x + size_t(tok0 + t) * d + c0 + c : x, ok);
      }
      for (int i = threadIdx.x; i < bits * (kLshChunk / 2); i += NT) {
        const int b = i / (kLshChunk / 2), c = (i % (kLshChunk / 2)) * 2;
        const bool ok = c0 + c < d;
        cp_async16(pd + b * PROW + c, ok ? proj + size_t(b) * d + c0 + c : proj, ok);
      }
    }
    cp_async_commit();
  };

  double dot = 0.0;
  for (int ch = 0; ch < kGateStages - 1; ++ch) issue(ch);
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait<kGateStages - 2>();
    __syncthreads();
    issue(ch + kGateStages - 1);
    const int cn = min(kLshChunk, d - ch * kLshChunk);  // a multiple of 8
    if (active) {
      const T* xrow = xs(ch % kGateStages) + local * XROW;
      const double2* prow = reinterpret_cast<const double2*>(ps(ch % kGateStages) + j * PROW);
      for (int c = 0; c < cn; c += 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(xrow + c);
        double xv[8];
        if constexpr (sizeof(T) == 2) {
          const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
          for (int i = 0; i < 8; ++i) xv[i] = double(load_as_f32(e, i));
        } else {
          const uint4 raw2 = *reinterpret_cast<const uint4*>(xrow + c + 4);
          const float* e = reinterpret_cast<const float*>(&raw);
          const float* e2 = reinterpret_cast<const float*>(&raw2);
#pragma unroll
          for (int i = 0; i < 4; ++i) { xv[i] = double(e[i]); xv[4 + i] = double(e2[i]); }
        }
        double prod[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 pp = prow[c / 2 + i];
          prod[2 * i] = __dmul_rn(xv[2 * i], pp.x);
          prod[2 * i + 1] = __dmul_rn(xv[2 * i + 1], pp.y);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) dot = __dadd_rn(dot, prod[i]);
      }
    }
  }
  cp_async_wait<0>();
  const unsigned mask = __ballot_sync(0xffffffffu, active && dot >= 0.0);
  if (active && j == 0) {
    const uint32_t code = (mask >> (sub * bits)) & ((1u << bits) - 1u);
    const int e = int(code % uint32_t(E));
    if (codes) codes[tok] = code;
    topk_idx[tok] = e;
    topk_w[tok] = 1.0f;
    atomicAdd(&counts[e], 1);
  }
}

// ------------------------------------------------------- N1b fast path ----
// The reference only consumes the SIGN of each sequential dot (bit j =
// dot >= 0, gating.hpp:76-79), so most bits can be decided without running
// the 4096-step dependent chain.  Certified fast path:
//   S  = sum_i x_i*w_i accumulated with DFMA in any order (lanes split d,
//        then a butterfly reduction);
//   |S_seq - S| <= (gamma_n + (1+u)gamma_{n-1} + u) * sum|x_i w_i|
//              <= 2.0003 n u ||x||_2 ||w||_2                  (Cauchy-Schwarz),
// where S_seq is the reference's left-to-right sum of the rounded products
// and u = 2^-53.  If |S| > thr = 8 n u ||x|| ||w|| (computed norms, a 4x
// margin), S_seq has S's sign and is nonzero, so the bit is S > 0.  An
// all-zero row gives S_seq = +0 (bit 1).  Anything else — |S| <= thr, NaN,
// Inf — re-runs the exact sequential chain for that (token, bit) pair, so the
// codes are identical to the reference's by construction.  Each warp owns
// kLshFastTW tokens; lanes take 8-element slices of d (16 B loads of x,
// streamed past L1; hyperplane rows are L1-resident).
constexpr int kLshFastTW = 2;      // tokens per warp
constexpr int kLshFastWarps = 8;   // warps per CTA (16 tokens)
constexpr int kLshFastChunk = 256; // columns per ring stage (8 per lane)

template <typename T, int BMAX>
struct LshFastCfg {
  static constexpr int TB = kLshFastWarps * kLshFastTW;
  static constexpr int XROW = kLshFastChunk + 16 / int(sizeof(T));  // +16 B
  static constexpr size_t XBYTES = size_t(TB) * XROW * sizeof(T);
  static constexpr size_t WBYTES = size_t(BMAX) * kLshFastChunk * sizeof(double);
  static constexpr size_t STAGE = XBYTES + WBYTES;
  static constexpr size_t SMEM = kGateStages * STAGE + size_t(kLshFastWarps) * BMAX * sizeof(double);
  // stage stride for `bits` hyperplane rows (the ring only holds what is used)
  static constexpr size_t stage_bytes(int bits) {
    return XBYTES + size_t(bits) * kLshFastChunk * sizeof(double);
  }
  static constexpr size_t smem_bytes(int bits) {
    return kGateStages * stage_bytes(bits) + size_t(kLshFastWarps) * BMAX * sizeof(double);
  }
};

template <typename T, int BMAX>
__global__ void __launch_bounds__(kLshFastWarps * 32) gate_lsh_fast_kernel(
    const T* __restrict__ x, int64_t N, int d, const double* __restrict__ proj, int bits, int E,
    int force_exact, uint32_t* __restrict__ codes, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_w, int32_t* __restrict__ counts) {
  using C = LshFastCfg<T, BMAX>;
  constexpr int TW = kLshFastTW, NT = kLshFastWarps * 32, CH = kLshFastChunk;
  constexpr int V = 16 / int(sizeof(T));
  extern __shared__ __align__(16) uint8_t lshf_smem[];
  const size_t stage = C::stage_bytes(bits);
  auto xs = [&](int st) { return reinterpret_cast<T*>(lshf_smem + st * stage); };
  auto ws = [&](int st) { return reinterpret_cast<double*>(lshf_smem + st * stage + C::XBYTES); };
  double* wnorm = reinterpret_cast<double*>(lshf_smem + kGateStages * stage);  // [warps][BMAX]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tok0 = int64_t(blockIdx.x) * C::TB;
  const int nch = (d + CH - 1) / CH;

  // per-thread copy assignments are the same for every chunk (only c0 moves):
  // x: TB*CH/V 16-B pieces, XPT per thread; w: one pair per thread per bit
  constexpr int XPT = C::TB * (CH / V) / NT;
  static_assert(C::TB * (CH / V) % NT == 0 && NT % (CH / 2) == 0, "LSH fast ring shape");
  // thread -> (row t = i / (CH/V), column c = (i % (CH/V)) * V), i = tid + NT*r:
  // the column is the same for every r (NT is a multiple of CH/V)
  static_assert(NT % (CH / V) == 0, "LSH fast ring shape");
  const int x_c = (threadIdx.x % (CH / V)) * V;
  const int x_t0 = threadIdx.x / (CH / V);
  // hyperplane pairs lane-interleaved: pair p (columns 2p, 2p+1 of the chunk)
  // of lane p/4 lands at slot (p%4)*32 + p/4, so the 16-B reads of one pair
  // index by the 32 lanes are contiguous (conflict-free)
  const int pr = threadIdx.x % (CH / 2), b_first = threadIdx.x / (CH / 2);
  const int w_dst = ((pr & 3) * 32 + (pr >> 2)) * 2;
  auto issue = [&](int ch) {
    if (ch < nch) {
      const int c0 = ch * CH;
      T* xd = xs(ch % kGateStages);
      double* wd = ws(ch % kGateStages);
      const bool cok = c0 + x_c < d;
#pragma unroll
      for (int r = 0; r < XPT; ++r) {
        const int t = x_t0 + r * (NT / (CH / V));
        const bool ok = cok && tok0 + t < N;
        cp_async16(xd + t * C::XROW + x_c, ok ? x + (tok0 + t) * int64_t(d) + c0 + x_c : x, ok);
      }
      const bool wok = c0 + 2 * pr < d;
      for (int b = b_first; b < bits; b += NT / (CH / 2))
        cp_async16(wd + b * CH + w_dst, wok ? proj + size_t(b) * d + c0 + 2 * pr : proj, wok);
    }
    cp_async_commit();
  };

  double acc[TW][BMAX], xx[TW], ww[BMAX];
#pragma unroll
  for (int t = 0; t < TW; ++t) {
    xx[t] = 0.0;
#pragma unroll
    for (int b = 0; b < BMAX; ++b) acc[t][b] = 0.0;
  }
#pragma unroll
  for (int b = 0; b < BMAX; ++b) ww[b] = 0.0;

  for (int ch = 0; ch < kGateStages - 1; ++ch) issue(ch);
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait<kGateStages - 2>();
    __syncthreads();
    issue(ch + kGateStages - 1);
    const T* xb = xs(ch % kGateStages) + (warp * TW) * C::XROW + lane * 8;
    const double* wb = ws(ch % kGateStages) + lane * 2;
    double xv[TW][8];
#pragma unroll
    for (int t = 0; t < TW; ++t) {
      if constexpr (sizeof(T) == 2) {
        const uint4 raw = *reinterpret_cast<const uint4*>(xb + t * C::XROW);
        const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int i = 0; i < 8; ++i) xv[t][i] = double(load_as_f32(e, i));
      } else {
        const float4 r0 = *reinterpret_cast<const float4*>(xb + t * C::XROW);
        const float4 r1 = *reinterpret_cast<const float4*>(xb + t * C::XROW + 4);
        xv[t][0] = r0.x; xv[t][1] = r0.y; xv[t][2] = r0.z; xv[t][3] = r0.w;
        xv[t][4] = r1.x; xv[t][5] = r1.y; xv[t][6] = r1.z; xv[t][7] = r1.w;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) xx[t] = fma(xv[t][i], xv[t][i], xx[t]);
    }
#pragma unroll
    for (int b = 0; b < BMAX; ++b) {
      if (b < bits) {
        double wv[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 q = *reinterpret_cast<const double2*>(wb + b * CH + k * 64);
          wv[2 * k] = q.x;
          wv[2 * k + 1] = q.y;
        }
        if ((b & (kLshFastWarps - 1)) == warp) {  // each warp sums the norms of its bits
#pragma unroll
          for (int i = 0; i < 8; ++i) ww[b] = fma(wv[i], wv[i], ww[b]);
        }
#pragma unroll
        for (int t = 0; t < TW; ++t)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[t][b] = fma(xv[t][i], wv[i], acc[t][b]);
      }
    }
  }
  cp_async_wait<0>();
  // butterfly: every lane ends with the full sums
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int t = 0; t < TW; ++t) {
      xx[t] += __shfl_xor_sync(0xffffffffu, xx[t], off);
#pragma unroll
      for (int b = 0; b < BMAX; ++b) acc[t][b] += __shfl_xor_sync(0xffffffffu, acc[t][b], off);
    }
#pragma unroll
    for (int b = 0; b < BMAX; ++b) ww[b] += __shfl_xor_sync(0xffffffffu, ww[b], off);
  }
  if (lane == 0)
#pragma unroll
    for (int b = 0; b < BMAX; ++b) wnorm[warp * BMAX + b] = ww[b];
  __syncthreads();
  // lane j < TW*bits decides pair (t, b) = (j / bits, j % bits) of this warp
  const int64_t wtok0 = tok0 + warp * TW;
  uint32_t mybit = 0;
  const int j = lane;
  const int t = j / bits, b = j % bits;
  if (j < TW * bits && wtok0 + t < N) {
    double S = 0.0, xn = 0.0;
#pragma unroll
    for (int tt = 0; tt < TW; ++tt)
#pragma unroll
      for (int bb = 0; bb < BMAX; ++bb)
        if (tt == t && bb == b) { S = acc[tt][bb]; xn = xx[tt]; }
    const double wn = wnorm[(b & (kLshFastWarps - 1)) * BMAX + b];
    const double thr = 8.0 * double(d) * 0x1p-53 * sqrt(xn) * sqrt(wn) + 0x1p-1000;
    bool bit;
    if (xn == 0.0) {
      bit = true;  // all products are +-0: the chain stays +0, and +0 >= 0
    } else if (!force_exact && fabs(S) > thr) {
      bit = S > 0.0;
    } else {  // ambiguous, NaN or Inf: the reference's sequential chain
      const T* xr = x + (wtok0 + t) * int64_t(d);
      const double* wr = proj + size_t(b) * d;
      double dot = 0.0;
      for (int i = 0; i < d; ++i)
        dot = __dadd_rn(dot, __dmul_rn(double(load_as_f32(xr, i)), wr[i]));
      bit = dot >= 0.0;
    }
    mybit = bit ? (1u << b) : 0u;
  }
  // OR the bits of each token: lanes t*bits .. t*bits+bits-1
  uint32_t code = 0;
#pragma unroll
  for (int tt = 0; tt < TW; ++tt) {
    uint32_t part = (j < TW * bits && t == tt) ? mybit : 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part |= __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == tt) code = part;
  }
  if (lane < TW && wtok0 + lane < N) {
    const int64_t tk = wtok0 + lane;
    const int e = int(code % uint32_t(E));
    if (codes) codes[tk] = code;
    topk_idx[tk] = e;
    topk_w[tk] = 1.0f;
    atomicAdd(&counts[e], 1);
  }
}

// INFMOE_LSH_FORCE_EXACT=1: every bit through the exact chain of the fast
// kernel (tests); INFMOE_LSH_FAST=0: the all-sequential ring kernel.
int lsh_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <typename T, int BMAX>
void lsh_fast_go(const void* x, int64_t N, int d, const double* proj, int bits, int E,
                 uint32_t* codes, int32_t* idx, float* w, int32_t* counts, cudaStream_t s) {
  static const int force = lsh_env("INFMOE_LSH_FORCE_EXACT", 0);
  using C = LshFastCfg<T, BMAX>;
  auto kern = gate_lsh_fast_kernel<T, BMAX>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), size_t(int(C::SMEM)));
  const unsigned blocks = unsigned((N + C::TB - 1) / C::TB);
  kern<<<blocks, kLshFastWarps * 32, C::smem_bytes(bits), s>>>(
      reinterpret_cast<const T*>(x), N, d, proj, bits, E, force, codes, idx, w, counts);
}

// ------------------------------------------- N1b fast path on fp64 MMA ----
// The same certified decision as gate_lsh_fast_kernel, with the parallel dot
// products on the fp64 tensor cores: S[16 tokens][8 bits] += X[16 x 4] .
// W[4 x 8] per mma.sync.m16n8k4.f64 (DMMA; 37 TF/s on B200, the DFMA pipe's
// rate, but 512 FMAs per instruction instead of 32, so the kernel is no longer
// issue-bound).  The reduction order is free (the bound covers any order), so
// the k index is permuted: thread (gid, tig) of a warp owns the 8 contiguous
// columns c0 + 8*tig .. +7 of every 32-column chunk and feeds them to 8
// consecutive mmas — its A fragment (x rows gid and gid+8) and B fragment
// (hyperplane row gid) are exactly the 16-byte / 64-byte slices it loads, so
// no shared memory or shuffles sit in the main loop.  A CTA owns 16 tokens;
// its 4 warps take the 32-column chunks round-robin and meet in shared memory
// for the final sums, norms and the certified decision.
constexpr int kLshMmaWarps = 8;  // 16 tokens per CTA, 8 warps splitting d (2 CTAs per SM: one wave)

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

template <typename T>
__global__ void __launch_bounds__(kLshMmaWarps * 32) gate_lsh_mma_kernel(
    const T* __restrict__ x, int64_t N, int d, const double* __restrict__ proj, int bits, int E,
    int force_exact, uint32_t* __restrict__ codes, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_w, int32_t* __restrict__ counts) {
  constexpr int W = kLshMmaWarps;
  __shared__ double s_part[W][16][9];  // per-warp partial S (padded)
  __shared__ double s_xx[W][16];
  __shared__ double s_ww[W][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int gid = lane / 4, tig = lane % 4;
  const int64_t tok0 = int64_t(blockIdx.x) * 16;
  const bool r0ok = tok0 + gid < N, r1ok = tok0 + gid + 8 < N;
  const bool bok = gid < bits;
  const T* x0 = x + (r0ok ? tok0 + gid : 0) * int64_t(d);
  const T* x1 = x + (r1ok ? tok0 + gid + 8 : 0) * int64_t(d);
  const double* w0 = proj + size_t(bok ? gid : 0) * d;

  double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};  // two independent mma chains
  double xx0 = 0.0, xx1 = 0.0, ww = 0.0;
  const int nch = (d + 31) / 32;
  // raw operands of the next chunk in flight ahead of the math (loads of
  // chunk ch + W issue before chunk ch's mmas); x stays raw until it is used
  constexpr int XV = sizeof(T) == 2 ? 1 : 2;  // 16-byte vectors per 8 x values
  struct Raw {
    uint4 x0[XV], x1[XV];
    double2 w[4];
  };
  auto load = [&](int ch, Raw& r) {
    const int c = ch * 32 + tig * 8;
    const bool cok = ch < nch && c < d;  // d % 8 == 0: a slice is all in or all out
#pragma unroll
    for (int v = 0; v < XV; ++v) {
      r.x0[v] = r0ok && cok ? __ldcs(reinterpret_cast<const uint4*>(x0 + c) + v) : make_uint4(0, 0, 0, 0);
      r.x1[v] = r1ok && cok ? __ldcs(reinterpret_cast<const uint4*>(x1 + c) + v) : make_uint4(0, 0, 0, 0);
    }
    const double2* wp = reinterpret_cast<const double2*>(w0 + c);
#pragma unroll
    for (int i = 0; i < 4; ++i) r.w[i] = bok && cok ? __ldg(wp + i) : make_double2(0.0, 0.0);
  };
  auto widen = [&](const uint4 (&raw)[XV], double (&v)[8]) {
    const T* e = reinterpret_cast<const T*>(&raw[0]);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = double(load_as_f32(e, i));
  };
  Raw cur, nxt;
  load(warp, cur);
  for (int ch = warp; ch < nch; ch += W) {
    load(ch + W, nxt);
    double a[8], b[8];
    widen(cur.x0, a);
    widen(cur.x1, b);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const double wm = (m & 1) ? cur.w[m / 2].y : cur.w[m / 2].x;
      dmma_16x8x4(acc[m & 1], a[m], b[m], wm);
      xx0 = fma(a[m], a[m], xx0);
      xx1 = fma(b[m], b[m], xx1);
      ww = fma(wm, wm, ww);
    }
    cur = nxt;
  }
  // D fragment: acc[.][0..1] = S[gid][2tig, 2tig+1], acc[.][2..3] = S[gid+8][...]
  s_part[warp][gid][2 * tig] = acc[0][0] + acc[1][0];
  s_part[warp][gid][2 * tig + 1] = acc[0][1] + acc[1][1];
  s_part[warp][gid + 8][2 * tig] = acc[0][2] + acc[1][2];
  s_part[warp][gid + 8][2 * tig + 1] = acc[0][3] + acc[1][3];
  // norms: sum over the 4 tig lanes of each row (the whole d of this warp's chunks)
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    xx0 += __shfl_xor_sync(0xffffffffu, xx0, off);
    xx1 += __shfl_xor_sync(0xffffffffu, xx1, off);
    ww += __shfl_xor_sync(0xffffffffu, ww, off);
  }
  if (tig == 0) {
    s_xx[warp][gid] = xx0;
    s_xx[warp][gid + 8] = xx1;
    s_ww[warp][gid] = ww;
  }
  __syncthreads();
  if (warp != 0) return;
  // lanes 0..15: one token each
  if (lane < 16 && tok0 + lane < N) {
    const int t = lane;
    double xn = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) xn += s_xx[w][t];
    uint32_t code = 0;
    for (int j = 0; j < bits; ++j) {
      double S = 0.0, wn = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        S += s_part[w][t][j];
        wn += s_ww[w][j];
      }
      const double thr = 8.0 * double(d) * 0x1p-53 * sqrt(xn) * sqrt(wn) + 0x1p-1000;
      bool bit;
      if (xn == 0.0) {
        bit = true;  // all products are +-0: the chain stays +0, and +0 >= 0
      } else if (!force_exact && fabs(S) > thr) {
        bit = S > 0.0;
      } else {  // ambiguous, NaN or Inf: the reference's sequential chain
        const T* xr = x + (tok0 + t) * int64_t(d);
        const double* wr = proj + size_t(j) * d;
        double dot = 0.0;
        for (int i = 0; i < d; ++i)
          dot = __dadd_rn(dot, __dmul_rn(double(load_as_f32(xr, i)), wr[i]));
        bit = dot >= 0.0;
      }
      if (bit) code |= 1u << j;
    }
    const int64_t tk = tok0 + t;
    const int e = int(code % uint32_t(E));
    if (codes) codes[tk] = code;
    topk_idx[tk] = e;
    topk_w[tk] = 1.0f;
    atomicAdd(&counts[e], 1);
  }
}

template <typename T>
void lsh_mma_go(const void* x, int64_t N, int d, const double* proj, int bits, int E,
                uint32_t* codes, int32_t* idx, float* w, int32_t* counts, cudaStream_t s) {
  static const int force = lsh_env("INFMOE_LSH_FORCE_EXACT", 0);
  gate_lsh_mma_kernel<T><<<unsigned((N + 15) / 16), kLshMmaWarps * 32, 0, s>>>(
      reinterpret_cast<const T*>(x), N, d, proj, bits, E, force, codes, idx, w, counts);
}

// ------------------------------------------------- N1a on tensor cores ----
// The CUDA-core gate above spends d FMAs per (token, expert) on the CUDA
// cores and is issue-bound (C5: 16384 x 64 x 4096, ~350 us).  For bf16 token
// rows and 2 <= top_k <= 8 the gate instead runs as
//  0. gate_split_kernel (once per gate matrix; a layer does it at set-up):
//     W_g (fp32) = hi + mid + lo, three bf16 matrices (3 x 8 significand bits
//     cover fp32's 24; a residual only where a part underflows, measured), and
//     the per-expert bound coefficient g_e (below).
//  1. gate_tc_kernel: L~[t, e] = x_t . (hi_e + mid_e + lo_e) on tcgen05
//     (kind::f16, 128-token tiles, the three parts against the same
//     TMA-staged x tile).  The hi products go to S fp32 TMEM accumulators, one
//     per K segment; mid and lo (<= 2^-8 of hi) share one more; the epilogue
//     sums them in a fixed order.  The 4 epilogue warps also read every staged
//     x tile (their row's 128 B) for ||x_t||_2, so x is streamed from HBM
//     exactly once.  Epilogue thread = token:
//       B_e = ||x_t|| g_e + 2^-22 |L~_e| + beta >= |L~_e - L_e|,
//     L_e the exact fmaf-chain logit of the CUDA-core gate (its reduction
//     order is the contract, oracle.c or_gate_softmax).  If the k largest
//     L~ are separated by their bounds (L~_(j) - B_(j) > L~_(j+1) + B_(j+1))
//     and from every other expert (L~_(k) - B_(k) > max_rest L~_e + B_e),
//     the exact chain would pick the same experts in the same order: the
//     token is CERTIFIED and its picks, softmax weights (from L~, renormalised
//     over the picks) and counts are written right there.
//  2. gate_tc_fallback_kernel (one CTA per uncertified token, listed by
//     step 1; the candidates' chains spread over its warps): every expert
//     whose upper bound reaches the k-th largest lower bound is a candidate
//     and gets its exact logit by the CUDA-core gate's fmaf chain and
//     butterfly; top-k over those (ties and NaN -> lower index).  A token with a non-finite value or more than kTcCandMax
//     candidates takes every expert through the exact chain.
// So indices and counts equal the exact gate's by construction; the weights
// carry the tensor-core logits' error (observed <= 1.5e-7 ||x|| ||w||).
// g_e = gamma_hi ||hi_e|| + gamma_ml ||mid_e + lo_e|| + gamma_w ||w_e|| +
// ||residual_e||, with gamma_hi/ml = 17 2^-23 (m + 1) for the m tcgen05.mma
// accumulated into one hi / the mid-lo accumulator (each MMA, 16 products plus
// the accumulator, is modelled as aligning its 17 addends to the largest and
// truncating each at 2^-23 of it; a wider alignment only tightens this), and
// gamma_w = (S + 1) 2^-24 (the epilogue's sum) + (dpad/32 + 8) 2^-23 (the
// exact chain's own fmaf/butterfly rounding), all against sum |x_i v_i| <=
// ||x|| ||v|| (Cauchy-Schwarz).  tests/test_gpu_gate_tc.py records the
// observed |L~ - x.w| against the model.
constexpr int kTcTok = 128;     // tokens per tile = UMMA M = TMEM lanes
constexpr int kTcThreads = 192; // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kTcMaxStages = 8;
constexpr int kTcParts = 3;     // hi, mid, lo
constexpr int kTcKMax = 8;
constexpr int kTcCandMax = 24;
constexpr int kTcSelWarps = 4;  // warps per fallback CTA (one token)
constexpr int kTcMaxD = 16384;  // the fallback stages the d bf16 of a row in shared memory
constexpr int kTcTmemCols = 512;
constexpr int kTcSplitSeg = 16; // column segments per expert row in the split

__global__ void __launch_bounds__(256) gate_split_kernel(const float* __restrict__ wg, int E,
                                                         int Ep, int d,
                                                         __nv_bfloat16* __restrict__ w3,
                                                         double* __restrict__ sums) {
  __shared__ double red[4][256];
  const int e = blockIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // w^2, hi^2, (mid + lo)^2, residual^2
  for (int c = blockIdx.y * 256 + threadIdx.x; c < d; c += kTcSplitSeg * 256) {
    const float w = e < E ? wg[size_t(e) * d + c] : 0.0f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    const float r1 = w - __bfloat162float(hi);  // exact (Sterbenz)
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
    w3[size_t(e) * d + c] = hi;
    w3[(size_t(Ep) + e) * d + c] = mid;
    w3[(size_t(2 * Ep) + e) * d + c] = lo;
    // exact in fp64 (0 unless a part underflows bf16's normal range)
    const double ml = double(__bfloat162float(mid)) + double(__bfloat162float(lo));
    const double res = double(w) - double(__bfloat162float(hi)) - ml;
    acc[0] += double(w) * double(w);
    acc[1] += double(__bfloat162float(hi)) * double(__bfloat162float(hi));
    acc[2] += ml * ml;
    acc[3] += res * res;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) red[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (int(threadIdx.x) < o)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 4) atomicAdd(&sums[4 * e + threadIdx.x], red[threadIdx.x][0]);
}

// g_e = gamma_hi ||hi_e|| + gamma_ml ||mid_e + lo_e|| + gamma_w ||w_e|| + ||res_e||
__global__ void gate_coef_kernel(const double* __restrict__ sums, int Ep, double gamma_hi,
                                 double gamma_ml, double gamma_w, float* __restrict__ gcoef) {
  for (int e = threadIdx.x; e < Ep; e += blockDim.x) {
    const double* q = sums + 4 * e;
    const double g = (gamma_hi * sqrt(q[1]) + gamma_ml * sqrt(q[2]) + gamma_w * sqrt(q[0]) +
                      sqrt(q[3])) *
                     (1.0 + 1e-6);
    gcoef[e] = __double2float_ru(g);
  }
}

struct TcGateArgs {
  int64_t N;
  int d, Ep, E, k, stages, seg_kb, n_seg, force_exact;  // n_seg hi segments (+1 mid/lo)
  const float* gcoef;
  const float* bias;
  int32_t* topk_idx;
  float* topk_w;
  int32_t* counts;
  int32_t* fb_list;    // uncertified tokens
  int32_t* fb_count;
  float* fb_logits;    // [fb slot][Ep] their L~ (no bias)
  float* approx;       // optional [N][Ep] L~ of every token (test hook)
  unsigned long long* stats;  // [2]: certified tokens
};

__device__ __forceinline__ float tc_bound(float nx, float g, float v) {
  return __fadd_ru(__fmaf_ru(nx, g, 1e-30f), __fmul_ru(fabsf(v), 2.4e-7f));
}

template <int K>
__global__ void __launch_bounds__(kTcThreads, 1) gate_tc_kernel(
    const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
    const TcGateArgs a) {
  using namespace gemm;
  extern __shared__ uint8_t tc_smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ int hist[128];
  const uint32_t base = (smem_u32(tc_smem) + 1023u) & ~1023u;
  const uint32_t A_BYTES = kTcTok * ROW_BYTES;
  const uint32_t P_BYTES = uint32_t(a.Ep) * ROW_BYTES;
  const uint32_t STAGE = A_BYTES + kTcParts * P_BYTES;
  const int stages = a.stages;
  const uint32_t bar0 = base + uint32_t(stages) * STAGE;
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kTcMaxStages + s); };
  const uint32_t accf_bar = bar0 + 8u * (2 * kTcMaxStages);
  const uint32_t acce_bar = accf_bar + 8u;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1 + 4);  // the MMA commit + the 4 norm/epilogue warps
    }
    mbar_init(accf_bar, 1);
    mbar_init(acce_bar, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "n"(kTcTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int64_t N = a.N;
  const int Ep = a.Ep;
  const int64_t n_tiles = (N + kTcTok - 1) / kTcTok;
  const int kblocks = a.d / (ROW_BYTES / 2);

  if (warp == 0) {  // ---- TMA producer: x tile + the W_g parts per K-block
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_first(), pol_w = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x)
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sA = base + uint32_t(stage) * STAGE;
          mbar_expect_tx(full_bar(stage), STAGE);
          tma_load_2d(sA, &tmap_x, full_bar(stage), kb * 64, int32_t(t * kTcTok), pol_x);
          for (int p = 0; p < kTcParts; ++p)
            tma_load_2d(sA + A_BYTES + p * P_BYTES, &tmap_w, full_bar(stage), kb * 64, p * Ep,
                        pol_w);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
    }
  } else if (warp == 1) {  // ---- MMA issuer (one elected lane)
    const uint32_t idesc = make_idesc<false>(uint32_t(Ep));
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      mbar_wait(acce_bar, acc_phase ^ 1);  // the previous tile's epilogue has read TMEM
      tc_fence_after();
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sA = base + uint32_t(stage) * STAGE;
          const uint64_t da = sdesc(sA);
          // hi -> its K segment's accumulator; mid and lo -> one shared accumulator
          const uint32_t d_hi = tmem + uint32_t((kb / a.seg_kb) * Ep);
          const uint32_t d_ml = tmem + uint32_t(a.n_seg * Ep);
          const bool first_hi = kb % a.seg_kb == 0;
          const uint64_t db_hi = sdesc(sA + A_BYTES);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma<false>(d_hi, da + 2 * kk, db_hi + 2 * kk, idesc, (first_hi && kk == 0) ? 0u : 1u);
#pragma unroll
          for (int p = 1; p < kTcParts; ++p) {
            const uint64_t db = sdesc(sA + A_BYTES + p * P_BYTES);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma<false>(d_ml, da + 2 * kk, db + 2 * kk, idesc,
                         (kb == 0 && p == 1 && kk == 0) ? 0u : 1u);
          }
          tc_commit(empty_bar(stage));
        }
        __syncwarp();
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit(accf_bar);
      __syncwarp();
      acc_phase ^= 1;
    }
  } else {  // ---- norm + certification epilogue: thread = token row
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
    const int r = quarter * 32 + lane;
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      // ||x_t||^2 from the staged tiles: row r's 8 16-byte chunks (SW128:
      // chunk j of row r sits at j ^ (r & 7))
      float ssj[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};  // 8 short chains
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(full_bar(stage), phase);
        const uint8_t* row = tc_smem + (base - smem_u32(tc_smem)) + size_t(stage) * STAGE +
                             size_t(r) * ROW_BYTES;
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          v[j] = *reinterpret_cast<const uint4*>(row + ((j ^ (r & 7)) << 4));
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(stage));  // the row is in registers
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float p = __uint_as_float(w4[i] << 16), q = __uint_as_float(w4[i] & 0xffff0000u);
            ssj[j] = fmaf(p, p, ssj[j]);
            ssj[j] = fmaf(q, q, ssj[j]);
          }
        }
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
      float ss = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += ssj[j];
      // >= ||x_t||_2 (the fp32 sum of d squares is within (d/8 + 8) 2^-24 of exact)
      const float nx = __fmul_ru(__fsqrt_ru(ss), 1.001f);
      mbar_wait(accf_bar, acc_phase);
      tc_fence_after();
      const int64_t tok = t * kTcTok + r;
      const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16);
      // running top-K by L~ (ties -> lower index: experts arrive ascending)
      float tv[K], tlo[K], tup[K];
      int ti[K];
#pragma unroll
      for (int j = 0; j < K; ++j) { tv[j] = -INFINITY; tlo[j] = tup[j] = -INFINITY; ti[j] = -1; }
      float rest_up = -INFINITY;
      bool bad = !(nx <= 3.0e38f);
      for (int cc = 0; cc < Ep / 32; ++cc) {
        float acc[32];
        uint32_t rr[32], r2[32];
        tmem_ld32(taddr + cc * 32, rr);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = __uint_as_float(rr[i]);
        int sg = 1;
        for (; sg + 1 < a.n_seg; sg += 2) {  // two segment loads in flight
          tmem_ld32_nowait(taddr + uint32_t(sg * Ep) + cc * 32, rr);
          tmem_ld32_nowait(taddr + uint32_t((sg + 1) * Ep) + cc * 32, r2);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] += __uint_as_float(rr[i]);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] += __uint_as_float(r2[i]);
        }
        if (sg < a.n_seg) {
          tmem_ld32(taddr + uint32_t(sg * Ep) + cc * 32, rr);
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] += __uint_as_float(rr[i]);
        }
        tmem_ld32(taddr + uint32_t(a.n_seg * Ep) + cc * 32, rr);  // + (mid + lo)
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] += __uint_as_float(rr[i]);
        if (a.approx && tok < N) {
          float4* dst = reinterpret_cast<float4*>(a.approx + tok * Ep + cc * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
        }
        if (a.fb_logits && tok < N) {  // kept for the fallback in case the token is not certified
          float4* dst = reinterpret_cast<float4*>(a.fb_logits + tok * Ep + cc * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int e = cc * 32 + i;
          if (e >= a.E) break;
          const float v = a.bias ? __fadd_rn(acc[i], a.bias[e]) : acc[i];
          const float B = tc_bound(nx, a.gcoef[e], v);
          if (!(fabsf(v) <= 3.0e38f) || !(B <= 3.0e38f)) bad = true;
          const float lo = __fsub_rd(v, B), up = __fadd_ru(v, B);
          // insert (v, e) into the sorted top-K; whatever falls out joins the rest
          float cv = v, clo = lo, cup = up;
          int ci = e;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            if (cv > tv[j]) {
              const float sv = tv[j], slo = tlo[j], sup = tup[j];
              const int si = ti[j];
              tv[j] = cv; tlo[j] = clo; tup[j] = cup; ti[j] = ci;
              cv = sv; clo = slo; cup = sup; ci = si;
            }
          }
          if (ci >= 0) rest_up = fmaxf(rest_up, cup);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acce_bar);  // TMEM may be overwritten now
      acc_phase ^= 1;
      if (tok < N) {
        bool ok = !bad && !a.force_exact && ti[K - 1] >= 0;
#pragma unroll
        for (int j = 0; j + 1 < K; ++j) ok = ok && tlo[j] > tup[j + 1];
        ok = ok && tlo[K - 1] > rest_up;
        if (ok) {  // certified: the exact chain picks the same experts in the same order
          float ps = 0.0f, pj[K];
#pragma unroll
          for (int j = 0; j < K; ++j) { pj[j] = expf(tv[j] - tv[0]); ps += pj[j]; }
#pragma unroll
          for (int j = 0; j < K; ++j) {
            a.topk_idx[tok * K + j] = ti[j];
            a.topk_w[tok * K + j] = pj[j] / ps;
            atomicAdd(&hist[ti[j]], 1);
          }
        } else {
          const int pos = atomicAdd(a.fb_count, 1);
          a.fb_list[pos] = int32_t(tok);
        }
        const unsigned m = __ballot_sync(__activemask(), ok);
        if (a.stats && (lane == __ffs(__activemask()) - 1))
          atomicAdd(&a.stats[0], static_cast<unsigned long long>(__popc(m)));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  for (int e = threadIdx.x; e < a.E; e += blockDim.x)
    if (hist[e]) atomicAdd(&a.counts[e], hist[e]);
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTcTmemCols)
                 : "memory");
  }
}

// the CUDA-core gate's logit for one (token, expert), by one warp: lane l's
// fmaf chain over columns 8l..8l+7 of every 256-column chunk (columns past d
// contribute fmaf(0, 0, acc)), butterfly, + bias.  x row from shared memory;
// the weight slices of 8 chunks are requested before the chain consumes them.
__device__ __forceinline__ void fma8(float& acc, const uint4 raw, const float4 a,
                                     const float4 b) {
  acc = fmaf(__uint_as_float(raw.x << 16), a.x, acc);
  acc = fmaf(__uint_as_float(raw.x & 0xffff0000u), a.y, acc);
  acc = fmaf(__uint_as_float(raw.y << 16), a.z, acc);
  acc = fmaf(__uint_as_float(raw.y & 0xffff0000u), a.w, acc);
  acc = fmaf(__uint_as_float(raw.z << 16), b.x, acc);
  acc = fmaf(__uint_as_float(raw.z & 0xffff0000u), b.y, acc);
  acc = fmaf(__uint_as_float(raw.w << 16), b.z, acc);
  acc = fmaf(__uint_as_float(raw.w & 0xffff0000u), b.w, acc);
}

__device__ __forceinline__ float exact_logit(const __nv_bfloat16* xs,
                                             const float* __restrict__ wr, int d, int lane,
                                             const float* bias, int e) {
  constexpr int G = 8;
  const int nch = (d + 255) / 256;
  float acc = 0.0f;
  for (int cb = 0; cb < nch; cb += G) {
    float4 wa[G], wb[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int c = (cb + j) * 256 + lane * 8;
      if (cb + j < nch && c < d) {
        wa[j] = __ldg(reinterpret_cast<const float4*>(wr + c));
        wb[j] = __ldg(reinterpret_cast<const float4*>(wr + c) + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      if (cb + j < nch) {
        const int c = (cb + j) * 256 + lane * 8;
        if (c < d) fma8(acc, *reinterpret_cast<const uint4*>(xs + c), wa[j], wb[j]);
        else acc = __fadd_rn(acc, 0.0f);  // == fmaf(0, 0, acc), also for acc = -0
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  return bias ? __fadd_rn(acc, bias[e]) : acc;
}

// one CTA (kTcSelWarps warps) per uncertified token listed by gate_tc_kernel,
// persistent over the list: the warps stage the x row in shared memory
// together, each derives the same candidate set, and candidate i's exact chain
// runs on warp i % kTcSelWarps; warp 0 then picks the top-k.
__global__ void __launch_bounds__(kTcSelWarps * 32) gate_tc_fallback_kernel(
    const __nv_bfloat16* __restrict__ x, int d, const float* __restrict__ wg,
    const float* __restrict__ bias, int E, int Ep, int k, const int32_t* __restrict__ fb_list,
    const int32_t* __restrict__ fb_count, const float* __restrict__ logits,
    const float* __restrict__ gcoef, int force_exact, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_w, int32_t* __restrict__ counts,
    unsigned long long* __restrict__ stats) {
  constexpr int SQ = 4;  // experts per lane (E <= 128)
  constexpr int W = kTcSelWarps;
  extern __shared__ __align__(16) uint8_t sel_smem[];
  __shared__ int hist[128];
  __shared__ float ss_w[W];
  __shared__ float ex_s[128];
  const int64_t n_fb = *fb_count;
  if (int64_t(blockIdx.x) >= n_fb) return;
  for (int i = threadIdx.x; i < E; i += blockDim.x) hist[i] = 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sel_smem);
  unsigned long long n_cand = 0, n_full = 0, n_tok = 0;
  for (int64_t it = blockIdx.x; it < n_fb; it += gridDim.x) {
    const int64_t tok = fb_list[it];
    const __nv_bfloat16* xr = x + tok * d;
    __syncthreads();  // the previous token is done with xs / ex_s
    // the row in 16-byte slices: slice j -> lane j % 32 of warp (j / 32) % W
    float ss = 0.0f;
    for (int c = (warp * 32 + lane) * 8; c < d; c += W * 256) {
      const uint4 raw = __ldg(reinterpret_cast<const uint4*>(xr + c));
      *reinterpret_cast<uint4*>(xs + c) = raw;
      const uint32_t wds[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float p = __uint_as_float(wds[i] << 16), q = __uint_as_float(wds[i] & 0xffff0000u);
        ss = fmaf(p, p, ss);
        ss = fmaf(q, q, ss);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) ss_w[warp] = ss;
    __syncthreads();
    ss = 0.0f;
#pragma unroll
    for (int w = 0; w < W; ++w) ss += ss_w[w];
    const float nx = __fmul_ru(__fsqrt_ru(ss), 1.001f);
    float lo_b[SQ], hi_b[SQ];
    bool live[SQ];
    bool bad = !(nx <= 3.0e38f);
#pragma unroll
    for (int q = 0; q < SQ; ++q) {
      const int e = lane + 32 * q;
      live[q] = e < E;
      lo_b[q] = hi_b[q] = 0.0f;
      if (live[q]) {
        float v = logits[tok * Ep + e];
        if (bias) v = __fadd_rn(v, bias[e]);
        const float B = tc_bound(nx, gcoef[e], v);
        lo_b[q] = __fsub_rd(v, B);
        hi_b[q] = __fadd_ru(v, B);
        if (!(fabsf(v) <= 3.0e38f) || !(B <= 3.0e38f)) bad = true;
      }
    }
    bad = __any_sync(0xffffffffu, bad);
    // v_k: the k-th largest lower bound
    float vk = 0.0f;
    {
      bool used[SQ] = {false, false, false, false};
      for (int j = 0; j < k; ++j) {
        float best = -INFINITY;
        int bi = -1;
#pragma unroll
        for (int q = 0; q < SQ; ++q)
          if (live[q] && !used[q] && (bi < 0 || lo_b[q] > best)) { best = lo_b[q]; bi = lane + 32 * q; }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const float ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (oi >= 0 && (bi < 0 || ob > best || (ob == best && oi < bi))) { best = ob; bi = oi; }
        }
#pragma unroll
        for (int q = 0; q < SQ; ++q)
          if (lane + 32 * q == bi) used[q] = true;
        vk = best;
      }
    }
    bool cand[SQ];
    int nc = 0;
#pragma unroll
    for (int q = 0; q < SQ; ++q) {
      cand[q] = live[q] && hi_b[q] >= vk;
      nc += __popc(__ballot_sync(0xffffffffu, cand[q]));
    }
    const bool full = bad || force_exact || nc > kTcCandMax;
    if (full) {
#pragma unroll
      for (int q = 0; q < SQ; ++q) cand[q] = live[q];
    }
    // candidate i (ascending expert index) -> warp i % W
    int rank = 0;
#pragma unroll
    for (int q = 0; q < SQ; ++q) {
      unsigned m = __ballot_sync(0xffffffffu, cand[q]);
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        if (rank++ % W == warp) {
          const int e = b + 32 * q;
          const float L = exact_logit(xs, wg + size_t(e) * d, d, lane, bias, e);
          if (lane == 0) ex_s[e] = L;
        }
      }
    }
    __syncthreads();
    if (warp == 0) {  // top-k over the exact candidate logits (ties and NaN -> lower index)
      float ex[SQ];
#pragma unroll
      for (int q = 0; q < SQ; ++q) ex[q] = cand[q] ? ex_s[lane + 32 * q] : 0.0f;
      float mx = -INFINITY;
#pragma unroll
      for (int q = 0; q < SQ; ++q)
        if (cand[q] && !isnan(ex[q])) mx = fmaxf(mx, ex[q]);
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float psum = 0.0f, pk_mine = 0.0f;
      int ik_mine = 0;
      for (int j = 0; j < k; ++j) {
        Cand best{0.0f, -1};
#pragma unroll
        for (int q = 0; q < SQ; ++q) {
          Cand c{ex[q], cand[q] ? lane + 32 * q : -1};
          if (better(c, best)) best = c;
        }
        for (int o = 16; o; o >>= 1) {
          Cand other{__shfl_xor_sync(0xffffffffu, best.v, o),
                     __shfl_xor_sync(0xffffffffu, best.i, o)};
          if (better(other, best)) best = other;
        }
        const float pj = expf(best.v - mx);
        psum += pj;
        if (lane == j) { pk_mine = pj; ik_mine = best.i; }
#pragma unroll
        for (int q = 0; q < SQ; ++q)
          if (lane + 32 * q == best.i) cand[q] = false;
      }
      if (lane < k) {
        topk_idx[tok * k + lane] = ik_mine;
        topk_w[tok * k + lane] = pk_mine / psum;
        atomicAdd(&hist[ik_mine], 1);
      }
    }
    n_cand += full ? unsigned(E) : unsigned(nc);
    n_full += full ? 1u : 0u;
    n_tok += 1;
  }
  if (stats && threadIdx.x == 0 && n_tok) {
    atomicAdd(&stats[1], n_tok);
    atomicAdd(&stats[2], n_cand);
    if (n_full) atomicAdd(&stats[3], n_full);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (hist[e]) atomicAdd(&counts[e], hist[e]);
}

struct TcGateWs {
  size_t w3, sums, gcoef, stats, fb_count, fb_list, fb_logits, total;
};
TcGateWs tc_gate_layout(int64_t N, int d, int Ep) {
  auto up = [](size_t v) { return (v + 1023) & ~size_t(1023); };
  const size_t n = size_t(std::max<int64_t>(N, 1));
  TcGateWs L;
  L.w3 = 0;
  L.sums = up(size_t(kTcParts) * Ep * d * 2);
  L.gcoef = up(L.sums + size_t(Ep) * 32);
  L.stats = up(L.gcoef + size_t(Ep) * 4);
  L.fb_count = L.stats + 32;
  L.fb_list = up(L.fb_count + 4);
  L.fb_logits = up(L.fb_list + n * 4);
  L.total = up(L.fb_logits + n * Ep * 4);
  return L;
}

int tc_gate_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

bool tc_gate_applies(int dtype, int64_t N, int d, int E, int k) {
  return dtype == kDtypeBf16 && k >= 2 && k <= kTcKMax && E <= 128 && d % 64 == 0 && d > 0 &&
         d <= kTcMaxD && N > 0 && tc_gate_env("INFMOE_GATE_TC", 1) != 0;
}

struct TcSeg {
  int n_seg, seg_kb;
};
TcSeg tc_segments(int d, int Ep) {
  const int kblocks = d / 64;
  const int max_seg = kTcTmemCols / Ep - 1;  // the last accumulator takes mid + lo
  TcSeg s;
  s.seg_kb = (kblocks + max_seg - 1) / max_seg;
  s.n_seg = (kblocks + s.seg_kb - 1) / s.seg_kb;
  return s;
}

// step 0 into ws: the bf16 parts of W_g and the per-expert bound coefficients
void tc_gate_prepare(const float* wg, int E, int d, uint8_t* ws, cudaStream_t s) {
  const int Ep = (E + 31) / 32 * 32;
  const TcGateWs L = tc_gate_layout(1, d, Ep);
  auto* sums = reinterpret_cast<double*>(ws + L.sums);
  INFMOE_CUDA(cudaMemsetAsync(sums, 0, size_t(Ep) * 32, s));
  gate_split_kernel<<<dim3(unsigned(Ep), kTcSplitSeg), 256, 0, s>>>(
      wg, E, Ep, d, reinterpret_cast<__nv_bfloat16*>(ws + L.w3), sums);
  INFMOE_LAUNCH_CHECK();
  const TcSeg sg = tc_segments(d, Ep);
  const int m_hi = 4 * sg.seg_kb;                      // tcgen05.mma per hi accumulator
  const int m_ml = 4 * (kTcParts - 1) * (d / 64);      // ... into the mid/lo accumulator
  const int dpad = (d + 255) / 256 * 256;
  const double gamma_hi = std::ldexp(17.0 * (m_hi + 1), -23);
  const double gamma_ml = std::ldexp(17.0 * (m_ml + 1), -23);
  const double gamma_w = std::ldexp(double(sg.n_seg + 1), -24) + std::ldexp(dpad / 32.0 + 8.0, -23);
  gate_coef_kernel<<<1, 128, 0, s>>>(sums, Ep, gamma_hi, gamma_ml, gamma_w,
                                     reinterpret_cast<float*>(ws + L.gcoef));
  INFMOE_LAUNCH_CHECK();
}

void tc_gate_go(const void* x, int64_t N, int d, const float* wg, const float* bias, int E, int k,
                int32_t* idx, float* w, int32_t* counts, uint8_t* ws, float* approx_out,
                unsigned long long* stats_out, cudaStream_t s) {
  const int Ep = (E + 31) / 32 * 32;
  const TcGateWs L = tc_gate_layout(N, d, Ep);
  const int force = tc_gate_env("INFMOE_GATE_TC_FORCE_EXACT", 0);
  auto* stats = reinterpret_cast<unsigned long long*>(ws + L.stats);
  auto* fb_count = reinterpret_cast<int32_t*>(ws + L.fb_count);
  auto* fb_list = reinterpret_cast<int32_t*>(ws + L.fb_list);
  auto* fb_logits = reinterpret_cast<float*>(ws + L.fb_logits);
  INFMOE_CUDA(cudaMemsetAsync(stats, 0, 32 + 4, s));  // stats[4] + fb_count

  const uint32_t stage_bytes = uint32_t(gemm::BM + kTcParts * Ep) * gemm::ROW_BYTES;
  const int stages = std::min<int>(kTcMaxStages, int((200u * 1024u) / stage_bytes));
  const size_t smem = size_t(stages) * stage_bytes + 1024 + 8 * (2 * kTcMaxStages + 2);
  const void* kern = nullptr;
  switch (k) {
    case 2: kern = reinterpret_cast<const void*>(gate_tc_kernel<2>); break;
    case 3: kern = reinterpret_cast<const void*>(gate_tc_kernel<3>); break;
    case 4: kern = reinterpret_cast<const void*>(gate_tc_kernel<4>); break;
    case 5: kern = reinterpret_cast<const void*>(gate_tc_kernel<5>); break;
    case 6: kern = reinterpret_cast<const void*>(gate_tc_kernel<6>); break;
    case 7: kern = reinterpret_cast<const void*>(gate_tc_kernel<7>); break;
    default: kern = reinterpret_cast<const void*>(gate_tc_kernel<8>); break;
  }
  ensure_dyn_smem(kern, smem);
  const CUtensorMap tx = gemm::make_tmap(x, uint64_t(N), uint64_t(d), false, kTcTok);
  const CUtensorMap tw =
      gemm::make_tmap(ws + L.w3, uint64_t(kTcParts * Ep), uint64_t(d), false, uint32_t(Ep));
  const TcSeg sg = tc_segments(d, Ep);
  TcGateArgs a;
  a.N = N; a.d = d; a.Ep = Ep; a.E = E; a.k = k; a.stages = stages;
  a.seg_kb = sg.seg_kb; a.n_seg = sg.n_seg; a.force_exact = force;
  a.gcoef = reinterpret_cast<const float*>(ws + L.gcoef);
  a.bias = bias; a.topk_idx = idx; a.topk_w = w; a.counts = counts;
  a.fb_list = fb_list; a.fb_count = fb_count; a.fb_logits = fb_logits;
  a.approx = nullptr; a.stats = stats;
  const int64_t tiles = (N + kTcTok - 1) / kTcTok;
  const int grid = int(std::min<int64_t>(tiles, device_sm_count()));
  void* kargs[] = {const_cast<CUtensorMap*>(&tx), const_cast<CUtensorMap*>(&tw), &a};
  INFMOE_CUDA(cudaLaunchKernel(kern, dim3(unsigned(grid)), dim3(kTcThreads), kargs, smem, s));
  INFMOE_LAUNCH_CHECK();

  const size_t sel_smem = size_t(d) * 2;  // one x row per CTA
  ensure_dyn_smem(reinterpret_cast<const void*>(gate_tc_fallback_kernel), sel_smem);
  int per_sm = 0;
  INFMOE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, gate_tc_fallback_kernel, kTcSelWarps * 32, sel_smem));
  const int64_t fb_grid = std::min<int64_t>(N, int64_t(std::max(per_sm, 1)) * device_sm_count());
  gate_tc_fallback_kernel<<<unsigned(fb_grid), kTcSelWarps * 32, sel_smem, s>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), d, wg, bias, E, Ep, k, fb_list, fb_count,
      fb_logits, a.gcoef, force, idx, w, counts, stats);
  INFMOE_LAUNCH_CHECK();
  if (approx_out)  // every token's L~ is in fb_logits (Ep-strided)
    INFMOE_CUDA(cudaMemcpy2DAsync(approx_out, size_t(E) * 4, fb_logits, size_t(Ep) * 4,
                                  size_t(E) * 4, size_t(N), cudaMemcpyDeviceToDevice, s));
  if (stats_out)
    INFMOE_CUDA(cudaMemcpyAsync(stats_out, stats, 32, cudaMemcpyDeviceToDevice, s));
}

template <typename T, int EB>
void softmax_go(const void* x, int64_t N, int d, const float* wg, const float* bias, int E, int k,
                int32_t* idx, float* w, int32_t* counts, cudaStream_t s) {
  using C = SoftCfg<T, EB>;
  auto kern = gate_softmax_kernel<T, EB>;
  const size_t smem = C::smem(E);
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  const int warps = (E + EB - 1) / EB;
  kern<<<unsigned((N + C::TT - 1) / C::TT), warps * 32, smem, s>>>(
      reinterpret_cast<const T*>(x), N, d, wg, bias, E, k, idx, w, counts);
}

template <typename T>
void softmax_launch(const void* x, int64_t N, int d, const float* wg, const float* bias, int E,
                    int k, int32_t* idx, float* w, int32_t* counts, cudaStream_t s) {
  // experts per warp EB (TT*EB = 64 accumulators per lane): 4 experts x 16
  // tokens up to 64 experts (measured best at E = 32 and 64: each CTA streams
  // all of W_g once, the weight slices stay in registers across 16 tokens),
  // 16 x 4 beyond
  if (E <= 64) softmax_go<T, 4>(x, N, d, wg, bias, E, k, idx, w, counts, s);
  else softmax_go<T, 16>(x, N, d, wg, bias, E, k, idx, w, counts, s);
}

}  // namespace

size_t gate_softmax_ws_bytes(int dtype, int64_t N, int d, int E, int k) {
  if (!tc_gate_applies(dtype, std::max<int64_t>(N, 1), d, E, k)) return 0;
  return tc_gate_layout(N, d, (E + 31) / 32 * 32).total;
}

void gate_softmax_prepare(const float* wg, int d, int E, void* ws, cudaStream_t stream) {
  require(ws != nullptr && wg != nullptr, "softmax gate prepare: NULL pointer");
  tc_gate_prepare(wg, E, d, static_cast<uint8_t*>(ws), stream);
}

void launch_gate_softmax(const void* x, int dtype, int64_t N, int d, const float* wg,
                         const float* bias, int E, int k, int32_t* topk_idx, float* topk_w,
                         int32_t* counts, cudaStream_t stream, void* ws, size_t ws_bytes,
                         bool ws_prepared, float* approx_logits, unsigned long long* tc_stats) {
  require(E >= 1 && E <= 128, "softmax gate: n_experts must be in [1, 128]");
  require(k >= 1 && k <= 8 && k <= E, "softmax gate: top_k must be in [1, min(8, E)]");
  require(d >= 1, "softmax gate: d_model must be >= 1");
  require(d % 8 == 0, "softmax gate: d_model must be a multiple of 8");
  require(reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(wg) % 16 == 0,
          "softmax gate: x and gate weights must be 16-byte aligned");
  INFMOE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * size_t(E), stream));
  if (N == 0) return;
  const size_t need = gate_softmax_ws_bytes(dtype, N, d, E, k);
  if (need) {  // tensor-core logits + certified exact selection
    require(reinterpret_cast<uintptr_t>(x) % 16 == 0, "softmax gate: x must be 16-byte aligned");
    uint8_t* w = static_cast<uint8_t*>(ws);
    const bool own = w == nullptr || ws_bytes < need;
    if (own) INFMOE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&w), need, stream));
    if (own || !ws_prepared) tc_gate_prepare(wg, E, d, w, stream);
    tc_gate_go(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, w, approx_logits, tc_stats,
               stream);
    if (own) INFMOE_CUDA(cudaFreeAsync(w, stream));
    return;
  }
  if (tc_stats) INFMOE_CUDA(cudaMemsetAsync(tc_stats, 0xff, 32, stream));  // not on this path
  if (dtype == kDtypeBf16)
    softmax_launch<__nv_bfloat16>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
  else
    softmax_launch<float>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
  INFMOE_LAUNCH_CHECK();
}

void launch_gate_lsh(const void* x, int dtype, int64_t N, int d, const double* proj, int bits,
                     int E, uint32_t* codes, int32_t* topk_idx, float* topk_w, int32_t* counts,
                     cudaStream_t stream) {
  require(bits >= 1 && bits <= 31, "gating: n_hash_bits must be in [1, 31]");
  require(E >= 1, "route_tokens: n_experts must be >= 1");
  require((1u << bits) >= uint32_t(E), "gating: 2^n_hash_bits must be >= n_experts");
  const size_t esz = dtype_bytes(dtype);
  require(d % 8 == 0, "lsh gate: d_model must be a multiple of 8");
  require(reinterpret_cast<uintptr_t>(proj) % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0,
          "lsh gate: x and proj must be 16-byte aligned");
  INFMOE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * size_t(E), stream));
  if (N == 0) return;
  static const int fast = lsh_env("INFMOE_LSH_FAST", 1);
  static const int mma = lsh_env("INFMOE_LSH_MMA", 1);
  if (fast && mma && bits <= 8 && d % 8 == 0) {  // certified fast path on fp64 MMA
    if (dtype == kDtypeBf16)
      lsh_mma_go<__nv_bfloat16>(x, N, d, proj, bits, E, codes, topk_idx, topk_w, counts, stream);
    else
      lsh_mma_go<float>(x, N, d, proj, bits, E, codes, topk_idx, topk_w, counts, stream);
    INFMOE_LAUNCH_CHECK();
    return;
  }
  if (fast && bits <= 8) {
    const bool bf = dtype == kDtypeBf16;
    if (bits <= 4) {
      if (bf) lsh_fast_go<__nv_bfloat16, 4>(x, N, d, proj, bits, E, codes, topk_idx, topk_w, counts, stream);
      else lsh_fast_go<float, 4>(x, N, d, proj, bits, E, codes, topk_idx, topk_w, counts, stream);
    } else {
      if (bf) lsh_fast_go<__nv_bfloat16, 8>(x, N, d, proj, bits, E, codes, topk_idx, topk_w, counts, stream);
      else lsh_fast_go<float, 8>(x, N, d, proj, bits, E, codes, topk_idx, topk_w, counts, stream);
    }
    INFMOE_LAUNCH_CHECK();
    return;
  }
  const int G = 32 / bits;
  const int TB = kLshWarps * G;
  const int64_t blocks = (N + TB - 1) / TB;
  const size_t smem = kGateStages * (size_t(TB) * (kLshChunk + 16 / esz) * esz +
                                     size_t(bits) * (kLshChunk + 2) * sizeof(double));
  if (dtype == kDtypeBf16) {
    auto kern = gate_lsh_kernel<__nv_bfloat16>;
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<unsigned(blocks), kLshWarps * 32, smem, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), N, d, proj, bits, E, codes, topk_idx, topk_w,
        counts);
  } else {
    auto kern = gate_lsh_kernel<float>;
    ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<unsigned(blocks), kLshWarps * 32, smem, stream>>>(reinterpret_cast<const float*>(x), N, d,
                                                             proj, bits, E, codes, topk_idx,
                                                             topk_w, counts);
  }
  INFMOE_LAUNCH_CHECK();
}

}  // namespace infmoe
