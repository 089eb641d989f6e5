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
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace infmoe {
namespace {

constexpr int kChunk = 32;  // d-chunk staged per iteration

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

template <typename T, int EQ, int TPW>
__global__ void __launch_bounds__(256) gate_softmax_kernel(
    const T* __restrict__ x, int64_t N, int d, const float* __restrict__ wg,
    const float* __restrict__ bias, int E, int k, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_w, int32_t* __restrict__ counts) {
  constexpr int EP = 32 * EQ;
  constexpr int TB = 8 * TPW;
  __shared__ float xs[TB][kChunk];
  __shared__ float ws[kChunk][EP + 1];
  __shared__ int hist[EP];

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t tok0 = int64_t(blockIdx.x) * TB;
  for (int i = threadIdx.x; i < EP; i += blockDim.x) hist[i] = 0;

  float acc[TPW][EQ];
#pragma unroll
  for (int t = 0; t < TPW; ++t)
#pragma unroll
    for (int q = 0; q < EQ; ++q) acc[t][q] = 0.0f;

  for (int c0 = 0; c0 < d; c0 += kChunk) {
    const int cn = min(kChunk, d - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < TB * kChunk; i += blockDim.x) {
      const int t = i / kChunk, c = i % kChunk;
      const int64_t tok = tok0 + t;
      xs[t][c] = (tok < N && c < cn) ? load_as_f32(x, size_t(tok) * d + c0 + c) : 0.0f;
    }
    for (int i = threadIdx.x; i < EP * kChunk; i += blockDim.x) {
      const int e = i / kChunk, c = i % kChunk;
      ws[c][e] = (e < E && c < cn) ? wg[size_t(e) * d + c0 + c] : 0.0f;
    }
    __syncthreads();
    for (int c = 0; c < cn; ++c) {
      float wv[EQ];
#pragma unroll
      for (int q = 0; q < EQ; ++q) wv[q] = ws[c][lane + 32 * q];
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const float xv = xs[warp * TPW + t][c];
#pragma unroll
        for (int q = 0; q < EQ; ++q) acc[t][q] = fmaf(xv, wv[q], acc[t][q]);
      }
    }
  }

#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int64_t tok = tok0 + warp * TPW + t;
    float lg[EQ];
    bool live[EQ];
#pragma unroll
    for (int q = 0; q < EQ; ++q) {
      const int e = lane + 32 * q;
      live[q] = e < E;
      lg[q] = live[q] ? (bias ? __fadd_rn(acc[t][q], bias[e]) : acc[t][q]) : 0.0f;
    }
    // softmax denominator over all experts (fp32; weights are tolerance-checked)
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < EQ; ++q)
      if (live[q] && !isnan(lg[q])) mx = fmaxf(mx, lg[q]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.0f;
#pragma unroll
    for (int q = 0; q < EQ; ++q)
      if (live[q]) se += expf(lg[q] - mx);
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);

    float pk[8];
    int ik[8];
    float psum = 0.0f;
    for (int j = 0; j < k; ++j) {
      Cand best{0.0f, -1};
#pragma unroll
      for (int q = 0; q < EQ; ++q) {
        Cand c{lg[q], live[q] ? lane + 32 * q : -1};
        if (better(c, best)) best = c;
      }
      for (int o = 16; o; o >>= 1) {
        Cand other{__shfl_xor_sync(0xffffffffu, best.v, o),
                   __shfl_xor_sync(0xffffffffu, best.i, o)};
        if (better(other, best)) best = other;
      }
      ik[j] = best.i;
      pk[j] = expf(best.v - mx) / se;
      psum += pk[j];
#pragma unroll
      for (int q = 0; q < EQ; ++q)
        if (lane + 32 * q == best.i) live[q] = false;  // exclude from the next pick
    }
    if (lane == 0 && tok < N) {
      for (int j = 0; j < k; ++j) {
        topk_idx[tok * k + j] = ik[j];
        topk_w[tok * k + j] = k > 1 ? pk[j] / psum : pk[j];
        atomicAdd(&hist[ik[j]], 1);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (hist[e]) atomicAdd(&counts[e], hist[e]);
}

// LSH: lane = (token sub-slot, hash bit); tokens per warp = 32 / bits.
template <typename T>
__global__ void __launch_bounds__(128) gate_lsh_kernel(
    const T* __restrict__ x, int64_t N, int d, const double* __restrict__ proj, int bits, int E,
    uint32_t* __restrict__ codes, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
    int32_t* __restrict__ counts) {
  constexpr int kWarps = 4;
  constexpr int kLshChunk = 32;
  __shared__ float xs[kWarps * 32][kLshChunk + 1];
  __shared__ double ps[kLshChunk][32];
  __shared__ int hist[1024];

  const int G = 32 / bits;  // tokens per warp
  const int TB = kWarps * G;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int sub = lane / bits, j = lane % bits;
  const bool active = sub < G;
  const int64_t tok0 = int64_t(blockIdx.x) * TB;
  const int local_tok = warp * G + (active ? sub : 0);
  for (int i = threadIdx.x; i < E && i < 1024; i += blockDim.x) hist[i] = 0;

  double dot = 0.0;
  for (int c0 = 0; c0 < d; c0 += kLshChunk) {
    const int cn = min(kLshChunk, d - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < TB * kLshChunk; i += blockDim.x) {
      const int t = i / kLshChunk, c = i % kLshChunk;
      const int64_t tok = tok0 + t;
      xs[t][c] = (tok < N && c < cn) ? load_as_f32(x, size_t(tok) * d + c0 + c) : 0.0f;
    }
    for (int i = threadIdx.x; i < bits * kLshChunk; i += blockDim.x) {
      const int b = i / kLshChunk, c = i % kLshChunk;
      ps[c][b] = c < cn ? proj[size_t(b) * d + c0 + c] : 0.0;
    }
    __syncthreads();
    if (active) {
      for (int c = 0; c < cn; ++c)
        dot = __dadd_rn(dot, __dmul_rn(double(xs[local_tok][c]), ps[c][j]));
    }
  }
  const unsigned mask = __ballot_sync(0xffffffffu, active && dot >= 0.0);
  const int64_t tok = tok0 + local_tok;
  if (active && j == 0 && tok < N) {
    const uint32_t code = (mask >> (sub * bits)) & ((bits >= 32) ? 0xffffffffu : ((1u << bits) - 1u));
    const int e = int(code % uint32_t(E));
    if (codes) codes[tok] = code;
    topk_idx[tok] = e;
    topk_w[tok] = 1.0f;
    if (E <= 1024) atomicAdd(&hist[e], 1);
    else atomicAdd(&counts[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E && e < 1024; e += blockDim.x)
    if (hist[e]) atomicAdd(&counts[e], hist[e]);
}

template <typename T, int EQ, int TPW>
void softmax_launch(const void* x, int64_t N, int d, const float* wg, const float* bias, int E,
                    int k, int32_t* idx, float* w, int32_t* counts, cudaStream_t s) {
  const int64_t blocks = (N + 8 * TPW - 1) / (8 * TPW);
  gate_softmax_kernel<T, EQ, TPW><<<unsigned(blocks), 256, 0, s>>>(
      reinterpret_cast<const T*>(x), N, d, wg, bias, E, k, idx, w, counts);
}

}  // namespace

void launch_gate_softmax(const void* x, int dtype, int64_t N, int d, const float* wg,
                         const float* bias, int E, int k, int32_t* topk_idx, float* topk_w,
                         int32_t* counts, cudaStream_t stream) {
  require(E >= 1 && E <= 128, "softmax gate: n_experts must be in [1, 128]");
  require(k >= 1 && k <= 8 && k <= E, "softmax gate: top_k must be in [1, min(8, E)]");
  require(d >= 1, "softmax gate: d_model must be >= 1");
  INFMOE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * size_t(E), stream));
  if (N == 0) return;
  const bool bf = dtype == kDtypeBf16;
  if (E <= 32) {
    if (bf) softmax_launch<__nv_bfloat16, 1, 4>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
    else softmax_launch<float, 1, 4>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
  } else if (E <= 64) {
    if (bf) softmax_launch<__nv_bfloat16, 2, 2>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
    else softmax_launch<float, 2, 2>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
  } else {
    if (bf) softmax_launch<__nv_bfloat16, 4, 1>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
    else softmax_launch<float, 4, 1>(x, N, d, wg, bias, E, k, topk_idx, topk_w, counts, stream);
  }
  INFMOE_LAUNCH_CHECK();
}

void launch_gate_lsh(const void* x, int dtype, int64_t N, int d, const double* proj, int bits,
                     int E, uint32_t* codes, int32_t* topk_idx, float* topk_w, int32_t* counts,
                     cudaStream_t stream) {
  require(bits >= 1 && bits <= 31, "gating: n_hash_bits must be in [1, 31]");
  require(E >= 1, "route_tokens: n_experts must be >= 1");
  require((1u << bits) >= uint32_t(E), "gating: 2^n_hash_bits must be >= n_experts");
  INFMOE_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * size_t(E), stream));
  if (N == 0) return;
  const int G = 32 / bits;
  const int64_t blocks = (N + 4 * G - 1) / (4 * G);
  if (dtype == kDtypeBf16)
    gate_lsh_kernel<<<unsigned(blocks), 128, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(x), N, d, proj, bits, E, codes, topk_idx, topk_w,
        counts);
  else
    gate_lsh_kernel<<<unsigned(blocks), 128, 0, stream>>>(reinterpret_cast<const float*>(x), N, d,
                                                           proj, bits, E, codes, topk_idx, topk_w,
                                                           counts);
  INFMOE_LAUNCH_CHECK();
}

}  // namespace infmoe
