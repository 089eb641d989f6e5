// dispatch.cu — N2 token dispatch (stable counting sort + row gather) and N5
// combine (its gate-weighted inverse).
//
// Dispatch is a stable counting sort over the N*k (token, slot) assignments,
// so the permutation is deterministic and equals oracle.c or_dispatch bit for
// bit.  Up to 32768 assignments and 128 experts it is one single-CTA launch
// (dispatch_small_kernel); beyond, three launches:
//   1. per-chunk histograms               (one CTA per 2048 assignments)
//   2. exclusive scan -> offsets[E+1] and each chunk's base per expert
//   3. per-chunk stable scatter: warps own contiguous sub-ranges, ranks inside a
//      warp come from __match_any_sync peer masks.
// The row gather and the combine move 16-byte vectors, one warp per row, and
// are HBM-bound.
#include "common.cuh"
#include "kernels.cuh"

namespace infmoe {
namespace {

constexpr int kChunkAssign = 2048;
constexpr int kScatterWarps = 8;
constexpr int kMaxExpertsDispatch = 1024;

__global__ void chunk_histogram_kernel(const int32_t* __restrict__ idx, int64_t n, int E,
                                       int32_t* __restrict__ chunk_hist) {
  extern __shared__ int h[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const int64_t a0 = int64_t(blockIdx.x) * kChunkAssign;
  const int64_t a1 = min(n, a0 + kChunkAssign);
  for (int64_t a = a0 + threadIdx.x; a < a1; a += blockDim.x) atomicAdd(&h[idx[a]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) chunk_hist[size_t(blockIdx.x) * E + e] = h[e];
}

// one CTA: per expert, running sum over chunks; then exclusive scan over experts
__global__ void dispatch_scan_kernel(int32_t* __restrict__ chunk_hist, int n_chunks, int E,
                                     int32_t* __restrict__ offsets) {
  extern __shared__ int tot[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = 0;
    for (int b = 0; b < n_chunks; ++b) {
      const int c = chunk_hist[size_t(b) * E + e];
      chunk_hist[size_t(b) * E + e] = run;  // becomes the chunk's base inside expert e
      run += c;
    }
    tot[e] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = acc;
      acc += tot[e];
    }
    offsets[E] = acc;
  }
}

__global__ void __launch_bounds__(kScatterWarps * 32)
    dispatch_scatter_kernel(const int32_t* __restrict__ idx, int64_t n, int E,
                            const int32_t* __restrict__ chunk_base,
                            const int32_t* __restrict__ offsets, int32_t* __restrict__ perm,
                            int32_t* __restrict__ inv) {
  extern __shared__ int wb[];  // [kScatterWarps][E]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kPerWarp = kChunkAssign / kScatterWarps;
  const int64_t a0 = int64_t(blockIdx.x) * kChunkAssign + int64_t(warp) * kPerWarp;
  const int64_t a1 = min(n, a0 + kPerWarp);
  for (int i = threadIdx.x; i < kScatterWarps * E; i += blockDim.x) wb[i] = 0;
  __syncthreads();
  for (int64_t a = a0 + lane; a < a1; a += 32) atomicAdd(&wb[warp * E + idx[a]], 1);
  __syncthreads();
  // warp bases: offsets[e] + chunk base + counts of earlier warps in this chunk
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int run = offsets[e] + chunk_base[size_t(blockIdx.x) * E + e];
    for (int w = 0; w < kScatterWarps; ++w) {
      const int c = wb[w * E + e];
      wb[w * E + e] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = a0; base < a1; base += 32) {
    const int64_t a = base + lane;
    const bool live = a < a1;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    if (live) {
      const int e = idx[a];
      const unsigned peers = __match_any_sync(act, e);
      const int pos = wb[warp * E + e] + __popc(peers & lt);
      perm[pos] = int32_t(a);
      inv[a] = pos;
      __syncwarp(act);
      if ((peers & lt) == 0) wb[warp * E + e] += __popc(peers);  // group leader advances
    }
    __syncwarp();
  }
}

// Small problems (<= kSmallAssign assignments, <= kSmallExperts experts):
// the same stable counting sort in ONE CTA of 32 warps — per-warp histograms
// of contiguous sub-ranges, one scan, then the match_any scatter — so the
// dispatch is one launch instead of three.
constexpr int kSmallWarps = 32;
constexpr int64_t kSmallAssign = 32768;
constexpr int kSmallExperts = 128;

__global__ void __launch_bounds__(kSmallWarps * 32)
    dispatch_small_kernel(const int32_t* __restrict__ idx, int64_t n, int E,
                          int32_t* __restrict__ offsets, int32_t* __restrict__ perm,
                          int32_t* __restrict__ inv) {
  __shared__ int wb[kSmallWarps * kSmallExperts];  // per-warp counts, then bases
  __shared__ int tot[kSmallExperts + 1];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t per = (n + kSmallWarps - 1) / kSmallWarps;
  const int64_t a0 = min(n, int64_t(warp) * per), a1 = min(n, a0 + per);
  for (int i = threadIdx.x; i < kSmallWarps * E; i += blockDim.x) wb[i] = 0;
  __syncthreads();
  for (int64_t a = a0 + lane; a < a1; a += 32) atomicAdd(&wb[warp * E + idx[a]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {  // running sum over warps
    int run = 0;
    for (int w = 0; w < kSmallWarps; ++w) {
      const int c = wb[w * E + e];
      wb[w * E + e] = run;
      run += c;
    }
    tot[e] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive scan over experts
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      const int c = tot[e];
      tot[e] = acc;
      offsets[e] = acc;
      acc += c;
    }
    offsets[E] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSmallWarps * E; i += blockDim.x) wb[i] += tot[i % E];
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = a0; base < a1; base += 32) {
    const int64_t a = base + lane;
    const bool live = a < a1;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    if (live) {
      const int e = idx[a];
      const unsigned peers = __match_any_sync(act, e);
      const int pos = wb[warp * E + e] + __popc(peers & lt);
      perm[pos] = int32_t(a);
      inv[a] = pos;
      __syncwarp(act);
      if ((peers & lt) == 0) wb[warp * E + e] += __popc(peers);  // group leader advances
    }
    __syncwarp();
  }
}

__global__ void gather_rows_kernel(const uint4* __restrict__ x, int64_t rows_out, int vec_per_row,
                                   int k, const int32_t* __restrict__ perm,
                                   uint4* __restrict__ xp) {
  const int warps = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int64_t p = int64_t(blockIdx.x) * warps + warp; p < rows_out;
       p += int64_t(gridDim.x) * warps) {
    const int64_t src = perm[p] / k;
    const uint4* s = x + src * vec_per_row;
    uint4* d = xp + p * vec_per_row;
    // 4 independent 16-byte loads in flight per lane before the stores (the
    // row copy is latency-bound at 1 load per lane: ~32 KB in flight per SM)
    int v = lane;
    for (; v + 96 < vec_per_row; v += 128) {
      uint4 r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = __ldg(s + v + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) d[v + 32 * u] = r[u];
    }
    for (; v < vec_per_row; v += 32) d[v] = __ldg(s + v);
  }
}

// token-major form of the same gather: warp per token, the row is read ONCE and
// written to its k positions x_perm[inv[t*k+j]] (the perm-driven form reads a
// token row k times, which misses L2 when x is larger than L2)
__global__ void gather_rows_by_token_kernel(const uint4* __restrict__ x, int64_t N,
                                            int vec_per_row, int k,
                                            const int32_t* __restrict__ inv,
                                            uint4* __restrict__ xp) {
  const int warps = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int64_t t = int64_t(blockIdx.x) * warps + warp; t < N; t += int64_t(gridDim.x) * warps) {
    int32_t dst[8];
    for (int j = 0; j < k; ++j) dst[j] = inv[t * k + j];
    const uint4* s = x + t * vec_per_row;
    int v = lane;
    for (; v + 96 < vec_per_row; v += 128) {
      uint4 r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = __ldg(s + v + 32 * u);
      for (int j = 0; j < k; ++j) {
        uint4* d = xp + int64_t(dst[j]) * vec_per_row;
#pragma unroll
        for (int u = 0; u < 4; ++u) d[v + 32 * u] = r[u];
      }
    }
    for (; v < vec_per_row; v += 32) {
      const uint4 r = __ldg(s + v);
      for (int j = 0; j < k; ++j) xp[int64_t(dst[j]) * vec_per_row + v] = r;
    }
  }
}

__global__ void scatter_rows_kernel(const uint4* __restrict__ src, int64_t rows, int vec_per_row,
                                    const int32_t* __restrict__ index, uint4* __restrict__ dst) {
  const int warps = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int64_t p = int64_t(blockIdx.x) * warps + warp; p < rows;
       p += int64_t(gridDim.x) * warps) {
    const uint4* s = src + p * vec_per_row;
    uint4* d = dst + int64_t(index[p]) * vec_per_row;
    for (int v = lane; v < vec_per_row; v += 32) d[v] = __ldg(s + v);
  }
}

template <typename T>
__global__ void combine_kernel(const T* __restrict__ yp, const int32_t* __restrict__ inv,
                               const float* __restrict__ w, int64_t N, int k, int d,
                               T* __restrict__ y) {
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte vector
  const int warps = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nvec = d / V;
  for (int64_t t = int64_t(blockIdx.x) * warps + warp; t < N; t += int64_t(gridDim.x) * warps) {
    int32_t rows[8];
    float ws[8];
    for (int j = 0; j < k; ++j) {
      rows[j] = inv[t * k + j];
      ws[j] = w[t * k + j];
    }
    // U vectors per lane per step: the k*U row loads of a step are issued
    // before any arithmetic (same fmaf chain per element, slot order 0..k-1)
    constexpr int U = 4;
    for (int v0 = lane; v0 < nvec; v0 += 32 * U) {
      float acc[U][V];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[u][i] = 0.0f;
      for (int j = 0; j < k; ++j) {
        const uint4* src = reinterpret_cast<const uint4*>(yp + size_t(rows[j]) * d);
        uint4 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (v0 + 32 * u < nvec) raw[u] = __ldg(src + v0 + 32 * u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const T* e = reinterpret_cast<const T*>(&raw[u]);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[u][i] = fmaf(ws[j], load_as_f32(e, i), acc[u][i]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v0 + 32 * u >= nvec) break;
        uint4 out;
        T* o = reinterpret_cast<T*>(&out);
#pragma unroll
        for (int i = 0; i < V; ++i) {
          if constexpr (sizeof(T) == 2) o[i] = __float2bfloat16_rn(acc[u][i]);
          else o[i] = acc[u][i];
        }
        reinterpret_cast<uint4*>(y + size_t(t) * d)[v0 + 32 * u] = out;
      }
    }
  }
}

int grid_for_rows(int64_t rows, int warps_per_block) {
  const int64_t want = (rows + warps_per_block - 1) / warps_per_block;
  return int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(device_sm_count()) * 8)));
}

}  // namespace

__global__ void counts_from_offsets_kernel(const int32_t* __restrict__ offsets, int E,
                                           int32_t* __restrict__ counts) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
    counts[e] = offsets[e + 1] - offsets[e];
}

void launch_counts_from_offsets(const int32_t* offsets, int E, int32_t* counts, cudaStream_t s) {
  counts_from_offsets_kernel<<<(E + 255) / 256, 256, 0, s>>>(offsets, E, counts);
  INFMOE_LAUNCH_CHECK();
}

size_t dispatch_workspace_bytes(int64_t n_assign, int E) {
  const int64_t chunks = std::max<int64_t>(1, (n_assign + kChunkAssign - 1) / kChunkAssign);
  return size_t(chunks) * size_t(E) * sizeof(int32_t);
}

void launch_dispatch(const int32_t* idx, int64_t n, int E, int32_t* offsets, int32_t* perm,
                     int32_t* inv, void* workspace, cudaStream_t s) {
  require(E >= 1 && E <= kMaxExpertsDispatch, "dispatch: n_experts must be in [1, 1024]");
  require(workspace != nullptr, "dispatch: workspace is NULL");
  if (n <= kSmallAssign && E <= kSmallExperts) {
    dispatch_small_kernel<<<1, kSmallWarps * 32, 0, s>>>(idx, n, E, offsets, perm, inv);
    INFMOE_LAUNCH_CHECK();
    return;
  }
  const int64_t chunks = std::max<int64_t>(1, (n + kChunkAssign - 1) / kChunkAssign);
  int32_t* ch = reinterpret_cast<int32_t*>(workspace);
  chunk_histogram_kernel<<<unsigned(chunks), 256, E * sizeof(int), s>>>(idx, n, E, ch);
  INFMOE_LAUNCH_CHECK();
  dispatch_scan_kernel<<<1, 256, E * sizeof(int), s>>>(ch, int(chunks), E, offsets);
  INFMOE_LAUNCH_CHECK();
  if (n == 0) return;
  dispatch_scatter_kernel<<<unsigned(chunks), kScatterWarps * 32,
                            kScatterWarps * E * sizeof(int), s>>>(idx, n, E, ch, offsets, perm,
                                                                  inv);
  INFMOE_LAUNCH_CHECK();
}

void launch_gather_rows(const void* x, int dtype, int64_t N, int d, int k, const int32_t* perm,
                        void* x_perm, cudaStream_t s) {
  const size_t row_bytes = size_t(d) * dtype_bytes(dtype);
  require(row_bytes % 16 == 0, "gather: row bytes must be a multiple of 16");
  const int64_t rows = N * k;
  if (rows == 0) return;
  gather_rows_kernel<<<grid_for_rows(rows, 8), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(x), rows, int(row_bytes / 16), k, perm,
      reinterpret_cast<uint4*>(x_perm));
  INFMOE_LAUNCH_CHECK();
}

void launch_gather_rows_by_token(const void* x, int dtype, int64_t N, int d, int k,
                                 const int32_t* inv, void* x_perm, cudaStream_t s) {
  const size_t row_bytes = size_t(d) * dtype_bytes(dtype);
  require(row_bytes % 16 == 0, "gather: row bytes must be a multiple of 16");
  require(k >= 1 && k <= 8, "gather: top_k must be in [1, 8]");
  if (N == 0) return;
  gather_rows_by_token_kernel<<<grid_for_rows(N, 8), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(x), N, int(row_bytes / 16), k, inv,
      reinterpret_cast<uint4*>(x_perm));
  INFMOE_LAUNCH_CHECK();
}

void launch_scatter_rows(const void* src, int dtype, int64_t rows, int d, const int32_t* index,
                         void* dst, cudaStream_t s) {
  const size_t row_bytes = size_t(d) * dtype_bytes(dtype);
  require(row_bytes % 16 == 0, "scatter: row bytes must be a multiple of 16");
  if (rows == 0) return;
  scatter_rows_kernel<<<grid_for_rows(rows, 8), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(src), rows, int(row_bytes / 16), index,
      reinterpret_cast<uint4*>(dst));
  INFMOE_LAUNCH_CHECK();
}

void launch_combine(const void* yp, int dtype, const int32_t* inv, const float* w, int64_t N,
                    int k, int d, void* y, cudaStream_t s) {
  require(k >= 1 && k <= 8, "combine: top_k must be in [1, 8]");
  require((size_t(d) * dtype_bytes(dtype)) % 16 == 0, "combine: row bytes must be a multiple of 16");
  if (N == 0) return;
  if (dtype == kDtypeBf16)
    combine_kernel<<<grid_for_rows(N, 8), 256, 0, s>>>(
        reinterpret_cast<const __nv_bfloat16*>(yp), inv, w, N, k, d,
        reinterpret_cast<__nv_bfloat16*>(y));
  else
    combine_kernel<<<grid_for_rows(N, 8), 256, 0, s>>>(reinterpret_cast<const float*>(yp), inv,
                                                        w, N, k, d, reinterpret_cast<float*>(y));
  INFMOE_LAUNCH_CHECK();
}

}  // namespace infmoe
