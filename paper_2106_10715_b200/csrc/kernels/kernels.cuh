// kernels.cuh — launchers of the non-GEMM sm_100a kernels (gate, dispatch,
// gather, combine, fill).  All take device pointers and a stream.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace infmoe {

void launch_fill_uniform(void* out, int dtype, uint64_t n, uint64_t seed, float scale,
                         cudaStream_t stream);
// test hooks (fill.cu): SM-occupying spinners and the flag that releases them
void launch_occupy(int n_ctas, size_t smem, const int32_t* release, uint64_t timeout_ns,
                   int32_t* timed_out, cudaStream_t s);
void launch_set_flag(int32_t* flag, cudaStream_t s);

// N1a: logits by a sequential fmaf chain per (token, expert), top-k by strict
// argmax (ties -> lower index), softmax weights.  counts must be zeroed by the
// launcher (it is: the launcher issues the memset).
// For bf16 x and top_k >= 2 (E <= 128, d % 64 == 0) the logits come from
// tcgen05 and only the candidates the error bound cannot exclude are re-run
// through the exact chain (gate.cu, "N1a on tensor cores"): same indices and
// counts.  It needs gate_softmax_ws_bytes() of device workspace (0 = the
// CUDA-core path); a NULL or short ws is allocated stream-ordered.  A caller
// with fixed gate weights runs gate_softmax_prepare(wg) into ws once and
// passes ws_prepared = true (the bf16 split of W_g lives in ws).
// approx_logits [N, E] / tc_stats {certified tokens, fallback tokens, exact
// chains, full-exact tokens} (device, optional) are test hooks; tc_stats is
// set to all-ones on the CUDA-core path.
size_t gate_softmax_ws_bytes(int dtype, int64_t N, int d, int E, int k);
void gate_softmax_prepare(const float* wg, int d, int E, void* ws, cudaStream_t stream);
void launch_gate_softmax(const void* x, int dtype, int64_t N, int d, const float* wg,
                         const float* bias, int E, int k, int32_t* topk_idx, float* topk_w,
                         int32_t* counts, cudaStream_t stream, void* ws = nullptr,
                         size_t ws_bytes = 0, bool ws_prepared = false,
                         float* approx_logits = nullptr,
                         unsigned long long* tc_stats = nullptr);
// N1b: LSH sign-bit code over the fp64 promotion of x (gating.hpp:61-104).
void launch_gate_lsh(const void* x, int dtype, int64_t N, int d, const double* proj, int bits,
                     int E, uint32_t* codes, int32_t* topk_idx, float* topk_w, int32_t* counts,
                     cudaStream_t stream);

// N2: stable counting sort.  workspace bytes from dispatch_workspace_bytes.
size_t dispatch_workspace_bytes(int64_t n_assign, int E);
void launch_dispatch(const int32_t* topk_idx, int64_t n_assign, int E, int32_t* offsets,
                     int32_t* perm, int32_t* inv, void* workspace, cudaStream_t stream);
// counts[e] = offsets[e+1] - offsets[e] (routing given by the caller)
void launch_counts_from_offsets(const int32_t* offsets, int E, int32_t* counts, cudaStream_t s);
void launch_gather_rows(const void* x, int dtype, int64_t N, int d, int k, const int32_t* perm,
                        void* x_perm, cudaStream_t stream);
// x_perm[inv[t*k+j]] = x[t]: the same x_perm, each token row read once
void launch_gather_rows_by_token(const void* x, int dtype, int64_t N, int d, int k,
                                 const int32_t* inv, void* x_perm, cudaStream_t s);
void launch_scatter_rows(const void* src, int dtype, int64_t rows, int d, const int32_t* index,
                         void* dst, cudaStream_t stream);
// N7 expert parallelism over peer memory (ep_peer.cu)
void launch_ep_counts_push(const int32_t* counts, int E, int me, int P, int32_t* const* peer_counts,
                           cudaStream_t s);
void launch_ep_plan(const int32_t* all_counts, int P, int E, int me, int32_t* dest_base,
                    int32_t* local_offsets, cudaStream_t s);
void launch_ep_dispatch_push(const void* x, const int32_t* perm, int k, int dtype, int64_t rows,
                             int d, const int32_t* offsets, int E, int P, const int32_t* dest_base,
                             int me, void* const* peer_x, int2* const* peer_ret, cudaStream_t s);
// cross-rank barrier on epoch flags in symmetric buffers (P <= 32)
void launch_ep_flag_barrier(uint32_t* const* peer_flags, uint32_t* my_flags, int me, int P,
                            uint32_t epoch, uint64_t timeout_ns, cudaStream_t s);
// N5
void launch_combine(const void* y_perm, int dtype, const int32_t* inv, const float* topk_w,
                    int64_t N, int k, int d, void* y, cudaStream_t stream);

}  // namespace infmoe
