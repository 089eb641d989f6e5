// expert_gemm.cuh — host interface of the tcgen05 grouped expert GEMM.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace infmoe {

constexpr int kMaxGroups = 128;
constexpr int kMaxPeers = 16;  // expert-parallel ranks reachable over peer memory

// One launch computes out[rows of group g, :] = epi(A[rows] . B[slot_g]^T) for
// every listed group.  A is [a_rows, K] row-major (token rows, K contiguous);
// B is [n_slots * N, K] (the weight of slot s occupies rows s*N .. s*N+N-1);
// out is [a_rows, N] row-major.  Rows of group g are
// [offsets[expert_g], offsets[expert_g + 1]).  epi: GeLU (gelu=1) or identity.
struct GroupedGemmArgs {
  const void* a;
  int64_t a_rows;
  const void* b;
  int32_t n_slots;
  int32_t N, K;
  int32_t dtype;  // 0 bf16 (kind::f16), 1 f32 (kind::tf32)
  const int32_t* offsets;  // device
  int32_t n_groups;
  int32_t experts[kMaxGroups];
  int32_t slots[kMaxGroups];
  void* out;  // bf16 or f32 (same as dtype)
  int32_t gelu;
  int32_t max_ctas;  // 0 = one CTA per SM
  int32_t max_rows_hint;  // largest group row count if known on the host, else 0
};

void launch_grouped_gemm(const GroupedGemmArgs& args, cudaStream_t stream);

// Both projections of the expert FFN in ONE persistent launch:
//   phase 1  h[rows(g)] = GeLU(x[rows(g)] . w_in[slot(g)]^T)     (N = d_ff,   K = d_model)
//   phase 2  y[rows(g)] = h[rows(g)] . w_out[slot(g)]^T           (N = d_model, K = d_ff)
// A phase-2 tile of group g starts as soon as every phase-1 tile of g has
// stored its H rows (per-group completion counters, release/acquire), so the
// wave tail of phase 1 and the launch gap disappear.  With `perm` and `topk_w`
// (top-1 only) the phase-2 epilogue also performs the combine:
//   y_out[perm[r]] = bf16(fmaf(topk_w[perm[r]], bf16(acc_r), 0))   (== N5 combine)
struct FusedFfnArgs {
  const void* x;        // [rows, d_model]
  int64_t rows;
  const void* w_in;     // [n_slots, d_ff, d_model]
  const void* w_out;    // [n_slots, d_model, d_ff]
  int32_t n_slots;
  int32_t d_model, d_ff;
  int32_t dtype;        // bf16 only (kind::f16)
  const int32_t* offsets;
  int32_t n_groups;
  int32_t experts[kMaxGroups];
  int32_t slots[kMaxGroups];
  void* h;              // [rows, d_ff] scratch
  void* y;              // [rows, d_model] (or [N, d_model] when the combine is fused)
  const int32_t* perm;  // fused top-1 combine: row -> token, or NULL
  const float* topk_w;  // weight per token (with perm)
  // expert-parallel return (PEER transport): row r of the output is stored at
  // row ret[r].y of peer_y[ret[r].x] (device pointers, one per rank)
  const int2* ret;
  void* peer_y[kMaxPeers];
  int32_t n_peers;
  int32_t* done;        // >= n_groups + 1 counters in device memory (zeroed by the launcher):
                        // per-group phase-1 completion, then the tile-claim counter
  int32_t max_ctas;
  int32_t max_rows_hint;
  // optional events recorded right around the kernel, after all host-side
  // preparation (tensor-map encoding), so a timed interval holds GPU work only
  cudaEvent_t ev_begin, ev_end;
};
void launch_expert_ffn_fused(const FusedFfnArgs& args, cudaStream_t stream);
bool ffn_pair_mode();

}  // namespace infmoe
