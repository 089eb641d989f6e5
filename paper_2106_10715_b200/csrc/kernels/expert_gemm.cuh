// expert_gemm.cuh — host interface of the tcgen05 grouped expert GEMM.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace infmoe {

constexpr int kMaxGroups = 128;

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

}  // namespace infmoe
