// ep_plan.hpp — expert-parallel exchange plan (see ep_plan.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace infmoe {

struct EpPlan {
  int P = 1, El = 0;
  std::vector<int64_t> send_off, send_rows;  // [P] rows of x_perm per destination
  std::vector<int64_t> recv_off, recv_rows;  // [P] receive-buffer segment per source
  int64_t n_recv = 0;
  std::vector<int32_t> local_offsets;        // [El+1] expert-contiguous layout
  std::vector<int32_t> local_index;          // [n_recv] local row <- receive row
};

EpPlan make_ep_plan(int P, int rank, int E, const int32_t* send_counts,
                    const int32_t* recv_counts);

}  // namespace infmoe
