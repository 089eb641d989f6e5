// ep_plan.cpp — expert-parallel exchange plan (no reference
// counterpart: multi-GPU placement is a SPEC non-goal).
//
// Experts are split into P contiguous blocks of E/P, so a rank's dispatch
// order (sorted by global expert) is already grouped by destination rank.
// After the count exchange each rank knows
//   send_counts[E]        rows it routes to every global expert, and
//   recv_counts[P][E/P]   rows every source routes to each of its local experts.
// The plan says which x_perm rows go to which peer, where each source's rows
// land in the receive buffer (source-major), and the permutation that makes
// the received rows expert-contiguous (expert-major, then source, then the
// source's token order) for the grouped GEMM.  With tokens sharded
// contiguously across ranks that is exactly the single-GPU row order of every
// expert, so EP outputs are bit-identical to the one-GPU layer.
#include "ep_plan.hpp"

#include "status.hpp"

namespace infmoe {

EpPlan make_ep_plan(int P, int rank, int E, const int32_t* send_counts,
                    const int32_t* recv_counts) {
  require(P >= 1 && rank >= 0 && rank < P, "ep_plan: bad rank / world size");
  require(E >= P && E % P == 0, "ep_plan: n_experts must be a multiple of the EP world size");
  require(send_counts && recv_counts, "ep_plan: NULL counts");
  const int El = E / P;
  EpPlan p;
  p.P = P;
  p.El = El;
  p.send_off.assign(size_t(P), 0);
  p.send_rows.assign(size_t(P), 0);
  p.recv_off.assign(size_t(P), 0);
  p.recv_rows.assign(size_t(P), 0);
  int64_t off = 0;
  for (int r = 0; r < P; ++r) {
    int64_t rows = 0;
    for (int e = r * El; e < (r + 1) * El; ++e) {
      require(send_counts[e] >= 0, "ep_plan: negative count");
      rows += send_counts[e];
    }
    p.send_off[size_t(r)] = off;
    p.send_rows[size_t(r)] = rows;
    off += rows;
  }
  off = 0;
  for (int s = 0; s < P; ++s) {
    int64_t rows = 0;
    for (int e = 0; e < El; ++e) {
      require(recv_counts[s * El + e] >= 0, "ep_plan: negative count");
      rows += recv_counts[s * El + e];
    }
    p.recv_off[size_t(s)] = off;
    p.recv_rows[size_t(s)] = rows;
    off += rows;
  }
  p.n_recv = off;
  // expert-contiguous local layout
  p.local_offsets.assign(size_t(El) + 1, 0);
  for (int e = 0; e < El; ++e) {
    int64_t n = 0;
    for (int s = 0; s < P; ++s) n += recv_counts[s * El + e];
    p.local_offsets[size_t(e) + 1] = p.local_offsets[size_t(e)] + int32_t(n);
  }
  p.local_index.assign(size_t(p.n_recv), 0);
  std::vector<int64_t> cursor(static_cast<size_t>(El));
  for (int e = 0; e < El; ++e) cursor[size_t(e)] = p.local_offsets[size_t(e)];
  for (int s = 0; s < P; ++s) {
    int64_t src_row = p.recv_off[size_t(s)];
    for (int e = 0; e < El; ++e)
      for (int i = 0; i < recv_counts[s * El + e]; ++i)
        p.local_index[size_t(cursor[size_t(e)]++)] = int32_t(src_row++);
  }
  return p;
}

}  // namespace infmoe
