// ep_peer.cu — expert-parallel exchange over peer memory (NVLink / NVSwitch):
// the device half of the PEER transport (layer.cu).
//
// Every rank owns symmetric buffers that its peers write into directly:
//   counts[P][E]   the routed-row histogram of every source rank,
//   x_recv[cap][d] dispatched token rows, already in this rank's
//                  expert-contiguous order (expert-major, then source-major,
//                  then the source's own row order = global token order),
//   ret[cap]       (source rank, source x_perm row) of every received row,
//   y_back[A][d]   expert outputs for this rank's own x_perm rows, written by
//                  the owners of the experts (fused into the FFN epilogue).
// The exchange plan is computed on the device from counts[P][E], so a
// resident layer needs no host round trip between its kernels.  Three
// stream-ordered barriers separate "counts pushed" / "rows pushed" / "results
// pushed" across ranks: device-side epoch flags in the symmetric flags[P]
// buffers (ep_flag_barrier_kernel: no collective, no host), or a 1-int NCCL
// all-reduce when the ranks share one process (layer.cu peer_barrier).
#include "common.cuh"
#include "kernels.cuh"

namespace infmoe {
namespace {

// my histogram into row `me` of every rank's counts[P][E]
__global__ void ep_counts_push_kernel(const int32_t* __restrict__ counts, int E, int me, int P,
                                      int32_t* const* __restrict__ peer_counts) {
  for (int i = threadIdx.x; i < P * E; i += blockDim.x) {
    const int r = i / E, e = i % E;
    peer_counts[r][size_t(me) * E + e] = counts[e];
  }
  __threadfence_system();
}

// dest_base[e]: row in the owner's x_recv where my rows of global expert e
// start; local_offsets[El+1]: this rank's expert-contiguous layout
__global__ void ep_plan_kernel(const int32_t* __restrict__ C, int P, int E, int El, int me,
                               int32_t* __restrict__ dest_base,
                               int32_t* __restrict__ local_offsets) {
  extern __shared__ int32_t tot[];  // [E]: rows of expert e over all sources
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t s = 0;
    for (int src = 0; src < P; ++src) s += C[size_t(src) * E + e];
    tot[e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int r = e / El, le = e % El;
    int32_t base = 0;
    for (int q = 0; q < le; ++q) base += tot[r * El + q];  // earlier experts of owner r
    for (int src = 0; src < me; ++src) base += C[size_t(src) * E + e];  // earlier sources
    dest_base[e] = base;
  }
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int q = 0; q < El; ++q) {
      local_offsets[q] = acc;
      acc += tot[me * El + q];
    }
    local_offsets[El] = acc;
  }
}

// one warp per x_perm row p: find its expert, push token row x[perm[p] / k]
// (16-byte stores over NVLink; no x_perm is materialised) and its return
// address into the owner's buffers
__global__ void ep_dispatch_push_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ perm,
                                        int k, int64_t rows, int vec_per_row,
                                        const int32_t* __restrict__ offsets, int E, int El,
                                        const int32_t* __restrict__ dest_base, int me,
                                        uint4* const* __restrict__ peer_x,
                                        int2* const* __restrict__ peer_ret) {
  const int warps = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int64_t p = int64_t(blockIdx.x) * warps + warp; p < rows; p += int64_t(gridDim.x) * warps) {
    int lo = 0, hi = E - 1;  // last expert e with offsets[e] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (offsets[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int e = lo, r = e / El;
    const int64_t dst = int64_t(dest_base[e]) + (p - offsets[e]);
    const uint4* s = x + int64_t(perm[p] / k) * vec_per_row;
    uint4* dptr = peer_x[r] + dst * vec_per_row;
    for (int v = lane; v < vec_per_row; v += 32) dptr[v] = __ldg(s + v);
    if (lane == 0) peer_ret[r][dst] = make_int2(me, int32_t(p));
  }
  __threadfence_system();
}

// Cross-rank barrier on epoch flags: rank `me` stores `epoch` into slot `me`
// of every rank's flags[P] (release, system scope, after a system fence that
// orders this rank's earlier peer stores), then waits until every slot of its
// own flags[] reached `epoch` (acquire).  Epochs only grow (wrap-safe compare).
// A rank that never arrives traps after `timeout_ns` instead of hanging.
__global__ void ep_flag_barrier_kernel(uint32_t* const* __restrict__ peer_flags,
                                       uint32_t* __restrict__ my_flags, int me, int P,
                                       uint32_t epoch, uint64_t timeout_ns) {
  const int t = threadIdx.x;
  __threadfence_system();
  __syncthreads();
  if (t < P) {
    uint32_t* dst = peer_flags[t] + me;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(epoch) : "memory");
    uint64_t t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flags + t) : "memory");
      if (int32_t(v - epoch) >= 0) break;
      __nanosleep(200);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) __trap();  // a peer never arrived
    }
  }
  __syncthreads();
  __threadfence_system();
}

}  // namespace

void launch_ep_flag_barrier(uint32_t* const* peer_flags, uint32_t* my_flags, int me, int P,
                            uint32_t epoch, uint64_t timeout_ns, cudaStream_t s) {
  ep_flag_barrier_kernel<<<1, 32, 0, s>>>(peer_flags, my_flags, me, P, epoch, timeout_ns);
  INFMOE_LAUNCH_CHECK();
}

void launch_ep_counts_push(const int32_t* counts, int E, int me, int P, int32_t* const* peer_counts,
                           cudaStream_t s) {
  ep_counts_push_kernel<<<1, 256, 0, s>>>(counts, E, me, P, peer_counts);
  INFMOE_LAUNCH_CHECK();
}

void launch_ep_plan(const int32_t* all_counts, int P, int E, int me, int32_t* dest_base,
                    int32_t* local_offsets, cudaStream_t s) {
  require(E % P == 0, "ep plan: E must be a multiple of P");
  ep_plan_kernel<<<1, 256, size_t(E) * sizeof(int32_t), s>>>(all_counts, P, E, E / P, me,
                                                             dest_base, local_offsets);
  INFMOE_LAUNCH_CHECK();
}

void launch_ep_dispatch_push(const void* x, const int32_t* perm, int k, int dtype, int64_t rows,
                             int d, const int32_t* offsets, int E, int P, const int32_t* dest_base,
                             int me, void* const* peer_x, int2* const* peer_ret, cudaStream_t s) {
  const size_t row_bytes = size_t(d) * dtype_bytes(dtype);
  require(row_bytes % 16 == 0, "ep dispatch: row bytes must be a multiple of 16");
  if (rows == 0) return;
  const int64_t want = (rows + 7) / 8;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(device_sm_count()) * 8)));
  ep_dispatch_push_kernel<<<grid, 256, 0, s>>>(
      reinterpret_cast<const uint4*>(x), perm, k, rows, int(row_bytes / 16), offsets, E, E / P,
      dest_base, me, reinterpret_cast<uint4* const*>(peer_x), peer_ret);
  INFMOE_LAUNCH_CHECK();
}

}  // namespace infmoe
