// layer.hpp — state owned by one infmoe_layer handle (device buffers sized for
// max_tokens, K+1 weight slots, copy stream, per-position events, and the
// expert-parallel exchange buffers).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../host/ep_plan.hpp"
#include "../kernels/codec.cuh"
#include "infmoe.h"

namespace infmoe {

// K+1 shared expert slots (infmoe_slot_pool)
struct SlotPool {
  int device = 0, K = 0, n_slots = 0;  // n_slots = sets * (K + 1)
  int sets = 1;
  size_t matrix_bytes = 0;
  uint8_t* slot_in = nullptr;
  uint8_t* slot_out = nullptr;
  // exp4 codec: one staging buffer per slot for the packed bytes (grown on demand)
  uint8_t* stage = nullptr;
  size_t stage_bytes = 0;
};

// exp4 packs of one host weight set (w_in, w_out of n experts), pinned, shared
// by every layer that points at the same host weights (HostPack::acquire)
struct HostPack {
  uint8_t* host = nullptr;          // pinned
  std::vector<uint64_t> off, size;  // per expert: [w_in pack | w_out pack], 16-aligned
  std::vector<uint64_t> in_size;    // bytes of the w_in pack (w_out pack follows)
  std::vector<codec::ExphLayout> lay_in, lay_out;  // exph: per-matrix layouts
  int codec_id = 0;
  uint64_t max_size = 0, total = 0, raw_bytes = 0;
  uint64_t digest = 0;              // content digest of the host weights packed
  int source = 1;                   // 1 encoded in this process, 2 read from the pack cache
  // the pack of (w_in, w_out): a live cached pack of the same buffers and the
  // same content digest is shared, unless `fresh` (always re-pack)
  // packs are also kept on disk when a pack cache directory is set
  // (infmoe_set_pack_cache_dir / INFMOE_PACK_CACHE_DIR): one file per content
  // digest, read back instead of re-encoding, verified by its own checksum
  static void set_cache_dir(const char* dir);
  static std::shared_ptr<HostPack> acquire(const void* w_in, const void* w_out, int n_experts,
                                           uint64_t matrix_elems, int codec_id, bool fresh);
  ~HostPack();
};

struct Layer {
  explicit Layer(const infmoe_layer_desc& d);
  ~Layer();
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;

  // given_idx / given_w (device [N*k], optional): the caller's routing instead
  // of the layer's gate (infmoe_layer_forward_routed)
  void forward(const void* x, int64_t N, void* y, infmoe_forward_out* out, cudaStream_t s,
               const int32_t* given_idx = nullptr, const float* given_w = nullptr);
  // fresh_pack: re-pack the host weights for the h2d codec even if a pack of
  // the same buffers is cached (explicit infmoe_layer_set_host_weights calls)
  void set_host_weights(const void* w_in, const void* w_out, bool fresh_pack = true);
  // SURVEY 8(f)-4 hot-expert pinning (not in the reference): keep these local
  // experts on the device across forwards; n = 0 unpins
  void pin_experts(const int32_t* experts, int n);
  // cache policy: pin the n experts with the highest running load estimate
  // (EMA of routed rows over offloaded forwards, decay 0.5; ties: lower index)
  std::vector<int32_t> pin_hottest(int n);
  int n_pinned_experts() const { return n_pinned; }
  // continuous_load_stream: the layer forwarded after this one
  void set_next(Layer* nxt);
  int pack_source() const { return pack ? pack->source : 0; }
  void h2d_bytes(uint64_t* packed, uint64_t* raw) const {
    const uint64_t r = uint64_t(n_local) * 2 * expert_in_bytes;
    if (raw) *raw = r;
    if (packed) *packed = pack ? pack->total : r;
  }

 private:
  // the rows one expert-compute pass works on
  struct Rows {
    const void* a;            // [rows, d_model] expert-contiguous token rows
    const int32_t* offsets;   // device [n_local + 1]
    int64_t rows;
    void* h;                  // [rows, d_ff]
    void* y;                  // [rows, d_model]
    const int32_t* counts;    // host [n_local] rows per local expert (may be NULL: resident)
  };
  void route(const void* x, int64_t N, cudaStream_t s, const int32_t* given_idx,
             const float* given_w);
  void compute_resident(const Rows& r, bool timed, cudaStream_t s);  // grouped GEMM pair
  void compute_offloaded(const Rows& r, bool timed, infmoe_forward_out* out, cudaStream_t s);
  void ffn(const Rows& r, const int32_t* experts, const int32_t* slots, int n, const void* w_in,
           const void* w_out, int n_w_slots, int max_ctas, int rows_hint, cudaStream_t s,
           cudaEvent_t ev_begin = nullptr, cudaEvent_t ev_end = nullptr);
  void ep_exchange_out(int64_t N, cudaStream_t s);   // dispatch all-to-allv
  void ep_exchange_back(cudaStream_t s);             // combine all-to-allv
  void peer_setup();                                 // PEER transport: map the peers
  void peer_barrier(cudaStream_t s);                 // stream-ordered, all ranks
  template <class T>
  T* grow(T*& p, size_t& cap, size_t n);

  infmoe_layer_desc desc;
  size_t esz = 2;
  int n_local = 0;  // experts held by this rank (E / ep_size)
  int n_scheduled = 0;  // experts loaded by the last offloaded forward
  std::vector<int32_t> exec_order;  // ... and their load order (local expert ids)
  std::vector<void*> owned;
  std::vector<void*> registered;
  // routing / dispatch buffers
  int32_t* idx = nullptr;
  float* wts = nullptr;
  int32_t* counts = nullptr;
  int32_t* offsets = nullptr;
  int32_t* perm = nullptr;
  int32_t* inv = nullptr;
  uint8_t* dws = nullptr;
  uint8_t* gws = nullptr;  // softmax gate workspace (tensor-core path), gws_bytes
  size_t gws_bytes = 0;
  uint8_t* xp = nullptr;
  uint8_t* hbuf = nullptr;
  uint8_t* yp = nullptr;
  double* proj = nullptr;
  float* gate_w = nullptr;
  float* gate_b = nullptr;
  int32_t* counts_host = nullptr;  // pinned [E + ep_size * n_local]
  int32_t* done_ctr = nullptr;     // fused FFN per-group completion counters
  void* fused_out = nullptr;       // y when the combine is fused into the GEMM2 epilogue
  // offload executor
  size_t expert_in_bytes = 0;  // = bytes of W_in = bytes of W_out of one expert
  int n_slots = 0;   // slots in the weight tensors (all sets of the pool)
  int n_rot = 0;     // slots this layer rotates through (K+1, or fewer experts + 1)
  int slot_base = 0; // first slot of this layer's set
  int slot_of(int j) const { return slot_base + j % n_rot; }
  // continuous_load_stream: prefetched leading positions of the next forward
  struct Prefetched {
    int expert;
  };
  Layer* next = nullptr;
  std::vector<Layer*> prevs;  // layers whose `next` is this one (unlinked on destroy)
  bool set_assigned = false;
  std::vector<Prefetched> pf;
  int pf_reused = 0;
  cudaEvent_t last_load = nullptr;
  cudaEvent_t in_half = nullptr;  // the last expert's W_in pack has landed
  void prefetch(cudaEvent_t after_loads, cudaEvent_t after_computes);
  std::vector<int> predicted_order(std::vector<int>* members) const;
  uint8_t* slot_in = nullptr;
  uint8_t* slot_out = nullptr;
  const uint8_t* host_in = nullptr;
  const uint8_t* host_out = nullptr;
  std::shared_ptr<HostPack> pack;   // exp4 codec: packed host weights
  SlotPool own_pool;                // staging when the layer owns its slots
  SlotPool* pool_ptr = nullptr;     // where the staging buffers live
  uint8_t* stage_of(int slot) const { return pool_ptr->stage + size_t(slot) * pool_ptr->stage_bytes; }
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> load_done, compute_done;
  std::vector<cudaEvent_t> t_load0, t_load1, t_comp0, t_comp1;
  cudaEvent_t t_start = nullptr;
  // pinned experts (pin_experts): pin_slot[e] = slot in pin_in/pin_out or -1
  std::vector<int32_t> pin_slot;
  std::vector<int32_t> pin_list;  // pinned experts, slot order
  int n_pinned = 0;
  int n_pinned_run = 0;               // pinned experts computed by the last forward
  std::vector<int32_t> pinned_run;
  std::vector<double> load_ema;  // per local expert (pin_hottest)
  bool ema_seen = false;
  uint8_t* pin_in = nullptr;
  uint8_t* pin_out = nullptr;
  cudaEvent_t t_pin0 = nullptr, t_pin1 = nullptr;
  void copy_pinned();
  // expert parallelism
  void* comm = nullptr;
  bool use_ep = false;
  EpPlan plan;
  int32_t* recv_counts_dev = nullptr;  // [ep_size * n_local]
  int32_t* plan_dev = nullptr;         // [n_local + 1 | n_recv] offsets + index
  int32_t* plan_host = nullptr;        // pinned staging for plan_dev
  size_t plan_cap = 0, plan_host_cap = 0;
  uint8_t* recv_x = nullptr;   // receive buffer, source-major
  uint8_t* loc_x = nullptr;    // expert-contiguous rows
  uint8_t* loc_h = nullptr;
  uint8_t* loc_y = nullptr;
  uint8_t* recv_y = nullptr;   // results in receive layout (sent back)
  size_t cap_x = 0, cap_lx = 0, cap_h = 0, cap_ly = 0, cap_ry = 0;
  // PEER transport (ep_peer.cu): symmetric buffers peers write into
  bool ep_peer = false;
  int64_t cap_recv = 0;           // rows this rank can receive (P * max_tokens * k)
  uint8_t* sym_x = nullptr;       // [cap_recv, d] received rows, expert-contiguous
  int2* sym_ret = nullptr;        // [cap_recv] (source rank, source row)
  uint8_t* sym_y = nullptr;       // [max_tokens*k, d] results for my rows
  int32_t* sym_counts = nullptr;  // [P, E] every source's histogram
  int32_t* dest_base = nullptr;   // [E]
  int32_t* loc_offsets = nullptr; // [n_local + 1]
  int32_t* bar_buf = nullptr;     // 1-int all-reduce of the barrier (ranks in one process)
  uint32_t* sym_flags = nullptr;  // [P] barrier epochs written by the peers
  uint32_t** d_peer_flags = nullptr;
  uint32_t bar_epoch = 0;
  bool dev_barrier = false;       // device flag barrier (peers in other processes)
  void** d_peer_x = nullptr;      // device arrays of the peers' buffers
  int2** d_peer_ret = nullptr;
  int32_t** d_peer_counts = nullptr;
  std::vector<void*> peer_y;      // host copy (FFN kernel parameter)
  std::vector<void*> ipc_opened;  // peer mappings to close
};

}  // namespace infmoe
