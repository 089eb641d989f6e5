// layer.cu — the MoE layer handle: N1 gate -> N2 dispatch -> [N7 EP exchange]
// -> N3/N4 expert FFN (resident grouped GEMM, or the N6 offload executor) ->
// [N7 EP return] -> N5 combine.
//
// Offloaded execution realises the two-lane recurrence of simulator.hpp:87-194
// (and PAPER.md:366, "by using different CUDA streams, parameter-loading and
// computation of different experts can be easily overlapped"):
//   * the order comes from the InfMoE scheduler on the routed counts
//     (cost_model.hpp:43-62 -> scheduler.hpp:243-248), identical to the
//     reference's order for the same counts / geometry / hardware / K;
//   * a copy stream streams expert j's W_in+W_out from pinned host memory into
//     device slot j mod (K+1) with cudaMemcpyAsync, after the expert that last
//     used that slot (position j-K-1) finished computing.  K+1 physical slots
//     are what the simulator's "K completed residents + one copy in flight"
//     semantics needs;
//   * the compute stream runs expert j's grouped-GEMM pair once load j landed.
// The per-layer counts read-back is the one device->host sync of the path.
//
// Expert parallelism: experts are split into ep_size contiguous
// blocks; after routing, a count exchange and a token all-to-allv (grouped
// NCCL send/recv over NVLink) move every routed row to its expert's owner, the
// owner runs its local experts (resident or offloaded), and the reverse
// all-to-allv brings the results home for the combine.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cstring>
#include <map>
#include <memory>
#include <atomic>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include <unistd.h>

#include "../host/planner.hpp"
#include "../kernels/codec.cuh"
#include "../kernels/common.cuh"
#include "../kernels/expert_gemm.cuh"
#include "../kernels/kernels.cuh"
#include "infmoe.h"
#include "layer.hpp"
#include "nccl_shim.hpp"

namespace infmoe {

namespace {
template <class T>
T* dalloc(size_t n, std::vector<void*>& owned) {
  void* p = nullptr;
  if (n == 0) n = 1;
  INFMOE_CUDA(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  return reinterpret_cast<T*>(p);
}
}  // namespace

template <class T>
T* Layer::grow(T*& p, size_t& cap, size_t n) {
  if (n > cap) {
    if (p) INFMOE_CUDA(cudaFree(p));
    p = nullptr;
    cap = std::max<size_t>(n, cap + cap / 2);
    INFMOE_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), cap * sizeof(T)));
  }
  return p;
}

Layer::Layer(const infmoe_layer_desc& d) : desc(d) {
  require(d.d_model > 0 && d.d_ff > 0 && d.n_experts > 0, "layer: dimensions must be > 0");
  require(d.top_k >= 1 && d.top_k <= 8 && d.top_k <= d.n_experts, "layer: bad top_k");
  require(d.dtype == INFMOE_DTYPE_BF16 || d.dtype == INFMOE_DTYPE_F32, "layer: bad dtype");
  require(d.max_tokens >= 1, "layer: max_tokens must be >= 1");
  require(d.w_in && d.w_out, "layer: expert weights are NULL");
  if (d.gate_kind == INFMOE_GATE_LSH) require(d.top_k == 1, "layer: the LSH gate is top-1");
  const int P = std::max(1, d.ep_size);
  require(d.n_experts % P == 0, "layer: n_experts must be a multiple of ep_size");
  require(d.ep_rank >= 0 && d.ep_rank < P, "layer: ep_rank out of range");
  require(P == 1 || d.ep_comm != nullptr, "layer: ep_size > 1 needs ep_comm");
  // (desc.ep_comm with ep_size == 1 runs the exchange path against itself)
  n_local = d.n_experts / P;
  require(n_local <= kMaxGroups, "layer: at most 128 experts per rank");
  desc.ep_size = P;
  comm = d.ep_comm;
  INFMOE_CUDA(cudaSetDevice(d.device));
  esz = dtype_bytes(d.dtype);
  const int64_t A = int64_t(d.max_tokens) * d.top_k;
  idx = dalloc<int32_t>(size_t(A), owned);
  wts = dalloc<float>(size_t(A), owned);
  counts = dalloc<int32_t>(size_t(d.n_experts), owned);
  offsets = dalloc<int32_t>(size_t(d.n_experts) + 1, owned);
  perm = dalloc<int32_t>(size_t(A), owned);
  inv = dalloc<int32_t>(size_t(A), owned);
  dws = dalloc<uint8_t>(dispatch_workspace_bytes(A, d.n_experts), owned);
  if (d.gate_kind != INFMOE_GATE_LSH) {  // the tensor-core softmax gate's workspace (or 0)
    gws_bytes = gate_softmax_ws_bytes(d.dtype, d.max_tokens, d.d_model, d.n_experts, d.top_k);
    if (gws_bytes) gws = dalloc<uint8_t>(gws_bytes, owned);
  }
  done_ctr = dalloc<int32_t>(size_t(d.n_experts) + 1, owned);  // + the tile-claim counter
  xp = dalloc<uint8_t>(size_t(A) * d.d_model * esz, owned);
  yp = dalloc<uint8_t>(size_t(A) * d.d_model * esz, owned);
  // the exchange path runs whenever a communicator is given (ep_size == 1 then
  // exchanges with itself, which exercises the NCCL transport on one GPU)
  use_ep = P > 1 || comm != nullptr;
  ep_peer = use_ep && d.ep_transport == INFMOE_EP_PEER;
  require(d.ep_transport == INFMOE_EP_NCCL || d.ep_transport == INFMOE_EP_PEER,
          "layer: unknown ep_transport");
  require(!ep_peer || (P <= kMaxPeers && d.dtype == INFMOE_DTYPE_BF16),
          "layer: the PEER transport takes bf16 and at most 16 ranks");
  if (!use_ep) hbuf = dalloc<uint8_t>(size_t(A) * d.d_ff * esz, owned);
  else recv_counts_dev = dalloc<int32_t>(size_t(P) * n_local, owned);
  if (ep_peer) {
    cap_recv = int64_t(P) * A;
    sym_x = dalloc<uint8_t>(size_t(cap_recv) * d.d_model * esz, owned);
    sym_ret = dalloc<int2>(size_t(cap_recv), owned);
    sym_y = dalloc<uint8_t>(size_t(A) * d.d_model * esz, owned);
    sym_counts = dalloc<int32_t>(size_t(P) * d.n_experts, owned);
    dest_base = dalloc<int32_t>(size_t(d.n_experts), owned);
    loc_offsets = dalloc<int32_t>(size_t(n_local) + 1, owned);
    bar_buf = dalloc<int32_t>(1, owned);
    sym_flags = reinterpret_cast<uint32_t*>(dalloc<int32_t>(size_t(P), owned));
    INFMOE_CUDA(cudaMemset(sym_flags, 0, sizeof(uint32_t) * size_t(P)));
    cap_h = size_t(cap_recv) * d.d_ff * esz;  // freed with the other exchange buffers
    INFMOE_CUDA(cudaMalloc(&loc_h, cap_h));
    peer_setup();
  }

  if (d.gate_kind == INFMOE_GATE_LSH) {
    std::vector<double> p = lsh_hyperplanes(d.lsh_seed, d.lsh_bits, d.d_model);
    proj = dalloc<double>(p.size(), owned);
    INFMOE_CUDA(cudaMemcpy(proj, p.data(), p.size() * sizeof(double), cudaMemcpyHostToDevice));
  } else {
    require(d.gate_weight != nullptr, "layer: softmax gate needs gate_weight [E, d]");
    const size_t n = size_t(d.n_experts) * d.d_model;
    gate_w = dalloc<float>(n, owned);
    INFMOE_CUDA(cudaMemcpy(gate_w, d.gate_weight, n * sizeof(float), cudaMemcpyHostToDevice));
    if (gws) {  // the tensor-core gate's bf16 split of W_g, once, on a private stream (a
                // device-wide sync could wait behind another EP rank's spinning barrier)
      cudaStream_t ps;
      INFMOE_CUDA(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
      gate_softmax_prepare(gate_w, d.d_model, d.n_experts, gws, ps);
      INFMOE_CUDA(cudaStreamSynchronize(ps));
      INFMOE_CUDA(cudaStreamDestroy(ps));
    }
    if (d.gate_bias) {
      gate_b = dalloc<float>(size_t(d.n_experts), owned);
      INFMOE_CUDA(cudaMemcpy(gate_b, d.gate_bias, sizeof(float) * d.n_experts,
                             cudaMemcpyHostToDevice));
    }
  }
  // [E] counts | [P * n_local] received counts (NCCL) or [n_local + 1] offsets (PEER)
  const int tail = std::max(P * n_local, n_local + 1);
  INFMOE_CUDA(cudaMallocHost(&counts_host, sizeof(int32_t) * size_t(d.n_experts + tail)));

  expert_in_bytes = size_t(d.d_ff) * d.d_model * esz;
  if (d.residency == INFMOE_OFFLOADED) {
    require(d.K >= 1, "layer: offloaded mode needs K >= 1");
    require(d.h2d_codec == INFMOE_CODEC_RAW || d.h2d_codec == INFMOE_CODEC_EXP4 ||
                d.h2d_codec == INFMOE_CODEC_EXPH,
            "layer: unknown h2d_codec");
    require(d.h2d_codec == INFMOE_CODEC_RAW || d.dtype == INFMOE_DTYPE_BF16,
            "layer: the exp4 / exph codecs pack bf16 weights");
    if (d.slot_pool) {  // K+1 slots shared with the other layers of the stack
      auto* pool = reinterpret_cast<SlotPool*>(d.slot_pool);
      pool_ptr = pool;
      require(pool->device == d.device, "layer: slot pool lives on another device");
      require(pool->K == d.K, "layer: slot pool K differs from the layer's K");
      require(pool->matrix_bytes == expert_in_bytes,
              "layer: slot pool expert size differs from the layer's");
      n_slots = pool->n_slots;
      n_rot = pool->K + 1;
      require(!d.continuous_load_stream || pool->sets >= 2,
              "layer: continuous_load_stream on a shared pool needs 2 slot sets "
              "(infmoe_slot_pool_create_ex)");
      slot_in = pool->slot_in;
      slot_out = pool->slot_out;
    } else {
      n_slots = std::min(d.K + 1, n_local + 1);
      n_rot = n_slots;
      slot_in = dalloc<uint8_t>(size_t(n_slots) * expert_in_bytes, owned);
      slot_out = dalloc<uint8_t>(size_t(n_slots) * expert_in_bytes, owned);
      own_pool.device = d.device;
      own_pool.K = d.K;
      own_pool.n_slots = n_slots;
      own_pool.matrix_bytes = expert_in_bytes;
      own_pool.slot_in = slot_in;
      own_pool.slot_out = slot_out;
      pool_ptr = &own_pool;
    }
    require(d.prefetch_depth >= 0, "layer: prefetch_depth must be >= 0");
    INFMOE_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    INFMOE_CUDA(cudaEventCreateWithFlags(&last_load, cudaEventDisableTiming));
    INFMOE_CUDA(cudaEventCreateWithFlags(&in_half, cudaEventDisableTiming));
    const size_t E = size_t(n_local);
    for (auto* v : {&load_done, &compute_done}) {
      v->resize(E);
      for (auto& e : *v) INFMOE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (auto* v : {&t_load0, &t_load1, &t_comp0, &t_comp1}) {
      v->resize(E);
      for (auto& e : *v) INFMOE_CUDA(cudaEventCreate(&e));
    }
    set_host_weights(d.w_in, d.w_out, /*fresh_pack=*/false);
  } else {
    t_comp0.resize(1);
    t_comp1.resize(1);
    INFMOE_CUDA(cudaEventCreate(&t_comp0[0]));
    INFMOE_CUDA(cudaEventCreate(&t_comp1[0]));
  }
  INFMOE_CUDA(cudaEventCreate(&t_start));
  INFMOE_CUDA(cudaEventCreate(&t_pin0));
  INFMOE_CUDA(cudaEventCreate(&t_pin1));
  pin_slot.assign(size_t(n_local), -1);
  load_ema.assign(size_t(n_local), 0.0);
}

void Layer::set_host_weights(const void* w_in, const void* w_out, bool fresh_pack) {
  require(desc.residency == INFMOE_OFFLOADED, "set_host_weights: layer is resident");
  require(w_in && w_out, "set_host_weights: NULL weights");
  const size_t bytes = expert_in_bytes * size_t(n_local);
  for (const void* p : {w_in, w_out}) {
    cudaPointerAttributes at;
    INFMOE_CUDA(cudaPointerGetAttributes(&at, p));
    // a packed-codec layer streams its pinned packs, never the raw weights
    // (they are only read by the host packer and by pin_experts' one-time
    // copies), so pageable raw weights stay pageable: half the pinned memory
    if (at.type == cudaMemoryTypeUnregistered && desc.h2d_codec != INFMOE_CODEC_RAW) continue;
    if (at.type == cudaMemoryTypeUnregistered) {
      INFMOE_CUDA(cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterDefault));
      registered.push_back(const_cast<void*>(p));
    } else {
      require(at.type == cudaMemoryTypeHost,
              "offloaded layer: expert weights must live in host memory");
    }
  }
  host_in = reinterpret_cast<const uint8_t*>(w_in);
  host_out = reinterpret_cast<const uint8_t*>(w_out);
  pf.clear();  // a prefetched slot would hold the old weights
  if (desc.h2d_codec != INFMOE_CODEC_RAW) {
    // packs are SNAPSHOTS of the host weights: an explicit set_host_weights
    // always re-packs (the caller may have refilled the buffer in place); at
    // create a cached pack of the same buffer is shared only if its content
    // digest still matches (HostPack::acquire)
    pack = HostPack::acquire(w_in, w_out, n_local, uint64_t(desc.d_ff) * desc.d_model,
                             desc.h2d_codec, fresh_pack);
    if (pool_ptr->stage_bytes < pack->max_size) {  // grow the shared staging buffers
      INFMOE_CUDA(cudaDeviceSynchronize());
      if (pool_ptr->stage) INFMOE_CUDA(cudaFree(pool_ptr->stage));
      pool_ptr->stage = nullptr;
      pool_ptr->stage_bytes = 0;
      INFMOE_CUDA(cudaMalloc(&pool_ptr->stage, size_t(pool_ptr->n_slots) * pack->max_size));
      pool_ptr->stage_bytes = pack->max_size;
    }
  }
  if (n_pinned) copy_pinned();  // pinned copies follow the new host weights
}

void Layer::copy_pinned() {
  INFMOE_CUDA(cudaStreamSynchronize(copy_stream));
  for (int i = 0; i < n_pinned; ++i) {
    const size_t e = size_t(pin_list[size_t(i)]);
    INFMOE_CUDA(cudaMemcpyAsync(pin_in + size_t(i) * expert_in_bytes,
                                host_in + e * expert_in_bytes, expert_in_bytes,
                                cudaMemcpyHostToDevice, copy_stream));
    INFMOE_CUDA(cudaMemcpyAsync(pin_out + size_t(i) * expert_in_bytes,
                                host_out + e * expert_in_bytes, expert_in_bytes,
                                cudaMemcpyHostToDevice, copy_stream));
  }
  INFMOE_CUDA(cudaStreamSynchronize(copy_stream));
}

void Layer::pin_experts(const int32_t* experts, int n) {
  require(desc.residency == INFMOE_OFFLOADED, "pin_experts: layer is resident");
  require(n >= 0 && n <= n_local, "pin_experts: n must be in [0, local experts]");
  require(n == 0 || experts, "pin_experts: NULL experts");
  std::vector<int32_t> slot(size_t(n_local), -1), list;
  for (int i = 0; i < n; ++i) {
    const int e = experts[i];
    require(e >= 0 && e < n_local, "pin_experts: expert out of range");
    require(slot[size_t(e)] < 0, "pin_experts: expert listed twice");
    slot[size_t(e)] = i;
    list.push_back(e);
  }
  INFMOE_CUDA(cudaSetDevice(desc.device));
  INFMOE_CUDA(cudaDeviceSynchronize());  // no forward may still read the old copies
  uint8_t *nin = nullptr, *nout = nullptr;
  if (n > 0) {
    const size_t bytes = size_t(n) * expert_in_bytes;
    if (cudaMalloc(&nin, bytes) != cudaSuccess || cudaMalloc(&nout, bytes) != cudaSuccess) {
      cudaGetLastError();
      if (nin) cudaFree(nin);
      fail(kCapacity, "pin_experts: not enough device memory for " + std::to_string(n) +
                          " pinned experts");
    }
    // experts that stay pinned are copied on the device; the others come over the link
    for (int i = 0; i < n; ++i) {
      const size_t e = size_t(list[size_t(i)]);
      const int old = pin_slot.empty() ? -1 : pin_slot[e];
      const size_t dst = size_t(i) * expert_in_bytes;
      if (old >= 0) {
        const size_t src = size_t(old) * expert_in_bytes;
        INFMOE_CUDA(cudaMemcpyAsync(nin + dst, pin_in + src, expert_in_bytes,
                                    cudaMemcpyDeviceToDevice, copy_stream));
        INFMOE_CUDA(cudaMemcpyAsync(nout + dst, pin_out + src, expert_in_bytes,
                                    cudaMemcpyDeviceToDevice, copy_stream));
      } else {
        INFMOE_CUDA(cudaMemcpyAsync(nin + dst, host_in + e * expert_in_bytes, expert_in_bytes,
                                    cudaMemcpyHostToDevice, copy_stream));
        INFMOE_CUDA(cudaMemcpyAsync(nout + dst, host_out + e * expert_in_bytes, expert_in_bytes,
                                    cudaMemcpyHostToDevice, copy_stream));
      }
    }
    INFMOE_CUDA(cudaStreamSynchronize(copy_stream));
  }
  if (pin_in) cudaFree(pin_in);
  if (pin_out) cudaFree(pin_out);
  pin_in = nin;
  pin_out = nout;
  pin_slot = slot;
  pin_list = list;
  n_pinned = n;
}

std::vector<int32_t> Layer::pin_hottest(int n) {
  require(n >= 0 && n <= n_local, "pin_hottest: n must be in [0, local experts]");
  std::vector<int32_t> idx(static_cast<size_t>(n_local));
  for (int e = 0; e < n_local; ++e) idx[size_t(e)] = e;
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
    return load_ema[size_t(a)] > load_ema[size_t(b)];
  });
  idx.resize(size_t(n));
  std::sort(idx.begin(), idx.end());
  pin_experts(idx.data(), n);
  return idx;
}

Layer::~Layer() {
  // continuous_load_stream links: nobody may prefetch into a destroyed layer
  for (Layer* p : prevs) p->next = nullptr;
  if (next) next->prevs.erase(std::remove(next->prevs.begin(), next->prevs.end(), this),
                              next->prevs.end());
  cudaSetDevice(desc.device);
  for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
  if (copy_stream) cudaStreamSynchronize(copy_stream);
  for (auto* v : {&load_done, &compute_done, &t_load0, &t_load1, &t_comp0, &t_comp1})
    for (cudaEvent_t e : *v) cudaEventDestroy(e);
  if (t_start) cudaEventDestroy(t_start);
  if (last_load) cudaEventDestroy(last_load);
  if (in_half) cudaEventDestroy(in_half);
  if (t_pin0) cudaEventDestroy(t_pin0);
  if (t_pin1) cudaEventDestroy(t_pin1);
  if (pin_in) cudaFree(pin_in);
  if (pin_out) cudaFree(pin_out);
  if (own_pool.stage) cudaFree(own_pool.stage);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  for (void* p : registered) cudaHostUnregister(p);
  if (counts_host) cudaFreeHost(counts_host);
  if (plan_host) cudaFreeHost(plan_host);
  for (void* p : {static_cast<void*>(plan_dev), static_cast<void*>(recv_x),
                  static_cast<void*>(loc_x), static_cast<void*>(loc_h),
                  static_cast<void*>(loc_y), static_cast<void*>(recv_y)})
    if (p) cudaFree(p);
  for (void* p : owned) cudaFree(p);
}

void Layer::route(const void* x, int64_t N, cudaStream_t s, const int32_t* given_idx,
                  const float* given_w) {
  const int E = desc.n_experts, k = desc.top_k;
  if (given_idx) {  // the caller's routing: assignments and weights, no gate
    const size_t A = size_t(N) * size_t(k);
    if (A) {
      INFMOE_CUDA(cudaMemcpyAsync(idx, given_idx, A * 4, cudaMemcpyDeviceToDevice, s));
      INFMOE_CUDA(cudaMemcpyAsync(wts, given_w, A * 4, cudaMemcpyDeviceToDevice, s));
    }
  } else if (desc.gate_kind == INFMOE_GATE_LSH) {
    launch_gate_lsh(x, desc.dtype, N, desc.d_model, proj, desc.lsh_bits, E, nullptr, idx, wts,
                    counts, s);
  } else {
    launch_gate_softmax(x, desc.dtype, N, desc.d_model, gate_w, gate_b, E, k, idx, wts, counts,
                        s, gws, gws_bytes, /*ws_prepared=*/true);
  }
  launch_dispatch(idx, N * k, E, offsets, perm, inv, dws, s);
  if (given_idx) launch_counts_from_offsets(offsets, E, counts, s);
  // the PEER transport pushes token rows straight from x (no x_perm)
  if (!ep_peer) {
    if (k > 1) launch_gather_rows_by_token(x, desc.dtype, N, desc.d_model, k, inv, xp, s);
    else launch_gather_rows(x, desc.dtype, N, desc.d_model, k, perm, xp, s);
  }
}

void Layer::ffn(const Rows& r, const int32_t* experts, const int32_t* slots, int n,
                const void* w_in, const void* w_out, int n_w_slots, int max_ctas, int rows_hint,
                cudaStream_t s, cudaEvent_t ev_begin, cudaEvent_t ev_end) {
  if (desc.dtype == INFMOE_DTYPE_BF16) {  // both projections in one persistent launch
    FusedFfnArgs a;
    std::memset(&a, 0, sizeof(a));
    a.x = r.a;
    a.rows = r.rows;
    a.w_in = w_in;
    a.w_out = w_out;
    a.n_slots = n_w_slots;
    a.d_model = desc.d_model;
    a.d_ff = desc.d_ff;
    a.dtype = desc.dtype;
    a.offsets = r.offsets;
    a.n_groups = n;
    for (int i = 0; i < n; ++i) {
      a.experts[i] = experts[i];
      a.slots[i] = slots[i];
    }
    a.h = r.h;
    a.y = r.y;
    if (ep_peer) {  // results straight back to the token owners over peer memory
      a.ret = sym_ret;
      a.n_peers = desc.ep_size;
      for (int q = 0; q < desc.ep_size; ++q) a.peer_y[q] = peer_y[size_t(q)];
    }
    if (fused_out) {  // top-1, no exchange: the GEMM2 epilogue writes y directly
      a.y = fused_out;
      a.perm = perm;
      a.topk_w = wts;
    }
    a.done = done_ctr;
    a.max_ctas = max_ctas;
    a.max_rows_hint = rows_hint;
    a.ev_begin = ev_begin;
    a.ev_end = ev_end;
    launch_expert_ffn_fused(a, s);
    return;
  }
  if (ev_begin) INFMOE_CUDA(cudaEventRecord(ev_begin, s));
  GroupedGemmArgs g;
  std::memset(&g, 0, sizeof(g));
  g.a = r.a;
  g.a_rows = r.rows;
  g.b = w_in;
  g.n_slots = n_w_slots;
  g.N = desc.d_ff;
  g.K = desc.d_model;
  g.dtype = desc.dtype;
  g.offsets = r.offsets;
  g.n_groups = n;
  for (int i = 0; i < n; ++i) {
    g.experts[i] = experts[i];
    g.slots[i] = slots[i];
  }
  g.out = r.h;
  g.gelu = 1;
  g.max_ctas = max_ctas;
  g.max_rows_hint = rows_hint;
  launch_grouped_gemm(g, s);
  g.a = r.h;
  g.b = w_out;
  g.N = desc.d_model;
  g.K = desc.d_ff;
  g.out = r.y;
  g.gelu = 0;
  launch_grouped_gemm(g, s);
  if (ev_end) INFMOE_CUDA(cudaEventRecord(ev_end, s));
}

// one grouped launch per projection over all local experts; no host round trip
void Layer::compute_resident(const Rows& r, bool timed, cudaStream_t s) {
  std::vector<int32_t> all(static_cast<size_t>(n_local));
  for (int e = 0; e < n_local; ++e) all[size_t(e)] = e;
  // token-tile width: the largest expert when the counts are on the host; else
  // the mean rows per expert when that alone exceeds the default 192-row tile
  // (top-k > 1 / many tokens: tensor-bound, the 256-row tile needs 12% fewer
  // operand bytes per FLOP), else 0 (the default tile for ~128-192 rows)
  int hint = 0;
  if (r.counts) hint = *std::max_element(r.counts, r.counts + n_local);
  else if (r.rows > 192 * int64_t(n_local)) hint = int((r.rows + n_local - 1) / n_local);
  cudaEvent_t e0 = timed ? t_comp0[0] : nullptr, e1 = timed ? t_comp1[0] : nullptr;
  if (r.rows > 0) {
    ffn(r, all.data(), all.data(), n_local, desc.w_in, desc.w_out, n_local, 0, hint, s, e0, e1);
  } else if (timed) {
    INFMOE_CUDA(cudaEventRecord(e0, s));
    INFMOE_CUDA(cudaEventRecord(e1, s));
  }
}

void Layer::compute_offloaded(const Rows& r, bool timed, infmoe_forward_out* out,
                              cudaStream_t s) {
  // experts taking part: all of them (reference default), or only those that
  // received rows when skip_empty_experts is set
  // running load estimate across forwards (pin_hottest's cache policy)
  for (int e = 0; e < n_local; ++e)
    load_ema[size_t(e)] = ema_seen ? 0.5 * load_ema[size_t(e)] + 0.5 * double(r.counts[e])
                                   : double(r.counts[e]);
  ema_seen = true;
  // pinned experts (pin_experts) need no load: they are computed first, in one
  // grouped launch from their device copies, while the first copy is in flight
  std::vector<int> members;
  std::vector<int32_t> pex, psl;
  int pin_rows = 0;
  for (int e = 0; e < n_local; ++e) {
    if (pin_slot[size_t(e)] >= 0) {
      if (r.counts[e] > 0) {
        pex.push_back(e);
        psl.push_back(pin_slot[size_t(e)]);
        pin_rows = std::max(pin_rows, int(r.counts[e]));
      }
    } else if (!desc.skip_empty_experts || r.counts[e] > 0) {
      members.push_back(e);
    }
  }
  n_pinned_run = int(pex.size());
  if (!pex.empty())
    ffn(r, pex.data(), psl.data(), int(pex.size()), pin_in, pin_out, n_pinned, 0, pin_rows, s,
        timed ? t_pin0 : nullptr, timed ? t_pin1 : nullptr);
  pinned_run = pex;
  const int E = int(members.size());
  n_scheduled = E;
  if (E == 0) {
    if (out && out->order)
      for (int j = 0; j < n_local; ++j) out->order[j] = -1;
    if (out && out->feasible) *out->feasible = 1;
    return;
  }
  std::vector<uint64_t> cnt(static_cast<size_t>(E));
  for (int i = 0; i < E; ++i) cnt[size_t(i)] = uint64_t(r.counts[members[size_t(i)]]);
  Geometry geo{1, 1, 1, desc.d_model, desc.d_ff, E, int(esz)};
  Hardware hw{desc.hw.peak_flops, desc.hw.h2d_bandwidth, desc.hw.device_memory,
              desc.hw.reserved_memory};
  Costs c = derive_costs(cnt.data(), E, geo, hw);
  Plan pl;
  switch (desc.policy) {
    case INFMOE_POLICY_NAIVE: pl = plan_identity(c, desc.K); break;
    case INFMOE_POLICY_GREEDY: pl = plan_greedy(c, desc.K); break;
    case INFMOE_POLICY_EXACT: pl = plan_exact(c, desc.K, 12); break;
    default: pl = plan_auto(c, desc.K, 12); break;
  }
  exec_order.resize(size_t(E));
  for (int j = 0; j < E; ++j) exec_order[size_t(j)] = members[size_t(pl.order[size_t(j)])];
  // continuous_load_stream: the leading positions the previous layer already
  // streamed in (prefetch) are reused while their expert matches the real
  // order; the first mismatch and everything after it load as usual (the
  // slot is simply overwritten, in copy-stream order)
  pf_reused = 0;
  while (pf_reused < int(pf.size()) && pf_reused < E &&
         pf[size_t(pf_reused)].expert == exec_order[size_t(pf_reused)])
    ++pf_reused;
  pf.clear();
  // ---- copy lane / compute lane ----
  // drain (simulator.hpp:131-133): this layer's own loads start after the
  // previous layer's computes (in either mode they also need this layer's
  // routing, which the counts read-back above already waited for)
  INFMOE_CUDA(cudaStreamWaitEvent(copy_stream, t_start, 0));
  for (int j = 0; j < E; ++j) {
    const int e = members[size_t(pl.order[size_t(j)])];
    const int slot = slot_of(j);
    const bool split_last = pack && j == E - 1 && j >= pf_reused && r.counts[e] > 0;
    bool w_in_decoded = false;
    if (j < pf_reused) {  // streamed in by the previous layer: no copy
      INFMOE_CUDA(cudaStreamWaitEvent(s, load_done[size_t(j)], 0));
    } else {
    if (j >= n_rot)
      INFMOE_CUDA(cudaStreamWaitEvent(copy_stream, compute_done[size_t(j - n_rot)], 0));
    if (timed) INFMOE_CUDA(cudaEventRecord(t_load0[size_t(j)], copy_stream));
    if (pack && split_last) {
      // the layer's LAST expert: its W_in pack is copied first and decoded
      // while the W_out pack is still on the link, so only one decode stays in
      // the layer's tail (elsewhere one copy per expert: one 108 MB copy ran at
      // 55.00 GB/s, two half copies at 54.82)
      const uint64_t a = pack->in_size[size_t(e)];
      INFMOE_CUDA(cudaMemcpyAsync(stage_of(slot), pack->host + pack->off[size_t(e)], a,
                                  cudaMemcpyHostToDevice, copy_stream));
      INFMOE_CUDA(cudaEventRecord(in_half, copy_stream));
      INFMOE_CUDA(cudaMemcpyAsync(stage_of(slot) + a, pack->host + pack->off[size_t(e)] + a,
                                  pack->size[size_t(e)] - a, cudaMemcpyHostToDevice,
                                  copy_stream));
    } else if (pack) {  // packed codec: one copy of the expert's pack pair into its staging buffer
      INFMOE_CUDA(cudaMemcpyAsync(stage_of(slot), pack->host + pack->off[size_t(e)],
                                  pack->size[size_t(e)], cudaMemcpyHostToDevice, copy_stream));
    } else {
      INFMOE_CUDA(cudaMemcpyAsync(slot_in + size_t(slot) * expert_in_bytes,
                                  host_in + size_t(e) * expert_in_bytes, expert_in_bytes,
                                  cudaMemcpyHostToDevice, copy_stream));
      INFMOE_CUDA(cudaMemcpyAsync(slot_out + size_t(slot) * expert_in_bytes,
                                  host_out + size_t(e) * expert_in_bytes, expert_in_bytes,
                                  cudaMemcpyHostToDevice, copy_stream));
    }
    // the reference's residency gate (simulator.hpp:147-155): load j COMPLETES
    // -- expert j becomes resident -- only once expert j-K has finished
    // computing, so at most K experts are resident at any time; the copy in
    // flight meanwhile occupies the (K+1)-th physical slot.  Like
    // the simulator's single load lane, the next copy starts after this point.
    if (j >= desc.K)
      INFMOE_CUDA(cudaStreamWaitEvent(copy_stream, compute_done[size_t(j - desc.K)], 0));
    if (timed) INFMOE_CUDA(cudaEventRecord(t_load1[size_t(j)], copy_stream));
    INFMOE_CUDA(cudaEventRecord(load_done[size_t(j)], copy_stream));

    if (pack && split_last) {  // W_in decode overlaps the W_out copy (part of the load)
      INFMOE_CUDA(cudaStreamWaitEvent(s, in_half, 0));
      auto* w1 = reinterpret_cast<uint16_t*>(slot_in + size_t(slot) * expert_in_bytes);
      if (pack->codec_id == INFMOE_CODEC_EXPH)
        codec::launch_exph_unpack(stage_of(slot), pack->lay_in[size_t(e)], w1, s);
      else
        codec::launch_exp4_unpack(stage_of(slot), uint64_t(desc.d_ff) * desc.d_model, w1, s);
      w_in_decoded = true;
    }
    INFMOE_CUDA(cudaStreamWaitEvent(s, load_done[size_t(j)], 0));
    }
    const int32_t ex = e, sl = slot;
    const int64_t n_e = int64_t(r.counts[e]);
    cudaEvent_t e0 = timed ? t_comp0[size_t(j)] : nullptr;
    cudaEvent_t e1 = timed ? t_comp1[size_t(j)] : nullptr;
    if (n_e > 0) {
      if (pack) {  // decode both matrices into the slot (counted as compute)
        if (e0) INFMOE_CUDA(cudaEventRecord(e0, s));
        const uint64_t elems = uint64_t(desc.d_ff) * desc.d_model;
        auto* w1 = reinterpret_cast<uint16_t*>(slot_in + size_t(slot) * expert_in_bytes);
        auto* w2 = reinterpret_cast<uint16_t*>(slot_out + size_t(slot) * expert_in_bytes);
        const uint8_t* p1 = stage_of(slot);
        const uint8_t* p2 = p1 + pack->in_size[size_t(e)];
        if (pack->codec_id == INFMOE_CODEC_EXPH) {
          if (!w_in_decoded) codec::launch_exph_unpack(p1, pack->lay_in[size_t(e)], w1, s);
          codec::launch_exph_unpack(p2, pack->lay_out[size_t(e)], w2, s);
        } else {
          if (!w_in_decoded) codec::launch_exp4_unpack(p1, elems, w1, s);
          codec::launch_exp4_unpack(p2, elems, w2, s);
        }
        e0 = nullptr;
      }
      const int tiles = int((n_e + 127) / 128) * (std::max(desc.d_ff, desc.d_model) / 128);
      ffn(r, &ex, &sl, 1, slot_in, slot_out, n_slots, tiles, int(n_e), s, e0, e1);
    } else if (timed) {
      INFMOE_CUDA(cudaEventRecord(e0, s));
      INFMOE_CUDA(cudaEventRecord(e1, s));
    }
    INFMOE_CUDA(cudaEventRecord(compute_done[size_t(j)], s));
  }
  // continuous_load_stream: keep the load lane flowing into the next layer
  if (desc.continuous_load_stream && next) {
    INFMOE_CUDA(cudaEventRecord(last_load, copy_stream));
    next->prefetch(last_load, t_start);
  }
  if (out) {
    if (out->prefetched) *out->prefetched = pf_reused;
    if (out->order) {
      for (int j = 0; j < n_local; ++j) out->order[j] = -1;  // -1: not loaded (skipped)
      for (int j = 0; j < E; ++j) out->order[j] = members[size_t(pl.order[size_t(j)])];
    }
    if (out->feasible) *out->feasible = pl.feasible ? 1 : 0;
  }
}

// The InfMoE order of this layer's PREDICTED counts (the EMA of its routed
// rows over its forwards, rounded): the same members rule and scheduler call
// as compute_offloaded, so a stable routing predicts the real order exactly.
std::vector<int> Layer::predicted_order(std::vector<int>* members_out) const {
  std::vector<int> members;
  std::vector<uint64_t> cnt;
  for (int e = 0; e < n_local; ++e) {
    const uint64_t c = uint64_t(std::llround(load_ema[size_t(e)]));
    if (pin_slot[size_t(e)] >= 0) continue;
    if (!desc.skip_empty_experts || c > 0) {
      members.push_back(e);
      cnt.push_back(c);
    }
  }
  std::vector<int> order;
  if (members.empty()) return order;
  const int E = int(members.size());
  Geometry geo{1, 1, 1, desc.d_model, desc.d_ff, E, int(esz)};
  Hardware hw{desc.hw.peak_flops, desc.hw.h2d_bandwidth, desc.hw.device_memory,
              desc.hw.reserved_memory};
  Costs c = derive_costs(cnt.data(), E, geo, hw);
  Plan pl;
  switch (desc.policy) {
    case INFMOE_POLICY_NAIVE: pl = plan_identity(c, desc.K); break;
    case INFMOE_POLICY_GREEDY: pl = plan_greedy(c, desc.K); break;
    case INFMOE_POLICY_EXACT: pl = plan_exact(c, desc.K, 12); break;
    default: pl = plan_auto(c, desc.K, 12); break;
  }
  for (int j = 0; j < E; ++j) order.push_back(members[size_t(pl.order[size_t(j)])]);
  if (members_out) *members_out = members;
  return order;
}

// Called by the previous layer once its last load is issued: stream the first
// prefetch_depth experts of this layer's predicted order into this layer's
// own slots, on this layer's copy lane after the previous layer's loads (one
// load lane) and after every compute that preceded the previous layer's
// forward (the last users of this layer's slot set).  No residency gate is
// needed for positions < K (simulator.hpp:147: the gate starts at j = K).
void Layer::prefetch(cudaEvent_t after_loads, cudaEvent_t after_computes) {
  pf.clear();
  if (!ema_seen || n_scheduled < 0) return;
  const std::vector<int> order = predicted_order(nullptr);
  const int depth = std::max(1, desc.prefetch_depth);
  const int m = std::min({depth, int(order.size()), desc.K, n_rot});
  if (m <= 0) return;
  INFMOE_CUDA(cudaStreamWaitEvent(copy_stream, after_loads, 0));
  INFMOE_CUDA(cudaStreamWaitEvent(copy_stream, after_computes, 0));
  for (int j = 0; j < m; ++j) {
    const int e = order[size_t(j)];
    const int slot = slot_of(j);
    INFMOE_CUDA(cudaEventRecord(t_load0[size_t(j)], copy_stream));
    if (pack) {
      INFMOE_CUDA(cudaMemcpyAsync(stage_of(slot), pack->host + pack->off[size_t(e)],
                                  pack->size[size_t(e)], cudaMemcpyHostToDevice, copy_stream));
    } else {
      INFMOE_CUDA(cudaMemcpyAsync(slot_in + size_t(slot) * expert_in_bytes,
                                  host_in + size_t(e) * expert_in_bytes, expert_in_bytes,
                                  cudaMemcpyHostToDevice, copy_stream));
      INFMOE_CUDA(cudaMemcpyAsync(slot_out + size_t(slot) * expert_in_bytes,
                                  host_out + size_t(e) * expert_in_bytes, expert_in_bytes,
                                  cudaMemcpyHostToDevice, copy_stream));
    }
    INFMOE_CUDA(cudaEventRecord(t_load1[size_t(j)], copy_stream));
    INFMOE_CUDA(cudaEventRecord(load_done[size_t(j)], copy_stream));
    pf.push_back({e});
  }
}

void Layer::set_next(Layer* nxt) {
  require(desc.residency == INFMOE_OFFLOADED && desc.continuous_load_stream,
          "set_next: the layer is not an offloaded continuous_load_stream layer");
  auto unlink = [&] {
    if (next) next->prevs.erase(std::remove(next->prevs.begin(), next->prevs.end(), this),
                                next->prevs.end());
    next = nullptr;
  };
  if (!nxt) {
    unlink();
    return;
  }
  require(nxt->desc.residency == INFMOE_OFFLOADED && nxt->desc.continuous_load_stream,
          "set_next: the next layer is not an offloaded continuous_load_stream layer");
  require(nxt->desc.device == desc.device, "set_next: layers on different devices");
  if (pool_ptr == nxt->pool_ptr && pool_ptr != &own_pool) {
    // one shared pool: consecutive layers use alternate slot sets
    if (!set_assigned) set_assigned = true;
    const int want = slot_base == 0 ? n_rot : 0;
    if (nxt->set_assigned && nxt->slot_base != want)
      fail(kArgument, "set_next: consecutive layers would share a slot set (odd cycle on one "
                      "pool)");
    nxt->slot_base = want;
    nxt->set_assigned = true;
  }
  unlink();
  next = nxt;
  nxt->prevs.push_back(this);
}

// PEER transport: publish (pid, pointers, IPC handles) of the symmetric
// buffers through an NCCL all-gather and map every peer's buffers: a raw
// pointer when the peer lives in this process (ranks as threads), else a CUDA
// IPC mapping (NVLink peer access is enabled lazily by the runtime).
void Layer::peer_setup() {
  struct Info {
    int64_t pid;
    uint64_t ptr[5];
    cudaIpcMemHandle_t h[5];
  };
  const int P = desc.ep_size, me = desc.ep_rank;
  Info mine{};
  mine.pid = int64_t(getpid());
  void* bufs[5] = {sym_x, sym_ret, sym_y, sym_counts, sym_flags};
  for (int i = 0; i < 5; ++i) {
    mine.ptr[i] = reinterpret_cast<uint64_t>(bufs[i]);
    INFMOE_CUDA(cudaIpcGetMemHandle(&mine.h[i], bufs[i]));
  }
  uint8_t* dev = nullptr;
  INFMOE_CUDA(cudaMalloc(&dev, sizeof(Info) * size_t(P + 1)));
  INFMOE_CUDA(cudaMemcpy(dev + sizeof(Info) * size_t(P), &mine, sizeof(Info),
                         cudaMemcpyHostToDevice));
  cudaStream_t s;
  INFMOE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const auto& nc = nccl::api();
  nccl::check(nc.AllGather(dev + sizeof(Info) * size_t(P), dev, sizeof(Info), nccl::kUint8,
                           reinterpret_cast<nccl::Comm>(comm), s),
              "ncclAllGather");
  INFMOE_CUDA(cudaStreamSynchronize(s));
  INFMOE_CUDA(cudaStreamDestroy(s));
  std::vector<Info> all(static_cast<size_t>(P));
  INFMOE_CUDA(cudaMemcpy(all.data(), dev, sizeof(Info) * size_t(P), cudaMemcpyDeviceToHost));
  INFMOE_CUDA(cudaFree(dev));
  std::vector<void*> px(static_cast<size_t>(P)), pr(static_cast<size_t>(P)), pc(static_cast<size_t>(P)),
      pf(static_cast<size_t>(P));
  peer_y.assign(size_t(P), nullptr);
  bool all_remote = true;  // every peer lives in another process
  for (int r = 0; r < P; ++r) {
    void* q[5];
    if (r != me && all[size_t(r)].pid == mine.pid) all_remote = false;
    for (int i = 0; i < 5; ++i) {
      if (r == me || all[size_t(r)].pid == mine.pid) {
        q[i] = reinterpret_cast<void*>(all[size_t(r)].ptr[i]);
      } else {
        INFMOE_CUDA(cudaIpcOpenMemHandle(&q[i], all[size_t(r)].h[i],
                                         cudaIpcMemLazyEnablePeerAccess));
        ipc_opened.push_back(q[i]);
      }
    }
    px[size_t(r)] = q[0];
    pr[size_t(r)] = q[1];
    peer_y[size_t(r)] = q[2];
    pc[size_t(r)] = q[3];
    pf[size_t(r)] = q[4];
  }
  // barriers: device epoch flags when the peers are other processes (one
  // process per GPU: no collective and no host per barrier); a 1-int NCCL
  // all-reduce when ranks share this process (threads: a spinning barrier
  // kernel could stall another rank's first kernel launch, e.g. a lazy module
  // load).  INFMOE_EP_BARRIER=device|nccl overrides.
  dev_barrier = all_remote;
  if (const char* m = std::getenv("INFMOE_EP_BARRIER")) {
    if (std::string(m) == "device") dev_barrier = true;
    else if (std::string(m) == "nccl") dev_barrier = false;
  }
  d_peer_flags = reinterpret_cast<uint32_t**>(dalloc<void*>(size_t(P), owned));
  INFMOE_CUDA(cudaMemcpy(d_peer_flags, pf.data(), sizeof(void*) * P, cudaMemcpyHostToDevice));
  d_peer_x = dalloc<void*>(size_t(P), owned);
  d_peer_ret = dalloc<int2*>(size_t(P), owned);
  d_peer_counts = dalloc<int32_t*>(size_t(P), owned);
  INFMOE_CUDA(cudaMemcpy(d_peer_x, px.data(), sizeof(void*) * P, cudaMemcpyHostToDevice));
  INFMOE_CUDA(cudaMemcpy(d_peer_ret, pr.data(), sizeof(void*) * P, cudaMemcpyHostToDevice));
  INFMOE_CUDA(cudaMemcpy(d_peer_counts, pc.data(), sizeof(void*) * P, cudaMemcpyHostToDevice));
}

// every rank's work enqueued before this point has finished before any rank's
// work after it starts: a 1-int all-reduce on the stream
void Layer::peer_barrier(cudaStream_t s) {
  if (dev_barrier) {
    static const uint64_t timeout_ns = [] {
      const char* t = std::getenv("INFMOE_EP_BARRIER_TIMEOUT_S");
      return uint64_t(t ? std::atof(t) * 1e9 : 60e9);
    }();
    launch_ep_flag_barrier(d_peer_flags, sym_flags, desc.ep_rank, desc.ep_size, ++bar_epoch,
                           timeout_ns, s);
    return;
  }
  const auto& nc = nccl::api();
  nccl::check(nc.AllReduce(bar_buf, bar_buf, 1, nccl::kInt32, nccl::kSum,
                           reinterpret_cast<nccl::Comm>(comm), s),
              "ncclAllReduce");
}

void Layer::ep_exchange_out(int64_t N, cudaStream_t s) {
  (void)N;
  const auto& nc = nccl::api();
  auto* cm = reinterpret_cast<nccl::Comm>(comm);
  const int P = desc.ep_size, E = desc.n_experts, El = n_local;
  // 1. count exchange: rows routed to each of the peer's experts
  nccl::check(nc.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < P; ++r) {
    nccl::check(nc.Send(counts + size_t(r) * El, size_t(El), nccl::kInt32, r, cm, s), "ncclSend");
    nccl::check(nc.Recv(recv_counts_dev + size_t(r) * El, size_t(El), nccl::kInt32, r, cm, s),
                "ncclRecv");
  }
  nccl::check(nc.GroupEnd(), "ncclGroupEnd");
  INFMOE_CUDA(cudaMemcpyAsync(counts_host, counts, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
  INFMOE_CUDA(cudaMemcpyAsync(counts_host + E, recv_counts_dev, sizeof(int32_t) * P * El,
                              cudaMemcpyDeviceToHost, s));
  INFMOE_CUDA(cudaStreamSynchronize(s));
  // 2. plan (host) + upload of the local layout
  plan = make_ep_plan(P, desc.ep_rank, E, counts_host, counts_host + E);
  const size_t pn = size_t(El) + 1 + size_t(plan.n_recv);
  grow(plan_dev, plan_cap, pn);
  if (pn > plan_host_cap) {
    if (plan_host) INFMOE_CUDA(cudaFreeHost(plan_host));
    plan_host_cap = std::max(pn, plan_host_cap * 2);
    INFMOE_CUDA(cudaMallocHost(&plan_host, plan_host_cap * sizeof(int32_t)));
  }
  std::memcpy(plan_host, plan.local_offsets.data(), sizeof(int32_t) * (El + 1));
  std::memcpy(plan_host + El + 1, plan.local_index.data(), sizeof(int32_t) * plan.n_recv);
  INFMOE_CUDA(cudaMemcpyAsync(plan_dev, plan_host, sizeof(int32_t) * pn, cudaMemcpyHostToDevice, s));
  const size_t rowb = size_t(desc.d_model) * esz;
  const size_t nr = size_t(std::max<int64_t>(plan.n_recv, 1));
  grow(recv_x, cap_x, nr * rowb);
  grow(loc_x, cap_lx, nr * rowb);
  grow(loc_h, cap_h, nr * size_t(desc.d_ff) * esz);
  grow(loc_y, cap_ly, nr * rowb);
  grow(recv_y, cap_ry, nr * rowb);
  // 3. token all-to-allv (dispatch)
  nccl::check(nc.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < P; ++r) {
    nccl::check(nc.Send(xp + size_t(plan.send_off[size_t(r)]) * rowb,
                        size_t(plan.send_rows[size_t(r)]) * rowb, nccl::kUint8, r, cm, s),
                "ncclSend");
    nccl::check(nc.Recv(recv_x + size_t(plan.recv_off[size_t(r)]) * rowb,
                        size_t(plan.recv_rows[size_t(r)]) * rowb, nccl::kUint8, r, cm, s),
                "ncclRecv");
  }
  nccl::check(nc.GroupEnd(), "ncclGroupEnd");
  // 4. expert-contiguous local rows
  launch_gather_rows(recv_x, desc.dtype, plan.n_recv, desc.d_model, 1, plan_dev + El + 1, loc_x,
                     s);
}

void Layer::ep_exchange_back(cudaStream_t s) {
  const auto& nc = nccl::api();
  auto* cm = reinterpret_cast<nccl::Comm>(comm);
  const int P = desc.ep_size, El = n_local;
  const size_t rowb = size_t(desc.d_model) * esz;
  launch_scatter_rows(loc_y, desc.dtype, plan.n_recv, desc.d_model, plan_dev + El + 1, recv_y, s);
  nccl::check(nc.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < P; ++r) {
    nccl::check(nc.Send(recv_y + size_t(plan.recv_off[size_t(r)]) * rowb,
                        size_t(plan.recv_rows[size_t(r)]) * rowb, nccl::kUint8, r, cm, s),
                "ncclSend");
    nccl::check(nc.Recv(yp + size_t(plan.send_off[size_t(r)]) * rowb,
                        size_t(plan.send_rows[size_t(r)]) * rowb, nccl::kUint8, r, cm, s),
                "ncclRecv");
  }
  nccl::check(nc.GroupEnd(), "ncclGroupEnd");
}

void Layer::forward(const void* x, int64_t N, void* y, infmoe_forward_out* out, cudaStream_t s,
                    const int32_t* given_idx, const float* given_w) {
  require(N >= 0 && N <= desc.max_tokens, "forward: N exceeds max_tokens");
  INFMOE_CUDA(cudaSetDevice(desc.device));
  const int E = desc.n_experts, k = desc.top_k;
  const bool offloaded = desc.residency == INFMOE_OFFLOADED;
  const bool timed = out && (out->events || out->exposed_copy_s);
  INFMOE_CUDA(cudaEventRecord(t_start, s));
  route(x, N, s, given_idx, given_w);
  if (out) {  // per-token routing outputs at the layer boundary (device to device)
    const size_t A = size_t(N) * size_t(k);
    if (out->topk_idx && A)
      INFMOE_CUDA(cudaMemcpyAsync(out->topk_idx, idx, A * 4, cudaMemcpyDeviceToDevice, s));
    if (out->topk_w && A)
      INFMOE_CUDA(cudaMemcpyAsync(out->topk_w, wts, A * 4, cudaMemcpyDeviceToDevice, s));
    if (out->perm && A)
      INFMOE_CUDA(cudaMemcpyAsync(out->perm, perm, A * 4, cudaMemcpyDeviceToDevice, s));
    if (out->offsets)
      INFMOE_CUDA(cudaMemcpyAsync(out->offsets, offsets, size_t(E + 1) * 4,
                                  cudaMemcpyDeviceToDevice, s));
  }

  Rows r;
  std::vector<int32_t> local_counts;
  if (!use_ep) {
    r = Rows{xp, offsets, N * k, hbuf, yp, nullptr};
    if (offloaded || (out && (out->counts || out->local_rows))) {
      INFMOE_CUDA(cudaMemcpyAsync(counts_host, counts, sizeof(int32_t) * E,
                                  cudaMemcpyDeviceToHost, s));
      if (offloaded) {
        INFMOE_CUDA(cudaStreamSynchronize(s));
        r.counts = counts_host;
      }
    }
  } else if (ep_peer) {
    // PEER transport: counts to every rank, plan on the device, rows pushed
    // into the owners' expert-contiguous buffers; no host round trip unless
    // the offload order (or the caller) needs the local counts
    const int P = desc.ep_size, me = desc.ep_rank;
    launch_ep_counts_push(counts, E, me, P, d_peer_counts, s);
    peer_barrier(s);
    launch_ep_plan(sym_counts, P, E, me, dest_base, loc_offsets, s);
    launch_ep_dispatch_push(x, perm, k, desc.dtype, N * k, desc.d_model, offsets, E, P,
                            dest_base, me, d_peer_x, d_peer_ret, s);
    peer_barrier(s);
    const bool need_counts = offloaded || (out && (out->local_rows || out->counts));
    if (need_counts) {
      INFMOE_CUDA(cudaMemcpyAsync(counts_host, counts, sizeof(int32_t) * E,
                                  cudaMemcpyDeviceToHost, s));
      INFMOE_CUDA(cudaMemcpyAsync(counts_host + E, loc_offsets, sizeof(int32_t) * (n_local + 1),
                                  cudaMemcpyDeviceToHost, s));
      INFMOE_CUDA(cudaStreamSynchronize(s));
      local_counts.resize(size_t(n_local));
      for (int e = 0; e < n_local; ++e)
        local_counts[size_t(e)] = counts_host[E + e + 1] - counts_host[E + e];
    }
    r = Rows{sym_x, loc_offsets, cap_recv, loc_h, sym_y,
             need_counts ? local_counts.data() : nullptr};
  } else {
    ep_exchange_out(N, s);
    local_counts.resize(size_t(n_local));
    for (int e = 0; e < n_local; ++e)
      local_counts[size_t(e)] = plan.local_offsets[size_t(e) + 1] - plan.local_offsets[size_t(e)];
    r = Rows{loc_x, plan_dev, plan.n_recv, loc_h, loc_y, local_counts.data()};
  }

  // top-1 without an exchange: the combine is fused into the GEMM2 epilogue
  fused_out = (k == 1 && !use_ep && desc.dtype == INFMOE_DTYPE_BF16) ? y : nullptr;
  if (offloaded) compute_offloaded(r, timed, out, s);
  else compute_resident(r, timed, s);

  if (ep_peer) {
    peer_barrier(s);  // every owner has written my rows' results into sym_y
    launch_combine(sym_y, desc.dtype, inv, wts, N, k, desc.d_model, y, s);
  } else {
    if (use_ep) ep_exchange_back(s);
    if (!fused_out) launch_combine(yp, desc.dtype, inv, wts, N, k, desc.d_model, y, s);
  }

  if (!out) return;
  const bool need_sync = timed || ((out->counts || out->local_rows) && !offloaded && !use_ep);
  if (need_sync) INFMOE_CUDA(cudaStreamSynchronize(s));
  if (out->counts) std::memcpy(out->counts, counts_host, sizeof(int32_t) * E);
  if (out->local_rows) {
    if (use_ep) std::memcpy(out->local_rows, local_counts.data(), sizeof(int32_t) * n_local);
    else std::memcpy(out->local_rows, counts_host, sizeof(int32_t) * n_local);
  }
  if (!timed) return;
  // event times are seconds from this forward's start, or from the caller's
  // origin event (out->time_origin) so a stack's layers share one time axis
  double base = 0.0;
  if (out->time_origin) {
    float o = 0;
    INFMOE_CUDA(cudaEventElapsedTime(&o, reinterpret_cast<cudaEvent_t>(out->time_origin),
                                     t_start));
    base = double(o) * 1e-3;
  }
  if (!offloaded) {
    float a = 0, b = 0;
    INFMOE_CUDA(cudaEventElapsedTime(&a, t_start, t_comp0[0]));
    INFMOE_CUDA(cudaEventElapsedTime(&b, t_start, t_comp1[0]));
    if (out->events)
      out->events[0] = {INFMOE_STREAM_COMPUTE, 0, -1, base + a * 1e-3, base + b * 1e-3};
    if (out->exposed_copy_s) *out->exposed_copy_s = 0.0;
    return;
  }
  double busy = 0.0, makespan = 0.0;
  if (out->events)
    for (int j = 0; j < 2 * n_local; ++j) out->events[j] = {-1, 0, -1, 0.0, 0.0};
  if (n_pinned_run > 0) {  // one grouped launch: a compute event per pinned expert, no load
    float a = 0, b = 0;
    INFMOE_CUDA(cudaEventElapsedTime(&a, t_start, t_pin0));
    INFMOE_CUDA(cudaEventElapsedTime(&b, t_start, t_pin1));
    if (out->events)
      for (int i = 0; i < n_pinned_run; ++i)
        out->events[2 * (n_scheduled + i) + 1] = {INFMOE_STREAM_COMPUTE, 0, pinned_run[size_t(i)],
                                                  base + a * 1e-3, base + b * 1e-3};
    busy += (b - a) * 1e-3;
    makespan = std::max(makespan, double(b) * 1e-3);
  }
  for (int j = 0; j < n_scheduled; ++j) {
    float a = 0, b = 0, c0 = 0, c1 = 0;
    INFMOE_CUDA(cudaEventElapsedTime(&a, t_start, t_load0[size_t(j)]));
    INFMOE_CUDA(cudaEventElapsedTime(&b, t_start, t_load1[size_t(j)]));
    INFMOE_CUDA(cudaEventElapsedTime(&c0, t_start, t_comp0[size_t(j)]));
    INFMOE_CUDA(cudaEventElapsedTime(&c1, t_start, t_comp1[size_t(j)]));
    const int e = exec_order[size_t(j)];
    if (out->events) {
      out->events[2 * j] = {INFMOE_STREAM_LOAD, 0, e, base + a * 1e-3, base + b * 1e-3};
      out->events[2 * j + 1] = {INFMOE_STREAM_COMPUTE, 0, e, base + c0 * 1e-3, base + c1 * 1e-3};
    }
    busy += (c1 - c0) * 1e-3;
    makespan = std::max(makespan, double(c1) * 1e-3);
  }
  if (out->exposed_copy_s) *out->exposed_copy_s = makespan - busy;
}

// ------------------------------------------------------- exp4 host packs --
namespace {
struct PackKey {
  const void* a;
  const void* b;
  int n;
  uint64_t elems;
  int codec_id;
  bool operator<(const PackKey& o) const {
    return std::tie(a, b, n, elems, codec_id) < std::tie(o.a, o.b, o.n, o.elems, o.codec_id);
  }
};
std::mutex g_pack_mu;
std::map<PackKey, std::weak_ptr<HostPack>> g_packs;
}  // namespace

// 64-bit content digest of both host matrices of every expert (threads over
// 1 MiB blocks, combined in block order): a cached pack is reused only for
// identical bytes
static uint64_t host_digest(const void* w_in, const void* w_out, uint64_t bytes_each) {
  constexpr uint64_t kBlock = 1 << 20;
  const uint64_t nb = (bytes_each + kBlock - 1) / kBlock;
  std::vector<uint64_t> part(size_t(2 * nb), 0);
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::atomic<uint64_t> next{0};
  auto work = [&] {
    for (uint64_t b = next++; b < 2 * nb; b = next++) {
      const auto* base = static_cast<const uint8_t*>(b < nb ? w_in : w_out);
      const uint64_t off = (b % nb) * kBlock, len = std::min(kBlock, bytes_each - off);
      uint64_t h = 0x9e3779b97f4a7c15ull ^ b, w = 0;
      const uint8_t* q = base + off;
      uint64_t i = 0;
      for (; i + 8 <= len; i += 8) {
        std::memcpy(&w, q + i, 8);
        h = (h ^ w) * 0x100000001b3ull + (h >> 29);
      }
      for (; i < len; ++i) h = (h ^ q[i]) * 0x100000001b3ull;
      part[size_t(b)] = h;
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  uint64_t h = bytes_each;
  for (uint64_t v : part) h = dev_mix64(h ^ v);
  return h;
}

// ---- on-disk pack cache ----------------------------------------------------
// <dir>/<digest>-<codec>-<experts>x<elems>.infmoe-pack:
//   "INFMOEPK" | u32 version | u32 codec | u64 experts | u64 elems | u64 digest |
//   u64 total | u64 max_size | u64 raw_bytes | u64 pack checksum |
//   per expert {off, size, in_size} | exph: per expert {lay_in, lay_out} |
//   the pack bytes.  The checksum covers the tables and the pack bytes; a file
//   whose header, tables or checksum do not match is ignored (and replaced by
//   the next encode).
namespace {
std::string g_pack_dir = [] {
  const char* e = std::getenv("INFMOE_PACK_CACHE_DIR");
  return std::string(e ? e : "");
}();
constexpr char kPackMagic[8] = {'I', 'N', 'F', 'M', 'O', 'E', 'P', 'K'};
constexpr uint32_t kPackVersion = 4;  // 2: 256-byte aligned pack parts; 3: exph (dist, m2) symbols; 4: pair residuals, 64-bit LUT

uint64_t pack_checksum(const uint8_t* p, uint64_t bytes) {
  // both halves (and an odd last byte)
  return host_digest(p, p + bytes / 2, bytes / 2) ^ dev_mix64(bytes + (bytes & 1 ? p[bytes - 1] : 0));
}

// digest of the per-expert tables (offsets, sizes, exph layouts) and the header
// sizes: the file's checksum covers them together with the pack bytes
uint64_t tables_digest(const HostPack& p) {
  uint64_t h = dev_mix64(p.total ^ (p.max_size << 1) ^ (p.raw_bytes << 2));
  auto mix = [&](const void* q, size_t bytes) {
    const auto* b = static_cast<const uint8_t*>(q);
    for (size_t i = 0; i < bytes; i += 8) {
      uint64_t w = 0;
      std::memcpy(&w, b + i, std::min<size_t>(8, bytes - i));
      h = dev_mix64(h ^ w);
    }
  };
  mix(p.off.data(), p.off.size() * 8);
  mix(p.size.data(), p.size.size() * 8);
  mix(p.in_size.data(), p.in_size.size() * 8);
  mix(p.lay_in.data(), p.lay_in.size() * sizeof(codec::ExphLayout));
  mix(p.lay_out.data(), p.lay_out.size() * sizeof(codec::ExphLayout));
  return h;
}

// the tables describe parts that lie inside the pack and layouts that fit their
// parts (a damaged file is rejected before any decode could read past a part)
bool tables_sane(const HostPack& p, uint64_t elems) {
  for (size_t e = 0; e < p.off.size(); ++e) {
    if (p.in_size[e] > p.size[e] || p.off[e] + p.size[e] > p.total || p.size[e] > p.max_size)
      return false;
    if (p.codec_id == INFMOE_CODEC_EXPH) {
      const codec::ExphLayout& a = p.lay_in[e];
      const codec::ExphLayout& b = p.lay_out[e];
      if (a.n != elems || b.n != elems || a.bytes > p.in_size[e] ||
          b.bytes > p.size[e] - p.in_size[e])
        return false;
    }
  }
  return true;
}

std::string pack_path(uint64_t digest, int codec_id, int n_experts, uint64_t elems) {
  char name[128];
  std::snprintf(name, sizeof(name), "%016llx-%d-%dx%llu.infmoe-pack",
                static_cast<unsigned long long>(digest), codec_id, n_experts,
                static_cast<unsigned long long>(elems));
  return g_pack_dir + "/" + name;
}

struct PackHeader {
  char magic[8];
  uint32_t version, codec;
  uint64_t experts, elems, digest, total, max_size, raw_bytes, checksum;
};

bool pack_load(const std::string& path, HostPack& p, int n_experts, uint64_t elems) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  PackHeader h;
  bool ok = std::fread(&h, sizeof(h), 1, f) == 1 && std::memcmp(h.magic, kPackMagic, 8) == 0 &&
            h.version == kPackVersion && int(h.codec) == p.codec_id &&
            h.experts == uint64_t(n_experts) && h.elems == elems && h.digest == p.digest;
  const size_t ne = size_t(n_experts);
  if (ok) {
    p.off.resize(ne);
    p.size.resize(ne);
    p.in_size.resize(ne);
    for (size_t e = 0; e < ne && ok; ++e) {
      uint64_t v[3];
      ok = std::fread(v, sizeof(v), 1, f) == 1;
      p.off[e] = v[0];
      p.size[e] = v[1];
      p.in_size[e] = v[2];
    }
  }
  if (ok && p.codec_id == INFMOE_CODEC_EXPH) {
    p.lay_in.resize(ne);
    p.lay_out.resize(ne);
    for (size_t e = 0; e < ne && ok; ++e)
      ok = std::fread(&p.lay_in[e], sizeof(codec::ExphLayout), 1, f) == 1 &&
           std::fread(&p.lay_out[e], sizeof(codec::ExphLayout), 1, f) == 1;
  }
  if (ok) {
    p.total = h.total;
    p.max_size = h.max_size;
    p.raw_bytes = h.raw_bytes;
    ok = tables_sane(p, elems);
  }
  if (ok) {
    INFMOE_CUDA(cudaMallocHost(&p.host, p.total));
    ok = std::fread(p.host, 1, p.total, f) == p.total &&
         (pack_checksum(p.host, p.total) ^ tables_digest(p)) == h.checksum;
    if (!ok) {
      cudaFreeHost(p.host);
      p.host = nullptr;
    }
  }
  std::fclose(f);
  if (!ok) {
    p.off.clear(); p.size.clear(); p.in_size.clear(); p.lay_in.clear(); p.lay_out.clear();
    p.total = p.max_size = p.raw_bytes = 0;
  }
  return ok;
}

void pack_save(const std::string& path, const HostPack& p, int n_experts, uint64_t elems) {
  const std::string tmp = path + ".tmp." + std::to_string(::getpid());
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return;  // an unwritable cache directory only costs the next re-encode
  PackHeader h;
  std::memcpy(h.magic, kPackMagic, 8);
  h.version = kPackVersion;
  h.codec = uint32_t(p.codec_id);
  h.experts = uint64_t(n_experts);
  h.elems = elems;
  h.digest = p.digest;
  h.total = p.total;
  h.max_size = p.max_size;
  h.raw_bytes = p.raw_bytes;
  h.checksum = pack_checksum(p.host, p.total) ^ tables_digest(p);
  bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1;
  for (int e = 0; e < n_experts && ok; ++e) {
    const uint64_t v[3] = {p.off[size_t(e)], p.size[size_t(e)], p.in_size[size_t(e)]};
    ok = std::fwrite(v, sizeof(v), 1, f) == 1;
  }
  if (p.codec_id == INFMOE_CODEC_EXPH)
    for (int e = 0; e < n_experts && ok; ++e)
      ok = std::fwrite(&p.lay_in[size_t(e)], sizeof(codec::ExphLayout), 1, f) == 1 &&
           std::fwrite(&p.lay_out[size_t(e)], sizeof(codec::ExphLayout), 1, f) == 1;
  ok = ok && std::fwrite(p.host, 1, p.total, f) == p.total;
  ok = (std::fclose(f) == 0) && ok;
  if (!ok || std::rename(tmp.c_str(), path.c_str()) != 0) std::remove(tmp.c_str());
}
}  // namespace

void HostPack::set_cache_dir(const char* dir) {
  std::lock_guard<std::mutex> lock(g_pack_mu);
  g_pack_dir = dir ? dir : "";
}

std::shared_ptr<HostPack> HostPack::acquire(const void* w_in, const void* w_out, int n_experts,
                                            uint64_t matrix_elems, int codec_id, bool fresh) {
  std::lock_guard<std::mutex> lock(g_pack_mu);
  const PackKey key{w_in, w_out, n_experts, matrix_elems, codec_id};
  const uint64_t digest = host_digest(w_in, w_out, uint64_t(n_experts) * matrix_elems * 2);
  auto it = g_packs.find(key);
  if (!fresh && it != g_packs.end())
    if (auto sp = it->second.lock())
      if (sp->digest == digest) return sp;
  auto p = std::make_shared<HostPack>();
  p->codec_id = codec_id;
  p->digest = digest;
  const std::string path =
      g_pack_dir.empty() ? std::string() : pack_path(digest, codec_id, n_experts, matrix_elems);
  if (!path.empty() && pack_load(path, *p, n_experts, matrix_elems)) {
    p->source = 2;
    g_packs[key] = p;
    return p;
  }
  const auto* in = static_cast<const uint16_t*>(w_in);
  const auto* out = static_cast<const uint16_t*>(w_out);
  const bool h = codec_id == INFMOE_CODEC_EXPH;
  std::vector<codec::Exp4Plan> p4;
  std::vector<codec::ExphPlan> ph;
  for (int e = 0; e < n_experts; ++e)
    for (const uint16_t* m : {in + uint64_t(e) * matrix_elems, out + uint64_t(e) * matrix_elems}) {
      if (h) ph.push_back(codec::exph_plan(m, matrix_elems));
      else p4.push_back(codec::exp4_plan(m, matrix_elems));
    }
  for (int e = 0; e < n_experts; ++e) {
    const size_t i1 = size_t(2 * e), i2 = i1 + 1;
    const uint64_t a = h ? ph[i1].L.bytes : p4[i1].bytes;
    const uint64_t b = h ? ph[i2].L.bytes : p4[i2].bytes;
    if (h) {
      p->lay_in.push_back(ph[i1].L);
      p->lay_out.push_back(ph[i2].L);
    }
    // every copy (an expert's pack pair, or its W_out part alone) starts on a
    // 256-byte boundary in host and device memory: 16-byte aligned starts ran
    // the host link 0.6% slower (tools/h2d_copy_probe.py)
    constexpr uint64_t kAl = 256;
    const uint64_t a_pad = (a + kAl - 1) / kAl * kAl;
    const uint64_t span = (a_pad + b + kAl - 1) / kAl * kAl;
    p->off.push_back(p->total);
    p->size.push_back(a_pad + b);
    p->in_size.push_back(a_pad);
    p->max_size = std::max(p->max_size, span);
    p->total += span;
  }
  p->raw_bytes = uint64_t(n_experts) * matrix_elems * 2 * 2;
  INFMOE_CUDA(cudaMallocHost(&p->host, p->total));
  for (int e = 0; e < n_experts; ++e) {
    uint8_t* dst = p->host + p->off[size_t(e)];
    const uint64_t a = h ? ph[size_t(2 * e)].L.bytes : p4[size_t(2 * e)].bytes;
    const uint64_t end = e + 1 < n_experts ? p->off[size_t(e + 1)] : p->total;
    std::memset(dst + a, 0, p->in_size[size_t(e)] - a);              // padding after W_in
    std::memset(dst + p->size[size_t(e)], 0, end - p->off[size_t(e)] - p->size[size_t(e)]);
    const uint16_t* m1 = in + uint64_t(e) * matrix_elems;
    const uint16_t* m2 = out + uint64_t(e) * matrix_elems;
    if (h) {
      codec::exph_fill(m1, ph[size_t(2 * e)], dst);
      codec::exph_fill(m2, ph[size_t(2 * e + 1)], dst + p->in_size[size_t(e)]);
    } else {
      codec::exp4_fill(m1, p4[size_t(2 * e)], dst);
      codec::exp4_fill(m2, p4[size_t(2 * e + 1)], dst + p->in_size[size_t(e)]);
    }
  }
  if (!path.empty()) pack_save(path, *p, n_experts, matrix_elems);
  g_packs[key] = p;
  return p;
}

HostPack::~HostPack() {
  if (host) cudaFreeHost(host);
}

}  // namespace infmoe
