// capi_device.cu — extern "C" entry points of the device path (infmoe.h,
// "Device path" section).  Every call is exception-guarded.
#include <cstring>
#include <vector>

#include "../host/status.hpp"
#include "../kernels/codec.cuh"
#include "../kernels/common.cuh"
#include "../kernels/expert_gemm.cuh"
#include "../kernels/kernels.cuh"
#include "infmoe.h"
#include "../host/ep_plan.hpp"
#include "layer.hpp"
#include "nccl_shim.hpp"

using namespace infmoe;

struct infmoe_layer {
  Layer* impl;
};

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int infmoe_fill_uniform(void* out, int32_t dtype, uint64_t n, uint64_t seed, float scale,
                        void* stream) {
  return guarded([&] {
    require(out != nullptr || n == 0, "fill: out is NULL");
    launch_fill_uniform(out, dtype, n, seed, scale, as_stream(stream));
  });
}

int infmoe_debug_occupy_sms(int32_t n_ctas, int32_t smem_bytes, const int32_t* release,
                            uint64_t timeout_ns, int32_t* timed_out, void* stream) {
  return guarded([&] {
    require(n_ctas >= 1 && smem_bytes >= 0 && release && timed_out, "occupy: bad arguments");
    launch_occupy(n_ctas, size_t(smem_bytes), release, timeout_ns, timed_out, as_stream(stream));
  });
}

int infmoe_debug_set_flag(int32_t* flag, void* stream) {
  return guarded([&] {
    require(flag != nullptr, "set_flag: NULL flag");
    launch_set_flag(flag, as_stream(stream));
  });
}

int infmoe_gate_softmax_topk(const void* x, int32_t dtype, int64_t N, int32_t d,
                             const float* wg, const float* bias, int32_t E, int32_t k,
                             int32_t* topk_idx, float* topk_w, int32_t* counts, void* stream) {
  return guarded([&] {
    require(x && wg && topk_idx && topk_w && counts, "gate: NULL pointer");
    launch_gate_softmax(x, dtype, N, d, wg, bias, E, k, topk_idx, topk_w, counts,
                        as_stream(stream));
  });
}

size_t infmoe_gate_softmax_ws_bytes(int32_t dtype, int64_t N, int32_t d, int32_t E, int32_t k) {
  size_t r = 0;
  guarded([&] { r = gate_softmax_ws_bytes(dtype, N, d, E, k); });
  return r;
}

int infmoe_gate_softmax_prepare(const float* wg, int32_t d, int32_t E, void* ws,
                                size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(wg && ws, "gate prepare: NULL pointer");
    require(ws_bytes >= gate_softmax_ws_bytes(kDtypeBf16, 1, d, E, 2),
            "gate prepare: workspace too small");
    gate_softmax_prepare(wg, d, E, ws, as_stream(stream));
  });
}

int infmoe_gate_softmax_topk_ws(const void* x, int32_t dtype, int64_t N, int32_t d,
                                const float* wg, const float* bias, int32_t E, int32_t k,
                                int32_t* topk_idx, float* topk_w, int32_t* counts, void* ws,
                                size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(x && wg && topk_idx && topk_w && counts, "gate: NULL pointer");
    const size_t need = gate_softmax_ws_bytes(dtype, N, d, E, k);
    require(need == 0 || (ws && ws_bytes >= need), "gate: workspace too small");
    launch_gate_softmax(x, dtype, N, d, wg, bias, E, k, topk_idx, topk_w, counts,
                        as_stream(stream), ws, ws_bytes, /*ws_prepared=*/true);
  });
}

int infmoe_gate_softmax_debug(const void* x, int32_t dtype, int64_t N, int32_t d,
                              const float* wg, const float* bias, int32_t E, int32_t k,
                              int32_t* topk_idx, float* topk_w, int32_t* counts,
                              float* approx_logits, uint64_t* stats, void* stream) {
  return guarded([&] {
    require(x && wg && topk_idx && topk_w && counts, "gate: NULL pointer");
    launch_gate_softmax(x, dtype, N, d, wg, bias, E, k, topk_idx, topk_w, counts,
                        as_stream(stream), nullptr, 0, false, approx_logits,
                        reinterpret_cast<unsigned long long*>(stats));
  });
}

int infmoe_gate_lsh(const void* x, int32_t dtype, int64_t N, int32_t d, const double* proj,
                    int32_t bits, int32_t E, uint32_t* codes, int32_t* topk_idx, float* topk_w,
                    int32_t* counts, void* stream) {
  return guarded([&] {
    require(x && proj && topk_idx && topk_w && counts, "lsh gate: NULL pointer");
    launch_gate_lsh(x, dtype, N, d, proj, bits, E, codes, topk_idx, topk_w, counts,
                    as_stream(stream));
  });
}

size_t infmoe_dispatch_workspace_bytes(int64_t n_assign, int32_t E) {
  return dispatch_workspace_bytes(n_assign, E);
}

int infmoe_dispatch(const int32_t* topk_idx, int64_t N, int32_t k, int32_t E, int32_t* offsets,
                    int32_t* perm, int32_t* inv, void* workspace, void* stream) {
  return guarded([&] {
    require(topk_idx && offsets && perm && inv, "dispatch: NULL pointer");
    launch_dispatch(topk_idx, N * k, E, offsets, perm, inv, workspace, as_stream(stream));
  });
}

int infmoe_gather_rows(const void* x, int32_t dtype, int64_t N, int32_t d, int32_t k,
                       const int32_t* perm, void* x_perm, void* stream) {
  return guarded([&] {
    require(x && perm && x_perm, "gather: NULL pointer");
    launch_gather_rows(x, dtype, N, d, k, perm, x_perm, as_stream(stream));
  });
}

int infmoe_gather_rows_by_token(const void* x, int32_t dtype, int64_t N, int32_t d, int32_t k,
                                const int32_t* inv, void* x_perm, void* stream) {
  return guarded([&] {
    require(x && inv && x_perm, "gather: NULL pointer");
    launch_gather_rows_by_token(x, dtype, N, d, k, inv, x_perm, as_stream(stream));
  });
}

int infmoe_expert_ffn(const void* x_perm, int64_t n_rows, int32_t d_model, int32_t d_ff,
                      int32_t dtype, const int32_t* offsets, int32_t E, const void* w_in,
                      const void* w_out, int32_t n_slots, const int32_t* experts,
                      const int32_t* slots, int32_t n_groups, void* h, void* y_perm,
                      void* stream) {
  return guarded([&] {
    require(x_perm && offsets && w_in && w_out && h && y_perm, "expert_ffn: NULL pointer");
    GroupedGemmArgs g;
    std::memset(&g, 0, sizeof(g));
    if (!experts) {
      n_groups = E;
      require(n_slots >= E, "expert_ffn: n_slots < E with experts == NULL");
    }
    require(n_groups >= 1 && n_groups <= kMaxGroups, "expert_ffn: n_groups out of range");
    for (int i = 0; i < n_groups; ++i) {
      g.experts[i] = experts ? experts[i] : i;
      g.slots[i] = experts ? slots[i] : i;
      require(g.experts[i] >= 0 && g.experts[i] < E, "expert_ffn: expert id out of range");
      require(g.slots[i] >= 0 && g.slots[i] < n_slots, "expert_ffn: slot out of range");
    }
    g.n_groups = n_groups;
    g.dtype = dtype;
    g.offsets = offsets;
    g.n_slots = n_slots;
    g.a = x_perm;
    g.a_rows = n_rows;
    g.b = w_in;
    g.N = d_ff;
    g.K = d_model;
    g.out = h;
    g.gelu = 1;
    if (n_rows == 0) return;
    launch_grouped_gemm(g, as_stream(stream));
    g.a = h;
    g.b = w_out;
    g.N = d_model;
    g.K = d_ff;
    g.out = y_perm;
    g.gelu = 0;
    launch_grouped_gemm(g, as_stream(stream));
  });
}

int infmoe_expert_ffn_fused(const void* x_perm, int64_t n_rows, int32_t d_model, int32_t d_ff,
                            const int32_t* offsets, int32_t E, const void* w_in,
                            const void* w_out, int32_t n_slots, const int32_t* experts,
                            const int32_t* slots, int32_t n_groups, void* h, void* y,
                            const int32_t* perm, const float* topk_w, int32_t* done,
                            void* stream) {
  return guarded([&] {
    FusedFfnArgs a;
    std::memset(&a, 0, sizeof(a));
    if (!experts) {
      n_groups = E;
      require(n_slots >= E, "expert_ffn_fused: n_slots < E with experts == NULL");
    }
    require(n_groups >= 1 && n_groups <= kMaxGroups, "expert_ffn_fused: n_groups out of range");
    for (int i = 0; i < n_groups; ++i) {
      a.experts[i] = experts ? experts[i] : i;
      a.slots[i] = experts ? slots[i] : i;
      require(a.experts[i] >= 0 && a.experts[i] < E, "expert_ffn_fused: expert id out of range");
      require(a.slots[i] >= 0 && a.slots[i] < n_slots, "expert_ffn_fused: slot out of range");
    }
    a.x = x_perm;
    a.rows = n_rows;
    a.w_in = w_in;
    a.w_out = w_out;
    a.n_slots = n_slots;
    a.d_model = d_model;
    a.d_ff = d_ff;
    a.dtype = INFMOE_DTYPE_BF16;
    a.offsets = offsets;
    a.n_groups = n_groups;
    a.h = h;
    a.y = y;
    a.perm = perm;
    a.topk_w = topk_w;
    a.done = done;
    if (n_rows == 0) return;
    launch_expert_ffn_fused(a, as_stream(stream));
  });
}

int infmoe_scatter_rows(const void* src, int32_t dtype, int64_t rows, int32_t d,
                        const int32_t* index, void* dst, void* stream) {
  return guarded([&] {
    require(src && index && dst, "scatter: NULL pointer");
    launch_scatter_rows(src, dtype, rows, d, index, dst, as_stream(stream));
  });
}

int infmoe_ep_plan(int32_t P, int32_t rank, int32_t E, const int32_t* send_counts,
                   const int32_t* recv_counts, int64_t* send_off, int64_t* send_rows,
                   int64_t* recv_off, int64_t* recv_rows, int32_t* local_offsets,
                   int32_t* local_index, int64_t* n_recv) {
  return guarded([&] {
    EpPlan p = make_ep_plan(P, rank, E, send_counts, recv_counts);
    auto put = [](int64_t* dst, const std::vector<int64_t>& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(int64_t));
    };
    put(send_off, p.send_off);
    put(send_rows, p.send_rows);
    put(recv_off, p.recv_off);
    put(recv_rows, p.recv_rows);
    if (local_offsets)
      std::memcpy(local_offsets, p.local_offsets.data(), p.local_offsets.size() * sizeof(int32_t));
    if (local_index)
      std::memcpy(local_index, p.local_index.data(), p.local_index.size() * sizeof(int32_t));
    if (n_recv) *n_recv = p.n_recv;
  });
}

int infmoe_ep_get_unique_id(uint8_t id[128]) {
  return guarded([&] {
    require(id != nullptr, "ep: NULL id");
    nccl::UniqueId u;
    nccl::check(nccl::api().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
  });
}

int infmoe_ep_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, void** comm) {
  return guarded([&] {
    require(id && comm && nranks >= 1 && rank >= 0 && rank < nranks, "ep: bad arguments");
    nccl::UniqueId u;
    std::memcpy(u.internal, id, 128);
    nccl::Comm c = nullptr;
    nccl::check(nccl::api().CommInitRank(&c, nranks, u, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int infmoe_ep_comm_destroy(void* comm) {
  return guarded([&] {
    if (comm) nccl::check(nccl::api().CommDestroy(reinterpret_cast<nccl::Comm>(comm)),
                          "ncclCommDestroy");
  });
}

int infmoe_combine(const void* y_perm, int32_t dtype, const int32_t* inv, const float* topk_w,
                   int64_t N, int32_t k, int32_t d, void* y, void* stream) {
  return guarded([&] {
    require(y_perm && inv && topk_w && y, "combine: NULL pointer");
    launch_combine(y_perm, dtype, inv, topk_w, N, k, d, y, as_stream(stream));
  });
}

int infmoe_slot_pool_create(int32_t device, int32_t K, uint64_t expert_matrix_bytes,
                            infmoe_slot_pool** out) {
  return infmoe_slot_pool_create_ex(device, K, expert_matrix_bytes, 1, out);
}

int infmoe_slot_pool_create_ex(int32_t device, int32_t K, uint64_t expert_matrix_bytes,
                               int32_t sets, infmoe_slot_pool** out) {
  return guarded([&] {
    require(out != nullptr, "slot_pool_create: NULL argument");
    *out = nullptr;
    require(K >= 1, "slot_pool_create: K must be >= 1");
    require(sets >= 1 && sets <= 2, "slot_pool_create: sets must be 1 or 2");
    require(expert_matrix_bytes > 0, "slot_pool_create: expert_matrix_bytes must be > 0");
    INFMOE_CUDA(cudaSetDevice(device));
    auto* p = new SlotPool{device, K, sets * (K + 1), sets, size_t(expert_matrix_bytes), nullptr,
                           nullptr};
    const size_t n = size_t(p->n_slots) * p->matrix_bytes;
    cudaError_t e1 = cudaMalloc(&p->slot_in, n);
    cudaError_t e2 = e1 == cudaSuccess ? cudaMalloc(&p->slot_out, n) : e1;
    if (e2 != cudaSuccess) {
      if (p->slot_in) cudaFree(p->slot_in);
      delete p;
      INFMOE_CUDA(e2);
    }
    *out = reinterpret_cast<infmoe_slot_pool*>(p);
  });
}

int infmoe_slot_pool_destroy(infmoe_slot_pool* pool) {
  return guarded([&] {
    if (!pool) return;
    auto* p = reinterpret_cast<SlotPool*>(pool);
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();  // no layer may still be copying into the slots
    cudaFree(p->slot_in);
    cudaFree(p->slot_out);
    if (p->stage) cudaFree(p->stage);
    delete p;
  });
}

int infmoe_layer_create(const infmoe_layer_desc* desc, infmoe_layer** out) {
  return guarded([&] {
    require(desc && out, "layer_create: NULL argument");
    *out = nullptr;
    Layer* impl = new Layer(*desc);
    *out = new infmoe_layer{impl};
  });
}

int infmoe_layer_set_next(infmoe_layer* layer, infmoe_layer* next) {
  return guarded([&] {
    require(layer && layer->impl, "set_next: NULL layer");
    layer->impl->set_next(next ? next->impl : nullptr);
  });
}

int infmoe_layer_forward_routed(infmoe_layer* layer, const void* x, int64_t N,
                                const int32_t* topk_idx, const float* topk_w, void* y,
                                infmoe_forward_out* out, void* stream) {
  return guarded([&] {
    require(layer && layer->impl && (N == 0 || (x && y && topk_idx && topk_w)),
            "layer_forward_routed: NULL argument");
    layer->impl->forward(x, N, y, out, as_stream(stream), topk_idx, topk_w);
  });
}

int infmoe_layer_forward(infmoe_layer* layer, const void* x, int64_t N, void* y,
                         infmoe_forward_out* out, void* stream) {
  return guarded([&] {
    require(layer && layer->impl && (N == 0 || (x && y)), "layer_forward: NULL argument");
    layer->impl->forward(x, N, y, out, as_stream(stream));
  });
}

int infmoe_layer_set_host_weights(infmoe_layer* layer, const void* w_in, const void* w_out) {
  return guarded([&] {
    require(layer && layer->impl, "set_host_weights: NULL layer");
    layer->impl->set_host_weights(w_in, w_out);
  });
}

int infmoe_layer_pin_experts(infmoe_layer* layer, const int32_t* experts, int32_t n) {
  return guarded([&] {
    require(layer && layer->impl, "pin_experts: NULL layer");
    layer->impl->pin_experts(experts, n);
  });
}

int infmoe_layer_pin_hottest(infmoe_layer* layer, int32_t n, int32_t* pinned) {
  return guarded([&] {
    require(layer && layer->impl, "pin_hottest: NULL layer");
    const std::vector<int32_t> got = layer->impl->pin_hottest(n);
    if (pinned) std::copy(got.begin(), got.end(), pinned);
  });
}

int infmoe_codec_roundtrip_host(int32_t codec_id, const uint16_t* in, uint64_t n, uint16_t* out,
                                uint64_t* pack_bytes) {
  return guarded([&] {
    require(in && out, "codec_roundtrip_host: NULL argument");
    require(codec_id == INFMOE_CODEC_EXP4 || codec_id == INFMOE_CODEC_EXPH,
            "codec_roundtrip_host: unknown codec");
    require(n > 0 && n % (codec_id == INFMOE_CODEC_EXPH ? 256 : 128) == 0,
            "codec_roundtrip_host: n must be a positive multiple of 256 (exph) / 128 (exp4)");
    std::vector<uint8_t> pk;
    if (codec_id == INFMOE_CODEC_EXP4) {
      const codec::Exp4Plan plan = codec::exp4_plan(in, n);
      pk.resize(plan.bytes);
      codec::exp4_fill(in, plan, pk.data());
      codec::exp4_unpack_host(pk.data(), n, out);
    } else {
      const codec::ExphPlan plan = codec::exph_plan(in, n);
      pk.resize(plan.L.bytes);
      codec::exph_fill(in, plan, pk.data());
      codec::exph_unpack_host(pk.data(), plan.L, out);
    }
    if (pack_bytes) *pack_bytes = pk.size();
  });
}

int infmoe_layer_pack_source(infmoe_layer* layer, int32_t* source) {
  return guarded([&] {
    require(layer && layer->impl && source, "pack_source: NULL argument");
    *source = layer->impl->pack_source();
  });
}

int infmoe_set_pack_cache_dir(const char* dir) {
  return guarded([&] { HostPack::set_cache_dir(dir); });
}

int infmoe_layer_h2d_bytes(infmoe_layer* layer, uint64_t* packed, uint64_t* raw) {
  return guarded([&] {
    require(layer && layer->impl, "h2d_bytes: NULL layer");
    layer->impl->h2d_bytes(packed, raw);
  });
}

int infmoe_codec_roundtrip(int32_t codec_id, const uint16_t* in, uint64_t n, uint16_t* out,
                           uint64_t* pack_bytes, int32_t device) {
  return guarded([&] {
    require(in && out, "codec_roundtrip: NULL argument");
    require(codec_id == INFMOE_CODEC_EXP4 || codec_id == INFMOE_CODEC_EXPH,
            "codec_roundtrip: unknown codec");
    require(n > 0 && n % (codec_id == INFMOE_CODEC_EXPH ? 256 : 128) == 0,
            "codec_roundtrip: n must be a positive multiple of 256 (exph) / 128 (exp4)");
    INFMOE_CUDA(cudaSetDevice(device));
    std::vector<uint8_t> pk;
    codec::ExphLayout hl;
    if (codec_id == INFMOE_CODEC_EXP4) {
      const codec::Exp4Plan plan = codec::exp4_plan(in, n);
      pk.resize(plan.bytes);
      codec::exp4_fill(in, plan, pk.data());
    } else {
      const codec::ExphPlan plan = codec::exph_plan(in, n);
      hl = plan.L;
      pk.resize(plan.L.bytes);
      codec::exph_fill(in, plan, pk.data());
    }
    if (pack_bytes) *pack_bytes = pk.size();
    uint8_t* dp = nullptr;
    uint16_t* dout = nullptr;
    INFMOE_CUDA(cudaMalloc(&dp, pk.size()));
    INFMOE_CUDA(cudaMalloc(&dout, n * 2));
    INFMOE_CUDA(cudaMemcpy(dp, pk.data(), pk.size(), cudaMemcpyHostToDevice));
    if (codec_id == INFMOE_CODEC_EXP4) codec::launch_exp4_unpack(dp, n, dout, nullptr);
    else codec::launch_exph_unpack(dp, hl, dout, nullptr);
    INFMOE_CUDA(cudaMemcpy(out, dout, n * 2, cudaMemcpyDeviceToHost));
    cudaFree(dp);
    cudaFree(dout);
  });
}

int infmoe_layer_destroy(infmoe_layer* layer) {
  return guarded([&] {
    if (!layer) return;
    delete layer->impl;
    delete layer;
  });
}

}  // extern "C"
