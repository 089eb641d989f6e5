// capi_device.cu — extern "C" entry points of the device path (infmoe.h,
// "Device path" section).  Every call is exception-guarded.
#include <cstring>

#include "../host/status.hpp"
#include "../kernels/common.cuh"
#include "../kernels/expert_gemm.cuh"
#include "../kernels/kernels.cuh"
#include "infmoe.h"
#include "layer.hpp"

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

int infmoe_gate_softmax_topk(const void* x, int32_t dtype, int64_t N, int32_t d,
                             const float* wg, const float* bias, int32_t E, int32_t k,
                             int32_t* topk_idx, float* topk_w, int32_t* counts, void* stream) {
  return guarded([&] {
    require(x && wg && topk_idx && topk_w && counts, "gate: NULL pointer");
    launch_gate_softmax(x, dtype, N, d, wg, bias, E, k, topk_idx, topk_w, counts,
                        as_stream(stream));
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

int infmoe_combine(const void* y_perm, int32_t dtype, const int32_t* inv, const float* topk_w,
                   int64_t N, int32_t k, int32_t d, void* y, void* stream) {
  return guarded([&] {
    require(y_perm && inv && topk_w && y, "combine: NULL pointer");
    launch_combine(y_perm, dtype, inv, topk_w, N, k, d, y, as_stream(stream));
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

int infmoe_layer_forward(infmoe_layer* layer, const void* x, int64_t N, void* y,
                         infmoe_forward_out* out, void* stream) {
  return guarded([&] {
    require(layer && layer->impl && x && y, "layer_forward: NULL argument");
    layer->impl->forward(x, N, y, out, as_stream(stream));
  });
}

int infmoe_layer_set_host_weights(infmoe_layer* layer, const void* w_in, const void* w_out) {
  return guarded([&] {
    require(layer && layer->impl, "set_host_weights: NULL layer");
    layer->impl->set_host_weights(w_in, w_out);
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
