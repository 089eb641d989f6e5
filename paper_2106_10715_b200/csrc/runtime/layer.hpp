// layer.hpp — state owned by one infmoe_layer handle (device buffers sized for
// max_tokens, K+1 weight slots, copy stream, per-position events).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "infmoe.h"

namespace infmoe {

struct Layer {
  explicit Layer(const infmoe_layer_desc& d);
  ~Layer();
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;

  void forward(const void* x, int64_t N, void* y, infmoe_forward_out* out, cudaStream_t s);
  void set_host_weights(const void* w_in, const void* w_out);

 private:
  void route(const void* x, int64_t N, cudaStream_t s);
  void ffn(const int32_t* experts, const int32_t* slots, int n, const void* w_in,
           const void* w_out, int n_w_slots, int64_t rows, int max_ctas, int rows_hint,
           cudaStream_t s);

  infmoe_layer_desc desc;
  size_t esz = 2;
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
  uint8_t* xp = nullptr;
  uint8_t* hbuf = nullptr;
  uint8_t* yp = nullptr;
  double* proj = nullptr;
  float* gate_w = nullptr;
  float* gate_b = nullptr;
  int32_t* counts_host = nullptr;
  // offload executor
  size_t expert_in_bytes = 0;  // = bytes of W_in = bytes of W_out of one expert
  int n_slots = 0;
  uint8_t* slot_in = nullptr;
  uint8_t* slot_out = nullptr;
  const uint8_t* host_in = nullptr;
  const uint8_t* host_out = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> load_done, compute_done;
  std::vector<cudaEvent_t> t_load0, t_load1, t_comp0, t_comp1;
  cudaEvent_t t_start = nullptr;
};

}  // namespace infmoe
