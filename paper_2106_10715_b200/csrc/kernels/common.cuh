// common.cuh — shared device helpers for the sm_100a kernels of libinfmoe.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "../host/status.hpp"

#define INFMOE_CUDA(call)                                                            \
  do {                                                                               \
    cudaError_t err__ = (call);                                                      \
    if (err__ != cudaSuccess)                                                        \
      ::infmoe::fail(::infmoe::kRuntime, std::string(#call) + ": " +                 \
                                             cudaGetErrorString(err__));            \
  } while (0)

#define INFMOE_LAUNCH_CHECK() INFMOE_CUDA(cudaGetLastError())

namespace infmoe {

constexpr int kDtypeBf16 = 0;
constexpr int kDtypeF32 = 1;

inline size_t dtype_bytes(int dtype) { return dtype == kDtypeBf16 ? 2 : 4; }

__host__ __device__ inline uint64_t dev_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ float load_as_f32(const __nv_bfloat16* p, size_t i) {
  return __bfloat162float(p[i]);
}
__device__ __forceinline__ float load_as_f32(const float* p, size_t i) { return p[i]; }

inline int device_sm_count() {
  int dev = 0, n = 0;
  INFMOE_CUDA(cudaGetDevice(&dev));
  INFMOE_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return n;
}

// Opt a kernel in to `bytes` of dynamic shared memory on the CURRENT device.
// The attribute is per (device, function), so the record is keyed on both and
// only ever grows; a mutex makes concurrent launchers (EP ranks as threads,
// layers on several GPUs) safe.  Cheap enough to call on every launch.
inline void ensure_dyn_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> configured;
  int dev = 0;
  INFMOE_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = configured[{dev, func}];
  if (bytes > cur) {
    INFMOE_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(bytes)));
    cur = bytes;
  }
}

}  // namespace infmoe
