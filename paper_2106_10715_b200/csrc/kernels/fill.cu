// fill.cu — synthetic-input generator (counter hash; bit-identical to
// oracle.c or_fill_uniform_* so CPU and GPU consume the same inputs).
//   h = splitmix64(seed ^ splitmix64(i)), u = (h >> 40) * 2^-24,
//   v = (2u - 1) * scale   (uniform, variance scale^2 / 3), rounded RNE to dtype.
#include "common.cuh"
#include "kernels.cuh"

namespace infmoe {

template <typename T>
__global__ void fill_uniform_kernel(T* out, uint64_t n, uint64_t seed, float scale) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = dev_mix64(seed ^ dev_mix64(i));
    const float u = float(h >> 40) * 5.9604644775390625e-8f;
    const float v = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
    if constexpr (sizeof(T) == 2) out[i] = __float2bfloat16_rn(v);
    else out[i] = v;
  }
}

void launch_fill_uniform(void* out, int dtype, uint64_t n, uint64_t seed, float scale,
                         cudaStream_t stream) {
  if (n == 0) return;
  const int threads = 256;
  const uint64_t want = (n + threads - 1) / threads;
  const int blocks = int(std::min<uint64_t>(want, uint64_t(device_sm_count()) * 16));
  if (dtype == kDtypeBf16)
    fill_uniform_kernel<<<blocks, threads, 0, stream>>>(reinterpret_cast<__nv_bfloat16*>(out),
                                                        n, seed, scale);
  else
    fill_uniform_kernel<<<blocks, threads, 0, stream>>>(reinterpret_cast<float*>(out), n, seed,
                                                        scale);
  INFMOE_LAUNCH_CHECK();
}

}  // namespace infmoe
