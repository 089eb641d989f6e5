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


// ---------------------------------------------------------------- test hooks
// n_ctas CTAs, each holding `smem` bytes of shared memory (so one per SM),
// spin until *release != 0 or timeout_ns elapsed (globaltimer); *timed_out is
// set if any CTA gave up.  Used to take SMs away from a concurrent launch.
__global__ void occupy_kernel(const volatile int32_t* release, uint64_t timeout_ns,
                              int32_t* timed_out) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x != 0) return;
  pad[0] = 0;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*release == 0) {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicExch(timed_out, 1);
      return;
    }
  }
}
// the same spinner in clusters of two: it takes whole TPCs, so the SMs left
// free come in pairs a cta_group::2 kernel can use
__global__ void __cluster_dims__(2, 1, 1)
    occupy_pair_kernel(const volatile int32_t* release, uint64_t timeout_ns, int32_t* timed_out) {
  extern __shared__ uint8_t pad2[];
  if (threadIdx.x != 0) return;
  pad2[0] = 0;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*release == 0) {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      atomicExch(timed_out, 1);
      return;
    }
  }
}
__global__ void set_flag_kernel(int32_t* flag) { *reinterpret_cast<volatile int32_t*>(flag) = 1; }

void launch_occupy(int n_ctas, size_t smem, const int32_t* release, uint64_t timeout_ns,
                   int32_t* timed_out, cudaStream_t s) {
  if (n_ctas % 2 == 0) {  // whole TPCs
    ensure_dyn_smem(reinterpret_cast<const void*>(occupy_pair_kernel), smem);
    occupy_pair_kernel<<<n_ctas, 32, smem, s>>>(release, timeout_ns, timed_out);
  } else {
    ensure_dyn_smem(reinterpret_cast<const void*>(occupy_kernel), smem);
    occupy_kernel<<<n_ctas, 32, smem, s>>>(release, timeout_ns, timed_out);
  }
  INFMOE_LAUNCH_CHECK();
}
void launch_set_flag(int32_t* flag, cudaStream_t s) {
  set_flag_kernel<<<1, 1, 0, s>>>(flag);
  INFMOE_LAUNCH_CHECK();
}

}  // namespace infmoe
