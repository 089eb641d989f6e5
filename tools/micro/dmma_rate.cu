// dmma_rate.cu — dev micro: fp64 tensor-core (DMMA m16n8k4) throughput and
// dependent-chain latency on this GPU, vs the fp64 DFMA pipe.
#include <cstdio>

template <int CHAINS>
__global__ void dmma_k(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 1.0 - a0, b0 = 0.5 + a0;
  double d[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
          : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
          : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_k(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
  const double m = 1.0000001, a = 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], m, a);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int iters = 20000;
  // latency: one warp, one chain
  dmma_k<1><<<1, 32>>>(out, 1000);
  cudaEventRecord(a);
  dmma_k<1><<<1, 32>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("DMMA m16n8k4 dependent chain: %.1f ns per mma (%.1f cycles at %d MHz)\n",
         ms * 1e6 / iters, ms * 1e6 / iters * clk / 1e6, clk / 1000);
  // throughput: 8 warps per SM x 4 chains
  for (int warps : {4, 8, 16}) {
    dmma_k<4><<<sms, 32 * warps>>>(out, 100);
    cudaEventRecord(a);
    dmma_k<4><<<sms, 32 * warps>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double flop = 2.0 * 16 * 8 * 4 * 4 * double(iters) * warps * sms;
    printf("DMMA %2d warps/SM: %.1f TFLOP/s fp64\n", warps, flop / (ms * 1e-3) / 1e12);
  }
  dfma_k<<<sms, 256>>>(out, 100);
  cudaEventRecord(a);
  dfma_k<<<sms * 4, 256>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("DFMA pipe: %.1f TFLOP/s fp64\n", 2.0 * 8 * double(iters) * 256 * sms * 4 / (ms * 1e-3) / 1e12);
  return 0;
}
