// Dependent-chain latency microbenchmark (dev tool): cycles per step of
// dadd, dmul+dadd (separate roundings), dfma and ffma chains on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
  double x = a, y = b;
  float fx = (float)a, fy = (float)b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, __dmul_rn(y, (double)i));
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, y, a);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) fx = __fmaf_rn(fx, fy, (float)b);
  long long t4 = clock64();
  out[threadIdx.x] = x + fx;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 64);
  int n = 1 << 16;
  k<<<1, 32>>>(o, c, n, 1.0000001, 1e-9); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n, 1.0000001, 1e-9); cudaDeviceSynchronize();
  printf("cycles/step: dadd %.2f  dmul+dadd %.2f  dfma %.2f  ffma %.2f\n", c[0] / double(n),
         c[1] / double(n), c[2] / double(n), c[3] / double(n));
  return 0;
}
