/*
 * oracle_ffn.c — CPU restatement of one expert's FFN (TEST INFRASTRUCTURE and
 * the CPU baseline arm; see oracle.h).  y = GeLU_erf(x . W_in^T) . W_out^T
 * with fp64 accumulation over fp32 (bf16-exact) inputs, H rounded to bf16
 * when round_h (the device path stores H in bf16).  Parity of the device FFN
 * against this is tolerance-checked, so the fp64 summation order is free:
 * eight interleaved partial sums let the compiler vectorise, and OpenMP
 * spreads (row, column) pairs over all host cores.  Compiled in its own
 * translation unit with -O3 -mavx2 (no effect on the bit-exact LSH code).
 */
#include <math.h>
#include <stdlib.h>

#include "oracle.h"

static double dot8(const float* a, const float* b, int n) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = 0;
  for (; c + 8 <= n; c += 8)
    for (int i = 0; i < 8; ++i) acc[i] += (double)a[c + i] * (double)b[c + i];
  double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  for (; c < n; ++c) s += (double)a[c] * (double)b[c];
  return s;
}

static double dot8d(const double* a, const float* b, int n) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int c = 0;
  for (; c + 8 <= n; c += 8)
    for (int i = 0; i < 8; ++i) acc[i] += a[c + i] * (double)b[c + i];
  double s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  for (; c < n; ++c) s += a[c] * (double)b[c];
  return s;
}

void or_expert_ffn(const float* x, uint64_t n, int d, int f, const float* w_in,
                   const float* w_out, int round_h, float* y) {
  if (n == 0) return;
  double* h = (double*)malloc(sizeof(double) * (size_t)n * (size_t)f);
  /* weight rows outermost: each weight row streams from memory once and meets
   * every token row while it is in cache */
#pragma omp parallel for schedule(static)
  for (int j = 0; j < f; ++j)
    for (uint64_t r = 0; r < n; ++r) {
      const double g = or_gelu(dot8(x + r * (uint64_t)d, w_in + (uint64_t)j * (uint64_t)d, d));
      h[r * (uint64_t)f + j] = round_h ? (double)or_bf16_to_f32(or_f32_to_bf16((float)g)) : g;
    }
#pragma omp parallel for schedule(static)
  for (int c = 0; c < d; ++c)
    for (uint64_t r = 0; r < n; ++r)
      y[r * (uint64_t)d + c] = (float)dot8d(h + r * (uint64_t)f, w_out + (uint64_t)c * (uint64_t)f, f);
  free(h);
}
