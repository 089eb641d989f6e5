/*
 * cpu_ffn.c — the CPU BASELINE's expert FFN (TEST / BASELINE INFRASTRUCTURE,
 * never the product; only bench.py's cpu_baseline leg and --impl reference
 * call it).  The reference (moesim) has no FFN at all, so the
 * CPU arm runs this port of the same arithmetic the GPU computes:
 *
 *   h = bf16( GeLU_erf( x . W_in^T ) )        fp32 accumulation
 *   y = x_h . W_out^T                          fp32 accumulation (caller rounds)
 *
 * over bf16 token rows and bf16 weights read in place (no conversion pass
 * outside the timed region).  The contraction is C[n, m] = A[n, K] . B[m, K]^T
 * blocked 4 weight rows x 4 token rows (16 accumulators); with AVX512-BF16 the
 * inner step is vdpbf16ps (32 bf16 products per instruction into 16 fp32
 * lanes), else an fp32 FMA loop over bf16->fp32 conversions (auto-vectorised).
 * OpenMP spreads weight-row blocks over all host cores.  Parity is NOT checked
 * against this (oracle_ffn.c's fp64 FFN is the parity oracle); bench.py reports
 * its error against the GPU next to its speed.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#if defined(__x86_64__)
#include <immintrin.h>
#define CPU_FFN_X86 1
#endif

static inline float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

/* ---- generic path: C[r][j] = sum_k A[r][k] * B[j][k], fp32 ------------- */
static void block_generic(const uint16_t* A, const uint16_t* B, int nr, int nj, int K,
                          float* acc /* [4][4] */) {
  float a32[4][64], b32[4][64];
  for (int i = 0; i < 16; ++i) acc[i] = 0.0f;
  for (int k0 = 0; k0 < K; k0 += 64) {
    const int kk = K - k0 < 64 ? K - k0 : 64;
    for (int r = 0; r < nr; ++r)
      for (int k = 0; k < kk; ++k) a32[r][k] = bf2f(A[(size_t)r * K + k0 + k]);
    for (int j = 0; j < nj; ++j)
      for (int k = 0; k < kk; ++k) b32[j][k] = bf2f(B[(size_t)j * K + k0 + k]);
    for (int r = 0; r < nr; ++r)
      for (int j = 0; j < nj; ++j) {
        float s = 0.0f;
#pragma omp simd reduction(+ : s)
        for (int k = 0; k < kk; ++k) s += a32[r][k] * b32[j][k];
        acc[r * 4 + j] += s;
      }
  }
}

#ifdef CPU_FFN_X86
/* 4 token rows x 4 weight rows over k in [k0, k1): partial sums kept as
 * vectors in acc (16 x 16 lanes, caller-owned, reduced once at the end) */
__attribute__((target("avx512f,avx512bf16")))
static void block_bf16dp(const uint16_t* A, const uint16_t* B, int nr, int nj, int K, int k0,
                         int k1, __m512* acc) {
  if (nr == 4 && nj == 4) {
    __m512 c00 = acc[0], c01 = acc[1], c02 = acc[2], c03 = acc[3];
    __m512 c10 = acc[4], c11 = acc[5], c12 = acc[6], c13 = acc[7];
    __m512 c20 = acc[8], c21 = acc[9], c22 = acc[10], c23 = acc[11];
    __m512 c30 = acc[12], c31 = acc[13], c32 = acc[14], c33 = acc[15];
    const uint16_t *a0 = A, *a1 = A + K, *a2 = A + 2 * (size_t)K, *a3 = A + 3 * (size_t)K;
    const uint16_t *b0 = B, *b1 = B + K, *b2 = B + 2 * (size_t)K, *b3 = B + 3 * (size_t)K;
    for (int k = k0; k < k1; k += 32) {
      const __m512bh w0 = (__m512bh)_mm512_loadu_si512((const void*)(b0 + k));
      const __m512bh w1 = (__m512bh)_mm512_loadu_si512((const void*)(b1 + k));
      const __m512bh w2 = (__m512bh)_mm512_loadu_si512((const void*)(b2 + k));
      const __m512bh w3 = (__m512bh)_mm512_loadu_si512((const void*)(b3 + k));
      __m512bh x = (__m512bh)_mm512_loadu_si512((const void*)(a0 + k));
      c00 = _mm512_dpbf16_ps(c00, x, w0); c01 = _mm512_dpbf16_ps(c01, x, w1);
      c02 = _mm512_dpbf16_ps(c02, x, w2); c03 = _mm512_dpbf16_ps(c03, x, w3);
      x = (__m512bh)_mm512_loadu_si512((const void*)(a1 + k));
      c10 = _mm512_dpbf16_ps(c10, x, w0); c11 = _mm512_dpbf16_ps(c11, x, w1);
      c12 = _mm512_dpbf16_ps(c12, x, w2); c13 = _mm512_dpbf16_ps(c13, x, w3);
      x = (__m512bh)_mm512_loadu_si512((const void*)(a2 + k));
      c20 = _mm512_dpbf16_ps(c20, x, w0); c21 = _mm512_dpbf16_ps(c21, x, w1);
      c22 = _mm512_dpbf16_ps(c22, x, w2); c23 = _mm512_dpbf16_ps(c23, x, w3);
      x = (__m512bh)_mm512_loadu_si512((const void*)(a3 + k));
      c30 = _mm512_dpbf16_ps(c30, x, w0); c31 = _mm512_dpbf16_ps(c31, x, w1);
      c32 = _mm512_dpbf16_ps(c32, x, w2); c33 = _mm512_dpbf16_ps(c33, x, w3);
    }
    acc[0] = c00; acc[1] = c01; acc[2] = c02; acc[3] = c03;
    acc[4] = c10; acc[5] = c11; acc[6] = c12; acc[7] = c13;
    acc[8] = c20; acc[9] = c21; acc[10] = c22; acc[11] = c23;
    acc[12] = c30; acc[13] = c31; acc[14] = c32; acc[15] = c33;
    return;
  }
  for (int r = 0; r < nr; ++r)
    for (int j = 0; j < nj; ++j) {
      __m512 c = acc[r * 4 + j];
      for (int k = k0; k < k1; k += 32)
        c = _mm512_dpbf16_ps(
            c, (__m512bh)_mm512_loadu_si512((const void*)(A + (size_t)r * K + k)),
            (__m512bh)_mm512_loadu_si512((const void*)(B + (size_t)j * K + k)));
      acc[r * 4 + j] = c;
    }
}
__attribute__((target("avx512f,avx512bf16")))
static void zero_acc(__m512* acc, int n) {
  for (int i = 0; i < n; ++i) acc[i] = _mm512_setzero_ps();
}
__attribute__((target("avx512f,avx512bf16")))
static float reduce_acc(const __m512* acc) { return _mm512_reduce_add_ps(*acc); }
#endif

static int use_bf16dp(int K) {
#ifdef CPU_FFN_X86
  static int have = -1;
  if (have < 0) {
    __builtin_cpu_init();
    have = __builtin_cpu_supports("avx512bf16") ? 1 : 0;
    const char* e = getenv("ORACLE_CPU_FFN_GENERIC");
    if (e && atoi(e)) have = 0;
  }
  return have && K % 32 == 0;
#else
  (void)K;
  return 0;
#endif
}

/* C = epi(A . B^T): A [n, K] bf16 rows, B [m, K] bf16 rows.
 * epi 0: C_f32[n][m] = acc; epi 1: C_bf16[n][m] = bf16(gelu_erf(acc)).
 * A thread owns a block of 4 weight rows and walks K in chunks of kKc
 * (4 x kKc x 2 B of weights stay in L1) across every token block, keeping each
 * block's 16 vector partial sums in a per-thread buffer. */
static void store_epi(int epi, void* C, int m, int r0, int j0, int nr, int nj,
                      const float* acc) {
  for (int r = 0; r < nr; ++r)
    for (int j = 0; j < nj; ++j) {
      const float v = acc[r * 4 + j];
      const size_t o = (size_t)(r0 + r) * m + j0 + j;
      if (epi == 1) {
        const float g = 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
        ((uint16_t*)C)[o] = f2bf(g);
      } else {
        ((float*)C)[o] = v;
      }
    }
}

static void gemm_bt(const uint16_t* A, int n, const uint16_t* B, int m, int K, int epi,
                    void* C) {
  const int dp = use_bf16dp(K);
  const int nrb = (n + 3) / 4;
#pragma omp parallel
  {
#ifdef CPU_FFN_X86
    __m512* vacc = dp ? (__m512*)aligned_alloc(64, sizeof(__m512) * 16 * (size_t)nrb) : NULL;
#endif
#pragma omp for schedule(dynamic, 1)
    for (int j0 = 0; j0 < m; j0 += 4) {
      const int nj = m - j0 < 4 ? m - j0 : 4;
      float acc[16];
#ifdef CPU_FFN_X86
      if (dp) {
        enum { kKc = 1024 };
        zero_acc(vacc, 16 * nrb);
        for (int k0 = 0; k0 < K; k0 += kKc) {
          const int k1 = K - k0 < kKc ? K : k0 + kKc;
          for (int rb = 0; rb < nrb; ++rb) {
            const int r0 = rb * 4, nr = n - r0 < 4 ? n - r0 : 4;
            block_bf16dp(A + (size_t)r0 * K, B + (size_t)j0 * K, nr, nj, K, k0, k1,
                         vacc + 16 * (size_t)rb);
          }
        }
        for (int rb = 0; rb < nrb; ++rb) {
          const int r0 = rb * 4, nr = n - r0 < 4 ? n - r0 : 4;
          for (int i = 0; i < 16; ++i) acc[i] = reduce_acc(vacc + 16 * (size_t)rb + i);
          store_epi(epi, C, m, r0, j0, nr, nj, acc);
        }
        continue;
      }
#endif
      for (int r0 = 0; r0 < n; r0 += 4) {
        const int nr = n - r0 < 4 ? n - r0 : 4;
        block_generic(A + (size_t)r0 * K, B + (size_t)j0 * K, nr, nj, K, acc);
        store_epi(epi, C, m, r0, j0, nr, nj, acc);
      }
    }
#ifdef CPU_FFN_X86
    free(vacc);
#endif
  }
}

void or_expert_ffn_bf16(const uint16_t* x, uint64_t n, int d, int f, const uint16_t* w_in,
                        const uint16_t* w_out, uint16_t* h, float* y) {
  if (n == 0) return;
  gemm_bt(x, (int)n, w_in, f, d, 1, h);
  gemm_bt(h, (int)n, w_out, d, f, 0, y);
}

int or_cpu_ffn_isa(void) { return use_bf16dp(32) ? 1 : 0; }
