// stream_bw.cu — dev microbenchmark: how fast can 148 persistent CTAs stream
// an expert weight matrix into shared memory, by access pattern?  No MMA; the
// consumer releases each stage as soon as it lands.  Mirrors the grouped
// GEMM's producer (4-6 stage mbarrier ring, 1 CTA per SM).
//   mode 0: 2D TMA boxes of 128 rows x 128 B (the GEMM's current W tile)
//   mode 1: 2D TMA, two 128-B boxes per row back to back (256 B per row/stage)
//   mode 2: 1D bulk copies of 16 KB contiguous (a pre-tiled weight layout)
//   mode 3: 2D TMA boxes 128 rows x 128 B with no L2 promotion
//   l2rows > 0: the tiles cycle over the first l2rows weight rows only (an
//   L2-resident working set): the L2 -> shared-memory TMA ceiling
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));     \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n));
}
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 "
      "bra W_%=;\n}" ::"r"(b),
      "r"(ph));
}
__device__ __forceinline__ void arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b));
}
__device__ __forceinline__ void tma2d(uint32_t dst, const void* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

constexpr int STAGES = 12;  // ring slots (mode 1 uses 6 slots of 32 KB)
constexpr uint32_t STAGE = 16384;

__global__ void __launch_bounds__(64, 1)
    stream_kernel(const __grid_constant__ CUtensorMap map, const uint8_t* base, int mode,
                  int tiles, int rows_total, int K, int nst_override) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const uint32_t sbase = (su32(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(su32(&full[s]), 1);
      mbar_init(su32(&empty[s]), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int kblocks = K / 64;  // 128-B K-blocks per row
  const int nst = nst_override > 0 ? nst_override : (mode == 1 ? STAGES / 2 : STAGES);
  const uint32_t sb = mode == 1 ? 2 * STAGE : STAGE;
  if (threadIdx.x == 0) {      // producer
    int stage = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int row0 = (t * 128) % rows_total;
      const int step = mode == 1 ? 2 : 1;
      for (int kb = 0; kb < kblocks; kb += step) {
        wait(su32(&empty[stage]), ph ^ 1);
        const uint32_t dst = sbase + stage * sb;
        if (mode == 0 || mode == 3) {
          expect_tx(su32(&full[stage]), 16384);
          tma2d(dst, &map, su32(&full[stage]), kb * 64, row0);
        } else if (mode == 1) {
          expect_tx(su32(&full[stage]), 32768);
          tma2d(dst, &map, su32(&full[stage]), kb * 64, row0);
          tma2d(dst + 16384, &map, su32(&full[stage]), (kb + 1) * 64, row0);
        } else {
          const size_t off = (size_t(row0) * K + size_t(kb) * 64 * 128) * 2;
          expect_tx(su32(&full[stage]), 16384);
          bulk1d(dst, base + off, 16384, su32(&full[stage]));
        }
        if (++stage == nst) { stage = 0; ph ^= 1; }
      }
    }
  } else if (threadIdx.x == 32) {  // consumer
    int stage = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int step = mode == 1 ? 2 : 1;
      for (int kb = 0; kb < kblocks; kb += step) {
        wait(su32(&full[stage]), ph);
        arrive(su32(&empty[stage]));
        if (++stage == nst) { stage = 0; ph ^= 1; }
      }
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

int main() {
  const int E = 32, f = 10240, d = 4096;
  const size_t rows = size_t(E) * f, bytes = rows * d * 2;
  uint8_t* w;
  CK(cudaMalloc(&w, bytes));
  CK(cudaMemset(w, 1, bytes));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = reinterpret_cast<EncFn>(fp);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          STAGES * STAGE + 1024));
  const int tiles = int(rows / 128);
  int runs[][3] = {{0, 0, 0}, {1, 0, 0}, {2, 0, 0}, {3, 0, 0}, {0, 3, 0}, {0, 4, 0}, {0, 5, 0},
                   {0, 6, 0}, {0, 8, 0}, {0, 10, 0}, {0, 6, 2048}, {0, 8, 2048}, {0, 12, 2048},
                   {1, 6, 2048}, {0, 12, 4096}, {0, 12, 8192}};
  for (auto& rr : runs) {
    const int mode = rr[0], nst = rr[1];
    const int l2rows = rr[2];
    CUtensorMap m;
    memset(&m, 0, sizeof(m));
    cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(rows)};
    cuuint64_t str[1] = {cuuint64_t(d) * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B,
        mode == 3 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a);
      stream_kernel<<<sms, 64, STAGES * STAGE + 1024>>>(m, w, mode, tiles,
                                                         l2rows ? l2rows : int(rows), d, nst);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    CK(cudaGetLastError());
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double gbs = bytes / (best * 1e-3) / 1e9;
    printf("mode %d stages %d l2rows %d (%s): %.3f ms  %.1f GB/s  %.1f B/clk/SM at %d MHz\n", mode,
           nst, l2rows, l2rows ? "L2-resident" : "HBM", best, gbs,
           gbs * 1e9 / (double(clk_khz) * 1e3) / sms, clk_khz / 1000);
  }
  return 0;
}
