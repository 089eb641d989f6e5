// gather4.cu — dev check: does cp.async.bulk.tensor.2d ... tile::gather4 place
// 4 indexed rows in shared memory exactly as a 4-row tile box of the same
// rows would (same 128-B swizzle)?  Prints MATCH / MISMATCH.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}

__global__ void k(const __grid_constant__ CUtensorMap tile_map, const __grid_constant__ CUtensorMap g4_map,
                  const int* rows, uint8_t* out_tile, uint8_t* out_g4) {
  __shared__ __align__(1024) uint8_t a[8 * 128];
  __shared__ __align__(1024) uint8_t b[8 * 128];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(2048));
    // two regular 4-row boxes: rows[0]..rows[0]+3 and rows[4]..rows[4]+3 (consecutive)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(su32(a)), "l"(&tile_map), "r"(0), "r"(rows[0]), "r"(su32(&bar)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(su32(a + 512)), "l"(&tile_map), "r"(0), "r"(rows[4]), "r"(su32(&bar)) : "memory");
    // the same 8 rows by index, 4 at a time
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(su32(b)), "l"(&g4_map), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(su32(&bar)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(su32(b + 512)), "l"(&g4_map), "r"(0), "r"(rows[4]), "r"(rows[5]), "r"(rows[6]), "r"(rows[7]), "r"(su32(&bar)) : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(su32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    out_tile[i] = a[i];
    out_g4[i] = b[i];
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

int main() {
  const int R = 64, D = 512;  // bf16 [R, D]
  std::vector<uint16_t> h(size_t(R) * D);
  for (size_t i = 0; i < h.size(); ++i) h[i] = uint16_t(i * 2654435761u >> 7);
  void* dx;
  cudaMalloc(&dx, h.size() * 2);
  cudaMemcpy(dx, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = reinterpret_cast<EncFn>(fp);
  cuuint64_t dims[2] = {cuuint64_t(D), cuuint64_t(R)};
  cuuint64_t str[1] = {cuuint64_t(D) * 2};
  cuuint32_t box_t[2] = {64, 4}, box_g[2] = {64, 1}, es[2] = {1, 1};
  CUtensorMap mt, mg;
  memset(&mt, 0, sizeof(mt));
  memset(&mg, 0, sizeof(mg));
  CUresult r1 = enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, str, box_t, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims, str, box_g, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode tile=%d gather=%d\n", int(r1), int(r2));
  int hr[8] = {8, 9, 10, 11, 12, 13, 14, 15};
  int* dr;
  cudaMalloc(&dr, sizeof(hr));
  cudaMemcpy(dr, hr, sizeof(hr), cudaMemcpyHostToDevice);
  uint8_t *ot, *og;
  cudaMalloc(&ot, 1024);
  cudaMalloc(&og, 1024);
  int hrows[8];
  memcpy(hrows, hr, sizeof(hr));
  int* rows_dev = dr;
  (void)rows_dev;
  // rows are passed through a device array read by thread 0
  k<<<1, 128>>>(mt, mg, dr, ot, og);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint8_t> a(1024), b(1024);
  cudaMemcpy(a.data(), ot, 1024, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), og, 1024, cudaMemcpyDeviceToHost);
  printf("%s\n", a == b ? "MATCH" : "MISMATCH");
  // also: permuted indices must land row by row
  return 0;
}
