// expert_gemm.cu — N3/N4: per-expert FFN projections as one persistent,
// warp-specialised tcgen05 grouped GEMM for sm_100a.
//
//   out[r, n] = epi( sum_k A[r, k] * B[slot(r) * N + n, k] )
//
// A = token rows of the dispatched activations (x_perm for W_in, H for W_out),
// B = the expert weight in nn.Linear [out, in] (K-major) layout, one slot per
// resident expert.  The shape of one expert follows model_config.hpp:12-13
// (d_model x d_ff and d_ff x d_model); the FLOP count is expert_flops
// (model_config.hpp:77-80).
//
// Tiling: a tile is (group, 128 weight rows = output features,
// up to TOK token rows).  The weight tile is the MMA's M operand (M = 128) and
// the ragged token set is N (a multiple of 16, <= 256), so an expert with
// ~128-150 tokens is ONE tile column: every weight byte is read from HBM once
// and the token rows (x_perm or H) are re-read from L2 in 32-row boxes.  With
// ~128 tokens per expert the layer is weight-streaming bound (128 FLOP/B <
// 251 FLOP/B ridge), so the ring is sized for bytes of weight in flight.
// Roles: warp 0 TMA producer, warp 1 MMA issuer (one elected thread,
// accumulators in TMEM, 2 accumulator stages), warps 2-5 epilogue
// (tcgen05.ld -> GeLU -> bf16 -> global; TMEM lane = feature, column = token,
// so each warp store writes 32 consecutive features of one token row).
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "expert_gemm.cuh"
#include "tc_ptx.cuh"

namespace infmoe {
namespace gemm {

constexpr int TOK_BOX = 32;      // token rows per TMA box
constexpr uint32_t W_TILE = BM * ROW_BYTES;  // 16 KiB
constexpr int NUM_THREADS = 192;

template <int TOK, int STAGES>
struct Cfg {
  static constexpr uint32_t X_TILE = TOK * ROW_BYTES;
  static constexpr uint32_t STAGE_BYTES = W_TILE + X_TILE;
  static constexpr int ACC = 2;
  static constexpr int ACC_COLS = TOK <= 128 ? 128 : 256;  // TMEM columns per accumulator
  static constexpr int TMEM_COLS = ACC * ACC_COLS;
  static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static_assert(TMEM_COLS <= 512, "TMEM budget");
  static_assert(TOK % TOK_BOX == 0 && TOK <= 256, "token tile");
};

struct Params {
  int32_t N, K;
  int32_t n_groups;
  int32_t ld_out;
  int64_t a_rows;
  const int32_t* offsets;
  void* out;
  int32_t experts[kMaxGroups];
  int32_t slots[kMaxGroups];
};

// -------------------------------------------------------------- tile table
struct TileTable {
  int32_t n_groups;
  int32_t fblocks;  // N / BM (feature blocks of the output)
  int32_t tile_start[kMaxGroups + 1];
  int32_t chunks[kMaxGroups];
  int32_t row0[kMaxGroups];
  int32_t rows[kMaxGroups];
  int32_t slot[kMaxGroups];
};

struct Tile {
  int32_t row0;    // first token row
  int32_t ntok;    // valid token rows (<= TOK)
  int32_t w_row0;  // first weight row
  int32_t f0;      // first output column (feature)
};

template <int TOK>
__device__ __forceinline__ Tile decode(const TileTable& tt, int32_t t, int32_t& g_cursor,
                                       int32_t N) {
  while (t >= tt.tile_start[g_cursor + 1]) ++g_cursor;
  const int32_t g = g_cursor;
  const int32_t local = t - tt.tile_start[g];
  const int32_t tc = local % tt.chunks[g];  // token chunks fastest: neighbours
  const int32_t fb = local / tt.chunks[g];  // share the same weight tile in L2
  Tile r;
  r.row0 = tt.row0[g] + tc * TOK;
  r.ntok = min(TOK, tt.rows[g] - tc * TOK);
  r.w_row0 = tt.slot[g] * N + fb * BM;
  r.f0 = fb * BM;
  return r;
}

// ------------------------------------------------------------------ kernel
template <bool kTF32, bool kGelu, int TOK, int STAGES>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmap_x,
                        const __grid_constant__ CUtensorMap tmap_w, const Params p) {
  using C = Cfg<TOK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ TileTable tt;
  __shared__ uint32_t tmem_base_slot;

  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SW128 atoms need 1 KiB alignment
  const uint32_t bar_base = base + STAGES * C::STAGE_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  auto accf_bar = [&](int a) { return bar_base + 8u * (2 * STAGES + a); };
  auto acce_bar = [&](int a) { return bar_base + 8u * (2 * STAGES + C::ACC + a); };

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    tt.n_groups = p.n_groups;
    tt.fblocks = p.N / BM;
    int32_t acc = 0;
    for (int g = 0; g < p.n_groups; ++g) {
      const int e = p.experts[g];
      const int32_t r0 = p.offsets[e];
      const int32_t rn = p.offsets[e + 1] - r0;
      tt.row0[g] = r0;
      tt.rows[g] = rn;
      tt.slot[g] = p.slots[g];
      tt.chunks[g] = (rn + TOK - 1) / TOK;
      tt.tile_start[g] = acc;
      acc += tt.chunks[g] * tt.fblocks;
    }
    tt.tile_start[p.n_groups] = acc;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      mbar_init(accf_bar(a), 1);
      mbar_init(acce_bar(a), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_slot;
  const int32_t n_tiles = tt.tile_start[tt.n_groups];
  const int32_t bk_elems = ROW_BYTES / (kTF32 ? 4 : 2);
  const int32_t kblocks = p.K / bk_elems;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once
      const uint64_t pol_x = policy_evict_last();   // token rows: re-read per feature block
      int stage = 0;
      uint32_t phase = 0;
      int32_t gc = 0;
      for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const Tile tile = decode<TOK>(tt, t, gc, p.N);
        const int boxes = (tile.ntok + TOK_BOX - 1) / TOK_BOX;
        const uint32_t bytes = W_TILE + boxes * (TOK_BOX * ROW_BYTES);
        for (int32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sW = base + stage * C::STAGE_BYTES;
          const uint32_t sX = sW + W_TILE;
          mbar_expect_tx(full_bar(stage), bytes);
          tma_load_2d(sW, &tmap_w, full_bar(stage), kb * bk_elems, tile.w_row0, pol_w);
          for (int b = 0; b < boxes; ++b)
            tma_load_2d(sX + b * (TOK_BOX * ROW_BYTES), &tmap_x, full_bar(stage), kb * bk_elems,
                        tile.row0 + b * TOK_BOX, pol_x);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int32_t gc = 0;
    for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tile = decode<TOK>(tt, t, gc, p.N);
      const uint32_t n_mma = uint32_t((tile.ntok + 15) & ~15);  // UMMA N: multiple of 16
      const uint32_t idesc = make_idesc<kTF32>(n_mma);
      mbar_wait(acce_bar(acc), acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
      for (int32_t kb = 0; kb < kblocks; ++kb) {
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sW = base + stage * C::STAGE_BYTES;
          const uint64_t dw = sdesc(sW);
          const uint64_t dx = sdesc(sW + W_TILE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // 4 x 32 B of K per 128 B row
            mma<kTF32>(d_tmem, dw + 2 * kk, dx + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
          tc_commit(empty_bar(stage));  // smem slot free once these MMAs retire
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit(accf_bar(acc));  // accumulator ready for the epilogue
      __syncwarp();
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ================= epilogue (warps 2..5) =================
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 are visible to this warp
    int acc = 0;
    uint32_t acc_phase = 0;
    int32_t gc = 0;
    for (int32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tile = decode<TOK>(tt, t, gc, p.N);
      mbar_wait(accf_bar(acc), acc_phase);
      tc_fence_after();
      const int feat = tile.f0 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + acc * C::ACC_COLS;
      const int chunks = (tile.ntok + 31) / 32;
      for (int cc = 0; cc < chunks; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        const int nvalid = min(32, tile.ntok - cc * 32);
        const int64_t row = int64_t(tile.row0) + cc * 32;
        if constexpr (kTF32) {
          float* dst = reinterpret_cast<float*>(p.out) + row * p.ld_out + feat;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float v = __uint_as_float(r[i]);
            if constexpr (kGelu) v = gelu_erf(v);
            if (i < nvalid) dst[int64_t(i) * p.ld_out] = v;
          }
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + row * p.ld_out + feat;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float v = __uint_as_float(r[i]);
            if constexpr (kGelu) v = gelu_erf(v);
            if (i < nvalid) dst[int64_t(i) * p.ld_out] = __float2bfloat16_rn(v);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acce_bar(acc));
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(C::TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------ host helpers
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!fn) fail(kRuntime, "cuTensorMapEncodeTiled unavailable from the driver");
  return fn;
}

CUtensorMap make_tmap(const void* base, uint64_t rows, uint64_t cols, bool f32,
                      uint32_t box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const uint64_t esz = f32 ? 4 : 2;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esz};
  cuuint32_t box[2] = {uint32_t(ROW_BYTES / esz), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(kRuntime, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

template <bool kTF32, bool kGelu, int TOK, int STAGES>
void launch_impl(const GroupedGemmArgs& a, cudaStream_t stream) {
  using C = Cfg<TOK, STAGES>;
  auto kern = grouped_gemm_kernel<kTF32, kGelu, TOK, STAGES>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), size_t(int(C::SMEM_BYTES)));
  const CUtensorMap tx = make_tmap(a.a, uint64_t(std::max<int64_t>(a.a_rows, 1)), uint64_t(a.K),
                                   kTF32, TOK_BOX);
  const CUtensorMap tw = make_tmap(a.b, uint64_t(a.n_slots) * uint64_t(a.N), uint64_t(a.K),
                                   kTF32, BM);
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.N = a.N;
  p.K = a.K;
  p.n_groups = a.n_groups;
  p.ld_out = a.N;
  p.a_rows = a.a_rows;
  p.offsets = a.offsets;
  p.out = a.out;
  for (int g = 0; g < a.n_groups; ++g) {
    p.experts[g] = a.experts[g];
    p.slots[g] = a.slots[g];
  }
  int grid = device_sm_count();
  if (a.max_ctas > 0) grid = std::min(grid, a.max_ctas);
  kern<<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(tx, tw, p);
  INFMOE_LAUNCH_CHECK();
}

// Token-tile width: as wide as the largest expert when the host knows it (one
// weight read per expert), else 192 (the ~128 +- 20 tokens/expert of a
// balanced top-1 layer fit in one column).  Narrower tiles buy ring depth.
template <bool kTF32, bool kGelu>
void dispatch_tok(const GroupedGemmArgs& a, cudaStream_t s) {
  const int hint = a.max_rows_hint;
  if constexpr (kTF32) {
    launch_impl<kTF32, kGelu, 128, 4>(a, s);  // f32 tiles are twice as wide in bytes per K
  } else if (hint > 0 && hint <= 128) {
    launch_impl<kTF32, kGelu, 128, 6>(a, s);
  } else if (hint > 192) {
    launch_impl<kTF32, kGelu, 256, 4>(a, s);
  } else {
    launch_impl<kTF32, kGelu, 192, 5>(a, s);
  }
}


// =================================================================== fused
// Two-phase persistent kernel (see FusedFfnArgs).  Tiles are numbered phase-1
// first (expert-major), then phase 2, and claimed in that order from a global
// counter (claim_tile), so every phase-1 tile is owned by a running CTA before
// any phase-2 tile is handed out and the per-group waits always make progress,
// whether or not the whole grid is resident (concurrent kernels, MPS / green
// contexts, EP ranks sharing a GPU).  Dynamic claiming also balances the 2.5x
// longer phase-2 tiles across CTAs (greedy list scheduling).
struct FusedParams {
  int32_t d, f;
  int32_t n_groups;
  const int32_t* offsets;
  void* h;
  void* y;
  int32_t* done;
  const int32_t* perm;
  const float* topk_w;
  // expert-parallel return (PEER transport): output row r goes to rank
  // ret[r].x's y_back at row ret[r].y (peer_y = every rank's y_back)
  const int2* ret;
  void* peer_y[kMaxPeers];
  int64_t band_bytes;  // L2 budget for one band of token rows (0: one band per expert)
  int32_t pol_w, pol_x;  // L2 policies of the weight / token-row loads (policy_of; w -1: by chunks)
  int32_t experts[kMaxGroups];
  int32_t slots[kMaxGroups];
};

struct FusedTable {
  int32_t n_groups, fb1, fb2, total1;
  int32_t band1, band2;  // token chunks per band (phase 1 / phase 2), see band_split
  int32_t start1[kMaxGroups + 1];
  int32_t start2[kMaxGroups + 1];
  int32_t chunks[kMaxGroups];
  int32_t row0[kMaxGroups];
  int32_t rows[kMaxGroups];
  int32_t slot[kMaxGroups];
};

struct FTile {
  int32_t phase;  // 0: x . w_in -> GeLU -> h ; 1: h . w_out -> y
  int32_t g;
  int32_t row0, ntok, w_row0, f0;
};

// The tiles of one expert are walked in bands of `band` token chunks, the token
// chunk fastest inside a band.  The tiles in flight at once (one per CTA/pair)
// then share a few weight blocks, and the band's token rows (x_perm or H) stay
// L2-resident across all the expert's weight blocks: an expert with C chunks
// reads its weights ceil(C / band) times instead of once per wave and its token
// rows once instead of once per weight block.  band >= C (every balanced top-1
// layer: one chunk per expert) is the plain chunk-fastest order.
__device__ __forceinline__ void band_split(int32_t local, int32_t chunks, int32_t nfb,
                                           int32_t band, int32_t& tc, int32_t& fb) {
  band = min(band, chunks);
  const int32_t per = band * nfb;
  const int32_t b = local / per;
  const int32_t rem = local - b * per;
  const int32_t w = min(band, chunks - b * band);
  tc = b * band + rem % w;
  fb = rem / w;
}

__device__ __forceinline__ int32_t band_size(int64_t budget, int64_t chunk_bytes) {
  if (budget <= 0) return 1 << 30;
  const int64_t b = budget / chunk_bytes;
  return b < 1 ? 1 : (b > (1 << 30) ? (1 << 30) : int32_t(b));
}

// L2 budget of one band of token rows; INFMOE_FFN_BAND_MB overrides (0 = one band)
static int64_t ffn_band_bytes() {
  static const int64_t v = [] {
    const char* e = std::getenv("INFMOE_FFN_BAND_MB");
    return int64_t(e ? std::atoi(e) : 64) << 20;
  }();
  return v;
}

// L2 policies of the fused FFN's loads.  Default (-1): token rows evict_last
// (re-read once per weight block); weights evict_first when the expert is one
// token chunk (read once) and evict_normal when it spans several (re-read once
// per band, by the CTAs working on the band's other chunks).
// INFMOE_FFN_POLICY="wx" (digits of policy_of) forces both.
static void ffn_policies(int32_t& w, int32_t& x) {
  static const int v = [] {
    const char* e = std::getenv("INFMOE_FFN_POLICY");
    return e ? std::atoi(e) : -1;
  }();
  w = v < 0 ? -1 : (v / 10) % 3;
  x = v < 0 ? 2 : v % 10 % 3;
}

template <int TOK>
__device__ __forceinline__ FTile fdecode(const FusedTable& tt, int32_t t, int32_t& c1,
                                         int32_t& c2, int32_t d, int32_t f) {
  FTile r;
  if (t < tt.total1) {
    while (t >= tt.start1[c1 + 1]) ++c1;
    int32_t tc, fb;
    band_split(t - tt.start1[c1], tt.chunks[c1], tt.fb1, tt.band1, tc, fb);
    r.phase = 0;
    r.g = c1;
    r.row0 = tt.row0[c1] + tc * TOK;
    r.ntok = min(TOK, tt.rows[c1] - tc * TOK);
    r.w_row0 = tt.slot[c1] * f + fb * BM;
    r.f0 = fb * BM;
  } else {
    t -= tt.total1;
    while (t >= tt.start2[c2 + 1]) ++c2;
    int32_t tc, fb;
    band_split(t - tt.start2[c2], tt.chunks[c2], tt.fb2, tt.band2, tc, fb);
    r.phase = 1;
    r.g = c2;
    r.row0 = tt.row0[c2] + tc * TOK;
    r.ntok = min(TOK, tt.rows[c2] - tc * TOK);
    r.w_row0 = tt.slot[c2] * d + fb * BM;
    r.f0 = fb * BM;
  }
  return r;
}

__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int32_t* p, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- dynamic tile claim (forward progress without co-residency) ----------
// The persistent FFN kernels do not assume that their whole grid is resident.
// One thread per CTA (per pair) claims tiles in global order from a counter
// (done[n_groups]); all phase-1 tiles precede all phase-2 tiles in that order,
// so when a phase-2 tile of expert g is claimed every phase-1 tile of g is
// already owned by a RUNNING CTA whose pipeline drains without further claims.
// A CTA that is never scheduled simply claims nothing.  The claimed index is
// handed to the CTA's other roles through a small ring in shared memory
// (full/empty mbarriers); in the pair kernel the leader also writes it into
// the follower's ring over DSMEM.  The claim for tile i+1 is issued while
// tile i's loads are being issued, so its latency is hidden.
constexpr int kTileRing = 4;
__device__ __forceinline__ void mbar_wait_cl(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_s32(uint32_t caddr, int32_t v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(caddr), "r"(v) : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr)
               : "memory");
}
__device__ __forceinline__ int32_t claim_tile(int32_t* ctr, int32_t n_tiles) {
  const int32_t t = atomicAdd(ctr, 1);
  return t < n_tiles ? t : -1;
}
// consumer side: the next claimed tile (-1 = no more), slot released at once
struct TileRing {
  uint32_t full0, empty0;  // barrier arrays (8 B apart)
  volatile int32_t* idx;
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ int32_t next(int lane, uint32_t empty_addr_of_slot0) {
    mbar_wait_cl(full0 + 8u * slot, phase);
    const int32_t t = idx[slot];
    __syncwarp(__activemask());  // a whole role warp, or the single producer lane
    if (lane == 0) arrive_cluster(empty_addr_of_slot0 + 8u * slot);
    if (++slot == kTileRing) { slot = 0; phase ^= 1; }
    return t;
  }
};

template <int TOK, int STAGES>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    fused_ffn_kernel(const __grid_constant__ CUtensorMap tmap_x,
                     const __grid_constant__ CUtensorMap tmap_w1,
                     const __grid_constant__ CUtensorMap tmap_h,
                     const __grid_constant__ CUtensorMap tmap_w2, const FusedParams p) {
  using C = Cfg<TOK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ FusedTable tt;
  __shared__ uint32_t tmem_base_slot;
  __shared__ int32_t tile_idx[kTileRing];
  __shared__ __align__(8) uint64_t tile_bar[2 * kTileRing];  // full[kTileRing] | empty[kTileRing]

  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar_base = base + STAGES * C::STAGE_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  auto accf_bar = [&](int a) { return bar_base + 8u * (2 * STAGES + a); };
  auto acce_bar = [&](int a) { return bar_base + 8u * (2 * STAGES + C::ACC + a); };
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    tt.n_groups = p.n_groups;
    tt.fb1 = p.f / BM;
    tt.fb2 = p.d / BM;
    tt.band1 = band_size(p.band_bytes, int64_t(TOK) * p.d * 2);
    tt.band2 = band_size(p.band_bytes, int64_t(TOK) * p.f * 2);
    int32_t a1 = 0, a2 = 0;
    for (int g = 0; g < p.n_groups; ++g) {
      const int e = p.experts[g];
      const int32_t r0 = p.offsets[e];
      const int32_t rn = p.offsets[e + 1] - r0;
      tt.row0[g] = r0;
      tt.rows[g] = rn;
      tt.slot[g] = p.slots[g];
      tt.chunks[g] = (rn + TOK - 1) / TOK;
      tt.start1[g] = a1;
      tt.start2[g] = a2;
      a1 += tt.chunks[g] * tt.fb1;
      a2 += tt.chunks[g] * tt.fb2;
    }
    tt.start1[p.n_groups] = a1;
    tt.start2[p.n_groups] = a2;
    tt.total1 = a1;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      mbar_init(accf_bar(a), 1);
      mbar_init(acce_bar(a), 4);
    }
    for (int i = 0; i < kTileRing; ++i) {
      mbar_init(smem_u32(&tile_bar[i]), 1);              // the claiming producer
      mbar_init(smem_u32(&tile_bar[kTileRing + i]), 5);  // MMA warp + 4 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_slot;
  const int32_t n_tiles = tt.total1 + tt.start2[tt.n_groups];
  constexpr int32_t bk = ROW_BYTES / 2;  // bf16 elements per K-block
  int32_t* const tile_ctr = p.done + p.n_groups;
  TileRing ring{smem_u32(&tile_bar[0]), smem_u32(&tile_bar[kTileRing]), tile_idx};

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol_w1 = policy_of(p.pol_w < 0 ? 0 : p.pol_w);  // single-chunk experts
      const uint64_t pol_wn = policy_of(p.pol_w < 0 ? 1 : p.pol_w);  // multi-chunk experts
      const uint64_t pol_x = policy_of(p.pol_x);
      int stage = 0;
      uint32_t phase = 0;
      int32_t c1 = 0, c2 = 0, ready_g = -1;
      int ts = 0;
      uint32_t tph = 0;
      int32_t t = claim_tile(tile_ctr, n_tiles);
      for (;;) {
        mbar_wait_cl(ring.empty0 + 8u * ts, tph ^ 1);  // publish t to the MMA / epilogue warps
        tile_idx[ts] = t;
        mbar_arrive(ring.full0 + 8u * ts);
        if (++ts == kTileRing) { ts = 0; tph ^= 1; }
        if (t < 0) break;
        const int32_t t_next = claim_tile(tile_ctr, n_tiles);  // latency hidden by this tile
        const FTile tile = fdecode<TOK>(tt, t, c1, c2, p.d, p.f);
        if (tile.phase == 1 && tile.g != ready_g) {
          // every phase-1 tile of this group has published its H rows
          const int32_t target = tt.chunks[tile.g] * tt.fb1;
          uint32_t spins = 0;
          while (ld_acquire(p.done + tile.g) < target) {
            __nanosleep(64);
            if (++spins == (1u << 28)) __trap();  // a broken invariant must not hang the GPU
          }
          fence_proxy_async_global();  // generic-proxy H stores -> async-proxy TMA reads
          ready_g = tile.g;
        }
        const CUtensorMap* ta = tile.phase ? &tmap_h : &tmap_x;
        const CUtensorMap* tb = tile.phase ? &tmap_w2 : &tmap_w1;
        const uint64_t pol_w = tt.chunks[tile.g] > 1 ? pol_wn : pol_w1;
        const int32_t kblocks = (tile.phase ? p.f : p.d) / bk;
        const int boxes = (tile.ntok + TOK_BOX - 1) / TOK_BOX;
        const uint32_t bytes = W_TILE + boxes * (TOK_BOX * ROW_BYTES);
        for (int32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sW = base + stage * C::STAGE_BYTES;
          const uint32_t sX = sW + W_TILE;
          mbar_expect_tx(full_bar(stage), bytes);
          tma_load_2d(sW, tb, full_bar(stage), kb * bk, tile.w_row0, pol_w);
          for (int b = 0; b < boxes; ++b)
            tma_load_2d(sX + b * (TOK_BOX * ROW_BYTES), ta, full_bar(stage), kb * bk,
                        tile.row0 + b * TOK_BOX, pol_x);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        t = t_next;
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int32_t c1 = 0, c2 = 0;
    for (int32_t t = ring.next(lane, ring.empty0); t >= 0; t = ring.next(lane, ring.empty0)) {
      const FTile tile = fdecode<TOK>(tt, t, c1, c2, p.d, p.f);
      const uint32_t n_mma = uint32_t((tile.ntok + 15) & ~15);
      const uint32_t idesc = make_idesc<false>(n_mma);
      const int32_t kblocks = (tile.phase ? p.f : p.d) / bk;
      mbar_wait(acce_bar(acc), acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
      for (int32_t kb = 0; kb < kblocks; ++kb) {
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sW = base + stage * C::STAGE_BYTES;
          const uint64_t dw = sdesc(sW);
          const uint64_t dx = sdesc(sW + W_TILE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma<false>(d_tmem, dw + 2 * kk, dx + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
          tc_commit(empty_bar(stage));
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tc_commit(accf_bar(acc));
      __syncwarp();
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ================= epilogue (warps 2..5) =================
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int32_t c1 = 0, c2 = 0;
    for (int32_t t = ring.next(lane, ring.empty0); t >= 0; t = ring.next(lane, ring.empty0)) {
      const FTile tile = fdecode<TOK>(tt, t, c1, c2, p.d, p.f);
      mbar_wait(accf_bar(acc), acc_phase);
      tc_fence_after();
      const int feat = tile.f0 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + acc * C::ACC_COLS;
      const int chunks = (tile.ntok + 31) / 32;
      for (int cc = 0; cc < chunks; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        const int nvalid = min(32, tile.ntok - cc * 32);
        const int64_t row = int64_t(tile.row0) + cc * 32;
        if (tile.phase == 0) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.h) + row * p.f + feat;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nvalid)
              dst[int64_t(i) * p.f] = __float2bfloat16_rn(gelu_erf(__uint_as_float(r[i])));
        } else if (p.ret != nullptr) {
          // expert-parallel return: each row straight into its source rank's
          // y_back over NVLink (the combine then runs at the source)
          const int2 rt_l = lane < nvalid ? p.ret[row + lane] : make_int2(0, 0);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int rk = __shfl_sync(0xffffffffu, rt_l.x, i);
            const int pos = __shfl_sync(0xffffffffu, rt_l.y, i);
            if (i < nvalid)
              reinterpret_cast<__nv_bfloat16*>(p.peer_y[rk])[int64_t(pos) * p.d + feat] =
                  __float2bfloat16_rn(__uint_as_float(r[i]));
          }
        } else if (p.perm == nullptr) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.y) + row * p.d + feat;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nvalid) dst[int64_t(i) * p.d] = __float2bfloat16_rn(__uint_as_float(r[i]));
        } else {
          // fused top-1 combine: token of each row and its gate weight, broadcast
          const int tok_l = lane < nvalid ? p.perm[row + lane] : 0;
          const float w_l = lane < nvalid ? p.topk_w[tok_l] : 0.0f;
          __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(p.y);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int tok = __shfl_sync(0xffffffffu, tok_l, i);
            const float w = __shfl_sync(0xffffffffu, w_l, i);
            if (i < nvalid) {
              const float yb16 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(r[i])));
              yb[int64_t(tok) * p.d + feat] = __float2bfloat16_rn(fmaf(w, yb16, 0.0f));
            }
          }
        }
      }
      tc_fence_before();
      if (tile.phase == 0) {
        // all four epilogue warps stored this tile's H rows -> publish
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) {
          __threadfence();
          fence_proxy_async_global();
          red_release_add(p.done + tile.g, 1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(acce_bar(acc));
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (p.ret) __threadfence_system();  // results stored to peers are visible system-wide
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(C::TMEM_COLS)
                 : "memory");
  }
}

template <int TOK, int STAGES>
void fused_launch(const FusedFfnArgs& a, cudaStream_t stream) {
  using C = Cfg<TOK, STAGES>;
  auto kern = fused_ffn_kernel<TOK, STAGES>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), size_t(int(C::SMEM_BYTES)));
  const uint64_t rows = uint64_t(std::max<int64_t>(a.rows, 1));
  const CUtensorMap tx = make_tmap(a.x, rows, uint64_t(a.d_model), false, TOK_BOX);
  const CUtensorMap tw1 = make_tmap(a.w_in, uint64_t(a.n_slots) * a.d_ff, uint64_t(a.d_model),
                                    false, BM);
  const CUtensorMap th = make_tmap(a.h, rows, uint64_t(a.d_ff), false, TOK_BOX);
  const CUtensorMap tw2 = make_tmap(a.w_out, uint64_t(a.n_slots) * a.d_model, uint64_t(a.d_ff),
                                    false, BM);
  FusedParams p;
  std::memset(&p, 0, sizeof(p));
  p.d = a.d_model;
  p.f = a.d_ff;
  p.n_groups = a.n_groups;
  p.offsets = a.offsets;
  p.h = a.h;
  p.y = a.y;
  p.done = a.done;
  p.perm = a.perm;
  p.topk_w = a.topk_w;
  p.ret = a.ret;
  p.band_bytes = ffn_band_bytes();
  ffn_policies(p.pol_w, p.pol_x);
  for (int r = 0; r < a.n_peers && r < kMaxPeers; ++r) p.peer_y[r] = a.peer_y[r];
  for (int g = 0; g < a.n_groups; ++g) {
    p.experts[g] = a.experts[g];
    p.slots[g] = a.slots[g];
  }
  int grid = device_sm_count();
  if (a.max_ctas > 0) grid = std::min(grid, a.max_ctas);
  if (a.ev_begin) INFMOE_CUDA(cudaEventRecord(a.ev_begin, stream));
  INFMOE_CUDA(cudaMemsetAsync(a.done, 0, sizeof(int32_t) * size_t(a.n_groups + 1), stream));
  kern<<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(tx, tw1, th, tw2, p);
  INFMOE_LAUNCH_CHECK();
  if (a.ev_end) INFMOE_CUDA(cudaEventRecord(a.ev_end, stream));
}


// ============================================================ 2-SM variant
// Same two-phase schedule, but a tile is owned by a CTA PAIR (cluster of 2 on
// one TPC) issuing cta_group::2 MMAs with M = 256: each CTA streams its 128
// weight rows and HALF of the token rows, the leader (rank 0) issues the MMAs
// for both, and each CTA's TMEM receives its 128 x N accumulator.  Halving the
// token bytes per SM leaves room for a deeper weight ring (7 stages at
// TOK=192), which is what the weight-streaming bound needs.
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the leader CTA

// mbarrier wait that traps instead of hanging if a pair-protocol invariant is
// ever broken (a legitimate wait here lasts microseconds)
__device__ __forceinline__ void mbar_wait_guarded(uint32_t bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (!done && ++spins == (1u << 24)) __trap();
  } while (!done);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const void* tmap, uint32_t bar,
                                                 int32_t c_inner, int32_t c_outer,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar & kPeerMask), "r"(c_inner), "r"(c_outer),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// MMA completion -> arrive on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(bar),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void arrive_leader(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar & kPeerMask) : "memory");
}

template <int TOK, int STAGES>
struct PairCfg {
  static constexpr int XH = TOK / 2;                      // token rows per CTA
  static constexpr uint32_t X_TILE = XH * ROW_BYTES;
  static constexpr uint32_t STAGE_BYTES = W_TILE + X_TILE;
  static constexpr int ACC = 2;
  static constexpr int ACC_COLS = TOK <= 128 ? 128 : 256;
  static constexpr int TMEM_COLS = ACC * ACC_COLS;
  static constexpr uint32_t SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static_assert(XH % TOK_BOX == 0, "token half-tile must be whole TMA boxes");
  static_assert(TMEM_COLS <= 512, "TMEM budget");
};

template <int TOK>
__device__ __forceinline__ FTile pdecode(const FusedTable& tt, int32_t t, int32_t& c1, int32_t& c2,
                                         int32_t d, int32_t f, uint32_t rank) {
  // identical to fdecode with 256-row weight tiles; this CTA owns half 'rank'
  FTile r = fdecode<TOK>(tt, t, c1, c2, d, f);
  const int32_t fb = r.f0 / BM;  // fdecode's fb counts 256-row pair tiles here (fb1/fb2 halved)
  const int32_t n = r.phase ? d : f;
  r.f0 = fb * 2 * BM + int32_t(rank) * BM;
  r.w_row0 = tt.slot[r.g] * n + r.f0;
  return r;
}

template <int TOK, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    fused_ffn_pair_kernel(const __grid_constant__ CUtensorMap tmap_x,
                          const __grid_constant__ CUtensorMap tmap_w1,
                          const __grid_constant__ CUtensorMap tmap_h,
                          const __grid_constant__ CUtensorMap tmap_w2, const FusedParams p) {
  using C = PairCfg<TOK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ FusedTable tt;
  __shared__ uint32_t tmem_base_slot;
  __shared__ int32_t tile_idx[kTileRing];
  __shared__ __align__(8) uint64_t tile_bar[2 * kTileRing];  // full[kTileRing] | empty[kTileRing]

  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar_base = base + STAGES * C::STAGE_BYTES;
  auto full_bar = [&](int s) { return bar_base + 8u * s; };
  auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
  auto accf_bar = [&](int a) { return bar_base + 8u * (2 * STAGES + a); };
  auto acce_bar = [&](int a) { return bar_base + 8u * (2 * STAGES + C::ACC + a); };
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    tt.n_groups = p.n_groups;
    tt.fb1 = p.f / (2 * BM);
    tt.fb2 = p.d / (2 * BM);
    tt.band1 = band_size(p.band_bytes, int64_t(TOK) * p.d * 2);
    tt.band2 = band_size(p.band_bytes, int64_t(TOK) * p.f * 2);
    int32_t a1 = 0, a2 = 0;
    for (int g = 0; g < p.n_groups; ++g) {
      const int e = p.experts[g];
      const int32_t r0 = p.offsets[e];
      const int32_t rn = p.offsets[e + 1] - r0;
      tt.row0[g] = r0;
      tt.rows[g] = rn;
      tt.slot[g] = p.slots[g];
      tt.chunks[g] = (rn + TOK - 1) / TOK;
      tt.start1[g] = a1;
      tt.start2[g] = a2;
      a1 += tt.chunks[g] * tt.fb1;
      a2 += tt.chunks[g] * tt.fb2;
    }
    tt.start1[p.n_groups] = a1;
    tt.start2[p.n_groups] = a2;
    tt.total1 = a1;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);   // leader producer's expect_tx; both CTAs' bytes land here
      mbar_init(empty_bar(s), 1);  // one multicast MMA commit per stage
    }
    for (int a = 0; a < C::ACC; ++a) {
      mbar_init(accf_bar(a), 1);   // one multicast commit per tile
      mbar_init(acce_bar(a), 8);   // 4 epilogue warps x 2 CTAs (the leader's copy is used)
    }
    for (int i = 0; i < kTileRing; ++i) {
      // full: the leader's producer publishes into both CTAs' rings; empty (the
      // leader's copy is used): leader MMA + 4 leader epilogue warps + the
      // follower's producer + 4 follower epilogue warps
      mbar_init(smem_u32(&tile_bar[i]), 1);
      mbar_init(smem_u32(&tile_bar[kTileRing + i]), 10);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {  // same warp id in both CTAs, same destination slot
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peer barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_slot;
  const int32_t n_tiles = tt.total1 + tt.start2[tt.n_groups];
  constexpr int32_t bk = ROW_BYTES / 2;
  int32_t* const tile_ctr = p.done + p.n_groups;
  TileRing ring{smem_u32(&tile_bar[0]), smem_u32(&tile_bar[kTileRing]), tile_idx};
  const uint32_t leader_empty0 = map_rank(ring.empty0, 0);  // consumers release the leader's slot

  if (warp == 0) {
    // ================= TMA producer (both CTAs) =================
    if (lane == 0) {
      const uint64_t pol_w1 = policy_of(p.pol_w < 0 ? 0 : p.pol_w);  // single-chunk experts
      const uint64_t pol_wn = policy_of(p.pol_w < 0 ? 1 : p.pol_w);  // multi-chunk experts
      const uint64_t pol_x = policy_of(p.pol_x);
      int stage = 0;
      uint32_t phase = 0;
      int32_t c1 = 0, c2 = 0, ready_g = -1;
      int ts = 0;
      uint32_t tph = 0;
      const uint32_t peer_idx0 = map_rank(smem_u32(&tile_idx[0]), 1);
      const uint32_t peer_full0 = map_rank(ring.full0, 1);
      int32_t t = leader ? claim_tile(tile_ctr, n_tiles) : -1;
      for (;;) {
        int32_t t_next = -1;
        if (leader) {  // claim and publish to both CTAs
          mbar_wait_cl(ring.empty0 + 8u * ts, tph ^ 1);
          tile_idx[ts] = t;
          st_cluster_s32(peer_idx0 + 4u * ts, t);
          arrive_cluster(peer_full0 + 8u * ts);
          mbar_arrive(ring.full0 + 8u * ts);
          if (++ts == kTileRing) { ts = 0; tph ^= 1; }
          if (t < 0) break;
          t_next = claim_tile(tile_ctr, n_tiles);  // latency hidden by this tile
        } else {
          t = ring.next(0, leader_empty0);
          if (t < 0) break;
        }
        const FTile tile = pdecode<TOK>(tt, t, c1, c2, p.d, p.f, rank);
        if (tile.phase == 1 && tile.g != ready_g) {
          const int32_t target = tt.chunks[tile.g] * tt.fb1 * 2;  // both halves of every tile
          uint32_t spins = 0;
          while (ld_acquire(p.done + tile.g) < target) {
            __nanosleep(64);
            if (++spins == (1u << 28)) __trap();
          }
          fence_proxy_async_global();
          ready_g = tile.g;
        }
        const int32_t n_mma = (tile.ntok + 15) & ~15;
        const int32_t half = n_mma / 2;
        const int32_t xrow0 = tile.row0 + int32_t(rank) * half;
        const int boxes = (half + TOK_BOX - 1) / TOK_BOX;
        const uint32_t bytes_pair = 2u * (W_TILE + boxes * (TOK_BOX * ROW_BYTES));
        const CUtensorMap* ta = tile.phase ? &tmap_h : &tmap_x;
        const CUtensorMap* tb = tile.phase ? &tmap_w2 : &tmap_w1;
        const uint64_t pol_w = tt.chunks[tile.g] > 1 ? pol_wn : pol_w1;
        const int32_t kblocks = (tile.phase ? p.f : p.d) / bk;
        for (int32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait_guarded(empty_bar(stage), phase ^ 1);
          const uint32_t sW = base + stage * C::STAGE_BYTES;
          const uint32_t sX = sW + W_TILE;
          if (leader) mbar_expect_tx(full_bar(stage), bytes_pair);
          tma_load_2d_pair(sW, tb, full_bar(stage), kb * bk, tile.w_row0, pol_w);
          for (int b = 0; b < boxes; ++b)
            tma_load_2d_pair(sX + b * (TOK_BOX * ROW_BYTES), ta, full_bar(stage), kb * bk,
                             xrow0 + b * TOK_BOX, pol_x);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        t = t_next;
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA only) =================
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int32_t c1 = 0, c2 = 0;
      for (int32_t t = ring.next(lane, ring.empty0); t >= 0; t = ring.next(lane, ring.empty0)) {
        const FTile tile = pdecode<TOK>(tt, t, c1, c2, p.d, p.f, rank);
        const uint32_t n_mma = uint32_t((tile.ntok + 15) & ~15);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((n_mma >> 3) << 17) |
                               (uint32_t((2 * BM) >> 4) << 24);  // M = 256
        const int32_t kblocks = (tile.phase ? p.f : p.d) / bk;
        mbar_wait_guarded(acce_bar(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
        for (int32_t kb = 0; kb < kblocks; ++kb) {
          mbar_wait_guarded(full_bar(stage), phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sW = base + stage * C::STAGE_BYTES;
            const uint64_t dw = sdesc(sW);
            const uint64_t dx = sdesc(sW + W_TILE);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_pair(d_tmem, dw + 2 * kk, dx + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
            commit_pair(empty_bar(stage));
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) commit_pair(accf_bar(acc));
        __syncwarp();
        if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ================= epilogue (warps 2..5, both CTAs) =================
    const int quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int32_t c1 = 0, c2 = 0;
    for (int32_t t = ring.next(lane, leader_empty0); t >= 0; t = ring.next(lane, leader_empty0)) {
      const FTile tile = pdecode<TOK>(tt, t, c1, c2, p.d, p.f, rank);
      mbar_wait_guarded(accf_bar(acc), acc_phase);
      tc_fence_after();
      const int feat = tile.f0 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + acc * C::ACC_COLS;
      const int chunks = (tile.ntok + 31) / 32;
      for (int cc = 0; cc < chunks; ++cc) {
        uint32_t r[32];
        tmem_ld32(taddr + cc * 32, r);
        const int nvalid = min(32, tile.ntok - cc * 32);
        const int64_t row = int64_t(tile.row0) + cc * 32;
        if (tile.phase == 0) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.h) + row * p.f + feat;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nvalid)
              dst[int64_t(i) * p.f] = __float2bfloat16_rn(gelu_erf(__uint_as_float(r[i])));
        } else if (p.ret != nullptr) {
          // expert-parallel return: each row straight into its source rank's
          // y_back over NVLink (the combine then runs at the source)
          const int2 rt_l = lane < nvalid ? p.ret[row + lane] : make_int2(0, 0);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int rk = __shfl_sync(0xffffffffu, rt_l.x, i);
            const int pos = __shfl_sync(0xffffffffu, rt_l.y, i);
            if (i < nvalid)
              reinterpret_cast<__nv_bfloat16*>(p.peer_y[rk])[int64_t(pos) * p.d + feat] =
                  __float2bfloat16_rn(__uint_as_float(r[i]));
          }
        } else if (p.perm == nullptr) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.y) + row * p.d + feat;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nvalid) dst[int64_t(i) * p.d] = __float2bfloat16_rn(__uint_as_float(r[i]));
        } else {
          const int tok_l = lane < nvalid ? p.perm[row + lane] : 0;
          const float w_l = lane < nvalid ? p.topk_w[tok_l] : 0.0f;
          __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(p.y);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int tok = __shfl_sync(0xffffffffu, tok_l, i);
            const float w = __shfl_sync(0xffffffffu, w_l, i);
            if (i < nvalid) {
              const float yb16 = __bfloat162float(__float2bfloat16_rn(__uint_as_float(r[i])));
              yb[int64_t(tok) * p.d + feat] = __float2bfloat16_rn(fmaf(w, yb16, 0.0f));
            }
          }
        }
      }
      tc_fence_before();
      if (tile.phase == 0) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) {
          __threadfence();
          fence_proxy_async_global();
          red_release_add(p.done + tile.g, 1);
        }
      }
      __syncwarp();
      if (lane == 0) arrive_leader(acce_bar(acc));
      if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (p.ret) __threadfence_system();  // results stored to peers are visible system-wide
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no MMA, TMA or remote arrive of either CTA is still in flight
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(C::TMEM_COLS)
                 : "memory");
  }
}

template <int TOK, int STAGES>
void fused_pair_launch(const FusedFfnArgs& a, cudaStream_t stream) {
  using C = PairCfg<TOK, STAGES>;
  auto kern = fused_ffn_pair_kernel<TOK, STAGES>;
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), size_t(int(C::SMEM_BYTES)));
  const uint64_t rows = uint64_t(std::max<int64_t>(a.rows, 1));
  const CUtensorMap tx = make_tmap(a.x, rows, uint64_t(a.d_model), false, TOK_BOX);
  const CUtensorMap tw1 = make_tmap(a.w_in, uint64_t(a.n_slots) * a.d_ff, uint64_t(a.d_model),
                                    false, BM);
  const CUtensorMap th = make_tmap(a.h, rows, uint64_t(a.d_ff), false, TOK_BOX);
  const CUtensorMap tw2 = make_tmap(a.w_out, uint64_t(a.n_slots) * a.d_model, uint64_t(a.d_ff),
                                    false, BM);
  FusedParams p;
  std::memset(&p, 0, sizeof(p));
  p.d = a.d_model;
  p.f = a.d_ff;
  p.n_groups = a.n_groups;
  p.offsets = a.offsets;
  p.h = a.h;
  p.y = a.y;
  p.done = a.done;
  p.perm = a.perm;
  p.topk_w = a.topk_w;
  p.ret = a.ret;
  p.band_bytes = ffn_band_bytes();
  ffn_policies(p.pol_w, p.pol_x);
  for (int r = 0; r < a.n_peers && r < kMaxPeers; ++r) p.peer_y[r] = a.peer_y[r];
  for (int g = 0; g < a.n_groups; ++g) {
    p.experts[g] = a.experts[g];
    p.slots[g] = a.slots[g];
  }
  int grid = device_sm_count() & ~1;
  if (a.max_ctas > 0) grid = std::min(grid, (a.max_ctas + 1) & ~1);
  grid = std::max(grid, 2);
  if (a.ev_begin) INFMOE_CUDA(cudaEventRecord(a.ev_begin, stream));
  INFMOE_CUDA(cudaMemsetAsync(a.done, 0, sizeof(int32_t) * size_t(a.n_groups + 1), stream));
  kern<<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(tx, tw1, th, tw2, p);
  INFMOE_LAUNCH_CHECK();
  if (a.ev_end) INFMOE_CUDA(cudaEventRecord(a.ev_end, stream));
}

}  // namespace gemm

void launch_grouped_gemm(const GroupedGemmArgs& a, cudaStream_t stream) {
  require(a.n_groups >= 1 && a.n_groups <= kMaxGroups, "grouped gemm: n_groups out of range");
  require(a.N % gemm::BM == 0, "grouped gemm: N must be a multiple of 128");
  const int bk = a.dtype == kDtypeF32 ? 32 : 64;
  require(a.K % bk == 0 && a.K > 0, "grouped gemm: K must be a multiple of 64 (bf16) / 32 (f32)");
  require(a.a && a.b && a.out && a.offsets, "grouped gemm: NULL pointer");
  const bool tf32 = a.dtype == kDtypeF32;
  if (tf32) {
    if (a.gelu) gemm::dispatch_tok<true, true>(a, stream);
    else gemm::dispatch_tok<true, false>(a, stream);
  } else {
    if (a.gelu) gemm::dispatch_tok<false, true>(a, stream);
    else gemm::dispatch_tok<false, false>(a, stream);
  }
}

void launch_expert_ffn_fused(const FusedFfnArgs& a, cudaStream_t stream) {
  require(a.dtype == kDtypeBf16, "fused expert FFN: bf16 only (f32 uses the two-launch path)");
  require(a.n_groups >= 1 && a.n_groups <= kMaxGroups, "fused expert FFN: n_groups out of range");
  require(a.d_model % gemm::BM == 0 && a.d_ff % gemm::BM == 0,
          "fused expert FFN: d_model and d_ff must be multiples of 128");
  require(a.x && a.w_in && a.w_out && a.h && a.y && a.offsets && a.done,
          "fused expert FFN: NULL pointer");
  require((a.perm == nullptr) == (a.topk_w == nullptr), "fused expert FFN: perm needs topk_w");
  require(a.ret == nullptr || (a.perm == nullptr && a.n_peers >= 1 && a.n_peers <= kMaxPeers),
          "fused expert FFN: return mode needs 1..16 peers and no fused combine");
  const int hint = a.max_rows_hint;
  if (ffn_pair_mode() && a.d_model % (2 * gemm::BM) == 0 && a.d_ff % (2 * gemm::BM) == 0) {
    if (hint > 0 && hint <= 128) gemm::fused_pair_launch<128, 8>(a, stream);
    else if (hint > 192) gemm::fused_pair_launch<256, 6>(a, stream);
    else gemm::fused_pair_launch<192, 7>(a, stream);
    return;
  }
  if (hint > 0 && hint <= 128) gemm::fused_launch<128, 6>(a, stream);
  else if (hint > 192) gemm::fused_launch<256, 4>(a, stream);
  else gemm::fused_launch<192, 5>(a, stream);
}

// The cta_group::2 kernel is the default; INFMOE_FFN_PAIR=0 selects one SM per tile
bool ffn_pair_mode() {
  static int mode = [] {
    const char* v = std::getenv("INFMOE_FFN_PAIR");
    return v ? std::atoi(v) : 1;
  }();
  return mode != 0;
}

}  // namespace infmoe
