/*
 * infmoe.h — C-ABI of the B200-native InfMoE MoE-layer hot path (libinfmoe.so).
 *
 * Plain C types only: pointers, sizes, POD structs.  No C++ exception crosses
 * this boundary; every entry point returns a status code:
 *   0 OK, 2 config (moesim::ConfigError), 3 capacity (moesim::CapacityError),
 *   4 invariant breach (moesim::InvariantError), 5 CUDA / NCCL runtime failure,
 *   6 invalid argument (std::invalid_argument: malformed call, NULL pointer,
 *     non-permutation order, K < 1, T > max_T).
 * (errors.hpp:8-21 and SPEC.md:382 exit-code convention.)  The message for the
 * last failure on the calling thread is infmoe_last_error().
 *
 * Each declaration names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/moesim/).  Device pointers
 * are raw CUDA addresses; `stream` is a cudaStream_t passed as void*.
 */
#ifndef INFMOE_H_
#define INFMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  INFMOE_OK = 0,
  INFMOE_ERR_CONFIG = 2,
  INFMOE_ERR_CAPACITY = 3,
  INFMOE_ERR_INVARIANT = 4,
  INFMOE_ERR_RUNTIME = 5,
  INFMOE_ERR_ARGUMENT = 6
};

const char* infmoe_last_error(void);
const char* infmoe_version(void);

/* ---- model_config.hpp -------------------------------------------------- */
/* = moesim::ModelGeometry (model_config.hpp:14-22) */
typedef struct {
  int32_t n_layers, n_heads, d_head, d_model, d_ff, n_experts_per_layer, bytes_per_param;
} infmoe_geometry;
/* = moesim::HardwareProfile (model_config.hpp:27-32) */
typedef struct {
  double peak_flops;    /* FLOP/s */
  double h2d_bandwidth; /* bytes/s */
  uint64_t device_memory, reserved_memory;
} infmoe_hardware;

/* validate(ModelGeometry) model_config.hpp:37-55; *warn = 1 when d_model != n_heads*d_head */
int infmoe_validate_geometry(const infmoe_geometry* g, int32_t* warn_dmodel);
/* validate(HardwareProfile) model_config.hpp:57-64 */
int infmoe_validate_hardware(const infmoe_hardware* hw);
/* expert_param_bytes model_config.hpp:69-73 */
uint64_t infmoe_expert_param_bytes(const infmoe_geometry* g);
/* expert_flops model_config.hpp:77-80 */
uint64_t infmoe_expert_flops(const infmoe_geometry* g, uint64_t n_tokens);
/* builtin_geometry_presets model_config.hpp:85-105 ("cpm2", "cpm-small") */
int infmoe_geometry_preset(const char* name, infmoe_geometry* out);

/* ---- prng.hpp ---------------------------------------------------------- */
uint64_t infmoe_splitmix64(uint64_t x);                 /* prng.hpp:18-23 */
uint64_t infmoe_derive_seed(uint64_t seed, uint64_t tag); /* prng.hpp:27-29 */
/* n consecutive draws of GaussianStream(seed).next() (prng.hpp:49-71) */
int infmoe_gaussian_fill(uint64_t seed, double* out, uint64_t n);

/* The synthetic tensors of SURVEY 8(d), host side: n_mats independent
 * GaussianStream(seeds[m]) sequences (prng.hpp:49-71, the generator of
 * gaussian_tokens gating.hpp:108-114), each value times scales[m], rounded to
 * dtype (INFMOE_DTYPE_BF16: double -> f32 round-to-nearest -> bf16 RNE;
 * INFMOE_DTYPE_F32: double -> f32), n_each values into outs[m] (host memory).
 * threads <= 0 uses every hardware thread; values do not depend on it. */
int infmoe_gaussian_fill_typed(int32_t dtype, int32_t n_mats, const uint64_t* seeds,
                               const double* scales, uint64_t n_each, void* const* outs,
                               int32_t threads);

/* ---- gating.hpp (host side) ------------------------------------------- */
/* gating_projection gating.hpp:47-56: bits*hidden doubles, bit-major */
int infmoe_gating_projection(uint64_t seed, int32_t n_hash_bits, int32_t hidden_dim,
                             double* out);
/* lsh_codes gating.hpp:61-82 on HOST fp64 rows x[n_tokens, hidden]
 * (GatingModel{seed, bits, hidden}): bit-identical codes (sequential fp64 dot,
 * no contraction).  Errors as the reference: bits outside [1, 31] or hidden < 1
 * -> 2 (ConfigError).  The device gate for bf16/f32 rows is infmoe_gate_lsh. */
int infmoe_lsh_codes(uint64_t seed, int32_t n_hash_bits, int32_t hidden_dim, const double* x,
                     uint64_t n_tokens, uint32_t* codes);
/* route_tokens gating.hpp:87-104: counts[n_experts] of code mod n_experts.
 * n_experts < 1 -> 6 (std::invalid_argument); 2^bits < n_experts -> 2 */
int infmoe_route_tokens(uint64_t seed, int32_t n_hash_bits, int32_t hidden_dim,
                        const double* x, uint64_t n_tokens, int32_t n_experts,
                        uint64_t* counts);
/* explicit_workload gating.hpp:167-175 (+ validate :25-33): *total = sum of
 * counts; no experts -> 2 */
int infmoe_explicit_workload(const uint64_t* counts, int32_t n_experts, uint64_t* total);
/* workload_from_csv gating.hpp:180-219: "expert_id,token_count" rows, optional
 * header line, ids in any order (missing ids count 0, duplicates -> 2).
 * *n_experts = max id + 1; counts (capacity entries, may be NULL to query the
 * size first) receives the per-expert counts; *total (may be NULL) their sum. */
int infmoe_workload_from_csv(const char* path, uint64_t* counts, int32_t capacity,
                             int32_t* n_experts, uint64_t* total);
/* synthetic_workload gating.hpp:122-165; kind 0 uniform, 1 zipf, 2 balanced */
int infmoe_synthetic_workload(int32_t kind, uint64_t total_tokens, int32_t n_experts,
                              uint64_t seed, double zipf_s, uint64_t* counts);

/* ---- cost_model.hpp ---------------------------------------------------- */
/* compute_costs cost_model.hpp:43-62 (counts has g->n_experts_per_layer entries) */
int infmoe_compute_costs(const infmoe_geometry* g, const infmoe_hardware* hw,
                         const uint64_t* counts, int32_t n_experts, double* alphas,
                         double* beta);
/* resident_capacity cost_model.hpp:65-78 */
int infmoe_resident_capacity(const infmoe_geometry* g, const infmoe_hardware* hw,
                             int32_t* K);
/* clamp_explicit_capacity cost_model.hpp:82-91; *clamped = 1 when the warning fired */
int infmoe_clamp_explicit_capacity(int32_t explicit_k, int32_t capacity, int32_t* K,
                                   int32_t* clamped);
/* with_event_overhead cost_model.hpp:96-101 (in place) */
int infmoe_with_event_overhead(double* alphas, int32_t T, double* beta, double eps);

/* ---- scheduler.hpp ----------------------------------------------------- */
enum { INFMOE_BOUND_LOWER = 0, INFMOE_BOUND_UPPER = 1 };
/* = moesim::ConstraintReport (scheduler.hpp:25-37); position = -1 when none */
typedef struct {
  int32_t feasible;
  int32_t position;
  int32_t bound;
  double prefix_sum, limit;
} infmoe_constraint_report;
/* check_constraints scheduler.hpp:70-95; slack[T] may be NULL */
int infmoe_check_constraints(const int32_t* order, const double* alphas, int32_t T,
                             double beta, int32_t K, double* slack,
                             infmoe_constraint_report* rep);

enum { /* OrderPolicy simulator.hpp:17 + the direct scheduler entry points */
  INFMOE_POLICY_AUTO = 0,   /* auto_order  scheduler.hpp:243-248 (greedy + exact fallback) */
  INFMOE_POLICY_GREEDY = 1, /* greedy_order scheduler.hpp:143-180 */
  INFMOE_POLICY_EXACT = 2,  /* exact_order scheduler.hpp:187-237 */
  INFMOE_POLICY_NAIVE = 3   /* naive_order scheduler.hpp:127-132 */
};
enum { INFMOE_DIAG_NONE = -1, INFMOE_DIAG_FEASIBLE = 0, INFMOE_DIAG_TOO_LITTLE_COMPUTE = 1,
       INFMOE_DIAG_IMBALANCED = 2 };
enum { INFMOE_METHOD_GREEDY = 0, INFMOE_METHOD_EXACT_FALLBACK = 1, INFMOE_METHOD_NAIVE = 2 };
/* = moesim::Schedule (scheduler.hpp:39-45) minus the vectors */
typedef struct {
  int32_t feasible;
  int32_t diagnosis; /* INFMOE_DIAG_*, NONE when unset */
  int32_t method;    /* INFMOE_METHOD_* */
} infmoe_schedule_info;
int infmoe_schedule(const double* alphas, int32_t T, double beta, int32_t K, int32_t policy,
                    int32_t exact_max_T, int32_t* order, double* slack,
                    infmoe_schedule_info* info);
/* diagnose scheduler.hpp:253-258 */
int infmoe_diagnose(const double* alphas, int32_t T, double beta, int32_t K,
                    int32_t exact_max_T, int32_t* diagnosis);

/* ---- simulator.hpp ----------------------------------------------------- */
enum { INFMOE_STREAM_LOAD = 0, INFMOE_STREAM_COMPUTE = 1 };
enum { INFMOE_MODE_OVERLAPPED = 0, INFMOE_MODE_SERIAL = 1 };
/* = moesim::TimelineEvent (simulator.hpp:19-25) */
typedef struct {
  int32_t stream, layer_id, expert_id;
  double start, end;
} infmoe_event;
/* = moesim::SimReport (simulator.hpp:40-48) without per_layer */
typedef struct {
  double makespan, compute_busy, load_busy, compute_stall;
  int32_t peak_resident_experts;
  double overlap_efficiency;
} infmoe_sim_report;
/* = moesim::LayerReport (simulator.hpp:27-38) without the schedule */
typedef struct {
  int32_t layer_id, n_experts;
  double start, end, compute_busy, load_busy, compute_stall;
  int32_t peak_resident;
  double lower_bound;
} infmoe_layer_report;
/* simulate(order, costs, K, mode) simulator.hpp:209-220; events[2T] */
int infmoe_simulate(const int32_t* order, const double* alphas, int32_t T, double beta,
                    int32_t K, int32_t mode, infmoe_event* events, infmoe_sim_report* rep);
/* run_layers (simulator.hpp:102-194) on GIVEN per-layer orders: simulate(schedule,
 * costs, K, mode) and simulate(order, costs, K, mode) (simulator.hpp:199-220) for
 * one layer, or a stack of layers with fixed orders (drain, or
 * continuous_load_stream != 0).  Orders are checked as permutations. */
int infmoe_simulate_orders(int32_t n_layers, const int32_t* T, const int32_t* orders,
                           const double* alphas, const double* betas, int32_t K, int32_t mode,
                           int32_t continuous_load_stream, infmoe_event* events,
                           infmoe_sim_report* rep, infmoe_layer_report* per_layer);
/* simulate_model(costs, K, opt) simulator.hpp:241-255.  Layer l has T[l] experts,
 * alphas concatenated, betas[l].  policy: INFMOE_POLICY_AUTO (= OrderPolicy::Greedy),
 * _NAIVE or _EXACT.  orders_out[sum T], events[2 sum T], per_layer[n_layers] (may be NULL). */
int infmoe_simulate_model(int32_t n_layers, const int32_t* T, const double* alphas,
                          const double* betas, int32_t K, int32_t mode, int32_t policy,
                          int32_t continuous_load_stream, int32_t exact_max_T,
                          int32_t* orders_out, infmoe_event* events, infmoe_sim_report* rep,
                          infmoe_layer_report* per_layer);
/* lower_bound simulator.hpp:53-56 */
double infmoe_lower_bound(const double* alphas, int32_t T, double beta);
/* Timeline audit (the rules of verification.hpp:108-198, re-implemented for
 * MEASURED timelines): per-stream exclusivity, load-before-compute per
 * (layer, expert), at most max_resident experts resident per layer (load end
 * to compute end, departures before arrivals at ties), malformed events, and
 * (check_durations != 0) event lengths equal to beta / alpha.  Returns the
 * violation count in *n_violations and per-kind counts in kinds[6] (overlap,
 * causality, residency, duration, makespan, malformed). */
int infmoe_replay_check(const infmoe_event* events, int32_t n_events, int32_t n_layers,
                        const int32_t* T, const double* alphas, const double* betas,
                        int32_t max_resident, int32_t check_durations, double tol_s,
                        int32_t* n_violations, int32_t* kinds);

/* ======================================================================
 * Device path: the MoE layer forward the paper's TensorRT plugin ran
 * (PAPER.md:345, :396).  No reference code exists for these;
 * the semantics are fixed by oracle/oracle.h.
 * ==================================================================== */
enum { INFMOE_DTYPE_BF16 = 0, INFMOE_DTYPE_F32 = 1 };
enum { INFMOE_GATE_SOFTMAX = 0, INFMOE_GATE_LSH = 1 };
enum { INFMOE_RESIDENT = 0, INFMOE_OFFLOADED = 1 };

/* counter-hash synthetic fill (oracle.h or_fill_uniform_*): out[i] = (2u-1)*scale */
int infmoe_fill_uniform(void* out, int32_t dtype, uint64_t n, uint64_t seed, float scale,
                        void* stream);

/* test hooks: n_ctas spinning CTAs holding smem_bytes of shared memory each
 * (one per SM at ~200 KB; an even n_ctas launches clusters of 2, i.e. whole
 * TPCs) until *release != 0 (device int) or timeout_ns;
 * *timed_out (device int) is set to 1 if any gave up.  infmoe_debug_set_flag
 * stores 1 to *flag in stream order.  Used to check that the persistent FFN
 * makes progress when part of the GPU is taken by a concurrent kernel. */
int infmoe_debug_occupy_sms(int32_t n_ctas, int32_t smem_bytes, const int32_t* release,
                            uint64_t timeout_ns, int32_t* timed_out, void* stream);
int infmoe_debug_set_flag(int32_t* flag, void* stream);

/* N1a softmax/top-k gate: x[N,d] (dtype), wg[E,d] f32, bias[E] f32 or NULL.
 * Outputs topk_idx[N,k] i32, topk_w[N,k] f32, counts[E] i32 (device). */
int infmoe_gate_softmax_topk(const void* x, int32_t dtype, int64_t N, int32_t d,
                             const float* wg, const float* bias, int32_t E, int32_t k,
                             int32_t* topk_idx, float* topk_w, int32_t* counts, void* stream);
/* The same gate with caller-owned workspace, for fixed gate weights: the
 * tensor-core path (bf16 x, 2 <= k <= 8, E <= 128, d % 64 == 0) keeps W_g's
 * bf16 split there.  ws_bytes() is 0 when the call takes the CUDA-core path
 * (ws may then be NULL); prepare(wg) fills ws once (stream-ordered), after
 * which topk_ws() runs without re-splitting W_g.  Results equal
 * infmoe_gate_softmax_topk's. */
size_t infmoe_gate_softmax_ws_bytes(int32_t dtype, int64_t N, int32_t d, int32_t E, int32_t k);
int infmoe_gate_softmax_prepare(const float* wg, int32_t d, int32_t E, void* ws,
                                size_t ws_bytes, void* stream);
int infmoe_gate_softmax_topk_ws(const void* x, int32_t dtype, int64_t N, int32_t d,
                                const float* wg, const float* bias, int32_t E, int32_t k,
                                int32_t* topk_idx, float* topk_w, int32_t* counts, void* ws,
                                size_t ws_bytes, void* stream);
/* Test hook of the same gate: also returns the tensor-core path's approximate
 * logits (approx_logits[N,E] f32 device, may be NULL) and its counters
 * (stats[4] u64 device: tokens certified from the tensor-core logits, tokens
 * sent to the exact fallback, exact-chain logits the fallback computed, tokens
 * that took every expert through the exact chain; all-ones when the call ran
 * on the CUDA-core path: f32 x, top_k == 1 or > 8, E > 128, d % 64 != 0). */
int infmoe_gate_softmax_debug(const void* x, int32_t dtype, int64_t N, int32_t d,
                              const float* wg, const float* bias, int32_t E, int32_t k,
                              int32_t* topk_idx, float* topk_w, int32_t* counts,
                              float* approx_logits, uint64_t* stats, void* stream);
/* N1b LSH gate (gating.hpp:61-104) on the fp64 promotion of x; proj[bits,d] f64 device.
 * Writes codes[N] u32 (may be NULL), topk_idx[N], topk_w[N]=1, counts[E]. */
int infmoe_gate_lsh(const void* x, int32_t dtype, int64_t N, int32_t d, const double* proj,
                    int32_t bits, int32_t E, uint32_t* codes, int32_t* topk_idx,
                    float* topk_w, int32_t* counts, void* stream);
/* N2 dispatch: stable counting sort of N*k assignments -> offsets[E+1], perm[N*k],
 * inv[N*k]; workspace >= infmoe_dispatch_workspace_bytes(N*k, E) bytes (device). */
size_t infmoe_dispatch_workspace_bytes(int64_t n_assign, int32_t E);
int infmoe_dispatch(const int32_t* topk_idx, int64_t N, int32_t k, int32_t E,
                    int32_t* offsets, int32_t* perm, int32_t* inv, void* workspace,
                    void* stream);
/* N2 gather: x_perm[p] = x[perm[p] / k] for p < N*k (row-vectorised) */
int infmoe_gather_rows(const void* x, int32_t dtype, int64_t N, int32_t d, int32_t k,
                       const int32_t* perm, void* x_perm, void* stream);
/* N2 gather, token-major: x_perm[inv[t*k+j]] = x[t] (the same x_perm as
 * infmoe_gather_rows; each token row is read once — the layer's path for k > 1) */
int infmoe_gather_rows_by_token(const void* x, int32_t dtype, int64_t N, int32_t d, int32_t k,
                                const int32_t* inv, void* x_perm, void* stream);
/* N3+N4 grouped expert FFN on tcgen05: for each listed expert e with rows
 * [offsets[e], offsets[e+1]) of x_perm:  h = GeLU(x_perm . w_in[slot]^T) (bf16 into h),
 * y_perm = h . w_out[slot]^T.  w_in is [n_slots, d_ff, d_model], w_out is
 * [n_slots, d_model, d_ff] (K-major).  experts/slots are HOST arrays of n_groups
 * entries; experts == NULL means all E with slot == expert. */
int infmoe_expert_ffn(const void* x_perm, int64_t n_rows, int32_t d_model, int32_t d_ff,
                      int32_t dtype, const int32_t* offsets, int32_t E,
                      const void* w_in, const void* w_out, int32_t n_slots,
                      const int32_t* experts, const int32_t* slots, int32_t n_groups,
                      void* h, void* y_perm, void* stream);
/* N3+N4 in ONE persistent launch (phase-2 tiles of an expert start once its
 * H rows are complete; see csrc/kernels/expert_gemm.cuh).  bf16 only.
 * done: >= n_groups + 1 int32 of device scratch (per-expert completion counters
 * and the tile-claim counter of the persistent launch).  perm/topk_w (top-1 only, or
 * NULL): fuse the combine, y[perm[r]] = bf16(fmaf(topk_w[perm[r]], bf16(acc_r), 0)),
 * in which case y is [N, d_model]; otherwise y is y_perm [n_rows, d_model]. */
int infmoe_expert_ffn_fused(const void* x_perm, int64_t n_rows, int32_t d_model, int32_t d_ff,
                            const int32_t* offsets, int32_t E, const void* w_in,
                            const void* w_out, int32_t n_slots, const int32_t* experts,
                            const int32_t* slots, int32_t n_groups, void* h, void* y,
                            const int32_t* perm, const float* topk_w, int32_t* done,
                            void* stream);
/* row scatter (inverse of the gather): dst[index[p]] = src[p] for p < rows */
int infmoe_scatter_rows(const void* src, int32_t dtype, int64_t rows, int32_t d,
                        const int32_t* index, void* dst, void* stream);
/* N5 combine: y[t] = fmaf-chain over j<k of topk_w[t,j] * y_perm[inv[t,j]] */
int infmoe_combine(const void* y_perm, int32_t dtype, const int32_t* inv,
                   const float* topk_w, int64_t N, int32_t k, int32_t d, void* y,
                   void* stream);

/* ---- the layer handle (N6 offload executor + N8) ---------------------- */
typedef struct infmoe_layer infmoe_layer;
/* A device pool of K+1 expert slots (W_in + W_out each) that offloaded layers
 * of one shape share: the InfMoE memory model, K experts resident on the GPU
 * for the whole stack plus the one load in flight (resident_capacity,
 * cost_model.hpp:65).  Layers sharing a pool must be forwarded one
 * after another on one stream (a layer's loads start after the previous
 * layer's computes: the reference's drain mode, simulator.hpp:131-133). */
typedef struct infmoe_slot_pool infmoe_slot_pool;
typedef struct {
  int32_t d_model, d_ff, n_experts, top_k;
  int32_t dtype;      /* INFMOE_DTYPE_* */
  int32_t gate_kind;  /* INFMOE_GATE_* */
  int32_t residency;  /* INFMOE_RESIDENT / INFMOE_OFFLOADED */
  int32_t K;          /* offloaded: resident capacity K; the handle owns K+1 slots (D6) */
  int32_t policy;     /* INFMOE_POLICY_* for the offload order */
  int32_t max_tokens; /* upper bound on N per forward */
  int32_t device;
  /* gate: softmax -> gate_weight[E,d] f32 (+ optional gate_bias[E]); lsh -> seed/bits */
  const float* gate_weight; /* host pointer, copied at create */
  const float* gate_bias;   /* host pointer or NULL */
  uint64_t lsh_seed;
  int32_t lsh_bits;
  /* expert weights: w_in [E, d_ff, d_model], w_out [E, d_model, d_ff] in dtype.
   * RESIDENT: device pointers (borrowed).  OFFLOADED: host pointers; page-locked
   * memory is used as is, pageable memory is registered by the handle. */
  const void* w_in;
  const void* w_out;
  infmoe_hardware hw; /* cost model inputs for the scheduler (alpha, beta) */
  /* expert parallelism: ep_size ranks, experts split into
   * contiguous blocks of n_experts/ep_size; w_in/w_out then hold only this
   * rank's block.  ep_comm from infmoe_ep_comm_init (NULL when ep_size == 1). */
  int32_t ep_size, ep_rank;
  void* ep_comm;
  /* skip_empty_experts (scenario.hpp:99; default off as in the
   * reference): experts that received no rows are neither scheduled nor loaded */
  int32_t skip_empty_experts;
  /* offloaded: shared slot pool (NULL: the handle owns its own K+1 slots) */
  infmoe_slot_pool* slot_pool;
  /* expert-parallel transport: INFMOE_EP_NCCL (grouped ncclSend/ncclRecv
   * all-to-allv, host-planned) or INFMOE_EP_PEER (rows pushed straight into the
   * owner's expert-contiguous buffer over peer memory, results written back by
   * the expert FFN's epilogue, plan computed on the device; peers are mapped
   * with CUDA IPC at create; NCCL only for 1-int barriers) */
  int32_t ep_transport;
  /* offloaded, bf16: how expert weights cross the host link.  INFMOE_CODEC_RAW
   * (default; the reference's model: expert_param_bytes per load) or
   * INFMOE_CODEC_EXP4 (lossless: the handle packs the host weights once into
   * pinned exp4 packs -- 12 bits per value, exponents coded against a per-block
   * base -- shared by every layer on the same host weights; each load copies
   * the pack and a decoder kernel restores the bf16 slot bit for bit before the
   * FFN).  INFMOE_CODEC_EXPH instead codes each value's (exponent distance
   * to its block or matrix base, top two mantissa bits) with a per-matrix
   * canonical Huffman code (<= 12 bits, length-limited optimally) and stores
   * the sign and low five mantissa bits raw: 256-value chunks with recorded
   * start bits, decoded one warp per 32 chunks (one lane per chunk) through a
   * shared-memory table; ~10.1-10.9 bits per value (uniform .. Laplace
   * weights; 10.61 on Gaussian).
   * Packs are SNAPSHOTS of the host weights taken at create and at every
   * infmoe_layer_set_host_weights call (which always re-packs); layers created
   * on the same host buffers share one pack only while its content digest
   * matches the buffers.  Refilling host weights in place without calling
   * infmoe_layer_set_host_weights leaves a codec layer on the old snapshot.
   * Outputs are identical; the scheduler's costs stay the reference's. */
  int32_t h2d_codec;
  /* continuous_load_stream (simulator.hpp:99-101, :131-133; scenario.hpp:98;
   * default 0 = the reference's drain mode).  A layer's loads depend on its
   * routing, i.e. on the previous layer's output, so the executor realises the
   * continuous lane SPECULATIVELY: once this layer's last load is issued, it
   * streams the first prefetch_depth experts of the layer set with
   * infmoe_layer_set_next, in the InfMoE order of that layer's predicted counts
   * (an EMA of its routed rows), into that layer's own slots; the next forward
   * reuses the leading positions whose expert matches its real order and loads
   * the rest as usual.  Outputs are unchanged.  Layers sharing a slot pool
   * need a pool with 2 slot sets (infmoe_slot_pool_create_ex): consecutive
   * layers use alternate sets ("each layer has its own K slots"). */
  int32_t continuous_load_stream;
  int32_t prefetch_depth; /* 0: 1 position; at most K */
} infmoe_layer_desc;
enum { INFMOE_EP_NCCL = 0, INFMOE_EP_PEER = 1 };
enum { INFMOE_CODEC_RAW = 0, INFMOE_CODEC_EXP4 = 1, INFMOE_CODEC_EXPH = 2 };

/* per-forward outputs (all optional; host pointers unless noted) */
typedef struct {
  int32_t* counts;       /* [E] routed tokens per expert */
  int32_t* order;        /* [E] executed expert order (offloaded) */
  int32_t* feasible;     /* scheduler verdict */
  infmoe_event* events;  /* [2E] measured timeline (seconds from layer start) */
  double* exposed_copy_s;/* makespan - compute_busy on the measured timeline */
  int32_t* local_rows;   /* [E/ep_size] rows this rank computed per local expert */
  /* per-token routing (SURVEY 8(b) infmoe_routing_out), DEVICE pointers filled
   * in stream order (no host sync): topk_idx[N*k] expert of (token t, slot j)
   * at t*k+j, topk_w[N*k] its gate weight, perm[N*k] the dispatch permutation
   * (perm[pos] = t*k+j, grouped by expert, token order inside an expert),
   * offsets[E+1] each expert's first position in perm.  Each may be NULL. */
  int32_t* topk_idx;
  float* topk_w;
  int32_t* perm;
  int32_t* offsets;
  /* input, optional: a cudaEvent_t recorded earlier on the stream; measured
   * event times are then seconds from it (not from this forward's start), so
   * the layers of a stack report on one time axis */
  void* time_origin;
  /* output, optional: leading positions of this forward's load order whose
   * copies the previous layer prefetched and that were reused (continuous) */
  int32_t* prefetched;
} infmoe_forward_out;

/* ---- expert parallelism (N7) ------------------------------------------ */
/* Exchange plan for one rank: send_counts[E] (rows this rank routes to every
 * global expert), recv_counts[P * E/P] (rows each source routes to this rank's
 * experts, source-major).  Outputs: send_off/send_rows[P], recv_off/recv_rows[P],
 * local_offsets[E/P + 1], local_index[n_recv] (local row <- receive row),
 * *n_recv.  local_index may be NULL to query n_recv first. */
int infmoe_ep_plan(int32_t P, int32_t rank, int32_t E, const int32_t* send_counts,
                   const int32_t* recv_counts, int64_t* send_off, int64_t* send_rows,
                   int64_t* recv_off, int64_t* recv_rows, int32_t* local_offsets,
                   int32_t* local_index, int64_t* n_recv);
/* NCCL communicator for the EP exchange (NCCL is loaded at run time) */
int infmoe_ep_get_unique_id(uint8_t id[128]);
int infmoe_ep_comm_init(const uint8_t id[128], int32_t nranks, int32_t rank, void** comm);
int infmoe_ep_comm_destroy(void* comm);

/* K+1 slots of expert_matrix_bytes (= d_ff * d_model * bytes/param) per matrix */
int infmoe_slot_pool_create(int32_t device, int32_t K, uint64_t expert_matrix_bytes,
                            infmoe_slot_pool** out);
/* the same with `sets` independent sets of K+1 slots (sets = 2 for stacks of
 * continuous_load_stream layers: consecutive layers use alternate sets) */
int infmoe_slot_pool_create_ex(int32_t device, int32_t K, uint64_t expert_matrix_bytes,
                               int32_t sets, infmoe_slot_pool** out);
int infmoe_slot_pool_destroy(infmoe_slot_pool* pool);

int infmoe_layer_create(const infmoe_layer_desc* desc, infmoe_layer** out);
/* x, y: device [N, d_model] in dtype; stream: cudaStream_t or NULL. */
int infmoe_layer_forward(infmoe_layer* layer, const void* x, int64_t N, void* y,
                         infmoe_forward_out* out, void* stream);
/* infmoe_layer_forward with the caller's routing instead of the layer's gate:
 * topk_idx[N*k] (device, every entry in [0, n_experts)) and topk_w[N*k]
 * (device) -- e.g. a scenario's synthetic / explicit / CSV workload realised
 * as token assignments.  Dispatch, executor and combine are unchanged. */
int infmoe_layer_forward_routed(infmoe_layer* layer, const void* x, int64_t N,
                                const int32_t* topk_idx, const float* topk_w, void* y,
                                infmoe_forward_out* out, void* stream);
/* continuous_load_stream: `next` is the layer forwarded after `layer` (may be
 * the first layer of the stack, closing the cycle for the next batch); both
 * offloaded with continuous_load_stream, on one device.  Layers sharing a
 * pool alternate slot sets along the chain (an odd cycle on one pool -> 6).
 * next == NULL unlinks. */
int infmoe_layer_set_next(infmoe_layer* layer, infmoe_layer* next);
/* point an offloaded layer at another host weight set of the same shape */
int infmoe_layer_set_host_weights(infmoe_layer* layer, const void* w_in, const void* w_out);
/* SURVEY 8(f)-4, NOT in the reference (its eviction is immediate):
 * hot-expert pinning for an offloaded layer.  The n listed local experts are
 * copied to device memory once and stay there across forwards (n = 0 unpins);
 * a forward then computes the pinned experts first, in one grouped launch with
 * no load, while the first streamed copy is in flight, and streams only the
 * others, in the InfMoE order over their own costs through the K+1 slots.
 * Outputs are bit-identical to the unpinned layer.  Returns 3 (CapacityError)
 * when the device copies do not fit, 6 for a resident layer or a bad list. */
int infmoe_layer_pin_experts(infmoe_layer* layer, const int32_t* experts, int32_t n);
/* The cross-batch cache policy over infmoe_layer_pin_experts: pin the n local
 * experts with the highest running load estimate (an EMA of each expert's
 * routed rows over this layer's offloaded forwards, decay 0.5; ties to the
 * lower index), re-using the device copies of experts that stay pinned.
 * pinned (optional, n entries) receives the chosen experts in ascending order. */
int infmoe_layer_pin_hottest(infmoe_layer* layer, int32_t n, int32_t* pinned);
int infmoe_layer_destroy(infmoe_layer* layer);
/* bytes one pass of an offloaded layer moves over the host link for its local
 * experts with its codec (packed) and without (raw = n_local * expert_param_bytes) */
int infmoe_layer_h2d_bytes(infmoe_layer* layer, uint64_t* packed, uint64_t* raw);
/* Where the layer's h2d-codec pack came from: 0 no pack (raw stream), 1 encoded
 * in this process, 2 read from the pack cache directory. */
int infmoe_layer_pack_source(infmoe_layer* layer, int32_t* source);
/* Pack cache directory (process-wide; NULL or "" disables; default: the
 * INFMOE_PACK_CACHE_DIR environment variable).  A codec layer looks up
 * <dir>/<content digest>-<codec>-<experts>x<elems>.infmoe-pack before
 * encoding its host weights and writes the file after encoding (tmp file +
 * rename).  The file name carries the digest of the host weights and the
 * file its own checksum, so a stale or damaged file is never used: it is
 * re-encoded and replaced.  Saves the one-time encode (~9 s per 10.7 GB of
 * bf16 weights on 16 host threads) on every later start. */
int infmoe_set_pack_cache_dir(const char* dir);
/* codec round trip (test hook): pack n bf16 values (host) with codec
 * (INFMOE_CODEC_EXP4 / EXPH) on the host, decode them on the device, copy the
 * result to out (host); pack_bytes (may be NULL) receives the pack size.  n must
 * be a positive multiple of 256 (exph) or 128 (exp4). */
int infmoe_codec_roundtrip(int32_t codec, const uint16_t* in, uint64_t n, uint16_t* out,
                           uint64_t* pack_bytes, int32_t device);
/* the same round trip decoded by the host reference decoder (no GPU needed) */
int infmoe_codec_roundtrip_host(int32_t codec, const uint16_t* in, uint64_t n, uint16_t* out,
                                uint64_t* pack_bytes);

/* ---- scenario.hpp + the CLI front door ------------------ */
/* parse_scenario (scenario.hpp:188-332: strict keys, presets from
 * builtin_geometry_presets + $MOE_SIM_PRESETS, K = integer or "auto", seed from
 * entropy when omitted) and to_json (scenario.hpp:350-406): the resolved
 * self-contained scenario, indented JSON with sorted keys, into out (cap bytes,
 * NUL-terminated; *len = bytes needed).  Errors 2 / 3 with the reference's
 * messages. */
int infmoe_scenario_resolve(const char* json_text, char* out, uint64_t cap, uint64_t* len);
int infmoe_scenario_resolve_file(const char* path, char* out, uint64_t cap, uint64_t* len);
typedef struct {
  const char* out_dir;   /* NULL: the scenario's output_dir */
  int32_t trace_format;  /* bit 0 Chrome trace JSON, bit 1 events CSV (0 = both) */
  int32_t execute;       /* 1: also run the layers on the GPU through the offload executor
                          * and write MEASURED timelines under <out>/measured/ */
  int32_t device;
  int32_t host_sets;     /* execute: distinct host weight sets aliased across layers */
  int32_t repeats;       /* execute: stack passes per policy (the last is reported) */
  int32_t jobs;          /* sweep: points simulated concurrently (results unchanged) */
  int32_t has_seed;      /* 1: seed overrides the config's seed (--seed) */
  uint64_t seed;
} infmoe_run_options;
/* run_scenario: per policy <out>/<policy>/{trace.json,
 * events.csv, report.json}, <out>/summary.csv, <out>/resolved.json, and
 * <out>/meta.json (the only file with timestamps: two runs of the same
 * resolved scenario give byte-identical artefacts otherwise).
 * The summary CSV is also returned in summary (cap bytes; *len needed). */
int infmoe_scenario_run(const char* config_path, const infmoe_run_options* opt, char* summary,
                        uint64_t cap, uint64_t* len);
/* sweep over axis "K" | "total_tokens" | "zipf_s" |
 * "bandwidth": one run per value under <out>/<axis>=<value>/ and
 * <out>/sweep.csv (rows in value order, whatever opt->jobs); an axis the
 * scenario cannot take -> 2. */
int infmoe_scenario_sweep(const char* config_path, const char* axis, const double* values,
                          int32_t n_values, const infmoe_run_options* opt, char* table,
                          uint64_t cap, uint64_t* len);

#ifdef __cplusplus
}
#endif
#endif /* INFMOE_H_ */
