/*
 * oracle.h — CPU restatement of InfMoE's MoE-layer hot path (TEST INFRASTRUCTURE).
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * (libinfmoe.so) never links, calls or falls back to anything in oracle/.
 *
 * Parity status
 *   - PINNED to the reference (moesim headers under /root/reference/proj/include,
 *     compiled by oracle/Makefile into oracle/_ref/libmoesim_ref.so and frozen as
 *     golden vectors in tests/golden/): PRNG stream, LSH gate, route_tokens,
 *     synthetic workloads, cost model, K, check_constraints, greedy/exact/auto
 *     order, diagnose, simulate/simulate_model, lower_bound, instance_digest.
 *   - PARITY UNPINNED by the reference (no reference implementation exists;
 *     SURVEY.md §0.1): softmax/top-k gate, dispatch permutation, expert FFN,
 *     combine.  For these the oracle below *is* the definition, written from the
 *     counts semantics of gating.hpp:96-103 and the two-matrix expert of
 *     model_config.hpp:12-13.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off (see oracle/Makefile).  No FMA
 * contraction: gating.hpp:76 compiles to separate mul+add in the reference build.
 */
#ifndef INFMOE_ORACLE_H
#define INFMOE_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- prng.hpp:18-71 ---------------------------------------------------- */
uint64_t or_splitmix64(uint64_t x);
uint64_t or_derive_seed(uint64_t seed, uint64_t tag);
uint64_t or_mt64_first(uint64_t seed); /* first mt19937_64 output (anchor) */
void or_gaussian_fill(uint64_t seed, double* out, uint64_t n);
/* counter-hash synthetic fill shared with the product's fill kernels */
void or_fill_uniform_f32(uint64_t seed, uint64_t n, float scale, float* out);
void or_fill_uniform_bf16(uint64_t seed, uint64_t n, float scale, uint16_t* out);
uint16_t or_f32_to_bf16(float f);
float or_bf16_to_f32(uint16_t h);

/* ---- gating.hpp ---------------------------------------------------------- */
int or_gating_projection(uint64_t seed, int bits, int hidden, double* out);
int or_lsh_codes(uint64_t seed, int bits, int hidden, const double* x, uint64_t n,
                 uint32_t* codes);
int or_route_tokens(uint64_t seed, int bits, int hidden, const double* x, uint64_t n,
                    int n_experts, uint64_t* counts);
/* kind: 0 uniform, 1 zipf, 2 balanced (gating.hpp:116) */
int or_synthetic_workload(int kind, uint64_t total, int n_experts, uint64_t seed,
                          double zipf_s, uint64_t* counts);

/* ---- model_config.hpp / cost_model.hpp --------------------------------- */
uint64_t or_expert_param_bytes(int d_model, int d_ff, int bytes_per_param);
uint64_t or_expert_flops(int d_model, int d_ff, uint64_t n_tokens);
int or_compute_costs(int d_model, int d_ff, int bytes_per_param, double peak_flops,
                     double h2d_bw, const uint64_t* counts, int T, double* alphas,
                     double* beta);
int or_resident_capacity(int d_model, int d_ff, int bytes_per_param,
                         uint64_t device_memory, uint64_t reserved, int* K);

/* ---- scheduler.hpp ------------------------------------------------------- */
/* returns 0 ok, 2 invalid argument; feasible / first violation through outs */
int or_check_constraints(const int* order, const double* alphas, int T, double beta,
                         int K, double* slack, int* feasible, int* viol_pos,
                         int* viol_side);
/* method: 0 greedy, 1 exact-fallback, 2 naive; diagnosis: -1 none, 0 feasible,
 * 1 too_little_compute, 2 imbalanced */
int or_greedy_order(const double* alphas, int T, double beta, int K, int* order,
                    int* feasible, int* diagnosis);
int or_exact_order(const double* alphas, int T, double beta, int K, int max_T,
                   int* order, int* feasible, int* diagnosis);
int or_auto_order(const double* alphas, int T, double beta, int K, int max_T,
                  int* order, int* feasible, int* diagnosis, int* method);
int or_diagnose(const double* alphas, int T, double beta, int K, int max_T);
uint64_t or_instance_digest(const double* alphas, int T, double beta, int K);
/* brute-force permutation oracle (verification.hpp:50-72), T <= 9 */
int or_enumerate_feasibility(const double* alphas, int T, double beta, int K,
                             int* witness);

/* ---- simulator.hpp ------------------------------------------------------- */
typedef struct {
  int stream; /* 0 load, 1 compute */
  int layer_id;
  int expert_id;
  double start, end;
} or_event;
typedef struct {
  double makespan, compute_busy, load_busy, compute_stall;
  int peak_resident;
  double overlap_efficiency;
} or_report;
/* orders: concatenated per-layer permutations; alphas concatenated; betas per
 * layer.  mode 0 overlapped, 1 serial. */
int or_run_layers(int n_layers, const int* T, const int* orders, const double* alphas,
                  const double* betas, int K, int mode, int continuous, or_event* ev,
                  or_report* rep, double* layer_stall, int* layer_peak);
double or_lower_bound(const double* alphas, int T, double beta);
/* replay_check (verification.hpp:108-198) on one layer set; returns number of
 * violations, kinds[] histogram indexed by verification.hpp:74-81 order. */
int or_replay_check(const or_event* ev, int n_ev, int n_layers, const int* T,
                    const double* alphas, const double* betas, int K,
                    int check_durations, int* kinds6);

/* ---- MoE layer forward (parity UNPINNED by the reference) --------------- */
/* softmax/top-k gate.  logits[t][e] = x[t] . wg[e] in fp32 in the gate
 * kernel's warp order: 32 lane-partial fmaf chains (lane l owns columns
 * 8l..8l+7 of every 256-column chunk, ascending, zero-padded to the chunk),
 * combined by the butterfly p[l] += p[l^off], off = 16..1; then + bias[e] (one
 * fp32 add).  top-k
 * by repeated strict-greater argmax (ties -> lower expert index, NaN never
 * wins; all-NaN -> expert 0 then 1).  Weights: softmax probabilities in fp64,
 * renormalised over the k picks when k > 1. */
void or_gate_softmax(const float* x, uint64_t N, int d, const float* wg,
                     const float* bias, int E, int k, int32_t* topk_idx,
                     float* topk_w, int32_t* counts);
/* LSH gate on the fp64 promotion of x (gating.hpp:61-104), weight 1.0 */
void or_gate_lsh(const float* x, uint64_t N, int d, const double* proj, int bits,
                 int E, int32_t* topk_idx, float* topk_w, int32_t* counts);
/* stable counting sort of the N*k assignments by expert (token-major order
 * within an expert).  offsets[E+1]; perm[pos] = assignment index t*k+j;
 * inv[t*k+j] = pos. */
void or_dispatch(const int32_t* topk_idx, uint64_t N, int k, int E, int32_t* offsets,
                 int32_t* perm, int32_t* inv);
/* expert FFN on the rows of one expert: y = GeLU_erf(x . W_in^T) . W_out^T.
 * x rows [n, d] fp32 (bf16-exact), W_in [f, d], W_out [d, f] (bf16-exact fp32),
 * fp64 accumulation, H rounded to bf16 (round_h=1) as the device path stores
 * it, output fp32 (caller rounds).  Threads: OpenMP over rows when available. */
void or_expert_ffn(const float* x, uint64_t n, int d, int f, const float* w_in,
                   const float* w_out, int round_h, float* y);
/* cpu_ffn.c — the CPU BASELINE's FFN (bench.py only; not a parity oracle):
 * bf16 rows x [n, d], W_in [f, d], W_out [d, f] read in place, fp32
 * accumulation (AVX512-BF16 dot products when the host has them), h [n, f]
 * bf16 scratch = bf16(gelu_erf(.)), y [n, d] fp32. */
void or_expert_ffn_bf16(const uint16_t* x, uint64_t n, int d, int f, const uint16_t* w_in,
                        const uint16_t* w_out, uint16_t* h, float* y);
/* 1 when or_expert_ffn_bf16 runs on AVX512-BF16 (vdpbf16ps), 0 generic fp32 */
int or_cpu_ffn_isa(void);
/* full layer in one call (gate -> dispatch -> FFN -> combine) */
void or_combine(const float* y_perm, const int32_t* inv, const float* topk_w,
                uint64_t N, int k, int d, float* y);
double or_gelu(double v);

#ifdef __cplusplus
}
#endif
#endif
