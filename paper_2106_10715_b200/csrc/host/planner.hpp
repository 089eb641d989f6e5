// planner.hpp — host-side planning layer of the offloaded MoE path:
// synthetic-input PRNG, geometry/hardware, cost model (α, β, K), the InfMoE
// prefix-band scheduler and the two-lane timeline recurrence that the CUDA
// executor realises.  Written from the paper and SPEC.md;
// results are bit-identical to the reference moesim headers (checked by
// tests/test_planner_parity.py against oracle/_ref and tests/golden/).
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <vector>

namespace infmoe {

// ---------------------------------------------------------------- PRNG ----
// prng.hpp:18-71 stream contract "mt19937_64/box-muller/v1".
std::uint64_t mix64(std::uint64_t x);                       // splitmix64
std::uint64_t child_seed(std::uint64_t seed, std::uint64_t tag);  // derive_seed
void normal_draws(std::uint64_t seed, double* out, std::uint64_t n);
// n_mats independent streams normal_draws(seeds[m]) x scales[m], rounded to
// dtype (0 bf16: double -> f32 RN -> bf16 RNE; 1 f32: double -> f32 RN; 2 f64), n_each
// values into outs[m]; `threads` host threads (<= 0: all)
void normal_fill_typed(int dtype, int n_mats, const std::uint64_t* seeds, const double* scales,
                       std::uint64_t n_each, void* const* outs, int threads);

// ------------------------------------------------------------ geometry ----
struct Geometry {  // model_config.hpp:14-22
  int n_layers = 0, n_heads = 0, d_head = 0, d_model = 0, d_ff = 0, experts = 0,
      bytes_per_param = 0;
};
struct Hardware {  // model_config.hpp:27-32
  double peak_flops = 0.0, h2d_bandwidth = 0.0;
  std::uint64_t device_memory = 0, reserved_memory = 0;
};
bool check_geometry(const Geometry& g);  // returns the d_model != heads*d_head warning
void check_hardware(const Hardware& hw);
std::uint64_t bytes_per_expert(const Geometry& g);
std::uint64_t flops_for_tokens(const Geometry& g, std::uint64_t tokens);
bool preset(const std::string& name, Geometry* out);

// --------------------------------------------------------------- gating ---
std::vector<double> lsh_hyperplanes(std::uint64_t seed, int bits, int hidden);
// lsh_codes gating.hpp:61-82 on host fp64 rows (bit-exact, threads over tokens)
void lsh_codes_host(std::uint64_t seed, int bits, int hidden, const double* x,
                    std::uint64_t n_tokens, std::uint32_t* codes);
// explicit_workload's validation (gating.hpp:25-33): returns the total
std::uint64_t explicit_total(const std::uint64_t* counts, int n);
// workload_from_csv gating.hpp:180-219: per-expert counts
std::vector<std::uint64_t> workload_csv(const std::string& path);
std::vector<std::uint64_t> workload_counts(int kind, std::uint64_t total, int experts,
                                           std::uint64_t seed, double zipf_s);

// ----------------------------------------------------------- cost model ---
struct Costs {  // α per expert (s), uniform β (s)
  std::vector<double> alpha;
  double beta = 0.0;
  int size() const { return static_cast<int>(alpha.size()); }
  double alpha_sum() const;
};
void check_costs(const Costs& c);
Costs derive_costs(const std::uint64_t* counts, int n, const Geometry& g, const Hardware& hw);
int capacity_slots(const Geometry& g, const Hardware& hw);

// ------------------------------------------------------------ scheduler ---
enum class Verdict { None = -1, Feasible = 0, TooLittleCompute = 1, Imbalanced = 2 };
enum class Method { Greedy = 0, ExactFallback = 1, Naive = 2 };
struct BandCheck {
  bool feasible = true;
  std::vector<double> slack;
  int position = -1;
  int side = -1;  // 0 lower, 1 upper
  double prefix = 0.0, limit = 0.0;
};
struct Plan {
  std::vector<int> order;
  bool feasible = false;
  std::vector<double> slack;
  Verdict verdict = Verdict::None;
  Method method = Method::Greedy;
};
BandCheck band_check(std::span<const int> order, const Costs& c, int K);
Plan plan_greedy(const Costs& c, int K);
Plan plan_exact(const Costs& c, int K, int max_T);
Plan plan_auto(const Costs& c, int K, int max_T);
Plan plan_identity(const Costs& c, int K);
Verdict classify(const Costs& c, int K, int max_T);

// ------------------------------------------------------------- timeline ---
struct Event {
  int stream;  // 0 load, 1 compute
  int layer, expert;
  double start, end;
};
struct LayerStats {
  int layer = 0, experts = 0;
  double start = 0, end = 0, compute_busy = 0, load_busy = 0, compute_stall = 0;
  int peak_resident = 0;
  double lower_bound = 0;
};
struct TimelineStats {
  double makespan = 0, compute_busy = 0, load_busy = 0, compute_stall = 0;
  int peak_resident = 0;
  double overlap_efficiency = 0;
  std::vector<LayerStats> layers;
};
double makespan_floor(const Costs& c);
// Two-lane recurrence (load lane, compute lane) over layers in sequence.
TimelineStats run_timeline(std::span<const std::vector<int>> orders,
                           std::span<const Costs> costs, int K, bool serial,
                           bool continuous_loads, std::vector<Event>* events);

// Timeline audit for measured (or simulated) event lists; kinds[6] counts
// overlap, causality, residency, duration, makespan, malformed violations.
int audit_timeline(const std::vector<Event>& ev, std::span<const Costs> costs, int max_resident,
                   bool check_durations, double tol_s, int kinds[6]);

}  // namespace infmoe
