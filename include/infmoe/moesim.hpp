// infmoe/moesim.hpp — drop-in C++ mirror of the reference moesim scheduler API
// (/root/reference/proj/include/moesim/{model_config,cost_model,scheduler,
// simulator}.hpp) implemented over the libinfmoe C-ABI (include/infmoe.h).
//
// A moesim user switches by replacing `#include "moesim/scheduler.hpp"` (etc.)
// with `#include "infmoe/moesim.hpp"` and `namespace moesim` with
// `namespace infmoe::moesim` (or a using-directive); types, function names,
// argument meaning, return values and exceptions (ConfigError, CapacityError,
// InvariantError, std::invalid_argument) are the reference's.  Results are
// bit-identical (tests/test_planner_parity.py, tests/cpp/test_moesim_compat.cpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <filesystem>
#include <map>
#include <numbers>
#include <optional>
#include <random>
#include <string_view>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "infmoe.h"

namespace infmoe::moesim {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvariantError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == INFMOE_OK) return;
  const std::string msg = infmoe_last_error();
  switch (rc) {
    case INFMOE_ERR_CONFIG: throw ConfigError(msg);
    case INFMOE_ERR_CAPACITY: throw CapacityError(msg);
    case INFMOE_ERR_ARGUMENT: throw std::invalid_argument(msg);
    case INFMOE_ERR_INVARIANT: throw InvariantError(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// ---- tolerance.hpp ---------------------------------------------------------
// the one comparison rule of the scheduler / simulator (tolerance.hpp:10-23)
inline constexpr double kRelTol = 1e-9;
inline constexpr double kAbsTol = 1e-15;
inline double cmp_tol(double a, double b) {
  return std::max(kAbsTol, kRelTol * std::max(std::fabs(a), std::fabs(b)));
}
inline bool approx_geq(double a, double b) { return a >= b - cmp_tol(a, b); }
inline bool approx_leq(double a, double b) { return a <= b + cmp_tol(a, b); }
inline bool approx_eq(double a, double b) { return std::fabs(a - b) <= cmp_tol(a, b); }
inline bool definitely_lt(double a, double b) { return !approx_geq(a, b); }

// ---- model_config.hpp ----------------------------------------------------
struct ModelGeometry {
  int n_layers = 0, n_heads = 0, d_head = 0, d_model = 0, d_ff = 0, n_experts_per_layer = 0,
      bytes_per_param = 0;
};
struct HardwareProfile {
  double peak_flops = 0.0, h2d_bandwidth = 0.0;
  std::uint64_t device_memory = 0, reserved_memory = 0;
};
namespace detail {
inline infmoe_geometry c(const ModelGeometry& g) {
  return {g.n_layers, g.n_heads, g.d_head, g.d_model, g.d_ff, g.n_experts_per_layer,
          g.bytes_per_param};
}
inline infmoe_hardware c(const HardwareProfile& h) {
  return {h.peak_flops, h.h2d_bandwidth, h.device_memory, h.reserved_memory};
}
}  // namespace detail
inline std::vector<std::string> validate(const ModelGeometry& g) {
  const infmoe_geometry cg = detail::c(g);
  int32_t warn = 0;
  detail::check(infmoe_validate_geometry(&cg, &warn));
  if (!warn) return {};
  return {"geometry: d_model (" + std::to_string(g.d_model) + ") != n_heads * d_head (" +
          std::to_string(g.n_heads * g.d_head) + ")"};
}
inline std::vector<std::string> validate(const HardwareProfile& hw) {
  const infmoe_hardware ch = detail::c(hw);
  detail::check(infmoe_validate_hardware(&ch));
  return {};
}
inline std::uint64_t expert_param_bytes(const ModelGeometry& g) {
  const infmoe_geometry cg = detail::c(g);
  return infmoe_expert_param_bytes(&cg);
}
inline std::uint64_t expert_flops(const ModelGeometry& g, std::uint64_t n_tokens) {
  const infmoe_geometry cg = detail::c(g);
  return infmoe_expert_flops(&cg, n_tokens);
}
inline const std::map<std::string, ModelGeometry>& builtin_geometry_presets() {
  static const std::map<std::string, ModelGeometry> presets = [] {
    std::map<std::string, ModelGeometry> m;
    for (const char* name : {"cpm2", "cpm-small"}) {
      infmoe_geometry g;
      detail::check(infmoe_geometry_preset(name, &g));
      m[name] = ModelGeometry{g.n_layers, g.n_heads, g.d_head, g.d_model, g.d_ff,
                              g.n_experts_per_layer, g.bytes_per_param};
    }
    return m;
  }();
  return presets;
}

// ---- prng.hpp -------------------------------------------------------------
inline constexpr std::string_view kPrngName = "mt19937_64/box-muller/v1";
inline std::uint64_t splitmix64(std::uint64_t x) { return infmoe_splitmix64(x); }
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) {
  return infmoe_derive_seed(seed, tag);
}
// The stream contract itself (prng.hpp:32-71): 53-bit uniforms and Box-Muller
// with a cached spare over std::mt19937_64, whose output sequence is
// standardised -- the library's generators produce the same values.
inline double uniform01(std::mt19937_64& rng) {
  return static_cast<double>(rng() >> 11) * 0x1.0p-53;
}
inline double uniform01_open0(std::mt19937_64& rng) {
  return (static_cast<double>(rng() >> 11) + 1.0) * 0x1.0p-53;
}
inline std::uint64_t uniform_below(std::mt19937_64& rng, std::uint64_t n) {
  return static_cast<std::uint64_t>(uniform01(rng) * static_cast<double>(n)) % n;
}
class GaussianStream {
 public:
  explicit GaussianStream(std::uint64_t seed) : rng_(seed) {}
  double next() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    const double u1 = uniform01_open0(rng_);
    const double u2 = uniform01(rng_);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * std::numbers::pi * u2;
    spare_ = r * std::sin(theta);
    has_spare_ = true;
    return r * std::cos(theta);
  }

 private:
  std::mt19937_64 rng_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// ---- gating.hpp -----------------------------------------------------------
struct ExpertWorkload {
  int layer_id = 0;
  std::vector<std::uint64_t> token_counts;
  std::uint64_t total_tokens = 0;
};
inline void validate(const ExpertWorkload& w) {
  std::uint64_t sum = 0;
  for (std::uint64_t c : w.token_counts) sum += c;
  if (sum != w.total_tokens)
    throw ConfigError("workload: token_counts sum to " + std::to_string(sum) +
                      ", expected total_tokens = " + std::to_string(w.total_tokens));
  if (w.token_counts.empty()) throw ConfigError("workload: no experts");
}
struct GatingModel {
  std::uint64_t projection_seed = 0;
  int n_hash_bits = 5;
  int hidden_dim = 0;
};
inline std::vector<double> gating_projection(const GatingModel& m) {
  std::vector<double> p(m.n_hash_bits > 0 && m.hidden_dim > 0
                            ? std::size_t(m.n_hash_bits) * std::size_t(m.hidden_dim)
                            : 0);
  detail::check(infmoe_gating_projection(m.projection_seed, m.n_hash_bits, m.hidden_dim,
                                         p.data()));
  return p;
}
inline std::vector<std::uint32_t> lsh_codes(const GatingModel& m,
                                            std::span<const double> hidden_states,
                                            std::size_t n_tokens) {
  if (hidden_states.size() != n_tokens * static_cast<std::size_t>(m.hidden_dim))
    throw std::invalid_argument("lsh_codes: hidden_states size != n_tokens * hidden_dim");
  std::vector<std::uint32_t> codes(n_tokens, 0);
  detail::check(infmoe_lsh_codes(m.projection_seed, m.n_hash_bits, m.hidden_dim,
                                 hidden_states.data(), n_tokens, codes.data()));
  return codes;
}
inline ExpertWorkload route_tokens(const GatingModel& m, std::span<const double> hidden_states,
                                   std::size_t n_tokens, int n_experts, int layer_id = 0) {
  if (n_experts < 1) throw std::invalid_argument("route_tokens: n_experts must be >= 1");
  if (m.n_hash_bits >= 0 &&
      (1u << std::min(m.n_hash_bits, 31)) < static_cast<std::uint32_t>(n_experts))
    throw ConfigError("gating: 2^n_hash_bits must be >= n_experts");
  if (hidden_states.size() != n_tokens * static_cast<std::size_t>(m.hidden_dim))
    throw std::invalid_argument("lsh_codes: hidden_states size != n_tokens * hidden_dim");
  ExpertWorkload w;
  w.layer_id = layer_id;
  w.token_counts.assign(std::size_t(n_experts), 0);
  detail::check(infmoe_route_tokens(m.projection_seed, m.n_hash_bits, m.hidden_dim,
                                    hidden_states.data(), n_tokens, n_experts,
                                    w.token_counts.data()));
  w.total_tokens = n_tokens;
  return w;
}
inline std::vector<double> gaussian_tokens(std::uint64_t seed, std::size_t n_tokens, int dim) {
  std::vector<double> out(n_tokens * static_cast<std::size_t>(dim));
  detail::check(infmoe_gaussian_fill(seed, out.data(), out.size()));
  return out;
}
enum class SyntheticKind { Uniform, Zipf, Balanced };
inline ExpertWorkload synthetic_workload(SyntheticKind kind, std::uint64_t total_tokens,
                                         int n_experts, std::uint64_t seed,
                                         double zipf_s = 1.0, int layer_id = 0) {
  ExpertWorkload w;
  w.layer_id = layer_id;
  w.total_tokens = total_tokens;
  w.token_counts.assign(n_experts > 0 ? std::size_t(n_experts) : 1, 0);
  const int k = kind == SyntheticKind::Uniform ? 0 : (kind == SyntheticKind::Zipf ? 1 : 2);
  detail::check(infmoe_synthetic_workload(k, total_tokens, n_experts, seed, zipf_s,
                                          w.token_counts.data()));
  return w;
}
inline ExpertWorkload explicit_workload(std::vector<std::uint64_t> counts, int layer_id = 0) {
  ExpertWorkload w;
  w.layer_id = layer_id;
  detail::check(infmoe_explicit_workload(counts.data(), int32_t(counts.size()),
                                         &w.total_tokens));
  w.token_counts = std::move(counts);
  return w;
}
inline ExpertWorkload workload_from_csv(const std::filesystem::path& path, int layer_id = 0) {
  int32_t n = 0;
  uint64_t total = 0;
  const std::string p = path.string();
  detail::check(infmoe_workload_from_csv(p.c_str(), nullptr, 0, &n, &total));
  std::vector<std::uint64_t> counts(std::size_t(n), 0);
  detail::check(infmoe_workload_from_csv(p.c_str(), counts.data(), n, &n, &total));
  return explicit_workload(std::move(counts), layer_id);
}

// ---- cost_model.hpp -------------------------------------------------------
struct CostVector {
  std::vector<double> alphas;
  double beta = 0.0;
  int size() const { return static_cast<int>(alphas.size()); }
  double total_alpha() const {
    double s = 0.0;
    for (double a : alphas) s += a;
    return s;
  }
};
inline CostVector compute_costs(const ExpertWorkload& w, const ModelGeometry& g,
                                const HardwareProfile& hw) {
  const infmoe_geometry cg = detail::c(g);
  const infmoe_hardware ch = detail::c(hw);
  CostVector c;
  c.alphas.resize(w.token_counts.size());
  detail::check(infmoe_compute_costs(&cg, &ch, w.token_counts.data(),
                                     int32_t(w.token_counts.size()), c.alphas.data(), &c.beta));
  return c;
}
inline int resident_capacity(const ModelGeometry& g, const HardwareProfile& hw) {
  const infmoe_geometry cg = detail::c(g);
  const infmoe_hardware ch = detail::c(hw);
  int32_t K = 0;
  detail::check(infmoe_resident_capacity(&cg, &ch, &K));
  return K;
}
inline int clamp_explicit_capacity(int explicit_k, int capacity,
                                   std::vector<std::string>& warnings) {
  int32_t K = 0, clamped = 0;
  detail::check(infmoe_clamp_explicit_capacity(explicit_k, capacity, &K, &clamped));
  if (clamped)
    warnings.push_back("K clamped from " + std::to_string(explicit_k) + " to capacity " +
                       std::to_string(capacity));
  return K;
}
inline CostVector with_event_overhead(CostVector c, double eps) {
  detail::check(infmoe_with_event_overhead(c.alphas.data(), c.size(), &c.beta, eps));
  return c;
}

// ---- scheduler.hpp --------------------------------------------------------
enum class Diagnosis { Feasible, TooLittleCompute, Imbalanced };
enum class ScheduleMethod { Greedy, ExactFallback, Naive };
enum class BoundSide { Lower, Upper };
struct ConstraintViolation {
  int position = 0;
  BoundSide bound = BoundSide::Lower;
  double prefix_sum = 0.0;
  double limit = 0.0;
};
struct ConstraintReport {
  bool feasible = false;
  std::vector<double> slack;
  std::optional<ConstraintViolation> first_violation;
};
struct Schedule {
  std::vector<int> order;
  bool feasible = false;
  std::vector<double> slack;
  std::optional<Diagnosis> diagnosis;
  ScheduleMethod method = ScheduleMethod::Greedy;
};
inline ConstraintReport check_constraints(std::span<const int> order, const CostVector& costs,
                                          int K) {
  ConstraintReport r;
  if (int(order.size()) != costs.size())
    throw std::invalid_argument("order size " + std::to_string(order.size()) +
                                " != expert count " + std::to_string(costs.size()));
  r.slack.resize(order.size());
  infmoe_constraint_report rep;
  std::vector<int32_t> o(order.begin(), order.end());
  detail::check(infmoe_check_constraints(o.data(), costs.alphas.data(), costs.size(), costs.beta,
                                         K, r.slack.data(), &rep));
  r.feasible = rep.feasible != 0;
  if (!r.feasible)
    r.first_violation = ConstraintViolation{
        rep.position, rep.bound == INFMOE_BOUND_LOWER ? BoundSide::Lower : BoundSide::Upper,
        rep.prefix_sum, rep.limit};
  return r;
}
namespace detail {
inline Schedule schedule(const CostVector& c, int K, int policy, int max_T) {
  Schedule s;
  s.order.resize(c.alphas.size());
  s.slack.resize(c.alphas.size());
  std::vector<int32_t> o(c.alphas.size());
  infmoe_schedule_info info;
  check(infmoe_schedule(c.alphas.data(), c.size(), c.beta, K, policy, max_T, o.data(),
                        s.slack.data(), &info));
  s.order.assign(o.begin(), o.end());
  s.feasible = info.feasible != 0;
  if (info.diagnosis >= 0) s.diagnosis = static_cast<Diagnosis>(info.diagnosis);
  s.method = static_cast<ScheduleMethod>(info.method);
  return s;
}
}  // namespace detail
inline Schedule naive_order(const CostVector& c, int K) {
  return detail::schedule(c, K, INFMOE_POLICY_NAIVE, 12);
}
inline Schedule greedy_order(const CostVector& c, int K) {
  return detail::schedule(c, K, INFMOE_POLICY_GREEDY, 12);
}
inline Schedule exact_order(const CostVector& c, int K, int max_T = 12) {
  return detail::schedule(c, K, INFMOE_POLICY_EXACT, max_T);
}
inline Schedule auto_order(const CostVector& c, int K, int exact_fallback_max_T = 12) {
  return detail::schedule(c, K, INFMOE_POLICY_AUTO, exact_fallback_max_T);
}
inline Diagnosis diagnose(const CostVector& c, int K, int exact_fallback_max_T = 12) {
  int32_t d = 0;
  detail::check(infmoe_diagnose(c.alphas.data(), c.size(), c.beta, K, exact_fallback_max_T, &d));
  return static_cast<Diagnosis>(d);
}

// ---- simulator.hpp --------------------------------------------------------
enum class StreamKind { Load, Compute };
enum class SimMode { Overlapped, Serial };
enum class OrderPolicy { Greedy, Naive, Exact };
struct TimelineEvent {
  StreamKind stream = StreamKind::Load;
  int layer_id = 0;
  int expert_id = 0;
  double start = 0.0;
  double end = 0.0;
};
struct LayerReport {
  int layer_id = 0;
  int n_experts = 0;
  double start = 0.0;
  double end = 0.0;
  double compute_busy = 0.0;
  double load_busy = 0.0;
  double compute_stall = 0.0;
  int peak_resident = 0;
  double lower_bound = 0.0;
  Schedule schedule;
};
struct SimReport {
  double makespan = 0.0, compute_busy = 0.0, load_busy = 0.0, compute_stall = 0.0;
  int peak_resident_experts = 0;
  double overlap_efficiency = 0.0;
  std::vector<LayerReport> per_layer;
};
struct ModelSimOptions {
  SimMode mode = SimMode::Overlapped;
  OrderPolicy policy = OrderPolicy::Greedy;
  bool continuous_load_stream = false;
  int exact_max_T = 12;
};
inline double lower_bound(const CostVector& c) {
  return infmoe_lower_bound(c.alphas.data(), c.size(), c.beta);
}
inline Schedule order_for_policy(const CostVector& costs, int K, OrderPolicy policy,
                                 int exact_max_T = 12) {
  switch (policy) {
    case OrderPolicy::Greedy: return auto_order(costs, K, exact_max_T);
    case OrderPolicy::Naive: return naive_order(costs, K);
    case OrderPolicy::Exact: return exact_order(costs, K, exact_max_T);
  }
  throw std::invalid_argument("unknown policy");
}
namespace detail {
// the recurrence of simulator.hpp:102-194 on fixed schedules (one per layer)
inline std::pair<std::vector<TimelineEvent>, SimReport> run(
    std::span<const Schedule> schedules, std::span<const CostVector> costs, int K, SimMode mode,
    bool continuous) {
  std::vector<int32_t> T, orders;
  std::vector<double> alphas, betas;
  for (std::size_t l = 0; l < costs.size(); ++l) {
    T.push_back(costs[l].size());
    alphas.insert(alphas.end(), costs[l].alphas.begin(), costs[l].alphas.end());
    betas.push_back(costs[l].beta);
    if (int(schedules[l].order.size()) != costs[l].size())
      throw std::invalid_argument("order size " + std::to_string(schedules[l].order.size()) +
                                  " != expert count " + std::to_string(costs[l].size()));
    orders.insert(orders.end(), schedules[l].order.begin(), schedules[l].order.end());
  }
  std::vector<infmoe_event> ev(2 * alphas.size());
  std::vector<infmoe_layer_report> pl(costs.size());
  infmoe_sim_report r;
  check(infmoe_simulate_orders(int32_t(T.size()), T.data(), orders.data(), alphas.data(),
                               betas.data(), K,
                               mode == SimMode::Overlapped ? INFMOE_MODE_OVERLAPPED
                                                           : INFMOE_MODE_SERIAL,
                               continuous ? 1 : 0, ev.data(), &r, pl.data()));
  std::vector<TimelineEvent> out;
  out.reserve(ev.size());
  for (const auto& e : ev)
    out.push_back({e.stream == INFMOE_STREAM_LOAD ? StreamKind::Load : StreamKind::Compute,
                   e.layer_id, e.expert_id, e.start, e.end});
  SimReport rep{r.makespan, r.compute_busy, r.load_busy, r.compute_stall,
                r.peak_resident_experts, r.overlap_efficiency, {}};
  for (std::size_t l = 0; l < pl.size(); ++l)
    rep.per_layer.push_back({pl[l].layer_id, pl[l].n_experts, pl[l].start, pl[l].end,
                             pl[l].compute_busy, pl[l].load_busy, pl[l].compute_stall,
                             pl[l].peak_resident, pl[l].lower_bound, schedules[l]});
  return {std::move(out), std::move(rep)};
}
}  // namespace detail
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate(
    const Schedule& schedule, const CostVector& costs, int K,
    SimMode mode = SimMode::Overlapped) {
  return detail::run(std::span<const Schedule>(&schedule, 1),
                     std::span<const CostVector>(&costs, 1), K, mode, false);
}
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate(
    std::span<const int> order, const CostVector& costs, int K,
    SimMode mode = SimMode::Overlapped) {
  ConstraintReport chk = check_constraints(order, costs, K);
  Schedule s;
  s.order.assign(order.begin(), order.end());
  s.feasible = chk.feasible;
  s.slack = std::move(chk.slack);
  s.method = ScheduleMethod::Naive;
  return simulate(s, costs, K, mode);
}
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate_model(
    std::span<const CostVector> layer_costs, int K, const ModelSimOptions& opt) {
  if (layer_costs.empty()) throw std::invalid_argument("simulate_model: no layers");
  std::vector<Schedule> schedules;
  schedules.reserve(layer_costs.size());
  for (const CostVector& c : layer_costs)
    schedules.push_back(order_for_policy(c, K, opt.policy, opt.exact_max_T));
  return detail::run(schedules, layer_costs, K, opt.mode, opt.continuous_load_stream);
}
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate_model(
    std::span<const ExpertWorkload> workloads, const ModelGeometry& geometry,
    const HardwareProfile& hw, int K, const ModelSimOptions& opt) {
  std::vector<CostVector> costs;
  costs.reserve(workloads.size());
  for (const ExpertWorkload& w : workloads) costs.push_back(compute_costs(w, geometry, hw));
  return simulate_model(costs, K, opt);
}
inline std::string to_string(StreamKind s) { return s == StreamKind::Load ? "load" : "compute"; }
inline std::string to_string(SimMode m) {
  return m == SimMode::Overlapped ? "overlapped" : "serial";
}

// ---- scenario.hpp + the CLI front door -------------------------------------
// The reference's parse_scenario / to_json work on nlohmann::json objects; the
// library exchanges the resolved scenario as JSON text (indent 2, sorted keys:
// byte-identical to the reference's to_json(parse_scenario(...)).dump(2)).
inline std::string resolve_scenario(const std::string& json_text) {
  uint64_t len = 0;
  detail::check(infmoe_scenario_resolve(json_text.c_str(), nullptr, 0, &len));
  std::string out(len, '\0');
  detail::check(infmoe_scenario_resolve(json_text.c_str(), out.data(), len, &len));
  out.resize(len ? len - 1 : 0);
  return out;
}
inline std::string resolve_scenario_file(const std::filesystem::path& path) {
  uint64_t len = 0;
  const std::string p = path.string();
  detail::check(infmoe_scenario_resolve_file(p.c_str(), nullptr, 0, &len));
  std::string out(len, '\0');
  detail::check(infmoe_scenario_resolve_file(p.c_str(), out.data(), len, &len));
  out.resize(len ? len - 1 : 0);
  return out;
}
// run_scenario / sweep: artefacts under opt.out_dir (or the
// scenario's output_dir); returns summary.csv / sweep.csv
inline std::string run_scenario(const std::filesystem::path& path,
                                const infmoe_run_options* opt = nullptr) {
  std::string out(1 << 20, '\0');
  uint64_t len = 0;
  const std::string p = path.string();
  detail::check(infmoe_scenario_run(p.c_str(), opt, out.data(), out.size(), &len));
  out.resize(std::min<uint64_t>(len ? len - 1 : 0, out.size()));
  return out;
}
inline std::string sweep_scenario(const std::filesystem::path& path, const std::string& axis,
                                  const std::vector<double>& values,
                                  const infmoe_run_options* opt = nullptr) {
  std::string out(1 << 20, '\0');
  uint64_t len = 0;
  const std::string p = path.string();
  detail::check(infmoe_scenario_sweep(p.c_str(), axis.c_str(), values.data(),
                                      int32_t(values.size()), opt, out.data(), out.size(),
                                      &len));
  out.resize(std::min<uint64_t>(len ? len - 1 : 0, out.size()));
  return out;
}

}  // namespace infmoe::moesim
