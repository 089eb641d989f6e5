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

#include <cstdint>
#include <optional>
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

// ---- gating.hpp (workload) ------------------------------------------------
struct ExpertWorkload {
  int layer_id = 0;
  std::vector<std::uint64_t> token_counts;
  std::uint64_t total_tokens = 0;
};
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
struct SimReport {
  double makespan = 0.0, compute_busy = 0.0, load_busy = 0.0, compute_stall = 0.0;
  int peak_resident_experts = 0;
  double overlap_efficiency = 0.0;
};
struct ModelSimOptions {
  SimMode mode = SimMode::Overlapped;
  OrderPolicy policy = OrderPolicy::Greedy;
  bool continuous_load_stream = false;
  int exact_max_T = 12;
};
namespace detail {
inline std::pair<std::vector<TimelineEvent>, SimReport> unpack(
    const std::vector<infmoe_event>& ev, const infmoe_sim_report& r) {
  std::vector<TimelineEvent> out;
  out.reserve(ev.size());
  for (const auto& e : ev)
    out.push_back({e.stream == INFMOE_STREAM_LOAD ? StreamKind::Load : StreamKind::Compute,
                   e.layer_id, e.expert_id, e.start, e.end});
  return {std::move(out), SimReport{r.makespan, r.compute_busy, r.load_busy, r.compute_stall,
                                    r.peak_resident_experts, r.overlap_efficiency}};
}
}  // namespace detail
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate(
    std::span<const int> order, const CostVector& costs, int K,
    SimMode mode = SimMode::Overlapped) {
  std::vector<int32_t> o(order.begin(), order.end());
  std::vector<infmoe_event> ev(2 * o.size());
  infmoe_sim_report r;
  detail::check(infmoe_simulate(o.data(), costs.alphas.data(), costs.size(), costs.beta, K,
                                mode == SimMode::Overlapped ? INFMOE_MODE_OVERLAPPED
                                                            : INFMOE_MODE_SERIAL,
                                ev.data(), &r));
  return detail::unpack(ev, r);
}
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate(
    const Schedule& s, const CostVector& costs, int K, SimMode mode = SimMode::Overlapped) {
  return simulate(std::span<const int>(s.order), costs, K, mode);
}
inline std::pair<std::vector<TimelineEvent>, SimReport> simulate_model(
    std::span<const CostVector> layer_costs, int K, const ModelSimOptions& opt) {
  std::vector<int32_t> T;
  std::vector<double> alphas, betas;
  for (const auto& c : layer_costs) {
    T.push_back(c.size());
    alphas.insert(alphas.end(), c.alphas.begin(), c.alphas.end());
    betas.push_back(c.beta);
  }
  std::vector<int32_t> orders(alphas.size());
  std::vector<infmoe_event> ev(2 * alphas.size());
  infmoe_sim_report r;
  const int pol = opt.policy == OrderPolicy::Greedy
                      ? INFMOE_POLICY_AUTO
                      : (opt.policy == OrderPolicy::Naive ? INFMOE_POLICY_NAIVE
                                                          : INFMOE_POLICY_EXACT);
  detail::check(infmoe_simulate_model(
      int32_t(T.size()), T.data(), alphas.data(), betas.data(), K,
      opt.mode == SimMode::Overlapped ? INFMOE_MODE_OVERLAPPED : INFMOE_MODE_SERIAL, pol,
      opt.continuous_load_stream ? 1 : 0, opt.exact_max_T, orders.data(), ev.data(), &r,
      nullptr));
  return detail::unpack(ev, r);
}
inline double lower_bound(const CostVector& c) {
  return infmoe_lower_bound(c.alphas.data(), c.size(), c.beta);
}

}  // namespace infmoe::moesim
