// ref_driver.cpp — TEST INFRASTRUCTURE.  A thin extern "C" shim that compiles
// the UNMODIFIED reference headers (/root/reference/proj/include/moesim/*.hpp,
// included in place via -I, never copied) into oracle/_ref/libmoesim_ref.so so
// tests and bench.py's reference arm can call the reference itself.
// Build recipe: oracle/Makefile (target _ref/libmoesim_ref.so).
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <vector>

#include "moesim/cost_model.hpp"
#include "moesim/gating.hpp"
#include "moesim/model_config.hpp"
#include "moesim/prng.hpp"
#include "moesim/scheduler.hpp"
#include "moesim/simulator.hpp"
#include "moesim/verification.hpp"

using namespace moesim;

namespace {
CostVector make_costs(const double* a, int T, double beta) {
  CostVector c;
  c.alphas.assign(a, a + T);
  c.beta = beta;
  return c;
}
int diag_code(const Schedule& s) {
  if (!s.diagnosis) return -1;
  switch (*s.diagnosis) {
    case Diagnosis::Feasible: return 0;
    case Diagnosis::TooLittleCompute: return 1;
    case Diagnosis::Imbalanced: return 2;
  }
  return -1;
}
int method_code(ScheduleMethod m) {
  return m == ScheduleMethod::Greedy ? 0 : (m == ScheduleMethod::ExactFallback ? 1 : 2);
}
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const CapacityError&) {
    return 3;
  } catch (const InvariantError&) {
    return 4;
  } catch (const ConfigError&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (...) {
    return 9;
  }
}
}  // namespace

extern "C" {

uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ref_derive_seed(uint64_t s, uint64_t t) { return derive_seed(s, t); }
uint64_t ref_mt64_first(uint64_t seed) {
  std::mt19937_64 r(seed);
  return r();
}
void ref_gaussian_tokens(uint64_t seed, uint64_t n_tokens, int dim, double* out) {
  auto v = gaussian_tokens(seed, n_tokens, dim);
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}
int ref_gating_projection(uint64_t seed, int bits, int hidden, double* out) {
  return guard([&] {
    auto v = gating_projection(GatingModel{seed, bits, hidden});
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}
int ref_lsh_codes(uint64_t seed, int bits, int hidden, const double* x, uint64_t n,
                  uint32_t* codes) {
  return guard([&] {
    auto v = lsh_codes(GatingModel{seed, bits, hidden},
                       std::span<const double>(x, n * (uint64_t)hidden), n);
    std::memcpy(codes, v.data(), v.size() * sizeof(uint32_t));
  });
}
int ref_route_tokens(uint64_t seed, int bits, int hidden, const double* x, uint64_t n,
                     int E, uint64_t* counts) {
  return guard([&] {
    auto w = route_tokens(GatingModel{seed, bits, hidden},
                          std::span<const double>(x, n * (uint64_t)hidden), n, E);
    std::memcpy(counts, w.token_counts.data(), sizeof(uint64_t) * E);
  });
}
// workload_from_csv / explicit_workload (gating.hpp:167-219); returns the
// guard code (2 = ConfigError); counts receives up to cap entries
int ref_workload_from_csv(const char* path, uint64_t* counts, int cap, int* n_experts,
                          uint64_t* total) {
  return guard([&] {
    auto w = workload_from_csv(path);
    *n_experts = int(w.token_counts.size());
    *total = w.total_tokens;
    for (int e = 0; e < *n_experts && e < cap; ++e) counts[e] = w.token_counts[size_t(e)];
  });
}
int ref_explicit_workload(const uint64_t* counts, int n, uint64_t* total) {
  return guard([&] {
    auto w = explicit_workload(std::vector<uint64_t>(counts, counts + n));
    *total = w.total_tokens;
  });
}
int ref_synthetic_workload(int kind, uint64_t total, int E, uint64_t seed, double s,
                           uint64_t* counts) {
  return guard([&] {
    SyntheticKind k = kind == 0 ? SyntheticKind::Uniform
                                : (kind == 1 ? SyntheticKind::Zipf : SyntheticKind::Balanced);
    auto w = synthetic_workload(k, total, E, seed, s);
    std::memcpy(counts, w.token_counts.data(), sizeof(uint64_t) * E);
  });
}
uint64_t ref_expert_param_bytes(int d, int f, int b) {
  ModelGeometry g{1, 1, 1, d, f, 1, b};
  return expert_param_bytes(g);
}
uint64_t ref_expert_flops(int d, int f, uint64_t n) {
  ModelGeometry g{1, 1, 1, d, f, 1, 2};
  return expert_flops(g, n);
}
int ref_compute_costs(int d, int f, int b, double peak, double bw, const uint64_t* counts,
                      int T, double* alphas, double* beta) {
  return guard([&] {
    ModelGeometry g{1, 1, 1, d, f, T, b};
    HardwareProfile hw{peak, bw, 2, 1};
    ExpertWorkload w = explicit_workload(std::vector<uint64_t>(counts, counts + T));
    CostVector c = compute_costs(w, g, hw);
    std::memcpy(alphas, c.alphas.data(), sizeof(double) * T);
    *beta = c.beta;
  });
}
int ref_resident_capacity(int d, int f, int b, uint64_t dev, uint64_t res, int* K) {
  return guard([&] {
    ModelGeometry g{1, 1, 1, d, f, 1, b};
    HardwareProfile hw{1.0, 1.0, dev, res};
    *K = resident_capacity(g, hw);
  });
}
int ref_check_constraints(const int* order, const double* a, int T, double beta, int K,
                          double* slack, int* feasible, int* vpos, int* vside) {
  return guard([&] {
    auto r = check_constraints(std::span<const int>(order, T), make_costs(a, T, beta), K);
    *feasible = r.feasible;
    for (int i = 0; i < T; ++i) slack[i] = r.slack[i];
    *vpos = r.first_violation ? r.first_violation->position : -1;
    *vside = r.first_violation ? (r.first_violation->bound == BoundSide::Lower ? 0 : 1) : -1;
  });
}
// policy: 0 auto(greedy+fallback), 1 greedy only, 2 exact, 3 naive
int ref_schedule(const double* a, int T, double beta, int K, int policy, int max_T,
                 int* order, int* feasible, int* diagnosis, int* method) {
  return guard([&] {
    CostVector c = make_costs(a, T, beta);
    Schedule s = policy == 0   ? auto_order(c, K, max_T)
                 : policy == 1 ? greedy_order(c, K)
                 : policy == 2 ? exact_order(c, K, max_T)
                               : naive_order(c, K);
    std::memcpy(order, s.order.data(), sizeof(int) * T);
    *feasible = s.feasible;
    *diagnosis = diag_code(s);
    *method = method_code(s.method);
  });
}
int ref_diagnose(const double* a, int T, double beta, int K, int max_T) {
  int out = -2;
  guard([&] {
    Diagnosis d = diagnose(make_costs(a, T, beta), K, max_T);
    out = d == Diagnosis::Feasible ? 0 : (d == Diagnosis::TooLittleCompute ? 1 : 2);
  });
  return out;
}
typedef struct {
  int stream, layer_id, expert_id;
  double start, end;
} ref_event;
typedef struct {
  double makespan, compute_busy, load_busy, compute_stall;
  int peak_resident;
  double overlap_efficiency;
} ref_report;
// Whole-model simulation through simulate_model(costs, K, opt) (simulator.hpp:241).
// policy: 0 greedy(auto), 1 naive, 2 exact.  orders_out receives chosen orders.
int ref_simulate_model(int L, const int* Ts, const double* alphas, const double* betas,
                       int K, int mode, int policy, int continuous, int max_T,
                       int* orders_out, ref_event* ev, ref_report* rep) {
  return guard([&] {
    std::vector<CostVector> cs;
    int off = 0;
    for (int l = 0; l < L; ++l) {
      cs.push_back(make_costs(alphas + off, Ts[l], betas[l]));
      off += Ts[l];
    }
    ModelSimOptions opt;
    opt.mode = mode == 0 ? SimMode::Overlapped : SimMode::Serial;
    opt.policy = policy == 0 ? OrderPolicy::Greedy
                             : (policy == 1 ? OrderPolicy::Naive : OrderPolicy::Exact);
    opt.continuous_load_stream = continuous != 0;
    opt.exact_max_T = max_T;
    auto [events, r] = simulate_model(std::span<const CostVector>(cs), K, opt);
    off = 0;
    for (auto& lr : r.per_layer) {
      std::memcpy(orders_out + off, lr.schedule.order.data(), sizeof(int) * lr.n_experts);
      off += lr.n_experts;
    }
    for (size_t i = 0; i < events.size(); ++i) {
      ev[i] = {events[i].stream == StreamKind::Load ? 0 : 1, events[i].layer_id,
               events[i].expert_id, events[i].start, events[i].end};
    }
    *rep = {r.makespan, r.compute_busy, r.load_busy, r.compute_stall,
            r.peak_resident_experts, r.overlap_efficiency};
  });
}
// Single layer under an explicit permutation (simulator.hpp:209-220).
int ref_simulate_order(const int* order, const double* a, int T, double beta, int K,
                       int mode, ref_event* ev, ref_report* rep) {
  return guard([&] {
    auto [events, r] = simulate(std::span<const int>(order, T), make_costs(a, T, beta), K,
                                mode == 0 ? SimMode::Overlapped : SimMode::Serial);
    for (size_t i = 0; i < events.size(); ++i) {
      ev[i] = {events[i].stream == StreamKind::Load ? 0 : 1, events[i].layer_id,
               events[i].expert_id, events[i].start, events[i].end};
    }
    *rep = {r.makespan, r.compute_busy, r.load_busy, r.compute_stall,
            r.peak_resident_experts, r.overlap_efficiency};
  });
}
double ref_lower_bound(const double* a, int T, double beta) {
  return lower_bound(make_costs(a, T, beta));
}
// Returns the 16-hex-digit FNV digest as uint64.
uint64_t ref_instance_digest(const double* a, int T, double beta, int K) {
  return std::stoull(instance_digest(make_costs(a, T, beta), K), nullptr, 16);
}
int ref_enumerate_feasibility(const double* a, int T, double beta, int K, int* witness) {
  int out = -2;
  guard([&] {
    auto r = enumerate_feasibility(make_costs(a, T, beta), K);
    out = r.oracle_feasible ? 1 : 0;
    if (r.witness_order && witness)
      std::memcpy(witness, r.witness_order->data(), sizeof(int) * T);
  });
  return out;
}
// replay_check on a single layer; returns violation count, kinds histogram.
int ref_replay_check(const ref_event* ev, int n, const double* a, int T, double beta,
                     int K, int* kinds6) {
  std::vector<TimelineEvent> events(n);
  for (int i = 0; i < n; ++i)
    events[i] = {ev[i].stream == 0 ? StreamKind::Load : StreamKind::Compute,
                 ev[i].layer_id, ev[i].expert_id, ev[i].start, ev[i].end};
  auto v = replay_check(std::span<const TimelineEvent>(events), make_costs(a, T, beta), K);
  std::memset(kinds6, 0, sizeof(int) * 6);
  for (auto& x : v) kinds6[static_cast<int>(x.kind)]++;
  return static_cast<int>(v.size());
}
}
