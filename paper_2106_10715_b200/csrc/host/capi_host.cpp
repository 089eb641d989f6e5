// capi_host.cpp — extern "C" entry points of the planning layer (infmoe.h,
// model_config / prng / gating / cost_model / scheduler / simulator sections).
#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "infmoe.h"
#include "planner.hpp"
#include "status.hpp"

namespace infmoe {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& m) { g_last_error = m; }

static Geometry to_geom(const infmoe_geometry* g) {
  require(g != nullptr, "geometry is NULL");
  return Geometry{g->n_layers, g->n_heads, g->d_head, g->d_model,
                  g->d_ff,     g->n_experts_per_layer, g->bytes_per_param};
}
static Hardware to_hw(const infmoe_hardware* h) {
  require(h != nullptr, "hardware is NULL");
  return Hardware{h->peak_flops, h->h2d_bandwidth, h->device_memory, h->reserved_memory};
}
static Costs to_costs(const double* alphas, int32_t T, double beta) {
  require(T >= 0 && (alphas != nullptr || T == 0), "alphas is NULL");
  Costs c;
  c.alpha.assign(alphas, alphas + T);
  c.beta = beta;
  return c;
}
static void emit_plan(const Plan& p, int32_t* order, double* slack,
                      infmoe_schedule_info* info) {
  if (order) std::memcpy(order, p.order.data(), sizeof(int32_t) * p.order.size());
  if (slack) std::memcpy(slack, p.slack.data(), sizeof(double) * p.slack.size());
  if (info) {
    info->feasible = p.feasible ? 1 : 0;
    info->diagnosis = static_cast<int32_t>(p.verdict);
    info->method = static_cast<int32_t>(p.method);
  }
}
}  // namespace infmoe

using namespace infmoe;

extern "C" {

const char* infmoe_last_error(void) { return g_last_error.c_str(); }
const char* infmoe_version(void) { return "infmoe-b200 0.1 (sm_100a)"; }

int infmoe_validate_geometry(const infmoe_geometry* g, int32_t* warn) {
  return guarded([&] {
    bool w = check_geometry(to_geom(g));
    if (warn) *warn = w ? 1 : 0;
  });
}
int infmoe_validate_hardware(const infmoe_hardware* hw) {
  return guarded([&] { check_hardware(to_hw(hw)); });
}
uint64_t infmoe_expert_param_bytes(const infmoe_geometry* g) {
  return g ? bytes_per_expert(to_geom(g)) : 0;
}
uint64_t infmoe_expert_flops(const infmoe_geometry* g, uint64_t n) {
  return g ? flops_for_tokens(to_geom(g), n) : 0;
}
int infmoe_geometry_preset(const char* name, infmoe_geometry* out) {
  return guarded([&] {
    require(name && out, "NULL argument");
    Geometry g;
    if (!preset(name, &g)) fail(kConfig, std::string("unknown geometry preset '") + name + "'");
    *out = {g.n_layers, g.n_heads, g.d_head, g.d_model, g.d_ff, g.experts, g.bytes_per_param};
  });
}

uint64_t infmoe_splitmix64(uint64_t x) { return mix64(x); }
uint64_t infmoe_derive_seed(uint64_t s, uint64_t t) { return child_seed(s, t); }
int infmoe_gaussian_fill(uint64_t seed, double* out, uint64_t n) {
  return guarded([&] {
    require(out != nullptr || n == 0, "out is NULL");
    normal_draws(seed, out, n);
  });
}
int infmoe_gaussian_fill_typed(int32_t dtype, int32_t n_mats, const uint64_t* seeds,
                               const double* scales, uint64_t n_each, void* const* outs,
                               int32_t threads) {
  return guarded([&] {
    require(dtype == INFMOE_DTYPE_BF16 || dtype == INFMOE_DTYPE_F32, "gaussian fill: bad dtype");
    require(n_mats >= 0 && (n_mats == 0 || (seeds && scales && outs)), "gaussian fill: NULL");
    for (int m = 0; m < n_mats; ++m) require(outs[m] != nullptr || n_each == 0, "out is NULL");
    normal_fill_typed(dtype, n_mats, seeds, scales, n_each, outs, threads);
  });
}
int infmoe_lsh_codes(uint64_t seed, int32_t bits, int32_t hidden, const double* x,
                     uint64_t n_tokens, uint32_t* codes) {
  return guarded([&] {
    if (bits < 1 || bits > 31) fail(kConfig, "gating: n_hash_bits must be in [1, 31]");
    if (hidden < 1) fail(kConfig, "gating: hidden_dim must be >= 1");
    require((x && codes) || n_tokens == 0, "lsh_codes: NULL argument");
    lsh_codes_host(seed, bits, hidden, x, n_tokens, codes);
  });
}
int infmoe_route_tokens(uint64_t seed, int32_t bits, int32_t hidden, const double* x,
                        uint64_t n_tokens, int32_t n_experts, uint64_t* counts) {
  return guarded([&] {
    if (n_experts < 1) fail(kArgument, "route_tokens: n_experts must be >= 1");
    if (bits >= 0 && (1u << std::min(bits, 31)) < uint32_t(n_experts))
      fail(kConfig, "gating: 2^n_hash_bits must be >= n_experts");
    if (bits < 1 || bits > 31) fail(kConfig, "gating: n_hash_bits must be in [1, 31]");
    if (hidden < 1) fail(kConfig, "gating: hidden_dim must be >= 1");
    require(counts && (x || n_tokens == 0), "route_tokens: NULL argument");
    std::vector<uint32_t> codes(n_tokens);
    lsh_codes_host(seed, bits, hidden, x, n_tokens, codes.data());
    std::memset(counts, 0, sizeof(uint64_t) * size_t(n_experts));
    for (uint32_t c : codes) ++counts[c % uint32_t(n_experts)];
  });
}
int infmoe_explicit_workload(const uint64_t* counts, int32_t n_experts, uint64_t* total) {
  return guarded([&] {
    require(counts || n_experts <= 0, "explicit_workload: counts is NULL");
    const uint64_t t = explicit_total(counts, n_experts);
    if (total) *total = t;
  });
}
int infmoe_workload_from_csv(const char* path, uint64_t* counts, int32_t capacity,
                             int32_t* n_experts, uint64_t* total) {
  return guarded([&] {
    require(path && n_experts, "workload_from_csv: NULL argument");
    const std::vector<uint64_t> c = workload_csv(path);
    if (c.size() > size_t(INT32_MAX)) fail(kConfig, "workload csv: expert id too large");
    *n_experts = int32_t(c.size());
    if (total) *total = explicit_total(c.data(), int(c.size()));
    if (counts) {
      require(capacity >= int32_t(c.size()), "workload_from_csv: counts buffer too small");
      std::memcpy(counts, c.data(), sizeof(uint64_t) * c.size());
    }
  });
}
int infmoe_gating_projection(uint64_t seed, int32_t bits, int32_t hidden, double* out) {
  return guarded([&] {
    require(out != nullptr, "out is NULL");
    auto p = lsh_hyperplanes(seed, bits, hidden);
    std::memcpy(out, p.data(), p.size() * sizeof(double));
  });
}
int infmoe_synthetic_workload(int32_t kind, uint64_t total, int32_t E, uint64_t seed,
                              double zipf_s, uint64_t* counts) {
  return guarded([&] {
    require(counts != nullptr, "counts is NULL");
    auto c = workload_counts(kind, total, E, seed, zipf_s);
    std::memcpy(counts, c.data(), c.size() * sizeof(uint64_t));
  });
}

int infmoe_compute_costs(const infmoe_geometry* g, const infmoe_hardware* hw,
                         const uint64_t* counts, int32_t n, double* alphas, double* beta) {
  return guarded([&] {
    require(counts && alphas && beta, "NULL argument");
    Costs c = derive_costs(counts, n, to_geom(g), to_hw(hw));
    std::memcpy(alphas, c.alpha.data(), sizeof(double) * c.alpha.size());
    *beta = c.beta;
  });
}
int infmoe_resident_capacity(const infmoe_geometry* g, const infmoe_hardware* hw,
                             int32_t* K) {
  return guarded([&] {
    require(K != nullptr, "K is NULL");
    *K = capacity_slots(to_geom(g), to_hw(hw));
  });
}
int infmoe_clamp_explicit_capacity(int32_t explicit_k, int32_t capacity, int32_t* K,
                                   int32_t* clamped) {
  return guarded([&] {
    require(K != nullptr, "K is NULL");
    if (explicit_k < 1) fail(kCapacity, "explicit K must be >= 1");
    const bool over = explicit_k > capacity;
    *K = over ? capacity : explicit_k;
    if (clamped) *clamped = over ? 1 : 0;
  });
}
int infmoe_with_event_overhead(double* alphas, int32_t T, double* beta, double eps) {
  return guarded([&] {
    if (eps < 0.0) fail(kConfig, "event_overhead must be >= 0");
    require(beta && (alphas || T == 0), "NULL argument");
    for (int32_t i = 0; i < T; ++i) alphas[i] += eps;
    *beta += eps;
  });
}

int infmoe_check_constraints(const int32_t* order, const double* alphas, int32_t T,
                             double beta, int32_t K, double* slack,
                             infmoe_constraint_report* rep) {
  return guarded([&] {
    require(order != nullptr, "order is NULL");
    BandCheck b = band_check(std::span<const int>(order, std::size_t(T)),
                             to_costs(alphas, T, beta), K);
    if (slack) std::memcpy(slack, b.slack.data(), sizeof(double) * b.slack.size());
    if (rep) *rep = {b.feasible ? 1 : 0, b.position, b.side, b.prefix, b.limit};
  });
}
int infmoe_schedule(const double* alphas, int32_t T, double beta, int32_t K, int32_t policy,
                    int32_t exact_max_T, int32_t* order, double* slack,
                    infmoe_schedule_info* info) {
  return guarded([&] {
    Costs c = to_costs(alphas, T, beta);
    Plan p;
    switch (policy) {
      case INFMOE_POLICY_AUTO: p = plan_auto(c, K, exact_max_T); break;
      case INFMOE_POLICY_GREEDY: p = plan_greedy(c, K); break;
      case INFMOE_POLICY_EXACT: p = plan_exact(c, K, exact_max_T); break;
      case INFMOE_POLICY_NAIVE: p = plan_identity(c, K); break;
      default: fail(kConfig, "unknown policy");
    }
    emit_plan(p, order, slack, info);
  });
}
int infmoe_diagnose(const double* alphas, int32_t T, double beta, int32_t K,
                    int32_t exact_max_T, int32_t* diagnosis) {
  return guarded([&] {
    require(diagnosis != nullptr, "diagnosis is NULL");
    *diagnosis = static_cast<int32_t>(classify(to_costs(alphas, T, beta), K, exact_max_T));
  });
}

static void emit_timeline(const TimelineStats& st, const std::vector<Event>& ev,
                          infmoe_event* events, infmoe_sim_report* rep,
                          infmoe_layer_report* per_layer) {
  if (events)
    for (std::size_t i = 0; i < ev.size(); ++i)
      events[i] = {ev[i].stream, ev[i].layer, ev[i].expert, ev[i].start, ev[i].end};
  if (rep)
    *rep = {st.makespan, st.compute_busy, st.load_busy, st.compute_stall, st.peak_resident,
            st.overlap_efficiency};
  if (per_layer)
    for (std::size_t l = 0; l < st.layers.size(); ++l) {
      const LayerStats& s = st.layers[l];
      per_layer[l] = {s.layer, s.experts, s.start, s.end, s.compute_busy, s.load_busy,
                      s.compute_stall, s.peak_resident, s.lower_bound};
    }
}

int infmoe_simulate(const int32_t* order, const double* alphas, int32_t T, double beta,
                    int32_t K, int32_t mode, infmoe_event* events, infmoe_sim_report* rep) {
  return guarded([&] {
    require(order != nullptr, "order is NULL");
    Costs c = to_costs(alphas, T, beta);
    check_costs(c);
    band_check(std::span<const int>(order, std::size_t(T)), c, K);  // validates the order
    std::vector<std::vector<int>> orders{std::vector<int>(order, order + T)};
    std::vector<Costs> cs{c};
    std::vector<Event> ev;
    TimelineStats st = run_timeline(orders, cs, K, mode == INFMOE_MODE_SERIAL, false, &ev);
    emit_timeline(st, ev, events, rep, nullptr);
  });
}

int infmoe_simulate_orders(int32_t n_layers, const int32_t* T, const int32_t* orders,
                           const double* alphas, const double* betas, int32_t K, int32_t mode,
                           int32_t continuous, infmoe_event* events, infmoe_sim_report* rep,
                           infmoe_layer_report* per_layer) {
  return guarded([&] {
    if (n_layers < 1) fail(kArgument, "simulate: no layers");
    require(T && orders && alphas && betas, "NULL argument");
    std::vector<Costs> cs;
    std::vector<std::vector<int>> ords;
    std::size_t off = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
      Costs c = to_costs(alphas + off, T[l], betas[l]);
      check_costs(c);
      band_check(std::span<const int>(orders + off, std::size_t(T[l])), c, K);  // validates
      ords.emplace_back(orders + off, orders + off + T[l]);
      cs.push_back(std::move(c));
      off += std::size_t(T[l]);
    }
    std::vector<Event> ev;
    TimelineStats st =
        run_timeline(ords, cs, K, mode == INFMOE_MODE_SERIAL, continuous != 0, &ev);
    emit_timeline(st, ev, events, rep, per_layer);
  });
}

int infmoe_simulate_model(int32_t n_layers, const int32_t* T, const double* alphas,
                          const double* betas, int32_t K, int32_t mode, int32_t policy,
                          int32_t continuous, int32_t exact_max_T, int32_t* orders_out,
                          infmoe_event* events, infmoe_sim_report* rep,
                          infmoe_layer_report* per_layer) {
  return guarded([&] {
    if (n_layers < 1) fail(kArgument, "simulate_model: no layers");
    require(T && alphas && betas, "NULL argument");
    std::vector<Costs> cs;
    std::vector<std::vector<int>> orders;
    std::size_t off = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
      Costs c = to_costs(alphas + off, T[l], betas[l]);
      check_costs(c);
      Plan p;
      switch (policy) {
        case INFMOE_POLICY_AUTO:
        case INFMOE_POLICY_GREEDY: p = plan_auto(c, K, exact_max_T); break;
        case INFMOE_POLICY_NAIVE: p = plan_identity(c, K); break;
        case INFMOE_POLICY_EXACT: p = plan_exact(c, K, exact_max_T); break;
        default: fail(kConfig, "unknown policy");
      }
      if (orders_out) std::memcpy(orders_out + off, p.order.data(), sizeof(int32_t) * T[l]);
      orders.push_back(std::move(p.order));
      cs.push_back(std::move(c));
      off += std::size_t(T[l]);
    }
    std::vector<Event> ev;
    TimelineStats st =
        run_timeline(orders, cs, K, mode == INFMOE_MODE_SERIAL, continuous != 0, &ev);
    emit_timeline(st, ev, events, rep, per_layer);
  });
}

int infmoe_replay_check(const infmoe_event* events, int32_t n_events, int32_t n_layers,
                        const int32_t* T, const double* alphas, const double* betas,
                        int32_t max_resident, int32_t check_durations, double tol_s,
                        int32_t* n_violations, int32_t* kinds) {
  return guarded([&] {
    require(events || n_events == 0, "replay_check: events is NULL");
    require(T && alphas && betas && n_layers >= 1, "replay_check: NULL costs");
    std::vector<Costs> cs;
    std::size_t off = 0;
    for (int32_t l = 0; l < n_layers; ++l) {
      cs.push_back(to_costs(alphas + off, T[l], betas[l]));
      off += std::size_t(T[l]);
    }
    std::vector<Event> ev(static_cast<std::size_t>(n_events));
    for (int32_t i = 0; i < n_events; ++i)
      ev[std::size_t(i)] = {events[i].stream, events[i].layer_id, events[i].expert_id,
                            events[i].start, events[i].end};
    int k6[6];
    const int n = audit_timeline(ev, cs, max_resident, check_durations != 0, tol_s, k6);
    if (n_violations) *n_violations = n;
    if (kinds) for (int i = 0; i < 6; ++i) kinds[i] = k6[i];
  });
}

double infmoe_lower_bound(const double* alphas, int32_t T, double beta) {
  if (!alphas || T < 1) return 0.0;
  return makespan_floor(to_costs(alphas, T, beta));
}

}  // extern "C"
