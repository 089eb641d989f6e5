// test_moesim_compat.cpp — the SPEC.md examples and acceptance properties,
// written against the moesim API.  Built twice by tests/test_cpp_compat.py:
//   -DUSE_INFMOE : infmoe::moesim (include/infmoe/moesim.hpp over libinfmoe.so)
//   (default)    : the reference headers in place (/root/reference, when present)
// Both builds must print identical output (a differential test) and pass.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#ifdef USE_INFMOE
#include "infmoe/moesim.hpp"
namespace ms = infmoe::moesim;
#else
#include "moesim/cost_model.hpp"
#include "moesim/gating.hpp"
#include "moesim/model_config.hpp"
#include "moesim/tolerance.hpp"
#include "moesim/prng.hpp"
#include "moesim/scheduler.hpp"
#include "moesim/simulator.hpp"
namespace ms = moesim;
#endif

static int failures = 0;
#define CHECK(cond)                                                 \
  do {                                                              \
    if (!(cond)) {                                                  \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);    \
      ++failures;                                                   \
    }                                                               \
  } while (0)

int main() {
  // model_config
  ms::ModelGeometry cpm2{24, 64, 64, 4096, 10240, 32, 2};
  CHECK(ms::expert_param_bytes(cpm2) == 167772160ull);
  CHECK(ms::expert_flops(cpm2, 1) == 167772160ull);
  CHECK(ms::validate(cpm2).empty());
  // cost model
  ms::HardwareProfile hw{1e12, 16e9, 16ull << 30, 8ull << 30};
  CHECK(ms::resident_capacity(cpm2, hw) == 51);
  bool threw = false;
  try {
    ms::resident_capacity(cpm2, ms::HardwareProfile{1e12, 16e9, 100, 10});
  } catch (const ms::CapacityError&) {
    threw = true;
  }
  CHECK(threw);
  // Figure 3 instance
  ms::CostVector c;
  c.alphas = {0.5, 2, 1, 0.5};
  c.beta = 1.0;
  ms::Schedule g = ms::greedy_order(c, 2);
  ms::Schedule e = ms::exact_order(c, 2);
  ms::Schedule n = ms::naive_order(c, 2);
  CHECK(g.feasible && !n.feasible);
  CHECK((g.order == std::vector<int>{2, 1, 0, 3}));
  CHECK((e.order == std::vector<int>{1, 0, 2, 3}));
  auto [ev, rep] = ms::simulate(g, c, 2);
  CHECK(rep.makespan == 5.0 && rep.compute_stall == 0.0);
  auto [evn, repn] = ms::simulate(n, c, 2);
  CHECK(repn.makespan == 5.5 && repn.compute_stall == 0.5);
  auto [evs, reps] = ms::simulate(g, c, 2, ms::SimMode::Serial);
  CHECK(reps.makespan == 8.0);
  // diagnosis
  ms::CostVector z;
  z.alphas = {0, 0, 0};
  z.beta = 1.0;
  CHECK(ms::diagnose(z, 1) == ms::Diagnosis::TooLittleCompute);
  ms::CostVector im;
  im.alphas = {10, 0, 0, 0, 0};
  im.beta = 1.0;
  CHECK(ms::diagnose(im, 1) == ms::Diagnosis::Imbalanced);
  // invalid arguments are std::invalid_argument (scheduler.hpp:49-62, :74)
  threw = false;
  try {
    std::vector<int> bad{0, 0, 1, 2};
    ms::check_constraints(bad, c, 2);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  // multi-layer
  ms::CostVector two;
  two.alphas = {1.5, 1, 1.25, 1};
  two.beta = 1.0;
  std::vector<ms::CostVector> layers{two, two};
  ms::ModelSimOptions opt;
  CHECK(ms::simulate_model(layers, 2, opt).second.makespan == 11.5);
  opt.continuous_load_stream = true;
  CHECK(ms::simulate_model(layers, 2, opt).second.makespan == 10.5);
  // a differential sweep: every order / makespan printed bit for bit
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0.0, 3.0);
  unsigned long long digest = 1469598103934665603ull;
  auto mix = [&](unsigned long long v) {
    digest ^= v;
    digest *= 1099511628211ull;
  };
  for (int t = 0; t < 400; ++t) {
    ms::CostVector cv;
    const int T = 1 + int(rng() % 24);
    for (int i = 0; i < T; ++i) cv.alphas.push_back(U(rng));
    cv.beta = 0.5 + U(rng) / 3.0;
    const int K = 1 + int(rng() % 6);
    ms::Schedule s = ms::auto_order(cv, K);
    for (int o : s.order) mix(unsigned(o));
    mix(s.feasible);
    auto [ev2, rep2] = ms::simulate(s, cv, K);
    unsigned long long bits;
    std::memcpy(&bits, &rep2.makespan, 8);
    mix(bits);
  }
  // ---- tolerance.hpp, builtin presets ----
  CHECK(ms::approx_eq(1.0, 1.0 + 1e-10) && !ms::approx_eq(1.0, 1.0 + 1e-8));
  CHECK(ms::approx_geq(1.0, 1.0 + 5e-10) && ms::definitely_lt(1.0, 1.0 + 1e-6));
  CHECK(ms::approx_leq(0.0, 1e-16) && !ms::approx_leq(0.0, -1e-14));
  mix(unsigned(ms::builtin_geometry_presets().size()));
  for (const auto& [name, geo] : ms::builtin_geometry_presets()) {
    mix(unsigned(name.size()));
    mix(unsigned(geo.d_model) + unsigned(geo.d_ff) + unsigned(geo.n_experts_per_layer) +
        unsigned(geo.bytes_per_param));
  }
  // ---- prng.hpp / gating.hpp: the LSH gate on host fp64 rows, workloads ----
  auto mixd = [&](double v) {
    unsigned long long b;
    std::memcpy(&b, &v, 8);
    mix(b);
  };
  mix(ms::derive_seed(1, 0));
  {
    ms::GaussianStream gs(0);
    for (int i = 0; i < 5; ++i) mixd(gs.next());
  }
  const ms::GatingModel gm{ms::derive_seed(20261018, 2), 5, 256};
  for (double v : ms::gating_projection(gm)) mixd(v);
  const std::vector<double> hid = ms::gaussian_tokens(ms::derive_seed(20261018, 0), 700, 256);
  mixd(hid.front());
  mixd(hid.back());
  const auto codes = ms::lsh_codes(gm, hid, 700);
  for (auto c2 : codes) mix(c2);
  const ms::ExpertWorkload rw = ms::route_tokens(gm, hid, 700, 24, 3);
  CHECK(rw.total_tokens == 700 && rw.layer_id == 3 && rw.token_counts.size() == 24);
  for (auto c2 : rw.token_counts) mix(c2);
  threw = false;
  try {
    ms::route_tokens(ms::GatingModel{1, 3, 256}, hid, 700, 9);  // 2^3 < 9 experts
  } catch (const ms::ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    ms::lsh_codes(gm, hid, 699);  // size mismatch
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    ms::gating_projection(ms::GatingModel{1, 32, 8});
  } catch (const ms::ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  const ms::ExpertWorkload ew = ms::explicit_workload({5, 0, 7}, 2);
  CHECK(ew.total_tokens == 12 && ew.layer_id == 2);
  threw = false;
  try {
    ms::explicit_workload({});
  } catch (const ms::ConfigError&) {
    threw = true;
  }
  CHECK(threw);
  const char* csv = "/tmp/infmoe_compat_workload.csv";
  {
    std::ofstream o(csv);
    o << "expert_id,token_count\r\n3,10\n\n0,4\n1,2,9\n";
  }
  const ms::ExpertWorkload cw = ms::workload_from_csv(csv, 1);
  CHECK((cw.token_counts == std::vector<std::uint64_t>{4, 2, 0, 10}) && cw.total_tokens == 16);
  for (auto c2 : cw.token_counts) mix(c2);
  for (const char* bad : {"0,1\n0,2\n", "0,\n", "x,1\n1,y\n", ""}) {
    std::ofstream(csv) << bad;
    threw = false;
    try {
      ms::workload_from_csv(csv);
    } catch (const ms::ConfigError&) {
      threw = true;
    }
    CHECK(threw);
  }
  // ---- simulate_model over workloads, per-layer reports, order_for_policy ----
  ms::ModelGeometry small{2, 8, 64, 512, 2048, 24, 2};
  ms::HardwareProfile hw2{2e12, 2e9, 8ull << 30, 1ull << 30};
  std::vector<ms::ExpertWorkload> wls{rw, ms::synthetic_workload(ms::SyntheticKind::Zipf, 900,
                                                                 24, 5, 1.0, 1)};
  for (bool cont : {false, true}) {
    for (ms::OrderPolicy pol : {ms::OrderPolicy::Greedy, ms::OrderPolicy::Naive}) {
      ms::ModelSimOptions o2;
      o2.policy = pol;
      o2.continuous_load_stream = cont;
      auto [evm, repm] = ms::simulate_model(wls, small, hw2, 3, o2);
      CHECK(repm.per_layer.size() == 2);
      mixd(repm.makespan);
      mixd(repm.compute_stall);
      mix(unsigned(repm.peak_resident_experts));
      for (const auto& lr : repm.per_layer) {
        mix(unsigned(lr.layer_id));
        mix(unsigned(lr.n_experts));
        mixd(lr.start);
        mixd(lr.end);
        mixd(lr.compute_busy);
        mixd(lr.compute_stall);
        mix(unsigned(lr.peak_resident));
        mixd(lr.lower_bound);
        for (int o : lr.schedule.order) mix(unsigned(o));
        mix(lr.schedule.feasible);
        mix(unsigned(lr.schedule.method));
      }
      for (const auto& e2 : evm) {
        mix(unsigned(e2.stream == ms::StreamKind::Load));
        mix(unsigned(e2.expert_id));
        mixd(e2.end);
      }
      const ms::Schedule sp = ms::order_for_policy(ms::compute_costs(wls[1], small, hw2), 3, pol);
      for (int o : sp.order) mix(unsigned(o));
    }
  }
  {
    auto [ev1, rep1] = ms::simulate(g, c, 2);
    CHECK(rep1.per_layer.size() == 1 && rep1.per_layer[0].schedule.order == g.order);
    mixd(rep1.per_layer[0].lower_bound);
    std::vector<int> ord{3, 2, 1, 0};
    auto [ev2, rep2] = ms::simulate(ord, c, 2);
    CHECK(rep2.per_layer[0].schedule.method == ms::ScheduleMethod::Naive);
    mixd(rep2.makespan);
    mix(rep2.per_layer[0].schedule.feasible);
  }
  std::printf("digest %016llx failures %d\n", digest, failures);
  return failures == 0 ? 0 : 1;
}
