// test_moesim_compat.cpp — the SPEC.md examples and acceptance properties,
// written against the moesim API.  Built twice by tests/test_cpp_compat.py:
//   -DUSE_INFMOE : infmoe::moesim (include/infmoe/moesim.hpp over libinfmoe.so)
//   (default)    : the reference headers in place (/root/reference, when present)
// Both builds must print identical output (a differential test) and pass.
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#ifdef USE_INFMOE
#include "infmoe/moesim.hpp"
namespace ms = infmoe::moesim;
#else
#include "moesim/cost_model.hpp"
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
  std::printf("digest %016llx failures %d\n", digest, failures);
  return failures == 0 ? 0 : 1;
}
