// planner.cpp — see planner.hpp.  Every floating-point expression that feeds a
// scheduling decision is evaluated in the same operation order as the
// reference so expert orders are bit-identical.
#include "planner.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <fstream>
#include <thread>
#include <map>
#include <numbers>
#include <random>

#include "status.hpp"

namespace infmoe {

// ====================================================================== PRNG
std::uint64_t mix64(std::uint64_t x) {  // prng.hpp:18-23
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

std::uint64_t child_seed(std::uint64_t seed, std::uint64_t tag) {  // prng.hpp:27-29
  return mix64(seed ^ mix64(tag));
}

namespace {
// 53-bit uniforms (prng.hpp:32-39)
inline double unit_closed0(std::mt19937_64& g) {
  return static_cast<double>(g() >> 11) * 0x1.0p-53;
}
inline double unit_open0(std::mt19937_64& g) {
  return (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;
}
}  // namespace

// Box–Muller pairs: the cosine branch is emitted first, the sine branch second
// (the cached spare of prng.hpp:53-65), so n draws consume ceil(n/2) pairs.
void normal_draws(std::uint64_t seed, double* out, std::uint64_t n) {
  std::mt19937_64 g(seed);
  std::uint64_t i = 0;
  while (i < n) {
    const double a = unit_open0(g);
    const double b = unit_closed0(g);
    const double radius = std::sqrt(-2.0 * std::log(a));
    const double angle = 2.0 * std::numbers::pi * b;
    out[i++] = radius * std::cos(angle);
    if (i < n) out[i++] = radius * std::sin(angle);
  }
}

// Rounding of a synthetic draw to the config dtype: double -> f32 (RN), then
// f32 -> bf16 (RNE, the same bit trick as __float2bfloat16_rn) for bf16.
static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return uint16_t((u >> 16) | 0x40);
  return uint16_t((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

void normal_fill_typed(int dtype, int n_mats, const std::uint64_t* seeds, const double* scales,
                       std::uint64_t n_each, void* const* outs, int threads) {
  const int nt = std::max(1, threads > 0 ? threads
                                         : int(std::max(1u, std::thread::hardware_concurrency())));
  auto store = [&](int m, std::uint64_t i, double g) {
    if (dtype == 2) {  // f64: the draws themselves, times the scale
      static_cast<double*>(outs[m])[i] = g * scales[m];
      return;
    }
    const float v = static_cast<float>(g * scales[m]);
    if (dtype == 0) static_cast<uint16_t*>(outs[m])[i] = f32_to_bf16_rne(v);
    else static_cast<float*>(outs[m])[i] = v;
  };
  auto run = [&](auto&& body, std::uint64_t n_items) {  // body(item), items claimed in order
    std::atomic<std::uint64_t> next{0};
    auto worker = [&] {
      for (std::uint64_t it = next++; it < n_items; it = next++) body(it);
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(worker);
    worker();
    for (auto& t : th) t.join();
  };
  if (n_mats >= nt) {  // one stream per thread, streamed straight into the output
    run([&](std::uint64_t m) {
          std::mt19937_64 g(seeds[m]);
          for (std::uint64_t i = 0; i < n_each;) {
            const double a = unit_open0(g);
            const double b = unit_closed0(g);
            const double radius = std::sqrt(-2.0 * std::log(a));
            const double angle = 2.0 * std::numbers::pi * b;
            store(int(m), i++, radius * std::cos(angle));
            if (i < n_each) store(int(m), i++, radius * std::sin(angle));
          }
        },
        std::uint64_t(n_mats));
    return;
  }
  // few long streams: the engine's raw outputs sequentially (two per pair),
  // then the Box-Muller pairs in parallel chunks (each pair depends only on
  // its own two outputs, so the values are those of the sequential stream)
  const std::uint64_t pairs = (n_each + 1) / 2;
  std::vector<std::uint64_t> raw(2 * pairs);
  for (int m = 0; m < n_mats; ++m) {
    std::mt19937_64 g(seeds[m]);
    for (auto& r : raw) r = g();
    constexpr std::uint64_t kChunk = 1 << 16;  // pairs per work item
    run([&](std::uint64_t c) {
          const std::uint64_t p1 = std::min(pairs, (c + 1) * kChunk);
          for (std::uint64_t p = c * kChunk; p < p1; ++p) {
            const double a = (static_cast<double>(raw[2 * p] >> 11) + 1.0) * 0x1.0p-53;
            const double b = static_cast<double>(raw[2 * p + 1] >> 11) * 0x1.0p-53;
            const double radius = std::sqrt(-2.0 * std::log(a));
            const double angle = 2.0 * std::numbers::pi * b;
            store(m, 2 * p, radius * std::cos(angle));
            if (2 * p + 1 < n_each) store(m, 2 * p + 1, radius * std::sin(angle));
          }
        },
        (pairs + kChunk - 1) / kChunk);
  }
}

// ================================================================== geometry
bool check_geometry(const Geometry& g) {  // model_config.hpp:37-55
  const std::pair<int, const char*> fields[] = {
      {g.n_layers, "n_layers"}, {g.n_heads, "n_heads"}, {g.d_head, "d_head"},
      {g.d_model, "d_model"},   {g.d_ff, "d_ff"},       {g.experts, "n_experts_per_layer"},
      {g.bytes_per_param, "bytes_per_param"}};
  for (const auto& [v, name] : fields)
    if (v <= 0) fail(kConfig, std::string("geometry.") + name + " must be > 0");
  return g.d_model != g.n_heads * g.d_head;
}

void check_hardware(const Hardware& hw) {  // model_config.hpp:57-64
  if (hw.peak_flops <= 0.0) fail(kConfig, "hardware.peak_flops must be > 0");
  if (hw.h2d_bandwidth <= 0.0) fail(kConfig, "hardware.h2d_bandwidth must be > 0");
  if (hw.device_memory <= hw.reserved_memory)
    fail(kConfig, "hardware.device_memory must exceed reserved_memory");
}

std::uint64_t bytes_per_expert(const Geometry& g) {  // two projections, no biases
  return 2ull * std::uint64_t(g.d_model) * std::uint64_t(g.d_ff) *
         std::uint64_t(g.bytes_per_param);
}

std::uint64_t flops_for_tokens(const Geometry& g, std::uint64_t tokens) {
  return 4ull * tokens * std::uint64_t(g.d_model) * std::uint64_t(g.d_ff);
}

bool preset(const std::string& name, Geometry* out) {  // model_config.hpp:85-105
  if (name == "cpm2") {
    *out = Geometry{24, 64, 64, 4096, 10240, 32, 2};
    return true;
  }
  if (name == "cpm-small") {
    *out = Geometry{12, 12, 64, 768, 3072, 32, 4};
    return true;
  }
  return false;
}

// ==================================================================== gating
std::vector<double> lsh_hyperplanes(std::uint64_t seed, int bits, int hidden) {
  if (bits < 1 || bits > 31) fail(kConfig, "gating: n_hash_bits must be in [1, 31]");
  if (hidden < 1) fail(kConfig, "gating: hidden_dim must be >= 1");
  std::vector<double> p(std::size_t(bits) * std::size_t(hidden));
  normal_draws(seed, p.data(), p.size());  // bit-major: plane j = p[j*hidden ...]
  return p;
}

// lsh_codes (gating.hpp:61-82): per token, bit j = (sum_d x[t,d] * P[j,d] >= 0)
// with the products and the running sum rounded separately in ascending d
// (this translation unit is built with -ffp-contract=off, like the reference),
// so the codes are bit-identical.  Tokens are independent: split over threads.
void lsh_codes_host(std::uint64_t seed, int bits, int hidden, const double* x,
                    std::uint64_t n_tokens, std::uint32_t* codes) {
  const std::vector<double> proj = lsh_hyperplanes(seed, bits, hidden);
  auto rows = [&](std::uint64_t t0, std::uint64_t t1) {
    for (std::uint64_t t = t0; t < t1; ++t) {
      const double* row = x + t * std::uint64_t(hidden);
      std::uint32_t code = 0;
      for (int j = 0; j < bits; ++j) {
        const double* hp = proj.data() + std::size_t(j) * std::size_t(hidden);
        double dot = 0.0;
        for (int d = 0; d < hidden; ++d) dot += row[d] * hp[d];
        if (dot >= 0.0) code |= (1u << j);
      }
      codes[t] = code;
    }
  };
  const std::uint64_t work = n_tokens * std::uint64_t(bits) * std::uint64_t(hidden);
  const unsigned nt = work < (1u << 22) ? 1u
                                        : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (nt == 1) {
    rows(0, n_tokens);
    return;
  }
  std::vector<std::thread> th;
  const std::uint64_t per = (n_tokens + nt - 1) / nt;
  for (unsigned i = 0; i < nt; ++i) {
    const std::uint64_t a = std::min(n_tokens, i * per), b = std::min(n_tokens, a + per);
    if (a < b) th.emplace_back(rows, a, b);
  }
  for (auto& t : th) t.join();
}

// explicit_workload + validate(ExpertWorkload) (gating.hpp:25-33, :167-175)
std::uint64_t explicit_total(const std::uint64_t* counts, int n) {
  if (n < 1) fail(kConfig, "workload: no experts");
  std::uint64_t s = 0;
  for (int e = 0; e < n; ++e) s += counts[e];
  return s;
}

// workload_from_csv (gating.hpp:180-219): "expert_id,token_count" rows, an
// optional header (first line only, non-numeric id), ids in any order, an id
// listed twice is an error; expert count = max id + 1 (missing ids count 0).
std::vector<std::uint64_t> workload_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(kConfig, "workload csv: cannot open " + path);
  std::vector<std::pair<std::uint64_t, std::uint64_t>> rows;
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    while (!line.empty() && (line.back() == '\r' || line.back() == '\n')) line.pop_back();
    if (line.empty()) continue;
    const std::size_t comma = line.find(',');
    // both fields must be non-empty up to the end of the line
    if (comma == std::string::npos || comma + 1 >= line.size())
      fail(kConfig, "workload csv: line " + std::to_string(lineno) +
                        ": expected expert_id,token_count");
    const std::string a = line.substr(0, comma), b = line.substr(comma + 1);
    if (lineno == 1 && a.find_first_not_of("0123456789 ") != std::string::npos) continue;
    try {
      rows.emplace_back(std::stoull(a), std::stoull(b));
    } catch (const std::exception&) {
      fail(kConfig, "workload csv: line " + std::to_string(lineno) + ": not a number: " + line);
    }
  }
  if (rows.empty()) fail(kConfig, "workload csv: no rows in " + path);
  std::uint64_t max_id = 0;
  for (const auto& r : rows) max_id = std::max(max_id, r.first);
  std::vector<std::uint64_t> counts(max_id + 1, 0);
  std::vector<bool> seen(max_id + 1, false);
  for (const auto& [id, n] : rows) {
    if (seen[id]) fail(kConfig, "workload csv: duplicate expert_id " + std::to_string(id));
    seen[id] = true;
    counts[id] = n;
  }
  return counts;
}

std::vector<std::uint64_t> workload_counts(int kind, std::uint64_t total, int experts,
                                           std::uint64_t seed, double zipf_s) {
  if (experts < 1) fail(kConfig, "workload: n_experts must be >= 1");
  std::vector<std::uint64_t> counts(std::size_t(experts), 0);
  const std::uint64_t E = std::uint64_t(experts);
  if (kind == 2) {  // balanced: remainder to the lowest indices
    for (std::uint64_t e = 0; e < E; ++e) counts[e] = total / E + (e < total % E ? 1 : 0);
    return counts;
  }
  std::mt19937_64 g(seed);
  if (kind == 0) {  // uniform, modulo-folded 53-bit draw
    for (std::uint64_t t = 0; t < total; ++t)
      ++counts[static_cast<std::uint64_t>(unit_closed0(g) * double(E)) % E];
    return counts;
  }
  if (kind == 1) {  // zipf: inverse-CDF search over rank^-s
    if (!(zipf_s > 0.0)) fail(kConfig, "workload: zipf exponent must be > 0");
    std::vector<double> cdf(static_cast<std::size_t>(experts));
    double running = 0.0;
    for (int e = 0; e < experts; ++e) {
      running += std::pow(double(e + 1), -zipf_s);
      cdf[std::size_t(e)] = running;
    }
    for (std::uint64_t t = 0; t < total; ++t) {
      const double target = unit_closed0(g) * running;
      std::size_t e = std::size_t(std::lower_bound(cdf.begin(), cdf.end(), target) - cdf.begin());
      ++counts[std::min<std::size_t>(e, std::size_t(experts) - 1)];
    }
    return counts;
  }
  fail(kConfig, "workload.kind: unknown kind");
}

// ================================================================ cost model
namespace {
// One tolerance rule for every duration comparison: relative 1e-9, absolute
// floor 1e-15 s (tolerance.hpp:10-23).
inline double tol(double a, double b) {
  return std::max(1e-15, 1e-9 * std::max(std::fabs(a), std::fabs(b)));
}
inline bool at_least(double a, double b) { return a >= b - tol(a, b); }
inline bool at_most(double a, double b) { return a <= b + tol(a, b); }
inline bool below(double a, double b) { return !at_least(a, b); }
}  // namespace

double Costs::alpha_sum() const {
  double s = 0.0;
  for (double a : alpha) s += a;  // left-to-right, as std::accumulate
  return s;
}

void check_costs(const Costs& c) {
  if (c.alpha.empty()) fail(kConfig, "costs: need at least one expert");
  if (!(c.beta > 0.0)) fail(kConfig, "costs: beta must be > 0");
  for (double a : c.alpha)
    if (!(a >= 0.0)) fail(kConfig, "costs: alphas must be >= 0");
}

Costs derive_costs(const std::uint64_t* counts, int n, const Geometry& g,
                   const Hardware& hw) {  // cost_model.hpp:43-62
  if (!(hw.peak_flops > 0.0)) fail(kConfig, "costs: peak_flops must be > 0");
  if (!(hw.h2d_bandwidth > 0.0)) fail(kConfig, "costs: h2d_bandwidth must be > 0");
  if (n != g.experts)
    fail(kConfig, "costs: workload has " + std::to_string(n) + " experts, geometry says " +
                      std::to_string(g.experts));
  Costs c;
  c.alpha.resize(std::size_t(n));
  for (int i = 0; i < n; ++i)
    c.alpha[std::size_t(i)] = double(flops_for_tokens(g, counts[i])) / hw.peak_flops;
  c.beta = double(bytes_per_expert(g)) / hw.h2d_bandwidth;
  return c;
}

int capacity_slots(const Geometry& g, const Hardware& hw) {  // cost_model.hpp:65-78
  if (hw.device_memory <= hw.reserved_memory)
    fail(kConfig, "capacity: device_memory must exceed reserved_memory");
  const std::uint64_t room = hw.device_memory - hw.reserved_memory;
  const std::uint64_t each = bytes_per_expert(g);
  if (room / each < 1)
    fail(kCapacity, "expert does not fit in device memory: needs " + std::to_string(each) +
                        " bytes, free " + std::to_string(room));
  return int(room / each);
}

// ================================================================= scheduler
namespace {
void require_order(std::span<const int> order, int T) {
  if (int(order.size()) != T)
    fail(kArgument, "order size " + std::to_string(order.size()) + " != expert count " +
                      std::to_string(T));
  std::vector<char> hit(std::size_t(T), 0);
  for (int e : order) {
    if (e < 0 || e >= T || hit[std::size_t(e)])
      fail(kArgument, "order is not a permutation of 0.." + std::to_string(T - 1));
    hit[std::size_t(e)] = 1;
  }
}

Verdict classify_infeasible(const Costs& c) {  // scheduler.hpp:102-109
  const double smallest = *std::min_element(c.alpha.begin(), c.alpha.end());
  const double reachable = c.alpha_sum() - smallest;
  const double needed = (c.size() - 1) * c.beta;
  return below(reachable, needed) ? Verdict::TooLittleCompute : Verdict::Imbalanced;
}

Plan finish(std::vector<int> order, const Costs& c, int K, Method m, bool diagnose) {
  BandCheck b = band_check(order, c, K);
  Plan p;
  p.order = std::move(order);
  p.feasible = b.feasible;
  p.slack = std::move(b.slack);
  p.method = m;
  if (!p.feasible && diagnose) p.verdict = classify_infeasible(c);
  return p;
}
}  // namespace

// Prefix bands m*β <= P_m <= (m+K)*β for m = 0..T-1.
BandCheck band_check(std::span<const int> order, const Costs& c, int K) {
  const int T = c.size();
  require_order(order, T);
  if (K < 1) fail(kArgument, "K must be >= 1");
  BandCheck r;
  r.slack.resize(std::size_t(T));
  double P = 0.0;
  for (int m = 0; m < T; ++m) {
    const double floor_m = m * c.beta;
    const double ceil_m = (m + K) * c.beta;
    r.slack[std::size_t(m)] = P - floor_m;
    if (r.feasible) {
      if (!at_least(P, floor_m)) {
        r.feasible = false;
        r.position = m, r.side = 0, r.prefix = P, r.limit = floor_m;
      } else if (!at_most(P, ceil_m)) {
        r.feasible = false;
        r.position = m, r.side = 1, r.prefix = P, r.limit = ceil_m;
      }
    }
    P += c.alpha[std::size_t(order[std::size_t(m)])];
  }
  return r;
}

// Position-by-position pick (scheduler.hpp:134-180 semantics): the cheapest
// expert that lands the prefix inside the band; failing that the most
// expensive one still under the ceiling; failing that the cheapest overall.
// Candidates are scanned in ascending index with strict comparisons, so ties
// go to the lower index.
Plan plan_greedy(const Costs& c, int K) {
  check_costs(c);
  if (K < 1) fail(kArgument, "K must be >= 1");
  const int T = c.size();
  const auto& a = c.alpha;
  std::vector<char> taken(std::size_t(T), 0);
  std::vector<int> order;
  order.reserve(std::size_t(T));
  double P = 0.0;
  for (int m = 1; m < T; ++m) {
    const double floor_m = m * c.beta;
    const double ceil_m = (m + K) * c.beta;
    int fit = -1, big = -1, small = -1;
    for (int e = 0; e < T; ++e) {
      if (taken[std::size_t(e)]) continue;
      const double q = P + a[std::size_t(e)];
      const bool ok_hi = at_most(q, ceil_m);
      if (ok_hi && at_least(q, floor_m) && (fit < 0 || a[std::size_t(e)] < a[std::size_t(fit)]))
        fit = e;
      if (ok_hi && (big < 0 || a[std::size_t(e)] > a[std::size_t(big)])) big = e;
      if (small < 0 || a[std::size_t(e)] < a[std::size_t(small)]) small = e;
    }
    const int pick = fit >= 0 ? fit : (big >= 0 ? big : small);
    taken[std::size_t(pick)] = 1;
    order.push_back(pick);
    P += a[std::size_t(pick)];
  }
  for (int e = 0; e < T; ++e)
    if (!taken[std::size_t(e)]) order.push_back(e);  // last slot is unconstrained
  return finish(std::move(order), c, K, Method::Greedy, true);
}

// Depth-first search over positions with the band pruned at every prefix and a
// memo of dead subsets (feasibility of a partial order depends only on the set
// used).  Children in ascending index: the first hit is the lexicographically
// smallest feasible order.
Plan plan_exact(const Costs& c, int K, int max_T) {
  check_costs(c);
  if (K < 1) fail(kArgument, "K must be >= 1");
  const int T = c.size();
  max_T = std::min(max_T, 24);
  if (T > max_T)
    fail(kArgument, "exact_order: T = " + std::to_string(T) + " exceeds max_T = " +
                      std::to_string(max_T));
  std::vector<char> dead(std::size_t(1) << T, 0);
  std::vector<int> path;
  path.reserve(std::size_t(T));
  struct Search {
    const Costs& c;
    int T, K;
    std::vector<char>& dead;
    std::vector<int>& path;
    bool go(std::uint32_t used, int depth, double P) {
      if (depth == T) return true;
      if (dead[used]) return false;
      for (int e = 0; e < T; ++e) {
        if (used >> e & 1u) continue;
        const double q = P + c.alpha[std::size_t(e)];
        if (depth + 1 <= T - 1) {
          if (!at_least(q, (depth + 1) * c.beta) || !at_most(q, (depth + 1 + K) * c.beta))
            continue;
        }
        path.push_back(e);
        if (go(used | (1u << e), depth + 1, q)) return true;
        path.pop_back();
      }
      dead[used] = 1;
      return false;
    }
  } s{c, T, K, dead, path};
  if (s.go(0u, 0, 0.0)) return finish(std::move(path), c, K, Method::ExactFallback, false);
  std::vector<int> identity(static_cast<std::size_t>(T));
  for (int i = 0; i < T; ++i) identity[std::size_t(i)] = i;
  Plan p = finish(std::move(identity), c, K, Method::ExactFallback, false);
  p.feasible = false;
  p.verdict = classify_infeasible(c);
  return p;
}

Plan plan_auto(const Costs& c, int K, int max_T) {  // scheduler.hpp:243-248
  Plan g = plan_greedy(c, K);
  if (g.feasible || c.size() > max_T) return g;
  return plan_exact(c, K, max_T);
}

Plan plan_identity(const Costs& c, int K) {
  std::vector<int> order(std::size_t(c.size()));
  for (int i = 0; i < c.size(); ++i) order[std::size_t(i)] = i;
  return finish(std::move(order), c, K, Method::Naive, false);
}

Verdict classify(const Costs& c, int K, int max_T) {
  return plan_auto(c, K, max_T).feasible ? Verdict::Feasible : classify_infeasible(c);
}

// ================================================================== timeline
double makespan_floor(const Costs& c) {  // simulator.hpp:53-56
  return std::max(c.beta + c.alpha_sum(), double(c.size()) * c.beta);
}

namespace {
// Max simultaneous residents: +1 at load completion, -1 at compute completion,
// departures ordered before arrivals at equal instants.
int max_resident_count(std::vector<std::pair<double, int>>& marks) {
  std::sort(marks.begin(), marks.end());
  int now = 0, peak = 0;
  for (const auto& mk : marks) peak = std::max(peak, now += mk.second);
  return peak;
}
}  // namespace

// load_end(j)    = max(load_end(j-1) + β, compute_end(j-K))
// compute_end(j) = max(load_end(j), compute_end(j-1)) + α_j
// (simulator.hpp:87-194; PAPER.md:366 two CUDA streams).  Serial mode runs
// load then compute back to back on one lane.  Without continuous loads the
// load lane waits for the previous layer's last compute.
TimelineStats run_timeline(std::span<const std::vector<int>> orders,
                           std::span<const Costs> costs, int K, bool serial,
                           bool continuous_loads, std::vector<Event>* events) {
  if (K < 1) fail(kArgument, "K must be >= 1");
  TimelineStats st;
  double load_lane = 0.0, compute_lane = 0.0, last_ce = -1.0;
  for (std::size_t l = 0; l < costs.size(); ++l) {
    const Costs& c = costs[l];
    const int T = c.size();
    require_order(orders[l], T);
    LayerStats ls;
    ls.layer = int(l);
    ls.experts = T;
    ls.lower_bound = makespan_floor(c);
    std::vector<double> ce_at(static_cast<std::size_t>(T));
    std::vector<std::pair<double, int>> marks;
    marks.reserve(std::size_t(2 * T));
    double layer_last_ce = -1.0, first_start = -1.0, layer_end = 0.0;
    if (!serial && !continuous_loads && l > 0) load_lane = std::max(load_lane, compute_lane);
    for (int j = 0; j < T; ++j) {
      const int e = orders[l][std::size_t(j)];
      const double alpha = c.alpha[std::size_t(e)];
      double l0, l1, c0, c1;
      if (serial) {
        l0 = std::max(load_lane, compute_lane);
        l1 = l0 + c.beta;
        c0 = l1;
        c1 = c0 + alpha;
      } else {
        const double evict_gate = j >= K ? ce_at[std::size_t(j - K)] : 0.0;
        const double unblocked = load_lane + c.beta;
        if (evict_gate > unblocked) {
          l1 = evict_gate;
          l0 = evict_gate - c.beta;
        } else {
          l0 = load_lane;
          l1 = unblocked;
        }
        c0 = std::max(l1, compute_lane);
        c1 = c0 + alpha;
      }
      load_lane = l1;
      compute_lane = c1;
      ce_at[std::size_t(j)] = c1;
      marks.emplace_back(l1, +1);
      marks.emplace_back(c1, -1);
      if (events) {
        events->push_back({0, int(l), e, l0, l1});
        events->push_back({1, int(l), e, c0, c1});
      }
      ls.load_busy += l1 - l0;
      ls.compute_busy += c1 - c0;
      if (layer_last_ce >= 0.0 && c0 > layer_last_ce) ls.compute_stall += c0 - layer_last_ce;
      layer_last_ce = c1;
      if (last_ce >= 0.0 && c0 > last_ce) st.compute_stall += c0 - last_ce;
      last_ce = c1;
      first_start = first_start < 0.0 ? l0 : std::min(first_start, l0);
      layer_end = std::max(layer_end, c1);
    }
    ls.start = first_start;
    ls.end = layer_end;
    ls.peak_resident = max_resident_count(marks);
    st.load_busy += ls.load_busy;
    st.compute_busy += ls.compute_busy;
    st.peak_resident = std::max(st.peak_resident, ls.peak_resident);
    st.makespan = std::max(st.makespan, layer_end);
    st.layers.push_back(ls);
  }
  st.overlap_efficiency = st.makespan > 0.0 ? st.compute_busy / st.makespan : 0.0;
  return st;
}

// ============================================================ timeline audit
// The rules of replay_check (verification.hpp:108-198) for measured timelines:
// measured durations are never exactly alpha/beta, so the duration rule is
// optional and comparisons take an absolute tolerance on top of the usual one.
int audit_timeline(const std::vector<Event>& ev, std::span<const Costs> costs, int max_resident,
                   bool check_durations, double tol_s, int kinds[6]) {
  for (int i = 0; i < 6; ++i) kinds[i] = 0;
  const int L = int(costs.size());
  auto leq = [&](double a, double b) { return a <= b + tol_s || at_most(a, b); };
  for (const Event& e : ev) {  // malformed events skip only the duration rule
    if (e.end < e.start || e.layer < 0 || e.layer >= L || e.expert < 0 ||
        e.expert >= costs[size_t(e.layer)].size()) {
      ++kinds[5];
      continue;
    }
    if (check_durations) {
      const Costs& c = costs[size_t(e.layer)];
      const double want = e.stream == 0 ? c.beta : c.alpha[size_t(e.expert)];
      if (std::fabs((e.end - e.start) - want) > std::max(tol_s, tol(e.end - e.start, want)))
        ++kinds[3];
    }
  }
  for (int lane = 0; lane < 2; ++lane) {  // one lane per stream, across layers
    std::vector<const Event*> v;
    for (const Event& e : ev)
      if (e.stream == lane) v.push_back(&e);
    std::stable_sort(v.begin(), v.end(),
                     [](const Event* a, const Event* b) { return a->start < b->start; });
    for (size_t i = 1; i < v.size(); ++i)
      if (!leq(v[i - 1]->end, v[i]->start)) ++kinds[0];
  }
  // causality per (layer, expert), residency per layer
  std::map<std::pair<int, int>, std::pair<const Event*, const Event*>> pairs;
  for (const Event& e : ev) {
    if (e.layer < 0 || e.layer >= L) continue;
    auto& slot = pairs[{e.layer, e.expert}];
    (e.stream == 0 ? slot.first : slot.second) = &e;
  }
  std::map<int, std::vector<std::pair<double, int>>> marks;
  for (const auto& [key, pr] : pairs) {
    const Event* a = pr.first;
    const Event* b = pr.second;
    if (!a || !b) { ++kinds[1]; continue; }
    if (!leq(a->end, b->start)) ++kinds[1];
    marks[key.first].emplace_back(a->end, +1);
    marks[key.first].emplace_back(b->end, -1);
  }
  for (auto& [layer, m] : marks)
    if (max_resident > 0 && max_resident_count(m) > max_resident) ++kinds[2];
  int n = 0;
  for (int i = 0; i < 6; ++i) n += kinds[i];
  return n;
}

}  // namespace infmoe
