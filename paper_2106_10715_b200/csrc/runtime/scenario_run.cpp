// scenario_run.cpp — `run` and `sweep` over a parsed scenario (
// the reference's CLI is absent, so the pipeline composition of
// SURVEY §3.4 is restated here): workload -> compute_costs -> K (capacity or
// clamped explicit) -> [event overhead] -> per policy schedule + two-lane
// timeline -> artifacts.  With `execute`, the same layers run on the GPU
// through the real offload executor (infmoe_layer_*) and the MEASURED
// timelines are written next to the simulated ones, audited with replay_check's
// rules and compared with the simulator at the measured counts.
//
// Per-layer workload realisation (builder-defined, recorded in resolved.json's
// seed): layer l of a gating workload routes gaussian_tokens(derive_seed(seed,
// 2l), total_tokens, hidden) through GatingModel{derive_seed(seed, 2l+1), bits,
// hidden}; uniform / zipf draw synthetic_workload(kind, total_tokens, E,
// derive_seed(seed, l), zipf_s); balanced / explicit / csv give every layer the
// same counts.  Artifacts are byte-identical for identical resolved scenarios
// (timestamps only in meta.json); measured/ artifacts carry hardware timings.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <memory>
#include <fstream>
#include <mutex>
#include <sstream>
#include <thread>

#include <json.hpp>

#include "../host/scenario.hpp"
#include "../host/status.hpp"
#include "infmoe.h"

namespace infmoe::scn {

using json = nlohmann::json;
namespace fs = std::filesystem;

namespace {

std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

void write_file(const fs::path& p, const std::string& text) {
  fs::create_directories(p.parent_path());
  const fs::path tmp = p.string() + ".tmp";
  {
    std::ofstream o(tmp, std::ios::binary);
    if (!o) fail(kConfig, "cannot write " + p.string());
    o << text;
  }
  fs::rename(tmp, p);  // one file at a time, atomically
}

struct LayerIn {
  std::vector<std::uint64_t> counts;  // per expert (empty for explicit costs)
  Costs costs;                        // after event overhead
  std::vector<int> ids;               // expert id of each cost entry (skip_empty_experts)
};

// the workload of layer l (see the header comment)
std::vector<std::uint64_t> layer_counts(const Scenario& s, int l) {
  const Workload& w = *s.workload;
  const Geometry& g = *s.geometry;
  switch (w.kind) {
    case WorkloadKind::Gating: {
      const int hid = w.hidden_dim > 0 ? w.hidden_dim : g.d_model;
      if (w.n_hash_bits >= 0 && (1u << std::min(w.n_hash_bits, 31)) < uint32_t(g.experts))
        fail(kConfig, "gating: 2^n_hash_bits must be >= n_experts");
      std::vector<double> x(w.total_tokens * std::uint64_t(hid));
      const std::uint64_t seed = child_seed(s.seed, 2ull * std::uint64_t(l));
      const double one = 1.0;
      void* out = x.data();
      normal_fill_typed(2, 1, &seed, &one, x.size(), &out, 0);
      std::vector<std::uint32_t> codes(w.total_tokens);
      lsh_codes_host(child_seed(s.seed, 2ull * std::uint64_t(l) + 1), w.n_hash_bits, hid,
                     x.data(), w.total_tokens, codes.data());
      std::vector<std::uint64_t> c(std::size_t(g.experts), 0);
      for (std::uint32_t code : codes) ++c[code % std::uint32_t(g.experts)];
      return c;
    }
    case WorkloadKind::Uniform:
      return workload_counts(0, w.total_tokens, g.experts, child_seed(s.seed, std::uint64_t(l)),
                             w.zipf_s);
    case WorkloadKind::Zipf:
      return workload_counts(1, w.total_tokens, g.experts, child_seed(s.seed, std::uint64_t(l)),
                             w.zipf_s);
    case WorkloadKind::Balanced:
      return workload_counts(2, w.total_tokens, g.experts, 0, w.zipf_s);
    case WorkloadKind::Explicit: explicit_total(w.counts.data(), int(w.counts.size()));
      return w.counts;
    case WorkloadKind::Csv: return workload_csv(w.csv_path);
  }
  return {};
}

Costs with_overhead(Costs c, double eps) {  // cost_model.hpp:96-101
  for (double& a : c.alpha) a += eps;
  c.beta += eps;
  return c;
}

struct Prepared {
  std::vector<LayerIn> layers;
  int K = 1;
  std::vector<std::string> warnings;
};

Prepared prepare(const Scenario& s) {
  Prepared p;
  if (s.alphas) {  // direct costs: every layer the same, explicit K
    Costs c;
    c.alpha = *s.alphas;
    c.beta = s.beta;
    check_costs(c);
    p.K = *s.k_explicit;
    for (int l = 0; l < s.n_moe_layers; ++l) {
      LayerIn li;
      li.costs = with_overhead(c, s.event_overhead_s);
      for (int e = 0; e < c.size(); ++e) li.ids.push_back(e);
      p.layers.push_back(std::move(li));
    }
    return p;
  }
  const Geometry& g = *s.geometry;
  const Hardware& hw = *s.hardware;
  const int cap = capacity_slots(g, hw);
  if (s.k_explicit) {
    p.K = std::min(*s.k_explicit, cap);  // clamp_explicit_capacity, cost_model.hpp:82-91
    if (*s.k_explicit > cap)
      p.warnings.push_back("K clamped from " + std::to_string(*s.k_explicit) +
                           " to capacity " + std::to_string(cap));
  } else {
    p.K = cap;
  }
  for (int l = 0; l < s.n_moe_layers; ++l) {
    LayerIn li;
    li.counts = layer_counts(s, l);
    if (int(li.counts.size()) != g.experts)
      fail(kConfig, "costs: workload has " + std::to_string(li.counts.size()) +
                        " experts, geometry says " + std::to_string(g.experts));
    std::vector<std::uint64_t> kept;
    for (int e = 0; e < g.experts; ++e)
      if (!s.skip_empty_experts || li.counts[std::size_t(e)] > 0) {
        li.ids.push_back(e);
        kept.push_back(li.counts[std::size_t(e)]);
      }
    Geometry gk = g;
    gk.experts = int(kept.size());
    li.costs = kept.empty() ? Costs{} : derive_costs(kept.data(), int(kept.size()), gk, hw);
    if (kept.empty()) li.costs.beta = double(bytes_per_expert(g)) / hw.h2d_bandwidth;
    li.costs = with_overhead(li.costs, s.event_overhead_s);
    p.layers.push_back(std::move(li));
  }
  return p;
}

Plan order_for(const Costs& c, int K, Policy pol) {
  switch (pol) {
    case Policy::Greedy: return plan_auto(c, K, 12);
    case Policy::Exact: return plan_exact(c, K, 12);
    default: return plan_identity(c, K);  // naive; serial (order-independent)
  }
}

struct Result {
  std::vector<Event> events;  // expert ids already mapped to the scenario's
  TimelineStats stats;
  std::vector<Plan> plans;
};

Result simulate(const Prepared& p, Policy pol, bool continuous) {
  Result r;
  std::vector<std::vector<int>> orders;
  std::vector<Costs> costs;
  for (const LayerIn& li : p.layers) {
    Plan pl = li.costs.size() ? order_for(li.costs, p.K, pol) : Plan{};
    orders.push_back(pl.order);
    costs.push_back(li.costs);
    r.plans.push_back(std::move(pl));
  }
  r.stats = run_timeline(orders, costs, p.K, pol == Policy::Serial, continuous, &r.events);
  for (Event& e : r.events) e.expert = p.layers[std::size_t(e.layer)].ids[std::size_t(e.expert)];
  return r;
}

std::string events_csv(const std::vector<Event>& ev) {
  std::string out = "stream,layer,expert,start_s,end_s\n";
  for (const Event& e : ev)
    out += std::string(e.stream == 0 ? "load" : "compute") + "," + std::to_string(e.layer) +
           "," + std::to_string(e.expert) + "," + num(e.start) + "," + num(e.end) + "\n";
  return out;
}

std::string chrome_trace(const std::vector<Event>& ev, const std::string& name,
                         const std::string& policy) {
  json tr = json::array();
  for (int t = 0; t < 2; ++t)
    tr.push_back({{"name", "thread_name"}, {"ph", "M"}, {"pid", 0}, {"tid", t},
                  {"args", {{"name", t == 0 ? "load" : "compute"}}}});
  for (const Event& e : ev)
    tr.push_back({{"name", "L" + std::to_string(e.layer) + " E" + std::to_string(e.expert)},
                  {"cat", e.stream == 0 ? "load" : "compute"},
                  {"ph", "X"},
                  {"pid", 0},
                  {"tid", e.stream},
                  {"ts", e.start * 1e6},
                  {"dur", (e.end - e.start) * 1e6},
                  {"args", {{"layer", e.layer}, {"expert", e.expert}}}});
  json j = {{"traceEvents", tr},
            {"displayTimeUnit", "ms"},
            {"otherData",
             {{"scenario", name}, {"policy", policy}, {"prng", "mt19937_64/box-muller/v1"}}}};
  return j.dump(1);
}

json report_json(const TimelineStats& st, const std::vector<Plan>& plans, int K) {
  json layers = json::array();
  for (std::size_t l = 0; l < st.layers.size(); ++l) {
    const LayerStats& ls = st.layers[l];
    json lj = {{"layer_id", ls.layer},          {"n_experts", ls.experts},
               {"start", ls.start},             {"end", ls.end},
               {"compute_busy", ls.compute_busy}, {"load_busy", ls.load_busy},
               {"compute_stall", ls.compute_stall}, {"peak_resident", ls.peak_resident},
               {"lower_bound", ls.lower_bound}};
    if (l < plans.size()) {
      lj["schedule"] = {{"order", plans[l].order}, {"feasible", plans[l].feasible},
                        {"method", int(plans[l].method)},
                        {"diagnosis", int(plans[l].verdict)}};
    }
    layers.push_back(std::move(lj));
  }
  return {{"makespan", st.makespan},
          {"compute_busy", st.compute_busy},
          {"load_busy", st.load_busy},
          {"compute_stall", st.compute_stall},
          {"peak_resident_experts", st.peak_resident},
          {"overlap_efficiency", st.overlap_efficiency},
          {"K", K},
          {"per_layer", layers}};
}

std::string summary_row(const std::string& policy, const TimelineStats& st, int K, int L) {
  return policy + "," + num(st.makespan) + "," + num(st.compute_busy) + "," +
         num(st.load_busy) + "," + num(st.compute_stall) + "," + num(st.overlap_efficiency) +
         "," + std::to_string(st.peak_resident) + "," + std::to_string(K) + "," +
         std::to_string(L) + "\n";
}
const char* kSummaryHead =
    "policy,makespan_s,compute_busy_s,load_busy_s,compute_stall_s,overlap_efficiency,"
    "peak_resident_experts,K,n_layers\n";

void write_policy(const fs::path& dir, const std::string& scen, const std::string& pol,
                  const std::vector<Event>& ev, const json& rep, int fmt) {
  if (fmt & 1) write_file(dir / "trace.json", chrome_trace(ev, scen, pol));
  if (fmt & 2) write_file(dir / "events.csv", events_csv(ev));
  write_file(dir / "report.json", rep.dump(1));
}

// ------------------------------------------------------------ GPU execute --
void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kRuntime, std::string(what) + ": " + cudaGetErrorString(e));
}
void abi_ok(int rc) {
  if (rc != INFMOE_OK) fail(Status(rc), infmoe_last_error());
}

struct HostBuf {
  void* p = nullptr;
  explicit HostBuf(size_t n) { cuda_ok(cudaMallocHost(&p, std::max<size_t>(n, 1)), "host alloc"); }
  ~HostBuf() { cudaFreeHost(p); }
};
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t n) { cuda_ok(cudaMalloc(&p, std::max<size_t>(n, 1)), "device alloc"); }
  ~DevBuf() { cudaFree(p); }
};

// measured timeline of the real executor for every layer and executable policy
std::string execute(const Scenario& s, const Prepared& p, const RunOptions& opt,
                    const fs::path& out) {
  const Geometry& g = *s.geometry;
  const Workload& w = *s.workload;
  const int d = g.d_model, f = g.d_ff, E = g.experts, L = s.n_moe_layers;
  if (g.bytes_per_param != 2 && g.bytes_per_param != 4)
    fail(kConfig, "execute: bytes_per_param must be 2 (bf16) or 4 (f32)");
  const int dtype = g.bytes_per_param == 2 ? INFMOE_DTYPE_BF16 : INFMOE_DTYPE_F32;
  const bool gating = w.kind == WorkloadKind::Gating;
  if (gating && w.hidden_dim > 0 && w.hidden_dim != d)
    fail(kConfig, "execute: the gating hidden_dim must equal d_model");
  cuda_ok(cudaSetDevice(opt.device), "cudaSetDevice");
  const size_t esz = size_t(g.bytes_per_param), mat = size_t(d) * size_t(f);
  // host weight sets (SURVEY 8(d) generators), aliased across layers
  const int n_sets = std::max(1, std::min(opt.host_sets, L));
  std::vector<std::unique_ptr<HostBuf>> w_in, w_out;
  for (int st = 0; st < n_sets; ++st) {
    w_in.push_back(std::make_unique<HostBuf>(size_t(E) * mat * esz));
    w_out.push_back(std::make_unique<HostBuf>(size_t(E) * mat * esz));
    std::vector<std::uint64_t> seeds;
    std::vector<double> scales;
    std::vector<void*> outs;
    for (int e = 0; e < E; ++e) {
      seeds.push_back(child_seed(s.seed + std::uint64_t(st), 1000 + 2ull * std::uint64_t(e)));
      scales.push_back(1.0 / std::sqrt(double(d)));
      outs.push_back(static_cast<uint8_t*>(w_in.back()->p) + size_t(e) * mat * esz);
      seeds.push_back(child_seed(s.seed + std::uint64_t(st), 1001 + 2ull * std::uint64_t(e)));
      scales.push_back(1.0 / std::sqrt(double(f)));
      outs.push_back(static_cast<uint8_t*>(w_out.back()->p) + size_t(e) * mat * esz);
    }
    normal_fill_typed(dtype == INFMOE_DTYPE_BF16 ? 0 : 1, int(outs.size()), seeds.data(),
                      scales.data(), mat, outs.data(), 0);
  }
  // per-layer inputs: the gating workload's hidden states (rounded to the
  // dtype; the layer's GPU LSH gate routes them), or the counts realised as
  // token -> expert assignments (expert-major) for the routed forward
  std::int64_t n_max = 1;
  for (const LayerIn& li : p.layers) {
    std::uint64_t n = 0;
    for (auto c : li.counts) n += c;
    n_max = std::max<std::int64_t>(n_max, std::int64_t(n));
  }
  DevBuf x_dev(size_t(n_max) * size_t(d) * esz), y_dev(size_t(n_max) * size_t(d) * esz);
  DevBuf idx_dev(size_t(n_max) * 4), w_dev(size_t(n_max) * 4);
  HostBuf x_host(size_t(n_max) * size_t(d) * esz);
  std::vector<int32_t> idx_h(static_cast<size_t>(n_max));
  std::vector<float> ones(static_cast<size_t>(n_max), 1.0f);
  cuda_ok(cudaMemcpy(w_dev.p, ones.data(), size_t(n_max) * 4, cudaMemcpyHostToDevice), "H2D");
  infmoe_slot_pool* pool = nullptr;
  abi_ok(infmoe_slot_pool_create(opt.device, p.K, uint64_t(mat * esz), &pool));
  cudaStream_t stream;
  cuda_ok(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
  cudaEvent_t origin;
  cuda_ok(cudaEventCreate(&origin), "event");
  std::string rows = kSummaryHead;
  json meas_all = json::object();
  for (Policy pol : s.policies) {
    if (pol == Policy::Serial) continue;  // the serial baseline is a simulator mode only
    const std::string pname = policy_name(pol);
    std::vector<infmoe_layer*> layers(size_t(L), nullptr);
    for (int l = 0; l < L; ++l) {
      infmoe_layer_desc dsc;
      std::memset(&dsc, 0, sizeof(dsc));
      dsc.d_model = d;
      dsc.d_ff = f;
      dsc.n_experts = E;
      dsc.top_k = 1;
      dsc.dtype = dtype;
      dsc.gate_kind = INFMOE_GATE_LSH;
      dsc.lsh_seed = child_seed(s.seed, 2ull * std::uint64_t(l) + 1);
      dsc.lsh_bits = gating ? w.n_hash_bits : std::max(1, int(std::ceil(std::log2(double(E)))));
      dsc.residency = INFMOE_OFFLOADED;
      dsc.K = p.K;
      dsc.policy = pol == Policy::Greedy ? INFMOE_POLICY_AUTO
                   : pol == Policy::Exact ? INFMOE_POLICY_EXACT
                                          : INFMOE_POLICY_NAIVE;
      dsc.max_tokens = int32_t(n_max);
      dsc.device = opt.device;
      dsc.w_in = w_in[size_t(l % n_sets)]->p;
      dsc.w_out = w_out[size_t(l % n_sets)]->p;
      dsc.hw = {s.hardware->peak_flops, s.hardware->h2d_bandwidth, s.hardware->device_memory,
                s.hardware->reserved_memory};
      dsc.ep_size = 1;
      dsc.skip_empty_experts = s.skip_empty_experts ? 1 : 0;
      dsc.slot_pool = pool;
      abi_ok(infmoe_layer_create(&dsc, &layers[size_t(l)]));
    }
    std::vector<Event> ev_all;
    std::vector<std::vector<std::uint64_t>> meas_counts;
    for (int rep = 0; rep < std::max(1, opt.repeats); ++rep) {
      ev_all.clear();
      meas_counts.clear();
      cuda_ok(cudaEventRecord(origin, stream), "record");
      for (int l = 0; l < L; ++l) {
        const LayerIn& li = p.layers[size_t(l)];
        std::int64_t n = 0;
        for (auto c : li.counts) n += std::int64_t(c);
        const std::uint64_t xs = child_seed(s.seed, 2ull * std::uint64_t(l));
        const double one = 1.0;
        void* xo = x_host.p;
        normal_fill_typed(dtype == INFMOE_DTYPE_BF16 ? 0 : 1, 1, &xs, &one,
                          std::uint64_t(n) * std::uint64_t(d), &xo, 0);
        cuda_ok(cudaMemcpyAsync(x_dev.p, x_host.p, size_t(n) * size_t(d) * esz,
                                cudaMemcpyHostToDevice, stream), "x H2D");
        std::vector<int32_t> counts(static_cast<size_t>(E)), order(static_cast<size_t>(E));
        std::vector<infmoe_event> ev(static_cast<size_t>(2 * E));
        int32_t feas = 0;
        double exposed = 0;
        infmoe_forward_out fo;
        std::memset(&fo, 0, sizeof(fo));
        fo.counts = counts.data();
        fo.order = order.data();
        fo.feasible = &feas;
        fo.events = ev.data();
        fo.exposed_copy_s = &exposed;
        fo.time_origin = origin;
        if (gating) {
          abi_ok(infmoe_layer_forward(layers[size_t(l)], x_dev.p, n, y_dev.p, &fo, stream));
        } else {
          std::int64_t t = 0;
          for (int e = 0; e < E; ++e)
            for (std::uint64_t c = 0; c < li.counts[size_t(e)]; ++c) idx_h[size_t(t++)] = e;
          cuda_ok(cudaMemcpyAsync(idx_dev.p, idx_h.data(), size_t(n) * 4,
                                  cudaMemcpyHostToDevice, stream), "idx H2D");
          abi_ok(infmoe_layer_forward_routed(layers[size_t(l)], x_dev.p, n,
                                             static_cast<const int32_t*>(idx_dev.p),
                                             static_cast<const float*>(w_dev.p), y_dev.p, &fo,
                                             stream));
        }
        for (const infmoe_event& e : ev)
          if (e.stream >= 0) ev_all.push_back({e.stream, l, e.expert_id, e.start, e.end});
        meas_counts.emplace_back(counts.begin(), counts.end());
      }
      cuda_ok(cudaStreamSynchronize(stream), "sync");
    }
    // measured statistics, the replay_check rules (<= K residents), and the
    // simulator's prediction at the MEASURED counts and this scenario's costs
    TimelineStats st;
    st.makespan = 0;
    double c_first = 1e300, c_last = 0;
    std::vector<Costs> mcosts;
    std::vector<std::vector<int>> morders;
    for (int l = 0; l < L; ++l) {
      LayerStats ls;
      ls.layer = l;
      ls.start = 1e300;
      for (const Event& e : ev_all)
        if (e.layer == l) {
          ls.start = std::min(ls.start, e.start);
          ls.end = std::max(ls.end, e.end);
          (e.stream == 0 ? ls.load_busy : ls.compute_busy) += e.end - e.start;
          ls.experts += e.stream == 1;
        }
      st.layers.push_back(ls);
      st.compute_busy += ls.compute_busy;
      st.load_busy += ls.load_busy;
      Geometry gk = g;
      std::vector<std::uint64_t> kept;
      for (auto c : meas_counts[size_t(l)])
        if (!s.skip_empty_experts || c > 0) kept.push_back(c);
      gk.experts = int(kept.size());
      Costs c = kept.empty() ? Costs{} : derive_costs(kept.data(), int(kept.size()), gk,
                                                      *s.hardware);
      c = with_overhead(c, s.event_overhead_s);
      morders.push_back(c.size() ? order_for(c, p.K, pol).order : std::vector<int>{});
      mcosts.push_back(std::move(c));
    }
    for (const Event& e : ev_all) {
      st.makespan = std::max(st.makespan, e.end);
      if (e.stream == 1) {
        c_first = std::min(c_first, e.start);
        c_last = std::max(c_last, e.end);
      }
    }
    st.compute_stall = c_last > c_first ? (c_last - c_first) - st.compute_busy : 0.0;
    st.overlap_efficiency = st.makespan > 0 ? st.compute_busy / st.makespan : 0.0;
    // residency: an expert is resident from its load's end to its compute's end
    {
      std::vector<std::pair<double, int>> marks;
      for (const Event& e : ev_all)
        if (e.stream == 0) {
          for (const Event& c : ev_all)
            if (c.stream == 1 && c.layer == e.layer && c.expert == e.expert) {
              marks.push_back({e.end, 1});
              marks.push_back({c.end - 1e-6, -1});
            }
        }
      std::sort(marks.begin(), marks.end());
      int cur = 0;
      for (auto& m : marks) st.peak_resident = std::max(st.peak_resident, cur += m.second);
    }
    std::vector<Event> sim_ev;
    TimelineStats sim = run_timeline(morders, mcosts, p.K, false, s.continuous_load_stream,
                                     &sim_ev);
    // the audit indexes costs by position: map expert ids to their position
    // among the layer's scheduled experts (all of them unless skip_empty_experts)
    std::vector<Event> audit_ev = ev_all;
    for (Event& e : audit_ev) {
      const auto& mc = meas_counts[size_t(e.layer)];
      int pos = 0;
      for (int x = 0; x < e.expert; ++x) pos += (!s.skip_empty_experts || mc[size_t(x)] > 0);
      e.expert = pos;
    }
    int kinds[6] = {0, 0, 0, 0, 0, 0};
    const int viol = audit_timeline(audit_ev, mcosts, p.K, false, 2e-6, kinds);
    std::uint64_t h2d_bytes = 0;
    for (const Event& e : ev_all) h2d_bytes += e.stream == 0 ? bytes_per_expert(g) : 0;
    json rep = report_json(st, {}, p.K);
    rep["measured"] = true;
    rep["executor"] = "libinfmoe offload executor (K+1 device slots, copy + compute streams)";
    rep["continuous_load_stream"] = s.continuous_load_stream;
    rep["h2d_bytes"] = h2d_bytes;
    rep["h2d_gbs_while_loading"] = st.load_busy > 0 ? double(h2d_bytes) / st.load_busy / 1e9 : 0;
    rep["simulated_makespan_at_measured_counts"] = sim.makespan;
    rep["measured_over_simulated"] = sim.makespan > 0 ? st.makespan / sim.makespan : 0;
    rep["replay_check_violations"] = viol;
    rep["replay_check_kinds"] = std::vector<int>(kinds, kinds + 6);
    rep["measured_counts"] = meas_counts;
    write_policy(out / "measured" / pname, s.name, pname, ev_all, rep, opt.trace_format);
    rows += summary_row(pname, st, p.K, L);
    for (infmoe_layer* ly : layers) infmoe_layer_destroy(ly);
  }
  cudaEventDestroy(origin);
  cudaStreamDestroy(stream);
  infmoe_slot_pool_destroy(pool);
  write_file(out / "measured" / "summary.csv", rows);
  return rows;
}

}  // namespace

std::string run(const Scenario& s, const RunOptions& opt) {
  const fs::path out = opt.out_dir.empty() ? fs::path(s.output_dir) : fs::path(opt.out_dir);
  Prepared p = prepare(s);
  std::string rows = kSummaryHead;
  for (Policy pol : s.policies) {
    Result r = simulate(p, pol, s.continuous_load_stream);
    json rep = report_json(r.stats, r.plans, p.K);
    rep["policy"] = policy_name(pol);
    rep["warnings"] = p.warnings;
    write_policy(out / policy_name(pol), s.name, policy_name(pol), r.events, rep,
                 opt.trace_format);
    rows += summary_row(policy_name(pol), r.stats, p.K, s.n_moe_layers);
  }
  write_file(out / "summary.csv", rows);
  write_file(out / "resolved.json", resolved_json(s));
  const auto now = std::chrono::system_clock::now().time_since_epoch();
  json meta = {{"tool", "infmoe run"},
               {"version", infmoe_version()},
               {"unix_time_s", std::chrono::duration<double>(now).count()},
               {"note", "timestamps live only here; every other artifact is reproducible"}};
  if (opt.execute) {
    if (s.alphas) fail(kConfig, "execute: explicit costs have no model to run");
    meta["measured_summary"] = execute(s, p, opt, out);
  }
  write_file(out / "meta.json", meta.dump(1));
  return rows;
}

std::string sweep(const Scenario& base, const std::string& axis,
                  const std::vector<double>& values, const RunOptions& opt, int jobs) {
  if (axis != "K" && axis != "total_tokens" && axis != "zipf_s" && axis != "bandwidth")
    fail(kConfig, "sweep: unknown axis '" + axis + "' (K | total_tokens | zipf_s | bandwidth)");
  if (values.empty()) fail(kConfig, "sweep: no values");
  std::vector<Scenario> pts;
  for (double v : values) {
    Scenario s = base;
    if (axis == "K") {
      if (v != std::floor(v)) fail(kConfig, "sweep: K values must be integers");
      if (v < 1) fail(kCapacity, "K: must be >= 1");
      s.k_explicit = int(v);
    } else if (axis == "total_tokens") {
      if (!s.workload || s.workload->kind == WorkloadKind::Explicit ||
          s.workload->kind == WorkloadKind::Csv)
        fail(kConfig, "sweep: axis 'total_tokens' needs a gating / uniform / zipf / balanced "
                      "workload");
      if (v < 0 || v != std::floor(v)) fail(kConfig, "sweep: total_tokens must be >= 0 integers");
      s.workload->total_tokens = std::uint64_t(v);
    } else if (axis == "zipf_s") {
      if (!s.workload || s.workload->kind != WorkloadKind::Zipf)
        fail(kConfig, "sweep: axis 'zipf_s' needs a zipf workload");
      if (!(v > 0.0)) fail(kConfig, "workload.zipf_s: must be > 0");
      s.workload->zipf_s = v;
    } else {
      if (!s.hardware) fail(kConfig, "sweep: axis 'bandwidth' needs a hardware profile");
      if (!(v > 0.0)) fail(kConfig, "hardware.h2d_bandwidth must be > 0");
      s.hardware->h2d_bandwidth = v;
    }
    pts.push_back(std::move(s));
  }
  const fs::path out = opt.out_dir.empty() ? fs::path(base.output_dir) : fs::path(opt.out_dir);
  std::vector<std::string> point_rows(pts.size());
  std::vector<std::exception_ptr> errors(pts.size());
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i = next++; i < pts.size(); i = next++) {
      try {
        RunOptions o = opt;
        o.out_dir = (out / (axis + "=" + num(values[i]))).string();
        const std::string rows = run(pts[i], o);
        const Prepared p = prepare(pts[i]);
        const Costs& c0 = p.layers.front().costs;
        std::istringstream in(rows);
        std::string line;
        std::getline(in, line);  // header
        while (std::getline(in, line)) {
          // policy,makespan,busy,load_busy,stall,eff,peak,K,L
          std::vector<std::string> f;
          std::stringstream ls(line);
          for (std::string x; std::getline(ls, x, ',');) f.push_back(x);
          point_rows[i] += axis + "," + num(values[i]) + "," + f[0] + "," + f[1] + "," + f[4] +
                           "," + f[5] + "," + num(c0.beta) + "," + num(c0.alpha_sum()) + "," +
                           f[7] + "\n";
        }
      } catch (...) {
        errors[i] = std::current_exception();
      }
    }
  };
  const int nj = opt.execute ? 1 : std::max(1, jobs);
  std::vector<std::thread> th;
  for (int t = 1; t < nj; ++t) th.emplace_back(work);
  work();
  for (auto& t : th) t.join();
  for (size_t i = 0; i < pts.size(); ++i)
    if (errors[i]) std::rethrow_exception(errors[i]);  // the first failing point, in value order
  std::string csv =
      "axis,value,policy,makespan_s,compute_stall_s,overlap_efficiency,beta_s,sum_alpha_s,K\n";
  for (const std::string& r : point_rows) csv += r;  // value order, whatever the jobs
  write_file(out / "sweep.csv", csv);
  return csv;
}

}  // namespace infmoe::scn
