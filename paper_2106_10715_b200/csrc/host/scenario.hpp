// scenario.hpp — the scenario front door: a strict JSON config
// (scenario.hpp:87-332 of the reference: unknown keys rejected, presets plus
// the MOE_SIM_PRESETS directory, K = integer or "auto", seed resolved from
// entropy when omitted), its resolved round-trip form (scenario.hpp:347-406),
// and the `run` / `sweep` pipelines of SPEC.md:356-388 that turn a scenario
// into per-policy simulated timelines and, on a GPU, MEASURED timelines of the
// real offload executor, written as Chrome trace / CSV / report JSON.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "planner.hpp"

namespace infmoe::scn {

enum class Policy { Greedy, Naive, Serial, Exact };
enum class WorkloadKind { Gating, Uniform, Zipf, Balanced, Explicit, Csv };

struct Workload {
  WorkloadKind kind = WorkloadKind::Balanced;
  std::uint64_t total_tokens = 0;
  double zipf_s = 1.0;
  std::vector<std::uint64_t> counts;  // explicit
  std::string csv_path;               // csv
  int n_hash_bits = 5;                // gating
  int hidden_dim = 0;                 // gating; 0 = d_model
};

struct Scenario {
  std::string name = "scenario";
  std::optional<Geometry> geometry;
  std::string geometry_preset;
  std::optional<Hardware> hardware;
  std::optional<Workload> workload;
  std::optional<std::vector<double>> alphas;  // explicit costs
  double beta = 0.0;
  std::optional<int> k_explicit;  // nullopt = "auto"
  std::vector<Policy> policies;
  std::uint64_t seed = 0;
  int n_moe_layers = 1;
  bool continuous_load_stream = false;
  bool skip_empty_experts = false;
  double event_overhead_s = 0.0;
  std::string output_dir = "out";
};

using Presets = std::map<std::string, Geometry>;

const char* policy_name(Policy p);
const char* workload_name(WorkloadKind k);
Presets builtin_presets();
Presets presets_from_dir(const std::string& dir);
Presets effective_presets();  // builtins + $MOE_SIM_PRESETS (shadowing)

// parse + validate a JSON document (errors: Error{kConfig | kCapacity})
Scenario parse(const std::string& json_text, const Presets& presets);
Scenario parse_file(const std::string& path, const Presets& presets);
// the resolved, self-contained form (indent 2, keys sorted)
std::string resolved_json(const Scenario& s);

struct RunOptions {
  std::string out_dir;       // empty: the scenario's output_dir
  int trace_format = 3;      // bit 0 chrome, bit 1 csv
  bool execute = false;      // also run the real offload executor on the GPU
  int device = 0;
  int host_sets = 1;         // distinct host weight sets aliased across layers (execute)
  int repeats = 1;           // measured forwards per layer (execute); the last is reported
};

// One scenario: per policy <out>/<policy>/{trace.json, events.csv, report.json},
// <out>/summary.csv, <out>/resolved.json, <out>/meta.json (timestamps only);
// with execute, the same under <out>/measured/.  Returns the summary rows.
std::string run(const Scenario& s, const RunOptions& opt);
// A sweep over one axis (K | total_tokens | zipf_s | bandwidth): one run per
// value under <out>/<axis>=<value>/ and <out>/sweep.csv, rows in value order;
// `jobs` points simulate concurrently (results do not depend on it).
std::string sweep(const Scenario& base, const std::string& axis,
                  const std::vector<double>& values, const RunOptions& opt, int jobs);

}  // namespace infmoe::scn
