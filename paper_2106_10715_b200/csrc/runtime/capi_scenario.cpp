// capi_scenario.cpp — extern "C" entry points of the scenario front door
// (include/infmoe.h "scenario.hpp" section).  Every call is exception-guarded.
#include <cstring>
#include <string>

#include "../host/scenario.hpp"
#include "../host/status.hpp"
#include "infmoe.h"

using namespace infmoe;

namespace {
void emit(const std::string& s, char* out, uint64_t cap, uint64_t* len) {
  if (len) *len = uint64_t(s.size()) + 1;
  if (out && cap > 0) {
    const size_t n = std::min<size_t>(s.size(), size_t(cap - 1));
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
}
scn::RunOptions options(const infmoe_run_options* o) {
  scn::RunOptions r;
  if (!o) return r;
  if (o->out_dir) r.out_dir = o->out_dir;
  r.trace_format = o->trace_format > 0 ? o->trace_format : 3;
  r.execute = o->execute != 0;
  r.device = o->device;
  r.host_sets = o->host_sets > 0 ? o->host_sets : 1;
  r.repeats = o->repeats > 0 ? o->repeats : 1;
  return r;
}
scn::Scenario load(const char* path, const infmoe_run_options* o) {
  require(path != nullptr, "scenario: NULL path");
  scn::Scenario s = scn::parse_file(path, scn::effective_presets());
  if (o && o->has_seed) s.seed = o->seed;  // --seed overrides the config
  return s;
}
}  // namespace

extern "C" {

int infmoe_scenario_resolve(const char* json_text, char* out, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    require(json_text != nullptr, "scenario: NULL text");
    emit(scn::resolved_json(scn::parse(json_text, scn::effective_presets())), out, cap, len);
  });
}

int infmoe_scenario_resolve_file(const char* path, char* out, uint64_t cap, uint64_t* len) {
  return guarded([&] { emit(scn::resolved_json(load(path, nullptr)), out, cap, len); });
}

int infmoe_scenario_run(const char* path, const infmoe_run_options* opt, char* summary,
                        uint64_t cap, uint64_t* len) {
  return guarded([&] { emit(scn::run(load(path, opt), options(opt)), summary, cap, len); });
}

int infmoe_scenario_sweep(const char* path, const char* axis, const double* values,
                          int32_t n_values, const infmoe_run_options* opt, char* table,
                          uint64_t cap, uint64_t* len) {
  return guarded([&] {
    require(axis && (values || n_values == 0), "sweep: NULL argument");
    std::vector<double> v(values, values + std::max(0, n_values));
    emit(scn::sweep(load(path, opt), axis, v, options(opt), opt ? opt->jobs : 1), table, cap,
         len);
  });
}

}  // extern "C"
