// scenario_demo.cpp — the scenario front door from C++ through the drop-in
// header (include/infmoe/moesim.hpp -> libinfmoe.so): resolve, run and sweep a
// scenario file.  Built and run by tests/test_scenario.py.
#include <cstdio>
#include <string>
#include <vector>

#include "infmoe/moesim.hpp"

namespace ms = infmoe::moesim;

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string cfg = argv[1], out = argv[2];
  const std::string resolved = ms::resolve_scenario_file(cfg);
  if (ms::resolve_scenario(resolved) != resolved) {  // the resolved form is a fixed point
    std::printf("resolve not idempotent\n");
    return 1;
  }
  infmoe_run_options o{};
  const std::string run_dir = out + "/run";
  o.out_dir = run_dir.c_str();
  const std::string summary = ms::run_scenario(cfg, &o);
  const std::string sweep_dir = out + "/sweep";
  o.out_dir = sweep_dir.c_str();
  o.jobs = 2;
  const std::string table = ms::sweep_scenario(cfg, "K", {1, 2, 4}, &o);
  bool threw = false;
  try {
    ms::sweep_scenario(cfg, "colour", {1});
  } catch (const ms::ConfigError&) {
    threw = true;
  }
  std::printf("%s---\n%s---\n%s\n", summary.c_str(), table.c_str(), threw ? "ok" : "no-throw");
  return threw ? 0 : 1;
}
