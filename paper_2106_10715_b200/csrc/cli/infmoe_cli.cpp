// infmoe — the scenario CLI: a thin front end over the
// C-ABI (include/infmoe.h).  Exit codes: 0 ok, 2 config error
// (including the library's 6, a malformed argument), 3 capacity, 4 invariant
// breach; 5 CUDA runtime (execute only).
//   infmoe run   <config.json> [--out DIR] [--seed S] [--trace-format chrome|csv|both]
//                [--execute] [--device N] [--host-sets N] [--repeats N]
//   infmoe sweep <config.json> --axis K|total_tokens|zipf_s|bandwidth --values a,b,c
//                [--jobs N] [same options]
//   infmoe resolve <config.json>      (the resolved, self-contained scenario JSON)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "infmoe.h"

static int usage() {
  std::fprintf(stderr,
               "usage: infmoe run|sweep|resolve <config.json> [--out DIR] [--seed S]\n"
               "       [--trace-format chrome|csv|both] [--execute] [--device N]\n"
               "       [--host-sets N] [--repeats N] [--axis A --values a,b,c] [--jobs N]\n");
  return 2;
}

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1];
  const char* path = argv[2];
  infmoe_run_options o;
  std::memset(&o, 0, sizeof(o));
  o.trace_format = 3;
  o.jobs = 1;
  std::string out, axis;
  std::vector<double> values;
  for (int i = 3; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> const char* {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "infmoe: %s needs a value\n", a.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--out") out = next();
    else if (a == "--seed") { o.seed = std::strtoull(next(), nullptr, 10); o.has_seed = 1; }
    else if (a == "--trace-format") {
      const std::string f = next();
      o.trace_format = f == "chrome" ? 1 : f == "csv" ? 2 : f == "both" ? 3 : -1;
      if (o.trace_format < 0) return usage();
    } else if (a == "--execute") o.execute = 1;
    else if (a == "--device") o.device = std::atoi(next());
    else if (a == "--host-sets") o.host_sets = std::atoi(next());
    else if (a == "--repeats") o.repeats = std::atoi(next());
    else if (a == "--jobs") o.jobs = std::atoi(next());
    else if (a == "--axis") axis = next();
    else if (a == "--values") {
      std::string v = next();
      for (size_t p = 0; p <= v.size();) {
        const size_t q = std::min(v.find(',', p), v.size());
        if (q > p) values.push_back(std::strtod(v.substr(p, q - p).c_str(), nullptr));
        p = q + 1;
      }
    } else return usage();
  }
  if (!out.empty()) o.out_dir = out.c_str();
  uint64_t len = 0;
  int rc;
  if (cmd == "resolve") {
    rc = infmoe_scenario_resolve_file(path, nullptr, 0, &len);
    if (rc == 0) {
      std::string s(len, '\0');
      rc = infmoe_scenario_resolve_file(path, s.data(), len, &len);
      std::printf("%s\n", s.c_str());
    }
  } else if (cmd == "run" || cmd == "sweep") {
    std::string s(1 << 20, '\0');
    rc = cmd == "run" ? infmoe_scenario_run(path, &o, s.data(), s.size(), &len)
                      : infmoe_scenario_sweep(path, axis.c_str(), values.data(),
                                              int32_t(values.size()), &o, s.data(), s.size(),
                                              &len);
    if (rc == 0) std::fputs(s.c_str(), stdout);
  } else {
    return usage();
  }
  if (rc != 0) std::fprintf(stderr, "infmoe: %s\n", infmoe_last_error());
  return rc == INFMOE_ERR_ARGUMENT ? INFMOE_ERR_CONFIG : rc;
}
