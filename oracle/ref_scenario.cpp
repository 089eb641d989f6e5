// ref_scenario.cpp — TEST INFRASTRUCTURE.  The reference's scenario parser and
// resolved form (scenario.hpp, UNMODIFIED, included in place) behind one
// extern "C" call, so tests/test_scenario.py can compare libinfmoe's
// infmoe_scenario_resolve with parse_scenario + to_json on the same documents.
#include <cstring>
#include <string>

#include "moesim/scenario.hpp"

using namespace moesim;

extern "C" {
// rc: 0 ok, 2 ConfigError, 3 CapacityError, 4 other; out gets the resolved
// JSON (dump(2)) or the error message
int ref_scenario_resolve(const char* text, char* out, unsigned long long cap) {
  std::string s;
  int rc = 0;
  try {
    s = to_json(parse_scenario(json::parse(text), effective_presets())).dump(2);
  } catch (const CapacityError& e) {
    rc = 3;
    s = e.what();
  } catch (const ConfigError& e) {
    rc = 2;
    s = e.what();
  } catch (const std::exception& e) {
    rc = 4;
    s = e.what();
  }
  std::strncpy(out, s.c_str(), cap - 1);
  out[cap - 1] = '\0';
  return rc;
}
}
