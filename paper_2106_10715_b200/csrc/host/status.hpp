// status.hpp — error taxonomy of libinfmoe and the exception→status-code guard
// used at every extern "C" entry point (no C++ exception crosses the C-ABI).
// Codes follow moesim's CLI mapping (errors.hpp:8-21).
#pragma once

#include <exception>
#include <stdexcept>
#include <string>

namespace infmoe {

enum Status : int {
  kOk = 0,
  kConfig = 2,     // moesim::ConfigError
  kCapacity = 3,   // moesim::CapacityError
  kInvariant = 4,  // moesim::InvariantError
  kRuntime = 5,    // CUDA / NCCL failure
  kArgument = 6,   // std::invalid_argument (malformed call, e.g. not a permutation)
};

struct Error : std::runtime_error {
  Status code;
  Error(Status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(Status c, const std::string& m) { throw Error(c, m); }
inline void require(bool ok, const std::string& m) {
  if (!ok) fail(kArgument, m);
}

void set_last_error(const std::string& m);

template <class F>
int guarded(F&& f) noexcept {
  try {
    f();
    return kOk;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return kArgument;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return kRuntime;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return kInvariant;
  } catch (...) {
    set_last_error("unknown C++ exception");
    return kInvariant;
  }
}

}  // namespace infmoe
