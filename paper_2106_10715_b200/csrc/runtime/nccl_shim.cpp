// nccl_shim.cpp — see nccl_shim.hpp.
#include "nccl_shim.hpp"

#include <dlfcn.h>

#include <cstdlib>

#include <mutex>
#include <string>

#include "../host/status.hpp"

namespace infmoe {
namespace nccl {

namespace {
Api g_api;
std::string g_error;

template <class F>
void bind(void* h, F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  if (!fn) g_error += std::string(" missing ") + name;
}
}  // namespace

const Api& api() {
  static std::once_flag once;
  std::call_once(once, [] {
    // INFMOE_NCCL_LIB names another implementation of these entry points
    // (tests/loopback_nccl: P ranks as threads on one GPU)
    const char* over = std::getenv("INFMOE_NCCL_LIB");
    void* h = over ? dlopen(over, RTLD_NOW | RTLD_LOCAL) : nullptr;
    if (over && !h) {
      g_error = std::string("cannot dlopen INFMOE_NCCL_LIB: ") + dlerror();
      return;
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_error = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    bind(h, g_api.GetUniqueId, "ncclGetUniqueId");
    bind(h, g_api.CommInitRank, "ncclCommInitRank");
    bind(h, g_api.CommDestroy, "ncclCommDestroy");
    bind(h, g_api.GroupStart, "ncclGroupStart");
    bind(h, g_api.GroupEnd, "ncclGroupEnd");
    bind(h, g_api.Send, "ncclSend");
    bind(h, g_api.Recv, "ncclRecv");
    bind(h, g_api.AllGather, "ncclAllGather");
    bind(h, g_api.AllReduce, "ncclAllReduce");
    bind(h, g_api.GetErrorString, "ncclGetErrorString");
    bind(h, g_api.GetVersion, "ncclGetVersion");
  });
  if (!g_error.empty()) fail(kRuntime, "NCCL unavailable:" + g_error);
  return g_api;
}

void check(int result, const char* what) {
  if (result != 0) {
    const char* msg = g_api.GetErrorString ? g_api.GetErrorString(result) : "?";
    fail(kRuntime, std::string(what) + ": NCCL error " + std::to_string(result) + " (" + msg + ")");
  }
}

}  // namespace nccl
}  // namespace infmoe
