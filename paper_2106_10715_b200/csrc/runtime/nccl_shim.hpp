// nccl_shim.hpp — the few NCCL entry points the EP exchange uses, resolved at
// run time with dlopen so libinfmoe.so has no link-time NCCL dependency and,
// inside a process that already loaded torch's NCCL, shares that copy
// (RTLD_NOLOAD first).  Only stable core API (since NCCL 2.7) is used.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace infmoe {
namespace nccl {

typedef struct ncclComm* Comm;
struct UniqueId {
  char internal[128];
};
enum DataType { kUint8 = 1, kInt32 = 2 };
enum RedOp { kSum = 0 };

struct Api {
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  int (*GetVersion)(int*) = nullptr;
};

// Loads NCCL on first use; throws Error(kRuntime) when it is unavailable.
const Api& api();
void check(int result, const char* what);

}  // namespace nccl
}  // namespace infmoe
