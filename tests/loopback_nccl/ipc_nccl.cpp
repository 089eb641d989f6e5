// ipc_nccl.cpp — TEST INFRASTRUCTURE.  A process-shared stand-in for the two
// NCCL collectives the PEER expert-parallel transport uses (nccl_shim.hpp):
// ncclAllGather (the one-time exchange of pids, pointers and CUDA IPC handles
// at layer create) and ncclAllReduce (the 1-int barriers, with
// INFMOE_EP_BARRIER=nccl).  P ranks are P PROCESSES on one GPU sharing a
// /dev/shm segment named after the unique id: each collective synchronises the
// caller's stream, meets the other ranks at a host barrier in shared memory,
// and copies through the segment -- so no kernel ever waits on another rank's
// kernel, while the layer's peer buffers really are CUDA-IPC mappings across
// processes.  Point-to-point send/recv are not provided (the PEER transport
// does not use them).  Loaded by setting INFMOE_NCCL_LIB to this library.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

namespace {
constexpr size_t kData = 1 << 20;  // bytes per rank slot
constexpr int kMaxRanks = 8;

struct Shared {
  std::atomic<uint32_t> arrived;
  std::atomic<uint32_t> generation;
  uint8_t data[kMaxRanks][kData];
};

struct Comm {
  int nranks, rank;
  Shared* sh;
  char name[64];
};

void barrier(Comm* c) {
  Shared* s = c->sh;
  const uint32_t gen = s->generation.load();
  if (s->arrived.fetch_add(1) + 1 == uint32_t(c->nranks)) {
    s->arrived.store(0);
    s->generation.fetch_add(1);
  } else {
    while (s->generation.load() == gen) sched_yield();
  }
}

size_t elem_size(int dt) {
  if (dt == 2 || dt == 3 || dt == 7) return 4;
  if (dt == 4 || dt == 5 || dt == 8) return 8;
  if (dt == 6 || dt == 9) return 2;
  return 1;
}
}  // namespace

extern "C" {
typedef struct {
  char internal[128];
} ncclUniqueId;

int ncclGetUniqueId(ncclUniqueId* id) {
  std::random_device rd;
  std::snprintf(id->internal, sizeof(id->internal), "infmoe_ipc_%08x%08x", rd(), rd());
  return 0;
}

int ncclCommInitRank(Comm** out, int nranks, ncclUniqueId id, int rank) {
  if (nranks > kMaxRanks) return 1;
  auto* c = new Comm{nranks, rank, nullptr, {}};
  // the unique id's bytes name the segment (any 128 bytes: hex of the first 16)
  char nm[64] = "/infmoe_ipc_";
  for (int i = 0; i < 16; ++i)
    std::snprintf(nm + 12 + 2 * i, 3, "%02x", uint8_t(id.internal[i]));
  std::memcpy(c->name, nm, sizeof(nm));
  const int fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return 1;
  if (ftruncate(fd, sizeof(Shared)) != 0) return 1;
  void* p = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return 1;
  c->sh = static_cast<Shared*>(p);  // zero-filled on creation: counters start at 0
  barrier(c);                        // every rank attached
  *out = c;
  return 0;
}

int ncclCommDestroy(Comm* c) {
  barrier(c);
  munmap(c->sh, sizeof(Shared));
  if (c->rank == 0) shm_unlink(c->name);
  delete c;
  return 0;
}

int ncclGroupStart() { return 0; }
int ncclGroupEnd() { return 0; }
int ncclSend(const void*, size_t, int, int, Comm*, cudaStream_t) { return 1; }
int ncclRecv(void*, size_t, int, int, Comm*, cudaStream_t) { return 1; }

int ncclAllGather(const void* send, void* recv, size_t count, int dt, Comm* c, cudaStream_t s) {
  const size_t b = count * elem_size(dt);
  if (b > kData) return 1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  if (cudaMemcpy(c->sh->data[c->rank], send, b, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  barrier(c);
  for (int r = 0; r < c->nranks; ++r)
    if (cudaMemcpy(static_cast<uint8_t*>(recv) + size_t(r) * b, c->sh->data[r], b,
                   cudaMemcpyHostToDevice) != cudaSuccess)
      return 1;
  barrier(c);  // nobody overwrites a slot before everyone read it
  return 0;
}

int ncclAllReduce(const void* send, void* recv, size_t count, int dt, int op, Comm* c,
                  cudaStream_t s) {
  if (dt != 2 || op != 0 || count * 4 > kData) return 1;  // int32 sum (the barrier)
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  if (cudaMemcpy(c->sh->data[c->rank], send, count * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 1;
  barrier(c);
  int32_t acc[256] = {};
  const size_t n = count < 256 ? count : 256;
  for (int r = 0; r < c->nranks; ++r)
    for (size_t i = 0; i < n; ++i) acc[i] += reinterpret_cast<int32_t*>(c->sh->data[r])[i];
  barrier(c);
  return cudaMemcpy(recv, acc, n * 4, cudaMemcpyHostToDevice) == cudaSuccess ? 0 : 1;
}

const char* ncclGetErrorString(int r) { return r ? "ipc stand-in transport error" : "no error"; }
int ncclGetVersion(int* v) {
  *v = 22809;
  return 0;
}
}
