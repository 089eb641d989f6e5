// loopback_nccl.cpp — TEST INFRASTRUCTURE.  A stand-in for the handful of NCCL
// entry points libinfmoe.so binds (nccl_shim.hpp), for running P expert-
// parallel ranks as P host threads on ONE GPU.  Each rank calls the real
// Layer::forward; ncclSend/ncclRecv become stream-ordered device-to-device
// copies matched on the host:
//   * GroupEnd posts every send (with an event recorded on the sender's
//     stream) and every receive, then for each receive waits on the host for
//     its matching send, makes the receiver's stream wait for the sender's
//     event, copies, and records a done-event; each send then waits on the host
//     for that done-event and makes the sender's stream wait on it.
// No kernel ever waits on another rank's kernel; the GPU only sees copies and
// event waits.  Loaded by setting INFMOE_NCCL_LIB to this library's path.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <tuple>
#include <vector>

namespace {

struct Comm {
  uint64_t key;
  int nranks, rank;
  std::map<int, uint64_t> send_seq, recv_seq;  // per peer
};

struct Slot {  // one matched send/recv pair
  bool sent = false, received = false;
  const void* src = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr;  // recorded on the sender's stream
  cudaEvent_t done = nullptr;   // recorded on the receiver's stream after the copy
};

std::mutex g_mu;
std::condition_variable g_cv;
std::map<std::tuple<uint64_t, int, int, uint64_t>, std::shared_ptr<Slot>> g_slots;

struct Op {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  Comm* comm;
  cudaStream_t stream;
};
thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;

size_t elem_size(int dt) {  // ncclDataType_t codes
  if (dt == 2 || dt == 3 || dt == 7) return 4;
  if (dt == 4 || dt == 5 || dt == 8) return 8;
  if (dt == 6 || dt == 9) return 2;
  return 1;
}

std::shared_ptr<Slot> slot(uint64_t key, int src, int dst, uint64_t seq) {
  auto& s = g_slots[{key, src, dst, seq}];
  if (!s) s = std::make_shared<Slot>();
  return s;
}

int run(const std::vector<Op>& ops) {
  std::vector<std::pair<Op, std::shared_ptr<Slot>>> sends, recvs;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (const Op& o : ops) {
      Comm* c = o.comm;
      if (o.send) {
        auto s = slot(c->key, c->rank, o.peer, c->send_seq[o.peer]++);
        cudaEventCreateWithFlags(&s->ready, cudaEventDisableTiming);
        cudaEventRecord(s->ready, o.stream);
        s->src = o.buf;
        s->bytes = o.bytes;
        s->sent = true;
        sends.push_back({o, s});
      } else {
        recvs.push_back({o, slot(c->key, o.peer, c->rank, c->recv_seq[o.peer]++)});
      }
    }
  }
  g_cv.notify_all();
  for (auto& [o, s] : recvs) {
    std::unique_lock<std::mutex> lk(g_mu);
    g_cv.wait(lk, [&] { return s->sent; });
    if (s->bytes != o.bytes) return 3;  // ncclInvalidArgument: size mismatch
    cudaStreamWaitEvent(o.stream, s->ready, 0);
    if (o.bytes) cudaMemcpyAsync(o.buf, s->src, o.bytes, cudaMemcpyDeviceToDevice, o.stream);
    cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming);
    cudaEventRecord(s->done, o.stream);
    s->received = true;
    lk.unlock();
    g_cv.notify_all();
  }
  for (auto& [o, s] : sends) {
    std::unique_lock<std::mutex> lk(g_mu);
    g_cv.wait(lk, [&] { return s->received; });
    cudaStreamWaitEvent(o.stream, s->done, 0);
  }
  return 0;
}

}  // namespace

extern "C" {
typedef struct { char internal[128]; } ncclUniqueId;

int ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof(*id));
  uint64_t key = std::random_device{}() ^ (uint64_t(std::random_device{}()) << 32);
  std::memcpy(id->internal, &key, sizeof(key));
  return 0;
}
int ncclCommInitRank(Comm** comm, int nranks, ncclUniqueId id, int rank) {
  uint64_t key;
  std::memcpy(&key, id.internal, sizeof(key));
  *comm = new Comm{key, nranks, rank, {}, {}};
  return 0;
}
int ncclCommDestroy(Comm* comm) {
  delete comm;
  return 0;
}
int ncclGroupStart() {
  ++t_depth;
  return 0;
}
int ncclGroupEnd() {
  if (--t_depth > 0) return 0;
  std::vector<Op> ops;
  ops.swap(t_ops);
  return run(ops);
}
int ncclSend(const void* buf, size_t count, int dt, int peer, Comm* comm, cudaStream_t s) {
  Op o{true, const_cast<void*>(buf), count * elem_size(dt), peer, comm, s};
  if (t_depth > 0) { t_ops.push_back(o); return 0; }
  return run({o});
}
int ncclRecv(void* buf, size_t count, int dt, int peer, Comm* comm, cudaStream_t s) {
  Op o{false, buf, count * elem_size(dt), peer, comm, s};
  if (t_depth > 0) { t_ops.push_back(o); return 0; }
  return run({o});
}
// collectives as P-1 sends + P-1 receives per rank through the same matcher,
// plus a local copy / reduction; a sum all-reduce of int32 or float only
int ncclAllGather(const void* send, void* recv, size_t count, int dt, Comm* comm,
                  cudaStream_t s) {
  const size_t bytes = count * elem_size(dt);
  std::vector<Op> ops;
  for (int r = 0; r < comm->nranks; ++r) {
    if (r == comm->rank) continue;
    ops.push_back(Op{true, const_cast<void*>(send), bytes, r, comm, s});
    ops.push_back(Op{false, static_cast<uint8_t*>(recv) + size_t(r) * bytes, bytes, r, comm, s});
  }
  if (bytes) cudaMemcpyAsync(static_cast<uint8_t*>(recv) + size_t(comm->rank) * bytes, send, bytes,
                             cudaMemcpyDeviceToDevice, s);
  return run(ops);
}
int ncclAllReduce(const void* send, void* recv, size_t count, int dt, int op, Comm* comm,
                  cudaStream_t s) {
  if (op != 0 || !(dt == 2 || dt == 7)) return 5;  // ncclInvalidUsage: sum of int32/f32 only
  const size_t bytes = count * 4;
  std::vector<uint8_t> mine(bytes), other(bytes), acc(bytes);
  void* stage = nullptr;
  cudaMalloc(&stage, bytes * size_t(comm->nranks));
  int rc = ncclAllGather(send, stage, count, dt, comm, s);
  if (rc) return rc;
  cudaStreamSynchronize(s);  // host reduction (test transport: correctness, not speed)
  std::vector<uint8_t> all(bytes * size_t(comm->nranks));
  cudaMemcpy(all.data(), stage, all.size(), cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < count; ++i) {
    if (dt == 2) {
      int32_t v = 0;
      for (int r = 0; r < comm->nranks; ++r) v += reinterpret_cast<int32_t*>(all.data() + r * bytes)[i];
      reinterpret_cast<int32_t*>(acc.data())[i] = v;
    } else {
      float v = 0.f;
      for (int r = 0; r < comm->nranks; ++r) v += reinterpret_cast<float*>(all.data() + r * bytes)[i];
      reinterpret_cast<float*>(acc.data())[i] = v;
    }
  }
  cudaMemcpy(recv, acc.data(), bytes, cudaMemcpyHostToDevice);
  cudaFree(stage);
  return 0;
}
const char* ncclGetErrorString(int r) { return r ? "loopback transport error" : "no error"; }
int ncclGetVersion(int* v) {
  *v = 22809;
  return 0;
}
}
