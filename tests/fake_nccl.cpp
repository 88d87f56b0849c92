// fake_nccl.cpp -- TEST INFRASTRUCTURE ONLY: an in-process stand-in for
// the libnccl point-to-point entry points libtsim opens at run time
// (TSIM_NCCL_LIB=<this .so>), so the library's native exchange path
// (ts_nccl_init, ts_exchange, ts_step with neighbours: nccl_exchange in
// tsim_api.cu) runs with real partners on ONE GPU: every rank is a handle
// of the same process driven from its own host thread.
//
// A send / recv pair is matched on the host (per sender, receiver and call
// order) and carried out as one device-to-device copy on the receiver's
// stream, after the sender's stream has reached the send (event) and
// before the sender's stream goes on (event): stream order only, nothing on
// the GPU waits on another kernel.  ncclGroupEnd posts the group's sends,
// then performs its receives (blocking on the host until the matching send
// is posted), then waits until its sends have been consumed -- the rendezvous
// semantics of NCCL's grouped point-to-point calls.  Only the entry points
// libtsim uses are provided; types are ABI-compatible stand-ins.
#include <cuda.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

extern "C" {
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // 0 = ncclSuccess
}

namespace {
constexpr ncclResult_t kOk = 0, kSystemError = 2, kInvalidArgument = 4, kInvalidUsage = 5;

struct Msg {
  CUdeviceptr src = 0;
  size_t bytes = 0;
  CUevent ready = nullptr, done = nullptr;
};
struct World {
  int n = 0;
  std::map<std::tuple<int, int, uint64_t>, Msg> msgs;  // (from, to, seq)
};
std::mutex g_mu;
std::condition_variable g_cv;
std::map<uint64_t, World> g_worlds;  // by unique id
uint64_t g_next_id = 1;

struct Comm {
  World *w;
  int rank;
  std::map<int, uint64_t> sent, recvd;  // per peer: calls so far
};
struct Op {
  bool send;
  CUdeviceptr buf;
  size_t bytes;
  int peer;
  Comm *comm;
  CUstream stream;
};
thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;

ncclResult_t run_group(std::vector<Op> &ops) {
  struct Posted {
    World *w;
    std::tuple<int, int, uint64_t> key;
    CUstream stream;
  };
  std::vector<Posted> posted;
  for (Op &o : ops)  // 1. post the sends
    if (o.send) {
      Msg m;
      m.src = o.buf;
      m.bytes = o.bytes;
      if (cuEventCreate(&m.ready, CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS ||
          cuEventRecord(m.ready, o.stream) != CUDA_SUCCESS)
        return kSystemError;
      std::lock_guard<std::mutex> lk(g_mu);
      const auto key = std::make_tuple(o.comm->rank, o.peer, o.comm->sent[o.peer]++);
      o.comm->w->msgs[key] = m;
      posted.push_back(Posted{o.comm->w, key, o.stream});
      g_cv.notify_all();
    }
  for (Op &o : ops)  // 2. the receives: copy once the matching send is posted
    if (!o.send) {
      std::unique_lock<std::mutex> lk(g_mu);
      const auto key = std::make_tuple(o.peer, o.comm->rank, o.comm->recvd[o.peer]++);
      auto &msgs = o.comm->w->msgs;
      g_cv.wait(lk, [&] { return msgs.count(key) != 0; });
      Msg &m = msgs[key];
      if (m.bytes != o.bytes) return kInvalidUsage;  // sizes must match, as in NCCL
      CUevent done;
      if (cuStreamWaitEvent(o.stream, m.ready, 0) != CUDA_SUCCESS ||
          (o.bytes && cuMemcpyDtoDAsync(o.buf, m.src, o.bytes, o.stream) != CUDA_SUCCESS) ||
          cuEventCreate(&done, CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS ||
          cuEventRecord(done, o.stream) != CUDA_SUCCESS)
        return kSystemError;
      m.done = done;
      g_cv.notify_all();
    }
  for (Posted &p : posted) {  // 3. the sender's stream goes on after the copy
    std::unique_lock<std::mutex> lk(g_mu);
    g_cv.wait(lk, [&] { return p.w->msgs[p.key].done != nullptr; });
    Msg m = p.w->msgs[p.key];
    p.w->msgs.erase(p.key);
    lk.unlock();
    if (cuStreamWaitEvent(p.stream, m.done, 0) != CUDA_SUCCESS) return kSystemError;
    cuEventDestroy(m.ready);  // released once their pending work completes
    cuEventDestroy(m.done);
  }
  return kOk;
}
}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId *id) {
  if (!id) return kInvalidArgument;
  std::lock_guard<std::mutex> lk(g_mu);
  memset(id, 0, sizeof *id);
  const uint64_t v = g_next_id++;
  memcpy(id->internal, &v, sizeof v);
  return kOk;
}

ncclResult_t ncclCommInitRank(void **comm, int nranks, ncclUniqueId id, int rank) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return kInvalidArgument;
  uint64_t v;
  memcpy(&v, id.internal, sizeof v);
  std::lock_guard<std::mutex> lk(g_mu);
  World &w = g_worlds[v];
  if (w.n == 0) w.n = nranks;
  if (w.n != nranks) return kInvalidUsage;
  *comm = new Comm{&w, rank, {}, {}};
  return kOk;
}

ncclResult_t ncclCommDestroy(void *comm) {
  delete static_cast<Comm *>(comm);
  return kOk;
}

ncclResult_t ncclGroupStart() {
  t_depth++;
  return kOk;
}

ncclResult_t ncclGroupEnd() {
  if (t_depth <= 0) return kInvalidUsage;
  if (--t_depth > 0) return kOk;
  std::vector<Op> ops;
  ops.swap(t_ops);
  return run_group(ops);
}

static ncclResult_t p2p(bool send, const void *buf, size_t count, int dtype, int peer, void *comm,
                        void *stream) {
  if (dtype != 0 && dtype != 1) return kInvalidArgument;  // ncclInt8 / ncclUint8 only
  Comm *c = static_cast<Comm *>(comm);
  if (!c || peer < 0 || peer >= c->w->n || peer == c->rank) return kInvalidArgument;
  t_ops.push_back(Op{send, (CUdeviceptr)buf, count, peer, c, (CUstream)stream});
  if (t_depth > 0) return kOk;
  std::vector<Op> ops;  // an ungrouped call is a group of one
  ops.swap(t_ops);
  return run_group(ops);
}

ncclResult_t ncclSend(const void *buf, size_t count, int dtype, int peer, void *comm, void *stream) {
  return p2p(true, buf, count, dtype, peer, comm, stream);
}

ncclResult_t ncclRecv(void *buf, size_t count, int dtype, int peer, void *comm, void *stream) {
  return p2p(false, buf, count, dtype, peer, comm, stream);
}

const char *ncclGetErrorString(ncclResult_t r) {
  return r == kOk ? "success" : r == kInvalidUsage ? "invalid usage (fake)" : "error (fake)";
}
}
