// Test-only NCCL stand-in: the subset of the NCCL API libfastusp calls, implemented for ranks
// that are THREADS of one process sharing a GPU (real NCCL refuses two ranks on one device,
// and this build only ever sees one B200).  Loaded with LD_PRELOAD so that fastusp's own
// NcclComm code path -- ncclCommInitRank, ncclCommSplit, grouped ncclSend/ncclRecv,
// ncclCommGetAsyncError, ncclCommAbort -- runs unchanged at world > 1.
//
// Semantics follow NCCL's point-to-point contract: inside ncclGroupStart/End every rank posts
// its sends, matching is by (communicator, peer, per-pair sequence number), and the transfer
// is stream-ordered on both sides.  A send posts (pointer, bytes, "ready" event on the
// sender's stream); the receiver's stream waits for it and PULLS the bytes with a copy-engine
// cudaMemcpy, then records "done"; the sender's stream waits for "done" before the buffer can
// be reused.  Errors are asynchronous like NCCL's: a rendezvous that does not complete within
// FUSP_SHIM_TIMEOUT_S seconds sets the communicator's async error (ncclRemoteError), which
// ncclCommGetAsyncError reports.  Graph capture is not supported (host rendezvous).
//
// This is test infrastructure (tests/test_gpu_nccl_shim.py); the product links the real NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <tuple>
#include <vector>

namespace {

double timeout_s() {
  const char* e = std::getenv("FUSP_SHIM_TIMEOUT_S");
  return e ? std::atof(e) : 60.0;
}

struct Shared {  // one communicator, shared by its member threads
  explicit Shared(int n) : n(n), send_seq(size_t(n) * n, 0), recv_seq(size_t(n) * n, 0) {}
  int n;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<uint64_t> send_seq, recv_seq;  // [src * n + dst]
  struct Post {
    const void* ptr = nullptr;
    size_t bytes = 0;
    int dev = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
    bool pulled = false;
  };
  std::map<std::tuple<int, int, uint64_t>, Post> posts;  // (src, dst, seq)
  // ncclCommSplit rounds
  struct Split {
    std::vector<std::tuple<int, int, int>> entries;  // (color, key, rank)
    int arrived = 0, left = 0;
    std::map<int, std::shared_ptr<Shared>> comms;  // color -> new communicator
    std::map<int, int> new_rank;                   // old rank -> new rank
    bool ready = false;
  };
  std::map<uint64_t, Split> splits;
  std::vector<uint64_t> split_seq = std::vector<uint64_t>(size_t(n), 0);
};

}  // namespace

struct ncclComm {
  std::shared_ptr<Shared> sh;
  int rank = 0;
  int dev = 0;
  std::atomic<int> err{ncclSuccess};
  bool aborted = false;
};

namespace {

std::mutex g_init_mu;
std::condition_variable g_init_cv;
struct Pending {
  std::shared_ptr<Shared> sh;
  int joined = 0;
};
std::map<std::string, Pending> g_pending;

struct Op {
  bool send;
  ncclComm* comm;
  int peer;
  void* buf;
  size_t bytes;
  cudaStream_t stream;
  uint64_t seq = 0;
};
thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;

template <typename Pred>
bool wait_for(std::unique_lock<std::mutex>& lk, std::condition_variable& cv, Pred p) {
  return cv.wait_until(lk, std::chrono::steady_clock::now() +
                               std::chrono::milliseconds(int64_t(timeout_s() * 1000)), p);
}

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 1;
  }
}

ncclResult_t run_ops(std::vector<Op>& ops) {
  // 1. post every send (ready = the sender's stream has produced the buffer)
  for (Op& o : ops) {
    if (!o.send) continue;
    Shared& sh = *o.comm->sh;
    cudaEvent_t ready;
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess) return ncclUnhandledCudaError;
    if (cudaEventRecord(ready, o.stream) != cudaSuccess) return ncclUnhandledCudaError;
    std::lock_guard<std::mutex> lk(sh.mu);
    o.seq = sh.send_seq[size_t(o.comm->rank) * sh.n + o.peer]++;
    Shared::Post p;
    p.ptr = o.buf;
    p.bytes = o.bytes;
    p.dev = o.comm->dev;
    p.ready = ready;
    sh.posts[{o.comm->rank, o.peer, o.seq}] = p;
    sh.cv.notify_all();
  }
  // 2. pull every receive on the receiver's stream (copy engines)
  for (Op& o : ops) {
    if (o.send) continue;
    Shared& sh = *o.comm->sh;
    std::unique_lock<std::mutex> lk(sh.mu);
    o.seq = sh.recv_seq[size_t(o.peer) * sh.n + o.comm->rank]++;
    const auto key = std::make_tuple(o.peer, o.comm->rank, o.seq);
    if (!wait_for(lk, sh.cv, [&] { return sh.posts.count(key) != 0; })) {
      o.comm->err = ncclRemoteError;
      return ncclSuccess;  // asynchronous error, as NCCL reports a dead peer
    }
    Shared::Post p = sh.posts[key];
    lk.unlock();
    if (p.bytes != o.bytes) {
      o.comm->err = ncclInvalidUsage;
      return ncclInvalidUsage;
    }
    if (cudaStreamWaitEvent(o.stream, p.ready, 0) != cudaSuccess) return ncclUnhandledCudaError;
    cudaError_t e = p.dev == o.comm->dev
                        ? cudaMemcpyAsync(o.buf, p.ptr, o.bytes, cudaMemcpyDeviceToDevice, o.stream)
                        : cudaMemcpyPeerAsync(o.buf, o.comm->dev, p.ptr, p.dev, o.bytes, o.stream);
    if (e != cudaSuccess) return ncclUnhandledCudaError;
    cudaEvent_t done;
    if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess) return ncclUnhandledCudaError;
    if (cudaEventRecord(done, o.stream) != cudaSuccess) return ncclUnhandledCudaError;
    lk.lock();
    sh.posts[key].done = done;
    sh.posts[key].pulled = true;
    sh.cv.notify_all();
  }
  // 3. the sender's stream may reuse its buffer once its receiver has pulled it
  for (Op& o : ops) {
    if (!o.send) continue;
    Shared& sh = *o.comm->sh;
    std::unique_lock<std::mutex> lk(sh.mu);
    const auto key = std::make_tuple(o.comm->rank, o.peer, o.seq);
    if (!wait_for(lk, sh.cv, [&] { return sh.posts[key].pulled; })) {
      o.comm->err = ncclRemoteError;
      return ncclSuccess;
    }
    Shared::Post p = sh.posts[key];
    sh.posts.erase(key);
    lk.unlock();
    if (cudaStreamWaitEvent(o.stream, p.done, 0) != cudaSuccess) return ncclUnhandledCudaError;
    cudaEventDestroy(p.ready);  // deferred by CUDA until the recorded work completes
    cudaEventDestroy(p.done);
  }
  return ncclSuccess;
}

ncclResult_t enqueue(bool send, const void* buf, size_t count, ncclDataType_t t, int peer,
                     ncclComm* comm, cudaStream_t stream) {
  if (comm == nullptr || comm->aborted) return ncclInvalidArgument;
  if (peer < 0 || peer >= comm->sh->n) return ncclInvalidArgument;
  if (comm->err != ncclSuccess) return ncclSuccess;  // already failed: NCCL keeps returning
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cs);
  if (cs != cudaStreamCaptureStatusNone) return ncclInvalidUsage;  // eager only
  t_ops.push_back(Op{send, comm, peer, const_cast<void*>(buf), count * type_size(t), stream});
  if (t_depth == 0) {
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_ops(ops);
  }
  return ncclSuccess;
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error";
    case ncclUnhandledCudaError: return "unhandled cuda error (shim)";
    case ncclSystemError: return "unhandled system error (shim)";
    case ncclInternalError: return "internal error (shim)";
    case ncclInvalidArgument: return "invalid argument (shim)";
    case ncclInvalidUsage: return "invalid usage (shim)";
    case ncclRemoteError: return "remote process exited or there was a network error (shim: peer timed out)";
    case ncclInProgress: return "NCCL operation in progress";
    default: return "unknown result code (shim)";
  }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::atomic<uint64_t> ctr{0};
  std::random_device rd;
  std::memset(id, 0, sizeof(*id));
  const uint64_t a = (uint64_t(rd()) << 32) ^ rd(), b = ctr.fetch_add(1);
  std::memcpy(id->internal, &a, 8);
  std::memcpy(id->internal + 8, &b, 8);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  const std::string key(id.internal, sizeof(id.internal));
  std::unique_lock<std::mutex> lk(g_init_mu);
  Pending& p = g_pending[key];
  if (!p.sh) p.sh = std::make_shared<Shared>(nranks);
  if (p.sh->n != nranks) return ncclInvalidUsage;
  auto sh = p.sh;
  p.joined++;
  g_init_cv.notify_all();
  if (!wait_for(lk, g_init_cv, [&] { return g_pending[key].joined >= nranks; })) return ncclRemoteError;
  auto* c = new ncclComm;
  c->sh = sh;
  c->rank = rank;
  cudaGetDevice(&c->dev);
  *out = c;
  return ncclSuccess;
}

ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm, ncclConfig_t*) {
  if (comm == nullptr || comm->aborted) return ncclInvalidArgument;
  Shared& sh = *comm->sh;
  std::unique_lock<std::mutex> lk(sh.mu);
  const uint64_t round = sh.split_seq[size_t(comm->rank)]++;
  Shared::Split& sp = sh.splits[round];
  sp.entries.emplace_back(color, key, comm->rank);
  if (++sp.arrived == sh.n) {
    std::map<int, std::vector<std::pair<int, int>>> by_color;  // color -> (key, rank)
    for (auto& [c, k, r] : sp.entries)
      if (c != NCCL_SPLIT_NOCOLOR) by_color[c].push_back({k, r});
    for (auto& [c, v] : by_color) {
      std::sort(v.begin(), v.end());
      sp.comms[c] = std::make_shared<Shared>(static_cast<int>(v.size()));
      for (size_t i = 0; i < v.size(); ++i) sp.new_rank[v[i].second] = static_cast<int>(i);
    }
    sp.ready = true;
    sh.cv.notify_all();
  } else if (!wait_for(lk, sh.cv, [&] { return sh.splits[round].ready; })) {
    comm->err = ncclRemoteError;
    return ncclRemoteError;
  }
  Shared::Split& done = sh.splits[round];
  *newcomm = nullptr;
  if (color != NCCL_SPLIT_NOCOLOR) {
    auto* c = new ncclComm;
    c->sh = done.comms[color];
    c->rank = done.new_rank[comm->rank];
    c->dev = comm->dev;
    *newcomm = c;
  }
  if (++done.left == sh.n) sh.splits.erase(round);
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t comm) {
  if (comm) {
    comm->aborted = true;
    delete comm;
  }
  return ncclSuccess;
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* r) {
  if (comm == nullptr || r == nullptr) return ncclInvalidArgument;
  *r = static_cast<ncclResult_t>(comm->err.load());
  return ncclSuccess;
}

ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  *count = comm->sh->n;
  return ncclSuccess;
}

ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  *rank = comm->rank;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++t_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (t_depth == 0) return ncclInvalidUsage;
  if (--t_depth > 0) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(t_ops);
  return run_ops(ops);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return enqueue(true, buf, count, t, peer, comm, stream);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  return enqueue(false, buf, count, t, peer, comm, stream);
}

}  // extern "C"
