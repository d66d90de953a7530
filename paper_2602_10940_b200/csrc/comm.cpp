// LocalComm (threads-as-ranks fabric with copy-engine pulls) and NcclComm.
#include "comm.h"

#include <algorithm>
#include <cstring>
#include <chrono>
#include <sstream>
#include <thread>

namespace fusp {

std::string Group::key() const {
  std::string k;
  for (size_t i = 0; i < members.size(); ++i) {
    if (i) k += ',';
    k += std::to_string(members[i]);
  }
  return k;
}

fusp_status nccl_error(ncclResult_t r, const std::string& where) {
  return set_error(FUSP_ERR_NCCL, where + ": " + ncclGetErrorString(r));
}

#define FUSP_NCCL(expr)                                   \
  do {                                                    \
    ncclResult_t _r = (expr);                             \
    if (_r != ncclSuccess) return nccl_error(_r, #expr);  \
  } while (0)

fusp_status Comm::wait(cudaStream_t s, double, const char*) {
  FUSP_CUDA(cudaStreamSynchronize(s));  // in-process fabric: its rendezvous carries the timeout
  return FUSP_OK;
}

// ---- LocalComm ----------------------------------------------------------------------------
LocalComm::LocalComm(LocalFabric* f, int rank, int device) : fabric_(f), rank_(rank), device_(device) {
  cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&done_, cudaEventDisableTiming);
}

LocalComm::~LocalComm() {
  if (ready_) cudaEventDestroy(ready_);
  if (done_) cudaEventDestroy(done_);
}

fusp_status LocalComm::exchange(const Group& g, const char* op, std::vector<const void*> sends,
                                const std::vector<Pull>& pulls, cudaStream_t s) {
  const int n = g.size();
  const std::string key = std::string(op) + ":" + g.key();
  // Sender side: my buffers are final once everything before this point on `s` ran.
  FUSP_CUDA(cudaEventRecord(ready_, s));
  std::unique_lock<std::mutex> lk(fabric_->mu);
  auto& seqv = fabric_->seq[key];
  if (seqv.empty()) seqv.assign(static_cast<size_t>(fabric_->world), 0);
  const uint64_t seq = seqv[rank_]++;
  auto& slot = fabric_->slots[{key, seq}];
  if (slot.posts.empty()) slot.posts.resize(static_cast<size_t>(n));
  slot.posts[g.pos].sends = std::move(sends);
  slot.posts[g.pos].device = device_;
  slot.posts[g.pos].ready = ready_;
  slot.posts[g.pos].done = done_;
  slot.arrived++;
  fabric_->cv.notify_all();
  auto deadline = std::chrono::steady_clock::now() +
                  std::chrono::milliseconds(static_cast<int64_t>(fabric_->timeout_s * 1000));
  auto stalled = [&](const char* what, int have) {
    std::ostringstream os;
    os << "deadlock: rank " << rank_ << " stalled in " << op << "(group=" << g.key()
       << ", round=" << seq << ", " << have << "/" << n << " " << what << ")";
    return set_error(FUSP_ERR_DEADLOCK, os.str());
  };
  if (!fabric_->cv.wait_until(lk, deadline, [&] { return slot.arrived == n; }))
    return stalled("arrived", slot.arrived);
  std::vector<LocalFabric::Post> posts = slot.posts;
  lk.unlock();
  // Receiver side: pull each chunk after its sender's ready event (copy engines).
  std::vector<bool> waited(n, false);
  for (const Pull& p : pulls) {
    const auto& post = posts[p.from];
    if (p.from != g.pos && !waited[p.from]) {
      FUSP_CUDA(cudaStreamWaitEvent(s, post.ready, 0));
      waited[p.from] = true;
    }
    const void* src = static_cast<const char*>(post.sends[p.part]) + p.src_off;
    if (src == p.dst || p.bytes == 0) continue;
    if (post.device == device_) {
      FUSP_CUDA(cudaMemcpyAsync(p.dst, src, p.bytes, cudaMemcpyDeviceToDevice, s));
    } else {
      FUSP_CUDA(cudaMemcpyPeerAsync(p.dst, device_, src, post.device, p.bytes, s));
    }
  }
  FUSP_CUDA(cudaEventRecord(done_, s));
  lk.lock();
  slot.done_arrived++;
  fabric_->cv.notify_all();
  if (!fabric_->cv.wait_until(lk, deadline, [&] { return slot.done_arrived == n; }))
    return stalled("pulled", slot.done_arrived);
  posts = slot.posts;
  if (++slot.left == n) fabric_->slots.erase({key, seq});
  lk.unlock();
  // Peers finished reading my buffers at their done events: later writes wait for them.
  for (int j = 0; j < n; ++j)
    if (j != g.pos) FUSP_CUDA(cudaStreamWaitEvent(s, posts[j].done, 0));
  return FUSP_OK;
}

fusp_status LocalComm::allgather_host(const void* mine, size_t bytes, void* all) {
  const int n = fabric_->world;
  std::unique_lock<std::mutex> lk(fabric_->mu);
  const std::string key = "allgather_host";
  auto& seqv = fabric_->seq[key];
  if (seqv.empty()) seqv.assign(static_cast<size_t>(n), 0);
  const uint64_t seq = seqv[rank_]++;
  auto& slot = fabric_->slots[{key, seq}];
  if (slot.posts.empty()) slot.posts.resize(static_cast<size_t>(n));
  slot.posts[rank_].sends = {mine};
  slot.arrived++;
  fabric_->cv.notify_all();
  const auto deadline = std::chrono::steady_clock::now() +
                        std::chrono::milliseconds(static_cast<int64_t>(fabric_->timeout_s * 1000));
  if (!fabric_->cv.wait_until(lk, deadline, [&] { return slot.arrived == n; }))
    return set_error(FUSP_ERR_DEADLOCK, "deadlock: rank " + std::to_string(rank_) +
                                            " stalled in allgather (" + std::to_string(slot.arrived) +
                                            "/" + std::to_string(n) + " arrived)");
  for (int j = 0; j < n; ++j)  // host memory of the posting threads, still alive: they wait below
    std::memcpy(static_cast<char*>(all) + size_t(j) * bytes, slot.posts[j].sends[0], bytes);
  slot.done_arrived++;
  fabric_->cv.notify_all();
  if (!fabric_->cv.wait_until(lk, deadline, [&] { return slot.done_arrived == n; }))
    return set_error(FUSP_ERR_DEADLOCK, "deadlock: rank " + std::to_string(rank_) + " stalled in allgather");
  if (++slot.left == n) fabric_->slots.erase({key, seq});
  return FUSP_OK;
}

fusp_status LocalComm::all_to_all(const Group& g, const void* send, void* recv, size_t stride,
                                  size_t bytes, cudaStream_t s) {
  const int n = g.size();
  if (n == 1) {  // self slot only: no rendezvous (keeps world-1 contexts graph-capturable)
    if (send != recv && bytes) FUSP_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    return FUSP_OK;
  }
  std::vector<Pull> pulls;
  for (int j = 0; j < n; ++j)  // member j's slot addressed to me lands in my slot j
    pulls.push_back({j, 0, static_cast<size_t>(g.pos) * stride,
                     static_cast<char*>(recv) + static_cast<size_t>(j) * stride, bytes});
  return exchange(g, "all_to_all", {send}, pulls, s);
}

fusp_status LocalComm::ring_exchange(const Group& g, const void* const* send, void* const* recv,
                                     const size_t* bytes, int nparts, cudaStream_t s) {
  const int n = g.size();
  if (n == 1) {
    for (int i = 0; i < nparts; ++i)
      if (send[i] != recv[i] && bytes[i])
        FUSP_CUDA(cudaMemcpyAsync(recv[i], send[i], bytes[i], cudaMemcpyDeviceToDevice, s));
    return FUSP_OK;
  }
  const int prev = (g.pos - 1 + n) % n;
  std::vector<Pull> pulls;
  for (int i = 0; i < nparts; ++i) pulls.push_back({prev, i, 0, recv[i], bytes[i]});
  return exchange(g, "send", std::vector<const void*>(send, send + nparts), pulls, s);
}

// ---- NcclComm -------------------------------------------------------------------------------
NcclComm::NcclComm(ncclComm_t world, int rank, int nranks)
    : world_(world), rank_(rank), nranks_(nranks) {}

NcclComm::~NcclComm() {
  if (aborted_) return;  // ncclCommAbort already released them
  for (auto& kv : subs_) ncclCommDestroy(kv.second);
  if (world_) ncclCommDestroy(world_);
}

fusp_status NcclComm::fail(const std::string& why) {
  if (!aborted_) {
    for (auto& kv : subs_) ncclCommAbort(kv.second);
    if (world_) ncclCommAbort(world_);
    subs_.clear();
    world_ = nullptr;
    aborted_ = true;
  }
  return set_error(FUSP_ERR_DEADLOCK, "deadlock: rank " + std::to_string(rank_) + " " + why);
}

fusp_status NcclComm::check_async(const char* op, const Group& g) {
  std::vector<ncclComm_t> all{world_};
  for (auto& kv : subs_) all.push_back(kv.second);
  for (ncclComm_t c : all) {
    ncclResult_t r = ncclSuccess;
    if (c == nullptr || ncclCommGetAsyncError(c, &r) != ncclSuccess) continue;
    if (r != ncclSuccess && r != ncclInProgress)
      return fail(std::string("stalled in ") + op + "(group=" + g.key() + "): NCCL " +
                  ncclGetErrorString(r) + "; communicators aborted");
  }
  return FUSP_OK;
}

fusp_status NcclComm::wait(cudaStream_t s, double timeout_s, const char* what) {
  if (aborted_) return set_error(FUSP_ERR_COMM, "NCCL communicators were aborted after a failure");
  const auto t0 = std::chrono::steady_clock::now();
  Group world;
  for (int i = 0; i < nranks_; ++i) world.members.push_back(i);
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return FUSP_OK;
    if (q != cudaErrorNotReady) return set_cuda_error(q, "cudaStreamQuery");
    FUSP_CHECK(check_async(what, world));
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > timeout_s) {
      std::ostringstream os;
      os << "timed out after " << timeout_s << " s waiting in " << what
         << " (a peer never joined its collective); communicators aborted";
      return fail(os.str());
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

fusp_status NcclComm::ensure_mesh(int r) {
  const int u = nranks_ / r;
  const int ring_idx = rank_ / u, uly_idx = rank_ % u;
  // Ulysses groups: contiguous rank blocks (mesh.cpp:44-47); ring groups stride by U (:48-53).
  Group ug, rg;
  for (int j = 0; j < u; ++j) ug.members.push_back(ring_idx * u + j);
  for (int i = 0; i < r; ++i) rg.members.push_back(i * u + uly_idx);
  ug.pos = uly_idx;
  rg.pos = ring_idx;
  if (!subs_.count(ug.key())) {
    ncclComm_t c;
    FUSP_NCCL(ncclCommSplit(world_, ring_idx, uly_idx, &c, nullptr));
    subs_[ug.key()] = c;
  }
  if (!subs_.count(rg.key())) {
    ncclComm_t c;
    FUSP_NCCL(ncclCommSplit(world_, uly_idx, ring_idx, &c, nullptr));
    subs_[rg.key()] = c;
  }
  return FUSP_OK;
}

fusp_status NcclComm::split_group(const Group& g) {
  // Collective over the world: members pass color = their group's smallest member (disjoint
  // groups of one call get distinct colors) and key = position; others opt out.
  const bool in = g.size() > 0 && g.pos >= 0;
  int color = NCCL_SPLIT_NOCOLOR;
  if (in) color = *std::min_element(g.members.begin(), g.members.end());
  ncclComm_t c = nullptr;
  FUSP_NCCL(ncclCommSplit(world_, color, in ? g.pos : 0, &c, nullptr));
  if (!in) return FUSP_OK;
  auto it = subs_.find(g.key());
  if (it != subs_.end()) ncclCommDestroy(it->second);
  subs_[g.key()] = c;
  return FUSP_OK;
}

fusp_status NcclComm::sub(const Group& g, ncclComm_t* out) {
  bool identity = g.size() == nranks_;
  for (int i = 0; i < g.size() && identity; ++i) identity = g.members[i] == i;
  if (identity) {  // the world communicator's ranks are the group positions
    *out = world_;
    return FUSP_OK;
  }
  auto it = subs_.find(g.key());
  if (it == subs_.end())
    return set_error(FUSP_ERR_COMM, "no NCCL sub-communicator for group " + g.key());
  *out = it->second;
  return FUSP_OK;
}

fusp_status NcclComm::all_to_all(const Group& g, const void* send, void* recv, size_t stride,
                                 size_t bytes, cudaStream_t s) {
  const int n = g.size();
  const char* sp = static_cast<const char*>(send);
  char* rp = static_cast<char*>(recv);
  if (sp + g.pos * stride != rp + g.pos * stride && bytes)
    FUSP_CUDA(cudaMemcpyAsync(rp + g.pos * stride, sp + g.pos * stride, bytes,
                              cudaMemcpyDeviceToDevice, s));
  if (n == 1 || bytes == 0) return FUSP_OK;
  if (aborted_) return set_error(FUSP_ERR_COMM, "NCCL communicators were aborted after a failure");
  ncclComm_t c;
  FUSP_CHECK(sub(g, &c));
  FUSP_NCCL(ncclGroupStart());
  for (int j = 0; j < n; ++j) {
    if (j == g.pos) continue;
    FUSP_NCCL(ncclSend(sp + j * stride, bytes, ncclUint8, j, c, s));
    FUSP_NCCL(ncclRecv(rp + j * stride, bytes, ncclUint8, j, c, s));
  }
  FUSP_NCCL(ncclGroupEnd());
  return check_async("all_to_all", g);
}

// Grouped point-to-point to and from every rank (what ncclAllGather does; send/recv keeps the
// set of NCCL calls fastusp makes small).  Setup only: synchronous.
fusp_status NcclComm::allgather_host(const void* mine, size_t bytes, void* all) {
  if (aborted_) return set_error(FUSP_ERR_COMM, "NCCL communicators were aborted after a failure");
  // Stream-ordered buffer and copies: no device-wide wait (ranks sharing a GPU may already have
  // peer-exchange kernels spinning on it for work this rank enqueues next).
  char* dev = nullptr;
  cudaStream_t s = nullptr;
  FUSP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  FUSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dev), bytes * size_t(nranks_), s));
  fusp_status st = FUSP_OK;
  auto run = [&]() -> fusp_status {
    FUSP_CUDA(cudaMemcpyAsync(dev + size_t(rank_) * bytes, mine, bytes, cudaMemcpyHostToDevice, s));
    if (nranks_ > 1) {
      FUSP_NCCL(ncclGroupStart());
      for (int j = 0; j < nranks_; ++j) {
        if (j == rank_) continue;
        FUSP_NCCL(ncclSend(dev + size_t(rank_) * bytes, bytes, ncclUint8, j, world_, s));
        FUSP_NCCL(ncclRecv(dev + size_t(j) * bytes, bytes, ncclUint8, j, world_, s));
      }
      FUSP_NCCL(ncclGroupEnd());
      Group w;
      for (int j = 0; j < nranks_; ++j) w.members.push_back(j);
      w.pos = rank_;
      FUSP_CHECK(check_async("allgather", w));
      FUSP_CHECK(wait(s, 120.0, "allgather"));
    }
    FUSP_CUDA(cudaMemcpyAsync(all, dev, bytes * size_t(nranks_), cudaMemcpyDeviceToHost, s));
    FUSP_CUDA(cudaStreamSynchronize(s));
    return FUSP_OK;
  };
  st = run();
  cudaFreeAsync(dev, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return st;
}

fusp_status NcclComm::ring_exchange(const Group& g, const void* const* send, void* const* recv,
                                    const size_t* bytes, int nparts, cudaStream_t s) {
  const int n = g.size();
  if (n == 1) {
    for (int i = 0; i < nparts; ++i)
      if (send[i] != recv[i] && bytes[i])
        FUSP_CUDA(cudaMemcpyAsync(recv[i], send[i], bytes[i], cudaMemcpyDeviceToDevice, s));
    return FUSP_OK;
  }
  if (aborted_) return set_error(FUSP_ERR_COMM, "NCCL communicators were aborted after a failure");
  ncclComm_t c;
  FUSP_CHECK(sub(g, &c));
  FUSP_NCCL(ncclGroupStart());
  for (int i = 0; i < nparts; ++i) {
    FUSP_NCCL(ncclSend(send[i], bytes[i], ncclUint8, (g.pos + 1) % n, c, s));
    FUSP_NCCL(ncclRecv(recv[i], bytes[i], ncclUint8, (g.pos - 1 + n) % n, c, s));
  }
  FUSP_NCCL(ncclGroupEnd());
  return check_async("send", g);
}

}  // namespace fusp
