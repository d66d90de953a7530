// Communication backends for the USP protocols.
//
// The reference moves bytes through an in-process fabric of threads
// (reference proj/src/fabric.cpp:147-226): eager send, blocking recv, and an
// all_to_all that is one logical round per group.  On B200 the same collective
// semantics are provided by
//   * NcclComm  -- one process (or thread) per GPU, NCCL grouped send/recv over
//                  NVLink/NVSwitch on Ulysses / ring sub-communicators split from
//                  the world communicator exactly like the mesh (mesh.cpp:44-53);
//   * LocalComm -- ranks living in one process (threads as ranks, like
//                  run_protocol): a host rendezvous exchanges buffer pointers and
//                  CUDA events, and each receiver PULLS its slots with copy-engine
//                  cudaMemcpyPeerAsync on its own stream.  Several ranks may share
//                  one GPU, which is how the multi-rank protocols are exercised on a
//                  single B200.
// All operations are stream-ordered: they enqueue on the given stream and return.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fastusp_internal.h"

namespace fusp {

struct Group {
  std::vector<int> members;  // world ranks, group order
  int pos = -1;              // my position
  std::string key() const;
  int size() const { return static_cast<int>(members.size()); }
};

class Comm {
 public:
  virtual ~Comm() = default;
  // Slot t (t = group position) of `send` goes to member t; slot j of `recv` receives
  // member j's slot for me.  `bytes` per slot, slots `stride` bytes apart.  The self
  // slot is copied locally unless send and recv alias.
  virtual fusp_status all_to_all(const Group& g, const void* send, void* recv, size_t stride,
                                 size_t bytes, cudaStream_t s) = 0;
  // Ring step: send `nparts` buffers to position (pos+1)%R and receive the same number
  // from (pos-1+R)%R (the reference sends K then V, protocols.cpp:253-257).
  virtual fusp_status ring_exchange(const Group& g, const void* const* send, void* const* recv,
                                    const size_t* bytes, int nparts, cudaStream_t s) = 0;
  virtual bool capturable() const = 0;
  // Host all-gather of `bytes` per rank over the whole world (blocking; setup only): rank r's
  // `mine` lands at all + r * bytes on every rank.
  virtual fusp_status allgather_host(const void* mine, size_t bytes, void* all) = 0;
  // Host wait until `s` drained, bounded by timeout_s: a stalled or failed peer becomes
  // FUSP_ERR_DEADLOCK (the reference's DeadlockError, fabric.hpp:112-116) instead of a hang.
  virtual fusp_status wait(cudaStream_t s, double timeout_s, const char* what);
  // SMs a transfer in flight occupies (its kernels must find free SMs while the persistent
  // attention kernel runs beside it): NCCL p2p kernels need some, copy engines none.
  virtual int sms_in_flight() const { return 0; }
};

// ---- in-process fabric -------------------------------------------------------------------
struct LocalFabric {
  explicit LocalFabric(int n) : world(n) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  struct Post {
    std::vector<const void*> sends;
    int device = 0;
    cudaEvent_t ready = nullptr;
    cudaEvent_t done = nullptr;
  };
  struct Slot {
    std::vector<Post> posts;
    int arrived = 0;
    int done_arrived = 0;
    int left = 0;
  };
  std::map<std::pair<std::string, uint64_t>, Slot> slots;
  std::map<std::string, std::vector<uint64_t>> seq;
  double timeout_s = 120.0;
};

class LocalComm : public Comm {
 public:
  LocalComm(LocalFabric* f, int rank, int device);
  ~LocalComm() override;
  fusp_status all_to_all(const Group& g, const void* send, void* recv, size_t stride, size_t bytes,
                         cudaStream_t s) override;
  fusp_status ring_exchange(const Group& g, const void* const* send, void* const* recv,
                            const size_t* bytes, int nparts, cudaStream_t s) override;
  bool capturable() const override { return fabric_->world == 1; }
  fusp_status allgather_host(const void* mine, size_t bytes, void* all) override;

 private:
  // Generic pull-based exchange: for every peer j in `srcs`, copy the chunk at
  // (peer send ptr + src_off[j]) into (recv + dst_off[j]).
  struct Pull {
    int from;        // group position of the sender
    int part;        // which of the sender's posted buffers
    size_t src_off;  // byte offset inside it
    void* dst;
    size_t bytes;
  };
  fusp_status exchange(const Group& g, const char* op, std::vector<const void*> sends,
                       const std::vector<Pull>& pulls, cudaStream_t s);
  LocalFabric* fabric_;
  int rank_, device_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
};

// ---- NCCL --------------------------------------------------------------------------------
class NcclComm : public Comm {
 public:
  NcclComm(ncclComm_t world, int rank, int nranks);
  ~NcclComm() override;
  fusp_status all_to_all(const Group& g, const void* send, void* recv, size_t stride, size_t bytes,
                         cudaStream_t s) override;
  fusp_status ring_exchange(const Group& g, const void* const* send, void* const* recv,
                            const size_t* bytes, int nparts, cudaStream_t s) override;
  bool capturable() const override { return true; }
  fusp_status allgather_host(const void* mine, size_t bytes, void* all) override;
  // FUSP_NCCL_SMS overrides; 8 covers the p2p channels NCCL uses for one send/recv pair.
  int sms_in_flight() const override {
    static const int n = [] {
      const char* e = std::getenv("FUSP_NCCL_SMS");
      return e ? std::atoi(e) : 8;
    }();
    return n;
  }
  // Collective over the world: make sure sub-communicators for every group of the
  // (R,U) mesh exist (ncclCommSplit, color = ring / ulysses index).
  fusp_status ensure_mesh(int r);
  // Collective over the world (fusp_group_create): a sub-communicator for `g` (g.pos < 0 or an
  // empty group: this rank joins the split call without a group).
  fusp_status split_group(const Group& g);
  // Polls ncclCommGetAsyncError on every communicator while the stream drains; on an error or
  // the timeout, ncclCommAbort on all of them (fabric.hpp:106-126 semantics).
  fusp_status wait(cudaStream_t s, double timeout_s, const char* what) override;

 private:
  fusp_status sub(const Group& g, ncclComm_t* out);
  // After an enqueue: a communicator that already reports an asynchronous error (a peer that
  // failed or never arrived) aborts the world -> FUSP_ERR_DEADLOCK naming the operation.
  fusp_status check_async(const char* op, const Group& g);
  fusp_status fail(const std::string& why);
  bool aborted_ = false;
  ncclComm_t world_;
  int rank_, nranks_;
  std::map<std::string, ncclComm_t> subs_;
};

fusp_status nccl_error(ncclResult_t r, const std::string& where);

// ---- peer-memory windows (peer.cu) --------------------------------------------------------
// One device window per rank, mapped by every rank of the world (one node): a 4 KB control
// block of uint32 words -- [kind][src] signals for kinds 0 input reshard, 1 output reshard,
// 2 ring chunk ready, 3 ring buffer free; [kPeerKinds + kind][src] completed waits per source;
// [2 kPeerKinds][0] timeout flag; src = world rank -- and the data region the Ulysses receive
// slots and the ring receive buffers live in.
constexpr int kPeerMaxWorld = 64;
constexpr int kPeerKinds = 4;
constexpr size_t kPeerCtlBytes = 4096;
constexpr uint64_t kPeerMagic = 0x46555350504545ull;  // "FUSPPEE"
struct PeerHandle {  // FUSP_PEER_HANDLE_BYTES on the wire
  uint64_t magic;
  int32_t pid, device;
  uint64_t ptr, bytes;
  cudaIpcMemHandle_t ipc;
  uint8_t pad[128 - 32 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(PeerHandle) == 128, "peer handle is 128 bytes");
struct PeerWindow {
  int device = -1, rank = 0, world = 0;
  char* base = nullptr;       // my window: control block + data
  size_t data_bytes = 0;
  std::vector<char*> peer;    // world rank -> that rank's window in my address space
  std::vector<bool> opened;   // mapped with cudaIpcOpenMemHandle (closed on destruction)
  std::vector<uint64_t> bytes_of;  // data bytes of every rank's window
  std::vector<bool> shares_device; // rank r is a thread of this process on my device
  std::string group;          // the one Ulysses group the peer path serves (usp.cpp)
  std::string ring_group;     // the one ring group the peer ring serves
  ~PeerWindow();
  char* data(int r) const { return peer[r] + kPeerCtlBytes; }
  uint32_t* ctl(int r) const { return reinterpret_cast<uint32_t*>(peer[r]); }
};
fusp_status peer_window_create(PeerWindow* w, int rank, int world, int device, size_t data_bytes,
                               PeerHandle* mine);
fusp_status peer_window_open(PeerWindow* w, const PeerHandle* all);
// kind 0: input reshard, 1: output reshard.  Signals every other member of g, then waits
// until each has signalled me once more than before (timeout -> the flag peer_window_check reads).
fusp_status launch_peer_exchange(const PeerWindow& w, int kind, const Group& g, double timeout_s,
                                 cudaStream_t s);
// Ring step over the windows (kinds 2 / 3): signal `to` (a world rank, -1: none) on `kind_sig`,
// then wait for one more signal from `from` (-1: none) on `kind_wait` than waited for before.
fusp_status launch_peer_signal_wait(const PeerWindow& w, int kind_sig, int to, int kind_wait,
                                    int from, double timeout_s, cudaStream_t s);
fusp_status peer_window_check(const PeerWindow& w, const char* what, cudaStream_t s);

}  // namespace fusp
