// Peer-memory Ulysses transport: every rank exposes one device window to the other ranks of its
// node (CUDA IPC across processes, the raw pointer between threads of one process), and the
// Ulysses all-to-alls become stores of the PRODUCING kernels straight into the members' windows
// over NVLink / NVSwitch:
//   * input reshard (protocols.cpp:125-180): the pack kernel writes slot t -- heads
//     [t*hp, (t+1)*hp) of Q, K, V (FP8 codes + scale trailers included) -- into member t's
//     receive region at my position;
//   * output reshard (protocols.cpp:182-203): the attention epilogue stores O (and the LSE)
//     rows [t*SL, (t+1)*SL) straight into member t's output region, tile by tile, so the
//     transfer overlaps the math and no output all-to-all is left.
// Each reshard then needs one tiny exchange kernel: it signals every member (a system-scope
// release add on the member's word for my world rank) and spins until every member has
// signalled me as often as I have waited for it (per-source counters in my own window, so the
// protocol is graph-replay safe: all state is on the device).
//
// Why single-buffered regions are safe: member A writes B's input region for layer i+1 only
// after A's output exchange of layer i observed B's signal, which B sends after its layer-i
// staging read that region; A writes B's output region for layer i+1 only after A's input
// exchange of layer i+1 observed B's signal, which B sends after copying out layer i.  This
// holds when every peer-path layer of a rank uses the same Ulysses group (usp.cpp enforces it).
#include "comm.h"

#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace fusp {
namespace {

struct ExchArgs {
  uint32_t* remote[kMaxPeerChunks];  // member t's word for me (null for myself)
  int src[kMaxPeerChunks];           // world rank of member t
  uint32_t* sig;                     // my words, indexed by source world rank
  uint32_t* expect;                  // my per-source counters of completed waits
  uint32_t* err;                     // timeout flag (read by PeerWindow::check)
  unsigned long long timeout_ns;
  int n, self;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One warp: lane t < n handles member t.
__global__ void peer_exchange_kernel(const __grid_constant__ ExchArgs a) {
  const int t = threadIdx.x;
  const bool peer = t < a.n && t != a.self;
  if (peer) {
    // everything this stream wrote before (the producing kernel fenced its remote stores
    // system-wide before exiting) happens-before the member's acquire of this add
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.remote[t]) : "memory");
  }
  if (peer) {
    const int src = a.src[t];
    const uint32_t target = a.expect[src] + 1u;
    const unsigned long long t0 = globaltimer();
    while (static_cast<int32_t>(ld_acquire_sys(&a.sig[src]) - target) < 0) {
      __nanosleep(100);
      if (globaltimer() - t0 > a.timeout_ns) {
        atomicOr(a.err, 1u);
        break;
      }
    }
    a.expect[src] = target;
  }
}

// One thread: signal one rank, then wait for one rank (the ring's point-to-point steps).
struct SigWaitArgs {
  uint32_t* remote;  // to's word for me (null: no signal)
  uint32_t* sig;     // my word for `from` (null: no wait)
  uint32_t* expect;  // my completed waits on `from`
  uint32_t* err;
  unsigned long long timeout_ns;
};
__global__ void peer_signal_wait_kernel(const __grid_constant__ SigWaitArgs a) {
  if (a.remote != nullptr) {
    __threadfence_system();  // the stream's copies / stores into to's window before the signal
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(a.remote) : "memory");
  }
  if (a.sig != nullptr) {
    const uint32_t target = *a.expect + 1u;
    const unsigned long long t0 = globaltimer();
    while (static_cast<int32_t>(ld_acquire_sys(a.sig) - target) < 0) {
      __nanosleep(100);
      if (globaltimer() - t0 > a.timeout_ns) {
        atomicOr(a.err, 1u);
        break;
      }
    }
    *a.expect = target;
  }
}

}  // namespace

fusp_status launch_peer_signal_wait(const PeerWindow& w, int kind_sig, int to, int kind_wait,
                                    int from, double timeout_s, cudaStream_t s) {
  SigWaitArgs a{};
  if (to >= 0) a.remote = w.ctl(to) + kind_sig * kPeerMaxWorld + w.rank;
  if (from >= 0) {
    a.sig = w.ctl(w.rank) + kind_wait * kPeerMaxWorld + from;
    a.expect = w.ctl(w.rank) + (kPeerKinds + kind_wait) * kPeerMaxWorld + from;
  }
  a.err = w.ctl(w.rank) + 2 * kPeerKinds * kPeerMaxWorld;
  a.timeout_ns = static_cast<unsigned long long>((timeout_s > 0 ? timeout_s : 120.0) * 1e9);
  peer_signal_wait_kernel<<<1, 1, 0, s>>>(a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "peer_signal_wait_kernel");
  return FUSP_OK;
}

PeerWindow::~PeerWindow() {
  if (device >= 0) cudaSetDevice(device);
  for (size_t r = 0; r < peer.size(); ++r)
    if (opened.size() > r && opened[r]) cudaIpcCloseMemHandle(peer[r]);
  if (base) cudaFree(base);
}

fusp_status peer_window_create(PeerWindow* w, int rank, int world, int device, size_t data_bytes,
                               PeerHandle* mine) {
  if (world > kPeerMaxWorld)
    return set_error(FUSP_ERR_UNSUPPORTED, "peer window: world above " + std::to_string(kPeerMaxWorld));
  FUSP_CUDA(cudaSetDevice(device));
  w->device = device;
  w->rank = rank;
  w->world = world;
  w->data_bytes = (data_bytes + 255) / 256 * 256;
  FUSP_CUDA(cudaMalloc(&w->base, kPeerCtlBytes + w->data_bytes));
  // The zeroed control words must be in memory before the handle leaves this rank: a member's
  // first signal (from its own non-blocking stream, unordered with this memset's stream) could
  // otherwise land before the memset and be wiped -- a lost signal, i.e. a deadlock.
  FUSP_CUDA(cudaMemset(w->base, 0, kPeerCtlBytes));
  FUSP_CUDA(cudaDeviceSynchronize());
  std::memset(mine, 0, sizeof(*mine));
  mine->magic = kPeerMagic;
  mine->pid = static_cast<int32_t>(getpid());
  mine->device = device;
  mine->ptr = reinterpret_cast<uint64_t>(w->base);
  mine->bytes = w->data_bytes;
  FUSP_CUDA(cudaIpcGetMemHandle(&mine->ipc, w->base));
  return FUSP_OK;
}

fusp_status peer_window_open(PeerWindow* w, const PeerHandle* all) {
  FUSP_CUDA(cudaSetDevice(w->device));
  w->peer.assign(static_cast<size_t>(w->world), nullptr);
  w->opened.assign(static_cast<size_t>(w->world), false);
  w->bytes_of.assign(static_cast<size_t>(w->world), 0);
  w->shares_device.assign(static_cast<size_t>(w->world), false);
  const int32_t pid = static_cast<int32_t>(getpid());
  // Ranks of this process sharing my device (threads as ranks): every one of them enqueues on
  // its own stream and side stream, and a spinning exchange kernel blocks whatever the
  // hardware queues behind it.  CUDA maps streams onto CUDA_DEVICE_MAX_CONNECTIONS hardware
  // queues (default 8); two ranks' streams in one queue make a rank's progress wait behind
  // another rank's spin on it -- a deadlock.  Refuse rather than hang.
  int sharing = 0;
  for (int r = 0; r < w->world; ++r) sharing += all[r].pid == pid && all[r].device == w->device;
  if (sharing > 1) {
    const char* e = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    const int conns = e != nullptr ? atoi(e) : 8;
    if (conns < 2 * sharing)
      return set_error(FUSP_ERR_UNSUPPORTED,
                       "peer window: " + std::to_string(sharing) + " ranks of this process share device " +
                           std::to_string(w->device) + "; their spinning exchange kernels need a hardware "
                           "queue per stream: set CUDA_DEVICE_MAX_CONNECTIONS >= " +
                           std::to_string(2 * sharing) + " (at most 32) before CUDA initialises");
  }
  for (int r = 0; r < w->world; ++r) {
    const PeerHandle& h = all[r];
    if (h.magic != kPeerMagic)
      return set_error(FUSP_ERR_COMM, "peer window: bad handle from rank " + std::to_string(r));
    w->bytes_of[r] = h.bytes;
    w->shares_device[r] = h.pid == pid && h.device == w->device;
    if (r == w->rank) {
      w->peer[r] = w->base;
      continue;
    }
    if (h.pid == pid) {  // ranks that are threads of this process: the pointer itself
      w->peer[r] = reinterpret_cast<char*>(h.ptr);
      if (h.device != w->device) {
        int can = 0;
        FUSP_CUDA(cudaDeviceCanAccessPeer(&can, w->device, h.device));
        if (!can)
          return set_error(FUSP_ERR_COMM, "peer window: device " + std::to_string(w->device) +
                                              " cannot access device " + std::to_string(h.device));
        cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return set_cuda_error(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
    } else {
      void* p = nullptr;
      FUSP_CUDA(cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess));
      w->peer[r] = static_cast<char*>(p);
      w->opened[r] = true;
    }
  }
  return FUSP_OK;
}

fusp_status launch_peer_exchange(const PeerWindow& w, int kind, const Group& g, double timeout_s,
                                 cudaStream_t s) {
  if (g.size() > kMaxPeerChunks) return set_error(FUSP_ERR_UNSUPPORTED, "peer exchange: group too large");
  ExchArgs a{};
  a.n = g.size();
  a.self = g.pos;
  for (int t = 0; t < a.n; ++t) {
    const int m = g.members[t];
    a.src[t] = m;
    a.remote[t] = t == g.pos ? nullptr : w.ctl(m) + kind * kPeerMaxWorld + w.rank;
  }
  a.sig = w.ctl(w.rank) + kind * kPeerMaxWorld;
  a.expect = w.ctl(w.rank) + (kPeerKinds + kind) * kPeerMaxWorld;
  a.err = w.ctl(w.rank) + 2 * kPeerKinds * kPeerMaxWorld;
  a.timeout_ns = static_cast<unsigned long long>((timeout_s > 0 ? timeout_s : 120.0) * 1e9);
  peer_exchange_kernel<<<1, 32, 0, s>>>(a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "peer_exchange_kernel");
  return FUSP_OK;
}

fusp_status peer_window_check(const PeerWindow& w, const char* what, cudaStream_t s) {
  uint32_t err = 0;  // (stream-ordered: a legacy-stream copy could wait on other ranks' spins)
  FUSP_CUDA(cudaMemcpyAsync(&err, w.ctl(w.rank) + 2 * kPeerKinds * kPeerMaxWorld, 4, cudaMemcpyDeviceToHost, s));
  FUSP_CUDA(cudaStreamSynchronize(s));
  if (err && getenv("FUSP_PEER_DEBUG") != nullptr) {  // post-mortem: who signalled whom
    std::vector<uint32_t> ctl((2 * kPeerKinds + 1) * kPeerMaxWorld);
    cudaMemcpy(ctl.data(), w.ctl(w.rank), ctl.size() * 4, cudaMemcpyDeviceToHost);
    std::string out;  // one write per rank: ranks may be threads printing at once
    for (int kind = 0; kind < kPeerKinds; ++kind) {
      out += "[peer] rank " + std::to_string(w.rank) + " kind " + std::to_string(kind) + " sig/expect:";
      for (int r = 0; r < w.world; ++r)
        out += " " + std::to_string(ctl[kind * kPeerMaxWorld + r]) + "/" +
               std::to_string(ctl[(kPeerKinds + kind) * kPeerMaxWorld + r]);
      out += "\n";
    }
    fputs(out.c_str(), stderr);
  }
  if (err)
    return set_error(FUSP_ERR_DEADLOCK, std::string("deadlock: rank ") + std::to_string(w.rank) +
                                            " stalled in " + what + " (peer-memory exchange timed out)");
  return FUSP_OK;
}

// Every kernel of this file, for preload_kernels() (lazy module loading, see runtime.cpp).
void append_kernels_peer(std::vector<const void*>& v) {
  v.push_back(reinterpret_cast<const void*>(peer_exchange_kernel));
  v.push_back(reinterpret_cast<const void*>(peer_signal_wait_kernel));
}

}  // namespace fusp
