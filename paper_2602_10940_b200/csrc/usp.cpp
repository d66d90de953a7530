// The USP protocols on B200: per-rank context, Ulysses all-to-all reshards, the
// (serial or double-buffered) ring with the LSE merge fused into the attention
// epilogue, FP8 K/V communication, and CUDA-Graph capture of the layer.
//
// Reference mapping (proj/src/protocols.cpp):
//   usp_attention            :321-340  -> run_layer(kUsp)
//   ulysses_attention        :207-214  -> run_layer(kUlysses)  (R = 1)
//   ring_attention_serial    :237-268  -> ring()  with pipelined = false
//   ring_attention_pipelined :270-319  -> ring()  with pipelined = true (side stream)
//   ulysses_input_reshard    :125-180  -> ulysses_in()   pack -> all_to_all -> unpack
//   ulysses_output_reshard   :182-203  -> ulysses_out()  epilogue writes send slots -> all_to_all
#include <cmath>
#include <cstring>
#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <tuple>
#include <sstream>
#include <string>
#include <vector>

#include "comm.h"
#include "fastusp_internal.h"

using namespace fusp;

struct fusp_fabric_s {
  explicit fusp_fabric_s(int n) : fabric(n) {}
  LocalFabric fabric;
};

// Device workspace of a layer: the arena (wire slots, operands, ring buffers, accumulators)
// and zero-initialised words (attention stream-K tickets, staging amax / tickets) that every
// kernel leaves zeroed.  A context owns one for eager calls; every captured graph owns its
// own, so eager calls may regrow the context's without touching memory a graph replays.
struct Workspace {
  void* arena = nullptr;
  size_t bytes = 0;
  fusp::CounterBuf words;
  void release() {
    if (arena) cudaFree(arena);
    if (words.ptr) cudaFree(words.ptr);
    arena = nullptr;
    bytes = 0;
    words = fusp::CounterBuf{};
  }
};

// Device staging of the host-buffer path: two slots of Q, K, V and output chunks, and the
// copy streams / events of its H2D || layer || D2H pipeline.  Owned by the context.
struct HostStage {
  void* d = nullptr;
  size_t bytes = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaStream_t h2d_x[2] = {nullptr, nullptr};  // extra H2D streams (FUSP_HOST_H2D_STREAMS)
  cudaEvent_t in_ready[2] = {nullptr, nullptr}, computed[2] = {nullptr, nullptr},
              out_done[2] = {nullptr, nullptr};
  cudaEvent_t in_ready_x[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  uint32_t* flag = nullptr;
  ~HostStage() {
    if (d) cudaFree(d);
    if (flag) cudaFree(flag);
    for (cudaStream_t x : {h2d, d2h, h2d_x[0], h2d_x[1]})
      if (x) cudaStreamDestroy(x);
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {in_ready[i], computed[i], out_done[i], in_ready_x[0][i], in_ready_x[1][i]})
        if (e) cudaEventDestroy(e);
  }
};

struct fusp_ctx_s {
  int rank = 0, world = 1, device = 0;
  std::unique_ptr<Comm> comm;
  NcclComm* nccl = nullptr;
  // peer-memory Ulysses transport (fusp_ctx_peer_enable): null = the comm backend moves bytes
  std::unique_ptr<PeerWindow> peer;
  bool peer_open = false;
  cudaStream_t last_stream = nullptr;  // stream of the previous layer call (workspace users)
  bool last_stream_valid = false;
  uint64_t peer_layers = 0;     // layers whose Ulysses reshards went through the windows
  uint64_t peer_fallbacks = 0;  // layers that could not (see peer_eligible) and used `comm`
  cudaStream_t side = nullptr;  // ring communication stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_recv[2] = {nullptr, nullptr}, ev_attn[2] = {nullptr, nullptr};
  static constexpr int kMaxSteps = 32;
  cudaEvent_t tc0[kMaxSteps], tc1[kMaxSteps], tm0[kMaxSteps], tm1[kMaxSteps];
  int timed_steps = 0;
  bool capturing = false;
  Workspace own;             // eager calls
  Workspace* ws = &own;      // the workspace in use (a graph's while it is being captured)
  int live_graphs = 0;       // graphs captured on this context and not yet destroyed
  void* block_ws = nullptr;  // Q, K, V and attention output of fusp_usp_block
  size_t block_ws_bytes = 0;
  std::unique_ptr<HostStage> host;  // fusp_usp_attention_host's staging (created on first use)
  // fusp_ctx_debug_wire: device copies of every payload this rank put on the wire (eager calls)
  struct WireRec {
    int kind, round;  // 0 Ulysses-in send slots, 1 / 2 ring K / V part (round = hop)
    void* dev;
    size_t bytes;
  };
  bool debug_wire = false;
  std::vector<WireRec> wire;
  void clear_wire() {
    for (auto& r : wire) cudaFree(r.dev);
    wire.clear();
  }
  uint64_t a2a_bytes = 0, send_bytes = 0;
  // TrafficLog mirror (fabric.hpp:32-60): one entry per sender-side op, self traffic excluded
  struct Traffic {
    std::string op, group;
    int round, rank;
    uint64_t bytes, msgs;
  };
  std::vector<Traffic> traffic;
  std::map<std::string, int> a2a_seq;  // per-group collective call index (fabric.cpp:211-213)
  // schedule of the last ring call, for the Timeline mirror (fabric.hpp:62-93)
  int tl_steps = 0;
  bool tl_pipelined = false;
  bool tl_valid = false;
  int tl_next = -1;
};

struct fusp_group_s {  // = uspsim::ProcessGroup (fabric.hpp:20-28) seen from one rank
  fusp::Group g;
  fusp_ctx_s* ctx = nullptr;
};

struct fusp_graph_s {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int device = 0;
  fusp_ctx_s* ctx = nullptr;  // its communicators are replayed: the context must outlive it
  Workspace ws;               // the arena and words the captured kernels address
  void* block_ws = nullptr;   // fusp_graph_capture_block: Q, K, V and attention output
};

namespace {

enum class Mode { kUsp, kUlysses, kRing };

const char* tag(Mode m) { return m == Mode::kUsp ? "usp" : m == Mode::kUlysses ? "ulysses" : "ring"; }

std::string sstr(const fusp_shape4& s) {
  std::ostringstream os;
  os << "[" << s.b << "," << s.h << "," << s.s << "," << s.d << "]";
  return os.str();
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bound of every host wait on collectives (FUSP_TIMEOUT_S, default 120 s like the in-process
// fabric's rendezvous): past it a stalled peer is reported as DeadlockError.
double sync_timeout_s() {
  static const double t = [] {
    const char* e = std::getenv("FUSP_TIMEOUT_S");
    const double v = e ? std::atof(e) : 120.0;
    return v > 0 ? v : 120.0;
  }();
  return t;
}

// TrafficLog entries as the reference's fabric records them (fabric.cpp:155-158, :343-351):
// all_to_all: one per collective and member, bytes sent to the other members; send: one per
// message, group "from->to", round = ring round.
void log_a2a(fusp_ctx_s* c, const Group& g, uint64_t bytes) {
  const std::string key = g.key();
  const int round = c->a2a_seq[key]++;
  c->traffic.push_back({"all_to_all", key, round, c->rank, bytes, uint64_t(g.size() - 1)});
}
// Debug capture of a wire payload (fusp_ctx_debug_wire): a device copy, stream-ordered.
fusp_status record_wire(fusp_ctx_s* c, int kind, int round, const void* p, size_t bytes,
                        cudaStream_t s) {
  if (!c->debug_wire || c->capturing) return FUSP_OK;
  void* d = nullptr;
  FUSP_CUDA(cudaMalloc(&d, bytes ? bytes : 1));
  FUSP_CUDA(cudaMemcpyAsync(d, p, bytes, cudaMemcpyDeviceToDevice, s));
  c->wire.push_back({kind, round, d, bytes});
  return FUSP_OK;
}

void log_send(fusp_ctx_s* c, const Group& g, int round, uint64_t bytes) {
  const int next = g.members[(g.pos + 1) % g.size()];
  c->traffic.push_back(
      {"send", std::to_string(c->rank) + "->" + std::to_string(next), round, c->rank, bytes, 1});
}

// Bump allocator over the context arena; the first (dry) pass only measures.
struct Carve {
  char* base = nullptr;
  size_t off = 0;
  void* take(size_t bytes) {
    off = align_up(off, 256);
    void* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
};

// Workspace growth is stream-ordered on the layer's stream `s` and never waits on the whole
// device: with peer windows, ranks sharing one GPU (tests) have exchange kernels spinning on it
// for work that another rank's thread has not enqueued yet, and a cudaDeviceSynchronize /
// cudaFree here would wait for them forever.  The old buffers' last users ran on the stream of
// the previous call (host-synchronized here when it differs) or on the side stream, which every
// layer joins back into its stream before returning.
fusp_status quiesce_previous(fusp_ctx_s* c, cudaStream_t s) {
  if (c->last_stream != s && c->last_stream_valid) FUSP_CUDA(cudaStreamSynchronize(c->last_stream));
  return FUSP_OK;
}

fusp_status ensure_arena(fusp_ctx_s* c, size_t bytes, cudaStream_t s) {
  Workspace& w = *c->ws;
  if (w.bytes >= bytes) return FUSP_OK;
  if (c->capturing)
    return set_error(FUSP_ERR_UNSUPPORTED, "workspace growth during graph capture");
  if (w.arena) {
    FUSP_CHECK(quiesce_previous(c, s));
    FUSP_CUDA(cudaFreeAsync(w.arena, s));
  }
  w.arena = nullptr;
  w.bytes = 0;
  FUSP_CUDA(cudaMallocAsync(&w.arena, bytes, s));
  w.bytes = bytes;
  return FUSP_OK;
}

fusp_status ensure_words(fusp_ctx_s* c, size_t words, cudaStream_t s) {
  if (c->ws->words.ptr != nullptr && c->ws->words.words >= words) return FUSP_OK;
  if (c->capturing)
    return set_error(FUSP_ERR_UNSUPPORTED, "workspace growth during graph capture");
  if (c->ws->words.ptr != nullptr) FUSP_CHECK(quiesce_previous(c, s));
  return ensure_counters(c->ws->words, words, s);
}

// Bump allocator over the zero-initialised words.
struct CarveWords {
  uint32_t* base = nullptr;
  size_t off = 0;
  uint32_t* take(size_t n) {
    uint32_t* p = base ? base + off : nullptr;
    off += (n + 31) / 32 * 32;
    return p;
  }
};

struct Layer {
  Mode mode;
  int B, H, SL, D, U, R, hp, heads_r, span;
  int64_t blk, C;  // elements per (Q|K|V) slot piece, elements per ring chunk (= U*blk)
  bool fp8, pipelined;
  int in_dt, out_dt;
  // MMA dtype of Q and K: bf16 for bf16 inputs (exact), f16 otherwise -- f32 inputs keep 11
  // significant bits instead of bf16's 8, and the FP8 path's decode(code)*scale values too.
  // Every staging into f16 from a wider-range source is range-guarded (fastusp_internal.h).
  int qk_dt;
  // operand dtypes of K and V as the attention kernel reads them: qk_dt and f16 on the tcgen05
  // path (D = 128); for other D (attention_generic.cu, f32 CUDA cores) the caller's dtype, or
  // f32 for dequantized FP8 chunks -- and no range guard (nothing is staged into f16)
  int k_op = FUSP_BF16, v_op = FUSP_F16;
  bool generic = false;
  size_t w_in;  // bytes per element of the caller's dtype = of the wire (non-FP8 Q/K/V, FP8 Q)
  size_t wout;
  Group ug, rg;
  // Ulysses wire slot: [Q blk][K blk][V blk] in the caller's dtype (the reference's f32 wire
  // for f32 inputs), or, FP8, [Q blk][K codes][V codes][k scales][v scales]; byte offsets
  size_t off_k = 0, off_v = 0, off_tr = 0;
  size_t slot_bytes, slot_stride;
  // FP8 scale counts: per-tensor (reference) = 1; per block = one per (b,h) slab
  bool fp8_block = false;
  int nsc_local = 1;  // scales of the caller's local K (or V): B*H per block
  int nsc_slot = 1;   // scales riding in one Ulysses slot: B*hp per block
  int nsc_chunk = 1;  // scales of a ring chunk: heads_r per block
  // fused QK prologue (fusp_qk_prologue): Q goes through norm/rope on its way into the slot
  // (or the attention operand); K likewise, except on the FP8 path, which normalizes K once
  // into an f32 scratch copy (k_dt = F32) that the quantizers then read
  const fusp_qk_prologue* pro = nullptr;
  bool pro_q = false, pro_k = false, pro_k_pre = false;
  int64_t pos0 = 0;
  int k_dt = 0;  // dtype of the K source the FP8 quantizers read
  // Q, K, V were written into the layer's own buffers by a producer (fusp_usp_block's QKV
  // projection): the Ulysses pack (U > 1) or the operand conversion (U = 1) is skipped
  bool prepacked = false;
  // consumer reads the output where it landed: with peer windows and B = 1 the output region
  // of my window IS the output (concatenation over heads), so *out_view = it and no copy runs
  const void** out_view = nullptr;
  // detail::ulysses_input_reshard (fusp_ulysses_input_reshard): the wire path runs even for a
  // one-member group and the unpack writes the caller's buffers in `reshard_dt`, unstaged
  bool force_wire = false;
  void *reshard_q = nullptr, *reshard_k = nullptr, *reshard_v = nullptr;
  int reshard_dt = FUSP_F32;
  bool wire() const { return mode != Mode::kRing && (U > 1 || force_wire); }
  // Peer-memory Ulysses (PeerWindow, peer.cu): the pack writes the members' receive regions and
  // the attention epilogue their output regions directly; offsets inside every window's data
  bool peer = false;
  char* pw[kMaxPeerChunks] = {};  // data region of member t's window (group order)
  size_t pw_out = 0, pw_lse = 0;  // output / LSE regions (the receive slots start at 0)
  size_t pw_need = 0;             // data bytes the layer needs in every member's window
  // Peer-memory ring (R > 1): the K / V chunk of every hop is copied into the next member's
  // window (ring buffers at pw_ring, [buffer][part] of pw_ring_part bytes), no backend call
  bool peer_ring = false;
  size_t pw_ring = 0, pw_ring_part = 0;
  int ring_next = -1, ring_prev = -1;  // world ranks
  char* ring_next_win = nullptr;       // the next member's data region
  char* ring_win_self = nullptr;       // my data region
};

// Window layout of a layer: Ulysses receive slots, output and LSE regions (U > 1), then the
// ring's two receive buffers of K and V parts (R > 1).  Shared by plan_peer and
// fusp_peer_window_bytes.
void peer_layout(Layer& l) {
  size_t off = 0;
  if (l.U > 1) {
    const size_t in = l.slot_stride * l.U;
    l.pw_out = align_up(in, 256);
    l.pw_lse = l.pw_out + align_up(size_t(l.blk) * l.wout * l.U, 256);
    off = l.pw_lse + align_up(size_t(l.blk / l.D) * 4 * l.U, 256);
  }
  l.pw_ring = off;
  l.pw_ring_part = l.R > 1 ? align_up(l.fp8 ? size_t(l.C) + 4 * size_t(l.nsc_chunk) : size_t(l.C) * l.w_in, 256) : 0;
  l.pw_need = off + 4 * l.pw_ring_part;
}

struct Buffers {
  // Ulysses in
  char *send_in = nullptr, *recv_in = nullptr;
  // attention operands of the local chunk, and their buffers when staged
  const void *Qr = nullptr, *Kr = nullptr, *Vr = nullptr;
  void *Qr_w = nullptr, *Kr_w = nullptr, *Vr_w = nullptr;
  // range-guard exponents of the local operands (null: not staged from a wider range)
  const int *q_exp = nullptr, *k_exp = nullptr, *v_exp = nullptr;
  int* exps = nullptr;  // [7][heads_r]: q, k, v, then K / V of ring buffer 0 and 1
  // sources of the U = 1 staging: Q / K as they come (caller, prologue or producer output)
  const void *Qs = nullptr, *Ks_src = nullptr, *Vs_src = nullptr;
  int qs_dt = 0, ks_dt = 0;
  void *Qtmp = nullptr, *Ktmp = nullptr, *Vtmp = nullptr;  // f32 prologue / producer outputs
  // the local K / V chunk in the wire dtype (first ring hop, non-FP8)
  const void *Kw = nullptr, *Vw = nullptr;
  // fp8 exact local chunk: codes [heads_r][span][D] + per-segment scales
  uint8_t *Kc = nullptr, *Vc = nullptr;
  const float *Ks = nullptr, *Vs = nullptr;
  int64_t s_stride = 1;     // floats between the scale arrays of consecutive sequence segments
  int64_t bh_stride = 0;    // floats between the scales of consecutive (b,h) slabs
  int seg_rows = 0;
  float* qscale = nullptr;  // K scales then V scales of a locally quantized chunk
  uint32_t* amax = nullptr;   // zero words: per-block amax of the FP8 passes (+ tickets)
  float* pscale = nullptr;    // FP8 Ulysses pack: K scales then V scales (amax pass output)
  // ring
  char* rb[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [buf][K|V] wire parts
  char* sw[2] = {nullptr, nullptr};                           // fp8 send wire parts
  void* Kd[2] = {nullptr, nullptr};                           // staged ring operands per buffer
  void* Vd[2] = {nullptr, nullptr};
  float *acc_o = nullptr, *acc_lse = nullptr;
  // Ulysses out (LSE rides a second all-to-all when the caller asks for it)
  char *send_out = nullptr, *recv_out = nullptr;
  float *lse_send = nullptr, *lse_recv = nullptr;
  // FP8 path with a K prologue: normalized + rotated K in f32
  float* Kpro = nullptr;
  // stream-K partials of the attention kernel
  void* attn_ws = nullptr;
  size_t attn_ws_bytes = 0;
  uint32_t* attn_cnt = nullptr;
  size_t attn_cnt_words = 0;
  // zero-initialised staging words: local operands (3), ring buffer x K/V
  uint32_t* stage_w[3] = {nullptr, nullptr, nullptr};
  uint32_t* ring_w[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
};

fusp_status plan_layer(fusp_ctx_s* c, Mode mode, int r, const fusp_shape4& ls, int in_dt,
                       const fusp_comm_options& o, Layer* L, const Group* grp = nullptr) {
  if (mode != Mode::kUsp) r = mode == Mode::kRing ? c->world : 1;
  if (grp != nullptr) {  // ulysses / ring over a caller's ProcessGroup (protocols.hpp:47-65)
    if (grp->pos < 0)
      return set_error(FUSP_ERR_COMM, "rank " + std::to_string(c->rank) + " not in group " + grp->key());
    r = mode == Mode::kRing ? grp->size() : 1;
  } else if (r < 1 || c->world % r != 0)
    return set_error(FUSP_ERR_MESH, "ring dimension " + std::to_string(r) +
                                        " does not divide worker count " + std::to_string(c->world));
  if (ls.b < 1 || ls.h < 1 || ls.s < 1 || ls.d < 1)
    return set_error(FUSP_ERR_SHAPE, std::string(tag(mode)) + ": bad local shape " + sstr(ls));
  if (in_dt != FUSP_F32 && in_dt != FUSP_BF16 && in_dt != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "input dtype must be f32, bf16 or f16");
  if (o.out_dtype != FUSP_F32 && o.out_dtype != FUSP_BF16 && o.out_dtype != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "out_dtype must be f32, bf16 or f16");
  Layer& l = *L;
  l.mode = mode;
  l.B = static_cast<int>(ls.b);
  l.H = static_cast<int>(ls.h);
  l.SL = static_cast<int>(ls.s);
  l.D = static_cast<int>(ls.d);
  l.R = r;
  l.U = mode == Mode::kRing ? 1 : (grp != nullptr ? grp->size() : c->world / r);
  if (l.H % l.U != 0)
    return set_error(FUSP_ERR_SHAPE, std::string(tag(mode)) + ": head count H=" +
                                         std::to_string(l.H) + " not divisible by ulysses dimension U=" +
                                         std::to_string(l.U));
  if (l.D != 128 && (l.D % 8 != 0 || l.D > 256))
    return set_error(FUSP_ERR_SHAPE, std::string(tag(mode)) + ": head dim D=" + std::to_string(l.D) +
                                         " unsupported (D = 128 on tcgen05; other D a multiple of 8 up to 256)");
  l.generic = l.D != 128;
  l.hp = l.H / l.U;
  l.heads_r = l.B * l.hp;
  l.span = l.U * l.SL;
  l.blk = int64_t(l.B) * l.hp * l.SL * l.D;
  l.C = l.blk * l.U;
  l.fp8 = o.fp8_kv != 0;
  l.pipelined = o.pipelined_ring != 0;
  l.in_dt = in_dt;
  l.k_dt = in_dt;
  l.qk_dt = (in_dt == FUSP_BF16 && !l.fp8) ? FUSP_BF16 : FUSP_F16;
  l.k_op = l.qk_dt;
  l.v_op = FUSP_F16;
  if (l.generic) {
    l.qk_dt = in_dt;
    l.k_op = l.v_op = l.fp8 ? FUSP_F32 : in_dt;
  }
  l.w_in = dtype_size(in_dt);
  l.out_dt = o.out_dtype;
  l.wout = dtype_size(o.out_dtype);
  if (grp != nullptr) {  // the caller's group on one axis, this rank alone on the other
    Group self;
    self.members = {c->rank};
    self.pos = 0;
    l.ug = mode == Mode::kRing ? self : *grp;
    l.rg = mode == Mode::kRing ? *grp : self;
  } else {
    // mesh groups (mesh.cpp:44-53): rank = ring_idx * U + uly_idx
    const int ri = c->rank / l.U, ui = c->rank % l.U;
    for (int j = 0; j < l.U; ++j) l.ug.members.push_back(ri * l.U + j);
    for (int i = 0; i < l.R; ++i) l.rg.members.push_back(i * l.U + ui);
    l.ug.pos = ui;
    l.rg.pos = ri;
  }
  l.fp8_block = l.fp8 && o.fp8_block != 0;
  if (l.fp8_block) {
    l.nsc_local = l.B * l.H;
    l.nsc_slot = l.B * l.hp;
    l.nsc_chunk = l.heads_r;
  }
  l.off_k = size_t(l.blk) * l.w_in;
  l.off_v = l.off_k + size_t(l.blk) * (l.fp8 ? 1 : l.w_in);
  l.off_tr = l.off_v + size_t(l.blk) * (l.fp8 ? 1 : l.w_in);
  l.slot_bytes = l.fp8 ? l.off_tr + 8 * size_t(l.nsc_slot) : l.off_tr;
  l.slot_stride = align_up(l.slot_bytes, 256);
  return FUSP_OK;
}

// Whether this layer's Ulysses reshards go through the peer windows (the fused pack / epilogue
// stores) or through c->comm.  The windows serve ONE Ulysses group per context (the hazard
// argument in peer.cu needs every peer-path exchange of a rank to involve the same members):
// the first eligible layer's group.  A producer (fusp_usp_block's QKV projection) stores into
// the members' windows itself: GEMM epilogue and all-to-all in one kernel, and so do the fused
// QK RMSNorm + RoPE packs.  Not on the peer path: other head dims, wire debugging, layers
// larger than any member's window.
bool plan_peer_ulysses(fusp_ctx_s* c, Layer& l) {
  l.peer = false;
  if (!l.wire() || l.force_wire || l.U < 2 || l.U > kMaxPeerChunks) return false;
  const std::string key = l.ug.key();
  if (!c->peer->group.empty() && c->peer->group != key) return false;
  if (l.slot_stride % 16 != 0 || (size_t(l.blk) * l.wout) % 16 != 0) return false;
  for (int t = 0; t < l.U; ++t)
    if (c->peer->bytes_of[size_t(l.ug.members[t])] < l.pw_need) return false;
  for (int t = 0; t < l.U; ++t) l.pw[t] = c->peer->data(l.ug.members[t]);
  c->peer->group = key;
  l.peer = true;
  return true;
}

// The ring's K / V hops through the windows: like the Ulysses path, ONE ring group per context
// (every ring signal of a rank then involves the same two neighbours, whose counters pair up).
// Ring members that are threads of this process on my device (the single-GPU test setup) keep
// the backend ring unless FUSP_PEER_RING=1: their streams share the device's hardware queues,
// and a queue holding one rank's spinning wait ahead of another rank's work can close a cycle
// through the ring that one-process-per-GPU ranks (separate queues, the deployment shape) and
// ranks in separate processes (time-sliced contexts; tested over CUDA IPC) cannot.
bool plan_peer_ring(fusp_ctx_s* c, Layer& l) {
  l.peer_ring = false;
  if (l.R < 2 || l.rg.size() < 2) return false;
  bool shared = true;
  for (int m : l.rg.members) shared = shared && c->peer->shares_device[size_t(m)];
  const char* force = getenv("FUSP_PEER_RING");
  if (shared && !(force != nullptr && atoi(force) == 1)) return false;
  const std::string key = l.rg.key();
  if (!c->peer->ring_group.empty() && c->peer->ring_group != key) return false;
  for (int m : l.rg.members)
    if (c->peer->bytes_of[size_t(m)] < l.pw_need) return false;
  const int R = l.rg.size();
  l.ring_next = l.rg.members[(l.rg.pos + 1) % R];
  l.ring_prev = l.rg.members[(l.rg.pos - 1 + R) % R];
  l.ring_next_win = c->peer->data(l.ring_next);
  l.ring_win_self = c->peer->data(c->rank);
  c->peer->ring_group = key;
  l.peer_ring = true;
  return true;
}

bool plan_peer(fusp_ctx_s* c, Layer& l) {
  l.peer = l.peer_ring = false;
  if (!c->peer || !c->peer_open || l.generic || c->debug_wire) return false;
  peer_layout(l);
  const bool u = plan_peer_ulysses(c, l);
  const bool r = plan_peer_ring(c, l);
  return u || r;
}

// Assign workspace for a layer. `q`, `k`, `v` are the caller's tensors (zero-copy when the
// attention can read them as they are).
void carve(const Layer& l, Carve& cv, CarveWords& cw, Buffers* b, const void* q, const void* k,
           const void* v, void* out) {
  const size_t CQ = size_t(l.C) * dtype_size(l.qk_dt);  // operand chunks in their dtypes
  const size_t CK = size_t(l.C) * dtype_size(l.k_op);
  const size_t CV = size_t(l.C) * dtype_size(l.v_op);
  const size_t C4 = size_t(l.C) * 4;
  const bool uly = l.mode != Mode::kRing;
  const int hr = l.heads_r;
  const bool wire = l.wire();
  b->exps = static_cast<int*>(cv.take(sizeof(int) * 7 * size_t(hr)));
  for (int i = 0; i < 3; ++i) b->stage_w[i] = cw.take(stage_words(hr));
  for (int i = 0; i < 2; ++i)
    for (int p = 0; p < 2; ++p) b->ring_w[i][p] = cw.take(stage_words(hr));
  if (wire) {
    if (l.peer) {  // receive slots in my window; the pack writes the members' windows
      b->recv_in = l.pw[l.ug.pos];
    } else {
      b->send_in = static_cast<char*>(cv.take(l.slot_stride * l.U));
      b->recv_in = static_cast<char*>(cv.take(l.slot_stride * l.U));
    }
    b->Qr = b->Qr_w = cv.take(CQ);
    b->Kr = b->Kr_w = cv.take(CK);
    b->Vr = b->Vr_w = cv.take(CV);
    if (l.fp8) {
      b->Kc = static_cast<uint8_t*>(cv.take(l.C));
      b->Vc = static_cast<uint8_t*>(cv.take(l.C));
    } else if (l.R > 1) {  // the ring forwards the chunk in the wire dtype
      b->Kw = l.in_dt == l.k_op ? b->Kr : cv.take(size_t(l.C) * l.w_in);
      b->Vw = l.in_dt == l.v_op ? b->Vr : cv.take(size_t(l.C) * l.w_in);
    }
  } else {
    // U == 1: no transfer; the operands are the caller's tensors when already in the MMA dtype.
    const bool fq = uly && l.fp8;  // Ulysses self slot still takes the FP8 round trip (D7)
    // Q source: the caller's q, or the prologue's output -- straight into the operand in the
    // MMA dtype when that is the caller's dtype, else an f32 copy that is staged
    if (l.pro_q || l.prepacked) {
      if (l.in_dt == l.qk_dt) {
        b->Qr = b->Qr_w = cv.take(CQ);
        b->Qs = b->Qr;
        b->qs_dt = l.qk_dt;
      } else {
        b->Qs = b->Qtmp = cv.take(C4);
        b->qs_dt = FUSP_F32;
      }
    } else {
      b->Qs = q;
      b->qs_dt = l.in_dt;
    }
    if (b->Qr == nullptr) {
      if (b->qs_dt == l.qk_dt) b->Qr = b->Qs;
      else b->Qr = b->Qr_w = cv.take(CQ);
    }
    // K source likewise (the FP8 path with a K prologue reads the f32 Kpro copy instead)
    if (l.pro_k || l.prepacked) {
      if (l.in_dt == l.k_op) {
        b->Kr = b->Kr_w = cv.take(CK);
        b->Ks_src = b->Kr;
        b->ks_dt = l.k_op;
      } else {
        b->Ks_src = b->Ktmp = cv.take(C4);
        b->ks_dt = FUSP_F32;
      }
    } else {
      b->Ks_src = k;  // (or Kpro, set by run_layer)
      b->ks_dt = l.k_dt;
    }
    if (b->Kr == nullptr) {
      if (b->ks_dt == l.k_op && !fq) b->Kr = b->Ks_src;
      else b->Kr = b->Kr_w = cv.take(CK);
    }
    if (l.prepacked && l.in_dt != l.v_op) {
      b->Vs_src = b->Vtmp = cv.take(size_t(l.C) * l.w_in);
    } else if (l.prepacked) {
      b->Vs_src = b->Vr = b->Vr_w = cv.take(CV);
    } else {
      b->Vs_src = v;
    }
    if (b->Vr == nullptr) {
      if (l.in_dt == l.v_op && !fq) b->Vr = b->Vs_src;
      else b->Vr = b->Vr_w = cv.take(CV);
    }
    b->Kw = b->Ks_src;
    b->Vw = b->Vs_src;
    if (fq) {
      b->Kc = static_cast<uint8_t*>(cv.take(l.C));
      b->Vc = static_cast<uint8_t*>(cv.take(l.C));
    }
  }
  if (l.pro_k_pre) b->Kpro = static_cast<float*>(cv.take(C4));
  const int nsc = l.nsc_local > l.nsc_chunk ? l.nsc_local : l.nsc_chunk;
  b->qscale = static_cast<float*>(cv.take(sizeof(float) * 2 * nsc));
  // amax words of the FP8 passes: zero-initialised, and the amax pass's last CTA leaves them
  // zero (launch_amax_scales), so no memset precedes a quantization
  b->amax = cw.take(4 * (size_t(nsc) + 1));
  b->pscale = static_cast<float*>(cv.take(sizeof(float) * 2 * (size_t(nsc) + 1)));
  if (l.R > 1) {
    const size_t part = l.fp8 ? align_up(size_t(l.C) + 4 * size_t(l.nsc_chunk), 256)
                              : size_t(l.C) * l.w_in;
    for (int i = 0; i < 2; ++i)
      for (int p = 0; p < 2; ++p)  // peer ring: my receive buffers are in my window
        b->rb[i][p] = l.peer_ring ? l.ring_win_self + l.pw_ring + (2 * i + p) * l.pw_ring_part
                                  : static_cast<char*>(cv.take(part));
    if (l.fp8)
      for (int p = 0; p < 2; ++p) b->sw[p] = static_cast<char*>(cv.take(part));
    for (int i = 0; i < 2; ++i) {
      if (l.fp8 || l.in_dt != l.k_op) b->Kd[i] = cv.take(CK);
      if (l.fp8 || l.in_dt != l.v_op) b->Vd[i] = cv.take(CV);
    }
    b->acc_o = static_cast<float*>(cv.take(C4));
    b->acc_lse = static_cast<float*>(cv.take(size_t(l.heads_r) * l.span * 4));
  }
  b->attn_ws_bytes = attention_workspace_bytes(l.heads_r, l.span, l.span);
  if (b->attn_ws_bytes) b->attn_ws = cv.take(b->attn_ws_bytes);
  if (wire && l.peer) {  // the epilogue stores into the members' windows; mine receives
    b->recv_out = l.pw[l.ug.pos] + l.pw_out;
    b->lse_recv = reinterpret_cast<float*>(l.pw[l.ug.pos] + l.pw_lse);
  } else if (wire) {
    b->send_out = static_cast<char*>(cv.take(size_t(l.blk) * l.wout * l.U));
    b->recv_out = l.B == 1 ? static_cast<char*>(out)
                           : static_cast<char*>(cv.take(size_t(l.blk) * l.wout * l.U));
    const size_t lb = size_t(l.blk / l.D) * 4 * l.U;  // [U][B][hp][SL] f32
    b->lse_send = static_cast<float*>(cv.take(lb));
    b->lse_recv = static_cast<float*>(cv.take(lb));
  }
}

// A staging op into the operand dtype `ddt`, range-guarded when that is f16 and the source has
// a wider range (fastusp_internal.h).
StageOp staged_op(const void* src, int sdt, void* dst, int ddt, int* exps, uint32_t* words) {
  StageOp o{};
  o.src = src;
  o.sdt = sdt;
  o.dst = dst;
  o.ddt = ddt;
  if (ddt == FUSP_F16 && sdt != FUSP_F16) {
    o.exps = exps;
    o.words = words;
  }
  return o;
}

// ---------------------------------------------------------------- Ulysses input reshard
fusp_status ulysses_in(fusp_ctx_s* c, const Layer& l, Buffers& b, const void* q, const void* k,
                       const void* v, cudaStream_t s) {
  const bool uly = l.mode != Mode::kRing;
  const int hr = l.heads_r;
  // norm/rope of Q (or K) written as `ddt` into slots of `stride` elements, u = 1: plain copy
  auto prologue = [&](bool is_q, const void* src, void* dst, int ddt, int64_t stride,
                      int u) -> fusp_status {
    const fusp_qk_prologue& p = *l.pro;
    return launch_norm_rope_pack(src, l.in_dt, dst, ddt, stride, l.B, l.H, l.SL, l.D, u,
                                 is_q ? p.q_norm_weight : p.k_norm_weight, p.eps, p.rope_cos,
                                 p.rope_sin, l.pos0, s);
  };
  if (!l.wire()) {
    // (the producer path wrote Qs / Ks_src / Vs_src itself)
    if (l.pro_q && !l.prepacked)
      FUSP_CHECK(prologue(true, q, const_cast<void*>(b.Qs), b.qs_dt, 0, 1));
    if (l.pro_k && !l.prepacked)
      FUSP_CHECK(prologue(false, k, const_cast<void*>(b.Ks_src), b.ks_dt, 0, 1));
    StageOp ops[3];
    int n = 0;
    if (b.Qr_w != nullptr && b.Qr != b.Qs) {
      ops[n++] = staged_op(b.Qs, b.qs_dt, b.Qr_w, l.qk_dt, b.exps, b.stage_w[0]);
      b.q_exp = ops[n - 1].exps;
    }
    if (uly && l.fp8) {
      // quantize the whole local K and V (protocols.cpp:139-142; or per (b,h) slab), and the
      // self slot takes the dequantized values (:163-179)
      const int64_t block = l.fp8_block ? int64_t(l.span) * l.D : l.C;
      const Fp8Src srcs[2] = {Fp8Src{b.Ks_src, b.ks_dt, nullptr, 0, 0, l.D, l.span, l.span},
                              Fp8Src{b.Vs_src, l.in_dt, nullptr, 0, 0, l.D, l.span, l.span}};
      uint32_t* works[2] = {b.amax, b.amax + (l.nsc_local + 1)};
      float* scs[2] = {b.qscale, b.qscale + l.nsc_local};
      uint8_t* cds[2] = {b.Kc, b.Vc};
      FUSP_CHECK(launch_quantize_fp8_multi(srcs, 2, l.C, block, works, scs, cds, nullptr, s));
      for (int p = 0; p < 2; ++p) {
        StageOp o = staged_op(cds[p], FUSP_E4M3, p == 0 ? b.Kr_w : b.Vr_w, p == 0 ? l.k_op : l.v_op,
                              b.exps + (1 + p) * hr, b.stage_w[1 + p]);
        o.scales = scs[p];
        o.scale_bh_stride = l.fp8_block ? 1 : 0;
        ops[n++] = o;
        (p == 0 ? b.k_exp : b.v_exp) = o.exps;
      }
      b.Ks = b.qscale;
      b.Vs = b.qscale + l.nsc_local;
      b.s_stride = 0;
      b.bh_stride = l.fp8_block ? 1 : 0;
      b.seg_rows = l.span;
    } else {
      if (b.Kr_w != nullptr && b.Kr != b.Ks_src) {
        ops[n++] = staged_op(b.Ks_src, b.ks_dt, b.Kr_w, l.k_op, b.exps + hr, b.stage_w[1]);
        b.k_exp = ops[n - 1].exps;
      }
      if (b.Vr_w != nullptr && b.Vr != b.Vs_src) {
        ops[n++] = staged_op(b.Vs_src, l.in_dt, b.Vr_w, l.v_op, b.exps + 2 * hr, b.stage_w[2]);
        b.v_exp = ops[n - 1].exps;
      }
    }
    return launch_stage(ops, n, hr, l.span, l.D, 1, s);
  }
  const int64_t sew = int64_t(l.slot_stride / l.w_in);  // slot stride in wire elements
  // Peer-memory pack: slot t is my slot in member t's receive region (its window), so the pack
  // kernel's stores ARE the all-to-all; slot 0's address plus per-slot byte offsets
  char* sbase = b.send_in;
  int64_t boff[kMaxPeerChunks] = {};
  if (l.peer) {
    sbase = l.pw[0] + size_t(l.ug.pos) * l.slot_stride;
    for (int t = 0; t < l.U; ++t) boff[t] = l.pw[t] - l.pw[0];
  }
  const int64_t* pboff = l.peer ? boff : nullptr;
  if (!l.prepacked) {
    // pack: destination slot t <- heads [t*hp, (t+1)*hp) (protocols.cpp:143-153); Q, K, V
    // keep the caller's dtype on the wire (the receiver stages them for the tensor cores)
    PackDesc p{};
    p.b = l.B;
    p.h = l.H;
    p.sl = l.SL;
    p.d = l.D;
    p.u = l.U;
    p.src = q;
    p.src_dtype = l.in_dt;
    p.dst = sbase;
    p.dst_dtype = l.in_dt;
    p.dst_slot_stride = sew;
    PackDesc ops[3];
    int nops = 0;
    if (!l.fp8 && (l.pro_q || l.pro_k)) {
      // one norm/RoPE/pack launch whose V operand is a plain pack
      const fusp_qk_prologue& pr = *l.pro;
      // (peer path: the fused prologue stores into the members' windows like the plain pack)
      const ProPack pops[3] = {
          {q, sbase, l.pro_q ? pr.q_norm_weight : nullptr, l.pro_q ? pr.rope_cos : nullptr,
           l.pro_q ? pr.rope_sin : nullptr, l.in_dt, l.in_dt},
          {k, sbase + l.off_k, l.pro_k ? pr.k_norm_weight : nullptr,
           l.pro_k ? pr.rope_cos : nullptr, l.pro_k ? pr.rope_sin : nullptr, l.in_dt, l.in_dt},
          {v, sbase + l.off_v, nullptr, nullptr, nullptr, l.in_dt, l.in_dt}};
      FUSP_CHECK(launch_norm_rope_pack_multi(pops, 3, sew, l.B, l.H, l.SL, l.D, l.U, pr.eps, l.pos0, s, pboff));
    } else if (!l.fp8) {
      ops[nops++] = p;
      p.src = k;
      p.dst = sbase + l.off_k;
      ops[nops++] = p;
      p.src = v;
      p.dst = sbase + l.off_v;
      ops[nops++] = p;
      FUSP_CHECK(launch_pack_multi(ops, nops, s, false, pboff));
    } else {
      if (l.pro_q) {
        const fusp_qk_prologue& pr = *l.pro;
        FUSP_CHECK(launch_norm_rope_pack(q, l.in_dt, sbase, l.in_dt, sew, l.B, l.H, l.SL, l.D, l.U,
                                         pr.q_norm_weight, pr.eps, pr.rope_cos, pr.rope_sin, l.pos0, s, pboff));
      }
      else ops[nops++] = p;
      // per-tensor scale over ALL local heads (fp8.cpp:107-123) -- or one per (b,h) slab --:
      // one amax launch for K and V, then Q, K, V leave in one pack launch whose E4M3
      // operands compute their scales from the amax words and write every slot's trailer
      const int64_t n = int64_t(l.B) * l.H * l.SL * l.D;
      const int64_t block = l.fp8_block ? int64_t(l.SL) * l.D : n;
      const Fp8Src srcs[2] = {Fp8Src{k, l.k_dt, nullptr, 0, 0, l.D, l.SL, l.SL},
                              Fp8Src{v, l.in_dt, nullptr, 0, 0, l.D, l.SL, l.SL}};
      uint32_t* am[2] = {b.amax, b.amax + l.nsc_local + 1};
      float* sc[2] = {b.pscale, b.pscale + l.nsc_local};
      for (int part = 0; part < 2; ++part) {
        p.src = srcs[part].x;
        p.src_dtype = srcs[part].dt;
        p.dst = sbase + (part == 0 ? l.off_k : l.off_v);
        p.dst_dtype = FUSP_E4M3;
        p.dst_slot_stride = int64_t(l.slot_stride);
        p.scale = sc[part];
        p.amax_bits = nullptr;
        p.scale_bh_stride = l.fp8_block ? 1 : 0;
        p.trailer = reinterpret_cast<float*>(sbase + l.off_tr) + part * l.nsc_slot;
        p.trailer_stride = int64_t(l.slot_stride / 4);
        ops[nops++] = p;
      }
      bool fused = false;  // small per-tensor case: amax + pack in one cooperative launch
      if (nops == 3 && !l.fp8_block)
        FUSP_CHECK(try_pack_fp8_fused(ops, am, sc, pboff, s, &fused));
      if (!fused) {
        FUSP_CHECK(launch_amax_scales(srcs, 2, block, l.nsc_local, am, sc, nullptr, s));
        // programmatic dependent of the amax pass: the Q copy overlaps it, the E4M3 operands
        // wait for its scales
        FUSP_CHECK(launch_pack_multi(ops, nops, s, /*pdl=*/true, pboff));
      }
    }
  }
  if (l.peer) {
    // the members' pack kernels wrote my receive slots: signal mine, wait for theirs
    FUSP_CHECK(launch_peer_exchange(*c->peer, 0, l.ug, sync_timeout_s(), s));
  } else {
    FUSP_CHECK(record_wire(c, 0, 0, b.send_in, l.slot_stride * l.U, s));
    FUSP_CHECK(c->comm->all_to_all(l.ug, b.send_in, b.recv_in, l.slot_stride, l.slot_bytes, s));
  }
  c->a2a_bytes += uint64_t(l.U - 1) * l.slot_bytes;
  log_a2a(c, l.ug, uint64_t(l.U - 1) * l.slot_bytes);
  // unpack + stage: source j contributed our heads over its sequence shard
  // (protocols.cpp:163-179); every operand leaves the receive slots in one launch
  StageOp ops[3];
  if (l.reshard_q != nullptr) {
    // detail::ulysses_input_reshard: the resharded Q, K, V themselves (FP8 K / V dequantized
    // exactly, decode(code) * scale in f32 as fp8.cpp:125-130), in the caller's dtype
    const float* scales = reinterpret_cast<const float*>(b.recv_in + l.off_tr);
    void* dst[3] = {l.reshard_q, l.reshard_k, l.reshard_v};
    for (int p = 0; p < 3; ++p) {
      StageOp o{};
      const bool codes = l.fp8 && p > 0;
      o.src = b.recv_in + (p == 0 ? 0 : p == 1 ? l.off_k : l.off_v);
      o.sdt = codes ? FUSP_E4M3 : l.in_dt;
      o.src_slot_stride = codes ? int64_t(l.slot_stride) : sew;
      if (codes) {
        o.scales = scales + (p - 1) * l.nsc_slot;
        o.scale_stride = int64_t(l.slot_stride / 4);
        o.scale_bh_stride = l.fp8_block ? 1 : 0;
      }
      o.dst = dst[p];
      o.ddt = l.reshard_dt;
      ops[p] = o;
    }
    return launch_stage(ops, 3, hr, l.SL, l.D, l.U, s);
  }
  StageOp oq = staged_op(b.recv_in, l.in_dt, b.Qr_w, l.qk_dt, b.exps, b.stage_w[0]);
  oq.src_slot_stride = sew;
  b.q_exp = oq.exps;
  ops[0] = oq;
  if (!l.fp8) {
    for (int p = 0; p < 2; ++p) {
      StageOp o = staged_op(b.recv_in + (p == 0 ? l.off_k : l.off_v), l.in_dt,
                            p == 0 ? b.Kr_w : b.Vr_w, p == 0 ? l.k_op : l.v_op,
                            b.exps + (1 + p) * hr, b.stage_w[1 + p]);
      o.src_slot_stride = sew;
      if (o.ddt != l.in_dt) {  // staged (range-guarded into f16): the ring forwards the wire copy
        o.raw = l.R > 1 ? const_cast<void*>(p == 0 ? b.Kw : b.Vw) : nullptr;
        (p == 0 ? b.k_exp : b.v_exp) = o.exps;
      }
      ops[1 + p] = o;
    }
    return launch_stage(ops, 3, hr, l.SL, l.D, l.U, s);
  }
  const float* scales = reinterpret_cast<const float*>(b.recv_in + l.off_tr);
  for (int p = 0; p < 2; ++p) {
    StageOp o = staged_op(b.recv_in + (p == 0 ? l.off_k : l.off_v), FUSP_E4M3,
                          p == 0 ? b.Kr_w : b.Vr_w, p == 0 ? l.k_op : l.v_op,
                          b.exps + (1 + p) * hr, b.stage_w[1 + p]);
    o.src_slot_stride = int64_t(l.slot_stride);
    o.scales = scales + p * l.nsc_slot;
    o.scale_stride = int64_t(l.slot_stride / 4);
    o.scale_bh_stride = l.fp8_block ? 1 : 0;
    o.raw = p == 0 ? static_cast<void*>(b.Kc) : static_cast<void*>(b.Vc);  // exact codes
    ops[1 + p] = o;
    (p == 0 ? b.k_exp : b.v_exp) = o.exps;
  }
  FUSP_CHECK(launch_stage(ops, 3, hr, l.SL, l.D, l.U, s));
  b.Ks = scales;
  b.Vs = scales + l.nsc_slot;
  b.s_stride = int64_t(l.slot_stride / 4);
  b.bh_stride = l.fp8_block ? 1 : 0;
  b.seg_rows = l.SL;
  return FUSP_OK;
}

// ---------------------------------------------------------------- attention step
fusp_status attend(const Layer& l, const Buffers& b, const void* K, const void* V, const int* k_exp,
                   const int* v_exp, bool first, bool last, void* out, float* lse_out,
                   cudaStream_t s, int reserve_sms = 0) {
  AttnLaunch a{};
  if (reserve_sms > 0) a.max_ctas = sm_count() - reserve_sms;
  a.split_ws = b.attn_ws;
  a.split_ws_bytes = b.attn_ws_bytes;
  a.split_counters = b.attn_cnt;
  a.split_counter_words = b.attn_cnt_words;
  a.qk_dtype = l.qk_dt;
  a.k_dtype = l.k_op;
  a.v_dtype = l.v_op;
  a.q = b.Qr;
  a.k = K;
  a.v = V;
  a.q_exp = b.q_exp;
  a.k_exp = k_exp;
  a.v_exp = v_exp;
  a.q_hs = a.k_hs = a.v_hs = int64_t(l.span) * l.D;
  a.heads = l.heads_r;
  a.sq = l.span;
  a.skv = l.span;
  a.d = l.D;
  const bool direct_out = l.mode == Mode::kRing || l.U == 1;
  if (last) {
    a.out = direct_out ? out : b.send_out;
    a.out_dtype = l.out_dt;
    if (direct_out) {
      a.out_chunk = l.span;
      a.out_hs = int64_t(l.span) * l.D;
      a.out_cs = 0;
      a.out_rs = l.D;
    } else {  // epilogue stores O straight into the output all-to-all slots (t = row / SL)
      a.out_chunk = l.SL;
      a.out_hs = int64_t(l.SL) * l.D;
      a.out_cs = l.blk;
      a.out_rs = l.D;
    }
    a.lse = lse_out;
    a.lse_hs = l.span;
    if (!direct_out && lse_out != nullptr) {  // LSE into its own all-to-all slots [U][B][hp][SL]
      a.lse = b.lse_send;
      a.lse_hs = l.SL;
      a.lse_cs = l.blk / l.D;
    }
    if (!direct_out && l.peer) {
      // the output reshard fused into the epilogue: rows [t*SL, (t+1)*SL) go straight to my
      // slot of member t's output region over NVLink (protocols.cpp:182-203)
      a.peer_chunks = l.U;
      const size_t os = size_t(l.blk) * l.wout, ls = size_t(l.blk / l.D) * 4;
      for (int t = 0; t < l.U; ++t) {
        a.out_peer[t] = l.pw[t] + l.pw_out + size_t(l.ug.pos) * os;
        a.lse_peer[t] = reinterpret_cast<float*>(l.pw[t] + l.pw_lse + size_t(l.ug.pos) * ls);
      }
      a.out = a.out_peer[0];
      if (lse_out != nullptr) a.lse = a.lse_peer[0];
    }
  } else {
    a.out = b.acc_o;
    a.out_dtype = FUSP_F32;
    a.out_chunk = l.span;
    a.out_hs = int64_t(l.span) * l.D;
    a.out_cs = 0;
    a.out_rs = l.D;
    a.lse = b.acc_lse;
    a.lse_hs = l.span;
  }
  if (!first) {  // merge_lse(acc, part) fused into the epilogue (protocols.cpp:265-266, :315-316)
    a.acc_o = b.acc_o;
    a.acc_lse = b.acc_lse;
  }
  return launch_attention(a, s);
}

// ---------------------------------------------------------------- ring
fusp_status ring(fusp_ctx_s* c, const Layer& l, Buffers& b, const void* k_src, const void* v_src,
                 void* out, float* lse_out, cudaStream_t s) {
  const int R = l.R;
  const int hr = l.heads_r;
  const bool timing = !c->capturing && R <= fusp_ctx_s::kMaxSteps;
  c->timed_steps = timing ? R : 0;
  // wire part per K and per V: codes + f32 scale(s) (the reference's 4-byte scale + codes), or
  // the chunk in the caller's dtype
  const size_t part_bytes = l.fp8 ? size_t(l.C) + 4 * size_t(l.nsc_chunk) : size_t(l.C) * l.w_in;
  const int64_t block = l.fp8_block ? int64_t(l.span) * l.D : l.C;  // quantization block
  if (R == 1) {
    if (timing) FUSP_CUDA(cudaEventRecord(c->tc0[0], s));
    FUSP_CHECK(attend(l, b, b.Kr, b.Vr, b.k_exp, b.v_exp, true, true, out, lse_out, s));
    if (timing) FUSP_CUDA(cudaEventRecord(c->tc1[0], s));
    return FUSP_OK;
  }
  const bool usp_local = l.mode != Mode::kRing;
  // Fill the FP8 send wire [codes][f32 scales] for one hop from the chunk we hold.
  auto quantize_hop = [&](int hop, int from_buf, cudaStream_t st) -> fusp_status {
    Fp8Src srcs[2];
    uint32_t* works[2];
    float* scs[2];
    uint8_t* cds[2];
    for (int p = 0; p < 2; ++p) {
      uint8_t* codes = reinterpret_cast<uint8_t*>(b.sw[p]);
      float* scales = reinterpret_cast<float*>(b.sw[p] + l.C);
      Fp8Src src{};
      if (hop == 1 && !usp_local) {  // pure ring: quantize the caller's local chunk
        src = Fp8Src{p == 0 ? k_src : v_src, p == 0 ? l.k_dt : l.in_dt, nullptr, 0, 0, l.D,
                      l.span, l.span};
      } else if (hop == 1) {  // USP: exact f32 values of the (multi-scale) resharded chunk
        src = Fp8Src{p == 0 ? b.Kc : b.Vc, FUSP_E4M3, p == 0 ? b.Ks : b.Vs, b.s_stride,
                     b.bh_stride, l.D, l.span, b.seg_rows};
      } else {  // forward: re-quantize the dequantized chunk just received (protocols.cpp:309-310)
        const char* w = b.rb[from_buf][p];
        src = Fp8Src{w, FUSP_E4M3, reinterpret_cast<const float*>(w + l.C), 0,
                     l.fp8_block ? 1 : 0, l.D, l.span, l.span};
      }
      srcs[p] = src;
      works[p] = b.amax + p * (l.nsc_chunk + 1);
      scs[p] = scales;
      cds[p] = codes;
    }
    // beside the attention (pipelined: the side stream) the two-pass form, which runs on the
    // SMs the compute leaves free; the one-launch form needs the whole GPU to start
    return launch_quantize_fp8_multi(srcs, 2, l.C, block, works, scs, cds, nullptr, st, st == s);
  };
  // Transfer hop `hop` into buffer hop % 2, then stage the received chunk for the tensor cores
  // on the same stream (under the previous step's compute when pipelined).
  auto exchange = [&](int hop, cudaStream_t st) -> fusp_status {
    const int into = hop % 2, from = (hop - 1) % 2;
    const void* snd[2];
    if (l.fp8) {
      if (hop == 1) {
        FUSP_CHECK(quantize_hop(hop, from, st));
        snd[0] = b.sw[0];
        snd[1] = b.sw[1];
      } else {
        // Forwarding a chunk that quantize produced as a whole (one scale per quantization
        // block): quantize(dequantize(chunk)) (protocols.cpp:309-310) keeps every code -- the
        // block's max |value| is decode(0x7E) * s = RN(448 s), and RN(RN(d s) / s') = d (1 +
        // O(2^-23)) rounds back to d for every E4M3 value d -- and only the scale becomes
        // RN(RN(448 s) / 448).  So the received buffer is forwarded in place with its trailer
        // updated (after its own staging read the old scale): no pass over the codes.
        // tests/test_gpu_wire.py pins the forwarded bytes to the reference quantizer.
        float* tr[2] = {reinterpret_cast<float*>(b.rb[from][0] + l.C),
                        reinterpret_cast<float*>(b.rb[from][1] + l.C)};
        FUSP_CHECK(launch_fp8_forward_scales(tr, 2, l.nsc_chunk, st));
        snd[0] = b.rb[from][0];
        snd[1] = b.rb[from][1];
      }
    } else if (hop == 1) {
      snd[0] = b.Kw;
      snd[1] = b.Vw;
    } else {
      snd[0] = b.rb[from][0];
      snd[1] = b.rb[from][1];
    }
    void* rcv[2] = {b.rb[into][0], b.rb[into][1]};
    const size_t bytes[2] = {part_bytes, part_bytes};
    FUSP_CHECK(record_wire(c, 1, hop, snd[0], part_bytes, st));
    FUSP_CHECK(record_wire(c, 2, hop, snd[1], part_bytes, st));
    if (l.peer_ring) {
      // Through the windows (protocols.cpp:253-257 as stores): my receive buffer `into` was
      // last read by my compute step hop-2 (the caller's event wait precedes this on `st`) and
      // by my forward of hop-1 (earlier on `st`), so I tell my previous member it may overwrite
      // it, and wait for the same word from my next member before writing into its buffer.  Then copy both parts (copy engines, over NVLink for a real peer),
      // signal the next member and wait for my previous member's chunk.
      // Released at EVERY hop, also for a buffer no hop has used yet (the pair of signals is
      // then a plain handshake): the first hops of a layer reuse the buffers of the previous
      // layer, and a captured graph replays the same kernels whatever ran before, so no host
      // state may decide which hops release.
      const double to = sync_timeout_s();
      FUSP_CHECK(launch_peer_signal_wait(*c->peer, 3, l.ring_prev, 3, l.ring_next, to, st));
      for (int p = 0; p < 2; ++p)
        FUSP_CUDA(cudaMemcpyAsync(l.ring_next_win + l.pw_ring + (2 * into + p) * l.pw_ring_part, snd[p],
                                  part_bytes, cudaMemcpyDeviceToDevice, st));
      FUSP_CHECK(launch_peer_signal_wait(*c->peer, 2, l.ring_next, 2, l.ring_prev, to, st));
    } else {
      FUSP_CHECK(c->comm->ring_exchange(l.rg, snd, rcv, bytes, 2, st));
    }
    c->send_bytes += 2 * part_bytes;
    log_send(c, l.rg, hop, part_bytes);  // K (protocols.cpp:253)
    log_send(c, l.rg, hop, part_bytes);  // V (protocols.cpp:254)
    StageOp ops[2];
    int n = 0;
    for (int p = 0; p < 2; ++p) {
      void* dst = p == 0 ? b.Kd[into] : b.Vd[into];
      if (dst == nullptr) continue;  // the chunk is already the MMA operand
      StageOp o = staged_op(b.rb[into][p], l.fp8 ? FUSP_E4M3 : l.in_dt, dst, p == 0 ? l.k_op : l.v_op,
                            b.exps + (3 + 2 * into + p) * hr, b.ring_w[into][p]);
      if (l.fp8) {
        o.scales = reinterpret_cast<const float*>(b.rb[into][p] + l.C);
        o.scale_bh_stride = l.fp8_block ? 1 : 0;
      }
      ops[n++] = o;
    }
    return launch_stage(ops, n, hr, l.span, l.D, 1, st);
  };
  auto operands = [&](int hop, const void** K, const void** V, const int** ke, const int** ve) {
    const int buf = hop % 2;
    *K = b.Kd[buf] ? b.Kd[buf] : b.rb[buf][0];
    *V = b.Vd[buf] ? b.Vd[buf] : b.rb[buf][1];
    *ke = b.Kd[buf] && l.k_op == FUSP_F16 ? b.exps + (3 + 2 * buf) * hr : nullptr;  // guarded
    *ve = b.Vd[buf] && l.v_op == FUSP_F16 ? b.exps + (4 + 2 * buf) * hr : nullptr;
  };

  if (!l.pipelined) {
    // ring_attention_serial (protocols.cpp:237-268): compute, then send/recv/compute per round.
    if (timing) FUSP_CUDA(cudaEventRecord(c->tc0[0], s));
    FUSP_CHECK(attend(l, b, b.Kr, b.Vr, b.k_exp, b.v_exp, true, false, out, lse_out, s));
    if (timing) FUSP_CUDA(cudaEventRecord(c->tc1[0], s));
    for (int i = 1; i < R; ++i) {
      if (timing) FUSP_CUDA(cudaEventRecord(c->tm0[i], s));
      FUSP_CHECK(exchange(i, s));
      if (timing) FUSP_CUDA(cudaEventRecord(c->tm1[i], s));
      const void *K, *V;
      const int *ke, *ve;
      operands(i, &K, &V, &ke, &ve);
      if (timing) FUSP_CUDA(cudaEventRecord(c->tc0[i], s));
      FUSP_CHECK(attend(l, b, K, V, ke, ve, false, i == R - 1, out, lse_out, s));
      if (timing) FUSP_CUDA(cudaEventRecord(c->tc1[i], s));
    }
    return FUSP_OK;
  }
  // ring_attention_pipelined (Alg. 2, protocols.cpp:270-319): round i+1's transfer runs on
  // the side stream while round i computes; buffers alternate, WAR hazards are events.
  cudaStream_t m = c->side;
  FUSP_CUDA(cudaEventRecord(c->ev_fork, s));
  FUSP_CUDA(cudaStreamWaitEvent(m, c->ev_fork, 0));
  if (timing) FUSP_CUDA(cudaEventRecord(c->tm0[1], m));
  FUSP_CHECK(exchange(1, m));
  if (timing) FUSP_CUDA(cudaEventRecord(c->tm1[1], m));
  FUSP_CUDA(cudaEventRecord(c->ev_recv[1], m));
  // compute steps that run beside a transfer leave its SMs free (NCCL kernels need them)
  const int reserve = l.peer_ring ? 0 : c->comm->sms_in_flight();  // (copy engines on the peer ring)
  if (timing) FUSP_CUDA(cudaEventRecord(c->tc0[0], s));
  FUSP_CHECK(attend(l, b, b.Kr, b.Vr, b.k_exp, b.v_exp, true, false, out, lse_out, s, reserve));
  if (timing) FUSP_CUDA(cudaEventRecord(c->tc1[0], s));
  FUSP_CUDA(cudaEventRecord(c->ev_attn[0], s));
  for (int i = 1; i < R; ++i) {
    FUSP_CUDA(cudaStreamWaitEvent(s, c->ev_recv[i % 2], 0));
    if (i < R - 1) {
      // buffer (i+1)%2 (and its staged operands) was last read by compute step i-1
      FUSP_CUDA(cudaStreamWaitEvent(m, c->ev_attn[(i - 1) % 2], 0));
      if (timing) FUSP_CUDA(cudaEventRecord(c->tm0[i + 1], m));
      FUSP_CHECK(exchange(i + 1, m));
      if (timing) FUSP_CUDA(cudaEventRecord(c->tm1[i + 1], m));
      FUSP_CUDA(cudaEventRecord(c->ev_recv[(i + 1) % 2], m));
    }
    const void *K, *V;
    const int *ke, *ve;
    operands(i, &K, &V, &ke, &ve);
    if (timing) FUSP_CUDA(cudaEventRecord(c->tc0[i], s));
    FUSP_CHECK(attend(l, b, K, V, ke, ve, false, i == R - 1, out, lse_out, s, i < R - 1 ? reserve : 0));
    if (timing) FUSP_CUDA(cudaEventRecord(c->tc1[i], s));
    FUSP_CUDA(cudaEventRecord(c->ev_attn[i % 2], s));
  }
  FUSP_CUDA(cudaEventRecord(c->ev_join, m));
  FUSP_CUDA(cudaStreamWaitEvent(s, c->ev_join, 0));
  return FUSP_OK;
}

// ---------------------------------------------------------------- Ulysses output reshard
fusp_status ulysses_out(fusp_ctx_s* c, const Layer& l, Buffers& b, void* out, float* lse_out,
                        cudaStream_t s) {
  if (!l.wire()) return FUSP_OK;  // epilogue wrote `out` (and `lse`) directly
  const size_t slot = size_t(l.blk) * l.wout;
  if (l.peer) {
    // the members' epilogues wrote my output region: signal mine, wait for theirs, then the
    // region is the concatenation over heads (B = 1: exactly `out`)
    FUSP_CHECK(launch_peer_exchange(*c->peer, 1, l.ug, sync_timeout_s(), s));
    if (l.B == 1 && l.out_view != nullptr && lse_out == nullptr) *l.out_view = b.recv_out;
    else if (l.B == 1) FUSP_CUDA(cudaMemcpyAsync(out, b.recv_out, slot * l.U, cudaMemcpyDeviceToDevice, s));
  } else {
    FUSP_CHECK(c->comm->all_to_all(l.ug, b.send_out, b.recv_out, slot, slot, s));
  }
  c->a2a_bytes += uint64_t(l.U - 1) * slot;
  log_a2a(c, l.ug, uint64_t(l.U - 1) * slot);
  if (l.B > 1)  // concat_heads (protocols.cpp:196-202)
    FUSP_CHECK(launch_unpack_heads(b.recv_out, l.blk, out, l.out_dt, l.B, l.hp, l.SL, l.D, l.U, s));
  if (lse_out != nullptr) {
    // The reference's usp_attention drops the LSE (protocols.cpp:339); fastusp returns it on
    // request: the rows' LSE ride a second, small all-to-all back to their sequence shards
    // (B = 1: straight into the caller's [1][H][SL] buffer, heads t*hp.. from member t).
    const size_t ls = size_t(l.blk / l.D) * 4;
    float* dst = l.B == 1 ? lse_out : b.lse_recv;
    if (l.peer) {  // already in my window with O (same exchange)
      if (l.B == 1) FUSP_CUDA(cudaMemcpyAsync(lse_out, b.lse_recv, ls * l.U, cudaMemcpyDeviceToDevice, s));
    } else {
      FUSP_CHECK(c->comm->all_to_all(l.ug, b.lse_send, dst, ls, ls, s));
    }
    c->a2a_bytes += uint64_t(l.U - 1) * ls;
    log_a2a(c, l.ug, uint64_t(l.U - 1) * ls);
    if (l.B > 1) {  // slot t [B][hp][SL] -> lse[b][t*hp + hl][SL]
      const size_t row = size_t(l.hp) * l.SL * 4;
      for (int t = 0; t < l.U; ++t)
        FUSP_CUDA(cudaMemcpy2DAsync(lse_out + size_t(t) * l.hp * l.SL, size_t(l.H) * l.SL * 4,
                                    reinterpret_cast<const char*>(b.lse_recv) + t * ls, row, row,
                                    l.B, cudaMemcpyDeviceToDevice, s));
    }
  }
  return FUSP_OK;
}

// detail::ulysses_output_reshard (protocols.cpp:182-203) on its own: o [B][hp][U*SL][D] ->
// slot t = rows [t*SL, (t+1)*SL) (one stage launch, the inverse of the unpack mapping) ->
// all_to_all -> concat_heads.
fusp_status output_reshard(fusp_ctx_s* c, const Layer& l, Buffers& b, const void* o, int dt,
                           void* out, cudaStream_t s) {
  StageOp op{};
  op.src = o;
  op.sdt = dt;
  op.src_slot_stride = int64_t(l.SL) * l.D;
  op.src_bh_stride = int64_t(l.span) * l.D;
  op.dst = b.send_out;
  op.ddt = dt;
  op.dst_slot_stride = l.blk;
  op.dst_bh_stride = int64_t(l.SL) * l.D;
  FUSP_CHECK(launch_stage(&op, 1, l.heads_r, l.SL, l.D, l.U, s));
  return ulysses_out(c, l, b, out, nullptr, s);
}

fusp_status check_inputs(fusp_ctx_s* c, Mode mode, const Layer& l, const void* q, const void* k,
                         const void* v, cudaStream_t s) {
  size_t need = 256;
  FUSP_CHECK(ensure_arena(c, need, s));
  uint32_t* flag = static_cast<uint32_t*>(c->ws->arena);
  FUSP_CUDA(cudaMemsetAsync(flag, 0, 4, s));
  const int64_t n = int64_t(l.B) * l.H * l.SL * l.D;
  FUSP_CHECK(launch_finite(q, l.in_dt, n, flag, s));
  FUSP_CHECK(launch_finite(k, l.in_dt, n, flag, s));
  FUSP_CHECK(launch_finite(v, l.in_dt, n, flag, s));
  uint32_t h = 0;
  FUSP_CUDA(cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, s));
  FUSP_CHECK(c->comm->wait(s, sync_timeout_s(), "check_finite"));
  if (h)  // check_local_qkv (protocols.cpp:102-104)
    return set_error(FUSP_ERR_INVALID_ARGUMENT,
                     std::string(tag(mode)) + ": non-finite element in protocol input");
  return FUSP_OK;
}

fusp_status validate_prologue(const fusp_qk_prologue* p) {
  if (!p) return FUSP_OK;
  const bool rope = p->rope_cos != nullptr || p->rope_sin != nullptr;
  if (rope && (p->rope_cos == nullptr || p->rope_sin == nullptr))
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "qk prologue: rope_cos and rope_sin go together");
  if (!(p->eps >= 0.f))
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "qk prologue: eps must be >= 0");
  return FUSP_OK;
}

fusp_status plan_prologue(fusp_ctx_s* c, const fusp_qk_prologue* p, Layer* L) {
  Layer& l = *L;
  if (!p) return FUSP_OK;
  FUSP_CHECK(validate_prologue(p));
  if (l.D != 128) return set_error(FUSP_ERR_SHAPE, "qk prologue: head dim must be 128");
  const bool rope = p->rope_cos != nullptr;
  l.pos0 = p->rope_pos0 < 0 ? int64_t(c->rank) * l.SL : p->rope_pos0;
  if (rope && (p->rope_rows < l.pos0 + l.SL))
    return set_error(FUSP_ERR_SHAPE, "qk prologue: rope table has " + std::to_string(p->rope_rows) +
                                         " rows, positions up to " +
                                         std::to_string(l.pos0 + l.SL) + " needed");
  l.pro = p;
  l.pro_q = rope || p->q_norm_weight != nullptr;
  const bool pk = rope || p->k_norm_weight != nullptr;
  if (pk && l.fp8) {  // quantizers read a normalized f32 copy of K
    l.pro_k_pre = true;
    l.k_dt = FUSP_F32;
  } else {
    l.pro_k = pk;
  }
  return FUSP_OK;
}

// Producer of the layer's Q, K, V, called with the layer's own operand buffers (slots).
using Produce = std::function<fusp_status(const QkvDst&)>;

// Variants of a layer call beyond the mesh protocols.
struct LayerCall {
  const Group* grp = nullptr;      // ulysses / ring over this ProcessGroup (null: mesh / world)
  bool reshard_in = false;         // detail::ulysses_input_reshard only: Q, K, V -> rq, rk, rv
  void *rq = nullptr, *rk = nullptr, *rv = nullptr;
  int rdt = FUSP_F32;
  const void* reshard_out = nullptr;  // detail::ulysses_output_reshard only: o -> out
  const void** out_view = nullptr;    // see Layer::out_view (fusp_usp_block's out projection)
};

fusp_status run_layer(fusp_ctx_s* c, Mode mode, int r, const void* q, const void* k,
                      const void* v, int in_dt, fusp_shape4 ls, void* out, float* lse_out,
                      const fusp_comm_options* opts, cudaStream_t s, bool size_only = false,
                      const fusp_qk_prologue* pro = nullptr, const Produce* produce = nullptr,
                      const LayerCall* call = nullptr) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  FUSP_CUDA(cudaSetDevice(c->device));
  fusp_comm_options o{};
  o.out_dtype = FUSP_F32;
  if (opts) o = *opts;
  const LayerCall none{};
  if (call == nullptr) call = &none;
  Layer l;
  FUSP_CHECK(plan_layer(c, mode, r, ls, in_dt, o, &l, call->grp));
  l.out_view = call->out_view;
  if (call->reshard_in || call->reshard_out != nullptr) {
    l.force_wire = true;
    if (call->reshard_in) {
      l.reshard_q = call->rq;
      l.reshard_k = call->rk;
      l.reshard_v = call->rv;
      l.reshard_dt = call->rdt;
    }
  }
  FUSP_CHECK(plan_prologue(c, pro, &l));
  if (c->nccl && l.U > 1 && l.R > 1) FUSP_CHECK(c->nccl->ensure_mesh(l.R));
  if (o.check_finite && !size_only) FUSP_CHECK(check_inputs(c, mode, l, q, k, v, s));
  if (produce != nullptr) {
    if (l.fp8 || l.pro != nullptr || l.mode == Mode::kRing || o.check_finite ||
        (l.in_dt != FUSP_BF16 && l.in_dt != FUSP_F16))
      return set_error(FUSP_ERR_UNSUPPORTED, "operand producer: bf16/f16 wire, no prologue, no check");
    l.prepacked = true;
  }
  if (c->peer && (l.wire() || l.R > 1)) {
    // a layer is on the peer path when every transfer it makes goes through the windows
    // (counted on the peer path when its Ulysses reshards -- or, without them, its ring --
    // went through the windows)
    plan_peer(c, l);
    const bool on = l.wire() ? l.peer : l.peer_ring;
    if (!size_only) ++(on ? c->peer_layers : c->peer_fallbacks);
  }
  if (c->capturing && !c->comm->capturable() && ((l.wire() && !l.peer) || (l.R > 1 && !l.peer_ring)))
    return set_error(FUSP_ERR_UNSUPPORTED,
                     "graph capture: this layer needs the in-process fabric's host rendezvous");
  Carve cv;
  CarveWords cw;
  Buffers b;
  const size_t cnt_words = attention_counter_words(l.heads_r, l.span);
  cw.take(cnt_words);
  carve(l, cv, cw, &b, q, k, v, out);
  FUSP_CHECK(ensure_arena(c, cv.off + 256, s));
  FUSP_CHECK(ensure_words(c, cw.off, s));
  c->last_stream = s;
  c->last_stream_valid = true;
  if (size_only) return FUSP_OK;
  cv = Carve{static_cast<char*>(c->ws->arena), 0};
  cw = CarveWords{c->ws->words.ptr, 0};
  b = Buffers{};
  b.attn_cnt = cw.take(cnt_words);
  b.attn_cnt_words = cnt_words;
  carve(l, cv, cw, &b, q, k, v, out);
  if (l.pro_k_pre) {
    FUSP_CHECK(launch_norm_rope_pack(k, l.in_dt, b.Kpro, FUSP_F32, 0, l.B, l.H, l.SL, l.D, 1,
                                     pro->k_norm_weight, pro->eps, pro->rope_cos, pro->rope_sin,
                                     l.pos0, s));
    k = b.Kpro;
    if (l.mode == Mode::kRing || l.U == 1) b.Ks_src = b.Kw = b.Kpro;
  }
  if (produce != nullptr) {
    QkvDst d{};
    int64_t boff[kMaxPeerChunks] = {};
    if (l.U > 1 && l.peer) {  // straight into my slot of every member's receive region
      char* sbase = l.pw[0] + size_t(l.ug.pos) * l.slot_stride;
      for (int t = 0; t < l.U; ++t) boff[t] = l.pw[t] - l.pw[0];
      d = QkvDst{sbase, sbase + l.off_k, sbase + l.off_v, l.in_dt, l.in_dt, l.U,
                 int64_t(l.slot_stride / l.w_in), boff};
    } else if (l.U > 1) {  // straight into the Ulysses send slots: [Q blk][K blk][V blk] per slot
      d = QkvDst{b.send_in, b.send_in + l.off_k, b.send_in + l.off_v, l.in_dt, l.in_dt, l.U,
                 int64_t(l.slot_stride / l.w_in)};
    } else {        // the staging sources (Q, K: the attention operands themselves)
      d = QkvDst{const_cast<void*>(b.Qs), const_cast<void*>(b.Ks_src), const_cast<void*>(b.Vs_src),
                 l.in_dt, l.in_dt, 1, 0};
    }
    FUSP_CHECK((*produce)(d));
  }
  if (call->reshard_out != nullptr) return output_reshard(c, l, b, call->reshard_out, l.out_dt, out, s);
  if (call->reshard_in) return ulysses_in(c, l, b, q, k, v, s);
  // the reference still runs a 1-member all_to_all (fabric.cpp:199-226)
  const bool uly1 = l.mode != Mode::kRing && !l.wire();
  if (uly1) log_a2a(c, l.ug, 0);
  FUSP_CHECK(ulysses_in(c, l, b, q, k, v, s));
  FUSP_CHECK(ring(c, l, b, k, v, out, lse_out, s));
  FUSP_CHECK(ulysses_out(c, l, b, out, lse_out, s));
  if (uly1) log_a2a(c, l.ug, 0);
  c->tl_steps = c->timed_steps;
  c->tl_pipelined = l.pipelined && l.R > 1;
  c->tl_valid = c->timed_steps > 0;
  c->tl_next = l.rg.members[(l.rg.pos + 1) % l.rg.size()];
  return FUSP_OK;
}

fusp_status init_ctx(fusp_ctx_s* c) {
  FUSP_CUDA(cudaSetDevice(c->device));
  FUSP_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  FUSP_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  FUSP_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    FUSP_CUDA(cudaEventCreateWithFlags(&c->ev_recv[i], cudaEventDisableTiming));
    FUSP_CUDA(cudaEventCreateWithFlags(&c->ev_attn[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < fusp_ctx_s::kMaxSteps; ++i) {
    FUSP_CUDA(cudaEventCreate(&c->tc0[i]));
    FUSP_CUDA(cudaEventCreate(&c->tc1[i]));
    FUSP_CUDA(cudaEventCreate(&c->tm0[i]));
    FUSP_CUDA(cudaEventCreate(&c->tm1[i]));
  }
  return FUSP_OK;
}

}  // namespace

extern "C" {

fusp_status fusp_fabric_create(int world, fusp_fabric* out) {
  clear_error();
  if (world < 1) return set_error(FUSP_ERR_COMM, "run_protocol: need at least one worker");
  *out = new fusp_fabric_s(world);
  return FUSP_OK;
}

fusp_status fusp_fabric_destroy(fusp_fabric f) {
  delete f;
  return FUSP_OK;
}

fusp_status fusp_ctx_create_local(fusp_fabric f, int rank, int device, fusp_ctx* out) {
  clear_error();
  if (!f) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null fabric");
  if (rank < 0 || rank >= f->fabric.world)
    return set_error(FUSP_ERR_COMM, "rank " + std::to_string(rank) + " out of range [0," +
                                        std::to_string(f->fabric.world) + ")");
  auto* c = new fusp_ctx_s;
  c->rank = rank;
  c->world = f->fabric.world;
  c->device = device;
  fusp_status st = init_ctx(c);
  if (st != FUSP_OK) {
    delete c;
    return st;
  }
  c->comm = std::make_unique<LocalComm>(&f->fabric, rank, device);
  *out = c;
  return FUSP_OK;
}

fusp_status fusp_nccl_unique_id(uint8_t uid[128]) {
  clear_error();
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(uid, &id, 128);
  return FUSP_OK;
}

fusp_status fusp_ctx_create_nccl(const uint8_t uid[128], int world, int rank, int device,
                                 fusp_ctx* out) {
  clear_error();
  auto* c = new fusp_ctx_s;
  c->rank = rank;
  c->world = world;
  c->device = device;
  fusp_status st = init_ctx(c);
  if (st != FUSP_OK) {
    delete c;
    return st;
  }
  ncclUniqueId id;
  std::memcpy(&id, uid, 128);
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_error(r, "ncclCommInitRank");
  }
  auto nc = std::make_unique<NcclComm>(comm, rank, world);
  c->nccl = nc.get();
  c->comm = std::move(nc);
  *out = c;
  return FUSP_OK;
}

fusp_status fusp_ctx_destroy(fusp_ctx c) {
  clear_error();
  if (!c) return FUSP_OK;
  if (c->live_graphs > 0)
    return set_error(FUSP_ERR_UNSUPPORTED, "context has " + std::to_string(c->live_graphs) +
                                               " live graph(s): destroy them first");
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  c->peer.reset();
  c->comm.reset();
  c->own.release();
  c->clear_wire();
  if (c->block_ws) cudaFree(c->block_ws);
  c->host.reset();
  if (c->side) cudaStreamDestroy(c->side);
  for (cudaEvent_t e : {c->ev_fork, c->ev_join, c->ev_recv[0], c->ev_recv[1], c->ev_attn[0], c->ev_attn[1]})
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < fusp_ctx_s::kMaxSteps; ++i)
    for (cudaEvent_t e : {c->tc0[i], c->tc1[i], c->tm0[i], c->tm1[i]})
      if (e) cudaEventDestroy(e);
  delete c;
  return FUSP_OK;
}

fusp_status fusp_ctx_peer_window(fusp_ctx c, size_t window_bytes, void* handle_out) {
  clear_error();
  if (!c || !handle_out) return set_error(FUSP_ERR_INVALID_ARGUMENT, "peer window: null argument");
  if (c->live_graphs > 0)
    return set_error(FUSP_ERR_UNSUPPORTED, "peer window: the context has live graphs");
  FUSP_CUDA(cudaSetDevice(c->device));
  FUSP_CUDA(cudaDeviceSynchronize());
  auto w = std::make_unique<PeerWindow>();
  PeerHandle h{};
  FUSP_CUDA(cudaSetDevice(c->device));
  FUSP_CHECK(preload_kernels());  // no lazy module load may wait behind a spinning exchange
  FUSP_CHECK(peer_window_create(w.get(), c->rank, c->world, c->device, window_bytes, &h));
  std::memcpy(handle_out, &h, sizeof(h));
  c->peer = std::move(w);
  c->peer_layers = c->peer_fallbacks = 0;
  c->peer_open = false;
  return FUSP_OK;
}

fusp_status fusp_ctx_peer_open(fusp_ctx c, const void* handles) {
  clear_error();
  if (!c || !c->peer || !handles)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "peer open: create the window first");
  fusp_status st = peer_window_open(c->peer.get(), static_cast<const PeerHandle*>(handles));
  if (st != FUSP_OK) {
    c->peer.reset();
    return st;
  }
  c->peer_open = true;
  return FUSP_OK;
}

fusp_status fusp_ctx_peer_enable(fusp_ctx c, size_t window_bytes) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  PeerHandle mine{};
  FUSP_CHECK(fusp_ctx_peer_window(c, window_bytes, &mine));
  std::vector<PeerHandle> all(static_cast<size_t>(c->world));
  fusp_status st = c->comm->allgather_host(&mine, sizeof(mine), all.data());
  if (st != FUSP_OK) {
    c->peer.reset();
    return st;
  }
  return fusp_ctx_peer_open(c, all.data());
}

fusp_status fusp_peer_window_bytes(int world, int ring_dim, fusp_dtype in_dtype, fusp_shape4 ls,
                                   const fusp_comm_options* opts, size_t* bytes) {
  clear_error();
  if (!bytes || world < 1) return set_error(FUSP_ERR_INVALID_ARGUMENT, "peer window bytes: bad argument");
  fusp_ctx_s tmp;
  tmp.world = world;
  tmp.rank = 0;
  fusp_comm_options o{};
  o.out_dtype = FUSP_F32;
  if (opts) o = *opts;
  Layer l;
  FUSP_CHECK(plan_layer(&tmp, Mode::kUsp, ring_dim, ls, in_dtype, o, &l));
  peer_layout(l);
  *bytes = l.pw_need;
  return FUSP_OK;
}

fusp_status fusp_ctx_peer_disable(fusp_ctx c) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  if (c->live_graphs > 0)
    return set_error(FUSP_ERR_UNSUPPORTED, "peer disable: the context has live graphs");
  FUSP_CUDA(cudaSetDevice(c->device));
  if (c->last_stream_valid) FUSP_CUDA(cudaStreamSynchronize(c->last_stream));
  FUSP_CUDA(cudaStreamSynchronize(c->side));
  c->peer.reset();
  c->peer_open = false;
  return FUSP_OK;
}

fusp_status fusp_ctx_peer_stats(fusp_ctx c, uint64_t* layers, uint64_t* fallbacks) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  if (layers) *layers = c->peer_layers;
  if (fallbacks) *fallbacks = c->peer_fallbacks;
  return FUSP_OK;
}

fusp_status fusp_ctx_synchronize(fusp_ctx c, fusp_stream_t stream, double timeout_s) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  FUSP_CUDA(cudaSetDevice(c->device));
  FUSP_CHECK(c->comm->wait(reinterpret_cast<cudaStream_t>(stream),
                           timeout_s > 0 ? timeout_s : sync_timeout_s(), "synchronize"));
  if (c->peer) FUSP_CHECK(peer_window_check(*c->peer, "synchronize", reinterpret_cast<cudaStream_t>(stream)));
  return FUSP_OK;
}

fusp_status fusp_ctx_debug_wire(fusp_ctx c, int enable) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  FUSP_CUDA(cudaSetDevice(c->device));
  FUSP_CUDA(cudaDeviceSynchronize());
  c->clear_wire();
  c->debug_wire = enable != 0;
  return FUSP_OK;
}

int fusp_ctx_debug_wire_count(fusp_ctx c) { return c ? static_cast<int>(c->wire.size()) : 0; }

fusp_status fusp_ctx_debug_wire_get(fusp_ctx c, int index, int* kind, int* round, void* host,
                                    size_t cap, size_t* bytes) {
  clear_error();
  if (!c || index < 0 || index >= static_cast<int>(c->wire.size()))
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "debug wire: no record " + std::to_string(index));
  const auto& r = c->wire[size_t(index)];
  if (kind) *kind = r.kind;
  if (round) *round = r.round;
  if (bytes) *bytes = r.bytes;
  if (host != nullptr) {
    FUSP_CUDA(cudaSetDevice(c->device));
    FUSP_CUDA(cudaMemcpy(host, r.dev, cap < r.bytes ? cap : r.bytes, cudaMemcpyDeviceToHost));
  }
  return FUSP_OK;
}

int fusp_ctx_rank(fusp_ctx c) { return c ? c->rank : -1; }
int fusp_ctx_world(fusp_ctx c) { return c ? c->world : 0; }

fusp_status fusp_ctx_traffic(fusp_ctx c, uint64_t* a2a, uint64_t* snd) {
  if (a2a) *a2a = c->a2a_bytes;
  if (snd) *snd = c->send_bytes;
  return FUSP_OK;
}

fusp_status fusp_ctx_reset_traffic(fusp_ctx c) {
  c->a2a_bytes = 0;
  c->send_bytes = 0;
  c->traffic.clear();
  c->a2a_seq.clear();
  return FUSP_OK;
}

static fusp_status put_json(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
    if (n < s.size()) return set_error(FUSP_ERR_INVALID_ARGUMENT, "json buffer too small");
  }
  return FUSP_OK;
}

fusp_status fusp_ctx_traffic_json(fusp_ctx c, char* buf, size_t cap, size_t* len) {
  clear_error();
  // TrafficLog::to_json (fabric.cpp:72-87): entries in (op, group, round, rank) order
  std::vector<fusp_ctx_s::Traffic> t = c->traffic;
  std::stable_sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
    return std::tie(a.op, a.group, a.round, a.rank) < std::tie(b.op, b.group, b.round, b.rank);
  });
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < t.size(); ++i) {
    if (i) os << ",";
    os << "{\"op\":\"" << t[i].op << "\",\"group\":\"" << t[i].group << "\",\"round\":"
       << t[i].round << ",\"rank\":" << t[i].rank << ",\"bytes\":" << t[i].bytes
       << ",\"msgs\":" << t[i].msgs << "}";
  }
  os << "]";
  return put_json(os.str(), buf, cap, len);
}

fusp_status fusp_ctx_timeline_json(fusp_ctx c, char* buf, size_t cap, size_t* len) {
  clear_error();
  // Timeline::to_json (fabric.cpp:115-125) of the last layer, with device timestamps (ms from
  // the first event).  Event order follows protocols.cpp:243-265 (serial) / :276-316 (pipelined);
  // the merge is fused into the attention epilogue, so it carries compute_end's time.
  if (!c->tl_valid) return put_json("[]", buf, cap, len);
  FUSP_CUDA(cudaSetDevice(c->device));
  const int R = c->tl_steps;
  cudaEvent_t t0 = c->tc0[0];
  if (R > 1 && c->tl_pipelined) t0 = c->tm0[1];
  FUSP_CUDA(cudaEventSynchronize(c->tc1[R - 1]));
  auto ms = [&](cudaEvent_t e) {
    float v = 0.f;
    cudaEventElapsedTime(&v, t0, e);
    return v < 0.f ? 0.f : v;
  };
  struct Ev {
    const char* kind;
    const char* tag;
    int round;
    float t;
  };
  std::vector<Ev> ev;
  if (c->tl_pipelined) {
    ev.push_back({"recv_issue", "kv", 1, ms(c->tm0[1])});
    ev.push_back({"send_issue", "kv", 1, ms(c->tm0[1])});
  }
  ev.push_back({"compute_begin", "attn", 0, ms(c->tc0[0])});
  ev.push_back({"compute_end", "attn", 0, ms(c->tc1[0])});
  for (int r = 1; r < R; ++r) {
    if (!c->tl_pipelined) {
      ev.push_back({"send_issue", "kv", r, ms(c->tm0[r])});
      ev.push_back({"recv_issue", "kv", r, ms(c->tm0[r])});
    }
    ev.push_back({"transfer_complete", "kv", r, ms(c->tm1[r])});
    if (c->tl_pipelined && r < R - 1) {
      ev.push_back({"recv_issue", "kv", r + 1, ms(c->tm0[r + 1])});
      ev.push_back({"send_issue", "kv", r + 1, ms(c->tm0[r + 1])});
    }
    ev.push_back({"compute_begin", "attn", r, ms(c->tc0[r])});
    ev.push_back({"compute_end", "attn", r, ms(c->tc1[r])});
    ev.push_back({"merge", "lse", r, ms(c->tc1[r])});
  }
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < ev.size(); ++i) {
    if (i) os << ",";
    os << "{\"seq\":" << i << ",\"rank\":" << c->rank << ",\"kind\":\"" << ev[i].kind
       << "\",\"tag\":\"" << ev[i].tag << "\",\"round\":" << ev[i].round << ",\"t_ms\":"
       << ev[i].t << "}";
  }
  os << "]";
  return put_json(os.str(), buf, cap, len);
}

fusp_status fusp_ctx_ring_timings(fusp_ctx c, int max_steps, float* compute_ms, float* comm_ms,
                                  int* steps) {
  clear_error();
  FUSP_CUDA(cudaSetDevice(c->device));
  const int n = c->timed_steps < max_steps ? c->timed_steps : max_steps;
  *steps = n;
  for (int i = 0; i < n; ++i) {
    FUSP_CUDA(cudaEventSynchronize(c->tc1[i]));
    FUSP_CUDA(cudaEventElapsedTime(&compute_ms[i], c->tc0[i], c->tc1[i]));
    comm_ms[i] = 0.f;
    if (i > 0) {
      FUSP_CUDA(cudaEventSynchronize(c->tm1[i]));
      FUSP_CUDA(cudaEventElapsedTime(&comm_ms[i], c->tm0[i], c->tm1[i]));
    }
  }
  return FUSP_OK;
}

fusp_status fusp_usp_attention(fusp_ctx c, int ring_dim, const void* q, const void* k,
                               const void* v, fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                               const fusp_comm_options* opts, fusp_stream_t stream) {
  return run_layer(c, Mode::kUsp, ring_dim, q, k, v, in_dtype, ls, out, nullptr, opts,
                   reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_usp_attention_ex(fusp_ctx c, int ring_dim, const void* q, const void* k,
                                  const void* v, fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                                  const fusp_comm_options* opts, const fusp_qk_prologue* prologue,
                                  fusp_stream_t stream) {
  return run_layer(c, Mode::kUsp, ring_dim, q, k, v, in_dtype, ls, out, nullptr, opts,
                   reinterpret_cast<cudaStream_t>(stream), false, prologue);
}

fusp_status fusp_usp_attention_proj(fusp_ctx c, int ring_dim, const void* q, const void* k,
                                    const void* v, fusp_dtype in_dtype, fusp_shape4 ls,
                                    void* attn_out, const fusp_comm_options* opts,
                                    const fusp_qk_prologue* prologue, const void* w_out,
                                    int64_t n_out, void* y, fusp_dtype y_dtype,
                                    fusp_stream_t stream) {
  const int odt = opts ? opts->out_dtype : FUSP_F32;
  if (odt != FUSP_BF16 && odt != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT,
                     "usp_attention_proj: the attention output feeding the projection must be bf16 or f16");
  FUSP_CHECK(run_layer(c, Mode::kUsp, ring_dim, q, k, v, in_dtype, ls, attn_out, nullptr, opts,
                       reinterpret_cast<cudaStream_t>(stream), false, prologue));
  // the consumer, on the same stream straight after the output reshard (and inside any
  // graph being captured)
  return fusp_out_projection(attn_out, static_cast<fusp_dtype>(odt), ls, w_out, n_out, y, y_dtype, stream);
}

fusp_status fusp_usp_block(fusp_ctx c, int ring_dim, const void* x, fusp_dtype x_dtype,
                           int64_t batch, int64_t s_local, int64_t channels, const void* w_qkv,
                           int heads, const fusp_qk_prologue* prologue, const void* w_out,
                           int64_t n_out, void* y, fusp_dtype y_dtype,
                           const fusp_comm_options* opts, fusp_stream_t stream) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  FUSP_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (x_dtype != FUSP_BF16 && x_dtype != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "usp_block: x must be bf16 or f16");
  if (batch <= 0 || s_local <= 0 || channels <= 0 || heads <= 0)
    return set_error(FUSP_ERR_SHAPE, "usp_block: empty shape");
  FUSP_CHECK(validate_prologue(prologue));  // the projection epilogue dereferences cos AND sin
  const int64_t pos0 = prologue && prologue->rope_pos0 >= 0 ? prologue->rope_pos0 : int64_t(c->rank) * s_local;
  if (prologue && prologue->rope_cos && prologue->rope_rows < pos0 + s_local)
    return set_error(FUSP_ERR_SHAPE, "qk prologue: rope table has " + std::to_string(prologue->rope_rows) +
                                         " rows, positions up to " + std::to_string(pos0 + s_local) + " needed");
  // Q, K, V and the attention output, one allocation per context (grown outside capture)
  const size_t one = align_up(size_t(batch) * heads * s_local * 128 * 2, 256);
  if (c->block_ws_bytes < 4 * one) {
    if (c->capturing) return set_error(FUSP_ERR_UNSUPPORTED, "workspace growth during graph capture");
    // stream-ordered like the layer workspace (no device-wide wait: see ensure_arena)
    if (c->block_ws) {
      FUSP_CHECK(quiesce_previous(c, st));
      FUSP_CUDA(cudaFreeAsync(c->block_ws, st));
    }
    c->block_ws = nullptr;
    c->block_ws_bytes = 0;
    FUSP_CUDA(cudaMallocAsync(&c->block_ws, 4 * one, st));
    c->block_ws_bytes = 4 * one;
  }
  char* ws = static_cast<char*>(c->block_ws);
  void *q = ws, *k = ws + one, *v = ws + 2 * one, *attn = ws + 3 * one;
  const void* attn_at = attn;
  fusp_comm_options o{};
  if (opts) o = *opts;
  o.out_dtype = x_dtype;  // the layer's output in the projection's input dtype
  const fusp_shape4 ls{batch, heads, s_local, 128};
  // producer: QKV projection with the QK RMSNorm + RoPE in its epilogue
  auto qkv = [&](const QkvDst& d) {
    return launch_qkv_proj_to(x, x_dtype, int(batch), int(s_local), int(channels), w_qkv, heads, d,
                              prologue ? prologue->q_norm_weight : nullptr,
                              prologue ? prologue->k_norm_weight : nullptr, prologue ? prologue->eps : 0.f,
                              prologue ? prologue->rope_cos : nullptr, prologue ? prologue->rope_sin : nullptr,
                              pos0, st);
  };
  if (!o.fp8_kv && !o.check_finite) {
    // the projection writes Q, K, V straight into the layer's Ulysses send slots (U = 1: the
    // attention operands, V already f16), so neither the pack nor the V conversion runs
    const Produce produce = qkv;
    // with peer windows the QKV projection's epilogue stores into the members' windows (GEMM +
    // input all-to-all in one kernel) and the out projection reads O where the members'
    // attention epilogues put it (the window is not rewritten before this rank's next input
    // exchange, which follows the out projection on this stream -- peer.cu)
    LayerCall call;
    call.out_view = &attn_at;
    FUSP_CHECK(run_layer(c, Mode::kUsp, ring_dim, q, k, v, x_dtype, ls, attn, nullptr, &o, st, false,
                         nullptr, &produce, &call));
  } else {
    FUSP_CHECK(qkv(QkvDst{q, k, v, x_dtype, x_dtype, 1, 0}));
    FUSP_CHECK(run_layer(c, Mode::kUsp, ring_dim, q, k, v, x_dtype, ls, attn, nullptr, &o, st));
  }
  // consumer: output projection
  return fusp_out_projection(attn_at, x_dtype, ls, w_out, n_out, y, y_dtype, stream);
}

fusp_status fusp_group_create(fusp_ctx c, const int* members, int n, fusp_group* out) {
  clear_error();
  if (!c || !out) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context or output");
  *out = nullptr;
  Group g;
  if (n < 0) return set_error(FUSP_ERR_COMM, "empty process group");
  for (int i = 0; i < n; ++i) g.members.push_back(members[i]);
  // validate_group (fabric.cpp:316-324)
  for (int i = 0; i < n; ++i) {
    const int m = members[i];
    if (m < 0 || m >= c->world)
      return set_error(FUSP_ERR_COMM, "group member " + std::to_string(m) + " out of range [0," +
                                          std::to_string(c->world) + ")");
    for (int j = 0; j < i; ++j)
      if (members[j] == m)
        return set_error(FUSP_ERR_COMM, "duplicate member " + std::to_string(m) + " in group " + g.key());
    if (m == c->rank) g.pos = i;
  }
  FUSP_CUDA(cudaSetDevice(c->device));
  if (c->nccl) FUSP_CHECK(c->nccl->split_group(g));  // collective over the world
  if (n == 0) return FUSP_OK;  // joined the split without a group
  if (g.pos < 0)
    return set_error(FUSP_ERR_COMM, "rank " + std::to_string(c->rank) + " not in group " + g.key());
  auto* h = new fusp_group_s;
  h->g = g;
  h->ctx = c;
  *out = h;
  return FUSP_OK;
}

fusp_status fusp_group_destroy(fusp_group g) {
  delete g;
  return FUSP_OK;
}

int fusp_group_size(fusp_group g) { return g ? g->g.size() : 0; }
int fusp_group_position(fusp_group g) { return g ? g->g.pos : -1; }

static fusp_status group_of(fusp_ctx c, fusp_group g, const Group** out) {
  *out = nullptr;
  if (g == nullptr) return FUSP_OK;  // the world
  if (g->ctx != c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "group belongs to another context");
  *out = &g->g;
  return FUSP_OK;
}

fusp_status fusp_usp_attention_lse(fusp_ctx c, int ring_dim, const void* q, const void* k,
                                   const void* v, fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                                   float* lse, const fusp_comm_options* opts, fusp_stream_t stream) {
  return run_layer(c, Mode::kUsp, ring_dim, q, k, v, in_dtype, ls, out, lse, opts,
                   reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_ulysses_attention_group(fusp_ctx c, fusp_group group, const void* q, const void* k,
                                         const void* v, fusp_dtype in_dtype, fusp_shape4 ls,
                                         void* out, float* lse, const fusp_comm_options* opts,
                                         fusp_stream_t stream) {
  clear_error();
  LayerCall call;
  FUSP_CHECK(group_of(c, group, &call.grp));
  return run_layer(c, Mode::kUlysses, 1, q, k, v, in_dtype, ls, out, lse, opts,
                   reinterpret_cast<cudaStream_t>(stream), false, nullptr, nullptr, &call);
}

fusp_status fusp_ring_attention_group(fusp_ctx c, fusp_group group, const void* q, const void* k,
                                      const void* v, fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                                      float* lse, const fusp_comm_options* opts,
                                      fusp_stream_t stream) {
  clear_error();
  LayerCall call;
  FUSP_CHECK(group_of(c, group, &call.grp));
  return run_layer(c, Mode::kRing, c ? c->world : 1, q, k, v, in_dtype, ls, out, lse, opts,
                   reinterpret_cast<cudaStream_t>(stream), false, nullptr, nullptr, &call);
}

fusp_status fusp_ulysses_input_reshard(fusp_ctx c, fusp_group group, const void* q, const void* k,
                                       const void* v, fusp_dtype in_dtype, fusp_shape4 ls,
                                       void* q_out, void* k_out, void* v_out, fusp_dtype out_dtype,
                                       const fusp_comm_options* opts, fusp_stream_t stream) {
  clear_error();
  if (out_dtype != FUSP_F32 && out_dtype != FUSP_BF16 && out_dtype != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "reshard: out_dtype must be f32, bf16 or f16");
  LayerCall call;
  FUSP_CHECK(group_of(c, group, &call.grp));
  call.reshard_in = true;
  call.rq = q_out;
  call.rk = k_out;
  call.rv = v_out;
  call.rdt = out_dtype;
  fusp_comm_options o{};
  o.out_dtype = FUSP_F32;
  if (opts) o = *opts;
  o.pipelined_ring = 0;
  return run_layer(c, Mode::kUlysses, 1, q, k, v, in_dtype, ls, nullptr, nullptr, &o,
                   reinterpret_cast<cudaStream_t>(stream), false, nullptr, nullptr, &call);
}

fusp_status fusp_ulysses_output_reshard(fusp_ctx c, fusp_group group, const void* o, fusp_dtype dtype,
                                        fusp_shape4 o_shape, void* out, fusp_stream_t stream) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  LayerCall call;
  FUSP_CHECK(group_of(c, group, &call.grp));
  const int u = call.grp ? call.grp->size() : c->world;
  if (o_shape.s % u != 0)  // protocols.cpp:185-188
    return set_error(FUSP_ERR_SHAPE, "ulysses: gathered sequence length S=" + std::to_string(o_shape.s) +
                                         " not divisible by ulysses dimension U=" + std::to_string(u));
  call.reshard_out = o;
  fusp_comm_options opt{};
  opt.out_dtype = dtype;
  const fusp_shape4 ls{o_shape.b, o_shape.h * u, o_shape.s / u, o_shape.d};
  return run_layer(c, Mode::kUlysses, 1, nullptr, nullptr, nullptr, dtype, ls, out, nullptr, &opt,
                   reinterpret_cast<cudaStream_t>(stream), false, nullptr, nullptr, &call);
}

fusp_status fusp_ulysses_attention(fusp_ctx c, const void* q, const void* k, const void* v,
                                   fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                                   const fusp_comm_options* opts, fusp_stream_t stream) {
  return run_layer(c, Mode::kUlysses, 1, q, k, v, in_dtype, ls, out, nullptr, opts,
                   reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_ring_attention(fusp_ctx c, const void* q, const void* k, const void* v,
                                fusp_dtype in_dtype, fusp_shape4 ls, void* out, float* lse,
                                const fusp_comm_options* opts, fusp_stream_t stream) {
  return run_layer(c, Mode::kRing, c ? c->world : 1, q, k, v, in_dtype, ls, out, lse, opts,
                   reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_usp_attention_host(fusp_ctx c, int ring_dim, const void* q, const void* k,
                                    const void* v, fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                                    const fusp_comm_options* opts, fusp_stream_t stream) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  FUSP_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fusp_comm_options o{};
  o.out_dtype = FUSP_F32;
  if (opts) o = *opts;
  const int out_dt = o.out_dtype;
  // Validate the whole call first (shape / mesh errors as the unchunked layer reports them).
  FUSP_CHECK(run_layer(c, Mode::kUsp, ring_dim, q, k, v, in_dtype, ls, out, nullptr, &o, s, true));
  // Heads are independent through the whole layer, so the host path pipelines head chunks:
  // H2D of chunk i+1 (copy stream) || layer on chunk i (caller's stream) || D2H of chunk i-1
  // (second copy stream).  Chunks are a multiple of the Ulysses degree so every chunk is a
  // valid USP layer; every rank picks the same chunking, so collectives stay matched.
  const int U = c->world / (ring_dim > 0 ? ring_dim : 1);
  // At most 4 equal chunks dividing H (tuning knob FUSP_HOST_CHUNKS): PCIe moves larger copies
  // faster (FLUX U=1: H2D per chunk ~50 GB/s at 4 chunks, ~45 GB/s at 8 with the D2H running
  // alongside), and that outweighs the longer pipeline tail -- 1.87 ms per layer vs 2.10 ms at
  // 8 chunks.  Chunks halving in size ([12, 6, 3, 2, 1] heads, a shorter tail) measured
  // 1.90-1.93 ms (tools/e2e_probe.py): the PCIe rate, not the tail, is what bounds this path.
  static const int max_chunks = [] {
    const char* e = getenv("FUSP_HOST_CHUNKS");
    const int n = e ? atoi(e) : 4;
    return n > 0 ? n : 4;
  }();
  // per-tensor FP8 quantizes over ALL local heads (fp8.cpp:107-123): one chunk keeps the
  // reference's single scale; per-block scales are per head, so chunking is exact there
  const bool whole = o.fp8_kv && !o.fp8_block;
  int hcu = static_cast<int>(ls.h);
  for (int cand = U; cand <= ls.h && !whole; cand += U)
    if (ls.h % cand == 0 && ls.h / cand <= max_chunks) { hcu = cand; break; }
  const std::vector<int> sizes(static_cast<size_t>(ls.h / hcu), hcu);
  const int nch = static_cast<int>(sizes.size());
  const int hc = sizes[0];  // the largest chunk sizes the staging slots
  const size_t esz_in = dtype_size(in_dtype), esz_out = dtype_size(out_dt);
  const size_t head_elems = size_t(ls.s * ls.d);
  const size_t chunk_in = size_t(ls.b) * hc * head_elems * esz_in;
  const size_t chunk_out = size_t(ls.b) * hc * head_elems * esz_out;
  // device staging (its own allocation: the arena belongs to the layer), two slots
  if (!c->host) {
    auto h = std::make_unique<HostStage>();
    FUSP_CUDA(cudaStreamCreateWithFlags(&h->h2d, cudaStreamNonBlocking));
    for (int x = 0; x < 2; ++x) {
      FUSP_CUDA(cudaStreamCreateWithFlags(&h->h2d_x[x], cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i)
        FUSP_CUDA(cudaEventCreateWithFlags(&h->in_ready_x[x][i], cudaEventDisableTiming));
    }
    FUSP_CUDA(cudaStreamCreateWithFlags(&h->d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      FUSP_CUDA(cudaEventCreateWithFlags(&h->in_ready[i], cudaEventDisableTiming));
      FUSP_CUDA(cudaEventCreateWithFlags(&h->computed[i], cudaEventDisableTiming));
      FUSP_CUDA(cudaEventCreateWithFlags(&h->out_done[i], cudaEventDisableTiming));
    }
    FUSP_CUDA(cudaMalloc(&h->flag, 256));
    c->host = std::move(h);
  }
  HostStage& st = *c->host;
  const size_t slot = 3 * align_up(chunk_in, 256) + align_up(chunk_out, 256);
  if (st.bytes < 2 * slot) {
    if (st.d) FUSP_CUDA(cudaFree(st.d));
    FUSP_CUDA(cudaMalloc(&st.d, 2 * slot));
    st.bytes = 2 * slot;
  }
  const bool check = o.check_finite != 0;
  o.check_finite = 0;  // checked per chunk on the device below, reported after the pipeline
  if (check) FUSP_CUDA(cudaMemsetAsync(st.flag, 0, 4, s));
  const size_t pitch_in = size_t(ls.h) * head_elems * esz_in, pitch_out = size_t(ls.h) * head_elems * esz_out;
  FUSP_CUDA(cudaEventRecord(st.computed[0], s));  // order the copy streams after prior work
  FUSP_CUDA(cudaStreamWaitEvent(st.h2d, st.computed[0], 0));
  // Q, K, V copies over 1-3 H2D streams (knob FUSP_HOST_H2D_STREAMS, default 1)
  static const int n_h2d = [] {
    const char* e = getenv("FUSP_HOST_H2D_STREAMS");
    const int n = e ? atoi(e) : 1;
    return n < 1 ? 1 : (n > 3 ? 3 : n);
  }();
  cudaStream_t h2ds[3] = {st.h2d, st.h2d_x[0], st.h2d_x[1]};
  for (int x = 1; x < n_h2d; ++x) FUSP_CUDA(cudaStreamWaitEvent(h2ds[x], st.computed[0], 0));
  int h0 = 0;  // first head of the chunk
  for (int i = 0; i < nch; h0 += sizes[i], ++i) {
    const int b = i % 2;
    const int hi = sizes[i];
    fusp_shape4 cs = ls;
    cs.h = hi;
    const size_t chunk_in = size_t(ls.b) * hi * head_elems * esz_in;
    const size_t chunk_out = size_t(ls.b) * hi * head_elems * esz_out;
    char* d = static_cast<char*>(st.d) + b * slot;
    void* dq = d;
    void* dk = d + align_up(size_t(ls.b) * hc * head_elems * esz_in, 256);
    void* dv = d + 2 * align_up(size_t(ls.b) * hc * head_elems * esz_in, 256);
    void* dout = d + 3 * align_up(size_t(ls.b) * hc * head_elems * esz_in, 256);
    const size_t off_in = size_t(h0) * head_elems * esz_in;
    const size_t off_out = size_t(h0) * head_elems * esz_out;
    // slot b's inputs were last read by the layer on chunk i-2
    if (i >= 2)
      for (int x = 0; x < n_h2d; ++x) FUSP_CUDA(cudaStreamWaitEvent(h2ds[x], st.computed[b], 0));
    const void* src[3] = {q, k, v};
    void* dst[3] = {dq, dk, dv};
    for (int t = 0; t < 3; ++t) {
      cudaStream_t hs = h2ds[t % n_h2d];
      if (ls.b == 1)
        FUSP_CUDA(cudaMemcpyAsync(dst[t], static_cast<const char*>(src[t]) + off_in, chunk_in,
                                  cudaMemcpyHostToDevice, hs));
      else
        FUSP_CUDA(cudaMemcpy2DAsync(dst[t], chunk_in / ls.b, static_cast<const char*>(src[t]) + off_in,
                                    pitch_in, chunk_in / ls.b, ls.b, cudaMemcpyHostToDevice, hs));
    }
    FUSP_CUDA(cudaEventRecord(st.in_ready[b], st.h2d));
    FUSP_CUDA(cudaStreamWaitEvent(s, st.in_ready[b], 0));
    for (int x = 1; x < n_h2d; ++x) {
      FUSP_CUDA(cudaEventRecord(st.in_ready_x[x - 1][b], h2ds[x]));
      FUSP_CUDA(cudaStreamWaitEvent(s, st.in_ready_x[x - 1][b], 0));
    }
    // slot b's output was last read by the D2H of chunk i-2
    if (i >= 2) FUSP_CUDA(cudaStreamWaitEvent(s, st.out_done[b], 0));
    if (check) {
      const int64_t n = int64_t(ls.b) * hi * int64_t(head_elems);
      FUSP_CHECK(launch_finite(dq, in_dtype, n, st.flag, s));
      FUSP_CHECK(launch_finite(dk, in_dtype, n, st.flag, s));
      FUSP_CHECK(launch_finite(dv, in_dtype, n, st.flag, s));
    }
    FUSP_CHECK(run_layer(c, Mode::kUsp, ring_dim, dq, dk, dv, in_dtype, cs, dout, nullptr, &o, s));
    FUSP_CUDA(cudaEventRecord(st.computed[b], s));
    FUSP_CUDA(cudaStreamWaitEvent(st.d2h, st.computed[b], 0));
    if (ls.b == 1)
      FUSP_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + off_out, dout, chunk_out, cudaMemcpyDeviceToHost,
                                st.d2h));
    else
      FUSP_CUDA(cudaMemcpy2DAsync(static_cast<char*>(out) + off_out, pitch_out, dout, chunk_out / ls.b,
                                  chunk_out / ls.b, ls.b, cudaMemcpyDeviceToHost, st.d2h));
    FUSP_CUDA(cudaEventRecord(st.out_done[b], st.d2h));
  }
  FUSP_CUDA(cudaStreamWaitEvent(s, st.out_done[(nch - 1) % 2], 0));
  if (nch >= 2) FUSP_CUDA(cudaStreamWaitEvent(s, st.out_done[(nch - 2) % 2], 0));
  uint32_t bad = 0;
  if (check) FUSP_CUDA(cudaMemcpyAsync(&bad, st.flag, 4, cudaMemcpyDeviceToHost, s));
  FUSP_CHECK(c->comm->wait(s, sync_timeout_s(), "usp_attention_host"));
  if (bad)  // check_local_qkv (protocols.cpp:102-104); the output is unspecified
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "usp: non-finite element in protocol input");
  return FUSP_OK;
}

fusp_status fusp_graph_capture_usp(fusp_ctx c, int ring_dim, const void* q, const void* k,
                                   const void* v, fusp_dtype in_dtype, fusp_shape4 ls, void* out,
                                   const fusp_comm_options* opts, int layers,
                                   int64_t in_stride, int64_t out_stride, fusp_stream_t stream,
                                   fusp_graph* graph) {
  clear_error();
  if (!c) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context");
  if (!c->comm->capturable() && !c->peer)
    return set_error(FUSP_ERR_UNSUPPORTED,
                     "graph capture needs an NCCL context, a world-1 local context, or peer windows");
  if (opts && opts->check_finite)
    return set_error(FUSP_ERR_UNSUPPORTED, "check_finite synchronizes; not capturable");
  FUSP_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // the graph gets its own workspace, sized before capture (no allocation inside the graph):
  // later eager calls on the context may regrow the context's without touching it
  auto* g = new fusp_graph_s;
  g->device = c->device;
  g->ctx = c;
  c->ws = &g->ws;
  fusp_status st0 = run_layer(c, Mode::kUsp, ring_dim, q, k, v, in_dtype, ls, out, nullptr, opts, s, true);
  if (st0 == FUSP_OK && cudaStreamSynchronize(s) != cudaSuccess) st0 = set_cuda_error(cudaGetLastError(), "cudaStreamSynchronize");
  if (st0 != FUSP_OK) {
    c->ws = &c->own;
    g->ws.release();
    delete g;
    return st0;
  }
  c->capturing = true;
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  fusp_status st = e == cudaSuccess ? FUSP_OK : set_cuda_error(e, "cudaStreamBeginCapture");
  for (int i = 0; i < layers && st == FUSP_OK; ++i) {
    const char* qi = static_cast<const char*>(q) + i * in_stride;
    const char* ki = static_cast<const char*>(k) + i * in_stride;
    const char* vi = static_cast<const char*>(v) + i * in_stride;
    char* oi = static_cast<char*>(out) + i * out_stride;
    st = run_layer(c, Mode::kUsp, ring_dim, qi, ki, vi, in_dtype, ls, oi, nullptr, opts, s);
  }
  cudaGraph_t graph_raw = nullptr;
  e = cudaStreamEndCapture(s, &graph_raw);
  c->capturing = false;
  c->ws = &c->own;
  if (st == FUSP_OK && e != cudaSuccess) st = set_cuda_error(e, "cudaStreamEndCapture");
  if (st == FUSP_OK) {
    g->graph = graph_raw;
    e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) st = set_cuda_error(e, "cudaGraphInstantiate");
  } else if (graph_raw) {
    cudaGraphDestroy(graph_raw);
  }
  if (st != FUSP_OK) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    g->ws.release();
    delete g;
    return st;
  }
  c->live_graphs++;
  *graph = g;
  return FUSP_OK;
}

fusp_status fusp_graph_launch(fusp_graph g, fusp_stream_t stream) {
  clear_error();
  FUSP_CUDA(cudaSetDevice(g->device));
  FUSP_CUDA(cudaGraphLaunch(g->exec, reinterpret_cast<cudaStream_t>(stream)));
  return FUSP_OK;
}

fusp_status fusp_graph_destroy(fusp_graph g) {
  if (!g) return FUSP_OK;
  cudaSetDevice(g->device);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  g->ws.release();  // cudaFree waits for a replay still in flight
  if (g->block_ws) cudaFree(g->block_ws);
  if (g->ctx) g->ctx->live_graphs--;
  delete g;
  return FUSP_OK;
}

// CUDA graph of `layers` back-to-back fusp_usp_block calls (the whole MMDiT attention block:
// QKV projection -> USP layer -> output projection).  Collective like the block itself.  The
// graph owns its layer workspace and block buffers: sized by one eager block (which also
// computes y for layer 0), then captured; eager calls on the context may later regrow the
// context's own without touching them.  At world > 1 only the peer-memory path (ring_dim 1)
// or an NCCL context is capturable -- the in-process fabric's rendezvous is host code.
fusp_status fusp_graph_capture_block(fusp_ctx c, int ring_dim, const void* x, fusp_dtype x_dtype,
                                     int64_t batch, int64_t s_local, int64_t channels,
                                     const void* w_qkv, int heads, const fusp_qk_prologue* prologue,
                                     const void* w_out, int64_t n_out, void* y, fusp_dtype y_dtype,
                                     const fusp_comm_options* opts, int layers, int64_t x_stride,
                                     int64_t y_stride, fusp_stream_t stream, fusp_graph* graph) {
  clear_error();
  if (!c || !graph) return set_error(FUSP_ERR_INVALID_ARGUMENT, "null context or graph");
  if (!c->comm->capturable() && !c->peer)
    return set_error(FUSP_ERR_UNSUPPORTED,
                     "graph capture needs an NCCL context, a world-1 local context, or peer windows");
  if (opts && opts->check_finite)
    return set_error(FUSP_ERR_UNSUPPORTED, "check_finite synchronizes; not capturable");
  if (layers < 1) return set_error(FUSP_ERR_INVALID_ARGUMENT, "graph capture: layers < 1");
  FUSP_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto* g = new fusp_graph_s;
  g->device = c->device;
  g->ctx = c;
  void* own_bws = c->block_ws;
  const size_t own_bbytes = c->block_ws_bytes;
  c->ws = &g->ws;
  c->block_ws = nullptr;
  c->block_ws_bytes = 0;
  auto restore = [&]() {
    c->ws = &c->own;
    g->block_ws = c->block_ws;
    c->block_ws = own_bws;
    c->block_ws_bytes = own_bbytes;
  };
  auto fail = [&](fusp_status st) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    cudaStreamSynchronize(s);
    g->ws.release();
    if (g->block_ws) cudaFree(g->block_ws);
    delete g;
    return st;
  };
  fusp_status st0 = fusp_usp_block(c, ring_dim, x, x_dtype, batch, s_local, channels, w_qkv, heads,
                                   prologue, w_out, n_out, y, y_dtype, opts, stream);
  if (st0 == FUSP_OK && cudaStreamSynchronize(s) != cudaSuccess)
    st0 = set_cuda_error(cudaGetLastError(), "cudaStreamSynchronize");
  if (st0 != FUSP_OK) {
    restore();
    return fail(st0);
  }
  c->capturing = true;
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  fusp_status st = e == cudaSuccess ? FUSP_OK : set_cuda_error(e, "cudaStreamBeginCapture");
  for (int i = 0; i < layers && st == FUSP_OK; ++i)
    st = fusp_usp_block(c, ring_dim, static_cast<const char*>(x) + i * x_stride, x_dtype, batch, s_local,
                        channels, w_qkv, heads, prologue, w_out, n_out,
                        static_cast<char*>(y) + i * y_stride, y_dtype, opts, stream);
  cudaGraph_t graph_raw = nullptr;
  e = cudaStreamEndCapture(s, &graph_raw);
  c->capturing = false;
  restore();
  if (st == FUSP_OK && e != cudaSuccess) st = set_cuda_error(e, "cudaStreamEndCapture");
  if (st == FUSP_OK) {
    g->graph = graph_raw;
    e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) st = set_cuda_error(e, "cudaGraphInstantiate");
  } else if (graph_raw) {
    cudaGraphDestroy(graph_raw);
  }
  if (st != FUSP_OK) return fail(st);
  c->live_graphs++;
  *graph = g;
  return FUSP_OK;
}

}  // extern "C"
