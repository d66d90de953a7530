// Header-only C++ façade that re-exposes the reference's uspsim API
// (/root/reference/proj/include/uspsim/{tensor,fp8,mesh,fabric,protocols}.hpp) on top of
// the fastusp C ABI (include/fastusp.h).  A harness written against uspsim:: compiles
// against fastusp::uspsim:: unchanged: host Tensor4 in, host Tensor4 out, one thread per
// rank under run_protocol, and the same exception classes carrying the same messages.
//
// Every computation runs in libfastusp.so's sm_100a kernels; host tensors are staged to
// the rank's device for each call (the reference's calling convention).  Link with
// -lfastusp -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../fastusp.h"

namespace fastusp {
namespace uspsim {

// ---- exceptions (tensor.hpp:13, mesh.hpp:17, fabric.hpp:106-126) ------------------------------
class ShapeError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class MeshError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class FabricError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeadlockError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class WorkerFailure : public std::runtime_error {
 public:
  WorkerFailure(int rank, const std::string& what)
      : std::runtime_error("worker " + std::to_string(rank) + " failed: " + what), rank_(rank) {}
  int rank() const { return rank_; }

 private:
  int rank_;
};

inline void check(fusp_status st) {
  if (st == FUSP_OK) return;
  const std::string msg = fusp_last_error();
  switch (st) {
    case FUSP_ERR_SHAPE: throw ShapeError(msg);
    case FUSP_ERR_MESH: throw MeshError(msg);
    case FUSP_ERR_COMM: throw FabricError(msg);
    case FUSP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FUSP_ERR_DEADLOCK: throw DeadlockError(msg);
    default: throw std::runtime_error("fastusp: " + msg);
  }
}

// ---- tensors (tensor.hpp:18-83) ----------------------------------------------------------------
struct Shape4 {
  int64_t b = 0, h = 0, s = 0, d = 0;
  int64_t count() const { return b * h * s * d; }
  bool operator==(const Shape4&) const = default;
  std::string str() const {
    return "[" + std::to_string(b) + "," + std::to_string(h) + "," + std::to_string(s) + "," +
           std::to_string(d) + "]";
  }
  fusp_shape4 c() const { return {b, h, s, d}; }
};

template <typename T>
struct Tensor4T {
  Shape4 shape{};
  std::vector<T> data;
  Tensor4T() = default;
  explicit Tensor4T(Shape4 sh) : shape(sh), data(static_cast<size_t>(sh.count()), T(0)) {}
  Tensor4T(Shape4 sh, std::vector<T> v) : shape(sh), data(std::move(v)) {
    if (static_cast<int64_t>(data.size()) != sh.count())
      throw ShapeError("tensor data length " + std::to_string(data.size()) +
                       " does not match shape " + sh.str());
  }
  int64_t index(int64_t b, int64_t h, int64_t s, int64_t d) const {
    return ((b * shape.h + h) * shape.s + s) * shape.d + d;
  }
  T& at(int64_t b, int64_t h, int64_t s, int64_t d) { return data[index(b, h, s, d)]; }
  const T& at(int64_t b, int64_t h, int64_t s, int64_t d) const { return data[index(b, h, s, d)]; }
  Tensor4T slice_heads(int64_t h0, int64_t count) const {  // tensor.cpp:35-46
    if (h0 < 0 || count < 0 || h0 + count > shape.h)
      throw ShapeError("head slice [" + std::to_string(h0) + "," + std::to_string(h0 + count) +
                       ") out of range for H=" + std::to_string(shape.h));
    Tensor4T r(Shape4{shape.b, count, shape.s, shape.d});
    for (int64_t b = 0; b < shape.b; ++b)
      for (int64_t h = 0; h < count; ++h)
        std::memcpy(&r.at(b, h, 0, 0), &at(b, h0 + h, 0, 0), sizeof(T) * shape.s * shape.d);
    return r;
  }
  Tensor4T slice_seq(int64_t s0, int64_t count) const {
    if (s0 < 0 || count < 0 || s0 + count > shape.s)
      throw ShapeError("sequence slice [" + std::to_string(s0) + "," + std::to_string(s0 + count) +
                       ") out of range for S=" + std::to_string(shape.s));
    Tensor4T r(Shape4{shape.b, shape.h, count, shape.d});
    for (int64_t b = 0; b < shape.b; ++b)
      for (int64_t h = 0; h < shape.h; ++h)
        std::memcpy(&r.at(b, h, 0, 0), &at(b, h, s0, 0), sizeof(T) * count * shape.d);
    return r;
  }
};
using Tensor4 = Tensor4T<float>;
using CodeTensor = Tensor4T<uint8_t>;

struct AttnResult {
  Tensor4 out;
  std::vector<float> lse;
};

// ---- device staging --------------------------------------------------------------------------
namespace detail {
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t n) {
    if (n && cudaMalloc(&p, n) != cudaSuccess) throw std::runtime_error("fastusp: cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};
inline void h2d(void* d, const void* h, size_t n) {
  if (n && cudaMemcpy(d, h, n, cudaMemcpyHostToDevice) != cudaSuccess)
    throw std::runtime_error("fastusp: H2D copy");
}
inline void d2h(void* h, const void* d, size_t n) {
  if (n && cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost) != cudaSuccess)
    throw std::runtime_error("fastusp: D2H copy");
}
}  // namespace detail

// ---- fp8 (fp8.hpp:15-49) ----------------------------------------------------------------------
inline constexpr float kFp8Max = 448.0f;
inline constexpr uint8_t kFp8MaxCode = 0x7E;
inline constexpr uint8_t kFp8NanCode = 0x7F;

struct QuantizedTensor {
  CodeTensor codes;
  float scale = 1.0f;
  const Shape4& shape() const { return codes.shape; }
  // fp8.cpp:100-105: a head slice keeps the tensor-wide scale
  QuantizedTensor slice_heads(int64_t h0, int64_t count) const {
    QuantizedTensor r;
    r.scale = scale;
    r.codes = codes.slice_heads(h0, count);
    return r;
  }
};

inline QuantizedTensor quantize(const Tensor4& x) {
  const size_t n = x.data.size();
  detail::DevBuf dx(n * 4), dc(n), ds(4);
  detail::h2d(dx.p, x.data.data(), n * 4);
  check(fusp_quantize_e4m3(dx.p, FUSP_F32, static_cast<int64_t>(n), dc.as<uint8_t>(),
                           ds.as<float>(), 1, nullptr));
  QuantizedTensor q;
  q.codes = CodeTensor(x.shape);
  detail::d2h(q.codes.data.data(), dc.p, n);
  detail::d2h(&q.scale, ds.p, 4);
  return q;
}

inline Tensor4 dequantize(const QuantizedTensor& q) {
  const size_t n = q.codes.data.size();
  detail::DevBuf dc(n), ds(4), dy(n * 4);
  detail::h2d(dc.p, q.codes.data.data(), n);
  detail::h2d(ds.p, &q.scale, 4);
  check(fusp_dequantize_e4m3(dc.as<uint8_t>(), ds.as<float>(), static_cast<int64_t>(n), dy.p,
                             FUSP_F32, nullptr));
  Tensor4 r(q.codes.shape);
  detail::d2h(r.data.data(), dy.p, n * 4);
  return r;
}

inline uint8_t encode_e4m3(float x) {
  detail::DevBuf dx(4), dc(1);
  detail::h2d(dx.p, &x, 4);
  check(fusp_encode_e4m3(dx.as<float>(), 1, dc.as<uint8_t>(), nullptr));
  uint8_t c = 0;
  detail::d2h(&c, dc.p, 1);
  return c;
}

inline float decode_e4m3(uint8_t code) {
  detail::DevBuf dc(1), dy(4);
  detail::h2d(dc.p, &code, 1);
  check(fusp_decode_e4m3(dc.as<uint8_t>(), 1, dy.as<float>(), nullptr));
  float y = 0;
  detail::d2h(&y, dy.p, 4);
  return y;
}

// ---- attention (tensor.hpp:85-98) --------------------------------------------------------------
inline AttnResult attention_with_lse(const Tensor4& q, const Tensor4& k, const Tensor4& v) {
  if (q.shape.h != k.shape.h || q.shape.h != v.shape.h)
    throw ShapeError("attention: head axis mismatch, Q H=" + std::to_string(q.shape.h) +
                     " K H=" + std::to_string(k.shape.h) + " V H=" + std::to_string(v.shape.h));
  if (k.shape.s != v.shape.s)
    throw ShapeError("attention: sequence axis mismatch between K S=" + std::to_string(k.shape.s) +
                     " and V S=" + std::to_string(v.shape.s));
  const size_t nq = q.data.size(), nk = k.data.size();
  detail::DevBuf dq(nq * 4), dk(nk * 4), dv(nk * 4), dout(nq * 4),
      dl(static_cast<size_t>(q.shape.b * q.shape.h * q.shape.s) * 4);
  detail::h2d(dq.p, q.data.data(), nq * 4);
  detail::h2d(dk.p, k.data.data(), nk * 4);
  detail::h2d(dv.p, v.data.data(), nk * 4);
  check(fusp_attention_with_lse(dq.p, dk.p, dv.p, FUSP_F32, q.shape.c(), k.shape.s, dout.p,
                                FUSP_F32, dl.as<float>(), nullptr));
  AttnResult r;
  r.out = Tensor4(q.shape);
  r.lse.resize(static_cast<size_t>(q.shape.b * q.shape.h * q.shape.s));
  detail::d2h(r.out.data.data(), dout.p, nq * 4);
  detail::d2h(r.lse.data(), dl.p, r.lse.size() * 4);
  return r;
}

// attention_reference (tensor.cpp:185-191): attention_with_lse without the LSE
inline Tensor4 attention_reference(const Tensor4& q, const Tensor4& k, const Tensor4& v) {
  return attention_with_lse(q, k, v).out;
}

// merge_lse (tensor.cpp:204-243) on the device merge kernel
inline AttnResult merge_lse(const AttnResult& a, const AttnResult& b) {
  if (!(a.out.shape == b.out.shape))
    throw ShapeError("merge_lse: output shapes differ, " + a.out.shape.str() + " vs " + b.out.shape.str());
  if (a.lse.size() != b.lse.size())
    throw ShapeError("merge_lse: lse lengths differ, " + std::to_string(a.lse.size()) + " vs " +
                     std::to_string(b.lse.size()));
  const size_t n = a.out.data.size(), m = a.lse.size();
  detail::DevBuf o1(n * 4), o2(n * 4), l1(m * 4), l2(m * 4), ro(n * 4), rl(m * 4);
  detail::h2d(o1.p, a.out.data.data(), n * 4);
  detail::h2d(o2.p, b.out.data.data(), n * 4);
  detail::h2d(l1.p, a.lse.data(), m * 4);
  detail::h2d(l2.p, b.lse.data(), m * 4);
  check(fusp_merge_lse(o1.as<float>(), l1.as<float>(), o2.as<float>(), l2.as<float>(), a.out.shape.c(),
                       ro.as<float>(), rl.as<float>(), nullptr));
  AttnResult r;
  r.out = Tensor4(a.out.shape);
  r.lse.resize(m);
  detail::d2h(r.out.data.data(), ro.p, n * 4);
  detail::d2h(r.lse.data(), rl.p, m * 4);
  return r;
}

// ---- mesh (mesh.hpp:22-50) ---------------------------------------------------------------------
struct ProcessGroup {
  std::vector<int> members;
  int size() const { return static_cast<int>(members.size()); }
  int position_of(int rank) const {
    for (size_t i = 0; i < members.size(); ++i)
      if (members[i] == rank) return static_cast<int>(i);
    return -1;
  }
  std::string key() const {
    std::string k;
    for (size_t i = 0; i < members.size(); ++i) k += (i ? "," : "") + std::to_string(members[i]);
    return k;
  }
};

struct Mesh2D {
  int n = 1, r = 1, u = 1;
  std::vector<ProcessGroup> ring_groups, ulysses_groups;
  int ring_index(int rank) const { return rank / u; }
  int ulysses_index(int rank) const { return rank % u; }
  const ProcessGroup& ring_group(int rank) const { return ring_groups.at(ulysses_index(rank)); }
  const ProcessGroup& ulysses_group(int rank) const { return ulysses_groups.at(ring_index(rank)); }
};

inline Mesh2D make_mesh(int n, int r) {
  std::vector<int> ug(static_cast<size_t>(n > 0 ? n : 1)), rg(ug.size());
  check(fusp_mesh_make(n, r, ug.data(), rg.data()));
  Mesh2D m;
  m.n = n;
  m.r = r;
  m.u = n / r;
  for (int i = 0; i < m.r; ++i)
    m.ulysses_groups.push_back({std::vector<int>(ug.begin() + i * m.u, ug.begin() + (i + 1) * m.u)});
  for (int j = 0; j < m.u; ++j)
    m.ring_groups.push_back({std::vector<int>(rg.begin() + j * m.r, rg.begin() + (j + 1) * m.r)});
  return m;
}

inline Mesh2D build_mesh(int n, int max_ring_dim_size, int heads) {
  int r = 0, u = 0;
  check(fusp_mesh_build(n, max_ring_dim_size, heads, &r, &u));
  return make_mesh(n, r);
}

// ---- ranks (fabric.hpp:136-180) ------------------------------------------------------------------
struct CommOptions {
  bool fp8_kv = false;
  bool pipelined_ring = false;
};

class WorkerContext {
 public:
  WorkerContext(fusp_ctx c) : c_(c) {}
  ~WorkerContext() {
    for (auto& g : groups_) fusp_group_destroy(g.second);
  }
  WorkerContext(const WorkerContext&) = delete;
  WorkerContext& operator=(const WorkerContext&) = delete;
  int rank() const { return fusp_ctx_rank(c_); }
  int world_size() const { return fusp_ctx_world(c_); }
  fusp_ctx handle() const { return c_; }
  // The fastusp handle of a ProcessGroup on this rank (created on first use; run_protocol's
  // in-process fabric needs no collective setup).  The world in rank order is NULL.
  fusp_group group(const ProcessGroup& g) {
    bool world = g.size() == world_size();
    for (int i = 0; i < g.size() && world; ++i) world = g.members[i] == i;
    if (world) return nullptr;
    for (auto& e : groups_)
      if (e.first == g.members) return e.second;
    fusp_group h = nullptr;
    check(fusp_group_create(c_, g.members.data(), g.size(), &h));
    groups_.emplace_back(g.members, h);
    return h;
  }

 private:
  fusp_ctx c_;
  std::vector<std::pair<std::vector<int>, fusp_group>> groups_;
};

using WorkerProgram = std::function<void(WorkerContext&)>;

// run_protocol (fabric.hpp:180): n host threads over an in-process fabric on `device`.
inline void run_protocol(int n, const WorkerProgram& program, int device = 0) {
  fusp_fabric fab = nullptr;
  check(fusp_fabric_create(n, &fab));
  std::vector<std::string> errs(static_cast<size_t>(n));
  std::vector<std::thread> th;
  for (int r = 0; r < n; ++r) {
    th.emplace_back([&, r] {
      try {
        cudaSetDevice(device);
        fusp_ctx c = nullptr;
        check(fusp_ctx_create_local(fab, r, device, &c));
        WorkerContext ctx(c);
        try {
          program(ctx);
        } catch (...) {
          fusp_ctx_destroy(c);
          throw;
        }
        fusp_ctx_destroy(c);
      } catch (const std::exception& e) {
        errs[r] = e.what();
      }
    });
  }
  for (auto& t : th) t.join();
  fusp_fabric_destroy(fab);
  for (int r = 0; r < n; ++r)
    if (!errs[r].empty()) throw WorkerFailure(r, errs[r]);
}

// ---- protocols (protocols.hpp:28-71) -------------------------------------------------------------
inline std::vector<Tensor4> split_sequence(const Tensor4& full, int count) {
  if (count < 1) throw ShapeError("split_sequence: count must be >= 1");
  if (full.shape.s % count != 0)
    throw ShapeError("split_sequence: S=" + std::to_string(full.shape.s) +
                     " not divisible by shard count " + std::to_string(count));
  std::vector<Tensor4> out;
  const int64_t c = full.shape.s / count;
  for (int i = 0; i < count; ++i) out.push_back(full.slice_seq(i * c, c));
  return out;
}

inline Tensor4 gather_output(const std::vector<Tensor4>& shards) {
  Shape4 s = shards.at(0).shape;
  int64_t total = 0;
  for (const auto& t : shards) total += t.shape.s;
  Tensor4 r(Shape4{s.b, s.h, total, s.d});
  int64_t off = 0;
  for (const auto& t : shards) {
    for (int64_t b = 0; b < s.b; ++b)
      for (int64_t h = 0; h < s.h; ++h)
        std::memcpy(&r.at(b, h, off, 0), &t.at(b, h, 0, 0), sizeof(float) * t.shape.s * s.d);
    off += t.shape.s;
  }
  return r;
}

// ShardSpec / gather_shards (protocols.hpp:17-35, protocols.cpp:25-50): reassembly with
// explicit coverage checking (host-side, like the reference).
struct ShardSpec {
  enum class Axis { kSequence, kHead };
  Axis axis = Axis::kSequence;
  int index = 0;
  int count = 1;
};

inline Tensor4 gather_shards(const std::vector<std::pair<ShardSpec, Tensor4>>& shards) {
  if (shards.empty()) throw ShapeError("gather_shards: no shards");
  const int count = shards.front().first.count;
  std::vector<const Tensor4*> ordered(static_cast<size_t>(count > 0 ? count : 0), nullptr);
  for (const auto& [spec, t] : shards) {
    if (spec.axis != ShardSpec::Axis::kSequence)
      throw ShapeError("gather_shards: only sequence-axis shards are gathered");
    if (spec.count != count)
      throw ShapeError("gather_shards: inconsistent shard counts " + std::to_string(spec.count) +
                       " vs " + std::to_string(count));
    if (spec.index < 0 || spec.index >= count)
      throw ShapeError("gather_shards: shard index " + std::to_string(spec.index) + " outside [0," +
                       std::to_string(count) + ")");
    auto& slot = ordered[static_cast<size_t>(spec.index)];
    if (slot != nullptr)
      throw ShapeError("gather_shards: shard index " + std::to_string(spec.index) + " covered twice");
    slot = &t;
  }
  std::vector<Tensor4> parts;
  for (int i = 0; i < count; ++i) {
    if (!ordered[static_cast<size_t>(i)])
      throw ShapeError("gather_shards: gap in coverage at shard index " + std::to_string(i));
    parts.push_back(*ordered[static_cast<size_t>(i)]);
  }
  return gather_output(parts);
}

namespace detail {
inline fusp_comm_options c_opts(const CommOptions& opts) {
  fusp_comm_options o{};
  o.fp8_kv = opts.fp8_kv;
  o.pipelined_ring = opts.pipelined_ring;
  o.out_dtype = FUSP_F32;
  o.check_finite = 1;
  return o;
}
inline void check_local(const Tensor4& q, const Tensor4& k, const Tensor4& v, const char* where) {
  if (!(q.shape == k.shape) || !(q.shape == v.shape))
    throw ShapeError(std::string(where) + ": local Q/K/V shapes differ: Q=" + q.shape.str() +
                     " K=" + k.shape.str() + " V=" + v.shape.str());
}
// Host tensors staged to the device around one collective call (the reference's convention).
struct Staged {
  DevBuf q, k, v;
  explicit Staged(const Tensor4& tq, const Tensor4& tk, const Tensor4& tv)
      : q(tq.data.size() * 4), k(tk.data.size() * 4), v(tv.data.size() * 4) {
    h2d(q.p, tq.data.data(), tq.data.size() * 4);
    h2d(k.p, tk.data.data(), tk.data.size() * 4);
    h2d(v.p, tv.data.data(), tv.data.size() * 4);
  }
};
}  // namespace detail

// ulysses_attention (protocols.hpp:47-48, protocols.cpp:207-214) over `group`
inline Tensor4 ulysses_attention(WorkerContext& ctx, const Tensor4& q, const Tensor4& k,
                                 const Tensor4& v, const ProcessGroup& group,
                                 const CommOptions& opts) {
  detail::check_local(q, k, v, "ulysses");
  const fusp_comm_options o = detail::c_opts(opts);
  detail::Staged d(q, k, v);
  detail::DevBuf out(q.data.size() * 4);
  check(fusp_ulysses_attention_group(ctx.handle(), ctx.group(group), d.q.p, d.k.p, d.v.p, FUSP_F32,
                                     q.shape.c(), out.p, nullptr, &o, nullptr));
  Tensor4 r(q.shape);
  detail::d2h(r.data.data(), out.p, q.data.size() * 4);
  return r;
}

namespace detail {
inline AttnResult ring(WorkerContext& ctx, const Tensor4& q, const Tensor4& k, const Tensor4& v,
                       const ProcessGroup& group, const CommOptions& opts, bool pipelined) {
  check_local(q, k, v, "ring");
  fusp_comm_options o = c_opts(opts);
  o.pipelined_ring = pipelined;
  Staged d(q, k, v);
  const size_t rows = static_cast<size_t>(q.shape.b * q.shape.h * q.shape.s);
  DevBuf out(q.data.size() * 4), lse(rows * 4);
  check(fusp_ring_attention_group(ctx.handle(), ctx.group(group), d.q.p, d.k.p, d.v.p, FUSP_F32,
                                  q.shape.c(), out.p, lse.as<float>(), &o, nullptr));
  AttnResult r;
  r.out = Tensor4(q.shape);
  r.lse.resize(rows);
  d2h(r.out.data.data(), out.p, q.data.size() * 4);
  d2h(r.lse.data(), lse.p, rows * 4);
  return r;
}
}  // namespace detail

// ring_attention_serial / _pipelined (protocols.hpp:54-65, protocols.cpp:237-319)
inline AttnResult ring_attention_serial(WorkerContext& ctx, const Tensor4& q, const Tensor4& k,
                                        const Tensor4& v, const ProcessGroup& group,
                                        const CommOptions& opts) {
  return detail::ring(ctx, q, k, v, group, opts, false);
}
inline AttnResult ring_attention_pipelined(WorkerContext& ctx, const Tensor4& q, const Tensor4& k,
                                           const Tensor4& v, const ProcessGroup& group,
                                           const CommOptions& opts) {
  return detail::ring(ctx, q, k, v, group, opts, true);
}

namespace detail {
// detail::Resharded / ulysses_input_reshard / ulysses_output_reshard (protocols.hpp:73-86)
struct Resharded {
  Tensor4 q, k, v;  // [B, H/U, S_span, D]
};

inline Resharded ulysses_input_reshard(WorkerContext& ctx, const Tensor4& q, const Tensor4& k,
                                       const Tensor4& v, const ProcessGroup& group,
                                       const CommOptions& opts) {
  check_local(q, k, v, "ulysses");
  const int u = group.size();
  if (u < 1 || q.shape.h % u != 0)
    throw ShapeError("ulysses: head count H=" + std::to_string(q.shape.h) +
                     " not divisible by ulysses dimension U=" + std::to_string(u));
  const fusp_comm_options o = c_opts(opts);
  Staged d(q, k, v);
  const Shape4 rs{q.shape.b, q.shape.h / u, q.shape.s * u, q.shape.d};
  const size_t n = static_cast<size_t>(rs.count()) * 4;
  DevBuf rq(n), rk(n), rv(n);
  check(fusp_ulysses_input_reshard(ctx.handle(), ctx.group(group), d.q.p, d.k.p, d.v.p, FUSP_F32,
                                   q.shape.c(), rq.p, rk.p, rv.p, FUSP_F32, &o, nullptr));
  Resharded r{Tensor4(rs), Tensor4(rs), Tensor4(rs)};
  d2h(r.q.data.data(), rq.p, n);
  d2h(r.k.data.data(), rk.p, n);
  d2h(r.v.data.data(), rv.p, n);
  return r;
}

inline Tensor4 ulysses_output_reshard(WorkerContext& ctx, const Tensor4& out, const ProcessGroup& group) {
  const int u = group.size();
  if (u < 1 || out.shape.s % u != 0)
    throw ShapeError("ulysses: gathered sequence length S=" + std::to_string(out.shape.s) +
                     " not divisible by ulysses dimension U=" + std::to_string(u));
  const size_t n = out.data.size() * 4;
  DevBuf o(n), res(n);
  h2d(o.p, out.data.data(), n);
  check(fusp_ulysses_output_reshard(ctx.handle(), ctx.group(group), o.p, FUSP_F32, out.shape.c(),
                                    res.p, nullptr));
  Tensor4 r(Shape4{out.shape.b, out.shape.h * u, out.shape.s / u, out.shape.d});
  d2h(r.data.data(), res.p, n);
  return r;
}
}  // namespace detail

inline Tensor4 usp_attention(WorkerContext& ctx, const Tensor4& q, const Tensor4& k,
                             const Tensor4& v, const Mesh2D& mesh, const CommOptions& opts) {
  if (mesh.n != ctx.world_size())
    throw MeshError("mesh covers " + std::to_string(mesh.n) + " workers but the fabric has " +
                    std::to_string(ctx.world_size()));
  if (!(q.shape == k.shape) || !(q.shape == v.shape))
    throw ShapeError("usp: local Q/K/V shapes differ: Q=" + q.shape.str() + " K=" + k.shape.str() +
                     " V=" + v.shape.str());
  fusp_comm_options o{};
  o.fp8_kv = opts.fp8_kv;
  o.pipelined_ring = opts.pipelined_ring;
  o.out_dtype = FUSP_F32;
  o.check_finite = 1;
  Tensor4 out(q.shape);
  check(fusp_usp_attention_host(ctx.handle(), mesh.r, q.data.data(), k.data.data(), v.data.data(),
                                FUSP_F32, q.shape.c(), out.data.data(), &o, nullptr));
  return out;
}

}  // namespace uspsim
}  // namespace fastusp
