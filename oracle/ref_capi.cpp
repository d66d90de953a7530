// TEST INFRASTRUCTURE ONLY -- the oracle's C entry points (oracle/_ref/libuspsim_ref.so).
//
// A thin extern "C" layer over the *reference's own* uspsim library, compiled
// from /root/reference/proj/src by oracle/Makefile (see oracle/shim/*.cpp for
// the two one-line compile fixes, applied without touching the sources).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this library, and only as the checker or the
// timed CPU baseline -- never as the product path.
//
// Every function returns 0 on success or an error class code:
//   1 ShapeError (tensor.hpp:13)      2 MeshError (mesh.hpp:17)
//   3 FabricError (fabric.hpp:106)    4 std::invalid_argument
//   5 DeadlockError (fabric.hpp:112)  6 WorkerFailure (fabric.hpp:118)
//   9 anything else
// and leaves the exception's what() in ref_last_error().
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "uspsim/fp8.hpp"
#include "uspsim/mesh.hpp"
#include "uspsim/protocols.hpp"
#include "uspsim/rng.hpp"
#include "uspsim/tensor.hpp"

using namespace uspsim;

namespace {

thread_local std::string g_err;

int classify(const std::exception& e) {
  if (dynamic_cast<const ShapeError*>(&e)) return 1;
  if (dynamic_cast<const MeshError*>(&e)) return 2;
  if (dynamic_cast<const FabricError*>(&e)) return 3;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 4;
  if (dynamic_cast<const DeadlockError*>(&e)) return 5;
  if (dynamic_cast<const WorkerFailure*>(&e)) return 6;
  return 9;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
  } catch (...) {
    g_err = "unknown exception";
    return 9;
  }
}

Tensor4 make(const float* p, int64_t b, int64_t h, int64_t s, int64_t d) {
  Shape4 sh{b, h, s, d};
  std::vector<float> v(p, p + sh.count());
  return Tensor4(sh, std::move(v));
}

void put(const Tensor4& t, float* out) { std::memcpy(out, t.data.data(), t.data.size() * 4); }

// Per-rank error capture inside run_protocol programs so the *inner*
// exception class survives the WorkerFailure wrapper (fabric.cpp:402-406).
struct RankErr {
  std::mutex mu;
  int code = 0;
  std::string what;
  void record(const std::exception& e) {
    std::lock_guard<std::mutex> lk(mu);
    if (code == 0) {
      code = classify(e);
      what = e.what();
    }
  }
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- fp8 codec (fp8.cpp:39-68, 107-130) ------------------------------------
int ref_encode_e4m3(const float* x, uint8_t* out, int64_t n) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) out[i] = encode_e4m3(x[i]);
  });
}

int ref_decode_e4m3(const uint8_t* c, float* out, int64_t n) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) out[i] = decode_e4m3(c[i]);
  });
}

int ref_quantize(const float* x, int64_t b, int64_t h, int64_t s, int64_t d, uint8_t* codes,
                 float* scale) {
  return guarded([&] {
    QuantizedTensor q = quantize(make(x, b, h, s, d));
    std::memcpy(codes, q.codes.data.data(), q.codes.data.size());
    *scale = q.scale;
  });
}

int ref_dequantize(const uint8_t* codes, float scale, int64_t b, int64_t h, int64_t s, int64_t d,
                   float* out) {
  return guarded([&] {
    QuantizedTensor q;
    q.scale = scale;
    q.codes = CodeTensor(Shape4{b, h, s, d});
    std::memcpy(q.codes.data.data(), codes, q.codes.data.size());
    put(dequantize(q), out);
  });
}

// ---- attention numerics (tensor.cpp:185-243) --------------------------------
int ref_attention_with_lse_f32(const float* q, const float* k, const float* v, int64_t b,
                               int64_t h, int64_t sq, int64_t skv, int64_t d, float* out,
                               float* lse) {
  return guarded([&] {
    AttnResult r = attention_with_lse(make(q, b, h, sq, d), make(k, b, h, skv, d),
                                      make(v, b, h, skv, d));
    put(r.out, out);
    std::memcpy(lse, r.lse.data(), r.lse.size() * 4);
  });
}

int ref_attention_with_lse_f64(const double* q, const double* k, const double* v, int64_t b,
                               int64_t h, int64_t sq, int64_t skv, int64_t d, double* out,
                               double* lse) {
  return guarded([&] {
    auto mk = [](const double* p, Shape4 sh) {
      return Tensor4d(sh, std::vector<double>(p, p + sh.count()));
    };
    AttnResultd r = attention_with_lse(mk(q, {b, h, sq, d}), mk(k, {b, h, skv, d}),
                                       mk(v, {b, h, skv, d}));
    std::memcpy(out, r.out.data.data(), r.out.data.size() * 8);
    std::memcpy(lse, r.lse.data(), r.lse.size() * 8);
  });
}

int ref_attention_reference_f32(const float* q, const float* k, const float* v, int64_t b,
                                int64_t h, int64_t sq, int64_t skv, int64_t d, float* out) {
  return guarded([&] {
    put(attention_reference(make(q, b, h, sq, d), make(k, b, h, skv, d), make(v, b, h, skv, d)),
        out);
  });
}

int ref_merge_lse_f32(const float* o1, const float* l1, const float* o2, const float* l2, int64_t b,
                      int64_t h, int64_t s, int64_t d, float* out, float* lse) {
  return guarded([&] {
    AttnResult a, c;
    a.out = make(o1, b, h, s, d);
    c.out = make(o2, b, h, s, d);
    a.lse.assign(l1, l1 + b * h * s);
    c.lse.assign(l2, l2 + b * h * s);
    AttnResult r = merge_lse(a, c);
    put(r.out, out);
    std::memcpy(lse, r.lse.data(), r.lse.size() * 4);
  });
}

// ---- mesh (mesh.cpp:34-79) ---------------------------------------------------
int ref_build_mesh(int n, int max_ring, int heads, int* r, int* u) {
  return guarded([&] {
    Mesh2D m = build_mesh(n, max_ring, heads);
    *r = m.r;
    *u = m.u;
  });
}

// groups written as flat member lists: ulysses [R][U], ring [U][R]
int ref_make_mesh(int n, int r, int* ulysses_groups, int* ring_groups) {
  return guarded([&] {
    Mesh2D m = make_mesh(n, r);
    int i = 0;
    for (const auto& g : m.ulysses_groups)
      for (int x : g.members) ulysses_groups[i++] = x;
    i = 0;
    for (const auto& g : m.ring_groups)
      for (int x : g.members) ring_groups[i++] = x;
  });
}

// ---- fixtures (rng.hpp:20-43) -------------------------------------------------
int ref_rng_uniform(uint64_t seed, int64_t n, float lo, float hi, float* out) {
  return guarded([&] {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
  });
}

// ---- protocols over the reference's deterministic fabric (protocols.cpp) ----
// Global q,k,v [B,H,S,D]; rank r holds split_sequence(..., n)[r] (protocols.cpp:10-21).
// out_global receives gather_output of every rank's result. a2a_bytes/send_bytes
// (length n, may be null) receive TrafficLog::bytes_for(op, rank) (fabric.cpp:44-49).
int ref_usp_attention(int n, int r, int fp8, int pipelined, const float* q, const float* k,
                      const float* v, int64_t b, int64_t h, int64_t s, int64_t d,
                      float* out_global, uint64_t* a2a_bytes, uint64_t* send_bytes) {
  return guarded([&] {
    Tensor4 Q = make(q, b, h, s, d), K = make(k, b, h, s, d), V = make(v, b, h, s, d);
    auto qs = split_sequence(Q, n), ks = split_sequence(K, n), vs = split_sequence(V, n);
    Mesh2D mesh = make_mesh(n, r);
    CommOptions opts{fp8 != 0, pipelined != 0};
    std::vector<Tensor4> outs(static_cast<size_t>(n));
    RankErr err;
    RunReport rep;
    try {
      rep = run_protocol(n, [&](WorkerContext& ctx) {
        const int rk = ctx.rank();
        try {
          outs[rk] = usp_attention(ctx, qs[rk], ks[rk], vs[rk], mesh, opts);
        } catch (const std::exception& e) {
          err.record(e);
          throw;
        }
      });
    } catch (const WorkerFailure&) {
      if (err.code == 1) throw ShapeError(err.what);
      if (err.code == 2) throw MeshError(err.what);
      if (err.code == 4) throw std::invalid_argument(err.what);
      throw;
    }
    put(gather_output(outs), out_global);
    for (int i = 0; i < n; ++i) {
      if (a2a_bytes) a2a_bytes[i] = rep.traffic.bytes_for("all_to_all", i);
      if (send_bytes) send_bytes[i] = rep.traffic.bytes_for("send", i);
    }
  });
}

// usp_attention returning the fabric's own report: TrafficLog::to_json and Timeline::to_json
// (fabric.cpp:72-87, :115-125) as JSON text.
int ref_usp_report(int n, int r, int fp8, int pipelined, const float* q, const float* k,
                   const float* v, int64_t b, int64_t h, int64_t s, int64_t d, char* traffic,
                   size_t traffic_cap, char* timeline, size_t timeline_cap) {
  return guarded([&] {
    Tensor4 Q = make(q, b, h, s, d), K = make(k, b, h, s, d), V = make(v, b, h, s, d);
    auto qs = split_sequence(Q, n), ks = split_sequence(K, n), vs = split_sequence(V, n);
    Mesh2D mesh = make_mesh(n, r);
    CommOptions opts{fp8 != 0, pipelined != 0};
    RunReport rep = run_protocol(n, [&](WorkerContext& ctx) {
      const int rk = ctx.rank();
      usp_attention(ctx, qs[rk], ks[rk], vs[rk], mesh, opts);
    });
    const std::string tj = rep.traffic.to_json().dump(), lj = rep.timeline.to_json().dump();
    std::snprintf(traffic, traffic_cap, "%s", tj.c_str());
    std::snprintf(timeline, timeline_cap, "%s", lj.c_str());
  });
}

// Pure Ulysses over the world group (protocols.cpp:207-214).
int ref_ulysses_attention(int n, int fp8, const float* q, const float* k, const float* v,
                          int64_t b, int64_t h, int64_t s, int64_t d, float* out_global) {
  return guarded([&] {
    Tensor4 Q = make(q, b, h, s, d), K = make(k, b, h, s, d), V = make(v, b, h, s, d);
    auto qs = split_sequence(Q, n), ks = split_sequence(K, n), vs = split_sequence(V, n);
    ProcessGroup g = make_world_group(n);
    CommOptions opts{fp8 != 0, false};
    std::vector<Tensor4> outs(static_cast<size_t>(n));
    run_protocol(n, [&](WorkerContext& ctx) {
      const int rk = ctx.rank();
      outs[rk] = ulysses_attention(ctx, qs[rk], ks[rk], vs[rk], g, opts);
    });
    put(gather_output(outs), out_global);
  });
}

// Ring over the world group (protocols.cpp:237-319): returns gathered out and lse
// (lse laid out [B,H,S] after gathering along S).
int ref_ring_attention(int n, int fp8, int pipelined, const float* q, const float* k,
                       const float* v, int64_t b, int64_t h, int64_t s, int64_t d,
                       float* out_global, float* lse_global) {
  return guarded([&] {
    Tensor4 Q = make(q, b, h, s, d), K = make(k, b, h, s, d), V = make(v, b, h, s, d);
    auto qs = split_sequence(Q, n), ks = split_sequence(K, n), vs = split_sequence(V, n);
    ProcessGroup g = make_world_group(n);
    CommOptions opts{fp8 != 0, pipelined != 0};
    std::vector<AttnResult> res(static_cast<size_t>(n));
    run_protocol(n, [&](WorkerContext& ctx) {
      const int rk = ctx.rank();
      res[rk] = pipelined ? ring_attention_pipelined(ctx, qs[rk], ks[rk], vs[rk], g, opts)
                          : ring_attention_serial(ctx, qs[rk], ks[rk], vs[rk], g, opts);
    });
    std::vector<Tensor4> outs;
    for (auto& x : res) outs.push_back(x.out);
    put(gather_output(outs), out_global);
    const int64_t sl = s / n;
    for (int rk = 0; rk < n; ++rk)
      for (int64_t bh = 0; bh < b * h; ++bh)
        for (int64_t i = 0; i < sl; ++i)
          lse_global[bh * s + rk * sl + i] = res[rk].lse[static_cast<size_t>(bh * sl + i)];
  });
}

// Ulysses input reshard on the world group (protocols.cpp:125-180). Writes each
// rank's resharded q/k/v [B,H/n,S,D] back to back (rank-major).
int ref_ulysses_input_reshard(int n, int fp8, const float* q, const float* k, const float* v,
                              int64_t b, int64_t h, int64_t s, int64_t d, float* rq, float* rk,
                              float* rv) {
  return guarded([&] {
    Tensor4 Q = make(q, b, h, s, d), K = make(k, b, h, s, d), V = make(v, b, h, s, d);
    auto qs = split_sequence(Q, n), ks = split_sequence(K, n), vs = split_sequence(V, n);
    ProcessGroup g = make_world_group(n);
    CommOptions opts{fp8 != 0, false};
    std::vector<detail::Resharded> res(static_cast<size_t>(n));
    run_protocol(n, [&](WorkerContext& ctx) {
      const int r = ctx.rank();
      res[r] = detail::ulysses_input_reshard(ctx, qs[r], ks[r], vs[r], g, opts);
    });
    const int64_t per = b * (h / n) * s * d;
    for (int r = 0; r < n; ++r) {
      std::memcpy(rq + r * per, res[r].q.data.data(), per * 4);
      std::memcpy(rk + r * per, res[r].k.data.data(), per * 4);
      std::memcpy(rv + r * per, res[r].v.data.data(), per * 4);
    }
  });
}

// ---- CPU baseline timing -------------------------------------------------------
// nthreads concurrent calls of the reference's attention_with_lse, each on one
// head: Q [1,1,sq,d] against K,V [1,1,skv,d] (tensor.cpp:193-202), inputs from
// uspsim::Rng. Returns the wall time of the concurrent section in *seconds.
int ref_time_attention(int nthreads, int64_t sq, int64_t skv, int64_t d, uint64_t seed,
                       double* seconds, float* checksum) {
  return guarded([&] {
    std::vector<Tensor4> qs, ks, vs;
    for (int t = 0; t < nthreads; ++t) {
      Rng rng(seed + static_cast<uint64_t>(t));
      Tensor4 Q(Shape4{1, 1, sq, d}), K(Shape4{1, 1, skv, d}), V(Shape4{1, 1, skv, d});
      rng.fill_uniform(Q, -1.f, 1.f);
      rng.fill_uniform(K, -1.f, 1.f);
      rng.fill_uniform(V, -1.f, 1.f);
      qs.push_back(std::move(Q));
      ks.push_back(std::move(K));
      vs.push_back(std::move(V));
    }
    std::vector<float> sums(static_cast<size_t>(nthreads), 0.f);
    std::vector<std::thread> th;
    auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < nthreads; ++t) {
      th.emplace_back([&, t] {
        AttnResult r = attention_with_lse(qs[t], ks[t], vs[t]);
        sums[t] = r.out.data[0] + r.lse[0];
      });
    }
    for (auto& x : th) x.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    float c = 0.f;
    for (float x : sums) c += x;
    *checksum = c;
  });
}

}  // extern "C"
