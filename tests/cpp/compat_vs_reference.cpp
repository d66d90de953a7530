// GPU parity test at the C++ boundary: the same harness code drives the reference's
// uspsim library (oracle/_ref, compiled from /root/reference/proj) and the fastusp
// façade (include/fastusp/uspsim_compat.hpp over libfastusp.so) on identical inputs.
// Exit code 0 = every check passed; one line of JSON per check on stdout.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "fastusp/uspsim_compat.hpp"
#include "uspsim/fp8.hpp"
#include "uspsim/mesh.hpp"
#include "uspsim/protocols.hpp"
#include "uspsim/rng.hpp"

namespace fu = fastusp::uspsim;

static int failures = 0;

static void report(const std::string& name, bool ok, double metric) {
  std::printf("{\"check\": \"%s\", \"ok\": %s, \"metric\": %.3e}\n", name.c_str(),
              ok ? "true" : "false", metric);
  if (!ok) ++failures;
}

// bf16-representable inputs from the reference RNG
static uspsim::Tensor4 fixture(uint64_t seed, uspsim::Shape4 sh) {
  uspsim::Tensor4 t(sh);
  uspsim::Rng(seed).fill_uniform(t, -1.f, 1.f);
  for (float& x : t.data) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000u;
    std::memcpy(&x, &b, 4);
  }
  return t;
}

// genuine f32 values (NOT bf16-representable): the facade's native calling convention
static uspsim::Tensor4 fixture_f32(uint64_t seed, uspsim::Shape4 sh, float lo, float hi) {
  uspsim::Tensor4 t(sh);
  uspsim::Rng(seed).fill_uniform(t, lo, hi);
  return t;
}

static fu::Tensor4 to_fu(const uspsim::Tensor4& t) {
  return fu::Tensor4(fu::Shape4{t.shape.b, t.shape.h, t.shape.s, t.shape.d}, t.data);
}

static double rel_l2(const std::vector<float>& a, const std::vector<float>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += double(a[i] - b[i]) * (a[i] - b[i]);
    den += double(b[i]) * b[i];
  }
  return std::sqrt(num / den);
}

int main() {
  const uspsim::Shape4 full{1, 8, 256, 128};
  auto Q = fixture(42, full), K = fixture(43, full), V = fixture(44, full);

  // quantize: codes and scale bit-exact (fp8.cpp:107-123)
  {
    auto rq = uspsim::quantize(K);
    auto fq = fu::quantize(to_fu(K));
    bool ok = rq.scale == fq.scale && rq.codes.data == fq.codes.data;
    report("quantize_bit_exact", ok, 0);
    report("encode_e4m3_known", fu::encode_e4m3(1000.f) == 0x7E && fu::encode_e4m3(-0.f) == 0x80, 0);
  }
  // attention_with_lse (tensor.cpp:193-202)
  {
    auto r = uspsim::attention_with_lse(Q, K, V);
    auto f = fu::attention_with_lse(to_fu(Q), to_fu(K), to_fu(V));
    double e = rel_l2(f.out.data, r.out.data);
    double le = 0;
    for (size_t i = 0; i < r.lse.size(); ++i) le = std::max(le, double(std::fabs(f.lse[i] - r.lse[i])));
    report("attention_with_lse_relL2", e <= 1e-3, e);
    report("attention_with_lse_lse_maxabs", le <= 1e-4, le);
  }
  // usp_attention over N ranks (protocols.cpp:321-340), same harness for both libraries
  for (int n : {1, 2, 4, 8}) {
    for (int r = 1; r <= n; r *= 2) {
      for (int fp8 = 0; fp8 < 2; ++fp8) {
        auto qs = uspsim::split_sequence(Q, n), ks = uspsim::split_sequence(K, n),
             vs = uspsim::split_sequence(V, n);
        std::vector<uspsim::Tensor4> ref_out(n);
        auto rmesh = uspsim::make_mesh(n, r);
        uspsim::run_protocol(n, [&](uspsim::WorkerContext& ctx) {
          ref_out[ctx.rank()] = uspsim::usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                      vs[ctx.rank()], rmesh, {fp8 != 0, true});
        });
        std::vector<fu::Tensor4> fu_out(n);
        auto fmesh = fu::make_mesh(n, r);
        fu::run_protocol(n, [&](fu::WorkerContext& ctx) {
          int k = ctx.rank();
          fu_out[k] = fu::usp_attention(ctx, to_fu(qs[k]), to_fu(ks[k]), to_fu(vs[k]), fmesh,
                                        {fp8 != 0, true});
        });
        double e = rel_l2(fu::gather_output(fu_out).data, uspsim::gather_output(ref_out).data);
        report("usp_n" + std::to_string(n) + "_r" + std::to_string(r) + (fp8 ? "_fp8" : ""),
               e <= (fp8 ? 2e-3 : 1e-3), e);
      }
    }
  }
  // f32 inputs that bf16 cannot represent, U[-1,1] and U[-3,3] (f16 Q.K^T + range guard)
  for (float hi : {1.f, 3.f}) {
    auto q = fixture_f32(71, full, -hi, hi), k = fixture_f32(72, full, -hi, hi),
         v = fixture_f32(73, full, -hi, hi);
    auto r = uspsim::attention_with_lse(q, k, v);
    auto f = fu::attention_with_lse(to_fu(q), to_fu(k), to_fu(v));
    double e = rel_l2(f.out.data, r.out.data);
    report("attention_f32_u" + std::to_string(int(hi)) + "_relL2", e <= 1e-3, e);
    auto qs = uspsim::split_sequence(q, 4), ks = uspsim::split_sequence(k, 4),
         vs = uspsim::split_sequence(v, 4);
    std::vector<uspsim::Tensor4> ref_out(4);
    auto rmesh = uspsim::make_mesh(4, 2);
    uspsim::run_protocol(4, [&](uspsim::WorkerContext& ctx) {
      ref_out[ctx.rank()] =
          uspsim::usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], rmesh, {false, true});
    });
    std::vector<fu::Tensor4> fu_out(4);
    auto fmesh = fu::make_mesh(4, 2);
    fu::run_protocol(4, [&](fu::WorkerContext& ctx) {
      int i = ctx.rank();
      fu_out[i] = fu::usp_attention(ctx, to_fu(qs[i]), to_fu(ks[i]), to_fu(vs[i]), fmesh, {false, true});
    });
    e = rel_l2(fu::gather_output(fu_out).data, uspsim::gather_output(ref_out).data);
    report("usp_f32_u" + std::to_string(int(hi)) + "_n4_r2", e <= 1e-3, e);
  }
  // |V| = 1e5 (beyond f16) and 1e-6 (f16 subnormal) through the facade
  for (float vs_ : {1e5f, 1e-6f}) {
    auto v = fixture_f32(73, full, -vs_, vs_);
    auto r = uspsim::attention_with_lse(Q, K, v);
    auto f = fu::attention_with_lse(to_fu(Q), to_fu(K), to_fu(v));
    double e = rel_l2(f.out.data, r.out.data);
    report(std::string("attention_v_") + (vs_ > 1 ? "1e5" : "1e-6"), e <= 1e-3 && std::isfinite(e), e);
  }
  // attention_reference / merge_lse (tensor.cpp:185-243)
  {
    auto half = [&](const uspsim::Tensor4& t, int i) { return t.slice_seq(i * 128, 128); };
    auto a = uspsim::attention_with_lse(Q, half(K, 0), half(V, 0));
    auto b = uspsim::attention_with_lse(Q, half(K, 1), half(V, 1));
    auto rm = uspsim::merge_lse(a, b);
    fu::AttnResult fa{to_fu(a.out), a.lse}, fb{to_fu(b.out), b.lse};
    auto fm = fu::merge_lse(fa, fb);
    double e = rel_l2(fm.out.data, rm.out.data);
    double le = 0;
    for (size_t i = 0; i < rm.lse.size(); ++i) le = std::max(le, double(std::fabs(fm.lse[i] - rm.lse[i])));
    report("merge_lse", e <= 1e-6 && le <= 1e-6, e);
    auto ar = fu::attention_reference(to_fu(Q), to_fu(K), to_fu(V));
    e = rel_l2(ar.data, uspsim::attention_reference(Q, K, V).data);
    report("attention_reference", e <= 1e-3, e);
    bool threw = false;
    try {
      fu::merge_lse(fa, fu::AttnResult{to_fu(half(Q, 0).slice_seq(0, 64)), {}});
    } catch (const fu::ShapeError& x) {
      threw = std::string(x.what()).find("merge_lse: output shapes differ") != std::string::npos;
    }
    report("merge_lse_error", threw, 0);
  }
  // ulysses_attention / ring_attention_* over SUB-groups of a 4-rank world (protocols.hpp:47-65):
  // two disjoint groups each run their own problem, same harness for both libraries
  for (int fp8 = 0; fp8 < 2; ++fp8) {
    const std::vector<std::vector<int>> ug = {{0, 1}, {2, 3}}, rg = {{0, 2}, {1, 3}};
    auto Q2 = fixture(52, full), K2 = fixture(53, full), V2 = fixture(54, full);
    auto pick = [&](int grp, const uspsim::Tensor4& a, const uspsim::Tensor4& b) { return grp ? b : a; };
    // rank -> (group index, position)
    auto loc = [&](const std::vector<std::vector<int>>& gs, int rank, int* gi, int* pos) {
      for (int g = 0; g < 2; ++g)
        for (int p = 0; p < 2; ++p)
          if (gs[g][p] == rank) { *gi = g; *pos = p; }
    };
    std::vector<uspsim::Tensor4> r_u(4), r_ro(4);
    std::vector<std::vector<float>> r_rl(4);
    uspsim::run_protocol(4, [&](uspsim::WorkerContext& ctx) {
      int g, p;
      loc(ug, ctx.rank(), &g, &p);
      uspsim::ProcessGroup pg{ug[g]};
      auto sq = uspsim::split_sequence(pick(g, Q, Q2), 2)[p], sk = uspsim::split_sequence(pick(g, K, K2), 2)[p],
           sv = uspsim::split_sequence(pick(g, V, V2), 2)[p];
      r_u[ctx.rank()] = uspsim::ulysses_attention(ctx, sq, sk, sv, pg, {fp8 != 0, false});
      loc(rg, ctx.rank(), &g, &p);
      uspsim::ProcessGroup pr{rg[g]};
      sq = uspsim::split_sequence(pick(g, Q, Q2), 2)[p];
      sk = uspsim::split_sequence(pick(g, K, K2), 2)[p];
      sv = uspsim::split_sequence(pick(g, V, V2), 2)[p];
      auto rr = uspsim::ring_attention_pipelined(ctx, sq, sk, sv, pr, {fp8 != 0, true});
      r_ro[ctx.rank()] = rr.out;
      r_rl[ctx.rank()] = rr.lse;
    });
    std::vector<fu::Tensor4> f_u(4), f_ro(4), f_so(4);
    std::vector<std::vector<float>> f_rl(4);
    fu::run_protocol(4, [&](fu::WorkerContext& ctx) {
      int g, p;
      loc(ug, ctx.rank(), &g, &p);
      fu::ProcessGroup pg{ug[g]};
      auto sq = uspsim::split_sequence(pick(g, Q, Q2), 2)[p], sk = uspsim::split_sequence(pick(g, K, K2), 2)[p],
           sv = uspsim::split_sequence(pick(g, V, V2), 2)[p];
      f_u[ctx.rank()] = fu::ulysses_attention(ctx, to_fu(sq), to_fu(sk), to_fu(sv), pg, {fp8 != 0, false});
      loc(rg, ctx.rank(), &g, &p);
      fu::ProcessGroup pr{rg[g]};
      sq = uspsim::split_sequence(pick(g, Q, Q2), 2)[p];
      sk = uspsim::split_sequence(pick(g, K, K2), 2)[p];
      sv = uspsim::split_sequence(pick(g, V, V2), 2)[p];
      auto fr = fu::ring_attention_pipelined(ctx, to_fu(sq), to_fu(sk), to_fu(sv), pr, {fp8 != 0, true});
      f_ro[ctx.rank()] = fr.out;
      f_rl[ctx.rank()] = fr.lse;
      f_so[ctx.rank()] = fu::ring_attention_serial(ctx, to_fu(sq), to_fu(sk), to_fu(sv), pr, {fp8 != 0, false}).out;
    });
    const double bar = fp8 ? 2e-3 : 1e-3;
    double eu = 0, er = 0, le = 0;
    bool same = true;
    for (int i = 0; i < 4; ++i) {
      eu = std::max(eu, rel_l2(f_u[i].data, r_u[i].data));
      er = std::max(er, rel_l2(f_ro[i].data, r_ro[i].data));
      for (size_t j = 0; j < r_rl[i].size(); ++j) le = std::max(le, double(std::fabs(f_rl[i][j] - r_rl[i][j])));
      same = same && f_so[i].data == f_ro[i].data;
    }
    const std::string sfx = fp8 ? "_fp8" : "";
    report("ulysses_subgroup" + sfx, eu <= bar, eu);
    report("ring_subgroup" + sfx, er <= bar && le <= (fp8 ? 2e-3 : 1e-4), er);
    report("ring_subgroup_serial_eq_pipelined" + sfx, same, 0);
  }
  // detail::ulysses_input_reshard / output_reshard (protocols.cpp:125-203): pure data movement
  // (and exact FP8 dequantization) -- bit-identical to the reference
  for (int fp8 = 0; fp8 < 2; ++fp8) {
    const int n = 4;
    auto qs = uspsim::split_sequence(Q, n), ks = uspsim::split_sequence(K, n), vs = uspsim::split_sequence(V, n);
    std::vector<uspsim::detail::Resharded> rr(n);
    std::vector<uspsim::Tensor4> ro(n);
    uspsim::ProcessGroup world{{0, 1, 2, 3}};
    uspsim::run_protocol(n, [&](uspsim::WorkerContext& ctx) {
      int i = ctx.rank();
      rr[i] = uspsim::detail::ulysses_input_reshard(ctx, qs[i], ks[i], vs[i], world, {fp8 != 0, false});
      ro[i] = uspsim::detail::ulysses_output_reshard(ctx, rr[i].v, world);
    });
    std::vector<fu::detail::Resharded> fr(n);
    std::vector<fu::Tensor4> fo(n);
    fu::ProcessGroup fworld{{0, 1, 2, 3}}, fsub{{1, 0}};
    std::vector<fu::detail::Resharded> fsubr(n);
    fu::run_protocol(n, [&](fu::WorkerContext& ctx) {
      int i = ctx.rank();
      fr[i] = fu::detail::ulysses_input_reshard(ctx, to_fu(qs[i]), to_fu(ks[i]), to_fu(vs[i]), fworld,
                                               {fp8 != 0, false});
      fo[i] = fu::detail::ulysses_output_reshard(ctx, to_fu(rr[i].v), fworld);
    });
    bool exact = true;
    for (int i = 0; i < n; ++i)
      exact = exact && fr[i].q.data == rr[i].q.data && fr[i].k.data == rr[i].k.data &&
              fr[i].v.data == rr[i].v.data && fo[i].data == ro[i].data;
    report(std::string("reshards_bit_exact") + (fp8 ? "_fp8" : ""), exact, 0);
  }
  // gather_shards (protocols.cpp:25-50) and QuantizedTensor::slice_heads (fp8.cpp:100-105)
  {
    auto parts = uspsim::split_sequence(Q, 4);
    std::vector<std::pair<uspsim::ShardSpec, uspsim::Tensor4>> rs;
    std::vector<std::pair<fu::ShardSpec, fu::Tensor4>> fs;
    for (int i : {2, 0, 3, 1}) {
      rs.push_back({uspsim::ShardSpec{uspsim::ShardSpec::Axis::kSequence, i, 4}, parts[i]});
      fs.push_back({fu::ShardSpec{fu::ShardSpec::Axis::kSequence, i, 4}, to_fu(parts[i])});
    }
    report("gather_shards", fu::gather_shards(fs).data == uspsim::gather_shards(rs).data, 0);
    fs.pop_back();
    std::string msg;
    try {
      fu::gather_shards(fs);
    } catch (const fu::ShapeError& e) {
      msg = e.what();
    }
    rs.pop_back();
    std::string rmsg;
    try {
      uspsim::gather_shards(rs);
    } catch (const uspsim::ShapeError& e) {
      rmsg = e.what();
    }
    report("gather_shards_gap_message", !msg.empty() && msg == rmsg, 0);
    auto rq = uspsim::quantize(K).slice_heads(2, 3);
    auto fq = fu::quantize(to_fu(K)).slice_heads(2, 3);
    report("quantized_slice_heads", rq.scale == fq.scale && rq.codes.data == fq.codes.data, 0);
  }
  // error classes map 1:1 (ShapeError on H % U, protocols.cpp:328-331)
  {
    bool ok = false;
    auto bad = fixture(1, {1, 3, 16, 128});
    try {
      auto m = fu::make_mesh(2, 1);
      fu::run_protocol(2, [&](fu::WorkerContext& ctx) {
        fu::usp_attention(ctx, to_fu(bad), to_fu(bad), to_fu(bad), m, {});
      });
    } catch (const fu::WorkerFailure& e) {
      ok = std::string(e.what()).find("usp: head count H=3 not divisible by ulysses dimension U=2") !=
           std::string::npos;
    }
    report("error_shape_message", ok, 0);
  }
  std::printf("{\"failures\": %d}\n", failures);
  return failures == 0 ? 0 : 1;
}
