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
