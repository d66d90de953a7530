// Times the layer's HBM-bound movers (Ulysses pack / unpack, FP8 amax+quantize, dequantize)
// at the BASELINE per-rank shapes with CUDA events: `hot` = back-to-back repetitions,
// `cold` = a 256 MiB L2 flush before every repetition.  Algorithmic bytes = compulsory reads +
// writes.  Links the library's internal launchers (exported C++ symbols of libfastusp.so).
//   make -C tools/cpp && tools/cpp/movers_bench
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <functional>
#include "../../paper_2602_10940_b200/csrc/fastusp_internal.h"

using namespace fusp;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
#define FK(x) do { fusp_status st = (x); if (st != FUSP_OK) { printf("fusp error %d at %d\n", int(st), __LINE__); return 1; } } while (0)

static void* flushbuf = nullptr;
static double peak = 6548.5;

static void* cpa = nullptr;
static void* cpb = nullptr;
static void report(const char* name, double bytes, const std::function<void()>& f, bool with_copy = true);
// The same algorithmic bytes moved by a device-to-device cudaMemcpy (bytes / 2 read + written):
// the practical ceiling for a kernel of that size, launch and DRAM ramp included.
static void copy_ref(double bytes) {
  const size_t half = static_cast<size_t>(bytes / 2) / 256 * 256;
  report("  (same bytes as cudaMemcpy D2D)", 2.0 * half,
         [&] { cudaMemcpyAsync(cpb, cpa, half, cudaMemcpyDeviceToDevice); }, false);
}
static void report(const char* name, double bytes, const std::function<void()>& f, bool with_copy) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  // MOVERS_ONCE=1: one warm-up and one timed call (for ncu: every kernel captured once)
  static const bool once = getenv("MOVERS_ONCE") != nullptr;
  for (int i = 0; i < (once ? 1 : 3); ++i) f();
  cudaDeviceSynchronize();
  const int reps = once ? 1 : 50;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float hot; cudaEventElapsedTime(&hot, a, b); hot /= reps;
  float cold = 0;
  const int creps = once ? 1 : 10;
  for (int i = 0; i < creps; ++i) {
    cudaMemsetAsync(flushbuf, i, 256u << 20);
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); cold += t / creps;
  }
  printf("{\"kernel\": \"%s\", \"bytes\": %.0f, \"hot_us\": %.2f, \"hot_gbs\": %.0f, \"cold_us\": %.2f, \"cold_gbs\": %.0f, \"cold_frac_of_hbm\": %.3f}\n",
         name, bytes, hot * 1e3, bytes / (hot * 1e-3) / 1e9, cold * 1e3, bytes / (cold * 1e-3) / 1e9,
         bytes / (cold * 1e-3) / 1e9 / peak);
  if (with_copy && getenv("MOVERS_ONCE") == nullptr) copy_ref(bytes);
}

int main() {
  CK(cudaMalloc(&flushbuf, 256u << 20));
  CK(cudaMalloc(&cpa, 128u << 20));
  CK(cudaMalloc(&cpb, 128u << 20));
  {  // operand staging at FLUX U = 1: V [24][4608][128] bf16 -> f16 (the layer's only mover)
    const int heads = 24, rows = 4608;
    const int64_t n = int64_t(heads) * rows * 128;
    void *x, *y, *x32;
    int* exps;
    uint32_t* words;
    CK(cudaMalloc(&x, n * 2)); CK(cudaMalloc(&y, n * 2)); CK(cudaMalloc(&x32, n * 4));
    CK(cudaMalloc(&exps, 4096)); CK(cudaMalloc(&words, 4096)); CK(cudaMemset(words, 0, 4096));
    {  // in-range data (the common path): bf16 / f32 1.0
      std::vector<uint16_t> hb(n, 0x3f80);
      std::vector<uint32_t> hf(n, 0x3f800000u);
      CK(cudaMemcpy(x, hb.data(), n * 2, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(x32, hf.data(), n * 4, cudaMemcpyHostToDevice));
    }
    StageOp g{};
    g.src = x; g.sdt = FUSP_BF16; g.dst = y; g.ddt = FUSP_F16; g.exps = exps; g.words = words;
    StageOp u = g;
    u.exps = nullptr; u.words = nullptr;
    StageOp g32 = g;
    g32.src = x32; g32.sdt = FUSP_F32;
    report("flux_u1 stage V bf16->f16 range-guarded (stage + decide)", n * 4.0,
           [&] { launch_stage(&g, 1, heads, rows, 128, 1, 0); });
    report("flux_u1 stage V bf16->f16 unguarded (stage only)", n * 4.0,
           [&] { launch_stage(&u, 1, heads, rows, 128, 1, 0); });
    report("flux_u1 bf16_to_f16_kernel (round-1 converter, no guard)", n * 4.0,
           [&] { launch_convert(x, FUSP_BF16, y, FUSP_F16, n, 0); });
    report("flux_u1 stage Q f32->f16 range-guarded", n * 6.0,
           [&] { launch_stage(&g32, 1, heads, rows, 128, 1, 0); });
    CK(cudaMemset(x, 0x3c, n * 2));  // |x| = 0.0115 < 2^-6: every head takes the rewrite
    report("flux_u1 stage V bf16->f16 range-guarded, RARE path (all 24 heads rewritten)", n * 4.0,
           [&] { launch_stage(&g, 1, heads, rows, 128, 1, 0); });
    for (void* p : std::vector<void*>{x, y, x32, exps, words}) cudaFree(p);
  }
  struct Cfg { const char* name; int h, sl, u; };
  const Cfg cfgs[] = {{"flux_u2", 24, 2304, 2}, {"flux_u8", 24, 576, 8}};
  for (const Cfg& c : cfgs) {
    const int64_t n = int64_t(c.h) * c.sl * 128;  // one local tensor [1,H,SL,128]
    void *q, *k, *v, *slots, *dq, *dk, *dv;
    CK(cudaMalloc(&q, n * 2)); CK(cudaMalloc(&k, n * 2)); CK(cudaMalloc(&v, n * 2));
    CK(cudaMalloc(&slots, n * 6 + 4096)); CK(cudaMalloc(&dq, n * 2)); CK(cudaMalloc(&dk, n * 2)); CK(cudaMalloc(&dv, n * 2));
    CK(cudaMemset(q, 0x3c, n * 2)); CK(cudaMemset(k, 0x3c, n * 2)); CK(cudaMemset(v, 0x3c, n * 2));
    const int64_t blk = n / c.u;          // elements per (Q|K|V) slot piece
    const int64_t se2 = 3 * blk;          // slot stride (16-bit elements): [Q][K][V]
    PackDesc p[3];
    for (int t = 0; t < 3; ++t) {
      p[t] = PackDesc{};
      p[t].src = t == 0 ? q : t == 1 ? k : v; p[t].src_dtype = FUSP_BF16;
      p[t].dst = static_cast<uint16_t*>(slots) + t * blk; p[t].dst_dtype = t == 2 ? FUSP_F16 : FUSP_BF16;
      p[t].dst_slot_stride = se2; p[t].b = 1; p[t].h = c.h; p[t].sl = c.sl; p[t].d = 128; p[t].u = c.u;
    }
    char nm[96];
    snprintf(nm, sizeof nm, "%s pack Q,K,V bf16 -> slots (one launch)", c.name);
    report(nm, 3.0 * n * 4, [&] { launch_pack_multi(p, 3, 0); });
    UnpackDesc u[3];
    for (int t = 0; t < 3; ++t) {
      u[t] = UnpackDesc{};
      u[t].src = static_cast<uint16_t*>(slots) + t * blk; u[t].src_dtype = t == 2 ? FUSP_F16 : FUSP_BF16;
      u[t].src_slot_stride = se2; u[t].dst = t == 0 ? dq : t == 1 ? dk : dv; u[t].dst_dtype = u[t].src_dtype;
      u[t].b = 1; u[t].hp = c.h / c.u; u[t].sl = c.sl; u[t].d = 128; u[t].u = c.u;
    }
    {  // FP8 Ulysses pack (Q bf16, K and V E4M3 with per-tensor scales + slot trailers)
      uint32_t* w8;
      float* sc8;
      CK(cudaMalloc(&w8, 4096)); CK(cudaMemset(w8, 0, 4096)); CK(cudaMalloc(&sc8, 4096));
      const int64_t blk8 = n / c.u;                       // elements per slot piece
      const int64_t slot_bytes = blk8 * 2 + 2 * blk8 + 256;  // [Q bf16][K codes][V codes][trailers]
      PackDesc f[3];
      for (int t = 0; t < 3; ++t) {
        f[t] = PackDesc{};
        f[t].src = t == 0 ? q : t == 1 ? k : v; f[t].src_dtype = FUSP_BF16;
        f[t].b = 1; f[t].h = c.h; f[t].sl = c.sl; f[t].d = 128; f[t].u = c.u;
        f[t].dst = static_cast<char*>(slots) + (t == 0 ? 0 : blk8 * 2 + (t - 1) * blk8);
        f[t].dst_dtype = t == 0 ? FUSP_BF16 : FUSP_E4M3;
        f[t].dst_slot_stride = t == 0 ? slot_bytes / 2 : slot_bytes;
        if (t > 0) {
          f[t].scale = sc8 + (t - 1);
          f[t].trailer = reinterpret_cast<float*>(static_cast<char*>(slots) + blk8 * 4) + (t - 1);
          f[t].trailer_stride = slot_bytes / 4;
        }
      }
      uint32_t* am8[2] = {w8, w8 + 2};
      float* scs8[2] = {sc8, sc8 + 1};
      const Fp8Src s8[2] = {Fp8Src{k, FUSP_BF16, nullptr, 0, 0, 128, c.sl, c.sl}, Fp8Src{v, FUSP_BF16, nullptr, 0, 0, 128, c.sl, c.sl}};
      if (int64_t(c.u) * slot_bytes <= n * 6 + 4096) {
        snprintf(nm, sizeof nm, "%s fp8 Ulysses pack: amax pass + pack (two launches)", c.name);
        report(nm, double(n) * (2 + 2 + 2 + 2 + 1 + 1), [&] {
          launch_amax_scales(s8, 2, n, 1, am8, scs8, nullptr, 0);
          launch_pack_multi(f, 3, 0, true);
        });
        snprintf(nm, sizeof nm, "%s fp8 Ulysses pack: one cooperative launch (when it fits)", c.name);
        report(nm, double(n) * (2 + 2 + 2 + 2 + 1 + 1), [&] {
          bool done = false;
          try_pack_fp8_fused(f, am8, scs8, nullptr, 0, &done);
          if (!done) { launch_amax_scales(s8, 2, n, 1, am8, scs8, nullptr, 0); launch_pack_multi(f, 3, 0, true); }
        });
      }
      cudaFree(w8); cudaFree(sc8);
    }
    snprintf(nm, sizeof nm, "%s unpack Q,K,V slots -> operands (one launch)", c.name);
    report(nm, 3.0 * n * 4, [&] { launch_unpack_multi(u, 3, 0); });
    // FP8: K and V amax + quantize (per-tensor block), codes into a buffer
    uint8_t *ck, *cv; float* sc; uint32_t* wk;
    CK(cudaMalloc(&ck, n)); CK(cudaMalloc(&cv, n)); CK(cudaMalloc(&sc, 4096)); CK(cudaMalloc(&wk, 4096)); CK(cudaMemset(wk, 0, 4096));  // zero words (the amax pass leaves them zero)
    Fp8Src src[2] = {Fp8Src{k, FUSP_BF16, nullptr, 0, 0, 128, c.sl, c.sl}, Fp8Src{v, FUSP_BF16, nullptr, 0, 0, 128, c.sl, c.sl}};
    uint32_t* works[2] = {wk, wk + 64};
    float* scs[2] = {sc, sc + 64};
    uint8_t* cds[2] = {ck, cv};
    snprintf(nm, sizeof nm, "%s fp8 amax+quantize K,V (2 passes; bytes: 2 read + 1 written per element)", c.name);
    report(nm, 2.0 * n * (2 + 1), [&] { launch_quantize_fp8_multi(src, 2, n, n, works, scs, cds, nullptr, 0); });
    snprintf(nm, sizeof nm, "%s fp8 dequantize K -> bf16", c.name);
    report(nm, double(n) * (1 + 2), [&] { launch_dequantize_blocks(ck, sc, n, n, dk, FUSP_BF16, 0); });
    // ring hop: re-quantize an E4M3 chunk (per-segment scales) -- the FP8 ring forward
    Fp8Src esrc[2] = {Fp8Src{ck, FUSP_E4M3, sc, 0, 0, 128, c.sl, c.sl}, Fp8Src{cv, FUSP_E4M3, sc + 64, 0, 0, 128, c.sl, c.sl}};
    uint8_t *ck2, *cv2;
    CK(cudaMalloc(&ck2, n)); CK(cudaMalloc(&cv2, n));
    uint8_t* cds2[2] = {ck2, cv2};
    snprintf(nm, sizeof nm, "%s fp8 ring hop re-quantize K,V from e4m3 (hop 1: multi-scale chunk; bytes: 1 read + 1 written)", c.name);
    report(nm, 2.0 * n * (1 + 1), [&] { launch_quantize_fp8_multi(esrc, 2, n, n, works, scs, cds2, nullptr, 0); });
    float* trs[2] = {sc, sc + 64};
    snprintf(nm, sizeof nm, "%s fp8 ring hop >= 2 forward (codes kept in place, scale trailer only)", c.name);
    report(nm, 2.0 * n * (1 + 1 + 1), [&] { launch_fp8_forward_scales(trs, 2, 1, 0); });
    for (void* x : {q, k, v, slots, dq, dk, dv}) cudaFree(x);
    for (void* x : std::vector<void*>{ck, cv, sc, wk, ck2, cv2}) cudaFree(x);
  }
  // reference: a plain device copy of 3 bf16 tensors (FLUX U=2 size)
  const int64_t n = int64_t(24) * 2304 * 128 * 3;
  void *a, *b;
  CK(cudaMalloc(&a, n * 2)); CK(cudaMalloc(&b, n * 2));
  report("reference cudaMemcpyAsync D2D (FLUX U=2 Q+K+V bytes)", 4.0 * n, [&] { cudaMemcpyAsync(b, a, n * 2, cudaMemcpyDeviceToDevice); });
  return 0;
}
