// QKV projection (with / without the QK prologue epilogue) and output projection timings at
// the FLUX shape and its per-rank token counts at N = 2, 4, 8 (S / N rows: the block's GEMMs at
// U = N), CUDA events over back-to-back launches.
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2602_10940_b200/csrc/fastusp_internal.h"
using namespace fusp;
// uniform(-a, a) bf16 from a hash of the index (random operands: tensor-core power, and so
// clocks, depend on the data; constant fills would flatter the numbers)
__global__ void fill_bf16(uint16_t* p, size_t n, float a, uint32_t seed) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    const float u = (h & 0xFFFFFF) * (1.0f / 16777216.0f) * 2.f - 1.f;
    p[i] = uint16_t(__float_as_uint(u * a) >> 16);
  }
}
int main() {
  const int s = 4608, c = 3072, h = 24, n = 3 * h * 128;  // allocation at the full sequence
  void *x, *w, *q, *k, *v, *wo, *y;
  float *wq, *cs;
  cudaMalloc(&x, size_t(s) * c * 2); cudaMalloc(&w, size_t(c) * n * 2);
  cudaMalloc(&q, size_t(s) * h * 128 * 2); cudaMalloc(&k, size_t(s) * h * 128 * 2); cudaMalloc(&v, size_t(s) * h * 128 * 2);
  cudaMalloc(&wo, size_t(h) * 128 * c * 2); cudaMalloc(&y, size_t(s) * c * 2);
  cudaMalloc(&wq, 128 * 4); cudaMalloc(&cs, size_t(s) * 64 * 4);
  fill_bf16<<<1184, 256>>>(static_cast<uint16_t*>(x), size_t(s) * c, 1.f, 1);
  fill_bf16<<<1184, 256>>>(static_cast<uint16_t*>(w), size_t(c) * n, 0.02f, 2);
  fill_bf16<<<1184, 256>>>(static_cast<uint16_t*>(wo), size_t(h) * 128 * c, 0.02f, 3);
  fill_bf16<<<1184, 256>>>(static_cast<uint16_t*>(q), size_t(s) * h * 128, 1.f, 4); cudaMemset(wq, 0, 128 * 4); cudaMemset(cs, 0, size_t(s) * 64 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int cur = s;  // the token count being timed (printed)
  auto run = [&](const char* name, double flop, auto f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
    printf("{\"kernel\": \"%s\", \"tokens\": %d, \"us\": %.1f, \"tflops\": %.1f}\n", name, cur, ms * 1e3, flop / (ms * 1e-3) / 1e12);
  };
  for (const int s : {4608, 2304, 1152, 576}) {
  cur = s;
  const double fq = 2.0 * s * c * n, fo = 2.0 * s * h * 128 * c;
  run("qkv projection, plain epilogue", fq, [&] { launch_qkv_proj(x, FUSP_BF16, 1, s, c, w, h, q, k, v, FUSP_BF16, nullptr, nullptr, 0.f, nullptr, nullptr, 0, 0); });
  run("qkv projection + RMSNorm + RoPE epilogue", fq, [&] { launch_qkv_proj(x, FUSP_BF16, 1, s, c, w, h, q, k, v, FUSP_BF16, wq, wq, 1e-6f, cs, cs, 0, 0); });
  run("output projection", fo, [&] { launch_out_proj(q, FUSP_BF16, 1, h, s, wo, c, y, FUSP_BF16, 0); });
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
