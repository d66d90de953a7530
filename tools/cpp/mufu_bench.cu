// Measures MUFU.EX2 and FFMA2 issue throughput per SM sub-partition on this GPU
// (warps per SMSP = 1..4, independent chains), in cycles per warp instruction.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned ex2h2(unsigned x) { unsigned y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ unsigned hmul2(unsigned a, unsigned b) { unsigned y; asm volatile("mul.rn.f16x2 %0, %1, %2;" : "=r"(y) : "r"(a), "r"(b)); return y; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  if (MODE == 2) {  // MUFU.EX2 on packed f16x2: two exponentials per instruction
    unsigned h[8];
    for (int i = 0; i < 8; ++i) h[i] = 0x3c00bc00u + threadIdx.x + i;
    const unsigned mh = 0xb800b800u;  // -0.5, -0.5
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) h[i] = hmul2(ex2h2(h[i]), mh);
    }
    long long t1 = clock64();
    unsigned s = 0; for (int i = 0; i < 8; ++i) s ^= h[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(s);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    return;
  }
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) * -0.5f;         // MUFU + FMUL
      else a[i] = fmaf(a[i], 0.999f, 1e-7f);           // FMA only
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, warps * 32>>>(out, cyc, iters);
        else if (mode == 1) k<1><<<148, warps * 32>>>(out, cyc, iters);
        else k<2><<<148, warps * 32>>>(out, cyc, iters);
        cudaDeviceSynchronize();
      }
      long long h[148]; cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
      double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
      const double per_smsp_warps = warps / 4.0;
      // instructions per warp: iters*8 (MUFU or FFMA); per SMSP: warps/4 * that
      printf("%s warps/SM=%2d: %.2f cycles per warp-instruction per SMSP\n",
             mode == 0 ? "MUFU.EX2(+FMUL)     " : mode == 1 ? "FFMA                " : "MUFU.EX2.F16x2(+HMUL2)",
             warps, c / (iters * 8.0 * per_smsp_warps));
    }
  }
  return 0;
}
