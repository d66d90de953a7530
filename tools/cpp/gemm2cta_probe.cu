// Probe for a 2-CTA (cta_group::2) tcgen05 GEMM: C[M][N] f32 = A[M][K] (K-major bf16) x
// B[K][N] (N-major bf16, like W_qkv / W_o), tile 256 x 256 per CTA pair (128 rows per CTA,
// each CTA holding half of B's 256 columns), checked against a naive GPU GEMM and timed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 gemm2cta_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2602_10940_b200/csrc/sm100_ptx.cuh"

using namespace fusp::ptx;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int kM = 128, kN = 256, kK = 64, kStages = 6, kThreads = 384;
constexpr uint32_t kABytes = kM * kK * 2;          // 16 KB: this CTA's 128 rows
constexpr uint32_t kBBytes = (kN / 2) * kK * 2;    // 16 KB: this CTA's 128 of the 256 columns
constexpr uint32_t kBChunk = 64 * kK * 2;          // 8 KB [64 k][64 n]

struct __align__(1024) Smem {
  uint8_t a[kStages][kABytes];
  uint8_t b[kStages][kBBytes];
  uint64_t full[kStages], empty[kStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2(uint64_t* bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

struct Args {
  int m_tiles, n_tiles, k_blocks, m, n, nostore;
  uint32_t idesc;
  float* c;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b, const Args p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int pairs = ((p.m_tiles + 1) / 2) * p.n_tiles;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 2);  // both producers arrive (leader with the pair's tx bytes)
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.acc_full[b], 1);
      mbar_init(&sm.acc_empty[b], 2);  // one arrive per CTA's epilogue
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tm_a);
      prefetch_tmap(&tm_b);
      uint32_t it = 0;
      for (int pr = cluster; pr < pairs; pr += nclusters) {
        const int nt = pr % p.n_tiles;
        const int mt = (pr / p.n_tiles) * 2 + static_cast<int>(rank);
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int st = it % kStages;
          mbar_wait(&sm.empty[st], ((it / kStages) & 1) ^ 1);
          const uint32_t full_leader = mapa(smem_u32(&sm.full[st]), 0);
          if (leader) mbar_expect_tx(&sm.full[st], 2 * (kABytes + kBBytes));
          else mbar_arrive_cluster(full_leader);
          tma_load_2d_2sm(sm.a[st], &tm_a, full_leader, kb * kK, mt * kM);
          for (int c = 0; c < 2; ++c)
            tma_load_2d_2sm(sm.b[st] + c * kBChunk, &tm_b, full_leader, nt * kN + static_cast<int>(rank) * 128 + c * 64,
                            kb * kK);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      uint32_t it = 0, lt = 0;
      for (int pr = cluster; pr < pairs; pr += nclusters, ++lt) {
        const int ab = lt & 1;
        mbar_wait(&sm.acc_empty[ab], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * kN;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int st = it % kStages;
          mbar_wait(&sm.full[st], (it / kStages) & 1);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(smem_u32(sm.a[st]), 16, 1024);
          const uint64_t bdesc = umma_desc_sw128(smem_u32(sm.b[st]), kBChunk, 1024);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kK / 16; ++k)
              mma2(d, adesc + uint64_t(k * 32 / 16), bdesc + uint64_t(k * 16 * 128 / 16), p.idesc,
                   (kb > 0 || k > 0) ? 1u : 0u);
            commit2(&sm.empty[st]);
          }
          __syncwarp();
        }
        if (elect_one()) commit2(&sm.acc_full[ab]);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int quad = warp & 3, eg = (warp - 4) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t acc_empty_leader0 = mapa(smem_u32(&sm.acc_empty[0]), 0);
    const uint32_t acc_empty_leader1 = mapa(smem_u32(&sm.acc_empty[1]), 0);
    uint32_t lt = 0;
    for (int pr = cluster; pr < pairs; pr += nclusters, ++lt) {
      const int ab = lt & 1;
      const int nt = pr % p.n_tiles;
      const int mt = (pr / p.n_tiles) * 2 + static_cast<int>(rank);
      mbar_wait(&sm.acc_full[ab], (lt >> 1) & 1);
      tc_fence_after();
      const int row = mt * kM + r;
      for (int c = eg * 4; c < eg * 4 + 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + ab * kN + c * 32, v);
        tmem_wait_ld();
        if (!p.nostore && row < p.m && mt < p.m_tiles) {
          float* y = p.c + static_cast<int64_t>(row) * p.n + nt * kN + c * 32;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(y)[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                          __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 128) mbar_arrive_cluster(ab ? acc_empty_leader1 : acc_empty_leader0);
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// 1-CTA comparison: the same pipeline with cta_group::1, 128 x 256 per CTA, full B per CTA
constexpr int kStages1 = 4;
struct __align__(1024) Smem1 {
  uint8_t a[kStages1][kABytes];
  uint8_t b[kStages1][2 * kBBytes];
  uint64_t full[kStages1], empty[kStages1];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};
__global__ void __launch_bounds__(kThreads, 1)
    gemm1(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b, const Args p) {
  extern __shared__ uint8_t smem_raw[];
  Smem1& sm = *reinterpret_cast<Smem1*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const int tiles = p.m_tiles * p.n_tiles;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages1; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.acc_full[b], 1);
      mbar_init(&sm.acc_empty[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int nt = t % p.n_tiles, mt = t / p.n_tiles;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
          const int st = it % kStages1;
          mbar_wait(&sm.empty[st], ((it / kStages1) & 1) ^ 1);
          mbar_expect_tx(&sm.full[st], kABytes + 2 * kBBytes);
          tma_load_2d(sm.a[st], &tm_a, &sm.full[st], kb * kK, mt * kM);
          for (int c = 0; c < 4; ++c)
            tma_load_2d(sm.b[st] + c * kBChunk, &tm_b, &sm.full[st], nt * kN + c * 64, kb * kK);
        }
      }
    }
  } else if (warp == 1) {
    uint32_t it = 0, lt = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      const int ab = lt & 1;
      mbar_wait(&sm.acc_empty[ab], ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < p.k_blocks; ++kb, ++it) {
        const int st = it % kStages1;
        mbar_wait(&sm.full[st], (it / kStages1) & 1);
        tc_fence_after();
        const uint64_t adesc = umma_desc_sw128(smem_u32(sm.a[st]), 16, 1024);
        const uint64_t bdesc = umma_desc_sw128(smem_u32(sm.b[st]), kBChunk, 1024);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kK / 16; ++k)
            mma_ss(tmem + ab * kN, adesc + uint64_t(k * 32 / 16), bdesc + uint64_t(k * 16 * 128 / 16), p.idesc,
                   (kb > 0 || k > 0) ? 1u : 0u);
          mma_commit(&sm.empty[st]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&sm.acc_full[ab]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int quad = warp & 3, eg = (warp - 4) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      const int ab = lt & 1, nt = t % p.n_tiles, mt = t / p.n_tiles;
      mbar_wait(&sm.acc_full[ab], (lt >> 1) & 1);
      tc_fence_after();
      const int row = mt * kM + r;
      for (int c = eg * 4; c < eg * 4 + 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + ab * kN + c * 32, v);
        tmem_wait_ld();
        if (!p.nostore && row < p.m) {
          float* y = p.c + static_cast<int64_t>(row) * p.n + nt * kN + c * 32;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(y)[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                          __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 128) mbar_arrive(&sm.acc_empty[ab]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

__global__ void ref_gemm(const __nv_bfloat16* a, const __nv_bfloat16* b, float* c, int m, int n, int k) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j >= n) return;
  float s = 0.f;
  for (int t = 0; t < k; ++t) s += __bfloat162float(a[int64_t(i) * k + t]) * __bfloat162float(b[int64_t(t) * n + j]);
  c[int64_t(i) * n + j] = s;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 4608, n = argc > 2 ? atoi(argv[2]) : 9216, k = argc > 3 ? atoi(argv[3]) : 3072;
  std::vector<__nv_bfloat16> ha(size_t(m) * k), hb(size_t(k) * n);
  srand(1);
  for (auto& x : ha) x = __float2bfloat16((rand() % 2001 - 1000) / 1000.f);
  for (auto& x : hb) x = __float2bfloat16((rand() % 2001 - 1000) / 50000.f);
  __nv_bfloat16 *a, *b;
  float *c, *cr;
  CK(cudaMalloc(&a, ha.size() * 2));
  CK(cudaMalloc(&b, hb.size() * 2));
  CK(cudaMalloc(&c, size_t(m) * n * 4));
  CK(cudaMalloc(&cr, size_t(m) * n * 4));
  CK(cudaMemcpy(a, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
  CUtensorMap ta, tb;
  {
    cuuint64_t dims[2] = {cuuint64_t(k), cuuint64_t(m)}, str[1] = {cuuint64_t(k) * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 2;
  }
  {
    cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(k)}, str[1] = {cuuint64_t(n) * 2};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 3;
  }
  Args p{};
  p.m_tiles = (m + kM - 1) / kM;
  p.n_tiles = n / kN;
  p.k_blocks = k / kK;
  p.m = m;
  p.n = n;
  p.idesc = idesc_f16(1, 1, 0, 1, 256, kN);
  p.nostore = getenv("NOSTORE") != nullptr;
  p.c = c;
  const bool one = getenv("ONE") != nullptr;
  const int smem = one ? int(sizeof(Smem1)) + 1024 : int(sizeof(Smem)) + 1024;
  CK(cudaFuncSetAttribute(gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(Smem)) + 1024));
  CK(cudaFuncSetAttribute(gemm1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(Smem1)) + 1024));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int pairs = ((p.m_tiles + 1) / 2) * p.n_tiles;
  int max_clusters = 0;
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((sms / 2) * 2);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.dynamicSmemBytes = sizeof(Smem) + 1024;
    CK(cudaOccupancyMaxActiveClusters(&max_clusters, gemm2, &cfg));
  }
  int grid = (sms / 2) * 2;
  if (getenv("CLUSTERS")) grid = 2 * atoi(getenv("CLUSTERS"));
  else if (max_clusters > 0 && 2 * max_clusters < grid) grid = 2 * max_clusters;
  fprintf(stderr, "max active clusters %d, grid %d\n", max_clusters, grid);
  if (pairs * 2 < grid) grid = pairs * 2;
  if (one) p.idesc = idesc_f16(1, 1, 0, 1, 128, kN);
  auto launch = [&] {
    if (one) gemm1<<<sms, kThreads, smem>>>(ta, tb, p);
    else gemm2<<<grid, kThreads, smem>>>(ta, tb, p);
  };
  launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  ref_gemm<<<dim3((n + 255) / 256, m), 256>>>(a, b, cr, m, n, k);
  CK(cudaDeviceSynchronize());
  std::vector<float> h1(size_t(m) * n), h2(size_t(m) * n);
  CK(cudaMemcpy(h1.data(), c, h1.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2.data(), cr, h2.size() * 4, cudaMemcpyDeviceToHost));
  double num = 0, den = 0;
  for (size_t i = 0; i < h1.size(); ++i) {
    num += (h1[i] - h2[i]) * double(h1[i] - h2[i]);
    den += double(h2[i]) * h2[i];
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) launch();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / 20, tf = 2.0 * m * n * k / (us * 1e-6) / 1e12;
  printf("{\"probe\": \"%s\", \"m\": %d, \"n\": %d, \"k\": %d, \"rel_l2\": %.3e, \"us\": %.1f, \"tflops\": %.1f}\n",
         one ? "gemm 1-CTA 128x256" : "gemm 2-CTA 256x256", m, n, k, std::sqrt(num / den), us, tf);
  return 0;
}
