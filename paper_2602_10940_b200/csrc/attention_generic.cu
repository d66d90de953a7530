// Attention for head dims other than 128 (D a multiple of 8, up to 256): the reference's
// attention_core (tensor.cpp:143-181) is generic in D, and SPEC.md's parity grids use small
// D.  The tcgen05 kernel (attention_sm100.cu) is specialised for D = 128 (the north-star
// FLUX / Qwen shapes); every other D runs here, on CUDA cores in f32 -- the reference's own
// arithmetic type, so the results match it to f32 rounding, whatever the magnitudes.
//
// One warp per query row, 8 rows per CTA sharing K / V tiles of 32 keys in shared memory.
// Per tile, lane j scores key j (a D-long dot product against the row's q in shared memory),
// the warp updates the online-softmax state (row max and sum through shuffles), and each lane
// accumulates the D/32 output dimensions it owns.  Same interface as the tcgen05 launch:
// chunked output / LSE addressing (Ulysses slots), the fused merge_lse into a running
// accumulator (ring steps), f32 / f16 / bf16 operands and outputs.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>

#include <vector>

#include "fastusp_internal.h"

namespace fusp {
namespace {

constexpr int kGRows = 8;   // query rows (warps) per CTA
constexpr int kGKeys = 32;  // keys per shared-memory tile
constexpr int kGMaxD = 256;

__device__ __forceinline__ float ld_any(const void* p, int dt, int64_t i) {
  switch (dt) {
    case FUSP_F32: return static_cast<const float*>(p)[i];
    case FUSP_F16: return __half2float(static_cast<const __half*>(p)[i]);
    default: return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  }
}
__device__ __forceinline__ void st_any(void* p, int dt, int64_t i, float v) {
  switch (dt) {
    case FUSP_F32: static_cast<float*>(p)[i] = v; break;
    case FUSP_F16: static_cast<__half*>(p)[i] = __float2half_rn(v); break;
    default: static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v); break;
  }
}

struct GParams {
  const void *q, *k, *v;
  int qdt, kdt, vdt;
  int64_t q_hs, k_hs, v_hs;  // element strides between heads (rows are d apart)
  int sq, skv, d;
  float scale;               // 1/sqrt(D)
  void* out;
  int out_dtype, out_chunk;
  int64_t out_hs, out_cs, out_rs;
  float* lse;
  int64_t lse_hs, lse_cs;
  const float* acc_o;        // merge into the running (acc_o, acc_lse) when non-null
  const float* acc_lse;
};

// grid (ceil(sq / kGRows), heads), kGRows warps
__global__ void __launch_bounds__(kGRows * 32) attn_generic_kernel(const GParams p) {
  extern __shared__ float gsm[];
  const int d = p.d;
  float* ks = gsm;                      // [kGKeys][d]
  float* vs = ks + kGKeys * d;          // [kGKeys][d]
  float* qs = vs + kGKeys * d;          // [kGRows][d]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int row = blockIdx.x * kGRows + warp;
  const bool live = row < p.sq;
  for (int i = lane; i < d; i += 32)
    qs[warp * d + i] = live ? ld_any(p.q, p.qdt, head * p.q_hs + int64_t(row) * d + i) : 0.f;
  constexpr int kPer = kGMaxD / 32;  // output dims per lane (lane, lane + 32, ...)
  float o[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) o[i] = 0.f;
  float m = -INFINITY, l = 0.f;
  for (int k0 = 0; k0 < p.skv; k0 += kGKeys) {
    __syncthreads();  // the previous tile is consumed (and q is written, first time)
    const int nk = p.skv - k0 < kGKeys ? p.skv - k0 : kGKeys;
    for (int i = threadIdx.x; i < nk * d; i += blockDim.x) {
      ks[i] = ld_any(p.k, p.kdt, head * p.k_hs + int64_t(k0) * d + i);
      vs[i] = ld_any(p.v, p.vdt, head * p.v_hs + int64_t(k0) * d + i);
    }
    __syncthreads();
    float s = -INFINITY;
    if (lane < nk) {
      float acc = 0.f;
      const float* kr = ks + lane * d;
      const float* qr = qs + warp * d;
      for (int i = 0; i < d; ++i) acc = fmaf(qr[i], kr[i], acc);
      s = acc * p.scale;  // (q.k) * 1/sqrt(D), as tensor.cpp:147
    }
    float tmax = s;
    for (int off = 16; off > 0; off >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
    const float m_new = fmaxf(m, tmax);
    const float alpha = m == -INFINITY ? 0.f : expf(m - m_new);
    const float pj = lane < nk ? expf(s - m_new) : 0.f;
    float psum = pj;
    for (int off = 16; off > 0; off >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
    l = l * alpha + psum;
    m = m_new;
#pragma unroll
    for (int i = 0; i < kPer; ++i) o[i] *= alpha;
    for (int j = 0; j < nk; ++j) {
      const float w = __shfl_sync(0xffffffffu, pj, j);
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int dd = lane + 32 * i;
        if (dd < d) o[i] = fmaf(w, vs[j * d + dd], o[i]);
      }
    }
  }
  if (!live) return;
  const float lse_b = m + logf(l);  // natural log (tensor.cpp:177)
  const float inv_l = 1.f / l;
  float c_acc = 0.f, c_new = 1.f, lse_out = lse_b;
  if (p.acc_o != nullptr) {  // merge_lse(acc, part) (tensor.cpp:219-240), identity rows pass
    const float l1 = p.acc_lse[int64_t(head) * p.sq + row];
    if (lse_b == -INFINITY) {
      c_acc = 1.f; c_new = 0.f; lse_out = l1;
    } else if (l1 == -INFINITY) {
      c_acc = 0.f; c_new = 1.f; lse_out = lse_b;
    } else {
      const float mm = l1 > lse_b ? l1 : lse_b;
      lse_out = mm + logf(expf(l1 - mm) + expf(lse_b - mm));
      c_acc = expf(l1 - lse_out);
      c_new = expf(lse_b - lse_out);
    }
  }
  const int64_t ob = int64_t(head) * p.out_hs + int64_t(row / p.out_chunk) * p.out_cs +
                     int64_t(row % p.out_chunk) * p.out_rs;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int dd = lane + 32 * i;
    if (dd >= d) continue;
    float y = o[i] * inv_l * c_new;
    if (p.acc_o != nullptr) y = fmaf(c_acc, p.acc_o[(int64_t(head) * p.sq + row) * d + dd], y);
    st_any(p.out, p.out_dtype, ob + dd, y);
  }
  if (lane == 0 && p.lse != nullptr)
    p.lse[int64_t(head) * p.lse_hs + int64_t(row / p.out_chunk) * p.lse_cs + row % p.out_chunk] = lse_out;
}

}  // namespace

fusp_status launch_attention_generic(const AttnLaunch& a, cudaStream_t stream) {
  if (a.d < 8 || a.d > kGMaxD || a.d % 8 != 0)
    return set_error(FUSP_ERR_SHAPE, "attention: head dim D=" + std::to_string(a.d) +
                                         " unsupported (D = 128 on tcgen05; other D a multiple of 8 up to 256)");
  if (a.sq <= 0 || a.heads <= 0) return FUSP_OK;
  if (a.skv <= 0) return set_error(FUSP_ERR_SHAPE, "attention kernel: empty KV (caller handles it)");
  if (a.heads > 65535) return set_error(FUSP_ERR_SHAPE, "attention: too many heads");
  GParams p{};
  p.q = a.q;
  p.k = a.k;
  p.v = a.v;
  p.qdt = a.qk_dtype;
  p.kdt = a.k_dtype >= 0 ? a.k_dtype : a.qk_dtype;
  p.vdt = a.v_dtype;
  p.q_hs = a.q_hs;
  p.k_hs = a.k_hs;
  p.v_hs = a.v_hs;
  p.sq = a.sq;
  p.skv = a.skv;
  p.d = a.d;
  p.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(a.d)));
  p.out = a.out;
  p.out_dtype = a.out_dtype;
  p.out_chunk = a.out_chunk > 0 ? a.out_chunk : a.sq;
  p.out_hs = a.out_hs;
  p.out_cs = a.out_cs;
  p.out_rs = a.out_rs;
  p.lse = a.lse;
  p.lse_hs = a.lse_hs;
  p.lse_cs = a.lse_cs;
  p.acc_o = a.acc_o;
  p.acc_lse = a.acc_lse;
  const int smem = static_cast<int>(sizeof(float)) * (2 * kGKeys + kGRows) * a.d;
  FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(attn_generic_kernel), smem, "attn_generic_kernel"));
  attn_generic_kernel<<<dim3((a.sq + kGRows - 1) / kGRows, a.heads), kGRows * 32, smem, stream>>>(p);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "attn_generic_kernel launch");
  return FUSP_OK;
}

// Every kernel of this file, for preload_kernels() (lazy module loading, see runtime.cpp).
void append_kernels_attention_generic(std::vector<const void*>& v) {
  v.push_back(reinterpret_cast<const void*>(attn_generic_kernel));
}

}  // namespace fusp
