// The producer side of the layer fused into the Ulysses pack:
// MMDiT joint attention applies RMSNorm to each Q and K head row and rotary position
// embedding before attention (FLUX QK-norm + RoPE).  Instead of a norm
// kernel, a RoPE kernel and the pack (three HBM round trips), one pass reads the
// projected row, normalizes, rotates and writes it straight into its destination's
// all-to-all slot (or into the attention operand when U = 1).
//
// One warp per (b, h, s) row of D = 128: each lane owns 4 consecutive elements = 2 RoPE
// pairs.  RMSNorm in f32: y = x * rsqrt(mean(x^2) + eps) * w.  RoPE on interleaved pairs
// (x0, x1) at position p: (x0 cos - x1 sin, x0 sin + x1 cos) with cos/sin[p][pair].
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include <vector>

#include "fastusp_internal.h"

namespace fusp {
namespace {


__device__ __forceinline__ void load4(const void* p, int dt, int64_t i, float* f) {
  if (dt == FUSP_F32) {
    const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(p) + i);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  } else {
    const uint2 w = *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(p) + i);
    if (dt == FUSP_BF16) {
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
      f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    } else {
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
      f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
    }
  }
}

__device__ __forceinline__ void store4(void* p, int dt, int64_t i, const float* f) {
  if (dt == FUSP_F32) {
    *reinterpret_cast<float4*>(static_cast<float*>(p) + i) = make_float4(f[0], f[1], f[2], f[3]);
  } else if (dt == FUSP_BF16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]), b = __floats2bfloat162_rn(f[2], f[3]);
    *reinterpret_cast<uint2*>(static_cast<uint16_t*>(p) + i) =
        make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  } else {
    __half2 a = __floats2half2_rn(f[0], f[1]), b = __floats2half2_rn(f[2], f[3]);
    *reinterpret_cast<uint2*>(static_cast<uint16_t*>(p) + i) =
        make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

struct ProOp {
  const void* src;
  void* dst;
  const float* w;     // RMSNorm weight [D] or null
  const float* cosv;  // RoPE tables [rows][D/2] or null (null: plain pack, e.g. V)
  const float* sinv;
  int sdt, ddt;
};
struct ProArgs {
  ProOp op[3];
  int64_t slot_stride;  // destination elements between slots
  int h, hp, sl;
  int rows;             // B * H * SL
  float eps;
  int64_t pos0;
  int peer;             // slot t at slot_boff[t] bytes from slot 0 (the members' peer windows)
  int64_t slot_boff[kMaxPeerChunks];
};

// src [B][H][SL][D] -> dst slot t = h / hp: [B][hp][SL][D] at t * slot_stride (elements);
// grid.y = operand (Q, K and, in the same launch, V as a plain pack).
__global__ void __launch_bounds__(256) norm_rope_pack_kernel(const __grid_constant__ ProArgs a) {
  constexpr int D = 128;
  const ProOp& o = a.op[blockIdx.y];
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < a.rows;
       row += (gridDim.x * blockDim.x) >> 5) {
    const int bh = row / a.sl;
    const int s = row - bh * a.sl;
    const int bb = bh / a.h;
    const int hh = bh - bb * a.h;
    float x[4];
    load4(o.src, o.sdt, int64_t(row) * D + lane * 4, x);
    if (o.w != nullptr) {  // RMSNorm over the head dim
      float ss = x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
      const float r = rsqrtf(ss * (1.0f / D) + a.eps);
      const float4 wv = *reinterpret_cast<const float4*>(o.w + lane * 4);
      x[0] *= r * wv.x;
      x[1] *= r * wv.y;
      x[2] *= r * wv.z;
      x[3] *= r * wv.w;
    }
    if (o.cosv != nullptr) {  // RoPE on the two interleaved pairs this lane owns
      const int64_t pos = a.pos0 + s;
      const float2 c = *reinterpret_cast<const float2*>(o.cosv + pos * (D / 2) + lane * 2);
      const float2 n = *reinterpret_cast<const float2*>(o.sinv + pos * (D / 2) + lane * 2);
      const float y0 = x[0] * c.x - x[1] * n.x, y1 = x[0] * n.x + x[1] * c.x;
      const float y2 = x[2] * c.y - x[3] * n.y, y3 = x[2] * n.y + x[3] * c.y;
      x[0] = y0; x[1] = y1; x[2] = y2; x[3] = y3;
    }
    const int t = hh / a.hp, hl = hh - t * a.hp;
    const int64_t slot0 = a.peer ? a.slot_boff[t] / (o.ddt == FUSP_F32 ? 4 : 2) : t * a.slot_stride;
    const int64_t dst = slot0 + ((int64_t(bb) * a.hp + hl) * a.sl + s) * D + lane * 4;
    store4(o.dst, o.ddt, dst, x);
  }
  if (a.peer) __threadfence_system();  // remote stores visible before the exchange signal
}

}  // namespace

fusp_status launch_norm_rope_pack_multi(const ProPack* ops, int n, int64_t slot_stride, int b,
                                        int h, int sl, int d, int u, float eps, int64_t pos0,
                                        cudaStream_t s, const int64_t* peer_slot_boff) {
  if (d != 128) return set_error(FUSP_ERR_SHAPE, "qk prologue: head dim must be 128");
  if (n < 1 || n > 3) return set_error(FUSP_ERR_INVALID_ARGUMENT, "qk prologue: 1..3 operands");
  const int64_t rows = int64_t(b) * h * sl;
  if (rows <= 0) return FUSP_OK;
  if (rows >= (int64_t(1) << 31)) return set_error(FUSP_ERR_SHAPE, "qk prologue: too many rows");
  ProArgs a{};
  for (int i = 0; i < n; ++i)
    a.op[i] = ProOp{ops[i].src, ops[i].dst, ops[i].w, ops[i].cosv, ops[i].sinv, ops[i].sdt, ops[i].ddt};
  a.slot_stride = slot_stride;
  a.h = h;
  a.hp = h / u;
  a.sl = sl;
  a.rows = static_cast<int>(rows);
  a.eps = eps;
  a.pos0 = pos0;
  if (peer_slot_boff != nullptr) {
    if (u > kMaxPeerChunks) return set_error(FUSP_ERR_UNSUPPORTED, "qk prologue: too many peer slots");
    a.peer = 1;
    for (int t = 0; t < u; ++t) {
      if (peer_slot_boff[t] % 16 != 0) return set_error(FUSP_ERR_INVALID_ARGUMENT, "qk prologue: misaligned peer slot");
      a.slot_boff[t] = peer_slot_boff[t];
    }
  }
  int64_t grid = (rows * 32 + 255) / 256;
  const int64_t cap = (int64_t(sm_count()) * 16 + n - 1) / n;
  if (grid > cap) grid = cap;
  norm_rope_pack_kernel<<<dim3(static_cast<unsigned>(grid), n), 256, 0, s>>>(a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "norm_rope_pack_kernel");
  return FUSP_OK;
}

fusp_status launch_norm_rope_pack(const void* src, int sdt, void* dst, int ddt,
                                  int64_t slot_stride, int b, int h, int sl, int d, int u,
                                  const float* w, float eps, const float* cosv, const float* sinv,
                                  int64_t pos0, cudaStream_t s, const int64_t* peer_slot_boff) {
  const ProPack op{src, dst, w, cosv, sinv, sdt, ddt};
  return launch_norm_rope_pack_multi(&op, 1, slot_stride, b, h, sl, d, u, eps, pos0, s, peer_slot_boff);
}

// Every kernel of this file, for preload_kernels() (lazy module loading, see runtime.cpp).
void append_kernels_prologue(std::vector<const void*>& v) {
  v.push_back(reinterpret_cast<const void*>(norm_rope_pack_kernel));
}

}  // namespace fusp
