// HBM-bound kernels of the USP layer: dtype conversion, the E4M3 codec and the per-tensor
// quantizer (bit-exact with the reference), the LSE merge, and the Ulysses pack/unpack.
//
// Grids are sized as a multiple of the 148 SMs and loop grid-stride; all global accesses
// are 16-byte vectors where the layout allows.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cmath>
#include <cstdint>

#include <vector>

#include "fastusp_internal.h"

namespace fusp {
namespace {

constexpr int kBlock = 256;
#ifndef FUSP_FP8_UNROLL
#define FUSP_FP8_UNROLL 8
#endif
constexpr int kFp8Unroll = FUSP_FP8_UNROLL;  // raw vectors in flight per thread (FP8 passes)
constexpr int kE4Unroll = 4;  // 16-code loads in flight per thread (E4M3 sources)

// Programmatic dependent launch (PDL): the kernel may become resident while the previous
// kernel on `s` drains; it must execute griddepcontrol.wait before touching that kernel's output.
template <typename Args>
cudaError_t launch_pdl(void (*kernel)(Args), dim3 grid, cudaStream_t s, const Args& args,
                       int block = 256) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args);
}

inline int grid_for(int64_t work_items, int per_sm = 8) {  // grid-stride kernels
  int64_t g = (work_items + kBlock - 1) / kBlock;
  if (g > int64_t(sm_count()) * per_sm) g = int64_t(sm_count()) * per_sm;
  return g < 1 ? 1 : static_cast<int>(g);
}

__device__ __forceinline__ float load_as_f32(const void* p, int dt, int64_t i) {
  switch (dt) {
    case FUSP_F32: return static_cast<const float*>(p)[i];
    case FUSP_F16: return __half2float(static_cast<const __half*>(p)[i]);
    default: return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  }
}
__device__ __forceinline__ void store_from_f32(void* p, int dt, int64_t i, float v) {
  switch (dt) {
    case FUSP_F32: static_cast<float*>(p)[i] = v; break;
    case FUSP_F16: static_cast<__half*>(p)[i] = __float2half_rn(v); break;
    default: static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v); break;
  }
}

// E4M3 encode == reference encode_e4m3 (fp8.cpp:45-68): hardware RNE satfinite cvt is
// bit-identical on every finite f32; NaN keeps its sign bit (0x7F / 0xFF).
__device__ __forceinline__ uint8_t enc_e4m3(float x) {
  if (isnan(x)) return signbit(x) ? 0xFF : 0x7F;
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.f), "f"(x));
  return static_cast<uint8_t>(r & 0xFF);
}
// Exact decode (fp8.cpp:39-43): sign | (exp==0 ? m*2^-9 : (8+m)*2^(e-10)); 0x7F/0xFF -> NaN.
__device__ __forceinline__ float dec_e4m3(uint8_t c) {
  const int e = (c >> 3) & 0xF, m = c & 7;
  float mag;
  if ((c & 0x7F) == 0x7F) mag = __int_as_float(0x7fc00000);
  else if (e == 0) mag = ldexpf(static_cast<float>(m), -9);
  else mag = ldexpf(static_cast<float>(8 + m), e - 10);
  return (c & 0x80) ? -mag : mag;
}

__global__ void convert_kernel(const void* __restrict__ x, int xdt, void* __restrict__ y, int ydt,
                               int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    store_from_f32(y, ydt, i, load_as_f32(x, xdt, i));
}

// bf16 -> f16 specialisation, 8 elements (16 B) per thread.
__global__ void bf16_to_f16_kernel(const uint4* __restrict__ x, uint4* __restrict__ y, int64_t n8) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8;
       i += int64_t(gridDim.x) * blockDim.x) {
    uint4 v = x[i];
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&w[e]);
      float2 f = __bfloat1622float2(b);
      __half2 h = __floats2half2_rn(f.x, f.y);
      w[e] = *reinterpret_cast<uint32_t*>(&h);
    }
    y[i] = v;
  }
}

__global__ void encode_kernel(const float* __restrict__ x, int64_t n, uint8_t* __restrict__ c) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    c[i] = enc_e4m3(x[i]);
}

__global__ void decode_kernel(const uint8_t* __restrict__ c, int64_t n, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = dec_e4m3(c[i]);
}

// Pass 1 of quantize (fp8.cpp:108-117): max|x| and a non-finite flag.
__global__ void amax_kernel(const void* __restrict__ x, int dt, int64_t n,
                            uint32_t* __restrict__ amax_bits, uint32_t* __restrict__ nonfinite) {
  float m = 0.f;
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float v = load_as_f32(x, dt, i);
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  bad = __any_sync(0xffffffffu, bad);
  __shared__ float wm[kBlock / 32];
  __shared__ int wb[kBlock / 32];
  if ((threadIdx.x & 31) == 0) {
    wm[threadIdx.x >> 5] = m;
    wb[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bm = 0.f;
    int bb = 0;
    for (int w = 0; w < kBlock / 32; ++w) {
      bm = fmaxf(bm, wm[w]);
      bb |= wb[w];
    }
    if (!(bm >= 0.f)) bm = 0.f;  // NaN max is reported through the flag
    atomicMax(amax_bits, __float_as_uint(bm));
    if (bb) atomicOr(nonfinite, 1u);
  }
}

// Pass 2 (fp8.cpp:119-121): scale = max/448 (1 if 0), codes = encode(x / scale), IEEE division.
__global__ void quantize_kernel(const void* __restrict__ x, int dt, int64_t n,
                                const uint32_t* __restrict__ amax_bits, float* __restrict__ scale_out,
                                uint8_t* __restrict__ codes) {
  const float amax = __uint_as_float(*amax_bits);
  const float scale = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    codes[i] = enc_e4m3(__fdiv_rn(load_as_f32(x, dt, i), scale));
}

__global__ void dequantize_kernel(const uint8_t* __restrict__ c, const float* __restrict__ scale,
                                  int64_t n, void* __restrict__ y, int ydt) {
  const float s = *scale;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    store_from_f32(y, ydt, i, __fmul_rn(dec_e4m3(c[i]), s));
}

// merge_lse (tensor.cpp:204-243): one warp per row, identity rows copied through.
__global__ void merge_kernel(const float* __restrict__ o1, const float* __restrict__ l1,
                             const float* __restrict__ o2, const float* __restrict__ l2,
                             int64_t rows, int d, float* out, float* lse) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; r < rows;
       r += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const float a = l1[r], b = l2[r];
    float c1 = 1.f, c2 = 0.f, ln;
    int ident = 0;  // 1: take o1 (b is the identity), 2: take o2
    if (b == -INFINITY) { ident = 1; ln = a; }
    else if (a == -INFINITY) { ident = 2; ln = b; }
    else {
      const float m = a > b ? a : b;
      ln = m + logf(expf(a - m) + expf(b - m));
      c1 = expf(a - ln);
      c2 = expf(b - ln);
    }
    const float* x1 = o1 + r * d;
    const float* x2 = o2 + r * d;
    float* y = out + r * d;
    for (int i = lane; i < d; i += 32) {
      const float v1 = x1[i], v2 = x2[i];
      y[i] = ident == 1 ? v1 : ident == 2 ? v2 : __fadd_rn(__fmul_rn(c1, v1), __fmul_rn(c2, v2));
    }
    __syncwarp();
    if (lane == 0) lse[r] = ln;
  }
}

__global__ void fill_kernel(void* p, int dt, int64_t n, float v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    store_from_f32(p, dt, i, v);
}

// Ulysses pack (protocols.cpp:143-153): destination slot t takes heads [t*hp, (t+1)*hp).
// One thread per 8 consecutive d-elements.
__global__ void pack_kernel(const void* __restrict__ src, int sdt, void* __restrict__ dst, int ddt,
                            int64_t slot_stride, int b, int h, int sl, int d, int u,
                            const float* __restrict__ scale, int64_t scale_bh_stride) {
  const int hp = h / u;
  const int64_t n = int64_t(b) * h * sl * d;  // multiple of 8 (d % 8 == 0)
  for (int64_t v8 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v8 < n / 8;
       v8 += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = v8 * 8;
    const int64_t row = i / d;       // (b, h, s) flattened
    const int dd = static_cast<int>(i - row * d);
    const int s = static_cast<int>(row % sl);
    const int64_t bh = row / sl;
    const int hh = static_cast<int>(bh % h);
    const int bb = static_cast<int>(bh / h);
    const int t = hh / hp, hl = hh % hp;
    const int64_t o = t * slot_stride + ((int64_t(bb) * hp + hl) * sl + s) * d + dd;
    float f[8];
    if (sdt == FUSP_BF16) {
      const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(src) + i);
      const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(p2[e]);
        f[2 * e] = x.x;
        f[2 * e + 1] = x.y;
      }
    } else if (sdt == FUSP_F16) {
      const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const __half*>(src) + i);
      const __half2* p2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x = __half22float2(p2[e]);
        f[2 * e] = x.x;
        f[2 * e + 1] = x.y;
      }
    } else {
      const float4* p4 = reinterpret_cast<const float4*>(static_cast<const float*>(src) + i);
      const float4 a = p4[0], c = p4[1];
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
      f[4] = c.x; f[5] = c.y; f[6] = c.z; f[7] = c.w;
    }
    if (ddt == FUSP_E4M3) {
      // per-tensor (stride 0) or per-(b,h)-slab scale of the local tensor
      const float qs = scale[bh * scale_bh_stride];
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) lo |= uint32_t(enc_e4m3(__fdiv_rn(f[e], qs))) << (8 * e);
#pragma unroll
      for (int e = 0; e < 4; ++e) hi |= uint32_t(enc_e4m3(__fdiv_rn(f[4 + e], qs))) << (8 * e);
      *reinterpret_cast<uint2*>(static_cast<uint8_t*>(dst) + o) = make_uint2(lo, hi);
    } else if (ddt == FUSP_F32) {
      float4* q4 = reinterpret_cast<float4*>(static_cast<float*>(dst) + o);
      q4[0] = make_float4(f[0], f[1], f[2], f[3]);
      q4[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (ddt == FUSP_F16) {
          __half2 x = __floats2half2_rn(f[2 * e], f[2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&x);
        } else {
          __nv_bfloat162 x = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&x);
        }
      }
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dst) + o) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// Ulysses unpack (protocols.cpp:163-179): slot j (group position j) holds our heads over the
// j-th sequence block; destination [B][hp][U*SL][D] in group-position sequence order.
__global__ void unpack_kernel(const void* __restrict__ src, int sdt, int64_t slot_stride,
                              const float* __restrict__ scales, int64_t scale_stride,
                              int64_t scale_bh_stride, void* __restrict__ dst, int ddt, int b,
                              int hp, int sl, int d, int u) {
  const int64_t per_slot = int64_t(b) * hp * sl * d;
  const int64_t n = per_slot * u;
  const int64_t span = int64_t(u) * sl;
  for (int64_t v8 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v8 < n / 8;
       v8 += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = v8 * 8;
    const int j = static_cast<int>(i / per_slot);
    const int64_t r = i - j * per_slot;
    const int64_t row = r / d;
    const int dd = static_cast<int>(r - row * d);
    const int s = static_cast<int>(row % sl);
    const int64_t bh = row / sl;
    const int64_t o = (bh * span + int64_t(j) * sl + s) * d + dd;
    const int64_t si = j * slot_stride + r;
    if (sdt == FUSP_E4M3 && ddt == FUSP_E4M3) {
      *reinterpret_cast<uint2*>(static_cast<uint8_t*>(dst) + o) =
          *reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(src) + si);
      continue;
    }
    if (sdt == ddt) {
      if (sdt == FUSP_F32) {
        const float4* a = reinterpret_cast<const float4*>(static_cast<const float*>(src) + si);
        float4* z = reinterpret_cast<float4*>(static_cast<float*>(dst) + o);
        z[0] = a[0];
        z[1] = a[1];
      } else {
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dst) + o) =
            *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(src) + si);
      }
      continue;
    }
    float f[8];
    if (sdt == FUSP_E4M3) {
      const float sc = scales[j * scale_stride + bh * scale_bh_stride];
      const uint2 w = *reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(src) + si);
#pragma unroll
      for (int e = 0; e < 4; ++e) f[e] = __fmul_rn(dec_e4m3((w.x >> (8 * e)) & 0xFF), sc);
#pragma unroll
      for (int e = 0; e < 4; ++e) f[4 + e] = __fmul_rn(dec_e4m3((w.y >> (8 * e)) & 0xFF), sc);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = load_as_f32(src, sdt, si + e);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) store_from_f32(dst, ddt, o + e, f[e]);
  }
}

__global__ void unpack_heads_kernel(const uint8_t* __restrict__ src, int64_t slot_stride_bytes,
                                    uint8_t* __restrict__ dst, int esz, int b, int hp, int sl,
                                    int d, int u) {
  // src slot j: [B][hp][SL][D] -> dst [B][H=u*hp][SL][D]; 16-byte granules.
  const int64_t row_bytes = int64_t(sl) * d * esz;  // one (b,h) slab
  const int64_t per_slot = int64_t(b) * hp * row_bytes;
  const int64_t n16 = per_slot * u / 16;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n16;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = g * 16;
    const int j = static_cast<int>(i / per_slot);
    const int64_t r = i - j * per_slot;
    const int64_t slab = r / row_bytes;
    const int64_t off = r - slab * row_bytes;
    const int hl = static_cast<int>(slab % hp);
    const int bb = static_cast<int>(slab / hp);
    const int64_t o = ((int64_t(bb) * u * hp + int64_t(j) * hp + hl) * row_bytes) + off;
    *reinterpret_cast<uint4*>(dst + o) =
        *reinterpret_cast<const uint4*>(src + j * slot_stride_bytes + r);
  }
}

// ---- blocked FP8 (per-tensor = one block; per-(b,h)-slab = the B200 per-block option) ----
// Source value i: a float tensor, or an E4M3 chunk [bh][span][d] whose value is
// decode(code) * scales[(row / seg_rows) * seg_stride + bh * bh_stride] -- exactly the f32
// values the reference's dequantize produced (fp8.cpp:125-130), so re-quantizing them
// reproduces the reference's ring hops (protocols.cpp:113-115, :303-311) bit for bit.
__device__ __forceinline__ float src_value(const Fp8Src& s, int64_t i) {
  if (s.dt != FUSP_E4M3) return load_as_f32(s.x, s.dt, i);
  const int64_t row = i / s.d;
  const int64_t bh = row / s.span;
  const int r = static_cast<int>(row - bh * s.span);
  return __fmul_rn(dec_e4m3(static_cast<const uint8_t*>(s.x)[i]),
                   s.scales[(r / s.seg_rows) * s.seg_stride + bh * s.bh_stride]);
}

// Pass 1 (fp8.cpp:108-117) per block: grid.y = block, grid.x strides inside it.
__global__ void amax_blocks_kernel(Fp8Src s, int64_t block_elems, uint32_t* __restrict__ amax,
                                   uint32_t* __restrict__ nonfinite) {
  const int64_t base = int64_t(blockIdx.y) * block_elems;
  float m = 0.f;
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < block_elems;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float v = src_value(s, base + i);
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  bad = __any_sync(0xffffffffu, bad);
  __shared__ float wm[kBlock / 32];
  __shared__ int wb[kBlock / 32];
  if ((threadIdx.x & 31) == 0) {
    wm[threadIdx.x >> 5] = m;
    wb[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bm = 0.f;
    int bb = 0;
    for (int w = 0; w < kBlock / 32; ++w) {
      bm = fmaxf(bm, wm[w]);
      bb |= wb[w];
    }
    if (!(bm >= 0.f)) bm = 0.f;
    atomicMax(&amax[blockIdx.y], __float_as_uint(bm));
    if (bb && nonfinite) atomicOr(nonfinite, 1u);
  }
}

// scale = max/448, 1 for an all-zero block (fp8.cpp:119).
__global__ void finalize_scales_kernel(const uint32_t* __restrict__ amax, int nblocks,
                                       float* __restrict__ scales) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nblocks; k += gridDim.x * blockDim.x) {
    const float a = __uint_as_float(amax[k]);
    scales[k] = a > 0.f ? __fdiv_rn(a, 448.0f) : 1.0f;
  }
}

// Pass 2 (fp8.cpp:121): codes = encode(x / scale[block]), IEEE division.
__global__ void quantize_blocks_kernel(Fp8Src s, int64_t n, int64_t block_elems,
                                       const float* __restrict__ scales,
                                       uint8_t* __restrict__ codes) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    codes[i] = enc_e4m3(__fdiv_rn(src_value(s, i), scales[i / block_elems]));
}

__global__ void dequantize_blocks_kernel(const uint8_t* __restrict__ c,
                                         const float* __restrict__ scales, int64_t block_elems,
                                         int64_t n, void* __restrict__ y, int ydt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    store_from_f32(y, ydt, i, __fmul_rn(dec_e4m3(c[i]), scales[i / block_elems]));
}

// Slot trailers of the Ulysses FP8 wire: slot t carries the scales of its destination's
// heads -- the tensor-wide scale (reference, QuantizedTensor::slice_heads, fp8.cpp:100-105)
// or, per block, the scales of slabs (b, t*hp + hl) in [b][hl] order.
__global__ void scatter_slot_scales_kernel(const float* __restrict__ scales, float* __restrict__ base,
                                           int64_t slot_stride_f, int b, int h, int u,
                                           int per_block) {
  const int hp = h / u;
  const int nsc = per_block ? b * hp : 1;
  for (int idx = threadIdx.x; idx < u * nsc; idx += blockDim.x) {
    const int t = idx / nsc, k = idx % nsc;
    const int src = per_block ? (k / hp) * h + t * hp + (k % hp) : 0;
    base[t * slot_stride_f + k] = scales[src];
  }
}

// Finite check over several tensors at once (check_local_qkv, protocols.cpp:102-104).
__global__ void finite_kernel(const void* __restrict__ x, int dt, int64_t n, uint32_t* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    bad |= !isfinite(load_as_f32(x, dt, i));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}


// ---- 16-byte-vector movers (the Ulysses pack / unpack and the FP8 passes) -----------------
// One (b,h) slab of a [B][H][SL][D] tensor is SL*D contiguous elements in the source and in
// its destination slot, so the copies are slab-to-slab: grid.y = slab, grid.z = tensor,
// 32-bit offsets inside the slab, no per-element index arithmetic.  8 elements per step.
struct Vec8 {
  float f[8];
};
// Raw 8-element vector (16 B for 16-bit types, 32 B for f32) and its f32 values: the FP8 passes
// issue every load of a thread's stride before converting any (bytes in flight per SM).
struct Raw8 {  // 8 source elements as loaded: f32 = a,b; 16-bit = a; e4m3 = a.x, a.y
  uint4 a, b;
};
__device__ __forceinline__ Raw8 load_raw8(const void* base, int sdt, int64_t i) {
  Raw8 r;
  if (sdt == FUSP_F32) {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const float*>(base) + i);
    r.a = __ldg(p);
    r.b = __ldg(p + 1);
  } else if (sdt == FUSP_E4M3) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(base) + i));
    r.a = make_uint4(w.x, w.y, 0u, 0u);
  } else {
    r.a = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + i));
  }
  return r;
}
__device__ __forceinline__ Vec8 cvt8(const Raw8& r, int dt) {
  Vec8 v;
  const uint32_t w[8] = {r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, r.b.z, r.b.w};
  if (dt == FUSP_F32) {
#pragma unroll
    for (int e = 0; e < 8; ++e) v.f[e] = __uint_as_float(w[e]);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = dt == FUSP_F16 ? __half22float2(*reinterpret_cast<const __half2*>(&w[e]))
                                      : __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
      v.f[2 * e] = x.x;
      v.f[2 * e + 1] = x.y;
    }
  }
  return v;
}
// |x| maximum of a raw vector on the bit patterns: sign-magnitude floats order like their
// magnitude bits, so the maximum is an integer SIMD max (no conversions).  `mag` accumulates
// magnitude bits (two 16-bit lanes, or one 32-bit value for f32); a vector holding a NaN
// (magnitude bits above the infinity pattern) is left to the float path (fmaxf ignores NaN,
// as the amax always did) and `inf_or_nan` is raised for it and for infinities.
__device__ __forceinline__ bool absmax_raw8(const Raw8& r, int dt, uint32_t& mag, bool& inf_or_nan) {
  if (dt == FUSP_F32) {
    const uint32_t w[8] = {r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, r.b.z, r.b.w};
    uint32_t m = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) m = max(m, w[e] & 0x7FFFFFFFu);
    if (m >= 0x7F800000u) {
      inf_or_nan = true;
      if (m > 0x7F800000u) return false;  // a NaN: float path
    }
    mag = max(mag, m);
    return true;
  }
  const uint32_t inf2 = dt == FUSP_F16 ? 0x7C007C00u : 0x7F807F80u;
  const uint32_t m = __vmaxu2(__vmaxu2(r.a.x & 0x7FFF7FFFu, r.a.y & 0x7FFF7FFFu),
                              __vmaxu2(r.a.z & 0x7FFF7FFFu, r.a.w & 0x7FFF7FFFu));
  if (__vcmpgeu2(m, inf2) != 0u) {
    inf_or_nan = true;
    if (__vcmpgtu2(m, inf2) != 0u) return false;
  }
  mag = __vmaxu2(mag, m);
  return true;
}
__device__ __forceinline__ float mag_to_f32(uint32_t mag, int dt) {
  if (dt == FUSP_F32) return __uint_as_float(mag);
  const uint32_t h = max(mag & 0xFFFFu, mag >> 16);
  return dt == FUSP_F16 ? __half2float(__ushort_as_half(static_cast<unsigned short>(h)))
                        : __uint_as_float(h << 16);
}
__device__ __forceinline__ Vec8 load8(const void* base, int dt, int64_t i) {
  Vec8 v;
  if (dt == FUSP_F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + i);
    const float4 a = __ldg(p), b = __ldg(p + 1);
    v.f[0] = a.x; v.f[1] = a.y; v.f[2] = a.z; v.f[3] = a.w;
    v.f[4] = b.x; v.f[5] = b.y; v.f[6] = b.z; v.f[7] = b.w;
  } else {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + i));
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 x;
      if (dt == FUSP_F16) x = __half22float2(*reinterpret_cast<const __half2*>(&ww[e]));
      else x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[e]));
      v.f[2 * e] = x.x;
      v.f[2 * e + 1] = x.y;
    }
  }
  return v;
}
__device__ __forceinline__ void store8(void* base, int dt, int64_t i, const Vec8& v) {
  if (dt == FUSP_F32) {
    float4* p = reinterpret_cast<float4*>(static_cast<float*>(base) + i);
    p[0] = make_float4(v.f[0], v.f[1], v.f[2], v.f[3]);
    p[1] = make_float4(v.f[4], v.f[5], v.f[6], v.f[7]);
    return;
  }
  uint32_t w[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (dt == FUSP_F16) {
      __half2 x = __floats2half2_rn(v.f[2 * e], v.f[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&x);
    } else {
      __nv_bfloat162 x = __floats2bfloat162_rn(v.f[2 * e], v.f[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&x);
    }
  }
  *reinterpret_cast<uint4*>(static_cast<uint16_t*>(base) + i) = make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ uint32_t enc_pair(float a, float b) {  // (a -> low byte, b -> high)
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(b), "f"(a));
  uint32_t x = r;
  if (isnan(a)) x = (x & 0xFF00u) | (signbit(a) ? 0xFFu : 0x7Fu);
  if (isnan(b)) x = (x & 0x00FFu) | ((signbit(b) ? 0xFFu : 0x7Fu) << 8);
  return x;
}
// RN(x / qs) as the E4M3 encoder sees it, bit-exact with IEEE division (fp8.cpp:121):
// q = x * RN(1/qs) is within 2.5 f32 ulp of RN(x/qs), so it encodes identically unless
// RN(x/qs) sits near an E4M3 rounding boundary -- the midpoint pattern 0x80000 in the low 20
// mantissa bits (normal range), or anywhere in the E4M3 subnormal range (|q| < 2^-6).  Those
// rare values take the exact division.  Above 448 everything saturates to 448 either way.
// The IEEE division, out of line: taken for |q| < 2^-6 (E4M3 subnormals) and near rounding
// boundaries only, and the unrolled FP8 loops would otherwise inline it at every element.
__device__ __noinline__ float qdiv_slow(float x, float qs) { return __fdiv_rn(x, qs); }
__device__ __forceinline__ float qdiv(float x, float qs, float inv) {
  const float q = x * inv;
  const uint32_t b = __float_as_uint(q) & 0x7fffffffu;
  if (b < 0x3c800000u || ((b & 0xFFFFFu) - 0x7FFF8u) < 16u) return qdiv_slow(x, qs);
  return q;
}
__device__ __forceinline__ uint2 encode8(const Vec8& v, float qs) {  // IEEE x / scale, RNE sat
  const float inv = __frcp_rn(qs);
  float q[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) q[e] = qdiv(v.f[e], qs, inv);
  return make_uint2(enc_pair(q[0], q[1]) | (enc_pair(q[2], q[3]) << 16),
                    enc_pair(q[4], q[5]) | (enc_pair(q[6], q[7]) << 16));
}
// Finite inputs only (the amax pass rejected non-finite ones): no NaN fix-ups.
__device__ __forceinline__ uint32_t enc_pair_finite(float a, float b) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(b), "f"(a));
  return r;
}
// x * inv for a pair with one FFMA2 (c = -0: RN(a b + -0) = RN(a b), signed zeros included).
__device__ __forceinline__ float2 fmul2_rn(float2 a, float b) {
  const float2 bb = make_float2(b, b), zz = make_float2(-0.f, -0.f);
  float2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(reinterpret_cast<unsigned long long&>(r))
      : "l"(reinterpret_cast<const unsigned long long&>(a)),
        "l"(reinterpret_cast<const unsigned long long&>(bb)),
        "l"(reinterpret_cast<const unsigned long long&>(zz)));
  return r;
}
// As qdiv on 8 values: the products packed in pairs, and one branch per vector to the exact
// divisions -- taken only when some product is in the E4M3 subnormal range or near a rounding
// boundary (then every element of the vector goes through qdiv, with the same results).
__device__ __forceinline__ uint2 encode8_finite(const Vec8& v, float qs, float inv) {
  float q[8];
  uint32_t slow = 0;
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    const float2 p = fmul2_rn(make_float2(v.f[e], v.f[e + 1]), inv);
    q[e] = p.x;
    q[e + 1] = p.y;
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t b = __float_as_uint(q[e]) & 0x7fffffffu;
    slow |= static_cast<uint32_t>(b < 0x3c800000u) | static_cast<uint32_t>(((b & 0xFFFFFu) - 0x7FFF8u) < 16u);
  }
  if (slow) {
#pragma unroll
    for (int e = 0; e < 8; ++e) q[e] = qdiv(v.f[e], qs, inv);
  }
  return make_uint2(enc_pair_finite(q[0], q[1]) | (enc_pair_finite(q[2], q[3]) << 16),
                    enc_pair_finite(q[4], q[5]) | (enc_pair_finite(q[6], q[7]) << 16));
}
// 8 codes -> f32, exact: the hardware e4m3x2 -> f16x2 conversion is exact (every E4M3 value
// is an f16; 0x7F / 0xFF -> NaN as in fp8.cpp:39-43), then f16 -> f32 and * scale (f32 RN).
__device__ __forceinline__ void dec4(uint32_t w, float sc, float* f) {
  uint32_t lo, hi;
  asm("{\n\t.reg .b16 a, b;\n\tmov.b32 {a, b}, %2;\n\t"
      "cvt.rn.f16x2.e4m3x2 %0, a;\n\tcvt.rn.f16x2.e4m3x2 %1, b;\n\t}"
      : "=r"(lo), "=r"(hi) : "r"(w));
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&lo));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&hi));
  f[0] = __fmul_rn(a.x, sc);
  f[1] = __fmul_rn(a.y, sc);
  f[2] = __fmul_rn(b.x, sc);
  f[3] = __fmul_rn(b.y, sc);
}
__device__ __forceinline__ Vec8 decode8(uint2 w, float sc) {
  Vec8 v;
  dec4(w.x, sc, v.f);
  dec4(w.y, sc, v.f + 4);
  return v;
}

constexpr int kMaxMoveOps = 6;  // tensors moved by one pack / unpack launch (grid.z)
struct PackOp {
  const void* src;
  void* dst;
  const float* scale;       // e4m3 destination: scale[slab * scale_bh_stride] ...
  const uint32_t* amax;     // ... or, when set, scale = amax[slab * scale_bh_stride] / 448 (1 if 0)
  float* trailer;           // e4m3: also write each slot's scales here (slot t at t * trailer_stride)
  int64_t trailer_stride;
  int64_t scale_bh_stride;
  int64_t slot_stride;      // destination elements between slots
  int sdt, ddt;
};
struct PackArgs {
  PackOp op[kMaxMoveOps];
  int h, hp, slab_vecs;  // slab_vecs = SL*D/8
  int64_t slab_elems;
  // Peer-memory Ulysses pack (peer = 1): slot t lives in member t's window, slot_boff[t] bytes
  // from slot 0 (ops' dst / trailer address slot 0); replaces t * slot_stride / trailer_stride.
  int peer;
  int64_t slot_boff[kMaxPeerChunks];
};
// Ulysses pack (protocols.cpp:143-153): slab (b, h) -> slot h / hp, position (b, h % hp).
__global__ void __launch_bounds__(256) pack_slab_kernel(const __grid_constant__ PackArgs a) {
  const PackOp& o = a.op[blockIdx.z];
  const int slab = blockIdx.y;
  const int hh = slab % a.h, bb = slab / a.h;
  const int t = hh / a.hp, hl = hh - t * a.hp;
  const int64_t s0 = int64_t(slab) * a.slab_elems;
  const int64_t desz = o.ddt == FUSP_E4M3 ? 1 : (o.ddt == FUSP_F32 ? 4 : 2);
  const int64_t d0 = (a.peer ? a.slot_boff[t] / desz : int64_t(t) * o.slot_stride) +
                     (int64_t(bb) * a.hp + hl) * a.slab_elems;
  float qs = 1.f;
  if (o.ddt == FUSP_E4M3) {
    // (programmatic dependent of the amax pass: its scales are complete after the wait; a
    // no-op for an ordinary launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (o.amax != nullptr) {  // finalize fused in: scale = amax / 448, 1 for an all-zero block
      const float am = __uint_as_float(o.amax[slab * o.scale_bh_stride]);
      qs = am > 0.f ? __fdiv_rn(am, 448.0f) : 1.0f;
    } else {
      qs = __ldcg(&o.scale[slab * o.scale_bh_stride]);
    }
    // slot trailer (QuantizedTensor::slice_heads keeps the tensor-wide scale, fp8.cpp:100-105;
    // per block: the scales of this slot's slabs in [b][hl] order)
    if (o.trailer != nullptr && blockIdx.x == 0 && threadIdx.x == 0 &&
        (o.scale_bh_stride != 0 || (bb == 0 && hl == 0)))
      o.trailer[(a.peer ? a.slot_boff[t] / 4 : t * o.trailer_stride) +
                (o.scale_bh_stride != 0 ? bb * a.hp + hl : 0)] = qs;
  }
  const int stride = gridDim.x * blockDim.x;
  const int v0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (o.sdt == o.ddt && o.sdt != FUSP_F32) {  // same 16-bit type: 4 x 16 B in flight per thread
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(o.src) + s0);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(o.dst) + d0);
    for (int v = v0; v < a.slab_vecs; v += 4 * stride) {
      uint4 x[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (v + e * stride < a.slab_vecs) x[e] = __ldg(src + v + e * stride);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (v + e * stride < a.slab_vecs) dst[v + e * stride] = x[e];
    }
    if (a.peer) __threadfence_system();  // remote stores visible before the exchange signal
    return;
  }
  for (int v = v0; v < a.slab_vecs; v += 4 * stride) {
    Vec8 x[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (v + e * stride < a.slab_vecs) x[e] = load8(o.src, o.sdt, s0 + int64_t(v + e * stride) * 8);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (v + e * stride >= a.slab_vecs) break;
      const int64_t i = int64_t(v + e * stride) * 8;
      if (o.ddt == FUSP_E4M3)
        *reinterpret_cast<uint2*>(static_cast<uint8_t*>(o.dst) + d0 + i) = encode8(x[e], qs);
      else
        store8(o.dst, o.ddt, d0 + i, x[e]);
    }
  }
  if (a.peer) __threadfence_system();
}

struct UnpackOp {
  const void* src;
  void* dst;
  const float* scales;  // e4m3 source: scales[j * scale_stride + bh * scale_bh_stride]
  int64_t src_slot_stride, scale_stride, scale_bh_stride;
  int sdt, ddt;
};
struct UnpackArgs {
  UnpackOp op[kMaxMoveOps];
  int bhp, sl, u, slab_vecs;  // bhp = B * hp
  int64_t slab_elems;
};
// Ulysses unpack (protocols.cpp:163-179): slot j's slab bh -> rows [j*SL, (j+1)*SL) of slab bh.
__global__ void __launch_bounds__(256) unpack_slab_kernel(const __grid_constant__ UnpackArgs a) {
  const UnpackOp& o = a.op[blockIdx.z];
  const int slab = blockIdx.y;
  const int j = slab / a.bhp, bh = slab - j * a.bhp;
  const int64_t s0 = int64_t(j) * o.src_slot_stride + int64_t(bh) * a.slab_elems;
  const int64_t d0 = (int64_t(bh) * a.u + j) * a.slab_elems;
  const float sc = o.sdt == FUSP_E4M3 ? o.scales[j * o.scale_stride + bh * o.scale_bh_stride] : 1.f;
  const int stride = gridDim.x * blockDim.x;
  const int v0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (o.sdt == o.ddt && (o.sdt == FUSP_F16 || o.sdt == FUSP_BF16)) {  // 4 x 16 B in flight
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(o.src) + s0);
    uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(o.dst) + d0);
    for (int v = v0; v < a.slab_vecs; v += 4 * stride) {
      uint4 x[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (v + e * stride < a.slab_vecs) x[e] = __ldg(src + v + e * stride);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (v + e * stride < a.slab_vecs) dst[v + e * stride] = x[e];
    }
    return;
  }
  if (o.sdt == FUSP_E4M3 && o.ddt != FUSP_E4M3) {  // dequantize: 4 x 8 codes in flight
    for (int v = v0; v < a.slab_vecs; v += 4 * stride) {
      uint2 c[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (v + e * stride < a.slab_vecs)
          c[e] = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(o.src) + s0 +
                                                      int64_t(v + e * stride) * 8));
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (v + e * stride < a.slab_vecs) store8(o.dst, o.ddt, d0 + int64_t(v + e * stride) * 8, decode8(c[e], sc));
    }
    return;
  }
  for (int v = v0; v < a.slab_vecs; v += stride) {
    const int64_t i = int64_t(v) * 8;
    if (o.sdt == o.ddt) {
      if (o.sdt == FUSP_E4M3)
        *reinterpret_cast<uint2*>(static_cast<uint8_t*>(o.dst) + d0 + i) =
            __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(o.src) + s0 + i));
      else if (o.sdt == FUSP_F32)
        store8(o.dst, FUSP_F32, d0 + i, load8(o.src, FUSP_F32, s0 + i));
      else
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(o.dst) + d0 + i) =
            __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(o.src) + s0 + i));
      continue;
    }
    const Vec8 x = o.sdt == FUSP_E4M3
                       ? decode8(__ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(o.src) + s0 + i)), sc)
                       : load8(o.src, o.sdt, s0 + i);
    store8(o.dst, o.ddt, d0 + i, x);
  }
}

// ---- operand staging with the f16 range guard (fastusp_internal.h, StageOp) ---------------
__device__ __forceinline__ void store_raw8(void* base, int sdt, int64_t i, const Raw8& r) {
  if (sdt == FUSP_F32) {
    uint4* p = reinterpret_cast<uint4*>(static_cast<float*>(base) + i);
    p[0] = r.a;
    p[1] = r.b;
  } else if (sdt == FUSP_E4M3) {
    *reinterpret_cast<uint2*>(static_cast<uint8_t*>(base) + i) = make_uint2(r.a.x, r.a.y);
  } else {
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(base) + i) = r.a;
  }
}
__device__ __forceinline__ Vec8 raw_to_f32(const Raw8& r, int sdt, float sc) {
  Vec8 v;
  if (sdt == FUSP_F32) {
    v.f[0] = __uint_as_float(r.a.x); v.f[1] = __uint_as_float(r.a.y);
    v.f[2] = __uint_as_float(r.a.z); v.f[3] = __uint_as_float(r.a.w);
    v.f[4] = __uint_as_float(r.b.x); v.f[5] = __uint_as_float(r.b.y);
    v.f[6] = __uint_as_float(r.b.z); v.f[7] = __uint_as_float(r.b.w);
  } else if (sdt == FUSP_E4M3) {
    v = decode8(make_uint2(r.a.x, r.a.y), sc);
  } else {
    const uint32_t ww[4] = {r.a.x, r.a.y, r.a.z, r.a.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 x;
      if (sdt == FUSP_F16) x = __half22float2(*reinterpret_cast<const __half2*>(&ww[e]));
      else x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[e]));
      v.f[2 * e] = x.x;
      v.f[2 * e + 1] = x.y;
    }
  }
  return v;
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
// Exponent of the f16 range guard: 0 while max|x| is in [2^-6, 2^15) (or zero / non-finite),
// else e with max|x| * 2^-e in [2^14, 2^15), clamped to [kGuardExpMin, kGuardExpMax].
__device__ __forceinline__ int guard_exp(float amax) {
  if (!(amax > 0.f) || !isfinite(amax)) return 0;
  if (amax >= 0x1p-6f && amax < 0x1p15f) return 0;
  const int e = static_cast<int>((__float_as_uint(amax) >> 23) & 0xFFu) - 127 - 14;
  return e < kGuardExpMin ? kGuardExpMin : (e > kGuardExpMax ? kGuardExpMax : e);
}

#ifndef FUSP_STAGE_MINB   // resident CTAs per SM the staging kernel is compiled for
#define FUSP_STAGE_MINB 4
#endif
#ifndef FUSP_STAGE_NV     // 16-byte vectors in flight per thread (f32 sources: half as many 32-byte)
#define FUSP_STAGE_NV 4
#endif
#ifndef FUSP_STAGE_WAVES  // grid cap: CTAs per SM (one resident wave at FUSP_STAGE_MINB)
#define FUSP_STAGE_WAVES FUSP_STAGE_MINB
#endif
struct StageArgs {
  StageOp op[kMaxStageOps];
  int bhp, u, slab_vecs;
  int64_t slab_elems;
};
// Main pass of one staging op, everything per element known at compile time: the source
// dtype, the destination mode (DDT = -1: copy of the source bytes), the range guard (max|x|)
// and the optional raw copy.  Pointers and offsets are hoisted out of the loop.  Registers:
// the f32 source keeps half as many (32-byte) vectors in flight per thread.
template <int SDT, int DDT, bool GUARD, bool RAW>
__device__ __forceinline__ float stage_main(const void* __restrict__ src, void* __restrict__ dst,
                                            void* __restrict__ raw, int slab_vecs, float sc) {
  constexpr int NV = SDT == FUSP_F32 ? (FUSP_STAGE_NV + 1) / 2 : FUSP_STAGE_NV;
  const int stride = gridDim.x * blockDim.x;
  float m = 0.f;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < slab_vecs; v += NV * stride) {
    Raw8 r[NV];
#pragma unroll
    for (int e = 0; e < NV; ++e)
      if (v + e * stride < slab_vecs) r[e] = load_raw8(src, SDT, int64_t(v + e * stride) * 8);
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      if (v + e * stride >= slab_vecs) break;
      const int64_t i = int64_t(v + e * stride) * 8;
      if (RAW) store_raw8(raw, SDT, i, r[e]);
      if (DDT < 0) {
        store_raw8(dst, SDT, i, r[e]);
      } else {
        const Vec8 x = raw_to_f32(r[e], SDT, sc);
        if (GUARD) {
#pragma unroll
          for (int k = 0; k < 8; ++k) m = fmaxf(m, fabsf(x.f[k]));
        }
        store8(dst, DDT, i, x);
      }
    }
  }
  return m;
}

template <int SDT>
__device__ __forceinline__ float stage_dispatch(const StageOp& o, const char* src, char* dst,
                                                char* raw, int slab_vecs, float sc) {
  const bool guard = o.exps != nullptr;
  if (o.dst == nullptr) return stage_main<SDT, -1, false, false>(src, raw, nullptr, slab_vecs, sc);
  if (o.ddt == SDT && !guard) {
    if (raw != nullptr) return stage_main<SDT, -1, false, true>(src, dst, raw, slab_vecs, sc);
    return stage_main<SDT, -1, false, false>(src, dst, nullptr, slab_vecs, sc);
  }
  if (guard) {
    if (raw != nullptr) return stage_main<SDT, FUSP_F16, true, true>(src, dst, raw, slab_vecs, sc);
    return stage_main<SDT, FUSP_F16, true, false>(src, dst, nullptr, slab_vecs, sc);
  }
  if (raw != nullptr) {  // e.g. FP8 codes kept exact beside an f32 operand (other head dims)
    switch (o.ddt) {
      case FUSP_F16: return stage_main<SDT, FUSP_F16, false, true>(src, dst, raw, slab_vecs, sc);
      case FUSP_BF16: return stage_main<SDT, FUSP_BF16, false, true>(src, dst, raw, slab_vecs, sc);
      default: return stage_main<SDT, FUSP_F32, false, true>(src, dst, raw, slab_vecs, sc);
    }
  }
  switch (o.ddt) {
    case FUSP_F16: return stage_main<SDT, FUSP_F16, false, false>(src, dst, nullptr, slab_vecs, sc);
    case FUSP_BF16: return stage_main<SDT, FUSP_BF16, false, false>(src, dst, nullptr, slab_vecs, sc);
    default: return stage_main<SDT, FUSP_F32, false, false>(src, dst, nullptr, slab_vecs, sc);
  }
}

// grid (x: part of a slab, y: slab (j, bh), z: op).  Plain copies, conversions, e4m3 decodes;
// guarded f16 destinations fold max|x| into their per-head word (fastusp_internal.h).
__global__ void __launch_bounds__(256, FUSP_STAGE_MINB) stage_kernel(const __grid_constant__ StageArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");  // let stage_decide_kernel get scheduled
  const StageOp& o = a.op[blockIdx.z];
  const int slab = blockIdx.y;
  const int j = slab / a.bhp, bh = slab - j * a.bhp;
  const int64_t s0 = int64_t(j) * o.src_slot_stride + int64_t(bh) * o.src_bh_stride;
  const int64_t d0 = int64_t(j) * o.dst_slot_stride + int64_t(bh) * o.dst_bh_stride;
  const int sdt = o.sdt;
  const float sc = sdt == FUSP_E4M3 ? o.scales[j * o.scale_stride + bh * o.scale_bh_stride] : 1.f;
  const bool guard = o.exps != nullptr;
  const int64_t ssz = sdt == FUSP_F32 ? 4 : sdt == FUSP_E4M3 ? 1 : 2;
  const int64_t dsz = o.dst == nullptr ? ssz : (o.ddt == FUSP_F32 ? 4 : 2);
  const char* src = static_cast<const char*>(o.src) + s0 * ssz;
  char* dst = o.dst != nullptr ? static_cast<char*>(o.dst) + d0 * dsz : nullptr;
  char* raw = o.raw != nullptr ? static_cast<char*>(o.raw) + d0 * ssz : nullptr;
  float m;
  switch (sdt) {
    case FUSP_F32: m = stage_dispatch<FUSP_F32>(o, src, dst, raw, a.slab_vecs, sc); break;
    case FUSP_F16: m = stage_dispatch<FUSP_F16>(o, src, dst, raw, a.slab_vecs, sc); break;
    case FUSP_BF16: m = stage_dispatch<FUSP_BF16>(o, src, dst, raw, a.slab_vecs, sc); break;
    default: m = stage_dispatch<FUSP_E4M3>(o, src, dst, raw, a.slab_vecs, sc); break;
  }
  if (!guard) return;
  // CTA max -> one relaxed atomic per CTA (per-warp atomics on the head's word serialised at
  // L2: ~4600 warps on 6 words at FLUX U=8); no fence: the per-head decision runs in
  // stage_decide_kernel, ordered after this kernel by the stream
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  __shared__ float wm[kBlock / 32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kBlock / 32; ++w) m = fmaxf(m, wm[w]);
    if (m > 0.f) atomicMax(&o.words[bh], __float_as_uint(m));
  }
}

// Per (head, guarded op), kFixParts CTAs: each derives e from the head's max|x| word; part 0
// publishes exps[bh]; the last part to count (relaxed ticket, words[bhp + bh]) resets both
// words for the next call.  A head outside [2^-6, 2^15) is rewritten as x * 2^-e, its slabs'
// vectors split over the parts -- the rare path; the common one exits after one load.
constexpr int kFixParts = 8;
__global__ void __launch_bounds__(256) stage_decide_kernel(const __grid_constant__ StageArgs a) {
  const StageOp& o = a.op[blockIdx.y];
  if (o.exps == nullptr) return;
  const int bh = blockIdx.x, part = blockIdx.z;
  // launched as a programmatic dependent of stage_kernel: resident early, and this waits for
  // the staging grid's completion and memory (griddepcontrol.wait)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ int s_e;
  if (threadIdx.x == 0) {
    const int e = guard_exp(__uint_as_float(__ldcg(&o.words[bh])));
    if (part == 0) o.exps[bh] = e;
    __threadfence();  // our read of the word before our ticket
    if (atomicAdd(&o.words[a.bhp + bh], 1u) + 1 == kFixParts) {
      o.words[bh] = 0u;
      o.words[a.bhp + bh] = 0u;
    }
    s_e = e;
  }
  __syncthreads();
  if (s_e == 0) return;
  const bool e4 = o.sdt == FUSP_E4M3;
  const float f = pow2f(-s_e);
  for (int jj = 0; jj < a.u; ++jj) {
    const int64_t sj = int64_t(jj) * o.src_slot_stride + int64_t(bh) * o.src_bh_stride;
    const int64_t dj = int64_t(jj) * o.dst_slot_stride + int64_t(bh) * o.dst_bh_stride;
    const float scj = e4 ? o.scales[jj * o.scale_stride + bh * o.scale_bh_stride] : 1.f;
    for (int v = part * blockDim.x + threadIdx.x; v < a.slab_vecs; v += kFixParts * blockDim.x) {
      Vec8 x = raw_to_f32(load_raw8(o.src, o.sdt, sj + int64_t(v) * 8), o.sdt, scj);
#pragma unroll
      for (int k = 0; k < 8; ++k) x.f[k] *= f;
      store8(o.dst, o.ddt, dj + int64_t(v) * 8, x);
    }
  }
}

// Element-wise staging (any alignment; no range guard): the stage_kernel mapping per element.
__global__ void stage_scalar_kernel(const __grid_constant__ StageArgs a, int64_t total) {
  const StageOp& o = a.op[blockIdx.y];
  const int esz = o.sdt == FUSP_F32 ? 4 : (o.sdt == FUSP_E4M3 ? 1 : 2);
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t slab = e / a.slab_elems, i = e - slab * a.slab_elems;
    const int j = static_cast<int>(slab / a.bhp), bh = static_cast<int>(slab - int64_t(j) * a.bhp);
    const int64_t si = int64_t(j) * o.src_slot_stride + int64_t(bh) * o.src_bh_stride + i;
    const int64_t di = int64_t(j) * o.dst_slot_stride + int64_t(bh) * o.dst_bh_stride + i;
    if (o.raw != nullptr)
      for (int b = 0; b < esz; ++b)
        static_cast<uint8_t*>(o.raw)[di * esz + b] = static_cast<const uint8_t*>(o.src)[si * esz + b];
    if (o.dst == nullptr) continue;
    float x;
    if (o.sdt == FUSP_E4M3)
      x = __fmul_rn(dec_e4m3(static_cast<const uint8_t*>(o.src)[si]),
                    o.scales[j * o.scale_stride + bh * o.scale_bh_stride]);
    else
      x = load_as_f32(o.src, o.sdt, si);
    store_from_f32(o.dst, o.ddt, di, x);
  }
}

// Unsigned division by a run-time constant as a multiply-high and a shift (x < 2^31):
// l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1, x / d = (umulhi(x, m) + x) >> l.  The
// E4M3 sources look up a per-segment scale for every 8 codes; three hardware-less 32-bit
// divisions per vector made those passes instruction-bound (ncu: issue-active 50 %).
struct FDiv {
  uint32_t d, m;
  int l;
};
inline FDiv make_fdiv(uint32_t d) {
  int l = 0;
  while ((uint64_t(1) << l) < d) ++l;
  return FDiv{d, static_cast<uint32_t>(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1), l};
}
__device__ __forceinline__ uint32_t fdiv(const FDiv& f, uint32_t x) {
  return (__umulhi(x, f.m) + x) >> f.l;
}
struct Fp8Div {  // i / d, row / span, r / seg_rows of an Fp8Src
  FDiv d, span, seg;
};
inline Fp8Div make_fp8div(const Fp8Src& s) {
  return Fp8Div{make_fdiv(uint32_t(s.d)), make_fdiv(uint32_t(s.span)), make_fdiv(uint32_t(s.seg_rows))};
}
// Scale of the segment holding element i of an E4M3 source.
__device__ __forceinline__ float e4m3_scale(const Fp8Src& s, const Fp8Div& dv, int64_t i) {
  const uint32_t row = fdiv(dv.d, static_cast<uint32_t>(i));
  const uint32_t bh = fdiv(dv.span, row);
  const uint32_t r = row - bh * static_cast<uint32_t>(s.span);
  return s.scales[int64_t(fdiv(dv.seg, r)) * s.seg_stride + int64_t(bh) * s.bh_stride];
}

// Source value of 8 consecutive elements (one row segment) for the FP8 passes.
__device__ __forceinline__ Vec8 src_vec8(const Fp8Src& s, const Fp8Div& dv, int64_t i) {  // i < 2^31
  if (s.dt != FUSP_E4M3) return load8(s.x, s.dt, i);
  return decode8(__ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(s.x) + i)),
                 e4m3_scale(s, dv, i));
}

// |value| maximum of 8 codes of an E4M3 source in one step: decode(c) * scale is monotone in
// the code magnitude (sign-magnitude encoding, RN multiply), so the maximum is the decoded
// largest magnitude -- a byte-SIMD max and one decode instead of eight.  A NaN code (0x7F)
// is the largest magnitude and decodes to NaN, which the caller flags as non-finite.
__device__ __forceinline__ float e4m3_vec_absmax(const Fp8Src& s, const Fp8Div& dv, int64_t i) {
  const float sc = e4m3_scale(s, dv, i);
  const uint2 w = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(s.x) + i));
  uint32_t m = __vmaxu4(w.x & 0x7F7F7F7Fu, w.y & 0x7F7F7F7Fu);
  m = max(max(m & 0xFFu, (m >> 8) & 0xFFu), max((m >> 16) & 0xFFu, m >> 24));
  float f[4];
  dec4(m, sc, f);
  return f[0];
}

// Wide (f32 / f16 / bf16) sources of the FP8 passes, specialised per dtype: every load of a
// thread's share (128 B: 8 vectors of 16-bit values, 4 of f32) is issued before any is used.
template <int DT>
__device__ __forceinline__ void amax_wide(const void* x, int64_t base, int64_t v0, int64_t stride,
                                          int64_t nv, float& m, bool& bad) {
  constexpr int U = DT == FUSP_F32 ? kFp8Unroll / 2 : kFp8Unroll;
  uint32_t mag = 0;
  for (int64_t v = v0; v < nv; v += U * stride) {
    Raw8 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v + u * stride < nv) r[u] = load_raw8(x, DT, (base + v + u * stride) * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v + u * stride >= nv) break;
      if (!absmax_raw8(r[u], DT, mag, bad)) {
        const Vec8 f = cvt8(r[u], DT);
#pragma unroll
        for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(f.f[e]));
      }
    }
  }
  m = fmaxf(m, mag_to_f32(mag, DT));
}
template <int DT>
__device__ __forceinline__ void quant_wide(const void* x, uint8_t* codes, int64_t base, int64_t v0,
                                           int64_t stride, int64_t nv, float qs, float inv) {
  constexpr int U = DT == FUSP_F32 ? kFp8Unroll / 2 : kFp8Unroll;
  for (int64_t v = v0; v < nv; v += U * stride) {
    Raw8 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v + u * stride < nv) r[u] = load_raw8(x, DT, (base + v + u * stride) * 8);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v + u * stride < nv)
        *reinterpret_cast<uint2*>(codes + (base + v + u * stride) * 8) = encode8_finite(cvt8(r[u], DT), qs, inv);
  }
}

// Pass 1 per block, 8 elements per step; grid.y = block, grid.z = tensor (K, V).
struct AmaxArgs {
  Fp8Src src[2];
  Fp8Div div[2];
  uint32_t* amax[2];  // zero on entry when `ticket` is set (the finalize leaves them zero)
  int64_t block_vecs;
  uint32_t* nonfinite;
  // Finalize in the last CTA (ticket != null): scales[p][blk] = amax / 448 (1 if 0), then the
  // amax words and the ticket are reset to zero for the next launch -- no memset before, no
  // separate finalize kernel after (threadFenceReduction pattern).
  float* scales[2];
  uint32_t* ticket;
  int nblocks, parts;
};
// SDT: the sources' dtype when every part shares it (the common case: each instance then
// holds only its own path's registers -- 4 resident CTAs per SM, one wave), -1 = per part.
template <int SDT>
__global__ void __launch_bounds__(256, 4) amax_vec_kernel(const __grid_constant__ AmaxArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");  // the quantize / pack pass gets scheduled
  const Fp8Src& s = a.src[blockIdx.z];
  const int sdt = SDT >= 0 ? SDT : s.dt;
  const int64_t base = int64_t(blockIdx.y) * a.block_vecs;
  float m = 0.f, nf = 0.f;
  bool bad = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (sdt == FUSP_E4M3 && s.d % 16 == 0 && a.block_vecs % 2 == 0) {
    // 16 codes (one row piece, one scale) per load, kFp8Unroll loads in flight per thread
    const int64_t nv = a.block_vecs / 2, e0 = base * 8;
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < nv; v += kE4Unroll * stride) {
      uint4 w[kE4Unroll];
      float sc[kE4Unroll];
#pragma unroll
      for (int u = 0; u < kE4Unroll; ++u)
        if (v + u * stride < nv) {
          const int64_t i = e0 + (v + u * stride) * 16;
          w[u] = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(s.x) + i));
          sc[u] = e4m3_scale(s, a.div[blockIdx.z], i);
        }
#pragma unroll
      for (int u = 0; u < kE4Unroll; ++u) {
        if (v + u * stride >= nv) break;
        uint32_t mm = __vmaxu4(__vmaxu4(w[u].x & 0x7F7F7F7Fu, w[u].y & 0x7F7F7F7Fu),
                               __vmaxu4(w[u].z & 0x7F7F7F7Fu, w[u].w & 0x7F7F7F7Fu));
        mm = max(max(mm & 0xFFu, (mm >> 8) & 0xFFu), max((mm >> 16) & 0xFFu, mm >> 24));
        float f[4];
        dec4(mm, sc[u], f);
        nf = fmaf(f[0], 0.f, nf);
        m = fmaxf(m, f[0]);
      }
    }
  } else if (sdt == FUSP_E4M3) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < a.block_vecs; v += stride) {
      const float x = e4m3_vec_absmax(s, a.div[blockIdx.z], (base + v) * 8);
      nf = fmaf(x, 0.f, nf);
      m = fmaxf(m, x);
    }
  } else {
    // 128 B of raw vectors in flight per thread; max |x| on the bit patterns
    const int64_t v0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (sdt == FUSP_F32) amax_wide<FUSP_F32>(s.x, base, v0, stride, a.block_vecs, m, bad);
    else if (sdt == FUSP_F16) amax_wide<FUSP_F16>(s.x, base, v0, stride, a.block_vecs, m, bad);
    else amax_wide<FUSP_BF16>(s.x, base, v0, stride, a.block_vecs, m, bad);
  }
  bad = bad || nf != 0.f;
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  bad = __any_sync(0xffffffffu, bad);
  __shared__ float wm[kBlock / 32];
  __shared__ int wb[kBlock / 32];
  if ((threadIdx.x & 31) == 0) {
    wm[threadIdx.x >> 5] = m;
    wb[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float bm = 0.f;
    int bb = 0;
    for (int w = 0; w < kBlock / 32; ++w) {
      bm = fmaxf(bm, wm[w]);
      bb |= wb[w];
    }
    if (!(bm >= 0.f)) bm = 0.f;
    atomicMax(&a.amax[blockIdx.z][blockIdx.y], __float_as_uint(bm));
    if (bb && a.nonfinite) atomicOr(a.nonfinite, 1u);
  }
  if (a.ticket == nullptr) return;
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();  // our amax contribution before our ticket
    last = atomicAdd(a.ticket, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < a.parts * a.nblocks; i += blockDim.x) {
    const int p = i / a.nblocks, blk = i - p * a.nblocks;
    const float am = __uint_as_float(__ldcg(&a.amax[p][blk]));
    a.scales[p][blk] = am > 0.f ? __fdiv_rn(am, 448.0f) : 1.0f;  // fp8.cpp:119
    a.amax[p][blk] = 0u;
  }
  if (threadIdx.x == 0) *a.ticket = 0u;
}

// Pass 2: scale = amax/448 (1 if 0) per block, written by the block's first vector;
// codes = encode(x / scale), IEEE division (fp8.cpp:119-121).
struct QuantArgs {
  Fp8Src src[2];
  Fp8Div div[2];
  const uint32_t* amax[2];   // scale = amax / 448 (1 if 0), written to scales[] ...
  const float* qscale[2];    // ... or, when set, the scale the amax pass finalized
  float* scales[2];
  uint8_t* codes[2];
  int64_t block_vecs;
};
// grid.y = block, grid.z = part: the block's scale is computed once per CTA.  Launched as a
// programmatic dependent of amax_vec_kernel: resident as the amax grid drains, waits for its
// completion (griddepcontrol.wait; a no-op for an ordinary launch) before reading the scale.
template <int SDT>  // as amax_vec_kernel
__global__ void __launch_bounds__(256, 4) quantize_vec_kernel(const __grid_constant__ QuantArgs a) {
  const int z = blockIdx.z, blk = blockIdx.y;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float qs;
  if (a.qscale[z] != nullptr) {
    qs = __ldcg(&a.qscale[z][blk]);
  } else {
    const float am = __uint_as_float(a.amax[z][blk]);
    qs = am > 0.f ? __fdiv_rn(am, 448.0f) : 1.0f;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.scales[z]) a.scales[z][blk] = qs;
  }
  const float inv = __frcp_rn(qs);
  const int64_t base = int64_t(blk) * a.block_vecs;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const Fp8Src& s = a.src[z];
  const int sdt = SDT >= 0 ? SDT : s.dt;
  if (sdt == FUSP_E4M3) {
    // Ring hop (protocols.cpp:113-115): codes = encode(RN(decode(c) * s_src) / s_new).  When
    // s_new == s_src the result is c itself: RN(RN(d * s) / s) = d (1 + e), |e| <= 2^-23, and
    // every E4M3 neighbour of d is >= 2^-4 away relatively (2^-9 absolutely near 0; 448 is
    // the saturation value), so the nearest code is d's own -- the vector is copied.  After the
    // first hop every segment of a chunk shares the chunk's scale, so later hops are copies.
    if (s.d % 16 == 0 && a.block_vecs % 2 == 0) {  // 16 codes per load, loads in flight
      const int64_t nv = a.block_vecs / 2, e0 = base * 8;
      for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < nv; v += kE4Unroll * stride) {
        uint4 w[kE4Unroll];
        float sc[kE4Unroll];
#pragma unroll
        for (int u = 0; u < kE4Unroll; ++u)
          if (v + u * stride < nv) {
            const int64_t i = e0 + (v + u * stride) * 16;
            w[u] = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(s.x) + i));
            sc[u] = e4m3_scale(s, a.div[z], i);
          }
#pragma unroll
        for (int u = 0; u < kE4Unroll; ++u)
          if (v + u * stride < nv) {
            uint4 o = w[u];
            if (sc[u] != qs) {
              const uint2 lo = encode8_finite(decode8(make_uint2(w[u].x, w[u].y), sc[u]), qs, inv);
              const uint2 hi = encode8_finite(decode8(make_uint2(w[u].z, w[u].w), sc[u]), qs, inv);
              o = make_uint4(lo.x, lo.y, hi.x, hi.y);
            }
            *reinterpret_cast<uint4*>(a.codes[z] + e0 + (v + u * stride) * 16) = o;
          }
      }
      return;
    }
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < a.block_vecs; v += stride) {
      const int64_t i = (base + v) * 8;
      const float sc = e4m3_scale(s, a.div[z], i);
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(static_cast<const uint8_t*>(s.x) + i));
      *reinterpret_cast<uint2*>(a.codes[z] + i) = sc == qs ? w : encode8_finite(decode8(w, sc), qs, inv);
    }
    return;
  }
  const int64_t v0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (sdt == FUSP_F32) quant_wide<FUSP_F32>(s.x, a.codes[z], base, v0, stride, a.block_vecs, qs, inv);
  else if (sdt == FUSP_F16) quant_wide<FUSP_F16>(s.x, a.codes[z], base, v0, stride, a.block_vecs, qs, inv);
  else quant_wide<FUSP_BF16>(s.x, a.codes[z], base, v0, stride, a.block_vecs, qs, inv);
}

// ---- one-launch per-tensor quantize for tensors that fit in the grid's registers ----------
// quantize (fp8.cpp:107-123) needs the whole tensor's amax before its first code, so it is two
// dependent passes -- two launches whose fixed costs dominate at the small per-rank sizes of
// U = 8 (FLUX: 3.5 MB per tensor; a memcpy of the same bytes reaches 0.1-0.2 of HBM).  Here
// one cooperative launch (every CTA co-resident) keeps each thread's share in registers
// (up to kFusedHold 16-byte pieces), reduces the amax, crosses a grid barrier, and encodes
// from the registers: one read of the source, one write of the codes, one launch.
// The barrier word (zero on entry, zero again on exit) packs arrivals in its low 16 bits and
// departures in its high 16 bits; the last CTA to depart also zeroes the amax words.
constexpr int kFusedHold = 6;
struct FusedQArgs {
  Fp8Src src[2];
  Fp8Div div[2];
  uint32_t* amax[2];      // one word per part (per-tensor), zero on entry and on exit
  float* scales[2];
  uint8_t* codes[2];
  int64_t units[2];       // 16-byte source pieces per part
  int cta0[3];            // CTAs [cta0[p], cta0[p+1]) serve part p
  uint32_t* barrier;      // zero on entry and on exit
  uint32_t* nonfinite;    // optional
  int parts;
};
template <int SDT>
__global__ void __launch_bounds__(256, 4) quantize_fused_kernel(const __grid_constant__ FusedQArgs a) {
  const int p = blockIdx.x >= static_cast<unsigned>(a.cta0[1]) ? 1 : 0;
  const Fp8Src& s = a.src[p];
  const int64_t per = int64_t(a.cta0[p + 1] - a.cta0[p]) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x - a.cta0[p]) * blockDim.x + threadIdx.x;
  constexpr int kElems = SDT == FUSP_E4M3 ? 16 : SDT == FUSP_F32 ? 4 : 8;  // per 16-byte piece
  uint4 w[kFusedHold];
  float sc[kFusedHold];
#pragma unroll
  for (int k = 0; k < kFusedHold; ++k) {
    const int64_t u = t0 + k * per;
    if (u < a.units[p]) {
      w[k] = __ldg(reinterpret_cast<const uint4*>(s.x) + u);
      if (SDT == FUSP_E4M3) sc[k] = e4m3_scale(s, a.div[p], u * 16);
    }
  }
  float m = 0.f;
  bool bad = false;
  uint32_t mag = 0;
#pragma unroll
  for (int k = 0; k < kFusedHold; ++k) {
    if (t0 + k * per >= a.units[p]) break;
    if (SDT == FUSP_E4M3) {
      uint32_t mm = __vmaxu4(__vmaxu4(w[k].x & 0x7F7F7F7Fu, w[k].y & 0x7F7F7F7Fu),
                             __vmaxu4(w[k].z & 0x7F7F7F7Fu, w[k].w & 0x7F7F7F7Fu));
      mm = max(max(mm & 0xFFu, (mm >> 8) & 0xFFu), max((mm >> 16) & 0xFFu, mm >> 24));
      float f[4];
      dec4(mm, sc[k], f);
      bad = bad || !(fabsf(f[0]) <= 3.402823466e38f);  // a NaN code (0x7F) decodes to NaN
      if (f[0] == f[0]) m = fmaxf(m, f[0]);
    } else {
      Raw8 r;
      r.a = w[k];
      r.b = make_uint4(0, 0, 0, 0);
      if (SDT == FUSP_F32) {  // 4 floats per piece: reuse the 8-lane helper on a padded vector
        uint32_t mm = max(max(w[k].x & 0x7FFFFFFFu, w[k].y & 0x7FFFFFFFu),
                          max(w[k].z & 0x7FFFFFFFu, w[k].w & 0x7FFFFFFFu));
        if (mm >= 0x7F800000u) {
          bad = true;
          const float f[4] = {__uint_as_float(w[k].x), __uint_as_float(w[k].y), __uint_as_float(w[k].z),
                              __uint_as_float(w[k].w)};
#pragma unroll
          for (int e = 0; e < 4; ++e) m = fmaxf(m, fabsf(f[e]));
        } else {
          mag = max(mag, mm);
        }
      } else if (!absmax_raw8(r, SDT, mag, bad)) {
        const Vec8 f = cvt8(r, SDT);
#pragma unroll
        for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(f.f[e]));
      }
    }
  }
  if (SDT != FUSP_E4M3) m = fmaxf(m, mag_to_f32(mag, SDT));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  bad = __any_sync(0xffffffffu, bad);
  __shared__ float wm[kBlock / 32];
  __shared__ int wb[kBlock / 32];
  __shared__ float qs_sh;
  if ((threadIdx.x & 31) == 0) {
    wm[threadIdx.x >> 5] = m;
    wb[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  const unsigned G = gridDim.x;
  if (threadIdx.x == 0) {
    float bm = 0.f;
    int bb = 0;
    for (int i = 0; i < kBlock / 32; ++i) {
      bm = fmaxf(bm, wm[i]);
      bb |= wb[i];
    }
    if (!(bm >= 0.f)) bm = 0.f;
    atomicMax(a.amax[p], __float_as_uint(bm));
    if (bb && a.nonfinite) atomicOr(a.nonfinite, 1u);
    // grid barrier: every CTA's amax contribution before anyone reads the amax
    __threadfence();
    atomicAdd(a.barrier, 1u);
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.barrier) : "memory");
      if ((v & 0xFFFFu) == G) break;
      __nanosleep(32);
    } while (true);
    const float am = __uint_as_float(__ldcg(a.amax[p]));
    const float qs = am > 0.f ? __fdiv_rn(am, 448.0f) : 1.0f;  // fp8.cpp:119
    qs_sh = qs;
    if (blockIdx.x == static_cast<unsigned>(a.cta0[p])) *a.scales[p] = qs;
  }
  __syncthreads();
  const float qs = qs_sh, inv = __frcp_rn(qs);
#pragma unroll
  for (int k = 0; k < kFusedHold; ++k) {
    const int64_t u = t0 + k * per;
    if (u >= a.units[p]) break;
    if (SDT == FUSP_E4M3) {
      uint4 o = w[k];
      if (sc[k] != qs) {  // same scale: the codes themselves (see quantize_vec_kernel)
        const uint2 lo = encode8_finite(decode8(make_uint2(w[k].x, w[k].y), sc[k]), qs, inv);
        const uint2 hi = encode8_finite(decode8(make_uint2(w[k].z, w[k].w), sc[k]), qs, inv);
        o = make_uint4(lo.x, lo.y, hi.x, hi.y);
      }
      reinterpret_cast<uint4*>(a.codes[p])[u] = o;
    } else if (SDT == FUSP_F32) {
      const float f0 = qdiv(__uint_as_float(w[k].x), qs, inv), f1 = qdiv(__uint_as_float(w[k].y), qs, inv);
      const float f2 = qdiv(__uint_as_float(w[k].z), qs, inv), f3 = qdiv(__uint_as_float(w[k].w), qs, inv);
      reinterpret_cast<uint32_t*>(a.codes[p])[u] = enc_pair_finite(f0, f1) | (enc_pair_finite(f2, f3) << 16);
    } else {
      Raw8 r;
      r.a = w[k];
      r.b = make_uint4(0, 0, 0, 0);
      reinterpret_cast<uint2*>(a.codes[p])[u] = encode8_finite(cvt8(r, SDT), qs, inv);
    }
  }
  if (threadIdx.x == 0) {  // depart; the last CTA out leaves the words zero for the next launch
    const uint32_t old = atomicAdd(a.barrier, 0x10000u);
    if ((old >> 16) == G - 1) {
      for (int q = 0; q < a.parts; ++q) *a.amax[q] = 0u;
      __threadfence();
      *a.barrier = 0u;
    }
  }
}

// ---- FP8 Ulysses pack in one cooperative launch (per-tensor scales, small tensors) ---------
// The FP8 input reshard quantizes the whole local K and V (fp8.cpp:107-123, protocols.cpp:
// 139-153) and packs them with Q into the slots: an amax launch, then the pack.  When K and V
// fit the registers of the grid (every FLUX U = 8 shape) one cooperative launch does both:
// each thread keeps its share of K or V, the CTAs reduce the two amaxes while ALL of them copy
// Q into its slots, cross a grid barrier, then encode from the registers straight into the
// slots (the members' windows on the peer path) and write the slot trailers.
struct FusedPackArgs {
  PackArgs pk;            // op[0] = Q (plain 16-bit copy), op[1] = K, op[2] = V (E4M3)
  FDiv slab_vecs, h, hp;  // vector -> slab, slab -> head, head -> slot
  uint32_t* amax[2];      // zero on entry and on exit
  float* scales[2];       // out: the K and V scales
  uint32_t* barrier;      // zero on entry and on exit (arrivals low, departures high 16 bits)
  int64_t nvec;           // 16-byte vectors per tensor (B*H*SL*D / 8)
  int cta0[3];            // CTAs [cta0[p], cta0[p+1]) hold part p (K, V)
};
__device__ __forceinline__ int64_t fused_pack_dst(const FusedPackArgs& a, int64_t v, int64_t desz,
                                                  int64_t slot_stride) {
  const PackArgs& k = a.pk;
  const uint32_t slab = fdiv(a.slab_vecs, static_cast<uint32_t>(v));
  const uint32_t off = static_cast<uint32_t>(v) - slab * a.slab_vecs.d;
  const uint32_t bb = fdiv(a.h, slab), hh = slab - bb * a.h.d;
  const uint32_t t = fdiv(a.hp, hh), hl = hh - t * a.hp.d;
  return (k.peer ? k.slot_boff[t] / desz : int64_t(t) * slot_stride) +
         (int64_t(bb) * k.hp + hl) * k.slab_elems + int64_t(off) * 8;
}
template <int SDT>
__global__ void __launch_bounds__(256, 4) pack_fp8_fused_kernel(const __grid_constant__ FusedPackArgs a) {
  const int p = blockIdx.x >= static_cast<unsigned>(a.cta0[1]) ? 1 : 0;
  const PackOp& o = a.pk.op[1 + p];
  const int64_t per = int64_t(a.cta0[p + 1] - a.cta0[p]) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x - a.cta0[p]) * blockDim.x + threadIdx.x;
  uint4 w[kFusedHold];
#pragma unroll
  for (int k = 0; k < kFusedHold; ++k)
    if (t0 + k * per < a.nvec) w[k] = __ldg(reinterpret_cast<const uint4*>(o.src) + t0 + k * per);
  float m = 0.f;
  bool bad = false;
  uint32_t mag = 0;
#pragma unroll
  for (int k = 0; k < kFusedHold; ++k) {
    if (t0 + k * per >= a.nvec) break;
    Raw8 r;
    r.a = w[k];
    r.b = make_uint4(0, 0, 0, 0);
    if (!absmax_raw8(r, SDT, mag, bad)) {
      const Vec8 f = cvt8(r, SDT);
#pragma unroll
      for (int e = 0; e < 8; ++e) m = fmaxf(m, fabsf(f.f[e]));
    }
  }
  m = fmaxf(m, mag_to_f32(mag, SDT));
  for (int q = 16; q > 0; q >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, q));
  __shared__ float wm[kBlock / 32];
  __shared__ float qs_sh;
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  const unsigned G = gridDim.x;
  if (threadIdx.x == 0) {
    float bm = 0.f;
    for (int i = 0; i < kBlock / 32; ++i) bm = fmaxf(bm, wm[i]);
    if (!(bm >= 0.f)) bm = 0.f;
    atomicMax(a.amax[p], __float_as_uint(bm));
    __threadfence();
    atomicAdd(a.barrier, 1u);
  }
  // Q needs no scale: every CTA copies its share into the slots while the others arrive
  {
    const PackOp& qo = a.pk.op[0];
    const int64_t qstride = int64_t(G) * blockDim.x;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < a.nvec; v += qstride)
      reinterpret_cast<uint4*>(qo.dst)[fused_pack_dst(a, v, 2, qo.slot_stride) / 8] =
          __ldg(reinterpret_cast<const uint4*>(qo.src) + v);
  }
  if (threadIdx.x == 0) {
    uint32_t bv;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(bv) : "l"(a.barrier) : "memory");
      if ((bv & 0xFFFFu) == G) break;
      __nanosleep(32);
    } while (true);
    const float am = __uint_as_float(__ldcg(a.amax[p]));
    const float qs = am > 0.f ? __fdiv_rn(am, 448.0f) : 1.0f;  // fp8.cpp:119
    qs_sh = qs;
    if (blockIdx.x == static_cast<unsigned>(a.cta0[p])) {
      *a.scales[p] = qs;
      // slot trailers: slice_heads keeps the tensor-wide scale (fp8.cpp:100-105)
      const int u = a.pk.h / a.pk.hp;
      for (int t = 0; t < u; ++t)
        o.trailer[a.pk.peer ? a.pk.slot_boff[t] / 4 : t * o.trailer_stride] = qs;
    }
  }
  __syncthreads();
  const float qs = qs_sh;
  (void)bad;  // (non-finite inputs are the caller's check_finite; the codes saturate like pack)
#pragma unroll
  for (int k = 0; k < kFusedHold; ++k) {
    const int64_t v = t0 + k * per;
    if (v >= a.nvec) break;
    Raw8 r;
    r.a = w[k];
    r.b = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint2*>(static_cast<uint8_t*>(o.dst) + fused_pack_dst(a, v, 1, o.slot_stride)) =
        encode8(cvt8(r, SDT), qs);
  }
  if (a.pk.peer) __threadfence_system();  // remote stores visible before the exchange signal
  __syncthreads();
  if (threadIdx.x == 0) {  // depart; the last CTA out leaves the words zero
    const uint32_t old = atomicAdd(a.barrier, 0x10000u);
    if ((old >> 16) == G - 1) {
      *a.amax[0] = 0u;
      *a.amax[1] = 0u;
      __threadfence();
      *a.barrier = 0u;
    }
  }
}

__global__ void __launch_bounds__(256) dequantize_vec_kernel(const uint8_t* __restrict__ c,
                                                             const float* __restrict__ scales,
                                                             FDiv block_vecs, int64_t n_vecs,
                                                             void* __restrict__ y, int ydt) {
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n_vecs;
       v += int64_t(gridDim.x) * blockDim.x)
    store8(y, ydt, v * 8, decode8(__ldg(reinterpret_cast<const uint2*>(c + v * 8)),
                                  scales[fdiv(block_vecs, static_cast<uint32_t>(v))]));
}

}  // namespace

size_t dtype_size(int dt) {
  switch (dt) {
    case FUSP_F32: return 4;
    case FUSP_F16:
    case FUSP_BF16: return 2;
    case FUSP_E4M3: return 1;
  }
  return 0;
}

#define FUSP_LAUNCHED(name)                                    \
  do {                                                         \
    count_launch();                                            \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return set_cuda_error(_e, name);    \
  } while (0)

fusp_status launch_convert(const void* x, int xdt, void* y, int ydt, int64_t n, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  if (xdt == FUSP_BF16 && ydt == FUSP_F16 && n % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) % 16 == 0) {
    bf16_to_f16_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(static_cast<const uint4*>(x),
                                                            static_cast<uint4*>(y), n / 8);
    FUSP_LAUNCHED("bf16_to_f16_kernel");
    return FUSP_OK;
  }
  convert_kernel<<<grid_for(n), kBlock, 0, s>>>(x, xdt, y, ydt, n);
  FUSP_LAUNCHED("convert_kernel");
  return FUSP_OK;
}

fusp_status launch_encode(const float* x, int64_t n, uint8_t* c, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  encode_kernel<<<grid_for(n), kBlock, 0, s>>>(x, n, c);
  FUSP_LAUNCHED("encode_kernel");
  return FUSP_OK;
}

fusp_status launch_decode(const uint8_t* c, int64_t n, float* y, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  decode_kernel<<<grid_for(n), kBlock, 0, s>>>(c, n, y);
  FUSP_LAUNCHED("decode_kernel");
  return FUSP_OK;
}

fusp_status launch_amax(const void* x, int dt, int64_t n, uint32_t* amax_bits, uint32_t* nonfinite,
                        cudaStream_t s) {
  FUSP_CUDA(cudaMemsetAsync(amax_bits, 0, sizeof(uint32_t), s));
  FUSP_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(uint32_t), s));
  if (n <= 0) return FUSP_OK;
  amax_kernel<<<grid_for(n, 4), kBlock, 0, s>>>(x, dt, n, amax_bits, nonfinite);
  FUSP_LAUNCHED("amax_kernel");
  return FUSP_OK;
}

fusp_status launch_quantize(const void* x, int dt, int64_t n, const uint32_t* amax_bits,
                            float* scale_out, uint8_t* codes, cudaStream_t s) {
  quantize_kernel<<<grid_for(n), kBlock, 0, s>>>(x, dt, n, amax_bits, scale_out, codes);
  FUSP_LAUNCHED("quantize_kernel");
  return FUSP_OK;
}

fusp_status launch_dequantize(const uint8_t* c, const float* scale, int64_t n, void* y, int ydt,
                              cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  dequantize_kernel<<<grid_for(n), kBlock, 0, s>>>(c, scale, n, y, ydt);
  FUSP_LAUNCHED("dequantize_kernel");
  return FUSP_OK;
}

fusp_status launch_merge(const float* o1, const float* l1, const float* o2, const float* l2,
                         int64_t rows, int d, float* out, float* lse, cudaStream_t s) {
  if (rows <= 0) return FUSP_OK;
  merge_kernel<<<grid_for(rows * 32), kBlock, 0, s>>>(o1, l1, o2, l2, rows, d, out, lse);
  FUSP_LAUNCHED("merge_kernel");
  return FUSP_OK;
}

fusp_status launch_fill(void* p, int dt, int64_t n, float v, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  fill_kernel<<<grid_for(n), kBlock, 0, s>>>(p, dt, n, v);
  FUSP_LAUNCHED("fill_kernel");
  return FUSP_OK;
}

fusp_status launch_pack_generic(const PackDesc& p, cudaStream_t s);
fusp_status launch_unpack_generic(const UnpackDesc& p, cudaStream_t s);
namespace {
bool aligned16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }
int slab_grid_x(int64_t slab_vecs, int64_t slabs) {
  // enough CTAs per slab to cover it once with 4 vectors per thread, capped near 16
  // resident CTAs per SM overall
  int64_t gx = (slab_vecs + 4 * kBlock - 1) / (4 * kBlock);
  const int64_t cap = (int64_t(sm_count()) * 16 + slabs - 1) / slabs;
  if (gx > cap) gx = cap;
  return gx < 1 ? 1 : static_cast<int>(gx);
}
}  // namespace

fusp_status launch_pack_multi(const PackDesc* ps, int n, cudaStream_t s, bool pdl,
                              const int64_t* peer_slot_boff) {
  if (n <= 0) return FUSP_OK;
  const PackDesc& p0 = ps[0];
  const int64_t slab_elems = int64_t(p0.sl) * p0.d;
  const int64_t slabs = int64_t(p0.b) * p0.h;
  bool fast = n <= kMaxMoveOps && p0.d % 8 == 0 && p0.h % p0.u == 0 && slabs <= 65535 &&
              slab_elems / 8 < (int64_t(1) << 31);
  for (int i = 0; i < n && fast; ++i) {
    const PackDesc& p = ps[i];
    fast = p.b == p0.b && p.h == p0.h && p.sl == p0.sl && p.d == p0.d && p.u == p0.u &&
           aligned16(p.src) && aligned16(p.dst) && (p.dst_dtype != FUSP_E4M3 || p.dst_slot_stride % 16 == 0) &&
           (p.dst_dtype == FUSP_E4M3 || (p.dst_slot_stride * int64_t(dtype_size(p.dst_dtype))) % 16 == 0) &&
           p.src_dtype != FUSP_E4M3;
  }
  if (!fast) {
    if (peer_slot_boff != nullptr)
      return set_error(FUSP_ERR_UNSUPPORTED, "peer pack: shape not 16-byte granular");
    for (int i = 0; i < n; ++i) FUSP_CHECK(launch_pack_generic(ps[i], s));
    return FUSP_OK;
  }
  if (slabs == 0 || slab_elems == 0) return FUSP_OK;
  PackArgs a{};
  if (peer_slot_boff != nullptr) {
    if (p0.u > kMaxPeerChunks) return set_error(FUSP_ERR_UNSUPPORTED, "peer pack: too many members");
    a.peer = 1;
    for (int t = 0; t < p0.u; ++t) {
      a.slot_boff[t] = peer_slot_boff[t];
      if (peer_slot_boff[t] % 16 != 0) return set_error(FUSP_ERR_INVALID_ARGUMENT, "peer pack: misaligned slot");
    }
  }
  for (int i = 0; i < n; ++i) {
    a.op[i] = PackOp{ps[i].src, ps[i].dst, ps[i].scale, ps[i].amax_bits, ps[i].trailer,
                     ps[i].trailer_stride, ps[i].scale_bh_stride, ps[i].dst_slot_stride,
                     ps[i].src_dtype, ps[i].dst_dtype};
  }
  a.h = p0.h;
  a.hp = p0.h / p0.u;
  a.slab_vecs = static_cast<int>(slab_elems / 8);
  a.slab_elems = slab_elems;
  const dim3 grid(slab_grid_x(a.slab_vecs, slabs * n), static_cast<unsigned>(slabs), n);
  if (pdl) FUSP_CUDA(launch_pdl(pack_slab_kernel, grid, s, a));
  else pack_slab_kernel<<<grid, kBlock, 0, s>>>(a);
  FUSP_LAUNCHED("pack_slab_kernel");
  return FUSP_OK;
}

fusp_status try_pack_fp8_fused(const PackDesc* ps, uint32_t* const* amax, float* const* scales,
                              const int64_t* peer_slot_boff, cudaStream_t s, bool* done) {
  *done = false;
  static const bool off = getenv("FUSP_FP8_FUSED") != nullptr && atoi(getenv("FUSP_FP8_FUSED")) == 0;
  const PackDesc& q = ps[0];
  const int dt = q.src_dtype;
  if (off || (dt != FUSP_BF16 && dt != FUSP_F16) || q.dst_dtype != dt) return FUSP_OK;
  const int64_t slab_elems = int64_t(q.sl) * q.d;
  const int64_t slabs = int64_t(q.b) * q.h;
  const int64_t n = slabs * slab_elems;
  if (n <= 0 || n % 8 != 0 || slab_elems % 8 != 0 || q.h % q.u != 0 || n / 8 >= (int64_t(1) << 31))
    return FUSP_OK;
  for (int i = 0; i < 3; ++i) {
    const PackDesc& p = ps[i];
    if (p.src_dtype != dt || p.b != q.b || p.h != q.h || p.sl != q.sl || p.d != q.d || p.u != q.u ||
        !aligned16(p.src) || !aligned16(p.dst))
      return FUSP_OK;
    if (i > 0 && (p.dst_dtype != FUSP_E4M3 || p.scale_bh_stride != 0 || p.trailer == nullptr ||
                  p.dst_slot_stride % 16 != 0))
      return FUSP_OK;
  }
  if ((q.dst_slot_stride * 2) % 16 != 0) return FUSP_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FUSP_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return FUSP_OK;
  FusedPackArgs a{};
  if (peer_slot_boff != nullptr) {
    if (q.u > kMaxPeerChunks) return FUSP_OK;
    a.pk.peer = 1;
    for (int t = 0; t < q.u; ++t) {
      if (peer_slot_boff[t] % 16 != 0) return FUSP_OK;
      a.pk.slot_boff[t] = peer_slot_boff[t];
    }
  }
  for (int i = 0; i < 3; ++i)
    a.pk.op[i] = PackOp{ps[i].src, ps[i].dst, ps[i].scale, ps[i].amax_bits, ps[i].trailer,
                        ps[i].trailer_stride, 0, ps[i].dst_slot_stride, ps[i].src_dtype, ps[i].dst_dtype};
  a.pk.h = q.h;
  a.pk.hp = q.h / q.u;
  a.pk.slab_vecs = static_cast<int>(slab_elems / 8);
  a.pk.slab_elems = slab_elems;
  a.slab_vecs = make_fdiv(static_cast<uint32_t>(slab_elems / 8));
  a.h = make_fdiv(static_cast<uint32_t>(q.h));
  a.hp = make_fdiv(static_cast<uint32_t>(q.h / q.u));
  a.nvec = n / 8;
  a.amax[0] = amax[0];
  a.amax[1] = amax[1];
  a.scales[0] = scales[0];
  a.scales[1] = scales[1];
  a.barrier = amax[0] + 1;  // the amax pass's ticket word (zero on entry and on exit)
  const int per_part = static_cast<int>((a.nvec + int64_t(kBlock) * kFusedHold - 1) / (int64_t(kBlock) * kFusedHold));
  a.cta0[0] = 0;
  a.cta0[1] = per_part;
  a.cta0[2] = 2 * per_part;
  void (*k)(FusedPackArgs) = dt == FUSP_BF16 ? pack_fp8_fused_kernel<FUSP_BF16> : pack_fp8_fused_kernel<FUSP_F16>;
  int dev = 0;
  FUSP_CUDA(cudaGetDevice(&dev));
  int occ = 0;
  static std::atomic<int> per_sm[16][2];
  const int slot = dt == FUSP_BF16 ? 0 : 1;
  if (dev < 16 && per_sm[dev][slot].load() > 0) {
    occ = per_sm[dev][slot].load();
  } else {
    FUSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBlock, 0));
    if (dev < 16) per_sm[dev][slot].store(occ);
  }
  const int grid = a.cta0[2];
  if (occ < 2 || grid > (occ - 1) * sm_count() || grid >= 0xFFFF) return FUSP_OK;  // see quantize
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FUSP_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  FUSP_LAUNCHED("pack_fp8_fused_kernel");
  *done = true;
  return FUSP_OK;
}

fusp_status launch_unpack_multi(const UnpackDesc* us, int n, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  const UnpackDesc& u0 = us[0];
  const int64_t slab_elems = int64_t(u0.sl) * u0.d;
  const int64_t slabs = int64_t(u0.u) * u0.b * u0.hp;
  bool fast = n <= kMaxMoveOps && u0.d % 8 == 0 && slabs <= 65535 && slab_elems / 8 < (int64_t(1) << 31);
  for (int i = 0; i < n && fast; ++i) {
    const UnpackDesc& u = us[i];
    const int64_t esz = u.src_dtype == FUSP_E4M3 ? 1 : int64_t(dtype_size(u.src_dtype));
    fast = u.b == u0.b && u.hp == u0.hp && u.sl == u0.sl && u.d == u0.d && u.u == u0.u &&
           aligned16(u.src) && aligned16(u.dst) && (u.src_slot_stride * esz) % 16 == 0 &&
           (u.dst_dtype != FUSP_E4M3 || u.src_dtype == FUSP_E4M3);
  }
  if (!fast) {
    for (int i = 0; i < n; ++i) FUSP_CHECK(launch_unpack_generic(us[i], s));
    return FUSP_OK;
  }
  if (slabs == 0 || slab_elems == 0) return FUSP_OK;
  UnpackArgs a{};
  for (int i = 0; i < n; ++i)
    a.op[i] = UnpackOp{us[i].src, us[i].dst, us[i].scales, us[i].src_slot_stride, us[i].scale_stride,
                       us[i].scale_bh_stride, us[i].src_dtype, us[i].dst_dtype};
  a.bhp = u0.b * u0.hp;
  a.sl = u0.sl;
  a.u = u0.u;
  a.slab_vecs = static_cast<int>(slab_elems / 8);
  a.slab_elems = slab_elems;
  unpack_slab_kernel<<<dim3(slab_grid_x(a.slab_vecs, slabs * n), static_cast<unsigned>(slabs), n),
                       kBlock, 0, s>>>(a);
  FUSP_LAUNCHED("unpack_slab_kernel");
  return FUSP_OK;
}

fusp_status launch_stage(const StageOp* ops, int n, int bhp, int sl, int d, int u, cudaStream_t s) {
  if (n <= 0 || bhp <= 0 || sl <= 0 || u <= 0) return FUSP_OK;
  if (n > kMaxStageOps) return set_error(FUSP_ERR_INVALID_ARGUMENT, "stage: too many operands");
  const int64_t slab_elems = int64_t(sl) * d;
  const int64_t slabs = int64_t(u) * bhp;
  if (d % 8 != 0 || slabs > 65535 || slab_elems / 8 >= (int64_t(1) << 31))
    return set_error(FUSP_ERR_SHAPE, "stage: unsupported operand shape");
  StageArgs a{};
  bool vec = true, guarded_any = false;
  for (int i = 0; i < n; ++i) {
    const StageOp& o = ops[i];
    const int64_t esz = int64_t(dtype_size(o.sdt));
    const bool ok = (o.sdt != FUSP_E4M3 || o.scales != nullptr) &&
                    (o.exps == nullptr || (o.words != nullptr && o.dst != nullptr && o.ddt == FUSP_F16)) &&
                    (o.dst == nullptr || o.ddt != FUSP_E4M3);
    if (!ok) return set_error(FUSP_ERR_INVALID_ARGUMENT, "stage: malformed operand");
    a.op[i] = o;
    StageOp& x = a.op[i];
    if (x.src_bh_stride == 0) x.src_bh_stride = slab_elems;
    if (x.dst_slot_stride == 0) x.dst_slot_stride = slab_elems;
    if (x.dst_bh_stride == 0) x.dst_bh_stride = int64_t(u) * slab_elems;
    const int64_t dsz = x.dst != nullptr ? int64_t(dtype_size(x.ddt)) : esz;
    vec = vec && aligned16(o.src) && (o.dst == nullptr || aligned16(o.dst)) &&
          (o.raw == nullptr || aligned16(o.raw)) && (x.src_slot_stride * esz) % 16 == 0 &&
          (x.src_bh_stride * esz) % 16 == 0 && (x.dst_slot_stride * dsz) % 16 == 0 &&
          (x.dst_bh_stride * dsz) % 16 == 0 &&
          (x.raw == nullptr || ((x.dst_slot_stride * esz) % 16 == 0 && (x.dst_bh_stride * esz) % 16 == 0));
    guarded_any = guarded_any || o.exps != nullptr;
  }
  if (!vec) {
    // small head dims (attention_generic.cu) can leave slabs off 16-byte boundaries: an
    // element-wise pass with the same mapping (never range-guarded: those operands are f32 or
    // the caller's dtype)
    if (guarded_any)
      return set_error(FUSP_ERR_INVALID_ARGUMENT, "stage: range-guarded operand not 16-byte aligned");
    a.bhp = bhp;
    a.u = u;
    a.slab_elems = slab_elems;
    const int64_t total = slab_elems * slabs;
    stage_scalar_kernel<<<dim3(static_cast<unsigned>(grid_for(total)), n), kBlock, 0, s>>>(a, total);
    FUSP_LAUNCHED("stage_scalar_kernel");
    return FUSP_OK;
  }
  a.bhp = bhp;
  a.u = u;
  a.slab_vecs = static_cast<int>(slab_elems / 8);
  a.slab_elems = slab_elems;
  // one resident wave (4 CTAs per SM): each CTA loops over its slab part, so the per-CTA
  // ticket of the range guard is paid once per CTA, not once per 16 KB
  int64_t gx = (a.slab_vecs + 4 * kBlock - 1) / (4 * kBlock);
  const int64_t cap = (int64_t(sm_count()) * FUSP_STAGE_WAVES + slabs * n - 1) / (slabs * n);
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  stage_kernel<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(slabs), n), kBlock, 0, s>>>(a);
  FUSP_LAUNCHED("stage_kernel");
  bool guarded = false;
  for (int i = 0; i < n; ++i) guarded = guarded || a.op[i].exps != nullptr;
  if (guarded) {
    // programmatic dependent launch: the decision kernel's launch latency hides under the
    // staging grid instead of following it
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(bhp), n, kFixParts);
    cfg.blockDim = dim3(kBlock);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FUSP_CUDA(cudaLaunchKernelEx(&cfg, stage_decide_kernel, a));
    FUSP_LAUNCHED("stage_decide_kernel");
  }
  return FUSP_OK;
}

fusp_status launch_pack(const PackDesc& p, cudaStream_t s) { return launch_pack_multi(&p, 1, s); }
fusp_status launch_unpack(const UnpackDesc& p, cudaStream_t s) { return launch_unpack_multi(&p, 1, s); }

fusp_status launch_pack_generic(const PackDesc& p, cudaStream_t s) {
  const int64_t n = int64_t(p.b) * p.h * p.sl * p.d;
  if (n <= 0) return FUSP_OK;
  if (p.d % 8 != 0) return set_error(FUSP_ERR_SHAPE, "pack: head dim must be a multiple of 8");
  const float* scale = p.scale;
  if (p.dst_dtype == FUSP_E4M3 && p.amax_bits != nullptr) {
    // unfused form of the fast path's scale + trailer handling: amax words -> scales in place
    const int nsc = p.scale_bh_stride != 0 ? p.b * p.h : 1;
    uint32_t* w = const_cast<uint32_t*>(p.amax_bits);
    finalize_scales_kernel<<<(nsc + kBlock - 1) / kBlock, kBlock, 0, s>>>(w, nsc, reinterpret_cast<float*>(w));
    FUSP_LAUNCHED("finalize_scales_kernel");
    scale = reinterpret_cast<const float*>(w);
  }
  if (p.dst_dtype == FUSP_E4M3 && p.trailer != nullptr)
    FUSP_CHECK(launch_scatter_slot_scales(scale, p.trailer, p.trailer_stride, p.b, p.h, p.u,
                                          p.scale_bh_stride != 0 ? 1 : 0, s));
  pack_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(p.src, p.src_dtype, p.dst, p.dst_dtype,
                                                  p.dst_slot_stride, p.b, p.h, p.sl, p.d, p.u,
                                                  scale, p.scale_bh_stride);
  FUSP_LAUNCHED("pack_kernel");
  return FUSP_OK;
}

fusp_status launch_unpack_generic(const UnpackDesc& p, cudaStream_t s) {
  const int64_t n = int64_t(p.b) * p.hp * p.sl * p.d * p.u;
  if (n <= 0) return FUSP_OK;
  if (p.d % 8 != 0) return set_error(FUSP_ERR_SHAPE, "unpack: head dim must be a multiple of 8");
  unpack_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(p.src, p.src_dtype, p.src_slot_stride, p.scales,
                                                    p.scale_stride, p.scale_bh_stride, p.dst,
                                                    p.dst_dtype, p.b, p.hp, p.sl, p.d, p.u);
  FUSP_LAUNCHED("unpack_kernel");
  return FUSP_OK;
}

fusp_status launch_unpack_heads(const void* src, int64_t slot_stride, void* dst, int dtype, int b,
                                int hp, int sl, int d, int u, cudaStream_t s) {
  const int esz = static_cast<int>(dtype_size(dtype));
  const int64_t bytes = int64_t(b) * hp * sl * d * esz * u;
  if (bytes <= 0) return FUSP_OK;
  if ((int64_t(sl) * d * esz) % 16 != 0)
    return set_error(FUSP_ERR_SHAPE, "unpack_heads: slab not 16-byte granular");
  unpack_heads_kernel<<<grid_for(bytes / 16), kBlock, 0, s>>>(
      static_cast<const uint8_t*>(src), slot_stride * esz, static_cast<uint8_t*>(dst), esz, b, hp,
      sl, d, u);
  FUSP_LAUNCHED("unpack_heads_kernel");
  return FUSP_OK;
}

}  // namespace fusp

namespace fusp {

fusp_status launch_amax_blocks_raw(const Fp8Src& src, int64_t block_elems, int nblocks,
                                   uint32_t* amax, cudaStream_t s) {  // amax zeroed by the caller
  if (block_elems <= 0 || nblocks <= 0) return FUSP_OK;
  int gx = grid_for(block_elems, 4);
  const int cap = (sm_count() * 8 + nblocks - 1) / nblocks;
  if (gx > cap) gx = cap < 1 ? 1 : cap;
  amax_blocks_kernel<<<dim3(gx, nblocks), kBlock, 0, s>>>(src, block_elems, amax, nullptr);
  FUSP_LAUNCHED("amax_blocks_kernel");
  return FUSP_OK;
}

namespace {
// CTAs along a block for the FP8 passes: every thread takes >= 8 vectors (two rounds of 4 in
// flight), at most 4 CTAs per SM over all blocks and parts -- few CTAs, so the per-CTA atomics
// on the block's amax word and the finalize ticket (one address each) stay off the critical
// path (ncu: 1184 CTAs x 2 same-address atomics cost ~3 us at FLUX U=8).
int fp8_grid_x(int64_t block_vecs, int blocks_total) {
  // one pass of kFp8Unroll vectors per thread when the grid allows, at most one resident
  // wave (the kernels' 4 CTAs per SM)
  int64_t gx = (block_vecs + kBlock * kFp8Unroll - 1) / (kBlock * kFp8Unroll);
  const int64_t cap = (int64_t(sm_count()) * 4 + blocks_total - 1) / blocks_total;
  if (gx > cap) gx = cap;
  return gx < 1 ? 1 : static_cast<int>(gx);
}
// The FP8 pass instance for the sources' common dtype (-1: mixed, resolved per part).
int fp8_common_dt(const Fp8Src* src, int parts) {
  for (int p = 1; p < parts; ++p)
    if (src[p].dt != src[0].dt) return -1;
  return src[0].dt;
}
using AmaxKern = void (*)(AmaxArgs);
using QuantKern = void (*)(QuantArgs);
AmaxKern amax_kernel_for(int dt) {
  switch (dt) {
    case FUSP_BF16: return amax_vec_kernel<FUSP_BF16>;
    case FUSP_F16: return amax_vec_kernel<FUSP_F16>;
    case FUSP_F32: return amax_vec_kernel<FUSP_F32>;
    case FUSP_E4M3: return amax_vec_kernel<FUSP_E4M3>;
    default: return amax_vec_kernel<-1>;
  }
}
QuantKern quantize_kernel_for(int dt) {
  switch (dt) {
    case FUSP_BF16: return quantize_vec_kernel<FUSP_BF16>;
    case FUSP_F16: return quantize_vec_kernel<FUSP_F16>;
    case FUSP_F32: return quantize_vec_kernel<FUSP_F32>;
    case FUSP_E4M3: return quantize_vec_kernel<FUSP_E4M3>;
    default: return quantize_vec_kernel<-1>;
  }
}
bool fp8_vec_ok(const Fp8Src& src, int64_t n, int64_t block_elems, const void* codes) {
  return n % 8 == 0 && block_elems % 8 == 0 && src.d % 8 == 0 && aligned16(src.x) &&
         aligned16(codes);
}
}  // namespace

fusp_status launch_amax_blocks(const Fp8Src& src, int64_t block_elems, int nblocks,
                               uint32_t* amax, uint32_t* nonfinite, cudaStream_t s) {
  FUSP_CUDA(cudaMemsetAsync(amax, 0, sizeof(uint32_t) * nblocks, s));
  if (nonfinite) FUSP_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(uint32_t), s));
  if (block_elems <= 0 || nblocks <= 0) return FUSP_OK;
  if (block_elems % 8 == 0 && src.d % 8 == 0 && aligned16(src.x) && nblocks <= 65535 &&
      block_elems * nblocks < (int64_t(1) << 31)) {
    AmaxArgs a{};
    a.src[0] = src;
    a.div[0] = make_fp8div(src);
    a.amax[0] = amax;
    a.block_vecs = block_elems / 8;
    a.nonfinite = nonfinite;
    const int gx = fp8_grid_x(a.block_vecs, nblocks);
    amax_kernel_for(src.dt)<<<dim3(gx, nblocks, 1), kBlock, 0, s>>>(a);
    FUSP_LAUNCHED("amax_vec_kernel");
    finalize_scales_kernel<<<(nblocks + kBlock - 1) / kBlock, kBlock, 0, s>>>(
        amax, nblocks, reinterpret_cast<float*>(amax));
    FUSP_LAUNCHED("finalize_scales_kernel");
    return FUSP_OK;
  }
  int gx = grid_for(block_elems, 4);
  const int cap = (sm_count() * 8 + nblocks - 1) / nblocks;  // ~8 CTAs per SM in total
  if (gx > cap) gx = cap < 1 ? 1 : cap;
  amax_blocks_kernel<<<dim3(gx, nblocks), kBlock, 0, s>>>(src, block_elems, amax, nonfinite);
  FUSP_LAUNCHED("amax_blocks_kernel");
  finalize_scales_kernel<<<(nblocks + kBlock - 1) / kBlock, kBlock, 0, s>>>(
      amax, nblocks, reinterpret_cast<float*>(amax));
  FUSP_LAUNCHED("finalize_scales_kernel");
  return FUSP_OK;
}

fusp_status launch_quantize_blocks(const Fp8Src& src, int64_t n, int64_t block_elems,
                                   const float* scales, uint8_t* codes, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  quantize_blocks_kernel<<<grid_for(n), kBlock, 0, s>>>(src, n, block_elems, scales, codes);
  FUSP_LAUNCHED("quantize_blocks_kernel");
  return FUSP_OK;
}


fusp_status launch_amax_multi(const Fp8Src* src, int parts, int64_t block_elems, int nblocks,
                              uint32_t* const* amax, cudaStream_t s) {
  bool fast = parts >= 1 && parts <= 2 && nblocks <= 65535 && block_elems % 8 == 0 &&
              block_elems * nblocks < (int64_t(1) << 31);
  for (int p = 0; p < parts && fast; ++p) fast = src[p].d % 8 == 0 && aligned16(src[p].x);
  if (!fast) {
    for (int p = 0; p < parts; ++p) {
      FUSP_CUDA(cudaMemsetAsync(amax[p], 0, sizeof(uint32_t) * nblocks, s));
      FUSP_CHECK(launch_amax_blocks_raw(src[p], block_elems, nblocks, amax[p], s));
    }
    return FUSP_OK;
  }
  if (parts == 2 && amax[1] == amax[0] + nblocks) {
    FUSP_CUDA(cudaMemsetAsync(amax[0], 0, sizeof(uint32_t) * 2 * nblocks, s));
  } else {
    for (int p = 0; p < parts; ++p) FUSP_CUDA(cudaMemsetAsync(amax[p], 0, sizeof(uint32_t) * nblocks, s));
  }
  AmaxArgs a{};
  for (int p = 0; p < parts; ++p) {
    a.src[p] = src[p];
    a.div[p] = make_fp8div(src[p]);
    a.amax[p] = amax[p];
  }
  a.block_vecs = block_elems / 8;
  const int gx = fp8_grid_x(a.block_vecs, nblocks * parts);
  amax_kernel_for(fp8_common_dt(src, parts))<<<dim3(gx, nblocks, parts), kBlock, 0, s>>>(a);
  FUSP_LAUNCHED("amax_vec_kernel");
  return FUSP_OK;
}

namespace {
// quantize_fused_kernel when the tensors fit the grid's registers (per-tensor scale, one common
// source dtype, 16-byte pieces, not under graph capture); *done = false otherwise.
fusp_status try_quantize_fused(const Fp8Src* src, int parts, int64_t n, uint32_t* const* work,
                               float* const* scales, uint8_t* const* codes, uint32_t* nonfinite,
                               cudaStream_t s, bool* done) {
  *done = false;
  static const bool off = getenv("FUSP_FP8_FUSED") != nullptr && atoi(getenv("FUSP_FP8_FUSED")) == 0;
  const int dt = fp8_common_dt(src, parts);
  if (off || dt < 0 || n <= 0) return FUSP_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FUSP_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return FUSP_OK;
  const int64_t w = static_cast<int64_t>(dtype_size(dt));
  FusedQArgs a{};
  a.parts = parts;
  a.cta0[0] = 0;
  for (int p = 0; p < parts; ++p) {
    if ((n * w) % 16 != 0 || !aligned16(src[p].x) || !aligned16(codes[p]) || scales[p] == nullptr) return FUSP_OK;
    if (dt == FUSP_E4M3 && src[p].d % 16 != 0) return FUSP_OK;
    a.src[p] = src[p];
    a.div[p] = make_fp8div(src[p]);
    a.amax[p] = work[p];
    a.scales[p] = scales[p];
    a.codes[p] = codes[p];
    a.units[p] = n * w / 16;
    a.cta0[p + 1] = a.cta0[p] + static_cast<int>((a.units[p] + int64_t(kBlock) * kFusedHold - 1) /
                                                  (int64_t(kBlock) * kFusedHold));
  }
  if (parts == 1) a.cta0[2] = a.cta0[1];
  a.barrier = work[0] + 1;  // the 2-pass finalize ticket word (zero on entry and exit)
  a.nonfinite = nonfinite;
  void (*k)(FusedQArgs) = dt == FUSP_BF16 ? quantize_fused_kernel<FUSP_BF16>
                        : dt == FUSP_F16 ? quantize_fused_kernel<FUSP_F16>
                        : dt == FUSP_F32 ? quantize_fused_kernel<FUSP_F32>
                                         : quantize_fused_kernel<FUSP_E4M3>;
  int dev = 0;
  FUSP_CUDA(cudaGetDevice(&dev));
  int occ = 0;  // resident CTAs per SM (per device and instance; racing threads agree)
  static std::atomic<int> per_sm[16][4];
  if (dev < 16 && per_sm[dev][dt].load() > 0) {
    occ = per_sm[dev][dt].load();
  } else {
    FUSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kBlock, 0));
    if (dev < 16) per_sm[dev][dt].store(occ);
  }
  // at most (occupancy - 1) CTAs per SM: a cooperative grid waits until ALL its CTAs fit, so
  // it leaves every SM room for a small kernel that may be resident meanwhile (an NCCL or
  // exchange kernel spinning on a peer whose progress could depend on this launch)
  const int grid = a.cta0[parts];
  if (occ < 2 || grid > (occ - 1) * sm_count() || grid >= 0xFFFF) return FUSP_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // every CTA resident before any runs: the barrier
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FUSP_CUDA(cudaLaunchKernelEx(&cfg, k, a));
  FUSP_LAUNCHED("quantize_fused_kernel");
  *done = true;
  return FUSP_OK;
}
}  // namespace

fusp_status launch_quantize_fp8_multi(const Fp8Src* src, int parts, int64_t n, int64_t block_elems,
                                      uint32_t* const* work, float* const* scales,
                                      uint8_t* const* codes, uint32_t* nonfinite, cudaStream_t s,
                                      bool one_launch) {
  const int nblocks = static_cast<int>((n + block_elems - 1) / block_elems);
  bool fast = parts >= 1 && parts <= 2 && nblocks <= 65535 && n < (int64_t(1) << 31);
  for (int p = 0; p < parts && fast; ++p) fast = fp8_vec_ok(src[p], n, block_elems, codes[p]);
  if (!fast) {
    for (int p = 0; p < parts; ++p)
      FUSP_CHECK(launch_quantize_fp8(src[p], n, block_elems, work[p], scales[p], codes[p], nonfinite, s));
    return FUSP_OK;
  }
  if (n <= 0) return FUSP_OK;
  for (int p = 0; p < parts; ++p)
    if (scales[p] == nullptr) return set_error(FUSP_ERR_INVALID_ARGUMENT, "quantize: no scale output");
  if (nonfinite) FUSP_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(uint32_t), s));
  if (nblocks == 1 && one_launch) {  // per tensor and small enough: one launch (quantize_fused_kernel)
    bool done = false;
    FUSP_CHECK(try_quantize_fused(src, parts, n, work, scales, codes, nonfinite, s, &done));
    if (done) return FUSP_OK;
  }
  // pass 1 finalizes the scales in its last CTA and leaves `work` zero again; pass 2 is its
  // programmatic dependent (launch latency hidden under pass 1, second read of x from L2)
  const int gx = fp8_grid_x(block_elems / 8, nblocks * parts);
  FUSP_CHECK(launch_amax_scales(src, parts, block_elems, nblocks, work, scales, nonfinite, s));
  QuantArgs q{};
  for (int p = 0; p < parts; ++p) {
    q.src[p] = src[p];
    q.div[p] = make_fp8div(src[p]);
    q.qscale[p] = scales[p];
    q.codes[p] = codes[p];
  }
  q.block_vecs = block_elems / 8;
  FUSP_CUDA(launch_pdl(quantize_kernel_for(fp8_common_dt(src, parts)), dim3(gx, nblocks, parts), s, q));
  FUSP_LAUNCHED("quantize_vec_kernel");
  return FUSP_OK;
}

fusp_status launch_amax_scales(const Fp8Src* src, int parts, int64_t block_elems, int nblocks,
                               uint32_t* const* work, float* const* scales, uint32_t* nonfinite,
                               cudaStream_t s) {
  if (parts < 1 || parts > 2 || nblocks <= 0 || nblocks > 65535 || block_elems % 8 != 0)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "amax: unsupported block layout");
  AmaxArgs a{};
  for (int p = 0; p < parts; ++p) {
    a.src[p] = src[p];
    a.div[p] = make_fp8div(src[p]);
    a.amax[p] = work[p];
    a.scales[p] = scales[p];
  }
  a.block_vecs = block_elems / 8;
  a.nonfinite = nonfinite;
  a.ticket = work[0] + nblocks;
  a.nblocks = nblocks;
  a.parts = parts;
  amax_kernel_for(fp8_common_dt(src, parts))<<<dim3(fp8_grid_x(a.block_vecs, nblocks * parts), nblocks, parts),
                                              kBlock, 0, s>>>(a);
  FUSP_LAUNCHED("amax_vec_kernel");
  return FUSP_OK;
}

fusp_status launch_quantize_fp8(const Fp8Src& src, int64_t n, int64_t block_elems, uint32_t* work,
                                float* scales, uint8_t* codes, uint32_t* nonfinite,
                                cudaStream_t s) {
  const int nblocks = static_cast<int>((n + block_elems - 1) / block_elems);
  if (fp8_vec_ok(src, n, block_elems, codes) && nblocks <= 65535)
    return launch_quantize_fp8_multi(&src, 1, n, block_elems, &work, &scales, &codes, nonfinite, s);
  FUSP_CHECK(launch_amax_blocks(src, block_elems, nblocks, work, nonfinite, s));
  FUSP_CUDA(cudaMemcpyAsync(scales, work, sizeof(float) * nblocks, cudaMemcpyDeviceToDevice, s));
  FUSP_CUDA(cudaMemsetAsync(work, 0, sizeof(uint32_t) * nblocks, s));  // zero again (contract)
  return launch_quantize_blocks(src, n, block_elems, scales, codes, s);
}

fusp_status launch_dequantize_blocks(const uint8_t* c, const float* scales, int64_t block_elems,
                                     int64_t n, void* y, int ydt, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  if (n % 8 == 0 && block_elems % 8 == 0 && aligned16(c) && aligned16(y) && ydt != FUSP_E4M3 &&
      n < (int64_t(1) << 31)) {
    dequantize_vec_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(c, scales, make_fdiv(uint32_t(block_elems / 8)),
                                                              n / 8, y, ydt);
    FUSP_LAUNCHED("dequantize_vec_kernel");
    return FUSP_OK;
  }
  dequantize_blocks_kernel<<<grid_for(n), kBlock, 0, s>>>(c, scales, block_elems, n, y, ydt);
  FUSP_LAUNCHED("dequantize_blocks_kernel");
  return FUSP_OK;
}

fusp_status launch_scatter_slot_scales(const float* scales, float* base, int64_t slot_stride_f,
                                       int b, int h, int u, int per_block, cudaStream_t s) {
  scatter_slot_scales_kernel<<<1, 256, 0, s>>>(scales, base, slot_stride_f, b, h, u, per_block);
  FUSP_LAUNCHED("scatter_slot_scales_kernel");
  return FUSP_OK;
}

fusp_status launch_finite(const void* x, int dt, int64_t n, uint32_t* flag, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
  finite_kernel<<<grid_for(n, 4), kBlock, 0, s>>>(x, dt, n, flag);
  FUSP_LAUNCHED("finite_kernel");
  return FUSP_OK;
}

}  // namespace fusp

namespace fusp {
namespace {
// quantize(dequantize(chunk)) of a chunk quantize produced as a whole: amax = decode(0x7E) * s
// (the block's largest code is +-448 by construction; an all-zero block has s = 1 and gives
// the same), scale' = amax / 448 (fp8.cpp:119), IEEE roundings as the reference.
__global__ void fp8_forward_scales_kernel(float* a, float* b, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    float* p = blockIdx.x == 0 ? a : b;
    const float amax = __fmul_rn(448.0f, p[i]);
    p[i] = amax > 0.f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  }
}
}  // namespace

fusp_status launch_fp8_forward_scales(float* const* scales, int parts, int n, cudaStream_t s) {
  if (n <= 0 || parts <= 0) return FUSP_OK;
  if (parts > 2) return set_error(FUSP_ERR_INVALID_ARGUMENT, "fp8 forward scales: at most 2 parts");
  fp8_forward_scales_kernel<<<parts, 256, 0, s>>>(scales[0], parts > 1 ? scales[1] : scales[0], n);
  FUSP_LAUNCHED("fp8_forward_scales_kernel");
  return FUSP_OK;
}

// Every kernel of this file, for preload_kernels() (lazy module loading, see runtime.cpp).
void append_kernels_kernels(std::vector<const void*>& v) {
  v.push_back(reinterpret_cast<const void*>(convert_kernel));
  v.push_back(reinterpret_cast<const void*>(bf16_to_f16_kernel));
  v.push_back(reinterpret_cast<const void*>(encode_kernel));
  v.push_back(reinterpret_cast<const void*>(decode_kernel));
  v.push_back(reinterpret_cast<const void*>(amax_kernel));
  v.push_back(reinterpret_cast<const void*>(quantize_kernel));
  v.push_back(reinterpret_cast<const void*>(dequantize_kernel));
  v.push_back(reinterpret_cast<const void*>(merge_kernel));
  v.push_back(reinterpret_cast<const void*>(fill_kernel));
  v.push_back(reinterpret_cast<const void*>(pack_kernel));
  v.push_back(reinterpret_cast<const void*>(unpack_kernel));
  v.push_back(reinterpret_cast<const void*>(unpack_heads_kernel));
  v.push_back(reinterpret_cast<const void*>(amax_blocks_kernel));
  v.push_back(reinterpret_cast<const void*>(finalize_scales_kernel));
  v.push_back(reinterpret_cast<const void*>(quantize_blocks_kernel));
  v.push_back(reinterpret_cast<const void*>(dequantize_blocks_kernel));
  v.push_back(reinterpret_cast<const void*>(scatter_slot_scales_kernel));
  v.push_back(reinterpret_cast<const void*>(finite_kernel));
  v.push_back(reinterpret_cast<const void*>(pack_slab_kernel));
  v.push_back(reinterpret_cast<const void*>(unpack_slab_kernel));
  v.push_back(reinterpret_cast<const void*>(stage_kernel));
  v.push_back(reinterpret_cast<const void*>(stage_decide_kernel));
  v.push_back(reinterpret_cast<const void*>(stage_scalar_kernel));
  for (const void* k : {reinterpret_cast<const void*>(amax_vec_kernel<-1>), reinterpret_cast<const void*>(amax_vec_kernel<FUSP_BF16>),
                        reinterpret_cast<const void*>(amax_vec_kernel<FUSP_F16>), reinterpret_cast<const void*>(amax_vec_kernel<FUSP_F32>),
                        reinterpret_cast<const void*>(amax_vec_kernel<FUSP_E4M3>)})
    v.push_back(k);
  for (const void* k : {reinterpret_cast<const void*>(quantize_vec_kernel<-1>), reinterpret_cast<const void*>(quantize_vec_kernel<FUSP_BF16>),
                        reinterpret_cast<const void*>(quantize_vec_kernel<FUSP_F16>), reinterpret_cast<const void*>(quantize_vec_kernel<FUSP_F32>),
                        reinterpret_cast<const void*>(quantize_vec_kernel<FUSP_E4M3>)})
    v.push_back(k);
  v.push_back(reinterpret_cast<const void*>(dequantize_vec_kernel));
  v.push_back(reinterpret_cast<const void*>(fp8_forward_scales_kernel));
  v.push_back(reinterpret_cast<const void*>(pack_fp8_fused_kernel<FUSP_BF16>));
  v.push_back(reinterpret_cast<const void*>(pack_fp8_fused_kernel<FUSP_F16>));
  for (const void* k : {reinterpret_cast<const void*>(quantize_fused_kernel<FUSP_BF16>), reinterpret_cast<const void*>(quantize_fused_kernel<FUSP_F16>),
                        reinterpret_cast<const void*>(quantize_fused_kernel<FUSP_F32>), reinterpret_cast<const void*>(quantize_fused_kernel<FUSP_E4M3>)})
    v.push_back(k);
}

}  // namespace fusp
