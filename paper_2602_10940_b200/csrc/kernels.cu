// HBM-bound kernels of the USP layer: dtype conversion, the E4M3 codec and the per-tensor
// quantizer (bit-exact with the reference), the LSE merge, and the Ulysses pack/unpack.
//
// Grids are sized as a multiple of the 148 SMs and loop grid-stride; all global accesses
// are 16-byte vectors where the layout allows.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>

#include "fastusp_internal.h"

namespace fusp {
namespace {

constexpr int kSMs = 148;
constexpr int kBlock = 256;

inline int grid_for(int64_t work_items, int per_sm = 8) {
  int64_t g = (work_items + kBlock - 1) / kBlock;
  if (g > int64_t(kSMs) * per_sm) g = int64_t(kSMs) * per_sm;
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

fusp_status launch_pack(const PackDesc& p, cudaStream_t s) {
  const int64_t n = int64_t(p.b) * p.h * p.sl * p.d;
  if (n <= 0) return FUSP_OK;
  if (p.d % 8 != 0) return set_error(FUSP_ERR_SHAPE, "pack: head dim must be a multiple of 8");
  pack_kernel<<<grid_for(n / 8), kBlock, 0, s>>>(p.src, p.src_dtype, p.dst, p.dst_dtype,
                                                  p.dst_slot_stride, p.b, p.h, p.sl, p.d, p.u,
                                                  p.scale, p.scale_bh_stride);
  FUSP_LAUNCHED("pack_kernel");
  return FUSP_OK;
}

fusp_status launch_unpack(const UnpackDesc& p, cudaStream_t s) {
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

fusp_status launch_amax_blocks(const Fp8Src& src, int64_t block_elems, int nblocks,
                               uint32_t* amax, uint32_t* nonfinite, cudaStream_t s) {
  FUSP_CUDA(cudaMemsetAsync(amax, 0, sizeof(uint32_t) * nblocks, s));
  if (nonfinite) FUSP_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(uint32_t), s));
  if (block_elems <= 0 || nblocks <= 0) return FUSP_OK;
  int gx = grid_for(block_elems, 4);
  const int cap = (kSMs * 8 + nblocks - 1) / nblocks;  // ~8 CTAs per SM in total
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

fusp_status launch_quantize_fp8(const Fp8Src& src, int64_t n, int64_t block_elems, uint32_t* work,
                                float* scales, uint8_t* codes, uint32_t* nonfinite,
                                cudaStream_t s) {
  const int nblocks = static_cast<int>((n + block_elems - 1) / block_elems);
  FUSP_CHECK(launch_amax_blocks(src, block_elems, nblocks, work, nonfinite, s));
  FUSP_CUDA(cudaMemcpyAsync(scales, work, sizeof(float) * nblocks, cudaMemcpyDeviceToDevice, s));
  return launch_quantize_blocks(src, n, block_elems, scales, codes, s);
}

fusp_status launch_dequantize_blocks(const uint8_t* c, const float* scales, int64_t block_elems,
                                     int64_t n, void* y, int ydt, cudaStream_t s) {
  if (n <= 0) return FUSP_OK;
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
