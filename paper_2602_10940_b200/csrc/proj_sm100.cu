// The consumer side of the layer (second half): the joint-attention
// block's output projection y = O · W_o, read straight from the output all-to-all's result.
//
// O is the layer output in its native layout [B][H][S][D = 128] (heads-major, the order the
// Ulysses output reshard delivers it), so the GEMM's K = H·D axis is walked as (head, d): a
// 4-D TMA map {d, s, h, b} with 64 x 128 boxes loads the A tile [128 tokens][64 k] of one
// head directly -- no transpose pass.  W_o is [H·D][N] row-major (N contiguous: MN-major B).
// y is token-major [B][S][N].
//
// tcgen05 GEMM, persistent (one CTA per SM): tiles of 128 tokens x 256 outputs, K in blocks
// of 64 through a 4-stage TMA ring (A 16 KB + B 32 KB per stage, 128B swizzle), one thread
// issues 4 MMAs (M=128, N=256, K=16) per block into a TMEM accumulator; two accumulators
// (2 x 256 columns) let the epilogue warpgroup drain tile i while tile i+1 accumulates.
//   warp 0   TMA producer        warp 1   TMEM allocator + MMA issuer
//   warps 4-11 epilogue, two warpgroups splitting the tile's columns (TMEM lane = token row)
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdlib>

#include <vector>

#include "fastusp_internal.h"
#include "sm100_ptx.cuh"

namespace fusp {
namespace {

using namespace ptx;

constexpr int kPM = 128;   // tokens per tile
constexpr int kPNMax = 256;  // outputs per tile (256, or 128 when that fills the SMs better)
constexpr int kPK = 64;    // K per stage (one 128-byte swizzle row of bf16)
constexpr int kPStages = 4;
constexpr int kPThreads = 384;  // producer / MMA warpgroup + 2 epilogue warpgroups
constexpr uint32_t kABytes = kPM * kPK * 2;  // 16 KB
constexpr uint32_t kBBytes = kPK * kPNMax * 2;  // up to 32 KB: chunks of [64 k][64 n]
constexpr uint32_t kBChunk = kPK * 64 * 2;   // 8 KB

struct __align__(1024) ProjSmem {
  uint8_t a[kPStages][kABytes];
  uint8_t b[kPStages][kBBytes];
  uint64_t full[kPStages], empty[kPStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  uint32_t ticket;  // stream-K: the tile's arrival count seen by this CTA
};

struct ProjParams {
  int m_tiles_per_b;  // ceil(S / 128)
  int n_tiles;        // ceil(N / 256)
  int tiles;          // B * m_tiles_per_b * n_tiles
  int m_tiles;        // B * m_tiles_per_b
  int m_fast;         // tile order: 1 = m-tiles fastest (consecutive CTAs share a B tile)
  int k_blocks;       // out-projection: H * 2; QKV projection: C / 64
  int s, n;           // tokens per batch row, outputs
  uint32_t idesc;
  void* y;
  int y_dtype;
  // QKV projection epilogue (kQkv): columns [part][head][d] of N = 3 * H * 128; Q and K rows
  // get RMSNorm (w != null) and interleaved RoPE (cos != null) and every part lands as
  // [B][H][S][128] at qkv[part]
  int heads;
  void* qkv[3];
  int part_dt[3];       // Q, K, V output dtypes (bf16 / f16)
  int u;                // Ulysses slots: head h -> slot h / (heads / u), position h % (heads / u)
  int64_t slot_stride;  // elements between slots (u = 1: unused)
  int peer;             // slot t at slot_eoff[t] elements from slot 0 (members' peer windows)
  int64_t slot_eoff[kMaxPeerChunks];
  // Stream-K over (tile, k-block) units (split = 1): CTA c owns units [c U / G, (c+1) U / G),
  // U = tiles * k_blocks, so a tile's K range may be cut between consecutive CTAs.  Every
  // segment of a cut tile but the finisher publishes its f32 partial (128 x kPN, [col/4][row]
  // float4s) to slot (cta, first/last segment) and counts on the tile's word; the segment that
  // brings the count to the tile's segment count sums all partials in K order (bit-identical
  // whoever finishes) back into its accumulator and runs the normal epilogue.
  int split;
  int64_t units;
  uint32_t* counters;   // one per tile, zero on entry, zeroed again by each tile's finisher
  float* slots;         // 2 * gridDim.x slots of 128 * kPN floats
  const float* norm_w[2];
  float eps;
  const float* cosv;
  const float* sinv;
  int64_t pos0;
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Tile raster: walk the m-tiles fastest when B (the weights) is the larger operand, so the
// CTAs in flight share a few B column blocks and stream A; otherwise n fastest.  Keeps the
// working set in L2 (QKV projection, W 56.6 MB vs x 28 MB at FLUX: 207 -> 179 us).
// FUSP_PROJ_MFAST=0/1 overrides.
bool proj_m_fast(int64_t a_bytes, int64_t b_bytes) {
  static const int v = [] {
    const char* e = getenv("FUSP_PROJ_MFAST");
    return e == nullptr ? -1 : atoi(e);
  }();
  return v < 0 ? b_bytes > a_bytes : v != 0;
}

// A CTA's work as segments (tile, k-blocks [kb0, kb1)): whole tiles strided by the grid, or
// its contiguous stream-K unit range.
struct PSeg {
  int tile, kb0, kb1;
};
__device__ __forceinline__ int64_t sk_begin(const ProjParams& p, int c) {
  return int64_t(c) * p.units / gridDim.x;
}
__device__ __forceinline__ int sk_cta_of(const ProjParams& p, int64_t u) {
  int c = static_cast<int>(u * gridDim.x / p.units);
  while (c + 1 < static_cast<int>(gridDim.x) && sk_begin(p, c + 1) <= u) ++c;
  while (c > 0 && sk_begin(p, c) > u) --c;
  return c;
}
struct PIter {
  int64_t u, end;
  __device__ explicit PIter(const ProjParams& p) {
    if (p.split) {
      u = sk_begin(p, blockIdx.x);
      end = sk_begin(p, blockIdx.x + 1);
    } else {
      u = blockIdx.x;
      end = p.tiles;
    }
  }
  __device__ bool next(const ProjParams& p, PSeg& g) {
    if (u >= end) return false;
    if (!p.split) {
      g.tile = static_cast<int>(u);
      g.kb0 = 0;
      g.kb1 = p.k_blocks;
      u += gridDim.x;
      return true;
    }
    g.tile = static_cast<int>(u / p.k_blocks);
    const int64_t t0 = int64_t(g.tile) * p.k_blocks;
    g.kb0 = static_cast<int>(u - t0);
    const int64_t lim = end < t0 + p.k_blocks ? end : t0 + p.k_blocks;
    g.kb1 = static_cast<int>(lim - t0);
    u = lim;
    return true;
  }
};
__device__ __forceinline__ uint32_t proj_atom_add_acq_rel(uint32_t* a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t proj_ld_acquire(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void epi_bar() {  // the 8 epilogue warps
  __syncwarp();
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

// kQkv = false: output projection, A = attention output [B][H][S][128] through a 4-D map.
// kQkv = true:  QKV projection, A = x [B*S][C] token-major through a 2-D map, epilogue does
//               the MMDiT QK RMSNorm + RoPE and writes Q, K, V head-major.
template <int kPN, bool kQkv>
__global__ void __launch_bounds__(kPThreads, 1)
    out_proj_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const ProjParams p) {
  extern __shared__ uint8_t smem_raw[];
  ProjSmem& sm = *reinterpret_cast<ProjSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.acc_full[b], 1);
      mbar_init(&sm.acc_empty[b], 256);
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
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      prefetch_tmap(&tm_a);
      prefetch_tmap(&tm_b);
      uint32_t it = 0;
      PIter pi(p);
      PSeg g;
      while (pi.next(p, g)) {
        const int tile = g.tile;
        const int nt = p.m_fast ? tile / p.m_tiles : tile % p.n_tiles;
        const int mt = p.m_fast ? tile % p.m_tiles : tile / p.n_tiles;
        const int bb = mt / p.m_tiles_per_b;
        const int s0 = (mt - bb * p.m_tiles_per_b) * kPM;
        for (int kb = g.kb0; kb < g.kb1; ++kb, ++it) {
          const int st = it % kPStages;
          mbar_wait(&sm.empty[st], ((it / kPStages) & 1) ^ 1);
          mbar_expect_tx(&sm.full[st], kABytes + kPK * kPN * 2);
          if (kQkv)  // A: x rows of batch bb, tokens s0.., channels kb*64..
            tma_load_2d(sm.a[st], &tm_a, &sm.full[st], kb * kPK, bb * p.s + s0);
          else       // A: head kb/2, d-half kb%2, 128 tokens from s0
            tma_load_4d(sm.a[st], &tm_a, &sm.full[st], (kb & 1) * 64, s0, kb >> 1, bb);
          // B: rows k = kb*64 .. +64, four 64-wide n-chunks
          for (int c = 0; c < kPN / 64; ++c)
            tma_load_2d(sm.b[st] + c * kBChunk, &tm_b, &sm.full[st], nt * kPN + c * 64, kb * kPK);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp walks, one lane issues) ----------------
    uint32_t it = 0, lt = 0;
    PIter pi(p);
    PSeg g;
    for (; pi.next(p, g); ++lt) {
      const int ab = lt & 1;
      mbar_wait(&sm.acc_empty[ab], ((lt >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      tc_fence_after();
      const uint32_t d_tmem = tmem + ab * kPN;
      for (int kb = g.kb0; kb < g.kb1; ++kb, ++it) {
        const int st = it % kPStages;
        mbar_wait(&sm.full[st], (it / kPStages) & 1);
        tc_fence_after();
        const uint64_t adesc = umma_desc_sw128(smem_u32(sm.a[st]), 16, 1024);
        // B MN-major SW128: LBO = stride between 64-wide n-chunks (8 KB), SBO = 8 k-rows (1 KB)
        const uint64_t bdesc = umma_desc_sw128(smem_u32(sm.b[st]), kBChunk, 1024);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kPK / 16; ++k)
            mma_ss(d_tmem, adesc + uint64_t(k * 32 / 16), bdesc + uint64_t(k * 16 * 128 / 16), p.idesc,
                   (kb > g.kb0 || k > 0) ? 1u : 0u);
          mma_commit(&sm.empty[st]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&sm.acc_full[ab]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int quad = warp & 3;
    const int eg = (warp - 4) >> 2;  // epilogue warpgroup: column half (QKV: head) of the tile
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    uint32_t lt = 0;
    PIter pi(p);
    PSeg g;
    for (; pi.next(p, g); ++lt) {
      const int tile = g.tile;
      const int ab = lt & 1;
      const int nt = p.m_fast ? tile / p.m_tiles : tile % p.n_tiles;
      const int mt = p.m_fast ? tile % p.m_tiles : tile / p.n_tiles;
      const int bb = mt / p.m_tiles_per_b;
      const int s = (mt - bb * p.m_tiles_per_b) * kPM + r;
      mbar_wait(&sm.acc_full[ab], (lt >> 1) & 1);
      tc_fence_after();
      if (p.split && (g.kb0 != 0 || g.kb1 != p.k_blocks)) {
        // a stream-K segment of a cut tile: publish, or finish (sum in K order into TMEM)
        const int64_t u0 = int64_t(tile) * p.k_blocks;
        const int cf = sk_cta_of(p, u0);
        const int nseg = sk_cta_of(p, u0 + p.k_blocks - 1) - cf + 1;
        const int kself = static_cast<int>(blockIdx.x) - cf;
        uint32_t* cnt = p.counters + tile;
        const uint32_t acc_col = tmem + lane_off + ab * kPN;
        constexpr int kHalf = kPN / 2;  // columns of this warpgroup: [eg * kHalf, +kHalf)
        auto slot_of = [&](int c) {     // the slot CTA c published this tile's segment to
          const int which = sk_begin(p, c) >= u0 ? 0 : 1;
          return reinterpret_cast<float4*>(p.slots + (int64_t(c) * 2 + which) * (int64_t(kPM) * kPN));
        };
        bool last = false;
        if (kself == 0) {  // processed last by its CTA: usually every other segment has counted
          if (threadIdx.x == 128) sm.ticket = proj_ld_acquire(cnt);
          epi_bar();
          last = *reinterpret_cast<volatile uint32_t*>(&sm.ticket) + 1 == static_cast<uint32_t>(nseg);
          epi_bar();
        }
        if (!last) {
          float4* q4 = slot_of(blockIdx.x);
#pragma unroll 1
          for (int c = 0; c < kHalf / 32; ++c) {
            const int col = eg * kHalf + c * 32;
            uint32_t v[32];
            tmem_ld32(acc_col + col, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i)
              __stcg(q4 + (col / 4 + i) * kPM + r, make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                              __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
          }
          epi_bar();  // every slot store happens-before thread 128's release
          if (threadIdx.x == 128) sm.ticket = proj_atom_add_acq_rel(cnt, 1u);
          epi_bar();
          last = *reinterpret_cast<volatile uint32_t*>(&sm.ticket) + 1 == static_cast<uint32_t>(nseg);
          if (!last) {
            tc_fence_before();
            mbar_arrive(&sm.acc_empty[ab]);
            continue;
          }
        }
        if (threadIdx.x == 128) *cnt = 0u;  // every segment has counted: zero for the next launch
#pragma unroll 1
        for (int c = 0; c < kHalf / 32; ++c) {
          const int col = eg * kHalf + c * 32;
          float v[32];
#pragma unroll 1
          for (int k = 0; k < nseg; ++k) {
            float x[32];
            if (k == kself) {
              uint32_t o[32];
              tmem_ld32(acc_col + col, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(o[i]);
            } else {
              const float4* q4 = slot_of(cf + k);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 y = __ldcg(q4 + (col / 4 + i) * kPM + r);
                x[4 * i] = y.x; x[4 * i + 1] = y.y; x[4 * i + 2] = y.z; x[4 * i + 3] = y.w;
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = k == 0 ? x[i] : v[i] + x[i];
          }
          uint32_t o[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(v[i]);
          tmem_st32(acc_col + col, o);
        }
        tmem_wait_st();
        tc_fence_before();
        epi_bar();  // both warpgroups' columns merged before either reads the other's head
        tc_fence_after();
      }
      const bool in_range = s < p.s;
      if constexpr (kQkv) {
        // two heads per 256-column tile (one per 128-column tile): RMSNorm needs the whole
        // head row, so each head is read from TMEM twice (sum of squares, then scale + rotate)
        const int hd = p.heads * 128;
#pragma unroll 1
        for (int hh = eg; hh < kPN / 128; hh += 2) {
          const int n0 = nt * kPN + hh * 128;
          const int part = n0 / hd, head = (n0 - part * hd) / 128;
          const uint32_t tcol = tmem + lane_off + ab * kPN + hh * 128;
          const float* w = part < 2 ? p.norm_w[part] : nullptr;
          const bool rope = part < 2 && p.cosv != nullptr;
          float rinv = 1.f;
          if (w != nullptr) {
            float ss = 0.f;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t v[32];
              tmem_ld32(tcol + c * 32, v);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) ss = fmaf(__uint_as_float(v[i]), __uint_as_float(v[i]), ss);
            }
            rinv = rsqrtf(ss * (1.0f / 128) + p.eps);
          }
          const int64_t pos = p.pos0 + s;
          const int hp = p.heads / p.u, slot = head / hp, hl = head - slot * hp;
          uint16_t* dst = static_cast<uint16_t*>(p.qkv[part]) +
                          (p.peer ? p.slot_eoff[slot] : slot * p.slot_stride) +
                          ((static_cast<int64_t>(bb) * hp + hl) * p.s + s) * 128;
          const bool o_f16 = p.part_dt[part] == FUSP_F16;
          const int e4 = lane & 3;  // stores: the 4 lanes of a group write one row's 64-byte chunk
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld32(tcol + c * 32, v);
            tmem_wait_ld();
            float x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(v[i]);
            if (w != nullptr && in_range) {
              const float4* w4 = reinterpret_cast<const float4*>(w + c * 32);
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4) {
                const float4 wv = __ldg(w4 + q4);
                x[4 * q4] *= rinv * wv.x;
                x[4 * q4 + 1] *= rinv * wv.y;
                x[4 * q4 + 2] *= rinv * wv.z;
                x[4 * q4 + 3] *= rinv * wv.w;
              }
            }
            if (rope && in_range) {  // this row's 16 (cos, sin) pairs of the chunk as float4 vectors
              const float4* c4 = reinterpret_cast<const float4*>(p.cosv + pos * 64 + c * 16);
              const float4* s4 = reinterpret_cast<const float4*>(p.sinv + pos * 64 + c * 16);
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                const float4 cv = __ldg(c4 + q4), sv = __ldg(s4 + q4);
                const float cc[4] = {cv.x, cv.y, cv.z, cv.w}, ss[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int i = q4 * 4 + e;
                  const float x0 = x[2 * i], x1 = x[2 * i + 1];
                  x[2 * i] = x0 * cc[e] - x1 * ss[e];
                  x[2 * i + 1] = x0 * ss[e] + x1 * cc[e];
                }
              }
            }
            uint32_t o16[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              o16[i] = o_f16 ? pack_f16x2(x[2 * i], x[2 * i + 1]) : pack_bf16x2(x[2 * i], x[2 * i + 1]);
            xpose4<4>(o16, lane);  // lane 4G+e now holds 16-byte piece e of rows 4G..4G+3
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (s - e4 + i < p.s)
                *reinterpret_cast<uint4*>(dst + (i - e4) * 128 + c * 32 + e4 * 8) =
                    make_uint4(o16[4 * i], o16[4 * i + 1], o16[4 * i + 2], o16[4 * i + 3]);
          }
        }
      } else {
      const int64_t ybase = (static_cast<int64_t>(bb) * p.s + s) * p.n + nt * kPN;
#pragma unroll 1
      for (int c = eg * (kPN / 64); c < (eg + 1) * (kPN / 64); ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + ab * kPN + c * 32, v);
        tmem_wait_ld();
        const int n0 = nt * kPN + c * 32;
        if (n0 >= p.n) continue;  // (uniform) N % 64 == 0: whole chunks
        // stores through 4-lane-group transposes: 4 lanes cover one row's chunk, 8 rows per
        // instruction (rows s - e4 + i are p.n elements apart)
        const int e4 = lane & 3;
        if (p.y_dtype == FUSP_F32) {
          xpose4<8>(v, lane);
          float* y = static_cast<float*>(p.y) + ybase + c * 32 + e4 * 8;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (s - e4 + i < p.s) {
              uint4* dst = reinterpret_cast<uint4*>(y + static_cast<int64_t>(i - e4) * p.n);
              dst[0] = make_uint4(v[8 * i], v[8 * i + 1], v[8 * i + 2], v[8 * i + 3]);
              dst[1] = make_uint4(v[8 * i + 4], v[8 * i + 5], v[8 * i + 6], v[8 * i + 7]);
            }
        } else {
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            w[i] = p.y_dtype == FUSP_F16 ? pack_f16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]))
                                         : pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
          xpose4<4>(w, lane);
          uint16_t* y = static_cast<uint16_t*>(p.y) + ybase + c * 32 + e4 * 8;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (s - e4 + i < p.s)
              *reinterpret_cast<uint4*>(y + static_cast<int64_t>(i - e4) * p.n) =
                  make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
      }
      }
      tc_fence_before();
      mbar_arrive(&sm.acc_empty[ab]);
    }
    // peer-memory slots: this thread's stores into other GPUs' windows are visible system-wide
    // before the stream's exchange kernel signals the members
    if constexpr (kQkv)
      if (p.peer) __threadfence_system();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

namespace {
// Tile width, stream-K split and grid of one projection launch.  128 x 256 tiles unless
// 128 x 128 fills the SMs' waves clearly better.  Stream-K (128 x 256 tiles, all SMs) when
// neither whole-tile width fills the waves to 90 % and every CTA still gets at least one
// tile's worth of units (two with a heavy epilogue: a cut tile's merge and epilogue run
// after its last segment, unoverlapped).  Measured (profiles/r02_proj_tokens.jsonl): the QKV
// projection at 1152 tokens 76.9 -> 56.0 us (plain epilogue) / 75.9 -> 66.4 us (RMSNorm +
// RoPE), at 576 tokens 41.1 -> 37.0 us (plain); the output projection (12 column tiles: few
// tiles, short segments) and the RMSNorm epilogue at 576 tokens lose, so they keep whole
// tiles.  FUSP_PROJ_SPLIT=0/1 overrides the choice.
template <bool kQkv>
fusp_status launch_proj_kernel(const CUtensorMap& ta, const CUtensorMap& tb, const ProjParams& p0,
                               int b, int n, bool allow256, uint32_t f, cudaStream_t stream,
                               const char* name, bool allow_split, bool heavy_epilogue) {
  const int sms = sm_count();
  auto tiles_for = [&](int pn) { return b * p0.m_tiles_per_b * ((n + pn - 1) / pn); };
  auto fill = [&](int pn) {
    const int t = tiles_for(pn);
    const int waves = (t + sms - 1) / sms;
    return static_cast<double>(t) / (static_cast<double>(waves) * sms);
  };
  static const int mode = [] {
    const char* e = getenv("FUSP_PROJ_SPLIT");
    return e == nullptr ? -1 : atoi(e);
  }();
  const int pn_split = allow256 ? 256 : 128;
  const int pn_whole = (!allow256 || fill(128) > 1.15 * fill(256)) ? 128 : 256;
  const double best_whole = allow256 && fill(256) > fill(128) ? fill(256) : fill(128);
  const bool want_split =
      mode == 1 || (mode < 0 && allow_split && p0.k_blocks >= 8 && best_whole < 0.9 &&
                    tiles_for(pn_split) >= (heavy_epilogue ? 2 : 1) * sms);
  auto launch = [&](uint32_t* cnt, float* slots) -> fusp_status {
    ProjParams p = p0;
    int pn = pn_whole;
    if (cnt != nullptr) {
      pn = pn_split;
      p.split = 1;
      p.counters = cnt;
      p.slots = slots;
    }
    p.n_tiles = (n + pn - 1) / pn;
    p.tiles = b * p.m_tiles_per_b * p.n_tiles;
    p.m_tiles = b * p.m_tiles_per_b;
    p.idesc = idesc_f16(f, f, 0, 1, kPM, pn);
    p.units = int64_t(p.tiles) * p.k_blocks;
    const int64_t work = p.split ? p.units : p.tiles;
    const int grid = static_cast<int>(work < sms ? work : sms);
    const int smem = static_cast<int>(sizeof(ProjSmem)) + 1024;
    if (pn == 256) out_proj_kernel<256, kQkv><<<grid, kPThreads, smem, stream>>>(ta, tb, p);
    else out_proj_kernel<128, kQkv><<<grid, kPThreads, smem, stream>>>(ta, tb, p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, name);
    return FUSP_OK;
  };
  if (want_split)
    return with_proj_workspace(stream, static_cast<size_t>(tiles_for(pn_split)),
                               size_t(2) * sms * kPM * pn_split * sizeof(float), launch);
  return launch(nullptr, nullptr);
}
}  // namespace

// y[B][S][N] = O[B][H][S][128] (as [B*S][H*128]) x W[H*128][N].  O and W: both bf16 or both
// f16; y: f32 / f16 / bf16.  N a multiple of 64 (TMA row pitch), pointers 16-byte aligned.
fusp_status launch_out_proj(const void* o, int o_dtype, int b, int h, int s, const void* w,
                            int n, void* y, int y_dtype, cudaStream_t stream) {
  if (b <= 0 || h <= 0 || s <= 0 || n <= 0) return FUSP_OK;
  if (o_dtype != FUSP_BF16 && o_dtype != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "out projection: O must be bf16 or f16");
  if (n % 64 != 0) return set_error(FUSP_ERR_SHAPE, "out projection: N must be a multiple of 64");
  if ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(y)) % 16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "out projection: pointers must be 16-byte aligned");
  const CUtensorMapDataType dt =
      o_dtype == FUSP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap ta, tb;
  {
    const cuuint64_t dims[4] = {128, static_cast<cuuint64_t>(s), static_cast<cuuint64_t>(h),
                                static_cast<cuuint64_t>(b)};
    const cuuint64_t strides[3] = {128 * 2, static_cast<cuuint64_t>(s) * 128 * 2,
                                   static_cast<cuuint64_t>(h) * s * 128 * 2};
    const cuuint32_t box[4] = {64, kPM, 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    FUSP_CHECK(encode_tmap(&ta, dt, 4, o, dims, strides, box, es));
  }
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(h) * 128};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * 2};
    const cuuint32_t box[2] = {64, kPK};
    const cuuint32_t es[2] = {1, 1};
    FUSP_CHECK(encode_tmap(&tb, dt, 2, w, dims, strides, box, es));
  }
  ProjParams p{};
  p.m_tiles_per_b = (s + kPM - 1) / kPM;
  p.k_blocks = h * 2;
  p.s = s;
  p.n = n;
  const uint32_t f = o_dtype == FUSP_BF16 ? 1u : 0u;
  p.y = y;
  p.y_dtype = y_dtype;
  p.m_fast = proj_m_fast(int64_t(b) * s * h * 128 * 2, int64_t(h) * 128 * n * 2) ? 1 : 0;
  const int smem = static_cast<int>(sizeof(ProjSmem)) + 1024;
  FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(out_proj_kernel<256, false>), smem, "out_proj_kernel<256>"));
  FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(out_proj_kernel<128, false>), smem, "out_proj_kernel<128>"));
  return launch_proj_kernel<false>(ta, tb, p, b, n, true, f, stream, "out_proj_kernel launch",
                                   /*allow_split=*/false, false);
}

// Q, K, V [B][H][S][128] (dtype qkv_dtype: bf16 or f16) = x[B][S][C] . W[C][3*H*128], with
// the QK prologue (RMSNorm weights wq / wk, interleaved RoPE tables [rows][64] at positions
// pos0 + s; null = skipped) applied in the epilogue.  x and W both bf16 or both f16; C a
// multiple of 64.
fusp_status launch_qkv_proj(const void* x, int x_dtype, int b, int s, int c, const void* w, int heads,
                            void* q, void* k, void* v, int qkv_dtype, const float* wq, const float* wk,
                            float eps, const float* cosv, const float* sinv, int64_t pos0,
                            cudaStream_t stream) {
  const QkvDst dst{q, k, v, qkv_dtype, qkv_dtype, 1, 0};
  return launch_qkv_proj_to(x, x_dtype, b, s, c, w, heads, dst, wq, wk, eps, cosv, sinv, pos0, stream);
}

// Same, writing Q, K, V straight into the layer's Ulysses send slots (dst.u > 1): head h of
// part P lands at P's base + (h / hp) * slot_stride + ((b * hp + h % hp) * S + s) * 128.
fusp_status launch_qkv_proj_to(const void* x, int x_dtype, int b, int s, int c, const void* w, int heads,
                               const QkvDst& dst, const float* wq, const float* wk, float eps,
                               const float* cosv, const float* sinv, int64_t pos0, cudaStream_t stream) {
  void *q = dst.q, *k = dst.k, *v = dst.v;
  const int qkv_dtype = dst.qk_dtype;
  if (b <= 0 || s <= 0 || c <= 0 || heads <= 0) return FUSP_OK;
  if (x_dtype != FUSP_BF16 && x_dtype != FUSP_F16)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "qkv projection: x must be bf16 or f16");
  for (int dt : {dst.qk_dtype, dst.v_dtype})
    if (dt != FUSP_BF16 && dt != FUSP_F16)
      return set_error(FUSP_ERR_INVALID_ARGUMENT, "qkv projection: Q/K/V must be bf16 or f16");
  if (dst.u < 1 || heads % dst.u != 0 || (dst.u > 1 && dst.slot_stride % 8 != 0))
    return set_error(FUSP_ERR_SHAPE, "qkv projection: heads must split evenly over the slots");
  if (c % 64 != 0) return set_error(FUSP_ERR_SHAPE, "qkv projection: C must be a multiple of 64");
  for (const void* ptr : {x, w, static_cast<const void*>(q), static_cast<const void*>(k), static_cast<const void*>(v)})
    if (reinterpret_cast<uintptr_t>(ptr) % 16)
      return set_error(FUSP_ERR_INVALID_ARGUMENT, "qkv projection: pointers must be 16-byte aligned");
  const CUtensorMapDataType dt =
      x_dtype == FUSP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const int n = 3 * heads * 128;
  CUtensorMap ta, tb;
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(b) * s};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(c) * 2};
    const cuuint32_t box[2] = {kPK, kPM};
    const cuuint32_t es[2] = {1, 1};
    FUSP_CHECK(encode_tmap(&ta, dt, 2, x, dims, strides, box, es));
  }
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(c)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(n) * 2};
    const cuuint32_t box[2] = {64, kPK};
    const cuuint32_t es[2] = {1, 1};
    FUSP_CHECK(encode_tmap(&tb, dt, 2, w, dims, strides, box, es));
  }
  ProjParams p{};
  p.m_tiles_per_b = (s + kPM - 1) / kPM;
  p.k_blocks = c / kPK;
  p.s = s;
  p.n = n;
  p.y_dtype = qkv_dtype;
  p.heads = heads;
  p.qkv[0] = q;
  p.qkv[1] = k;
  p.qkv[2] = v;
  p.part_dt[0] = p.part_dt[1] = qkv_dtype;
  p.part_dt[2] = dst.v_dtype;
  p.u = dst.u;
  p.slot_stride = dst.slot_stride;
  if (dst.slot_boff != nullptr) {
    if (dst.u > kMaxPeerChunks) return set_error(FUSP_ERR_UNSUPPORTED, "qkv projection: too many peer slots");
    p.peer = 1;
    for (int t = 0; t < dst.u; ++t) {
      if (dst.slot_boff[t] % 16 != 0)
        return set_error(FUSP_ERR_INVALID_ARGUMENT, "qkv projection: misaligned peer slot");
      p.slot_eoff[t] = dst.slot_boff[t] / 2;
    }
  }
  p.norm_w[0] = wq;
  p.norm_w[1] = wk;
  p.eps = eps;
  p.cosv = cosv;
  p.sinv = sinv;
  p.pos0 = pos0;
  // 256-column tiles hold two whole heads, 128-column tiles one (heads never straddle tiles)
  p.m_fast = proj_m_fast(int64_t(b) * s * c * 2, int64_t(c) * n * 2) ? 1 : 0;
  const uint32_t f = x_dtype == FUSP_BF16 ? 1u : 0u;
  const int smem = static_cast<int>(sizeof(ProjSmem)) + 1024;
  FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(out_proj_kernel<256, true>), smem, "out_proj_kernel<256>"));
  FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(out_proj_kernel<128, true>), smem, "out_proj_kernel<128>"));
  return launch_proj_kernel<true>(ta, tb, p, b, n, n % 256 == 0, f, stream, "qkv_proj kernel launch",
                                  /*allow_split=*/true, wq != nullptr || wk != nullptr || cosv != nullptr);
}

// Every kernel of this file, for preload_kernels() (lazy module loading, see runtime.cpp).
void append_kernels_proj(std::vector<const void*>& v) {
  v.push_back(reinterpret_cast<const void*>(out_proj_kernel<128, false>));
  v.push_back(reinterpret_cast<const void*>(out_proj_kernel<128, true>));
  v.push_back(reinterpret_cast<const void*>(out_proj_kernel<256, false>));
  v.push_back(reinterpret_cast<const void*>(out_proj_kernel<256, true>));
}

}  // namespace fusp
