// tcgen05 / TMEM / TMA flash-attention forward for sm_100a with natural-log LSE
// output and an optional fused online-softmax merge into a running accumulator.
//
// Replaces the reference's scalar attention_with_lse -> attention_core
// (reference proj/src/tensor.cpp:143-202) and, when `acc_o` is given, folds in
// merge_lse (tensor.cpp:204-243) so a ring step's partial result is merged in
// the epilogue instead of in a separate pass.
//
// Non-causal, head dim D = 128.  Q/K are bf16, V is f16 (P.V runs in f16:
// bf16 P cannot meet rel-L2 <= 1e-3 against the fp32 oracle).
//
// Persistent kernel, one CTA per SM.  The work is (q-block of 256 rows) x (KV tile of 128
// keys) units, q-block-major over heads.  Two schedules:
//   whole  -- CTA c takes q-blocks c, c+G, c+2G, ... (used when the q-blocks fill the SMs
//             in near-full waves);
//   split  -- stream-K: CTA c takes the contiguous unit range [c*T/G, (c+1)*T/G), so a
//             q-block may be cut into segments owned by consecutive CTAs.  Every segment but
//             the last to finish writes its unnormalised (O, m, l) to a workspace slot; the
//             last arriver (atomic ticket per q-block tile) merges them in segment order and
//             runs the normal epilogue.  Nobody waits on a CTA that has not started, so the
//             protocol is deadlock-free even when other kernels hold SMs.
// This keeps every SM busy at the small per-rank head counts the USP meshes produce
// (FLUX U=8: 3 heads = 54 q-blocks on 148 SMs).
//
// CTA = two 128-row Q tiles that ping-pong on the tensor core; KV tiles of 128 rows
// stream through a 2-stage TMA ring.
//   warp 0      TMA producer for Q and K
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warp 2      TMA producer for V
//   warp 3      idle
//   warps 4-7   softmax / correction / epilogue for Q tile 0 (one row per thread)
//   warps 8-11  same for Q tile 1
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_t (f16
// pairs) overwrites columns [0,64) of S_t after the softmax has read S_t.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <array>
#include <atomic>
#include <map>
#include <mutex>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "fastusp_internal.h"
#include "sm100_ptx.cuh"

namespace fusp {
namespace {

using namespace ptx;

constexpr int kBM = 128;   // rows per Q tile (one softmax warpgroup)
constexpr int kQB = 2 * kBM;  // rows per q-block (one CTA work item)
constexpr int kBN = 128;   // keys per KV tile
constexpr int kD = 128;    // head dim
#ifndef FUSP_SPLIT_S  // 1: S_t(j+1) in two 64-key halves, the upper half issued while the
#define FUSP_SPLIT_S 1   // softmax still works on S_t(j); P.V in two 64-key halves
#endif
constexpr bool kSplitS = FUSP_SPLIT_S != 0;
constexpr int kStages = 2;  // V ring depth
constexpr int kKStages = kSplitS ? 3 : 2;  // K ring depth (split S: K(j+1) is read one step early)
constexpr int kThreads = 384;
constexpr uint32_t kTileBytes = kBM * kD * 2;  // 32 KB: [2 halves][128 rows][128 B]
constexpr uint32_t kHalfBytes = kTileBytes / 2;
constexpr uint32_t kTmemS = 0;    // S_t / P_t at columns [128 t, 128 t + 128)
constexpr uint32_t kTmemO = 256;  // O_t at columns [256 + 128 t, ...)
constexpr float kRescaleThreshold = 8.0f;  // log2 units: lazy O rescale (P <= 2^8 in f16)
#ifndef FUSP_EMU_EVERY
#define FUSP_EMU_EVERY 4
#endif
#ifndef FUSP_PRODUCER_REGS  // setmaxnreg split; the CTA pool is 168 x 384 registers, so
#define FUSP_PRODUCER_REGS 56  // 128 * (168 - producer) >= 256 * (softmax - 168)
#endif
#ifndef FUSP_MMA_UNROLL  // unroll of the issuer's per-k MMA loops (code size vs issue cost)
#define FUSP_MMA_UNROLL 8
#endif
#ifndef FUSP_SOFTMAX_REGS
#define FUSP_SOFTMAX_REGS 224
#endif
static_assert(128 * (168 - FUSP_PRODUCER_REGS) >= 256 * (FUSP_SOFTMAX_REGS - 168),
              "setmaxnreg split exceeds the CTA register pool");
constexpr int kMmaUnroll = FUSP_MMA_UNROLL;
constexpr int kEmuEvery = FUSP_EMU_EVERY;  // 1 exp2 pair in kEmuEvery runs on the FMA pipe
// Stream-K partial slot for one 128-row tile: O as [32 column quads][128 rows][4] f32 (a
// warp's float4 accesses to one quad are contiguous), then m[128], l[128].
constexpr int kSlotTileFloats = kD * kBM + 2 * kBM;
constexpr int kMaxGrid = 160;  // persistent grid cap (B200: 148 SMs)
constexpr size_t kSlotBytes = size_t(2) * kSlotTileFloats * 4;  // both tiles of a q-block

struct __align__(1024) Smem {
  uint8_t q[2][kTileBytes];
  uint8_t k[kKStages][kTileBytes];
  uint8_t v[kStages][kTileBytes];
  uint64_t q_full[2], q_empty[2];
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_full[2], o_done[2];
  uint64_t s_read[2], p_half[2];  // split S: S_t loaded by the softmax / first half of P_t stored
  uint32_t tmem_base;
  uint32_t ticket[2];
};

struct Sched {
  int n_kv;         // KV tiles per q-block
  int qb_per_head;  // q-blocks per head
  int n_qb;         // heads * qb_per_head
  int split;        // 1: stream-K unit ranges; 0: whole q-blocks, strided by gridDim.x
  int total;        // n_qb * n_kv units (< 2^31)
  int begin[kMaxGrid + 1];  // split: CTA c owns units [begin[c], begin[c+1]) = c*total/grid
};

struct Params {
  int sq, skv, heads;
  uint32_t idesc_qk;  // bf16 x bf16 or f16 x f16 Q.K^T
  float scale_log2;  // log2(e) / sqrt(D)
  void* out;
  int out_dtype;     // FUSP_F32 / FUSP_F16 / FUSP_BF16
  int out_chunk;     // rows per output chunk (row -> (row / chunk, row % chunk))
  int64_t out_hs, out_cs, out_rs;  // element strides: head, chunk, row
  float* lse;        // [heads][lse_hs] natural-log LSE or null
  int64_t lse_hs;
  int64_t lse_cs;    // floats between output chunks (the output all-to-all slots), like out_cs
  // Peer-memory output reshard (usp.cpp, PeerWindow): chunk t of the rows is stored straight
  // into Ulysses member t's window over NVLink; its element offset relative to `out` / `lse`
  // (one unified address space) replaces t * out_cs / t * lse_cs.  0 chunks: the strided form.
  int peer_chunks;
  int64_t out_coff[kMaxPeerChunks], lse_coff[kMaxPeerChunks];
  const float* acc_o;    // fp32 [heads][sq][D] running accumulator or null
  const float* acc_lse;  // [heads][sq]
  const int* q_exp;      // per-head f16 range-guard exponents of the operands (null = 0)
  const int* k_exp;
  const int* v_exp;
  Sched sc;
  uint32_t* counters;    // split: [n_qb][2 tiles][arrive, written], zero between launches
  float* slots;          // split: [gridDim.x][2 (first/last segment)][2 tiles][kSlotTileFloats]
  unsigned long long* trace;  // optional per-CTA globaltimer events (attention_trace), or null
};
__device__ __forceinline__ int64_t out_chunk_off(const Params& p, int t) {
  return p.peer_chunks ? p.out_coff[t] : static_cast<int64_t>(t) * p.out_cs;
}
__device__ __forceinline__ int64_t lse_chunk_off(const Params& p, int t) {
  return p.peer_chunks ? p.lse_coff[t] : static_cast<int64_t>(t) * p.lse_cs;
}
// per CTA (SM cycles): start, end, [4 segments][2 tiles][8 events], 70: end (warp 4); then
// [2 tiles][64 KV steps of the first segment][S ready, P published]
constexpr int kTraceSlots = 72 + 2 * 64 * 2;

__device__ __forceinline__ unsigned long long gtimer() {  // SM cycle counter (per-CTA deltas)
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
#ifndef FUSP_TRACE_AT  // debug: which softmax point the per-step trace's 2nd event records
#define FUSP_TRACE_AT 0  // (0 P published, 1 S loaded, 2 row max, 3 exp loop done)
#endif
#ifndef FUSP_TRACE_EPI  // debug: epilogue sub-steps into the (whole-mode unused) slots 3..6
#define FUSP_TRACE_EPI 0
#endif
#ifndef FUSP_TRACE_BUILD  // 1: per-CTA clock64 tracing compiled in (a debug build: the trace
#define FUSP_TRACE_BUILD 0   // checks cost 1-2 % in the KV loop); 0: fusp_attention_trace returns -2
#endif
#define FUSP_TRACE(p, slot)                                                        \
  do {                                                                             \
    if (FUSP_TRACE_BUILD && (p).trace != nullptr)                                  \
      (p).trace[blockIdx.x * kTraceSlots + (slot)] = gtimer();                     \
  } while (0)

// ---- schedule (identical in every role) -------------------------------------------------
// The CTA whose unit range holds unit u: max c with begin[c] <= u (estimate, then correct).
__device__ __forceinline__ int sk_cta_of(const Sched& s, int u) {
  int c = static_cast<int>(static_cast<float>(u) * gridDim.x / static_cast<float>(s.total));
  c = c < 0 ? 0 : (c >= static_cast<int>(gridDim.x) ? gridDim.x - 1 : c);
  while (c > 0 && s.begin[c] > u) --c;
  while (c + 1 < static_cast<int>(gridDim.x) && s.begin[c + 1] <= u) ++c;
  return c;
}
// ctaid / nctaid read through volatile asm: values derived from them at a tile's end are
// not hoisted out of the KV loop (where they would hold registers across the softmax)
__device__ __forceinline__ int cta_id_v() {
  int v;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(v));
  return v;
}
__device__ __forceinline__ int n_cta_v() {
  int v;
  asm volatile("mov.u32 %0, %%nctaid.x;" : "=r"(v));
  return v;
}
__device__ __forceinline__ int sk_cta_of_v(const Sched& s, int u) {
  const int g = n_cta_v();
  int c = static_cast<int>(static_cast<float>(u) * g / static_cast<float>(s.total));
  c = c < 0 ? 0 : (c >= g ? g - 1 : c);
  while (c > 0 && s.begin[c] > u) --c;
  while (c + 1 < g && s.begin[c + 1] <= u) ++c;
  return c;
}
struct Seg {
  int qb, j0, j1;
};
struct SegIter {  // unit indices fit in 32 bits (the planner checks total < 2^31)
  int u, end, qb;
  __device__ explicit SegIter(const Sched& s) {
    u = s.split ? s.begin[blockIdx.x] : 0;
    end = s.split ? s.begin[blockIdx.x + 1] : 0;
    qb = blockIdx.x;
  }
  __device__ bool next(const Sched& s, Seg& g) {
    if (s.split) {
      if (u >= end) return false;
      g.qb = u / s.n_kv;
      g.j0 = u - g.qb * s.n_kv;
      const int left = end - u;
      g.j1 = left < s.n_kv - g.j0 ? g.j0 + left : s.n_kv;
      u += g.j1 - g.j0;
      return true;
    }
    if (qb >= s.n_qb) return false;
    g.qb = qb;
    g.j0 = 0;
    g.j1 = s.n_kv;
    qb += gridDim.x;
    return true;
  }
};
// Workspace slot CTA c uses for its segment of q-block qb (0: its first segment, 1: last).
__device__ __forceinline__ float* seg_slot(const Params& p, int c, int qb, int t) {
  const int first_qb = p.sc.begin[c] / p.sc.n_kv;
  const int which = qb == first_qb ? 0 : 1;
  return p.slots + (static_cast<size_t>(c) * 2 + which) * (2 * kSlotTileFloats) +
         static_cast<size_t>(t) * kSlotTileFloats;
}

// Slot of segment k of a tile whose segments start at CTA c_first: segments k >= 1 are their
// CTAs' first (slot 0); segment 0 is CTA c_first's first only when that CTA's range starts
// inside the tile (which0 = 0), else its last (slot 1).
__device__ __forceinline__ float* tile_slot(float* slots, int c_first, int which0, int k) {
  const int which = k == 0 ? which0 : 0;
  return slots + (static_cast<size_t>(c_first + k) * 2 + which) * (2 * kSlotTileFloats);
}

// The 128 threads of softmax warpgroup t.  bar.sync counts a diverged warp once per divergent
// arrival, so the warp reconverges first (callers often let lane 0 do a global op just before).
__device__ __forceinline__ void wg_bar(int t) {
  __syncwarp();
  if (t == 0) asm volatile("bar.sync 1, 128;" ::: "memory");
  else asm volatile("bar.sync 2, 128;" ::: "memory");
}
// Ticket: release orders this warpgroup's slot stores (seen through the preceding bar.sync)
// before the count; acquire orders the last arriver's slot reads after it.
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float merge_coeffs(float l1, float l2, float& c1, float& c2) {
  // merge_lse per row (reference tensor.cpp:219-240), identity rows pass through.
  if (l2 == -INFINITY) { c1 = 1.f; c2 = 0.f; return l1; }
  if (l1 == -INFINITY) { c1 = 0.f; c2 = 1.f; return l2; }
  const float m = l1 > l2 ? l1 : l2;
  const float lse = m + logf(expf(l1 - m) + expf(l2 - m));
  c1 = expf(l1 - lse);
  c2 = expf(l2 - lse);
  return lse;
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  // shfl from lane 0: the compiler then knows the warp index (and every role branch on it)
  // is warp-uniform, so schedule state and UMMA descriptors can live in uniform registers.
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const Sched& sc = p.sc;

  if (warp == 0 && lane == 0) {
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.q_full[t], 1);
      mbar_init(&sm.q_empty[t], 1);
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], kBM);
      mbar_init(&sm.s_read[t], kBM);
      mbar_init(&sm.p_half[t], kBM);
      mbar_init(&sm.o_done[t], 1);
    }
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
  __syncwarp();  // reconverge warp 0 (lane 0 initialised the barriers) before bar.sync
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // 512 columns is the whole TMEM, so the allocation always starts at lane 0, column 0; the
  // MMA and softmax roles use that constant base (uniform, foldable into the instructions).
  if (tmem != 0u) __trap();
  if (threadIdx.x == 0) FUSP_TRACE(p, 0);
  // Register split: the producer/MMA warpgroup gives registers to the softmax warpgroups.
  if (warp < 4) {
  reg_dealloc<FUSP_PRODUCER_REGS>();  // warpgroup-collective: every warp of the group sets the same limit
  if (warp == 0) {
    // ---------------- TMA producer: Q tiles, then K tiles ----------------
    if (lane == 0) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      SegIter si(sc);
      Seg g;
      uint32_t it = 0, ns = 0;
      while (si.next(sc, g)) {
        const int head = g.qb / sc.qb_per_head;
        const int row0 = (g.qb - head * sc.qb_per_head) * kQB;
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.q_empty[t], (ns & 1) ^ 1);
          mbar_expect_tx(&sm.q_full[t], kTileBytes);
          for (int h = 0; h < 2; ++h)
            tma_load_3d(sm.q[t] + h * kHalfBytes, &tm_q, &sm.q_full[t], h * 64, row0 + t * kBM, head);
        }
        for (int j = g.j0; j < g.j1; ++j, ++it) {
          const int st = it % kKStages;
          const uint32_t ph = (it / kKStages) & 1;
          mbar_wait(&sm.k_empty[st], ph ^ 1);
          mbar_expect_tx(&sm.k_full[st], kTileBytes);
          for (int h = 0; h < 2; ++h)
            tma_load_3d(sm.k[st] + h * kHalfBytes, &tm_k, &sm.k_full[st], h * 64, j * kBN, head);
        }
        ++ns;
      }
    }
  } else if (warp == 2) {
    // ---------------- TMA producer: V tiles ----------------
    if (lane == 0) {
      prefetch_tmap(&tm_v);
      SegIter si(sc);
      Seg g;
      uint32_t it = 0;
      while (si.next(sc, g)) {
        const int head = g.qb / sc.qb_per_head;
        for (int j = g.j0; j < g.j1; ++j, ++it) {
          const int st = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&sm.v_empty[st], ph ^ 1);
          mbar_expect_tx(&sm.v_full[st], kTileBytes);
          for (int h = 0; h < 2; ++h)
            tma_load_3d(sm.v[st] + h * kHalfBytes, &tm_v, &sm.v_full[st], h * 64, j * kBN, head);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- tcgen05.mma issuer ----------------
    // The whole warp walks the schedule (so descriptors stay in uniform registers); lane 0
    // issues every MMA and commit (tcgen05.commit tracks the issuing thread's MMAs).
    const uint32_t idesc_qk = p.idesc_qk;                           // K-major x K-major
    constexpr uint32_t idesc_pv = idesc_f16(0, 0, 0, 1, kBM, kD);   // f16 P(tmem) x f16 V(MN)
    // Descriptors are built once per operand tile, outside the elected region, and advanced
    // by adding the 16-byte-unit offset to the start-address field (smem < 256 KB: no carry).
    // O_t (+)= P_t V(stage st); `first` starts the segment's accumulation.
    auto issue_pv = [&](int t, int st, bool first) {
      // B = V tile, MN-major SW128: LBO = d-half stride (16 KB), SBO = 8-row group (1 KB)
      const uint64_t vdesc = umma_desc_sw128(smem_u32(sm.v[st]), kHalfBytes, 1024);
      if (elect_one()) {
#pragma unroll kMmaUnroll
        for (int k = 0; k < kBN / 16; ++k)
          mma_ts(kTmemO + t * 128, kTmemS + t * 128 + k * 8, vdesc + uint64_t(k * 16 * 128 / 16),
                 idesc_pv, (!first || k > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    // S_t = Q_t K^T over D = 128 in 8 K-steps of 16 (two 64-element swizzle halves).
    auto issue_qk = [&](int t, int st) {
      const uint64_t qdesc = umma_desc_sw128(smem_u32(sm.q[t]), 16, 1024);
      const uint64_t kdesc = umma_desc_sw128(smem_u32(sm.k[st]), 16, 1024);
      if (elect_one()) {
#pragma unroll kMmaUnroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint64_t off16 = ((k >> 2) * kHalfBytes + (k & 3) * 32) / 16;
          mma_ss(kTmemS + t * 128, qdesc + off16, kdesc + off16, idesc_qk, k > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    // Split S: S_t[:, 64 half ..] = Q_t K[64 half ..]^T (N = 64) into S_t columns 64 half ..
    const uint32_t idesc_qk_h = (idesc_qk & ~(0x3Fu << 17)) | ((64u >> 3) << 17);
    auto issue_qk_half = [&](int t, int sk, int half) {
      const uint64_t qdesc = umma_desc_sw128(smem_u32(sm.q[t]), 16, 1024);
      const uint64_t kdesc = umma_desc_sw128(smem_u32(sm.k[sk]) + half * 64 * 128, 16, 1024);
      if (elect_one()) {
#pragma unroll kMmaUnroll
        for (int k = 0; k < kD / 16; ++k) {
          const uint64_t off16 = ((k >> 2) * kHalfBytes + (k & 3) * 32) / 16;
          mma_ss(kTmemS + t * 128 + half * 64, qdesc + off16, kdesc + off16, idesc_qk_h, k > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    // O_t (+)= P_t[:, keys 64 half ..] V[keys 64 half ..]
    auto issue_pv_half = [&](int t, int st, int half, bool first) {
      const uint64_t vdesc = umma_desc_sw128(smem_u32(sm.v[st]), kHalfBytes, 1024);
      if (elect_one()) {
#pragma unroll
        for (int k = half * 4; k < half * 4 + 4; ++k)
          mma_ts(kTmemO + t * 128, kTmemS + t * 128 + k * 8, vdesc + uint64_t(k * 16 * 128 / 16),
                 idesc_pv, (!first || k > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    auto commit = [&](uint64_t* bar) {  // elect.sync picks the same lane as the MMAs
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
    SegIter si(sc);
    Seg g;
    uint32_t it = 0, ns = 0;
    if constexpr (kSplitS) {
      // Per tile t and KV step j (it = global step):
      //   [S_t(j+1) keys 64..127 -> columns 64..127]   once the softmax has loaded S_t(j)
      //   O_t (+)= P_t(j)[keys 0..63] V                 once the first half of P_t(j) is out
      //   O_t  += P_t(j)[keys 64..127] V                once all of P_t(j) is out
      //   [S_t(j+1) keys 0..63 -> columns 0..63]        (P_t(j) lives there: after the P.V)
      // so only 2 of the 4 64-key MMA groups sit between "P_t(j) published" and "S_t(j+1)
      // complete" -- the dependency chain that bounds the kernel.
      while (si.next(sc, g)) {
        {
          const int sk = it % kKStages;
          mbar_wait(&sm.k_full[sk], (it / kKStages) & 1);
          tc_fence_after();
          for (int t = 0; t < 2; ++t) {
            mbar_wait(&sm.q_full[t], ns & 1);
            tc_fence_after();
            issue_qk(t, sk);
            commit(&sm.s_full[t]);
          }
        }
        for (int j = g.j0; j < g.j1; ++j, ++it) {
          const bool nxt = j + 1 < g.j1;
          const int st = it % kStages, sk = it % kKStages, sn = (it + 1) % kKStages;
          if (nxt) {
            mbar_wait(&sm.k_full[sn], ((it + 1) / kKStages) & 1);
            tc_fence_after();
          }
          for (int t = 0; t < 2; ++t) {
            // every s_read phase is consumed (also a segment's last step, where nothing is
            // issued early): arrive/wait stay paired, as compute-sanitizer synccheck requires
            mbar_wait(&sm.s_read[t], it & 1);
            if (nxt) {
              tc_fence_after();
              issue_qk_half(t, sn, 1);
            }
            mbar_wait(&sm.p_half[t], it & 1);
            if (t == 0) mbar_wait(&sm.v_full[st], (it / kStages) & 1);
            tc_fence_after();
            issue_pv_half(t, st, 0, j == g.j0);
            mbar_wait(&sm.p_full[t], it & 1);
            tc_fence_after();
            issue_pv_half(t, st, 1, false);
            if (nxt) {
              issue_qk_half(t, sn, 0);
              commit(&sm.s_full[t]);
            } else {
              commit(&sm.o_done[t]);  // (Q_t is released by the softmax warpgroup)
            }
          }
          commit(&sm.k_empty[sk]);  // S(j) was issued in the previous step / segment start
          commit(&sm.v_empty[st]);
        }
        ++ns;
      }
    } else {
      while (si.next(sc, g)) {
        for (int j = g.j0; j < g.j1; ++j, ++it) {
          const int st = it % kStages;
          const int sk = it % kKStages;
          mbar_wait(&sm.k_full[sk], (it / kKStages) & 1);
          tc_fence_after();
          for (int t = 0; t < 2; ++t) {
            if (j > g.j0) {
              // O_t += P_t(j-1) V(j-1): needs the softmax to have published P_t(j-1)
              const uint32_t ip = it - 1;
              mbar_wait(&sm.p_full[t], ip & 1);
              if (t == 0) mbar_wait(&sm.v_full[ip % kStages], (ip / kStages) & 1);
              tc_fence_after();
              issue_pv(t, ip % kStages, j - 1 == g.j0);
              if (t == 1) commit(&sm.v_empty[ip % kStages]);
            } else {
              mbar_wait(&sm.q_full[t], ns & 1);
              tc_fence_after();
            }
            // S_t = Q_t K_j^T  (executes after PV_t(j-1) has read P_t: tcgen05.mma is in-order)
            issue_qk(t, sk);
            commit(&sm.s_full[t]);
          }
          commit(&sm.k_empty[sk]);
        }
        const uint32_t ip = it - 1;
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.p_full[t], ip & 1);
          if (t == 0) mbar_wait(&sm.v_full[ip % kStages], (ip / kStages) & 1);
          tc_fence_after();
          issue_pv(t, ip % kStages, g.j1 - 1 == g.j0);
          commit(&sm.o_done[t]);
        }
        commit(&sm.v_empty[ip % kStages]);
        ++ns;
      }
    }
  }
  } else {
    reg_alloc<FUSP_SOFTMAX_REGS>();
    // ---------------- softmax warpgroups ----------------
    const int t = (warp - 4) >> 2;          // Q tile 0 / 1
    const int quad = warp & 3;              // TMEM lane quadrant of this warp
    const int r_in_tile = quad * 32 + lane; // row within the 128-row tile
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t t_s = kTmemS + lane_off + t * 128;
    const uint32_t t_o = kTmemO + lane_off + t * 128;

    SegIter si(sc);
    Seg g;
    uint32_t it = 0, ns = 0;
    while (si.next(sc, g)) {
      const int tslot = ns < 4 ? 2 + (ns * 2 + t) * 8 : -1;
      const bool tr = r_in_tile == 0 && tslot >= 0;
      if (tr) FUSP_TRACE(p, tslot);
      const int head = g.qb / sc.qb_per_head;
      // f16 range guard (fastusp_internal.h): Q, K, V of this head were staged as x * 2^-e;
      // 2^(eq + ek) folds into the softmax scale, 2^ev into the output
      const int e_qk = (p.q_exp != nullptr ? p.q_exp[head] : 0) + (p.k_exp != nullptr ? p.k_exp[head] : 0);
      const float sl2 = p.scale_log2 * __int_as_float((127 + e_qk) << 23);
      const float v_scale = p.v_exp != nullptr ? __int_as_float((127 + p.v_exp[head]) << 23) : 1.f;
      const float2 sl2x2 = make_float2(sl2, sl2);
      const int row = (g.qb - head * sc.qb_per_head) * kQB + t * kBM + r_in_tile;
      float m_use = -INFINITY;  // max used for the exponent (raw logit units)
      float l_sum = 0.f;
      for (int j = g.j0; j < g.j1; ++j, ++it) {
        mbar_wait(&sm.s_full[t], it & 1);
        tc_fence_after();
        if (tr && j == g.j0) FUSP_TRACE(p, tslot + 1);
        if (tr && ns == 0 && j - g.j0 < 64) FUSP_TRACE(p, 72 + t * 128 + 2 * (j - g.j0));
        uint32_t s[128];
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
        tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
        tmem_wait_ld();
        if (FUSP_TRACE_AT == 1 && tr && ns == 0 && j - g.j0 < 64) FUSP_TRACE(p, 72 + t * 128 + 2 * (j - g.j0) + 1);
        if constexpr (kSplitS) {  // S_t(j) is in registers: the MMA may overwrite columns 64..127
          tc_fence_before();
          mbar_arrive(&sm.s_read[t]);
        }
        const int valid = p.skv - j * kBN;  // keys in this tile (mask the tail)
        if (valid < kBN) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= valid) s[c] = __float_as_uint(-INFINITY);
        }
        // row max with independent chains (FMNMX3)
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 128; c += 8) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            mx4[i] = fmaxf(mx4[i], fmaxf(__uint_as_float(s[c + i]), __uint_as_float(s[c + 4 + i])));
        }
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        if (FUSP_TRACE_AT == 2 && tr && ns == 0 && j - g.j0 < 64) FUSP_TRACE(p, 72 + t * 128 + 2 * (j - g.j0) + 1);
        // Lazy rescale: keep the old max unless the new one exceeds it by > 8 (log2 units).
        float alpha = 1.f;
        if (m_use == -INFINITY) {
          m_use = mx;
        } else if ((mx - m_use) * sl2 > kRescaleThreshold) {
          alpha = ex2((m_use - mx) * sl2);
          m_use = mx;
        }
        if constexpr (kSplitS) {
          // Rescale O before the first half of P is published (that half's P.V follows it).
          // PV_t(j-1) has completed: the s_full commit for S_t(j) covers every MMA before it.
          if (__any_sync(0xffffffffu, alpha != 1.f) && j > g.j0) {
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              tmem_ld32(t_o + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(t_o + c * 32, o);
            }
          }
        }
        const float neg_m = -m_use * sl2;
        const float2 negm2 = make_float2(neg_m, neg_m);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int pi = 0; pi < 64; ++pi) {
          const float2 x = ffma2(make_float2(__uint_as_float(s[2 * pi]), __uint_as_float(s[2 * pi + 1])),
                                 sl2x2, negm2);
          // one pair in kEmuEvery goes to the FMA pipe, the rest to MUFU.EX2
          const float2 pp = (pi % kEmuEvery == kEmuEvery - 1) ? exp2_poly2(x)
                                                             : make_float2(ex2(x.x), ex2(x.y));
          acc[pi & 3] = fadd2(acc[pi & 3], pp);
          s[pi] = pack_f16x2(pp.x, pp.y);  // P packs into the first 64 slots
          if (pi == 31) {  // first half of P goes out early
            tmem_st32(t_s + 0, &s[0]);
            if constexpr (kSplitS) {
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&sm.p_half[t]);
            }
          }
        }
        if (FUSP_TRACE_AT == 3 && tr && ns == 0 && j - g.j0 < 64) FUSP_TRACE(p, 72 + t * 128 + 2 * (j - g.j0) + 1);
        tmem_st32(t_s + 32, &s[32]);
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        const float2 a = fadd2(a01, a23);
        l_sum = fmaf(l_sum, alpha, a.x + a.y);
        // Rescale the O accumulator when the max moved. PV_t(j-1) has completed: the
        // s_full commit for S_t(j) covers every MMA issued before it.
        if (!kSplitS && __any_sync(0xffffffffu, alpha != 1.f) && j > g.j0) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(t_o + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(t_o + c * 32, o);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        if (FUSP_TRACE_AT == 0 && tr && ns == 0 && j - g.j0 < 64) FUSP_TRACE(p, 72 + t * 128 + 2 * (j - g.j0) + 1);
        mbar_arrive(&sm.p_full[t]);
      }

      // ---------------- segment end: O accumulated for keys of tiles [j0, j1) ----------------
      mbar_wait(&sm.o_done[t], ns & 1);
      tc_fence_after();
      if (tr) FUSP_TRACE(p, tslot + 2);
      // Every MMA of the segment has completed: Q_t may be reloaded.
      if (r_in_tile == 0) mbar_arrive(&sm.q_empty[t]);
      ++ns;
      int nseg = 1, kself = 0, c_first = 0;
      if (sc.split) {
        const int u0 = g.qb * sc.n_kv;
        c_first = sk_cta_of(sc, u0);
        nseg = sk_cta_of(sc, u0 + sc.n_kv - 1) - c_first + 1;
        kself = static_cast<int>(blockIdx.x) - c_first;
      }
      float m_fin = m_use, l_fin = l_sum;
      if (nseg > 1) {
        // Publish-then-count: every segment but the finisher stores its (O, m, l) slot, then
        // bumps the q-block tile's count; whoever brings it to nseg is last and merges.  The
        // lowest CTA's segment (kself 0: the q-block's first keys, processed at the END of
        // that CTA's range) checks the count first and, if every other segment has published,
        // merges without publishing its own.  Nobody ever waits on another CTA.
        // The merge accumulates in this tile's TMEM O: O = w_0 O_0, then O = fma(w_k, O_k, O)
        // for k = 1.. in segment order -- the same fma sequence whichever CTA finishes, so
        // results are bit-identical run to run.  Each step streams one whole 64 KB slot (32
        // float4 loads per thread in flight) and does one TMEM read-modify-write.
        uint32_t* cnt = p.counters + (static_cast<size_t>(g.qb) * 2 + t) * 2;
        bool last = false, published = false;
        if (kself == 0) {
          if (r_in_tile == 0) sm.ticket[t] = ld_acquire(&cnt[0]);
          wg_bar(t);
          last = *reinterpret_cast<volatile uint32_t*>(&sm.ticket[t]) + 1 == static_cast<uint32_t>(nseg);
        }
        if (!last) {
          float* slot = seg_slot(p, blockIdx.x, g.qb, t);
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(t_o + c * 32, o);
            tmem_wait_ld();
            float4* q4 = reinterpret_cast<float4*>(slot) + (c * 8) * kBM + r_in_tile;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              __stcg(q4 + i * kBM, make_float4(__uint_as_float(o[4 * i]), __uint_as_float(o[4 * i + 1]),
                                               __uint_as_float(o[4 * i + 2]), __uint_as_float(o[4 * i + 3])));
          }
          __stcg(slot + kD * kBM + r_in_tile, m_use);
          __stcg(slot + kD * kBM + kBM + r_in_tile, l_sum);
          if (tr) FUSP_TRACE(p, tslot + 4);
          wg_bar(t);  // the warpgroup's stores happen-before thread 0's release (cumulativity)
          if (r_in_tile == 0) {
            sm.ticket[t] = atom_add_acq_rel(&cnt[0], 1u);
          }
          wg_bar(t);
          published = true;
          last = *reinterpret_cast<volatile uint32_t*>(&sm.ticket[t]) + 1 == static_cast<uint32_t>(nseg);
          if (!last) {
            if (tr) FUSP_TRACE(p, tslot + 7);
            tc_fence_before();
            continue;
          }
        }
        if (tr) FUSP_TRACE(p, tslot + 3);
        if (r_in_tile == 0) cnt[0] = 0u;  // every segment has counted: reset for the next launch
        // (m_k, l_k) of every segment (own values for k == kself when unpublished): the loads of
        // up to kMl segments are issued together (one L2 round trip), the rest stream after.
        constexpr int kMl = 8;
        float mk_r[kMl], lk_r[kMl];
#pragma unroll
        for (int k = 0; k < kMl; ++k) {
          mk_r[k] = m_use;
          lk_r[k] = l_sum;
          if (k < nseg && (k != kself || published)) {
            const float* sl = seg_slot(p, c_first + k, g.qb, t);
            mk_r[k] = __ldcg(sl + kD * kBM + r_in_tile);
            lk_r[k] = __ldcg(sl + kD * kBM + kBM + r_in_tile);
          }
        }
        auto seg_ml = [&](int k, float& mk, float& lk) {
          if (k < kMl) {
#pragma unroll
            for (int q = 0; q < kMl; ++q)
              if (q == k) { mk = mk_r[q]; lk = lk_r[q]; }
            return;
          }
          mk = m_use;
          lk = l_sum;
          if (k != kself || published) {
            const float* sl = seg_slot(p, c_first + k, g.qb, t);
            mk = __ldcg(sl + kD * kBM + r_in_tile);
            lk = __ldcg(sl + kD * kBM + kBM + r_in_tile);
          }
        };
        m_fin = -INFINITY;
        for (int k = 0; k < nseg; ++k) {
          float mk, lk;
          seg_ml(k, mk, lk);
          m_fin = fmaxf(m_fin, mk);
        }
        l_fin = 0.f;
        for (int k = 0; k < nseg; ++k) {
          float mk, lk;
          seg_ml(k, mk, lk);
          l_fin = fmaf(ex2((mk - m_fin) * sl2), lk, l_fin);
        }
        if (tr) FUSP_TRACE(p, tslot + 5);
        // k = 0 term: own TMEM tile scaled in place (fast path), or slot 0 stored over it
        float m0, l0;
        seg_ml(0, m0, l0);
        const float w0 = ex2((m0 - m_fin) * sl2);
        if (!published) {
          if (__any_sync(0xffffffffu, w0 != 1.f)) {  // tcgen05.ld/st are warp-collective
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o[32];
              tmem_ld32(t_o + c * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(w0 * __uint_as_float(o[i]));
              tmem_st32(t_o + c * 32, o);
            }
          }
        } else {
          const float4* x4 = reinterpret_cast<const float4*>(seg_slot(p, c_first, g.qb, t)) + r_in_tile;
          float4 x[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = __ldcg(x4 + i * kBM);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              o[4 * i] = __float_as_uint(w0 * x[c * 8 + i].x);
              o[4 * i + 1] = __float_as_uint(w0 * x[c * 8 + i].y);
              o[4 * i + 2] = __float_as_uint(w0 * x[c * 8 + i].z);
              o[4 * i + 3] = __float_as_uint(w0 * x[c * 8 + i].w);
            }
            tmem_st32(t_o + c * 32, o);
          }
        }
        // k >= 1 terms from the slots
#pragma unroll 1
        for (int k = 1; k < nseg; ++k) {
          const float* sl = seg_slot(p, c_first + k, g.qb, t);
          const float4* x4 = reinterpret_cast<const float4*>(sl) + r_in_tile;
          float4 x[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = __ldcg(x4 + i * kBM);
          float mk, lk;
          seg_ml(k, mk, lk);
          const float w = ex2((mk - m_fin) * sl2);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(t_o + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              o[4 * i] = __float_as_uint(fmaf(w, x[c * 8 + i].x, __uint_as_float(o[4 * i])));
              o[4 * i + 1] = __float_as_uint(fmaf(w, x[c * 8 + i].y, __uint_as_float(o[4 * i + 1])));
              o[4 * i + 2] = __float_as_uint(fmaf(w, x[c * 8 + i].z, __uint_as_float(o[4 * i + 2])));
              o[4 * i + 3] = __float_as_uint(fmaf(w, x[c * 8 + i].w, __uint_as_float(o[4 * i + 3])));
            }
            tmem_st32(t_o + c * 32, o);
          }
        }
        tmem_wait_st();
        if (tr) FUSP_TRACE(p, tslot + 6);
      }

      // ---------------- epilogue: O / l, LSE, optional merge, store ----------------
      const bool in_range = row < p.sq;
      // natural-log LSE in accurate math: m/sqrt(D) + ln(l)  (tensor.cpp:177)
      const float lse_b = m_fin * (sl2 * 0.69314718055994530942f) + logf(l_fin);
      const float inv_l = 1.f / l_fin;
      float c_acc = 0.f, c_new = 1.f, lse_out = lse_b;
      if (p.acc_o != nullptr && in_range) {
        const float l1 = p.acc_lse[static_cast<int64_t>(head) * p.sq + row];
        lse_out = merge_coeffs(l1, lse_b, c_acc, c_new);
      }
      const float scale_new = c_new * inv_l * v_scale;
      const int64_t obase = static_cast<int64_t>(head) * p.out_hs +
                            out_chunk_off(p, row / p.out_chunk) +
                            static_cast<int64_t>(row % p.out_chunk) * p.out_rs;
      // O leaves (and the ring accumulator comes in) through accesses where the 4 lanes of a
      // group cover one row's contiguous 32-column chunk: row addresses of the group's 4 rows
      const int e4 = lane & 3;
      int64_t ob_g[4];
      bool in_g[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ob_g[i] = __shfl_sync(0xffffffffu, obase, (lane & ~3) + i);
        in_g[i] = row - e4 + i < p.sq;
      }
      const float* acc_h = p.acc_o != nullptr ? p.acc_o + static_cast<int64_t>(head) * p.sq * kD : nullptr;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld32(t_o + c * 32, o);
        tmem_wait_ld();
        if (FUSP_TRACE_EPI && tr && c == 0) FUSP_TRACE(p, tslot + 3);
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(o[i]) * scale_new;
        if (acc_h != nullptr) {  // merge_lse: O = c_acc * acc + c_new * O / l
          uint32_t a[32];        // piece e (8 floats) of rows 4G+i, then transposed to own row
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
            if (in_g[i]) {
              const float4* src =
                  reinterpret_cast<const float4*>(acc_h + static_cast<int64_t>(row - e4 + i) * kD + c * 32 + e4 * 8);
              x0 = src[0];
              x1 = src[1];
            }
            a[8 * i + 0] = __float_as_uint(x0.x); a[8 * i + 1] = __float_as_uint(x0.y);
            a[8 * i + 2] = __float_as_uint(x0.z); a[8 * i + 3] = __float_as_uint(x0.w);
            a[8 * i + 4] = __float_as_uint(x1.x); a[8 * i + 5] = __float_as_uint(x1.y);
            a[8 * i + 6] = __float_as_uint(x1.z); a[8 * i + 7] = __float_as_uint(x1.w);
          }
          xpose4<8>(a, lane);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaf(c_acc, __uint_as_float(a[i]), v[i]);
        }
        if (p.out_dtype != FUSP_F32) {
          const bool f16 = p.out_dtype == FUSP_F16;
          uint32_t w[16];  // piece q (16 B) = words 4q..4q+3 = columns 32c + 8q ..
#pragma unroll
          for (int e = 0; e < 16; ++e)
            w[e] = f16 ? pack_f16x2(v[2 * e], v[2 * e + 1]) : pack_bf16x2(v[2 * e], v[2 * e + 1]);
          xpose4<4>(w, lane);
          uint16_t* o16p = static_cast<uint16_t*>(p.out);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (in_g[i])
              *reinterpret_cast<uint4*>(o16p + ob_g[i] + c * 32 + e4 * 8) =
                  make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        } else {
          uint32_t w[32];  // piece q (32 B) = floats 8q..8q+7
#pragma unroll
          for (int i = 0; i < 32; ++i) w[i] = __float_as_uint(v[i]);
          xpose4<8>(w, lane);
          float* o32p = static_cast<float*>(p.out);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (in_g[i]) {
              uint4* dst = reinterpret_cast<uint4*>(o32p + ob_g[i] + c * 32 + e4 * 8);
              dst[0] = make_uint4(w[8 * i], w[8 * i + 1], w[8 * i + 2], w[8 * i + 3]);
              dst[1] = make_uint4(w[8 * i + 4], w[8 * i + 5], w[8 * i + 6], w[8 * i + 7]);
            }
        }
      }
      if (FUSP_TRACE_EPI && tr) FUSP_TRACE(p, tslot + 4);
      if (in_range && p.lse != nullptr)
        p.lse[static_cast<int64_t>(head) * p.lse_hs + lse_chunk_off(p, row / p.out_chunk) +
              row % p.out_chunk] = lse_out;
      if (tr) FUSP_TRACE(p, tslot + 7);
      tc_fence_before();
    }
  }

  // bar.sync counts a diverged warp once per divergent arrival: reconverge first, or the
  // producer warps (lane 0 vs 1..31) would release the barrier before the softmax warps finish.
  __syncwarp();
  // peer-memory output: every store this thread made to another GPU's window is visible
  // system-wide before the exchange kernel that follows signals it
  if (p.peer_chunks) __threadfence_system();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) FUSP_TRACE(p, 1);
  if (threadIdx.x == 128) FUSP_TRACE(p, 70);  // same barrier, seen from softmax warp 4
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---- KV-split variant for few q-blocks ----------------------------------------------------
// When a rank's launch has fewer 128-row Q tiles than SMs (FLUX U=8: 3 heads x 36 = 108 tiles
// on 148 SMs) the stream-K schedule above cuts 256-row q-blocks over ~2.7 CTAs and pays the
// partial-slot publish and finisher merge.  Here a work item is ONE 128-row Q tile, whole,
// and the CTA's two softmax warpgroups split its KV range instead of taking two Q tiles:
// chain t processes KV tiles j0 + t, j0 + t + 2, ... with its own S_t / O_t in TMEM, so the
// two chains still ping-pong on the tensor core.  At the tile's end the chains merge inside
// the CTA: (m, l) through shared memory, O through TMEM (warp w of either warpgroup reads the
// same 32 lanes), each warpgroup finishing half of the columns.  No workspace, no tickets.
// SMEM: Q 32 KB + K 4 x 32 KB (each chain keeps its next K tile in flight) + V 2 x 32 KB.
#ifndef FUSP_KV2_KSTAGES
#define FUSP_KV2_KSTAGES 4
#endif
#ifndef FUSP_KV2_VSTAGES
#define FUSP_KV2_VSTAGES 2
#endif
#ifndef FUSP_KV2_EARLY_K
#define FUSP_KV2_EARLY_K 1
#endif
constexpr int kKv2KStages = FUSP_KV2_KSTAGES;
constexpr int kKv2VStages = FUSP_KV2_VSTAGES;
struct __align__(1024) SmemKv2 {
  uint8_t q[kTileBytes];
  uint8_t k[kKv2KStages][kTileBytes];
  uint8_t v[kKv2VStages][kTileBytes];
  uint64_t q_full, q_empty;
  uint64_t k_full[kKv2KStages], k_empty[kKv2KStages];
  uint64_t v_full[kKv2VStages], v_empty[kKv2VStages];
  uint64_t s_full[2], p_full[2], o_done[2];
  uint64_t s_read[2], p_half[2];
  uint32_t tmem_base;
  uint32_t ticket;  // stream-K: the tile's arrival count seen by this CTA
};

// Named barrier over the 8 softmax warps (ids 1, 2 are the per-warpgroup ones).
__device__ __forceinline__ void softmax_bar() {
  __syncwarp();
  asm volatile("bar.sync 3, 256;" ::: "memory");
}

template <bool kSplit>  // kSplit: stream-K segments over the tiles (sc.split == 1)
__global__ void __launch_bounds__(kThreads, 1)
    attn_kv2_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  SmemKv2& sm = *reinterpret_cast<SmemKv2*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                            ~uintptr_t(1023));
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const Sched& sc = p.sc;  // qb = 128-row tile index; stream-K unit ranges when kSplit

  if (warp == 0 && lane == 0) {
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 2);  // both warpgroups release the Q tile
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], kBM);
      mbar_init(&sm.s_read[t], kBM);
      mbar_init(&sm.p_half[t], kBM);
      mbar_init(&sm.o_done[t], 1);
    }
    for (int s = 0; s < kKv2KStages; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kKv2VStages; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  if (tmem != 0u) __trap();
  if (threadIdx.x == 0) FUSP_TRACE(p, 0);
  if (warp < 4) {
    reg_dealloc<FUSP_PRODUCER_REGS>();
    if (warp == 0) {
      // ---------------- TMA producer: the Q tile, then the K tiles in KV order ----------------
      if (lane == 0) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        SegIter si(sc);
        Seg g;
        uint32_t kt = 0, ns = 0;
        while (si.next(sc, g)) {
          const int head = g.qb / sc.qb_per_head;
          const int row0 = (g.qb - head * sc.qb_per_head) * kBM;
          mbar_wait(&sm.q_empty, (ns & 1) ^ 1);
          mbar_expect_tx(&sm.q_full, kTileBytes);
          for (int h = 0; h < 2; ++h)
            tma_load_3d(sm.q + h * kHalfBytes, &tm_q, &sm.q_full, h * 64, row0, head);
          for (int j = g.j0; j < g.j1; ++j, ++kt) {
            const int st = kt % kKv2KStages;
            mbar_wait(&sm.k_empty[st], ((kt / kKv2KStages) & 1) ^ 1);
            mbar_expect_tx(&sm.k_full[st], kTileBytes);
            for (int h = 0; h < 2; ++h)
              tma_load_3d(sm.k[st] + h * kHalfBytes, &tm_k, &sm.k_full[st], h * 64, j * kBN, head);
          }
          ++ns;
        }
      }
    } else if (warp == 2) {
      // ---------------- TMA producer: V tiles in KV order ----------------
      if (lane == 0) {
        prefetch_tmap(&tm_v);
        SegIter si(sc);
        Seg g;
        uint32_t kt = 0;
        while (si.next(sc, g)) {
          const int head = g.qb / sc.qb_per_head;
          for (int j = g.j0; j < g.j1; ++j, ++kt) {
            const int st = kt % kKv2VStages;
            mbar_wait(&sm.v_empty[st], ((kt / kKv2VStages) & 1) ^ 1);
            mbar_expect_tx(&sm.v_full[st], kTileBytes);
            for (int h = 0; h < 2; ++h)
              tma_load_3d(sm.v[st] + h * kHalfBytes, &tm_v, &sm.v_full[st], h * 64, j * kBN, head);
          }
        }
      }
    } else if (warp == 1) {
      // ---------------- tcgen05.mma issuer: two KV chains on one Q tile ----------------
      const uint32_t idesc_qk = p.idesc_qk;
      constexpr uint32_t idesc_pv = idesc_f16(0, 0, 0, 1, kBM, kD);
      const uint32_t idesc_qk_h = (idesc_qk & ~(0x3Fu << 17)) | ((64u >> 3) << 17);
      const uint64_t qdesc = umma_desc_sw128(smem_u32(sm.q), 16, 1024);
      auto issue_qk = [&](int t, int sk) {
        const uint64_t kdesc = umma_desc_sw128(smem_u32(sm.k[sk]), 16, 1024);
        if (elect_one()) {
#pragma unroll kMmaUnroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint64_t off16 = ((k >> 2) * kHalfBytes + (k & 3) * 32) / 16;
            mma_ss(kTmemS + t * 128, qdesc + off16, kdesc + off16, idesc_qk, k > 0 ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto issue_qk_half = [&](int t, int sk, int half) {
        const uint64_t kdesc = umma_desc_sw128(smem_u32(sm.k[sk]) + half * 64 * 128, 16, 1024);
        if (elect_one()) {
#pragma unroll kMmaUnroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint64_t off16 = ((k >> 2) * kHalfBytes + (k & 3) * 32) / 16;
            mma_ss(kTmemS + t * 128 + half * 64, qdesc + off16, kdesc + off16, idesc_qk_h, k > 0 ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto issue_pv_half = [&](int t, int st, int half, bool first) {
        const uint64_t vdesc = umma_desc_sw128(smem_u32(sm.v[st]), kHalfBytes, 1024);
        if (elect_one()) {
#pragma unroll
          for (int k = half * 4; k < half * 4 + 4; ++k)
            mma_ts(kTmemO + t * 128, kTmemS + t * 128 + k * 8, vdesc + uint64_t(k * 16 * 128 / 16),
                   idesc_pv, (!first || k > 0) ? 1u : 0u);
        }
        __syncwarp();
      };
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) mma_commit(bar);
        __syncwarp();
      };
      SegIter si(sc);
      Seg g;
      uint32_t kt0 = 0, ns = 0, cnt[2] = {0, 0};
      while (si.next(sc, g)) {
        const int nt = g.j1 - g.j0;
        const int nc[2] = {(nt + 1) / 2, nt / 2};
        mbar_wait(&sm.q_full, ns & 1);
        tc_fence_after();
        for (int t = 0; t < 2; ++t) {  // each chain's first S
          if (nc[t] == 0) continue;
          const uint32_t kt = kt0 + t;
          mbar_wait(&sm.k_full[kt % kKv2KStages], (kt / kKv2KStages) & 1);
          tc_fence_after();
          issue_qk(t, kt % kKv2KStages);
          commit(&sm.s_full[t]);
#if FUSP_KV2_EARLY_K
          commit(&sm.k_empty[kt % kKv2KStages]);  // K(kt) is free once S(kt) completed
#endif
        }
        for (int s = 0; s < nc[0]; ++s) {
          for (int t = 0; t < 2; ++t) {
            if (s >= nc[t]) continue;
            const uint32_t kt = kt0 + 2 * s + t, ktn = kt + 2;
            const bool nxt = s + 1 < nc[t];
            const int sk = kt % kKv2KStages, sn = ktn % kKv2KStages, sv = kt % kKv2VStages;
            const uint32_t c = cnt[t]++;
            if (nxt) {
              mbar_wait(&sm.k_full[sn], (ktn / kKv2KStages) & 1);
              tc_fence_after();
            }
            mbar_wait(&sm.s_read[t], c & 1);  // every phase consumed (synccheck)
            if (nxt) {
              tc_fence_after();
              issue_qk_half(t, sn, 1);
            }
            mbar_wait(&sm.p_half[t], c & 1);
            mbar_wait(&sm.v_full[sv], (kt / kKv2VStages) & 1);
            tc_fence_after();
            issue_pv_half(t, sv, 0, s == 0);
            mbar_wait(&sm.p_full[t], c & 1);
            tc_fence_after();
            issue_pv_half(t, sv, 1, false);
            if (nxt) {
              issue_qk_half(t, sn, 0);
              commit(&sm.s_full[t]);
#if FUSP_KV2_EARLY_K
              // K(ktn) is released as soon as S(ktn) completes -- a chain step before its
              // P.V -- so the producer refills the stage a step earlier (the next-next tile's
              // S is needed right after the softmax loads this one: a short window)
              commit(&sm.k_empty[sn]);
#endif
            } else {
              commit(&sm.o_done[t]);
            }
#if !FUSP_KV2_EARLY_K
            commit(&sm.k_empty[sk]);  // S(kt) completed before this point
#endif
            commit(&sm.v_empty[sv]);
          }
        }
        kt0 += nt;
        ++ns;
      }
    }
  } else {
    reg_alloc<FUSP_SOFTMAX_REGS>();
    // ---------------- softmax warpgroups: chain t of the Q tile ----------------
    const int t = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int r_in_tile = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t t_s = kTmemS + lane_off + t * 128;
    const uint32_t t_o0 = kTmemO + lane_off;  // chain 0's O (chain 1's at +128)
    SegIter si(sc);
    Seg g;
    uint32_t c = 0, nd = 0;  // bit u: o_done[u] phase
    int seg_no = 0;  // debug trace: per-segment events at slots 2 + 8 seg + e (8 segments)
    const bool tr = threadIdx.x == 128;
    while (si.next(sc, g)) {
      const int tslot = 2 + 8 * (seg_no < 8 ? seg_no : 7);
      ++seg_no;
      const int head = g.qb / sc.qb_per_head;
      const int e_qk = (p.q_exp != nullptr ? p.q_exp[head] : 0) + (p.k_exp != nullptr ? p.k_exp[head] : 0);
      const float sl2 = p.scale_log2 * __int_as_float((127 + e_qk) << 23);
      const float v_scale = p.v_exp != nullptr ? __int_as_float((127 + p.v_exp[head]) << 23) : 1.f;
      const float2 sl2x2 = make_float2(sl2, sl2);
      const int row = (g.qb - head * sc.qb_per_head) * kBM + r_in_tile;
      const int nt = g.j1 - g.j0;
      const int nc[2] = {(nt + 1) / 2, nt / 2};
      float m_use = -INFINITY;
      float l_sum = 0.f;
      for (int i = 0; i < nc[t]; ++i, ++c) {
        const int j = g.j0 + 2 * i + t;
        mbar_wait(&sm.s_full[t], c & 1);
        tc_fence_after();
        if (tr && i == 0) FUSP_TRACE(p, tslot + 0);
        uint32_t s[128];
        tmem_ld32(t_s + 0, *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld32(t_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&s[64]));
        tmem_ld32(t_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&s[96]));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&sm.s_read[t]);
        const int valid = p.skv - j * kBN;
        if (valid < kBN) {
#pragma unroll
          for (int cc = 0; cc < 128; ++cc)
            if (cc >= valid) s[cc] = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int cc = 0; cc < 128; cc += 8) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mx4[q] = fmaxf(mx4[q], fmaxf(__uint_as_float(s[cc + q]), __uint_as_float(s[cc + 4 + q])));
        }
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        float alpha = 1.f;
        if (m_use == -INFINITY) {
          m_use = mx;
        } else if ((mx - m_use) * sl2 > kRescaleThreshold) {
          alpha = ex2((m_use - mx) * sl2);
          m_use = mx;
        }
        if (__any_sync(0xffffffffu, alpha != 1.f) && i > 0) {
#pragma unroll 1
          for (int cc = 0; cc < 4; ++cc) {
            uint32_t o[32];
            tmem_ld32(t_o0 + t * 128 + cc * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 32; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha);
            tmem_st32(t_o0 + t * 128 + cc * 32, o);
          }
        }
        const float neg_m = -m_use * sl2;
        const float2 negm2 = make_float2(neg_m, neg_m);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int pi = 0; pi < 64; ++pi) {
          const float2 x = ffma2(make_float2(__uint_as_float(s[2 * pi]), __uint_as_float(s[2 * pi + 1])),
                                 sl2x2, negm2);
          const float2 pp = (pi % kEmuEvery == kEmuEvery - 1) ? exp2_poly2(x)
                                                             : make_float2(ex2(x.x), ex2(x.y));
          acc[pi & 3] = fadd2(acc[pi & 3], pp);
          s[pi] = pack_f16x2(pp.x, pp.y);
          if (pi == 31) {
            tmem_st32(t_s + 0, &s[0]);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.p_half[t]);
          }
        }
        tmem_st32(t_s + 32, &s[32]);
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        const float2 a = fadd2(a01, a23);
        l_sum = fmaf(l_sum, alpha, a.x + a.y);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&sm.p_full[t]);
      }
      // ---------------- tile end: both chains' MMAs complete, then merge ----------------
      if (tr) FUSP_TRACE(p, tslot + 1);
      for (int u = 0; u < 2; ++u) {
        if (nc[u] == 0) continue;
        mbar_wait(&sm.o_done[u], (nd >> u) & 1);
        nd ^= 1u << u;
      }
      tc_fence_after();
      // (m, l) exchange through the Q tile's shared memory: nothing reads Q any more (every
      // MMA of the tile completed) and it is only reloaded after both warpgroups release it
      float2* ml = reinterpret_cast<float2*>(sm.q);
      ml[t * kBM + r_in_tile] = make_float2(m_use, l_sum);
      softmax_bar();
      const float2 o_ml = ml[(1 - t) * kBM + r_in_tile];
      softmax_bar();
      if (r_in_tile == 0) mbar_arrive(&sm.q_empty);
      if (tr) FUSP_TRACE(p, tslot + 2);
      const float m0 = t == 0 ? m_use : o_ml.x, l0 = t == 0 ? l_sum : o_ml.y;
      const float m1 = t == 0 ? o_ml.x : m_use, l1 = t == 0 ? o_ml.y : l_sum;
      const bool has1 = nc[1] > 0;
      const float m_self = has1 ? fmaxf(m0, m1) : m0;
      const float w0 = ex2((m0 - m_self) * sl2);
      const float w1 = has1 ? ex2((m1 - m_self) * sl2) : 0.f;
      const float l_self = w0 * l0 + w1 * l1;
      // this CTA's part of the tile, columns [32 cc, 32 cc + 32): X = w0 O0 + w1 O1 (frame m_self)
      auto self_chunk = [&](int cc, float (&v)[32], float a0, float a1, bool h1) {
        uint32_t o[32];
        tmem_ld32(t_o0 + cc * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = a0 * __uint_as_float(o[q]);
        if (h1) {  // (warp-uniform: the tile's chain count)
          tmem_ld32(t_o0 + 128 + cc * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = fmaf(a1, __uint_as_float(o[q]), v[q]);
        }
      };
      // Stream-K over whole tiles (sc.split): the tile's key range may be cut into segments
      // owned by consecutive CTAs.  Same publish-then-count protocol as attn_fwd_kernel, one
      // ticket per tile: every segment but the finisher stores X and (m_self, l_self) to its
      // slot and counts; the segment that brings the count to nseg merges all of them in
      // segment order (its own X from TMEM, bit-equal to what it would have stored), so the
      // result does not depend on which CTA finishes.  The tile's first segment (processed last
      // by its CTA) checks the count first and skips publishing when it is already the last.
      int nseg = 1, kself = 0, c_first = 0, which0 = 0;
      if (kSplit) {
        const int u0 = g.qb * sc.n_kv;
        c_first = sk_cta_of_v(sc, u0);
        nseg = sk_cta_of_v(sc, u0 + sc.n_kv - 1) - c_first + 1;
        kself = cta_id_v() - c_first;
        which0 = sc.begin[c_first] >= u0 ? 0 : 1;
      }
      float m_fin = m_self, l_fin = l_self;
      float e_w0 = w0, e_w1 = w1;  // epilogue weights of O0 / O1
      bool e_has1 = has1;
      if (nseg > 1) {
        uint32_t* cnt = p.counters + static_cast<size_t>(g.qb) * 2;
        bool last = false;
        if (kself == 0) {
          if (threadIdx.x == 128) sm.ticket = ld_acquire(cnt);
          softmax_bar();
          last = *reinterpret_cast<volatile uint32_t*>(&sm.ticket) + 1 == static_cast<uint32_t>(nseg);
          softmax_bar();  // every thread read the ticket before it is rewritten
        }
        if (!last) {
          float* slot = tile_slot(p.slots, c_first, which0, kself);
#pragma unroll 1
          for (int cc = 2 * t; cc < 2 * t + 2; ++cc) {
            float v[32];
            self_chunk(cc, v, w0, w1, has1);
            float4* q4 = reinterpret_cast<float4*>(slot) + (cc * 8) * kBM + r_in_tile;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              __stcg(q4 + i * kBM, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
          }
          if (t == 0) {
            __stcg(slot + kD * kBM + r_in_tile, m_self);
            __stcg(slot + kD * kBM + kBM + r_in_tile, l_self);
          }
          if (tr) FUSP_TRACE(p, tslot + 3);
          softmax_bar();  // every slot store happens-before thread 128's release
          if (threadIdx.x == 128) sm.ticket = atom_add_acq_rel(cnt, 1u);
          softmax_bar();
          last = *reinterpret_cast<volatile uint32_t*>(&sm.ticket) + 1 == static_cast<uint32_t>(nseg);
          if (!last) {
            if (tr) FUSP_TRACE(p, tslot + 6);
            // both chains' O were read before the next tile's P.V overwrites them
            tc_fence_before();
            softmax_bar();
            continue;
          }
        }
        if (tr) FUSP_TRACE(p, tslot + 4);
        if (threadIdx.x == 128) *cnt = 0u;  // every segment has counted: zero for the next launch
        m_fin = -INFINITY;
        for (int k = 0; k < nseg; ++k) {
          const float mk = k == kself ? m_self : __ldcg(tile_slot(p.slots, c_first, which0, k) + kD * kBM + r_in_tile);
          m_fin = fmaxf(m_fin, mk);
        }
        l_fin = 0.f;
        for (int k = 0; k < nseg; ++k) {
          const float* sl = tile_slot(p.slots, c_first, which0, k);
          const float mk = k == kself ? m_self : __ldcg(sl + kD * kBM + r_in_tile);
          const float lk = k == kself ? l_self : __ldcg(sl + kD * kBM + kBM + r_in_tile);
          l_fin = fmaf(ex2((mk - m_fin) * sl2), lk, l_fin);
        }
        // merged O (frame m_fin) over this warpgroup's columns, back into O0's TMEM columns:
        // the epilogue below then reads it with weights (1, -)
#pragma unroll 1
        for (int cc = 2 * t; cc < 2 * t + 2; ++cc) {
          float v[32];
#pragma unroll 1
          for (int k = 0; k < nseg; ++k) {
            const float* sl = tile_slot(p.slots, c_first, which0, k);
            const float mk = k == kself ? m_self : __ldcg(sl + kD * kBM + r_in_tile);
            const float wk = ex2((mk - m_fin) * sl2);
            // 16 columns at a time (register pressure here spills the KV loop's state)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float x[16];
              if (k == kself) {  // X_self exactly as self_chunk computes (and publishes) it
                uint32_t o[16];
                tmem_ld16(t_o0 + cc * 32 + hh * 16, o);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 16; ++q) x[q] = w0 * __uint_as_float(o[q]);
                if (has1) {
                  tmem_ld16(t_o0 + 128 + cc * 32 + hh * 16, o);
                  tmem_wait_ld();
#pragma unroll
                  for (int q = 0; q < 16; ++q) x[q] = fmaf(w1, __uint_as_float(o[q]), x[q]);
                }
              } else {
                const float4* x4 = reinterpret_cast<const float4*>(sl) + (cc * 8 + hh * 4) * kBM + r_in_tile;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float4 y = __ldcg(x4 + i * kBM);
                  x[4 * i] = y.x; x[4 * i + 1] = y.y; x[4 * i + 2] = y.z; x[4 * i + 3] = y.w;
                }
              }
              if (k == 0) {
#pragma unroll
                for (int q = 0; q < 16; ++q) v[hh * 16 + q] = wk * x[q];
              } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) v[hh * 16 + q] = fmaf(wk, x[q], v[hh * 16 + q]);
              }
            }
          }
          uint32_t vo[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) vo[q] = __float_as_uint(v[q]);
          tmem_st32(t_o0 + cc * 32, vo);
        }
        tmem_wait_st();
        e_w0 = 1.f;
        e_has1 = false;
        if (tr) FUSP_TRACE(p, tslot + 5);
      }
      const bool in_range = row < p.sq;
      const float lse_b = m_fin * (sl2 * 0.69314718055994530942f) + logf(l_fin);
      const float inv_l = 1.f / l_fin;
      float c_acc = 0.f, c_new = 1.f, lse_out = lse_b;
      if (p.acc_o != nullptr && in_range) {
        const float la = p.acc_lse[static_cast<int64_t>(head) * p.sq + row];
        lse_out = merge_coeffs(la, lse_b, c_acc, c_new);
      }
      const float scale_new = c_new * inv_l * v_scale;
      const int64_t obase = static_cast<int64_t>(head) * p.out_hs +
                            out_chunk_off(p, row / p.out_chunk) +
                            static_cast<int64_t>(row % p.out_chunk) * p.out_rs;
      const int e4 = lane & 3;
      int64_t ob_g[4];
      bool in_g[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ob_g[q] = __shfl_sync(0xffffffffu, obase, (lane & ~3) + q);
        in_g[q] = row - e4 + q < p.sq;
      }
      const float* acc_h = p.acc_o != nullptr ? p.acc_o + static_cast<int64_t>(head) * p.sq * kD : nullptr;
      // warpgroup t finishes columns [64 t, 64 t + 64): O = (w0 O0 + w1 O1) / l
#pragma unroll 1
      for (int cc = 2 * t; cc < 2 * t + 2; ++cc) {
        float v[32];
        self_chunk(cc, v, e_w0, e_w1, e_has1);
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] *= scale_new;
        if (acc_h != nullptr) {
          uint32_t av[32];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), x1 = x0;
            if (in_g[q]) {
              const float4* src =
                  reinterpret_cast<const float4*>(acc_h + static_cast<int64_t>(row - e4 + q) * kD + cc * 32 + e4 * 8);
              x0 = src[0];
              x1 = src[1];
            }
            av[8 * q + 0] = __float_as_uint(x0.x); av[8 * q + 1] = __float_as_uint(x0.y);
            av[8 * q + 2] = __float_as_uint(x0.z); av[8 * q + 3] = __float_as_uint(x0.w);
            av[8 * q + 4] = __float_as_uint(x1.x); av[8 * q + 5] = __float_as_uint(x1.y);
            av[8 * q + 6] = __float_as_uint(x1.z); av[8 * q + 7] = __float_as_uint(x1.w);
          }
          xpose4<8>(av, lane);
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = fmaf(c_acc, __uint_as_float(av[q]), v[q]);
        }
        if (p.out_dtype != FUSP_F32) {
          const bool f16 = p.out_dtype == FUSP_F16;
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            w[e] = f16 ? pack_f16x2(v[2 * e], v[2 * e + 1]) : pack_bf16x2(v[2 * e], v[2 * e + 1]);
          xpose4<4>(w, lane);
          uint16_t* o16p = static_cast<uint16_t*>(p.out);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (in_g[q])
              *reinterpret_cast<uint4*>(o16p + ob_g[q] + cc * 32 + e4 * 8) =
                  make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        } else {
          uint32_t w[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) w[q] = __float_as_uint(v[q]);
          xpose4<8>(w, lane);
          float* o32p = static_cast<float*>(p.out);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (in_g[q]) {
              uint4* dst = reinterpret_cast<uint4*>(o32p + ob_g[q] + cc * 32 + e4 * 8);
              dst[0] = make_uint4(w[8 * q], w[8 * q + 1], w[8 * q + 2], w[8 * q + 3]);
              dst[1] = make_uint4(w[8 * q + 4], w[8 * q + 5], w[8 * q + 6], w[8 * q + 7]);
            }
        }
      }
      if (t == 0 && in_range && p.lse != nullptr)
        p.lse[static_cast<int64_t>(head) * p.lse_hs + lse_chunk_off(p, row / p.out_chunk) +
              row % p.out_chunk] = lse_out;
      if (tr) FUSP_TRACE(p, tslot + 6);
      // both chains' O have been read before either chain's next-tile P.V can overwrite them
      tc_fence_before();
      softmax_bar();
    }
  }
  __syncwarp();
  if (p.peer_chunks) __threadfence_system();  // as attn_fwd_kernel
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 128) FUSP_TRACE(p, 1);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---- host-side schedule ------------------------------------------------------------------
// (tuning knobs set by fusp_attention_schedule from any thread: atomics, read once per plan)
std::atomic<int> g_sched_mode{0};  // 0 auto, 1 whole q-blocks, 2 stream-K split, 3-5 variants
unsigned long long* g_trace = nullptr;  // debug event buffer (attention_trace), device memory
bool g_trace_on = false;
std::atomic<int> g_max_ctas{0};    // 0 = every SM

}  // namespace
int sm_count() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() <= static_cast<size_t>(dev)) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}
namespace {

struct Plan {
  Sched sc;
  int grid;
  int kv2;  // 1: attn_kv2_kernel over whole 128-row Q tiles (chains split the KV range)
};

Plan plan_attention(int heads, int sq, int skv, bool have_ws, int max_ctas) {
  Plan pl{};
  const int g_sched_mode = fusp::g_sched_mode.load(std::memory_order_relaxed);
  const int g_max_ctas = fusp::g_max_ctas.load(std::memory_order_relaxed);
  int sms = sm_count();
  if (g_max_ctas > 0 && g_max_ctas < sms) sms = g_max_ctas;
  if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;
  if (sms > kMaxGrid) sms = kMaxGrid;
  pl.sc.n_kv = (skv + kBN - 1) / kBN;
  pl.sc.qb_per_head = (sq + kQB - 1) / kQB;
  pl.sc.n_qb = heads * pl.sc.qb_per_head;
  const int64_t total = static_cast<int64_t>(pl.sc.n_qb) * pl.sc.n_kv;
  pl.sc.total = total < (int64_t(1) << 31) ? static_cast<int>(total) : 0;
  const int waves = (pl.sc.n_qb + sms - 1) / sms;
  const double fill = static_cast<double>(pl.sc.n_qb) / (static_cast<double>(waves) * sms);
  bool split = have_ws && pl.sc.n_kv >= 2 && fill < 0.96 && pl.sc.total > 0;
  if (g_sched_mode == 1) split = false;
  if (g_sched_mode >= 2) split = have_ws && pl.sc.n_kv >= 2 && pl.sc.total > 0;
  pl.sc.split = split ? 1 : 0;
  // KV-split CTAs (attn_kv2_kernel): whole 128-row Q tiles, one wave, no partial merges.
  // Chosen (auto) where stream-K would otherwise cut 256-row q-blocks and the 128-row tiles
  // fill most of one wave; mode 4 forces it.
  {
    const int tiles = heads * ((sq + kBM - 1) / kBM);
    const int64_t units = static_cast<int64_t>(tiles) * pl.sc.n_kv;
    // KV-split CTAs with stream-K over whole tiles: every SM busy, at least 4 KV tiles per
    // CTA (two per chain); mode 5 forces it
    if (g_sched_mode == 5 && have_ws && pl.sc.n_kv >= 2 && units < (int64_t(1) << 31)) {
      Plan k{};
      k.kv2 = 1;
      k.sc.n_kv = pl.sc.n_kv;
      k.sc.qb_per_head = (sq + kBM - 1) / kBM;
      k.sc.n_qb = tiles;
      k.sc.split = 1;
      k.sc.total = static_cast<int>(units);
      const int g = k.sc.total / 4;
      k.grid = g < sms ? (g > 0 ? g : 1) : sms;
      for (int c = 0; c <= k.grid; ++c)
        k.sc.begin[c] = static_cast<int>(static_cast<int64_t>(c) * k.sc.total / k.grid);
      return k;
    }
    const bool fits = tiles <= sms && pl.sc.n_kv >= 4;
    const bool auto_kv2 = split && g_sched_mode == 0 && fits && 10 * tiles >= 6 * sms;
    if ((g_sched_mode == 4 && fits) || auto_kv2) {
      Plan k{};
      k.kv2 = 1;
      k.sc.n_kv = pl.sc.n_kv;
      k.sc.qb_per_head = (sq + kBM - 1) / kBM;
      k.sc.n_qb = tiles;
      k.sc.split = 0;
      k.sc.total = tiles * pl.sc.n_kv;
      k.grid = tiles;
      return k;
    }
  }
  // aligned split: every q-block cut into nseg equal KV segments, one per CTA (grid =
  // n_qb * nseg <= SMs): one partial merge per extra segment instead of stream-K's
  // arbitrary cuts (2-3 partial slots per q-block at FLUX U=8)
  const int nseg = pl.sc.n_qb > 0 ? sms / pl.sc.n_qb : 0;
  if (split && g_sched_mode == 3 && nseg >= 2 && pl.sc.n_kv >= 2 * nseg) {
    pl.grid = pl.sc.n_qb * nseg;
    for (int c = 0; c <= pl.grid; ++c) {
      const int qb = c / nseg, k = c % nseg;
      pl.sc.begin[c] = qb * pl.sc.n_kv + (k * pl.sc.n_kv) / nseg;
    }
    return pl;
  }
  if (split) {
    // at least 2 KV tiles per CTA so each segment amortises its Q load and epilogue
    const int g = pl.sc.total / 2;
    pl.grid = g < sms ? (g > 0 ? g : 1) : sms;
    for (int c = 0; c <= pl.grid; ++c)
      pl.sc.begin[c] = static_cast<int>(static_cast<int64_t>(c) * pl.sc.total / pl.grid);
  } else {
    pl.grid = pl.sc.n_qb < sms ? pl.sc.n_qb : sms;
  }
  return pl;
}

}  // namespace

// Host launcher. q,k: bf16 [heads][sq|skv][128] (row stride 128); v: f16 [heads][skv][128].
fusp_status launch_attention(const AttnLaunch& a, cudaStream_t stream) {
  if (a.d != kD) return launch_attention_generic(a, stream);  // CUDA-core f32 path for other D
  if (a.sq <= 0 || a.heads <= 0) return FUSP_OK;
  if (a.skv <= 0) return set_error(FUSP_ERR_SHAPE, "attention kernel: empty KV (caller handles it)");
  CUtensorMap tq, tk, tv;
  fusp_status st;
  const bool qk16 = a.qk_dtype == FUSP_F16;
  const CUtensorMapDataType qkt = qk16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  if ((st = make_tmap_rows(&tq, a.q, qkt, a.heads, a.sq, a.q_hs)) != FUSP_OK) return st;
  if ((st = make_tmap_rows(&tk, a.k, qkt, a.heads, a.skv, a.k_hs)) != FUSP_OK) return st;
  if ((st = make_tmap_rows(&tv, a.v, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, a.heads, a.skv, a.v_hs)) != FUSP_OK)
    return st;
  Params p{};
  p.sq = a.sq;
  p.skv = a.skv;
  p.heads = a.heads;
  p.idesc_qk = qk16 ? idesc_f16(0, 0, 0, 0, kBM, kBN) : idesc_f16(1, 1, 0, 0, kBM, kBN);
  p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(a.d)));
  p.out = a.out;
  p.out_dtype = a.out_dtype;
  p.out_chunk = a.out_chunk > 0 ? a.out_chunk : a.sq;
  p.out_hs = a.out_hs;
  p.out_cs = a.out_cs;
  p.out_rs = a.out_rs;
  p.lse = a.lse;
  p.lse_hs = a.lse_hs;
  p.lse_cs = a.lse_cs;
  if (a.peer_chunks > 0) {
    if (a.peer_chunks > kMaxPeerChunks || (p.sq + p.out_chunk - 1) / p.out_chunk > a.peer_chunks)
      return set_error(FUSP_ERR_INVALID_ARGUMENT, "attention: peer chunk table too small");
    p.peer_chunks = a.peer_chunks;
    const int64_t esz = a.out_dtype == FUSP_F32 ? 4 : 2;
    for (int t = 0; t < a.peer_chunks; ++t) {
      const int64_t d = reinterpret_cast<const char*>(a.out_peer[t]) - static_cast<const char*>(a.out);
      if (d % esz != 0) return set_error(FUSP_ERR_INVALID_ARGUMENT, "attention: misaligned peer chunk");
      p.out_coff[t] = d / esz;
      if (a.lse != nullptr) {
        const int64_t dl = reinterpret_cast<const char*>(a.lse_peer[t]) - reinterpret_cast<const char*>(a.lse);
        if (dl % 4 != 0) return set_error(FUSP_ERR_INVALID_ARGUMENT, "attention: misaligned peer LSE chunk");
        p.lse_coff[t] = dl / 4;
      }
    }
  }
  p.acc_o = a.acc_o;
  p.acc_lse = a.acc_lse;
  p.q_exp = a.q_exp;
  p.k_exp = a.k_exp;
  p.v_exp = a.v_exp;
  const size_t need = attention_workspace_bytes(a.heads, a.sq, a.skv);
  const bool have_ws = a.split_ws != nullptr && need > 0 && a.split_ws_bytes >= need &&
                       a.split_counters != nullptr &&
                       a.split_counter_words >= attention_counter_words(a.heads, a.sq);
  // plans are pure functions of the shape and the knobs: cached (no per-launch host work)
  Plan pl;
  {
    static std::mutex mu;
    static std::map<std::array<int, 8>, Plan> cache;
    const std::array<int, 8> key{a.heads, a.sq, a.skv, have_ws ? 1 : 0, a.max_ctas, g_sched_mode,
                                 g_max_ctas, sm_count()};
    std::lock_guard<std::mutex> lk(mu);
    auto itp = cache.find(key);
    if (itp == cache.end()) {
      if (cache.size() > 256) cache.clear();
      itp = cache.emplace(key, plan_attention(a.heads, a.sq, a.skv, have_ws, a.max_ctas)).first;
    }
    pl = itp->second;
  }
  p.sc = pl.sc;
  if (pl.sc.split) {
    p.counters = a.split_counters;
    p.slots = static_cast<float*>(a.split_ws);
  }
  if (g_trace_on) {
    if (g_trace == nullptr) FUSP_CUDA(cudaMalloc(&g_trace, sizeof(unsigned long long) * kMaxGrid * kTraceSlots));
    FUSP_CUDA(cudaMemsetAsync(g_trace, 0, sizeof(unsigned long long) * kMaxGrid * kTraceSlots, stream));
    p.trace = g_trace;
  }
  if (pl.kv2) {
    const int smem2 = static_cast<int>(sizeof(SmemKv2)) + 1024;
    auto* kern = pl.sc.split ? attn_kv2_kernel<true> : attn_kv2_kernel<false>;
    FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(kern), smem2, "attn_kv2_kernel"));
    kern<<<pl.grid, kThreads, smem2, stream>>>(tq, tk, tv, p);
    count_launch();
    cudaError_t e2 = cudaGetLastError();
    if (e2 != cudaSuccess) return set_cuda_error(e2, "attn_kv2_kernel launch");
    return FUSP_OK;
  }
  const int smem = static_cast<int>(sizeof(Smem)) + 1024;
  FUSP_CHECK(ensure_smem_attr(reinterpret_cast<const void*>(attn_fwd_kernel), smem, "attn_fwd_kernel"));
  attn_fwd_kernel<<<pl.grid, kThreads, smem, stream>>>(tq, tk, tv, p);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "attn_fwd_kernel launch");
  return FUSP_OK;
}

// Stream-K partial slots: two per CTA, sized for every SM so they are valid for any grid the
// planner picks.  Contents need no initialisation.
size_t attention_workspace_bytes(int heads, int sq, int skv) {
  if (heads <= 0 || sq <= 0 || skv <= 0) return 0;
  return static_cast<size_t>(sm_count()) * 2 * kSlotBytes;
}
// Stream-K ticket counters: [n_qb][2 tiles][arrive, written].  They must be zero when first
// used and live in memory nothing else writes; the finisher of each split q-block tile
// resets its pair, so they are zero again after every launch.
size_t attention_counter_words(int heads, int sq) {
  if (heads <= 0 || sq <= 0) return 0;
  return static_cast<size_t>(heads) * ((sq + kQB - 1) / kQB) * 4;
}

fusp_status ensure_counters(CounterBuf& b, size_t words, cudaStream_t s) {
  int dev = 0;
  FUSP_CUDA(cudaGetDevice(&dev));
  if (b.ptr != nullptr && b.words >= words && b.device == dev) return FUSP_OK;
  if (b.ptr != nullptr) {
    FUSP_CUDA(cudaFreeAsync(b.ptr, s));
    b.ptr = nullptr;
    b.words = 0;
  }
  const size_t n = words < 4096 ? 4096 : words;
  FUSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&b.ptr), n * 4, s));
  FUSP_CUDA(cudaMemsetAsync(b.ptr, 0, n * 4, s));
  b.words = n;
  b.device = dev;
  return FUSP_OK;
}

// Debug timeline: per-CTA globaltimer events of the most recent traced launch.
int attention_trace(int enable, unsigned long long* host, size_t n) {
  if (!FUSP_TRACE_BUILD) return -2;  // tools/build_variants.sh trace:-DFUSP_TRACE_BUILD=1
  g_trace_on = enable != 0;
  if (host != nullptr && g_trace != nullptr) {
    const size_t m = n < size_t(kMaxGrid) * kTraceSlots ? n : size_t(kMaxGrid) * kTraceSlots;
    if (cudaMemcpy(host, g_trace, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
      return -1;
    return static_cast<int>(m);
  }
  return 0;
}

void set_attention_schedule(int mode, int max_ctas) {
  g_sched_mode = mode;
  g_max_ctas = max_ctas;
}

// Every kernel of this file, for preload_kernels() (lazy module loading, see runtime.cpp).
void append_kernels_attention(std::vector<const void*>& v) {
  v.push_back(reinterpret_cast<const void*>(attn_fwd_kernel));
  v.push_back(reinterpret_cast<const void*>(attn_kv2_kernel<false>));
  v.push_back(reinterpret_cast<const void*>(attn_kv2_kernel<true>));
}

}  // namespace fusp
