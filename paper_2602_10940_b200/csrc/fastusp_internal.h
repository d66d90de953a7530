// Internal declarations shared by the fastusp translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>

#include "../../include/fastusp.h"

namespace fusp {

// ---- errors (thread-local last error, fastusp.h) --------------------------------------
fusp_status set_error(fusp_status code, const std::string& msg);
fusp_status set_cuda_error(cudaError_t e, const std::string& where);
void clear_error();

#define FUSP_CHECK(expr)                      \
  do {                                        \
    fusp_status _st = (expr);                 \
    if (_st != FUSP_OK) return _st;           \
  } while (0)
#define FUSP_CUDA(expr)                                              \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) return set_cuda_error(_e, #expr);         \
  } while (0)

void count_launch(int n = 1);
// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device (per-context) attribute: set it
// once per (kernel, device), thread-safely, before the first launch on that device.
fusp_status ensure_smem_attr(const void* kernel, int bytes, const char* name);
// The projection GEMMs' stream-K workspace of stream `s` (>= `words` zeroed counters, >= `bytes`
// of partial slots), held while `launch` enqueues its kernel; launch(nullptr, nullptr) when it
// cannot grow (graph capture): the caller then runs without the split.
fusp_status with_proj_workspace(cudaStream_t s, size_t words, size_t bytes,
                                const std::function<fusp_status(uint32_t*, float*)>& launch);
// Load every kernel of the library on the current device now (lazy module loading; runtime.cpp).
fusp_status preload_kernels();

// ---- TMA descriptors ------------------------------------------------------------------
// 3-D map over [heads][rows][128] 16-bit elements with a head stride of `head_stride`
// elements (rows are 128 elements apart); box = 64 elements x 128 rows x 1 head, 128B swizzle.
// Generic tiled tensor map (128B swizzle, L2 256B promotion, zero OOB fill).
fusp_status encode_tmap(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
                        const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                        const cuuint32_t* elem_strides);
fusp_status make_tmap_rows(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int heads,
                           int rows, int64_t head_stride);

// ---- output projection (proj_sm100.cu) ---------------------------------------------------
fusp_status launch_out_proj(const void* o, int o_dtype, int b, int h, int s, const void* w, int n,
                            void* y, int y_dtype, cudaStream_t stream);
struct QkvDst {  // where the QKV projection writes: plain [B][H][S][128] (u = 1) or Ulysses slots
  void *q, *k, *v;
  int qk_dtype, v_dtype;
  int u;
  int64_t slot_stride;  // elements between slots
  // Peer-memory Ulysses (csrc/peer.cu): slot t lives in member t's window, slot_boff[t] bytes
  // from slot 0 (q / k / v address slot 0); null = t * slot_stride in one buffer
  const int64_t* slot_boff = nullptr;
};
fusp_status launch_qkv_proj_to(const void* x, int x_dtype, int b, int s, int c, const void* w, int heads,
                               const QkvDst& dst, const float* wq, const float* wk, float eps,
                               const float* cosv, const float* sinv, int64_t pos0, cudaStream_t stream);
fusp_status launch_qkv_proj(const void* x, int x_dtype, int b, int s, int c, const void* w, int heads,
                            void* q, void* k, void* v, int qkv_dtype, const float* wq, const float* wk,
                            float eps, const float* cosv, const float* sinv, int64_t pos0,
                            cudaStream_t stream);

// ---- attention kernel -----------------------------------------------------------------
constexpr int kMaxPeerChunks = 16;  // Ulysses members a kernel stores into directly (NVLink domain)
struct AttnLaunch {
  const void* q;  // bf16|f16 [heads][sq][128], head stride q_hs elements
  const void* k;  // bf16|f16 [heads][skv][128]
  const void* v;  // f16  [heads][skv][128]
  int64_t q_hs, k_hs, v_hs;
  int heads, sq, skv, d;
  int qk_dtype;   // FUSP_BF16 (default) or FUSP_F16 for Q and K
  void* out;
  int out_dtype;
  int out_chunk;  // rows per output chunk; 0 = sq
  int64_t out_hs, out_cs, out_rs;
  float* lse;
  int64_t lse_hs;
  int64_t lse_cs = 0;  // floats between output chunks (LSE riding the output all-to-all)
  // Peer-memory output reshard: chunk t (rows [t*out_chunk, ...)) is written at out_peer[t]
  // (+ head * out_hs + row % out_chunk * out_rs) -- Ulysses member t's window, mapped here --
  // instead of out + t * out_cs; LSE likewise at lse_peer[t].  0: the strided form.
  int peer_chunks = 0;
  void* out_peer[kMaxPeerChunks] = {};
  float* lse_peer[kMaxPeerChunks] = {};
  const float* acc_o;    // merge into (acc_o, acc_lse) when non-null
  const float* acc_lse;
  void* split_ws;        // stream-K partial slots (attention_workspace_bytes)
  size_t split_ws_bytes;
  uint32_t* split_counters;    // stream-K tickets (attention_counter_words): zero-initialised,
  size_t split_counter_words;  // never written by anything else
  int max_ctas;  // persistent grid cap (0 = every SM): leaves SMs to a concurrent transfer
  const int* q_exp = nullptr;  // per-head range-guard exponents (StageOp.exps) or null
  const int* k_exp = nullptr;
  const int* v_exp = nullptr;
  // D != 128 (attention_generic.cu, CUDA cores in f32): operand dtypes F32 / F16 / BF16 each
  int k_dtype = -1;            // -1: qk_dtype
  int v_dtype = FUSP_F16;
};
// D = 128: the tcgen05 kernels; any other D (a multiple of 8 up to 256): launch_attention_generic.
fusp_status launch_attention(const AttnLaunch& a, cudaStream_t stream);
fusp_status launch_attention_generic(const AttnLaunch& a, cudaStream_t stream);
// Workspace the persistent attention kernel needs for a (heads, sq, skv) problem (0 when the
// q-blocks are scheduled whole).
size_t attention_workspace_bytes(int heads, int sq, int skv);
size_t attention_counter_words(int heads, int sq);
int sm_count();  // SMs of the current device (cached)
// Tuning/test knob: schedule 0 = auto, 1 = whole q-blocks, 2 = stream-K split; max_ctas 0 =
// every SM (a smaller grid leaves SMs to concurrent NCCL kernels).
void set_attention_schedule(int mode, int max_ctas);
// Debug: enable per-CTA globaltimer tracing of attention launches / copy the last trace out.
int attention_trace(int enable, unsigned long long* host, size_t n);
// Zero-initialised counter buffer that only grows (never during graph capture).
struct CounterBuf {
  uint32_t* ptr = nullptr;
  size_t words = 0;
  int device = -1;
};
// Growth is stream-ordered on `s` (cudaFreeAsync / cudaMallocAsync / cudaMemsetAsync): never a
// device-wide wait -- with peer windows, ranks sharing a GPU have exchange kernels spinning on
// it for work another rank's thread has not enqueued yet.  The caller guarantees the old buffer's
// users are ordered before `s`.
fusp_status ensure_counters(CounterBuf& b, size_t words, cudaStream_t s = nullptr);

// ---- elementwise / data-movement kernels (kernels.cu) -----------------------------------
fusp_status launch_convert(const void* x, int x_dtype, void* y, int y_dtype, int64_t n,
                           cudaStream_t s);
fusp_status launch_encode(const float* x, int64_t n, uint8_t* codes, cudaStream_t s);
fusp_status launch_decode(const uint8_t* c, int64_t n, float* y, cudaStream_t s);
// amax over n elements of x (any float dtype) into *amax_bits (u32 float bits, atomicMax),
// sets *nonfinite = 1 on NaN/Inf.  The buffer must be zeroed first (done by launch_amax).
fusp_status launch_amax(const void* x, int dtype, int64_t n, uint32_t* amax_bits,
                        uint32_t* nonfinite, cudaStream_t s);
// scale = amax/448 (1 if 0) from amax_bits; codes = RNE(x/scale)
fusp_status launch_quantize(const void* x, int dtype, int64_t n, const uint32_t* amax_bits,
                            float* scale_out, uint8_t* codes, cudaStream_t s);
fusp_status launch_dequantize(const uint8_t* codes, const float* scale, int64_t n, void* y,
                              int y_dtype, cudaStream_t s);
fusp_status launch_merge(const float* o1, const float* l1, const float* o2, const float* l2,
                         int64_t rows, int d, float* out, float* lse, cudaStream_t s);
fusp_status launch_fill(void* p, int dtype, int64_t n, float value, cudaStream_t s);

// Ulysses pack: src [B][H][SL][D] (dtype src_dt) -> dst [U][B][hp][SL][D] (dst_dt), slot-major.
struct PackDesc {
  const void* src;
  int src_dtype;
  void* dst;
  int dst_dtype;
  int64_t dst_slot_stride;  // elements (or bytes for e4m3) between destination slots
  int b, h, sl, d, u;
  const float* scale;       // e4m3: quantization scale(s) (device)
  int64_t scale_bh_stride;  // 0: one tensor-wide scale; 1: one scale per (b,h) slab
  const uint32_t* amax_bits = nullptr;  // e4m3: scales from amax words instead (amax/448)
  float* trailer = nullptr;             // e4m3: write each slot's scales (slot t at t*trailer_stride)
  int64_t trailer_stride = 0;           // floats
};
fusp_status launch_pack(const PackDesc& p, cudaStream_t s);
// Up to 6 packs / unpacks with one launch (same B, H, SL, D, U; else one launch each).
// pdl: launched as a programmatic dependent of the previous kernel (the FP8 amax pass): only
// the E4M3 operands wait for it (griddepcontrol.wait), plain copies run alongside.
// peer_slot_boff (peer-memory Ulysses): slot t is peer_slot_boff[t] bytes from slot 0 (member
// t's window) instead of t * dst_slot_stride; every CTA fences system-wide before it exits.
fusp_status launch_pack_multi(const PackDesc* ps, int n, cudaStream_t s, bool pdl = false,
                              const int64_t* peer_slot_boff = nullptr);
// The FP8 input reshard's amax + pack as ONE cooperative launch (pack_fp8_fused_kernel) when
// ps = {Q plain 16-bit, K E4M3, V E4M3} with per-tensor scales fit the grid's registers and the
// stream is not capturing; amax[p] (and amax[0][1], the barrier) zero on entry and on exit,
// scales[p] receive the K / V scales.  *done = false: nothing launched, use the two passes.
fusp_status try_pack_fp8_fused(const PackDesc* ps, uint32_t* const* amax, float* const* scales,
                              const int64_t* peer_slot_boff, cudaStream_t s, bool* done);
// Fused QK RMSNorm (w != null) + interleaved RoPE (cosv != null, rows pos0 + s) + pack into
// slot t = h / (H/u) at t * slot_stride elements (u = 1: plain [B][H][SL][D] output).
// One operand of a batched prologue pack (w / cos / sin null = that step skipped).
struct ProPack {
  const void* src;
  void* dst;
  const float* w;
  const float* cosv;
  const float* sinv;
  int sdt, ddt;
};
fusp_status launch_norm_rope_pack_multi(const ProPack* ops, int n, int64_t slot_stride, int b,
                                        int h, int sl, int d, int u, float eps, int64_t pos0,
                                        cudaStream_t s,
                                        const int64_t* peer_slot_boff = nullptr);
fusp_status launch_norm_rope_pack(const void* src, int sdt, void* dst, int ddt,
                                  int64_t slot_stride, int b, int h, int sl, int d, int u,
                                  const float* w, float eps, const float* cosv, const float* sinv,
                                  int64_t pos0, cudaStream_t s,
                                  const int64_t* peer_slot_boff = nullptr);
// Ulysses unpack: src slots [U][B][hp][SL][D] -> dst [B][hp][U*SL][D]; e4m3 src uses per-slot
// scales scale[j] (device) -- value = decode(code) * scale[j] in f32, then cast to dst dtype.
struct UnpackDesc {
  const void* src;
  int src_dtype;
  int64_t src_slot_stride;
  const float* scales;       // [U] for e4m3
  int64_t scale_stride;      // floats between consecutive slot scale arrays
  int64_t scale_bh_stride;   // 0: one scale per slot; 1: one per (b,h) slab inside the slot
  void* dst;
  int dst_dtype;
  int b, hp, sl, d, u;
};
fusp_status launch_unpack(const UnpackDesc& p, cudaStream_t s);
fusp_status launch_unpack_multi(const UnpackDesc* us, int n, cudaStream_t s);
// Output unpack for B>1: src slots [U][B][hp][SL][D] -> dst [B][H][SL][D].
fusp_status launch_unpack_heads(const void* src, int64_t slot_stride, void* dst, int dtype, int b,
                                int hp, int sl, int d, int u, cudaStream_t s);

size_t dtype_size(int dt);

// ---- operand staging (kernels.cu) --------------------------------------------------------
// The tensor-core operands of the attention kernel are bf16 (Q, K of bf16 inputs) or f16.  f16
// has 5 exponent bits, so every staging pass INTO f16 from a wider-range source (f32, bf16, or
// decode(code) * scale of an FP8 chunk) is range-guarded: it records max|x| per head, and a
// head whose maximum falls outside [2^-6, 2^15) is stored as x * 2^-e with the power of two
// e = exps[head] chosen so that max|x| * 2^-e lies in [2^14, 2^15) -- exact scaling, no
// overflow to inf, no loss to f16 subnormals.  The attention kernel folds 2^(eq + ek) into
// its softmax scale and 2^ev into the output, so results are the unscaled ones.  The decision
// needs the whole head's maximum: the staging kernel converts with e = 0 and folds max|x| into
// a per-(op, head) word (one relaxed atomic per warp); a small per-head kernel then sets
// exps[head], resets the word and, only when e != 0, rewrites that head (the rare path; one
// CTA per affected head, heads in parallel).
//
// Layout (the Ulysses unpack; u = 1 is plain staging of a [bhp][sl][d] tensor): slab (j, bh)
// of the source, at src + j * src_slot_stride + bh * sl * d, lands at rows [j*sl, (j+1)*sl)
// of operand slab bh: dst + (bh * u + j) * sl * d.
constexpr int kGuardExpMin = -40, kGuardExpMax = 60;  // clamp (eq + ek, ev stay normal f32)
struct StageOp {
  const void* src;
  int sdt;                  // F32 / BF16 / F16 / E4M3
  int64_t src_slot_stride;  // source elements (bytes for e4m3) between slots j
  const float* scales;      // e4m3: value = decode(c) * scales[j * scale_stride + bh * scale_bh_stride]
  int64_t scale_stride, scale_bh_stride;
  void* dst;                // operand in ddt (F16 / BF16 / F32), or null (raw only)
  int ddt;
  void* raw;                // optional: the source bytes unchanged, in operand layout
  int* exps;                // non-null: guarded f16 destination, per-bh exponent out
  uint32_t* words;          // guarded: bhp zero-initialised words (max|x| bits), left zeroed
  // Layout overrides (elements; 0 = the unpack layout above): slab (j, bh) reads
  // src + j * src_slot_stride + bh * src_bh_stride and writes dst/raw + j * dst_slot_stride +
  // bh * dst_bh_stride.  The inverse mapping (operand rows -> slots) is the output-reshard pack.
  int64_t src_bh_stride = 0, dst_slot_stride = 0, dst_bh_stride = 0;
};
constexpr int kMaxStageOps = 6;
fusp_status launch_stage(const StageOp* ops, int n, int bhp, int sl, int d, int u, cudaStream_t s);
// zeroed words one guarded StageOp needs
inline size_t stage_words(int bhp) { return 2 * static_cast<size_t>(bhp); }

// FP8 helpers for the protocols (blocked quantizer; one block = per-tensor reference mode).
// Source of the values to quantize: a float tensor (dt = F32/F16/BF16), or an E4M3 chunk
// [bh][span][d] whose value is decode(code) * scales[(row/seg_rows)*seg_stride + bh*bh_stride].
struct Fp8Src {
  const void* x;
  int dt;
  const float* scales;
  int64_t seg_stride, bh_stride;
  int d, span, seg_rows;
};
// amax words of 1-2 sources (K, V) in one launch (zeroed first; no finalize: the pack reads
// the words and computes amax/448 itself).
fusp_status launch_amax_multi(const Fp8Src* src, int parts, int64_t block_elems, int nblocks,
                              uint32_t* const* amax, cudaStream_t s);
fusp_status launch_amax_blocks_raw(const Fp8Src& src, int64_t block_elems, int nblocks,
                                   uint32_t* amax, cudaStream_t s);
// amax per block of `block_elems` (into work[0..nblocks)), then work[k] = scale bits.
fusp_status launch_amax_blocks(const Fp8Src& src, int64_t block_elems, int nblocks,
                               uint32_t* work, uint32_t* nonfinite, cudaStream_t s);
fusp_status launch_quantize_blocks(const Fp8Src& src, int64_t n, int64_t block_elems,
                                   const float* scales, uint8_t* codes, cudaStream_t s);
// amax + scales + codes in one call; `work` holds >= nblocks + 1 ZERO words (left zero).
fusp_status launch_quantize_fp8(const Fp8Src& src, int64_t n, int64_t block_elems, uint32_t* work,
                                float* scales, uint8_t* codes, uint32_t* nonfinite,
                                cudaStream_t s);
// Pass 1 of the quantizer for 1-2 sources (K, V) in one launch: per-block amax into the ZERO
// words work[p][0..nblocks) (work[0][nblocks] is the launch's ticket, so work[1] starts past
// it); the last CTA writes scales[p][blk] = amax / 448 (1 if 0) and zeroes the words again.
fusp_status launch_amax_scales(const Fp8Src* src, int parts, int64_t block_elems, int nblocks,
                               uint32_t* const* work, float* const* scales, uint32_t* nonfinite,
                               cudaStream_t s);
// K and V (parts = 2) quantized with one amax launch (scales finalized in it) and one quantize
// launch (its programmatic dependent).  `work` as for launch_amax_scales.  one_launch: per-tensor
// scales on tensors that fit one resident wave's registers run as ONE cooperative launch
// (quantize_fused_kernel) -- which needs the whole GPU free to start, so callers running
// beside another kernel (the pipelined ring's side stream, beside the attention) pass false
// and keep the two passes, which fill whatever SMs the compute leaves free.
fusp_status launch_quantize_fp8_multi(const Fp8Src* src, int parts, int64_t n, int64_t block_elems,
                                      uint32_t* const* work, float* const* scales,
                                      uint8_t* const* codes, uint32_t* nonfinite, cudaStream_t s,
                                      bool one_launch = true);
fusp_status launch_dequantize_blocks(const uint8_t* c, const float* scales, int64_t block_elems,
                                     int64_t n, void* y, int ydt, cudaStream_t s);
// Ring forward of an E4M3 chunk that quantize produced as a whole: scales[i] <- RN(RN(448 s) /
// 448) in place for `parts` trailers of n scales (the codes are unchanged; see usp.cpp ring()).
fusp_status launch_fp8_forward_scales(float* const* scales, int parts, int n, cudaStream_t s);
fusp_status launch_scatter_slot_scales(const float* scales, float* base, int64_t slot_stride_f,
                                       int b, int h, int u, int per_block, cudaStream_t s);
fusp_status launch_finite(const void* x, int dt, int64_t n, uint32_t* flag, cudaStream_t s);

}  // namespace fusp
