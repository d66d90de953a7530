/* fastusp -- B200-native USP (Ulysses x Ring) joint-attention layer, C ABI.
 *
 * Drop-in for the reference's uspsim USP attention API
 * (/root/reference/proj/include/uspsim/protocols.hpp, tensor.hpp, fp8.hpp, mesh.hpp).
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers unless a function says "_host".
 *  - Tensors are dense [B,H,S,D], row-major, d fastest (= uspsim::Tensor4T, tensor.hpp:29-61).
 *  - Every function returns fusp_status; the message of the last failure on the calling
 *    thread is fusp_last_error() (same text as the reference exception's what()).
 *  - Stream-ordered: functions enqueue on `stream` and return; they do not synchronize
 *    unless documented (options.check_finite, the _host variants).
 *  - Collective functions (usp/ulysses/ring) must be called by every rank of the mesh in
 *    the same order, like uspsim::run_protocol programs (fabric.cpp:211-213) and NCCL.
 */
#ifndef FASTUSP_H_
#define FASTUSP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fusp_stream_t; /* == cudaStream_t; NULL = legacy default stream */

/* Status codes map 1:1 onto the reference's exception classes. */
typedef enum {
  FUSP_OK = 0,
  FUSP_ERR_SHAPE = 1,            /* uspsim::ShapeError           tensor.hpp:13-16  */
  FUSP_ERR_MESH = 2,             /* uspsim::MeshError            mesh.hpp:17-20    */
  FUSP_ERR_COMM = 3,             /* uspsim::FabricError          fabric.hpp:106    */
  FUSP_ERR_INVALID_ARGUMENT = 4, /* std::invalid_argument (non-finite input) protocols.cpp:103, fp8.cpp:112 */
  FUSP_ERR_DEADLOCK = 5,         /* uspsim::DeadlockError        fabric.hpp:112    */
  FUSP_ERR_CUDA = 10,
  FUSP_ERR_NCCL = 11,
  FUSP_ERR_OOM = 12,
  FUSP_ERR_UNSUPPORTED = 13
} fusp_status;

typedef enum { FUSP_F32 = 0, FUSP_F16 = 1, FUSP_BF16 = 2, FUSP_E4M3 = 3 } fusp_dtype;

/* = uspsim::Shape4 (tensor.hpp:18-26) */
typedef struct {
  int64_t b, h, s, d;
} fusp_shape4;

/* = uspsim::CommOptions (protocols.hpp:12-15) plus B200 extensions. */
typedef struct {
  int fp8_kv;         /* quantize K/V payloads (scale + E4M3 codes), protocols.hpp:13 */
  int pipelined_ring; /* double-buffered ring on a side stream, protocols.hpp:14 */
  int out_dtype;      /* fusp_dtype of the layer output (F32 = reference) */
  int check_finite;   /* 1: validate inputs like check_local_qkv (protocols.cpp:97-105); syncs */
  int fp8_block;      /* 0 = per-tensor scale (reference); 1 = one scale per (b,h) head slab */
} fusp_comm_options;

const char* fusp_last_error(void);
const char* fusp_version(void);
/* Number of fastusp CUDA kernels launched so far by this process (all devices). */
uint64_t fusp_kernel_launch_count(void);
/* Tuning knob (no reference counterpart): attention work schedule, 0 = auto, 1 = whole
 * 256-row q-blocks per CTA, 2 = stream-K split of (q-block x KV tile) units over the SMs,
 * 3 = aligned split (equal KV segments per q-block), 4 = KV-split CTAs (whole 128-row Q tiles,
 * the two softmax warpgroups splitting the KV range; auto picks it for one-wave shapes),
 * 5 = KV-split CTAs with stream-K over the 128-row tiles (every SM busy);
 * max_ctas caps the persistent grid (0 = every SM; leave SMs free for concurrent NCCL). */
fusp_status fusp_attention_schedule(int mode, int max_ctas);
/* Debug timeline (no reference counterpart): enable != 0 records per-CTA globaltimer events
 * of subsequent attention launches; copies up to n u64 events of the last launch to host
 * (layout: 72 per CTA = start, end, [8 segments][2 Q tiles][start, first S, O done, stored]).
 * Returns the number copied; -2 in the shipped library, where the tracing is compiled out (a
 * debug build: nvcc -DFUSP_TRACE_BUILD=1, tools/build_variants.sh trace:-DFUSP_TRACE_BUILD=1). */
int fusp_attention_trace(int enable, uint64_t* host, size_t n);

/* ---- FP8 E4M3 codec (fp8.hpp:23-49) ---------------------------------------------------- */
/* encode_e4m3 (fp8.cpp:45-68), elementwise: f32 -> code.  Bit-exact. */
fusp_status fusp_encode_e4m3(const float* x, int64_t n, uint8_t* codes, fusp_stream_t stream);
/* decode_e4m3 (fp8.cpp:39-43), elementwise: code -> f32 (NaN codes -> NaN). */
fusp_status fusp_decode_e4m3(const uint8_t* codes, int64_t n, float* y, fusp_stream_t stream);
/* quantize (fp8.cpp:107-123): *scale_dev = max|x|/448 (1 if all zero), codes = RNE(x/scale).
 * x dtype F32/F16/BF16.  Bit-exact codes and scale.  Non-finite input -> FUSP_ERR_INVALID_ARGUMENT
 * (synchronizes to report it; pass check_finite=0 to skip the check and stay async). */
fusp_status fusp_quantize_e4m3(const void* x, fusp_dtype dtype, int64_t n, uint8_t* codes,
                               float* scale_dev, int check_finite, fusp_stream_t stream);
/* Per-block variant (B200 extension; SPEC.md:167 makes per-block a reference non-goal): every
 * run of `block` consecutive elements is quantized exactly as uspsim::quantize would quantize
 * that slice alone -> scales_dev[n / block].  block = n is the reference's per-tensor case. */
fusp_status fusp_quantize_e4m3_blocks(const void* x, fusp_dtype dtype, int64_t n, int64_t block,
                                      uint8_t* codes, float* scales_dev, fusp_stream_t stream);
fusp_status fusp_dequantize_e4m3_blocks(const uint8_t* codes, const float* scales_dev, int64_t n,
                                        int64_t block, void* y, fusp_dtype dtype,
                                        fusp_stream_t stream);
/* Ring-hop re-quantization (protocols.cpp:113-115, 309-310): quantize(dequantize(chunk)) where
 * every run of `seg` consecutive codes carries its own scale seg_scales_dev[i / seg] (the
 * resharded chunk holds rows from several senders) -> one scale *scale_dev and codes_out.
 * Bit-exact with uspsim::quantize of the dequantized f32 values; seg % 8 == 0, n % seg == 0. */
fusp_status fusp_requantize_e4m3(const uint8_t* codes, const float* seg_scales_dev, int64_t n,
                                 int64_t seg, uint8_t* codes_out, float* scale_dev,
                                 fusp_stream_t stream);
/* dequantize (fp8.cpp:125-130): y = decode(code) * (*scale_dev), written as `dtype`. */
fusp_status fusp_dequantize_e4m3(const uint8_t* codes, const float* scale_dev, int64_t n, void* y,
                                 fusp_dtype dtype, fusp_stream_t stream);

/* ---- single-GPU attention numerics (tensor.hpp:91-98) ----------------------------------- */
/* attention_with_lse (tensor.cpp:193-202): q [B,H,Sq,D], k,v [B,H,Skv,D], all `in_dtype`
 * (F32/BF16/F16; Q.K^T in bf16 for bf16 inputs, f16 otherwise, P.V in f16, f32 accumulation;
 * every f16 staging range-guarded per head by an exact power of two).
 * out [B,H,Sq,D] in out_dtype; lse [B,H,Sq] f32 natural log (nullable). Skv = 0 gives
 * out = 0, lse = -inf (tensor.cpp:161-164).  D = 128 runs on the tcgen05 kernel; any other D
 * that is a multiple of 8 (up to 256) on an f32 CUDA-core kernel (the protocols below too). */
fusp_status fusp_attention_with_lse(const void* q, const void* k, const void* v,
                                    fusp_dtype in_dtype, fusp_shape4 q_shape, int64_t skv,
                                    void* out, fusp_dtype out_dtype, float* lse,
                                    fusp_stream_t stream);
/* Same, with the operand dtypes the tensor cores consume given separately: Q,K in qk_dtype
 * (BF16 or F16) and V in v_dtype (F16 runs with no staging pass at all). */
fusp_status fusp_attention_with_lse_ex(const void* q, const void* k, const void* v,
                                       fusp_dtype qk_dtype, fusp_dtype v_dtype,
                                       fusp_shape4 q_shape, int64_t skv, void* out,
                                       fusp_dtype out_dtype, float* lse, fusp_stream_t stream);
/* Range-guarded f16 staging of a tensor-core operand (B200 extension; what every
 * fusp_attention* / protocol call does to f32, bf16 and FP8-decoded operands internally):
 * x [heads][rows][128] (F32/BF16/F16) -> y f16 = x * 2^-exps[h], exps[heads] int32 out, with
 * exps[h] = 0 while max|x[h]| lies in [2^-6, 2^15), else the power of two that brings it into
 * [2^14, 2^15) (see fastusp_internal.h).  Exact power-of-two scaling: no inf, no f16 subnormal. */
fusp_status fusp_stage_f16(const void* x, fusp_dtype dtype, int64_t heads, int64_t rows, void* y,
                           int* exps, fusp_stream_t stream);
/* merge_lse (tensor.cpp:204-243): f32 o1,o2 [B,H,S,D], l1,l2 [B,H,S] -> out, lse (may alias o1/l1). */
fusp_status fusp_merge_lse(const float* o1, const float* l1, const float* o2, const float* l2,
                           fusp_shape4 shape, float* out, float* lse, fusp_stream_t stream);

/* ---- mesh (mesh.hpp:27-50) -------------------------------------------------------------- */
/* build_mesh (mesh.cpp:57-79): largest feasible R <= max_ring with n%R==0 and heads%(n/R)==0. */
fusp_status fusp_mesh_build(int n, int max_ring_dim_size, int heads, int* r, int* u);
/* make_mesh (mesh.cpp:34-55): ulysses_groups [R][U], ring_groups [U][R] (rank = ring*U + uly). */
fusp_status fusp_mesh_make(int n, int r, int* ulysses_groups, int* ring_groups);

/* ---- per-rank context (replaces uspsim::WorkerContext, fabric.hpp:136-166) --------------- */
typedef struct fusp_fabric_s* fusp_fabric; /* in-process fabric: threads as ranks (fabric.cpp:280) */
typedef struct fusp_ctx_s* fusp_ctx;

fusp_status fusp_fabric_create(int world, fusp_fabric* out);
fusp_status fusp_fabric_destroy(fusp_fabric f);
/* A rank of an in-process fabric; `device` may be shared by several ranks (tests). */
fusp_status fusp_ctx_create_local(fusp_fabric f, int rank, int device, fusp_ctx* out);
/* One process (or thread) per GPU over NCCL; uid from fusp_nccl_unique_id on one rank. */
fusp_status fusp_nccl_unique_id(uint8_t uid[128]);
fusp_status fusp_ctx_create_nccl(const uint8_t uid[128], int world, int rank, int device,
                                 fusp_ctx* out);
fusp_status fusp_ctx_destroy(fusp_ctx ctx);
/* Wait for `stream` on the host, bounded: the NCCL backend polls ncclCommGetAsyncError while
 * the stream drains, and a peer that failed or never joined its collective (or timeout_s
 * elapsing; <= 0: FUSP_TIMEOUT_S, default 120) aborts every communicator of the context and
 * returns FUSP_ERR_DEADLOCK ("deadlock: rank R ...", DeadlockError, fabric.hpp:106-126)
 * instead of hanging.  Later collectives on an aborted context return FUSP_ERR_COMM. */
fusp_status fusp_ctx_synchronize(fusp_ctx ctx, fusp_stream_t stream, double timeout_s);
int fusp_ctx_rank(fusp_ctx ctx);
int fusp_ctx_world(fusp_ctx ctx);
/* Bytes this rank put on the wire since creation, self-traffic excluded, per op:
 * = TrafficLog::bytes_for("all_to_all"|"send", rank) (fabric.cpp:44-49). */
fusp_status fusp_ctx_traffic(fusp_ctx ctx, uint64_t* all_to_all_bytes, uint64_t* send_bytes);
fusp_status fusp_ctx_reset_traffic(fusp_ctx ctx);
/* TrafficLog::to_json (fabric.cpp:72-87): [{"op","group","round","rank","bytes","msgs"}, ...]
 * in (op, group, round, rank) order.  Writes at most cap bytes (NUL-terminated), *len = size. */
fusp_status fusp_ctx_traffic_json(fusp_ctx ctx, char* buf, size_t cap, size_t* len);
/* Timeline::to_json (fabric.cpp:115-125) of the last layer call, protocol event order, plus
 * "t_ms": device time of the event from the first one (CUDA events on both streams). */
fusp_status fusp_ctx_timeline_json(fusp_ctx ctx, char* buf, size_t cap, size_t* len);
/* Debug (no reference counterpart): enable != 0 keeps a device copy of every payload this
 * rank puts on the wire in later eager calls -- kind 0: the Ulysses-in send slots (all U
 * slots, slot stride apart), kind 1 / 2: the ring K / V part of hop `round` -- so tests can
 * compare FP8 codes and scale trailers byte for byte with the reference quantizer.  Enabling
 * (or disabling) drops the records. */
fusp_status fusp_ctx_debug_wire(fusp_ctx ctx, int enable);
int fusp_ctx_debug_wire_count(fusp_ctx ctx);
fusp_status fusp_ctx_debug_wire_get(fusp_ctx ctx, int index, int* kind, int* round, void* host,
                                    size_t cap, size_t* bytes);
/* Per-step device timings of the last ring call (ms): compute[i], comm[i] for i < R. */
fusp_status fusp_ctx_ring_timings(fusp_ctx ctx, int max_steps, float* compute_ms, float* comm_ms,
                                  int* steps);

/* ---- peer-memory Ulysses transport (no reference counterpart: B200 / NVSwitch) ----------------
 * The reference moves the Ulysses payloads through its fabric (all_to_all, fabric.cpp:199-226);
 * with peer windows enabled, the two Ulysses reshards of usp_attention / ulysses_attention
 * (protocols.cpp:125-203) are fused into the kernels around them: the pack kernel stores every
 * member's slot straight into that member's window and the attention epilogue stores O (and the
 * LSE) rows straight into their owner's window, over NVLink / NVSwitch, each followed by one tiny
 * signal-and-wait kernel.  Results and TrafficLog bytes are identical to the comm path.  The
 * ring's hops (R > 1) go through the windows too (copies into the next member's ring buffers,
 * signals both ways) when the ring's members are separate processes or devices.  Windows
 * serve one Ulysses group and one ring group per context (the first layer's); other layers
 * (other groups, D != 128, wire debugging, shapes larger than a window) fall back to the
 * backend -- counted by fusp_ctx_peer_stats.  The fused QK RMSNorm + RoPE packs store into the
 * windows like the plain pack.  fusp_usp_block's QKV projection is the producer on this path: its
 * epilogue stores Q, K, V into the members' windows (GEMM and input all-to-all in one kernel),
 * and its output projection reads O where the members' epilogues stored it.  A peer-path layer
 * needs no host rendezvous, so it is graph-capturable on any context.
 * Every kernel of the library is loaded when the window is created (lazy module loading could
 * otherwise synchronise the context behind a spinning exchange).  Ranks that are threads of one
 * process sharing one device need a hardware queue per stream: CUDA_DEVICE_MAX_CONNECTIONS >=
 * 2 x those ranks, set before CUDA initialises; fusp_ctx_peer_open refuses (FUSP_ERR_UNSUPPORTED)
 * otherwise, since streams sharing a queue would wait behind another rank's spin.
 * fusp_ctx_peer_enable is collective over the world: every rank allocates `window_bytes` of
 * device memory (fusp_peer_window_bytes sizes it for a layer), the 128-byte handles are
 * all-gathered through the context's own backend and mapped (CUDA IPC between processes of one
 * node; the pointer itself between threads of one process). */
#define FUSP_PEER_HANDLE_BYTES 128
fusp_status fusp_ctx_peer_enable(fusp_ctx ctx, size_t window_bytes);
/* The same in two steps for callers with their own bootstrap: create this rank's window and
 * its handle; then map the world's handles (world x FUSP_PEER_HANDLE_BYTES, rank order). */
fusp_status fusp_ctx_peer_window(fusp_ctx ctx, size_t window_bytes, void* handle_out);
fusp_status fusp_ctx_peer_open(fusp_ctx ctx, const void* handles);
/* Window bytes one layer needs on every member (world ranks, mesh make_mesh(world, ring_dim)). */
fusp_status fusp_peer_window_bytes(int world, int ring_dim, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                   const fusp_comm_options* opts, size_t* bytes);
/* Drop the windows (waits for the context's device work): later layers use the backend again.
 * Collective in effect: every rank of a group must agree on the transport of each layer. */
fusp_status fusp_ctx_peer_disable(fusp_ctx ctx);
/* Layers whose Ulysses reshards used the windows / fell back to the backend since enabling. */
fusp_status fusp_ctx_peer_stats(fusp_ctx ctx, uint64_t* layers, uint64_t* fallbacks);

/* ---- distributed protocols (protocols.hpp:47-71) ------------------------------------------ */
/* usp_attention (protocols.cpp:321-340) on mesh make_mesh(world, ring_dim).
 * q,k,v: local shards [B,H,S/N,D] (in_dtype F32/BF16/F16); out: [B,H,S/N,D] in opts->out_dtype. */
fusp_status fusp_usp_attention(fusp_ctx ctx, int ring_dim, const void* q, const void* k,
                               const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                               void* out, const fusp_comm_options* opts, fusp_stream_t stream);
/* ulysses_attention (protocols.cpp:207-214) over the whole world. */
fusp_status fusp_ulysses_attention(fusp_ctx ctx, const void* q, const void* k, const void* v,
                                   fusp_dtype in_dtype, fusp_shape4 local_shape, void* out,
                                   const fusp_comm_options* opts, fusp_stream_t stream);
/* ring_attention_{serial,pipelined} (protocols.cpp:237-319) over the whole world:
 * out [B,H,S/N,D] in opts->out_dtype and lse [B,H,S/N] f32 (nullable). */
fusp_status fusp_ring_attention(fusp_ctx ctx, const void* q, const void* k, const void* v,
                                fusp_dtype in_dtype, fusp_shape4 local_shape, void* out,
                                float* lse, const fusp_comm_options* opts, fusp_stream_t stream);

/* usp_attention (protocols.cpp:321-340) that also returns the rows' natural-log LSE:
 * lse [B,H,S/N] f32 (nullable).  The reference drops it (protocols.cpp:339); here it rides a
 * second, small all-to-all back with the output ([B][H/U][S/N] f32 per member). */
fusp_status fusp_usp_attention_lse(fusp_ctx ctx, int ring_dim, const void* q, const void* k,
                                   const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                   void* out, float* lse, const fusp_comm_options* opts,
                                   fusp_stream_t stream);

/* ---- process groups (uspsim::ProcessGroup, fabric.hpp:20-28) ----------------------------- */
typedef struct fusp_group_s* fusp_group;
/* A group of world ranks members[0..n) in group order (position = index).  Collective over the
 * WORLD for NCCL contexts (one ncclCommSplit): every rank calls it, with the group it belongs
 * to (the groups of one call must be disjoint) or n = 0 to take part without a group (*out =
 * NULL).  Errors as validate_group (fabric.cpp:316-324) / all_to_all (:204-205): FUSP_ERR_COMM
 * "group member X out of range [0,N)", "duplicate member X in group K", "rank R not in group K". */
fusp_status fusp_group_create(fusp_ctx ctx, const int* members, int n, fusp_group* out);
fusp_status fusp_group_destroy(fusp_group group);
int fusp_group_size(fusp_group group);
int fusp_group_position(fusp_group group);
/* ulysses_attention(ctx, q, k, v, group, opts) (protocols.hpp:47-48, protocols.cpp:207-214)
 * over `group` (NULL = the world); lse [B,H,S/U,D...] -> [B,H,S/U] f32, nullable. */
fusp_status fusp_ulysses_attention_group(fusp_ctx ctx, fusp_group group, const void* q,
                                         const void* k, const void* v, fusp_dtype in_dtype,
                                         fusp_shape4 local_shape, void* out, float* lse,
                                         const fusp_comm_options* opts, fusp_stream_t stream);
/* ring_attention_{serial,pipelined}(ctx, q, k, v, group, opts) (protocols.hpp:54-65) over
 * `group` (NULL = the world): out and lse [B,H,S/R] (lse nullable); opts->pipelined_ring. */
fusp_status fusp_ring_attention_group(fusp_ctx ctx, fusp_group group, const void* q, const void* k,
                                      const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                      void* out, float* lse, const fusp_comm_options* opts,
                                      fusp_stream_t stream);
/* detail::ulysses_input_reshard (protocols.hpp:81-83, protocols.cpp:125-180): local q, k, v
 * [B,H,S_l,D] -> q_out, k_out, v_out [B,H/U,U*S_l,D] in out_dtype (F32 = the reference's
 * Resharded; with opts->fp8_kv, K and V are the exact dequantized values decode(code)*scale). */
fusp_status fusp_ulysses_input_reshard(fusp_ctx ctx, fusp_group group, const void* q, const void* k,
                                       const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                       void* q_out, void* k_out, void* v_out, fusp_dtype out_dtype,
                                       const fusp_comm_options* opts, fusp_stream_t stream);
/* detail::ulysses_output_reshard (protocols.hpp:85-86, protocols.cpp:182-203):
 * o [B,H/U,S,D] (o_shape) -> out [B,H,S/U,D], same dtype. */
fusp_status fusp_ulysses_output_reshard(fusp_ctx ctx, fusp_group group, const void* o,
                                        fusp_dtype dtype, fusp_shape4 o_shape, void* out,
                                        fusp_stream_t stream);

/* Producer prologue fused into the Ulysses pack (B200 extension): the MMDiT
 * joint-attention block's per-head RMSNorm of Q and K and rotary embedding, applied to the
 * caller's projected rows on their way into the all-to-all slot, instead of as separate
 * kernels before fusp_usp_attention.  Per row x of D = 128 elements at sequence position p:
 *   y = x * rsqrt(mean(x^2) + eps) * w          (w = q_norm_weight / k_norm_weight; NULL = skip)
 *   (y[2i], y[2i+1]) <- (y[2i] cos[p][i] - y[2i+1] sin[p][i], y[2i] sin[p][i] + y[2i+1] cos[p][i])
 * RoPE (rope_cos/rope_sin NULL = skip) applies to Q and K.  All arrays f32 on the device.
 * p = rope_pos0 + local row; rope_pos0 = -1 means rank * S_local (split_sequence order). */
typedef struct {
  const float* q_norm_weight; /* [D] */
  const float* k_norm_weight; /* [D] */
  float eps;
  const float* rope_cos;      /* [rope_rows][D/2] */
  const float* rope_sin;      /* [rope_rows][D/2] */
  int64_t rope_rows;
  int64_t rope_pos0;
} fusp_qk_prologue;
/* fusp_usp_attention with the fused prologue (prologue NULL = fusp_usp_attention). */
fusp_status fusp_usp_attention_ex(fusp_ctx ctx, int ring_dim, const void* q, const void* k,
                                  const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                  void* out, const fusp_comm_options* opts,
                                  const fusp_qk_prologue* prologue, fusp_stream_t stream);

/* The joint-attention block's output projection, the layer's consumer (no reference
 * counterpart): y[B][S][N] = O[B][H][S][128] (read as [B*S][H*128], the
 * layout the output reshard delivers) x W[H*128][N].  O and W both bf16 or both f16; y f32,
 * f16 or bf16; N a multiple of 64; 16-byte aligned pointers.  tcgen05 GEMM, stream-ordered. */
fusp_status fusp_out_projection(const void* o, fusp_dtype o_dtype, fusp_shape4 o_shape,
                                const void* w, int64_t n_out, void* y, fusp_dtype y_dtype,
                                fusp_stream_t stream);

/* fusp_usp_attention_ex followed by fusp_out_projection of its output on the same stream:
 * attn_out [B,H,S/N,128] (opts->out_dtype bf16 or f16) -> y [B,S/N,n_out] = attn_out x w_out. */
fusp_status fusp_usp_attention_proj(fusp_ctx ctx, int ring_dim, const void* q, const void* k,
                                    const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                    void* attn_out, const fusp_comm_options* opts,
                                    const fusp_qk_prologue* prologue, const void* w_out,
                                    int64_t n_out, void* y, fusp_dtype y_dtype,
                                    fusp_stream_t stream);

/* The whole MMDiT joint-attention block on this rank's tokens: QKV projection (tcgen05 GEMM,
 * x [batch][s_local][channels] x w_qkv [channels][3*heads*128], the QK RMSNorm + RoPE of
 * `prologue` in its epilogue) -> the USP layer -> output projection (w_out [heads*128][n_out])
 * -> y [batch][s_local][n_out].  x and both weights bf16 or f16 (the layer computes and
 * hands its output over in that dtype); rope_pos0 < 0 means rank * s_local. */
fusp_status fusp_usp_block(fusp_ctx ctx, int ring_dim, const void* x, fusp_dtype x_dtype,
                           int64_t batch, int64_t s_local, int64_t channels, const void* w_qkv,
                           int heads, const fusp_qk_prologue* prologue, const void* w_out,
                           int64_t n_out, void* y, fusp_dtype y_dtype,
                           const fusp_comm_options* opts, fusp_stream_t stream);

/* Host-buffer variant of fusp_usp_attention (the reference's calling convention: host
 * tensors in, host tensor out).  Copies H2D, runs, copies D2H, synchronizes. */
fusp_status fusp_usp_attention_host(fusp_ctx ctx, int ring_dim, const void* q, const void* k,
                                    const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                    void* out, const fusp_comm_options* opts,
                                    fusp_stream_t stream);

/* ---- CUDA Graph of the per-layer launch sequence (no reference counterpart) -------------- */
typedef struct fusp_graph_s* fusp_graph;
/* Captures `layers` back-to-back fusp_usp_attention calls (layer i reads q/k/v + i*layer_stride
 * bytes and writes out + i*out_stride bytes) into one CUDA graph. NCCL or world-1 contexts. */
fusp_status fusp_graph_capture_usp(fusp_ctx ctx, int ring_dim, const void* q, const void* k,
                                   const void* v, fusp_dtype in_dtype, fusp_shape4 local_shape,
                                   void* out, const fusp_comm_options* opts, int layers,
                                   int64_t in_layer_stride_bytes, int64_t out_layer_stride_bytes,
                                   fusp_stream_t stream, fusp_graph* graph);
/* The same for `layers` back-to-back fusp_usp_block calls (x / y of layer i at i * x_stride /
 * i * y_stride bytes): the whole MMDiT attention block -- QKV projection, the USP layer and the
 * output projection -- as one graph.  Runs layer 0 once eagerly to size the graph's own
 * workspace.  Capturable at world > 1 through NCCL or with peer windows (see above). */
fusp_status fusp_graph_capture_block(fusp_ctx ctx, int ring_dim, const void* x, fusp_dtype x_dtype,
                                     int64_t batch, int64_t s_local, int64_t channels,
                                     const void* w_qkv, int heads, const fusp_qk_prologue* prologue,
                                     const void* w_out, int64_t n_out, void* y, fusp_dtype y_dtype,
                                     const fusp_comm_options* opts, int layers, int64_t x_stride,
                                     int64_t y_stride, fusp_stream_t stream, fusp_graph* graph);
fusp_status fusp_graph_launch(fusp_graph graph, fusp_stream_t stream);
fusp_status fusp_graph_destroy(fusp_graph graph);

#ifdef __cplusplus
}
#endif
#endif /* FASTUSP_H_ */
