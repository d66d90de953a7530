// fastusp runtime: error state, TMA descriptor encoding, per-device scratch, and the
// single-GPU C-ABI entry points (codec, attention_with_lse, merge_lse, mesh).
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>
#include <string>
#include <vector>

#include "fastusp_internal.h"

namespace fusp {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

fusp_status set_error(fusp_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

fusp_status set_cuda_error(cudaError_t e, const std::string& where) {
  if (e == cudaErrorMemoryAllocation)
    return set_error(FUSP_ERR_OOM, where + ": " + cudaGetErrorString(e));
  return set_error(FUSP_ERR_CUDA, where + ": " + cudaGetErrorString(e));
}

void clear_error() { g_last_error.clear(); }

void count_launch(int n) { g_launches.fetch_add(static_cast<uint64_t>(n)); }

fusp_status ensure_smem_attr(const void* kernel, int bytes, const char* name) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;  // (kernel, device, bytes)
  int dev = 0;
  FUSP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(kernel, dev, bytes);
  if (done.count(key)) return FUSP_OK;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, std::string("cudaFuncSetAttribute(") + name + ")");
  done.insert(key);
  return FUSP_OK;
}

// With lazy module loading (CUDA_MODULE_LOADING=LAZY, the default since CUDA 12.2) the first
// launch of a kernel loads it, and loading may synchronize the whole context.  A rank whose
// peer-exchange kernel spins for another rank's signal (peer.cu) would then block every rank
// sharing the context that launches a kernel for the first time -- a deadlock when that
// launch is on the path to the awaited signal (ranks as threads of one process, or the
// side stream of one rank).  So every kernel of the library is loaded up front, before the
// first spinning kernel can exist (fusp_ctx_peer_window), once per device.
void append_kernels_kernels(std::vector<const void*>& v);
void append_kernels_attention(std::vector<const void*>& v);
void append_kernels_attention_generic(std::vector<const void*>& v);
void append_kernels_prologue(std::vector<const void*>& v);
void append_kernels_proj(std::vector<const void*>& v);
void append_kernels_peer(std::vector<const void*>& v);

fusp_status preload_kernels() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  FUSP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(dev)) return FUSP_OK;
  std::vector<const void*> ks;
  append_kernels_kernels(ks);
  append_kernels_attention(ks);
  append_kernels_attention_generic(ks);
  append_kernels_prologue(ks);
  append_kernels_proj(ks);
  append_kernels_peer(ks);
  for (const void* k : ks) {
    cudaFuncAttributes a{};
    FUSP_CUDA(cudaFuncGetAttributes(&a, k));
  }
  done.insert(dev);
  return FUSP_OK;
}

// ---- TMA ------------------------------------------------------------------------------
namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
}  // namespace

fusp_status encode_tmap(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
                        const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                        const cuuint32_t* elem_strides) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(FUSP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUresult r = enc(m, dt, static_cast<cuuint32_t>(rank), const_cast<void*>(base), dims, strides, box,
                   elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(FUSP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return FUSP_OK;
}

fusp_status make_tmap_rows(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int heads,
                           int rows, int64_t head_stride) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(FUSP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "attention operand not 16-byte aligned");
  cuuint64_t dims[3] = {128, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(heads)};
  cuuint64_t strides[2] = {128 * 2, static_cast<cuuint64_t>(head_stride) * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(FUSP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return FUSP_OK;
}

// ---- per-(device, stream) workspace of the context-free single-GPU API -------------------
// Every use of a workspace is ordered on its stream, and a call holds the workspace's mutex
// from handing out its pointers until its kernels are enqueued, so two host threads (or two
// streams) never share scratch words, and a buffer is only freed after its stream drained.
namespace {
struct StreamWs {
  std::mutex mu;
  void* ptr = nullptr;
  size_t bytes = 0;
  CounterBuf cnt;  // zero-initialised words (stream-K tickets, staging amax / tickets)
  CounterBuf qw;   // zero-initialised words of the FP8 amax pass (left zero by each launch)
  CounterBuf pc;   // projection GEMM stream-K tile counters (left zero by each launch)
  void* pslots = nullptr;  // projection GEMM stream-K partial slots
  size_t pbytes = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, std::unique_ptr<StreamWs>> g_ws;

fusp_status stream_ws(cudaStream_t s, StreamWs** out) {
  int dev = 0;
  FUSP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  auto& w = g_ws[{dev, s}];
  if (!w) w = std::make_unique<StreamWs>();
  *out = w.get();
  return FUSP_OK;
}

// Call with w->mu held.
fusp_status ws_scratch(StreamWs* w, cudaStream_t s, size_t bytes, void** out) {
  if (w->bytes < bytes) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    FUSP_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return set_error(FUSP_ERR_UNSUPPORTED, "workspace growth during graph capture");
    if (w->ptr) {
      FUSP_CUDA(cudaFreeAsync(w->ptr, s));  // the old buffer's last users ran on `s`
      w->ptr = nullptr;
      w->bytes = 0;
    }
    const size_t n = bytes < (size_t(1) << 20) ? (size_t(1) << 20) : bytes;
    FUSP_CUDA(cudaMallocAsync(&w->ptr, n, s));
    w->bytes = n;
  }
  *out = w->ptr;
  return FUSP_OK;
}

fusp_status ws_words(StreamWs* w, cudaStream_t s, size_t words, uint32_t** out) {
  if (w->cnt.words < words || w->cnt.ptr == nullptr) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    FUSP_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return set_error(FUSP_ERR_UNSUPPORTED, "workspace growth during graph capture");
  }
  FUSP_CHECK(ensure_counters(w->cnt, words, s));  // stream-ordered: the old words' users ran on s
  *out = w->cnt.ptr;
  return FUSP_OK;
}

fusp_status ws_qwords(StreamWs* w, cudaStream_t s, size_t words, uint32_t** out) {
  if (w->qw.words < words || w->qw.ptr == nullptr) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    FUSP_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      return set_error(FUSP_ERR_UNSUPPORTED, "workspace growth during graph capture");
  }
  FUSP_CHECK(ensure_counters(w->qw, words, s));
  *out = w->qw.ptr;
  return FUSP_OK;
}

std::string shape_str(const fusp_shape4& s) {
  std::ostringstream os;
  os << "[" << s.b << "," << s.h << "," << s.s << "," << s.d << "]";
  return os.str();
}

bool valid_float_dtype(int dt) { return dt == FUSP_F32 || dt == FUSP_F16 || dt == FUSP_BF16; }
}  // namespace

fusp_status with_proj_workspace(cudaStream_t s, size_t words, size_t bytes,
                                const std::function<fusp_status(uint32_t*, float*)>& launch) {
  StreamWs* w = nullptr;
  FUSP_CHECK(stream_ws(s, &w));
  std::lock_guard<std::mutex> lk(w->mu);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FUSP_CUDA(cudaStreamIsCapturing(s, &cs));
  // under capture: whole tiles (a graph must not address this stream's workspace, which a
  // later eager call may regrow)
  if (cs != cudaStreamCaptureStatusNone) return launch(nullptr, nullptr);
  FUSP_CHECK(ensure_counters(w->pc, words, s));
  if (w->pbytes < bytes) {
    if (w->pslots) FUSP_CUDA(cudaFreeAsync(w->pslots, s));  // its last users ran on `s`
    w->pslots = nullptr;
    w->pbytes = 0;
    FUSP_CUDA(cudaMallocAsync(&w->pslots, bytes, s));
    w->pbytes = bytes;
  }
  return launch(w->pc.ptr, static_cast<float*>(w->pslots));
}

}  // namespace fusp

using namespace fusp;

extern "C" {

const char* fusp_last_error(void) { return g_last_error.c_str(); }
const char* fusp_version(void) { return "fastusp 0.1 (sm_100a)"; }
uint64_t fusp_kernel_launch_count(void) { return g_launches.load(); }

int fusp_attention_trace(int enable, uint64_t* host, size_t n) {
  return attention_trace(enable, reinterpret_cast<unsigned long long*>(host), n);
}

fusp_status fusp_out_projection(const void* o, fusp_dtype o_dtype, fusp_shape4 o_shape,
                                const void* w, int64_t n_out, void* y, fusp_dtype y_dtype,
                                fusp_stream_t stream) {
  clear_error();
  if (o_shape.d != 128)
    return set_error(FUSP_ERR_SHAPE, "out projection: head dim D=" + std::to_string(o_shape.d) +
                                         " unsupported (D=128)");
  if (o_shape.b < 0 || o_shape.h < 0 || o_shape.s < 0 || n_out < 0 || o_shape.b * o_shape.s > (1 << 30) ||
      n_out > (1 << 30))
    return set_error(FUSP_ERR_SHAPE, "out projection: bad shape " + shape_str(o_shape));
  if (!valid_float_dtype(y_dtype))
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "out projection: bad output dtype");
  return launch_out_proj(o, o_dtype, static_cast<int>(o_shape.b), static_cast<int>(o_shape.h),
                         static_cast<int>(o_shape.s), w, static_cast<int>(n_out), y, y_dtype,
                         reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_attention_schedule(int mode, int max_ctas) {
  clear_error();
  if (mode < 0 || mode > 5 || max_ctas < 0)
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "attention schedule: mode in {0,...,5}, max_ctas >= 0");
  set_attention_schedule(mode, max_ctas);
  return FUSP_OK;
}

fusp_status fusp_encode_e4m3(const float* x, int64_t n, uint8_t* codes, fusp_stream_t stream) {
  clear_error();
  return launch_encode(x, n, codes, reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_decode_e4m3(const uint8_t* codes, int64_t n, float* y, fusp_stream_t stream) {
  clear_error();
  return launch_decode(codes, n, y, reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_quantize_e4m3(const void* x, fusp_dtype dtype, int64_t n, uint8_t* codes,
                               float* scale_dev, int check_finite, fusp_stream_t stream) {
  clear_error();
  if (!valid_float_dtype(dtype)) return set_error(FUSP_ERR_INVALID_ARGUMENT, "quantize: bad dtype");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StreamWs* w = nullptr;
  FUSP_CHECK(stream_ws(s, &w));
  std::lock_guard<std::mutex> lk(w->mu);
  void* ws = nullptr;
  FUSP_CHECK(ws_scratch(w, s, 256, &ws));
  uint32_t* amax = static_cast<uint32_t*>(ws);
  uint32_t* bad = amax + 1;
  if (n > 0 && n % 8 == 0 && n / 8 < (int64_t(1) << 31) &&
      (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(codes)) % 16 == 0) {
    // the vectorised per-tensor passes (one cooperative launch when the tensor fits the
    // grid's registers); the non-finite flag comes out of the same amax reduction
    uint32_t* work = nullptr;
    FUSP_CHECK(ws_qwords(w, s, 2, &work));
    const int rows = static_cast<int>(n / 8);
    const Fp8Src src{x, dtype, nullptr, 0, 0, 8, rows, rows};
    FUSP_CHECK(launch_quantize_fp8_multi(&src, 1, n, n, &work, &scale_dev, &codes, bad, s));
    if (check_finite) {
      uint32_t flag = 0;
      FUSP_CUDA(cudaMemcpyAsync(&flag, bad, 4, cudaMemcpyDeviceToHost, s));
      FUSP_CUDA(cudaStreamSynchronize(s));
      if (!flag) return FUSP_OK;
    } else {
      return FUSP_OK;
    }
  }
  FUSP_CHECK(launch_amax(x, dtype, n, amax, bad, s));
  if (check_finite) {
    uint32_t flag = 0;
    FUSP_CUDA(cudaMemcpyAsync(&flag, bad, 4, cudaMemcpyDeviceToHost, s));
    FUSP_CUDA(cudaStreamSynchronize(s));
    if (flag) {
      // locate the first non-finite element like the reference message (fp8.cpp:112-113)
      std::vector<float> hv;
      int64_t idx = -1;
      const size_t es = dtype_size(dtype);
      std::vector<uint8_t> raw(static_cast<size_t>(n) * es);
      FUSP_CUDA(cudaMemcpy(raw.data(), x, raw.size(), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n && idx < 0; ++i) {
        float f;
        if (dtype == FUSP_F32) {
          std::memcpy(&f, &raw[i * 4], 4);
        } else {
          uint16_t h;
          std::memcpy(&h, &raw[i * 2], 2);
          if (dtype == FUSP_BF16) {
            uint32_t u = uint32_t(h) << 16;
            std::memcpy(&f, &u, 4);
          } else {
            const bool exp_all = ((h >> 10) & 0x1F) == 0x1F;
            f = exp_all ? NAN : 0.f;
          }
        }
        if (!std::isfinite(f)) idx = i;
      }
      return set_error(FUSP_ERR_INVALID_ARGUMENT,
                       "quantize: non-finite element at flat index " + std::to_string(idx));
    }
  }
  return launch_quantize(x, dtype, n, amax, scale_dev, codes, s);
}

fusp_status fusp_quantize_e4m3_blocks(const void* x, fusp_dtype dtype, int64_t n, int64_t block,
                                      uint8_t* codes, float* scales_dev, fusp_stream_t stream) {
  clear_error();
  if (!valid_float_dtype(dtype)) return set_error(FUSP_ERR_INVALID_ARGUMENT, "quantize: bad dtype");
  if (block <= 0 || n % block != 0)
    return set_error(FUSP_ERR_SHAPE, "quantize: block " + std::to_string(block) +
                                         " does not divide " + std::to_string(n) + " elements");
  const int64_t nblocks = n / block;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StreamWs* w = nullptr;
  FUSP_CHECK(stream_ws(s, &w));
  std::lock_guard<std::mutex> lk(w->mu);
  uint32_t* work = nullptr;
  FUSP_CHECK(ws_qwords(w, s, static_cast<size_t>(nblocks) + 1, &work));
  // rows of 8 elements when they tile the blocks (the vectorised passes), else scalar
  const bool v8 = n % 8 == 0 && block % 8 == 0 && n / 8 < (int64_t(1) << 31);
  const int rows = v8 ? static_cast<int>(n / 8) : 1;
  const Fp8Src src{x, dtype, nullptr, 0, 0, v8 ? 8 : 1, rows, rows};
  return launch_quantize_fp8(src, n, block, work, scales_dev, codes, nullptr, s);
}

fusp_status fusp_requantize_e4m3(const uint8_t* codes, const float* seg_scales_dev, int64_t n,
                                 int64_t seg, uint8_t* codes_out, float* scale_dev,
                                 fusp_stream_t stream) {
  clear_error();
  if (seg <= 0 || seg % 8 != 0 || n % seg != 0 || n / 8 >= (int64_t(1) << 31))
    return set_error(FUSP_ERR_SHAPE, "requantize: segment " + std::to_string(seg) +
                                         " must be a multiple of 8 dividing " + std::to_string(n));
  if (n == 0) return FUSP_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StreamWs* w = nullptr;
  FUSP_CHECK(stream_ws(s, &w));
  std::lock_guard<std::mutex> lk(w->mu);
  uint32_t* work = nullptr;
  FUSP_CHECK(ws_qwords(w, s, 2, &work));
  // the ring-hop source: rows of 8 codes, one bh, a scale per `seg / 8` rows
  const Fp8Src src{codes, FUSP_E4M3, seg_scales_dev, 1, 0, 8, static_cast<int>(n / 8),
                   static_cast<int>(seg / 8)};
  return launch_quantize_fp8_multi(&src, 1, n, n, &work, &scale_dev, &codes_out, nullptr, s);
}

fusp_status fusp_dequantize_e4m3_blocks(const uint8_t* codes, const float* scales_dev, int64_t n,
                                        int64_t block, void* y, fusp_dtype dtype,
                                        fusp_stream_t stream) {
  clear_error();
  if (!valid_float_dtype(dtype)) return set_error(FUSP_ERR_INVALID_ARGUMENT, "dequantize: bad dtype");
  if (block <= 0) return set_error(FUSP_ERR_SHAPE, "dequantize: bad block");
  return launch_dequantize_blocks(codes, scales_dev, block, n, y, dtype,
                                  reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_dequantize_e4m3(const uint8_t* codes, const float* scale_dev, int64_t n, void* y,
                                 fusp_dtype dtype, fusp_stream_t stream) {
  clear_error();
  if (!valid_float_dtype(dtype)) return set_error(FUSP_ERR_INVALID_ARGUMENT, "dequantize: bad dtype");
  return launch_dequantize(codes, scale_dev, n, y, dtype, reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_attention_with_lse_ex(const void* q, const void* k, const void* v,
                                       fusp_dtype qk_dtype, fusp_dtype v_dtype, fusp_shape4 qs,
                                       int64_t skv, void* out, fusp_dtype out_dtype, float* lse,
                                       fusp_stream_t stream) {
  clear_error();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!valid_float_dtype(qk_dtype) || !valid_float_dtype(v_dtype) || !valid_float_dtype(out_dtype))
    return set_error(FUSP_ERR_INVALID_ARGUMENT, "attention: bad dtype");
  if (qs.b < 0 || qs.h < 0 || qs.s < 0 || qs.d <= 0 || skv < 0)
    return set_error(FUSP_ERR_SHAPE, "attention: bad shape " + shape_str(qs));
  const int64_t heads = qs.b * qs.h;
  const int64_t nq = heads * qs.s * qs.d;
  if (heads == 0 || qs.s == 0) return FUSP_OK;
  if (skv == 0) {  // merge identity: out 0, lse -inf (tensor.cpp:161-164)
    FUSP_CHECK(launch_fill(out, out_dtype, nq, 0.f, s));
    if (lse) FUSP_CHECK(launch_fill(lse, FUSP_F32, heads * qs.s, -INFINITY, s));
    return FUSP_OK;
  }
  if (qs.d != 128) {
    // other head dims: CUDA cores in f32, reading the caller's operands as they are
    AttnLaunch g{};
    g.q = q;
    g.k = k;
    g.v = v;
    g.qk_dtype = qk_dtype;
    g.k_dtype = qk_dtype;
    g.v_dtype = v_dtype;
    g.q_hs = qs.s * qs.d;
    g.k_hs = skv * qs.d;
    g.v_hs = skv * qs.d;
    g.heads = static_cast<int>(heads);
    g.sq = static_cast<int>(qs.s);
    g.skv = static_cast<int>(skv);
    g.d = static_cast<int>(qs.d);
    g.out = out;
    g.out_dtype = out_dtype;
    g.out_chunk = static_cast<int>(qs.s);
    g.out_hs = qs.s * qs.d;
    g.out_rs = qs.d;
    g.lse = lse;
    g.lse_hs = qs.s;
    return launch_attention_generic(g, s);
  }
  const int64_t nkv = heads * skv * qs.d;
  if (heads > 65535 / 1 || qs.s > (int64_t(1) << 30) || skv > (int64_t(1) << 30))
    return set_error(FUSP_ERR_SHAPE, "attention: shape too large " + shape_str(qs));
  // Operand staging: bf16 Q, K feed the bf16 MMA as they are; f16 operands too.  f32 Q, K run
  // the f16 MMA and any non-f16 V the f16 P.V MMA: one range-guarded staging pass each
  // (fastusp_internal.h), with per-head power-of-two exponents the kernel folds back in.
  const int qk_dt = qk_dtype == FUSP_BF16 ? FUSP_BF16 : FUSP_F16;
  const bool stage_qk = qk_dtype != qk_dt;
  const bool stage_v = v_dtype != FUSP_F16;
  const int nh = static_cast<int>(heads);
  const size_t split =
      attention_workspace_bytes(nh, static_cast<int>(qs.s), static_cast<int>(skv));
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t need = up(split) + up(sizeof(int) * 3 * heads);
  if (stage_qk) need += up(static_cast<size_t>(nq) * 2) + up(static_cast<size_t>(nkv) * 2);
  if (stage_v) need += up(static_cast<size_t>(nkv) * 2);
  StreamWs* w = nullptr;
  FUSP_CHECK(stream_ws(s, &w));
  std::lock_guard<std::mutex> lk(w->mu);
  uint8_t* ws = nullptr;
  FUSP_CHECK(ws_scratch(w, s, need, reinterpret_cast<void**>(&ws)));
  const size_t cnt_words = attention_counter_words(nh, static_cast<int>(qs.s));
  uint32_t* words = nullptr;
  FUSP_CHECK(ws_words(w, s, cnt_words + 3 * stage_words(nh), &words));
  size_t off = up(split);  // the stream-K workspace comes first
  int* exps = reinterpret_cast<int*>(ws + off);
  off += up(sizeof(int) * 3 * heads);
  const void* qb = q;
  const void* kb = k;
  const void* vh = v;
  uint32_t* sw = words + cnt_words;
  auto guarded = [&](const void* src, int sdt, void* dst, int part) {
    StageOp o{};
    o.src = src;
    o.sdt = sdt;
    o.dst = dst;
    o.ddt = FUSP_F16;
    o.exps = exps + part * heads;
    o.words = sw + part * stage_words(nh);
    return o;
  };
  StageOp kv[2];
  int nkv_ops = 0;
  if (stage_qk) {
    void* tq = ws + off;
    off += up(static_cast<size_t>(nq) * 2);
    void* tk = ws + off;
    off += up(static_cast<size_t>(nkv) * 2);
    const StageOp oq = guarded(q, qk_dtype, tq, 0);
    FUSP_CHECK(launch_stage(&oq, 1, nh, static_cast<int>(qs.s), 128, 1, s));
    kv[nkv_ops++] = guarded(k, qk_dtype, tk, 1);
    qb = tq;
    kb = tk;
  }
  if (stage_v) {
    void* tv = ws + off;
    kv[nkv_ops++] = guarded(v, v_dtype, tv, 2);
    vh = tv;
  }
  FUSP_CHECK(launch_stage(kv, nkv_ops, nh, static_cast<int>(skv), 128, 1, s));
  AttnLaunch a{};
  a.q = qb;
  a.k = kb;
  a.v = vh;
  a.qk_dtype = qk_dt;
  if (stage_qk) {
    a.q_exp = exps;
    a.k_exp = exps + heads;
  }
  if (stage_v) a.v_exp = exps + 2 * heads;
  a.q_hs = qs.s * 128;
  a.k_hs = skv * 128;
  a.v_hs = skv * 128;
  a.heads = nh;
  a.sq = static_cast<int>(qs.s);
  a.skv = static_cast<int>(skv);
  a.d = static_cast<int>(qs.d);
  a.out = out;
  a.out_dtype = out_dtype;
  a.out_chunk = static_cast<int>(qs.s);
  a.out_hs = qs.s * 128;
  a.out_cs = 0;
  a.out_rs = 128;
  a.lse = lse;
  a.lse_hs = qs.s;
  a.split_ws = split ? ws : nullptr;
  a.split_ws_bytes = split;
  a.split_counters = words;
  a.split_counter_words = cnt_words;
  return launch_attention(a, s);
}

fusp_status fusp_stage_f16(const void* x, fusp_dtype dtype, int64_t heads, int64_t rows, void* y,
                           int* exps, fusp_stream_t stream) {
  clear_error();
  if (!valid_float_dtype(dtype)) return set_error(FUSP_ERR_INVALID_ARGUMENT, "stage: bad dtype");
  if (heads < 0 || rows < 0 || heads > 65535 || rows > (int64_t(1) << 30))
    return set_error(FUSP_ERR_SHAPE, "stage: bad shape");
  if (heads == 0 || rows == 0) return FUSP_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StreamWs* w = nullptr;
  FUSP_CHECK(stream_ws(s, &w));
  std::lock_guard<std::mutex> lk(w->mu);
  uint32_t* words = nullptr;
  FUSP_CHECK(ws_words(w, s, stage_words(static_cast<int>(heads)), &words));
  StageOp o{};
  o.src = x;
  o.sdt = dtype;
  o.dst = y;
  o.ddt = FUSP_F16;
  o.exps = exps;
  o.words = words;
  return launch_stage(&o, 1, static_cast<int>(heads), static_cast<int>(rows), 128, 1, s);
}

fusp_status fusp_attention_with_lse(const void* q, const void* k, const void* v,
                                    fusp_dtype in_dtype, fusp_shape4 qs, int64_t skv, void* out,
                                    fusp_dtype out_dtype, float* lse, fusp_stream_t stream) {
  return fusp_attention_with_lse_ex(q, k, v, in_dtype, in_dtype, qs, skv, out, out_dtype, lse,
                                    stream);
}

fusp_status fusp_merge_lse(const float* o1, const float* l1, const float* o2, const float* l2,
                           fusp_shape4 shape, float* out, float* lse, fusp_stream_t stream) {
  clear_error();
  return launch_merge(o1, l1, o2, l2, shape.b * shape.h * shape.s, static_cast<int>(shape.d), out,
                      lse, reinterpret_cast<cudaStream_t>(stream));
}

fusp_status fusp_mesh_build(int n, int max_ring, int heads, int* r, int* u) {
  clear_error();
  if (n < 1) return set_error(FUSP_ERR_MESH, "worker count must be >= 1, got " + std::to_string(n));
  if (max_ring < 1)
    return set_error(FUSP_ERR_MESH,
                     "max_ring_dim_size must be >= 1, got " + std::to_string(max_ring));
  if (heads < 1) return set_error(FUSP_ERR_MESH, "head count must be >= 1, got " + std::to_string(heads));
  for (int rr = (n < max_ring ? n : max_ring); rr >= 1; --rr) {
    if (n % rr != 0 || heads % (n / rr) != 0) continue;
    *r = rr;
    *u = n / rr;
    return FUSP_OK;
  }
  std::ostringstream os;
  os << "no feasible (R,U) mesh for N=" << n << ", max_ring_dim_size=" << max_ring
     << ", H=" << heads << ":";
  for (int rr = 1; rr <= n; ++rr) {
    if (n % rr != 0) continue;
    os << " (R=" << rr << ",U=" << n / rr << ")";
    if (rr > max_ring) os << " violates R<=" << max_ring << ";";
    else os << " violates H%" << n / rr << "==0;";
  }
  return set_error(FUSP_ERR_MESH, os.str());
}

fusp_status fusp_mesh_make(int n, int r, int* ulysses_groups, int* ring_groups) {
  clear_error();
  if (n < 1) return set_error(FUSP_ERR_MESH, "worker count must be >= 1, got " + std::to_string(n));
  if (r < 1 || n % r != 0)
    return set_error(FUSP_ERR_MESH, "ring dimension " + std::to_string(r) +
                                        " does not divide worker count " + std::to_string(n));
  const int u = n / r;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < u; ++j) ulysses_groups[i * u + j] = i * u + j;
  for (int j = 0; j < u; ++j)
    for (int i = 0; i < r; ++i) ring_groups[j * r + i] = i * u + j;
  return FUSP_OK;
}

}  // extern "C"
