// star_api.cu -- the C ABI (include/star.h): host-side validation, TMA descriptor set-up,
// tile/split planning and kernel launches.  No compute happens on the host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "lenpred_kernels.cuh"
#include "star_internal.h"

namespace star {

int g_num_sms = 148;

static thread_local std::string t_err;

static star_status fail(star_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return st;
}

static star_status cuda_fail(cudaError_t e, const char* where) {
  return fail(STAR_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define STAR_CUDA(call)                                 \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// Checks (once per device) that we run on sm_100 and records the SM count.
static star_status ensure_device() {
  static std::mutex mu;
  static int checked_dev = -1;
  static star_status checked_st = STAR_OK;
  static std::string checked_msg;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  if (checked_dev == dev) {
    if (checked_st != STAR_OK) t_err = checked_msg;
    return checked_st;
  }
  int major = 0, minor = 0, sms = 0;
  if ((e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute");
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  checked_dev = dev;
  if (major != 10 || minor != 0) {
    checked_st = fail(STAR_ENOTSUP, "star: device %d is sm_%d%d; this library is built for sm_100a (B200) only",
                      dev, major, minor);
    checked_msg = t_err;
    return checked_st;
  }
  g_num_sms = sms;
  checked_st = STAR_OK;
  return STAR_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D K-major tile map: inner = K (contiguous), outer = rows; box = 128 bytes x box_rows, SWIZZLE_128B.
static star_status make_tmap(CUtensorMap* m, const void* base, bool f32, uint64_t inner, uint64_t rows,
                             uint64_t row_stride_bytes, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (row_stride_bytes & 15u))
    return fail(STAR_EINVAL, "operand base/row stride must be 16-byte aligned");
  const uint32_t elem = f32 ? 4u : 2u;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {128u / elem, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(STAR_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return STAR_OK;
}

template <int BN, bool TF32>
static cudaError_t launch_gemm_t(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int m_tiles,
                                 cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(umma_gemm_kernel<BN, TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)GemmSmem<BN>::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(m_tiles, p.N / BN, p.splits);
  umma_gemm_kernel<BN, TF32><<<grid, 192, GemmSmem<BN>::BYTES, st>>>(a, b, p);
  return cudaGetLastError();
}

static cudaError_t launch_gemm(int BN, bool tf32, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p,
                               int m_tiles, cudaStream_t st) {
  if (tf32) {
    if (BN == 256) return launch_gemm_t<256, true>(a, b, p, m_tiles, st);
    if (BN == 128) return launch_gemm_t<128, true>(a, b, p, m_tiles, st);
    return launch_gemm_t<64, true>(a, b, p, m_tiles, st);
  }
  if (BN == 256) return launch_gemm_t<256, false>(a, b, p, m_tiles, st);
  if (BN == 128) return launch_gemm_t<128, false>(a, b, p, m_tiles, st);
  return launch_gemm_t<64, false>(a, b, p, m_tiles, st);
}

// Timing events must be real event-record nodes inside a captured graph (External flag);
// outside capture a plain record.  Errors are cleared so they cannot leak into a launch check.
static void record_timing_event(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else
    cudaEventRecord(ev, st);
  cudaGetLastError();
}

static int pick_bn(int N) {
  if (N % 256 == 0) return 256;
  if (N % 128 == 0) return 128;
  return 64;
}

// Split-K so that tiles * splits fills (but does not exceed) the SMs; every split gets >= 2 K blocks.
static void plan_splits(int m_tiles, int n_tiles, int num_kb, int* splits, int* kb_per_split) {
  const int tiles = m_tiles * n_tiles;
  int s = 1;
  if (tiles < g_num_sms) {
    s = g_num_sms / tiles;
    const int max_s = num_kb / 2 > 0 ? num_kb / 2 : 1;
    if (s > max_s) s = max_s;
    if (s < 1) s = 1;
  }
  int kps = (num_kb + s - 1) / s;
  s = (num_kb + kps - 1) / kps;
  *splits = s;
  *kb_per_split = kps;
}

}  // namespace star

using namespace star;

struct star_predictor {
  int d, m1, m2, m3, max_rows;
  bool f32;
  const void *W1, *W2, *W3;
  const float *w4, *b1, *b2, *b3, *b4;
  int bn1, bn2;
  // library-owned device memory
  float *W1s = nullptr, *W2s = nullptr, *W3s = nullptr;   // 3xTF32 [hi|lo|hi] weights (f32 mode)
  void* hs = nullptr;                                      // 3xTF32 [hi|hi|lo] h (f32 mode)
  void *Z1 = nullptr, *Z2 = nullptr;
  float* ws = nullptr;
  int* counters = nullptr;
  size_t ws_floats = 0;
  CUtensorMap tmA1, tmB1, tmA2, tmB2, tmA3, tmB3;
  const void* last_h = nullptr;
  int64_t last_ld = 0;
  int last_R = -1;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

extern "C" {

const char* star_last_error(void) { return t_err.c_str(); }
const char* star_version(void) { return "star-b200 0.1 sm_100a"; }

static void free_pred(star_predictor* p) {
  if (!p) return;
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  cudaFree(p->W1s);
  cudaFree(p->W2s);
  cudaFree(p->W3s);
  cudaFree(p->hs);
  cudaFree(p->Z1);
  cudaFree(p->Z2);
  cudaFree(p->ws);
  cudaFree(p->counters);
  delete p;
}

star_status star_predictor_create(star_predictor** out, int d, int m1, int m2, int m3, star_dtype dt, const void* W1,
                                  const void* W2, const void* W3, const float* w4, const float* b1, const float* b2,
                                  const float* b3, const float* b4, int max_rows, star_stream_t stream_) {
  if (!out) return fail(STAR_EINVAL, "out is NULL");
  *out = nullptr;
  star_status st = ensure_device();
  if (st != STAR_OK) return st;
  if (dt != STAR_F32 && dt != STAR_BF16) return fail(STAR_EINVAL, "dtype must be STAR_F32 or STAR_BF16");
  if (!W1 || !W2 || !W3 || !w4) return fail(STAR_EINVAL, "W1, W2, W3, w4 must be non-NULL");
  if (d < 8 || d % 8) return fail(STAR_EINVAL, "d=%d must be a positive multiple of 8", d);
  if (m1 < 64 || m1 % 64 || m2 < 64 || m2 % 64) return fail(STAR_ENOTSUP, "m1, m2 must be multiples of 64");
  if (m3 != 64) return fail(STAR_ENOTSUP, "m3 must be 64 (PAPER.md:241)");
  if (max_rows < 1 || max_rows > (1 << 20)) return fail(STAR_ERANGE, "max_rows=%d outside [1, 2^20]", max_rows);
  const bool f32 = dt == STAR_F32;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  star_predictor* p = new star_predictor();
  p->d = d;
  p->m1 = m1;
  p->m2 = m2;
  p->m3 = m3;
  p->max_rows = max_rows;
  p->f32 = f32;
  p->W1 = W1;
  p->W2 = W2;
  p->W3 = W3;
  p->w4 = w4;
  p->b1 = b1;
  p->b2 = b2;
  p->b3 = b3;
  p->b4 = b4;
  p->bn1 = pick_bn(m1);
  p->bn2 = pick_bn(m2);
  const size_t esz = f32 ? 4 : 2;
  const int kx = f32 ? 3 : 1;   // K expansion of the 3xTF32 operand layout
  auto alloc = [&](void** ptr, size_t bytes) -> bool { return cudaMalloc(ptr, bytes) == cudaSuccess; };
  bool ok = true;
  ok &= alloc(&p->Z1, (size_t)max_rows * m1 * esz * kx);
  ok &= alloc(&p->Z2, (size_t)max_rows * m2 * esz * kx);
  p->ws_floats = (size_t)g_num_sms * 128 * 256;
  ok &= alloc(reinterpret_cast<void**>(&p->ws), p->ws_floats * 4);
  ok &= alloc(reinterpret_cast<void**>(&p->counters), 4096 * sizeof(int));
  if (f32) {
    ok &= alloc(&p->hs, (size_t)max_rows * d * 4 * 3);
    ok &= alloc(reinterpret_cast<void**>(&p->W1s), (size_t)m1 * d * 4 * 3);
    ok &= alloc(reinterpret_cast<void**>(&p->W2s), (size_t)m2 * m1 * 4 * 3);
    ok &= alloc(reinterpret_cast<void**>(&p->W3s), (size_t)m3 * m2 * 4 * 3);
  }
  if (!ok) {
    cudaGetLastError();
    free_pred(p);
    return fail(STAR_ENOMEM, "device allocation failed");
  }
  cudaError_t e = cudaMemsetAsync(p->counters, 0, 4096 * sizeof(int), stream);
  if (e == cudaSuccess && f32) {
    tf32x3_split_kernel<<<1024, 256, 0, stream>>>(static_cast<const float*>(W1), d, m1, d, p->W1s, 1);
    tf32x3_split_kernel<<<256, 256, 0, stream>>>(static_cast<const float*>(W2), m1, m2, m1, p->W2s, 1);
    tf32x3_split_kernel<<<64, 256, 0, stream>>>(static_cast<const float*>(W3), m2, m3, m2, p->W3s, 1);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) {
    free_pred(p);
    return cuda_fail(e, "star_predictor_create");
  }
  const void* B1 = f32 ? (const void*)p->W1s : W1;
  const void* B2 = f32 ? (const void*)p->W2s : W2;
  const void* B3 = f32 ? (const void*)p->W3s : W3;
  const uint64_t K1 = (uint64_t)d * kx, K2 = (uint64_t)m1 * kx, K3 = (uint64_t)m2 * kx;
  if ((st = make_tmap(&p->tmB1, B1, f32, K1, m1, K1 * esz, p->bn1)) != STAR_OK ||
      (st = make_tmap(&p->tmB2, B2, f32, K2, m2, K2 * esz, p->bn2)) != STAR_OK ||
      (st = make_tmap(&p->tmB3, B3, f32, K3, m3, K3 * esz, 64)) != STAR_OK ||
      (st = make_tmap(&p->tmA2, p->Z1, f32, K2, max_rows, K2 * esz, 128)) != STAR_OK ||
      (st = make_tmap(&p->tmA3, p->Z2, f32, K3, max_rows, K3 * esz, 128)) != STAR_OK ||
      (f32 && (st = make_tmap(&p->tmA1, p->hs, true, K1, max_rows, K1 * 4, 128)) != STAR_OK)) {
    free_pred(p);
    return st;
  }
  *out = p;
  return STAR_OK;
}

star_status star_predictor_destroy(star_predictor* p) {
  if (!p) return STAR_OK;
  cudaError_t e = cudaDeviceSynchronize();
  free_pred(p);
  if (e != cudaSuccess) return cuda_fail(e, "star_predictor_destroy");
  return STAR_OK;
}

star_status star_predictor_layer1_timing(star_predictor* p, int enable) {
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  if (enable && !p->ev0) {
    STAR_CUDA(cudaEventCreate(&p->ev0));
    STAR_CUDA(cudaEventCreate(&p->ev1));
  } else if (!enable && p->ev0) {
    cudaEventDestroy(p->ev0);
    cudaEventDestroy(p->ev1);
    p->ev0 = p->ev1 = nullptr;
  }
  return STAR_OK;
}

star_status star_predictor_layer1_ms(star_predictor* p, float* ms) {
  if (!p || !ms) return fail(STAR_EINVAL, "predictor / ms is NULL");
  if (!p->ev0) return fail(STAR_EINVAL, "layer-1 timing is not enabled");
  STAR_CUDA(cudaEventSynchronize(p->ev1));
  STAR_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
  return STAR_OK;
}

star_status lenpred_forward(star_predictor* p, const void* h, int64_t ld_h, int R, const int32_t* n_tok,
                            int32_t max_ctx_len, float* y_hat, int32_t* n_hat, star_stream_t stream_) {
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  if (R < 0 || R > p->max_rows) return fail(STAR_ERANGE, "R=%d outside [0, max_rows=%d]", R, p->max_rows);
  if (R == 0) return STAR_OK;
  if (!h) return fail(STAR_EINVAL, "h is NULL");
  if (ld_h < p->d) return fail(STAR_EINVAL, "ld_h=%lld < d=%d", (long long)ld_h, p->d);
  if (max_ctx_len < 0) return fail(STAR_EINVAL, "max_ctx_len < 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  star_status s;
  const bool f32 = p->f32;
  const int kx = f32 ? 3 : 1;
  const int m_tiles = (R + 127) / 128;
  if (f32) {
    const int64_t total = (int64_t)R * p->d;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 4 * g_num_sms * 8) blocks = 4 * g_num_sms * 8;
    tf32x3_split_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(h), ld_h, R, p->d,
                                                 static_cast<float*>(p->hs), 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tf32x3_split_kernel");
  } else if (h != p->last_h || ld_h != p->last_ld || R != p->last_R) {
    if ((s = make_tmap(&p->tmA1, h, false, p->d, R, (uint64_t)ld_h * 2, 128)) != STAR_OK) return s;
    p->last_h = h;
    p->last_ld = ld_h;
    p->last_R = R;
  }
  GemmArgs g{};
  g.M = R;
  g.max_ctx = max_ctx_len;
  g.ws = p->ws;
  g.counters = p->counters;
  // ---- layer 1: Z1 = relu(W1 h + b1) ----
  {
    const int num_kb = (p->d * kx * (f32 ? 4 : 2) + 127) / 128;
    g.N = p->m1;
    g.num_kb = num_kb;
    plan_splits(m_tiles, p->m1 / p->bn1, num_kb, &g.splits, &g.kb_per_split);
    g.epi = f32 ? EPI_RELU_TF32X3 : EPI_RELU_BF16;
    g.out = p->Z1;
    g.ld_out = (int64_t)p->m1 * kx;
    g.bias = p->b1;
    if (p->ev0) record_timing_event(p->ev0, st);
    cudaError_t e = launch_gemm(p->bn1, f32, p->tmA1, p->tmB1, g, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "layer-1 GEMM launch");
    if (p->ev1) record_timing_event(p->ev1, st);
  }
  // ---- layer 2: Z2 = relu(W2 Z1 + b2) ----
  {
    const int num_kb = (p->m1 * kx * (f32 ? 4 : 2)) / 128;
    g.N = p->m2;
    g.num_kb = num_kb;
    plan_splits(m_tiles, p->m2 / p->bn2, num_kb, &g.splits, &g.kb_per_split);
    g.epi = f32 ? EPI_RELU_TF32X3 : EPI_RELU_BF16;
    g.out = p->Z2;
    g.ld_out = (int64_t)p->m2 * kx;
    g.bias = p->b2;
    cudaError_t e = launch_gemm(p->bn2, f32, p->tmA2, p->tmB2, g, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "layer-2 GEMM launch");
  }
  // ---- layer 3 + head: z3 = relu(W3 Z2 + b3); y = w4 . z3 + b4; N_hat = quantize(y) ----
  {
    const int num_kb = (p->m2 * kx * (f32 ? 4 : 2)) / 128;
    g.N = p->m3;
    g.num_kb = num_kb;
    plan_splits(m_tiles, 1, num_kb, &g.splits, &g.kb_per_split);
    g.epi = EPI_HEAD;
    g.out = nullptr;
    g.ld_out = 0;
    g.bias = p->b3;
    g.w4 = p->w4;
    g.b4 = p->b4;
    g.n_tok = n_tok;
    g.y_hat = y_hat;
    g.n_hat = n_hat;
    cudaError_t e = launch_gemm(64, f32, p->tmA3, p->tmB3, g, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "layer-3/head GEMM launch");
  }
  return STAR_OK;
}

star_status lenpred_quantize(const float* y_hat, const int32_t* n_tok, int R, int32_t max_ctx_len, int32_t* n_hat,
                             star_stream_t stream_) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  if (R < 0) return fail(STAR_EINVAL, "R < 0");
  if (R == 0) return STAR_OK;
  if (!y_hat || !n_hat) return fail(STAR_EINVAL, "y_hat and n_hat must be non-NULL");
  if (max_ctx_len < 0) return fail(STAR_EINVAL, "max_ctx_len < 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  int blocks = (R + 255) / 256;
  if (blocks > 8 * g_num_sms) blocks = 8 * g_num_sms;
  quantize_kernel<<<blocks, 256, 0, st>>>(y_hat, n_tok, R, max_ctx_len, n_hat);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "quantize_kernel");
  return STAR_OK;
}

size_t star_project_workspace_bytes(int n_inst, int H) {
  if (n_inst < 1 || H < 0) return 0;
  return project_workspace_bytes(n_inst, H);
}

int star_project_single_cta_max_rows(void) { return project_single_cta_max_rows(); }

star_status project_instance_load(int R, int n_inst, int inst_base, int H, const int32_t* inst, const int32_t* n_tok,
                                  const int32_t* n_hat, const uint32_t* beta_q, int64_t* L, int64_t* W,
                                  int64_t* peak, int64_t* growth, int32_t* count, void* workspace,
                                  int32_t* err_flag, star_stream_t stream_) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  if (R < 0) return fail(STAR_EINVAL, "R < 0");
  if (n_inst < 1 || n_inst > (1 << 16)) return fail(STAR_ERANGE, "n_inst=%d outside [1, 65536]", n_inst);
  if (H < 0 || H > 256) return fail(STAR_ERANGE, "H=%d outside [0, 256]", H);
  if (!L || !beta_q) return fail(STAR_EINVAL, "L and beta_q must be non-NULL");
  if (R > 0 && (!inst || !n_tok || !n_hat)) return fail(STAR_EINVAL, "inst, n_tok, n_hat must be non-NULL");
  if ((size_t)n_inst * (H + 2) > 12288 && !workspace)
    return fail(STAR_EINVAL, "n_inst*(H+2) > 12288 requires a workspace");
  cudaError_t e = launch_project(R, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                                 workspace, err_flag, reinterpret_cast<cudaStream_t>(stream_), nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "project_kernel launch");
  return STAR_OK;
}

static star_status check_plan_params(const star_plan_params* p) {
  if (!p) return fail(STAR_EINVAL, "params is NULL");
  if (p->n_inst < 1) return fail(STAR_EINVAL, "n_inst < 1");
  if (p->H < 0 || p->H > 256) return fail(STAR_ERANGE, "H outside [0, 256]");
  if (p->max_moves < 0 || p->max_moves > 1024) return fail(STAR_ERANGE, "max_moves outside [0, 1024]");
  if (p->theta_den < 1 || p->theta_num < 0) return fail(STAR_EINVAL, "theta must be num/den with num>=0, den>=1");
  if (!p->beta_q) return fail(STAR_EINVAL, "beta_q is NULL");
  if (p->flags & ~3u) return fail(STAR_EINVAL, "unknown flag bits");
  return STAR_OK;
}

star_status plan_reschedule_segmented(const star_plan_params* p, const star_plan_segments* sg, star_move* moves,
                                      int32_t* n_moves, int32_t* err_flag, star_stream_t stream_) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  if ((s = check_plan_params(p)) != STAR_OK) return s;
  if (!sg || !sg->L) return fail(STAR_EINVAL, "segments / L is NULL");
  if (!n_moves || (p->max_moves > 0 && !moves)) return fail(STAR_EINVAL, "moves / n_moves is NULL");
  if (sg->world < 1 || sg->n_loc < 1 || (int64_t)sg->world * sg->n_loc != p->n_inst)
    return fail(STAR_EINVAL, "world*n_loc must equal n_inst");
  if (sg->r_cap < 0) return fail(STAR_EINVAL, "r_cap < 0");
  if (sg->r_cap > 0 && (!sg->req_id || !sg->inst || !sg->n_tok || !sg->n_hat))
    return fail(STAR_EINVAL, "request arrays must be non-NULL");
  if ((int64_t)sg->world * sg->r_cap > (1 << 20)) return fail(STAR_ERANGE, "more than 2^20 request slots");
  if (sg->world > 1 && sg->seg_stride <= 0) return fail(STAR_EINVAL, "seg_stride must be > 0 when world > 1");
  const size_t smem = plan_smem_bytes(p->n_inst, p->H, sg->world, sg->r_cap) + 2048;  // + static smem
  if (smem > (size_t)kMaxSmemBytes)
    return fail(STAR_ENOTSUP, "plan state (%zu B) exceeds shared memory: n_inst*(H+1) too large", smem);
  cudaError_t e = launch_plan(p, sg, moves, n_moves, err_flag, reinterpret_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "plan_kernel launch");
  return STAR_OK;
}

star_status plan_reschedule(const star_plan_params* p, const int64_t* L, int R_total, const int32_t* req_id,
                            const int32_t* inst, const int32_t* n_tok, const int32_t* n_hat, const uint8_t* pinned,
                            star_move* moves, int32_t* n_moves, int32_t* err_flag, star_stream_t stream) {
  if (!p) return fail(STAR_EINVAL, "params is NULL");
  if (R_total < 0) return fail(STAR_EINVAL, "R_total < 0");
  star_plan_segments sg{};
  sg.world = 1;
  sg.n_loc = p->n_inst;
  sg.r_cap = R_total;
  sg.seg_stride = 0;
  sg.L = L;
  sg.r_count = nullptr;
  sg.req_id = req_id;
  sg.inst = inst;
  sg.n_tok = n_tok;
  sg.n_hat = n_hat;
  sg.pinned = pinned;
  return plan_reschedule_segmented(p, &sg, moves, n_moves, err_flag, stream);
}

}  // extern "C"
