// star_api.cu -- the C ABI (include/star.h): host-side validation, TMA descriptor set-up,
// tile/split planning and kernel launches.  No compute happens on the host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "lenpred_f32.cuh"
#include "lenpred_kernels.cuh"
#include "lenpred_small.cuh"
#include "lenpred_tail.cuh"
#include "lenpred_tail2.cuh"
#include "plan_core.cuh"
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

cudaError_t func_attr(const void* func, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(dev, func, (int)attr);
  auto it = done.find(key);
  const bool grow = attr == cudaFuncAttributeMaxDynamicSharedMemorySize;
  if (it != done.end() && (grow ? it->second >= value : true)) return cudaSuccess;
  e = cudaFuncSetAttribute(func, attr, value);
  if (e == cudaSuccess) done[key] = value;
  return e;
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
static cudaError_t launch_gemm_t(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmArgs& p,
                                 int m_tiles, cudaStream_t st) {
  {
    cudaError_t e = func_attr((const void*)umma_gemm_kernel<BN, TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)GemmSmem<BN>::BYTES);
    if (e != cudaSuccess) return e;
  }
  // grid (m tiles, n tiles, K splits); the splits of one output tile form a cluster along z
  // (co-scheduled, so they can exchange partials behind a cluster barrier).  Programmatic
  // dependent launch lets the prologue overlap the previous kernel; the kernel calls
  // griddepcontrol.wait before touching memory.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = p.mn_swap ? dim3(p.N / BN, m_tiles, p.splits) : dim3(m_tiles, p.N / BN, p.splits);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = GemmSmem<BN>::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = (unsigned)p.splits;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, umma_gemm_kernel<BN, TF32>, a, b, c, p);
}

static cudaError_t launch_gemm(int BN, bool tf32, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                               const GemmArgs& p, int m_tiles, cudaStream_t st) {
  if (tf32) {
    if (BN == 256) return launch_gemm_t<256, true>(a, b, c, p, m_tiles, st);
    if (BN == 128) return launch_gemm_t<128, true>(a, b, c, p, m_tiles, st);
    return launch_gemm_t<64, true>(a, b, c, p, m_tiles, st);
  }
  if (BN == 256) return launch_gemm_t<256, false>(a, b, c, p, m_tiles, st);
  if (BN == 128) return launch_gemm_t<128, false>(a, b, c, p, m_tiles, st);
  return launch_gemm_t<64, false>(a, b, c, p, m_tiles, st);
}

// CTA-pair layer-1 GEMM: grid (m tiles rounded up to even, n tiles), clusters of 2 along M, PDL.
static cudaError_t launch_pair_gemm(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmArgs& p,
                                   int m_tiles, cudaStream_t st, bool nu = false) {
  {
    cudaError_t e = func_attr((const void*)umma_pair_gemm_kernel<256, false>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairSmem<256>::BYTES);
    if (e == cudaSuccess)
      e = func_attr((const void*)umma_pair_gemm_kernel<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                    (int)PairSmem<256>::BYTES);
    if (e == cudaSuccess)
      e = func_attr((const void*)umma_pair_gemm_kernel<256, false, true>,
                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairSmem<256>::BYTES);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  // nu: N = 2048 as 9 tiles of 224 / 240 columns; splits: K ranges (one wave, <= SMs)
  cfg.gridDim = dim3((m_tiles + 1) & ~1, nu ? 9 : p.N / 256, p.splits);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = PairSmem<256>::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (nu) return cudaLaunchKernelEx(&cfg, umma_pair_gemm_kernel<256, false, true>, a, b, c, p);
  return p.splits > 1 ? cudaLaunchKernelEx(&cfg, umma_pair_gemm_kernel<256, true>, a, b, c, p)
                      : cudaLaunchKernelEx(&cfg, umma_pair_gemm_kernel<256, false>, a, b, c, p);
}

// Persistent 9-column-tile pairs, two tiles per pair (umma_pair_nu2_kernel): one wave of
// 2 * ceil(tiles / 2) CTAs.  STAR_L1_PERSIST=0 keeps the two-wave grid (A/B measurements).
static bool l1_persist_enabled() {
  static const bool v = [] {
    const char* e = getenv("STAR_L1_PERSIST");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}
static cudaError_t launch_pair_nu2(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int m_tiles,
                                   cudaStream_t st) {
  cudaError_t e = func_attr((const void*)umma_pair_nu2_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)PairSmem<256>::BYTES);
  if (e != cudaSuccess) return e;
  const int ntiles = ((m_tiles + 1) / 2) * 9;
  const int npairs = (ntiles + 1) / 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * npairs, 1, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = PairSmem<256>::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, umma_pair_nu2_kernel<256>, a, b, p, ntiles);
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

// Split-K choice.  splits is a power of two <= 8 (one portable cluster) with tiles*splits <=
// SMs, owned width BN/splits >= 16 columns and >= 2 K blocks per split.  Among those, pick the
// split count with the lowest modelled time (cycles), from B200 measurements
// (tools/tma_bench.cu, tools/timeline.py):
//   operand delivery  per-CTA bytes / 60 B/clk (per-SM TMA ingest with a 4-stage ring)
//   MMA               128 * BN * K_split / 4096 MAC/clk   (bf16; x2 for the 3xTF32 layout)
//   reduction         (splits > 1) 2 * (S-1)/S * 128*BN*4 B / 25 B/clk + 1500 (cluster barrier)
// (delivery dominates large tiles; the exchange and barrier dominate small ones, e.g. the
// 64-column head, which is fastest unsplit).
static void plan_splits(int tiles, int num_kb, int bn, bool tf32, int* splits, int* kb_per_split) {
  int best_s = 1, best_k = num_kb;
  double best_t = 1e30;
  for (int s = 1; s <= 8; s *= 2) {
    if (s > 1 && (tiles * s > g_num_sms || bn / s < 16 || num_kb / s < 2)) break;
    const int k = (num_kb + s - 1) / s;
    if (s > 1 && (s - 1) * k >= num_kb) break;
    const double cta_bytes = (128.0 + bn) * 128.0 * k;
    const double load = cta_bytes / 60.0;
    const double mma = 128.0 * bn * (k * (tf32 ? 32.0 : 64.0)) / 4096.0 * (tf32 ? 2.0 : 1.0);
    const double red = s > 1 ? 2.0 * (s - 1) / s * 128.0 * bn * 4.0 / 25.0 + 1500.0 : 0.0;
    const double t = std::max(load, mma) + red;
    if (t < best_t * 0.97) {   // prefer fewer splits unless clearly faster
      best_t = t;
      best_s = s;
      best_k = k;
    }
  }
  *splits = best_s;
  *kb_per_split = best_k;
}


// The one-launch small-batch predictor (lenpred_small.cuh) needs all of its CTAs resident at
// once (phases hand off through counters): 64 clusters of 2 CTAs of ~218 KB shared memory.
// STAR_SMALL=0 disables it (A/B measurements).
static bool small_path_available() {
  const char* e = getenv("STAR_SMALL");
  if (e && atoi(e) == 0) return false;
  if (func_attr((const void*)lenpred_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)SmallSmem::BYTES) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2, 16, 4);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = SmallSmem::BYTES;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)lenpred_small_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return ncl >= 64;
}

// The one-launch fp32 predictor (lenpred_f32.cuh, <= 128 rows) needs its 128 CTAs (~161 KB of
// shared memory, 512 TMEM columns each) resident at once.  STAR_F32_SMALL=0 disables it (A/B measurements).
static bool f32_small_available() {
  const char* e = getenv("STAR_F32_SMALL");
  if (e && atoi(e) == 0) return false;
  if (func_attr((const void*)lenpred_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)F32Smem::BYTES) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lenpred_f32_kernel, 320, F32Smem::BYTES) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return per_sm >= 1 && per_sm * g_num_sms >= 128;
}

struct SmallRefresh {   // refresh mode: the compacted batch and the slots it scatters into
  int rows_expected;      // sizes the grid (the count itself is on the device)
  const int32_t* M_dev;
  const int32_t* idx;
  const int32_t* gen;
  int32_t* g_last;
  int32_t* nhat_last;
  int32_t* n_hat;
};
static cudaError_t launch_small(star_predictor* p, int R, const int32_t* n_tok, int32_t max_ctx, float* y_hat,
                                int32_t* n_hat, const ProjArgs* proj, cudaStream_t st,
                                const CUtensorMap* tmH = nullptr, const SmallRefresh* rf = nullptr);
static cudaError_t launch_f32_small(star_predictor* p, int R, const int32_t* n_tok, int32_t max_ctx, float* y_hat,
                                    int32_t* n_hat, const ProjArgs* proj, cudaStream_t st);

// The large-batch tail: clusters of 4 per m-tile (lenpred_tail2.cuh); STAR_TAIL2=0 selects the
// round-1 split-K tail (A/B measurements).
static bool tail2_enabled() {
  static const bool v = [] {
    const char* e = getenv("STAR_TAIL2");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

// Whether a one-rank single-round plan runs in the fused tail's last CTA (STAR_PLAN_FUSE=1, read
// once) instead of the cluster plan kernel launched after it (default).  Measured at TGT with a
// move (Alg. 1 past Phase 1): 117.3 us fused (192 threads score the candidates) vs 99.4 us with
// the 8-CTA plan kernel; without candidates (C2) the two are within 0.4 us.
static bool plan_fuse_enabled() {
  static const bool v = [] {
    const char* e = getenv("STAR_PLAN_FUSE");
    return e ? atoi(e) != 0 : false;
  }();
  return v;
}

// Fused tail (layer 2 -> layer 3 -> head -> quantizer [-> projection]) launch: grid
// (m_tiles, n2, S), one cluster per layer-2 tile (its S split-K CTAs), PDL.
static cudaError_t launch_tail(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& w3, const TailArgs& t,
                               int m_tiles, cudaStream_t st) {
  {
    cudaError_t e = func_attr((const void*)tail_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)TailSmem::BYTES);
    if (e == cudaSuccess)
      e = func_attr((const void*)tail_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                    (int)TailSmem::BYTES);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = t.mn_swap ? dim3(t.n2_tiles, m_tiles, t.splits) : dim3(m_tiles, t.n2_tiles, t.splits);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = TailSmem::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = (unsigned)t.splits;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return t.plan ? cudaLaunchKernelEx(&cfg, tail_kernel<true>, a, b, w3, t)
                : cudaLaunchKernelEx(&cfg, tail_kernel<false>, a, b, w3, t);
}

// Split count of the fused tail: S = 4 when m_tiles * n2 * 4 CTAs fit one wave, else 2
// (n2 * S <= 8 keeps the workspace bounds).  Returns 0 when the shape cannot use the tail.
static int tail_splits(int m_tiles, int n2, int num_kb) {
  for (int s = 4; s >= 2; s /= 2) {
    if (n2 * s > 8 || num_kb / s < 2) continue;
    if (s == 4 && m_tiles * n2 * s > g_num_sms) continue;
    return s;
  }
  return 0;
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
  float* ws = nullptr;        // split-K partials
  float* head_ws = nullptr;   // split-K head partial dots
  float* ws3 = nullptr;       // fused tail: layer-3 partials [m_tiles][16][64][128]
  int* tail_cnt = nullptr;    // fused tail: per (m-tile, split) arrival counters
  int* l1_cnt = nullptr;      // layer-1 CTA-pair split-K: per CTA tile arrival / done counters
  uint64_t* tl = nullptr;     // diagnostics: fused-tail phase timeline [ctas][16]
  int tl_ctas = 0;            // CTAs of the most recent timed tail launch
  // refresh cadence (NEXT-1) scratch: compacted rows and their hidden states
  int32_t *r_idx = nullptr, *r_pos = nullptr, *r_ntok = nullptr, *r_nhat = nullptr, *r_M = nullptr;
  void* r_h = nullptr;
  float* r_ws = nullptr;      // layer-1 split-K partials for the refresh grid (all m-tiles x 4 splits)
  CUtensorMap tmA_r;          // compacted hidden states [max_rows][d]
  uint64_t* tl_l1 = nullptr;  // diagnostics: layer-1 (CTA-pair) GEMM phase timeline
  int tl_l1_ctas = 0;
  size_t ws_floats = 0;
  CUtensorMap tmA1, tmB1, tmA2, tmB2, tmA3, tmB3;
  CUtensorMap tmC1, tmC2;     // TMA-store maps of Z1 / Z2 (bf16, 64 x 32 boxes)
  CUtensorMap tmB1p;          // W1 with 128-row boxes (CTA-pair kernel: each CTA loads half of B)
  // one-launch predictor for <= 512 rows (lenpred_small.cuh)
  CUtensorMap tmW2s;          // W2 with 32-row boxes
  CUtensorMap tmW2t;          // W2 with 128-row boxes (tail2)
  CUtensorMap tmW1n[2];       // W1 with 32- / 64-row boxes (the small-batch kernel's narrow layer-1 tiles)
  int* tail2_done = nullptr;  // tail2: m-tiles finished (zero between launches)
  int* small_cnt = nullptr;   // its phase counters (zero between launches)
  int* r_blk = nullptr;       // refresh: the multi-CTA select's counts and counters (zero between launches)
  bool small_ok = false;      // shape supported and 32 clusters of 4 co-resident
  uint64_t* tl_small = nullptr;
  // one-launch fp32 predictor for <= 128 rows (lenpred_f32.cuh): raw fp32 operand maps
  CUtensorMap tmHf, tmW1f, tmW2f, tmW3f, tmZ1f, tmZ2f;
  int* f32_cnt = nullptr;     // its arrival counters (zero between launches)
  float *W1p = nullptr, *W2p = nullptr, *W3p = nullptr;   // its weights as [hi; lo] tf32 planes
  bool f32_ok = false;
  const void* last_hf = nullptr;
  int64_t last_ldf = 0;
  int last_Rf = -1;
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
  cudaFree(p->head_ws);
  cudaFree(p->ws3);
  cudaFree(p->tail_cnt);
  cudaFree(p->l1_cnt);
  cudaFree(p->tl);
  cudaFree(p->tl_l1);
  cudaFree(p->small_cnt);
  cudaFree(p->f32_cnt);
  cudaFree(p->W1p);
  cudaFree(p->W2p);
  cudaFree(p->W3p);
  cudaFree(p->r_blk);
  cudaFree(p->tail2_done);
  cudaFree(p->tl_small);
  cudaFree(p->r_idx);
  cudaFree(p->r_pos);
  cudaFree(p->r_ntok);
  cudaFree(p->r_nhat);
  cudaFree(p->r_M);
  cudaFree(p->r_h);
  cudaFree(p->r_ws);
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
  // split-K partials (128 x 256 fp32 per CTA tile and split): layer-1 split-K and CTA-pair grids
  // stay within one wave (<= SMs tiles x splits); the fused tail needs m_tiles x (m2/256) x S with
  // S = 4 (S = 2 only bounds the grid to one wave for the plain forward; the refresh grid may
  // run every m-tile with the S chosen for its row estimate)
  const size_t tail_tiles = (size_t)((max_rows + 127) / 128) * (m2 / 256 > 0 ? m2 / 256 : 1) * 4;
  p->ws_floats = (tail_tiles > (size_t)g_num_sms ? tail_tiles : (size_t)g_num_sms) * 128 * 256;
  ok &= alloc(reinterpret_cast<void**>(&p->ws), p->ws_floats * 4);
  ok &= alloc(reinterpret_cast<void**>(&p->head_ws), (size_t)g_num_sms * 128 * 4);
  ok &= alloc(reinterpret_cast<void**>(&p->ws3), (size_t)((max_rows + 127) / 128) * 16 * 64 * 128 * 4);
  ok &= alloc(reinterpret_cast<void**>(&p->tail_cnt), (size_t)((max_rows + 127) / 128) * 8 * sizeof(int));
  ok &= alloc(reinterpret_cast<void**>(&p->l1_cnt), (size_t)2 * g_num_sms * sizeof(int));
  if (!f32) {
    ok &= alloc(reinterpret_cast<void**>(&p->r_idx), (size_t)max_rows * 4);
    ok &= alloc(reinterpret_cast<void**>(&p->r_pos), (size_t)max_rows * 4);
    ok &= alloc(reinterpret_cast<void**>(&p->r_ntok), (size_t)max_rows * 4);
    ok &= alloc(reinterpret_cast<void**>(&p->r_nhat), (size_t)max_rows * 4);
    ok &= alloc(reinterpret_cast<void**>(&p->r_M), 16);
    ok &= alloc(&p->r_h, (size_t)max_rows * d * 2);
    ok &= alloc(reinterpret_cast<void**>(&p->r_ws),
                (size_t)((max_rows + 127) / 128) * (m1 / 256 > 0 ? m1 / 256 : 1) * 4 * 256 * 128 * 4);
  }
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
  cudaError_t e = cudaMemsetAsync(p->tail_cnt, 0, (size_t)((max_rows + 127) / 128) * 8 * sizeof(int), stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(p->l1_cnt, 0, (size_t)2 * g_num_sms * sizeof(int), stream);
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
      (f32 && (st = make_tmap(&p->tmA1, p->hs, true, K1, max_rows, K1 * 4, 128)) != STAR_OK) ||
      (!f32 && (st = make_tmap(&p->tmC1, p->Z1, false, m1, max_rows, (uint64_t)m1 * 2, 32)) != STAR_OK) ||
      (!f32 && (st = make_tmap(&p->tmB1p, B1, false, K1, m1, K1 * esz, 128)) != STAR_OK) ||
      (!f32 && (st = make_tmap(&p->tmA_r, p->r_h, false, (uint64_t)d, max_rows, (uint64_t)d * 2, 128)) != STAR_OK) ||
      (!f32 && (st = make_tmap(&p->tmC2, p->Z2, false, m2, max_rows, (uint64_t)m2 * 2, 32)) != STAR_OK)) {
    free_pred(p);
    return st;
  }
  if (f32 && m1 == 2048 && m2 == 512 && d % 128 == 0 && p->ws_floats >= (size_t)F32_WS_FLOATS) {
    const size_t n1 = (size_t)m1 * d, n2 = (size_t)m2 * m1, n3 = (size_t)m3 * m2;
    if (cudaMalloc(reinterpret_cast<void**>(&p->W1p), 2 * n1 * 4) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&p->W2p), 2 * n2 * 4) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&p->W3p), 2 * n3 * 4) != cudaSuccess) {
      cudaGetLastError();
      free_pred(p);
      return fail(STAR_ENOMEM, "device allocation failed");
    }
    tf32_planes_kernel<<<1024, 256, 0, stream>>>(static_cast<const float*>(W1), (int64_t)n1, p->W1p);
    tf32_planes_kernel<<<512, 256, 0, stream>>>(static_cast<const float*>(W2), (int64_t)n2, p->W2p);
    tf32_planes_kernel<<<64, 256, 0, stream>>>(static_cast<const float*>(W3), (int64_t)n3, p->W3p);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess) {
      free_pred(p);
      return cuda_fail(e, "tf32_planes_kernel");
    }
    if ((st = make_tmap(&p->tmW1f, p->W1p, true, (uint64_t)d, 2 * m1, (uint64_t)d * 4, 64)) != STAR_OK ||
        (st = make_tmap(&p->tmW2f, p->W2p, true, (uint64_t)m1, 2 * m2, (uint64_t)m1 * 4, 32)) != STAR_OK ||
        (st = make_tmap(&p->tmW3f, p->W3p, true, (uint64_t)m2, 2 * m3, (uint64_t)m2 * 4, 64)) != STAR_OK ||
        (st = make_tmap(&p->tmZ1f, p->Z1, true, (uint64_t)m1, max_rows, (uint64_t)m1 * 4, 128)) != STAR_OK ||
        (st = make_tmap(&p->tmZ2f, p->Z2, true, (uint64_t)m2, max_rows, (uint64_t)m2 * 4, 128)) != STAR_OK) {
      free_pred(p);
      return st;
    }
    p->f32_ok = f32_small_available();
    if (p->f32_ok && (cudaMalloc(reinterpret_cast<void**>(&p->f32_cnt), F32Cnt::N * sizeof(int)) != cudaSuccess ||
                      cudaMemset(p->f32_cnt, 0, F32Cnt::N * sizeof(int)) != cudaSuccess)) {
      cudaGetLastError();
      free_pred(p);
      return fail(STAR_ENOMEM, "device allocation failed");
    }
  }
  if (!f32 && m1 == 2048 && m2 == 512 && d % 256 == 0) {
    if ((st = make_tmap(&p->tmW2s, W2, false, (uint64_t)m1, m2, (uint64_t)m1 * 2, 32)) != STAR_OK ||
        (st = make_tmap(&p->tmW2t, W2, false, (uint64_t)m1, m2, (uint64_t)m1 * 2, 128)) != STAR_OK ||
        (st = make_tmap(&p->tmW1n[0], W1, false, (uint64_t)d, m1, (uint64_t)d * 2, 32)) != STAR_OK ||
        (st = make_tmap(&p->tmW1n[1], W1, false, (uint64_t)d, m1, (uint64_t)d * 2, 64)) != STAR_OK) {
      free_pred(p);
      return st;
    }
    p->small_ok = small_path_available();
    if (cudaMalloc(reinterpret_cast<void**>(&p->tail2_done), 16) != cudaSuccess ||
        cudaMemset(p->tail2_done, 0, 16) != cudaSuccess) {
      cudaGetLastError();
      free_pred(p);
      return fail(STAR_ENOMEM, "device allocation failed");
    }
    func_attr((const void*)tail2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Tail2Smem::BYTES);
    if (p->small_ok) {
      const size_t ncnt = (size_t)SmallSmem::DONE + 16, nblk = 2 * (size_t)g_num_sms + 16;
      if (cudaMalloc(reinterpret_cast<void**>(&p->small_cnt), ncnt * sizeof(int)) != cudaSuccess ||
          cudaMemset(p->small_cnt, 0, ncnt * sizeof(int)) != cudaSuccess ||
          cudaMalloc(reinterpret_cast<void**>(&p->r_blk), nblk * sizeof(int)) != cudaSuccess ||
          cudaMemset(p->r_blk, 0, nblk * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        free_pred(p);
        return fail(STAR_ENOMEM, "device allocation failed");
      }
    }
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

star_status star_predictor_timeline(star_predictor* p, int enable, uint64_t* host_out, int max_ctas, int* n_ctas) {
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  const size_t rows = (size_t)g_num_sms * 4 > (size_t)kTailPlanTlRow + 2 ? (size_t)g_num_sms * 4
                                                                        : (size_t)kTailPlanTlRow + 2;
  if (enable) {
    if (!p->tl) {
      STAR_CUDA(cudaMalloc(&p->tl, rows * kTailTlStride * sizeof(uint64_t)));
      STAR_CUDA(cudaMemset(p->tl, 0, rows * kTailTlStride * sizeof(uint64_t)));
    }
    if (enable == 2 && !p->tl_l1) {
      STAR_CUDA(cudaMalloc(&p->tl_l1, rows * 16 * sizeof(uint64_t)));
      STAR_CUDA(cudaMemset(p->tl_l1, 0, rows * 16 * sizeof(uint64_t)));
    }
  } else {
    cudaFree(p->tl);
    cudaFree(p->tl_l1);
    p->tl = nullptr;
    p->tl_l1 = nullptr;
  }
  if (host_out) {
    STAR_CUDA(cudaDeviceSynchronize());
    const bool l1 = enable == 2;
    const uint64_t* src = l1 ? p->tl_l1 : p->tl;
    const int have = l1 ? p->tl_l1_ctas : p->tl_ctas;
    // copies min(max_ctas, allocated rows) rows (rows past the grid hold auxiliary stamps:
    // the fused plan's, see TailArgs::tl); *n_ctas = rows that belong to CTAs of the last launch
    const int n = src ? (have < max_ctas ? have : max_ctas) : 0;
    const int ncopy = src ? (max_ctas < (int)rows ? max_ctas : (int)rows) : 0;
    const size_t stride = l1 ? 16 : kTailTlStride;
    if (ncopy > 0)
      STAR_CUDA(cudaMemcpy(host_out, src, (size_t)ncopy * stride * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (n_ctas) *n_ctas = n;
  }
  return STAR_OK;
}

star_status star_predictor_path(star_predictor* p, int R, int* path) {
  if (!p || !path) return fail(STAR_EINVAL, "predictor / path is NULL");
  *path = (!p->f32 && p->small_ok && R >= 1 && R <= 512) ? 1 : ((p->f32 && p->f32_ok && R >= 1 && R <= 128) ? 2 : 0);
  return STAR_OK;
}

star_status star_predictor_layer1_ms(star_predictor* p, float* ms) {
  if (!p || !ms) return fail(STAR_EINVAL, "predictor / ms is NULL");
  if (!p->ev0) return fail(STAR_EINVAL, "layer-1 timing is not enabled");
  STAR_CUDA(cudaEventSynchronize(p->ev1));
  STAR_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
  return STAR_OK;
}

// Forward of Eq. 2 (+ optionally the projection of its N_hat, `proj`).  bf16 predictors run
// 2 launches (layer-1 GEMM, fused tail); fp32 predictors run the 3 GEMM launches (+ the
// standalone projection kernel when `proj` is set).
static star_status forward_impl(star_predictor* p, const void* h, int64_t ld_h, int R, const int32_t* n_tok,
                                int32_t max_ctx_len, float* y_hat, int32_t* n_hat, const ProjArgs* proj,
                                void* proj_ws, cudaStream_t st, const PlanArgs* plan = nullptr,
                                bool* plan_fused = nullptr) {
  if (plan_fused) *plan_fused = false;
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  if (R < 0 || R > p->max_rows) return fail(STAR_ERANGE, "R=%d outside [0, max_rows=%d]", R, p->max_rows);
  star_status s;
  const bool f32 = p->f32;
  const int kx = f32 ? 3 : 1;
  const int m_tiles = (R + 127) / 128;
  if (f32 && p->f32_ok && R >= 1 && R <= 128 &&
      (!proj || (size_t)proj->n_inst * (proj->H + 2) * 12 + (size_t)(proj->H + 1) * 4 <= F32Smem::HIST_MAX)) {
    // one launch: Eq. 2 in 3xTF32 + quantizer (+ projection)
    if (h != p->last_hf || ld_h != p->last_ldf || R != p->last_Rf) {
      if ((s = make_tmap(&p->tmHf, h, true, p->d, R, (uint64_t)ld_h * 4, 128)) != STAR_OK) return s;
      p->last_hf = h;
      p->last_ldf = ld_h;
      p->last_Rf = R;
    }
    if (p->ev0) record_timing_event(p->ev0, st);
    cudaError_t e = launch_f32_small(p, R, n_tok, max_ctx_len, y_hat, n_hat, proj, st);
    if (e != cudaSuccess) return cuda_fail(e, "lenpred_f32_kernel launch");
    if (p->ev1) record_timing_event(p->ev1, st);
    return STAR_OK;
  }
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
  if (!f32 && p->small_ok && R >= 1 && R <= 512) {   // one launch: Eq. 2 + quantizer (+ projection)
    if (p->ev0) record_timing_event(p->ev0, st);
    cudaError_t e = launch_small(p, R, n_tok, max_ctx_len, y_hat, n_hat, proj, st);
    if (e != cudaSuccess) return cuda_fail(e, "lenpred_small_kernel launch");
    if (p->ev1) record_timing_event(p->ev1, st);
    return STAR_OK;
  }
  GemmArgs g{};
  g.M = R;
  g.max_ctx = max_ctx_len;
  g.ws = p->ws;
  g.head_ws = p->head_ws;
  const CUtensorMap& tmC1 = f32 ? p->tmA1 : p->tmC1;   // unused in fp32 mode (direct stores)
  const CUtensorMap& tmC2 = f32 ? p->tmA1 : p->tmC2;
  // ---- layer 1: Z1 = relu(W1 h + b1) ----
  {
    const int num_kb = (p->d * kx * (f32 ? 4 : 2) + 127) / 128;
    g.N = p->m1;
    g.num_kb = num_kb;
    plan_splits(m_tiles * (p->m1 / p->bn1), num_kb, p->bn1, f32, &g.splits, &g.kb_per_split);
    g.epi = f32 ? EPI_RELU_TF32X3 : EPI_RELU_BF16;
    g.tma_store = (!f32 && (p->bn1 / g.splits) % 64 == 0) ? 1 : 0;
    g.out = p->Z1;
    g.ld_out = (int64_t)p->m1 * kx;
    g.bias = p->b1;
    // CTA pairs (bf16): split K over the pairs until one wave of <= SMs CTAs is filled
    int pair_splits = 0;
    if (!f32 && p->bn1 == 256) {
      const int pairs = ((m_tiles + 1) / 2) * (p->m1 / 256);
      pair_splits = 1;
      // split-K pairs only for one pair row (129..256 requests: measured 12.5 us vs 13.2 us for the
      // 1-CTA split-4 kernel at d = 4096); at 257..1024 rows the 1-CTA split-K kernel is faster
      // (tools/gemm_bench.cu), at <= 128 rows as well (no padding rows)
      if (m_tiles == 2)
        while (pair_splits < 8 && pairs * pair_splits * 2 * 2 <= g_num_sms && num_kb / (pair_splits * 2) >= 4)
          pair_splits *= 2;
      if (pairs * pair_splits * 2 < (g_num_sms * 5) / 8) pair_splits = 0;   // too few CTAs either way
    }
    const bool pair = pair_splits > 0;
    if (pair) {
      g.splits = pair_splits;
      g.kb_per_split = (num_kb + pair_splits - 1) / pair_splits;
      g.tma_store = 1;
      g.l1_cnt = p->l1_cnt;
      // L2 prefetch by one CTA per tile row / column: cold L2 (the in-step case) 30.8 us vs 33.0 us
      // when every consumer prefetches, warm 24.8 vs 24.3 us (M = 2048, tools/gemm_bench.cu)
      g.prefetch = 2;
      g.tl = p->tl_l1;
      p->tl_l1_ctas = ((m_tiles + 1) & ~1) * (p->m1 / 256) * pair_splits;
    }
    // unsplit pairs over N = 2048: 9 non-uniform column tiles when they still fit one wave
    // (also over several waves: 9 tiles of <= 240 columns win whenever they need no more waves
    // than 8 tiles of 256, e.g. M = 4096: 2 waves of 144 CTAs instead of 148 + 108)
    const int slots = (g_num_sms / 2) * 2, npairs = (m_tiles + 1) / 2;
    const int w8 = (npairs * 16 + slots - 1) / slots, w9 = (npairs * 18 + slots - 1) / slots;
    const bool nu = pair && pair_splits == 1 && p->m1 == 2048 && w9 * 240 < w8 * 256;
    if (nu) p->tl_l1_ctas = ((m_tiles + 1) & ~1) * 9;
    if (!pair) {   // diagnostics timeline of the 1-CTA layer-1 kernel (rows: m x n x split CTAs)
      g.tl = p->tl_l1;
      p->tl_l1_ctas = m_tiles * (p->m1 / p->bn1) * g.splits;
    }
    if (p->ev0) record_timing_event(p->ev0, st);
    // two 9-tile waves fit one wave of pairs with two tiles each
    const int nu_tiles = ((m_tiles + 1) / 2) * 9;
    const bool nu2 = nu && nu_tiles * 2 > slots && (nu_tiles + 1) / 2 * 2 <= slots && l1_persist_enabled();
    cudaError_t e = nu2 ? launch_pair_nu2(p->tmA1, p->tmB1p, g, m_tiles, st)
                  : pair ? launch_pair_gemm(p->tmA1, p->tmB1p, tmC1, g, m_tiles, st, nu)
                         : launch_gemm(p->bn1, f32, p->tmA1, p->tmB1, tmC1, g, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "layer-1 GEMM launch");
    if (p->ev1) record_timing_event(p->ev1, st);
    g.tl = nullptr;
  }
  // ---- fused tail, large batches: one cluster of 4 per m-tile, no split-K (lenpred_tail2.cuh) ----
  if (!f32 && p->tail2_done && p->m2 == 512 && p->m3 == 64 && m_tiles >= 5 && tail2_enabled() &&
      !(proj && plan && plan->world == 1 && plan->max_moves <= 1 && plan_fuse_enabled())) {
    Tail2Args t{};
    t.M = R;
    t.num_kb = p->m1 / 64;
    t.b2 = p->b2;
    t.b3 = p->b3;
    t.w4 = p->w4;
    t.b4 = p->b4;
    t.n_tok = n_tok;
    t.max_ctx = max_ctx_len;
    t.y_hat = y_hat;
    t.n_hat = n_hat;
    t.done = p->tail2_done;
    t.project = proj ? 1 : 0;
    if (proj) t.pa = *proj;
    t.tl = p->tl;
    if (p->tl) p->tl_ctas = 4 * m_tiles;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(4, m_tiles, 1);
    cfg.blockDim = dim3(192, 1, 1);
    cfg.dynamicSmemBytes = Tail2Smem::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, tail2_kernel, p->tmA2, p->tmW2t, p->tmB3, t);
    if (e != cudaSuccess) return cuda_fail(e, "tail2 launch");
    return STAR_OK;
  }
  // ---- fused tail: layer 2 -> layer 3 -> head -> quantizer [-> projection] ----
  const int n2 = p->m2 / 256;
  const int num_kb2 = p->m1 * 2 / 128;
  const int ts = (!f32 && p->bn2 == 256 && p->m3 == 64) ? tail_splits(m_tiles, n2, num_kb2) : 0;
  if (ts) {
    TailArgs t{};
    t.M = R;
    t.num_kb = num_kb2;
    t.splits = ts;
    t.kb_per_split = (num_kb2 + ts - 1) / ts;
    t.n2_tiles = n2;
    t.b2 = p->b2;
    t.b3 = p->b3;
    t.w4 = p->w4;
    t.b4 = p->b4;
    t.n_tok = n_tok;
    t.max_ctx = max_ctx_len;
    t.y_hat = y_hat;
    t.n_hat = n_hat;
    t.ws2 = p->ws;
    t.ws3a = p->ws3;
    t.ws3b = p->ws3 + (size_t)m_tiles * n2 * ts * 64 * 128;
    t.cnt = p->tail_cnt;
    t.tl = p->tl;
    p->tl_ctas = m_tiles * n2 * ts;
    t.project = proj ? 1 : 0;
    if (proj) t.pa = *proj;
    // fused only for a single-round plan: the fused form runs on the tail's 192 threads, where a
    // multi-round plan (C4, max_moves = 4: ~17 us per round) is slower than the 512-thread plan
    // kernel it would save the launch of
    if (proj && plan && plan->world == 1 && plan->max_moves <= 1 && plan_fuse_enabled() &&
        plan_fast_smem_layout(plan->n, plan->H, 1, plan->r_cap) + 256 <= (size_t)TailSmem::OFF_W3) {
      t.plan = 1;   // Alg. 1 by the projection's last finisher: no plan launch, no kernel boundary
      t.pl = *plan;
      // round-0 W_i from the projection itself when it writes them into the plan's own L record:
      // W = sum beta_t L[t] in int64 is exact in the projection's validated domain (<= 65536
      // requests per instance, N <= 2^17, H <= 256: every term < 2^49, the sum < 2^57)
      if (proj->W && proj->L == plan->L) t.pl.W0 = proj->W;
      if (plan_fused) *plan_fused = true;
    }
    cudaError_t e = launch_tail(p->tmA2, p->tmB2, p->tmB3, t, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "fused tail launch");
    return STAR_OK;
  }
  // ---- layer 2: Z2 = relu(W2 Z1 + b2) ----
  {
    const int num_kb = (p->m1 * kx * (f32 ? 4 : 2)) / 128;
    g.N = p->m2;
    g.num_kb = num_kb;
    plan_splits(m_tiles * (p->m2 / p->bn2), num_kb, p->bn2, f32, &g.splits, &g.kb_per_split);
    g.epi = f32 ? EPI_RELU_TF32X3 : EPI_RELU_BF16;
    g.tma_store = (!f32 && (p->bn2 / g.splits) % 64 == 0) ? 1 : 0;
    g.out = p->Z2;
    g.ld_out = (int64_t)p->m2 * kx;
    g.bias = p->b2;
    cudaError_t e = launch_gemm(p->bn2, f32, p->tmA2, p->tmB2, tmC2, g, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "layer-2 GEMM launch");
  }
  // ---- layer 3 + head: z3 = relu(W3 Z2 + b3); y = w4 . z3 + b4; N_hat = quantize(y) ----
  {
    const int num_kb = (p->m2 * kx * (f32 ? 4 : 2)) / 128;
    g.N = p->m3;
    g.num_kb = num_kb;
    plan_splits(m_tiles, num_kb, 64, f32, &g.splits, &g.kb_per_split);
    g.epi = EPI_HEAD;
    g.tma_store = 0;
    g.out = nullptr;
    g.ld_out = 0;
    g.bias = p->b3;
    g.w4 = p->w4;
    g.b4 = p->b4;
    g.n_tok = n_tok;
    g.y_hat = y_hat;
    g.n_hat = n_hat;
    cudaError_t e = launch_gemm(64, f32, p->tmA3, p->tmB3, p->tmA3, g, m_tiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "layer-3/head GEMM launch");
  }
  if (proj) {   // unfused shapes: the standalone projection kernel on the forward's N_hat
    cudaError_t e = launch_project(R, proj->n_inst, proj->inst_base, proj->H, proj->inst, n_tok, n_hat, proj->beta_q,
                                   proj->L, proj->W, proj->peak, proj->growth, proj->count, proj_ws, proj->err, st,
                                   nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "project_kernel launch");
  }
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
  return forward_impl(p, h, ld_h, R, n_tok, max_ctx_len, y_hat, n_hat, nullptr, nullptr,
                      reinterpret_cast<cudaStream_t>(stream_));
}

star_status lenpred_forward_project(star_predictor* p, const void* h, int64_t ld_h, int R, const int32_t* n_tok,
                                    int32_t max_ctx_len, float* y_hat, int32_t* n_hat, int n_inst, int inst_base,
                                    int H, const int32_t* inst, const uint32_t* beta_q, int64_t* L, int64_t* W,
                                    int64_t* peak, int64_t* growth, int32_t* count, void* workspace,
                                    int32_t* err_flag, star_stream_t stream_) {
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  if (R < 0 || R > p->max_rows) return fail(STAR_ERANGE, "R=%d outside [0, max_rows=%d]", R, p->max_rows);
  if (n_inst < 1 || n_inst > (1 << 16)) return fail(STAR_ERANGE, "n_inst=%d outside [1, 65536]", n_inst);
  if (H < 0 || H > 256) return fail(STAR_ERANGE, "H=%d outside [0, 256]", H);
  if (!L || !beta_q || !workspace || !n_hat) return fail(STAR_EINVAL, "L, beta_q, workspace and n_hat must be non-NULL");
  if (max_ctx_len < 0) return fail(STAR_EINVAL, "max_ctx_len < 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  if (R == 0) {   // empty batch: zero loads from the standalone kernel
    cudaError_t e = launch_project(0, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                                   workspace, err_flag, st, nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "project_kernel launch");
    return STAR_OK;
  }
  if (!h || !inst || !n_tok) return fail(STAR_EINVAL, "h, inst and n_tok must be non-NULL");
  if (ld_h < p->d) return fail(STAR_EINVAL, "ld_h=%lld < d=%d", (long long)ld_h, p->d);
  ProjArgs pa = make_proj_args(R, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                               workspace, err_flag);
  return forward_impl(p, h, ld_h, R, n_tok, max_ctx_len, y_hat, n_hat, &pa, workspace, st);
}

static star_status check_plan_params(const star_plan_params* p);

star_status lenpred_forward_project_plan(star_predictor* p, const void* h, int64_t ld_h, int R,
                                         const int32_t* n_tok, int32_t max_ctx_len, float* y_hat, int32_t* n_hat,
                                         int n_inst, int H, const int32_t* inst, const uint32_t* beta_q, int64_t* L,
                                         int64_t* W, int64_t* peak, int64_t* growth, int32_t* count, void* workspace,
                                         const star_plan_params* pp, const star_plan_segments* sg,
                                         star_move* moves, int32_t* n_moves, int32_t* err_flag,
                                         star_stream_t stream_) {
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  star_status s = check_plan_params(pp);
  if (s != STAR_OK) return s;
  if (!sg || !sg->L) return fail(STAR_EINVAL, "segments / L is NULL");
  if (sg->world != 1 || sg->n_loc != n_inst || pp->n_inst != n_inst || pp->H != H)
    return fail(STAR_EINVAL, "one-rank step: segments world must be 1 and n_inst / H must match the plan");
  if (!n_moves || (pp->max_moves > 0 && !moves)) return fail(STAR_EINVAL, "moves / n_moves is NULL");
  if (sg->r_cap < R) return fail(STAR_EINVAL, "segment r_cap=%d < R=%d", sg->r_cap, R);
  if (sg->r_cap > 0 && (!sg->req_id || !sg->inst || !sg->n_tok || !sg->n_hat))
    return fail(STAR_EINVAL, "request arrays must be non-NULL");
  const size_t smem = plan_smem_bytes(pp->n_inst, pp->H, 1, sg->r_cap) + 2048;
  if (smem > (size_t)kMaxSmemBytes)
    return fail(STAR_ENOTSUP, "plan state (%zu B) exceeds shared memory: n_inst*(H+1) too large", smem);
  if (R < 0 || R > p->max_rows) return fail(STAR_ERANGE, "R=%d outside [0, max_rows=%d]", R, p->max_rows);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  bool fused = false;
  if (R > 0) {
    if (n_inst < 1 || n_inst > (1 << 16)) return fail(STAR_ERANGE, "n_inst=%d outside [1, 65536]", n_inst);
    if (H < 0 || H > 256) return fail(STAR_ERANGE, "H=%d outside [0, 256]", H);
    if (!L || !beta_q || !workspace || !n_hat) return fail(STAR_EINVAL, "L, beta_q, workspace and n_hat must be non-NULL");
    if (max_ctx_len < 0) return fail(STAR_EINVAL, "max_ctx_len < 0");
    if (!h || !inst || !n_tok) return fail(STAR_EINVAL, "h, inst and n_tok must be non-NULL");
    if (ld_h < p->d) return fail(STAR_EINVAL, "ld_h=%lld < d=%d", (long long)ld_h, p->d);
    ProjArgs pa = make_proj_args(R, n_inst, 0, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count, workspace,
                                 err_flag);
    const PlanArgs pl = make_plan_args(pp, sg, moves, n_moves, err_flag);
    s = forward_impl(p, h, ld_h, R, n_tok, max_ctx_len, y_hat, n_hat, &pa, workspace, st, &pl, &fused);
  } else {
    s = lenpred_forward_project(p, h, ld_h, 0, n_tok, max_ctx_len, y_hat, n_hat, n_inst, 0, H, inst, beta_q, L, W,
                                peak, growth, count, workspace, err_flag, stream_);
  }
  if (s != STAR_OK || fused) return s;
  cudaError_t e = launch_plan(pp, sg, moves, n_moves, err_flag, st);
  if (e != cudaSuccess) return cuda_fail(e, "plan_kernel launch");
  return STAR_OK;
}

static star_status refresh_impl(star_predictor* p, const void* h, int64_t ld_h, int R, const int32_t* n_tok,
                                int32_t max_ctx_len, const int32_t* gen, int32_t* g_last, int32_t* nhat_last,
                                int32_t k, int32_t* n_hat, int32_t* n_refreshed, const ProjArgs* proj,
                                star_stream_t stream_) {
  if (!p) return fail(STAR_EINVAL, "predictor is NULL");
  if (p->f32 || p->bn2 != 256 || p->m3 != 64)
    return fail(STAR_ENOTSUP, "refresh mode needs a bf16 predictor (m2 %% 256 == 0, m3 == 64)");
  if (R < 0 || R > p->max_rows) return fail(STAR_ERANGE, "R=%d outside [0, max_rows=%d]", R, p->max_rows);
  if (k < 1) return fail(STAR_EINVAL, "k=%d must be >= 1", k);
  if (max_ctx_len < 0) return fail(STAR_EINVAL, "max_ctx_len < 0");
  if (R == 0) return STAR_OK;
  if (!h || !gen || !g_last || !nhat_last || !n_hat)
    return fail(STAR_EINVAL, "h, gen, g_last, nhat_last, n_hat must be non-NULL");
  if (ld_h < p->d) return fail(STAR_EINVAL, "ld_h=%lld < d=%d", (long long)ld_h, p->d);
  if ((reinterpret_cast<uintptr_t>(h) | (uintptr_t)(ld_h * 2)) & 15u)
    return fail(STAR_EINVAL, "h rows must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  cudaError_t e;
  if (p->small_ok && R <= refresh_select_fused_max_rows() && R <= 64 * 512) {
    // one-launch path: the multi-CTA select compacts + gathers the due rows, ages the others (and
    // projects them); the small-batch predictor runs the due rows in 512-row chunks, scatters their
    // N_hat into their slots, adds them to the projection and finalises it
    if ((e = launch_refresh_select_fused(R, gen, g_last, nhat_last, k, n_tok, h, ld_h * 2, p->d * 2, p->r_idx,
                                         p->r_ntok, p->r_h, n_hat, p->r_M, n_refreshed, p->r_blk, proj, st, p->tl)) !=
        cudaSuccess)
      return cuda_fail(e, "refresh select launch");
    SmallRefresh rf{(R + k - 1) / k, p->r_M, p->r_idx, gen, g_last, nhat_last, n_hat};
    if ((e = launch_small(p, R, n_tok ? p->r_ntok : nullptr, max_ctx_len, nullptr, nullptr, proj, st, &p->tmA_r,
                          &rf)) != cudaSuccess)
      return cuda_fail(e, "refresh small-batch launch");
    return STAR_OK;
  }
  if ((e = launch_refresh_select(R, gen, g_last, k, n_tok, p->r_idx, p->r_ntok, p->r_pos, p->r_M, st)) != cudaSuccess)
    return cuda_fail(e, "refresh_select launch");
  if ((e = launch_refresh_gather(R, h, ld_h * 2, p->d * 2, p->r_idx, p->r_M, p->r_h, st)) != cudaSuccess)
    return cuda_fail(e, "refresh_gather launch");
  const int skip_le = 0;   // (the 2-launch kernels run every row here)
  // layer 1 on the compacted rows: 1-CTA tiles + cluster split-K sized for the expected row count
  // ~R/k (the grid covers R rows; tiles beyond the device-side count leave before any setup)
  const int m_tiles = (R + 127) / 128;
  const int m_est = ((R + k - 1) / k + 127) / 128;
  GemmArgs g{};
  g.M = R;
  g.M_dev = p->r_M;
  g.skip_le = skip_le;
  g.max_ctx = max_ctx_len;
  g.head_ws = p->head_ws;
  g.N = p->m1;
  g.num_kb = (p->d * 2 + 127) / 128;
  plan_splits((m_est < 1 ? 1 : m_est) * (p->m1 / p->bn1), g.num_kb, p->bn1, false, &g.splits, &g.kb_per_split);
  if (g.splits > 4) {   // the refresh partial workspace holds 4 splits of every m-tile
    g.splits = 4;
    g.kb_per_split = (g.num_kb + 3) / 4;
  }
  g.ws = p->r_ws;
  g.mn_swap = 1;   // the device-side row count leaves most m-tiles empty: launch the real ones first
  g.epi = EPI_RELU_BF16;
  g.tma_store = (p->bn1 / g.splits) % 64 == 0 ? 1 : 0;
  g.out = p->Z1;
  g.ld_out = p->m1;
  g.bias = p->b1;
  if ((e = launch_gemm(p->bn1, false, p->tmA_r, p->tmB1, p->tmC1, g, m_tiles, st)) != cudaSuccess)
    return cuda_fail(e, "refresh layer-1 launch");
  const int n2 = p->m2 / 256;
  const int num_kb2 = p->m1 * 2 / 128;
  const int ts = tail_splits(m_est < 1 ? 1 : m_est, n2, num_kb2);
  if (!ts) return fail(STAR_ENOTSUP, "shape not supported by the fused tail");
  TailArgs t{};
  t.M = R;
  t.M_dev = p->r_M;
  t.skip_le = skip_le;
  t.mn_swap = 1;
  t.num_kb = num_kb2;
  t.splits = ts;
  t.kb_per_split = (num_kb2 + ts - 1) / ts;
  t.n2_tiles = n2;
  t.b2 = p->b2;
  t.b3 = p->b3;
  t.w4 = p->w4;
  t.b4 = p->b4;
  t.n_tok = n_tok ? p->r_ntok : nullptr;
  t.max_ctx = max_ctx_len;
  t.y_hat = nullptr;
  t.n_hat = p->r_nhat;
  t.ws2 = p->ws;
  t.ws3a = p->ws3;
  t.ws3b = p->ws3 + (size_t)m_tiles * n2 * ts * 64 * 128;
  t.cnt = p->tail_cnt;
  t.project = 0;
  if ((e = launch_tail(p->tmA2, p->tmB2, p->tmB3, t, m_tiles, st)) != cudaSuccess)
    return cuda_fail(e, "refresh tail launch");
  if (proj && R <= 8192 && refresh_scatter_project_smem(proj->n_inst, proj->H) <= (size_t)200 * 1024) {
    // aging scatter fused with the projection of the resulting N_hat (one CTA)
    if ((e = launch_refresh_scatter_project(*proj, p->r_pos, p->r_nhat, gen, g_last, nhat_last, p->r_M, n_refreshed,
                                            st)) != cudaSuccess)
      return cuda_fail(e, "refresh_scatter_project launch");
    return STAR_OK;
  }
  if ((e = launch_refresh_scatter(R, p->r_pos, p->r_nhat, gen, g_last, nhat_last, n_hat, p->r_M, n_refreshed, st)) !=
      cudaSuccess)
    return cuda_fail(e, "refresh_scatter launch");
  if (proj) {
    const ProjArgs& a = *proj;
    if ((e = launch_project(a.R, a.n_inst, a.inst_base, a.H, a.inst, a.n_tok, a.n_hat, a.beta_q, a.L, a.W, a.peak,
                            a.growth, a.count, a.ws_sum, a.err, st, nullptr)) != cudaSuccess)
      return cuda_fail(e, "projection launch");
  }
  return STAR_OK;
}

star_status lenpred_forward_refresh(star_predictor* p, const void* h, int64_t ld_h, int R, const int32_t* n_tok,
                                    int32_t max_ctx_len, const int32_t* gen, int32_t* g_last, int32_t* nhat_last,
                                    int32_t k, int32_t* n_hat, int32_t* n_refreshed, star_stream_t stream_) {
  return refresh_impl(p, h, ld_h, R, n_tok, max_ctx_len, gen, g_last, nhat_last, k, n_hat, n_refreshed, nullptr,
                      stream_);
}

star_status lenpred_forward_refresh_project(star_predictor* p, const void* h, int64_t ld_h, int R,
                                            const int32_t* n_tok, int32_t max_ctx_len, const int32_t* gen,
                                            int32_t* g_last, int32_t* nhat_last, int32_t k, int32_t* n_hat,
                                            int32_t* n_refreshed, int n_inst, int inst_base, int H,
                                            const int32_t* inst, const uint32_t* beta_q, int64_t* L, int64_t* W,
                                            int64_t* peak, int64_t* growth, int32_t* count, void* workspace,
                                            int32_t* err_flag, star_stream_t stream_) {
  if (n_inst < 1 || n_inst > (1 << 16)) return fail(STAR_ERANGE, "n_inst=%d outside [1, 65536]", n_inst);
  if (H < 0 || H > 256) return fail(STAR_ERANGE, "H=%d outside [0, 256]", H);
  if (!L || !beta_q || !workspace) return fail(STAR_EINVAL, "L, beta_q and workspace must be non-NULL");
  if (R > 0 && (!inst || !n_tok)) return fail(STAR_EINVAL, "inst and n_tok must be non-NULL");
  if (R == 0)
    return project_instance_load(0, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                                 workspace, err_flag, stream_);
  const ProjArgs a = make_proj_args(R, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                                    workspace, err_flag);
  return refresh_impl(p, h, ld_h, R, n_tok, max_ctx_len, gen, g_last, nhat_last, k, n_hat, n_refreshed, &a, stream_);
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
  if ((size_t)n_inst * (H + 2) > 16384 && !workspace)
    return fail(STAR_EINVAL, "n_inst*(H+2) > 16384 requires a workspace");
  cudaError_t e = launch_project(R, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                                 workspace, err_flag, reinterpret_cast<cudaStream_t>(stream_), nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "project_kernel launch");
  return STAR_OK;
}

size_t star_dispatch_workspace_bytes(int n_inst, int H) {
  if (n_inst < 1 || H < 0) return 0;
  return dispatch_workspace_bytes(n_inst, H);
}

star_status dispatch_requests(int policy, int n_inst, int H, const uint32_t* beta_q, int64_t* L, const int64_t* c_mem,
                              const int64_t* reserved, int A, const int32_t* n_tok, const int32_t* n_hat,
                              int32_t counter, int32_t* assign, void* workspace, star_stream_t stream_) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  if (policy < STAR_DISPATCH_ROUND_ROBIN || policy > STAR_DISPATCH_PROJECTED)
    return fail(STAR_EINVAL, "unknown dispatch policy %d", policy);
  if (n_inst < 1 || n_inst > (1 << 16)) return fail(STAR_ERANGE, "n_inst=%d outside [1, 65536]", n_inst);
  if (H < 0 || H > 256) return fail(STAR_ERANGE, "H=%d outside [0, 256]", H);
  if (A < 0) return fail(STAR_EINVAL, "A < 0");
  if (counter < 0) return fail(STAR_EINVAL, "counter < 0");
  if (A == 0) return STAR_OK;
  if (!L || !beta_q || !n_tok || !n_hat || !assign) return fail(STAR_EINVAL, "L, beta_q, n_tok, n_hat, assign must be non-NULL");
  if (policy == STAR_DISPATCH_PROJECTED && !workspace)
    return fail(STAR_EINVAL, "the projected policy needs a workspace of star_dispatch_workspace_bytes()");
  cudaError_t e = launch_dispatch(policy, n_inst, H, beta_q, L, c_mem, reserved, A, n_tok, n_hat, counter, assign,
                                  workspace, reinterpret_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "dispatch_kernel launch");
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

star_status star_plan_timeline(uint64_t* host64) {
  if (!host64) return fail(STAR_EINVAL, "host64 is NULL");
  STAR_CUDA(cudaDeviceSynchronize());
  STAR_CUDA(plan_timeline(host64));
  return STAR_OK;
}

size_t star_plan_workspace_bytes(int n_inst, int H, int64_t request_slots) {
  if (n_inst < 1 || H < 0 || request_slots < 0) return 0;
  return plan_large_workspace_bytes(n_inst, H, request_slots);
}

star_status plan_reschedule_segmented_ws(const star_plan_params* p, const star_plan_segments* sg, star_move* moves,
                                         int32_t* n_moves, int32_t* err_flag, void* workspace,
                                         star_stream_t stream_) {
  if (!workspace) return plan_reschedule_segmented(p, sg, moves, n_moves, err_flag, stream_);
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
  if (!plan_large_supported(p->n_inst)) return fail(STAR_ENOTSUP, "n_inst=%d above the multi-CTA plan limit", p->n_inst);
  const PlanArgs a = make_plan_args(p, sg, moves, n_moves, err_flag);
  cudaError_t e = launch_plan_large(a, workspace, reinterpret_cast<cudaStream_t>(stream_));
  if (e != cudaSuccess) return cuda_fail(e, "plan_large launch");
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

star_status kv_pack(const star_kv_pool* src, const int32_t* table, int n, void* staging, int32_t* err_flag,
                    star_stream_t stream) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  std::string msg;
  if (!src) return fail(STAR_EINVAL, "kv_pack: src is NULL");
  s = kv_copy_checked(src, table, nullptr, nullptr, n, nullptr, staging, err_flag,
                      reinterpret_cast<cudaStream_t>(stream), &msg);
  return s == STAR_OK ? s : fail(s, "kv_pack: %s", msg.c_str());
}

star_status kv_unpack(const void* staging, const star_kv_pool* dst, const int32_t* table, int n, int32_t* err_flag,
                      star_stream_t stream) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  std::string msg;
  if (!dst) return fail(STAR_EINVAL, "kv_unpack: dst is NULL");
  s = kv_copy_checked(nullptr, nullptr, dst, table, n, const_cast<void*>(staging), nullptr, err_flag,
                      reinterpret_cast<cudaStream_t>(stream), &msg);
  return s == STAR_OK ? s : fail(s, "kv_unpack: %s", msg.c_str());
}

star_status kv_migrate(const star_kv_pool* src, const int32_t* src_table, const star_kv_pool* dst,
                       const int32_t* dst_table, int n, int32_t* err_flag, star_stream_t stream) {
  star_status s = ensure_device();
  if (s != STAR_OK) return s;
  std::string msg;
  if (!src || !dst) return fail(STAR_EINVAL, "kv_migrate: src and dst must be non-NULL");
  s = kv_copy_checked(src, src_table, dst, dst_table, n, nullptr, nullptr, err_flag,
                      reinterpret_cast<cudaStream_t>(stream), &msg);
  return s == STAR_OK ? s : fail(s, "kv_migrate: %s", msg.c_str());
}

}  // extern "C"

namespace star {
static cudaError_t launch_small(star_predictor* p, int R, const int32_t* n_tok, int32_t max_ctx, float* y_hat,
                                int32_t* n_hat, const ProjArgs* proj, cudaStream_t st, const CUtensorMap* tmH,
                                const SmallRefresh* rf) {
  SmallArgs a{};
  if (rf) {
    a.M_dev = rf->M_dev;
    a.r_idx = rf->idx;
    a.r_gen = rf->gen;
    a.r_glast = rf->g_last;
    a.r_nhat_last = rf->nhat_last;
    a.r_nhat = rf->n_hat;
  }
  a.M = R;
  a.kb1 = p->d / 64;
  a.b1 = p->b1;
  a.b2 = p->b2;
  a.b3 = p->b3;
  a.w4 = p->w4;
  a.b4 = p->b4;
  a.n_tok = n_tok;
  a.max_ctx = max_ctx;
  a.y_hat = y_hat;
  a.n_hat = n_hat;
  a.Z1 = static_cast<__nv_bfloat16*>(p->Z1);
  a.Z2 = static_cast<__nv_bfloat16*>(p->Z2);
  a.cnt = p->small_cnt;
  a.project = proj ? 1 : 0;
  if (proj) a.pa = *proj;
  a.tl = p->tl;   // diagnostics (star_predictor_timeline): [CTAs][32] phase stamps
  if (p->tl) p->tl_ctas = 128;
  cudaLaunchConfig_t cfg{};
  // 128 CTAs whatever the row count: 1 m-tile -> 32-column layer-1 tiles (64 per m-tile), 2 -> 64,
  // 3-4 -> 128 (refresh: sized for the expected due rows; more rows run in further chunks)
  const int rows = rf ? (rf->rows_expected < R ? rf->rows_expected : R) : R;
  int mt = (rows + 127) / 128;
  mt = mt < 1 ? 1 : (mt > 4 ? 4 : mt);
  const int n1 = mt == 1 ? 32 : (mt == 2 ? 64 : 128);
  a.n1 = n1;
  cfg.gridDim = dim3(2, 2048 / n1, mt);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = SmallSmem::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const CUtensorMap& tmW1 = n1 == 32 ? p->tmW1n[0] : (n1 == 64 ? p->tmW1n[1] : p->tmB1p);
  return cudaLaunchKernelEx(&cfg, lenpred_small_kernel, tmH ? *tmH : p->tmA1, tmW1, p->tmA2, p->tmW2s, p->tmA3,
                            p->tmB3, a);
}

static cudaError_t launch_f32_small(star_predictor* p, int R, const int32_t* n_tok, int32_t max_ctx, float* y_hat,
                                    int32_t* n_hat, const ProjArgs* proj, cudaStream_t st) {
  F32Args a{};
  a.M = R;
  a.kb1 = p->d / 32;
  a.b1 = p->b1;
  a.b2 = p->b2;
  a.b3 = p->b3;
  a.w4 = p->w4;
  a.b4 = p->b4;
  a.n_tok = n_tok;
  a.max_ctx = max_ctx;
  a.y_hat = y_hat;
  a.n_hat = n_hat;
  a.Z1 = static_cast<float*>(p->Z1);
  a.Z2 = static_cast<float*>(p->Z2);
  a.P1 = p->ws;
  a.P2 = a.P1 + 4 * 32 * 16 * 512;
  a.P3 = a.P2 + 8 * 16 * 8 * 512;
  a.yp = a.P3 + 8 * 16 * 512;
  a.cnt = p->f32_cnt;
  a.project = proj ? 1 : 0;
  if (proj) a.pa = *proj;
  a.tl = p->tl;   // diagnostics (star_predictor_timeline): [128][32] phase stamps
  if (p->tl) p->tl_ctas = 128;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(128, 1, 1);
  cfg.blockDim = dim3(320, 1, 1);
  cfg.dynamicSmemBytes = F32Smem::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lenpred_f32_kernel, p->tmHf, p->tmW1f, p->tmZ1f, p->tmW2f, p->tmZ2f, p->tmW3f, a);
}
}  // namespace star
