// refresh.cu -- prediction cadence k (NEXT-1): the paper predicts "at regular
// intervals" and sets the interval to k = 20 decode iterations to cut the
// predictor's overhead from 7.68% to 0.38%.  A request is re-predicted when
// it has no prediction yet or has generated >= k tokens since its last one (SPEC.md:164-172
// should_refresh); in between, its remaining-length prediction ages by the tokens generated since
// (reading A27): N_hat = max(0, N_hat_last - (g - g_last)).
//
//   refresh_select_kernel   one CTA: flags, block scan -> compacted row list idx[0..M), the
//                           rows' N(r), each row's compact position (or -1) and M on the device
//   refresh_gather_kernel   copies the M selected hidden-state rows into a contiguous buffer
//                           (16-byte vectors); the predictor kernels then run on it with the
//                           device-side row count (CTAs beyond M exit at once)
//   refresh_scatter_kernel  per row: refreshed -> new N_hat, g_last = g, N_hat_last = N_hat;
//                           else the aged value
//   refresh_scatter_project_kernel  the scatter fused with the per-instance projection of the
//                           resulting N_hat (one CTA, shared-memory histogram + finalize): one
//                           launch and one N_hat round trip fewer per step
#include <cstdint>
#include <cuda_runtime.h>
#include "project_core.cuh"
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

constexpr int kSelThreads = 1024;

__global__ void __launch_bounds__(kSelThreads) refresh_select_kernel(int R, const int32_t* __restrict__ gen,
                                                                     const int32_t* __restrict__ g_last, int32_t k,
                                                                     const int32_t* __restrict__ n_tok,
                                                                     int32_t* __restrict__ idx,
                                                                     int32_t* __restrict__ ntok_c,
                                                                     int32_t* __restrict__ pos,
                                                                     int32_t* __restrict__ M_out) {
  __shared__ int wsum[kSelThreads / 32];
  __shared__ int s_base;
  pdl_wait();
  pdl_launch_dependents();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int base = 0; base < R; base += kSelThreads) {
    const int r = base + tid;
    bool f = false;
    if (r < R) {
      const int gl = g_last[r];
      f = gl < 0 || gen[r] - gl >= k;   // should_refresh
    }
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the 32 warp counts
      const int v = wsum[lane];
      int x = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
      }
      wsum[lane] = x - v;
    }
    __syncthreads();
    const int p = s_base + wsum[warp] + __popc(m & ((1u << lane) - 1u));
    if (r < R) {
      pos[r] = f ? p : -1;
      if (f) {
        idx[p] = r;
        ntok_c[p] = n_tok ? n_tok[r] : 0;
      }
    }
    __syncthreads();
    if (tid == kSelThreads - 1) s_base = p + (f ? 1 : 0);
    __syncthreads();
  }
  if (tid == 0) *M_out = s_base;
}

__global__ void __launch_bounds__(256) refresh_gather_kernel(const uint8_t* __restrict__ h, int64_t ld_bytes,
                                                             int row_bytes, const int32_t* __restrict__ idx,
                                                             const int32_t* __restrict__ M_dev,
                                                             uint8_t* __restrict__ hc) {
  pdl_wait();
  pdl_launch_dependents();
  const int M = __ldcg(M_dev);
  const int nvec = row_bytes / 16;
  for (int p = blockIdx.x; p < M; p += gridDim.x) {
    const int4* src = reinterpret_cast<const int4*>(h + (int64_t)idx[p] * ld_bytes);
    int4* dst = reinterpret_cast<int4*>(hc + (int64_t)p * row_bytes);
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = __ldg(src + v);
  }
}

__global__ void __launch_bounds__(256) refresh_scatter_kernel(int R, const int32_t* __restrict__ pos,
                                                              const int32_t* __restrict__ nhat_c,
                                                              const int32_t* __restrict__ gen, int32_t* g_last,
                                                              int32_t* nhat_last, int32_t* __restrict__ n_hat,
                                                              const int32_t* __restrict__ M_dev,
                                                              int32_t* __restrict__ n_refreshed) {
  pdl_wait();
  pdl_launch_dependents();
  if (n_refreshed && blockIdx.x == 0 && threadIdx.x == 0) *n_refreshed = *M_dev;   // (no memcpy node in the chain)
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const int p = pos[r];
    const int g = gen[r];
    int nh;
    if (p >= 0) {
      nh = nhat_c[p];
      g_last[r] = g;
      nhat_last[r] = nh;
    } else {
      const int aged = nhat_last[r] - (g - g_last[r]);   // reading A27
      nh = aged > 0 ? aged : 0;
    }
    n_hat[r] = nh;
  }
}

constexpr int kScatProjThreads = 1024;
__global__ void __launch_bounds__(kScatProjThreads) refresh_scatter_project_kernel(
    const ProjArgs a, const int32_t* __restrict__ pos, const int32_t* __restrict__ nhat_c,
    const int32_t* __restrict__ gen, int32_t* g_last, int32_t* nhat_last, const int32_t* __restrict__ M_dev,
    int32_t* __restrict__ n_refreshed) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int nb = a.n_inst * (a.H + 2);
  unsigned long long* ssum = reinterpret_cast<unsigned long long*>(sm);
  uint32_t* scnt = reinterpret_cast<uint32_t*>(ssum + nb);
  __shared__ uint32_t sbeta[257];
  for (int k = threadIdx.x; k < nb; k += blockDim.x) {
    ssum[k] = 0;
    scnt[k] = 0;
  }
  pdl_wait();
  pdl_launch_dependents();
  for (int t = threadIdx.x; t <= a.H; t += blockDim.x) sbeta[t] = a.beta_q[t];
  if (n_refreshed && threadIdx.x == 0) *n_refreshed = *M_dev;
  __syncthreads();
  uint32_t errbits = 0;
  int32_t* n_hat = const_cast<int32_t*>(a.n_hat);
  for (int base = 0; base < a.R; base += blockDim.x) {   // CTA-uniform trip count: whole warps call
    const int r = base + (int)threadIdx.x;
    const bool valid = r < a.R;
    int nh = 0, ins = 0, nt = 0;
    if (valid) {
      const int p = pos[r];
      const int g = gen[r];
      if (p >= 0) {                       // re-predicted this step
        nh = nhat_c[p];
        g_last[r] = g;
        nhat_last[r] = nh;
      } else {                            // aged (reading A27)
        const int aged = nhat_last[r] - (g - g_last[r]);
        nh = aged > 0 ? aged : 0;
      }
      n_hat[r] = nh;
      ins = a.inst[r];
      nt = a.n_tok[r];
    }
    proj_accumulate<true>(a, valid, ins, nt, nh, scnt, ssum, errbits);
  }
  if (errbits && a.err) atomicOr(a.err, (int)errbits);
  __syncthreads();
  proj_finalize(a, scnt, ssum, sbeta, threadIdx.x >> 5, blockDim.x >> 5);
}

// Multi-CTA select for the one-launch predictor (refresh_select_gather_age_kernel): grid
// ceil(R / 1024) CTAs, all resident (<= SMs, checked on the host).  Per CTA: the due flags of its
// 1024 rows and their block scan; the CTA counts meet in global memory (arrival counter) so every
// CTA knows its base -- the compaction keeps row order, as the single-CTA select does; the CTA
// then writes idx / N(r) of its due rows and copies their hidden states into the compacted
// buffer (one warp per row, 16-byte vectors).  Rows that are NOT due age in place (reading A27)
// and, with the projection fused, go into its histogram here -- they do not depend on the
// predictor -- while the predictor adds the due rows and finalises.
struct SelArgs {
  int R;
  const int32_t* gen;
  const int32_t* g_last;
  const int32_t* nhat_last;
  int32_t k;
  const int32_t* n_tok;
  const uint8_t* h;
  int64_t ld_bytes;
  int row_bytes;
  int32_t* idx;          // [R] compacted position -> row
  int32_t* ntok_c;       // [R] N(r) of the compacted rows
  uint8_t* hc;           // [R][row_bytes] compacted hidden states
  int32_t* n_hat;        // [R] aged N_hat of the rows that are not due
  int32_t* M_out;        // device row count
  int32_t* n_refreshed;  // nullable
  int* blk;              // [grid] CTA counts | [grid] arrival | [grid + 1] done  (zero between launches)
  int project;
  ProjArgs pa;
  uint64_t* tl;          // diagnostics: rows [400 + CTA][32] of the predictor's timeline buffer, or nullptr
};

constexpr int kSelHistBins = 2560;
#define SEL_TS(k)                                                                 \
  do {                                                                            \
    if (a.tl && threadIdx.x == 0) a.tl[(400 + blockIdx.x) * 32 + (k)] = globaltimer_ns(); \
  } while (0)   // shared histogram of the aged rows (n_inst * (H + 2) <= this)

// 128 rows per CTA (the gather of the due rows' hidden states spreads over R / 128 SMs: with 1024
// rows per CTA, two CTAs gathered the C2 step's ~100 rows and the kernel took ~21 us)
constexpr int kSel2Threads = 128;

constexpr uint32_t kSelStageBytes = 160u * 1024u;   // gather staging: the CTA's due rows, chunked

__global__ void __launch_bounds__(kSel2Threads) refresh_select_gather_age_kernel(const SelArgs a) {
  extern __shared__ __align__(128) uint8_t stage[];   // kSelStageBytes
  __shared__ uint64_t gbar;
  __shared__ int wsum[kSel2Threads / 32];
  __shared__ int s_base, s_cnt;
  __shared__ int s_rows[kSel2Threads];
  __shared__ unsigned long long s_sum[kSelHistBins];
  __shared__ uint32_t s_hc[kSelHistBins];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = a.project ? a.pa.n_inst * (a.pa.H + 2) : 0;
  const bool shist = nb <= kSelHistBins;   // else the aged rows go straight to the global histogram
  if (shist)
    for (int j = tid; j < nb; j += kSel2Threads) {
      s_sum[j] = 0;
      s_hc[j] = 0;
    }
  SEL_TS(0);
  pdl_wait();
  pdl_launch_dependents();
  SEL_TS(1);
  const int G = gridDim.x, b = blockIdx.x;
  const int r = b * kSel2Threads + tid;
  bool f = false;
  int gl = 0, g = 0, nl = 0, ins = 0, nt = 0;
  if (r < a.R) {   // every per-row input in one round of loads
    gl = a.g_last[r];
    g = a.gen[r];
    nl = a.nhat_last[r];
    if (a.project) ins = a.pa.inst[r];
    if (a.n_tok) nt = a.n_tok[r];
    f = gl < 0 || g - gl >= a.k;   // should_refresh
  }
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
  if (lane == 0) wsum[warp] = __popc(m);
  __syncthreads();
  if (warp == 0) {   // exclusive scan of the 8 warp counts
    const int v = lane < kSel2Threads / 32 ? wsum[lane] : 0;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      __syncwarp();
      const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
      if (lane >= off) x += y;
    }
    if (lane < kSel2Threads / 32) wsum[lane] = x - v;
    if (lane == 31) s_cnt = x;
  }
  __syncthreads();
  const int lp = wsum[warp] + __popc(m & ((1u << lane) - 1u));   // position among this CTA's due rows
  if (f) s_rows[lp] = r;
  __syncthreads();
  // gather, part 1: the due rows' hidden states start streaming into shared memory now (bulk
  // copies, all in flight at once) -- their compacted position is known only after the CTA counts
  // meet below, but the loads do not need it
  const int cnt0 = s_cnt;
  const int rows_per_chunk = (int)(kSelStageBytes / (uint32_t)a.row_bytes);
  if (tid == 0) {   // publish this CTA's count first (the other CTAs wait for it)
    a.blk[b] = cnt0;
    fence_acq_rel_gpu();
    atomicAdd(a.blk + G, 1);
    mbar_init(&gbar, 1);
    fence_barrier_init();
    const int n = cnt0 < rows_per_chunk ? cnt0 : rows_per_chunk;
    if (n > 0) {
      mbar_arrive_expect_tx(&gbar, (uint32_t)(n * a.row_bytes));
      for (int j = 0; j < n; ++j)
        bulk_g2s(stage + (size_t)j * a.row_bytes, a.h + (int64_t)s_rows[j] * a.ld_bytes, (uint32_t)a.row_bytes, &gbar);
    }
  }
  SEL_TS(2);
  // rows that are not due age in place and (fused projection) enter the histogram now
  int nh = 0;
  if (r < a.R && !f) {
    const int aged = nl - (g - gl);   // reading A27
    nh = aged > 0 ? aged : 0;
    a.n_hat[r] = nh;
  }
  if (a.project) {
    // the long-tailed batch puts most rows of an instance in one bin (N_hat > H): aggregate per
    // warp (match_any) into a shared histogram, then one global add per non-empty bin per CTA
    uint32_t errbits = 0;
    const bool valid = r < a.R && !f;
    if (shist)
      proj_accumulate<true>(a.pa, valid, ins, nt, nh, s_hc, s_sum, errbits);
    else
      proj_accumulate(a.pa, valid, ins, nt, nh, a.pa.ws_cnt, a.pa.ws_sum, errbits);
    if (errbits && a.pa.err) atomicOr(a.pa.err, (int)errbits);
    if (shist) {
      __syncthreads();
      for (int j = tid; j < nb; j += kSel2Threads) {
        const uint32_t c = s_hc[j];
        if (c) {
          atomicAdd(a.pa.ws_cnt + j, c);
          atomicAdd(a.pa.ws_sum + j, s_sum[j]);
        }
      }
    }
  }
  SEL_TS(3);
  if (warp == 0) {   // every CTA's count is in: this CTA's base is the sum of the lower CTAs' counts
    if (lane == 0) spin_wait_geq(a.blk + G, G);
    __syncwarp();   // orders the lanes' loads after lane 0's acquire
    int part = 0;   // lanes load the lower CTAs' counts together (one round trip, not b of them)
    for (int j = lane; j < b; j += 32) part += __ldcg(a.blk + j);
    const int base = (int)__reduce_add_sync(0xFFFFFFFFu, (uint32_t)part);
    if (lane == 0) {
      s_base = base;
      if (b == G - 1) {
        *a.M_out = base + s_cnt;
        if (a.n_refreshed) *a.n_refreshed = base + s_cnt;
      }
      if (atomicAdd(a.blk + G + 1, 1) == G - 1) {   // the last reader re-arms the counters
        a.blk[G] = 0;
        a.blk[G + 1] = 0;
      }
    }
  }
  __syncthreads();
  SEL_TS(4);
  const int base = s_base, cnt = s_cnt;
  if (f) {
    a.idx[base + lp] = r;
    a.ntok_c[base + lp] = nt;
  }
  // gather, part 2: each chunk of staged rows goes out to its compacted position (bulk stores);
  // the next chunk (more due rows than shared memory holds) streams in after the stores read it
  if (tid == 0) {
    uint32_t ph = 0;
    for (int j0 = 0; j0 < cnt; j0 += rows_per_chunk) {
      const int n = cnt - j0 < rows_per_chunk ? cnt - j0 : rows_per_chunk;
      mbar_wait(&gbar, ph);
      ph ^= 1u;
      for (int j = 0; j < n; ++j)
        bulk_s2g(a.hc + (int64_t)(base + j0 + j) * a.row_bytes, stage + (size_t)j * a.row_bytes, (uint32_t)a.row_bytes);
      bulk_commit();
      const int j1 = j0 + rows_per_chunk;
      if (j1 < cnt) {
        bulk_wait_read_all();   // the staging buffer was read by the stores
        const int n1 = cnt - j1 < rows_per_chunk ? cnt - j1 : rows_per_chunk;
        mbar_arrive_expect_tx(&gbar, (uint32_t)(n1 * a.row_bytes));
        for (int j = 0; j < n1; ++j)
          bulk_g2s(stage + (size_t)j * a.row_bytes, a.h + (int64_t)s_rows[j1 + j] * a.ld_bytes, (uint32_t)a.row_bytes,
                   &gbar);
      }
    }
    bulk_wait_all();   // the compacted rows are in global memory before the grid completes
  }
  SEL_TS(5);
}

static cudaLaunchConfig_t pdl_cfg(dim3 grid, dim3 block, cudaStream_t st, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cfg;
}

cudaError_t launch_refresh_select(int R, const int32_t* gen, const int32_t* g_last, int32_t k, const int32_t* n_tok,
                                  int32_t* idx, int32_t* ntok_c, int32_t* pos, int32_t* M_out, cudaStream_t st) {
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = pdl_cfg(dim3(1), dim3(kSelThreads), st, at);
  return cudaLaunchKernelEx(&cfg, refresh_select_kernel, R, gen, g_last, k, n_tok, idx, ntok_c, pos, M_out);
}

cudaError_t launch_refresh_gather(int R, const void* h, int64_t ld_bytes, int row_bytes, const int32_t* idx,
                                  const int32_t* M_dev, void* hc, cudaStream_t st) {
  cudaLaunchAttribute at[1];
  int grid = R < 4 * g_num_sms ? (R > 0 ? R : 1) : 4 * g_num_sms;
  cudaLaunchConfig_t cfg = pdl_cfg(dim3(grid), dim3(256), st, at);
  return cudaLaunchKernelEx(&cfg, refresh_gather_kernel, static_cast<const uint8_t*>(h), ld_bytes, row_bytes, idx,
                            M_dev, static_cast<uint8_t*>(hc));
}

cudaError_t launch_refresh_scatter(int R, const int32_t* pos, const int32_t* nhat_c, const int32_t* gen,
                                   int32_t* g_last, int32_t* nhat_last, int32_t* n_hat, const int32_t* M_dev,
                                   int32_t* n_refreshed, cudaStream_t st) {
  cudaLaunchAttribute at[1];
  int grid = (R + 255) / 256;
  grid = grid < 1 ? 1 : (grid > 4 * g_num_sms ? 4 * g_num_sms : grid);
  cudaLaunchConfig_t cfg = pdl_cfg(dim3(grid), dim3(256), st, at);
  return cudaLaunchKernelEx(&cfg, refresh_scatter_kernel, R, pos, nhat_c, gen, g_last, nhat_last, n_hat, M_dev,
                            n_refreshed);
}

size_t refresh_scatter_project_smem(int n_inst, int H) { return (size_t)n_inst * (H + 2) * 12; }

cudaError_t launch_refresh_scatter_project(const ProjArgs& a, const int32_t* pos, const int32_t* nhat_c,
                                           const int32_t* gen, int32_t* g_last, int32_t* nhat_last,
                                           const int32_t* M_dev, int32_t* n_refreshed, cudaStream_t st) {
  const size_t smem = refresh_scatter_project_smem(a.n_inst, a.H);
  if (smem > 48 * 1024) {
    cudaError_t e = func_attr((const void*)refresh_scatter_project_kernel,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute at[1];
  cudaLaunchConfig_t cfg = pdl_cfg(dim3(1), dim3(kScatProjThreads), st, at);
  cfg.dynamicSmemBytes = smem;
  return cudaLaunchKernelEx(&cfg, refresh_scatter_project_kernel, a, pos, nhat_c, gen, g_last, nhat_last, M_dev,
                            n_refreshed);
}

cudaError_t launch_refresh_select_fused(int R, const int32_t* gen, const int32_t* g_last, const int32_t* nhat_last,
                                        int32_t k, const int32_t* n_tok, const void* h, int64_t ld_bytes, int row_bytes,
                                        int32_t* idx, int32_t* ntok_c, void* hc, int32_t* n_hat, int32_t* M_out,
                                        int32_t* n_refreshed, int* blk, const ProjArgs* proj, cudaStream_t st,
                                        uint64_t* tl) {
  SelArgs a{};
  a.tl = tl;
  a.R = R;
  a.gen = gen;
  a.g_last = g_last;
  a.nhat_last = nhat_last;
  a.k = k;
  a.n_tok = n_tok;
  a.h = static_cast<const uint8_t*>(h);
  a.ld_bytes = ld_bytes;
  a.row_bytes = row_bytes;
  a.idx = idx;
  a.ntok_c = ntok_c;
  a.hc = static_cast<uint8_t*>(hc);
  a.n_hat = n_hat;
  a.M_out = M_out;
  a.n_refreshed = n_refreshed;
  a.blk = blk;
  a.project = proj ? 1 : 0;
  if (proj) a.pa = *proj;
  cudaLaunchAttribute at[1];
  if ((row_bytes & 15) || (ld_bytes & 15) || (reinterpret_cast<uintptr_t>(h) & 15) || (uint32_t)row_bytes > kSelStageBytes)
    return cudaErrorInvalidValue;
  cudaError_t e = func_attr((const void*)refresh_select_gather_age_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSelStageBytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = pdl_cfg(dim3((R + kSel2Threads - 1) / kSel2Threads), dim3(kSel2Threads), st, at);
  cfg.dynamicSmemBytes = kSelStageBytes;
  return cudaLaunchKernelEx(&cfg, refresh_select_gather_age_kernel, a);
}

int refresh_select_fused_max_rows() { return kSel2Threads * g_num_sms; }

}  // namespace star
