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

}  // namespace star
