// project.cu -- worker-side local future-state simulation:
//   L_i[0] = sum_{r in B_i} N(r)                        current token load
//   L_i[t] = sum_{r in B_i, t < N_hat_r} (N(r) + t)     predicted load N_hat_i(B_{i,t})
//   W_i = sum_{t=1}^{H} beta_t L_i[t]  (w_i, Alg. 1 line 13), peak_i, growth_i, count_i
//
// Design (B200): the per-request work is a keyed histogram, not an O(R*H) loop.  A request
// with b = min(N_hat, H+1) is resident exactly for t in [1, b) (and always at t = 0), so with
// per-(instance, b) counts C and token sums S:
//   L_i[t] = sum_{b > t} (S_i[b] + t * C_i[b])   (t >= 1),   L_i[0] = sum_b S_i[b]
//   growth_i = sum_b C_i[b] * min(b, H)
// Pass 1 streams (inst, N, N_hat) with coalesced 16-byte loads (4 requests / thread / load),
// aggregates equal keys inside each warp (__match_any_sync + __reduce_add_sync; the hot bin
// b = H+1 holds ~78% of a long-tailed CoT batch), and adds into a shared-memory histogram.
// Multi-CTA grids merge through a global workspace; the last CTA to arrive finalises and
// re-zeroes the workspace.  Pass 2 (one CTA) is a suffix scan per instance.
#include <cstdint>
#include <cuda_runtime.h>
#include "project_core.cuh"
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

constexpr int kProjThreads = 1024;
constexpr int kProjMaxSmemBins = 16384;   // n_inst*(H+2) handled in shared memory (<= 192 KB)

// SMEM_BINS: histogram lives in shared memory (else directly in the global workspace).
template <bool SMEM_BINS>
__global__ void __launch_bounds__(kProjThreads) project_kernel(const ProjArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int nb = a.n_inst * (a.H + 2);
  unsigned long long* ssum;
  uint32_t* scnt;
  if (SMEM_BINS) {
    ssum = reinterpret_cast<unsigned long long*>(sm);
    scnt = reinterpret_cast<uint32_t*>(ssum + nb);
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
      ssum[k] = 0;
      scnt[k] = 0;
    }
  } else {
    ssum = a.ws_sum;
    scnt = a.ws_cnt;
  }
  __shared__ int s_last;
  __shared__ uint32_t sbeta[257];
  pdl_wait();   // inputs may come from the previous kernel (PDL launch)
  for (int t = threadIdx.x; t <= a.H; t += blockDim.x) sbeta[t] = a.beta_q[t];
  __syncthreads();   // zeroed bins and beta visible
  uint32_t errbits = 0;
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int64_t done = 0;
  if (a.vec_ok) {
    const int64_t nvec = a.R / 4;
    const int4* vi = reinterpret_cast<const int4*>(a.inst);
    const int4* vn = reinterpret_cast<const int4*>(a.n_tok);
    const int4* vh = reinterpret_cast<const int4*>(a.n_hat);
    // Each CTA streams one contiguous chunk (so an instance-grouped batch touches few
    // histogram bins per CTA and the merge below stays small); warps stride inside it.  The
    // stream is software-pipelined: the next 3 x 16 B of every lane are in flight while the
    // current 4 requests are aggregated (HBM latency hiding at bandwidth scale).
    const int64_t chunk = (nvec + gridDim.x - 1) / gridDim.x;
    const int64_t c_beg = (int64_t)blockIdx.x * chunk;
    const int64_t c_end = c_beg + chunk < nvec ? c_beg + chunk : nvec;
    const int64_t stride = (int64_t)(blockDim.x >> 5) * 32;
    int64_t g = c_beg + (int64_t)(threadIdx.x >> 5) * 32 + lane;
    int4 x = make_int4(0, 0, 0, 0), n = x, h = x;
    if (g < c_end) {
      x = ld_stream_int4(vi + g);
      n = ld_stream_int4(vn + g);
      h = ld_stream_int4(vh + g);
    }
    for (int64_t base = c_beg + (int64_t)(threadIdx.x >> 5) * 32; base < c_end; base += stride) {
      const bool valid = g < c_end;
      const int64_t g2 = g + stride;
      int4 x2 = make_int4(0, 0, 0, 0), n2 = x2, h2 = x2;
      if (g2 < c_end) {
        x2 = ld_stream_int4(vi + g2);
        n2 = ld_stream_int4(vn + g2);
        h2 = ld_stream_int4(vh + g2);
      }
      proj_accumulate4<SMEM_BINS>(a, valid, x, n, h, scnt, ssum, errbits);
      x = x2;
      n = n2;
      h = h2;
      g = g2;
    }
    done = nvec * 4;
  }
  for (int64_t base = done + (int64_t)warp_global * 32; base < a.R; base += (int64_t)nwarps * 32) {
    const int64_t r = base + lane;
    const bool valid = r < a.R;
    proj_accumulate<SMEM_BINS>(a, valid, valid ? a.inst[r] : 0, valid ? a.n_tok[r] : 0, valid ? a.n_hat[r] : 0, scnt, ssum,
                    errbits);
  }
  if (errbits && a.err) atomicOr(a.err, (int)errbits);
  __syncthreads();

  if (gridDim.x == 1) {
    proj_finalize(a, scnt, ssum, sbeta, threadIdx.x >> 5, blockDim.x >> 5);
    if (!SMEM_BINS) {  // leave the workspace zeroed
      __syncthreads();
      for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        a.ws_sum[k] = 0;
        a.ws_cnt[k] = 0;
      }
    }
    return;
  }
  if (SMEM_BINS) {
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
      if (scnt[k]) {
        atomicAdd(a.ws_cnt + k, scnt[k]);
        atomicAdd(a.ws_sum + k, ssum[k]);
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(a.ws_arrive, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (SMEM_BINS) {
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
      scnt[k] = __ldcg(a.ws_cnt + k);
      ssum[k] = __ldcg(a.ws_sum + k);
      a.ws_cnt[k] = 0;
      a.ws_sum[k] = 0;
    }
    __syncthreads();
    proj_finalize(a, scnt, ssum, sbeta, threadIdx.x >> 5, blockDim.x >> 5);
  } else {
    proj_finalize(a, a.ws_cnt, a.ws_sum, sbeta, threadIdx.x >> 5, blockDim.x >> 5);
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
      a.ws_sum[k] = 0;
      a.ws_cnt[k] = 0;
    }
  }
  if (threadIdx.x == 0) *a.ws_arrive = 0;
}

size_t project_workspace_bytes(int n_inst, int H) {
  const size_t nb = (size_t)n_inst * (size_t)(H + 2);
  return nb * 8 + nb * 4 + 16;
}

int project_single_cta_max_rows() { return 1 << 15; }

ProjArgs make_proj_args(int R, int n_inst, int inst_base, int H, const int32_t* inst, const int32_t* n_tok,
                        const int32_t* n_hat, const uint32_t* beta_q, int64_t* L, int64_t* W, int64_t* peak,
                        int64_t* growth, int32_t* count, void* workspace, int32_t* err_flag) {
  ProjArgs a{};
  a.R = R;
  a.n_inst = n_inst;
  a.inst_base = inst_base;
  a.H = H;
  a.inst = inst;
  a.n_tok = n_tok;
  a.n_hat = n_hat;
  a.beta_q = beta_q;
  a.L = L;
  a.W = W;
  a.peak = peak;
  a.growth = growth;
  a.count = count;
  a.err = err_flag;
  const size_t nb = (size_t)n_inst * (size_t)(H + 2);
  if (workspace) {
    a.ws_sum = reinterpret_cast<unsigned long long*>(workspace);
    a.ws_cnt = reinterpret_cast<uint32_t*>(a.ws_sum + nb);
    a.ws_arrive = reinterpret_cast<unsigned int*>(reinterpret_cast<uint8_t*>(workspace) + nb * 12);
  }
  a.vec_ok = ((reinterpret_cast<uintptr_t>(inst) | reinterpret_cast<uintptr_t>(n_tok) |
               reinterpret_cast<uintptr_t>(n_hat)) & 15u) == 0;
  return a;
}

cudaError_t launch_project(int R, int n_inst, int inst_base, int H, const int32_t* inst, const int32_t* n_tok,
                           const int32_t* n_hat, const uint32_t* beta_q, int64_t* L, int64_t* W, int64_t* peak,
                           int64_t* growth, int32_t* count, void* workspace, int32_t* err_flag,
                           cudaStream_t stream, int* grid_out) {
  ProjArgs a = make_proj_args(R, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, L, W, peak, growth, count,
                              workspace, err_flag);
  const size_t nb = (size_t)n_inst * (size_t)(H + 2);
  const bool smem_bins = nb <= (size_t)kProjMaxSmemBins;
  int grid = 1;
  if (workspace && R > project_single_cta_max_rows() / 8) {
    const int64_t per_cta = (int64_t)kProjThreads * 16;   // 4 vec loads of 4 requests per thread
    grid = (int)((R + per_cta - 1) / per_cta);
    // CTAs per SM: shared-memory histogram size bound, at most 2 x 1024 threads
    const size_t cta_smem = smem_bins ? nb * 12 + 2048 : 2048;
    int per_sm = (int)((200u * 1024u) / cta_smem);
    per_sm = per_sm < 1 ? 1 : (per_sm > 2 ? 2 : per_sm);
    const int max_grid = g_num_sms * per_sm;
    if (grid > max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
  }
  if (!smem_bins && !workspace) return cudaErrorInvalidValue;
  if (grid_out) *grid_out = grid;
  const size_t smem = smem_bins ? nb * 12 : 0;
  // Programmatic dependent launch: the kernel zeroes its shared histogram before
  // griddepcontrol.wait, overlapping the previous kernel's tail.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kProjThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (smem_bins) {
    static int attr_bytes = 48 * 1024;
    if ((int)smem > attr_bytes) {
      cudaError_t e = cudaFuncSetAttribute(project_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      attr_bytes = (int)smem;
    }
    static bool carve = false;
    if (!carve) {   // streaming kernel: prefer shared memory (several CTAs per SM), L1 is bypassed
      cudaFuncSetAttribute(project_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      carve = true;
    }
    return cudaLaunchKernelEx(&cfg, project_kernel<true>, a);
  }
  return cudaLaunchKernelEx(&cfg, project_kernel<false>, a);
}

}  // namespace star
