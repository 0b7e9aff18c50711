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
#include <cstdlib>
#include <cuda_runtime.h>
#include "project_core.cuh"
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

constexpr int kProjThreads = 1024;
constexpr int kProjMaxSmemBins = 16384;   // n_inst*(H+2) handled in shared memory (<= 192 KB)

// Grid-wide merge of the per-CTA histograms (shared-memory bins -> global workspace atomics) and
// the last-arriving CTA's finalize; leaves the workspace zeroed.  Every thread of the CTA calls it
// after a __syncthreads that follows its own accumulation.
template <bool SMEM_BINS>
__device__ __forceinline__ void proj_merge_finalize(const ProjArgs& a, uint32_t* scnt, unsigned long long* ssum,
                                                    const uint32_t* sbeta, int* s_last) {
  const int nb = a.n_inst * (a.H + 2);
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
  fence_acq_rel_gpu();
  __syncthreads();
  if (threadIdx.x == 0) *s_last = (atomicAdd(a.ws_arrive, 1u) == gridDim.x - 1) ? 1 : 0;
  __syncthreads();
  if (!*s_last) return;
  fence_acq_rel_gpu();
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

  proj_merge_finalize<SMEM_BINS>(a, scnt, ssum, sbeta, &s_last);
}

// ---------------------------------------------------------------------------------------
// Bandwidth form for large batches (R >= kStreamMinRows, 16-byte aligned arrays, workspace):
// project_ldg_kernel streams each CTA's contiguous slice of the three arrays with ld.global.nc
// int4 loads (two CTAs per SM), aggregates into a shared-memory histogram window and merges it
// into the 64-bit global workspace; project_finalize_kernel (PDL-launched) then finalises every
// instance in parallel, one warp per instance, and re-zeroes the workspace.  (Measured on this
// B200, tools/read_bench.cu: per-CTA-contiguous int4 loads reach 4.7-5.0 TB/s, cp.async.bulk
// rings cap at ~4.4 TB/s; a finalize by the last-arriving CTA cost ~10-30 us at 8-256 instances.)
// The per-request aggregation is the branch-light proj_acc4_stream (ncu: the general
// proj_accumulate4 spent ~270 warp-instructions per 128 requests, mostly compares, branches and
// reconvergence, and capped the kernel at ~45% of HBM): validity as bit masks, hot requests
// (N_hat > H, ~78% of a long-tailed CoT batch) reduced per distinct instance with ballot +
// REDUX (one round for an instance-grouped batch), cold requests added straight to their bin.
// Bins are 32-bit in shared memory with the token sum split as S = lo + hi * 2^12 (lo adds N mod
// 2^12, hi adds N >> 12 <= 32), so no bin can wrap while a CTA sees at most 2^20 requests
// (checked at launch) and no periodic flush (a CTA-wide barrier) is needed.
constexpr int kStreamWinBins = 3072;                      // 36 KB window of 32-bit bins
constexpr int64_t kStreamMaxPerCta = 1 << 20;             // requests per CTA (32-bit split-sum bins)
constexpr int64_t kStreamMinRows = 1 << 18;

// Shared-memory bins cover a WINDOW of instances [wbase, wbase + wn) (all of them when the
// histogram fits; otherwise the instances around the first request of the CTA's slice, which for
// an instance-grouped batch is every instance the slice touches).  A request of an instance
// outside the window is added straight to the 64-bit global workspace (correct for any order,
// slow only for inputs that are neither grouped nor small in instance count).
struct BinWin {
  int wbase, wn, HB;
};
__device__ __forceinline__ void bin_add(const ProjArgs& a, const BinWin& w, int inst, int b, uint32_t c,
                                        unsigned long long s, uint32_t* cnt, uint32_t* slo, uint32_t* shi) {
  const int wi = inst - w.wbase;
  if ((unsigned)wi < (unsigned)w.wn) {
    const int key = wi * w.HB + b;
    atomicAdd(cnt + key, c);
    atomicAdd(slo + key, (uint32_t)(s & 0xFFFu));
    atomicAdd(shi + key, (uint32_t)(s >> 12));
  } else {
    const int key = inst * w.HB + b;
    atomicAdd(a.ws_cnt + key, c);
    atomicAdd(a.ws_sum + key, s);
  }
}

// Warp-uniform running total of hot requests (N_hat > H) of one instance, kept in registers
// across stages: an instance-grouped stream touches the shared hot bin only when the instance
// changes (and once at the end).
struct HotAcc {
  int inst = -1;
  uint32_t c = 0;
  unsigned long long s = 0;
};
__device__ __forceinline__ void hot_acc_push(const ProjArgs& a, const BinWin& w, HotAcc& acc, uint32_t* cnt,
                                             uint32_t* slo, uint32_t* shi) {
  if (acc.inst >= 0 && (threadIdx.x & 31) == 0) bin_add(a, w, acc.inst, a.H + 1, acc.c, acc.s, cnt, slo, shi);
  acc.inst = -1;
  acc.c = 0;
  acc.s = 0;
}

// Four requests per lane; every lane of the warp calls it.  Bins: count and token sum, 32-bit.
// Written for issue slots (the kernel is issue-bound once the stream is decoupled): one OR of
// three range tests per request, the detailed error bits only in a warp that saw a bad request,
// the lane's hot merge through selects.
__device__ __forceinline__ void proj_acc4_stream(const ProjArgs& a, bool valid, const int4& x, const int4& n,
                                                 const int4& h, const BinWin& w, uint32_t* cnt, uint32_t* slo,
                                                 uint32_t* shi, uint32_t& errbits, HotAcc& acc) {
  const int ins[4] = {x.x - a.inst_base, x.y - a.inst_base, x.z - a.inst_base, x.w - a.inst_base};
  const int nt[4] = {n.x, n.y, n.z, n.w};
  const int nh[4] = {h.x, h.y, h.z, h.w};
  // range checks for the four requests at once (unsigned max over the lane's four values):
  // instance < n_inst, N - 1 < 2^17 (N in [1, 2^17]), N_hat >= 0
  const unsigned mi = max(max((unsigned)ins[0], (unsigned)ins[1]), max((unsigned)ins[2], (unsigned)ins[3]));
  const unsigned mn = max(max((unsigned)(nt[0] - 1), (unsigned)(nt[1] - 1)),
                          max((unsigned)(nt[2] - 1), (unsigned)(nt[3] - 1)));
  const unsigned sh = (unsigned)(nh[0] | nh[1] | nh[2] | nh[3]) >> 31;
  const bool lane_bad = valid && (mi >= (unsigned)a.n_inst || mn >= (1u << 17) || sh);
  uint32_t okm = valid ? 15u : 0u;
  if (__any_sync(0xFFFFFFFFu, lane_bad)) {   // rare: per-request checks and error bits
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t e = ((unsigned)ins[j] >= (unsigned)a.n_inst ? 1u : 0u) |
                         ((unsigned)(nt[j] - 1) >= (1u << 17) ? 2u : 0u) | (nh[j] < 0 ? 4u : 0u);
      if (valid && e) {
        errbits |= e;
        okm &= ~(1u << j);
      }
    }
  }
  uint32_t hot = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) hot |= nh[j] > a.H ? (1u << j) : 0u;
  hot &= okm;
  const uint32_t cold = okm & ~hot;
  // lane merge: hot requests of the lane's first hot instance (all four when the lane's
  // requests share one instance, the common case of an instance-grouped batch)
  int li = -1;
  uint32_t same = 0, ls = 0;
  if (ins[0] == ins[1] && ins[0] == ins[2] && ins[0] == ins[3]) {
    li = hot ? ins[0] : -1;
    same = hot;
#pragma unroll
    for (int j = 0; j < 4; ++j) ls += ((hot >> j) & 1u) ? (uint32_t)nt[j] : 0u;
  } else {
    li = (hot & 1u) ? ins[0] : (hot & 2u) ? ins[1] : (hot & 4u) ? ins[2] : (hot & 8u) ? ins[3] : -1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool sj = ((hot >> j) & 1u) && ins[j] == li;
      same |= sj ? (1u << j) : 0u;
      ls += sj ? (uint32_t)nt[j] : 0u;
    }
  }
  const uint32_t lc = __popc(same);
  const uint32_t direct = cold | (hot & ~same);   // to their bins one by one
  if (__any_sync(0xFFFFFFFFu, direct != 0)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((direct >> j) & 1u) bin_add(a, w, ins[j], (hot >> j) & 1u ? a.H + 1 : nh[j], 1u, (uint32_t)nt[j], cnt, slo, shi);
    }
  }
  // one ballot + REDUX round per distinct lane instance (one for an instance-grouped batch)
  __syncwarp();
  uint32_t pend = __ballot_sync(0xFFFFFFFFu, li >= 0);
  while (pend) {   // warp-uniform
    const int ki = __shfl_sync(0xFFFFFFFFu, li, __ffs(pend) - 1);
    const bool mine = li == ki;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, mine);
    const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, mine ? lc : 0u);
    const uint32_t ws = __reduce_add_sync(0xFFFFFFFFu, mine ? ls : 0u);   // <= 128 * 2^17
    if (ki != acc.inst) {
      hot_acc_push(a, w, acc, cnt, slo, shi);
      acc.inst = ki;
    }
    acc.c += wc;
    acc.s += ws;
    pend &= ~m;
  }
}

// Each CTA adds its window bins (split 32-bit sums) into the 64-bit global workspace.
__device__ __forceinline__ void window_merge(const ProjArgs& a, const BinWin& w, const uint32_t* scnt,
                                             const uint32_t* slo, const uint32_t* shi) {
  const int nbw = w.wn * w.HB, wofs = w.wbase * w.HB;
  for (int k = threadIdx.x; k < nbw; k += blockDim.x) {
    const uint32_t c = scnt[k];
    if (c) {
      atomicAdd(a.ws_cnt + wofs + k, c);
      atomicAdd(a.ws_sum + wofs + k, (unsigned long long)slo[k] + ((unsigned long long)shi[k] << 12));
    }
  }
}

// Finalize of the bandwidth form: one warp per instance straight from the (L2-resident) global
// workspace -- the bins of an instance are two coalesced loads per lane, the suffix scan runs on
// shuffles -- then the warp re-zeroes its instance's bins.  PDL: waits for the merging kernel.
constexpr int kFinWarps = 8;
__global__ void __launch_bounds__(kFinWarps * 32) project_finalize_kernel(const ProjArgs a) {
  __shared__ uint32_t sbeta[257];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t <= a.H; t += blockDim.x) sbeta[t] = a.beta_q[t];
  pdl_wait();
  __syncthreads();
  const int HB = a.H + 2;
  const int i0 = blockIdx.x * kFinWarps;
  ProjArgs ab = a;
  ab.n_inst = a.n_inst - i0 < kFinWarps ? a.n_inst - i0 : kFinWarps;
  ab.L = a.L + (int64_t)i0 * (a.H + 1);
  ab.W = a.W ? a.W + i0 : nullptr;
  ab.peak = a.peak ? a.peak + i0 : nullptr;
  ab.growth = a.growth ? a.growth + i0 : nullptr;
  ab.count = a.count ? a.count + i0 : nullptr;
  const int64_t o = (int64_t)i0 * HB;
  proj_finalize(ab, a.ws_cnt + o, a.ws_sum + o, sbeta, warp, kFinWarps);
  __syncthreads();
  if (warp < ab.n_inst) {
    for (int b = lane; b < HB; b += 32) {
      a.ws_cnt[o + (int64_t)warp * HB + b] = 0;
      a.ws_sum[o + (int64_t)warp * HB + b] = 0;
    }
  }
}

// Bandwidth kernel: the three arrays are read with ld.global.nc int4 loads, software-pipelined
// two iterations deep (the next iteration's 3 x 16 B per lane are in flight while the current
// ones are aggregated), one int4 of each array (4 requests) per lane per iteration.
constexpr int kLdgThreads = 512;
__global__ void __launch_bounds__(kLdgThreads, 2) project_ldg_kernel(const ProjArgs a, const int win_n) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int HB = a.H + 2;
  const int nbw = win_n * HB;
  uint32_t* scnt = reinterpret_cast<uint32_t*>(sm);
  uint32_t* slo = scnt + nbw;
  uint32_t* shi = slo + nbw;
  __shared__ int s_wbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < nbw; k += blockDim.x) {
    scnt[k] = 0;
    slo[k] = 0;
    shi[k] = 0;
  }
  const int64_t nvec = a.R / 4;
  const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t v_beg = (int64_t)blockIdx.x * per;
  const int64_t v_end = v_beg + per < nvec ? v_beg + per : nvec;
  pdl_wait();
  if (threadIdx.x == 0) {
    int wb = 0;
    if (win_n < a.n_inst && v_beg < v_end) {
      wb = __ldg(a.inst + v_beg * 4) - a.inst_base;
      wb = wb > a.n_inst - win_n ? a.n_inst - win_n : wb;
      wb = wb < 0 ? 0 : wb;
    }
    s_wbase = wb;
  }
  __syncthreads();
  const BinWin w{s_wbase, win_n, HB};
  const int4* vi = reinterpret_cast<const int4*>(a.inst);
  const int4* vn = reinterpret_cast<const int4*>(a.n_tok);
  const int4* vh = reinterpret_cast<const int4*>(a.n_hat);
  const int64_t stride = (int64_t)kLdgThreads;   // vectors per CTA sweep (16 warps x 32 lanes)
  uint32_t errbits = 0;
  HotAcc acc;
  const int4 z = make_int4(0, 0, 0, 0);
  int64_t ga = v_beg + threadIdx.x, gb = ga + stride;
  int4 xa = z, na = z, ha = z, xb = z, nb = z, hb = z;
  if (ga < v_end) {
    xa = ld_stream_int4(vi + ga);
    na = ld_stream_int4(vn + ga);
    ha = ld_stream_int4(vh + ga);
  }
  if (gb < v_end) {
    xb = ld_stream_int4(vi + gb);
    nb = ld_stream_int4(vn + gb);
    hb = ld_stream_int4(vh + gb);
  }
  // warp-uniform trip conditions: the warp's first vector of the sweep is inside the slice
  for (int64_t base = v_beg + warp * 32; base < v_end; base += 2 * stride) {
    proj_acc4_stream(a, ga < v_end, xa, na, ha, w, scnt, slo, shi, errbits, acc);
    ga += 2 * stride;
    if (ga < v_end) {
      xa = ld_stream_int4(vi + ga);
      na = ld_stream_int4(vn + ga);
      ha = ld_stream_int4(vh + ga);
    }
    if (base + stride < v_end) proj_acc4_stream(a, gb < v_end, xb, nb, hb, w, scnt, slo, shi, errbits, acc);
    gb += 2 * stride;
    if (gb < v_end) {
      xb = ld_stream_int4(vi + gb);
      nb = ld_stream_int4(vn + gb);
      hb = ld_stream_int4(vh + gb);
    }
  }
  if (blockIdx.x == 0 && warp == 0) {   // the R % 4 trailing requests, one per lane
    const int64_t r = nvec * 4 + lane;
    if (r < a.R) {
      const int i = a.inst[r] - a.inst_base, nt = a.n_tok[r], nh = a.n_hat[r];
      const bool in_rng = (unsigned)i < (unsigned)a.n_inst, nt_ok = (unsigned)(nt - 1) < (1u << 17), nh_ok = nh >= 0;
      errbits |= (in_rng ? 0u : 1u) | (nt_ok ? 0u : 2u) | (nh_ok ? 0u : 4u);
      if (in_rng && nt_ok && nh_ok) bin_add(a, w, i, nh > a.H + 1 ? a.H + 1 : nh, 1u, (uint32_t)nt, scnt, slo, shi);
    }
  }
  hot_acc_push(a, w, acc, scnt, slo, shi);
  if (errbits && a.err) atomicOr(a.err, (int)errbits);
  __syncthreads();
  window_merge(a, w, scnt, slo, shi);
  pdl_launch_dependents();   // after this CTA's merge: the finalize kernel's wait covers it
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
  if (workspace && a.vec_ok && (int64_t)R >= kStreamMinRows && (int64_t)R <= kStreamMaxPerCta * 2 * g_num_sms &&
      H + 2 <= kStreamWinBins) {
    // shared-memory window: every instance when the histogram fits, else a window of instances
    const int win_n = nb <= (size_t)kStreamWinBins ? n_inst : kStreamWinBins / (H + 2);
    const size_t smem = (size_t)win_n * (H + 2) * 12;
    const int grid = g_num_sms * 2;   // two 512-thread CTAs per SM
    if (grid_out) *grid_out = grid;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kLdgThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, project_ldg_kernel, a, win_n);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3((n_inst + kFinWarps - 1) / kFinWarps, 1, 1);
    cfg.blockDim = dim3(kFinWarps * 32, 1, 1);
    cfg.dynamicSmemBytes = 0;
    return cudaLaunchKernelEx(&cfg, project_finalize_kernel, a);
  }
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
    if (smem > 48 * 1024) {
      cudaError_t e = func_attr((const void*)project_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
      if (e != cudaSuccess) return e;
    }
    // streaming kernel: prefer shared memory (several CTAs per SM), L1 is bypassed
    func_attr((const void*)project_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return cudaLaunchKernelEx(&cfg, project_kernel<true>, a);
  }
  return cudaLaunchKernelEx(&cfg, project_kernel<false>, a);
}

}  // namespace star
