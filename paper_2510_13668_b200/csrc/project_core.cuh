// project_core.cuh -- device pieces of the per-instance projection (
// readings A4-A6) shared by the standalone projection kernel (project.cu) and the fused
// predictor tail (lenpred_tail.cuh):
//   proj_accumulate  warp-aggregated keyed histogram over (instance, b = min(N_hat, H+1)):
//                    C[i][b] = #requests, S[i][b] = sum N(r)
//   proj_finalize    L_i[0] = sum_b S, L_i[t] = sum_{b > t} (S[b] + t C[b]), W, peak, growth, count
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace star {

struct ProjArgs {
  int R, n_inst, inst_base, H;
  const int32_t* inst;
  const int32_t* n_tok;
  const int32_t* n_hat;
  const uint32_t* beta_q;
  int64_t* L;
  int64_t* W;
  int64_t* peak;
  int64_t* growth;
  int32_t* count;
  uint32_t* ws_cnt;                // [nb]
  unsigned long long* ws_sum;      // [nb]
  unsigned int* ws_arrive;         // [1]
  int32_t* err;
  int vec_ok;                      // all three arrays 16-byte aligned
};

__device__ __forceinline__ int4 ld_stream_int4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// One request per lane; all 32 lanes of the warp must call this (valid may be false).
__device__ __forceinline__ void proj_accumulate(const ProjArgs& a, bool valid, int32_t inst, int32_t ntok,
                                                int32_t nhat, uint32_t* scnt, unsigned long long* ssum,
                                                uint32_t& errbits) {
  const int i = inst - a.inst_base;
  bool ok = valid;
  if (valid) {
    if (i < 0 || i >= a.n_inst) { errbits |= 1u; ok = false; }
    if (ntok < 1 || ntok > (1 << 17)) { errbits |= 2u; ok = false; }
    if (nhat < 0) { errbits |= 4u; ok = false; }
  }
  const int b = nhat > a.H + 1 ? a.H + 1 : nhat;
  const uint32_t key = ok ? (uint32_t)(i * (a.H + 2) + b) : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xFFFFFFFFu, key);
  const uint32_t s = __reduce_add_sync(peers, ok ? (uint32_t)ntok : 0u);   // 32 * 2^17 < 2^32
  const int leader = __ffs(peers) - 1;
  if (ok && (int)(threadIdx.x & 31) == leader) {
    atomicAdd(scnt + key, (uint32_t)__popc(peers));
    atomicAdd(ssum + key, (unsigned long long)s);
  }
}

// Finalize one instance per warp (lanes over histogram bins b, processed in 32-bin chunks from
// the top): suffix sums SS[b] = sum_{b' >= b} S[b'], CC[b] = sum_{b' >= b} C[b'] by a warp
// shuffle scan plus a carry, then L[t] = SS[t+1] + t*CC[t+1] for t = 1..H, and warp reductions
// of L0, count, growth, W = sum beta_t L[t], peak.  beta comes from shared memory.
// `warp` / `nwarps`: this warp's index among the warps taking part (whole warps only).
__device__ __forceinline__ void proj_finalize(const ProjArgs& a, const uint32_t* cnt, const unsigned long long* sum,
                              const uint32_t* sbeta, int warp, int nwarps) {
  const int HB = a.H + 2;
  const int lane = threadIdx.x & 31;
  for (int i = warp; i < a.n_inst; i += nwarps) {
    const uint32_t* c = cnt + (int64_t)i * HB;
    const unsigned long long* s = sum + (int64_t)i * HB;
    int64_t* Li = a.L + (int64_t)i * (a.H + 1);
    int64_t L0 = 0, cnt_all = 0, grow = 0, w = 0, peak = 0, carry_s = 0, carry_c = 0;
    for (int base = ((HB - 1) / 32) * 32; base >= 0; base -= 32) {
      const int b = base + lane;
      const int64_t sv = b < HB ? (int64_t)s[b] : 0;
      const int64_t cv = b < HB ? (int64_t)c[b] : 0;
      L0 += sv;
      cnt_all += cv;
      grow += cv * (b < a.H ? b : a.H);
      int64_t ss = sv, cc = cv;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t ts = __shfl_down_sync(0xFFFFFFFFu, ss, off);
        const int64_t tc = __shfl_down_sync(0xFFFFFFFFu, cc, off);
        if (lane + off < 32) {
          ss += ts;
          cc += tc;
        }
      }
      ss += carry_s;
      cc += carry_c;
      carry_s = __shfl_sync(0xFFFFFFFFu, ss, 0);
      carry_c = __shfl_sync(0xFFFFFFFFu, cc, 0);
      if (b >= 2 && b <= a.H + 1) {   // t = b - 1 in [1, H]
        const int t = b - 1;
        const int64_t lt = ss + (int64_t)t * cc;
        Li[t] = lt;
        w += (int64_t)sbeta[t] * lt;
        peak = lt > peak ? lt : peak;
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      L0 += __shfl_xor_sync(0xFFFFFFFFu, L0, off);
      cnt_all += __shfl_xor_sync(0xFFFFFFFFu, cnt_all, off);
      grow += __shfl_xor_sync(0xFFFFFFFFu, grow, off);
      w += __shfl_xor_sync(0xFFFFFFFFu, w, off);
      const int64_t pk = __shfl_xor_sync(0xFFFFFFFFu, peak, off);
      peak = pk > peak ? pk : peak;
    }
    if (lane == 0) {
      Li[0] = L0;
      if (a.W) a.W[i] = w;
      if (a.peak) a.peak[i] = L0 > peak ? L0 : peak;
      if (a.growth) a.growth[i] = grow;
      if (a.count) a.count[i] = (int32_t)cnt_all;
      if (cnt_all > 65536 && a.err) atomicOr(a.err, 8);
    }
  }
}

}  // namespace star
