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

// 64-bit histogram add.  In shared memory a 64-bit atomicAdd compiles to a CAS spin loop
// (ATOMS.CAST.SPIN.64), which serialises badly on the hot bins; there the add is done as a
// native 32-bit add on the low word plus a carry into the high word (v < 2^32 so at most one
// carry).  Global memory has a native 64-bit reduction.
template <bool kShared>
__device__ __forceinline__ void hist_add64(unsigned long long* p, uint32_t v) {
  if constexpr (kShared) {
    uint32_t* w = reinterpret_cast<uint32_t*>(p);
    const uint32_t old = atomicAdd(w, v);
    if (old + v < old) atomicAdd(w + 1, 1u);
  } else {
    atomicAdd(p, (unsigned long long)v);
  }
}

// One request per lane; all 32 lanes of the warp must call this (valid may be false).
template <bool kShared = false>
__device__ __forceinline__ void proj_accumulate(const ProjArgs& a, bool valid, int32_t inst, int32_t ntok,
                                                int32_t nhat, uint32_t* scnt, unsigned long long* ssum,
                                                uint32_t& errbits) {
  __syncwarp();   // reconverge first: collectives of a diverged warp take a slow path
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
    hist_add64<kShared>(ssum + key, s);
  }
}

// Four requests per lane (one int4 of each array), all 32 lanes of the warp must call this.
// Fast path for instance-grouped batches (each decode instance's requests contiguous, the
// natural layout of a worker's batch): a lane merges its requests that fall in the hot bin
// b = H+1 (~78% of a long-tailed CoT batch) of its first such instance; if every lane's merged
// hot instance is the same, one full-warp REDUX per field and one leader atomic pair cover them,
// and the remaining (cold-bin) requests go straight to their bins.  Otherwise (e.g. round-robin
// instance order) every request takes the match_any aggregation of proj_accumulate.
template <bool kShared>
__device__ __forceinline__ void proj_accumulate4(const ProjArgs& a, bool valid, const int4& x, const int4& n,
                                                 const int4& h, uint32_t* scnt, unsigned long long* ssum,
                                                 uint32_t& errbits) {
  __syncwarp();
  const int ins[4] = {x.x - a.inst_base, x.y - a.inst_base, x.z - a.inst_base, x.w - a.inst_base};
  const int nt[4] = {n.x, n.y, n.z, n.w};
  const int nh[4] = {h.x, h.y, h.z, h.w};
  const int HB = a.H + 2;
  bool ok[4];
  int hot_i = -1;
  uint32_t hc = 0, hs = 0, merged = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    ok[j] = valid;
    if (valid) {
      if (ins[j] < 0 || ins[j] >= a.n_inst) { errbits |= 1u; ok[j] = false; }
      if (nt[j] < 1 || nt[j] > (1 << 17)) { errbits |= 2u; ok[j] = false; }
      if (nh[j] < 0) { errbits |= 4u; ok[j] = false; }
    }
    if (ok[j] && nh[j] > a.H) {
      if (hot_i < 0) hot_i = ins[j];
      if (ins[j] == hot_i) {
        ++hc;
        hs += (uint32_t)nt[j];
        merged |= 1u << j;
      }
    }
  }
  const uint32_t has = __ballot_sync(0xFFFFFFFFu, hot_i >= 0);
  const int c_i = has ? __shfl_sync(0xFFFFFFFFu, hot_i, __ffs(has) - 1) : -1;
  if (__all_sync(0xFFFFFFFFu, hot_i < 0 || hot_i == c_i)) {
    if (has) {
      const uint32_t wc = __reduce_add_sync(0xFFFFFFFFu, hc);
      const uint32_t wsum = __reduce_add_sync(0xFFFFFFFFu, hs);   // <= 128 * 2^17 < 2^32
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(scnt + c_i * HB + a.H + 1, wc);
        hist_add64<kShared>(ssum + c_i * HB + a.H + 1, wsum);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (ok[j] && !((merged >> j) & 1u)) {
        const int key = ins[j] * HB + (nh[j] > a.H + 1 ? a.H + 1 : nh[j]);
        atomicAdd(scnt + key, 1u);
        hist_add64<kShared>(ssum + key, (uint32_t)nt[j]);
      }
    }
  } else {
    uint32_t dummy = 0;   // error bits were recorded above
    proj_accumulate<kShared>(a, ok[0], x.x, n.x, h.x, scnt, ssum, dummy);
    proj_accumulate<kShared>(a, ok[1], x.y, n.y, h.y, scnt, ssum, dummy);
    proj_accumulate<kShared>(a, ok[2], x.z, n.z, h.z, scnt, ssum, dummy);
    proj_accumulate<kShared>(a, ok[3], x.w, n.w, h.w, scnt, ssum, dummy);
  }
}

// Finalize one instance per warp (lanes over histogram bins b, processed in 32-bin chunks from
// the top): suffix sums SS[b] = sum_{b' >= b} S[b'], CC[b] = sum_{b' >= b} C[b'] by a warp
// shuffle scan plus a carry, then L[t] = SS[t+1] + t*CC[t+1] for t = 1..H, and warp reductions
// of L0, count, growth, W = sum beta_t L[t], peak.  beta comes from shared memory.
// `warp` / `nwarps`: this warp's index among the warps taking part (whole warps only).
// Many instances (n_inst > 2 * nwarps): one LANE per instance instead, a sequential suffix sum
// from the top bin (the warp form costs a dependent chain of shuffles per instance, ~1.5 us, and a
// warp walks n_inst / nwarps instances one after the other).
__device__ __forceinline__ void proj_finalize_lanes(const ProjArgs& a, const uint32_t* cnt,
                                                    const unsigned long long* sum, const uint32_t* sbeta, int tid,
                                                    int nthreads) {
  const int HB = a.H + 2;
  for (int i = tid; i < a.n_inst; i += nthreads) {
    const uint32_t* c = cnt + (int64_t)i * HB;
    const unsigned long long* s = sum + (int64_t)i * HB;
    int64_t* Li = a.L + (int64_t)i * (a.H + 1);
    int64_t ss = 0, cc = 0, grow = 0, w = 0, peak = 0;
    for (int b = HB - 1; b >= 1; --b) {   // b = H+1 .. 1: SS[b], CC[b] suffix sums
      const int64_t cv = (int64_t)c[b];
      ss += (int64_t)s[b];
      cc += cv;
      grow += cv * (b < a.H ? b : a.H);
      if (b >= 2) {   // t = b - 1 in [1, H]: L[t] = SS[t+1] + t * CC[t+1]
        const int t = b - 1;
        const int64_t lt = ss + (int64_t)t * cc;
        Li[t] = lt;
        w += (int64_t)sbeta[t] * lt;
        peak = lt > peak ? lt : peak;
      }
    }
    ss += (int64_t)s[0];
    cc += (int64_t)c[0];
    Li[0] = ss;
    if (a.W) a.W[i] = w;
    if (a.peak) a.peak[i] = ss > peak ? ss : peak;
    if (a.growth) a.growth[i] = grow;
    if (a.count) a.count[i] = (int32_t)cc;
    if (cc > 65536 && a.err) atomicOr(a.err, 8);
  }
}

// Warp sum of int64 (mod 2^64, i.e. exact two's complement) by redux.sync over four 16-bit chunks
// (each chunk sum < 2^21 fits 32 bits; the four reductions are independent), and warp max of int64 as
// (high word signed, then low word unsigned among the lanes holding that high word).
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
  const uint64_t u = (uint64_t)v;
  const uint64_t c0 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(u & 0xFFFFu));
  const uint64_t c1 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)((u >> 16) & 0xFFFFu));
  const uint64_t c2 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)((u >> 32) & 0xFFFFu));
  const uint64_t c3 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)(u >> 48));
  return (int64_t)(c0 + (c1 << 16) + (c2 << 32) + (c3 << 48));
}
__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
  const int32_t hi = (int32_t)(v >> 32);
  const uint32_t lo = (uint32_t)v;
  const int32_t mh = __reduce_max_sync(0xFFFFFFFFu, hi);
  const uint32_t ml = __reduce_max_sync(0xFFFFFFFFu, hi == mh ? lo : 0u);
  return (int64_t)(((uint64_t)(uint32_t)mh << 32) | ml);
}

// kLanes: allow the lane-per-instance form (the fused tail, whose projection covers one rank's
// few instances, instantiates the warp form only and keeps its register budget).
template <bool kLanes = true>
__device__ __forceinline__ void proj_finalize(const ProjArgs& a, const uint32_t* cnt, const unsigned long long* sum,
                              const uint32_t* sbeta, int warp, int nwarps) {
  const int HB = a.H + 2;
  const int lane = threadIdx.x & 31;
  if (kLanes && a.n_inst > 2 * nwarps) {
    proj_finalize_lanes(a, cnt, sum, sbeta, warp * 32 + lane, nwarps * 32);
    return;
  }
  for (int i = warp; i < a.n_inst; i += nwarps) {
    __syncwarp();
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
    L0 = warp_sum_i64(L0);   // independent hardware reductions instead of five dependent shuffle rounds
    cnt_all = warp_sum_i64(cnt_all);
    grow = warp_sum_i64(grow);
    w = warp_sum_i64(w);
    peak = warp_max_i64(peak);
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
