// plan_core.cuh -- device pieces of Alg. 1 shared by the single-CTA plan
// (plan.cu) and the multi-CTA cluster-scale plan (plan_large.cu): arguments, segment addressing,
// the (gain desc, req_id asc, dst asc) candidate order (reading A20), int128 shuffles and the
// per-request best-target scoring with filters (a)/(b) (readings A15-A18).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/star.h"

namespace star {

typedef __int128 i128;

struct PlanArgs {
  int n, H, max_moves;
  int32_t theta_num, theta_den;
  const uint32_t* beta_q;
  const int64_t* c_mem;
  const int64_t* reserved;
  int64_t a_ps, b_ps, c0_ps, c1_ps;
  uint32_t flags;
  int world, n_loc, r_cap;
  int64_t seg_stride;
  const int64_t* L;
  const int32_t* r_count;   // nullptr -> every segment holds r_cap requests
  const int32_t* req_id;
  const int32_t* inst;
  const int32_t* n_tok;
  const int32_t* n_hat;
  const uint8_t* pinned;
  star_move* moves;
  int32_t* n_moves;
  int32_t* err;
};

template <typename T>
__device__ __forceinline__ const T* seg_ptr(const T* base, int k, int64_t stride) {
  return reinterpret_cast<const T*>(reinterpret_cast<const uint8_t*>(base) + (int64_t)k * stride);
}

struct Cand {
  i128 score;
  int32_t id, dst, g;   // g = flat request slot (k * r_cap + j), -1 = none
};

__device__ __forceinline__ bool cand_better(const Cand& x, const Cand& y) {  // x strictly better than y
  if (x.g < 0) return false;
  if (y.g < 0) return true;
  if (x.score != y.score) return x.score > y.score;
  if (x.id != y.id) return x.id < y.id;
  return x.dst < y.dst;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src_lane) {
  Cand o;
  const uint64_t lo = (uint64_t)c.score, hi = (uint64_t)(c.score >> 64);
  const uint64_t lo2 = __shfl_sync(0xFFFFFFFFu, lo, src_lane);
  const uint64_t hi2 = __shfl_sync(0xFFFFFFFFu, hi, src_lane);
  o.score = (i128)(((unsigned __int128)hi2 << 64) | lo2);
  o.id = __shfl_sync(0xFFFFFFFFu, c.id, src_lane);
  o.dst = __shfl_sync(0xFFFFFFFFu, c.dst, src_lane);
  o.g = __shfl_sync(0xFFFFFFFFu, c.g, src_lane);
  return o;
}

__device__ __forceinline__ Cand warp_argmax(Cand c) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    Cand o = shfl_cand(c, lane ^ off);
    if (cand_better(o, c)) c = o;
  }
  return c;
}

__device__ __forceinline__ i128 shfl_up_i128(i128 v, int off) {
  const unsigned long long lo = __shfl_up_sync(0xFFFFFFFFu, (unsigned long long)v, off);
  const long long hi = __shfl_up_sync(0xFFFFFFFFu, (long long)(v >> 64), off);
  return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}
__device__ __forceinline__ i128 shfl_idx_i128(i128 v, int src) {
  const unsigned long long lo = __shfl_sync(0xFFFFFFFFu, (unsigned long long)v, src);
  const long long hi = __shfl_sync(0xFFFFFFFFu, (long long)(v >> 64), src);
  return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}
__device__ __forceinline__ i128 shfl_xor_i128(i128 v, int m) {
  const unsigned long long lo = __shfl_xor_sync(0xFFFFFFFFu, (unsigned long long)v, m);
  const long long hi = __shfl_xor_sync(0xFFFFFFFFu, (long long)(v >> 64), m);
  return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}


// Best target of one request (slot g, on source instance src) over the target list ulist[0..nU):
// filter (a) N_hat * T_exec(u) > C_mig(r) (skipped in CURRENT_ONLY), filter (b) memory safety,
// closed-form gain score (plan.cu header); only positive scores count.  Ls / P0 / P1 / B may live
// in shared or global memory.
__device__ __forceinline__ Cand best_target(const PlanArgs& a, bool strict, bool cur_only, int g, int src, int64_t N,
                                            int64_t nh, int32_t rid, const int* ulist, int nU, const int64_t* Ls,
                                            const i128* P0, const i128* P1, const i128* B, int H1) {
  Cand best;
  best.score = 0;
  best.id = 0;
  best.dst = 0;
  best.g = -1;
  int T = (int)(nh - 1 < 0 ? 0 : (nh - 1 > a.H ? a.H : nh - 1));
  if (cur_only) T = 0;
  const i128 self = (i128)N * N * B[T] + (i128)2 * N * B[H1 + T] + B[2 * H1 + T];
  const i128 src_part = (i128)N * P0[(int64_t)src * H1 + T] + P1[(int64_t)src * H1 + T];
  const i128 mig = (i128)a.c0_ps + (i128)a.c1_ps * N;
  for (int q = 0; q < nU; ++q) {
    const int u = ulist[q];
    const int64_t Lu0 = Ls[(int64_t)u * H1];
    if (!cur_only) {  // filter (a): N_hat * T_exec(u) > C_mig(r)
      if (!((i128)nh * ((i128)a.a_ps + (i128)a.b_ps * Lu0) > mig)) continue;
    }
    if (a.c_mem) {    // filter (b): memory safety on the target
      i128 need = Lu0;
      if (strict) {
        if (!cur_only) need += nh;
      } else {
        need += (a.reserved ? a.reserved[u] : 0) + N + (cur_only ? 0 : nh);
      }
      if (!(need <= (i128)a.c_mem[u])) continue;
    }
    const i128 score = src_part - ((i128)N * P0[(int64_t)u * H1 + T] + P1[(int64_t)u * H1 + T]) - self;
    if (score <= 0) continue;
    Cand c;
    c.score = score;
    c.id = rid;
    c.dst = u;
    c.g = g;
    if (cand_better(c, best)) best = c;
  }
  return best;
}

// Warp-cooperative variant of best_target: the lanes split the target list (lane q, q+32, ...),
// so the per-target loads are coalesced and a request with hundreds of targets costs
// ceil(nU / 32) iterations instead of nU.  Every lane must call it with identical request
// arguments; returns the best candidate of the warp in every lane (warp_argmax, total order).
__device__ __forceinline__ Cand best_target_warp(const PlanArgs& a, bool strict, bool cur_only, int g, int src,
                                                 int64_t N, int64_t nh, int32_t rid, const int* ulist, int nU,
                                                 const int64_t* Ls, const i128* P0, const i128* P1, const i128* B,
                                                 int H1) {
  Cand best;
  best.score = 0;
  best.id = 0;
  best.dst = 0;
  best.g = -1;
  int T = (int)(nh - 1 < 0 ? 0 : (nh - 1 > a.H ? a.H : nh - 1));
  if (cur_only) T = 0;
  const i128 self = (i128)N * N * B[T] + (i128)2 * N * B[H1 + T] + B[2 * H1 + T];
  const i128 src_part = (i128)N * P0[(int64_t)src * H1 + T] + P1[(int64_t)src * H1 + T];
  const i128 mig = (i128)a.c0_ps + (i128)a.c1_ps * N;
  for (int q = (int)(threadIdx.x & 31); q < nU; q += 32) {
    const int u = ulist[q];
    const int64_t Lu0 = Ls[(int64_t)u * H1];
    if (!cur_only) {
      if (!((i128)nh * ((i128)a.a_ps + (i128)a.b_ps * Lu0) > mig)) continue;
    }
    if (a.c_mem) {
      i128 need = Lu0;
      if (strict) {
        if (!cur_only) need += nh;
      } else {
        need += (a.reserved ? a.reserved[u] : 0) + N + (cur_only ? 0 : nh);
      }
      if (!(need <= (i128)a.c_mem[u])) continue;
    }
    const i128 score = src_part - ((i128)N * P0[(int64_t)u * H1 + T] + P1[(int64_t)u * H1 + T]) - self;
    if (score <= 0) continue;
    Cand c;
    c.score = score;
    c.id = rid;
    c.dst = u;
    c.g = g;
    if (cand_better(c, best)) best = c;
  }
  return warp_argmax(best);
}

}  // namespace star
