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
  int bulk;                 // every segment array 16-byte aligned: the table may be bulk-copied
  const int64_t* W0;        // nullable: W_i of the input L (round 0), e.g. the projection's own
  uint64_t* cl_tl;          // diagnostics: per-CTA %globaltimer stamps of the cluster plan [8][8], or nullptr
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

// Warp argmax in the order (score desc, id asc, dst asc, g asc) -- plan_fast.cuh cand_better_g --
// by hardware reductions: the key as seven order-preserving
// 32-bit words (the score complemented, so its maximum is the minimum; id, dst, g with the sign bit
// flipped; an empty candidate all ones), minimised word by word among the lanes still tied
// (redux.sync: one instruction per word instead of a five-step shuffle tree).  Every lane returns
// the winner.
__device__ __forceinline__ Cand warp_argmax_g(const Cand& c) {
  __syncwarp();   // reconverge first
  const bool v = c.g >= 0;
  const unsigned __int128 us = v ? ~((unsigned __int128)c.score ^ ((unsigned __int128)1 << 127)) : ~(unsigned __int128)0;
  const uint32_t w[4] = {(uint32_t)(us >> 96), (uint32_t)(us >> 64), (uint32_t)(us >> 32), (uint32_t)us};
  const uint32_t wid = v ? (uint32_t)c.id ^ 0x80000000u : 0xFFFFFFFFu;
  const uint32_t wdst = v ? (uint32_t)c.dst ^ 0x80000000u : 0xFFFFFFFFu;
  const uint32_t wg = v ? (uint32_t)c.g ^ 0x80000000u : 0xFFFFFFFFu;
  uint32_t m[4];
  bool eq = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    m[k] = __reduce_min_sync(0xFFFFFFFFu, eq ? w[k] : 0xFFFFFFFFu);
    eq &= w[k] == m[k];
  }
  const uint32_t mid = __reduce_min_sync(0xFFFFFFFFu, eq ? wid : 0xFFFFFFFFu);
  eq &= wid == mid;
  const uint32_t mdst = __reduce_min_sync(0xFFFFFFFFu, eq ? wdst : 0xFFFFFFFFu);
  eq &= wdst == mdst;
  const uint32_t mg = __reduce_min_sync(0xFFFFFFFFu, eq ? wg : 0xFFFFFFFFu);
  Cand r;
  if (mg == 0xFFFFFFFFu) {   // no candidate in the warp (valid slots are < 2^31 - 1)
    r.score = 0;
    r.id = 0;
    r.dst = 0;
    r.g = -1;
  } else {
    const unsigned __int128 um = ((unsigned __int128)m[0] << 96) | ((unsigned __int128)m[1] << 64) |
                                 ((unsigned __int128)m[2] << 32) | (unsigned __int128)m[3];
    r.score = (i128)(~um ^ ((unsigned __int128)1 << 127));
    r.id = (int32_t)(mid ^ 0x80000000u);
    r.dst = (int32_t)(mdst ^ 0x80000000u);
    r.g = (int32_t)(mg ^ 0x80000000u);
  }
  return r;
}
__device__ __forceinline__ Cand warp_argmax(const Cand& c) { return warp_argmax_g(c); }

// a * b (mod 2^128) for a 32-bit unsigned b: four 32x32->64 multiply-adds over the limbs of a
// (the generic __int128 product costs ~4x as many IMADs and dominated the candidate scoring).
__device__ __forceinline__ i128 mul_u32(i128 a, uint32_t b) {
  const unsigned __int128 ua = (unsigned __int128)a;
  const uint64_t lo = (uint64_t)ua, hi = (uint64_t)(ua >> 64);
  const uint64_t p0 = (uint64_t)(uint32_t)lo * b;
  const uint64_t p1 = (lo >> 32) * b + (p0 >> 32);
  const uint64_t p2 = (uint64_t)(uint32_t)hi * b + (p1 >> 32);
  const uint64_t p3 = (hi >> 32) * b + (p2 >> 32);
  const uint64_t rlo = (p0 & 0xFFFFFFFFull) | (p1 << 32);
  const uint64_t rhi = (p2 & 0xFFFFFFFFull) | (p3 << 32);
  return (i128)(((unsigned __int128)rhi << 64) | rlo);
}
// a * b (mod 2^128) for a 32-bit signed b
__device__ __forceinline__ i128 mul_i32(i128 a, int32_t b) {
  const uint32_t m = b < 0 ? (uint32_t)(-(int64_t)b) : (uint32_t)b;
  const i128 r = mul_u32(a, m);
  return b < 0 ? -r : r;
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

// Barriers for plan_cta: the whole CTA, or the 128 epilogue threads of the fused tail.
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct NamedSync128 {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 1, 128;" ::: "memory"); }
};

// Shared-memory state of the plan (dynamic part; see plan_smem_bytes for the layout).
struct PlanSmem {
  i128* P0;        // [n][H+1]
  i128* P1;        // [n][H+1]
  i128* B;         // [3][H+1]
  i128* Wv;        // [n]
  int64_t* Ls;     // [n][H+1]
  uint32_t* beta;  // [H+1]
  int32_t* rid;    // [slots] staged request table (only when `staged`)
  int32_t* rinst;
  int32_t* rntok;
  int32_t* rnhat;
  uint8_t* rpin;
  uint32_t* moved; // bitmap [slots]
  int* seg_count;  // [world]
  int* ulist;      // [n]
  uint8_t* inO;    // [n]
  uint8_t* inU;    // [n]
};

// The whole plan executed by `nthreads` threads of one CTA (thread index tid; `sync` is the
// barrier over exactly those threads): the body of plan_kernel, also called by the fused
// predictor tail's finishing CTA (lenpred_forward_project_plan) so no extra launch is needed.
template <class Sync, bool staged>
__device__ __forceinline__ void plan_cta(const PlanArgs& a, uint8_t* smraw, const int tid,
                                         const int nthreads, Sync sync, Cand* warp_best, int* shv,
                                         uint64_t* tl = nullptr) {
#define PLAN_TS(k)                                       \
  do {                                                   \
    if (tl && tid == 0) {                                \
      uint64_t t_;                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
      tl[k] = t_;                                        \
    }                                                    \
  } while (0)
  const int n = a.n, H1 = a.H + 1;
  const bool strict = (a.flags & 1u) != 0;
  const bool cur_only = (a.flags & 2u) != 0;
  const int nslots = a.world * a.r_cap;
  const int nstage = staged ? nslots : 0;
  PlanSmem s;
  {
    uint8_t* p = smraw;
    s.P0 = reinterpret_cast<i128*>(p); p += sizeof(i128) * n * H1;
    s.P1 = reinterpret_cast<i128*>(p); p += sizeof(i128) * n * H1;
    s.B = reinterpret_cast<i128*>(p); p += sizeof(i128) * 3 * H1;
    s.Wv = reinterpret_cast<i128*>(p); p += sizeof(i128) * n;
    s.Ls = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * n * H1;
    s.rid = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * nstage;
    s.rinst = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * nstage;
    s.rntok = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * nstage;
    s.rnhat = reinterpret_cast<int32_t*>(p); p += sizeof(int32_t) * nstage;
    s.beta = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * H1;
    s.moved = reinterpret_cast<uint32_t*>(p); p += sizeof(uint32_t) * ((nslots + 31) / 32);
    s.seg_count = reinterpret_cast<int*>(p); p += sizeof(int) * a.world;
    s.ulist = reinterpret_cast<int*>(p); p += sizeof(int) * n;
    s.rpin = p; p += nstage;
    s.inO = p; p += n;
    s.inU = p; p += n;
  }
  int& s_stop = shv[0];
  int& s_nU = shv[1];
  int& s_nmoves = shv[2];
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthreads >> 5;
  // ---- stage inputs in shared memory (all loads issued in parallel) ----
  for (int e = tid; e < n * H1; e += nthreads) {   // segment k holds instances [k*n_loc, (k+1)*n_loc)
    const int i = e / H1, t = e % H1;
    const int k = i / a.n_loc, il = i % a.n_loc;
    s.Ls[e] = seg_ptr(a.L, k, a.seg_stride)[(int64_t)il * H1 + t];
  }
  for (int t = tid; t < H1; t += nthreads) s.beta[t] = a.beta_q[t];
  for (int w = tid; w < (nslots + 31) / 32; w += nthreads) s.moved[w] = 0u;
  for (int k = tid; k < a.world; k += nthreads) {
    int c = a.r_cap;
    if (a.r_count) {
      c = *seg_ptr(a.r_count, k, a.seg_stride);
      if (c < 0 || c > a.r_cap) {
        if (a.err) atomicOr(a.err, 16);
        c = c < 0 ? 0 : a.r_cap;
      }
    }
    s.seg_count[k] = c;
  }
  for (int g = tid; g < nstage; g += nthreads) {
    const int k = g / a.r_cap, j = g % a.r_cap;
    s.rid[g] = seg_ptr(a.req_id, k, a.seg_stride)[j];
    s.rinst[g] = seg_ptr(a.inst, k, a.seg_stride)[j];
    s.rntok[g] = seg_ptr(a.n_tok, k, a.seg_stride)[j];
    s.rnhat[g] = seg_ptr(a.n_hat, k, a.seg_stride)[j];
    s.rpin[g] = a.pinned ? seg_ptr(a.pinned, k, a.seg_stride)[j] : (uint8_t)0;
  }
  if (tid == 0) s_nmoves = 0;
  sync(); PLAN_TS(2);
  if (warp == nwarps - 1) {   // B0/B1/B2[T] = sum_{t<=T} beta_t {1, t, t^2}: warp scan (last warp)
    i128 c0 = 0, c1 = 0, c2 = 0;
    for (int base = 0; base < H1; base += 32) {
      const int u = base + lane;
      const i128 bt = u < H1 ? (i128)s.beta[u] : (i128)0;
      i128 x0 = bt, x1 = bt * u, x2 = bt * u * u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const i128 y0 = shfl_up_i128(x0, off), y1 = shfl_up_i128(x1, off), y2 = shfl_up_i128(x2, off);
        if (lane >= off) {
          x0 += y0;
          x1 += y1;
          x2 += y2;
        }
      }
      x0 += c0;
      x1 += c1;
      x2 += c2;
      if (u < H1) {
        s.B[u] = x0;
        s.B[H1 + u] = x1;
        s.B[2 * H1 + u] = x2;
      }
      c0 = shfl_idx_i128(x0, 31);
      c1 = shfl_idx_i128(x1, 31);
      c2 = shfl_idx_i128(x2, 31);
    }
  }
  const int p1_warps = nwarps - 1;   // Phase-1 warps (the last one built B above)

  for (int round = 0; round < a.max_moves; ++round) {
    // ---- Phase 1: InstanceClassification ----
    // one warp per instance: W_i (warp reduction) and the Phase-3 prefix sums
    //   P0_i[T] = sum_{t<=T} beta_t L_i[t],  P1_i[T] = sum_{t<=T} t beta_t L_i[t]  (warp scan)
    for (int i = warp; i < n && warp < p1_warps; i += p1_warps) {
      __syncwarp();
      const int64_t* Li = s.Ls + (int64_t)i * H1;
      i128 wpart = 0, c0 = 0, c1 = 0;
      for (int base = 0; base < H1; base += 32) {
        const int t = base + lane;
        const i128 x = t < H1 ? (i128)s.beta[t] * Li[t] : (i128)0;
        if (t >= 1) wpart += x;
        i128 x0 = x, x1 = x * t;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const i128 y0 = shfl_up_i128(x0, off), y1 = shfl_up_i128(x1, off);
          if (lane >= off) {
            x0 += y0;
            x1 += y1;
          }
        }
        x0 += c0;
        x1 += c1;
        if (t < H1) {
          s.P0[(int64_t)i * H1 + t] = x0;
          s.P1[(int64_t)i * H1 + t] = x1;
        }
        c0 = shfl_idx_i128(x0, 31);
        c1 = shfl_idx_i128(x1, 31);
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) wpart += shfl_xor_i128(wpart, m);
      if (lane == 0) s.Wv[i] = cur_only ? (i128)s.beta[0] * Li[0] : wpart;
    }
    sync(); PLAN_TS(3);
    __syncwarp();
    if (warp == 0) {   // classification: lanes over instances, ballots build the ordered U list
      i128 wsum = 0;
      for (int i = lane; i < n; i += 32) wsum += s.Wv[i];
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) wsum += shfl_xor_i128(wsum, m);
      const i128 rhs = (i128)(a.theta_den + a.theta_num) * wsum;
      bool anyO = false;
      int nU = 0;
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        bool o = false, u = false;
        if (i < n) {
          o = (i128)n * a.theta_den * s.Wv[i] > rhs;
          u = !o && ((i128)n * a.theta_den * (i128)65536 * s.Ls[(int64_t)i * H1] < rhs);
          s.inO[i] = o ? 1 : 0;
          s.inU[i] = u ? 1 : 0;
        }
        anyO |= __any_sync(0xFFFFFFFFu, o) != 0;
        const uint32_t um = __ballot_sync(0xFFFFFFFFu, u);
        if (u) s.ulist[nU + __popc(um & ((1u << lane) - 1u))] = i;
        nU += __popc(um);
      }
      if (lane == 0) {
        s_nU = nU;
        s_stop = anyO ? 0 : 1;
      }
    }
    sync(); PLAN_TS(4);
    if (s_stop) break;

    // ---- Phase 2 + 3: per-request best target, then block argmax ----
    Cand best;
    best.score = 0;
    best.id = 0;
    best.dst = 0;
    best.g = -1;
    const int nU = s_nU;
    PLAN_TS(11);
    for (int g = tid; g < nslots; g += nthreads) {
      const int k = g / a.r_cap, j = g % a.r_cap;
      if (j >= s.seg_count[k]) continue;
      if ((s.moved[g >> 5] >> (g & 31)) & 1u) continue;
      const int32_t src = staged ? s.rinst[g] : seg_ptr(a.inst, k, a.seg_stride)[j];
      if (src < 0 || src >= n) {
        if (a.err) atomicOr(a.err, 1);
        continue;
      }
      if (!s.inO[src]) continue;
      if (staged ? s.rpin[g] : (a.pinned && seg_ptr(a.pinned, k, a.seg_stride)[j])) continue;
      const int64_t N = staged ? s.rntok[g] : seg_ptr(a.n_tok, k, a.seg_stride)[j];
      const int64_t nh = staged ? s.rnhat[g] : seg_ptr(a.n_hat, k, a.seg_stride)[j];
      const int32_t rid = staged ? s.rid[g] : seg_ptr(a.req_id, k, a.seg_stride)[j];
      const Cand c = best_target(a, strict, cur_only, g, src, N, nh, rid, s.ulist, nU, s.Ls, s.P0, s.P1, s.B, H1);
      if (cand_better(c, best)) best = c;
    }
    PLAN_TS(12);
    best = warp_argmax(best);
    PLAN_TS(13);
    if (lane == 0) warp_best[warp] = best;
    sync(); PLAN_TS(5);
    if (warp == 0) {
      Cand c;
      if (lane < nwarps) {
        c = warp_best[lane];
      } else {
        c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
      }
      c = warp_argmax(c);   // butterfly: every lane holds the winner
      PLAN_TS(8);
      if (c.g < 0) {
        if (lane == 0) s_stop = 1;
      } else {
        // ExecuteMigration is out of the path: apply m* to the loads for the next round.
        const int k = c.g / a.r_cap, j = c.g % a.r_cap;
        const int src = staged ? s.rinst[c.g] : seg_ptr(a.inst, k, a.seg_stride)[j];
        const int64_t N = staged ? s.rntok[c.g] : seg_ptr(a.n_tok, k, a.seg_stride)[j];
        const int64_t nh = staged ? s.rnhat[c.g] : seg_ptr(a.n_hat, k, a.seg_stride)[j];
        for (int t = lane; t < H1; t += 32) {
          const int64_t ct = (t == 0) ? N : (t < nh ? N + t : 0);
          s.Ls[(int64_t)src * H1 + t] -= ct;
          s.Ls[(int64_t)c.dst * H1 + t] += ct;
        }
        PLAN_TS(9);
        if (lane == 0) {
          s.moved[c.g >> 5] |= 1u << (c.g & 31);
          const i128 gain = (i128)2 * n * c.score;
          star_move mv;
          mv.req_id = c.id;
          mv.src = src;
          mv.dst = c.dst;
          mv.round = round;
          mv.gain_hi = (int64_t)(gain >> 64);
          mv.gain_lo = (uint64_t)gain;
          a.moves[s_nmoves] = mv;
          s_nmoves = s_nmoves + 1;
        }
        PLAN_TS(10);
      }
    }
    sync(); PLAN_TS(6);
    if (s_stop) break;
  }
  PLAN_TS(7);
  if (tid == 0) *a.n_moves = s_nmoves;
#undef PLAN_TS
}


// Dynamic shared memory of plan_kernel (staged = request table copied into shared memory).
inline size_t plan_smem_layout(int n, int H, int world, int r_cap, bool staged) {
  const size_t H1 = (size_t)H + 1, nn = (size_t)n, slots = (size_t)world * r_cap;
  size_t b = 16 * nn * H1 * 2 + 16 * 3 * H1 + 16 * nn + 8 * nn * H1;
  if (staged) b += 16 * slots + slots;
  b += 4 * H1 + 4 * ((slots + 31) / 32) + 4 * (size_t)world + 4 * nn + 2 * nn;
  return (b + 15) & ~size_t(15);
}


}  // namespace star
