// plan_large.cu -- Alg. 1 at cluster scale (NEXT-3: hundreds of instances,
// tens of thousands of running requests; the paper's budget is <= 300 ms at 256 instances,
// PAPER.md:460).  Same exact-integer semantics and candidate order as plan.cu (the GPU parity
// tests compare both against the CPU oracle); the state lives in a global workspace instead of
// one CTA's shared memory; round 0 is two launches, every later round one:
//   plan_prep_kernel   (round 0) per-instance W_i and the beta-weighted prefix sums P0_i / P1_i
//                      (one warp per instance), the B0/B1/B2 prefix sums of beta, the gathered
//                      loads copied, the moved bitmap cleared
//   plan_scan_kernel   every CTA classifies (Phase 1) from the global W (a thread per instance),
//                      reads a strided share of the slots (a thread per slot, one round trip for
//                      the request fields), compacts its candidates in shared memory, and scores
//                      its (candidate, target in U) pairs spread over all threads (Phase 2/3,
//                      loads batched four deep), folding the results into per-thread bests that
//                      are reduced once to a CTA candidate; the last CTA to arrive picks m* in the
//                      total order (gain desc, req_id asc, dst asc), applies it to the loads,
//                      rebuilds the two touched instances' W and prefix sums and records the move
//                      (or sets the stop flag).
// The scan is L2-latency bound (a few hundred candidates x a few hundred targets of exact int128
// arithmetic): every step is laid out to keep dependent global round trips few.
// Kernel boundaries are the grid-wide synchronisation; every kernel exits immediately once the
// stop flag is set, so the host can enqueue max_moves rounds without reading anything back.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "plan_core.cuh"
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

constexpr int kScanThreads = 256;
constexpr int kPrepThreads = 256;
constexpr int kMaxScanCtas = 1024;
constexpr int kLargeMaxInst = 16384;   // U list + flags in shared memory

struct LargeWS {
  int64_t* Ls;        // [n][H+1]
  i128* P0;           // [n][H+1]
  i128* P1;           // [n][H+1]
  i128* Wv;           // [n]
  i128* Bt;           // [3][H+1] B0/B1/B2 prefix sums of beta (prep, round 0)
  uint32_t* moved;    // [ceil(slots/32)]
  Cand* cta_best;     // [kMaxScanCtas]
  uint32_t* ctr;      // arrival counter
  int* state;         // [0] stop, [1] moves so far, [2] dirty s, [3] dirty t
};

static size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

static LargeWS carve(void* ws, int n, int H, int64_t slots, size_t* total) {
  const size_t H1 = (size_t)H + 1;
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  size_t o = 0;
  LargeWS w{};
  w.Ls = reinterpret_cast<int64_t*>(p + o); o = align16(o + 8 * (size_t)n * H1);
  w.P0 = reinterpret_cast<i128*>(p + o); o = align16(o + 16 * (size_t)n * H1);
  w.P1 = reinterpret_cast<i128*>(p + o); o = align16(o + 16 * (size_t)n * H1);
  w.Wv = reinterpret_cast<i128*>(p + o); o = align16(o + 16 * (size_t)n);
  w.Bt = reinterpret_cast<i128*>(p + o); o = align16(o + 16 * 3 * H1);
  w.moved = reinterpret_cast<uint32_t*>(p + o); o = align16(o + 4 * (size_t)((slots + 31) / 32));
  w.cta_best = reinterpret_cast<Cand*>(p + o); o = align16(o + sizeof(Cand) * kMaxScanCtas);
  w.ctr = reinterpret_cast<uint32_t*>(p + o); o = align16(o + 16);
  w.state = reinterpret_cast<int*>(p + o); o = align16(o + 16);
  if (total) *total = o;
  return w;
}

// One warp: W_i and prefix sums of instance i from the workspace copy of its loads.
__device__ void large_prefix_row(const PlanArgs& a, const LargeWS& w, int i, bool cur_only) {
  const int lane = threadIdx.x & 31, H1 = a.H + 1;
  const int64_t* Li = w.Ls + (int64_t)i * H1;
  i128 wpart = 0, c0 = 0, c1 = 0;
  for (int base = 0; base < H1; base += 32) {
    const int t = base + lane;
    const i128 x = t < H1 ? mul_u32((i128)Li[t], a.beta_q[t]) : (i128)0;
    if (t >= 1) wpart += x;
    i128 x0 = x, x1 = mul_u32(x, (uint32_t)t);
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
      w.P0[(int64_t)i * H1 + t] = x0;
      w.P1[(int64_t)i * H1 + t] = x1;
    }
    c0 = shfl_idx_i128(x0, 31);
    c1 = shfl_idx_i128(x1, 31);
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) wpart += shfl_xor_i128(wpart, m);
  if (lane == 0) w.Wv[i] = cur_only ? (i128)a.beta_q[0] * Li[0] : wpart;
}

__global__ void __launch_bounds__(kPrepThreads) plan_prep_kernel(const PlanArgs a, const LargeWS w, int first,
                                                                 int64_t slots) {
  pdl_wait();
  pdl_launch_dependents();
  const bool cur_only = (a.flags & 2u) != 0;
  const int H1 = a.H + 1;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  if (first) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      w.state[0] = a.max_moves > 0 ? 0 : 1;
      w.state[1] = 0;
      *w.ctr = 0;
      *a.n_moves = 0;
    }
    if (blockIdx.x == gridDim.x - 1 && (threadIdx.x >> 5) == (blockDim.x >> 5) - 1) {   // B0/B1/B2 (warp scan)
      i128 c0 = 0, c1 = 0, c2 = 0;
      for (int base = 0; base < H1; base += 32) {
        const int u = base + lane;
        const i128 bt = u < H1 ? (i128)a.beta_q[u] : (i128)0;
        i128 x0 = bt, x1 = mul_u32(bt, (uint32_t)u), x2 = mul_u32(x1, (uint32_t)u);
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
          w.Bt[u] = x0;
          w.Bt[H1 + u] = x1;
          w.Bt[2 * H1 + u] = x2;
        }
        c0 = shfl_idx_i128(x0, 31);
        c1 = shfl_idx_i128(x1, 31);
        c2 = shfl_idx_i128(x2, 31);
      }
    }
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (slots + 31) / 32;
         k += (int64_t)gridDim.x * blockDim.x)
      w.moved[k] = 0u;
    for (int i = gw; i < a.n; i += nw) {   // copy instance i's gathered loads, then its prefix sums
      const int k = i / a.n_loc, il = i % a.n_loc;
      for (int t = lane; t < H1; t += 32) w.Ls[(int64_t)i * H1 + t] = seg_ptr(a.L, k, a.seg_stride)[(int64_t)il * H1 + t];
      __syncwarp();
      large_prefix_row(a, w, i, cur_only);
    }
  }
}

// Branch-free candidate order (gain desc, req_id asc, dst asc, then the slot: warp_argmax_g's order)
// for the per-thread running best.
__device__ __forceinline__ bool lg_better(const Cand& x, const Cand& y) {
  const bool tie = (x.id < y.id) | ((x.id == y.id) & ((x.dst < y.dst) | ((x.dst == y.dst) & (x.g < y.g))));
  return (x.g >= 0) & ((y.g < 0) | (x.score > y.score) | ((x.score == y.score) & tie));
}
__device__ __forceinline__ void lg_take(Cand& c, const Cand& o) {
  const bool b = lg_better(o, c);
  c.score = b ? o.score : c.score;
  c.id = b ? o.id : c.id;
  c.dst = b ? o.dst : c.dst;
  c.g = b ? o.g : c.g;
}

// Per-candidate terms of the score (closed-form gain 2n * score; same arithmetic
// as plan.cu's best_target with the int128 products taken by 32-bit limbs: N, N_hat are int32):
//   score(u) = N (P0_src[T] - P0_u[T]) + (P1_src[T] - P1_u[T]) - (N^2 B0[T] + 2N B1[T] + B2[T]).
struct LgCands {
  int src[kScanThreads], rid[kScanThreads], g[kScanThreads], N[kScanThreads], nh[kScanThreads], T[kScanThreads];
  int64_t need[kScanThreads];                       // C_mem demand (reading A18)
  i128 self[kScanThreads], p0[kScanThreads], p1[kScanThreads], mig[kScanThreads];
};

// Phase 2/3 over the CTA's (candidate, target) pairs, spread over all threads (the scoring is a
// dependent chain of int128 steps, so spreading the pairs, not the candidates, shortens the
// slowest thread); four pairs per thread and step with every load issued before any score is
// formed.  kSm: the per-target terms a + b L_u[0] and the C_mem slack are staged in shared memory
// (else formed here from global memory: tables too large to stage).
template <bool kSm>
__device__ __forceinline__ void lg_score_pairs(const PlanArgs& a, bool strict, bool cur_only, const LgCands& cs,
                                               int nc, const int* ulist, const i128* utex, const int64_t* uslack,
                                               int nU, const LargeWS& w, int H1, Cand& best) {
  constexpr int kU = 4;
  const int npairs = nc * nU, bd = blockDim.x;
  for (int pi0 = threadIdx.x; pi0 < npairs; pi0 += kU * bd) {
    int ci[kU], u[kU];
    i128 p0[kU], p1[kU], tex[kU];
    int64_t slack[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int pi = pi0 + k * bd;
      const bool v = pi < npairs;
      const int c = v ? pi / nU : 0, q = v ? pi - c * nU : 0;
      ci[k] = c;
      u[k] = v ? ulist[q] : -1;
      const int uu = v ? u[k] : 0;   // loads of row 0 stand in for absent pairs
      const int64_t o = (int64_t)uu * H1 + cs.T[c];
      p0[k] = w.P0[o];
      p1[k] = w.P1[o];
      if (kSm) {
        tex[k] = utex[q];
        slack[k] = uslack[q];
      } else {
        const int64_t L0 = w.Ls[(int64_t)uu * H1];
        tex[k] = (i128)a.a_ps + (i128)a.b_ps * L0;
        slack[k] = 0;
        if (a.c_mem) {
          const i128 sl = (i128)a.c_mem[uu] - L0 - (strict ? 0 : (a.reserved ? a.reserved[uu] : 0));
          slack[k] = sl > (i128)INT64_MAX ? INT64_MAX : (sl < (i128)INT64_MIN ? INT64_MIN : (int64_t)sl);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int c = ci[k];
      bool ok = u[k] >= 0;
      if (!cur_only) ok &= mul_i32(tex[k], cs.nh[c]) > cs.mig[c];   // (a): N_hat (a + b L_u[0]) > c0 + c1 N
      if (a.c_mem) ok &= cs.need[c] <= slack[k];                    // (b): C_mem
      Cand cd;
      cd.score = mul_i32(cs.p0[c] - p0[k], cs.N[c]) + (cs.p1[c] - p1[k]) - cs.self[c];
      cd.id = cs.rid[c];
      cd.dst = u[k];
      cd.g = (ok & (cd.score > 0)) ? cs.g[c] : -1;
      lg_take(best, cd);
    }
  }
}

// One request slot's fields (slot g < slots: every segment holds r_cap slots of storage, so the
// loads are in bounds before the slot is checked against the segment's request count).
struct LgSlot {
  int32_t src, rid, N, nh;
  uint32_t mw;   // the slot's word of the moved bitmap
  int pin;
};
__device__ __forceinline__ void lg_load_slot(const PlanArgs& a, const LargeWS& w, int64_t g, int64_t slots,
                                             LgSlot& f) {
  f.src = f.rid = f.N = f.nh = 0;
  f.mw = 0u;
  f.pin = 0;
  if (g < slots) {
    const int k = (int)(g / a.r_cap), j = (int)(g % a.r_cap);
    f.mw = w.moved[g >> 5];
    f.src = seg_ptr(a.inst, k, a.seg_stride)[j];
    f.N = seg_ptr(a.n_tok, k, a.seg_stride)[j];
    f.nh = seg_ptr(a.n_hat, k, a.seg_stride)[j];
    f.rid = seg_ptr(a.req_id, k, a.seg_stride)[j];
    f.pin = a.pinned ? seg_ptr(a.pinned, k, a.seg_stride)[j] : 0;
  }
}

__global__ void __launch_bounds__(kScanThreads) plan_scan_kernel(const PlanArgs a, const LargeWS w,
                                                                    int64_t slots, int round, int lu_smem) {
  extern __shared__ __align__(16) uint8_t smraw[];
  pdl_wait();
  pdl_launch_dependents();
  const int n = a.n, H1 = a.H + 1;
  const bool strict = (a.flags & 1u) != 0;
  const bool cur_only = (a.flags & 2u) != 0;
  const int64_t grid = gridDim.x;
  // every independent load of the round is issued here, together (the kernel is a chain of global
  // round trips): the stop flag, this thread's first slot, its instance's W and L[0], the B table
  LgSlot f;
  lg_load_slot(a, w, (int64_t)blockIdx.x + grid * threadIdx.x, slots, f);
  i128 w_own = 0;
  int64_t l_own = 0;
  if ((int)threadIdx.x < n) {
    w_own = w.Wv[threadIdx.x];
    l_own = w.Ls[(int64_t)threadIdx.x * H1];
  }
  if (w.state[0]) return;
  i128* B = reinterpret_cast<i128*>(smraw);                              // [3][H+1]
  i128* utex = B + 3 * H1;                                               // [n] (lu_smem): a + b L_u[0] of ulist[q]
  int64_t* uslack = reinterpret_cast<int64_t*>(utex + (lu_smem ? n : 0)); // [n] (lu_smem): C_mem slack of ulist[q]
  int* ulist = reinterpret_cast<int*>(uslack + (lu_smem ? n : 0));        // [n]
  int* seg_count = ulist + n;                                            // [world]
  uint8_t* inO = reinterpret_cast<uint8_t*>(seg_count + a.world);
  __shared__ Cand warp_best[kScanThreads / 32];
  __shared__ i128 s_wpart[kScanThreads / 32];
  __shared__ int s_nU, s_nc, s_last;
  __shared__ LgCands cs;   // the CTA's candidates of the current slot chunk
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int bd = blockDim.x;

  if (tid == 0) {
    s_nU = 0;
    s_nc = 0;
  }
  for (int k = tid; k < a.world; k += bd) {
    int c = a.r_cap;
    if (a.r_count) {
      c = *seg_ptr(a.r_count, k, a.seg_stride);
      if (c < 0 || c > a.r_cap) {
        if (a.err) atomicOr(a.err, 16);
        c = c < 0 ? 0 : a.r_cap;
      }
    }
    seg_count[k] = c;
  }
  // Phase 1 from the global W: every thread sums / classifies its instances
  i128 wpart = w_own;
  for (int i = tid + bd; i < n; i += bd) wpart += w.Wv[i];
  __syncwarp();   // reconverge first: shuffles of a diverged warp take a slow path
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) wpart += shfl_xor_i128(wpart, m);
  if (lane == 0) s_wpart[warp] = wpart;
  for (int t = tid; t < 3 * H1; t += bd) B[t] = w.Bt[t];
  __syncthreads();
  i128 wsum = 0;
  for (int k = 0; k < nwarps; ++k) wsum += s_wpart[k];
  const i128 rhs = mul_u32(wsum, (uint32_t)a.theta_den + (uint32_t)a.theta_num);   // den >= 1, num >= 0
  bool any_o = false;
  for (int i = tid; i < n; i += bd) {
    const i128 Wi = i == tid ? w_own : w.Wv[i];
    const int64_t L0 = i == tid ? l_own : w.Ls[(int64_t)i * H1];
    const bool o = mul_u32(mul_u32(Wi, (uint32_t)n), (uint32_t)a.theta_den) > rhs;
    const bool u = !o && (mul_u32(mul_u32(mul_u32((i128)L0, (uint32_t)n), (uint32_t)a.theta_den), 65536u) < rhs);
    inO[i] = o ? 1 : 0;
    any_o |= o;
    if (u) {   // U in any order: the argmax is over a total order
      const int q = atomicAdd(&s_nU, 1);
      ulist[q] = i;
      if (lu_smem) {
        utex[q] = (i128)a.a_ps + (i128)a.b_ps * L0;
        int64_t sk = 0;
        if (a.c_mem) {
          const i128 sl = (i128)a.c_mem[i] - L0 - (strict ? 0 : (a.reserved ? a.reserved[i] : 0));
          sk = sl > (i128)INT64_MAX ? INT64_MAX : (sl < (i128)INT64_MIN ? INT64_MIN : (int64_t)sl);
        }
        uslack[q] = sk;
      }
    }
  }
  const int anyO = __syncthreads_or(any_o ? 1 : 0);
  const int nU = s_nU;

  Cand best;
  best.score = 0;
  best.id = 0;
  best.dst = 0;
  best.g = -1;
  if (anyO) {
    // Thread t of CTA b reads slot b + grid * (t + bd * it) (an instance's contiguous slots land in
    // different CTAs), the CTA's candidates are compacted in shared memory, and the warps take them
    // round-robin: every warp scores about the same number of candidates.
    for (int64_t it0 = (int64_t)blockIdx.x; it0 < slots; it0 += grid * bd) {
      const int64_t g = it0 + grid * tid;
      if (it0 != (int64_t)blockIdx.x) lg_load_slot(a, w, g, slots, f);   // the first chunk is in f already
      bool cand = false;
      if (g < slots) {
        const int k = (int)(g / a.r_cap), j = (int)(g % a.r_cap);
        if (j < seg_count[k]) {
          const bool moved = (f.mw >> (g & 31)) & 1u;
          const bool bad = f.src < 0 || f.src >= n;
          if (bad && !moved && a.err) atomicOr(a.err, 1);
          cand = !bad && !moved && !f.pin && inO[f.src];
        }
      }
      if (cand) {
        const int q = atomicAdd(&s_nc, 1);
        cs.src[q] = f.src;
        cs.rid[q] = f.rid;
        cs.g[q] = (int)g;
        cs.N[q] = f.N;
        cs.nh[q] = f.nh;
      }
      __syncthreads();
      const int nc = s_nc;
      if (tid < nc) {   // the candidate's own terms, once
        const int c_src = cs.src[tid], c_N = cs.N[tid], c_nh = cs.nh[tid];
        int T = c_nh - 1 < 0 ? 0 : (c_nh - 1 > a.H ? a.H : c_nh - 1);
        if (cur_only) T = 0;
        cs.T[tid] = T;
        cs.p0[tid] = w.P0[(int64_t)c_src * H1 + T];
        cs.p1[tid] = w.P1[(int64_t)c_src * H1 + T];
        cs.self[tid] = mul_i32(mul_i32(B[T], c_N), c_N) + mul_i32(B[H1 + T], c_N) * 2 + B[2 * H1 + T];
        cs.mig[tid] = (i128)a.c0_ps + mul_i32((i128)a.c1_ps, c_N);
        cs.need[tid] = strict ? (cur_only ? 0 : (int64_t)c_nh) : (int64_t)c_N + (cur_only ? 0 : (int64_t)c_nh);
      }
      __syncthreads();
      if (lu_smem)
        lg_score_pairs<true>(a, strict, cur_only, cs, nc, ulist, utex, uslack, nU, w, H1, best);
      else
        lg_score_pairs<false>(a, strict, cur_only, cs, nc, ulist, nullptr, nullptr, nU, w, H1, best);
      __syncthreads();
      if (tid == 0) s_nc = 0;
      __syncthreads();
    }
  }
  best = warp_argmax_g(best);
  if (lane == 0) warp_best[warp] = best;
  __syncthreads();
  if (warp == 0) {
    Cand c;
    if (lane < nwarps) {
      c = warp_best[lane];
    } else {
      c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
    }
    c = warp_argmax_g(c);
    if (lane == 0) {
      w.cta_best[blockIdx.x] = c;
      fence_acq_rel_gpu();
      s_last = (atomicAdd(w.ctr, 1u) == gridDim.x - 1) ? 1 : 0;
    }
  }
  __syncthreads();
  if (!s_last) return;
  // ---- last CTA: m* over the CTA candidates (a total order, so the reduction order is free) ----
  fence_acq_rel_gpu();
  Cand c;
  c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
  for (int b = tid; b < (int)gridDim.x; b += bd) {   // written by other CTAs before fence + arrival: L2 reads
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(w.cta_best + b);
    const ulonglong2 v0 = __ldcg(src), v1 = __ldcg(src + 1);
    Cand o;
    o.score = (i128)(((unsigned __int128)v0.y << 64) | v0.x);
    o.id = (int32_t)(uint32_t)v1.x;
    o.dst = (int32_t)(uint32_t)(v1.x >> 32);
    o.g = (int32_t)(uint32_t)v1.y;
    lg_take(c, o);
  }
  c = warp_argmax_g(c);
  if (lane == 0) warp_best[warp] = c;
  const int m0 = w.state[1];   // read by every thread before warp 0 updates it (after the barrier)
  __syncthreads();
  if (warp >= 2) return;
  if (lane < nwarps) {
    c = warp_best[lane];
  } else {
    c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
  }
  c = warp_argmax_g(c);   // warps 0 and 1 hold the same m*
  if (c.g < 0 || !anyO) {
    if (warp == 0 && lane == 0) {
      w.state[0] = 1;   // no improving move: stop
      *w.ctr = 0;
    }
    return;
  }
  // ExecuteMigration is out of the path: apply m* to the loads for the next round and rebuild the
  // two touched instances' W and prefix sums here (no per-round prep launch): warp 0 takes the
  // source row, warp 1 the destination row.
  const int k = c.g / a.r_cap, j = c.g % a.r_cap;
  const int src = seg_ptr(a.inst, k, a.seg_stride)[j];
  const int64_t N = seg_ptr(a.n_tok, k, a.seg_stride)[j];
  const int64_t nh = seg_ptr(a.n_hat, k, a.seg_stride)[j];
  const int row = warp == 0 ? src : c.dst;
  for (int t = lane; t < H1; t += 32) {
    const int64_t ct = (t == 0) ? N : (t < nh ? N + t : 0);
    w.Ls[(int64_t)row * H1 + t] += warp == 0 ? -ct : ct;
  }
  __syncwarp();
  if (m0 + 1 < a.max_moves) large_prefix_row(a, w, row, cur_only);   // each lane re-reads what it wrote
  if (warp == 0 && lane == 0) {
    w.moved[c.g >> 5] |= 1u << (c.g & 31);
    const i128 gain = (i128)2 * n * c.score;
    star_move mv;
    mv.req_id = c.id;
    mv.src = src;
    mv.dst = c.dst;
    mv.round = round;
    mv.gain_hi = (int64_t)(gain >> 64);
    mv.gain_lo = (uint64_t)gain;
    a.moves[m0] = mv;
    w.state[1] = m0 + 1;
    *a.n_moves = m0 + 1;
    w.state[2] = src;
    w.state[3] = c.dst;
    if (m0 + 1 >= a.max_moves) w.state[0] = 1;
    *w.ctr = 0;
  }
}

size_t plan_large_workspace_bytes(int n, int H, int64_t slots) {
  size_t total = 0;
  carve(nullptr, n, H, slots, &total);
  return total;
}

bool plan_large_supported(int n) { return n <= kLargeMaxInst; }

static_assert(sizeof(Cand) == 32, "Cand layout (score | id, dst | g) read back with 16-byte loads");

cudaError_t launch_plan_large(const PlanArgs& a, void* workspace, cudaStream_t stream) {
  const int64_t slots = (int64_t)a.world * a.r_cap;
  const LargeWS w = carve(workspace, a.n, a.H, slots, nullptr);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cp{};
  cp.blockDim = dim3(kPrepThreads, 1, 1);
  cp.stream = stream;
  cp.attrs = at;
  cp.numAttrs = 1;
  int prep_grid = (a.n + (kPrepThreads / 32) - 1) / (kPrepThreads / 32);
  prep_grid = prep_grid < 1 ? 1 : (prep_grid > 4 * g_num_sms ? 4 * g_num_sms : prep_grid);
  cp.gridDim = dim3(prep_grid, 1, 1);
  cudaError_t e = cudaLaunchKernelEx(&cp, plan_prep_kernel, a, w, 1, slots);
  if (e != cudaSuccess) return e;
  int scan_grid = (int)((slots + (kScanThreads / 32) - 1) / (kScanThreads / 32));   // a warp per request
  scan_grid = scan_grid < 1 ? 1 : (scan_grid > 2 * g_num_sms ? 2 * g_num_sms : scan_grid);
  const size_t H1 = (size_t)a.H + 1;
  const size_t smem0 = 16 * 3 * H1 + 4 * (size_t)a.n + 4 * (size_t)a.world + (size_t)a.n + 16;
  static const bool force_global = [] {   // STAR_PLAN_LARGE_GLOBAL=1: per-target terms from global memory
    const char* e = getenv("STAR_PLAN_LARGE_GLOBAL");   // (the > ~6500-instance form, testable at any size)
    return e && e[0] == '1';
  }();
  const int lu_smem = !force_global && smem0 + 24 * (size_t)a.n <= 160 * 1024 ? 1 : 0;   // U's per-target terms
  const size_t smem = smem0 + (lu_smem ? 24 * (size_t)a.n : 0);
  if (smem > 48 * 1024) {
    e = func_attr((const void*)plan_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cs{};
  cs.gridDim = dim3(scan_grid, 1, 1);
  cs.blockDim = dim3(kScanThreads, 1, 1);
  cs.dynamicSmemBytes = smem;
  cs.stream = stream;
  cs.attrs = at;
  cs.numAttrs = 1;
  for (int r = 0; r < a.max_moves; ++r)   // round r's last CTA rebuilds the rows round r + 1 reads
    if ((e = cudaLaunchKernelEx(&cs, plan_scan_kernel, a, w, slots, r, lu_smem)) != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace star
