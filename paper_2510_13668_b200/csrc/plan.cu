// plan.cu -- Alg. 1 on the GPU, exact integers, one CTA.
//
// Objective (Eq. 3-4; readings A11/A12), Q16 weights beta_q:
//   Phi*n^2 = sum_{t=0}^{H} beta_q[t] * (n sum_i L_i[t]^2 - (sum_i L_i[t])^2)
// Moving request r (N = N(r), contribution c_t = N + t for t <= T_r, T_r = min(H, max(0, N_hat-1)))
// from s to u changes sum_i L_i[t]^2 by -2 c_t (L_s[t] - L_u[t] - c_t) and leaves sum_i L_i[t]
// unchanged, so the exact objective decrease is
//   gain = 2n * score,  score = sum_{t<=T_r} beta_t c_t (L_s[t] - L_u[t] - c_t)
//        = N (P0_s[T] - P0_u[T]) + (P1_s[T] - P1_u[T]) - (N^2 B0[T] + 2N B1[T] + B2[T])
// with per-instance prefix sums P0_i[T] = sum_{t<=T} beta_t L_i[t], P1_i[T] = sum_{t<=T} t beta_t L_i[t]
// and B0/B1/B2[T] = sum_{t<=T} beta_t {1, t, t^2}.  (The CPU oracle instead rebuilds the loads and
// recomputes Phi from scratch per candidate; parity between the two is a real check.)
// For a fixed request only -(N P0_u[T] + P1_u[T]) depends on the target, so each thread scores
// its requests against every target in U (filters (a)/(b) applied) and keeps the best; a
// warp-shuffle + shared-memory argmax over requests then picks m* with the key
// (gain desc, req_id asc, dst asc) (reading A20).  Greedy rounds (reading A21).
#include <cstdint>
#include <cuda_runtime.h>
#include "plan_core.cuh"
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

constexpr int kPlanThreads = 512;

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

__global__ void __launch_bounds__(kPlanThreads, 1) plan_kernel(const PlanArgs a, const int staged) {
  extern __shared__ __align__(16) uint8_t smraw[];
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
  __shared__ Cand warp_best[kPlanThreads / 32];
  __shared__ int s_stop, s_nU, s_nmoves;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  pdl_wait();   // inputs come from the projection / all-gather (PDL launch)
  pdl_launch_dependents();
  // ---- stage inputs in shared memory (all loads issued in parallel) ----
  for (int e = tid; e < n * H1; e += blockDim.x) {   // segment k holds instances [k*n_loc, (k+1)*n_loc)
    const int i = e / H1, t = e % H1;
    const int k = i / a.n_loc, il = i % a.n_loc;
    s.Ls[e] = seg_ptr(a.L, k, a.seg_stride)[(int64_t)il * H1 + t];
  }
  for (int t = tid; t < H1; t += blockDim.x) s.beta[t] = a.beta_q[t];
  for (int w = tid; w < (nslots + 31) / 32; w += blockDim.x) s.moved[w] = 0u;
  for (int k = tid; k < a.world; k += blockDim.x) {
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
  for (int g = tid; g < nstage; g += blockDim.x) {
    const int k = g / a.r_cap, j = g % a.r_cap;
    s.rid[g] = seg_ptr(a.req_id, k, a.seg_stride)[j];
    s.rinst[g] = seg_ptr(a.inst, k, a.seg_stride)[j];
    s.rntok[g] = seg_ptr(a.n_tok, k, a.seg_stride)[j];
    s.rnhat[g] = seg_ptr(a.n_hat, k, a.seg_stride)[j];
    s.rpin[g] = a.pinned ? seg_ptr(a.pinned, k, a.seg_stride)[j] : (uint8_t)0;
  }
  if (tid == 0) s_nmoves = 0;
  __syncthreads();
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
    __syncthreads();
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
    __syncthreads();
    if (s_stop) break;

    // ---- Phase 2 + 3: per-request best target, then block argmax ----
    Cand best;
    best.score = 0;
    best.id = 0;
    best.dst = 0;
    best.g = -1;
    const int nU = s_nU;
    for (int g = tid; g < nslots; g += blockDim.x) {
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
    best = warp_argmax(best);
    if (lane == 0) warp_best[warp] = best;
    __syncthreads();
    if (warp == 0) {
      Cand c;
      if (lane < nwarps) {
        c = warp_best[lane];
      } else {
        c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
      }
      c = warp_argmax(c);   // butterfly: every lane holds the winner
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
      }
    }
    __syncthreads();
    if (s_stop) break;
  }
  if (tid == 0) *a.n_moves = s_nmoves;
}

// Dynamic shared memory of plan_kernel (staged = request table copied into shared memory).
static size_t plan_smem_layout(int n, int H, int world, int r_cap, bool staged) {
  const size_t H1 = (size_t)H + 1, nn = (size_t)n, slots = (size_t)world * r_cap;
  size_t b = 16 * nn * H1 * 2 + 16 * 3 * H1 + 16 * nn + 8 * nn * H1;
  if (staged) b += 16 * slots + slots;
  b += 4 * H1 + 4 * ((slots + 31) / 32) + 4 * (size_t)world + 4 * nn + 2 * nn;
  return (b + 15) & ~size_t(15);
}

// Minimum dynamic shared memory (request table read from global memory).
size_t plan_smem_bytes(int n, int H, int world, int r_cap) { return plan_smem_layout(n, H, world, r_cap, false); }

PlanArgs make_plan_args(const star_plan_params* p, const star_plan_segments* sg, star_move* moves, int32_t* n_moves,
                        int32_t* err_flag) {
  PlanArgs a{};
  a.n = p->n_inst;
  a.H = p->H;
  a.max_moves = p->max_moves;
  a.theta_num = p->theta_num;
  a.theta_den = p->theta_den;
  a.beta_q = p->beta_q;
  a.c_mem = p->c_mem;
  a.reserved = p->reserved;
  a.a_ps = p->t_exec_a_ps;
  a.b_ps = p->t_exec_b_ps;
  a.c0_ps = p->mig_c0_ps;
  a.c1_ps = p->mig_c1_ps;
  a.flags = p->flags;
  a.world = sg->world;
  a.n_loc = sg->n_loc;
  a.r_cap = sg->r_cap;
  a.seg_stride = sg->seg_stride;
  a.L = sg->L;
  a.r_count = sg->r_count;
  a.req_id = sg->req_id;
  a.inst = sg->inst;
  a.n_tok = sg->n_tok;
  a.n_hat = sg->n_hat;
  a.pinned = sg->pinned;
  a.moves = moves;
  a.n_moves = n_moves;
  a.err = err_flag;
  return a;
}

cudaError_t launch_plan(const star_plan_params* p, const star_plan_segments* sg, star_move* moves, int32_t* n_moves,
                        int32_t* err_flag, cudaStream_t stream) {
  const PlanArgs a = make_plan_args(p, sg, moves, n_moves, err_flag);
  // Stage the request table in shared memory when it fits (it is re-read every round).
  const size_t lim = (size_t)kMaxSmemBytes - 4096;   // static shared memory + slack
  const bool staged = plan_smem_layout(a.n, a.H, a.world, a.r_cap, true) <= lim;
  const size_t smem = plan_smem_layout(a.n, a.H, a.world, a.r_cap, staged);
  static int attr_bytes = 48 * 1024;
  if ((int)smem > attr_bytes) {
    cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_bytes = (int)smem;
  }
  static bool carve = false;
  if (!carve) {   // same L1/shared split as the GEMM kernels before it: no SM reconfiguration between launches
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carve = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, 1, 1);
  cfg.blockDim = dim3(kPlanThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, plan_kernel, a, staged ? 1 : 0);
}

}  // namespace star
