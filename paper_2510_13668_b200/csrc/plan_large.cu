// plan_large.cu -- Alg. 1 at cluster scale (NEXT-3: hundreds of instances,
// tens of thousands of running requests; the paper's budget is <= 300 ms at 256 instances,
// PAPER.md:460).  Same exact-integer semantics and candidate order as plan.cu (the GPU parity
// tests compare both against the CPU oracle); the state lives in a global workspace instead of
// one CTA's shared memory and every round is two launches:
//   plan_prep_kernel   per-instance W_i and the beta-weighted prefix sums P0_i / P1_i (one warp
//                      per instance; round 0 also copies the gathered loads and clears the
//                      moved bitmap; later rounds rebuild only the two instances the last move
//                      touched)
//   plan_scan_kernel   every CTA classifies (Phase 1) from the global W, scores its slice of the
//                      requests against every target in U (Phase 2/3, best_target), reduces to a
//                      CTA candidate; the last CTA to arrive picks m* in the total order
//                      (gain desc, req_id asc, dst asc), applies it to the loads, records the
//                      move and marks the round's dirty instances (or sets the stop flag).
// Kernel boundaries are the grid-wide synchronisation; every kernel exits immediately once the
// stop flag is set, so the host can enqueue max_moves rounds without reading anything back.
#include <cstdint>
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
    const i128 x = t < H1 ? (i128)a.beta_q[t] * Li[t] : (i128)0;
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
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < (slots + 31) / 32;
         k += (int64_t)gridDim.x * blockDim.x)
      w.moved[k] = 0u;
    for (int i = gw; i < a.n; i += nw) {   // copy instance i's gathered loads, then its prefix sums
      const int k = i / a.n_loc, il = i % a.n_loc;
      for (int t = lane; t < H1; t += 32) w.Ls[(int64_t)i * H1 + t] = seg_ptr(a.L, k, a.seg_stride)[(int64_t)il * H1 + t];
      __syncwarp();
      large_prefix_row(a, w, i, cur_only);
    }
  } else {
    if (w.state[0]) return;
    if (gw < 2) large_prefix_row(a, w, w.state[2 + gw], cur_only);   // the two rows the last move touched
  }
}

__global__ void __launch_bounds__(kScanThreads) plan_scan_kernel(const PlanArgs a, const LargeWS w,
                                                                    int64_t slots, int round) {
  extern __shared__ __align__(16) uint8_t smraw[];
  pdl_wait();
  pdl_launch_dependents();
  if (w.state[0]) return;
  const int n = a.n, H1 = a.H + 1;
  const bool strict = (a.flags & 1u) != 0;
  const bool cur_only = (a.flags & 2u) != 0;
  i128* B = reinterpret_cast<i128*>(smraw);                      // [3][H+1]
  int* ulist = reinterpret_cast<int*>(B + 3 * H1);               // [n]
  int* seg_count = ulist + n;                                    // [world]
  uint8_t* inO = reinterpret_cast<uint8_t*>(seg_count + a.world);
  __shared__ Cand warp_best[kScanThreads / 32];
  __shared__ int s_nU, s_anyO, s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  for (int k = tid; k < a.world; k += blockDim.x) {
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
  __syncwarp();   // reconverge first: shuffles of a diverged warp take a slow path
  if (warp == nwarps - 1) {   // B0/B1/B2 prefix (warp scan)
    i128 c0 = 0, c1 = 0, c2 = 0;
    for (int base = 0; base < H1; base += 32) {
      const int u = base + lane;
      const i128 bt = u < H1 ? (i128)a.beta_q[u] : (i128)0;
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
        B[u] = x0;
        B[H1 + u] = x1;
        B[2 * H1 + u] = x2;
      }
      c0 = shfl_idx_i128(x0, 31);
      c1 = shfl_idx_i128(x1, 31);
      c2 = shfl_idx_i128(x2, 31);
    }
  }
  __syncwarp();
  if (warp == 0) {   // Phase 1 from the global W
    i128 wsum = 0;
    for (int i = lane; i < n; i += 32) wsum += w.Wv[i];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) wsum += shfl_xor_i128(wsum, m);
    const i128 rhs = (i128)(a.theta_den + a.theta_num) * wsum;
    bool anyO = false;
    int nU = 0;
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      bool o = false, u = false;
      if (i < n) {
        o = (i128)n * a.theta_den * w.Wv[i] > rhs;
        u = !o && ((i128)n * a.theta_den * (i128)65536 * w.Ls[(int64_t)i * H1] < rhs);
        inO[i] = o ? 1 : 0;
      }
      anyO |= __any_sync(0xFFFFFFFFu, o) != 0;
      const uint32_t um = __ballot_sync(0xFFFFFFFFu, u);
      if (u) ulist[nU + __popc(um & ((1u << lane) - 1u))] = i;
      nU += __popc(um);
    }
    if (lane == 0) {
      s_nU = nU;
      s_anyO = anyO ? 1 : 0;
    }
  }
  __syncthreads();

  Cand best;
  best.score = 0;
  best.id = 0;
  best.dst = 0;
  best.g = -1;
  if (s_anyO) {   // one request per warp at a time, lanes over the targets
    const int nU = s_nU;
    const int64_t gwarp = (int64_t)blockIdx.x * nwarps + warp, nwarp_all = (int64_t)gridDim.x * nwarps;
    for (int64_t g = gwarp; g < slots; g += nwarp_all) {
      const int k = (int)(g / a.r_cap), j = (int)(g % a.r_cap);
      if (j >= seg_count[k]) continue;
      if ((w.moved[g >> 5] >> (g & 31)) & 1u) continue;
      const int32_t src = seg_ptr(a.inst, k, a.seg_stride)[j];
      if (src < 0 || src >= n) {
        if (a.err && lane == 0) atomicOr(a.err, 1);
        continue;
      }
      if (!inO[src]) continue;
      if (a.pinned && seg_ptr(a.pinned, k, a.seg_stride)[j]) continue;
      const int64_t N = seg_ptr(a.n_tok, k, a.seg_stride)[j];
      const int64_t nh = seg_ptr(a.n_hat, k, a.seg_stride)[j];
      const int32_t rid = seg_ptr(a.req_id, k, a.seg_stride)[j];
      const Cand c = best_target_warp(a, strict, cur_only, (int)g, src, N, nh, rid, ulist, nU, w.Ls, w.P0, w.P1, B,
                                      H1);
      if (cand_better(c, best)) best = c;
    }
  }
  best = warp_argmax(best);
  if (lane == 0) warp_best[warp] = best;
  __syncthreads();
  __syncwarp();
  if (warp == 0) {
    Cand c;
    if (lane < nwarps) {
      c = warp_best[lane];
    } else {
      c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
    }
    c = warp_argmax(c);
    if (lane == 0) {
      w.cta_best[blockIdx.x] = c;
      fence_acq_rel_gpu();
      s_last = (atomicAdd(w.ctr, 1u) == gridDim.x - 1) ? 1 : 0;
    }
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  // ---- last CTA: m* over the CTA candidates (a total order, so the reduction order is free) ----
  fence_acq_rel_gpu();
  Cand c;
  c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
  for (int b = lane; b < (int)gridDim.x; b += 32) {   // written by other CTAs before fence + arrival: L2 reads
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(w.cta_best + b);
    const ulonglong2 v0 = __ldcg(src), v1 = __ldcg(src + 1);
    Cand o;
    o.score = (i128)(((unsigned __int128)v0.y << 64) | v0.x);
    o.id = (int32_t)(uint32_t)v1.x;
    o.dst = (int32_t)(uint32_t)(v1.x >> 32);
    o.g = (int32_t)(uint32_t)v1.y;
    if (cand_better(o, c)) c = o;
  }
  c = warp_argmax(c);
  if (c.g < 0 || !s_anyO) {
    if (lane == 0) {
      w.state[0] = 1;   // no improving move: stop
      *w.ctr = 0;
    }
    return;
  }
  // ExecuteMigration is out of the path: apply m* to the loads for the next round.
  const int k = c.g / a.r_cap, j = c.g % a.r_cap;
  const int src = seg_ptr(a.inst, k, a.seg_stride)[j];
  const int64_t N = seg_ptr(a.n_tok, k, a.seg_stride)[j];
  const int64_t nh = seg_ptr(a.n_hat, k, a.seg_stride)[j];
  for (int t = lane; t < H1; t += 32) {
    const int64_t ct = (t == 0) ? N : (t < nh ? N + t : 0);
    w.Ls[(int64_t)src * H1 + t] -= ct;
    w.Ls[(int64_t)c.dst * H1 + t] += ct;
  }
  if (lane == 0) {
    w.moved[c.g >> 5] |= 1u << (c.g & 31);
    const int m = w.state[1];
    const i128 gain = (i128)2 * n * c.score;
    star_move mv;
    mv.req_id = c.id;
    mv.src = src;
    mv.dst = c.dst;
    mv.round = round;
    mv.gain_hi = (int64_t)(gain >> 64);
    mv.gain_lo = (uint64_t)gain;
    a.moves[m] = mv;
    w.state[1] = m + 1;
    *a.n_moves = m + 1;
    w.state[2] = src;
    w.state[3] = c.dst;
    if (m + 1 >= a.max_moves) w.state[0] = 1;
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
  const size_t smem = 16 * 3 * H1 + 4 * (size_t)a.n + 4 * (size_t)a.world + (size_t)a.n + 16;
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
  cudaLaunchConfig_t cp1 = cp;
  cp1.gridDim = dim3(1, 1, 1);
  for (int r = 0; r < a.max_moves; ++r) {
    if (r > 0 && (e = cudaLaunchKernelEx(&cp1, plan_prep_kernel, a, w, 0, slots)) != cudaSuccess) return e;
    if ((e = cudaLaunchKernelEx(&cs, plan_scan_kernel, a, w, slots, r)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace star
