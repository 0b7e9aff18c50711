// plan_fast.cuh -- the single-CTA Alg. 1 with the request table in shared
// memory.  Same arithmetic, filters and candidate order as plan_cta (plan_core.cuh: closed-form
// score, readings A15-A21); what changes is how the work of a round is laid out:
//   * staging: static inputs are fetched before griddepcontrol.wait (overlapping the predictor
//     tail), N_hat and the loads after it; the request table (needed only once an instance is
//     overloaded) streams in with bulk copies behind Phase 1 and the classification
//   * Phase 1 is split: the W pass (W_i, T_exec(i): one dot product per instance) feeds the
//     classification; the P pass (prefix sums P0/P1, warp scans) runs only when some instance
//     is overloaded; both touch only the instances the previous move changed (all in round 0)
//   * Phases 2-3 first compact the requests of overloaded instances (warp ballots + one shared
//     counter), so every lane scores a real candidate; the all-slots scan left most lanes of a
//     warp idle while one lane evaluated a candidate (~4.6k cycles per warp iteration on B200)
//   * warp collectives follow an explicit __syncwarp: a warp does not reconverge at a CTA
//     barrier, and shuffles of a diverged warp take the slow path (measured 9k cycles for one
//     5-step argmax)
// The candidate order is extended by the slot index (cand_better_g), a total order, so the
// compaction order does not matter.
#pragma once
#include "plan_core.cuh"
#include "ptx.cuh"

namespace star {

struct FastSmem {
  i128* P0;        // [n][H+1]
  i128* P1;        // [n][H+1]
  i128* B;         // [3][H+1]
  i128* Wv;        // [n]
  i128* texec;     // [n]  T_exec(i) = a + b * L_i[0]   (filter (a))
  int64_t* Ls;     // [n][H+1]
  int64_t* cmem;   // [n]  C_mem(i) - reserved(i) (non-strict) or C_mem(i) (strict); nullptr if no memory filter
  uint32_t* beta;  // [H+1]
  int32_t* rid;    // [slots] request table (slot order), cp.async
  int32_t* rinst;  // [slots] source instance; after round 0's compaction -1 marks "never a candidate"
  int32_t* rntok;
  int32_t* rnhat;
  int32_t* cidx;   // [slots] this round's candidates (slot indices)
  uint32_t* moved; // bitmap [slots]
  uint8_t* rpin;   // [slots]
  int* seg_count;  // [world]
  int* ulist;      // [n]
  uint8_t* inO;    // [n]
  uint8_t* wdirty; // [n] W_i / T_exec(i) stale
  uint8_t* pdirty; // [n] P0_i / P1_i stale
  uint64_t* bar;   // request-table bulk copies
};

// Shared-memory slot pitch per segment: a multiple of 16 so every segment's table block starts on
// 16 bytes (bulk copies); slots with j >= r_cap are never valid.
__host__ __device__ inline int plan_fast_pitch(int r_cap) { return (r_cap + 15) & ~15; }

inline size_t plan_fast_smem_layout(int n, int H, int world, int r_cap) {
  const size_t H1 = (size_t)H + 1, nn = (size_t)n, slots = (size_t)world * plan_fast_pitch(r_cap);
  size_t b = 16 * (2 * nn * H1 + 3 * H1 + 2 * nn) + 8 * (nn * H1 + nn) + 4 * H1;
  b += 4 * 5 * slots + 4 * ((slots + 31) / 32) + slots;
  b += 4 * (size_t)world + 4 * nn + 3 * nn;
  return b + 16 * 22;   // mbarrier + alignment slack (each of the 19 arrays starts on 16 bytes)
}

// Cand order extended by the slot index, so the winner does not depend on enumeration order.
// Branch-free (one predicate from comparisons, no early returns): used between shuffle steps, where
// a divergent select would send the next shuffle down the slow (BRA.DIV) path.
__device__ __forceinline__ bool cand_better_g(const Cand& x, const Cand& y) {
  const bool s_gt = x.score > y.score, s_eq = x.score == y.score;
  const bool tie = (x.id < y.id) | ((x.id == y.id) & ((x.dst < y.dst) | ((x.dst == y.dst) & (x.g < y.g))));
  return (x.g >= 0) & ((y.g < 0) | s_gt | (s_eq & tie));
}


template <class T>
__device__ __forceinline__ T* carve(uint8_t*& p, size_t count) {
  // align by pointer arithmetic (an integer round trip would lose the shared address space and
  // turn every access to the plan state into a generic LD/ST)
  p += (16u - (uint32_t)(reinterpret_cast<uintptr_t>(p) & 15u)) & 15u;
  T* r = reinterpret_cast<T*>(p);
  p += sizeof(T) * count;
  return r;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Whole plan by one CTA of `nthreads` threads (multiple of 32).  tl: optional %globaltimer stamps.
// kFused: called by the predictor tail's last CTA after the projection (no griddepcontrol.wait
// period to hide the static staging in; the loads are issued together with it instead).
// kCl > 1: the plan runs on a thread-block cluster of kCl CTAs.  Every CTA stages the whole state
// and runs the (cheap, per-instance) Phase-1 / prefix-sum work itself; the candidate compaction
// and scoring -- the instruction-bound part, one int128 score per (request, target) -- are split
// over the CTAs (4-slot groups interleaved by CTA rank, so the requests of an overloaded instance
// spread over every SM); each round's CTA winners meet in distributed shared memory and every
// CTA takes the same argmax (a total order), applies m* to its own copy of the loads and goes on.
// Only CTA 0 writes the move list.  cl_best: [2] shared Cands (round-parity double buffer).
// (Measured and rejected: pushing the last round's CTA winners to CTA 0 with st.async +
// mbarrier instead of the cluster barrier -- the plan went 11.0 -> 15.4 us.)
template <bool kFused = false, int kCl = 1>
__device__ __forceinline__ void plan_cta_fast(const PlanArgs& a, uint8_t* smraw, const int tid, const int nthreads,
                                              Cand* warp_best, int* shv, uint64_t* tl, Cand* cl_best = nullptr) {
  const int crank = kCl > 1 ? (int)cluster_ctarank() : 0;
  if (kCl > 1 && crank != 0) tl = nullptr;
#define PLAN_TS(k)                                           \
  do {                                                       \
    if (tl && tid == 0) {                                    \
      uint64_t t_;                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \
      tl[k] = t_;                                            \
      tl[32 + (k)] = clock64();                              \
    }                                                        \
  } while (0)
  const int n = a.n, H1 = a.H + 1;
  const bool strict = (a.flags & 1u) != 0;
  const bool cur_only = (a.flags & 2u) != 0;
  const int rp = plan_fast_pitch(a.r_cap);   // slot g = k * rp + j
  const int nslots = a.world * rp;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nthreads >> 5;
  FastSmem s;
  {
    uint8_t* p = smraw;
    s.P0 = carve<i128>(p, (size_t)n * H1);
    s.P1 = carve<i128>(p, (size_t)n * H1);
    s.B = carve<i128>(p, 3 * (size_t)H1);
    s.Wv = carve<i128>(p, n);
    s.texec = carve<i128>(p, n);
    s.Ls = carve<int64_t>(p, (size_t)n * H1);
    s.cmem = a.c_mem ? carve<int64_t>(p, n) : nullptr;
    s.beta = carve<uint32_t>(p, H1);
    s.rid = carve<int32_t>(p, nslots);
    s.rinst = carve<int32_t>(p, nslots);
    s.rntok = carve<int32_t>(p, nslots);
    s.rnhat = carve<int32_t>(p, nslots);
    s.cidx = carve<int32_t>(p, nslots);
    s.moved = carve<uint32_t>(p, (nslots + 31) / 32);
    s.rpin = carve<uint8_t>(p, nslots);
    s.seg_count = carve<int>(p, a.world);
    s.ulist = carve<int>(p, n);
    s.inO = carve<uint8_t>(p, n);
    s.wdirty = carve<uint8_t>(p, n);
    s.pdirty = carve<uint8_t>(p, n);
    s.bar = carve<uint64_t>(p, 1);
  }
  int& s_stop = shv[0];
  int& s_nU = shv[1];
  int& s_nmoves = shv[2];
  int& s_ncand = shv[3];
  int& s_reuse = shv[4];   // round > 0 with an unchanged overloaded set: last round's candidates stand

  // ---- staging ----
  // Static inputs (request ids, instances, token counts, pins, counts, beta, capacities) are not
  // written by this library's kernels, so they are fetched BEFORE griddepcontrol.wait, while the
  // predictor tail is still running; N_hat and the loads L come from the predecessor and are
  // fetched after it.  The request table is consumed only after the classification, so it
  // streams in behind it: one thread issues a bulk copy (TMA, 16-byte granules) per segment and
  // array when the segment arrays are 16-byte aligned (a.bulk, checked on the host), the
  // sub-16-byte tails go through plain loads; otherwise 4-byte cp.async per element.
  auto tab_src = [&](int arr, int k) -> const uint8_t* {
    const void* base = arr == 0 ? (const void*)a.req_id : arr == 1 ? (const void*)a.inst
                     : arr == 2 ? (const void*)a.n_tok : arr == 3 ? (const void*)a.n_hat : (const void*)a.pinned;
    return reinterpret_cast<const uint8_t*>(base) + (int64_t)k * a.seg_stride;
  };
  auto tab_dst = [&](int arr) -> uint8_t* {
    return arr == 0 ? (uint8_t*)s.rid : arr == 1 ? (uint8_t*)s.rinst : arr == 2 ? (uint8_t*)s.rntok
         : arr == 3 ? (uint8_t*)s.rnhat : (uint8_t*)s.rpin;
  };
  const int tail_elems = a.bulk ? (a.r_cap & 3) : 0;   // int32 elements past the last 16-byte granule
  const int tail_pin = (a.bulk && a.pinned) ? (a.r_cap & 15) : 0;
  const uint32_t fl32 = (uint32_t)(a.r_cap * 4) & ~15u, fl8 = (uint32_t)a.r_cap & ~15u;
  const int issuer = nthreads - 1;   // the last thread: it rarely has a synchronous item below
  // bulk copies of the table arrays (all but N_hat, or only N_hat), by the issuer thread
  auto issue_table = [&](bool init, bool static_part, bool nhat_part) {
    if (init) {
      mbar_init(s.bar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(s.bar, (uint32_t)a.world * (4 * fl32 + (a.pinned ? fl8 : 0)));
    }
    // N_hat written through the generic proxy by THIS kernel (fused form) needs the proxy fence;
    // after griddepcontrol.wait the predecessor grid's completion has published it
    if (nhat_part && kFused) fence_proxy_async_global();
    for (int k = 0; k < a.world; ++k)
      for (int arr = 0; arr < 5; ++arr) {
        if (arr == 4 && !a.pinned) continue;
        if (arr == 3 ? !nhat_part : !static_part) continue;
        const uint32_t fl = arr < 4 ? fl32 : fl8;
        if (fl) bulk_g2s(tab_dst(arr) + (size_t)k * rp * (arr < 4 ? 4 : 1), tab_src(arr, k), fl, s.bar);
      }
  };
  // the fused form issues the whole table only once some instance is overloaded (below)
  bool table_issued = !(kFused && a.bulk);
  if (a.bulk) {
    if (!kFused && tid == issuer) issue_table(true, true, false);
  } else {
    for (int g = tid; g < nslots; g += nthreads) {
      const int k = g / rp, j = g - k * rp;
      if (j >= a.r_cap) continue;
      cp_async4(s.rid + g, seg_ptr(a.req_id, k, a.seg_stride) + j);
      cp_async4(s.rinst + g, seg_ptr(a.inst, k, a.seg_stride) + j);
      cp_async4(s.rntok + g, seg_ptr(a.n_tok, k, a.seg_stride) + j);
    }
  }
  // loads L and the N_hat tails, four per thread per batch, all in flight before any store
  auto load_dynamic = [&]() {
    const int nL = n * H1, total = nL + a.world * tail_elems;
    for (int base = 0; base < total; base += 4 * nthreads) {
      int64_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + 4 * tid + u;
        v[u] = 0;
        if (e < nL) {   // segment k holds instances [k*n_loc, (k+1)*n_loc)
          const int i = e / H1, t = e - i * H1;
          const int k = i / a.n_loc, il = i - k * a.n_loc;
          v[u] = seg_ptr(a.L, k, a.seg_stride)[(int64_t)il * H1 + t];
        } else if (e < total) {
          const int r = e - nL, k = r / tail_elems, j = (a.r_cap & ~3) + (r - k * tail_elems);
          v[u] = reinterpret_cast<const int32_t*>(tab_src(3, k))[j];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = base + 4 * tid + u;
        if (e < nL) {
          s.Ls[e] = v[u];
        } else if (e < total) {
          const int r = e - nL, k = r / tail_elems, j = (a.r_cap & ~3) + (r - k * tail_elems);
          s.rnhat[(size_t)k * rp + j] = (int32_t)v[u];
        }
      }
    }
  };
  if constexpr (kFused) load_dynamic();   // no wait period: the L loads on the low threads
  // synchronous static items, one per thread where it fits (all loads in flight together), on
  // the high threads (the fused form's L loads occupy the low ones)
  {
    const int nTail = a.world * (3 * tail_elems + tail_pin);
    const int nPin = (!a.bulk && a.pinned) ? nslots : 0;
    const int total = H1 + n + a.world + nTail + nPin;
    for (int e = nthreads - 1 - tid; e < total; e += nthreads) {
      int r = e;
      if (r < H1) {
        s.beta[r] = a.beta_q[r];
        continue;
      }
      r -= H1;
      if (r < n) {
        if (s.cmem)   // filter (b) capacity: strict needs L_u[0] + N_hat <= C_mem; otherwise
                      // L_u[0] + reserved + N + N_hat <= C_mem  (readings A17/A18)
          s.cmem[r] = a.c_mem[r] - (strict ? 0 : (a.reserved ? a.reserved[r] : 0));
        if (a.W0 && !cur_only) {   // round-0 W_i given (the projection's own, exact in int64)
          s.Wv[r] = (i128)a.W0[r];
          s.wdirty[r] = 2;
        } else {
          s.wdirty[r] = 1;
        }
        s.pdirty[r] = 1;
        continue;
      }
      r -= n;
      if (r < a.world) {
        int c = a.r_cap;
        if (a.r_count) {
          c = *seg_ptr(a.r_count, r, a.seg_stride);
          if (c < 0 || c > a.r_cap) {
            if (a.err) atomicOr(a.err, 16);
            c = c < 0 ? 0 : a.r_cap;
          }
        }
        s.seg_count[r] = c;
        continue;
      }
      r -= a.world;
      if (r < nTail) {
        const int per = 3 * tail_elems + tail_pin;
        const int k = r / per;
        const int q = r - k * per;
        if (q < 3 * tail_elems) {
          const int arr = q / tail_elems, j = (a.r_cap & ~3) + (q - arr * tail_elems);
          reinterpret_cast<int32_t*>(tab_dst(arr))[(size_t)k * rp + j] =
              reinterpret_cast<const int32_t*>(tab_src(arr, k))[j];
        } else {
          const int j = (a.r_cap & ~15) + (q - 3 * tail_elems);
          s.rpin[(size_t)k * rp + j] = tab_src(4, k)[j];
        }
        continue;
      }
      r -= nTail;
      {   // pinned flags, cp.async path
        const int k = r / rp, j = r - k * rp;
        if (j < a.r_cap) s.rpin[r] = seg_ptr(a.pinned, k, a.seg_stride)[j];
      }
    }
  }
  if (!a.pinned)
    for (int g = tid; g < nslots; g += nthreads) s.rpin[g] = 0;
  for (int w = tid; w < (nslots + 31) / 32; w += nthreads) s.moved[w] = 0u;
  if (tid == 0) s_nmoves = 0;
  PLAN_TS(12);
  pdl_wait();   // N_hat and L are written by the predecessor (predictor tail / projection / all-gather)
  if (kCl > 1 && a.cl_tl && tid == 0) a.cl_tl[crank * 8 + 1] = globaltimer_ns();
  PLAN_TS(13);
  if (a.bulk) {
    if (!kFused && tid == issuer) issue_table(false, false, true);
  } else {
    for (int g = tid; g < nslots; g += nthreads) {
      const int k = g / rp, j = g - k * rp;
      if (j < a.r_cap) cp_async4(s.rnhat + g, seg_ptr(a.n_hat, k, a.seg_stride) + j);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if constexpr (!kFused) load_dynamic();
  PLAN_TS(15);
  __syncthreads();
  __syncwarp();
  PLAN_TS(2);

  for (int round = 0; round < a.max_moves; ++round) {
    // ---- Phase 1: InstanceClassification, changed instances only ----
    // One warp per changed instance builds the prefix sums Phases 2-3 need, P0_i[T] = sum_{t<=T}
    // beta_t L_i[t] and P1_i[T] = sum_{t<=T} t beta_t L_i[t] (warp scans), and takes
    // W_i = sum_{t>=1} beta_t L_i[t] = P0_i[H] - beta_0 L_i[0] from them, plus T_exec(i).
    for (int i = warp; i < n; i += nwarps) {
      __syncwarp();
      const int d = s.wdirty[i];
      __syncwarp();   // every lane has read the flag before lane 0 clears it
      if (!d) continue;
      const int64_t* Li = s.Ls + (int64_t)i * H1;
      i128 c0 = 0, c1 = 0;
      for (int base = 0; base < H1; base += 32) {
        const int t = base + lane;
        const i128 x = t < H1 ? mul_u32((i128)Li[t], s.beta[t]) : (i128)0;
        i128 x0 = x, x1 = mul_u32(x, (uint32_t)t);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          __syncwarp();   // the add below diverges: reconverge before the next shuffle
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
      if (lane == 0) {   // c0 = P0_i[H] (lanes past H add zeros)
        if (d != 2) s.Wv[i] = cur_only ? (i128)s.beta[0] * Li[0] : c0 - (i128)s.beta[0] * Li[0];
        s.texec[i] = (i128)a.a_ps + (i128)a.b_ps * Li[0];
        s.wdirty[i] = 0;
        s.pdirty[i] = 0;
      }
    }
    __syncthreads();
    PLAN_TS(3);
    __syncwarp();
    if (warp == 0) {   // classification: lanes over instances, ballots build the ordered U list
      i128 wsum = 0;
      for (int i = lane; i < n; i += 32) wsum += s.Wv[i];
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) wsum += shfl_xor_i128(wsum, m);
      const i128 rhs = mul_u32(wsum, (uint32_t)a.theta_den + (uint32_t)a.theta_num);   // den >= 1, num >= 0
      bool anyO = false, chO = false;
      int nU = 0;
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        bool o = false, u = false, ch = false;
        if (i < n) {
          o = mul_u32(mul_u32(s.Wv[i], (uint32_t)n), (uint32_t)a.theta_den) > rhs;
          u = !o && (mul_u32(mul_u32((i128)s.Ls[(int64_t)i * H1], (uint32_t)n), (uint32_t)a.theta_den) << 16) < rhs;
          ch = s.inO[i] != (o ? 1 : 0);
          s.inO[i] = o ? 1 : 0;
        }
        anyO |= __any_sync(0xFFFFFFFFu, o) != 0;
        chO |= __any_sync(0xFFFFFFFFu, ch) != 0;
        const uint32_t um = __ballot_sync(0xFFFFFFFFu, u);
        if (u) s.ulist[nU + __popc(um & ((1u << lane) - 1u))] = i;
        nU += __popc(um);
      }
      if (lane == 0) {
        s_nU = nU;
        s_stop = anyO ? 0 : 1;
        // the candidate set is {valid, unpinned, source in O, not moved}: with O unchanged it is
        // last round's list minus the request just moved (skipped in the evaluation below)
        s_reuse = (round > 0 && !chO) ? 1 : 0;
        if (!s_reuse) s_ncand = 0;
      }
    }
    __syncthreads();
    PLAN_TS(4);
    if (s_stop) break;
    if (round == 0) {   // the request table must have landed (a stopping plan never waits here)
      if (a.bulk) {
        if (!table_issued) {   // fused form: issue it now (CTA-uniform branch)
          if (tid == issuer) issue_table(true, true, true);
          table_issued = true;
        }
        mbar_wait(s.bar, 0);   // the transaction barrier publishes the bulk copies to its waiters
      } else {
        cp_async_wait_all();
        __syncthreads();       // publishes every thread's cp.async
      }
    }

    // ---- P pass: P0_i[T] = sum_{t<=T} beta_t L_i[t], P1_i[T] = sum_{t<=T} t beta_t L_i[t] (warp
    // scans) for the instances whose loads changed; the same warps then join the compaction.
    // Round 0 also builds B0/B1/B2 here (needed only by the scoring). ----
    __syncwarp();
    if (round == 0 && warp == nwarps - 1) {   // B0/B1/B2[T] = sum_{t<=T} beta_t {1, t, t^2}: warp scan (last warp)
      i128 c0 = 0, c1 = 0, c2 = 0;
      for (int base = 0; base < H1; base += 32) {
        const int u = base + lane;
        const i128 bt = u < H1 ? (i128)s.beta[u] : (i128)0;
        i128 x0 = bt, x1 = mul_u32(bt, (uint32_t)u), x2 = mul_u32(x1, (uint32_t)u);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          __syncwarp();   // the add below diverges: reconverge before the next shuffle
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
    for (int i = warp; i < n; i += nwarps) {
      __syncwarp();
      const bool d = s.pdirty[i] != 0;
      __syncwarp();
      if (!d) continue;
      const int64_t* Li = s.Ls + (int64_t)i * H1;
      i128 c0 = 0, c1 = 0;
      for (int base = 0; base < H1; base += 32) {
        const int t = base + lane;
        const i128 x = t < H1 ? mul_u32((i128)Li[t], s.beta[t]) : (i128)0;
        i128 x0 = x, x1 = mul_u32(x, (uint32_t)t);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          __syncwarp();   // the add below diverges: reconverge before the next shuffle
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
      if (lane == 0) s.pdirty[i] = 0;
    }
    // ---- candidate compaction: requests on overloaded instances, not pinned, not yet moved ----
    // (round 0 also validates each slot once and marks the slots that can never be candidates)
    // four consecutive slots per lane (one 16-byte shared load), one atomic per warp; in a
    // cluster, CTA `crank` takes the 4-slot groups with (group index mod kCl) == crank
    for (int base = 0; base < (s_reuse ? 0 : nslots); base += 4 * nthreads * kCl) {
      const int g0 = base + 4 * (tid * kCl + crank);
      uint32_t cm = 0;   // candidate bits of slots g0..g0+3
      if (g0 < nslots) {   // nslots is a multiple of 16 (pitch)
        int4 sv = *reinterpret_cast<const int4*>(s.rinst + g0);
        int src4[4] = {sv.x, sv.y, sv.z, sv.w};
        const uint32_t mv = (s.moved[g0 >> 5] >> (g0 & 31)) & 15u;
        if (round == 0) {
          const int k = g0 / rp, j0 = g0 - k * rp, cnt = s.seg_count[k];
          bool changed = false;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            int src = src4[q];
            if (j0 + q >= cnt) {
              src = -1;
            } else if (src < 0 || src >= n) {
              if (a.err) atomicOr(a.err, 1);
              src = -1;
            } else if (s.rpin[g0 + q]) {
              src = -1;
            }
            changed |= src != src4[q];
            src4[q] = src;
          }
          if (changed) *reinterpret_cast<int4*>(s.rinst + g0) = make_int4(src4[0], src4[1], src4[2], src4[3]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (src4[q] >= 0 && s.inO[src4[q]] && !((mv >> q) & 1u)) cm |= 1u << q;
      }
      __syncwarp();
      const int cntl = __popc(cm);
      int x = cntl;   // inclusive warp scan of the per-lane counts
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        __syncwarp();
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, off);
        if (lane >= off) x += y;
      }
      int pos = 0;
      if (lane == 31 && x) pos = atomicAdd(&s_ncand, x);
      pos = __shfl_sync(0xFFFFFFFFu, pos, 31) + x - cntl;
      while (cm) {
        const int q = __ffs(cm) - 1;
        cm &= cm - 1;
        s.cidx[pos++] = g0 + q;
      }
    }
    __syncthreads();
    PLAN_TS(9);

    // ---- Phase 2 + 3: candidates x targets in U, then block argmax ----
    Cand best;
    best.score = 0;
    best.id = 0;
    best.dst = 0;
    best.g = -1;
    const int nU = s_nU, ncand = s_ncand;
    // one (candidate, target) pair per thread: the scoring is a dependent chain of int128 steps,
    // so spreading the pairs (not the candidates) over the threads shortens each thread's chain
    const int npairs = ncand * nU;
    const long long ev_t0 = (a.cl_tl && round == 0) ? clock64() : 0;
    for (int pi = tid; pi < npairs; pi += nthreads) {
      const int c = pi / nU, qq = pi - c * nU;
      const int g = s.cidx[c];
      if ((s.moved[g >> 5] >> (g & 31)) & 1u) continue;   // moved earlier in this call (reused list)
      const int src = s.rinst[g];
      const int32_t N = s.rntok[g], nh = s.rnhat[g];
      const int u = s.ulist[qq];
      if (!cur_only && !(mul_i32(s.texec[u], nh) > (i128)a.c0_ps + mul_i32((i128)a.c1_ps, N))) continue;  // filter (a)
      const int64_t need_r = strict ? (cur_only ? 0 : (int64_t)nh) : (int64_t)N + (cur_only ? 0 : (int64_t)nh);
      if (s.cmem && !(s.Ls[(int64_t)u * H1] + need_r <= s.cmem[u])) continue;                         // filter (b)
      int T = nh - 1 < 0 ? 0 : (nh - 1 > a.H ? a.H : nh - 1);
      if (cur_only) T = 0;
      // score = N (P0_src[T] - P0_u[T]) + (P1_src[T] - P1_u[T]) - (N^2 B0[T] + 2N B1[T] + B2[T])
      const i128 self = mul_i32(mul_i32(s.B[T], N), N) + mul_i32(s.B[H1 + T], N) * 2 + s.B[2 * H1 + T];
      const i128 score = mul_i32(s.P0[(int64_t)src * H1 + T] - s.P0[(int64_t)u * H1 + T], N) +
                         (s.P1[(int64_t)src * H1 + T] - s.P1[(int64_t)u * H1 + T]) - self;
      if (score <= 0) continue;
      Cand cd;
      cd.score = score;
      cd.id = s.rid[g];
      cd.dst = u;
      cd.g = g;
      if (cand_better_g(cd, best)) best = cd;
    }
    if (a.cl_tl && round == 0) {   // diagnostics: slowest thread's evaluation cycles, pairs, candidates
      const unsigned long long dt = (unsigned long long)(clock64() - ev_t0);
      atomicMax(reinterpret_cast<unsigned long long*>(a.cl_tl + crank * 8 + 6), dt);
      if (tid == 0) a.cl_tl[crank * 8 + 7] = ((uint64_t)ncand << 32) | (uint64_t)(uint32_t)nU;
    }
    PLAN_TS(10);
    __syncwarp();
    best = warp_argmax_g(best);
    PLAN_TS(11);
    if (lane == 0) warp_best[warp] = best;
    __syncthreads();
    PLAN_TS(5);
    __syncwarp();
    Cand c;
    c.score = 0; c.id = 0; c.dst = 0; c.g = -1;
    const bool last = round == a.max_moves - 1;
    if (warp == 0) {
      if (lane < nwarps) c = warp_best[lane];
      c = warp_argmax_g(c);   // every lane holds the CTA's winner
      if (kCl > 1 && lane == 0) cl_best[round & 1] = c;
    }
    if constexpr (kCl > 1) {
      // cluster argmax: every CTA published its winner; meet (all threads), then warp 0 of every
      // CTA reads all kCl winners from distributed shared memory and takes the same argmax
      if (a.cl_tl && tid == 0) a.cl_tl[crank * 8 + 2 + 2 * (round & 1)] = globaltimer_ns();
      cluster_sync_all();
      if (a.cl_tl && tid == 0) a.cl_tl[crank * 8 + 3 + 2 * (round & 1)] = globaltimer_ns();
      if (warp == 0) {
        Cand o;
        o.score = 0; o.id = 0; o.dst = 0; o.g = -1;
        if (lane < kCl) {
          const uint32_t ra = mapa_shared(smem_u32(cl_best + (round & 1)), (uint32_t)lane);
          uint64_t lo, hi;
          int32_t id, dst, g;
          asm volatile("ld.shared::cluster.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "r"(ra) : "memory");
          asm volatile("ld.shared::cluster.v2.s32 {%0, %1}, [%2];" : "=r"(id), "=r"(dst) : "r"(ra + 16u) : "memory");
          asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(g) : "r"(ra + 24u) : "memory");
          o.score = (i128)(((unsigned __int128)hi << 64) | lo);
          o.id = id;
          o.dst = dst;
          o.g = g;
        }
        c = warp_argmax_g(o);
      }
    }
    if (warp == 0) {
      PLAN_TS(8);
      if (c.g < 0) {
        if (lane == 0) s_stop = 1;
      } else {
        // ExecuteMigration is out of the path: apply m* to the loads for the next round (not
        // after the last one)
        const int src = s.rinst[c.g];
        const int64_t N = s.rntok[c.g], nh = s.rnhat[c.g];
        for (int t = lane; t < (last ? 0 : H1); t += 32) {
          const int64_t ct = (t == 0) ? N : (t < nh ? N + t : 0);
          s.Ls[(int64_t)src * H1 + t] -= ct;
          s.Ls[(int64_t)c.dst * H1 + t] += ct;
        }
        if (lane == 0) {
          s.moved[c.g >> 5] |= 1u << (c.g & 31);
          s.wdirty[src] = s.wdirty[c.dst] = 1;
          s.pdirty[src] = s.pdirty[c.dst] = 1;
        }
        if (lane == 0 && crank == 0) {
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
    PLAN_TS(6);
    if (s_stop) break;
  }
  // no copy may still be in flight when the CTA exits (a plan that stopped before round 0's wait)
  if (a.bulk) {
    if (table_issued) mbar_wait(s.bar, 0);
  } else {
    cp_async_wait_all();
  }
  PLAN_TS(7);
  if (tid == 0 && crank == 0) *a.n_moves = s_nmoves;
  if constexpr (kCl > 1) cluster_sync_all();   // no CTA leaves while a peer may still read its cl_best
#undef PLAN_TS
}

}  // namespace star
