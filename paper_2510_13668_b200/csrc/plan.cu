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
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "plan_core.cuh"
#include "plan_fast.cuh"
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

constexpr int kPlanThreads = 512;

// diagnostics: %globaltimer stamps of the most recent single-CTA plan (star_plan_timeline)
__device__ uint64_t g_plan_tl[64];
__device__ uint64_t g_plan_cl_tl[64];   // per-CTA stamps of the cluster plan: [rank][entry, pdl, pre-sync, post-sync, ...]

cudaError_t plan_timeline(uint64_t* host64) {
  cudaError_t e = cudaMemcpyFromSymbol(host64, g_plan_tl, sizeof(uint64_t) * 64);
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(host64 + 64, g_plan_cl_tl, sizeof(uint64_t) * 64);
  return e;
}


template <bool kStaged>
__global__ void __launch_bounds__(kPlanThreads, 1) plan_kernel(const PlanArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  __shared__ Cand warp_best[kPlanThreads / 32];
  __shared__ int shv[8];
  if (threadIdx.x == 0) g_plan_tl[0] = globaltimer_ns();
  if constexpr (!kStaged) pdl_wait();   // inputs come from the projection / all-gather (PDL launch)
  pdl_launch_dependents();   // (the fast path waits itself, after fetching its static inputs)
  if (threadIdx.x == 0) {
    g_plan_tl[1] = globaltimer_ns();
    g_plan_tl[33] = clock64();
  }
  if constexpr (kStaged)
    plan_cta_fast(a, smraw, (int)threadIdx.x, (int)blockDim.x, warp_best, shv, g_plan_tl);
  else
    plan_cta<CtaSync, false>(a, smraw, (int)threadIdx.x, (int)blockDim.x, CtaSync{}, warp_best, shv, g_plan_tl);
}

// Alg. 1 on a thread-block cluster of kCl CTAs (plan_fast.cuh: candidate compaction and scoring
// split over the CTAs, the round's argmax in distributed shared memory).
static_assert(offsetof(Cand, id) == 16 && offsetof(Cand, dst) == 20 && offsetof(Cand, g) == 24,
              "plan_cta_fast reads peers' Cand fields at these offsets");
template <int kCl>
__global__ void __launch_bounds__(kPlanThreads, 1) plan_cluster_kernel(const PlanArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  __shared__ Cand warp_best[kPlanThreads / 32];
  __shared__ Cand cl_best[2];
  __shared__ int shv[8];
  const bool lead = cluster_ctarank() == 0;
  if (threadIdx.x == 0) {
    g_plan_cl_tl[cluster_ctarank() * 8] = globaltimer_ns();
    g_plan_cl_tl[cluster_ctarank() * 8 + 6] = 0;   // max evaluation cycles (atomicMax below)
  }
  __syncthreads();
  PlanArgs ac = a;
  if (lead && threadIdx.x == 0) g_plan_tl[0] = globaltimer_ns();
  pdl_launch_dependents();
  if (lead && threadIdx.x == 0) {
    g_plan_tl[1] = globaltimer_ns();
    g_plan_tl[33] = clock64();
  }
  ac.cl_tl = g_plan_cl_tl;
  plan_cta_fast<false, kCl>(ac, smraw, (int)threadIdx.x, (int)blockDim.x, warp_best, shv, g_plan_tl, cl_best);
}

// Cluster size of the staged plan by request slots: 8 CTAs split the compaction and the pair
// scoring of a 4096-slot table best, but a cluster of 8 rarely finds a free GPC while the
// predictor holds 128 SMs, so for small tables a smaller cluster that launches early (its static
// staging under the predictor, PDL) wins (same-box A/B: C1, 128 slots: 36.0 us with 2 CTAs vs
// 36.9 us with 8; one rank at 256 requests (2048 gathered slots): 43.0 vs 44.3 us with 4; TGT,
// 4096 slots: 80.2 us with 8 vs 80.7 with 4).  STAR_PLAN_CLUSTER (1, 2, 4 or 8; read once)
// overrides it for A/B measurements.
static int plan_cluster_size(int slots) {
  static int v = [] {
    const char* e = getenv("STAR_PLAN_CLUSTER");
    const int x = e ? atoi(e) : 0;
    return (x == 1 || x == 2 || x == 4 || x == 8) ? x : 0;
  }();
  if (v) return v;
  return slots <= 256 ? 2 : (slots <= 2048 ? 4 : 8);
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
  auto al = [&](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  a.bulk = al(a.req_id) && al(a.inst) && al(a.n_tok) && al(a.n_hat) && (!a.pinned || al(a.pinned)) &&
           (a.world == 1 || (a.seg_stride & 15) == 0);
  return a;
}

cudaError_t launch_plan(const star_plan_params* p, const star_plan_segments* sg, star_move* moves, int32_t* n_moves,
                        int32_t* err_flag, cudaStream_t stream) {
  const PlanArgs a = make_plan_args(p, sg, moves, n_moves, err_flag);
  // Stage the request table in shared memory when it fits (it is re-read every round).
  const size_t lim = (size_t)kMaxSmemBytes - 4096;   // static shared memory + slack
  const bool staged = plan_fast_smem_layout(a.n, a.H, a.world, a.r_cap) <= lim;
  const size_t smem = staged ? plan_fast_smem_layout(a.n, a.H, a.world, a.r_cap)
                             : plan_smem_layout(a.n, a.H, a.world, a.r_cap, false);
  const int ncl = staged ? plan_cluster_size(a.world * plan_fast_pitch(a.r_cap)) : 1;
  auto kern = !staged ? plan_kernel<false>
            : ncl == 8 ? plan_cluster_kernel<8> : ncl == 4 ? plan_cluster_kernel<4>
            : ncl == 2 ? plan_cluster_kernel<2> : plan_kernel<true>;
  if (smem > 48 * 1024) {
    cudaError_t e = func_attr((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // same L1/shared split as the GEMM kernels before it: no SM reconfiguration
  func_attr((const void*)kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ncl, 1, 1);
  cfg.blockDim = dim3(kPlanThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = (unsigned)ncl;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = ncl > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace star
