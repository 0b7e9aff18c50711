// dispatch.cu -- P -> D placement of newly prefilled requests (NEXT-2).
// a finished prefill "will be forwarded to a decode instance according to its input
// length, predicted output length, and the current load of each decode instance"; baselines
// round robin and current KV load.
//
// Projected policy (reading A28): place arrival r on the feasible instance that minimises the
// objective Phi (Eq. 3-4) after the placement.  Adding r's contribution c_t (c_0 = N,
// c_t = (N+t)[t < N_hat]) to instance i raises sum_j L_j[t]^2 by 2 c_t L_i[t] + c_t^2 and leaves
// the i-independent (sum_j L_j[t])^2 term alone, so the argmin is
//     argmin_i  sum_{t<=T} beta_t (N + t) L_i[t]  =  N * P0_i[T] + P1_i[T]
// with the same per-instance beta-weighted prefix sums the plan uses (T = min(H, max(0, N_hat-1))).
// The CPU oracle instead recomputes Phi from scratch for every placement.
//
// One CTA; arrivals are sequential (each placement changes the loads the next one sees):
// threads over instances score, a block argmin on (score, instance id) picks the instance, the
// chosen instance's load row gets c_r and its prefix-sum row is rebuilt by one warp scan.
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
#include "star_internal.h"

namespace star {

typedef __int128 i128;
constexpr int kDispThreads = 512;

struct DispArgs {
  int policy, n, H, A;
  int32_t counter;
  const uint32_t* beta_q;
  int64_t* L;              // [n][H+1] in/out
  const int64_t* c_mem;    // nullable
  const int64_t* reserved; // nullable
  const int32_t* n_tok;
  const int32_t* n_hat;
  int32_t* assign;
  i128* P0;                // [n][H+1] workspace
  i128* P1;
};

__device__ __forceinline__ i128 shfl_up_i128d(i128 v, int off) {
  const unsigned long long lo = __shfl_up_sync(0xFFFFFFFFu, (unsigned long long)v, off);
  const long long hi = __shfl_up_sync(0xFFFFFFFFu, (long long)(v >> 64), off);
  return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}
__device__ __forceinline__ i128 shfl_idx_i128d(i128 v, int src) {
  const unsigned long long lo = __shfl_sync(0xFFFFFFFFu, (unsigned long long)v, src);
  const long long hi = __shfl_sync(0xFFFFFFFFu, (long long)(v >> 64), src);
  return (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
}

// One warp: P0_i[T] = sum_{t<=T} beta_t L_i[t], P1_i[T] = sum_{t<=T} t beta_t L_i[t].
__device__ void disp_prefix_row(const DispArgs& a, const uint32_t* sbeta, int i) {
  __syncwarp();   // reconverge first: shuffles of a diverged warp take a slow path
  const int lane = threadIdx.x & 31, H1 = a.H + 1;
  const int64_t* Li = a.L + (int64_t)i * H1;
  i128 c0 = 0, c1 = 0;
  for (int base = 0; base < H1; base += 32) {
    const int t = base + lane;
    const i128 x = t < H1 ? (i128)sbeta[t] * Li[t] : (i128)0;
    i128 x0 = x, x1 = x * t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const i128 y0 = shfl_up_i128d(x0, off), y1 = shfl_up_i128d(x1, off);
      if (lane >= off) {
        x0 += y0;
        x1 += y1;
      }
    }
    x0 += c0;
    x1 += c1;
    if (t < H1) {
      a.P0[(int64_t)i * H1 + t] = x0;
      a.P1[(int64_t)i * H1 + t] = x1;
    }
    c0 = shfl_idx_i128d(x0, 31);
    c1 = shfl_idx_i128d(x1, 31);
  }
}

struct DKey {
  i128 score;
  int i;   // -1 = none
};
__device__ __forceinline__ bool dkey_less(const DKey& x, const DKey& y) {   // x strictly better
  if (x.i < 0) return false;
  if (y.i < 0) return true;
  if (x.score != y.score) return x.score < y.score;
  return x.i < y.i;
}
__device__ __forceinline__ DKey dkey_shfl(const DKey& k, int m) {
  DKey o;
  const unsigned long long lo = __shfl_xor_sync(0xFFFFFFFFu, (unsigned long long)k.score, m);
  const long long hi = __shfl_xor_sync(0xFFFFFFFFu, (long long)(k.score >> 64), m);
  o.score = (i128)(((unsigned __int128)(unsigned long long)hi << 64) | lo);
  o.i = __shfl_xor_sync(0xFFFFFFFFu, k.i, m);
  return o;
}

__global__ void __launch_bounds__(kDispThreads) dispatch_kernel(const DispArgs a) {
  __shared__ uint32_t sbeta[257];
  __shared__ DKey wbest[kDispThreads / 32];
  __shared__ int s_best;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int H1 = a.H + 1;
  pdl_wait();
  for (int t = tid; t < H1; t += blockDim.x) sbeta[t] = a.beta_q[t];
  __syncthreads();
  if (a.policy == 2)
    for (int i = warp; i < a.n; i += nwarps) disp_prefix_row(a, sbeta, i);
  __syncthreads();
  for (int r = 0; r < a.A; ++r) {
    const int64_t N = a.n_tok[r], nh = a.n_hat[r];
    const int T = (int)(nh - 1 < 0 ? 0 : (nh - 1 > a.H ? a.H : nh - 1));
    if (a.policy == 0) {
      if (tid == 0) s_best = (int)(((int64_t)a.counter + r) % a.n);
    } else {
      DKey best;
      best.score = 0;
      best.i = -1;
      for (int i = tid; i < a.n; i += blockDim.x) {
        DKey k;
        k.i = i;
        if (a.policy == 1) {
          k.score = (i128)a.L[(int64_t)i * H1];
        } else {
          if (a.c_mem) {
            const i128 need = (i128)a.L[(int64_t)i * H1] + (a.reserved ? a.reserved[i] : 0) + N + nh;
            if (!(need <= (i128)a.c_mem[i])) continue;
          }
          k.score = (i128)N * a.P0[(int64_t)i * H1 + T] + a.P1[(int64_t)i * H1 + T];
        }
        if (dkey_less(k, best)) best = k;
      }
      __syncwarp();
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) {
        const DKey o = dkey_shfl(best, m);
        if (dkey_less(o, best)) best = o;
      }
      if (lane == 0) wbest[warp] = best;
      __syncthreads();
      __syncwarp();
      if (warp == 0) {
        DKey k;
        if (lane < nwarps) {
          k = wbest[lane];
        } else {
          k.score = 0;
          k.i = -1;
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
          const DKey o = dkey_shfl(k, m);
          if (dkey_less(o, k)) k = o;
        }
        if (lane == 0) s_best = k.i;
      }
    }
    __syncthreads();
    const int b = s_best;
    if (tid == 0) a.assign[r] = b;
    if (b >= 0) {
      for (int t = tid; t < H1; t += blockDim.x) {   // L_b[t] += c_r[t] (reading A5)
        const int64_t c = t == 0 ? N : (t < nh ? N + t : 0);
        a.L[(int64_t)b * H1 + t] += c;
      }
      __syncthreads();
      if (a.policy == 2 && warp == 0) disp_prefix_row(a, sbeta, b);
    }
    __syncthreads();
  }
}

size_t dispatch_workspace_bytes(int n, int H) { return (size_t)n * (size_t)(H + 1) * 32; }

cudaError_t launch_dispatch(int policy, int n, int H, const uint32_t* beta_q, int64_t* L, const int64_t* c_mem,
                            const int64_t* reserved, int A, const int32_t* n_tok, const int32_t* n_hat,
                            int32_t counter, int32_t* assign, void* workspace, cudaStream_t stream) {
  DispArgs a{};
  a.policy = policy;
  a.n = n;
  a.H = H;
  a.A = A;
  a.counter = counter;
  a.beta_q = beta_q;
  a.L = L;
  a.c_mem = c_mem;
  a.reserved = reserved;
  a.n_tok = n_tok;
  a.n_hat = n_hat;
  a.assign = assign;
  a.P0 = reinterpret_cast<i128*>(workspace);
  a.P1 = a.P0 + (size_t)n * (H + 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, 1, 1);
  cfg.blockDim = dim3(kDispThreads, 1, 1);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dispatch_kernel, a);
}

}  // namespace star
