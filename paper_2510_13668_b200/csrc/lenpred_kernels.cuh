// lenpred_kernels.cuh -- Eq. 2 on sm_100a tensor cores.
//
//   y_hat = w4 . phi(W3 phi(W2 phi(W1 h)))
//
// Each of the three dense layers is one launch of `umma_gemm_kernel`: a warp-specialised
// tcgen05 GEMM  C[M x N] = A[M x K] . B[N x K]^T  with both operands K-major (A = the
// activations, one row per running request; B = the nn.Linear weight [out][in]).
//   warp 0      TMA producer   (cp.async.bulk.tensor 2D, SWIZZLE_128B, STAGES-deep ring)
//   warp 1      MMA issuer     (one elected lane, tcgen05.mma cta_group::1, M=128, N=BN,
//                               accumulator in TMEM; tcgen05.commit frees smem slots)
//   warps 2..5  epilogue       (tcgen05.ld 32x32b -> registers -> fused epilogue -> HBM)
// Epilogues:  EPI_RELU_BF16   z = relu(acc + b) stored bf16 (next layer's A operand)
//             EPI_RELU_TF32X3 z = relu(acc + b) stored as [hi | hi | lo] tf32 split
//                             (3xTF32: next layer computes hi*hi + hi*lo + lo*hi)
//             EPI_HEAD        z3 = relu(acc + b3); y = w4 . z3 + b4; N_hat = quantize(y)
// Split-K (grid.z) when the tile count cannot fill the 148 SMs: each split writes its fp32
// partial tile, the last-arriving CTA of a tile sums the partials in fixed split order
// (deterministic, run-to-run bit-identical) and runs the epilogue.
#pragma once
#include "ptx.cuh"
#include <cuda_bf16.h>

namespace star {

enum : int { EPI_RELU_BF16 = 0, EPI_RELU_TF32X3 = 1, EPI_HEAD = 2 };

struct GemmArgs {
  int M, N;              // output rows (requests) / columns
  int num_kb;            // number of 128-byte K blocks
  int kb_per_split;      // K blocks per split (grid.z splits)
  int splits;
  int epi;
  void* out;             // EPI_RELU_*: output matrix
  int64_t ld_out;        // elements between output rows
  const float* bias;     // [N] or nullptr
  // EPI_HEAD
  const float* w4;       // [N] (N == 64)
  const float* b4;       // [1] or nullptr
  const int32_t* n_tok;  // [M] or nullptr
  int32_t max_ctx;
  float* y_hat;          // [M] or nullptr
  int32_t* n_hat;        // [M] or nullptr
  // split-K
  float* ws;             // [splits][M][N] fp32 partials
  int* counters;         // [tiles] arrival counters (zero between launches)
};

// Quantizer (readings A8-A10): cap = max(0, L_ctx - N(r)) (no n_tok -> L_ctx);
// N_hat = rint_half_even(fminf(fmaxf(y, 0), cap)).  fmaxf returns the non-NaN operand.
__device__ __forceinline__ int32_t quantize_nhat(float y, const int32_t* n_tok, int r, int32_t max_ctx) {
  int32_t cap = max_ctx;
  if (n_tok) cap = max_ctx - n_tok[r];
  cap = cap < 0 ? 0 : cap;
  float v = fmaxf(y, 0.0f);
  v = fminf(v, (float)cap);
  return __float2int_rn(v);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <int BN>
struct GemmSmem {
  static constexpr uint32_t A_BYTES = 128u * 128u;
  static constexpr uint32_t B_BYTES = (uint32_t)BN * 128u;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (int)((196u * 1024u) / STAGE_BYTES) > 8 ? 8 : (int)((196u * 1024u) / STAGE_BYTES);
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr uint32_t BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/;
};

// Epilogue warps: apply the fused epilogue to 32 consecutive columns [c0, c0+32) of one row.
template <int BN, bool TF32>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& p, int row, int col0, float (&f)[32],
                                               float& head_acc) {
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] += __ldg(p.bias + col0 + j);
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = fmaxf(f[j], 0.0f);
  if (p.epi == EPI_HEAD) {
#pragma unroll
    for (int j = 0; j < 32; ++j) head_acc = fmaf(__ldg(p.w4 + col0 + j), f[j], head_acc);
    return;
  }
  if (row >= p.M) return;
  if (p.epi == EPI_RELU_BF16) {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&b2);
    }
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.ld_out + col0);
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  } else {  // EPI_RELU_TF32X3: row = [hi (N) | hi (N) | lo (N)]
    float* base = reinterpret_cast<float*>(p.out) + (int64_t)row * p.ld_out + col0;
    float hi[32], lo[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      hi[j] = tf32_rna(f[j]);
      lo[j] = f[j] - hi[j];
    }
    float4* d0 = reinterpret_cast<float4*>(base);
    float4* d1 = reinterpret_cast<float4*>(base + p.N);
    float4* d2 = reinterpret_cast<float4*>(base + 2 * p.N);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 h4 = make_float4(hi[4 * j], hi[4 * j + 1], hi[4 * j + 2], hi[4 * j + 3]);
      d0[j] = h4;
      d1[j] = h4;
      d2[j] = make_float4(lo[4 * j], lo[4 * j + 1], lo[4 * j + 2], lo[4 * j + 3]);
    }
  }
}

template <int BN, bool TF32>
__global__ void __launch_bounds__(192, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs p) {
  using S = GemmSmem<BN>;
  constexpr int BM = 128;
  constexpr int ELEM = TF32 ? 4 : 2;
  constexpr int BK = 128 / ELEM;              // elements per 128-byte K block
  constexpr int UMMA_K = 32 / ELEM;           // K per tcgen05.mma (32 bytes)
  constexpr uint32_t IDESC = umma_idesc(TF32, BM, BN);
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S::STAGES * S::B_BYTES);
  uint64_t* empty = full + S::STAGES;
  uint64_t* accum = empty + S::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.num_kb, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<S::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_first();   // activations: streamed once per n-tile column
      const uint64_t pol_b = policy_evict_last();    // weights: re-read by every m-tile
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
        const int kc = (kb0 + i) * BK;
        tma_load_2d(sA + s * S::A_BYTES, &tmA, &full[s], kc, m_tile * BM, pol_a);
        tma_load_2d(sB + s * S::B_BYTES, &tmB, &full[s], kc, n_tile * BN, pol_b);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * S::A_BYTES));
        const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * S::B_BYTES));
#pragma unroll
        for (int k = 0; k < BK / UMMA_K; ++k) {
          // advance the start address by k*32 bytes inside the 128-byte swizzle atom
          umma_ss<TF32>(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), IDESC, (i | k) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(accum);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int row = m_tile * BM + q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int n0 = n_tile * BN;
    mbar_wait(accum, 0);
    tc_fence_after();
    float head_acc = 0.0f;
    if (p.splits == 1) {
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(trow + c * 32, v);
        tmem_ld_wait();
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        epilogue_chunk<BN, TF32>(p, row, n0 + c * 32, f, head_acc);
      }
    } else {
      // 1) publish this split's fp32 partial tile
      float* mine = p.ws + ((int64_t)split * p.M + row) * p.N + n0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(trow + c * 32, v);
        tmem_ld_wait();
        if (row < p.M) {
          float4* d = reinterpret_cast<float4*>(mine + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            d[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                               __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int tile_id = blockIdx.y * gridDim.x + blockIdx.x;
      if (warp == 2 && lane == 0) {
        const int prev = atomicAdd(p.counters + tile_id, 1);
        *last_flag = (prev == p.splits - 1) ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
        __threadfence();
        // 2) last arriving split: fixed-order reduction of all partials + epilogue
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float f[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] = 0.0f;
          if (row < p.M) {
            for (int s = 0; s < p.splits; ++s) {
              const float4* src = reinterpret_cast<const float4*>(p.ws + ((int64_t)s * p.M + row) * p.N + n0 + c * 32);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 x = __ldcg(src + j);
                f[4 * j] += x.x;
                f[4 * j + 1] += x.y;
                f[4 * j + 2] += x.z;
                f[4 * j + 3] += x.w;
              }
            }
          }
          epilogue_chunk<BN, TF32>(p, row, n0 + c * 32, f, head_acc);
        }
        if (warp == 2 && lane == 0) p.counters[tile_id] = 0;  // re-arm for the next launch
      }
    }
    if (p.epi == EPI_HEAD && (p.splits == 1 || *last_flag) && row < p.M) {
      const float y = head_acc + (p.b4 ? __ldg(p.b4) : 0.0f);
      if (p.y_hat) p.y_hat[row] = y;
      if (p.n_hat) p.n_hat[row] = quantize_nhat(y, p.n_tok, row, p.max_ctx);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<S::TMEM_COLS>(tmem);
  }
}

// 3xTF32 operand preparation: x [R][K] fp32 (row stride ld) -> out [R][3K]
//   pattern A: [hi | hi | lo]   (activations)     pattern B: [hi | lo | hi] (weights)
// so that A'.B'^T = hi.hi + hi.lo + lo.hi (the lo.lo term, ~2^-22 relative, is dropped).
__global__ void tf32x3_split_kernel(const float* __restrict__ x, int64_t ld, int R, int K, float* __restrict__ out,
                                    int pattern_b) {
  const int64_t total = (int64_t)R * K;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx / K), k = (int)(idx % K);
    const float v = x[(int64_t)r * ld + k];
    const float hi = tf32_rna(v);
    const float lo = v - hi;
    float* o = out + (int64_t)r * 3 * K;
    o[k] = hi;
    o[K + k] = pattern_b ? lo : hi;
    o[2 * K + k] = pattern_b ? hi : lo;
  }
}

__global__ void quantize_kernel(const float* __restrict__ y, const int32_t* __restrict__ n_tok, int R,
                                int32_t max_ctx, int32_t* __restrict__ n_hat) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x)
    n_hat[r] = quantize_nhat(y[r], n_tok, r, max_ctx);
}

}  // namespace star
