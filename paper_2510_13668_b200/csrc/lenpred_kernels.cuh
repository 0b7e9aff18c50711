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
// Epilogues:  EPI_RELU_BF16   z = relu(acc + b) -> bf16, staged in 128B-swizzled smem and
//                             written with TMA stores (next layer's A operand)
//             EPI_RELU_TF32X3 z = relu(acc + b) stored as [hi | hi | lo] tf32 split
//                             (3xTF32: next layer computes hi*hi + hi*lo + lo*hi)
//             EPI_HEAD        z3 = relu(acc + b3); y = w4 . z3 + b4; N_hat = quantize(y)
// Split-K (grid.z = S splits, launched as a thread-block cluster of S CTAs along z) when
// the tile count cannot fill the 148 SMs.  Every split owns BN/S of the tile's columns.
// Phase 1: each CTA publishes its fp32 partial of the columns the OTHER splits own, in a
// lane-contiguous layout ([col/4][row][4]: a warp's 32 rows are 512 contiguous bytes);
// cluster barrier; phase 2: each CTA sums the S partials of its own columns in fixed split
// order 0..S-1 (deterministic, run-to-run bit-identical) and runs the epilogue on them.
// The reduction is spread over all S CTAs of the cluster instead of one "last" CTA.
// EPI_HEAD adds a second cluster step: per-owner partial dots w4 . z3 are summed by split 0
// in fixed order.
#pragma once
#include "ptx.cuh"
#include <cuda_bf16.h>

namespace star {

enum : int { EPI_RELU_BF16 = 0, EPI_RELU_TF32X3 = 1, EPI_HEAD = 2 };

struct GemmArgs {
  int M, N;              // output rows (requests) / columns
  int num_kb;            // number of 128-byte K blocks
  int kb_per_split;      // K blocks per split (grid.z splits)
  int splits;            // power of two <= 8, BN/splits multiple of 16
  int epi;
  int tma_store;         // EPI_RELU_BF16: stage in smem + TMA store (owned width % 64 == 0)
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
  float* ws;             // [tiles][splits (producer)][splits (owner)][OW/4][128][4] fp32 partials
  float* head_ws;        // [tiles][splits][128] per-owner partial dots (EPI_HEAD)
  uint64_t* tl;          // diagnostics: [ctas][16] %globaltimer phase stamps, or nullptr
  const int32_t* M_dev;  // device-side row count (refresh mode: rows selected on the device), or nullptr
  int skip_le;           // refresh mode: leave when M_dev <= skip_le (the one-launch small path ran them)
  int* l1_cnt;           // CTA-pair split-K: [cta tiles][2] arrival / done counters (zeroed, self re-arming)
  int prefetch;          // CTA-pair L2 prefetch: 0 = every CTA, 1 = none, 2 = one CTA per tile row / column
  int mn_swap;           // 1-CTA kernel: grid (n tiles, m tiles, splits) instead of (m, n, splits)
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
  static_assert(STAGES * STAGE_BYTES >= 4u * (BN / 64 > 0 ? BN / 64 : 1) * 4096u, "epilogue staging fits");
  // split-K: [0, 32 KB) epilogue staging, [32 KB, +(S-1) x OW x 512 B <= 7/8 x BN x 512 B) partner partials
  static_assert(STAGES * STAGE_BYTES >= 32768u + (uint32_t)BN * 448u, "split-K partials fit");
};

// Fused epilogue on 16 consecutive columns [col0, col0+16) of one row.
//   stage: this warp's 32x128B swizzled staging box (TMA-store path) or nullptr
//   cb   : 16B-chunk index of col0 inside the 64-column box (0, 2, 4, 6)
template <bool TF32>
__device__ __forceinline__ void epilogue16(const GemmArgs& p, int row, int col0, float (&f)[16], float& head_acc,
                                           uint8_t* stage, int cb) {
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] += __ldg(p.bias + col0 + j);
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = fmaxf(f[j], 0.0f);
  if (p.epi == EPI_HEAD) {
#pragma unroll
    for (int j = 0; j < 16; ++j) head_acc = fmaf(__ldg(p.w4 + col0 + j), f[j], head_acc);
    return;
  }
  if (p.epi == EPI_RELU_BF16) {
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&b2);
    }
    if (stage) {   // 128B swizzle: 16B chunk c of row r lives at chunk (c ^ (r & 7))
      const int r = threadIdx.x & 31;
      uint4* rowp = reinterpret_cast<uint4*>(stage + r * 128);
      rowp[(cb) ^ (r & 7)] = make_uint4(w[0], w[1], w[2], w[3]);
      rowp[(cb + 1) ^ (r & 7)] = make_uint4(w[4], w[5], w[6], w[7]);
    } else if (row < p.M) {
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)row * p.ld_out + col0);
      dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
      dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
    return;
  }
  // EPI_RELU_TF32X3: row = [hi (N) | hi (N) | lo (N)]
  if (row >= p.M) return;
  float* base = reinterpret_cast<float*>(p.out) + (int64_t)row * p.ld_out + col0;
  float hi[16], lo[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    hi[j] = tf32_rna(f[j]);
    lo[j] = f[j] - hi[j];
  }
  float4* d0 = reinterpret_cast<float4*>(base);
  float4* d1 = reinterpret_cast<float4*>(base + p.N);
  float4* d2 = reinterpret_cast<float4*>(base + 2 * p.N);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float4 h4 = make_float4(hi[4 * j], hi[4 * j + 1], hi[4 * j + 2], hi[4 * j + 3]);
    d0[j] = h4;
    d1[j] = h4;
    d2[j] = make_float4(lo[4 * j], lo[4 * j + 1], lo[4 * j + 2], lo[4 * j + 3]);
  }
}

template <int BN, bool TF32>
__global__ void __launch_bounds__(192, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const GemmArgs p) {
  using S = GemmSmem<BN>;
  constexpr int BM = 128;
  constexpr int ELEM = TF32 ? 4 : 2;
  constexpr int BK = 128 / ELEM;              // elements per 128-byte K block
  constexpr int UMMA_K = 32 / ELEM;           // K per tcgen05.mma (32 bytes)
  constexpr uint32_t IDESC = umma_idesc(TF32, BM, BN);
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms) by pointer arithmetic on the shared array itself, so
  // the compiler keeps the shared address space (LDS/STS, not generic LD/ST through an integer)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S::STAGES * S::B_BYTES);
  uint64_t* empty = full + S::STAGES;
  uint64_t* accum = empty + S::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  uint64_t* pbar = accum + 2;   // split-K: the partner partial blocks' bulk copies

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint64_t* tl = p.tl ? p.tl + (((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 : nullptr;
  if (tl && threadIdx.x == 0) {
    tl[0] = globaltimer_ns();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tl[15] = smid;
  }
  // mn_swap: grid (n, m, S) -- m-tiles vary slowest, so with a device-side row count the real
  // (low) m-tiles are launched first instead of interleaved with the tiles that leave at once
  const int m_tile = p.mn_swap ? blockIdx.y : blockIdx.x, n_tile = p.mn_swap ? blockIdx.x : blockIdx.y;
  const int split = blockIdx.z;
  const int splits = p.splits;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.num_kb, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;   // >= 1 (host guarantees)

  if (p.M_dev) {   // refresh mode: tiles beyond the device-side row count leave before any setup
    pdl_wait();
    const int md = __ldcg(p.M_dev);
    if (m_tile * BM >= md || md <= p.skip_le) return;   // the whole cluster (same m-tile) leaves
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.tma_store) tma_prefetch_desc(&tmC);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    mbar_init(pbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<S::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tl && threadIdx.x == 0) tl[1] = globaltimer_ns();
  // PDL: the prologue above overlapped the previous kernel's tail; from here on we read
  // (and overwrite) memory it may own.
  pdl_wait();
  pdl_launch_dependents();
  if (tl && threadIdx.x == 0) tl[2] = globaltimer_ns();

  const int OW = BN / splits;                 // columns owned by each split
  const int own0 = split * OW;                // first owned column (tile-relative)
  const int q = warp & 3;                     // TMEM lane quarter accessible to this warp
  const int row_in_tile = q * 32 + lane;
  const int row = m_tile * BM + row_in_tile;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int n0 = n_tile * BN;
  const int tile_id = blockIdx.y * gridDim.x + blockIdx.x;
  float* wsb = p.ws + (int64_t)tile_id * splits * BN * BM;   // this tile's partial blocks

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
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (tl && i == 0) tl[3] = globaltimer_ns();
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
      if (tl) tl[9] = globaltimer_ns();
    }
    __syncwarp();
  } else {
    // ---------------- epilogue phase 1: wait for the accumulator, publish partials --------
    mbar_wait(accum, 0);
    tc_fence_after();
    if (tl && threadIdx.x == 64) tl[10] = globaltimer_ns();
    if (splits > 1) {
      for (int o = 0; o < splits; ++o) {
        if (o == split) continue;
        float4* dst = reinterpret_cast<float4*>(wsb + (int64_t)(split * splits + o) * OW * BM) + row_in_tile;
#pragma unroll 1
        for (int c = 0; c < OW; c += 16) {
          uint32_t v[16];
          tmem_ld_32x32b_x16(trow + (uint32_t)(o * OW + c), v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            dst[(c / 4 + j) * BM] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
      }
      fence_proxy_async_global();   // the owners read these blocks with bulk copies
    }
  }
  if (tl && threadIdx.x == 64) tl[7] = globaltimer_ns();
  if (splits > 1) cluster_sync_all();   // partials of every split of this tile are visible
  if (tl && threadIdx.x == 64) tl[8] = globaltimer_ns();

  float head_acc = 0.0f;
  if (warp >= 2) {
    // ---------------- epilogue phase 2: reduce owned columns (fixed split order) + epilogue ----
    if (splits > 1) {   // partner partials -> shared memory [32 KB, ...) (the ring is free now)
      const uint32_t pblk = (uint32_t)OW * BM * 4u;
      if (threadIdx.x == 64) {
        fence_proxy_async_global();
        mbar_arrive_expect_tx(pbar, (uint32_t)(splits - 1) * pblk);
        for (int s = 0, k = 0; s < splits; ++s) {
          if (s == split) continue;
          bulk_g2s(smem + 32768 + (size_t)(k++) * pblk, wsb + (int64_t)(s * splits + split) * OW * BM, pblk, pbar);
        }
      }
      mbar_wait(pbar, 0);
    }
    uint8_t* stage_base = p.tma_store ? smem + (q * (OW / 64)) * 4096 : nullptr;
#pragma unroll 1
    for (int c = 0; c < OW; c += 16) {
      float f[16];
      if (splits == 1) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(trow + (uint32_t)c, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
      } else {
        // the S-1 partner partial blocks of the owned columns (OW x 128 fp32 each, contiguous)
        // came into shared memory by bulk copy (one L2 round trip); sum in split order 0..S-1
        const float* sP = reinterpret_cast<const float*>(smem + 32768);
        uint32_t v[16];
        tmem_ld_32x32b_x16(trow + (uint32_t)(own0 + c), v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = 0.0f;
        for (int s = 0, k = 0; s < splits; ++s) {
          if (s == split) {
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] += __uint_as_float(v[j]);
          } else {
            const float4* src = reinterpret_cast<const float4*>(sP + (int64_t)(k++) * OW * BM) + row_in_tile;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 x = src[(c / 4 + j) * BM];
              f[4 * j] += x.x;
              f[4 * j + 1] += x.y;
              f[4 * j + 2] += x.z;
              f[4 * j + 3] += x.w;
            }
          }
        }
      }
      uint8_t* stage = stage_base ? stage_base + (c / 64) * 4096 : nullptr;
      epilogue16<TF32>(p, row, n0 + own0 + c, f, head_acc, stage, (c % 64) / 8);
      if (stage && (c % 64) == 48) {   // a 32-row x 64-column box is complete: TMA store it
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, stage, n0 + own0 + (c / 64) * 64, m_tile * BM + q * 32);
          bulk_commit();
        }
      }
    }
    if (stage_base && lane == 0) bulk_wait_all();
    if (tl && threadIdx.x == 64) tl[11] = globaltimer_ns();
    if (p.epi == EPI_HEAD && splits > 1) p.head_ws[((int64_t)tile_id * splits + split) * BM + row_in_tile] = head_acc;
  }
  if (p.epi == EPI_HEAD && splits > 1) cluster_sync_all();   // per-owner partial dots visible
  if (warp >= 2 && p.epi == EPI_HEAD && (splits == 1 || split == 0) && row < p.M) {
    float y = head_acc;
    if (splits > 1) {
      y = 0.0f;
#pragma unroll 8   // splits <= 8: the loads issue together, the sum keeps split order
      for (int s = 0; s < splits; ++s) y += __ldcg(p.head_ws + ((int64_t)tile_id * splits + s) * BM + row_in_tile);
    }
    y += p.b4 ? __ldg(p.b4) : 0.0f;
    if (p.y_hat) p.y_hat[row] = y;
    if (p.n_hat) p.n_hat[row] = quantize_nhat(y, p.n_tok, row, p.max_ctx);
  }
  tc_fence_before();
  __syncthreads();
  if (tl && threadIdx.x == 0) tl[12] = globaltimer_ns();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<S::TMEM_COLS>(tmem);
  }
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2) for the large bf16 layer-1 GEMM: a cluster of two
// CTAs on neighbouring SMs computes one 256 x BN tile.  Each CTA stages its own 128 rows of A
// and HALF of the BN rows of B (so every SM ingests 32 KB per 64-wide K block instead of 48 KB
// for a 128 x 256 single-CTA tile: the per-SM TMA ingest, ~75 B/clk measured, is what bounds
// the single-CTA kernel); the leader CTA issues the 256 x BN MMAs, which read the A and B
// halves from both CTAs' shared memory, and each CTA's TMEM receives its 128 x BN accumulator.
//   full[s]  lives in the leader: both CTAs' TMA loads complete their bytes on it
//   empty[s] / accum live in both CTAs: the leader's commits multicast to the pair
// Epilogue (both CTAs): relu(acc + b) -> bf16 -> 128B-swizzled smem -> TMA store.
constexpr int kPrefetchKB = 8;   // L2 prefetch distance (K blocks) of the GEMM producers

template <int BN>
struct PairSmem {
  static constexpr uint32_t A_BYTES = 128u * 128u;
  static constexpr uint32_t B_BYTES = (uint32_t)(BN / 2) * 128u;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (int)((196u * 1024u) / STAGE_BYTES) > 8 ? 8 : (int)((196u * 1024u) / STAGE_BYTES);
  static constexpr uint32_t BYTES = 1024 + STAGES * STAGE_BYTES + 256;
  static_assert(STAGES * STAGE_BYTES >= 4u * (BN / 64) * 4096u, "epilogue staging fits");
  static_assert(STAGES * STAGE_BYTES >= 32768u + (uint32_t)BN * 448u, "split-K partials fit");
};

// kSplit: the split-K instantiation (grid.z > 1).  A separate instantiation because merely
// compiling the split-K epilogue into the unsplit kernel cost the C2 step ~2 us (measured A/B).
// kNU: N = 2048 as 9 pair tiles of 224 (x7) and 240 (x2) columns instead of 8 x 256, so that
// 8 m-pairs occupy 144 of the 148 SMs (72 pairs) instead of 128; the epilogue stores directly.
template <int BN, bool kSplit = false, bool kNU = false>
__global__ void __launch_bounds__(192, 1)
    umma_pair_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmC, const GemmArgs p) {
  using S = PairSmem<BN>;
  constexpr int BK = 64;
  constexpr uint32_t IDESC = umma_idesc(false, 256, BN);
  static_assert(BN % 64 == 0 && BN >= 64 && BN <= 256, "BN");
  static_assert(!(kNU && kSplit), "non-uniform N tiles are an unsplit form");
  const uint32_t idesc = kNU ? umma_idesc(false, 256, blockIdx.y < 7 ? 224u : 240u) : IDESC;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms) by pointer arithmetic on the shared array itself, so
  // the compiler keeps the shared address space (LDS/STS, not generic LD/ST through an integer)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S::STAGES * S::B_BYTES);
  uint64_t* empty = full + S::STAGES;
  uint64_t* accum = empty + S::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  uint64_t* pbar = accum + 2;   // split-K: the partner partial blocks' bulk copies

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();       // 0 = leader (issues the MMAs), 1 = peer
  uint64_t* tl = p.tl ? p.tl + (((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 : nullptr;
  if (tl && threadIdx.x == 0) {
    tl[0] = globaltimer_ns();
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tl[15] = smid;
  }
  const int m_row0 = blockIdx.x * 128;           // this CTA's 128 rows (pair covers 256)
  const int n_tile = blockIdx.y;
  const int split = blockIdx.z, splits = p.splits;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.num_kb, kb0 + p.kb_per_split) - kb0;   // >= 1 (host guarantees)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    mbar_init(pbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<BN>(tmem_slot);
  tc_fence_before();
  cluster_sync_relaxed();   // barriers of both CTAs initialised (fence.mbarrier_init released them)
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  if (tl && threadIdx.x == 0) tl[1] = globaltimer_ns();

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);   // leader's full[0]
      const int nw_p = kNU ? (n_tile < 7 ? 224 : 240) : BN;
      const int n0_p = kNU ? n_tile * 224 + (n_tile > 7 ? (n_tile - 7) * 16 : 0) : n_tile * BN;
      const int b_row = n0_p + (int)rank * (nw_p / 2);
      auto kcol = [&](int i) { return (kb0 + i) * BK; };
      // the weights do not depend on the previous kernel: their first stages go out before
      // griddepcontrol.wait (PDL overlap)
      const int pre = nkb < S::STAGES ? nkb : S::STAGES;
      for (int i = 0; i < pre; ++i) {
        if (rank == 0) mbar_arrive_expect_tx(&full[i], 2 * S::STAGE_BYTES);
        tma_load_2d_pair(sB + i * S::B_BYTES, &tmB, full0 + (uint32_t)(i * 8), kcol(i), b_row, pol_b);
      }
      pdl_wait();
      if (tl) tl[2] = globaltimer_ns();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        if (i >= pre) {
          mbar_wait(&empty[s], ph ^ 1u);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * S::STAGE_BYTES);
          tma_load_2d_pair(sB + s * S::B_BYTES, &tmB, full0 + (uint32_t)(s * 8), kcol(i), b_row, pol_b);
        }
        tma_load_2d_pair(sA + s * S::A_BYTES, &tmA, full0 + (uint32_t)(s * 8), kcol(i), m_row0, pol_a);
        if (i + kPrefetchKB < nkb && p.prefetch != 1) {   // pull a later K block into L2 (TMA hits L2)
          // prefetch 2: one prefetch per tile row / column (the pair column n_tile 0 fetches A,
          // the pair row 0 fetches B) instead of one per consumer
          if (p.prefetch != 2 || n_tile == 0) tma_prefetch_2d(&tmA, kcol(i + kPrefetchKB), m_row0);
          if (p.prefetch != 2 || blockIdx.x < 2) tma_prefetch_2d(&tmB, kcol(i + kPrefetchKB), b_row);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (rank == 0 && elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (tl && (i & 15) == 0 && i / 16 < 6) tl[3 + i / 16] = globaltimer_ns();   // slots 3..6
        const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * S::A_BYTES));
        const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * S::B_BYTES));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma_pair(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (i | k) != 0 ? 1u : 0u);
        umma_commit_pair(&empty[s], (uint16_t)3);
      }
      umma_commit_pair(accum, (uint16_t)3);
      if (tl) tl[9] = globaltimer_ns();
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (both CTAs): own 128 lanes x BN columns ----------------
    const int q = warp & 3;
    const int row = m_row0 + q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int n0 = kNU ? n_tile * 224 + (n_tile > 7 ? (n_tile - 7) * 16 : 0) : n_tile * BN;
    pdl_wait();   // Z1 may still be read by the previous kernel
    mbar_wait(accum, 0);
    tc_fence_after();
    if (tl && threadIdx.x == 64) tl[10] = globaltimer_ns();
    float head_acc = 0.0f;
    if (kSplit) {
      // ---- split-K: the S CTAs computing this CTA's 128 x BN block over disjoint K ranges meet
      // through an arrival counter in global memory (the grid is one wave of <= 148 CTAs, every
      // CTA resident, so the wait cannot starve).  Each split publishes the columns the other
      // splits own (fp32, lane-contiguous [col/4][row][4]), then reduces its own BN/S columns in
      // the fixed split order 0..S-1 (deterministic) and runs the epilogue on them.
      const int OW = BN / splits, own0 = split * OW;
      const int row_in_tile = q * 32 + lane;
      const int cta_tile = blockIdx.y * gridDim.x + blockIdx.x;
      float* wsb = p.ws + (int64_t)cta_tile * splits * BN * 128;
      for (int o = 0; o < splits; ++o) {
        if (o == split) continue;
        float4* dst = reinterpret_cast<float4*>(wsb + (int64_t)(split * splits + o) * OW * 128) + row_in_tile;
#pragma unroll 1
        for (int c = 0; c < OW; c += 32) {
          uint32_t v[16], u[16];
          tmem_ld_32x32b_x16(trow + (uint32_t)(o * OW + c), v);
          tmem_ld_32x32b_x16(trow + (uint32_t)(o * OW + c + 16), u);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            dst[(c / 4 + j) * 128] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                 __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
            dst[(c / 4 + 4 + j) * 128] = make_float4(__uint_as_float(u[4 * j]), __uint_as_float(u[4 * j + 1]),
                                                     __uint_as_float(u[4 * j + 2]), __uint_as_float(u[4 * j + 3]));
          }
        }
      }
      fence_proxy_async_global();   // the owners read these blocks with bulk copies
      fence_acq_rel_gpu();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tl && threadIdx.x == 64) tl[7] = globaltimer_ns();
      if (threadIdx.x == 64) {
        int* ctr = p.l1_cnt + 2 * cta_tile;
        atomicAdd(ctr, 1);
        spin_wait_geq(ctr, splits);   // co-residency checked on the host; traps after ~2 s
        if (tl) tl[8] = globaltimer_ns();
        // the S-1 partner blocks of the owned columns -> shared memory [32 KB, ...) (ring is free)
        const uint32_t pblk = (uint32_t)OW * 128u * 4u;
        fence_proxy_async_global();
        mbar_arrive_expect_tx(pbar, (uint32_t)(splits - 1) * pblk);
        for (int s = 0, k = 0; s < splits; ++s) {
          if (s == split) continue;
          bulk_g2s(smem + 32768 + (size_t)(k++) * pblk, wsb + (int64_t)(s * splits + split) * OW * 128, pblk, pbar);
        }
      }
      mbar_wait(pbar, 0);
      uint8_t* stage_base = (OW % 64 == 0) ? smem + (q * (OW / 64)) * 4096 : nullptr;
#pragma unroll 1
      for (int c = 0; c < OW; c += 16) {
        const float* sP = reinterpret_cast<const float*>(smem + 32768);
        uint32_t v[16];
        tmem_ld_32x32b_x16(trow + (uint32_t)(own0 + c), v);
        tmem_ld_wait();
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = 0.0f;
        for (int s = 0, k = 0; s < splits; ++s) {   // fixed split order (deterministic)
          if (s == split) {
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] += __uint_as_float(v[j]);
          } else {
            const float4* src = reinterpret_cast<const float4*>(sP + (int64_t)(k++) * OW * 128) + row_in_tile;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 x = src[(c / 4 + j) * 128];
              f[4 * j] += x.x;
              f[4 * j + 1] += x.y;
              f[4 * j + 2] += x.z;
              f[4 * j + 3] += x.w;
            }
          }
        }
        uint8_t* stage = stage_base ? stage_base + (c / 64) * 4096 : nullptr;
        epilogue16<false>(p, row, n0 + own0 + c, f, head_acc, stage, (c % 64) / 8);
        if (stage && (c % 64) == 48) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, stage, n0 + own0 + (c / 64) * 64, m_row0 + q * 32);
            bulk_commit();
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) {   // the last split to finish re-arms the counter for the next launch
        int* ctr = p.l1_cnt + 2 * cta_tile;
        if (atomicAdd(ctr + 1, 1) == splits - 1) {
          ctr[0] = 0;
          ctr[1] = 0;
        }
      }
    } else if (kNU) {   // 224- or 240-column tile: 16-column chunks, direct 32-byte row stores
      const int nw = n_tile < 7 ? 224 : 240;
#pragma unroll 1
      for (int c = 0; c < nw; c += 32) {
        uint32_t v[16], u[16];
        tmem_ld_32x32b_x16(trow + (uint32_t)c, v);
        if (c + 16 < nw) tmem_ld_32x32b_x16(trow + (uint32_t)(c + 16), u);
        tmem_ld_wait();
        float f[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
        epilogue16<false>(p, row, n0 + c, f, head_acc, nullptr, 0);
        if (c + 16 < nw) {
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(u[j]);
          epilogue16<false>(p, row, n0 + c + 16, f, head_acc, nullptr, 0);
        }
      }
    } else {
    uint8_t* stage_base = smem + (q * (BN / 64)) * 4096;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[16], u[16];
      tmem_ld_32x32b_x16(trow + (uint32_t)c, v);
      tmem_ld_32x32b_x16(trow + (uint32_t)(c + 16), u);
      tmem_ld_wait();
      float f[16], g[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        f[j] = __uint_as_float(v[j]);
        g[j] = __uint_as_float(u[j]);
      }
      uint8_t* stage = stage_base + (c / 64) * 4096;
      epilogue16<false>(p, row, n0 + c, f, head_acc, stage, (c % 64) / 8);
      epilogue16<false>(p, row, n0 + c + 16, g, head_acc, stage, (c % 64) / 8 + 2);
      if ((c % 64) == 32) {   // a 32-row x 64-column box is complete: TMA store it
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, stage, n0 + (c / 64) * 64, m_row0 + q * 32);
          bulk_commit();
        }
      }
    }
    }
    if (lane == 0) bulk_wait_all();
    if (tl && threadIdx.x == 64) tl[11] = globaltimer_ns();
  }
  tc_fence_before();
  cluster_sync_relaxed();   // the pair's MMAs and TMEM reads are done before the pair frees TMEM
  if (tl && threadIdx.x == 0) tl[12] = globaltimer_ns();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<BN>(tmem);
  }
}

// Persistent form of the 9-column-tile pair GEMM for layer 1 over two tiles per CTA pair (e.g.
// M = 4096: 16 row pairs x 9 column tiles = 144 pair tiles on 72 pairs): the grid is one wave;
// pair P computes tiles P and P + npairs (tile t = row pair t / 9, column tile t % 9), the second
// tile's mainloop into the other half of a 512-column TMEM allocation while the epilogue stores
// the first (the epilogue no longer idles the tensor core, and there is no second-wave launch).
template <int BN>
__global__ void __launch_bounds__(192, 1)
    umma_pair_nu2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const GemmArgs p, int ntiles) {
  using S = PairSmem<BN>;
  constexpr int BK = 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S::STAGES * S::B_BYTES);
  uint64_t* empty = full + S::STAGES;
  uint64_t* accum = empty + S::STAGES;   // [2]: one per tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();       // 0 = leader (issues the MMAs), 1 = peer
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nmine = (pair + npairs < ntiles) ? 2 : 1;
  const int nkb = p.num_kb;
  auto tile_geom = [&](int j, int& m_row0, int& n0, int& nw) {
    const int t = pair + j * npairs;
    const int mp = t / 9, nt = t % 9;
    m_row0 = mp * 256 + (int)rank * 128;
    nw = nt < 7 ? 224 : 240;
    n0 = nt * 224 + (nt > 7 ? (nt - 7) * 16 : 0);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&accum[0], 1);
    mbar_init(&accum[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync_relaxed();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {   // TMA producer (both CTAs): the two tiles back to back through one ring
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
      const int pre = nkb < S::STAGES ? nkb : S::STAGES;
      int m_row0, n0, nw;
      tile_geom(0, m_row0, n0, nw);
      for (int i = 0; i < pre; ++i) {   // weights before griddepcontrol.wait
        if (rank == 0) mbar_arrive_expect_tx(&full[i], 2 * S::STAGE_BYTES);
        tma_load_2d_pair(sB + i * S::B_BYTES, &tmB, full0 + (uint32_t)(i * 8), i * BK, n0 + (int)rank * (nw / 2), pol_b);
      }
      pdl_wait();
      for (int j = 0; j < nmine; ++j) {
        tile_geom(j, m_row0, n0, nw);
        const int b_row = n0 + (int)rank * (nw / 2);
        for (int i = 0; i < nkb; ++i) {
          const int it = j * nkb + i, s = it % S::STAGES;
          const uint32_t ph = (uint32_t)(it / S::STAGES) & 1u;
          if (it >= pre) {
            mbar_wait(&empty[s], ph ^ 1u);
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * S::STAGE_BYTES);
            tma_load_2d_pair(sB + s * S::B_BYTES, &tmB, full0 + (uint32_t)(s * 8), i * BK, b_row, pol_b);
          }
          tma_load_2d_pair(sA + s * S::A_BYTES, &tmA, full0 + (uint32_t)(s * 8), i * BK, m_row0, pol_a);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {   // MMA issuer (leader): tile j into TMEM columns [256 j, +nw)
      for (int j = 0; j < nmine; ++j) {
        int m_row0, n0, nw;
        tile_geom(j, m_row0, n0, nw);
        const uint32_t idesc = umma_idesc(false, 256, (uint32_t)nw);
        for (int i = 0; i < nkb; ++i) {
          const int it = j * nkb + i, s = it % S::STAGES;
          mbar_wait(&full[s], (uint32_t)(it / S::STAGES) & 1u);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * S::A_BYTES));
          const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * S::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_pair(tmem + 256u * j, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), idesc, (i | k) != 0 ? 1u : 0u);
          umma_commit_pair(&empty[s], (uint16_t)3);
        }
        umma_commit_pair(&accum[j], (uint16_t)3);
      }
    }
    __syncwarp();
  } else {
    // epilogue (both CTAs): own 128 lanes of each tile; tile 0's stores overlap tile 1's mainloop
    const int q = warp & 3;
    const uint32_t trow0 = tmem + ((uint32_t)(q * 32) << 16);
    pdl_wait();   // Z1 may still be read by the previous kernel
    float head_acc = 0.0f;
    for (int j = 0; j < nmine; ++j) {
      int m_row0, n0, nw;
      tile_geom(j, m_row0, n0, nw);
      const int row = m_row0 + q * 32 + lane;
      const uint32_t trow = trow0 + 256u * j;
      mbar_wait(&accum[j], 0);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < nw; c += 32) {
        uint32_t v[16], u[16];
        tmem_ld_32x32b_x16(trow + (uint32_t)c, v);
        if (c + 16 < nw) tmem_ld_32x32b_x16(trow + (uint32_t)(c + 16), u);
        tmem_ld_wait();
        float f[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) f[jj] = __uint_as_float(v[jj]);
        epilogue16<false>(p, row, n0 + c, f, head_acc, nullptr, 0);
        if (c + 16 < nw) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) f[jj] = __uint_as_float(u[jj]);
          epilogue16<false>(p, row, n0 + c + 16, f, head_acc, nullptr, 0);
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_relaxed();   // the pair's MMAs and TMEM reads are done before the pair frees TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
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
