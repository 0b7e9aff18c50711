// lenpred_tail.cuh -- fused predictor tail of Eq. 2 for bf16 predictors:
//
//   Z2 = phi(W2 Z1 + b2)   ->   Z3 = phi(W3 Z2 + b3)   ->   y = w4 . Z3 + b4   ->   N_hat = q(y)
//   [-> keyed projection histogram of (instance, min(N_hat, H+1)) -> per-instance loads]
//
// in ONE launch, so Z2 / Z3 never leave the chip and the head and projection kernels (each a
// full launch + global round trips) disappear from the step.
//
// Grid (m_tiles, n2_tiles = m2/256, S splits); one thread-block cluster = the S split-K CTAs
// of one 128 x 256 layer-2 tile (clusters of 8 do not all fit at once on a 148-SM B200: at most
// 15 are co-resident, so the m-tile's n2 clusters meet through an arrival counter instead).
// Per CTA (192 threads, warp-specialised like umma_gemm_kernel):
//   1. layer 2: split-K tcgen05 GEMM of a 128 x 256 tile over K/S (TMA -> SMEM ring -> TMEM).
//   2. split-K exchange inside the cluster: each CTA publishes the fp32 partials of the columns
//      the other splits own (lane-contiguous layout), cluster barrier, and reduces its own
//      OW = 256/S columns in fixed split order (deterministic).
//   3. epilogue: + b2, ReLU, bf16 -> written straight into SMEM as the 128B-swizzled K-major
//      A operand of layer 3 (no global Z2).
//   4. layer 3 partial: tcgen05 M=128, N=64, K=OW against the W3[:, owned columns] block
//      (TMA-loaded at kernel start) -> TMEM columns [256, 320).
//   5. Z3 partials (128 x 64 fp32 per CTA) are published; cluster barrier; split r reduces rows
//      [r*128/S, (r+1)*128/S) over the S partials (fixed order) into the tile's n-tile partial;
//      the last of the n2 tiles to finish that row group (arrival counter) sums the n2 partials
//      in n-tile order, applies + b3, ReLU, the w4 dot (fixed shuffle tree), + b4 and the
//      quantizer.
//   6. (optional) the row owners add (instance, N_hat bin, N) into the global projection
//      histogram (warp-aggregated atomics); the last finisher of the grid finalises L/W/peak/
//      growth/count exactly like the standalone projection and re-zeroes the workspace.
#pragma once
#include "lenpred_kernels.cuh"
#include "project_core.cuh"
#include "plan_fast.cuh"

namespace star {

struct TailArgs {
  int M;               // rows (requests)
  int num_kb;          // layer-2 K blocks (m1 / 64)
  int kb_per_split;
  int splits;          // S in {2, 4}
  int n2_tiles;        // m2 / 256
  const float* b2;     // [m2] or nullptr
  const float* b3;     // [64] or nullptr
  const float* w4;     // [64]
  const float* b4;     // [1] or nullptr
  const int32_t* n_tok;
  int32_t max_ctx;
  float* y_hat;        // [M] or nullptr
  int32_t* n_hat;      // [M] or nullptr
  float* ws2;          // layer-2 partials [tile][S][S][OW/4][128][4]
  float* ws3a;         // layer-3 split partials [m_tile][n2][S][16][128][4]
  float* ws3b;         // layer-3 n-tile partials [m_tile][n2][128][64]
  int* cnt;            // [m_tiles][S] arrival counters (zero between launches)
  int project;         // fuse the projection (pa valid)
  ProjArgs pa;         // R / inst / n_tok / beta_q / outputs / workspace (ws_cnt, ws_sum, ws_arrive)
  uint64_t* tl;        // diagnostics: [ctas][16] %globaltimer phase stamps, or nullptr
  const int32_t* M_dev;  // device-side row count (refresh mode), or nullptr (then M)
  int skip_le;           // refresh mode: leave when M_dev <= skip_le (the one-launch small path ran them)
  int mn_swap;           // grid (n2 tiles, m tiles, splits): real m-tiles launch first (refresh mode)
  int plan;            // the projection's last finisher then runs Alg. 1 (one rank: pl reads this
                       // rank's own record), with the whole CTA, in the freed stage ring
  PlanArgs pl;
};

// Phase timestamp (diagnostics only; one designated thread per phase).  Row stride
// kTailTlStride: slots 0-14 phases, 15 the SM id, 16-19 the last finisher's projection finalize.
constexpr int kTailTlStride = 32;
constexpr int kTailPlanTlRow = 4 * 148 - 2;   // rows 590-591 of the [4 * SMs][32] buffer: fused-plan stamps
#define TAIL_TS(k)                                                                                        \
  do {                                                                                                    \
    if (p.tl) p.tl[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * kTailTlStride + (k)] = globaltimer_ns(); \
  } while (0)

struct TailSmem {
  static constexpr uint32_t A_BYTES = 128u * 128u;   // 128 rows x 64 bf16
  static constexpr uint32_t B_BYTES = 256u * 128u;   // 256 rows x 64 bf16
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = 4;
  static constexpr uint32_t W3_BYTES = 2u * 64u * 128u;   // W3 block, up to 2 K blocks (OW <= 128)
  static constexpr uint32_t OFF_W3 = STAGES * STAGE_BYTES;
  static constexpr uint32_t OFF_BAR = OFF_W3 + W3_BYTES;
  static constexpr uint32_t OFF_CONST = OFF_BAR + 256;
  static constexpr uint32_t CONST_BYTES = (128 + 64 + 64 + 260) * 4;
  static constexpr uint32_t BYTES = 1024 + OFF_CONST + CONST_BYTES;
};

// kPlan: the instantiation with the fused Alg. 1 (one rank); the others do not carry the plan's
// code (its mere presence in a kernel measurably changes the code generated for the rest).
template <bool kPlan>
__global__ void __launch_bounds__(192, 1)
    tail_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmW3, const TailArgs p) {
  using S = TailSmem;
  constexpr int BM = 128, BN = 256, BK = 64;
  constexpr uint32_t IDESC2 = umma_idesc(false, BM, BN);
  constexpr uint32_t IDESC3 = umma_idesc(false, BM, 64);

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms) by pointer arithmetic on the shared array itself, so
  // the compiler keeps the shared address space (LDS/STS, not generic LD/ST through an integer)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S::STAGES * S::A_BYTES;
  uint8_t* sW3 = smem + S::OFF_W3;
  // after layer 2 the stage ring is reused: [0, 32K) layer-3 A operand (Z2 owned block),
  // [32K, 128K) the other splits' layer-2 partial blocks, [128K, 160K) layer-3 partial blocks
  uint8_t* sA3 = smem;
  float* sP2 = reinterpret_cast<float*>(smem + 32768);
  float* sZ3 = reinterpret_cast<float*>(smem + 131072);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  uint64_t* empty = full + S::STAGES;
  uint64_t* accum = empty + S::STAGES;
  uint64_t* w3bar = accum + 1;
  uint64_t* a3bar = w3bar + 1;
  uint64_t* l3bar = a3bar + 1;
  uint64_t* pbar = l3bar + 1;   // layer-2 partial blocks landed in shared memory
  uint64_t* zbar = pbar + 1;    // layer-3 partial blocks landed in shared memory
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(zbar + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* sb2 = reinterpret_cast<float*>(smem + S::OFF_CONST);   // [OW] owned slice of b2
  float* sb3 = sb2 + 128;                                       // [64]
  float* sw4 = sb3 + 64;                                        // [64]
  uint32_t* sbeta = reinterpret_cast<uint32_t*>(sw4 + 64);      // [H+1] (projection)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    TAIL_TS(0);
    if (p.tl) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.tl[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * kTailTlStride + 15] = smid;
    }
  }
  const int m_tile = p.mn_swap ? blockIdx.y : blockIdx.x, n_tile = p.mn_swap ? blockIdx.x : blockIdx.y;
  const int split = blockIdx.z;
  const int splits = p.splits;
  const int OW = BN / splits;                  // owned Z2 columns (128 or 64)
  const int OWK = OW / 64;                     // layer-3 K blocks (2 or 1)
  const int own0 = split * OW;
  const int n0 = n_tile * BN;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.num_kb, kb0 + p.kb_per_split) - kb0;

  int Mrows = p.M;
  if (p.M_dev) {   // refresh mode: the row count was produced on the device by the previous kernels
    pdl_wait();
    Mrows = __ldcg(p.M_dev);
    if (m_tile * BM >= Mrows || Mrows <= p.skip_le) return;   // every CTA of this m-tile (and its cluster) leaves
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmW3);
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    mbar_init(w3bar, 1);
    *s_last = 0;
    mbar_init(a3bar, 4);   // one arrive per epilogue warp
    mbar_init(l3bar, 1);
    mbar_init(pbar, 1);
    mbar_init(zbar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  if (threadIdx.x == 0) TAIL_TS(1);

  const int q = warp & 3;
  const int row_in_tile = q * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int tile_id = m_tile * p.n2_tiles + n_tile;
  float* wsb = p.ws2 + (int64_t)tile_id * splits * BN * BM;

  // final-reduction geometry: split r owns rows [r*rpr, (r+1)*rpr) of the m-tile
  const int rpr = BM / splits;                 // rows per split (32 or 64)
  const int tpr = splits;                      // threads per row (4 or 2)
  const int cpt = 64 / tpr;                    // Z3 columns per thread (16 or 32)
  const int te = threadIdx.x - 64;             // epilogue thread index 0..127
  const int red_row = split * rpr + (te >= 0 ? te / tpr : 0);
  const int red_g = te >= 0 ? te % tpr : 0;
  const int grow = m_tile * BM + red_row;
  int32_t my_ntok = 0, my_inst = 0;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_first();
      const uint64_t pol_b = policy_evict_last();
      // weights do not depend on the previous kernel: W3 block + the first W2 stages go out
      // before griddepcontrol.wait (PDL overlap)
      mbar_arrive_expect_tx(w3bar, (uint32_t)OWK * 8192u);
      for (int kk = 0; kk < OWK; ++kk) tma_load_2d(sW3 + kk * 8192, &tmW3, w3bar, n0 + own0 + kk * 64, 0, pol_b);
      const int pre = nkb < S::STAGES ? nkb : S::STAGES;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], S::STAGE_BYTES);
        tma_load_2d(sB + i * S::B_BYTES, &tmB, &full[i], (kb0 + i) * BK, n0, pol_b);
      }
      pdl_wait();
      TAIL_TS(2);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        if (i >= pre) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
          tma_load_2d(sB + s * S::B_BYTES, &tmB, &full[s], (kb0 + i) * BK, n0, pol_b);
        }
        tma_load_2d(sA + s * S::A_BYTES, &tmA, &full[s], (kb0 + i) * BK, m_tile * BM, pol_a);
      }
      TAIL_TS(3);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (layer 2) ----------------
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % S::STAGES;
        const uint32_t ph = (uint32_t)(i / S::STAGES) & 1u;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * S::A_BYTES));
        const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * S::B_BYTES));
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_ss<false>(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), IDESC2, (i | k) != 0 ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(accum);
      TAIL_TS(4);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps: constants, then layer-2 split-K publish ----------------
    for (int i = te; i < OW; i += 128) sb2[i] = p.b2 ? __ldg(p.b2 + n0 + own0 + i) : 0.0f;
    for (int i = te; i < 64; i += 128) {
      sb3[i] = p.b3 ? __ldg(p.b3 + i) : 0.0f;
      sw4[i] = __ldg(p.w4 + i);
    }
    pdl_wait();
    if (p.project)
      for (int t = te; t <= p.pa.H; t += 128) sbeta[t] = p.pa.beta_q[t];
    if (red_g == 0 && grow < Mrows) {
      if (p.n_tok) my_ntok = p.n_tok[grow];
      if (p.project) my_inst = p.pa.inst[grow];
    }
    if (te == 0) TAIL_TS(5);
    mbar_wait(accum, 0);
    tc_fence_after();
    if (te == 0) TAIL_TS(6);
    for (int o = 0; o < splits; ++o) {
      if (o == split) continue;
      float4* dst = reinterpret_cast<float4*>(wsb + (int64_t)(split * splits + o) * OW * BM) + row_in_tile;
#pragma unroll 1
      for (int c = 0; c < OW; c += 32) {
        uint32_t v[16], u[16];
        tmem_ld_32x32b_x16(trow + (uint32_t)(o * OW + c), v);
        tmem_ld_32x32b_x16(trow + (uint32_t)(o * OW + c + 16), u);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dst[(c / 4 + j) * BM] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                              __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          dst[(c / 4 + 4 + j) * BM] = make_float4(__uint_as_float(u[4 * j]), __uint_as_float(u[4 * j + 1]),
                                                  __uint_as_float(u[4 * j + 2]), __uint_as_float(u[4 * j + 3]));
        }
      }
    }
    fence_proxy_async_global();   // the partner CTAs read these blocks with bulk copies
  }
  if (te == 0) TAIL_TS(7);
  cluster_sync_all();   // #1: layer-2 partials of every split visible (also orders sb2/sb3/sw4)
  if (te == 0) TAIL_TS(8);

  if (warp >= 2) {
    // ---------------- reduce owned Z2 columns -> relu(. + b2) -> bf16 A operand of layer 3 ----
    // the S-1 partner partial blocks (OW x 128 fp32 each, contiguous) come in by bulk copy
    const uint32_t pblk = (uint32_t)OW * BM * 4u;
    if (te == 0) {
      fence_proxy_async_global();
      mbar_arrive_expect_tx(pbar, (uint32_t)(splits - 1) * pblk);
      for (int s = 0, k = 0; s < splits; ++s) {
        if (s == split) continue;
        bulk_g2s(reinterpret_cast<uint8_t*>(sP2) + (k++) * pblk, wsb + (int64_t)(s * splits + split) * OW * BM, pblk,
                 pbar);
      }
    }
    mbar_wait(pbar, 0);
#pragma unroll 1
    for (int c = 0; c < OW; c += 16) {
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) f[j] = 0.0f;
      uint32_t v[16];
      tmem_ld_32x32b_x16(trow + (uint32_t)(own0 + c), v);
      tmem_ld_wait();
      for (int s = 0, k = 0; s < splits; ++s) {   // fixed split order (deterministic)
        if (s == split) {
#pragma unroll
          for (int j = 0; j < 16; ++j) f[j] += __uint_as_float(v[j]);
        } else {
          const float4* src = reinterpret_cast<const float4*>(sP2 + (int64_t)(k++) * OW * BM) + row_in_tile;
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
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a0 = fmaxf(f[2 * j] + sb2[c + 2 * j], 0.0f);
        const float a1 = fmaxf(f[2 * j + 1] + sb2[c + 2 * j + 1], 0.0f);
        __nv_bfloat162 b2v = __floats2bfloat162_rn(a0, a1);
        w[j] = *reinterpret_cast<uint32_t*>(&b2v);
      }
      // 128B-swizzled K-major tile: row r = row_in_tile, 16B chunk cb of K block kk
      uint4* rowp = reinterpret_cast<uint4*>(sA3 + (c / 64) * 16384 + row_in_tile * 128);
      const int cb = (c % 64) / 8;
      rowp[cb ^ (row_in_tile & 7)] = make_uint4(w[0], w[1], w[2], w[3]);
      rowp[(cb + 1) ^ (row_in_tile & 7)] = make_uint4(w[4], w[5], w[6], w[7]);
    }
    fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
    __syncwarp();
    if (lane == 0) mbar_arrive(a3bar);
    if (te == 0) TAIL_TS(9);
  } else if (warp == 1) {
    // ---------------- layer-3 partial MMA: Z3p = Z2[:, owned] . W3[:, owned]^T ----------------
    if (elect_one()) {
      mbar_wait(w3bar, 0);
      mbar_wait(a3bar, 0);
      tc_fence_after();
      for (int kk = 0; kk < OWK; ++kk) {
        const uint64_t ad = umma_desc_sw128(smem_u32(sA3 + kk * 16384));
        const uint64_t bd = umma_desc_sw128(smem_u32(sW3 + kk * 8192));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_ss<false>(tmem + 256, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), IDESC3, (kk | k) != 0 ? 1u : 0u);
      }
      umma_commit(l3bar);
    }
    __syncwarp();
  }
  if (warp >= 2) {
    // ---------------- publish this split's Z3 partial (128 x 64 fp32, lane-contiguous) ----------
    mbar_wait(l3bar, 0);
    tc_fence_after();
    if (te == 0) TAIL_TS(10);
    // layout [m][n][producer split][row group r][col4][rpr][4]: the block one consumer needs
    // from one producer is contiguous (bulk-copyable) and each warp store is 512 B contiguous
    const int rg = row_in_tile / rpr, rl = row_in_tile % rpr;
    float4* dst = reinterpret_cast<float4*>(p.ws3a + ((((int64_t)m_tile * p.n2_tiles + n_tile) * splits + split) * splits + rg) *
                                                         64 * rpr) + rl;
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
      uint32_t v[16], u[16];
      tmem_ld_32x32b_x16(trow + 256u + (uint32_t)c, v);
      tmem_ld_32x32b_x16(trow + 256u + (uint32_t)(c + 16), u);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dst[(c / 4 + j) * rpr] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                             __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        dst[(c / 4 + 4 + j) * rpr] = make_float4(__uint_as_float(u[4 * j]), __uint_as_float(u[4 * j + 1]),
                                                 __uint_as_float(u[4 * j + 2]), __uint_as_float(u[4 * j + 3]));
      }
    }
    fence_proxy_async_global();
  }
  if (te == 0) TAIL_TS(11);
  cluster_sync_all();   // #2: the S split partials of this (m, n) tile are visible
  if (te == 0) TAIL_TS(12);

  if (warp >= 2) {
    // ---- stage A: split r reduces rows [r*rpr, (r+1)*rpr) over the S partials (fixed order) ----
    const uint32_t zblk = 64u * (uint32_t)rpr * 4u;
    if (te == 0) {
      fence_proxy_async_global();
      mbar_arrive_expect_tx(zbar, (uint32_t)splits * zblk);
      for (int pr = 0; pr < splits; ++pr)
        bulk_g2s(reinterpret_cast<uint8_t*>(sZ3) + pr * zblk,
                 p.ws3a + ((((int64_t)m_tile * p.n2_tiles + n_tile) * splits + pr) * splits + split) * 64 * rpr, zblk,
                 zbar);
    }
    mbar_wait(zbar, 0);
    const int c0 = red_g * cpt;
    const int rl = red_row - split * rpr;
    float* zrow = p.ws3b + (((int64_t)m_tile * p.n2_tiles + n_tile) * BM + red_row) * 64;
#pragma unroll 1
    for (int cc = 0; cc < cpt; cc += 8) {
      float z[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) z[j] = 0.0f;
      for (int pr = 0; pr < splits; ++pr) {
        const float4* src = reinterpret_cast<const float4*>(sZ3 + (int64_t)pr * 64 * rpr) + rl;
        const float4 x0 = src[((c0 + cc) / 4) * rpr];
        const float4 x1 = src[((c0 + cc) / 4 + 1) * rpr];
        z[0] += x0.x; z[1] += x0.y; z[2] += x0.z; z[3] += x0.w;
        z[4] += x1.x; z[5] += x1.y; z[6] += x1.z; z[7] += x1.w;
      }
      float4* d4 = reinterpret_cast<float4*>(zrow + c0 + cc);
      d4[0] = make_float4(z[0], z[1], z[2], z[3]);
      d4[1] = make_float4(z[4], z[5], z[6], z[7]);
    }
    // ---- the last of the n2 tiles to finish a row group completes it (arrival counter) ----
    fence_acq_rel_gpu();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      int* ctr = p.cnt + m_tile * splits + split;
      const int last = atomicAdd(ctr, 1) == p.n2_tiles - 1;
      if (last) *ctr = 0;   // re-arm for the next launch (every arrival of this launch is in)
      *s_last = last;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) TAIL_TS(13);
    if (*s_last) {
      fence_acq_rel_gpu();
      // ---- Z3 = relu(sum over n-tiles + b3); y = w4 . Z3 + b4; N_hat = q(y) ----
      float dot = 0.0f;
#pragma unroll 1
      for (int cc = 0; cc < cpt; cc += 16) {   // all n-tile loads of a 16-column chunk in flight at once
        float4 x[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (nt < p.n2_tiles) {
            const float4* src = reinterpret_cast<const float4*>(
                p.ws3b + (((int64_t)m_tile * p.n2_tiles + nt) * BM + red_row) * 64 + c0 + cc);
#pragma unroll
            for (int j = 0; j < 4; ++j) x[nt][j] = __ldcg(src + j);
          }
        }
        float z[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) z[j] = 0.0f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {   // fixed n-tile order (deterministic)
          if (nt < p.n2_tiles) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              z[4 * j] += x[nt][j].x;
              z[4 * j + 1] += x[nt][j].y;
              z[4 * j + 2] += x[nt][j].z;
              z[4 * j + 3] += x[nt][j].w;
            }
          }
        }
        for (int nt = 2; nt < p.n2_tiles; ++nt) {   // m2 > 512 (rare): remaining n-tiles
          const float4* src = reinterpret_cast<const float4*>(
              p.ws3b + (((int64_t)m_tile * p.n2_tiles + nt) * BM + red_row) * 64 + c0 + cc);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 y4 = __ldcg(src + j);
            z[4 * j] += y4.x;
            z[4 * j + 1] += y4.y;
            z[4 * j + 2] += y4.z;
            z[4 * j + 3] += y4.w;
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) dot = fmaf(sw4[c0 + cc + j], fmaxf(z[j] + sb3[c0 + cc + j], 0.0f), dot);
      }
      __syncwarp();   // reconverge before the collectives (a CTA barrier does not)
      for (int off = 1; off < tpr; off <<= 1) dot += __shfl_xor_sync(0xFFFFFFFFu, dot, off);
      const bool owner = red_g == 0 && grow < Mrows;
      int32_t nh = 0;
      if (owner) {
        const float y = dot + (p.b4 ? __ldg(p.b4) : 0.0f);
        int32_t cap = p.max_ctx - (p.n_tok ? my_ntok : 0);
        cap = cap < 0 ? 0 : cap;
        nh = __float2int_rn(fminf(fmaxf(y, 0.0f), (float)cap));   // quantize_nhat (readings A8-A10)
        if (p.y_hat) p.y_hat[grow] = y;
        if (p.n_hat) p.n_hat[grow] = nh;
      }
      if (p.project) {
        // ---------------- fused projection: global histogram + last-finisher finalize ----------
        uint32_t errbits = 0;
        proj_accumulate(p.pa, owner, my_inst, my_ntok, nh, p.pa.ws_cnt, p.pa.ws_sum, errbits);
        if (errbits && p.pa.err) atomicOr(p.pa.err, (int)errbits);
        fence_acq_rel_gpu();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (te == 0) {
          const unsigned int finishers = (p.mn_swap ? gridDim.y : gridDim.x) * (unsigned)splits;   // per (m-tile, row group)
          *s_last = (atomicAdd(p.pa.ws_arrive, 1u) == finishers - 1) ? 1 : 0;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (*s_last) {
          if (te == 0) TAIL_TS(16);
          fence_acq_rel_gpu();
          const int nb = p.pa.n_inst * (p.pa.H + 2);
          const uint32_t* hc = p.pa.ws_cnt;
          const unsigned long long* hs = p.pa.ws_sum;
          if (nb * 12 <= 65536) {   // stage the histogram in shared memory (one round trip)
            unsigned long long* ss = reinterpret_cast<unsigned long long*>(sZ3);
            uint32_t* sc = reinterpret_cast<uint32_t*>(ss + nb);
            constexpr int kB = 8;   // all loads of a batch in flight before any store
            for (int base = 0; base < nb; base += kB * 128) {
              unsigned long long vs[kB];
              uint32_t vc[kB];
#pragma unroll
              for (int u = 0; u < kB; ++u) {
                const int k = base + u * 128 + te;
                if (k < nb) {
                  vs[u] = __ldcg(p.pa.ws_sum + k);
                  vc[u] = __ldcg(p.pa.ws_cnt + k);
                }
              }
#pragma unroll
              for (int u = 0; u < kB; ++u) {
                const int k = base + u * 128 + te;
                if (k < nb) {
                  ss[k] = vs[u];
                  sc[k] = vc[u];
                }
              }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            hc = sc;
            hs = ss;
          }
          if (te == 0) TAIL_TS(17);
          proj_finalize<false>(p.pa, hc, hs, sbeta, warp - 2, 4);
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (te == 0) TAIL_TS(18);
          for (int k = te; k < nb; k += 128) {
            p.pa.ws_cnt[k] = 0;
            p.pa.ws_sum[k] = 0;
          }
          if (te == 0) *p.pa.ws_arrive = 0;
          if (te == 0) TAIL_TS(19);
        }
      }
    }
  }
  if (te == 0) TAIL_TS(14);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (kPlan && p.plan && *s_last) {   // CTA-uniform: s_last was published by the barrier above
    // the stage ring is free (every TMA load and MMA of this CTA has completed); the plan's
    // shared state fits below OFF_W3 - 256 (checked on the host), warp_best / shv above it
    Cand* wb = reinterpret_cast<Cand*>(smem + S::OFF_W3 - 256);
    int* shv = reinterpret_cast<int*>(wb + 6);
    // diagnostics: the plan's stamps go to the two last timeline rows (never a CTA's)
    uint64_t* ptl = p.tl ? p.tl + (size_t)(gridDim.x * gridDim.y * gridDim.z > 0 ? kTailPlanTlRow : 0) * kTailTlStride
                         : nullptr;
    plan_cta_fast<true>(p.pl, smem, (int)threadIdx.x, (int)blockDim.x, wb, shv, ptl);
  }
}

}  // namespace star
