// lenpred_f32.cuh -- the fp32 predictor (Eq. 2) + quantizer + the fused
// projection for one decode batch of up to 128 requests in ONE launch:
// BASELINE.json configs[0] (2 instances x 64 requests, hidden 896, fp32).
//
// fp32 products by 3xTF32: a.b ~ a_hi.b_hi + a_hi.b_lo + a_lo.b_hi with hi = rna_tf32(x) and
// lo = x - hi (the dropped lo.lo term is ~2^-22 relative).  Shared-memory bandwidth, not the
// tensor pipe, bounds small-N 3xTF32 (each M=128 MMA re-reads its A tile; a first version that
// split both operands in shared memory spent ~1000 cycles per 32-wide K block), so:
//   * the weights are split once, at predictor creation, into hi / lo planes in global memory
//     (TMA loads both planes: no runtime conversion of B);
//   * the activations (h, Z1, Z2) land raw (1x bytes); each epilogue thread reads its row of the
//     landed block, splits it and writes the hi / lo halves into TENSOR memory (tcgen05.st), and
//     the MMAs take A from TMEM (tcgen05.mma ... [a_tmem]): A costs no shared-memory reads.
//
// Grid: 128 CTAs, one per SM, all resident at once (checked on the host), so the phases hand
// off through arrival counters in global memory instead of kernel boundaries:
//   L1  CTA c: Z1 columns [64 j1, +64) (j1 = c % 32) over the K quarter s1 = c / 32, tcgen05
//       kind::tf32 M=128 N=64 -> fp32 partial to global in a lane-contiguous layout
//       [s1][j1][16 column groups][128 rows][4]; once the 4 quarters of n-tile j1 are in
//       (p1_cnt[j1] = 4), CTA (j1, s1) adds columns [64 j1 + 16 s1, +16) in split order 0..3
//       (deterministic), + b1, ReLU -> Z1 (fp32, L2-resident) and bumps z1_cnt[j1 / 4].
//   L2  CTA c: Z2 columns [32 j2, +32) (j2 = c % 16) over Z1 columns [256 s2, +256) (s2 = c / 16:
//       L1 n-tiles 4 s2 .. 4 s2 + 3, z1_cnt[s2] = 16), N=32; the W2 blocks are in flight before
//       the wait.  Same partial / reduce: 8 splits, CTA (j2, s2) owns 4 columns -> Z2, z2_cnt[j2 / 2].
//   L3  CTAs 0..7: Z3 (64 columns) over Z2 columns [64 s3, +64) (z2_cnt[s3] = 16), N=64 ->
//       partial; CTA s3 adds columns [8 s3, +8) in split order, + b3, ReLU, the w4 dot over its
//       8 columns (column order) -> y partial; the last of the eight adds the y partials in order
//       0..7, + b4, the quantizer (readings A8-A10), the rows' projection histogram in shared
//       memory, the finalize (L/W/peak/growth/count), and re-arms every counter.
// Roles (320 threads): warp 0 TMA producer, warp 1 MMA issuer (one elected lane), warps 2-9 the
// operand split (warps 2-5 columns 0-15 of each block, 6-9 columns 16-31; TMEM lane quarter =
// warp % 4), warps 2-5 the epilogues.
#pragma once
#include "lenpred_kernels.cuh"
#include "project_core.cuh"

namespace star {

struct F32Args {
  int M;                 // rows (1..128)
  int kb1;               // layer-1 K blocks of 32 fp32 (d / 32), a multiple of 4
  const float* b1;       // [2048] or nullptr
  const float* b2;       // [512] or nullptr
  const float* b3;       // [64] or nullptr
  const float* w4;       // [64]
  const float* b4;       // [1] or nullptr
  const int32_t* n_tok;  // [M] or nullptr
  int32_t max_ctx;
  float* y_hat;          // [M] or nullptr
  int32_t* n_hat;        // [M] or nullptr
  float* Z1;             // [>= M][2048]
  float* Z2;             // [>= M][512]
  float* P1;             // [4][32][16][128][4] layer-1 partials
  float* P2;             // [8][16][8][128][4]
  float* P3;             // [8][16][128][4]
  float* yp;             // [8][128]
  int* cnt;              // F32Cnt counters (all zero between launches)
  int project;           // fused projection (histogram in shared memory)
  ProjArgs pa;
  uint64_t* tl;          // diagnostics: [128][32] %globaltimer phase stamps, or nullptr
};

// scratch floats: P1 + P2 + P3 + y partials
constexpr int F32_WS_FLOATS = 4 * 32 * 16 * 512 + 8 * 16 * 8 * 512 + 8 * 16 * 512 + 8 * 128;

struct F32Cnt {
  static constexpr int P1 = 0, Z1 = 32, P2 = 40, Z2 = 56, P3 = 64, Y = 65, N = 72;
};

struct F32Smem {
  static constexpr int STAGES = 5;
  // stage s at STAGE * s: A raw (128 rows x 32 fp32 = 16 KB, SW128) | B hi (<= 64 rows, 8 KB) | B lo
  static constexpr uint32_t STAGE = 32u * 1024u;
  static constexpr uint32_t A_RAW = 0, B_HI = 16384u, B_LO = 24576u;
  static constexpr uint32_t BAR = STAGES * STAGE;
  static constexpr uint32_t BYTES = 1024u + BAR + 256u + 2048u;
  static constexpr uint32_t HIST_MAX = BAR - 4096u;   // finalize: histogram + beta (ring idle)
  static constexpr uint32_t CBETA = BAR + 256u;        // beta [<= 512], prefetched by the layer-3 CTAs
  static constexpr int CBETA_MAX = 512;
};
// TMEM columns (512 allocated): accumulators L1 [0, 64), L2 [64, 96), L3 [128, 192); the A operand
// of ring stage s at [192 + 64 s, +32) (hi) and [+32, +64) (lo).
struct F32Tmem {
  static constexpr uint32_t ACC1 = 0, ACC2 = 64, ACC3 = 128, A0 = 192;
};
static_assert(F32Tmem::A0 + 64 * F32Smem::STAGES <= 512, "fp32 predictor TMEM");
static_assert(F32Smem::BYTES <= 227u * 1024u, "fp32 predictor smem");

#define F32_TS(k)                                                  \
  do {                                                             \
    if (p.tl) p.tl[(int64_t)blockIdx.x * 32 + (k)] = globaltimer_ns(); \
  } while (0)

__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_release_add_f(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Weight planes for the kernel below, once at predictor creation: x [n] (row-major [rows][K])
// -> out [2][n]: hi = rna_tf32(x), lo = x - hi.
__global__ void tf32_planes_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const float h = tf32_rna(v);
    out[i] = h;
    out[n + i] = v - h;
  }
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] . B[smem]^T, kind::tf32 (A: M rows in TMEM lanes, one element per column).
__device__ __forceinline__ void umma_ts_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// One phase's operand split, 8 warps (row = TMEM lane, `half` = which 16 of the block's 32
// columns): for every landed stage, read this row's 16 fp32 of the A block (SW128: 16-byte chunk
// c of row r sits at c ^ (r & 7)), split into hi = rna_tf32(x) and lo = x - hi, write both into
// the stage's TMEM A slot, signal the MMA warp.  `it0` = ring iterations before this phase
// (stage = it % NS), nkb K blocks of 32.
__device__ __forceinline__ void f32_convert(const uint8_t* smem, uint64_t* full, uint64_t* conv, int it0, int nkb,
                                            int row, int half, uint32_t trow, int lane, long long* dbg) {
  using S = F32Smem;
  for (int i = 0; i < nkb; ++i) {
    const int it = it0 + i, s = it % S::STAGES;
    const long long t0 = clock64();
    mbar_wait(&full[s], (uint32_t)(it / S::STAGES) & 1u);
    const long long t1 = clock64();
    const uint8_t* rp = smem + S::STAGE * s + S::A_RAW + row * 128;
    float4 x[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = *reinterpret_cast<const float4*>(rp + (((4 * half + c) ^ (row & 7)) << 4));
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float v[4] = {x[c].x, x[c].y, x[c].z, x[c].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float h = tf32_rna(v[e]);
        hi[4 * c + e] = __float_as_uint(h);
        lo[4 * c + e] = __float_as_uint(v[e] - h);
      }
    }
    const uint32_t ta = trow + F32Tmem::A0 + 64u * (uint32_t)s + 16u * (uint32_t)half;
    tmem_st_32x32b_x16(ta, hi);
    tmem_st_32x32b_x16(ta + 32u, lo);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&conv[s]);
    if (dbg) {
      dbg[0] += t1 - t0;
      dbg[1] += clock64() - t1;
    }
  }
}

__device__ __forceinline__ void f32_mma(uint8_t* smem, uint64_t* conv, uint64_t* empty, uint64_t* acc, int it0, int nkb,
                                        uint32_t tmem, uint32_t acc_col, uint32_t idesc, long long* dbg) {
  using S = F32Smem;
  for (int i = 0; i < nkb; ++i) {
    const int it = it0 + i, s = it % S::STAGES;
    const long long t0 = clock64();
    mbar_wait(&conv[s], (uint32_t)(it / S::STAGES) & 1u);
    if (dbg) dbg[0] += clock64() - t0;
    tc_fence_after();
    const uint32_t base = smem_u32(smem + S::STAGE * s);
    const uint64_t bhi = umma_desc_sw128(base + S::B_HI), blo = umma_desc_sw128(base + S::B_LO);
    const uint32_t ahi = tmem + F32Tmem::A0 + 64u * (uint32_t)s, alo = ahi + 32u, d = tmem + acc_col;
#pragma unroll
    for (int k = 0; k < 4; ++k) {   // 4 x K=8 per 32-wide block
      const uint64_t o = (uint64_t)(k * 2);
      umma_ts_tf32(d, ahi + 8u * k, bhi + o, idesc, (i | k) != 0 ? 1u : 0u);
      umma_ts_tf32(d, ahi + 8u * k, blo + o, idesc, 1u);
      umma_ts_tf32(d, alo + 8u * k, bhi + o, idesc, 1u);
    }
    umma_commit(&empty[s]);
  }
  umma_commit(acc);
}

// TMEM columns [c0, c0 + 4*ng) of this thread's row -> ng lane-contiguous float4 groups at
// dst + g * 128 rows (group stride 512 floats).
__device__ __forceinline__ void f32_store_partial(uint32_t trow, int c0, int ng, float* dst, int row) {
#pragma unroll 1
  for (int c = 0; c < ng * 4; c += 16) {
    uint32_t v[16];
    tmem_ld_32x32b_x16(trow + (uint32_t)(c0 + c), v);
    tmem_ld_wait();
    float4* d = reinterpret_cast<float4*>(dst) + row;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      __stcg(d + (c / 4 + j) * 128, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
  }
}

__global__ void __launch_bounds__(320, 1)
    lenpred_f32_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW1,
                       const __grid_constant__ CUtensorMap tmZ1, const __grid_constant__ CUtensorMap tmW2,
                       const __grid_constant__ CUtensorMap tmZ2, const __grid_constant__ CUtensorMap tmW3,
                       const F32Args p) {
  using S = F32Smem;
  using C = F32Cnt;
  constexpr int NS = S::STAGES;
  constexpr uint32_t ID1 = umma_idesc(true, 128, 64), ID2 = umma_idesc(true, 128, 32), ID3 = umma_idesc(true, 128, 64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR);
  uint64_t* conv = full + NS;
  uint64_t* empty = conv + NS;
  uint64_t* acc = empty + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int j1 = c & 31, s1 = c >> 5;   // layer 1: n-tile (64 columns), K quarter
  const int j2 = c & 15, s2 = c >> 4;   // layer 2: n-tile (32 columns), K eighth
  const bool l3 = c < 8;                // layer 3: K eighth s3 = c
  const int te = threadIdx.x - 64;
  const int M = p.M;
  if (threadIdx.x == 0) F32_TS(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH);
    tma_prefetch_desc(&tmW1);
    tma_prefetch_desc(&tmZ1);
    tma_prefetch_desc(&tmW2);
    if (l3) {
      tma_prefetch_desc(&tmZ2);
      tma_prefetch_desc(&tmW3);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 8);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();

  const int kq = p.kb1 / 4;                   // layer-1 K blocks of this quarter
  const int n1_it = kq, n2_it = 8, n3_it = 2;  // ring iterations per phase
  const int q = warp & 3, row = q * 32 + lane, half = warp >= 6 ? 1 : 0;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  int* cnt = p.cnt;
  long long dc[6] = {0, 0, 0, 0, 0, 0};   // diagnostics, converter te = 0: cycles waiting for / splitting stages

  if (warp == 0) {
    if (elect_one()) {   // ---------------- TMA producer
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      // B = the weight planes: hi rows [0, m), lo rows [m, 2m) of the plane map
      auto load_b = [&](const CUtensorMap* tm, int s, int k, int r, int m_rows, uint32_t bbytes) {
        tma_load_2d(smem + S::STAGE * s + S::B_HI, tm, &full[s], k, r, pol_b);
        tma_load_2d(smem + S::STAGE * s + S::B_LO, tm, &full[s], k, m_rows + r, pol_b);
        (void)bbytes;
      };
      const int pre = kq < NS ? kq : NS;
      // layer 1: the W1 blocks of the first stages before griddepcontrol.wait (independent of
      // the predecessor), then the hidden states
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], 16384u + 2u * 8192u);
        load_b(&tmW1, i, (s1 * kq + i) * 32, j1 * 64, 2048, 8192u);
      }
      for (int i = 0; i < 8; ++i) {   // into L2 early
        tma_prefetch_2d(&tmW2, (s2 * 8 + i) * 32, j2 * 32);
        tma_prefetch_2d(&tmW2, (s2 * 8 + i) * 32, 512 + j2 * 32);
      }
      if (l3)
        for (int i = 0; i < 2; ++i) {
          tma_prefetch_2d(&tmW3, (c * 2 + i) * 32, 0);
          tma_prefetch_2d(&tmW3, (c * 2 + i) * 32, 64);
        }
      pdl_wait();
      F32_TS(1);
      for (int i = 0; i < kq; ++i) {
        const int it = i, s = it % NS;
        if (i >= pre) {
          mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 2u * 8192u);
          load_b(&tmW1, s, (s1 * kq + i) * 32, j1 * 64, 2048, 8192u);
        }
        tma_load_2d(smem + S::STAGE * s + S::A_RAW, &tmH, &full[s], (s1 * kq + i) * 32, 0, pol_a);
      }
      // layer 2: W2 blocks first, the Z1 blocks once their 4 n-tiles are reduced
      const int it2 = n1_it;
      const int pre2 = NS < n2_it ? NS : n2_it;
      for (int i = 0; i < pre2; ++i) {
        const int it = it2 + i, s = it % NS;
        mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], 16384u + 2u * 4096u);
        load_b(&tmW2, s, (s2 * 8 + i) * 32, j2 * 32, 512, 4096u);
      }
      spin_wait_geq(cnt + C::Z1 + s2, 16);
      fence_proxy_async_global();
      F32_TS(5);
      for (int i = 0; i < n2_it; ++i) {
        const int it = it2 + i, s = it % NS;
        if (i >= pre2) {
          mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 2u * 4096u);
          load_b(&tmW2, s, (s2 * 8 + i) * 32, j2 * 32, 512, 4096u);
        }
        tma_load_2d(smem + S::STAGE * s + S::A_RAW, &tmZ1, &full[s], (s2 * 8 + i) * 32, 0, pol_a);
      }
      if (l3) {   // layer 3: W3 blocks, then the Z2 blocks after their 2 n-tiles
        const int it3 = n1_it + n2_it;
        for (int i = 0; i < n3_it; ++i) {
          const int it = it3 + i, s = it % NS;
          mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 2u * 8192u);
          load_b(&tmW3, s, (c * 2 + i) * 32, 0, 64, 8192u);
        }
        spin_wait_geq(cnt + C::Z2 + c, 16);
        fence_proxy_async_global();
        for (int i = 0; i < n3_it; ++i) {
          const int it = it3 + i, s = it % NS;
          tma_load_2d(smem + S::STAGE * s + S::A_RAW, &tmZ2, &full[s], (c * 2 + i) * 32, 0, pol_a);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {   // ---------------- MMA issuer
      long long dm[3] = {0, 0, 0};
      const long long t0 = clock64();
      f32_mma(smem, conv, empty, acc, 0, n1_it, tmem, F32Tmem::ACC1, ID1, dm);
      const long long t1 = clock64();
      f32_mma(smem, conv, empty, acc, n1_it, n2_it, tmem, F32Tmem::ACC2, ID2, dm + 1);
      if (l3) f32_mma(smem, conv, empty, acc, n1_it + n2_it, n3_it, tmem, F32Tmem::ACC3, ID3, dm + 2);
      if (p.tl) {   // diagnostics: MMA-thread cycles waiting for converted stages (L1, L2, L3), L1 span
        p.tl[(int64_t)blockIdx.x * 32 + 20] = (uint64_t)dm[0];
        p.tl[(int64_t)blockIdx.x * 32 + 21] = (uint64_t)dm[1];
        p.tl[(int64_t)blockIdx.x * 32 + 22] = (uint64_t)dm[2];
        p.tl[(int64_t)blockIdx.x * 32 + 23] = (uint64_t)(t1 - t0);
      }
    }
    __syncwarp();
  } else if (warp >= 6) {
    // ---------------- operand split, columns 16..31 of every block (no epilogue work)
    f32_convert(smem, full, conv, 0, n1_it, row, 1, trow, lane, nullptr);
    f32_convert(smem, full, conv, n1_it, n2_it, row, 1, trow, lane, nullptr);
    if (l3) f32_convert(smem, full, conv, n1_it + n2_it, n3_it, row, 1, trow, lane, nullptr);
  } else {
    // ---------------- operand split (columns 0..15) + epilogues (128 threads, row = TMEM lane)
    pdl_wait();
    // ===== layer 1
    f32_convert(smem, full, conv, 0, n1_it, row, 0, trow, lane, te == 0 ? dc : nullptr);
    mbar_wait(acc, 0);
    tc_fence_after();
    if (te == 0) F32_TS(2);
    f32_store_partial(trow, F32Tmem::ACC1, 16, p.P1 + (size_t)(s1 * 32 + j1) * 16 * 512, row);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      red_release_add_f(cnt + C::P1 + j1, 1);
      spin_wait_geq(cnt + C::P1 + j1, 4);
      F32_TS(3);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    {
      float4 x[4][4];
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int g = 0; g < 4; ++g)
          x[s][g] = __ldcg(reinterpret_cast<const float4*>(p.P1 + ((size_t)(s * 32 + j1) * 16 + s1 * 4 + g) * 512) + row);
      if (row < M) {
        float4* z = reinterpret_cast<float4*>(p.Z1 + (size_t)row * 2048 + j1 * 64 + s1 * 16);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int col = j1 * 64 + s1 * 16 + g * 4;
          float4 f = x[0][g];
#pragma unroll
          for (int s = 1; s < 4; ++s) {
            f.x += x[s][g].x;
            f.y += x[s][g].y;
            f.z += x[s][g].z;
            f.w += x[s][g].w;
          }
          if (p.b1) {
            f.x += __ldg(p.b1 + col);
            f.y += __ldg(p.b1 + col + 1);
            f.z += __ldg(p.b1 + col + 2);
            f.w += __ldg(p.b1 + col + 3);
          }
          z[g] = make_float4(fmaxf(f.x, 0.f), fmaxf(f.y, 0.f), fmaxf(f.z, 0.f), fmaxf(f.w, 0.f));
        }
      }
    }
    fence_proxy_async_global();   // Z1 (generic stores) -> the layer-2 TMA loads (async proxy)
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      red_release_add_f(cnt + C::Z1 + (j1 >> 2), 1);
      F32_TS(4);
    }
    // ===== layer 2
    f32_convert(smem, full, conv, n1_it, n2_it, row, 0, trow, lane, te == 0 ? dc + 2 : nullptr);
    mbar_wait(acc, 1);
    tc_fence_after();
    if (te == 0) F32_TS(6);
    f32_store_partial(trow, F32Tmem::ACC2, 8, p.P2 + (size_t)(s2 * 16 + j2) * 8 * 512, row);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      red_release_add_f(cnt + C::P2 + j2, 1);
      spin_wait_geq(cnt + C::P2 + j2, 8);
      F32_TS(7);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    {
      float4 x[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        x[s] = __ldcg(reinterpret_cast<const float4*>(p.P2 + ((size_t)(s * 16 + j2) * 8 + s2) * 512) + row);
      if (row < M) {
        const int col = j2 * 32 + s2 * 4;
        float4 f = x[0];
#pragma unroll
        for (int s = 1; s < 8; ++s) {
          f.x += x[s].x;
          f.y += x[s].y;
          f.z += x[s].z;
          f.w += x[s].w;
        }
        if (p.b2) {
          f.x += __ldg(p.b2 + col);
          f.y += __ldg(p.b2 + col + 1);
          f.z += __ldg(p.b2 + col + 2);
          f.w += __ldg(p.b2 + col + 3);
        }
        *reinterpret_cast<float4*>(p.Z2 + (size_t)row * 512 + col) =
            make_float4(fmaxf(f.x, 0.f), fmaxf(f.y, 0.f), fmaxf(f.z, 0.f), fmaxf(f.w, 0.f));
      }
    }
    fence_proxy_async_global();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      red_release_add_f(cnt + C::Z2 + (j2 >> 1), 1);
      F32_TS(8);
    }
    // ===== layer 3 + head (CTAs 0..7)
    if (l3) {
      const bool owner = row < M;
      int32_t ntok = 0, inst = 0;   // fetched while layer 3 runs
      if (owner) {
        if (p.n_tok) ntok = p.n_tok[row];
        if (p.project) inst = p.pa.inst[row];
      }
      if (p.project && p.pa.H + 1 <= S::CBETA_MAX)   // the finalize's beta, while layer 3 runs
        for (int t = te; t <= p.pa.H; t += 128) reinterpret_cast<uint32_t*>(smem + S::CBETA)[t] = p.pa.beta_q[t];
      float w4s[8], b3s[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        w4s[j] = __ldg(p.w4 + c * 8 + j);
        b3s[j] = p.b3 ? __ldg(p.b3 + c * 8 + j) : 0.0f;
      }
      f32_convert(smem, full, conv, n1_it + n2_it, n3_it, row, 0, trow, lane, te == 0 ? dc + 4 : nullptr);
      mbar_wait(acc, 0);
      tc_fence_after();
      if (te == 0) F32_TS(9);
      f32_store_partial(trow, F32Tmem::ACC3, 16, p.P3 + (size_t)c * 16 * 512, row);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        red_release_add_f(cnt + C::P3, 1);
        spin_wait_geq(cnt + C::P3, 8);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      float y = 0.0f;
      {
        float4 x[8][2];
#pragma unroll
        for (int s = 0; s < 8; ++s)
#pragma unroll
          for (int g = 0; g < 2; ++g)
            x[s][g] = __ldcg(reinterpret_cast<const float4*>(p.P3 + ((size_t)s * 16 + c * 2 + g) * 512) + row);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float4 f = x[0][g];
#pragma unroll
          for (int s = 1; s < 8; ++s) {
            f.x += x[s][g].x;
            f.y += x[s][g].y;
            f.z += x[s][g].z;
            f.w += x[s][g].w;
          }
          y = fmaf(w4s[4 * g], fmaxf(f.x + b3s[4 * g], 0.0f), y);
          y = fmaf(w4s[4 * g + 1], fmaxf(f.y + b3s[4 * g + 1], 0.0f), y);
          y = fmaf(w4s[4 * g + 2], fmaxf(f.z + b3s[4 * g + 2], 0.0f), y);
          y = fmaf(w4s[4 * g + 3], fmaxf(f.w + b3s[4 * g + 3], 0.0f), y);
        }
      }
      __stcg(p.yp + c * 128 + row, y);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        F32_TS(10);
        *s_last = atom_add_acq_rel(cnt + C::Y, 1) == 7 ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*s_last) {
        fence_acq_rel_gpu();
        float yy = __ldcg(p.yp + row);
#pragma unroll
        for (int s = 1; s < 8; ++s) yy += __ldcg(p.yp + s * 128 + row);
        yy += p.b4 ? __ldg(p.b4) : 0.0f;
        int32_t nh = 0;
        if (owner) {
          int32_t cap = p.max_ctx - ntok;
          cap = cap < 0 ? 0 : cap;
          nh = __float2int_rn(fminf(fmaxf(yy, 0.0f), (float)cap));   // quantize_nhat (readings A8-A10)
          if (p.y_hat) p.y_hat[row] = yy;
          if (p.n_hat) p.n_hat[row] = nh;
        }
        if (p.project) {
          // the ring is idle: histogram [nb] u64 sums, [nb] u32 counts, beta [H + 1]
          const int nb = p.pa.n_inst * (p.pa.H + 2);
          unsigned long long* ss = reinterpret_cast<unsigned long long*>(smem);
          uint32_t* sc = reinterpret_cast<uint32_t*>(ss + nb);
          uint32_t* sbeta = reinterpret_cast<uint32_t*>(smem + S::CBETA);   // prefetched
          for (int k = te; k < nb; k += 128) {
            ss[k] = 0ull;
            sc[k] = 0u;
          }
          if (p.pa.H + 1 > S::CBETA_MAX) {
            sbeta = sc + nb;
            for (int t = te; t <= p.pa.H; t += 128) sbeta[t] = p.pa.beta_q[t];
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          uint32_t errbits = 0;
          proj_accumulate<true>(p.pa, owner, inst, ntok, nh, sc, ss, errbits);
          if (errbits && p.pa.err) atomicOr(p.pa.err, (int)errbits);
          asm volatile("bar.sync 1, 128;" ::: "memory");
          proj_finalize<false>(p.pa, sc, ss, sbeta, warp - 2, 4);
        }
        // every counter of this launch has been consumed (each CTA's last wait precedes the
        // arrivals that led here): re-arm them for the next launch
        if (te < C::N) cnt[te] = 0;
        if (te == 0) F32_TS(11);
      }
    }
  }
  if (p.tl && threadIdx.x == 64)
    for (int k = 0; k < 6; ++k) p.tl[(int64_t)blockIdx.x * 32 + 24 + k] = (uint64_t)dc[k];
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace star
