// lenpred_small.cuh -- the whole predictor (Eq. 2) + quantizer + the fused
// projection for one rank's batch of up to 512 requests in ONE persistent launch: the per-rank
// shape of the north-star job (one decode instance of 512 running requests per B200).
//
//   Z1 = phi(W1 h + b1) -> Z2 = phi(W2 Z1 + b2) -> Z3 = phi(W3 Z2 + b3) -> y = w4 . Z3 + b4
//   -> N_hat = q(y) [-> keyed projection histogram -> per-instance loads]
//
// Grid (2, 16, m_tiles) in clusters of 2 CTAs (a K-split pair) along x: cluster (m, n), CTA rank
// r.  Every CTA is resident at once (one per SM, <= 128 CTAs, checked on the host), so the
// phases hand off through per-m-tile counters in global memory instead of kernel boundaries:
//   L1  tile 128 x 128 of Z1 (rows of m-tile m, columns of n-tile n) over the K half r:
//       TMA -> 6-stage SMEM ring -> tcgen05 (M=128, N=128) -> TMEM.  Split-K reduction in
//       distributed shared memory: each CTA stages the 64 partial columns its partner owns in its
//       (now free) ring, one cluster barrier, one 32 KB bulk copy shared::cta -> shared::cluster
//       into the partner's receive slot (completion on its mbarrier); each CTA adds its own 64
//       columns in fixed split order (deterministic), + b1, ReLU, bf16 -> Z1 (L2-resident
//       global), then bumps z1_cnt[m][n / 8] (release).
//       (Clusters of 2 and not 4: DSMEM moves only ~14-17 B/clk per SM on B200
//       (tools/dsmem_bench.cu), so the split-K exchange -- (S-1)/S of the 128 x N partial -- must
//       stay small: 32 KB at S = 2 against 96 KB at S = 4, for one third more operand ingest.)
//   L2  tile 128 x 32 of Z2 (n2 = n) over the K half r (= Z1 columns of n-tiles 8r..8r+7): the W2
//       blocks stream in first (independent), the Z1 blocks after z1_cnt[m][r] = 16 (acquire);
//       tcgen05 N=32; the same DSMEM reduction (8 KB, owned 16 columns) -> + b2, ReLU, bf16 ->
//       Z2, bump z2_cnt[m].
//   L3  (CTA 0 of cluster (m, 0): one per m-tile) Z3 = W3 Z2 over the full K = 512 after
//       z2_cnt[m] = 32 (no split: no exchange, no cluster barrier), + b3, ReLU, the w4 dot in
//       column order, + b4, the quantizer (readings A8-A10) and the rows' projection histogram;
//       the last m-tile to finish finalises L/W/peak/growth/count and re-arms every counter.
// Roles (192 threads, as in umma_gemm_kernel): warp 0 TMA producer, warp 1 MMA issuer (one
// elected lane), warps 2-5 epilogue (TMEM lane quarter = warp % 4).
#pragma once
#include "lenpred_kernels.cuh"
#include "project_core.cuh"

namespace star {

struct SmallArgs {
  int M;                 // rows (<= 512 per chunk)
  int kb1;               // layer-1 K blocks (d / 64), even
  int n1;                // layer-1 tile width: 128 (3-4 m-tiles), 64 (2), 32 (1): always 2048 / n1 column
                         // tiles x m-tiles x 2 K halves = 128 CTAs
  const float* b1;       // [2048] or nullptr
  const float* b2;       // [512] or nullptr
  const float* b3;       // [64] or nullptr
  const float* w4;       // [64]
  const float* b4;       // [1] or nullptr
  const int32_t* n_tok;  // [M] or nullptr
  int32_t max_ctx;
  float* y_hat;          // [M] or nullptr
  int32_t* n_hat;        // [M] or nullptr
  __nv_bfloat16* Z1;     // [>= M][2048]
  __nv_bfloat16* Z2;     // [>= M][512]
  int* cnt;              // per 512-row chunk c: [c*16 + 0..7] z1_cnt [4][2], [c*16 + 8..11] z2_cnt [4];
                         // [SmallSmem::DONE] layer-3 completions (all zero between launches)
  int project;
  ProjArgs pa;
  uint64_t* tl;          // diagnostics: [ctas][32] %globaltimer phase stamps (slot 15 = SM id), or nullptr
  const int32_t* M_dev;  // refresh mode: the row count comes from the device, or nullptr (then M)
  // refresh mode (cadence k): row p of the batch is request slot r_idx[p]; its N_hat, g_last = gen
  // and N_hat_last are scattered there (the aged slots were handled by the select kernel)
  const int32_t* r_idx;
  const int32_t* r_gen;
  int32_t* r_glast;
  int32_t* r_nhat_last;
  int32_t* r_nhat;
};

struct SmallSmem {
  static constexpr int STAGES = 6;
  // stage s: A (128 rows x 64 bf16, 16 KB) @ 16K*s; B @ B0 + 16K*s (L1: 128 rows = 16 KB,
  // L2: 32 rows = 4 KB, L3: 64 rows = 8 KB)
  static constexpr uint32_t B0 = 96u * 1024u;
  static constexpr uint32_t L1_SEND = 0;                  // 32 KB (after the L1 mainloop)
  static constexpr uint32_t L1_RECV = 32u * 1024u;        // 32 KB (after the cluster barrier)
  static constexpr uint32_t SEND23 = 0;                   // L2 / L3 send (A slots are idle then)
  static constexpr uint32_t R2 = 192u * 1024u;            // layer-2 receive 8 KB (dedicated)
  static constexpr uint32_t BAR = 200u * 1024u;
  // layer-3 CTAs: w4 [64], b3 [64], beta [<= 512] prefetched while layer 1 runs
  static constexpr uint32_t CW4 = BAR + 256u, CB3 = CW4 + 256u, CBETA = CB3 + 256u;
  static constexpr int CBETA_MAX = 512;
  static constexpr uint32_t BYTES = 1024u + CBETA + 4u * CBETA_MAX;
  static constexpr uint32_t HIST = 0;                     // finalize: histogram staging (ring idle), <= 96 KB
  static constexpr int DONE = 16 * 256;                   // index of the completion counter in cnt (<= 256 chunks)
};
static_assert(SmallSmem::BYTES <= 227u * 1024u, "small predictor smem");

#define SMALL_TS(k)                                                                                     \
  do {                                                                                                  \
    if (p.tl) p.tl[(((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 32 + (k)] = \
        globaltimer_ns();                                                                               \
  } while (0)

__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, const void* src_cta, uint32_t bytes,
                                               uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(smem_u32(src_cta)), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stages this warp's 32 rows x `cols` fp32 TMEM columns [c0, c0 + cols) into a lane-contiguous
// block [cols/4][128 rows][4] (conflict-free 16-byte stores).
__device__ __forceinline__ void tmem_to_block(uint32_t trow, int c0, int cols, float* blk, int row) {
#pragma unroll 1
  for (int c = 0; c < cols; c += 16) {
    uint32_t v[16];
    tmem_ld_32x32b_x16(trow + (uint32_t)(c0 + c), v);
    tmem_ld_wait();
    float4* d = reinterpret_cast<float4*>(blk) + row;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      d[(c / 4 + j) * 128] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                         __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
  }
}

// Owned columns [c0, c0 + 16) of this row: the two split partials (own from TMEM, the partner's
// from the received block at column-group offset cl/4) summed in split order 0, 1 (deterministic).
__device__ __forceinline__ void reduce16(uint32_t trow, int c0, const float* recv, int cl, int rank, int row,
                                         float (&f)[16]) {
  uint32_t v[16];
  tmem_ld_32x32b_x16(trow + (uint32_t)c0, v);
  const float4* src = reinterpret_cast<const float4*>(recv) + row;
  float4 x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = src[(cl / 4 + j) * 128];
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float o[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float mine = __uint_as_float(v[4 * j + e]);
      f[4 * j + e] = rank == 0 ? mine + o[e] : o[e] + mine;
    }
  }
}

__device__ __forceinline__ void relu_bf16_16(const float (&f)[16], const float* bias, int col, uint32_t (&w)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float a0 = fmaxf(f[2 * j] + (bias ? __ldg(bias + col + 2 * j) : 0.0f), 0.0f);
    const float a1 = fmaxf(f[2 * j + 1] + (bias ? __ldg(bias + col + 2 * j + 1) : 0.0f), 0.0f);
    __nv_bfloat162 b = __floats2bfloat162_rn(a0, a1);
    w[j] = *reinterpret_cast<uint32_t*>(&b);
  }
}

// The projection's last step (by the last m-tile to finish, or by CTA 0 when a refresh step has no
// due row): L/W/peak/growth/count from the global histogram (one warp per instance), then the
// histogram is re-zeroed.  The histogram comes into shared memory with L2 loads (other SMs'
// atomics) when it fits the ring's A slots.  Epilogue warps 2..5 (te = thread - 64).
__device__ __forceinline__ void small_finalize(const SmallArgs& p, uint8_t* smem, int te, int warp, bool beta_ready) {
  using S = SmallSmem;
  const int nb = p.pa.n_inst * (p.pa.H + 2);
  uint32_t* sbeta = reinterpret_cast<uint32_t*>(smem + S::CBETA);   // prefetched (H + 1 <= CBETA_MAX)
  if (!beta_ready || p.pa.H + 1 > S::CBETA_MAX) {
    sbeta = reinterpret_cast<uint32_t*>(smem + S::R2);   // consumed by now
    for (int t = te; t <= p.pa.H; t += 128) sbeta[t] = p.pa.beta_q[t];
  }
  const uint32_t* hc = p.pa.ws_cnt;
  const unsigned long long* hs = p.pa.ws_sum;
  if ((uint32_t)nb * 12u <= 96u * 1024u) {
    unsigned long long* ss = reinterpret_cast<unsigned long long*>(smem + S::HIST);
    uint32_t* sc = reinterpret_cast<uint32_t*>(ss + nb);
    for (int k = te; k < nb; k += 128) {
      ss[k] = __ldcg(p.pa.ws_sum + k);
      sc[k] = __ldcg(p.pa.ws_cnt + k);
    }
    hc = sc;
    hs = ss;
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  proj_finalize<false>(p.pa, hc, hs, sbeta, warp - 2, 4);
  asm volatile("bar.sync 1, 128;" ::: "memory");
  for (int k = te; k < nb; k += 128) {
    p.pa.ws_cnt[k] = 0;
    p.pa.ws_sum[k] = 0;
  }
  if (te == 0) *p.pa.ws_arrive = 0;
}

__global__ void __launch_bounds__(192, 1)
    lenpred_small_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW1,
                         const __grid_constant__ CUtensorMap tmZ1, const __grid_constant__ CUtensorMap tmW2,
                         const __grid_constant__ CUtensorMap tmZ2, const __grid_constant__ CUtensorMap tmW3,
                         const SmallArgs p) {
  using S = SmallSmem;
  constexpr int NS = S::STAGES;
  constexpr uint32_t ID2 = umma_idesc(false, 128, 32);
  constexpr uint32_t ID3 = umma_idesc(false, 128, 64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR);
  uint64_t* empty = full + NS;
  uint64_t* acc1 = empty + NS;
  uint64_t* acc2 = acc1 + 1;
  uint64_t* acc3 = acc2 + 1;
  uint64_t* r1bar = acc3 + 1;
  uint64_t* r2bar = r1bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r2bar + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = blockIdx.x, n = blockIdx.y, m = blockIdx.z;
  const int partner = rank ^ 1;
  const int te = threadIdx.x - 64;     // epilogue thread 0..127
  int M = p.M;
  const bool dev_rows = p.M_dev != nullptr;   // refresh mode: the row count comes from the predecessor
  if (!dev_rows && m * 128 >= M) return;      // (the host sizes the grid to M)
  const bool l2 = n < 16;                // layer 2 has 16 column tiles (32 wide) per m-tile
  const bool l3 = n == 0 && rank == 0;   // this CTA also runs layer 3 + head for its m-tile
  if (threadIdx.x == 0) {
    SMALL_TS(0);
    if (p.tl) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.tl[(((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 32 + 15] = smid;
    }
  }
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
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc1, 1);
    mbar_init(acc2, 1);
    mbar_init(acc3, 1);
    mbar_init(r1bar, 1);
    mbar_init(r2bar, 1);
    // the partner's bulk copies complete bytes on these: armed for the first chunk before the
    // barrier below; every later chunk's arm happens right after the previous chunk's data was
    // consumed (still before that chunk's cluster barrier, after which the partner pushes)
    mbar_arrive_expect_tx(r1bar, (uint32_t)p.n1 * 256u);   // the partner's n1/2 columns x 128 rows x 4 B
    mbar_arrive_expect_tx(r2bar, 8192u);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();   // barriers of both CTAs initialised and armed
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) SMALL_TS(1);
  pdl_launch_dependents();

  const int kh = p.kb1 / 2;            // layer-1 K blocks of this split
  const int N1 = p.n1, half1 = N1 / 2;  // layer-1 tile width; each CTA of the pair owns half of it
  const uint32_t l1_stage = 16384u + (uint32_t)N1 * 128u, l1_xchg = (uint32_t)half1 * 512u;
  const uint32_t ID1 = umma_idesc(false, 128, (uint32_t)N1);
  const int pre = kh < NS ? kh : NS;   // layer-1 W1 blocks issued before griddepcontrol.wait (PDL overlap)
  int pre_done = 0;
  if (dev_rows) {
    // the weight blocks of the first stages do not depend on the predecessor: out before its end
    if (warp == 0) {
      if (elect_one()) {
        const uint64_t pol_b = policy_evict_last();
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full[i], l1_stage);
          tma_load_2d(smem + S::B0 + 16384 * i, &tmW1, &full[i], (rank * kh + i) * 64, n * N1, pol_b);
        }
        if (n < 16)
          for (int i = 0; i < 16; ++i) tma_prefetch_2d(&tmW2, rank * 1024 + i * 64, n * 32);
      }
      __syncwarp();
    }
    pre_done = pre;
    pdl_wait();
    M = __ldcg(p.M_dev);
    if (m * 128 >= M) {
      // this m-tile is empty in every chunk (both CTAs of the cluster): complete the issued stages
      // (their h boxes are zero-filled or unused rows) and leave; with no due row at all, CTA 0
      // still finalises the projection of the aged rows
      if (warp == 0) {
        if (elect_one()) {
          for (int i = 0; i < pre; ++i) {
            tma_load_2d(smem + 16384 * i, &tmH, &full[i], (rank * kh + i) * 64, m * 128, policy_evict_first());
            mbar_wait(&full[i], 0);
          }
        }
        __syncwarp();
      }
      __syncthreads();
      if (M == 0 && p.project && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && warp >= 2)
        small_finalize(p, smem, te, warp, false);
      tc_fence_before();
      __syncthreads();
      if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
      }
      return;
    }
  }
  // rows are processed in chunks of 512 (4 m-tiles): one chunk unless a refresh step has more
  // due rows; chunk c's m-tile m covers rows [512 c + 128 m, +128)
  const int chunk_rows = 128 * (int)gridDim.z;   // rows per chunk: the grid's m-tiles
  const int nchunks = (M + chunk_rows - 1) / chunk_rows;
  const int total_mt = (M + 127) / 128;     // m-tiles over all chunks (= layer-3 completions)
  const int q = warp & 3;
  const int row = q * 32 + lane;       // row of the tile (epilogue warps)
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  // TMEM columns: L1 [0, 128), L2 [128, 160), L3 [160, 224)
  const int per_chunk = kh + (l2 ? 16 : 0) + (l3 ? 8 : 0);   // ring iterations of one chunk (stage = it % NS)
  int act = 0;                                     // chunks this CTA has processed (barrier parity)

  for (int chunk = 0; chunk < nchunks; ++chunk) {
    const int row0 = chunk * chunk_rows + m * 128;   // first row of this CTA's m-tile in this chunk
    if (row0 >= M) break;                     // CTA-uniform (and cluster-uniform: same m)
    const int grow = row0 + row;
    const bool more = chunk + 1 < nchunks && row0 + chunk_rows < M;   // this CTA runs another chunk
    const uint32_t par = (uint32_t)act & 1u;
    const int it1 = act * per_chunk, it2 = it1 + kh, it3 = it2 + (l2 ? 16 : 0);
    int* z1_cnt = p.cnt + chunk * 16;        // [4][2]: Z1 column halves published
    int* z2_cnt = p.cnt + chunk * 16 + 8;    // [4]

    // ============================ phase A: layer-1 mainloop ============================
    if (warp == 0) {
      if (elect_one()) {   // TMA producer
        const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
        for (int i = (act == 0 ? pre_done : 0); i < pre; ++i) {   // W1 blocks before griddepcontrol.wait
          const int it = it1 + i, s = it % NS;
          mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], l1_stage);
          tma_load_2d(smem + S::B0 + 16384 * s, &tmW1, &full[s], (rank * kh + i) * 64, n * N1, pol_b);
        }
        if (act == 0 && !pre_done) {
          if (l2)
            for (int i = 0; i < 16; ++i) tma_prefetch_2d(&tmW2, rank * 1024 + i * 64, n * 32);   // into L2 early
          pdl_wait();
          SMALL_TS(2);
        }
        for (int i = 0; i < kh; ++i) {
          const int it = it1 + i, s = it % NS;
          if (i >= pre) {
            mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
            mbar_arrive_expect_tx(&full[s], l1_stage);
            tma_load_2d(smem + S::B0 + 16384 * s, &tmW1, &full[s], (rank * kh + i) * 64, n * N1, pol_b);
          }
          tma_load_2d(smem + 16384 * s, &tmH, &full[s], (rank * kh + i) * 64, row0, pol_a);
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (elect_one()) {   // MMA issuer
        for (int i = 0; i < kh; ++i) {
          const int it = it1 + i, s = it % NS;
          mbar_wait(&full[s], (uint32_t)(it / NS) & 1u);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
          const uint64_t bd = umma_desc_sw128(smem_u32(smem + S::B0 + 16384 * s));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_ss<false>(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID1, (i | k) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(acc1);
      }
      __syncwarp();
    } else {
      // epilogue: stage the 64 columns the partner owns (lane-contiguous 32 KB block, free ring)
      if (act == 0) {
        if (l3) {   // constants of the head and the finalize, fetched while layer 1 runs
          float* cw4 = reinterpret_cast<float*>(smem + S::CW4);
          float* cb3 = reinterpret_cast<float*>(smem + S::CB3);
          if (te < 64) {
            cw4[te] = p.w4[te];
            cb3[te] = p.b3 ? p.b3[te] : 0.0f;
          }
          if (p.project && p.pa.H + 1 <= S::CBETA_MAX)
            for (int t = te; t <= p.pa.H; t += 128)
              reinterpret_cast<uint32_t*>(smem + S::CBETA)[t] = p.pa.beta_q[t];
        }
        pdl_wait();
      }
      mbar_wait(acc1, par);
      tc_fence_after();
      if (te == 0) SMALL_TS(3);
      tmem_to_block(trow, half1 * partner, half1, reinterpret_cast<float*>(smem + S::L1_SEND), row);
      fence_proxy_async_smem();   // generic smem writes -> the bulk copy (async proxy)
    }
    // the partner's ring is free (its layer-1 MMAs completed) and its send block is staged
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();

    // ============================ phase B: layer-1 reduce, layer 2, layer 3 ============================
    if (warp == 0) {
      asm volatile("bar.sync 2, 160;" ::: "memory");   // the epilogue released the ring
      if (l2 && elect_one()) {
        const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
        // layer 2: W2 blocks first (independent), the Z1 blocks once their half is published
        for (int i = 0; i < NS; ++i) {
          const int it = it2 + i, s = it % NS;
          mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 4096u);
          tma_load_2d(smem + S::B0 + 16384 * s, &tmW2, &full[s], rank * 1024 + i * 64, n * 32, pol_b);
        }
        spin_wait_geq(z1_cnt + m * 2 + rank, 2048 / N1);   // every n-tile pair of this K half
        fence_proxy_async_global();
        SMALL_TS(5);
        for (int i = 0; i < 16; ++i) {
          const int it = it2 + i, s = it % NS;
          if (i >= NS) {
            mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
            mbar_arrive_expect_tx(&full[s], 16384u + 4096u);
            tma_load_2d(smem + S::B0 + 16384 * s, &tmW2, &full[s], rank * 1024 + i * 64, n * 32, pol_b);
          }
          tma_load_2d(smem + 16384 * s, &tmZ1, &full[s], rank * 1024 + i * 64, row0, pol_a);
        }
        if (l3) {   // layer 3 (full K = 512): W3 blocks, then the Z2 blocks after all 32 layer-2 CTAs of the m-tile
          for (int i = 0; i < NS; ++i) {
            const int it = it3 + i, s = it % NS;
            mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
            mbar_arrive_expect_tx(&full[s], 16384u + 8192u);
            tma_load_2d(smem + S::B0 + 16384 * s, &tmW3, &full[s], i * 64, 0, pol_b);
          }
          spin_wait_geq(z2_cnt + m, 32);
          fence_proxy_async_global();
          for (int i = 0; i < 8; ++i) {
            const int it = it3 + i, s = it % NS;
            if (i >= NS) {
              mbar_wait(&empty[s], ((uint32_t)(it / NS) & 1u) ^ 1u);
              mbar_arrive_expect_tx(&full[s], 16384u + 8192u);
              tma_load_2d(smem + S::B0 + 16384 * s, &tmW3, &full[s], i * 64, 0, pol_b);
            }
            tma_load_2d(smem + 16384 * s, &tmZ2, &full[s], i * 64, row0, pol_a);
          }
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (l2 && elect_one()) {   // (l3 implies l2)
        for (int i = 0; i < 16; ++i) {
          const int it = it2 + i, s = it % NS;
          mbar_wait(&full[s], (uint32_t)(it / NS) & 1u);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
          const uint64_t bd = umma_desc_sw128(smem_u32(smem + S::B0 + 16384 * s));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_ss<false>(tmem + 128, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID2, (i | k) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(acc2);
        if (l3) {
          for (int i = 0; i < 8; ++i) {
            const int it = it3 + i, s = it % NS;
            mbar_wait(&full[s], (uint32_t)(it / NS) & 1u);
            tc_fence_after();
            const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
            const uint64_t bd = umma_desc_sw128(smem_u32(smem + S::B0 + 16384 * s));
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_ss<false>(tmem + 160, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID3, (i | k) != 0 ? 1u : 0u);
            umma_commit(&empty[s]);
          }
          umma_commit(acc3);
        }
      }
      __syncwarp();
    } else {
      // ---- layer-1 split-K: push the staged block into the partner, reduce the owned 64 columns ----
      if (te == 0) {
        SMALL_TS(4);
        bulk_s2cluster(mapa_shared(smem_u32(smem + S::L1_RECV), (uint32_t)partner), smem + S::L1_SEND, l1_xchg,
                       mapa_shared(smem_u32(r1bar), (uint32_t)partner));
        bulk_commit();
      }
      mbar_wait(r1bar, par);
      if (te == 0) SMALL_TS(12);
      const float* recv = reinterpret_cast<const float*>(smem + S::L1_RECV);
#pragma unroll 1
      for (int c = 0; c < half1; c += 16) {   // the row's owned columns, 16 (32 bytes) at a time
        float f[16];
        uint32_t w[8];
        reduce16(trow, half1 * rank + c, recv, c, rank, row, f);
        relu_bf16_16(f, p.b1, n * N1 + half1 * rank + c, w);
        if (grow < M) {
          uint4* d = reinterpret_cast<uint4*>(p.Z1 + (int64_t)grow * 2048 + n * N1 + half1 * rank + c);
          d[0] = make_uint4(w[0], w[1], w[2], w[3]);
          d[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      if (te == 0) SMALL_TS(13);
      asm volatile("bar.sync 1, 128;" ::: "memory");   // every thread has read the received block
      if (te == 0 && more) mbar_arrive_expect_tx(r1bar, l1_xchg);   // armed for the next chunk
      if (te == 0) bulk_wait_read_all();   // the send block was read: the ring may be reused
      fence_proxy_async_global();          // Z1 (generic stores) -> the layer-2 TMA loads (async proxy)
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        red_release_add(z1_cnt + m * 2 + (n * N1) / 1024, 1);
        SMALL_TS(6);
      }
      asm volatile("bar.sync 2, 160;" ::: "memory");   // the producer may refill the ring
    }
    if (l2 && warp >= 2) {
      // ---- layer 2: reduce the owned 16 columns of the 128 x 32 tile ----
      mbar_wait(acc2, par);
      tc_fence_after();
      if (te == 0) SMALL_TS(7);
      tmem_to_block(trow, 128 + 16 * partner, 16, reinterpret_cast<float*>(smem + S::SEND23), row);
      fence_proxy_async_smem();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        bulk_s2cluster(mapa_shared(smem_u32(smem + S::R2), (uint32_t)partner), smem + S::SEND23, 8192u,
                       mapa_shared(smem_u32(r2bar), (uint32_t)partner));
        bulk_commit();
      }
      mbar_wait(r2bar, par);
      if (te == 0) SMALL_TS(14);
      {
        float f[16];
        uint32_t w2[8];
        reduce16(trow, 128 + 16 * rank, reinterpret_cast<const float*>(smem + S::R2), 0, rank, row, f);
        asm volatile("bar.sync 1, 128;" ::: "memory");   // every thread has read the received block
        if (te == 0 && more) mbar_arrive_expect_tx(r2bar, 8192u);   // armed for the next chunk
        relu_bf16_16(f, p.b2, n * 32 + 16 * rank, w2);
        if (grow < M) {
          uint4* d = reinterpret_cast<uint4*>(p.Z2 + (int64_t)grow * 512 + n * 32 + 16 * rank);
          d[0] = make_uint4(w2[0], w2[1], w2[2], w2[3]);
          d[1] = make_uint4(w2[4], w2[5], w2[6], w2[7]);
        }
      }
      if (te == 0) bulk_wait_read_all();
      fence_proxy_async_global();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        red_release_add(z2_cnt + m, 1);
        SMALL_TS(8);
      }
    }

    if (l3 && warp >= 2) {
      // ---- layer 3 (this CTA holds the whole 128 x 64 Z3 tile): + b3, ReLU, w4 dot, + b4 ----
      const bool owner = grow < M;
      int32_t ntok = 0, inst = 0, r = grow;   // the row's N(r), instance and (refresh) slot, fetched
      if (owner) {                            // while layer 3 runs
        if (p.r_idx) r = p.r_idx[grow];
        if (p.n_tok) ntok = p.n_tok[grow];
        if (p.project) inst = p.pa.inst[r];
      }
      mbar_wait(acc3, par);
      tc_fence_after();
      if (te == 0) SMALL_TS(9);
      float y = 0.0f;
      const float* cw4 = reinterpret_cast<const float*>(smem + S::CW4);
      const float* cb3 = reinterpret_cast<const float*>(smem + S::CB3);
#pragma unroll 1
      for (int c = 0; c < 64; c += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(trow + 160u + (uint32_t)c, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) y = fmaf(cw4[c + j], fmaxf(__uint_as_float(v[j]) + cb3[c + j], 0.0f), y);
      }
      y += p.b4 ? __ldg(p.b4) : 0.0f;
      int32_t nh = 0;
      if (owner) {
        int32_t cap = p.max_ctx - ntok;
        cap = cap < 0 ? 0 : cap;
        nh = __float2int_rn(fminf(fmaxf(y, 0.0f), (float)cap));   // quantize_nhat (readings A8-A10)
        if (p.y_hat) p.y_hat[grow] = y;
        if (p.n_hat) p.n_hat[grow] = nh;
        if (p.r_idx) {   // refresh: scatter into the request's slot and restart its cadence (reading A27)
          p.r_nhat[r] = nh;
          p.r_glast[r] = p.r_gen[r];
          p.r_nhat_last[r] = nh;
        }
      }
      if (p.project) {
        uint32_t errbits = 0;
        proj_accumulate(p.pa, owner, inst, ntok, nh, p.pa.ws_cnt, p.pa.ws_sum, errbits);
        if (errbits && p.pa.err) atomicOr(p.pa.err, (int)errbits);
      }
      fence_acq_rel_gpu();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        SMALL_TS(10);
        *s_last = (atomicAdd(p.cnt + S::DONE, 1) == total_mt - 1) ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*s_last) {
        fence_acq_rel_gpu();
        if (p.project) small_finalize(p, smem, te, warp, true);
        // every counter of this launch has been consumed: re-arm them for the next one
        for (int k = te; k < nchunks * 16; k += 128) p.cnt[k] = 0;
        if (te == 0) p.cnt[S::DONE] = 0;
        if (te == 0) SMALL_TS(11);
      }
    }
    ++act;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

}  // namespace star
