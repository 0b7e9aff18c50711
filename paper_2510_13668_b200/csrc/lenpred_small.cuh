// lenpred_small.cuh -- the whole predictor (Eq. 2) + quantizer + the fused
// projection for one rank's batch of up to 512 requests in ONE persistent launch: the per-rank
// shape of the north-star job (one decode instance of 512 running requests per B200).
//
//   Z1 = phi(W1 h + b1) -> Z2 = phi(W2 Z1 + b2) -> Z3 = phi(W3 Z2 + b3) -> y = w4 . Z3 + b4
//   -> N_hat = q(y) [-> keyed projection histogram -> per-instance loads]
//
// Grid (4, 8, m_tiles) in clusters of 4 CTAs along x: cluster (m, n) and CTA rank r.  Every
// CTA is resident at once (one CTA per SM, <= 128 CTAs, checked on the host), so the phases
// hand off through per-m-tile counters in global memory instead of kernel boundaries:
//   L1  tile 128 x 256 of Z1 (rows of m-tile m, columns of n-tile n) over the K quarter r:
//       TMA -> 4-stage SMEM ring -> tcgen05 (M=128, N=256) -> TMEM.  Split-K reduction in
//       DISTRIBUTED SHARED MEMORY: each CTA stages the partial columns its three partners own in
//       its (now free) ring, one cluster barrier, three 32 KB bulk copies shared::cta ->
//       shared::cluster (TMA engine) into the partners' receive slots, completion on their
//       mbarriers; each CTA sums its 64 owned columns in fixed split order (deterministic),
//       + b1, ReLU, bf16 -> Z1 (L2-resident global), then bumps z1_cnt[m][n] (release).
//   L2  tile 128 x 64 of Z2 (n2 = n) over the K quarter r (= Z1 columns of n-tiles 2r, 2r+1):
//       the W2 block streams in first (independent), the Z1 block after z1_cnt[m][2r..2r+1]
//       reach 4 (acquire); tcgen05 N=64; the same DSMEM reduction (8 KB blocks, owned 16
//       columns) -> + b2, ReLU, bf16 -> Z2, bump z2_cnt[m].
//   L3  (clusters n == 0: one per m-tile) Z3 = W3 Z2 over the K quarter r after z2_cnt[m] = 32;
//       DSMEM reduction (owned 16 columns), + b3, ReLU, the partial w4 dot of the owned
//       columns -> CTA 0 of the cluster (DSMEM), which sums the four partial dots in rank order,
//       + b4, quantizes (readings A8-A10) and adds the rows to the projection histogram; the
//       last m-tile to finish finalises L/W/peak/growth/count and re-arms every counter.
// Roles (192 threads, as in umma_gemm_kernel): warp 0 TMA producer, warp 1 MMA issuer (one
// elected lane), warps 2-5 epilogue (TMEM lane quarter = warp % 4).
#pragma once
#include "lenpred_kernels.cuh"
#include "project_core.cuh"

namespace star {

struct SmallArgs {
  int M;                 // rows (<= 512)
  int kb1;               // layer-1 K blocks (d / 64), multiple of 4
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
  int* cnt;              // z1_cnt [4][8] | z2_cnt [4] | done [1]   (zero between launches)
  int project;
  ProjArgs pa;
  uint64_t* tl;          // diagnostics: [ctas][16] %globaltimer phase stamps, or nullptr
};

struct SmallSmem {
  static constexpr uint32_t RING = 192u * 1024u;          // L1 stages: A 16 KB @ 16K*s, B 32 KB @ 64K + 32K*s
  static constexpr uint32_t L1_SEND = 0;                  // [3][32 KB]
  static constexpr uint32_t L1_RECV = 96u * 1024u;        // [3][32 KB]
  static constexpr uint32_t SEND23 = 96u * 1024u;         // layer-2 send [3][8 KB] (beyond the L2/L3 stages)
  static constexpr uint32_t SEND3 = 120u * 1024u;         // layer-3 send [3][8 KB]
  static constexpr uint32_t R3 = 168u * 1024u;            // layer-3 receive [3][8 KB]
  static constexpr uint32_t R2 = 192u * 1024u;            // layer-2 receive [3][8 KB]
  static constexpr uint32_t DOT = 216u * 1024u;           // [4][128] fp32 partial dots (CTA 0)
  static constexpr uint32_t BAR = DOT + 2048u;
  static constexpr uint32_t BYTES = 1024u + BAR + 256u;
};
static_assert(SmallSmem::BYTES <= 227u * 1024u, "small predictor smem");

#define SMALL_TS(k)                                                                                     \
  do {                                                                                                  \
    if (p.tl) p.tl[(((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + (k)] = \
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
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stages 32 lanes x `cols` fp32 TMEM columns [c0, c0 + cols) of this warp's rows into a
// lane-contiguous block [cols/4][128 rows][4] (conflict-free 16-byte stores).
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

// Owned columns [c0, c0 + 16) of this row: own TMEM partial + the 3 received blocks, summed in
// split order 0..3 (deterministic).  recv slot of sender s = s - (s > rank).
__device__ __forceinline__ void reduce16(uint32_t trow, int c0, const float* recv, uint32_t blk_bytes, int cl,
                                         int rank, int row, float (&f)[16]) {
  uint32_t v[16];
  tmem_ld_32x32b_x16(trow + (uint32_t)c0, v);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = 0.0f;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s == rank) {
#pragma unroll
      for (int j = 0; j < 16; ++j) f[j] += __uint_as_float(v[j]);
    } else {
      const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(recv) +
                                                          (size_t)(s - (s > rank)) * blk_bytes) + row;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 x = src[(cl / 4 + j) * 128];
        f[4 * j] += x.x;
        f[4 * j + 1] += x.y;
        f[4 * j + 2] += x.z;
        f[4 * j + 3] += x.w;
      }
    }
  }
}

__global__ void __launch_bounds__(192, 1)
    lenpred_small_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW1,
                         const __grid_constant__ CUtensorMap tmZ1, const __grid_constant__ CUtensorMap tmW2,
                         const __grid_constant__ CUtensorMap tmZ2, const __grid_constant__ CUtensorMap tmW3,
                         const SmallArgs p) {
  using S = SmallSmem;
  constexpr uint32_t ID1 = umma_idesc(false, 128, 256);
  constexpr uint32_t ID64 = umma_idesc(false, 128, 64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR);
  uint64_t* empty = full + 4;
  uint64_t* acc1 = empty + 4;
  uint64_t* acc2 = acc1 + 1;
  uint64_t* acc3 = acc2 + 1;
  uint64_t* r1bar = acc3 + 1;
  uint64_t* r2bar = r1bar + 1;
  uint64_t* r3bar = r2bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r3bar + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = blockIdx.x, n = blockIdx.y, m = blockIdx.z;
  const int m_tiles = gridDim.z;
  const bool l3 = n == 0;   // this cluster also runs layer 3 + head for m-tile m
  int* z1_cnt = p.cnt;       // [4][8]
  int* z2_cnt = p.cnt + 32;  // [4]
  int* done = p.cnt + 36;
  if (threadIdx.x == 0) SMALL_TS(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH);
    tma_prefetch_desc(&tmW1);
    tma_prefetch_desc(&tmZ1);
    tma_prefetch_desc(&tmW2);
    if (l3) {
      tma_prefetch_desc(&tmZ2);
      tma_prefetch_desc(&tmW3);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc1, 1);
    mbar_init(acc2, 1);
    mbar_init(acc3, 1);
    mbar_init(r1bar, 1);
    mbar_init(r2bar, 1);
    mbar_init(r3bar, 1);
    // the partners' bulk copies complete bytes on these: arm them before anyone can send
    mbar_arrive_expect_tx(r1bar, 3u * 32768u);
    mbar_arrive_expect_tx(r2bar, 3u * 8192u);
    if (l3) mbar_arrive_expect_tx(r3bar, 3u * 8192u);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  // every CTA of the cluster has armed its receive barriers before any partner's first send
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) SMALL_TS(1);

  const int kq = p.kb1 / 4;            // layer-1 K blocks of this split
  const int q = warp & 3;
  const int row = q * 32 + lane;       // row of the tile (epilogue warps)
  const int grow = m * 128 + row;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int te = threadIdx.x - 64;     // epilogue thread 0..127

  pdl_launch_dependents();

  // ============================ phase A: layer-1 mainloop ============================
  if (warp == 0) {
    if (elect_one()) {   // TMA producer
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      // W1 blocks of the first stages before griddepcontrol.wait (PDL overlap)
      const int pre = kq < 4 ? kq : 4;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], 16384u + 32768u);
        tma_load_2d(smem + 65536 + 32768 * i, &tmW1, &full[i], (rank * kq + i) * 64, n * 256, pol_b);
      }
      // the layer-2 weight blocks this CTA needs later: into L2 now (independent of h)
      for (int i = 0; i < 8; ++i) tma_prefetch_2d(&tmW2, rank * 512 + i * 64, n * 64);
      pdl_wait();
      SMALL_TS(2);
      for (int i = 0; i < kq; ++i) {
        const int s = i & 3;
        if (i >= pre) {
          mbar_wait(&empty[s], ((uint32_t)(i >> 2) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 32768u);
          tma_load_2d(smem + 65536 + 32768 * s, &tmW1, &full[s], (rank * kq + i) * 64, n * 256, pol_b);
        }
        tma_load_2d(smem + 16384 * s, &tmH, &full[s], (rank * kq + i) * 64, m * 128, pol_a);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {   // MMA issuer
      for (int i = 0; i < kq; ++i) {
        const int s = i & 3;
        mbar_wait(&full[s], (uint32_t)(i >> 2) & 1u);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
        const uint64_t bd = umma_desc_sw128(smem_u32(smem + 65536 + 32768 * s));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_ss<false>(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID1, (i | k) != 0 ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(acc1);
    }
    __syncwarp();
  } else {
    // epilogue: stage the columns each partner owns (lane-contiguous 32 KB blocks, free ring)
    pdl_wait();
    mbar_wait(acc1, 0);
    tc_fence_after();
    if (te == 0) SMALL_TS(3);
    for (int pr = 0; pr < 4; ++pr) {
      if (pr == rank) continue;
      tmem_to_block(trow, 64 * pr, 64, reinterpret_cast<float*>(smem + S::L1_SEND + 32768u * (pr - (pr > rank))), row);
    }
    fence_proxy_async_smem();   // generic smem writes -> the bulk copies (async proxy)
  }
  // every partner's ring is free (its layer-1 MMAs completed) and its send blocks are staged
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();

  // ============================ phase B: layer-1 reduce, layer 2, layer 3 ============================
  const int it2 = kq, it3 = kq + 8;   // ring iteration numbers (stage = it % 4, phase = (it / 4) & 1)
  if (warp == 0) {
    asm volatile("bar.sync 2, 160;" ::: "memory");   // the epilogue released the ring
    if (elect_one()) {
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      // layer 2: W2 blocks first (independent), the Z1 blocks once their producers published
      for (int i = 0; i < 4; ++i) {
        const int it = it2 + i, s = it & 3;
        mbar_wait(&empty[s], ((uint32_t)(it >> 2) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], 16384u + 8192u);
        tma_load_2d(smem + 65536 + 8192 * s, &tmW2, &full[s], rank * 512 + i * 64, n * 64, pol_b);
      }
      spin_wait_geq(z1_cnt + m * 8 + 2 * rank, 4);
      spin_wait_geq(z1_cnt + m * 8 + 2 * rank + 1, 4);
      fence_proxy_async_global();
      SMALL_TS(5);
      for (int i = 0; i < 8; ++i) {
        const int it = it2 + i, s = it & 3;
        if (i >= 4) {
          mbar_wait(&empty[s], ((uint32_t)(it >> 2) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 8192u);
          tma_load_2d(smem + 65536 + 8192 * s, &tmW2, &full[s], rank * 512 + i * 64, n * 64, pol_b);
        }
        tma_load_2d(smem + 16384 * s, &tmZ1, &full[s], rank * 512 + i * 64, m * 128, pol_a);
      }
      if (l3) {   // layer 3: W3 blocks, then the Z2 blocks after all 32 layer-2 CTAs of m-tile m
        for (int i = 0; i < 2; ++i) {
          const int it = it3 + i, s = it & 3;
          mbar_wait(&empty[s], ((uint32_t)(it >> 2) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 16384u + 8192u);
          tma_load_2d(smem + 65536 + 8192 * s, &tmW3, &full[s], rank * 128 + i * 64, 0, pol_b);
        }
        spin_wait_geq(z2_cnt + m, 32);
        fence_proxy_async_global();
        for (int i = 0; i < 2; ++i) {
          const int it = it3 + i, s = it & 3;
          tma_load_2d(smem + 16384 * s, &tmZ2, &full[s], rank * 128 + i * 64, m * 128, pol_a);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      for (int i = 0; i < 8; ++i) {
        const int it = it2 + i, s = it & 3;
        mbar_wait(&full[s], (uint32_t)(it >> 2) & 1u);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
        const uint64_t bd = umma_desc_sw128(smem_u32(smem + 65536 + 8192 * s));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_ss<false>(tmem + 256, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID64, (i | k) != 0 ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(acc2);
      if (l3) {
        for (int i = 0; i < 2; ++i) {
          const int it = it3 + i, s = it & 3;
          mbar_wait(&full[s], (uint32_t)(it >> 2) & 1u);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
          const uint64_t bd = umma_desc_sw128(smem_u32(smem + 65536 + 8192 * s));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_ss<false>(tmem + 320, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID64, (i | k) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(acc3);
      }
    }
    __syncwarp();
  } else {
    // ---- layer-1 split-K: push the staged blocks into the partners, reduce the owned 64 columns ----
    if (te == 0) {
      SMALL_TS(4);
      for (int pr = 0; pr < 4; ++pr) {
        if (pr == rank) continue;
        const uint32_t dst = mapa_shared(smem_u32(smem + S::L1_RECV + 32768u * (rank - (rank > pr))), (uint32_t)pr);
        bulk_s2cluster(dst, smem + S::L1_SEND + 32768u * (pr - (pr > rank)), 32768u,
                       mapa_shared(smem_u32(r1bar), (uint32_t)pr));
      }
      bulk_commit();
    }
    mbar_wait(r1bar, 0);
    const float* recv = reinterpret_cast<const float*>(smem + S::L1_RECV);
#pragma unroll 1
    for (int c = 0; c < 64; c += 16) {
      float f[16];
      reduce16(trow, 64 * rank + c, recv, 32768u, c, rank, row, f);
      const int col = n * 256 + 64 * rank + c;
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a0 = fmaxf(f[2 * j] + (p.b1 ? __ldg(p.b1 + col + 2 * j) : 0.0f), 0.0f);
        const float a1 = fmaxf(f[2 * j + 1] + (p.b1 ? __ldg(p.b1 + col + 2 * j + 1) : 0.0f), 0.0f);
        __nv_bfloat162 b = __floats2bfloat162_rn(a0, a1);
        w[j] = *reinterpret_cast<uint32_t*>(&b);
      }
      if (grow < p.M) {
        uint4* d = reinterpret_cast<uint4*>(p.Z1 + (int64_t)grow * 2048 + col);
        d[0] = make_uint4(w[0], w[1], w[2], w[3]);
        d[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    if (te == 0) bulk_wait_read_all();   // the send blocks were read: the ring may be reused
    fence_proxy_async_global();          // Z1 (generic stores) -> the layer-2 TMA loads (async proxy)
    fence_acq_rel_gpu();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      red_release_add(z1_cnt + m * 8 + n, 1);
      SMALL_TS(6);
    }
    asm volatile("bar.sync 2, 160;" ::: "memory");   // the producer may refill the ring

    // ---- layer 2: reduce the owned 16 columns of the 128 x 64 tile ----
    mbar_wait(acc2, 0);
    tc_fence_after();
    if (te == 0) SMALL_TS(7);
    for (int pr = 0; pr < 4; ++pr) {
      if (pr == rank) continue;
      tmem_to_block(trow, 256 + 16 * pr, 16, reinterpret_cast<float*>(smem + S::SEND23 + 8192u * (pr - (pr > rank))), row);
    }
    fence_proxy_async_smem();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      for (int pr = 0; pr < 4; ++pr) {
        if (pr == rank) continue;
        const uint32_t dst = mapa_shared(smem_u32(smem + S::R2 + 8192u * (rank - (rank > pr))), (uint32_t)pr);
        bulk_s2cluster(dst, smem + S::SEND23 + 8192u * (pr - (pr > rank)), 8192u,
                       mapa_shared(smem_u32(r2bar), (uint32_t)pr));
      }
      bulk_commit();
    }
    mbar_wait(r2bar, 0);
    {
      float f[16];
      reduce16(trow, 256 + 16 * rank, reinterpret_cast<const float*>(smem + S::R2), 8192u, 0, rank, row, f);
      const int col = n * 64 + 16 * rank;
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a0 = fmaxf(f[2 * j] + (p.b2 ? __ldg(p.b2 + col + 2 * j) : 0.0f), 0.0f);
        const float a1 = fmaxf(f[2 * j + 1] + (p.b2 ? __ldg(p.b2 + col + 2 * j + 1) : 0.0f), 0.0f);
        __nv_bfloat162 b = __floats2bfloat162_rn(a0, a1);
        w[j] = *reinterpret_cast<uint32_t*>(&b);
      }
      if (grow < p.M) {
        uint4* d = reinterpret_cast<uint4*>(p.Z2 + (int64_t)grow * 512 + col);
        d[0] = make_uint4(w[0], w[1], w[2], w[3]);
        d[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
    if (te == 0) bulk_wait_read_all();
    fence_proxy_async_global();
    fence_acq_rel_gpu();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (te == 0) {
      red_release_add(z2_cnt + m, 1);
      SMALL_TS(8);
    }
  }

  if (l3) {
    float dot = 0.0f;
    if (warp >= 2) {
      // ---- L3: reduce the owned 16 Z3 columns, + b3, ReLU, partial w4 dot ----
      mbar_wait(acc3, 0);
      tc_fence_after();
      if (te == 0) SMALL_TS(9);
      for (int pr = 0; pr < 4; ++pr) {
        if (pr == rank) continue;
        tmem_to_block(trow, 320 + 16 * pr, 16, reinterpret_cast<float*>(smem + S::SEND3 + 8192u * (pr - (pr > rank))), row);
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        for (int pr = 0; pr < 4; ++pr) {
          if (pr == rank) continue;
          const uint32_t dst = mapa_shared(smem_u32(smem + S::R3 + 8192u * (rank - (rank > pr))), (uint32_t)pr);
          bulk_s2cluster(dst, smem + S::SEND3 + 8192u * (pr - (pr > rank)), 8192u,
                         mapa_shared(smem_u32(r3bar), (uint32_t)pr));
        }
        bulk_commit();
      }
      mbar_wait(r3bar, 0);
      float f[16];
      reduce16(trow, 320 + 16 * rank, reinterpret_cast<const float*>(smem + S::R3), 8192u, 0, rank, row, f);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int c = 16 * rank + j;
        dot = fmaf(__ldg(p.w4 + c), fmaxf(f[j] + (p.b3 ? __ldg(p.b3 + c) : 0.0f), 0.0f), dot);
      }
      // partial dot -> CTA 0's DOT[rank][row] (distributed shared memory)
      const uint32_t da = mapa_shared(smem_u32(smem + S::DOT + 4u * (uint32_t)(rank * 128 + row)), 0u);
      asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(da), "f"(dot) : "memory");
      if (te == 0) bulk_wait_read_all();
    }
    cluster_sync_all();   // the four partial dots are in CTA 0
    if (rank == 0 && warp >= 2) {
      const float* D = reinterpret_cast<const float*>(smem + S::DOT);
      float y = 0.0f;
#pragma unroll
      for (int s = 0; s < 4; ++s) y += D[s * 128 + row];   // rank order (deterministic)
      y += p.b4 ? __ldg(p.b4) : 0.0f;
      const bool owner = grow < p.M;
      int32_t nh = 0, ntok = 0, inst = 0;
      if (owner) {
        if (p.n_tok) ntok = p.n_tok[grow];
        if (p.project) inst = p.pa.inst[grow];
        int32_t cap = p.max_ctx - ntok;
        cap = cap < 0 ? 0 : cap;
        nh = __float2int_rn(fminf(fmaxf(y, 0.0f), (float)cap));   // quantize_nhat (readings A8-A10)
        if (p.y_hat) p.y_hat[grow] = y;
        if (p.n_hat) p.n_hat[grow] = nh;
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
        *s_last = (atomicAdd(done, 1) == m_tiles - 1) ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*s_last) {
        fence_acq_rel_gpu();
        if (p.project) {
          // finalize from the global histogram (one warp per instance), re-zero it; the
          // histogram comes into shared memory with L2 loads (other SMs' atomics) when it fits
          const int nb = p.pa.n_inst * (p.pa.H + 2);
          uint32_t* sbeta = reinterpret_cast<uint32_t*>(smem + S::DOT);   // the dots are consumed
          for (int t = te; t <= p.pa.H; t += 128) sbeta[t] = p.pa.beta_q[t];
          const uint32_t* hc = p.pa.ws_cnt;
          const unsigned long long* hs = p.pa.ws_sum;
          if ((uint32_t)nb * 12u <= 48u * 1024u) {   // R3 + R2 (both consumed)
            unsigned long long* ss = reinterpret_cast<unsigned long long*>(smem + S::R3);
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
        // every counter of this launch has been consumed: re-arm them for the next one
        for (int k = te; k < 37; k += 128) p.cnt[k] = 0;
        if (te == 0) SMALL_TS(11);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace star
