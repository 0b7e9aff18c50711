// lenpred_tail2.cuh -- the predictor tail of Eq. 2 for large batches (> 512 rows):
//
//   Z2 = phi(W2 Z1 + b2) -> Z3 = phi(W3 Z2 + b3) -> y = w4 . Z3 + b4 -> N_hat = q(y) [-> projection]
//
// after the layer-1 GEMM, in one launch of clusters of 4 CTAs, one cluster per 128-row m-tile:
//   * CTA r of the cluster computes Z2[:, 128 r .. 128 r + 128) over the FULL K = m1 (no split-K, so
//     no layer-2 partial exchange): TMA -> 6-stage ring -> tcgen05 M=128 N=128 -> TMEM; the W2
//     blocks of the first stages and the CTA's W3 slice (64 x 128) load before griddepcontrol.wait;
//   * the epilogue writes relu(Z2 + b2) in bf16 straight into shared memory as the 128B-swizzled
//     A operand of layer 3 (no global Z2) and the CTA multiplies it by its W3 slice: the layer-3
//     partial over K = its 128 Z2 columns (tcgen05 N = 64);
//   * the four layer-3 partials of the m-tile meet in distributed shared memory (reduce-scatter:
//     each CTA owns 16 of the 64 Z3 columns; three 8 KB bulk copies per CTA), each CTA sums its
//     columns in rank order (deterministic), + b3, ReLU and its part of the w4 dot; the four
//     partial dots go to CTA 0 (DSMEM), which adds them in rank order, + b4, quantizes (readings
//     A8-A10) and adds the rows to the projection histogram; the last m-tile to finish finalises
//     L/W/peak/growth/count (as the small-batch kernel does).
// Compared with tail_kernel (split-K over 2 CTAs with partials through global memory, layer-3
// partials through global memory and an arrival counter), the two global exchanges go; the
// mainloop streams 1 MB instead of 768 KB per CTA.
#pragma once
#include "lenpred_kernels.cuh"
#include "lenpred_small.cuh"
#include "project_core.cuh"

namespace star {

struct Tail2Args {
  int M;                 // rows
  int num_kb;            // layer-2 K blocks (m1 / 64)
  const float* b2;       // [512] or nullptr
  const float* b3;       // [64] or nullptr
  const float* w4;       // [64]
  const float* b4;       // [1] or nullptr
  const int32_t* n_tok;  // [M] or nullptr
  int32_t max_ctx;
  float* y_hat;          // [M] or nullptr
  int32_t* n_hat;        // [M] or nullptr
  int* done;             // [1] m-tiles finished (zero between launches)
  int project;
  ProjArgs pa;
  uint64_t* tl;          // diagnostics: [ctas][32] %globaltimer stamps, or nullptr
};

struct Tail2Smem {
  static constexpr int STAGES = 6;
  static constexpr uint32_t B0 = 96u * 1024u;        // stage s: A @ 16K*s, B (128 rows) @ B0 + 16K*s
  static constexpr uint32_t W3 = 192u * 1024u;       // W3 slice: 2 K blocks x 64 rows (16 KB)
  static constexpr uint32_t A3 = 0;                  // layer-3 A operand (ring idle): 2 x 16 KB
  static constexpr uint32_t SEND = 32u * 1024u;      // Z3 partial blocks for the 3 partners: 3 x 8 KB
  static constexpr uint32_t RECV = 64u * 1024u;      // from the 3 partners: 3 x 8 KB
  static constexpr uint32_t DOT = 208u * 1024u;      // [4][128] partial dots (CTA 0)
  static constexpr uint32_t BAR = DOT + 2048u;
  static constexpr uint32_t HIST = 96u * 1024u;      // finalize: histogram staging (ring idle), <= 96 KB
  // constants fetched while layer 2 runs: this rank's w4 / b3 slices, beta [<= 512] (rank 0)
  static constexpr uint32_t CW4 = BAR + 256u, CB3 = CW4 + 64u, CBETA = CB3 + 64u;
  static constexpr int CBETA_MAX = 512;
  static constexpr uint32_t BYTES = 1024u + CBETA + 4u * CBETA_MAX;
};
static_assert(Tail2Smem::BYTES <= 227u * 1024u, "tail2 smem");

#define TAIL2_TS(k)                                                                               \
  do {                                                                                            \
    if (p.tl) p.tl[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 32 + (k)] = globaltimer_ns(); \
  } while (0)

__global__ void __launch_bounds__(192, 1)
    tail2_kernel(const __grid_constant__ CUtensorMap tmZ1, const __grid_constant__ CUtensorMap tmW2,
                 const __grid_constant__ CUtensorMap tmW3, const Tail2Args p) {
  using S = Tail2Smem;
  constexpr int NS = S::STAGES;
  constexpr uint32_t ID2 = umma_idesc(false, 128, 128);
  constexpr uint32_t ID3 = umma_idesc(false, 128, 64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR);
  uint64_t* empty = full + NS;
  uint64_t* acc2 = empty + NS;
  uint64_t* w3bar = acc2 + 1;
  uint64_t* a3bar = w3bar + 1;
  uint64_t* acc3 = a3bar + 1;
  uint64_t* rbar = acc3 + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = blockIdx.x, m = blockIdx.y;
  const int te = threadIdx.x - 64;
  if (threadIdx.x == 0) {
    TAIL2_TS(0);
    if (p.tl) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.tl[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 32 + 15] = smid;
    }
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmZ1);
    tma_prefetch_desc(&tmW2);
    tma_prefetch_desc(&tmW3);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc2, 1);
    mbar_init(w3bar, 1);
    mbar_init(a3bar, 4);   // one arrive per epilogue warp
    mbar_init(acc3, 1);
    mbar_init(rbar, 1);
    mbar_arrive_expect_tx(rbar, 3u * 8192u);   // the partners' Z3 blocks (pushed after a cluster barrier)
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_launch_dependents();
  if (threadIdx.x == 0) TAIL2_TS(1);
  const int q = warp & 3;
  const int row = q * 32 + lane;
  const int grow = m * 128 + row;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int nkb = p.num_kb;

  if (warp == 0) {
    if (elect_one()) {   // TMA producer
      const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
      // independent of the layer-1 kernel: the W3 slice and the first W2 stages
      mbar_arrive_expect_tx(w3bar, 2u * 8192u);
      for (int kk = 0; kk < 2; ++kk) tma_load_2d(smem + S::W3 + 8192 * kk, &tmW3, w3bar, rank * 128 + kk * 64, 0, pol_b);
      const int pre = nkb < NS ? nkb : NS;
      for (int i = 0; i < pre; ++i) {
        mbar_arrive_expect_tx(&full[i], 32768u);
        tma_load_2d(smem + S::B0 + 16384 * i, &tmW2, &full[i], i * 64, rank * 128, pol_b);
      }
      pdl_wait();
      if (threadIdx.x == 0) TAIL2_TS(2);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % NS;
        if (i >= pre) {
          mbar_wait(&empty[s], ((uint32_t)(i / NS) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], 32768u);
          tma_load_2d(smem + S::B0 + 16384 * s, &tmW2, &full[s], i * 64, rank * 128, pol_b);
        }
        tma_load_2d(smem + 16384 * s, &tmZ1, &full[s], i * 64, m * 128, pol_a);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {   // MMA issuer: layer 2, then the layer-3 partial
      for (int i = 0; i < nkb; ++i) {
        const int s = i % NS;
        mbar_wait(&full[s], (uint32_t)(i / NS) & 1u);
        tc_fence_after();
        const uint64_t ad = umma_desc_sw128(smem_u32(smem + 16384 * s));
        const uint64_t bd = umma_desc_sw128(smem_u32(smem + S::B0 + 16384 * s));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_ss<false>(tmem, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID2, (i | k) != 0 ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(acc2);
      mbar_wait(w3bar, 0);
      mbar_wait(a3bar, 0);
      tc_fence_after();
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t ad = umma_desc_sw128(smem_u32(smem + S::A3 + 16384 * kk));
        const uint64_t bd = umma_desc_sw128(smem_u32(smem + S::W3 + 8192 * kk));
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_ss<false>(tmem + 128, ad + (uint64_t)(k * 2), bd + (uint64_t)(k * 2), ID3, (kk | k) != 0 ? 1u : 0u);
      }
      umma_commit(acc3);
    }
    __syncwarp();
  }
  // CTA 0's epilogue threads own the rows' outputs: fetch N(r) and the instance now, off the
  // critical path (after griddepcontrol.wait: the predecessor may have written them)
  int32_t ntok = 0, inst = 0;
  if (warp >= 2) {
    if (te < 16) {   // the head's constants (static: before griddepcontrol.wait)
      reinterpret_cast<float*>(smem + S::CW4)[te] = p.w4[16 * rank + te];
      reinterpret_cast<float*>(smem + S::CB3)[te] = p.b3 ? p.b3[16 * rank + te] : 0.0f;
    }
    if (rank == 0 && p.project && p.pa.H + 1 <= S::CBETA_MAX)
      for (int t = te; t <= p.pa.H; t += 128) reinterpret_cast<uint32_t*>(smem + S::CBETA)[t] = p.pa.beta_q[t];
    pdl_wait();   // the outputs below may still be read by the previous kernel
    if (rank == 0 && grow < p.M) {
      if (p.n_tok) ntok = p.n_tok[grow];
      if (p.project) inst = p.pa.inst[grow];
    }
  }
  if (warp >= 2) {
    // ---- layer-2 epilogue: relu(Z2 + b2) -> bf16 -> the swizzled layer-3 A operand in smem ----
    mbar_wait(acc2, 0);
    tc_fence_after();
    if (te == 0) TAIL2_TS(3);
#pragma unroll 1
    for (int c = 0; c < 128; c += 16) {
      uint32_t v[16];
      tmem_ld_32x32b_x16(trow + (uint32_t)c, v);
      tmem_ld_wait();
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) f[j] = __uint_as_float(v[j]);
      uint32_t w[8];
      relu_bf16_16(f, p.b2, rank * 128 + c, w);
      // 128B-swizzled K-major tile: row `row`, 16-byte chunk cb of K block c / 64
      uint4* rowp = reinterpret_cast<uint4*>(smem + S::A3 + (c / 64) * 16384 + row * 128);
      const int cb = (c % 64) / 8;
      rowp[cb ^ (row & 7)] = make_uint4(w[0], w[1], w[2], w[3]);
      rowp[(cb + 1) ^ (row & 7)] = make_uint4(w[4], w[5], w[6], w[7]);
    }
    fence_proxy_async_smem();   // generic smem writes -> the tensor core
    __syncwarp();
    if (lane == 0) mbar_arrive(a3bar);
    // ---- layer-3 partial: stage the columns each partner owns ----
    mbar_wait(acc3, 0);
    tc_fence_after();
    if (te == 0) TAIL2_TS(4);
    for (int pr = 0; pr < 4; ++pr) {
      if (pr == rank) continue;
      tmem_to_block(trow, 128 + 16 * pr, 16, reinterpret_cast<float*>(smem + S::SEND + 8192u * (pr - (pr > rank))), row);
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  cluster_sync_all();   // every partner staged its blocks (and its RECV slots are free: ring idle)
  tc_fence_after();
  float dot = 0.0f;
  if (warp >= 2) {
    if (te == 0) {
      TAIL2_TS(5);
      for (int pr = 0; pr < 4; ++pr) {
        if (pr == rank) continue;
        bulk_s2cluster(mapa_shared(smem_u32(smem + S::RECV + 8192u * (rank - (rank > pr))), (uint32_t)pr),
                       smem + S::SEND + 8192u * (pr - (pr > rank)), 8192u, mapa_shared(smem_u32(rbar), (uint32_t)pr));
      }
      bulk_commit();
    }
    mbar_wait(rbar, 0);
    // own 16 Z3 columns: the four partials in rank order (deterministic), + b3, ReLU, w4 dot
    uint32_t v[16];
    tmem_ld_32x32b_x16(trow + 128u + (uint32_t)(16 * rank), v);
    tmem_ld_wait();
    float f[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = 0.0f;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s == rank) {
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] += __uint_as_float(v[j]);
      } else {
        const float4* src = reinterpret_cast<const float4*>(smem + S::RECV + 8192u * (s - (s > rank))) + row;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 x = src[j * 128];
          f[4 * j] += x.x;
          f[4 * j + 1] += x.y;
          f[4 * j + 2] += x.z;
          f[4 * j + 3] += x.w;
        }
      }
    }
    const float* cw4 = reinterpret_cast<const float*>(smem + S::CW4);
    const float* cb3 = reinterpret_cast<const float*>(smem + S::CB3);
#pragma unroll
    for (int j = 0; j < 16; ++j) dot = fmaf(cw4[j], fmaxf(f[j] + cb3[j], 0.0f), dot);
    const uint32_t da = mapa_shared(smem_u32(smem + S::DOT + 4u * (uint32_t)(rank * 128 + row)), 0u);
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(da), "f"(dot) : "memory");
    if (te == 0) bulk_wait_read_all();
  }
  cluster_sync_all();   // the four partial dots are in CTA 0
  if (rank == 0 && warp >= 2) {
    const float* D = reinterpret_cast<const float*>(smem + S::DOT);
    float y = ((D[row] + D[128 + row]) + D[256 + row]) + D[384 + row];   // rank order
    y += p.b4 ? __ldg(p.b4) : 0.0f;
    const bool owner = grow < p.M;
    int32_t nh = 0;
    if (owner) {
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
      fence_acq_rel_gpu();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (te == 0) {
        TAIL2_TS(6);
        *s_last = (atomicAdd(p.done, 1) == (int)gridDim.y - 1) ? 1 : 0;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*s_last) {
        fence_acq_rel_gpu();
        // the ring, RECV and DOT are idle: reuse the small-batch kernel's finalize on this layout
        const int nb = p.pa.n_inst * (p.pa.H + 2);
        uint32_t* sbeta = reinterpret_cast<uint32_t*>(smem + S::CBETA);   // prefetched
        if (p.pa.H + 1 > S::CBETA_MAX) {
          sbeta = reinterpret_cast<uint32_t*>(smem + S::W3);   // W3 consumed by the layer-3 MMA
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
        if (te == 0) {
          *p.pa.ws_arrive = 0;
          *p.done = 0;
          TAIL2_TS(7);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

}  // namespace star
