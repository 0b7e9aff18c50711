// tma_bench.cu -- microbenchmark (development tool): per-SM TMA ingest rate on B200.
// Each CTA streams `nkb` k-blocks of (A box 128 x 128B + B box BROWS x 128B) through an
// S-stage mbarrier ring (no MMA: the consumer warp just releases the slot), like the
// mainloop of the predictor GEMMs.  Reports bytes/clk per SM and chip TB/s for a sweep of
// grid sizes, stage counts and data reuse patterns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2510_13668_b200/csrc
//        tma_bench.cu -o tma_bench -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "ptx.cuh"

using namespace star;

template <int STAGES, int BROWS>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap ta,
                                                       const __grid_constant__ CUtensorMap tb, int nkb, int a_rows,
                                                       int b_rows, int share) {
  constexpr uint32_t AB = 128 * 128, BB = BROWS * 128, SB = AB + BB;
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // share = 0: every CTA reads its own rows; share = 1: all CTAs read the same rows (L2 hits);
  // share = 2: GEMM-like (16 m-tiles x 8 n-tiles: each A tile read by 8 CTAs, each B tile by 16)
  int arow = share ? 0 : (blockIdx.x * 128) % a_rows;
  int brow = share ? 0 : (blockIdx.x * BROWS) % b_rows;
  if (share == 2) {
    arow = (blockIdx.x % 16) * 128;
    brow = (blockIdx.x / 16) * BROWS;
  }
  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], SB);
        tma_load_2d(smem + s * SB, &ta, &full[s], i * 64, arow, 0);
        tma_load_2d(smem + s * SB + AB, &tb, &full[s], i * 64, brow, 0);
      }
    }
  } else {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
        mbar_wait(&full[s], ph);
        mbar_arrive(&empty[s]);
      }
    }
  }
  __syncthreads();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap make(void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

template <int STAGES, int BROWS>
static void run(const CUtensorMap& ta, const CUtensorMap& tb, int grid, int nkb, int a_rows, int b_rows, int share,
                void* flush, size_t flush_bytes) {
  constexpr uint32_t SB = 128 * 128 + BROWS * 128;
  const int smem = 1024 + STAGES * SB + 256;
  cudaFuncSetAttribute(stream_kernel<STAGES, BROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    if (flush_bytes) cudaMemsetAsync(flush, rep, flush_bytes);
    cudaEventRecord(e0);
    stream_kernel<STAGES, BROWS><<<grid, 64, smem>>>(ta, tb, nkb, a_rows, b_rows, share);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double bytes_cta = (double)nkb * SB;
  const double clk = best * 1e-3 * 1.965e9;
  printf("stages %d brows %3d grid %3d share %d nkb %3d : %8.2f us  per-SM %6.1f B/clk  chip %6.2f TB/s\n", STAGES,
         BROWS, grid, share, nkb, best * 1e3, bytes_cta / clk, bytes_cta * grid / (best * 1e-3) / 1e12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
}

int main() {
  const int K = 8192;                 // 128 k-blocks of 64 bf16
  const int a_rows = 148 * 128, b_rows = 148 * 256;
  void *A, *B, *flush;
  const size_t flush_bytes = 256ull << 20;
  cudaMalloc(&A, (size_t)a_rows * K * 2);
  cudaMalloc(&B, (size_t)b_rows * K * 2);
  cudaMalloc(&flush, flush_bytes);
  cudaMemset(A, 0, (size_t)a_rows * K * 2);
  cudaMemset(B, 0, (size_t)b_rows * K * 2);
  CUtensorMap ta = make(A, K, a_rows, 128), tb = make(B, K, b_rows, 256), tb128 = make(B, K, b_rows, 128);
  for (int grid : {64, 128}) {
    run<4, 256>(ta, tb, grid, 64, a_rows, b_rows, 2, flush, flush_bytes);
    run<6, 128>(ta, tb128, grid, 64, a_rows, b_rows, 2, flush, flush_bytes);
    run<4, 256>(ta, tb, grid, 64, a_rows, b_rows, 1, flush, flush_bytes);
    run<6, 128>(ta, tb128, grid, 64, a_rows, b_rows, 1, flush, flush_bytes);
  }
  // no flush: warm L2 (share 1: every CTA streams the same blocks, the most L2 reuse possible)
  for (int grid : {32, 64, 128, 148}) {
    run<6, 128>(ta, tb128, grid, 64, a_rows, b_rows, 2, flush, 0);
    run<6, 128>(ta, tb128, grid, 64, a_rows, b_rows, 1, flush, 0);
  }
  return 0;
}
