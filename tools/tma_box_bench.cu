// tma_box_bench.cu -- microbenchmark (development tool): does the per-SM TMA ingest rate depend on
// the size of each TMA operation?  Each CTA streams K blocks of A (128 rows) and B (128 rows) of
// a bf16 GEMM-like operand pair through an mbarrier ring (no MMA), either as one 2D box per
// operand and 64-wide K block (16 KB per TMA op) or as one 3D box per operand covering KB
// consecutive K blocks ({64, 128 rows, KB}: KB x 16 KB per op, landing as KB consecutive SW128
// tiles -- the layout the UMMA descriptors expect), at the same bytes in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2510_13668_b200/csrc
//        tma_box_bench.cu -o tma_box_bench -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cuda_bf16.h>
#include "ptx.cuh"

using namespace star;

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// KB = K blocks per TMA op (1: 2D boxes); STAGES ring slots of KB K blocks each
template <int STAGES, int KB>
__global__ void __launch_bounds__(64, 1) box_kernel(const __grid_constant__ CUtensorMap ta,
                                                    const __grid_constant__ CUtensorMap tb, int nkb) {
  constexpr uint32_t OP = KB * 16384u, SB = 2 * OP;
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
  // GEMM-like reuse: 16 m-tiles x 8 n-tiles
  const int arow = (blockIdx.x % 16) * 128, brow = (blockIdx.x / 16) * 128;
  const int nit = nkb / KB;
  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nit; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((uint32_t)(i / STAGES) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], SB);
        if (KB == 1) {
          tma_load_2d(smem + s * SB, &ta, &full[s], i * 64, arow, 0);
          tma_load_2d(smem + s * SB + OP, &tb, &full[s], i * 64, brow, 0);
        } else {
          tma_load_3d(smem + s * SB, &ta, &full[s], 0, arow, i * KB);
          tma_load_3d(smem + s * SB + OP, &tb, &full[s], 0, brow, i * KB);
        }
      }
    }
  } else {
    if (elect_one()) {
      for (int i = 0; i < nit; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (uint32_t)(i / STAGES) & 1u);
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

static CUtensorMap make2(void* base, uint64_t K, uint64_t rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {K * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("make2 failed %d\n", (int)r);
  return m;
}
// dims {64 (K within a block), rows, K blocks}: strides rows = K*2 bytes, K blocks = 128 bytes
static CUtensorMap make3(void* base, uint64_t K, uint64_t rows, uint32_t kb) {
  CUtensorMap m;
  cuuint64_t dims[3] = {64, rows, K / 64};
  cuuint64_t strides[2] = {K * 2, 128};
  cuuint32_t box[3] = {64, 128, kb};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("make3(kb=%u) failed %d\n", kb, (int)r);
  return m;
}

template <int STAGES, int KB>
static void run(const CUtensorMap& ta, const CUtensorMap& tb, int grid, int nkb, void* flush, size_t flush_bytes) {
  constexpr uint32_t SB = 2 * KB * 16384u;
  const int smem = 1024 + STAGES * SB + 256;
  cudaFuncSetAttribute(box_kernel<STAGES, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    if (flush_bytes) cudaMemsetAsync(flush, rep, flush_bytes);
    cudaEventRecord(e0);
    box_kernel<STAGES, KB><<<grid, 64, smem>>>(ta, tb, nkb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double bytes_cta = (double)nkb * 32768.0;
  const double clk = best * 1e-3 * 1.965e9;
  printf("stages %d  KB/op %d (%3u KB per TMA op, %3u KB in flight)  grid %3d  %s: %8.2f us  per-SM %6.1f B/clk  "
         "chip %6.2f TB/s\n",
         STAGES, KB, KB * 16, STAGES * SB / 1024, grid, flush_bytes ? "cold" : "warm", best * 1e3, bytes_cta / clk,
         bytes_cta * grid / (best * 1e-3) / 1e12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
}


// A through the TMA unit, B through the LSU (cp.async 16-byte, .cg) by 4 warps writing the same
// SW128 layout (chunk c of row r at c ^ (r & 7)); cp.async.mbarrier.arrive.noinc tracks them.
template <int STAGES>
__global__ void __launch_bounds__(192, 1) mixed_kernel(const __grid_constant__ CUtensorMap ta,
                                                       const __nv_bfloat16* __restrict__ B, int K, int nkb) {
  constexpr uint32_t OP = 16384u, SB = 2 * OP;
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SB);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1 + 128);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int arow = (blockIdx.x % 16) * 128, brow = (blockIdx.x / 16) * 128;
  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((uint32_t)(i / STAGES) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], OP);
        tma_load_2d(smem + s * SB, &ta, &full[s], i * 64, arow, 0);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (uint32_t)(i / STAGES) & 1u);
        mbar_arrive(&empty[s]);
      }
    }
  } else {
    const int t = threadIdx.x - 64;   // 128 loader threads: 1024 chunks of 16 B per stage, 8 each
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&empty[s], ((uint32_t)(i / STAGES) & 1u) ^ 1u);
      uint8_t* dst = smem + s * SB + OP;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = t + 128 * j, r = c >> 3, ch = c & 7;
        const __nv_bfloat16* src = B + (size_t)(brow + r) * K + i * 64 + ch * 8;
        const uint32_t d = smem_u32(dst + r * 128 + ((ch ^ (r & 7)) << 4));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
  }
  __syncthreads();
}

template <int STAGES>
static void run_mixed(const CUtensorMap& ta, const __nv_bfloat16* B, int K, int grid, int nkb, void* flush,
                      size_t flush_bytes) {
  constexpr uint32_t SB = 2 * 16384u;
  const int smem = 1024 + STAGES * SB + 256;
  cudaFuncSetAttribute(mixed_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    if (flush_bytes) cudaMemsetAsync(flush, rep, flush_bytes);
    cudaEventRecord(e0);
    mixed_kernel<STAGES><<<grid, 192, smem>>>(ta, B, K, nkb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double bytes_cta = (double)nkb * 32768.0;
  const double clk = best * 1e-3 * 1.965e9;
  printf("MIXED stages %d (A TMA 16 KB + B cp.async 16 KB)  grid %3d  %s: %8.2f us  per-SM %6.1f B/clk  chip %6.2f TB/s\n",
         STAGES, grid, flush_bytes ? "cold" : "warm", best * 1e3, bytes_cta / clk, bytes_cta * grid / (best * 1e-3) / 1e12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
}

// in-flight sweep: one 16 KB A box per stage, STAGES deep
template <int STAGES>
__global__ void __launch_bounds__(64, 1) depth_kernel(const __grid_constant__ CUtensorMap ta, int nkb) {
  constexpr uint32_t SB = 16384u;
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
  const int arow = (blockIdx.x % 16) * 128;
  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((uint32_t)(i / STAGES) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], SB);
        tma_load_2d(smem + s * SB, &ta, &full[s], (i % 128) * 64, arow, 0);
      }
    }
  } else {
    if (elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (uint32_t)(i / STAGES) & 1u);
        mbar_arrive(&empty[s]);
      }
    }
  }
  __syncthreads();
}
template <int STAGES>
static void run_depth(const CUtensorMap& ta, int grid, int nkb, void* flush, size_t flush_bytes) {
  const int smem = 1024 + STAGES * 16384 + 256;
  cudaFuncSetAttribute(depth_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    if (flush_bytes) cudaMemsetAsync(flush, rep, flush_bytes);
    cudaEventRecord(e0);
    depth_kernel<STAGES><<<grid, 64, smem>>>(ta, nkb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const double bytes_cta = (double)nkb * 16384.0;
  const double clk = best * 1e-3 * 1.965e9;
  printf("DEPTH %2d x 16 KB in flight (%3d KB)  grid %3d  %s: %8.2f us  per-SM %6.1f B/clk\n", STAGES, STAGES * 16, grid,
         flush_bytes ? "cold" : "warm", best * 1e3, bytes_cta / clk);
}

int main() {
  const int K = 8192;   // 128 K blocks of 64 bf16
  const int rows = 16 * 128;
  void *A, *B, *flush;
  const size_t flush_bytes = 256ull << 20;
  cudaMalloc(&A, (size_t)rows * K * 2);
  cudaMalloc(&B, (size_t)rows * K * 2);
  cudaMalloc(&flush, flush_bytes);
  cudaMemset(A, 0, (size_t)rows * K * 2);
  cudaMemset(B, 0, (size_t)rows * K * 2);
  const CUtensorMap a2 = make2(A, K, rows), b2 = make2(B, K, rows);
  const CUtensorMap a3 = make3(A, K, rows, 2), b3 = make3(B, K, rows, 2);
  for (size_t fb : {flush_bytes, (size_t)0}) {
    run_depth<2>(a2, 128, 128, flush, fb);
    run_depth<4>(a2, 128, 128, flush, fb);
    run_depth<6>(a2, 128, 128, flush, fb);
    run_depth<8>(a2, 128, 128, flush, fb);
    run_depth<10>(a2, 128, 128, flush, fb);
    run_depth<12>(a2, 128, 128, flush, fb);
    run<6, 1>(a2, b2, 128, 64, flush, fb);
  }
  return 0;
}
