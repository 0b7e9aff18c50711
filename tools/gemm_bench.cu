// gemm_bench.cu -- microbenchmark (development tool): the predictor's layer-1 GEMM kernels in
// isolation, N back-to-back launches timed with CUDA events (per-launch cost incl. launch
// overhead amortised), warm L2 and with an L2 flush before the batch.  Compares the CTA-pair
// kernel and the 1-CTA split-K kernel on the same shapes; checks one output tile against the
// pair kernel for sanity.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2510_13668_b200/csrc
//        -I../include gemm_bench.cu -o gemm_bench -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "lenpred_kernels.cuh"

using namespace star;

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

template <typename F>
static float time_batch(F launch, int n, void* flush, size_t fb) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) launch();
  if (fb) cudaMemsetAsync(flush, 1, fb);
  cudaEventRecord(e0);
  for (int i = 0; i < n; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / n;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 2048, K = argc > 2 ? atoi(argv[2]) : 4096, N = 2048;
  const int nrep = 20;
  void *A, *B, *C, *flush;
  const size_t fb = 256ull << 20;
  cudaMalloc(&A, (size_t)M * K * 2);
  cudaMalloc(&B, (size_t)N * K * 2);
  cudaMalloc(&C, (size_t)M * N * 2);
  cudaMalloc(&flush, fb);
  std::vector<uint16_t> h((size_t)std::max(M, N) * K);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 0x3c00 + (uint16_t)(i % 7);   // small bf16 values
  cudaMemcpy(A, h.data(), (size_t)M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), (size_t)N * K * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA = make(A, K, M, 128), tB256 = make(B, K, N, 256), tB128 = make(B, K, N, 128), tC = make(C, N, M, 32);
  const double flop = 2.0 * M * N * K;
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.num_kb = K / 64;
  g.kb_per_split = K / 64;
  g.splits = 1;
  g.epi = EPI_RELU_BF16;
  g.tma_store = 1;
  g.out = C;
  g.ld_out = N;
  const int m_tiles = (M + 127) / 128;
  // ---- CTA-pair kernel ----
  cudaFuncSetAttribute(umma_pair_gemm_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)PairSmem<256>::BYTES);
  cudaFuncSetAttribute(umma_pair_gemm_kernel<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)PairSmem<256>::BYTES);
  auto pair = [&]() {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((m_tiles + 1) & ~1, N / 256, 1);
    cfg.blockDim = dim3(192, 1, 1);
    cfg.dynamicSmemBytes = PairSmem<256>::BYTES;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, umma_pair_gemm_kernel<256>, tA, tB128, tC, g);
  };
  // ---- 1-CTA kernel (no split) ----
  cudaFuncSetAttribute(umma_gemm_kernel<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)GemmSmem<256>::BYTES);
  auto single = [&]() {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(m_tiles, N / 256, 1);
    cfg.blockDim = dim3(192, 1, 1);
    cfg.dynamicSmemBytes = GemmSmem<256>::BYTES;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, umma_gemm_kernel<256, false>, tA, tB256, tC, g);
  };
  // ---- 1-CTA kernel with cluster split-K ----
  std::vector<float> ws_buf;
  float* ws;
  cudaMalloc(&ws, (size_t)148 * 128 * 256 * 4);
  for (int S : {2, 4, 8}) {
    GemmArgs gs = g;
    gs.splits = S;
    gs.kb_per_split = (K / 64 + S - 1) / S;
    gs.ws = ws;
    gs.tma_store = (256 / S) % 64 == 0;
    if (m_tiles * (N / 256) * S > 148) continue;
    auto split = [&]() {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(m_tiles, N / 256, S);
      cfg.blockDim = dim3(192, 1, 1);
      cfg.dynamicSmemBytes = GemmSmem<256>::BYTES;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 1;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = S;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      cudaLaunchKernelEx(&cfg, umma_gemm_kernel<256, false>, tA, tB256, tC, gs);
    };
    const float w = time_batch(split, nrep, flush, 0), c = time_batch(split, 1, flush, fb);
    printf("M=%d K=%d N=%d  1-CTA split %d: %.2f us warm (%.0f TF/s), %.2f us cold\n", M, K, N, S, w, flop / w / 1e6, c);
  }
  // ---- CTA-pair kernel with split-K (arrival counters in global memory) ----
  int* cnt;
  cudaMalloc(&cnt, 4096 * sizeof(int));
  cudaMemset(cnt, 0, 4096 * sizeof(int));
  for (int S : {2, 4, 8}) {
    const int pairs = ((m_tiles + 1) / 2) * (N / 256);
    if (pairs * S > 74 || (K / 64) / S < 2) continue;
    GemmArgs gs = g;
    gs.splits = S;
    gs.kb_per_split = (K / 64 + S - 1) / S;
    gs.ws = ws;
    gs.l1_cnt = cnt;
    auto psplit = [&]() {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((m_tiles + 1) & ~1, N / 256, S);
      cfg.blockDim = dim3(192, 1, 1);
      cfg.dynamicSmemBytes = PairSmem<256>::BYTES;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      cudaLaunchKernelEx(&cfg, umma_pair_gemm_kernel<256, true>, tA, tB128, tC, gs);
    };
    const float w = time_batch(psplit, nrep, flush, 0), c = time_batch(psplit, 1, flush, fb);
    printf("M=%d K=%d N=%d  pair split %d: %.2f us warm (%.0f TF/s), %.2f us cold  [%s]\n", M, K, N, S, w,
           flop / w / 1e6, c, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  for (int pf : {0, 1, 2}) {
    g.prefetch = pf;
    const float w = time_batch(pair, nrep, flush, 0), c = time_batch(pair, 1, flush, fb);
    printf("M=%d K=%d N=%d  pair prefetch=%d: %.2f us warm (%.0f TF/s), %.2f us cold\n", M, K, N, pf, w,
           flop / w / 1e6, c);
  }
  g.prefetch = 2;
  float tp_w = time_batch(pair, nrep, flush, 0), tp_c = time_batch(pair, 1, flush, fb);
  float ts_w = time_batch(single, nrep, flush, 0), ts_c = time_batch(single, 1, flush, fb);
  printf("M=%d K=%d N=%d  pair: %.2f us warm (%.0f TF/s), %.2f us cold   1-CTA: %.2f us warm (%.0f TF/s), %.2f us cold\n",
         M, K, N, tp_w, flop / tp_w / 1e6, tp_c, ts_w, flop / ts_w / 1e6, ts_c);
  return 0;
}
