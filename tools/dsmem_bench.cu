// DSMEM throughput microbenchmark (development): a cluster of 4 CTAs, each moves 96 KB of fp32
// partials to its 3 partners (32 KB each) by (0) bulk copy shared::cta -> shared::cluster,
// (1) ld.shared::cluster pulls by 128 threads (16-byte), (2) st.shared::cluster pushes from
// registers (16-byte).  Prints cycles per CTA (median over CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_bench tools/dsmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
template <int CL>
__global__ void __launch_bounds__(128, 1) k(int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* send = sm;            // [3][32K]
  uint8_t* recv = sm + 98304;    // [3][32K]
  uint64_t* bar = (uint64_t*)(sm + 196608);
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 98304 / 4; i += 128) ((float*)send)[i] = i;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(32768u * (CL - 1)));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  csync();
  long long t0 = clock64();
  if (mode == 0) {
    if (threadIdx.x == 0) {
      for (uint32_t p = 0; p < CL; ++p) {
        if (p == rank) continue;
        uint32_t dst = mapa(su32(recv + 32768u * (rank - (rank > p))), p);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "r"(su32(send + 32768u * (p - (p > rank)))), "r"(32768u), "r"(mapa(su32(bar), p)) : "memory");
      }
    }
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0,1,0,P;\n}" : "=r"(ok) : "r"(su32(bar)) : "memory");
  } else if (mode == 1) {
    // pull: CTA reads the block each partner staged for it
    float acc = 0;
    for (uint32_t p = 0; p < CL; ++p) {
      if (p == rank) continue;
      uint32_t src = mapa(su32(send + 32768u * (rank - (rank > p))), p);
      #pragma unroll 4
      for (int i = threadIdx.x; i < 2048; i += 128) {
        float4 v; asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(src + 16u * i));
        acc += v.x + v.y + v.z + v.w;
      }
    }
    ((float*)recv)[threadIdx.x] = acc;
  } else {
    for (uint32_t p = 0; p < CL; ++p) {
      if (p == rank) continue;
      uint32_t dst = mapa(su32(recv + 32768u * (rank - (rank > p))), p);
      #pragma unroll 4
      for (int i = threadIdx.x; i < 2048; i += 128) {
        float4 v = ((float4*)(send + 32768u * (p - (p > rank))))[i];
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(dst + 16u * i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
      }
    }
    csync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  csync();
}
template <int CL>
void run() {
  int n = 128;
  long long* d; cudaMalloc(&d, n * sizeof(long long));
  cudaFuncSetAttribute(k<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[3] = {"bulk push", "ld.shared::cluster pull", "st.shared::cluster push"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(n); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 3; ++rep) cudaLaunchKernelEx(&cfg, k<CL>, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(n); cudaMemcpy(h.data(), d, n * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    printf("cluster %d %-26s %s median %lld cyc  max %lld cyc  (%d KB per CTA: %.1f B/clk)\n", CL, names[mode],
           cudaGetErrorString(e), h[n / 2], h[n - 1], 32 * (CL - 1), 32768.0 * (CL - 1) / h[n / 2]);
  }
}
int main() {
  run<2>();
  run<4>();
  return 0;
}
