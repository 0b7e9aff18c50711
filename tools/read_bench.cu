// read_bench.cu -- HBM read ceiling on this B200 (development tool): one 192 MB array read by
// (1) grid-stride int4 loads, (2) per-CTA contiguous chunks of int4 loads, (3) cp.async.bulk
// rings of different depths; L2 flushed (256 MB write) before every timed run, median of 9.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 read_bench.cu -o read_bench
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
__device__ __forceinline__ int4 ldnc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int U>
__global__ void grid_stride(const int4* a, int64_t nvec, int* out) {
  int acc = 0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nvec; g += (int64_t)gridDim.x * blockDim.x * U) {
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = g + (int64_t)u * gridDim.x * blockDim.x;
      x[u] = k < nvec ? ldnc(a + k) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= x[u].x ^ x[u].w;
  }
  if (acc == 0x12345678) *out = acc;
}
__device__ __forceinline__ int4 ldnc256(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// per-CTA contiguous chunk, each thread U consecutive-by-blockDim int4 in flight
template <int U, bool HINT>
__global__ void chunked(const int4* a, int64_t nvec, int* out) {
  const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t beg = blockIdx.x * per, end = min(beg + per, nvec);
  int acc = 0;
  for (int64_t g = beg + threadIdx.x; g < end; g += (int64_t)blockDim.x * U) {
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = g + (int64_t)u * blockDim.x;
      x[u] = k < end ? (HINT ? ldnc256(a + k) : ldnc(a + k)) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= x[u].x ^ x[u].w;
  }
  if (acc == 0x12345678) *out = acc;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b)) : "memory");
}
// ring of S stages of B bytes; warp 0 lane 0 produces, (blockDim/32 - 1) consumer warps touch one int4 per lane
__global__ void bulk_ring(const int4* a, int64_t nvec, int* out, int S, int B) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * B);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nc = (blockDim.x >> 5) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nc); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t beg = blockIdx.x * per, end = min(beg + per, nvec);
  const int vps = B / 16;
  const int64_t nch = end > beg ? (end - beg + vps - 1) / vps : 0;
  int acc = 0;
  if (warp == 0) {
    if (lane == 0)
      for (int64_t c = 0; c < nch; ++c) {
        const int s = c % S; const uint32_t ph = (c / S) & 1;
        wait(&empty[s], ph ^ 1);
        const int64_t v0 = beg + c * vps;
        const int nv = (int)min((int64_t)vps, end - v0);
        expect_tx(&full[s], nv * 16);
        bulk(sm + (size_t)s * B, a + v0, nv * 16, &full[s]);
      }
  } else {
    for (int64_t c = 0; c < nch; ++c) {
      const int s = c % S; const uint32_t ph = (c / S) & 1;
      wait(&full[s], ph);
      const int4* st = reinterpret_cast<const int4*>(sm + (size_t)s * B);
      for (int j = (warp - 1) * 32 + lane; j < vps; j += nc * 32) acc ^= st[j].x;
      __syncwarp();
      if (lane == 0) arrive(&empty[s]);
    }
  }
  if (acc == 0x12345678) *out = acc;
}
template <typename F>
float timed(F f, void* fl) {
  std::vector<float> v;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 11; ++i) {
    cudaMemsetAsync(fl, i, 256 << 20);
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (i >= 2) v.push_back(ms);
  }
  std::sort(v.begin(), v.end());
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return v[v.size() / 2];
}
int main() {
  const int64_t bytes = 192ll << 20, nvec = bytes / 16;
  int4* a; int* out; void* fl;
  cudaMalloc(&a, bytes); cudaMalloc(&out, 4); cudaMalloc(&fl, 256 << 20);
  cudaMemset(a, 1, bytes);
  auto gb = [&](float ms) { return bytes / (ms * 1e-3) / 1e9; };
  if (0) for (int grid : {148, 296, 592, 1184})
    for (int blk : {256, 512, 1024}) {
      if ((int64_t)grid * blk > 600000) continue;
      float t4 = timed([&] { grid_stride<4><<<grid, blk>>>(a, nvec, out); }, fl);
      float t8 = timed([&] { grid_stride<8><<<grid, blk>>>(a, nvec, out); }, fl);
      printf("grid_stride grid %4d x %4d: U4 %.0f GB/s  U8 %.0f GB/s\n", grid, blk, gb(t4), gb(t8));
    }
  for (int cps : {1, 2, 4, 8})
    for (int blk : {256, 512, 1024}) {
      if (cps * blk > 2048) continue;
      const int grid = 148 * cps;
      float t8 = timed([&] { chunked<8, false><<<grid, blk>>>(a, nvec, out); }, fl);
      float t16 = timed([&] { chunked<16, false><<<grid, blk>>>(a, nvec, out); }, fl);
      float t8h = timed([&] { chunked<8, true><<<grid, blk>>>(a, nvec, out); }, fl);
      printf("chunked %d CTA/SM x %4d: U8 %.0f  U16 %.0f  U8+L2::256B %.0f GB/s\n", cps, blk, gb(t8), gb(t16), gb(t8h));
    }
  for (int ctas_per_sm : {1, 2, 3})
    for (int S : {3, 4})
      for (int B : {16384, 32768}) {
        const size_t smem = (size_t)S * B + 2 * S * 8;
        if (smem * ctas_per_sm > 220 * 1024) continue;
        cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int grid = 148 * ctas_per_sm;
        float t = timed([&] { bulk_ring<<<grid, 288, smem>>>(a, nvec, out, S, B); }, fl);
        printf("bulk_ring %d CTA/SM, %d stages x %5d B (%3zu KB/SM in flight): %.0f GB/s\n", ctas_per_sm, S, B,
               smem * ctas_per_sm / 1024, gb(t));
      }
  return 0;
}
