// stream_bench.cu -- what read bandwidth do 3 x 64 MB int4 streams reach with the projection
// kernel's access pattern (development tool)?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ int4 ldnc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int UNROLL>
__global__ void stream3(const int4* a, const int4* b, const int4* c, int64_t nvec, int* out, int chunked) {
  int acc = 0;
  if (chunked) {
    const int64_t chunk = (nvec + gridDim.x - 1) / gridDim.x;
    const int64_t beg = blockIdx.x * chunk, end = min(beg + chunk, nvec);
    for (int64_t g = beg + threadIdx.x; g < end; g += (int64_t)blockDim.x * UNROLL) {
      int4 x[UNROLL], y[UNROLL], z[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t k = g + (int64_t)u * blockDim.x;
        if (k < end) { x[u] = ldnc(a + k); y[u] = ldnc(b + k); z[u] = ldnc(c + k); } else { x[u] = y[u] = z[u] = make_int4(0,0,0,0); }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc += x[u].x ^ y[u].y ^ z[u].z ^ x[u].w;
    }
  } else {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nvec; g += (int64_t)gridDim.x * blockDim.x * UNROLL) {
      int4 x[UNROLL], y[UNROLL], z[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const int64_t k = g + (int64_t)u * gridDim.x * blockDim.x;
        if (k < nvec) { x[u] = ldnc(a + k); y[u] = ldnc(b + k); z[u] = ldnc(c + k); } else { x[u] = y[u] = z[u] = make_int4(0,0,0,0); }
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) acc += x[u].x ^ y[u].y ^ z[u].z ^ x[u].w;
    }
  }
  if (acc == 0x12345678) out[0] = acc;
}
template <int U>
void run(const int4* a, const int4* b, const int4* c, int64_t nvec, int* out, void* fl, int grid, int threads, int chunked) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaMemsetAsync(fl, r, 256 << 20);
    cudaEventRecord(e0);
    stream3<U><<<grid, threads>>>(a, b, c, nvec, out, chunked);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  printf("unroll %d grid %4d x %4d chunked %d: %.1f us  %.0f GB/s\n", U, grid, threads, chunked, best * 1e3, 3.0 * nvec * 16 / (best * 1e-3) / 1e9);
}
int main() {
  const int64_t n = 1 << 24, nvec = n / 4;
  int4 *a, *b, *c; int* out; void* fl;
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&c, n * 4); cudaMalloc(&out, 4); cudaMalloc(&fl, 256 << 20);
  cudaMemset(a, 1, n * 4); cudaMemset(b, 2, n * 4); cudaMemset(c, 3, n * 4);
  for (int ch = 0; ch <= 1; ++ch) {
    run<1>(a, b, c, nvec, out, fl, 148, 1024, ch);
    run<2>(a, b, c, nvec, out, fl, 148, 1024, ch);
    run<4>(a, b, c, nvec, out, fl, 148, 1024, ch);
    run<2>(a, b, c, nvec, out, fl, 296, 1024, ch);
    run<4>(a, b, c, nvec, out, fl, 592, 512, ch);
  }
}
