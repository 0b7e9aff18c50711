// gtimer.cu -- calibrates %globaltimer against %clock64 and CUDA events (diagnostics).
#include <cstdio>
#include <cstdint>
__global__ void spin(unsigned long long cycles, unsigned long long* out) {
  unsigned long long g0, g1, c0 = clock64(), c1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  do { c1 = clock64(); } while (c1 - c0 < cycles);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = g1 - g0; out[1] = c1 - c0; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (unsigned long long cyc : {20000ull, 200000ull, 2000000ull}) {
    spin<<<1, 32>>>(cyc, d); cudaDeviceSynchronize();
    cudaEventRecord(e0); spin<<<148, 32>>>(cyc, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("cycles %llu: globaltimer %llu ns, event %.2f us, clock %.3f GHz (by globaltimer)\n", h[1], h[0], ms * 1e3,
           (double)h[1] / h[0]);
  }
}
