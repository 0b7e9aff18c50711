// gather4_check.cu -- does `cp.async.bulk.tensor.2d ... tile::gather4` land 4 arbitrary rows of a
// SW128 K-major bf16 map at consecutive 128-byte rows of a 1024-aligned tile, swizzled by smem
// address like a plain 2D box?  (development tool; prints OK / the first mismatch)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_2510_13668_b200/csrc gather4_check.cu -o g4 -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"
using namespace star;

__global__ void k(const __grid_constant__ CUtensorMap tm, const int* rows, int kblk, uint16_t* out) {
  __shared__ __align__(1024) uint8_t buf[16384];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, 16384u);
  __syncwarp();
  if (threadIdx.x < 32) {   // lane j gathers rows 4j..4j+3 of the 128-row tile
    const int j = threadIdx.x;
    const uint32_t d = smem_u32(buf + 512 * j);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar)), "r"(kblk * 64), "r"(rows[4 * j]), "r"(rows[4 * j + 1]),
        "r"(rows[4 * j + 2]), "r"(rows[4 * j + 3])
        : "memory");
  }
  mbar_wait(&bar, 0);
  // unswizzle: element (r, c) of the tile sits at r*128 + ((c/8) ^ (r&7))*16 + (c%8)*2
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    const int r = e / 64, c = e % 64;
    out[e] = *reinterpret_cast<const uint16_t*>(buf + r * 128 + (((c / 8) ^ (r & 7)) << 4) + (c % 8) * 2);
  }
}

int main() {
  const int R = 1000, D = 512;
  std::vector<uint16_t> h((size_t)R * D);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 16);
  uint16_t* dh;
  cudaMalloc(&dh, h.size() * 2);
  cudaMemcpy(dh, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dh, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box {64,1}: %d\n", (int)cr);
  std::vector<int> rows(128);
  for (int i = 0; i < 128; ++i) rows[i] = (i * 37 + 11) % R;
  rows[127] = R + 5;   // out of range: zero fill expected
  int* drows;
  cudaMalloc(&drows, 128 * 4);
  cudaMemcpy(drows, rows.data(), 128 * 4, cudaMemcpyHostToDevice);
  uint16_t* dout;
  cudaMalloc(&dout, 128 * 64 * 2);
  const int kblk = 3;
  k<<<1, 128>>>(tm, drows, kblk, dout);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> out(128 * 64);
  cudaMemcpy(out.data(), dout, out.size() * 2, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128 && bad < 5; ++r)
    for (int c = 0; c < 64; ++c) {
      const uint16_t want = rows[r] < R ? h[(size_t)rows[r] * D + kblk * 64 + c] : 0;
      if (out[r * 64 + c] != want) {
        if (bad < 5) printf("mismatch r=%d c=%d got %u want %u\n", r, c, out[r * 64 + c], want);
        ++bad;
        break;
      }
    }
  printf(bad ? "FAIL\n" : "OK\n");
  return 0;
}
