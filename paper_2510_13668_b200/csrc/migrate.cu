// migrate.cu -- ExecuteMigration's data movement (NEXT-4; Alg. 1 line 10 "ExecuteMigration(m*)",
// PAPER.md:418; §5.4 "the paused request's KV cache is transferred to the target instance without
// blocking the execution of other requests"; transfer cost vs bandwidth,
// PAPER.md:631, Fig. 9).
//
// A paged KV pool (vLLM-style) is [n_layers][n_blocks][block_bytes] with a byte stride between
// layers; a request owns the blocks its block table lists.  Moving request r from instance s to
// instance t copies, for every layer, each of its blocks from s's pool into the blocks t
// allocated for it.  Three forms, one kernel:
//   kv_pack     pool --(table)--> contiguous staging [n_layers][n][block_bytes]
//   kv_unpack   staging --(table)--> pool
//   kv_migrate  pool_s --(table_s, table_t)--> pool_t directly (no staging).  With peer access
//               enabled the source pool may live on another GPU: the kernel, launched on the
//               destination GPU, pulls the blocks over NVLink (one kernel, no per-block copies).
// The copy is HBM-bound: 16-byte vector loads (read-only, no L1 allocation) and streaming
// stores, 64 bytes per thread in flight, several CTAs per SM, one (layer, block) item per CTA
// iteration so the block-table lookup is amortised over block_bytes.
#include <cuda_runtime.h>

#include <cstdint>

#include "star_internal.h"

namespace star {
namespace {

constexpr int kCopyThreads = 512;
constexpr int kUnroll = 4;   // 16-byte vectors per thread per iteration

struct CopyArgs {
  const uint8_t* src;
  int64_t src_layer_stride;
  int64_t src_nblocks;
  const int32_t* src_table;   // nullptr: identity (staging)
  uint8_t* dst;
  int64_t dst_layer_stride;
  int64_t dst_nblocks;
  const int32_t* dst_table;   // nullptr: identity (staging)
  int n_layers;
  int n;                      // blocks of the request
  int64_t block_bytes;        // multiple of 16
  int32_t* err_flag;
};

__device__ __forceinline__ int4 ld_nc_v4(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cs_v4(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(kCopyThreads) kv_copy_kernel(CopyArgs a) {
  const int64_t items = (int64_t)a.n_layers * a.n;
  const int64_t vecs = a.block_bytes >> 4;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int layer = (int)(it / a.n);
    const int j = (int)(it - (int64_t)layer * a.n);
    const int64_t sb = a.src_table ? (int64_t)__ldg(a.src_table + j) : j;
    const int64_t db = a.dst_table ? (int64_t)__ldg(a.dst_table + j) : j;
    if (sb < 0 || sb >= a.src_nblocks || db < 0 || db >= a.dst_nblocks) {   // CTA-uniform
      if (threadIdx.x == 0 && a.err_flag) atomicOr(a.err_flag, STAR_ERRF_BLOCK);
      continue;
    }
    const int4* s = reinterpret_cast<const int4*>(a.src + layer * a.src_layer_stride + sb * a.block_bytes);
    int4* d = reinterpret_cast<int4*>(a.dst + layer * a.dst_layer_stride + db * a.block_bytes);
    int64_t v = threadIdx.x;
    for (; v + (kUnroll - 1) * kCopyThreads < vecs; v += kUnroll * kCopyThreads) {
      int4 r[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) r[u] = ld_nc_v4(s + v + u * kCopyThreads);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) st_cs_v4(d + v + u * kCopyThreads, r[u]);
    }
    for (; v < vecs; v += kCopyThreads) st_cs_v4(d + v, ld_nc_v4(s + v));
  }
}

star_status validate_pool(const star_kv_pool* p, const char* what, std::string* msg) {
  if (!p || !p->base || p->n_layers <= 0 || p->n_blocks <= 0 || p->block_bytes <= 0 || (p->block_bytes & 15) ||
      (p->layer_stride & 15) || (reinterpret_cast<uintptr_t>(p->base) & 15) ||
      p->layer_stride < p->n_blocks * p->block_bytes) {
    *msg = std::string(what) + ": pool needs a 16-byte aligned base, block_bytes and layer_stride multiples of 16, "
                               "n_layers, n_blocks > 0 and layer_stride >= n_blocks * block_bytes";
    return STAR_EINVAL;
  }
  return STAR_OK;
}

cudaError_t launch_copy(const CopyArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  const int64_t items = (int64_t)a.n_layers * a.n;
  // 4 CTAs of 512 threads per SM (64 B in flight per thread: 128 KB per SM), capped by the items
  int64_t grid = (int64_t)g_num_sms * 4;
  if (grid > items) grid = items;
  kv_copy_kernel<<<(unsigned)grid, kCopyThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

star_status kv_copy_checked(const star_kv_pool* src, const int32_t* src_table, const star_kv_pool* dst,
                            const int32_t* dst_table, int n, void* staging_in, void* staging_out, int32_t* err_flag,
                            cudaStream_t stream, std::string* msg) {
  if (n < 0) {
    *msg = "n_blocks must be >= 0";
    return STAR_EINVAL;
  }
  const star_kv_pool* ref = src ? src : dst;
  star_status s = validate_pool(ref, src ? "src" : "dst", msg);
  if (s != STAR_OK) return s;
  if (src && dst) {
    if ((s = validate_pool(dst, "dst", msg)) != STAR_OK) return s;
    if (src->n_layers != dst->n_layers || src->block_bytes != dst->block_bytes) {
      *msg = "kv_migrate: source and destination pools differ in n_layers or block_bytes";
      return STAR_EINVAL;
    }
  }
  if (n > 0 && ((src && !src_table) || (dst && !dst_table))) {
    *msg = "block table is NULL";
    return STAR_EINVAL;
  }
  if (n == 0) return STAR_OK;   // nothing to copy (staging may be an empty allocation)
  void* stg = staging_in ? staging_in : staging_out;
  if (!(src && dst) && (!stg || (reinterpret_cast<uintptr_t>(stg) & 15))) {
    *msg = "staging must be a 16-byte aligned device buffer of n_layers * n * block_bytes bytes";
    return STAR_EINVAL;
  }
  CopyArgs a{};
  a.n_layers = ref->n_layers;
  a.n = n;
  a.block_bytes = ref->block_bytes;
  a.err_flag = err_flag;
  const int64_t stg_stride = (int64_t)n * ref->block_bytes;
  if (src) {
    a.src = static_cast<const uint8_t*>(src->base);
    a.src_layer_stride = src->layer_stride;
    a.src_nblocks = src->n_blocks;
    a.src_table = src_table;
  } else {
    a.src = static_cast<const uint8_t*>(staging_in);
    a.src_layer_stride = stg_stride;
    a.src_nblocks = n;
    a.src_table = nullptr;
  }
  if (dst) {
    a.dst = static_cast<uint8_t*>(dst->base);
    a.dst_layer_stride = dst->layer_stride;
    a.dst_nblocks = dst->n_blocks;
    a.dst_table = dst_table;
  } else {
    a.dst = static_cast<uint8_t*>(staging_out);
    a.dst_layer_stride = stg_stride;
    a.dst_nblocks = n;
    a.dst_table = nullptr;
  }
  cudaError_t e = launch_copy(a, stream);
  if (e != cudaSuccess) {
    *msg = std::string("kv copy launch: ") + cudaGetErrorString(e);
    return STAR_ECUDA;
  }
  return STAR_OK;
}

}  // namespace star
