// star_internal.h -- declarations shared by the product's CUDA translation units.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>
#include "../../include/star.h"
#include "project_core.cuh"

namespace star {

constexpr int kMaxSmemBytes = 227 * 1024;
extern int g_num_sms;   // set once by ensure_device()

// Function attributes belong to each device's context: set them per (device, kernel, attribute),
// under a lock.  cudaFuncAttributeMaxDynamicSharedMemorySize is raised to at least `value`;
// any other attribute is set to `value` once.  (star_api.cu)
cudaError_t func_attr(const void* func, cudaFuncAttribute attr, int value);

// project.cu
size_t project_workspace_bytes(int n_inst, int H);
int project_single_cta_max_rows();
cudaError_t launch_project(int R, int n_inst, int inst_base, int H, const int32_t* inst, const int32_t* n_tok,
                           const int32_t* n_hat, const uint32_t* beta_q, int64_t* L, int64_t* W, int64_t* peak,
                           int64_t* growth, int32_t* count, void* workspace, int32_t* err_flag,
                           cudaStream_t stream, int* grid_out);

ProjArgs make_proj_args(int R, int n_inst, int inst_base, int H, const int32_t* inst, const int32_t* n_tok,
                        const int32_t* n_hat, const uint32_t* beta_q, int64_t* L, int64_t* W, int64_t* peak,
                        int64_t* growth, int32_t* count, void* workspace, int32_t* err_flag);

// plan.cu
size_t plan_smem_bytes(int n, int H, int world, int r_cap);
cudaError_t launch_plan(const star_plan_params* p, const star_plan_segments* sg, star_move* moves, int32_t* n_moves,
                        int32_t* err_flag, cudaStream_t stream);

cudaError_t plan_timeline(uint64_t* host64);

// plan_large.cu (multi-CTA plan over a global workspace)
struct PlanArgs;
PlanArgs make_plan_args(const star_plan_params* p, const star_plan_segments* sg, star_move* moves, int32_t* n_moves,
                        int32_t* err_flag);
size_t plan_large_workspace_bytes(int n, int H, int64_t slots);
bool plan_large_supported(int n);
cudaError_t launch_plan_large(const PlanArgs& a, void* workspace, cudaStream_t stream);

// refresh.cu (prediction cadence k)
cudaError_t launch_refresh_select(int R, const int32_t* gen, const int32_t* g_last, int32_t k, const int32_t* n_tok,
                                  int32_t* idx, int32_t* ntok_c, int32_t* pos, int32_t* M_out, cudaStream_t st);
cudaError_t launch_refresh_gather(int R, const void* h, int64_t ld_bytes, int row_bytes, const int32_t* idx,
                                  const int32_t* M_dev, void* hc, cudaStream_t st);
cudaError_t launch_refresh_scatter(int R, const int32_t* pos, const int32_t* nhat_c, const int32_t* gen,
                                   int32_t* g_last, int32_t* nhat_last, int32_t* n_hat, const int32_t* M_dev,
                                   int32_t* n_refreshed, cudaStream_t st);
struct ProjArgs;
// multi-CTA select + gather + aging (+ projection of the aged rows) for the one-launch predictor
cudaError_t launch_refresh_select_fused(int R, const int32_t* gen, const int32_t* g_last, const int32_t* nhat_last,
                                        int32_t k, const int32_t* n_tok, const void* h, int64_t ld_bytes, int row_bytes,
                                        int32_t* idx, int32_t* ntok_c, void* hc, int32_t* n_hat, int32_t* M_out,
                                        int32_t* n_refreshed, int* blk, const ProjArgs* proj, cudaStream_t st,
                                        uint64_t* tl = nullptr);
int refresh_select_fused_max_rows();
size_t refresh_scatter_project_smem(int n_inst, int H);
cudaError_t launch_refresh_scatter_project(const ProjArgs& a, const int32_t* pos, const int32_t* nhat_c,
                                           const int32_t* gen, int32_t* g_last, int32_t* nhat_last,
                                           const int32_t* M_dev, int32_t* n_refreshed, cudaStream_t st);

// migrate.cu (KV migration, NEXT-4): src/dst NULL select the staging side
star_status kv_copy_checked(const star_kv_pool* src, const int32_t* src_table, const star_kv_pool* dst,
                            const int32_t* dst_table, int n, void* staging_in, void* staging_out, int32_t* err_flag,
                            cudaStream_t stream, std::string* msg);

// dispatch.cu
size_t dispatch_workspace_bytes(int n, int H);
cudaError_t launch_dispatch(int policy, int n, int H, const uint32_t* beta_q, int64_t* L, const int64_t* c_mem,
                            const int64_t* reserved, int A, const int32_t* n_tok, const int32_t* n_hat,
                            int32_t counter, int32_t* assign, void* workspace, cudaStream_t stream);

}  // namespace star
