/*
 * star.h -- C ABI of the B200-native hot path of STAR (arxiv 2510.13668,
 * "Adaptive Rescheduling in Prefill-Decode Disaggregated LLM Inference").
 *
 * Per decode iteration, on every decode instance (one instance or a block of instances per
 * B200), the path is:
 *   lenpred_forward        Eq. 2: remaining-length prediction from each
 *                          running request's last-token, last-layer hidden state, quantized
 *                          to integer tokens N_hat (readings A8-A10).
 *   project_instance_load  worker-side local future-state simulation:
 *                          current token load N_i(B_i) and projected loads
 *                          N_hat_i(B_{i,t}), t = 1..H, w_i (Alg. 1 line 13).
 *   (NCCL all-gather of the per-rank records -- done by the caller)
 *   plan_reschedule        Alg. 1: InstanceClassification,
 *                          CandidateEnumeration, OptimalSelection over Eq. 3-4's objective,
 *                          exact integers, greedy rounds.
 *
 * Conventions (all entry points):
 *  - Return star_status: 0 = OK, < 0 = error.  No exception crosses the ABI.  On error
 *    star_last_error() returns a thread-local message valid until the next call on that
 *    thread; nothing was enqueued unless the error is STAR_ECUDA from the launch itself.
 *  - Array pointers are DEVICE pointers (cudaMalloc / torch CUDA memory) owned by the caller,
 *    unless stated otherwise.  The library never frees caller memory.
 *  - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream) and the call
 *    returns immediately; results are valid after the stream is synchronised.
 *  - Hot-path calls (lenpred_forward, project_instance_load, plan_reschedule*) do no
 *    allocation and no host synchronisation, so they can be captured in a CUDA graph.
 *  - Scalar arguments are validated on the host (STAR_EINVAL / STAR_ERANGE).  Per-element
 *    problems found on the device (instance id out of range, N(r) outside [1, 2^17],
 *    N_hat < 0, count overflow) set bits in *err_flag (device int32, nullable, never
 *    cleared by the library) and the offending element is ignored.
 *  - Only sm_100a (B200) is supported; every call fails with STAR_ENOTSUP elsewhere.  There
 *    is no CPU fallback.
 *  - A predictor (and a projection / plan workspace) holds scratch and arrival counters that
 *    one call uses at a time: calls on the same predictor must be ordered (one stream, or
 *    streams joined by events); distinct predictors are independent.
 *  - The one-launch kernels (small-batch bf16, fp32, refresh select, multi-CTA plans) hand
 *    phases off between CTAs through device counters and assume their grid is co-resident
 *    (checked with the occupancy API when the predictor is created); if other work holds the
 *    SMs (MPS partitions, green contexts) a wait traps after ~2 s (STAR_ECUDA on the next
 *    synchronisation) instead of hanging the device.
 */
#ifndef STAR_H_
#define STAR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* star_stream_t;   /* ABI-identical to cudaStream_t */

typedef enum {
  STAR_OK = 0,
  STAR_EINVAL = -1,   /* bad pointer / shape / flag combination */
  STAR_ERANGE = -2,   /* a size exceeds the exactness bounds documented below */
  STAR_ECUDA = -3,    /* CUDA runtime / driver error (message has the CUDA error string) */
  STAR_ENOTSUP = -4,  /* device is not sm_100 or the shape is outside what the kernels tile */
  STAR_ENOMEM = -5    /* allocation failed (create only) */
} star_status;

typedef enum { STAR_F32 = 0, STAR_BF16 = 1 } star_dtype;

/* err_flag bits (device side) */
#define STAR_ERRF_INST   1  /* instance id outside [inst_base, inst_base + n_inst) */
#define STAR_ERRF_NTOK   2  /* N(r) outside [1, 2^17] */
#define STAR_ERRF_NHAT   4  /* N_hat(r) < 0 */
#define STAR_ERRF_COUNT  8  /* more than 2^16 requests on one instance */
#define STAR_ERRF_PLAN   16 /* plan input inconsistent (segment count > capacity, etc.) */

const char* star_last_error(void);
/* Library version string, e.g. "star-b200 0.1 sm_100a". */
const char* star_version(void);

/* =====================================================================================
 * Length predictor  (Eq. 2)
 *     y_hat = w4 . phi(W3 phi(W2 phi(W1 h)))      phi = ReLU
 * d = hidden size (any multiple of 8), m1 = 2048, m2 = 512, m3 = 64 for the paper's model
 * (reading A2: the widths are fixed for every d).  Supported: m1, m2 multiples
 * of 256 (bf16) / 128 (f32), m3 == 64.
 * Precision: STAR_BF16 -> bf16 operands on tcgen05 kind::f16, fp32 accumulation in TMEM,
 * Z1/Z2 rounded to bf16; STAR_F32 -> fp32 operands via 3xTF32 (hi/lo split,
 * hi*hi + hi*lo + lo*hi, tcgen05 kind::tf32), fp32 accumulation, Z1/Z2 kept in fp32 (the
 * one-launch fp32 kernel for R <= 128 splits the activations into tensor memory and the
 * MMAs read A from there; its split-K sums run in a different order than the multi-launch
 * path's, so the two agree within the fp32 tolerance, not bit for bit).  Layer 4 and the
 * biases are fp32 on the CUDA cores.
 * ===================================================================================== */
typedef struct star_predictor star_predictor;  /* opaque: TMA descriptors, scratch Z1/Z2 */

/* Creates a predictor bound to caller-owned device weights (they must outlive the handle):
 *   W1 [m1][d], W2 [m2][m1], W3 [m3][m2] row-major in `dt` (nn.Linear [out][in] layout =
 *   K-major, the UMMA B operand as-is);  w4 [m3] fp32;  b1 [m1], b2 [m2], b3 [m3], b4 [1] fp32
 *   or NULL (NULL reproduces Eq. 2 literally, reading A1).
 * max_rows bounds R of later forward calls.  For STAR_F32 the weights are split into tf32
 * hi/lo copies here (library-owned: the multi-launch path's [hi|lo|hi] rows and, for m1 = 2048,
 * m2 = 512, d % 128 == 0, the one-launch kernel's hi / lo planes).  This is the only call that allocates device memory;
 * it synchronises `stream` before returning. */
star_status star_predictor_create(star_predictor** out, int d, int m1, int m2, int m3, star_dtype dt,
                                  const void* W1, const void* W2, const void* W3, const float* w4,
                                  const float* b1, const float* b2, const float* b3, const float* b4,
                                  int max_rows, star_stream_t stream);
star_status star_predictor_destroy(star_predictor* p);

/* Forward for R rows of h (row r at h + r*ld_h elements, dtype of the predictor, ld_h >= d,
 * ld_h*elem_size a multiple of 16 bytes).  Outputs (each nullable):
 *   y_hat [R] fp32      the regression output of Eq. 2
 *   n_hat [R] int32     N_hat = (int) rint(fminf(fmaxf(y_hat, 0), cap_r)),
 *                       cap_r = max(0, max_ctx_len - n_tok[r])   (n_tok NULL => cap = max_ctx_len)
 *                       round-half-to-even, NaN -> 0 (readings A8-A10; PAPER.md:491 32K context)
 * R = 0 is legal (nothing enqueued).  R <= max_rows.  Not thread-safe per handle. */
star_status lenpred_forward(star_predictor* p, const void* h, int64_t ld_h, int R,
                            const int32_t* n_tok, int32_t max_ctx_len,
                            float* y_hat, int32_t* n_hat, star_stream_t stream);

/* Forward fused with the projection of its own N_hat (the worker-side "predict, then simulate
 * the local future state" of PAPER.md:384): exactly lenpred_forward followed by
 * project_instance_load(R, n_inst, inst_base, H, inst, n_tok, n_hat, beta_q, ...), with the same
 * outputs bit for bit, but for bf16 predictors with m2 a multiple of 256 and m3 == 64 it runs as
 * TWO launches: the layer-1 GEMM and one fused tail kernel (layer 2 -> layer 3 -> w4 dot ->
 * quantizer -> keyed projection histogram -> last-CTA finalize), so Z2, Z3 and N_hat never
 * make a round trip through HBM before the projection.  Other predictors run the unfused
 * kernels.  n_hat (the N_hat output) must be non-NULL; n_tok and inst are required when R > 0;
 * workspace (star_project_workspace_bytes(n_inst, H) bytes, zero-filled once by the caller) is
 * required and is left zeroed.  R = 0 writes zero loads.  Argument meaning, layouts and
 * err_flag bits are those of lenpred_forward and project_instance_load below. */
star_status lenpred_forward_project(star_predictor* p, const void* h, int64_t ld_h, int R,
                                    const int32_t* n_tok, int32_t max_ctx_len, float* y_hat, int32_t* n_hat,
                                    int n_inst, int inst_base, int H, const int32_t* inst, const uint32_t* beta_q,
                                    int64_t* L, int64_t* W, int64_t* peak, int64_t* growth, int32_t* count,
                                    void* workspace, int32_t* err_flag, star_stream_t stream);

/* Prediction cadence k (NEXT-1): the paper predicts "at regular intervals" and
 * sets the interval to k = 20 decode iterations.  Per request slot r:
 *   gen[r]        tokens generated so far (device, in)
 *   g_last[r]     gen at the request's last prediction, -1 = never predicted (device, in/out)
 *   nhat_last[r]  that prediction (device, in/out)
 * Rows with g_last < 0 or gen - g_last >= k (SPEC.md:164-172 should_refresh) are re-predicted from
 * their hidden state exactly as lenpred_forward (Eq. 2 + quantizer with cap max_ctx_len - n_tok[r])
 * and get g_last = gen, nhat_last = N_hat; every other row ages (reading A27):
 *   N_hat = max(0, nhat_last - (gen - g_last)).
 * n_hat [R] (out) = this step's N_hat for every row; n_refreshed (device int32, nullable) = number of
 * rows re-predicted.  The selection, the gather of the selected rows and the predictor run on the
 * device (the row count never visits the host), so the call stays graph-capturable.  bf16
 * predictors with m2 % 256 == 0 and m3 == 64 only (STAR_ENOTSUP otherwise). */
star_status lenpred_forward_refresh(star_predictor* p, const void* h, int64_t ld_h, int R,
                                    const int32_t* n_tok, int32_t max_ctx_len, const int32_t* gen,
                                    int32_t* g_last, int32_t* nhat_last, int32_t k, int32_t* n_hat,
                                    int32_t* n_refreshed, star_stream_t stream);

/* lenpred_forward_refresh followed by project_instance_load(R, n_inst, inst_base, H, inst, n_tok,
 * n_hat, beta_q, L, W, peak, growth, count, workspace, err_flag) on the resulting N_hat -- the
 * cadence-k step of one worker -- with identical outputs bit for bit.  For
 * R <= 8192 and n_inst * (H + 2) bins that fit one CTA's shared memory, the aging scatter and the
 * projection run as ONE kernel (one CTA: shared-memory histogram, suffix-scan finalize; the
 * workspace is not touched); otherwise the two kernels follow each other.  Argument meaning,
 * layouts and errors: lenpred_forward_refresh and project_instance_load. */
star_status lenpred_forward_refresh_project(star_predictor* p, const void* h, int64_t ld_h, int R,
                                            const int32_t* n_tok, int32_t max_ctx_len, const int32_t* gen,
                                            int32_t* g_last, int32_t* nhat_last, int32_t k, int32_t* n_hat,
                                            int32_t* n_refreshed, int n_inst, int inst_base, int H,
                                            const int32_t* inst, const uint32_t* beta_q, int64_t* L, int64_t* W,
                                            int64_t* peak, int64_t* growth, int32_t* count, void* workspace,
                                            int32_t* err_flag, star_stream_t stream);

/* The quantizer alone, on a caller-given fp32 y_hat (the exact device function the forward
 * epilogue uses).  Lets quantizer parity be tested on identical fp32 inputs. */
star_status lenpred_quantize(const float* y_hat, const int32_t* n_tok, int R, int32_t max_ctx_len,
                             int32_t* n_hat, star_stream_t stream);

/* Optional per-handle timing of the dominant kernel: with enable != 0 the handle creates two
 * CUDA events and every later lenpred_forward records them around the layer-1 GEMM launch on
 * its stream (also inside a captured CUDA graph).  star_predictor_layer1_ms() returns the
 * elapsed milliseconds of the most recent completed forward (it synchronises on the end event). */
star_status star_predictor_layer1_timing(star_predictor* p, int enable);
/* Diagnostics: with enable != 0 every later fused-tail launch (see lenpred_forward_project)
 * records per-CTA %globaltimer stamps (ns) of its phases into a library-owned device buffer
 * [CTAs][16] (slot 15 = SM id).  With host_out != NULL the call synchronises the device and
 * copies the stamps of the most recent launch (at most max_ctas CTAs) to host_out, writing the
 * CTA count to *n_ctas; enable == 2 copies the layer-1 (CTA-pair GEMM) stamps instead.  enable == 0
 * frees the buffers.  Not for the hot path. */
star_status star_predictor_timeline(star_predictor* p, int enable, uint64_t* host_out, int max_ctas, int* n_ctas);
star_status star_predictor_layer1_ms(star_predictor* p, float* ms);
/* Which kernels a forward of R rows runs: *path = 1 for the one-launch small-batch predictor
 * (bf16, m1 = 2048, m2 = 512, d % 256 == 0, 1 <= R <= 512, and its 128 CTAs co-resident on this
 * device; the layer-1 timing events then bracket that whole launch), 2 for the one-launch fp32
 * predictor (fp32, m1 = 2048, m2 = 512, d % 128 == 0, 1 <= R <= 128, 128 CTAs co-resident; with a
 * fused projection only while n_inst * (H + 2) * 12 + (H + 1) * 4 bytes fit its shared memory,
 * ~156 KB, else the multi-launch path runs), 0 for the layer-1 GEMM + fused tail (bf16) or the
 * 3 GEMMs (fp32). */
star_status star_predictor_path(star_predictor* p, int R, int* path);

/* =====================================================================================
 * Projected per-instance load  (readings A4-A6)
 * For instance i in [0, n_inst) (request r belongs to i = inst[r] - inst_base):
 *   L[i][0] = sum_{r in B_i} N(r)                                 N(r) = n_tok[r] (prompt + generated)
 *   L[i][t] = sum_{r in B_i, t < N_hat(r)} (N(r) + t),  t = 1..H    (a request stays resident while
 *                                                                  t < N_hat, growing one token/step)
 *   W[i]    = sum_{t=1}^{H} beta_q[t] * L[i][t]                    (w_i of Alg. 1 line 13, Q16 units)
 *   peak[i] = max_{0<=t<=H} L[i][t]   growth[i] = sum min(N_hat, H)   count[i] = |B_i|
 * Exact int64 integers: bounds N(r) <= 2^17, count <= 2^16, H <= 256, beta_q <= 2^16
 * (then L <= 2^33, W <= 2^57).  Any output pointer except L may be NULL.
 * workspace: device buffer of star_project_workspace_bytes(n_inst, H) bytes, ZERO-FILLED by
 * the caller once at allocation; each call leaves it zeroed again.  May be NULL when
 * R <= star_project_single_cta_max_rows(): then one CTA does the whole reduction.
 * Implementation: vectorised coalesced int4 loads, warp-aggregated (match_any + redux) shared-
 * memory histogram over (instance, min(N_hat, H+1)), suffix scan -> L, W, peak, growth.  From
 * 2^18 requests (16-byte aligned arrays, workspace given) the bandwidth form runs as two launches:
 * a streaming kernel (two CTAs per SM, per-CTA contiguous slices, shared-memory bins for a window
 * of instances -- fastest when each instance's requests are contiguous -- merged into the
 * workspace) and a PDL-launched finalize kernel (one warp per instance).
 * ===================================================================================== */
size_t star_project_workspace_bytes(int n_inst, int H);
int star_project_single_cta_max_rows(void);
star_status project_instance_load(int R, int n_inst, int inst_base, int H,
                                  const int32_t* inst, const int32_t* n_tok, const int32_t* n_hat,
                                  const uint32_t* beta_q,
                                  int64_t* L, int64_t* W, int64_t* peak, int64_t* growth, int32_t* count,
                                  void* workspace, int32_t* err_flag, star_stream_t stream);

/* =====================================================================================
 * Reschedule plan  (Alg. 1; objective Eq. 3-4)
 * Exact integer semantics (reading A11): with Q = 65536 and the Q16 schedule beta_q,
 *   Phi*n^2 = sum_{t=0}^{H} beta_q[t] * (n * sum_i L[i][t]^2 - (sum_i L[i][t])^2)
 * Per round (at most max_moves rounds, a request moves at most once per call):
 *   Phase 1  W_i as above (STAR_CURRENT_ONLY: W_i = beta_q[0]*L[i][0]);
 *            O = { i : n*den*W_i > (den+num)*sum_j W_j }                 (w_i > (1+theta) w_bar)
 *            U = { i not in O : n*den*Q*L[i][0] < (den+num)*sum_j W_j }  (reading A13)
 *            O empty -> stop.
 *   Phase 2  candidates (r, s in O, t in U), r on s, not pinned, not yet moved, with
 *            (a) N_hat(r) * (a + b*L[t][0]) > c0 + c1*N(r)    (N_hat > C_mig / T_exec, PAPER.md:435,
 *                readings A15-A17; skipped in STAR_CURRENT_ONLY)
 *            (b) L[t][0] + reserved[t] + N(r) + N_hat(r) <= c_mem[t]  (reading A18;
 *                STAR_STRICT_MEM: L[t][0] + N_hat(r) <= c_mem[t]; CURRENT_ONLY drops N_hat;
 *                c_mem NULL disables the filter)
 *   Phase 3  gain = Phi*n^2(before) - Phi*n^2(r moved s->t) (reading A19), exact __int128;
 *            keep gain > 0 (sigma2_max starts at 0); best = max gain, ties ->
 *            lowest req_id, then lowest target (reading A20).  Apply, emit, next round.
 * The whole plan runs in one CTA: per-request warp argmax over target instances of the
 * closed-form score, then a block argmax over requests.
 * Stream ordering: the plan is launched with programmatic dependent launch.  It reads L and
 * n_hat only after the preceding kernel in the stream has completed; its static inputs
 * (req_id, inst, n_tok, pinned, counts, beta_q, c_mem, reserved) may be read while a preceding
 * kernel of THIS library is still running (none of them writes those arrays).  A preceding
 * kernel of another library cannot overlap (it does not trigger the dependent launch).
 * ===================================================================================== */
#define STAR_STRICT_MEM    1u
#define STAR_CURRENT_ONLY  2u

typedef struct {
  int n_inst, H, max_moves;            /* n_inst >= 1, 0 <= H <= 256, 0 <= max_moves <= 1024 */
  int32_t theta_num, theta_den;        /* theta = num/den >= 0, den >= 1 (default 1/10) */
  const uint32_t* beta_q;              /* [H+1] device, Q16 (beta_q[0] weights sigma0^2) */
  const int64_t* c_mem;                /* [n_inst] device tokens, NULL = no memory filter */
  const int64_t* reserved;             /* [n_inst] device tokens in flight inbound, NULL = 0 */
  int64_t t_exec_a_ps, t_exec_b_ps;    /* T_exec(t) = a + b*L[t][0] picoseconds (Fig. 6 linearity) */
  int64_t mig_c0_ps, mig_c1_ps;        /* C_mig(r) = c0 + c1*N(r) picoseconds (KV bytes / bandwidth) */
  uint32_t flags;                      /* STAR_STRICT_MEM | STAR_CURRENT_ONLY */
} star_plan_params;

typedef struct {
  int32_t req_id, src, dst, round;
  int64_t gain_hi;                     /* gain = Phi*n^2 decrease as signed __int128 (hi:lo) */
  uint64_t gain_lo;
} star_move;                           /* 32 bytes */

/* Contiguous form: L [n_inst][H+1] and R_total requests (SoA, device).  inst[] holds global
 * instance ids in [0, n_inst).  pinned nullable.  moves [max_moves] and n_moves (device int32)
 * are outputs. */
star_status plan_reschedule(const star_plan_params* p, const int64_t* L, int R_total,
                            const int32_t* req_id, const int32_t* inst, const int32_t* n_tok,
                            const int32_t* n_hat, const uint8_t* pinned,
                            star_move* moves, int32_t* n_moves, int32_t* err_flag, star_stream_t stream);

/* Segmented form, reading the gathered per-rank records in place (no unpack copy):
 * segment k (k < world) owns instances [k*n_loc, (k+1)*n_loc) and for every pointer P below
 * its data lives at (char*)P + k*seg_stride:  L [n_loc][H+1] int64, r_count (int32, number of
 * valid requests in the segment, <= r_cap), req_id/inst/n_tok/n_hat [r_cap] int32,
 * pinned [r_cap] uint8 (nullable).  world*n_loc must equal p->n_inst. */
typedef struct {
  int world, n_loc, r_cap;
  int64_t seg_stride;                  /* bytes */
  const int64_t* L;
  const int32_t* r_count;
  const int32_t* req_id;
  const int32_t* inst;
  const int32_t* n_tok;
  const int32_t* n_hat;
  const uint8_t* pinned;
} star_plan_segments;

star_status plan_reschedule_segmented(const star_plan_params* p, const star_plan_segments* seg,
                                      star_move* moves, int32_t* n_moves, int32_t* err_flag,
                                      star_stream_t stream);

/* One-rank step (world == 1): lenpred_forward_project (inst_base 0) followed by
 * plan_reschedule_segmented on this rank's own state; outputs identical to the two calls in
 * sequence.  The segments (world 1, n_loc == n_inst) normally alias the projection output L and
 * n_hat.  When the fused tail runs, the plan has a single round (max_moves <= 1) and its state
 * fits in the tail's freed stage ring, Alg. 1 is executed by the projection's last finishing CTA
 * (one launch fewer, no kernel boundary between the projection and the plan); otherwise the
 * 512-thread plan kernel follows (faster for several rounds).  Argument meaning and errors:
 * lenpred_forward_project and plan_reschedule_segmented. */
star_status lenpred_forward_project_plan(star_predictor* p, const void* h, int64_t ld_h, int R,
                                         const int32_t* n_tok, int32_t max_ctx_len, float* y_hat, int32_t* n_hat,
                                         int n_inst, int H, const int32_t* inst, const uint32_t* beta_q, int64_t* L,
                                         int64_t* W, int64_t* peak, int64_t* growth, int32_t* count, void* workspace,
                                         const star_plan_params* pp, const star_plan_segments* sg,
                                         star_move* moves, int32_t* n_moves, int32_t* err_flag,
                                         star_stream_t stream);

/* Diagnostics: %globaltimer stamps (ns) of the most recent single-CTA plan launch: [0] entry,
 * [1] launched, [12] static inputs staged, [13] after griddepcontrol.wait, [2] inputs staged,
 * [3] W pass, [4] classification, [9] candidates compacted, [5] candidate argmax, [6] move
 * applied, [7] end (per-round stamps hold the last round); [32 + k] the same as clock64;
 * [64 + 8 r + j] per CTA r of the cluster plan: j = 0 entry, 1 after griddepcontrol.wait,
 * 2/4 before and 3/5 after the round's cluster barrier (round parity).  host64 holds 128 values.
 * Synchronises the device. */
star_status star_plan_timeline(uint64_t* host64);

/* Cluster-scale form (NEXT-3: hundreds of instances, up to 2^20 request slots; the paper's
 * budget is <= 300 ms at 256 instances): identical semantics and outputs, but the
 * state lives in `workspace` (star_plan_workspace_bytes(n_inst, H, world*r_cap) bytes, no
 * initialisation needed) and each round runs as two multi-CTA launches (per-instance prefix
 * sums; candidate scan over all SMs + last-CTA selection), so n_inst is limited only by
 * 16384 and by memory, not by one SM's shared memory.  workspace == NULL falls back to
 * plan_reschedule_segmented (single CTA). */
size_t star_plan_workspace_bytes(int n_inst, int H, int64_t request_slots);
star_status plan_reschedule_segmented_ws(const star_plan_params* p, const star_plan_segments* seg,
                                         star_move* moves, int32_t* n_moves, int32_t* err_flag, void* workspace,
                                         star_stream_t stream);

/* =====================================================================================
 * P -> D dispatch of newly prefilled requests  (NEXT-2; a request "will be
 * forwarded to a decode instance according to its input length, predicted output length, and
 * the current load of each decode instance"; baselines PAPER.md:98-99)
 * Arrivals a = 0..A-1 (n_tok[a] = N, n_hat[a] = predicted remaining length) are placed in
 * order; the chosen instance's loads L [n_inst][H+1] (device, in/out: the projected loads of
 * project_instance_load) get the request's contribution (c_0 = N, c_t = (N+t)[t < N_hat]) before
 * the next arrival is placed.  assign[a] = instance, or -1 when no instance is feasible.
 *   STAR_DISPATCH_ROUND_ROBIN   (counter + a) mod n_inst
 *   STAR_DISPATCH_CURRENT_LOAD  argmin L[i][0], ties -> lowest id
 *   STAR_DISPATCH_PROJECTED     (reading A28) among instances with
 *                               L[i][0] + reserved[i] + N + N_hat <= c_mem[i] (c_mem NULL -> all),
 *                               the one minimising the Eq. 3-4 objective after the placement
 *                               (exact integers: argmin sum_{t<=T} beta_q[t] (N+t) L[i][t]),
 *                               ties -> lowest id.  Needs `workspace`
 *                               (star_dispatch_workspace_bytes(n_inst, H) bytes, no init).
 * One CTA; sequential over arrivals by definition.  A = 0 enqueues nothing.
 * ===================================================================================== */
#define STAR_DISPATCH_ROUND_ROBIN  0
#define STAR_DISPATCH_CURRENT_LOAD 1
#define STAR_DISPATCH_PROJECTED    2

size_t star_dispatch_workspace_bytes(int n_inst, int H);
star_status dispatch_requests(int policy, int n_inst, int H, const uint32_t* beta_q, int64_t* L,
                              const int64_t* c_mem, const int64_t* reserved, int A, const int32_t* n_tok,
                              const int32_t* n_hat, int32_t counter, int32_t* assign, void* workspace,
                              star_stream_t stream);

/* =====================================================================================
 * KV-cache migration  (NEXT-4; Alg. 1 line 10 "ExecuteMigration(m*)"; §5.4: "the
 * paused request's KV cache is transfered to the target instance without blocking the execution
 * of other requests"; transfer time vs bandwidth, Fig. 9)
 * A paged KV pool is n_layers x n_blocks blocks of block_bytes bytes (block b of layer l at
 * base + l*layer_stride + b*block_bytes; e.g. vLLM's K and V of block_size tokens of one layer);
 * a request owns the n blocks its block table lists (int32 block ids, device memory).
 *   kv_pack     copies the request's blocks into a contiguous staging buffer laid out
 *               [n_layers][n][block_bytes] (layer-major, table order);
 *   kv_unpack   copies a staging buffer into the blocks `table` lists (the destination's
 *               freshly allocated blocks);
 *   kv_migrate  copies block src_table[j] of src to block dst_table[j] of dst for every layer and
 *               j, with no staging.  src->base may be a PEER device's pointer (cudaDeviceEnablePeerAccess):
 *               the kernel runs on the calling (destination) device and pulls over NVLink.
 * Requirements: bases, block_bytes and layer_stride 16-byte aligned, layer_stride >= n_blocks *
 * block_bytes, equal n_layers and block_bytes for kv_migrate.  A block id outside [0, n_blocks)
 * sets STAR_ERRF_BLOCK in *err_flag and that (layer, block) copy is skipped.  Asynchronous on
 * `stream`, no allocation, graph capturable; n = 0 enqueues nothing.  Overlap with decode by
 * issuing on a separate (low-priority) stream.  The copies of one call run concurrently: a block
 * must not be both read and written by the same call (src and dst may be the same pool when the
 * two tables are disjoint; a destination block listed twice gets either copy).
 * ===================================================================================== */
#define STAR_ERRF_BLOCK 4  /* KV block id outside the pool */

typedef struct {
  void* base;            /* device pointer of layer 0, block 0 */
  int n_layers;
  int64_t layer_stride;  /* bytes between consecutive layers */
  int64_t n_blocks;      /* blocks per layer */
  int64_t block_bytes;   /* bytes of one block of one layer */
} star_kv_pool;

star_status kv_pack(const star_kv_pool* src, const int32_t* table, int n, void* staging, int32_t* err_flag,
                    star_stream_t stream);
star_status kv_unpack(const void* staging, const star_kv_pool* dst, const int32_t* table, int n, int32_t* err_flag,
                      star_stream_t stream);
star_status kv_migrate(const star_kv_pool* src, const int32_t* src_table, const star_kv_pool* dst,
                       const int32_t* dst_table, int n, int32_t* err_flag, star_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* STAR_H_ */
