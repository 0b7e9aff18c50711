// STAR CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// Plain, slow, obviously-correct C++17 implementation of the hot path of
// arxiv 2510.13668 (STAR, "Adaptive Rescheduling in Prefill-Decode Disaggregated
// LLM Inference").  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no code,
// header, table or constant with the CUDA product path (paper_2510_13668_b200/).
//
// Conventions: scalar loops, fp64 accumulation for the predictor, exact __int128 for
// every integer the plan depends on, no blocking / fusion / reordering beyond the
// definitions cited.  Compiled with -O2 -ffp-contract=off (no FMA contraction).
//
// Pins (tests/test_oracle_*.py): closed forms, SPEC/PAPER worked examples, a pure-Python
// Fraction brute force (oracle/brute.py), invariants.  Every function below is pinned;
// see DESIGN.md "Oracle pins".
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>

typedef __int128 i128;

extern "C" {

// ---------------------------------------------------------------------------------
// Eq. 2 (§4.2 "MLP Predictor"):
//     y_hat = w4 * phi(W3 * phi(W2 * phi(W1 * h))),   phi = ReLU
// W1 [m1 x d], W2 [m2 x m1], W3 [m3 x m2], w4 [m3] row-major [out][in].
// Optional biases (reading A1: Eq. 2 has none; NULL reproduces it literally).
// Inputs are the exact fp32 values (bf16 inputs are widened exactly by the caller);
// every product and sum is carried in fp64, intermediates are not rounded.
// ---------------------------------------------------------------------------------
int oracle_lenpred(int R, int d, int m1, int m2, int m3,
                   const float* h, long ld_h,
                   const float* W1, const float* W2, const float* W3, const float* w4,
                   const float* b1, const float* b2, const float* b3, const float* b4,
                   double* y_out, int nthreads) {
  if (R < 0 || d <= 0 || m1 <= 0 || m2 <= 0 || m3 <= 0 || ld_h < d) return -1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int r = 0; r < R; ++r) {
    std::vector<double> z1(m1), z2(m2), z3(m3);
    const float* hr = h + (long)r * ld_h;
    // layer 1: z1 = phi(W1 h (+ b1))
    for (int j = 0; j < m1; ++j) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc += (double)W1[(long)j * d + k] * (double)hr[k];
      if (b1) acc += (double)b1[j];
      z1[j] = acc > 0.0 ? acc : 0.0;
    }
    // layer 2: z2 = phi(W2 z1 (+ b2))
    for (int j = 0; j < m2; ++j) {
      double acc = 0.0;
      for (int k = 0; k < m1; ++k) acc += (double)W2[(long)j * m1 + k] * z1[k];
      if (b2) acc += (double)b2[j];
      z2[j] = acc > 0.0 ? acc : 0.0;
    }
    // layer 3: z3 = phi(W3 z2 (+ b3))
    for (int j = 0; j < m3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < m2; ++k) acc += (double)W3[(long)j * m2 + k] * z2[k];
      if (b3) acc += (double)b3[j];
      z3[j] = acc > 0.0 ? acc : 0.0;
    }
    // output: y = w4 z3 (+ b4)
    double y = 0.0;
    for (int k = 0; k < m3; ++k) y += (double)w4[k] * z3[k];
    if (b4) y += (double)b4[0];
    y_out[r] = y;
  }
  return 0;
}

// ---------------------------------------------------------------------------------
// Quantizer (reading A8-A10; the paper treats y as a real-valued regression output,
// PAPER.md:201-206): cap_r = max(0, L_ctx - N_r) (N_r = n_tok[r]; n_tok NULL => cap = L_ctx),
// N_hat_r = (int) rint(fminf(fmaxf(y_r, 0), cap_r)), round-half-to-even, fp32.
// fmaxf(NaN, 0) = 0 (IEEE maxNum) so NaN -> 0; +Inf -> cap; negative -> 0.
// ---------------------------------------------------------------------------------
void oracle_quantize(int R, const float* y, const int32_t* n_tok, int32_t l_ctx, int32_t* n_hat) {
  for (int r = 0; r < R; ++r) {
    int32_t cap = l_ctx;
    if (n_tok) cap = l_ctx - n_tok[r];
    if (cap < 0) cap = 0;
    float v = fmaxf(y[r], 0.0f);
    v = fminf(v, (float)cap);
    n_hat[r] = (int32_t)rintf(v);
  }
}

// ---------------------------------------------------------------------------------
// Per-request projected contribution (reading A5):
//   c_r[0] = N_r;   c_r[t] = (N_r + t) if t < N_hat_r else 0,   t = 1..H
// ---------------------------------------------------------------------------------
static inline int64_t contrib(int64_t N, int64_t nhat, int t) {
  if (t == 0) return N;
  return (t < nhat) ? (N + t) : 0;
}

// ---------------------------------------------------------------------------------
// Worker-side local future-state simulation (Alg. 1 line 13):
//   L_i[0] = N_i(B_i) = sum_{r in B_i} N(r)
//   L_i[t] = N_hat_i(B_{i,t}) = sum_{r in B_i} c_r[t],  t = 1..H
//   W_i    = w_i = sum_{t=1}^{H} beta_t L_i[t]  (beta in Q16)
//   peak_i = max_{0<=t<=H} L_i[t];  G_i = sum min(N_hat_r, H);  count_i = |B_i|
// Literal O(R*H) double loop.  Instance of request r = inst[r] - inst_base.
// Returns 0, or -2 if an instance id is out of range.
// ---------------------------------------------------------------------------------
int oracle_project(int R, int n_inst, int inst_base, int H,
                   const int32_t* inst, const int32_t* n_tok, const int32_t* n_hat,
                   const uint32_t* beta_q,
                   int64_t* L, int64_t* W, int64_t* peak, int64_t* growth, int32_t* count) {
  for (int i = 0; i < n_inst; ++i) {
    for (int t = 0; t <= H; ++t) L[(long)i * (H + 1) + t] = 0;
    W[i] = 0; peak[i] = 0; growth[i] = 0; count[i] = 0;
  }
  for (int r = 0; r < R; ++r) {
    int i = inst[r] - inst_base;
    if (i < 0 || i >= n_inst) return -2;
    for (int t = 0; t <= H; ++t) L[(long)i * (H + 1) + t] += contrib(n_tok[r], n_hat[r], t);
    growth[i] += std::min<int64_t>(n_hat[r], H);
    count[i] += 1;
  }
  for (int i = 0; i < n_inst; ++i) {
    int64_t w = 0, pk = 0;
    for (int t = 1; t <= H; ++t) w += (int64_t)beta_q[t] * L[(long)i * (H + 1) + t];
    for (int t = 0; t <= H; ++t) pk = std::max(pk, L[(long)i * (H + 1) + t]);
    W[i] = w; peak[i] = pk;
  }
  return 0;
}

// ---------------------------------------------------------------------------------
// Objective, Eq. 3-4 truncated at H (Alg. 1 line 13), exact integers
// (reading A11/A12):  Phi * n^2 = sum_{t=0}^{H} beta_q[t] * (n * sum_i L_i[t]^2 - (sum_i L_i[t])^2)
// = n^2 * sum_t beta_t Var_t (population variance); beta_q[0] weights sigma0^2.
// With current_only (reading A25) only the t = 0 term (sigma0^2) is kept.
// ---------------------------------------------------------------------------------
static i128 phi_n2(int n, int H, const std::vector<int64_t>& L, const uint32_t* beta_q, bool current_only) {
  i128 total = 0;
  int Tmax = current_only ? 0 : H;
  for (int t = 0; t <= Tmax; ++t) {
    i128 s = 0, s2 = 0;
    for (int i = 0; i < n; ++i) {
      i128 x = L[(long)i * (H + 1) + t];
      s += x;
      s2 += x * x;
    }
    total += (i128)beta_q[t] * ((i128)n * s2 - s * s);
  }
  return total;
}

void oracle_objective(int n, int H, const int64_t* L, const uint32_t* beta_q, int current_only,
                      int64_t* hi, uint64_t* lo) {
  std::vector<int64_t> v(L, L + (long)n * (H + 1));
  i128 x = phi_n2(n, H, v, beta_q, current_only != 0);
  *hi = (int64_t)(x >> 64);
  *lo = (uint64_t)x;
}

// ---------------------------------------------------------------------------------
// Algorithm 1, greedy rounds (reading A20/A21), exact integers.
// flags: 1 = STRICT_MEM (filter (b) literal: L_t[0] + N_hat <= C_mem)
//        2 = CURRENT_ONLY ("vLLM + rescheduling" baseline, reading A25)
// Moves written to out arrays (capacity max_moves); returns #moves, or <0 on bad input.
// ---------------------------------------------------------------------------------
int oracle_plan(int n, int H, int max_moves, int32_t theta_num, int32_t theta_den,
                const uint32_t* beta_q, const int64_t* c_mem, const int64_t* reserved,
                int64_t a_ps, int64_t b_ps, int64_t c0_ps, int64_t c1_ps, uint32_t flags,
                const int64_t* L_in, int R, const int32_t* req_id, const int32_t* inst,
                const int32_t* n_tok, const int32_t* n_hat, const uint8_t* pinned,
                int32_t* mv_req, int32_t* mv_src, int32_t* mv_dst, int32_t* mv_round,
                int64_t* mv_gain_hi, uint64_t* mv_gain_lo) {
  const bool strict_mem = (flags & 1u) != 0;
  const bool current_only = (flags & 2u) != 0;
  const i128 Q = 65536;
  std::vector<int64_t> L(L_in, L_in + (long)n * (H + 1));
  std::vector<char> moved(R, 0);
  for (int r = 0; r < R; ++r)
    if (inst[r] < 0 || inst[r] >= n) return -2;
  int nm = 0;
  for (int round = 0; round < max_moves; ++round) {
    // ---- Phase 1: InstanceClassification (Alg. 1 lines 23-30) ----
    // w_i = sum_{t=1}^{H} beta_t N_hat_i(B_{i,t}); w_bar = mean_i w_i (reading A14)
    std::vector<i128> w(n);
    i128 wsum = 0;
    for (int i = 0; i < n; ++i) {
      i128 wi = 0;
      if (current_only) {
        wi = (i128)beta_q[0] * L[(long)i * (H + 1)];
      } else {
        for (int t = 1; t <= H; ++t) wi += (i128)beta_q[t] * L[(long)i * (H + 1) + t];
      }
      w[i] = wi;
      wsum += wi;
    }
    // O = { i : w_i > (1+theta) w_bar }  <=>  n*den*w_i > (den+num)*sum_j w_j
    std::vector<char> inO(n, 0), inU(n, 0);
    bool anyO = false;
    for (int i = 0; i < n; ++i) {
      if ((i128)n * theta_den * w[i] > (i128)(theta_den + theta_num) * wsum) { inO[i] = 1; anyO = true; }
    }
    if (!anyO) break;  // Alg. 1 line 14
    // U = { i not in O : N_i(B_{i,0}) < (1+theta) w_bar } (reading A13: L_i[0] scaled by Q)
    for (int i = 0; i < n; ++i) {
      if (inO[i]) continue;
      if ((i128)n * theta_den * Q * L[(long)i * (H + 1)] < (i128)(theta_den + theta_num) * wsum) inU[i] = 1;
    }
    // ---- Phase 2 + 3: CandidateEnumeration and OptimalSelection (lines 32-51) ----
    const i128 phi_before = phi_n2(n, H, L, beta_q, current_only);
    bool have = false;
    i128 best_g = 0;
    int best_r = -1, best_t = -1;
    for (int r = 0; r < R; ++r) {
      int s = inst[r];
      if (!inO[s] || moved[r] || (pinned && pinned[r])) continue;
      for (int tg = 0; tg < n; ++tg) {
        if (!inU[tg]) continue;
        // filter (a): N_hat(r) > C_mig / T_exec  (readings A15-A17)
        //   cross-multiplied in integer ps: N_hat * (a + b * L_t[0]) > c0 + c1 * N(r)
        if (!current_only) {
          i128 lhs = (i128)n_hat[r] * ((i128)a_ps + (i128)b_ps * L[(long)tg * (H + 1)]);
          i128 rhs = (i128)c0_ps + (i128)c1_ps * n_tok[r];
          if (!(lhs > rhs)) continue;
        }
        // filter (b): memory safety (reading A18)
        if (c_mem) {
          i128 need = L[(long)tg * (H + 1)];
          if (strict_mem) {
            if (!current_only) need += n_hat[r];
          } else {
            need += (reserved ? reserved[tg] : 0) + n_tok[r];
            if (!current_only) need += n_hat[r];
          }
          if (!(need <= (i128)c_mem[tg])) continue;
        }
        // AggregateSimulations + SimulateFutureVariance (reading A19): rebuild the
        // load vectors with r moved s -> tg and recompute the objective from scratch.
        std::vector<int64_t> L2 = L;
        for (int t = 0; t <= H; ++t) {
          int64_t c = contrib(n_tok[r], n_hat[r], t);
          L2[(long)s * (H + 1) + t] -= c;
          L2[(long)tg * (H + 1) + t] += c;
        }
        i128 g = phi_before - phi_n2(n, H, L2, beta_q, current_only);
        // UpdateBestCandidate (sigma2_max starts at 0 => strictly positive gain; ties by
        // lowest request id, then lowest target id -- reading A20)
        if (g <= 0) continue;
        bool better = !have || g > best_g ||
                      (g == best_g && (req_id[r] < req_id[best_r] ||
                                       (req_id[r] == req_id[best_r] && tg < best_t)));
        if (better) { have = true; best_g = g; best_r = r; best_t = tg; }
      }
    }
    if (!have) break;
    // ExecuteMigration is out of scope; apply m* to the snapshot for the next round.
    int s = inst[best_r];
    for (int t = 0; t <= H; ++t) {
      int64_t c = contrib(n_tok[best_r], n_hat[best_r], t);
      L[(long)s * (H + 1) + t] -= c;
      L[(long)best_t * (H + 1) + t] += c;
    }
    moved[best_r] = 1;
    mv_req[nm] = req_id[best_r];
    mv_src[nm] = s;
    mv_dst[nm] = best_t;
    mv_round[nm] = round;
    mv_gain_hi[nm] = (int64_t)(best_g >> 64);
    mv_gain_lo[nm] = (uint64_t)best_g;
    ++nm;
  }
  return nm;
}

// ---------------------------------------------------------------------------------
// P -> D dispatch of newly prefilled requests (NEXT-2; "forwarded to a decode
// instance according to its input length, predicted output length, and the current load";
// baselines PAPER.md:98-99).  Arrivals a = 0..A-1 are placed in order.
//   policy 0 (round robin):   i = (counter + a) mod n
//   policy 1 (current load):  i = argmin_i L_i[0]                 (ties -> lowest id)
//   policy 2 (projected, STAR, reading A28): among instances passing the memory filter
//     L_i[0] + reserved_i + N + N_hat <= C_mem_i (reading A18; c_mem NULL -> all), the one whose
//     objective Phi (Eq. 3-4, exact integer Phi*n^2) AFTER placing the request is smallest
//     (ties -> lowest id); none feasible -> -1 (not placed).  The objective is recomputed from
//     scratch for every candidate placement.
// The chosen instance's loads are updated with the request's contribution c_r[t] (reading A5)
// before the next arrival.  Returns the number placed.
// ---------------------------------------------------------------------------------
int oracle_dispatch(int policy, int n, int H, const uint32_t* beta_q, int64_t* L, const int64_t* c_mem,
                    const int64_t* reserved, int A, const int32_t* n_tok, const int32_t* n_hat, int32_t counter,
                    int32_t* assign) {
  std::vector<int64_t> Lv(L, L + (long)n * (H + 1));
  int placed = 0;
  for (int a = 0; a < A; ++a) {
    int best = -1;
    if (policy == 0) {
      best = (int)(((int64_t)counter + a) % n);
    } else if (policy == 1) {
      for (int i = 0; i < n; ++i)
        if (best < 0 || Lv[(long)i * (H + 1)] < Lv[(long)best * (H + 1)]) best = i;
    } else {
      i128 best_phi = 0;
      for (int i = 0; i < n; ++i) {
        if (c_mem) {
          i128 need = (i128)Lv[(long)i * (H + 1)] + (reserved ? reserved[i] : 0) + n_tok[a] + n_hat[a];
          if (!(need <= (i128)c_mem[i])) continue;
        }
        std::vector<int64_t> L2 = Lv;
        for (int t = 0; t <= H; ++t) L2[(long)i * (H + 1) + t] += contrib(n_tok[a], n_hat[a], t);
        i128 ph = phi_n2(n, H, L2, beta_q, false);
        if (best < 0 || ph < best_phi) { best = i; best_phi = ph; }
      }
    }
    assign[a] = best;
    if (best >= 0) {
      for (int t = 0; t <= H; ++t) Lv[(long)best * (H + 1) + t] += contrib(n_tok[a], n_hat[a], t);
      ++placed;
    }
  }
  for (long k = 0; k < (long)n * (H + 1); ++k) L[k] = Lv[k];
  return placed;
}

}  // extern "C"
