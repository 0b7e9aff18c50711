"""Independent pure-Python brute force for tiny inputs -- TEST INFRASTRUCTURE ONLY.

Written directly from the paper's real-valued statements with exact rationals
(fractions.Fraction), sharing nothing with oracle.cpp:
  * projection per request, straight from SPEC.md:96 / reading A5 (no histogram, no sums
    of prefixes),
  * variance as the textbook population variance with the mean subtracted (Eq. 3,
    PAPER.md:373), weighted sum over t with beta_t = beta_q[t] / 65536 (Eq. 4),
  * Phase 1 with real w_bar and real (1+theta),
  * filter (a) as the paper's quotient N_hat > C_mig / T_exec,
  * Phase 3 by re-projecting the whole request set with r reassigned and recomputing the
    objective, exhaustive over every candidate,
  * exhaustive optimal assignment over all n^R placements (lower bound pin).
"""
from __future__ import annotations

import itertools
from fractions import Fraction

Q = 65536


def request_load(N: int, nhat: int, t: int) -> int:
    """a request contributes N + t while t < predicted_remaining, else 0;
    at t = 0 the current token count N(r)."""
    if t == 0:
        return N
    return N + t if t < nhat else 0


def project(n, H, inst, n_tok, n_hat):
    L = [[0] * (H + 1) for _ in range(n)]
    for i_r, N, nh in zip(inst, n_tok, n_hat):
        for t in range(H + 1):
            L[int(i_r)][t] += request_load(int(N), int(nh), t)
    return L


def pop_variance(xs):
    xs = [Fraction(int(x)) for x in xs]
    mu = sum(xs, Fraction(0)) / len(xs)
    return sum(((x - mu) ** 2 for x in xs), Fraction(0)) / len(xs)


def phi(L, beta_q, current_only=False):
    """sigma_hat^2 = sigma0^2 + sum_{t=1}^{H} beta_t Var_t (Eq. 4 truncated), beta_t = beta_q[t]/Q;
    beta_q[0]/Q weights sigma0^2 (=1 with the default schedule)."""
    n = len(L)
    H = len(L[0]) - 1
    T = 0 if current_only else H
    total = Fraction(0)
    for t in range(T + 1):
        total += Fraction(int(beta_q[t]), Q) * pop_variance([L[i][t] for i in range(n)])
    return total


def classify(L, beta_q, theta, current_only=False):
    n = len(L)
    H = len(L[0]) - 1
    if current_only:
        w = [Fraction(int(beta_q[0]), Q) * L[i][0] for i in range(n)]
    else:
        w = [sum((Fraction(int(beta_q[t]), Q) * L[i][t] for t in range(1, H + 1)), Fraction(0)) for i in range(n)]
    wbar = sum(w, Fraction(0)) / n
    O = [i for i in range(n) if w[i] > (1 + theta) * wbar]
    U = [i for i in range(n) if i not in O and L[i][0] < (1 + theta) * wbar]
    return O, U


def plan(params, req_id, inst, n_tok, n_hat, pinned=None):
    """Exhaustive Alg. 1 with greedy rounds; returns [(req_id, src, dst, round, gain_int)],
    gain_int = n^2 * Q * (Phi_before - Phi_after) (the ABI's unit)."""
    n, H = params.n_inst, params.H
    beta_q = [int(b) for b in params.beta_q]
    theta = Fraction(params.theta_num, params.theta_den)
    strict = bool(params.flags & 1)
    cur = bool(params.flags & 2)
    inst = [int(x) for x in inst]
    R = len(inst)
    moved = set()
    out = []
    for rnd in range(params.max_moves):
        L = project(n, H, inst, n_tok, n_hat)
        O, U = classify(L, beta_q, theta, cur)
        if not O:
            break
        phi0 = phi(L, beta_q, cur)
        best = None
        for r in range(R):
            s = inst[r]
            if s not in O or r in moved or (pinned is not None and pinned[r]):
                continue
            N, nh = int(n_tok[r]), int(n_hat[r])
            for tg in U:
                if not cur:
                    T_exec = params.t_exec_a_ps + params.t_exec_b_ps * L[tg][0]
                    C_mig = params.mig_c0_ps + params.mig_c1_ps * N
                    if T_exec == 0 or not (Fraction(nh) > Fraction(C_mig, T_exec)):
                        continue
                if params.c_mem is not None:
                    if strict:
                        need = L[tg][0] + (0 if cur else nh)
                    else:
                        res = 0 if params.reserved is None else int(params.reserved[tg])
                        need = L[tg][0] + res + N + (0 if cur else nh)
                    if need > int(params.c_mem[tg]):
                        continue
                inst2 = list(inst)
                inst2[r] = tg
                phi1 = phi(project(n, H, inst2, n_tok, n_hat), beta_q, cur)
                red = phi0 - phi1
                if red <= 0:
                    continue
                key = (-red, int(req_id[r]), tg)
                if best is None or key < best[0]:
                    best = (key, r, tg, red)
        if best is None:
            break
        _, r, tg, red = best
        g = red * n * n * Q
        assert g.denominator == 1
        out.append((int(req_id[r]), inst[r], tg, rnd, int(g)))
        inst[r] = tg
        moved.add(r)
    return out


def optimal_assignment_phi(n, H, n_tok, n_hat, beta_q, current_only=False):
    """min Phi over all n^R placements (tiny R only)."""
    best = None
    R = len(n_tok)
    for a in itertools.product(range(n), repeat=R):
        v = phi(project(n, H, a, n_tok, n_hat), beta_q, current_only)
        if best is None or v < best:
            best = v
    return best


def dispatch(policy, L, beta_q, n_tok, n_hat, c_mem=None, reserved=None, counter=0):
    """P -> D placement in arrival order (reading A28), real-valued
    objective with exact rationals: for the projected policy every feasible placement is tried
    and the textbook weighted variance (phi) of the resulting loads is compared."""
    L = [list(map(int, row)) for row in L]
    n, H = len(L), len(L[0]) - 1
    out = []
    for a, (N, nh) in enumerate(zip(n_tok, n_hat)):
        N, nh = int(N), int(nh)
        if policy == 0:
            best = (counter + a) % n
        elif policy == 1:
            best = min(range(n), key=lambda i: (L[i][0], i))
        else:
            best, best_phi = -1, None
            for i in range(n):
                if c_mem is not None:
                    res = 0 if reserved is None else int(reserved[i])
                    if L[i][0] + res + N + nh > int(c_mem[i]):
                        continue
                L2 = [row[:] for row in L]
                for t in range(H + 1):
                    L2[i][t] += request_load(N, nh, t)
                ph = phi(L2, beta_q)
                if best < 0 or ph < best_phi:
                    best, best_phi = i, ph
        out.append(best)
        if best >= 0:
            for t in range(H + 1):
                L[best][t] += request_load(N, nh, t)
    return out, L
