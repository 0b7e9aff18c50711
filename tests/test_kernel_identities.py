"""CPU checks of the closed forms the CUDA kernels use in place of the paper's from-scratch
arithmetic (no GPU; plain integer numpy / Python ints, so every value is exact).

* Placing a request (N, N_hat) on instance i adds c_t (c_0 = N, c_t = (N + t)[t < N_hat],
  reading A5) to L_i.  The beta-weighted prefix sums P0_i[T] = sum_{t<=T} beta_t L_i[t] and
  P1_i[T] = sum_{t<=T} t beta_t L_i[t] (the plan's target term, Eq. 3-4) then
  grow by N B0[m] + B1[m] and N B1[m] + B2[m], m = min(T, clamp(N_hat - 1, 0, H)), with B0/B1/B2
  the prefix sums of beta_t, t beta_t, t^2 beta_t -- what dispatch_seq_kernel adds instead of
  rebuilding the row after each placement (csrc/dispatch.cu).
* The score of moving a request from s to u, N (P0_s[T] - P0_u[T]) + (P1_s[T] - P1_u[T]) -
  (N^2 B0[T] + 2 N B1[T] + B2[T]), is half the drop of sum_t beta_t sum_i L_i[t]^2 -- the only part
  of the objective (n times the beta-weighted variance) a move changes, so the gain is 2 n score.
* The 16-bit-chunk warp sum the projection finalize uses is the int64 sum mod 2^64.
"""
import numpy as np
import pytest


def _prefix(L_row, beta):
    P0, P1, a0, a1 = [], [], 0, 0
    for t, (l, b) in enumerate(zip(L_row, beta)):
        a0 += int(b) * int(l)
        a1 += t * int(b) * int(l)
        P0.append(a0)
        P1.append(a1)
    return P0, P1


def _btab(beta):
    B0, B1, B2, a0, a1, a2 = [], [], [], 0, 0, 0
    for t, b in enumerate(beta):
        a0 += int(b)
        a1 += t * int(b)
        a2 += t * t * int(b)
        B0.append(a0)
        B1.append(a1)
        B2.append(a2)
    return B0, B1, B2


def _contrib(N, nh, H):
    return [N if t == 0 else (N + t if t < nh else 0) for t in range(H + 1)]


@pytest.mark.parametrize("seed", range(12))
def test_prefix_growth_closed_form(seed):
    g = np.random.default_rng(seed)
    H = int(g.integers(0, 60))
    beta = [65536] + [int(x) for x in g.integers(1, 65537, H)]
    B0, B1, B2 = _btab(beta)
    L = [int(x) for x in g.integers(0, 10**6, H + 1)]
    for _ in range(20):
        N, nh = int(g.integers(0, 2**31 - 1)), int(g.integers(-3, H + 40))
        Tp = min(max(nh - 1, 0), H)
        before = _prefix(L, beta)
        L = [a + c for a, c in zip(L, _contrib(N, nh, H))]
        after = _prefix(L, beta)
        for T in range(H + 1):
            m = min(T, Tp)
            assert after[0][T] - before[0][T] == N * B0[m] + B1[m]
            assert after[1][T] - before[1][T] == N * B1[m] + B2[m]


@pytest.mark.parametrize("seed", range(12))
def test_move_score_closed_form(seed):
    g = np.random.default_rng(100 + seed)
    n, H = int(g.integers(2, 7)), int(g.integers(0, 30))
    beta = [65536] + [int(x) for x in g.integers(1, 65537, H)]
    B0, B1, B2 = _btab(beta)
    L = [[int(x) for x in g.integers(0, 10**5, H + 1)] for _ in range(n)]
    N, nh = int(g.integers(1, 5000)), int(g.integers(0, H + 10))
    s, u = 0, 1
    c = _contrib(N, nh, H)
    L[s] = [a + x for a, x in zip(L[s], c)]   # the request sits on s
    T = min(max(nh - 1, 0), H)
    P0s, P1s = _prefix(L[s], beta)
    P0u, P1u = _prefix(L[u], beta)
    score = N * (P0s[T] - P0u[T]) + (P1s[T] - P1u[T]) - (N * N * B0[T] + 2 * N * B1[T] + B2[T])

    def sq(Ls):
        return sum(int(beta[t]) * sum(Ls[i][t] ** 2 for i in range(n)) for t in range(H + 1))

    moved = [row[:] for row in L]
    moved[s] = [a - x for a, x in zip(moved[s], c)]
    moved[u] = [a + x for a, x in zip(moved[u], c)]
    # sum_i L_i[t] is unchanged by a move, so n * Var_t changes only through sum_i L_i[t]^2
    assert sq(L) - sq(moved) == 2 * score


def test_chunked_int64_sum():
    g = np.random.default_rng(7)
    for _ in range(200):
        v = [int(x) for x in g.integers(-2**63, 2**63 - 1, 32, dtype=np.int64)]
        chunks = [sum((x & 0xFFFFFFFFFFFFFFFF) >> (16 * k) & 0xFFFF for x in v) for k in range(4)]
        assert all(c < 2**32 for c in chunks)   # each redux.add.u32 is exact
        got = sum(c << (16 * k) for k, c in enumerate(chunks)) & 0xFFFFFFFFFFFFFFFF
        assert got == sum(v) & 0xFFFFFFFFFFFFFFFF
