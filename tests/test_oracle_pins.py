"""Oracle pins (CPU, `-m "not gpu"`): the oracle is checked against things other than
itself -- the paper's and SPEC's worked examples, hand-derived closed forms, invariants,
and an independent exact-rational brute force (oracle/brute.py)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import datagen
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# =============================================================================== predictor
def test_param_count_pins_layer_widths():
    """PAPER.md:241 widths (d=3584, m1=2048, m2=512, m3=64) give Table 1's '8.4 M'
    (PAPER.md:302): 3584*2048 + 2048*512 + 512*64 + 64 = 8,421,440 (reading A2)."""
    pw = datagen.make_predictor_weights(0, 3584, "bf16")
    n = pw.W1.size + pw.W2.size + pw.W3.size + pw.w4.size
    assert n == 8_421_440
    assert round(n / 1e6, 1) == 8.4


def test_predictor_hand_example(oracle_mod):
    g = _gold("predictor_tiny.json")
    y = oracle_mod.lenpred(np.array(g["h"], np.float32), np.array(g["W1"], np.float32),
                           np.array(g["W2"], np.float32), np.array(g["W3"], np.float32),
                           np.array(g["w4"], np.float32))
    assert y.tolist() == g["expected_y"]


def test_predictor_closed_form_identity(oracle_mod):
    """W1=W2=W3=I, w4=(1..8): h>=0 -> y = sum_j j*h_j; h<=0 -> y = 0 (ReLU kills it)."""
    d = 8
    eye = np.eye(d, dtype=np.float32)
    w4 = np.arange(1, d + 1, dtype=np.float32)
    g = datagen.rng(3)
    hp = np.abs(g.standard_normal((5, d))).astype(np.float32)
    y = oracle_mod.lenpred(hp, eye, eye, eye, w4)
    exact = [sum(Fraction(float(hp[r, j])) * (j + 1) for j in range(d)) for r in range(5)]
    np.testing.assert_allclose(y, [float(e) for e in exact], rtol=1e-15)
    y0 = oracle_mod.lenpred(-hp, eye, eye, eye, w4)
    assert np.all(y0 == 0.0)


def test_predictor_bias_closed_form(oracle_mod):
    """With zero weights the output is w4 . relu(b3) + b4 (biases propagate through phi)."""
    d, m = 4, 3
    Z = lambda a, b: np.zeros((a, b), np.float32)
    b3 = np.array([1.0, -2.0, 0.5], np.float32)
    w4 = np.array([2.0, 5.0, 4.0], np.float32)
    y = oracle_mod.lenpred(np.ones((2, d), np.float32), Z(m, d), Z(m, m), Z(m, m), w4,
                           b1=np.ones(m, np.float32), b2=np.ones(m, np.float32), b3=b3, b4=-1.5)
    assert y.tolist() == [2.0 + 0.0 + 2.0 - 1.5] * 2


@pytest.mark.parametrize("alpha", [2.0, 0.25, 1024.0])
def test_predictor_positive_homogeneity(oracle_mod, alpha):
    """Bias-free Eq. 2 with ReLU is positively homogeneous: y(a h) = a y(h), a > 0.
    Power-of-two a keeps a*h exact in fp32, so only fp64 summation rounding remains."""
    pw = datagen.make_predictor_weights(1, 96, "f32", m1=64, m2=32, m3=16)
    h = datagen.make_hidden(1, 7, 96, "f32")
    y1 = oracle_mod.lenpred_weights(h, pw)
    y2 = oracle_mod.lenpred_weights((h * np.float32(alpha)).astype(np.float32), pw)
    np.testing.assert_allclose(y2, alpha * y1, rtol=1e-12)


def test_predictor_row_permutation_and_batch_independence(oracle_mod):
    pw = datagen.make_predictor_weights(2, 64, "bf16", m1=48, m2=32, m3=8)
    h = datagen.make_hidden(2, 9, 64, "bf16")
    y = oracle_mod.lenpred_weights(h, pw)
    perm = np.random.default_rng(0).permutation(9)
    assert np.array_equal(oracle_mod.lenpred_weights(h[perm], pw), y[perm])
    assert np.array_equal(oracle_mod.lenpred_weights(h[3:4], pw), y[3:4])


def test_predictor_matches_exact_rational_small(oracle_mod):
    """Brute force: exact rational evaluation of Eq. 2 on a small net; fp64 accumulation
    must agree to ~1e-13 relative (rounding of the fp64 sums only)."""
    pw = datagen.make_predictor_weights(4, 12, "bf16", m1=10, m2=6, m3=4)
    h = datagen.make_hidden(4, 3, 12, "bf16")
    y = oracle_mod.lenpred_weights(h, pw)

    def layer(W, x):
        return [max(Fraction(0), sum((Fraction(float(W[j, k])) * x[k] for k in range(len(x))), Fraction(0)))
                for j in range(W.shape[0])]

    for r in range(3):
        x = [Fraction(float(v)) for v in h[r]]
        z3 = layer(pw.W3, layer(pw.W2, layer(pw.W1, x)))
        exact = sum((Fraction(float(pw.w4[k])) * z3[k] for k in range(len(z3))), Fraction(0))
        assert abs(y[r] - float(exact)) <= 1e-12 * max(1.0, abs(float(exact)))


# =============================================================================== quantizer
def test_quantizer_ieee_pins(oracle_mod):
    """Reading A8-A10: round-half-even, clamp to [0, cap], NaN->0, +Inf->cap."""
    y = np.array([2.5, 3.5, -0.4, np.nan, np.inf, -np.inf, 0.49999997, 1e9, 7.5], np.float32)
    out = oracle_mod.quantize(y)
    assert out.tolist() == [2, 4, 0, 0, 32768, 0, 0, 32768, 8]
    n_tok = np.array([100, 32768, 40000, 0], np.int32)
    out2 = oracle_mod.quantize(np.array([40000, 5, 5, 32767.5], np.float32), n_tok)
    assert out2.tolist() == [32668, 0, 0, 32768]


# =============================================================================== projection
def test_projection_spec_examples(oracle_mod):
    g = _gold("spec_core.json")
    for ex in g["token_load"]:
        reqs = ex["requests"]
        n_tok = np.array([q["prompt"] + q["generated"] for q in reqs], np.int32)
        P = oracle_mod.project(np.zeros(len(reqs), np.int32), n_tok, np.full(len(reqs), 7, np.int32),
                               1, 3, datagen.beta_schedule_q16(3))
        assert P["L"][0, 0] == ex["expected"], ex["cite"]
    for ex in g["project_load"]:
        H = 6
        P = oracle_mod.project([0], [ex["prompt"] + ex["generated"]], [ex["n_hat"]], 1, H,
                               datagen.beta_schedule_q16(H))
        assert P["L"][0, ex["t"]] == ex["expected"], ex["cite"]


def test_projection_closed_form_all_long(oracle_mod):
    """Every N_hat > H: L[t] = L[0] + t*count, W = L0*S0[H] + count*S1[H] (S0 = sum beta_t,
    S1 = sum t beta_t, t=1..H); peak = L[H]; G = count*H."""
    g = datagen.rng(11)
    R, n, H = 57, 3, 20
    inst = g.integers(0, n, R)
    n_tok = g.integers(1, 5000, R)
    n_hat = g.integers(H + 1, 3000, R)
    beta = datagen.beta_schedule_q16(H)
    P = oracle_mod.project(inst, n_tok, n_hat, n, H, beta)
    S0 = sum(int(beta[t]) for t in range(1, H + 1))
    S1 = sum(t * int(beta[t]) for t in range(1, H + 1))
    for i in range(n):
        m = inst == i
        L0, c = int(n_tok[m].sum()), int(m.sum())
        assert P["L"][i].tolist() == [L0 + t * c for t in range(H + 1)]
        assert P["W"][i] == L0 * S0 + c * S1
        assert P["peak"][i] == L0 + H * c
        assert P["growth"][i] == c * H and P["count"][i] == c


def test_projection_all_finished_is_zero(oracle_mod):
    """every N_hat <= t -> projected load 0 at t."""
    P = oracle_mod.project([0, 0, 0], [5, 9, 11], [0, 1, 3], 1, 6, datagen.beta_schedule_q16(6))
    assert P["L"][0].tolist() == [25, 12, 13, 0, 0, 0, 0]   # only N=11 (N_hat=3) alive at t=1,2


@pytest.mark.parametrize("seed", range(30))
def test_projection_matches_brute(oracle_mod, seed):
    g = datagen.rng(100 + seed)
    n, H, R = int(g.integers(1, 6)), int(g.integers(0, 12)), int(g.integers(0, 40))
    inst = g.integers(0, n, R)
    n_tok = g.integers(1, 1 << 17, R)
    n_hat = g.integers(0, H + 4, R)
    beta = np.concatenate([[65536], g.integers(0, 65537, H)]).astype(np.uint32)
    P = oracle_mod.project(inst, n_tok, n_hat, n, H, beta)
    L = brute.project(n, H, inst, n_tok, n_hat)
    assert P["L"].tolist() == L
    for i in range(n):
        assert P["W"][i] == sum(int(beta[t]) * L[i][t] for t in range(1, H + 1))
        assert P["peak"][i] == max(L[i])
        m = inst == i
        assert P["growth"][i] == int(np.minimum(n_hat[m], H).sum())
        assert P["count"][i] == int(m.sum())


def test_projection_additive_and_unimodal(oracle_mod):
    """SPEC.md:114 additivity over disjoint batches; SPEC.md:117 each request's contribution
    grows by 1/step then drops to 0."""
    g = datagen.rng(5)
    H = 15
    beta = datagen.beta_schedule_q16(H)
    n_tok, n_hat = g.integers(1, 100, 30), g.integers(0, 25, 30)
    z = np.zeros(30, np.int32)
    A = oracle_mod.project(z[:13], n_tok[:13], n_hat[:13], 1, H, beta)["L"]
    B = oracle_mod.project(z[13:], n_tok[13:], n_hat[13:], 1, H, beta)["L"]
    AB = oracle_mod.project(z, n_tok, n_hat, 1, H, beta)["L"]
    assert np.array_equal(A + B, AB)
    for k in range(30):
        row = oracle_mod.project([0], [n_tok[k]], [n_hat[k]], 1, H, beta)["L"][0]
        alive = [t for t in range(1, H + 1) if row[t] > 0]
        assert alive == list(range(1, min(int(n_hat[k]), H + 1)))
        assert all(row[t] == n_tok[k] + t for t in alive)


def test_projection_inst_base_and_bad_ids(oracle_mod):
    beta = datagen.beta_schedule_q16(2)
    P = oracle_mod.project([4, 5, 4], [3, 4, 5], [9, 9, 9], 2, 2, beta, inst_base=4)
    assert P["L"].tolist() == [[8, 10, 12], [4, 5, 6]]
    with pytest.raises(ValueError):
        oracle_mod.project([3], [1], [1], 2, 2, beta, inst_base=4)


# =============================================================================== objective
def test_objective_spec_variance_examples(oracle_mod):
    g = _gold("spec_core.json")
    for ex in g["current_variance"]:
        loads = np.array(ex["loads"], np.int64)[:, None]
        n = loads.shape[0]
        phi = oracle_mod.objective(loads, np.array([65536], np.uint32))
        assert Fraction(phi, n * n * 65536) == Fraction(ex["expected_num"], ex["expected_den"]), ex["cite"]


@pytest.mark.parametrize("seed", range(20))
def test_objective_matches_brute_and_invariants(oracle_mod, seed):
    g = datagen.rng(200 + seed)
    n, H = int(g.integers(1, 7)), int(g.integers(0, 9))
    L = g.integers(0, 1 << 33, (n, H + 1))
    beta = np.concatenate([[65536], g.integers(0, 65537, H)]).astype(np.uint32)
    phi = oracle_mod.objective(L, beta)
    assert Fraction(phi, n * n * 65536) == brute.phi(L.tolist(), beta)
    assert phi >= 0
    assert oracle_mod.objective(L[np.random.default_rng(seed).permutation(n)], beta) == phi
    sym = np.repeat(L[:1], n, axis=0)
    assert oracle_mod.objective(sym, beta) == 0
    assert oracle_mod.objective(L[:, :1], beta[:1]) == oracle_mod.objective(L, beta, current_only=True)


# =============================================================================== plan
def _run_plan(oracle_mod, snap, n_hat, params):
    P = oracle_mod.project(snap.inst, snap.n_tok, n_hat, params.n_inst, params.H, params.beta_q)
    return P, oracle_mod.plan(params, P["L"], snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)


def test_plan_worked_example(oracle_mod):
    g = _gold("worked_example.json")
    rq = g["requests"]
    beta = np.array(g["beta_q"], np.uint32)
    P = oracle_mod.project(rq["inst"], rq["n_tok"], rq["n_hat"], g["n"], g["H"], beta)
    assert P["L"].tolist() == g["expected_L"]
    phi = oracle_mod.objective(P["L"], beta)
    assert phi == g["expected_phi_n2_q"] and Fraction(phi, 4 * 65536) == g["expected_phi_fraction"]
    for case in g["cases"]:
        params = datagen.PlanParams(n_inst=2, H=2, beta_q=beta, theta_num=g["theta_num"], theta_den=g["theta_den"],
                                    max_moves=1, c_mem=None if case["c_mem"] is None else np.array(case["c_mem"], np.int64),
                                    t_exec_a_ps=case["a_ps"], t_exec_b_ps=case["b_ps"],
                                    mig_c0_ps=case["c0_ps"], mig_c1_ps=case["c1_ps"])
        moves = oracle_mod.plan(params, P["L"], rq["req_id"], rq["inst"], rq["n_tok"], rq["n_hat"])
        assert [list(m) for m in moves] == case["expected_moves"], case["name"]
        assert brute.plan(params, rq["req_id"], rq["inst"], rq["n_tok"], rq["n_hat"]) == moves


def test_plan_classification_spec_fixture():
    """3 instances, one long request on instance 0, theta=0.1 -> O={0}, U={1,2};
    SPEC.md:249 symmetric -> O empty; SPEC.md:251 theta -> inf -> O empty."""
    H = 50
    beta = datagen.beta_schedule_q16(H)
    L = brute.project(3, H, [0], [500], [1000])
    O, U = brute.classify(L, beta, Fraction(1, 10))
    assert (O, U) == ([0], [1, 2])
    Ls = brute.project(3, H, [0, 1, 2], [7, 7, 7], [9, 9, 9])
    assert brute.classify(Ls, beta, Fraction(1, 10))[0] == []
    assert brute.classify(L, beta, Fraction(10 ** 9))[0] == []


@pytest.mark.parametrize("seed", range(220))
def test_plan_matches_brute_force(oracle_mod, seed):
    """SPEC.md:271/286/541: select_optimal equals exhaustive search on >=200 random fixtures
    with <=5 instances and <=20 requests, including tie-breaks and all flag modes."""
    g = datagen.rng(seed)
    n = int(g.integers(1, 6))
    R = int(g.integers(0, 21))
    H = int(g.integers(0, 7))
    snap, n_hat, params = datagen.tiny_fixture(1000 + seed, n, R, H)
    if seed % 7 == 0 and R >= 2:           # force exact ties: duplicate a request under a new id
        snap.n_tok[1], n_hat[1], snap.inst[1] = snap.n_tok[0], n_hat[0], snap.inst[0]
        snap.pinned[:2] = 0
    _, moves = _run_plan(oracle_mod, snap, n_hat, params)
    assert moves == brute.plan(params, snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)


def test_plan_tie_breaks():
    """Two identical requests -> lowest request id; two identical targets -> lowest dst."""
    import oracle
    H = 3
    beta = datagen.beta_schedule_q16(H)
    params = datagen.PlanParams(n_inst=3, H=H, beta_q=beta, max_moves=1, t_exec_a_ps=1, t_exec_b_ps=0,
                                mig_c0_ps=0, mig_c1_ps=0)
    inst = np.array([0, 0, 0, 0], np.int32)
    n_tok = np.array([50, 50, 50, 50], np.int32)
    n_hat = np.array([9, 9, 9, 9], np.int32)
    ids = np.array([40, 17, 23, 99], np.int32)
    P = oracle.project(inst, n_tok, n_hat, 3, H, beta)
    moves = oracle.plan(params, P["L"], ids, inst, n_tok, n_hat)
    assert [(m[0], m[1], m[2]) for m in moves] == [(17, 0, 1)]


@pytest.mark.parametrize("seed", range(40))
def test_plan_invariants(oracle_mod, seed):
    """Conservation of sum_i L_i[t] (north star), strict decrease of Phi per move,
    filters hold at decision time, reported gain = replayed Phi decrease,
    determinism."""
    g = datagen.rng(5000 + seed)
    n, R, H = int(g.integers(2, 7)), int(g.integers(5, 40)), int(g.integers(1, 10))
    snap, n_hat, params = datagen.tiny_fixture(7000 + seed, n, R, H)
    params.max_moves = 6
    cur = bool(params.flags & 2)
    P, moves = _run_plan(oracle_mod, snap, n_hat, params)
    assert moves == _run_plan(oracle_mod, snap, n_hat, params)[1]
    inst = snap.inst.copy()
    L = P["L"].copy()
    tot = L.sum(axis=0)
    idx = {int(r): k for k, r in enumerate(snap.req_id)}
    for (rid, s, t, rnd, gain) in moves:
        k = idx[rid]
        assert inst[k] == s and s != t and not snap.pinned[k]
        if not cur:
            assert n_hat[k] * (params.t_exec_a_ps + params.t_exec_b_ps * L[t, 0]) > \
                params.mig_c0_ps + params.mig_c1_ps * snap.n_tok[k]
        if params.c_mem is not None:
            need = L[t, 0] + (0 if cur else n_hat[k]) + \
                (0 if params.flags & 1 else int(params.reserved[t]) + int(snap.n_tok[k]))
            assert need <= params.c_mem[t]
        before = oracle_mod.objective(L, params.beta_q, cur)
        inst[k] = t
        L = oracle_mod.project(inst, snap.n_tok, n_hat, n, H, params.beta_q)["L"]
        after = oracle_mod.objective(L, params.beta_q, cur)
        assert gain == before - after and gain > 0
        assert np.array_equal(L.sum(axis=0), tot)


@pytest.mark.parametrize("seed", range(25))
def test_plan_local_optimum_and_optimal_bound(oracle_mod, seed):
    """Large max_moves ends at a local optimum over not-yet-moved requests;
    Phi(final) >= Phi(optimal assignment over all n^R placements) (brute force)."""
    g = datagen.rng(9000 + seed)
    n, R, H = int(g.integers(2, 4)), int(g.integers(2, 7)), int(g.integers(0, 5))
    snap, n_hat, params = datagen.tiny_fixture(9100 + seed, n, R, H, with_mem=False, with_cost=False)
    snap.pinned[:] = 0
    params.flags = 0
    params.max_moves = 50
    P, moves = _run_plan(oracle_mod, snap, n_hat, params)
    inst = snap.inst.copy()
    idx = {int(r): k for k, r in enumerate(snap.req_id)}
    for (rid, s, t, _, _) in moves:
        inst[idx[rid]] = t
    final_L = brute.project(n, H, inst, snap.n_tok, n_hat)
    opt = brute.optimal_assignment_phi(n, H, snap.n_tok, n_hat, params.beta_q)
    assert brute.phi(final_L, params.beta_q) >= opt
    # local optimality: no further positive-gain single move of an unmoved request
    moved = {idx[m[0]] for m in moves}
    keep = np.array([k not in moved for k in range(R)])
    if len(moves) < params.max_moves:
        p2 = datagen.PlanParams(**{**params.__dict__, "max_moves": 1})
        sub_pinned = (~keep).astype(np.uint8)
        L2 = oracle_mod.project(inst, snap.n_tok, n_hat, n, H, params.beta_q)["L"]
        assert oracle_mod.plan(p2, L2, snap.req_id, inst, snap.n_tok, n_hat, sub_pinned) == []


def test_plan_fixed_point_on_frozen_snapshot(oracle_mod):
    """repeated ticks on a frozen snapshot converge (no further decisions)."""
    snap = datagen.make_snapshot(3, 4, 16)
    n_hat = snap.true_rem.copy()
    params = datagen.make_plan_params(snap, H=50, mem_factor=10.0)
    params.mig_c1_ps = 0
    inst = snap.inst.copy()
    for tick in range(200):
        L = oracle_mod.project(inst, snap.n_tok, n_hat, 4, 50, params.beta_q)["L"]
        moves = oracle_mod.plan(params, L, snap.req_id, inst, snap.n_tok, n_hat)
        if not moves:
            break
        idx = {int(r): k for k, r in enumerate(snap.req_id)}
        for m in moves:
            inst[idx[m[0]]] = m[2]
    else:
        pytest.fail("no fixed point within 200 ticks")
    assert tick > 0


def test_plan_current_only_max_to_min(oracle_mod):
    """moving load c from the max- to the min-loaded instance with c < gap strictly
    decreases sigma0^2; in CURRENT_ONLY mode the plan finds such a move (reading A25)."""
    H = 4
    beta = datagen.beta_schedule_q16(H)
    inst = np.array([0, 0, 0, 1, 2], np.int32)
    n_tok = np.array([300, 200, 100, 120, 90], np.int32)
    n_hat = np.zeros(5, np.int32)   # no predictions in this mode
    params = datagen.PlanParams(n_inst=3, H=H, beta_q=beta, max_moves=1, flags=datagen.PlanParams.CURRENT_ONLY)
    P = oracle_mod.project(inst, n_tok, n_hat, 3, H, beta)
    moves = oracle_mod.plan(params, P["L"], np.arange(5, dtype=np.int32), inst, n_tok, n_hat)
    assert len(moves) == 1 and moves[0][1] == 0 and moves[0][2] == 2
    # plain H = 0 in predictive mode is NOT this baseline: w == 0 -> O empty
    p0 = datagen.PlanParams(n_inst=3, H=0, beta_q=beta[:1], max_moves=1)
    P0 = oracle_mod.project(inst, n_tok, n_hat, 3, 0, beta[:1])
    assert oracle_mod.plan(p0, P0["L"], np.arange(5, dtype=np.int32), inst, n_tok, n_hat) == []


# =============================================================================== P -> D dispatch (NEXT-2)
def test_dispatch_round_robin_spec_examples(oracle_mod):
    """counter 0, n 3 -> 0; counter 7, n 3 -> 1; 300 assignments -> 100 each."""
    L = np.zeros((3, 3), np.int64)
    beta = datagen.beta_schedule_q16(2)
    a, _ = oracle_mod.dispatch(0, L, beta, [5], [5], counter=0)
    assert a.tolist() == [0]
    a, _ = oracle_mod.dispatch(0, L, beta, [5], [5], counter=7)
    assert a.tolist() == [1]
    a, _ = oracle_mod.dispatch(0, L, beta, [5] * 300, [5] * 300, counter=0)
    assert np.bincount(a, minlength=3).tolist() == [100, 100, 100]


def test_dispatch_current_load_spec_examples(oracle_mod):
    """loads [500,200,900] -> 1; [200,200,900] -> 0 (lowest id); after assigning a
    request of N tokens the re-query sees the increased load (two-step fixture)."""
    beta = datagen.beta_schedule_q16(0)
    a, _ = oracle_mod.dispatch(1, np.array([[500], [200], [900]]), beta, [10], [1])
    assert a.tolist() == [1]
    a, _ = oracle_mod.dispatch(1, np.array([[200], [200], [900]]), beta, [10], [1])
    assert a.tolist() == [0]
    a, L = oracle_mod.dispatch(1, np.array([[200], [150], [900]]), beta, [100, 10], [1, 1])
    assert a.tolist() == [1, 0] and L[:, 0].tolist() == [210, 250, 900]


def test_dispatch_projected_closed_forms(oracle_mod):
    """Projected policy (reading A28): (i) with N_hat <= 1 only t = 0 carries the request, so the
    choice is the current-load argmin; (ii) identical instances -> lowest id; (iii) a long request
    avoids the instance whose FUTURE load is high even though its current load is lower
    (the paper's point: current load alone misleads)."""
    beta = datagen.beta_schedule_q16(4)
    L = np.array([[300, 0, 0, 0, 0], [100, 100, 100, 100, 100], [200, 10, 10, 10, 10]], np.int64)
    a, _ = oracle_mod.dispatch(2, L, beta, [50], [1])
    assert a.tolist() == [1]                                    # (i) argmin L[0]
    a, _ = oracle_mod.dispatch(2, np.zeros((3, 5), np.int64), beta, [50], [9])
    assert a.tolist() == [0]                                    # (ii)
    a, _ = oracle_mod.dispatch(2, L, beta, [50], [100])
    assert a.tolist() == [2]                                    # (iii) hand-checked below
    # hand check of (iii): score_i = sum_t beta_t (50+t) L_i[t] over t = 0..4
    sc = [sum(int(beta[t]) * (50 + t) * int(L[i][t]) for t in range(5)) for i in range(3)]
    assert int(np.argmin(sc)) == 2
    # memory filter (reading A18): 200 + 50 + 100 = 350 > 349 excludes instance 2 -> next best (0)
    a, _ = oracle_mod.dispatch(2, L, beta, [50], [100], c_mem=np.array([10**9, 10**9, 349]))
    assert a.tolist() == [0]
    a, _ = oracle_mod.dispatch(2, L, beta, [50], [100], c_mem=np.array([10**9, 10**9, 350]))
    assert a.tolist() == [2]                                    # boundary: exactly C_mem is admitted
    a, L2 = oracle_mod.dispatch(2, L, beta, [50], [100], c_mem=np.array([1, 1, 1]))
    assert a.tolist() == [-1] and np.array_equal(L2, L)       # nowhere feasible: not placed


@pytest.mark.parametrize("seed", range(60))
def test_dispatch_matches_brute_force(oracle_mod, seed):
    """Exact-integer oracle == exact-rational brute force (real beta, textbook variance) on tiny
    random batches, all three policies, with and without the memory filter."""
    g = datagen.rng(7000 + seed)
    n, H, A = int(g.integers(1, 5)), int(g.integers(0, 6)), int(g.integers(0, 8))
    L = g.integers(0, 200, (n, H + 1)).astype(np.int64)
    beta = np.concatenate([[65536], g.integers(1, 65537, H)]).astype(np.uint32)
    n_tok = g.integers(1, 60, A).astype(np.int32)
    n_hat = g.integers(0, H + 3, A).astype(np.int32)
    c_mem = g.integers(100, 600, n).astype(np.int64) if seed % 2 else None
    reserved = g.integers(0, 50, n).astype(np.int64) if seed % 3 == 0 else None
    for policy in (0, 1, 2):
        a, L_o = oracle_mod.dispatch(policy, L, beta, n_tok, n_hat, c_mem, reserved, counter=seed)
        b, L_b = brute.dispatch(policy, L, beta, n_tok, n_hat, c_mem, reserved, counter=seed)
        assert a.tolist() == b
        assert L_o.tolist() == L_b


# =============================================================================== prediction cadence (NEXT-1)
def test_should_refresh_spec_examples(oracle_mod):
    """(last 100, gen 120, k 20) -> true; (100, 119, 20) -> false; fresh -> true."""
    assert oracle_mod.should_refresh([120], [100], 20).tolist() == [True]
    assert oracle_mod.should_refresh([119], [100], 20).tolist() == [False]
    assert oracle_mod.should_refresh([0], [-1], 20).tolist() == [True]


def test_prediction_overhead_formula():
    """PAPER.md:466-469 / SPEC.md:180-183: overhead = 1.40 / (18.23 k): 7.68% at k=1, 0.38% at k=20."""
    ov = lambda k: 1.40 / (18.23 * k)
    assert round(100 * ov(1), 2) == 7.68
    assert round(100 * ov(20), 2) == 0.38
    assert abs(ov(10) - 2 * ov(20)) < 1e-15


def test_refresh_schedule_and_aging(oracle_mod):
    """over a request's lifetime the refresh fires ceil(L/k) times (the initial
    prediction included); between refreshes the prediction ages one token per generated token
    and never goes negative."""
    pw = datagen.make_predictor_weights(0, 16, "f32", m1=32, m2=16, m3=8)
    k, L_out = 20, 93
    h = datagen.make_hidden(0, 1, 16, "f32")
    g_last, nhat_last = np.array([-1], np.int32), np.array([0], np.int32)
    fires, prev = 0, None
    for g in range(L_out):
        nh, g_last, nhat_last, due = oracle_mod.refresh_step(h, pw, [10 + g], [g], g_last, nhat_last, k)
        fires += int(due[0])
        if not due[0]:
            assert nh[0] == max(0, prev - 1)
        assert nh[0] >= 0
        prev = int(nh[0])
    assert fires == -(-L_out // k)


# ============================================================================ KV migration (NEXT-4)
def test_kv_oracle_hand_example(oracle_mod):
    """2 layers x 4 blocks of 2 bytes; the request owns blocks [3, 0] at the source and gets blocks
    [1, 2] at the destination (worked by hand)."""
    src = np.arange(16, dtype=np.uint8).reshape(2, 4, 2)      # layer l, block b holds (8l+2b, 8l+2b+1)
    stg = oracle_mod.kv_pack(src, [3, 0])
    assert stg.tolist() == [[[6, 7], [0, 1]], [[14, 15], [8, 9]]]
    dst = np.full((2, 4, 2), 255, np.uint8)
    out = oracle_mod.kv_unpack(stg, dst, [1, 2])
    assert out.tolist() == [[[255, 255], [6, 7], [0, 1], [255, 255]], [[255, 255], [14, 15], [8, 9], [255, 255]]]
    assert np.array_equal(oracle_mod.kv_migrate(src, [3, 0], dst, [1, 2]), out)


def test_kv_oracle_invariants(oracle_mod):
    g = np.random.default_rng(0)
    pool = g.integers(0, 256, (3, 10, 32), dtype=np.uint8)
    ident = list(range(10))
    assert np.array_equal(oracle_mod.kv_pack(pool, ident), pool)                     # identity table
    perm = g.permutation(10)
    stg = oracle_mod.kv_pack(pool, perm)
    back = oracle_mod.kv_unpack(stg, np.zeros_like(pool), perm)                       # round trip
    assert np.array_equal(back, pool)
    # untouched destination blocks keep their bytes; the bytes moved are conserved as a multiset
    dst = g.integers(0, 256, (3, 10, 32), dtype=np.uint8)
    out = oracle_mod.kv_migrate(pool, perm[:4], dst, [9, 0, 5, 2])
    keep = [b for b in range(10) if b not in (9, 0, 5, 2)]
    assert np.array_equal(out[:, keep], dst[:, keep])
    assert np.array_equal(np.sort(out[:, [9, 0, 5, 2]].ravel()), np.sort(pool[:, perm[:4]].ravel()))
