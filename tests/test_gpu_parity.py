"""GPU parity tests (`-m gpu`, B200 only): the CUDA path, called through the C ABI, against
the CPU oracle on the same seeded inputs.  Bars (BASELINE.json north_star):
  * predictor: max_r |y_gpu - y_ref| / max(|y_ref|, 1) <= 1e-3 (fp32) / 2e-2 (bf16)  (reading A7)
  * quantizer, projected loads, plans: bit-exact (plans on the oracle's N_hat)."""
import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-3, "bf16": 2e-2}


@pytest.fixture(scope="module")
def star():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2510_13668_b200 as star
    star.version()   # loads libstar.so; raises if missing
    return star


def _dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _weights_dev(pw, biases=False):
    tdt = torch.bfloat16 if pw.dtype == "bf16" else torch.float32
    W = [_dev(pw.W1, tdt), _dev(pw.W2, tdt), _dev(pw.W3, tdt), _dev(pw.w4)]
    b = [None] * 4
    if biases:
        b = [_dev(pw.b1), _dev(pw.b2), _dev(pw.b3), _dev(np.array([pw.b4], np.float32))]
    return W, b


def _rel_err(y, ref):
    return float(np.max(np.abs(y.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1.0)))


# ============================================================================ quantizer
def test_quantizer_bitexact(star, oracle_mod):
    g = datagen.rng(1)
    y = np.concatenate([g.normal(3000, 8000, 5000).astype(np.float32),
                        np.array([2.5, 3.5, -0.4, np.nan, np.inf, -np.inf, 32767.5, 1e30, -0.0, 0.5],
                                 np.float32)])
    y[:200] = np.round(y[:200]) + 0.5   # exact halves
    n_tok = g.integers(1, 40000, y.shape[0]).astype(np.int32)
    for nt in (None, n_tok):
        ref = oracle_mod.quantize(y, nt)
        got = star.lenpred_quantize(_dev(y), None if nt is None else _dev(nt)).cpu().numpy()
        assert np.array_equal(got, ref)


# ============================================================================ projection
@pytest.mark.parametrize("seed,n,R,H", [(0, 1, 0, 50), (1, 1, 1, 50), (2, 8, 2048, 50), (3, 8, 4096, 50),
                                       (4, 3, 1001, 7), (5, 5, 333, 0), (6, 64, 12345, 50), (7, 2, 77, 256),
                                       (8, 8, 300_000, 50), (9, 300, 50_000, 50), (10, 32, 1_000_003, 50),
                                       (11, 32, (1 << 20) + 1, 20), (12, 150, 600_001, 50)])
def test_projection_bitexact(star, oracle_mod, seed, n, R, H):
    snap = datagen.make_snapshot(seed, n, max(R // n, 1))
    g = datagen.rng(seed)
    if R != snap.R:
        idx = g.integers(0, snap.R, R) if snap.R else np.zeros(0, np.int64)
        inst, n_tok, n_hat = snap.inst[idx], snap.n_tok[idx], snap.true_rem[idx]
    else:
        inst, n_tok, n_hat = snap.inst, snap.n_tok, snap.true_rem
    n_hat = np.where(g.random(R) < 0.2, g.integers(0, H + 3, R), n_hat).astype(np.int32)
    beta = datagen.beta_schedule_q16(H)
    ref = oracle_mod.project(inst, n_tok, n_hat, n, H, beta)
    ws = torch.zeros(star.project_workspace_bytes(n, H), dtype=torch.uint8, device="cuda")
    for use_ws in (False, True) if n * (H + 2) <= 16384 else (True,):
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        out = star.project_instance_load(_dev(inst.astype(np.int32)), _dev(n_tok), _dev(n_hat), n, H,
                                         _dev(beta.astype(np.int32)), workspace=ws if use_ws else None,
                                         err_flag=err)
        torch.cuda.synchronize()
        assert err.item() == 0
        assert np.array_equal(out.L.cpu().numpy(), ref["L"])
        for k in ("W", "peak", "growth", "count"):
            assert np.array_equal(getattr(out, k).cpu().numpy(), ref[k]), k
    assert int(ws.sum().item()) == 0   # workspace left zeroed


@pytest.mark.parametrize("seed,n,R,H,grouped,base", [(20, 256, (1 << 20) + 3, 50, True, 0),
                                                    (21, 200, 300_001, 50, False, 0),
                                                    (22, 96, 500_000, 50, True, 1000),
                                                    (23, 40, 400_002, 256, True, 0),
                                                    (24, 64, 262_144, 50, False, 0)])
def test_projection_stream_window(star, oracle_mod, seed, n, R, H, grouped, base):
    """Bandwidth form (R >= 2^18): shared-memory bins over a window of instances, requests of
    instances outside the window added to the global workspace; grouped and interleaved orders,
    a nonzero inst_base, H = 256 -- bit-exact against the oracle."""
    g = datagen.rng(seed)
    snap = datagen.make_snapshot(seed, 8, 256)
    idx = g.integers(0, snap.R, R)
    inst = g.integers(0, n, R).astype(np.int32)
    if grouped:
        inst = np.sort(inst).astype(np.int32)
    n_tok, n_hat = snap.n_tok[idx], snap.true_rem[idx].astype(np.int32)
    n_hat = np.where(g.random(R) < 0.2, g.integers(0, H + 3, R), n_hat).astype(np.int32)
    beta = datagen.beta_schedule_q16(H)
    ref = oracle_mod.project(inst, n_tok, n_hat, n, H, beta)
    ws = torch.zeros(star.project_workspace_bytes(n, H), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(2):   # the workspace is left zeroed and reused
        out = star.project_instance_load(_dev(inst + base), _dev(n_tok), _dev(n_hat), n, H,
                                         _dev(beta.astype(np.int32)), inst_base=base, workspace=ws, err_flag=err)
        torch.cuda.synchronize()
        assert err.item() == 0
        assert np.array_equal(out.L.cpu().numpy(), ref["L"])
        for k in ("W", "peak", "growth", "count"):
            assert np.array_equal(getattr(out, k).cpu().numpy(), ref[k]), k
    assert int(ws.sum().item()) == 0


def test_projection_inst_base_and_errors(star, oracle_mod):
    inst = np.array([4, 5, 4, 9, 5], np.int32)
    n_tok = np.array([3, 4, 5, 6, 0], np.int32)   # inst 9 out of range, N=0 invalid
    n_hat = np.array([9, 9, 9, 9, 9], np.int32)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    beta = datagen.beta_schedule_q16(2).astype(np.int32)
    out = star.project_instance_load(_dev(inst), _dev(n_tok), _dev(n_hat), 2, 2, _dev(beta), inst_base=4,
                                     err_flag=err)
    torch.cuda.synchronize()
    assert out.L.cpu().numpy().tolist() == [[8, 10, 12], [4, 5, 6]]   # invalid rows ignored
    assert err.item() & 1 and err.item() & 2


@pytest.mark.parametrize("R,n,grouped", [(300_003, 8, True), (400_000, 200, False)])
def test_projection_bandwidth_form_errors(star, oracle_mod, R, n, grouped):
    """Bandwidth form (R >= 2^18) with invalid rows (instance out of range, N = 0, N > 2^17,
    N_hat < 0) scattered through the batch, incl. the R % 4 tail: every invalid row is skipped
    and flagged in err_flag (bits 1 / 2 / 4), the valid rows project bit-exactly."""
    g = datagen.rng(R)
    snap = datagen.make_snapshot(3, 8, 256)
    idx = g.integers(0, snap.R, R)
    inst = g.integers(0, n, R).astype(np.int32)
    if grouped:
        inst = np.sort(inst).astype(np.int32)
    n_tok, n_hat = snap.n_tok[idx].copy(), snap.true_rem[idx].astype(np.int32)
    bad = g.choice(R - 3, 40, replace=False)
    bad = np.concatenate([bad, [R - 1, R - 2]])   # two in the R % 4 tail
    kinds = np.arange(len(bad)) % 4
    inst[bad[kinds == 0]] = n + 5
    n_tok[bad[kinds == 1]] = 0
    n_tok[bad[kinds == 2]] = (1 << 17) + 1
    n_hat[bad[kinds == 3]] = -3
    ok = np.ones(R, bool)
    ok[bad] = False
    beta = datagen.beta_schedule_q16(50)
    ref = oracle_mod.project(inst[ok], n_tok[ok], n_hat[ok], n, 50, beta)
    ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = star.project_instance_load(_dev(inst), _dev(n_tok), _dev(n_hat), n, 50, _dev(beta.astype(np.int32)),
                                     workspace=ws, err_flag=err)
    torch.cuda.synchronize()
    assert err.item() & 7 == 7
    assert np.array_equal(out.L.cpu().numpy(), ref["L"])
    for k in ("W", "peak", "growth", "count"):
        assert np.array_equal(getattr(out, k).cpu().numpy(), ref[k]), k
    assert int(ws.sum().item()) == 0


# ============================================================================ plan
def _plan_gpu(star, params_h, L, snap, n_hat):
    pp = star.PlanParams.from_host(params_h)
    moves, nm = star.plan_reschedule(pp, _dev(L), _dev(snap.req_id), _dev(snap.inst), _dev(snap.n_tok),
                                     _dev(n_hat.astype(np.int32)), _dev(snap.pinned))
    torch.cuda.synchronize()
    return star.decode_moves(moves, nm)


@pytest.mark.parametrize("seed", range(240))
def test_plan_bitexact_tiny(star, oracle_mod, seed):
    g = datagen.rng(seed)
    n, R, H = int(g.integers(1, 7)), int(g.integers(0, 30)), int(g.integers(0, 9))
    snap, n_hat, params = datagen.tiny_fixture(3000 + seed, n, R, H)
    if seed % 5 == 0 and R >= 2:
        snap.n_tok[1], n_hat[1], snap.inst[1] = snap.n_tok[0], n_hat[0], snap.inst[0]
        snap.pinned[:2] = 0
    params.max_moves = int(g.integers(0, 6))
    L = oracle_mod.project(snap.inst, snap.n_tok, n_hat, n, H, params.beta_q)["L"]
    ref = oracle_mod.plan(params, L, snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)
    assert _plan_gpu(star, params, L, snap, n_hat) == ref


@pytest.mark.parametrize("cfg,seed,flags", [("C1", 0, 0), ("C2", 1, 0), ("C3", 2, 0), ("C4", 3, 0), ("TGT", 4, 0),
                                            ("C2", 5, 1), ("C4", 6, 2), ("C4", 7, 3), ("TGT", 0, 0), ("TGT", 8, 1),
                                            ("TGT", 9, 0), ("C3", 10, 1)])
def test_plan_bitexact_full_configs(star, oracle_mod, cfg, seed, flags):
    c = datagen.CONFIGS[cfg]
    snap = datagen.make_snapshot(seed, c["n_inst"], c["r_per_inst"], skewed=c.get("skewed", False),
                                 pinned_frac=0.05)
    n_hat = snap.true_rem.copy()   # STAR-Oracle predictions (north-star parity rule)
    params = datagen.make_plan_params(snap, mem_factor=c.get("mem_factor", 1.10), max_moves=max(c["max_moves"], 4),
                                      flags=flags, reserved_seed=seed)
    L = oracle_mod.project(snap.inst, snap.n_tok, n_hat, snap.n_inst, params.H, params.beta_q)["L"]
    ref = oracle_mod.plan(params, L, snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)
    if c.get("skewed") and flags == 0:
        assert len(ref) >= 1   # the skewed configs put Alg. 1 past Phase 1: candidates scored, moves made
    assert _plan_gpu(star, params, L, snap, n_hat) == ref


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_segmented_equals_contiguous(star, oracle_mod, world):
    """c9: the plan over gathered per-rank records equals the plan on the concatenated state."""
    n_loc, r_per = 8 // world, 96
    snap = datagen.make_snapshot(11, 8, r_per)
    n_hat = snap.true_rem.astype(np.int32)
    params = datagen.make_plan_params(snap, max_moves=4)
    H = params.H
    order = np.argsort(snap.inst, kind="stable")   # group requests by owning rank
    inst, n_tok, ids, pin, nh = (a[order] for a in (snap.inst, snap.n_tok, snap.req_id, snap.pinned, n_hat))
    L = oracle_mod.project(inst, n_tok, nh, 8, H, params.beta_q)["L"]
    ref = oracle_mod.plan(params, L, ids, inst, n_tok, nh, pin)
    # build a [world][record] buffer: L block | count | req_id | inst | n_tok | n_hat | pinned
    r_cap = r_per * n_loc + 5
    rec_i64 = n_loc * (H + 1) + 1 + (4 * r_cap + (r_cap + 7) // 8 * 2 + 1) // 2 + 1
    buf = np.zeros((world, rec_i64), np.int64)
    offs = {}
    for k in range(world):
        sel = (inst >= k * n_loc) & (inst < (k + 1) * n_loc)
        cnt = int(sel.sum())
        rec = buf[k].view(np.uint8)
        o = 0
        rec[o:o + 8 * n_loc * (H + 1)] = L[k * n_loc:(k + 1) * n_loc].reshape(-1).view(np.uint8); offs["L"] = o
        o += 8 * n_loc * (H + 1)
        rec[o:o + 4] = np.array([cnt], np.int32).view(np.uint8); offs["cnt"] = o; o += 8
        for name, arr in (("id", ids), ("inst", inst), ("ntok", n_tok), ("nhat", nh)):
            v = np.zeros(r_cap, np.int32)
            v[:cnt] = arr[sel]
            rec[o:o + 4 * r_cap] = v.view(np.uint8); offs[name] = o; o += 4 * r_cap
        v = np.zeros(r_cap, np.uint8)
        v[:cnt] = pin[sel]
        rec[o:o + r_cap] = v; offs["pin"] = o
    d = _dev(buf)
    base = d.data_ptr()
    seg = star._lib.PlanSegmentsC(world, n_loc, r_cap, rec_i64 * 8, base + offs["L"], base + offs["cnt"],
                                  base + offs["id"], base + offs["inst"], base + offs["ntok"], base + offs["nhat"],
                                  base + offs["pin"])
    pp = star.PlanParams.from_host(params)
    moves, nm = star.plan_reschedule_segmented(pp, seg)
    torch.cuda.synchronize()
    assert star.decode_moves(moves, nm) == ref


@pytest.mark.parametrize("world,r_cap", [(4, 60000), (8, 20000)])
def test_plan_large_segmented_many_slots(star, oracle_mod, world, r_cap):
    """The cluster-scale plan over gathered records whose capacity far exceeds their requests:
    240k / 160k slots (several strided slot chunks per CTA of the scan, the later ones loaded
    inside the chunk loop), 96 requests per rank at the front of each segment, 4 moves; == the
    oracle on the concatenated state."""
    n_loc, r_per = 8 // world, 96
    snap = datagen.make_snapshot(31, 8, r_per)
    n_hat = snap.true_rem.astype(np.int32)
    params = datagen.make_plan_params(snap, max_moves=4)
    H = params.H
    order = np.argsort(snap.inst, kind="stable")
    inst, n_tok, ids, pin, nh = (a[order] for a in (snap.inst, snap.n_tok, snap.req_id, snap.pinned, n_hat))
    L = oracle_mod.project(inst, n_tok, nh, 8, H, params.beta_q)["L"]
    ref = oracle_mod.plan(params, L, ids, inst, n_tok, nh, pin)
    assert len(ref) > 0
    rec_i64 = n_loc * (H + 1) + 1 + (4 * r_cap + (r_cap + 7) // 8 * 2 + 1) // 2 + 1
    buf = np.zeros((world, rec_i64), np.int64)
    offs = {}
    for k in range(world):
        sel = (inst >= k * n_loc) & (inst < (k + 1) * n_loc)
        cnt = int(sel.sum())
        rec = buf[k].view(np.uint8)
        o = 0
        rec[o:o + 8 * n_loc * (H + 1)] = L[k * n_loc:(k + 1) * n_loc].reshape(-1).view(np.uint8); offs["L"] = o
        o += 8 * n_loc * (H + 1)
        rec[o:o + 4] = np.array([cnt], np.int32).view(np.uint8); offs["cnt"] = o; o += 8
        for name, arr in (("id", ids), ("inst", inst), ("ntok", n_tok), ("nhat", nh)):
            v = np.zeros(r_cap, np.int32)
            v[:cnt] = arr[sel]
            rec[o:o + 4 * r_cap] = v.view(np.uint8); offs[name] = o; o += 4 * r_cap
        v = np.zeros(r_cap, np.uint8)
        v[:cnt] = pin[sel]
        rec[o:o + r_cap] = v; offs["pin"] = o
    d = _dev(buf)
    base = d.data_ptr()
    seg = star._lib.PlanSegmentsC(world, n_loc, r_cap, rec_i64 * 8, base + offs["L"], base + offs["cnt"],
                                  base + offs["id"], base + offs["inst"], base + offs["ntok"], base + offs["nhat"],
                                  base + offs["pin"])
    pp = star.PlanParams.from_host(params)
    ws = torch.empty(star.plan_workspace_bytes(8, H, world * r_cap), dtype=torch.uint8, device="cuda")
    moves, nm = star.plan_reschedule_segmented_ws(pp, seg, ws)
    torch.cuda.synchronize()
    assert star.decode_moves(moves, nm) == ref


# ============================================================================ predictor
def _predict(star, pw, h, biases=False, n_tok=None, max_rows=None):
    W, b = _weights_dev(pw, biases)
    pred = star.Predictor(*W, *b, max_rows=max_rows or max(h.shape[0], 1))
    tdt = torch.bfloat16 if pw.dtype == "bf16" else torch.float32
    y, nh = star.lenpred_forward(pred, _dev(h, tdt), None if n_tok is None else _dev(n_tok))
    torch.cuda.synchronize()
    return pred, y.cpu().numpy(), nh.cpu().numpy()


@pytest.mark.parametrize("d,dtype,R,biases", [(896, "f32", 128, False), (896, "f32", 333, True),
                                              (4096, "bf16", 300, False), (4096, "bf16", 129, True),
                                              (5120, "bf16", 257, False), (1024, "bf16", 1, False),
                                              (896, "bf16", 640, False),
                                              # layer 1 as 9 non-uniform column tiles (6-8 row pairs):
                                              # odd m-tile count (phantom rows) and a ragged last tile
                                              (4096, "bf16", 1300, True), (4096, "bf16", 1537, False),
                                              # hidden sizes that are multiples of 8 only (the last K block
                                              # is partly out of bounds: TMA zero fill)
                                              (72, "bf16", 50, True), (520, "bf16", 700, False),
                                              (200, "f32", 33, False), (104, "f32", 128, True)])
def test_predictor_parity(star, oracle_mod, d, dtype, R, biases):
    pw = datagen.make_predictor_weights(d, d, dtype, biases=biases)
    h = datagen.make_hidden(d + 1, R, d, dtype)
    n_tok = datagen.make_snapshot(d, 1, R).n_tok
    _, y, nh = _predict(star, pw, h, biases, n_tok)
    ref = oracle_mod.lenpred_weights(h, pw)
    err = _rel_err(y, ref)
    assert err <= TOL[dtype], f"max rel err {err:.3e}"
    # the forward's quantizer equals the oracle quantizer on the GPU's own fp32 y_hat
    assert np.array_equal(nh, oracle_mod.quantize(y, n_tok))


@pytest.mark.parametrize("d,dtype,m1,m2,R", [(512, "bf16", 1024, 256, 300), (1024, "bf16", 768, 512, 700),
                                             (256, "f32", 512, 256, 100), (384, "f32", 384, 128, 200)])
def test_predictor_parity_other_widths(star, oracle_mod, d, dtype, m1, m2, R):
    """Eq. 2 with hidden widths other than the paper's 2048 / 512 (star.h: m1, m2 multiples of 256
    for bf16, 128 for fp32; m3 = 64): the general kernels, against the fp64 oracle."""
    pw = datagen.make_predictor_weights(d + m1, d, dtype, m1=m1, m2=m2)
    h = datagen.make_hidden(d + 3, R, d, dtype)
    n_tok = datagen.make_snapshot(d, 1, R).n_tok
    pred, y, nh = _predict(star, pw, h, False, n_tok)
    assert pred.path(R) == 0
    err = _rel_err(y, oracle_mod.lenpred_weights(h, pw))
    assert err <= TOL[dtype], f"max rel err {err:.3e}"
    assert np.array_equal(nh, oracle_mod.quantize(y, n_tok))
    pred.close()


@pytest.mark.parametrize("cfg,R", [("C2", 2048), ("C3", 4096), ("C4", 4096), ("TGT", 4096), ("TGT", 512),
                                   ("C2", 256)])
def test_predictor_full_size_all_rows(star, oracle_mod, cfg, R):
    """Full BASELINE sizes (and the per-rank sizes of the W = 8 jobs) in the bench's launch
    configuration, EVERY row against the fp64 oracle; N_hat == the oracle quantizer of the GPU's
    own y_hat on every row."""
    c = datagen.CONFIGS[cfg]
    pw = datagen.make_predictor_weights(0, c["d"], c["dtype"])
    snap = datagen.make_snapshot(0, c["n_inst"], (R + c["n_inst"] - 1) // c["n_inst"],
                                 skewed=c.get("skewed", False))
    scale = np.maximum(snap.true_rem[:R], 1).astype(np.float32) / 60.0   # long-tailed, as in the bench
    h = datagen.make_hidden(0, R, c["d"], c["dtype"], scale=scale)
    pred, y, nh = _predict(star, pw, h, n_tok=snap.n_tok[:R])
    # the per-rank sizes run the one-launch small-batch kernel on a B200, the rest the 2-launch path
    assert pred.path(R) == (1 if R <= 512 else 0)
    ref = oracle_mod.lenpred_weights(h, pw)
    err = _rel_err(y, ref)
    assert err <= TOL[c["dtype"]], f"max rel err {err:.3e} over all {R} rows"
    assert np.array_equal(nh, oracle_mod.quantize(y, snap.n_tok[:R]))


def test_predictor_homogeneity_bitexact(star):
    """Pin (ii): bias-free Eq. 2 is positively homogeneous; scaling h by 2 scales every
    product, partial sum and bf16 rounding by 2, so y(2h) == 2 y(h) bit for bit."""
    pw = datagen.make_predictor_weights(3, 4096, "bf16")
    h = datagen.make_hidden(3, 700, 4096, "bf16")
    pred, y1, _ = _predict(star, pw, h, max_rows=700)
    y2, _ = star.lenpred_forward(pred, _dev(h * 2, torch.bfloat16))
    assert np.array_equal(y2.cpu().numpy(), 2 * y1)


def test_predictor_deterministic_and_row_independent(star):
    pw = datagen.make_predictor_weights(4, 4096, "bf16")
    h = datagen.make_hidden(4, 512, 4096, "bf16")
    pred, y1, _ = _predict(star, pw, h, max_rows=512)
    y2, _ = star.lenpred_forward(pred, _dev(h, torch.bfloat16))
    assert np.array_equal(y2.cpu().numpy(), y1)                      # run-to-run (fixed-order split-K)
    perm = datagen.rng(0).permutation(512)
    y3, _ = star.lenpred_forward(pred, _dev(h[perm], torch.bfloat16))
    np.testing.assert_allclose(y3.cpu().numpy(), y1[perm], rtol=1e-5)  # rows independent


def test_fused_step_projection_equals_oracle(star, oracle_mod):
    """Fused = standalone: the projection of the GPU predictor's own N_hat equals the oracle
    projection of that N_hat bit for bit (c3 pin)."""
    c = datagen.CONFIGS["C2"]
    snap = datagen.make_snapshot(5, c["n_inst"], c["r_per_inst"])
    pw = datagen.make_predictor_weights(5, c["d"], "bf16")
    h = datagen.make_hidden(5, snap.R, c["d"], "bf16")
    _, _, nh = _predict(star, pw, h, n_tok=snap.n_tok)
    beta = datagen.beta_schedule_q16(50)
    out = star.project_instance_load(_dev(snap.inst), _dev(snap.n_tok), _dev(nh), c["n_inst"], 50,
                                     _dev(beta.astype(np.int32)))
    ref = oracle_mod.project(snap.inst, snap.n_tok, nh, c["n_inst"], 50, beta)
    assert np.array_equal(out.L.cpu().numpy(), ref["L"])


# ============================================================================ fused forward+projection
@pytest.mark.parametrize("cfg,R,seed", [("C2", 2048, 0), ("C2", 2047, 1), ("C2", 1, 2), ("C2", 100, 3),
                                        ("C3", 4096, 4), ("TGT", 512, 5), ("C2", 256, 6), ("C1", 128, 7),
                                        ("C4", 4096, 8), ("C2", 3000, 9), ("C2", 8192, 10)])
def test_fused_forward_project_equals_standalone(star, oracle_mod, cfg, R, seed):
    """lenpred_forward_project == lenpred_forward + project_instance_load, bit for bit (y_hat,
    N_hat, L, W, peak, growth, count), and its projection equals the oracle projection of the
    GPU's own N_hat (c3 "fused = standalone" pin).  Ragged R (not a multiple of 128) included."""
    c = datagen.CONFIGS[cfg]
    n = c["n_inst"]
    snap = datagen.make_snapshot(seed, n, (R + n - 1) // n)
    inst, n_tok = snap.inst[:R].copy(), snap.n_tok[:R].copy()
    pw = datagen.make_predictor_weights(seed, c["d"], c["dtype"], biases=(seed % 2 == 1))
    scale = np.exp(datagen.rng(seed).normal(0.0, 1.5, R)).astype(np.float32)   # long-tailed N_hat
    h = datagen.make_hidden(seed, R, c["d"], c["dtype"], scale=scale)
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    W, b = _weights_dev(pw, biases=(seed % 2 == 1))
    pred = star.Predictor(*W, *b, max_rows=R)
    H = 50
    beta = datagen.beta_schedule_q16(H)
    bq = _dev(beta.astype(np.int32))
    hd, ntd, ind = _dev(h, tdt), _dev(n_tok), _dev(inst)
    ws = torch.zeros(star.project_workspace_bytes(n, H), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    y1, nh1, out1 = star.lenpred_forward_project(pred, hd, ntd, ind, n, H, bq, ws, err_flag=err)
    y2, nh2 = star.lenpred_forward(pred, hd, ntd)
    out2 = star.project_instance_load(ind, ntd, nh2, n, H, bq)
    torch.cuda.synchronize()
    assert err.item() == 0
    assert np.array_equal(y1.cpu().numpy(), y2.cpu().numpy())
    assert np.array_equal(nh1.cpu().numpy(), nh2.cpu().numpy())
    for k in ("L", "W", "peak", "growth", "count"):
        assert np.array_equal(getattr(out1, k).cpu().numpy(), getattr(out2, k).cpu().numpy()), k
    ref = oracle_mod.project(inst, n_tok, nh1.cpu().numpy(), n, H, beta)
    for k in ("L", "W", "peak", "growth", "count"):
        assert np.array_equal(getattr(out1, k).cpu().numpy(), ref[k]), k
    assert int(ws.sum().item()) == 0
    # predictor parity on sampled rows (full-size case) against the fp64 oracle
    rows = np.unique(np.concatenate([datagen.rng(seed + 1).integers(0, R, 24), [0, R - 1]]))
    y_ref = oracle_mod.lenpred_weights(h[rows], pw)
    assert _rel_err(y1.cpu().numpy()[rows], y_ref) <= TOL[c["dtype"]]
    # repeated calls: workspace re-armed, results identical
    y3, nh3, out3 = star.lenpred_forward_project(pred, hd, ntd, ind, n, H, bq, ws)
    torch.cuda.synchronize()
    assert np.array_equal(out3.L.cpu().numpy(), out1.L.cpu().numpy())
    pred.close()


# ============================================================================ P -> D dispatch (NEXT-2)
@pytest.mark.parametrize("seed", range(40))
def test_dispatch_bitexact_tiny(star, oracle_mod, seed):
    g = datagen.rng(9000 + seed)
    n, H, A = int(g.integers(1, 9)), int(g.integers(0, 12)), int(g.integers(0, 20))
    L = g.integers(0, 5000, (n, H + 1)).astype(np.int64)
    beta = np.concatenate([[65536], g.integers(1, 65537, H)]).astype(np.uint32)
    n_tok = g.integers(1, 3000, A).astype(np.int32)
    n_hat = g.integers(0, H + 5, A).astype(np.int32)
    c_mem = g.integers(2000, 12000, n).astype(np.int64) if seed % 2 else None
    reserved = g.integers(0, 500, n).astype(np.int64) if seed % 3 == 0 else None
    for policy in (0, 1, 2):
        ref_a, ref_L = oracle_mod.dispatch(policy, L, beta, n_tok, n_hat, c_mem, reserved, counter=seed)
        Ld = _dev(L)
        got = star.dispatch_requests(policy, Ld, _dev(beta.astype(np.int32)), _dev(n_tok), _dev(n_hat),
                                     None if c_mem is None else _dev(c_mem),
                                     None if reserved is None else _dev(reserved), counter=seed)
        torch.cuda.synchronize()
        assert got.cpu().numpy().tolist() == ref_a.tolist(), policy
        assert np.array_equal(Ld.cpu().numpy(), ref_L), policy


@pytest.mark.parametrize("n,A", [(8, 64), (64, 256), (256, 64)])
def test_dispatch_bitexact_cluster_scale(star, oracle_mod, n, A):
    """Projected loads of a real snapshot (8 .. 256 instances, H = 50) + a burst of arrivals with
    long-tailed predicted lengths; all policies bit-exact vs the from-scratch oracle."""
    snap = datagen.make_snapshot(n, n, 32)
    beta = datagen.beta_schedule_q16(50)
    L = oracle_mod.project(snap.inst, snap.n_tok, snap.true_rem, n, 50, beta)["L"]
    arr = datagen.make_snapshot(n + 1, 1, A)
    c_mem = np.full(n, int(L[:, 0].mean() * 1.05), np.int64)
    for policy in (0, 1, 2):
        ref_a, ref_L = oracle_mod.dispatch(policy, L, beta, arr.n_tok, arr.true_rem, c_mem, None, counter=3)
        Ld = _dev(L)
        got = star.dispatch_requests(policy, Ld, _dev(beta.astype(np.int32)), _dev(arr.n_tok),
                                     _dev(arr.true_rem.astype(np.int32)), _dev(c_mem), counter=3)
        torch.cuda.synchronize()
        assert got.cpu().numpy().tolist() == ref_a.tolist(), policy
        assert np.array_equal(Ld.cpu().numpy(), ref_L), policy


@pytest.mark.parametrize("n,A,H", [(1, 40, 50), (33, 300, 7), (1024, 48, 50), (1100, 24, 50), (16, 4096, 50),
                                   (40, 4100, 3)])
def test_dispatch_bitexact_kernel_limits(star, oracle_mod, n, A, H):
    """Both dispatch kernels and their boundary: the sequential one-instance-per-thread kernel
    (n <= 1024, A <= 4096: closed-form prefix corrections instead of row rebuilds) and the
    row-rebuilding kernel above either limit; every policy bit-exact vs the from-scratch oracle,
    with C_mem and reserved KV."""
    g = datagen.rng(n * 7 + A)
    L = g.integers(0, 20000, (n, H + 1)).astype(np.int64)
    beta = datagen.beta_schedule_q16(H)
    n_tok = g.integers(1, 4000, A).astype(np.int32)
    n_hat = np.minimum(g.pareto(1.2, A) * 40, 20000).astype(np.int32)
    c_mem = (L[:, 0] + g.integers(0, 60000, n)).astype(np.int64)
    reserved = g.integers(0, 300, n).astype(np.int64)
    for policy in (0, 1, 2):
        ref_a, ref_L = oracle_mod.dispatch(policy, L, beta, n_tok, n_hat, c_mem, reserved, counter=5)
        Ld = _dev(L)
        got = star.dispatch_requests(policy, Ld, _dev(beta.astype(np.int32)), _dev(n_tok), _dev(n_hat), _dev(c_mem),
                                     _dev(reserved), counter=5)
        torch.cuda.synchronize()
        assert got.cpu().numpy().tolist() == ref_a.tolist(), policy
        assert np.array_equal(Ld.cpu().numpy(), ref_L), policy


# ============================================================================ cluster-scale plan (NEXT-3)
def _plan_gpu_large(star, params_h, L, snap, n_hat):
    pp = star.PlanParams.from_host(params_h)
    moves, nm = star.plan_reschedule_large(pp, _dev(L), _dev(snap.req_id), _dev(snap.inst), _dev(snap.n_tok),
                                           _dev(n_hat.astype(np.int32)), _dev(snap.pinned))
    torch.cuda.synchronize()
    return star.decode_moves(moves, nm)


@pytest.mark.parametrize("seed", range(0, 240, 3))
def test_plan_large_bitexact_tiny(star, oracle_mod, seed):
    """The multi-CTA plan (workspace path) on the same tiny fixtures as the single-CTA plan."""
    g = datagen.rng(seed)
    n, R, H = int(g.integers(1, 7)), int(g.integers(0, 30)), int(g.integers(0, 9))
    snap, n_hat, params = datagen.tiny_fixture(3000 + seed, n, R, H)
    params.max_moves = int(g.integers(0, 6))
    L = oracle_mod.project(snap.inst, snap.n_tok, n_hat, n, H, params.beta_q)["L"]
    ref = oracle_mod.plan(params, L, snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)
    assert _plan_gpu_large(star, params, L, snap, n_hat) == ref


@pytest.mark.parametrize("n,r_per,moves,flags", [(256, 8, 3, 0), (64, 64, 4, 0), (128, 16, 2, 1), (96, 24, 3, 2),
                                                  (8, 256, 4, 0),
                                                  # more instances than scan threads (Phase 1 loops)
                                                  (300, 4, 2, 0), (600, 2, 2, 1)])
def test_plan_large_bitexact_cluster_scale(star, oracle_mod, n, r_per, moves, flags):
    """Cluster-scale shapes (up to 600 instances) vs the from-scratch oracle."""
    snap = datagen.make_snapshot(n + r_per, n, r_per, pinned_frac=0.03)
    n_hat = snap.true_rem.copy()
    params = datagen.make_plan_params(snap, mem_factor=1.10, max_moves=moves, flags=flags, reserved_seed=n)
    L = oracle_mod.project(snap.inst, snap.n_tok, n_hat, n, params.H, params.beta_q)["L"]
    ref = oracle_mod.plan(params, L, snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)
    got = _plan_gpu_large(star, params, L, snap, n_hat)
    assert got == ref
    if n <= 64:   # the single-CTA kernel agrees where its state fits one SM
        assert _plan_gpu(star, params, L, snap, n_hat) == ref


_PLAN_GLOBAL_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import datagen, oracle
import paper_2510_13668_b200 as star
for n, r_per, moves, flags in ((256, 8, 3, 0), (128, 16, 2, 1), (96, 24, 3, 2), (40, 30, 3, 0)):
    snap = datagen.make_snapshot(n + r_per, n, r_per, pinned_frac=0.03)
    n_hat = snap.true_rem.copy()
    params = datagen.make_plan_params(snap, mem_factor=1.10, max_moves=moves, flags=flags, reserved_seed=n)
    L = oracle.project(snap.inst, snap.n_tok, n_hat, n, params.H, params.beta_q)["L"]
    ref = oracle.plan(params, L, snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    pp = star.PlanParams.from_host(params)
    moves_t, nm = star.plan_reschedule_large(pp, d(L), d(snap.req_id), d(snap.inst), d(snap.n_tok),
                                             d(n_hat.astype(np.int32)), d(snap.pinned))
    torch.cuda.synchronize()
    got = star.decode_moves(moves_t, nm)
    assert got == ref, (n, got, ref)
    assert len(ref) > 0 or n == 40
print("global ok")
'''


def test_plan_large_global_terms_subprocess(star):
    """The cluster-scale plan's per-target terms read from global memory (the form above ~6500
    instances, where they do not fit shared memory), forced by STAR_PLAN_LARGE_GLOBAL=1 in a fresh
    process at sizes the oracle finishes: bit-exact vs the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _PLAN_GLOBAL_SCRIPT, root],
                       env={**os.environ, "STAR_PLAN_LARGE_GLOBAL": "1"}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "global ok" in r.stdout


# ============================================================================ prediction cadence (NEXT-1)
def _nhat_close(got, ref_y, n_tok, tol):
    """Refreshed rows: the GPU's N_hat within the bf16 tolerance of the quantized fp64 oracle."""
    ref = np.clip(np.rint(ref_y), 0, np.maximum(0, 32768 - n_tok))
    return np.all(np.abs(got.astype(np.float64) - ref) <= np.maximum(1.0, tol * np.abs(ref)) + 1.0)


@pytest.mark.parametrize("R,k,seed,d", [(2048, 20, 0, 4096), (2047, 20, 1, 4096), (300, 7, 2, 4096), (4096, 20, 3, 4096),
                                        (64, 1, 4, 4096),
                                        # more due rows than one 512-row chunk of the one-launch predictor
                                        (2048, 2, 5, 4096), (1000, 1, 6, 1024),
                                        # d % 256 != 0: the multi-launch refresh path
                                        (300, 5, 7, 896)])
def test_refresh_step_parity(star, oracle_mod, R, k, seed, d):
    g = datagen.rng(seed)
    snap = datagen.make_snapshot(seed, 8, (R + 7) // 8)
    n_tok = snap.n_tok[:R].copy()
    pw = datagen.make_predictor_weights(seed, d, "bf16")
    scale = np.exp(g.normal(0.0, 1.5, R)).astype(np.float32)
    h = datagen.make_hidden(seed, R, d, "bf16", scale=scale)
    gen = g.integers(0, 5000, R).astype(np.int32)
    g_last = np.where(g.random(R) < 0.1, -1, gen - g.integers(0, 2 * k + 1, R)).astype(np.int32)
    nhat_last = g.integers(0, 30000, R).astype(np.int32)
    W, _ = _weights_dev(pw)
    pred = star.Predictor(*W, max_rows=R)
    gl_d, nl_d = _dev(g_last), _dev(nhat_last)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    nh = star.lenpred_forward_refresh(pred, _dev(h, torch.bfloat16), _dev(n_tok), _dev(gen), gl_d, nl_d, k,
                                      n_refreshed=cnt)
    torch.cuda.synchronize()
    # the oracle's cadence step (oracle.refresh_step: SPEC.md:164-172 + reading A27, Eq. 2 in fp64)
    nh_ref, gl_ref, nl_ref, due = oracle_mod.refresh_step(h, pw, n_tok, gen, g_last, nhat_last, k)
    assert cnt.item() == int(due.sum())
    nh, gl2, nl2 = nh.cpu().numpy(), gl_d.cpu().numpy(), nl_d.cpu().numpy()
    aged = ~due   # aged rows: exact integers
    assert np.array_equal(nh[aged], nh_ref[aged])
    assert np.array_equal(gl2, gl_ref)                               # cadence state: exact everywhere
    assert np.array_equal(nl2[aged], nl_ref[aged]) and np.array_equal(nl2[due], nh[due])
    # refreshed rows (all of them): the GPU's N_hat within the bf16 tolerance of the oracle's
    d_ = np.abs(nh[due].astype(np.float64) - nh_ref[due])
    assert np.all(d_ <= np.maximum(1.0, 2e-2 * np.abs(nh_ref[due])) + 1.0)
    pred.close()


@pytest.mark.parametrize("R,k,seed,n", [(2048, 20, 0, 8), (777, 7, 1, 3), (64, 1, 2, 1), (5000, 20, 3, 64),
                                        (6000, 20, 4, 8), (512, 20, 5, 1), (4096, 20, 6, 8)])
def test_refresh_project_fused_equals_separate(star, oracle_mod, R, k, seed, n):
    """lenpred_forward_refresh_project (aging scatter fused with the projection, one CTA) ==
    lenpred_forward_refresh + project_instance_load, bit for bit (N_hat, cadence state, L, W, peak,
    growth, count), and == the oracle projection of that N_hat."""
    from paper_2510_13668_b200 import _lib
    c = datagen.CONFIGS["C2"]
    g = datagen.rng(seed)
    snap = datagen.make_snapshot(seed, n, (R + n - 1) // n)
    n_tok, inst = snap.n_tok[:R].copy(), snap.inst[:R].astype(np.int32)
    pw = datagen.make_predictor_weights(seed, c["d"], "bf16")
    scale = np.exp(g.normal(0.0, 1.5, R)).astype(np.float32)
    h = _dev(datagen.make_hidden(seed, R, c["d"], "bf16", scale=scale), torch.bfloat16)
    gen = g.integers(0, 5000, R).astype(np.int32)
    g_last = np.where(g.random(R) < 0.1, -1, gen - g.integers(0, 2 * k + 1, R)).astype(np.int32)
    if R >= 6000:   # first step of a batch: no prediction yet, every row due (12 chunks of 512 rows)
        g_last[:] = -1
    if seed == 5:   # no row due this step: only the aged rows, the projection must still be finalised
        g_last[:] = gen
    nhat_last = g.integers(0, 30000, R).astype(np.int32)
    W, _ = _weights_dev(pw)
    pred = star.Predictor(*W, max_rows=R)
    beta = datagen.beta_schedule_q16(50)
    bq = _dev(beta.astype(np.int32))
    res = []
    for fused in (True, False):
        gl_d, nl_d = _dev(g_last), _dev(nhat_last)
        ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        if fused:
            nh, out = _lib.lenpred_forward_refresh_project(pred, h, _dev(n_tok), _dev(gen), gl_d, nl_d, k,
                                                           _dev(inst), n, 50, bq, ws, err_flag=err)
        else:
            nh = star.lenpred_forward_refresh(pred, h, _dev(n_tok), _dev(gen), gl_d, nl_d, k)
            out = star.project_instance_load(_dev(inst), _dev(n_tok), nh, n, 50, bq, workspace=ws, err_flag=err)
        torch.cuda.synchronize()
        assert err.item() == 0 and int(ws.sum().item()) == 0
        res.append([nh.cpu().numpy(), gl_d.cpu().numpy(), nl_d.cpu().numpy()] +
                   [getattr(out, k_).cpu().numpy() for k_ in ("L", "W", "peak", "growth", "count")])
    for a, b in zip(*res):
        assert np.array_equal(a, b)
    ref = oracle_mod.project(inst, n_tok, res[0][0], n, 50, beta)
    assert np.array_equal(res[0][3], ref["L"]) and np.array_equal(res[0][4], ref["W"])
    pred.close()


def test_refresh_schedule_on_device(star, oracle_mod):
    """45 decode steps (gen += 1 per step), k = 20: every row refreshes at its first step and then
    every 20 generated tokens; in between the device ages it exactly like the oracle."""
    R, k, d = 512, 20, 4096
    pw = datagen.make_predictor_weights(9, d, "bf16")
    h = datagen.make_hidden(9, R, d, "bf16", scale=np.exp(datagen.rng(9).normal(0, 1.5, R)).astype(np.float32))
    W, _ = _weights_dev(pw)
    pred = star.Predictor(*W, max_rows=R)
    hd = _dev(h, torch.bfloat16)
    start = datagen.rng(10).integers(0, 30, R).astype(np.int32)
    n_tok0 = datagen.make_snapshot(9, 1, R).n_tok
    gl_d = _dev(np.full(R, -1, np.int32))
    nl_d = _dev(np.zeros(R, np.int32))
    g_last = np.full(R, -1, np.int32)
    nhat_last = np.zeros(R, np.int32)
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for step in range(45):
        gen = (start + step).astype(np.int32)
        n_tok = (n_tok0 + step).astype(np.int32)
        nh = star.lenpred_forward_refresh(pred, hd, _dev(n_tok), _dev(gen), gl_d, nl_d, k, n_refreshed=cnt)
        torch.cuda.synchronize()
        due = oracle_mod.should_refresh(gen, g_last, k)
        assert cnt.item() == int(due.sum()), step
        assert step != 0 or due.all()
        nh = nh.cpu().numpy()
        gl2, nl2 = gl_d.cpu().numpy(), nl_d.cpu().numpy()
        aged = ~due
        assert np.array_equal(nh[aged], np.maximum(0, nhat_last[aged] - (gen[aged] - g_last[aged])))
        assert np.array_equal(gl2[due], gen[due])
        g_last, nhat_last = gl2, nl2
    pred.close()


# ============================================================================ one-rank step (fused plan)
@pytest.mark.parametrize("cfg,R,seed", [("C2", 2048, 0), ("C4", 4096, 1), ("TGT", 4096, 2), ("C2", 1000, 3),
                                        ("C1", 128, 4), ("C4", 777, 5)])
def test_step_world1_fused_plan_equals_oracle(star, oracle_mod, cfg, R, seed):
    """Step.run at world 1 (lenpred_forward_project_plan: Alg. 1 run by the fused tail's last CTA
    when it fits) == the separate calls == the oracle plan on the GPU's own N_hat, bit for bit."""
    from paper_2510_13668_b200.step import Step
    c = datagen.CONFIGS[cfg]
    n = c["n_inst"]
    snap = datagen.make_snapshot(seed, n, (R + n - 1) // n, skewed=c.get("skewed", False), pinned_frac=0.05)
    sl = slice(0, R)
    ids, inst, n_tok, pin = snap.req_id[sl], snap.inst[sl], snap.n_tok[sl], snap.pinned[sl]
    pw = datagen.make_predictor_weights(seed, c["d"], c["dtype"])
    scale = np.maximum(snap.true_rem[sl], 1).astype(np.float32) / 60.0   # long-tailed self-predictions
    h = datagen.make_hidden(seed, R, c["d"], c["dtype"], scale=scale)
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    W, b = _weights_dev(pw, False)
    pred = star.Predictor(*W, *b, max_rows=R)
    params_h = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10),
                                        max_moves=max(c["max_moves"], 4))
    params = star.PlanParams.from_host(params_h)
    st = Step(pred, params, n, r_cap=R)
    st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in (ids, inst, n_tok)),
                     pinned=torch.from_numpy(np.ascontiguousarray(pin)))
    hd = _dev(h, tdt)
    st.run(hd)
    torch.cuda.synchronize()
    got = st.result()
    nh = st.v["n_hat"][:R].cpu().numpy()
    L = st.v["L"].cpu().numpy()
    assert st.err.item() == 0
    # the fused projection equals the oracle projection of the GPU's own N_hat ...
    ref_p = oracle_mod.project(inst, n_tok, nh, n, 50, params_h.beta_q)
    assert np.array_equal(L, ref_p["L"])
    # ... and the plan equals the oracle plan on that state
    ref = oracle_mod.plan(params_h, ref_p["L"], ids, inst, n_tok, nh, pin)
    assert got == ref
    if cfg in ("TGT", "C4"):
        assert len(got) >= 1   # skewed: the plan gets past Phase 1 on the GPU's own predictions
    # the separate calls (projection, then the plan kernel) give the same moves
    moves2, nm2 = star.plan_reschedule_segmented(params, st.seg)
    torch.cuda.synchronize()
    assert star.decode_moves(moves2, nm2) == got
    # repeated step: identical (workspace re-armed, plan state rebuilt)
    st.run(hd)
    torch.cuda.synchronize()
    assert st.result() == got
    pred.close()


# ============================================================================ W-rank step, one GPU
@pytest.mark.parametrize("cfg,world,r_per,seed", [("TGT", 8, 512, 0), ("C2", 4, 256, 1), ("C4", 2, 300, 2)])
def test_step_gathered_ranks_plan_equals_oracle(star, oracle_mod, cfg, world, r_per, seed):
    """Every rank of a W-rank job on one GPU (Step(gathered=...): the ranks' records written into
    one shared gathered buffer, as the all-gather delivers them): each rank's fused projection of
    its own N_hat equals the oracle's, and every rank's plan over the gathered records equals the
    oracle plan on the concatenated state, bit for bit."""
    from paper_2510_13668_b200.step import RecordLayout, Step, split_snapshot_by_rank
    c = datagen.CONFIGS[cfg]
    n = c["n_inst"]
    snap = datagen.make_snapshot(seed, n, r_per, skewed=c.get("skewed", False), pinned_frac=0.05)
    pw = datagen.make_predictor_weights(seed, c["d"], c["dtype"])
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    W, b = _weights_dev(pw, False)
    params_h = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10),
                                        max_moves=max(c["max_moves"], 2))
    params = star.PlanParams.from_host(params_h)
    idxs = [split_snapshot_by_rank(snap.inst, n, world, k) for k in range(world)]
    r_cap = max(len(i) for i in idxs)
    pred = star.Predictor(*W, *b, max_rows=r_cap)
    buf = torch.zeros(world * RecordLayout(n // world, 50, r_cap).nbytes, dtype=torch.uint8, device="cuda")
    steps = []
    for k, idx in enumerate(idxs):
        scale = np.maximum(snap.true_rem[idx], 1).astype(np.float32) / 60.0
        h = datagen.make_hidden(seed * 100 + k, len(idx), c["d"], c["dtype"], scale=scale)
        st = Step(pred, params, n, r_cap=r_cap, rank=k, world=world, gathered=buf)
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                      snap.n_tok)),
                         pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
        st.run(_dev(h, tdt))
        steps.append(st)
    torch.cuda.synchronize()
    order = np.concatenate(idxs)
    nh = np.concatenate([st.v["n_hat"][:len(i)].cpu().numpy() for st, i in zip(steps, idxs)])
    ids, inst, n_tok, pin = (a[order] for a in (snap.req_id, snap.inst, snap.n_tok, snap.pinned))
    ref_p = oracle_mod.project(inst, n_tok, nh, n, 50, params_h.beta_q)
    for k, st in enumerate(steps):
        assert st.err.item() == 0
        loc = slice(k * (n // world), (k + 1) * (n // world))
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"][loc])
    ref = oracle_mod.plan(params_h, ref_p["L"], ids, inst, n_tok, nh, pin)
    if c.get("skewed"):
        assert len(ref) >= 1   # Phases 2-3 reached, a request moves
    # the last rank ran with every record in place; re-plan on the final buffer from every rank
    for st in steps:
        moves, nm = star.plan_reschedule_segmented(params, st.seg)
        torch.cuda.synchronize()
        assert star.decode_moves(moves, nm) == ref
    assert steps[-1].result() == ref
    pred.close()


def test_step_gathered_with_an_empty_rank(star, oracle_mod):
    """A decode instance block with no running requests (rank 3 of 4: instances 6 and 7 empty):
    its rank runs the step on R = 0 and must still publish a valid record (zero loads, count 0)
    over whatever the gathered buffer held before; every rank's plan == the oracle's."""
    from paper_2510_13668_b200.step import RecordLayout, Step, split_snapshot_by_rank
    n, world, r_per, d = 8, 4, 96, 1024
    snap0 = datagen.make_snapshot(5, n, r_per, skewed=True, pinned_frac=0.05)
    keep = snap0.inst < 6
    pw = datagen.make_predictor_weights(5, d, "bf16")
    W, b = _weights_dev(pw, False)
    params_h = datagen.make_plan_params(snap0, H=50, max_moves=2)
    params = star.PlanParams.from_host(params_h)
    idxs = [i[keep[i]] for i in (split_snapshot_by_rank(snap0.inst, n, world, k) for k in range(world))]
    assert len(idxs[3]) == 0
    r_cap = max(len(i) for i in idxs)
    pred = star.Predictor(*W, *b, max_rows=r_cap)
    buf = torch.full((world * RecordLayout(n // world, 50, r_cap).nbytes,), 0xAB, dtype=torch.uint8, device="cuda")
    steps = []
    for k, idx in enumerate(idxs):
        h = datagen.make_hidden(500 + k, len(idx), d, "bf16")
        st = Step(pred, params, n, r_cap=r_cap, rank=k, world=world, gathered=buf)
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap0.req_id, snap0.inst,
                                                                                      snap0.n_tok)),
                         pinned=torch.from_numpy(np.ascontiguousarray(snap0.pinned[idx])))
        st.run(_dev(h, torch.bfloat16))
        steps.append(st)
    torch.cuda.synchronize()
    order = np.concatenate(idxs)
    nh = np.concatenate([st.v["n_hat"][:len(i)].cpu().numpy() for st, i in zip(steps, idxs)])
    ids, inst, n_tok, pin = (a[order] for a in (snap0.req_id, snap0.inst, snap0.n_tok, snap0.pinned))
    ref_p = oracle_mod.project(inst, n_tok, nh, n, 50, params_h.beta_q)
    assert not ref_p["L"][6:].any()
    for k, st in enumerate(steps):
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"][2 * k:2 * k + 2])
    assert steps[-1].err.item() == 0   # the last rank planned with every record in place
    ref = oracle_mod.plan(params_h, ref_p["L"], ids, inst, n_tok, nh, pin)
    assert steps[-1].result() == ref
    # (the earlier ranks planned while later records still held the 0xAB fill: re-plan on the final buffer)
    for st in steps:
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        moves, nm = star.plan_reschedule_segmented(params, st.seg, err_flag=err)
        torch.cuda.synchronize()
        assert err.item() == 0
        assert star.decode_moves(moves, nm) == ref
    pred.close()


@pytest.mark.parametrize("case", ["world1_empty", "refresh_empty", "no_moves_allowed", "one_instance", "fp32_world1"])
def test_step_edge_cases(star, oracle_mod, case):
    """Degenerate steps through the public Step API, each against the oracle: no running request
    on a one-rank step (zero loads, no move) and in the cadence-k mode; max_moves = 0 on an
    overloaded snapshot (no move, loads exact); a single instance (no target, no move); an fp32
    one-rank step (the one-launch fp32 predictor, then the plan)."""
    from paper_2510_13668_b200.step import Step
    n, r_per, d, dt = 4, 64, 1024, "bf16"
    if case == "one_instance":
        n = 1
    if case == "fp32_world1":
        n, r_per, d, dt = 2, 64, 896, "f32"
    snap = datagen.make_snapshot(9, n, r_per, skewed=n > 1)
    params_h = datagen.make_plan_params(snap, H=50, max_moves=0 if case == "no_moves_allowed" else 2)
    params = star.PlanParams.from_host(params_h)
    pw = datagen.make_predictor_weights(9, d, dt)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    W, b = _weights_dev(pw, False)
    pred = star.Predictor(*W, *b, max_rows=snap.R)
    idx = np.arange(0 if case.endswith("empty") else snap.R)
    st = Step(pred, params, n, r_cap=snap.R, refresh_k=20 if case == "refresh_empty" else None)
    st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst, snap.n_tok)))
    scale = np.maximum(snap.true_rem[idx], 1).astype(np.float32) / 60.0
    h = datagen.make_hidden(90, len(idx), d, dt, scale=scale if len(idx) else None)
    st.run(_dev(h, tdt) if len(idx) else torch.empty((0, d), dtype=tdt, device="cuda"))
    torch.cuda.synchronize()
    assert st.err.item() == 0
    nh = st.v["n_hat"][:len(idx)].cpu().numpy()
    ref_p = oracle_mod.project(snap.inst[idx].astype(np.int32), snap.n_tok[idx], nh, n, 50, params_h.beta_q)
    assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"])
    ref = oracle_mod.plan(params_h, ref_p["L"], snap.req_id[idx], snap.inst[idx], snap.n_tok[idx], nh, None)
    assert st.result() == ref
    if case in ("world1_empty", "refresh_empty", "no_moves_allowed", "one_instance"):
        assert ref == []
    pred.close()


@pytest.mark.parametrize("H,world", [(0, 1), (256, 1), (256, 4), (1, 4)])
def test_step_horizon_extremes(star, oracle_mod, H, world):
    """Projection horizons at the ends of the supported range (H = 0: current loads only; H = 256)
    through the Step API, one rank and the gathered 4-rank form: loads and plan == oracle."""
    from paper_2510_13668_b200.step import RecordLayout, Step, split_snapshot_by_rank
    n, r_per, d = 8, 64, 1024
    snap = datagen.make_snapshot(13 + H, n, r_per, skewed=True)
    params_h = datagen.make_plan_params(snap, H=H, max_moves=3)
    params = star.PlanParams.from_host(params_h)
    pw = datagen.make_predictor_weights(13, d, "bf16")
    W, b = _weights_dev(pw, False)
    idxs = [split_snapshot_by_rank(snap.inst, n, world, k) for k in range(world)]
    r_cap = max(len(i) for i in idxs)
    pred = star.Predictor(*W, *b, max_rows=r_cap)
    buf = (torch.zeros(world * RecordLayout(n // world, H, r_cap).nbytes, dtype=torch.uint8, device="cuda")
           if world > 1 else None)
    steps = []
    for k, idx in enumerate(idxs):
        st = Step(pred, params, n, r_cap=r_cap, rank=k, world=world, gathered=buf)
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                      snap.n_tok)))
        h = datagen.make_hidden(130 + k, len(idx), d, "bf16",
                                scale=np.maximum(snap.true_rem[idx], 1).astype(np.float32) / 60.0)
        st.run(_dev(h, torch.bfloat16))
        steps.append(st)
    torch.cuda.synchronize()
    order = np.concatenate(idxs)
    nh = np.concatenate([st.v["n_hat"][:len(i)].cpu().numpy() for st, i in zip(steps, idxs)])
    ids, inst, n_tok = (a[order] for a in (snap.req_id, snap.inst, snap.n_tok))
    ref_p = oracle_mod.project(inst, n_tok, nh, n, H, params_h.beta_q)
    for k, st in enumerate(steps):
        loc = slice(k * (n // world), (k + 1) * (n // world))
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"][loc])
        assert np.array_equal(st.v["W"].cpu().numpy(), ref_p["W"][loc])
    ref = oracle_mod.plan(params_h, ref_p["L"], ids, inst, n_tok, nh, None)
    assert steps[-1].result() == ref
    assert steps[-1].err.item() == 0
    pred.close()


def test_step_refresh_gathered_ranks(star, oracle_mod):
    """The cadence-k mode on every rank of a 4-rank job (gathered records on one GPU): each rank's
    refreshed / aged N_hat and cadence state follow oracle.refresh_step (aged rows and state
    exact, refreshed rows within the bf16 tolerance), its loads equal the oracle projection of its
    own N_hat, and every rank's plan over the gathered records equals the oracle's."""
    from paper_2510_13668_b200.step import RecordLayout, Step, split_snapshot_by_rank
    n, world, r_per, d, k = 8, 4, 96, 1024, 5
    snap = datagen.make_snapshot(17, n, r_per, skewed=True)
    params_h = datagen.make_plan_params(snap, H=50, max_moves=2)
    params = star.PlanParams.from_host(params_h)
    pw = datagen.make_predictor_weights(17, d, "bf16")
    W, b = _weights_dev(pw, False)
    g = datagen.rng(17)
    idxs = [split_snapshot_by_rank(snap.inst, n, world, q) for q in range(world)]
    r_cap = max(len(i) for i in idxs)
    pred = star.Predictor(*W, *b, max_rows=r_cap)
    buf = torch.zeros(world * RecordLayout(n // world, 50, r_cap).nbytes, dtype=torch.uint8, device="cuda")
    steps, states = [], []
    for q, idx in enumerate(idxs):
        R = len(idx)
        h = datagen.make_hidden(170 + q, R, d, "bf16", scale=np.maximum(snap.true_rem[idx], 1).astype(np.float32) / 60.0)
        gen = g.integers(10, 3000, R).astype(np.int32)
        g_last = np.where(g.random(R) < 0.2, -1, gen - g.integers(0, 2 * k, R)).astype(np.int32)
        nhat_last = g.integers(0, 5000, R).astype(np.int32)
        st = Step(pred, params, n, r_cap=r_cap, rank=q, world=world, gathered=buf, refresh_k=k)
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                      snap.n_tok)))
        st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last), torch.from_numpy(nhat_last))
        st.run(_dev(h, torch.bfloat16))
        steps.append(st)
        states.append((h, gen, g_last, nhat_last))
    torch.cuda.synchronize()
    nhs = []
    for st, idx, (h, gen, g_last, nhat_last) in zip(steps, idxs, states):
        R = len(idx)
        nh_ref, gl_ref, nl_ref, due = oracle_mod.refresh_step(h, pw, snap.n_tok[idx], gen, g_last, nhat_last, k)
        nh = st.v["n_hat"][:R].cpu().numpy()
        assert np.array_equal(nh[~due], nh_ref[~due])
        assert np.array_equal(st.g_last[:R].cpu().numpy(), gl_ref)
        d_ = np.abs(nh[due].astype(np.float64) - nh_ref[due])
        assert np.all(d_ <= np.maximum(1.0, 2e-2 * np.abs(nh_ref[due])) + 1.0)
        assert int(st.n_refreshed.item()) == int(due.sum())
        nhs.append(nh)
    order = np.concatenate(idxs)
    nh_all = np.concatenate(nhs)
    ids, inst, n_tok = (a[order] for a in (snap.req_id, snap.inst, snap.n_tok))
    ref_p = oracle_mod.project(inst, n_tok, nh_all, n, 50, params_h.beta_q)
    for q, st in enumerate(steps):
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"][2 * q:2 * q + 2])
    ref = oracle_mod.plan(params_h, ref_p["L"], ids, inst, n_tok, nh_all, None)
    assert steps[-1].result() == ref and steps[-1].err.item() == 0
    pred.close()


def test_step_refresh_over_many_steps(star, oracle_mod):
    """The cadence state evolving over 12 decode steps (every request generates one token per step,
    the hidden states change every step): each step's N_hat, g_last and N_hat_last follow
    oracle.refresh_step from the previous step's oracle state (aged rows exact; refreshed rows
    within the bf16 tolerance, the oracle then continues from the GPU's own N_hat so the
    comparison does not drift), loads and plan == oracle."""
    from paper_2510_13668_b200.step import Step
    n, r_per, d, k = 4, 64, 1024, 4
    snap = datagen.make_snapshot(19, n, r_per, skewed=True)
    R = snap.R
    params_h = datagen.make_plan_params(snap, H=50, max_moves=1)
    params = star.PlanParams.from_host(params_h)
    pw = datagen.make_predictor_weights(19, d, "bf16")
    W, b = _weights_dev(pw, False)
    pred = star.Predictor(*W, *b, max_rows=R)
    st = Step(pred, params, n, r_cap=R, refresh_k=k)
    n_tok = snap.n_tok.copy()
    gen = np.zeros(R, np.int32)
    g_last = np.full(R, -1, np.int32)
    nhat_last = np.zeros(R, np.int32)
    st.load_requests(*(torch.from_numpy(a) for a in (snap.req_id, snap.inst, n_tok)))
    st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last), torch.from_numpy(nhat_last))
    for step in range(12):
        h = datagen.make_hidden(1900 + step, R, d, "bf16", scale=np.maximum(snap.true_rem, 1).astype(np.float32) / 60.0)
        st.v["n_tok"][:R].copy_(torch.from_numpy(n_tok))
        st.set_generation(torch.from_numpy(gen))
        st.run(_dev(h, torch.bfloat16))
        torch.cuda.synchronize()
        nh_ref, gl_ref, nl_ref, due = oracle_mod.refresh_step(h, pw, n_tok, gen, g_last, nhat_last, k)
        nh = st.v["n_hat"][:R].cpu().numpy()
        assert np.array_equal(nh[~due], nh_ref[~due]), step
        assert np.array_equal(st.g_last[:R].cpu().numpy(), gl_ref), step
        d_ = np.abs(nh[due].astype(np.float64) - nh_ref[due])
        assert np.all(d_ <= np.maximum(1.0, 2e-2 * np.abs(nh_ref[due])) + 1.0), step
        nl = st.nhat_last[:R].cpu().numpy()
        assert np.array_equal(nl[~due], nl_ref[~due]) and np.array_equal(nl[due], nh[due]), step
        ref_p = oracle_mod.project(snap.inst, n_tok, nh, n, 50, params_h.beta_q)
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"]), step
        assert st.result() == oracle_mod.plan(params_h, ref_p["L"], snap.req_id, snap.inst, n_tok, nh, None), step
        # next step: continue from the GPU's own state; every request generates one token
        g_last, nhat_last = gl_ref, nl.copy()
        gen = gen + 1
        n_tok = n_tok + 1
    assert st.err.item() == 0
    pred.close()


def test_step_capture_replay_guards(star, oracle_mod):
    """Step.capture / replay (the public one-launch-per-step API): a replay after new request data
    of the same count equals a fresh run; a changed request count refuses to replay stale grids."""
    from paper_2510_13668_b200.step import Step
    n, r_per, d = 4, 64, 1024
    snap = datagen.make_snapshot(11, n, r_per, skewed=True)
    params_h = datagen.make_plan_params(snap, H=50, max_moves=2)
    params = star.PlanParams.from_host(params_h)
    pw = datagen.make_predictor_weights(11, d, "bf16")
    W, b = _weights_dev(pw, False)
    pred = star.Predictor(*W, *b, max_rows=snap.R)
    st = Step(pred, params, n, r_cap=snap.R)
    with pytest.raises(RuntimeError):
        st.replay()
    st.load_requests(*(torch.from_numpy(a) for a in (snap.req_id, snap.inst, snap.n_tok)))
    h = _dev(datagen.make_hidden(110, snap.R, d, "bf16",
                                 scale=np.maximum(snap.true_rem, 1).astype(np.float32) / 60.0), torch.bfloat16)
    st.capture(h)
    # new hidden states and token counts, same count: replay == the oracle on the new inputs
    h2 = datagen.make_hidden(111, snap.R, d, "bf16", scale=np.maximum(snap.true_rem, 1).astype(np.float32) / 50.0)
    h.copy_(_dev(h2, torch.bfloat16))
    st.load_requests(*(torch.from_numpy(a) for a in (snap.req_id, snap.inst, snap.n_tok + 3)))
    st.replay()
    torch.cuda.synchronize()
    nh = st.v["n_hat"][:snap.R].cpu().numpy()
    ref_p = oracle_mod.project(snap.inst, snap.n_tok + 3, nh, n, 50, params_h.beta_q)
    assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"])
    assert st.result() == oracle_mod.plan(params_h, ref_p["L"], snap.req_id, snap.inst, snap.n_tok + 3, nh, None)
    st.load_requests(*(torch.from_numpy(a[:-1]) for a in (snap.req_id, snap.inst, snap.n_tok)))
    with pytest.raises(RuntimeError):
        st.replay()
    pred.close()


def test_two_predictors_concurrent_streams(star, oracle_mod):
    """Two predictors on two streams at once (bf16 one-launch at 512 rows, fp32 one-launch at
    128 rows, each fused with its projection, then a plan each): the results equal the same calls
    run one after the other -- no state is shared between predictors."""
    beta = datagen.beta_schedule_q16(50)
    bq = _dev(beta.astype(np.int32))
    cases = []
    for seed, d, dt, R, n in ((21, 4096, "bf16", 512, 4), (22, 896, "f32", 128, 2)):
        pw = datagen.make_predictor_weights(seed, d, dt)
        snap = datagen.make_snapshot(seed, n, R // n, skewed=True)
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        W, b = _weights_dev(pw, False)
        pred = star.Predictor(*W, *b, max_rows=R)
        h = _dev(datagen.make_hidden(seed, R, d, dt, scale=np.maximum(snap.true_rem, 1).astype(np.float32) / 60.0),
                 tdt)
        params_h = datagen.make_plan_params(snap, H=50, max_moves=2)
        cases.append((pred, h, snap, n, star.PlanParams.from_host(params_h), params_h))

    def run(stream_of):
        outs = []
        for k, (pred, h, snap, n, pp, _) in enumerate(cases):
            st = stream_of(k)
            with torch.cuda.stream(st):
                ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
                y, nh, out = star.lenpred_forward_project(pred, h, _dev(snap.n_tok), _dev(snap.inst), n, 50, bq, ws)
                moves, nm = star.plan_reschedule(pp, out.L, _dev(snap.req_id), _dev(snap.inst), _dev(snap.n_tok), nh)
                outs.append((y, nh, out.L, moves, nm))
        torch.cuda.synchronize()
        return [(y.cpu().numpy(), nh.cpu().numpy(), L.cpu().numpy(), star.decode_moves(m, c)) for y, nh, L, m, c in outs]

    seq = run(lambda k: torch.cuda.current_stream())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(3):
        par = run(lambda k: streams[k])
        for a, b_ in zip(seq, par):
            assert np.array_equal(a[0], b_[0]) and np.array_equal(a[1], b_[1]) and np.array_equal(a[2], b_[2])
            assert a[3] == b_[3]
    for (pred, h, snap, n, pp, params_h), (y, nh, L, moves) in zip(cases, seq):
        ref_p = oracle_mod.project(snap.inst, snap.n_tok, nh, n, 50, beta)
        assert np.array_equal(L, ref_p["L"])
        assert moves == oracle_mod.plan(params_h, ref_p["L"], snap.req_id, snap.inst, snap.n_tok, nh, None)
        pred.close()


# ============================================================================ one-launch small-batch predictor
@pytest.mark.parametrize("d,R,biases,n,ld_pad", [(4096, 512, True, 1, 0), (4096, 384, False, 3, 64), (4096, 129, False, 8, 0),
                                                 (5120, 511, True, 2, 0), (1024, 64, False, 1, 0), (4096, 1, True, 1, 8),
                                                 (4096, 256, False, 300, 0), (2048, 200, True, 5, 0)])
def test_small_path_forward_project(star, oracle_mod, d, R, biases, n, ld_pad):
    """The one-launch predictor (<= 512 rows: layers 1-3, head, quantizer and the projection in
    one persistent kernel, DSMEM split-K reductions): every row within the bf16 tolerance of the
    fp64 oracle, N_hat == the oracle quantizer of its y_hat, L/W/peak/growth/count == the oracle
    projection of that N_hat bit for bit; repeated launches (counters re-armed) are bit-identical,
    also with a row stride > d and max_rows > R."""
    pw = datagen.make_predictor_weights(d + R, d, "bf16", biases=biases)
    snap = datagen.make_snapshot(R + n, n, (R + n - 1) // n)
    n_tok, inst = snap.n_tok[:R].copy(), snap.inst[:R].astype(np.int32)
    scale = np.maximum(snap.true_rem[:R], 1).astype(np.float32) / 60.0
    h = datagen.make_hidden(d + R, R, d, "bf16", scale=scale)
    hpad = np.zeros((R, d + ld_pad), np.float32)
    hpad[:, :d] = h
    hd = _dev(hpad, torch.bfloat16)[:, :d]
    W, b = _weights_dev(pw, biases)
    pred = star.Predictor(*W, *b, max_rows=max(R, 600))
    assert pred.path(R) == 1
    beta = datagen.beta_schedule_q16(50)
    bq = _dev(beta.astype(np.int32))
    ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    runs = []
    for _ in range(3):
        y, nh, out = star.lenpred_forward_project(pred, hd, _dev(n_tok), _dev(inst), n, 50, bq, ws, err_flag=err)
        torch.cuda.synchronize()
        runs.append([y.cpu().numpy(), nh[:R].cpu().numpy()] +
                    [getattr(out, k).cpu().numpy() for k in ("L", "W", "peak", "growth", "count")])
    for r in runs[1:]:
        for a_, b_ in zip(runs[0], r):
            assert np.array_equal(a_, b_)
    y, nh = runs[0][0], runs[0][1]
    ref = oracle_mod.lenpred_weights(h, pw)
    assert _rel_err(y, ref) <= TOL["bf16"]
    assert np.array_equal(nh, oracle_mod.quantize(y, n_tok))
    rp = oracle_mod.project(inst, n_tok, nh, n, 50, beta)
    for k, v in zip(("L", "W", "peak", "growth", "count"), runs[0][2:]):
        assert np.array_equal(v, rp[k]), k
    assert err.item() == 0 and int(ws.sum().item()) == 0
    pred.close()


# ============================================================================ one-launch fp32 predictor
@pytest.mark.parametrize("d,R,biases,n,ld_pad,max_rows", [(896, 128, False, 2, 0, 128), (896, 64, True, 1, 0, 600),
                                                          (128, 1, True, 1, 8, 1), (4096, 128, False, 8, 0, 256),
                                                          (1024, 77, True, 3, 32, 77), (2048, 100, False, 200, 0, 128),
                                                          (512, 5, False, 2, 0, 5)])
def test_f32_small_path_forward_project(star, oracle_mod, d, R, biases, n, ld_pad, max_rows):
    """The one-launch fp32 predictor (<= 128 rows: 3xTF32 layers 1-3 with the operands split in
    shared memory, head, quantizer and the projection in one kernel; BASELINE configs[0] shape
    first): every row within the fp32 tolerance of the fp64 oracle, N_hat == the oracle quantizer
    of its y_hat, L/W/peak/growth/count == the oracle projection of that N_hat bit for bit;
    repeated launches (counters re-armed) bit-identical, also with a row stride > d and
    max_rows < 128 (TMA zero-fills the rows past the map)."""
    pw = datagen.make_predictor_weights(d + R + 7, d, "f32", biases=biases)
    snap = datagen.make_snapshot(R + n + 7, n, (R + n - 1) // n)
    n_tok, inst = snap.n_tok[:R].copy(), snap.inst[:R].astype(np.int32)
    scale = np.maximum(snap.true_rem[:R], 1).astype(np.float32) / 60.0
    h = datagen.make_hidden(d + R + 7, R, d, "f32", scale=scale)
    hpad = np.zeros((R, d + ld_pad), np.float32)
    hpad[:, :d] = h
    hd = _dev(hpad)[:, :d]
    W, b = _weights_dev(pw, biases)
    pred = star.Predictor(*W, *b, max_rows=max_rows)
    assert pred.path(R) == 2
    beta = datagen.beta_schedule_q16(50)
    bq = _dev(beta.astype(np.int32))
    ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    runs = []
    for _ in range(3):
        y, nh, out = star.lenpred_forward_project(pred, hd, _dev(n_tok), _dev(inst), n, 50, bq, ws, err_flag=err)
        torch.cuda.synchronize()
        runs.append([y.cpu().numpy(), nh[:R].cpu().numpy()] +
                    [getattr(out, k).cpu().numpy() for k in ("L", "W", "peak", "growth", "count")])
    for r in runs[1:]:
        for a_, b_ in zip(runs[0], r):
            assert np.array_equal(a_, b_)
    y, nh = runs[0][0], runs[0][1]
    ref = oracle_mod.lenpred_weights(h, pw)
    assert _rel_err(y, ref) <= TOL["f32"]
    assert np.array_equal(nh, oracle_mod.quantize(y, n_tok))
    rp = oracle_mod.project(inst, n_tok, nh, n, 50, beta)
    for k, v in zip(("L", "W", "peak", "growth", "count"), runs[0][2:]):
        assert np.array_equal(v, rp[k]), k
    assert err.item() == 0
    # the plain forward (no projection, no n_tok) through the same kernel
    y2, nh2 = star.lenpred_forward(pred, hd)
    torch.cuda.synchronize()
    assert np.array_equal(y2.cpu().numpy(), y)
    assert np.array_equal(nh2.cpu().numpy(), oracle_mod.quantize(y, None))
    pred.close()


def test_f32_small_path_many_instances_falls_back(star, oracle_mod):
    """A projection histogram too large for the kernel's shared memory (600 instances x 52 bins)
    runs the multi-launch fp32 path: same tolerance, projection bit-exact."""
    d, R, n = 896, 128, 600
    pw = datagen.make_predictor_weights(11, d, "f32")
    snap = datagen.make_snapshot(12, n, 1)
    idx = np.arange(R)
    n_tok, inst = snap.n_tok[idx].copy(), snap.inst[idx].astype(np.int32)
    h = datagen.make_hidden(13, R, d, "f32")
    W, b = _weights_dev(pw)
    pred = star.Predictor(*W, *b, max_rows=R)
    beta = datagen.beta_schedule_q16(50)
    ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
    y, nh, out = star.lenpred_forward_project(pred, _dev(h), _dev(n_tok), _dev(inst), n, 50,
                                              _dev(beta.astype(np.int32)), ws)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    assert _rel_err(y, oracle_mod.lenpred_weights(h, pw)) <= TOL["f32"]
    nh = nh[:R].cpu().numpy()
    assert np.array_equal(nh, oracle_mod.quantize(y, n_tok))
    rp = oracle_mod.project(inst, n_tok, nh, n, 50, beta)
    for k in ("L", "W", "peak", "growth", "count"):
        assert np.array_equal(getattr(out, k).cpu().numpy(), rp[k]), k
    pred.close()


def test_example_decode_loop(star):
    """examples/decode_loop.py (the serving-loop example of the README) runs end to end through the
    public API, in both prediction modes."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "decode_loop.py")
    spec = importlib.util.spec_from_file_location("decode_loop", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.main(["--steps", "6", "--requests", "32", "--d", "1024"]) >= 0
    assert mod.main(["--steps", "6", "--requests", "32", "--d", "1024", "--k", "4"]) >= 0
    assert mod.main(["--steps", "12", "--requests", "32", "--d", "1024", "--kv"]) >= 0


_FALLBACK_SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import datagen, oracle
import paper_2510_13668_b200 as star
from paper_2510_13668_b200.step import Step
out = []
for dt, d, R, n in (("bf16", 1024, 384, 4), ("f32", 896, 128, 2)):
    pw = datagen.make_predictor_weights(31, d, dt)
    snap = datagen.make_snapshot(31, n, R // n, skewed=True)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    W = [torch.from_numpy(w).to(tdt).cuda() for w in (pw.W1, pw.W2, pw.W3)]
    pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=R)
    assert pred.path(R) == 0, "the one-launch forms are switched off"
    params_h = datagen.make_plan_params(snap, H=50, max_moves=2)
    st = Step(pred, star.PlanParams.from_host(params_h), n, r_cap=R)
    st.load_requests(*(torch.from_numpy(a) for a in (snap.req_id, snap.inst, snap.n_tok)))
    h = datagen.make_hidden(31, R, d, dt, scale=np.maximum(snap.true_rem, 1).astype(np.float32) / 60.0)
    st.run(torch.from_numpy(h).to(tdt).cuda())
    torch.cuda.synchronize()
    nh = st.v["n_hat"][:R].cpu().numpy()
    y, _ = star.lenpred_forward(pred, torch.from_numpy(h).to(tdt).cuda())
    torch.cuda.synchronize()
    ref = oracle.lenpred_weights(h, pw)
    err = float(np.max(np.abs(y.cpu().numpy() - ref) / np.maximum(np.abs(ref), 1.0)))
    assert err <= (2e-2 if dt == "bf16" else 1e-3), err
    rp = oracle.project(snap.inst, snap.n_tok, nh, n, 50, params_h.beta_q)
    assert np.array_equal(st.v["L"].cpu().numpy(), rp["L"])
    assert st.result() == oracle.plan(params_h, rp["L"], snap.req_id, snap.inst, snap.n_tok, nh, None)
    out.append(err)
print("fallback ok", out)
'''


@pytest.mark.parametrize("env", [{"STAR_SMALL": "0", "STAR_F32_SMALL": "0"},
                                 {"STAR_TAIL2": "0", "STAR_SMALL": "0", "STAR_F32_SMALL": "0"},
                                 {"STAR_PLAN_FUSE": "1", "STAR_SMALL": "0", "STAR_F32_SMALL": "0"}])
def test_fallback_paths_subprocess(star, env):
    """The paths a device takes when the one-launch forms are unavailable (their co-residency
    check fails, e.g. on an MPS partition) or switched off, in a fresh process: the multi-launch
    predictor (round-1 fused tail, 3xTF32 GEMMs), the fused plan in the tail's last CTA; Step ==
    oracle (loads, plan), predictor within tolerance."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FALLBACK_SCRIPT, root], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fallback ok" in r.stdout
