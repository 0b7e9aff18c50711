"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module holds NONE of the method's arithmetic (no predictor, no projection, no
variance, no plan). It only draws numbers: hidden states, predictor weights, a running
request snapshot with long-tailed reasoning-style lengths, and the plan parameters.
Both sides consume exactly the bytes produced here.

Recipe (PAPER.md citations):
  * h ~ N(0,1), rounded RNE to bf16 (bf16 configs) or kept fp32 (C1).  h is the
    last-token, last-layer hidden state, one d-vector per running request
    (§4.2 "LLM-native Predictor").
  * W1, W2, W3 ~ He-normal N(0, 2/fan_in); w4_j = 50*|N(0,1)| (>= 0, so the output layer
    has no cancellation); Eq. 2 widths m1=2048, m2=512, m3=64.
  * prompt p = round(lognormal(ln 36, 2.4)) clipped to [1, 4096]  (Table 2).
  * output L_out: with prob 0.173 near-cap (L_ctx - p, "17.3%"), else
    round(lognormal(7.16, 0.668)) clipped to [1, 30000] and to L_ctx - p.
  * running snapshot: L_out length-biased (long requests occupy slots longer),
    g ~ U{0..L_out-1}, N = p + g, true remaining = L_out - g (STAR-Oracle N̂).
  * instance assignment round-robin; "skewed": instance 0 gets 2x the share
    of near-cap requests (configs C3, C4, TGT: the overloaded instance puts Alg. 1 past Phase 1,
    PAPER.md:428-451, so every planned step scores candidates and moves a request).
  * plan params: H=50, beta_q[t] = round(65536*0.95^t) (SPEC.md:122 reading A6),
    theta = 1/10, T_exec = 5 ms + 10 ns/token, C_mig = c1 * N with
    c1 = KV bytes/token * 8 / bandwidth (Llama-3-8B bf16 KV 131072 B/token over 900 GB/s).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

L_CTX = 32768          # PAPER.md:491 "up to 32K tokens" (reading A10: total-context cap)
M1, M2, M3 = 2048, 512, 64
Q16 = 65536


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------- bf16 bits
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (uint16). NaN stays NaN."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_to_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    """Returns float32 values exactly representable in `dtype` ('bf16' or 'f32')."""
    x = np.asarray(x, dtype=np.float32)
    if dtype == "bf16":
        return bf16_bits_to_f32(f32_to_bf16_bits(x))
    if dtype == "f32":
        return x.copy()
    raise ValueError(dtype)


# ----------------------------------------------------------------------------- predictor
@dataclasses.dataclass
class PredictorWeights:
    d: int
    dtype: str                      # 'bf16' | 'f32' : storage of W1, W2, W3
    W1: np.ndarray                  # [m1, d] float32 (values representable in dtype)
    W2: np.ndarray                  # [m2, m1]
    W3: np.ndarray                  # [m3, m2]
    w4: np.ndarray                  # [m3] float32 (always fp32: used by the fp32 epilogue)
    b1: Optional[np.ndarray] = None  # [m1] fp32 or None (Eq. 2 has no bias, reading A1)
    b2: Optional[np.ndarray] = None
    b3: Optional[np.ndarray] = None
    b4: Optional[float] = None

    @property
    def m1(self):
        return self.W1.shape[0]

    @property
    def m2(self):
        return self.W2.shape[0]

    @property
    def m3(self):
        return self.W3.shape[0]


def make_predictor_weights(seed: int, d: int, dtype: str = "bf16", m1: int = M1, m2: int = M2,
                           m3: int = M3, biases: bool = False, b4: Optional[float] = None,
                           w4_scale: float = 50.0) -> PredictorWeights:
    g = rng(seed)

    def he(out_f, in_f):
        return round_to_dtype(g.standard_normal((out_f, in_f), dtype=np.float32)
                              * np.float32(math.sqrt(2.0 / in_f)), dtype)

    W1 = he(m1, d)
    W2 = he(m2, m1)
    W3 = he(m3, m2)
    w4 = round_to_dtype(np.abs(g.standard_normal(m3, dtype=np.float32)) * np.float32(w4_scale), dtype)
    pw = PredictorWeights(d=d, dtype=dtype, W1=W1, W2=W2, W3=W3, w4=w4)
    if biases:
        pw.b1 = (g.standard_normal(m1, dtype=np.float32) * np.float32(0.1)).astype(np.float32)
        pw.b2 = (g.standard_normal(m2, dtype=np.float32) * np.float32(0.1)).astype(np.float32)
        pw.b3 = (g.standard_normal(m3, dtype=np.float32) * np.float32(0.1)).astype(np.float32)
        pw.b4 = float(np.float32(g.standard_normal() * 10.0))
    if b4 is not None:
        pw.b4 = float(np.float32(b4))
    return pw


def make_hidden(seed: int, R: int, d: int, dtype: str = "bf16", scale: Optional[np.ndarray] = None) -> np.ndarray:
    """[R, d] float32 hidden states, representable in dtype. `scale` (per-row, >0) lets the
    bench steer the predicted lengths (positive homogeneity of bias-free Eq. 2)."""
    g = rng(seed + 7919)
    h = g.standard_normal((R, d), dtype=np.float32)
    if scale is not None:
        h = h * np.asarray(scale, dtype=np.float32)[:, None]
    return round_to_dtype(h, dtype)


# ----------------------------------------------------------------------------- requests
@dataclasses.dataclass
class Snapshot:
    n_inst: int
    req_id: np.ndarray      # [R] int32, globally unique
    inst: np.ndarray        # [R] int32 in [0, n_inst)
    prompt: np.ndarray      # [R] int32
    gen: np.ndarray         # [R] int32 generated so far
    n_tok: np.ndarray       # [R] int32  N(r) = prompt + generated (reading A4)
    true_rem: np.ndarray    # [R] int32  true remaining length (STAR-Oracle N̂)
    pinned: np.ndarray      # [R] uint8  migrating requests (never candidates)

    @property
    def R(self):
        return int(self.req_id.shape[0])


def sample_lengths(g: np.random.Generator, n: int, l_ctx: int = L_CTX, p_cap: float = 0.173):
    p = np.clip(np.rint(g.lognormal(math.log(36.0), 2.4, n)), 1, 4096).astype(np.int64)
    short = np.clip(np.rint(g.lognormal(7.16, 0.668, n)), 1, 30000).astype(np.int64)
    near_cap = g.random(n) < p_cap
    out = np.where(near_cap, l_ctx - p, short)
    out = np.minimum(out, l_ctx - p)
    out = np.maximum(out, 1)
    return p, out, near_cap


def make_snapshot(seed: int, n_inst: int, r_per_inst: int, l_ctx: int = L_CTX, skewed: bool = False,
                  pinned_frac: float = 0.0, id_base: int = 0) -> Snapshot:
    """Running-batch snapshot of n_inst * r_per_inst requests (length-biased draw)."""
    g = rng(seed + 104729)
    R = n_inst * r_per_inst
    pool = max(8 * R, 4096)
    p, out, near = sample_lengths(g, pool, l_ctx)
    w = out.astype(np.float64)
    w /= w.sum()
    pick = g.choice(pool, size=R, replace=True, p=w)
    p, out, near = p[pick], out[pick], near[pick]
    gen = (g.random(R) * out).astype(np.int64)
    gen = np.minimum(gen, out - 1)
    if skewed:
        # instance 0 receives 2x the share of near-cap requests (config C4)
        order = np.argsort(~near, kind="stable")
        inst = np.empty(R, dtype=np.int64)
        slots = np.tile(np.arange(n_inst), r_per_inst)
        weights = np.ones(n_inst)
        weights[0] = 2.0
        cap = np.full(n_inst, r_per_inst)
        # greedily place near-cap requests with a weighted preference for instance 0
        filled = np.zeros(n_inst, dtype=np.int64)
        for k, r in enumerate(order):
            if near[r]:
                prob = weights * (filled < cap)
                prob = prob / prob.sum()
                i = int(g.choice(n_inst, p=prob))
            else:
                free = np.nonzero(filled < cap)[0]
                i = int(free[np.argmin(filled[free])])
            inst[r] = i
            filled[i] += 1
        del slots
    else:
        inst = np.arange(R) % n_inst
    ids = (id_base + g.permutation(R)).astype(np.int32)
    pinned = (g.random(R) < pinned_frac).astype(np.uint8)
    return Snapshot(n_inst=n_inst, req_id=ids, inst=inst.astype(np.int32), prompt=p.astype(np.int32),
                    gen=gen.astype(np.int32), n_tok=(p + gen).astype(np.int32),
                    true_rem=(out - gen).astype(np.int32), pinned=pinned)


# ----------------------------------------------------------------------------- plan params
@dataclasses.dataclass
class PlanParams:
    n_inst: int
    H: int
    beta_q: np.ndarray            # [H+1] uint32, Q16; beta_q[0] = 65536 weights sigma0^2
    theta_num: int = 1
    theta_den: int = 10
    max_moves: int = 1
    c_mem: Optional[np.ndarray] = None      # [n_inst] int64 tokens (None = unlimited)
    reserved: Optional[np.ndarray] = None   # [n_inst] int64 tokens in flight inbound
    t_exec_a_ps: int = 5_000_000_000        # 5 ms
    t_exec_b_ps: int = 10_000               # 10 ns / token
    mig_c0_ps: int = 0
    mig_c1_ps: int = 145_636                # 131072 B/token * 8 / 7.2e12 bit/s (900 GB/s)
    flags: int = 0

    STRICT_MEM = 1
    CURRENT_ONLY = 2


def beta_schedule_q16(H: int, gamma: float = 0.95) -> np.ndarray:
    """beta_q[t] = round(65536 * gamma^t); beta_q[0] = 65536 (reading A6/A11)."""
    return np.array([int(round(Q16 * gamma ** t)) for t in range(H + 1)], dtype=np.uint32)


def make_plan_params(snap: Snapshot, H: int = 50, gamma: float = 0.95, mem_factor: float = 1.10,
                     max_moves: int = 1, flags: int = 0, reserved_seed: Optional[int] = None) -> PlanParams:
    """C_mem_i = floor(mem_factor * mean_j sum_{r in B_j} (N_r + H)) -- a raw-input recipe
    (not the method's projected peak) so that the memory filter binds on some targets."""
    n = snap.n_inst
    per = np.zeros(n, dtype=np.int64)
    np.add.at(per, snap.inst.astype(np.int64), snap.n_tok.astype(np.int64) + H)
    c = int(math.floor(mem_factor * float(per.mean()))) if n > 0 else 0
    c_mem = np.full(n, c, dtype=np.int64)
    reserved = np.zeros(n, dtype=np.int64)
    if reserved_seed is not None:
        g = rng(reserved_seed)
        reserved = (g.random(n) < 0.3).astype(np.int64) * g.integers(0, 20000, n)
    return PlanParams(n_inst=n, H=H, beta_q=beta_schedule_q16(H, gamma), max_moves=max_moves,
                      c_mem=c_mem, reserved=reserved, flags=flags)


# ----------------------------------------------------------------------------- tiny fixtures
def tiny_fixture(seed: int, n: int, R: int, H: int, max_N: int = 40, max_nhat: int = 12,
                 random_beta: bool = True, with_mem: bool = True, with_cost: bool = True):
    """Small random fixtures for brute-force pins: returns (snap, n_hat, params)."""
    g = rng(seed)
    inst = g.integers(0, n, R).astype(np.int32)
    n_tok = g.integers(1, max_N + 1, R).astype(np.int32)
    n_hat = g.integers(0, max_nhat + 1, R).astype(np.int32)
    ids = g.permutation(R * 3)[:R].astype(np.int32)
    pinned = (g.random(R) < 0.1).astype(np.uint8)
    snap = Snapshot(n_inst=n, req_id=ids, inst=inst, prompt=n_tok.copy(), gen=np.zeros(R, np.int32),
                    n_tok=n_tok, true_rem=n_hat.copy(), pinned=pinned)
    if random_beta:
        beta = np.concatenate([[Q16], g.integers(1, Q16 + 1, H)]).astype(np.uint32)
    else:
        beta = beta_schedule_q16(H)
    theta_den = int(g.integers(1, 11))
    theta_num = int(g.integers(0, theta_den + 1))
    c_mem = None
    reserved = None
    if with_mem:
        c_mem = g.integers(max_N, max_N * max(R, 1) + 2, n).astype(np.int64)
        reserved = g.integers(0, max_N, n).astype(np.int64) * (g.random(n) < 0.5)
    a = int(g.integers(0, 50)) if with_cost else 1
    b = int(g.integers(0, 3)) if with_cost else 0
    c0 = int(g.integers(0, 200)) if with_cost else 0
    c1 = int(g.integers(0, 4)) if with_cost else 0
    params = PlanParams(n_inst=n, H=H, beta_q=beta, theta_num=theta_num, theta_den=theta_den,
                        max_moves=int(g.integers(1, 4)), c_mem=c_mem, reserved=reserved,
                        t_exec_a_ps=a, t_exec_b_ps=b, mig_c0_ps=c0, mig_c1_ps=c1,
                        flags=int(g.integers(0, 4)))
    return snap, n_hat, params


# ----------------------------------------------------------------------------- configs
CONFIGS = {
    # BASELINE.json configs[0..4] (+ the north-star target point TGT)
    "C1": dict(n_inst=2, r_per_inst=64, d=896, dtype="f32", max_moves=1,
               desc="2 decode instances x 64 requests, hidden 896 (Qwen2.5-0.5B-shaped), fp32, 1 reschedule round"),
    "C2": dict(n_inst=8, r_per_inst=256, d=4096, dtype="bf16", max_moves=1,
               desc="8 instances x 256 requests, hidden 4096 (Llama-3-8B-shaped), bf16, long-tailed CoT lengths"),
    "C3": dict(n_inst=8, r_per_inst=512, d=5120, dtype="bf16", max_moves=1, skewed=True,
               desc="8 instances x 512 requests, hidden 5120 (Qwen-32B-shaped), per-step prediction + rebalance "
                    "(instance 0 holds 2x the near-cap share, so Alg. 1 moves a request every step)"),
    "C4": dict(n_inst=4, r_per_inst=1024, d=4096, dtype="bf16", max_moves=4, skewed=True, mem_factor=1.02,
               desc="4 instances x 1024 requests, hidden 4096, skewed arrivals near KV-OOM"),
    "C5": dict(n_inst=8, r_per_inst=512, d=4096, dtype="bf16", max_moves=1, skewed=True,
               r_sweep=(64, 128, 256, 512, 1024, 2048),
               desc="scaling sweep: one instance per GPU, 64-2048 requests per instance, hidden 4096, bf16, "
                    "skewed (r_per_inst is the sweep variable)"),
    "TGT": dict(n_inst=8, r_per_inst=512, d=4096, dtype="bf16", max_moves=1, skewed=True,
                desc="north-star target: 8 instances x 512 requests, hidden 4096, bf16, skewed (instance 0 holds "
                     "2x the near-cap share: overloaded, so Alg. 1 reaches Phases 2-3 and moves a request)"),
}
