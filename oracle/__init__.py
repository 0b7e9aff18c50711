"""STAR CPU oracle -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over oracle/liboracle.so (oracle/oracle.cpp) plus the independent
pure-Python brute force in oracle/brute.py.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this package.  It never
imports the product package (paper_2510_13668_b200) and the product never imports it.

Function map (each cites the passage it follows in oracle.cpp):
  lenpred(...)    Eq. 2, PAPER.md:237-241 (fp64 accumulation)
  quantize(...)   readings A8-A10 (round-half-even, total-context cap)
  project(...)    PAPER.md:366, 375, 384, 425 (literal O(R*H) loop)
  objective(...)  Eq. 3-4, PAPER.md:368-380 (exact integer Phi*n^2)
  plan(...)       Alg. 1, PAPER.md:405-453 (from-scratch objective per candidate)
  dispatch(...)   P -> D placement (reading A28), objective from scratch
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++, -O2 -ffp-contract=off, OpenMP over requests only)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-std=c++17", "-Wall", _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        I = C.c_int
        _lib.oracle_lenpred.argtypes = [I, I, I, I, I, P, C.c_long, P, P, P, P, P, P, P, P, P, I]
        _lib.oracle_lenpred.restype = I
        _lib.oracle_quantize.argtypes = [I, P, P, C.c_int32, P]
        _lib.oracle_quantize.restype = None
        _lib.oracle_project.argtypes = [I, I, I, I, P, P, P, P, P, P, P, P, P]
        _lib.oracle_project.restype = I
        _lib.oracle_objective.argtypes = [I, I, P, P, I, P, P]
        _lib.oracle_objective.restype = None
        _lib.oracle_plan.argtypes = [I, I, I, C.c_int32, C.c_int32, P, P, P, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_uint32, P, I, P, P, P, P, P,
                                     P, P, P, P, P, P]
        _lib.oracle_plan.restype = I
        _lib.oracle_dispatch.argtypes = [I, I, I, P, P, P, P, I, P, P, C.c_int32, P]
        _lib.oracle_dispatch.restype = I
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def lenpred(h, W1, W2, W3, w4, b1=None, b2=None, b3=None, b4=None, nthreads=None):
    """y_hat [R] float64 = Eq. 2 on exact fp32 inputs with fp64 accumulation."""
    h = _c(h, np.float32)
    R, d = h.shape
    W1, W2, W3, w4 = (_c(x, np.float32) for x in (W1, W2, W3, w4))
    m1, m2, m3 = W1.shape[0], W2.shape[0], W3.shape[0]
    assert W1.shape == (m1, d) and W2.shape == (m2, m1) and W3.shape == (m3, m2) and w4.shape == (m3,)
    b1, b2, b3 = _c(b1, np.float32), _c(b2, np.float32), _c(b3, np.float32)
    b4a = None if b4 is None else np.array([b4], dtype=np.float32)
    y = np.zeros(R, dtype=np.float64)
    nt = nthreads if nthreads else (os.cpu_count() or 1)
    rc = lib().oracle_lenpred(R, d, m1, m2, m3, _p(h), d, _p(W1), _p(W2), _p(W3), _p(w4),
                              _p(b1), _p(b2), _p(b3), _p(b4a), _p(y), nt)
    assert rc == 0, rc
    return y


def lenpred_weights(h, pw, nthreads=None):
    return lenpred(h, pw.W1, pw.W2, pw.W3, pw.w4, pw.b1, pw.b2, pw.b3, pw.b4, nthreads)


def quantize(y, n_tok=None, l_ctx=32768):
    y = _c(y, np.float32)
    out = np.zeros(y.shape[0], dtype=np.int32)
    n_tok = _c(n_tok, np.int32)
    lib().oracle_quantize(y.shape[0], _p(y), _p(n_tok), l_ctx, _p(out))
    return out


def project(inst, n_tok, n_hat, n_inst, H, beta_q, inst_base=0):
    inst, n_tok, n_hat = _c(inst, np.int32), _c(n_tok, np.int32), _c(n_hat, np.int32)
    beta_q = _c(beta_q, np.uint32)
    assert beta_q.shape[0] == H + 1
    L = np.zeros((n_inst, H + 1), dtype=np.int64)
    W = np.zeros(n_inst, dtype=np.int64)
    peak = np.zeros(n_inst, dtype=np.int64)
    G = np.zeros(n_inst, dtype=np.int64)
    cnt = np.zeros(n_inst, dtype=np.int32)
    rc = lib().oracle_project(inst.shape[0], n_inst, inst_base, H, _p(inst), _p(n_tok), _p(n_hat),
                              _p(beta_q), _p(L), _p(W), _p(peak), _p(G), _p(cnt))
    if rc != 0:
        raise ValueError(f"oracle_project: bad instance id (rc={rc})")
    return dict(L=L, W=W, peak=peak, growth=G, count=cnt)


def objective(L, beta_q, current_only=False):
    """Exact Phi * n^2 (Eq. 3-4 truncated at H) as a Python int."""
    L = _c(L, np.int64)
    n, H1 = L.shape
    hi = C.c_int64()
    lo = C.c_uint64()
    lib().oracle_objective(n, H1 - 1, _p(L), _p(_c(beta_q, np.uint32)), int(current_only),
                           C.byref(hi), C.byref(lo))
    return (hi.value << 64) | lo.value


def plan(params, L, req_id, inst, n_tok, n_hat, pinned=None):
    """Greedy Alg. 1 rounds; returns list of (req_id, src, dst, round, gain:int)."""
    L = _c(L, np.int64)
    n, H1 = L.shape
    H = H1 - 1
    assert n == params.n_inst and H == params.H
    R = int(np.asarray(req_id).shape[0])
    mm = max(params.max_moves, 0)
    cap = max(mm, 1)
    mv = [np.zeros(cap, dtype=np.int32) for _ in range(4)]
    ghi = np.zeros(cap, dtype=np.int64)
    glo = np.zeros(cap, dtype=np.uint64)
    args = [_c(req_id, np.int32), _c(inst, np.int32), _c(n_tok, np.int32), _c(n_hat, np.int32)]
    pin = _c(pinned, np.uint8)
    rc = lib().oracle_plan(n, H, mm, params.theta_num, params.theta_den, _p(_c(params.beta_q, np.uint32)),
                           _p(_c(params.c_mem, np.int64)), _p(_c(params.reserved, np.int64)),
                           params.t_exec_a_ps, params.t_exec_b_ps, params.mig_c0_ps, params.mig_c1_ps,
                           params.flags, _p(L), R, *(_p(a) for a in args), _p(pin),
                           *(_p(a) for a in mv), _p(ghi), _p(glo))
    if rc < 0:
        raise ValueError(f"oracle_plan: bad input (rc={rc})")
    out = []
    for k in range(rc):
        g = (int(ghi[k]) << 64) | int(glo[k])
        out.append((int(mv[0][k]), int(mv[1][k]), int(mv[2][k]), int(mv[3][k]), g))
    return out


DISPATCH_RR, DISPATCH_CURRENT_LOAD, DISPATCH_PROJECTED = 0, 1, 2


def dispatch(policy, L, beta_q, n_tok, n_hat, c_mem=None, reserved=None, counter=0):
    """Places arrivals in order; returns (assign [A] int32 (-1 = not placed), updated L)."""
    L = np.array(L, dtype=np.int64, copy=True)
    n, H1 = L.shape
    A = int(np.asarray(n_tok).shape[0])
    out = np.zeros(max(A, 1), dtype=np.int32)
    lib().oracle_dispatch(int(policy), n, H1 - 1, _p(_c(beta_q, np.uint32)), _p(L), _p(_c(c_mem, np.int64)),
                          _p(_c(reserved, np.int64)), A, _p(_c(n_tok, np.int32)), _p(_c(n_hat, np.int32)),
                          int(counter), _p(out))
    return out[:A], L


def should_refresh(gen, g_last, k):
    """true iff no prediction yet (g_last < 0) or gen - g_last >= k."""
    return (np.asarray(g_last) < 0) | (np.asarray(gen, np.int64) - np.asarray(g_last) >= k)


def refresh_step(h, pw, n_tok, gen, g_last, nhat_last, k, l_ctx=32768):
    """One step of the prediction cadence (NEXT-1, reading A27), plain loops:
    rows due for a refresh get N_hat = quantize(Eq. 2(h_r)) (fp64 oracle value rounded to fp32
    before the quantizer) and g_last = gen, nhat_last = N_hat; the others age by the tokens
    generated since their last prediction.  Returns (n_hat, g_last', nhat_last', refreshed mask)."""
    gen = np.asarray(gen, np.int64)
    g_last = np.array(g_last, np.int32, copy=True)
    nhat_last = np.array(nhat_last, np.int32, copy=True)
    due = should_refresh(gen, g_last, k)
    n_hat = np.zeros(gen.shape[0], np.int32)
    rows = np.nonzero(due)[0]
    if rows.size:
        y = lenpred_weights(h[rows], pw)
        q = quantize(y.astype(np.float32), np.asarray(n_tok)[rows], l_ctx)
        n_hat[rows] = q
        g_last[rows] = gen[rows]
        nhat_last[rows] = q
    for r in np.nonzero(~due)[0]:
        n_hat[r] = max(0, int(nhat_last[r]) - int(gen[r] - g_last[r]))
    return n_hat, g_last, nhat_last, due


# ----------------------------------------------------------------------------- KV migration (NEXT-4)
# ExecuteMigration(m*) (Alg. 1 line 10; §5.4) moves the request's
# KV cache: for every layer l and every block j of the request, block src_table[j] of the source
# pool becomes block dst_table[j] of the destination pool.  Plain loops over (l, j) with slice
# copies; a pool is a numpy array [n_layers][n_blocks][block_bytes] (uint8).
def kv_pack(pool, table):
    """staging[l][j] = pool[l][table[j]]."""
    pool = np.asarray(pool)
    n_layers, _, bb = pool.shape
    out = np.zeros((n_layers, len(table), bb), dtype=pool.dtype)
    for layer in range(n_layers):
        for j, b in enumerate(table):
            out[layer, j, :] = pool[layer, int(b), :]
    return out


def kv_unpack(staging, pool, table):
    """Returns a copy of pool with pool[l][table[j]] = staging[l][j]."""
    pool = np.array(pool, copy=True)
    for layer in range(pool.shape[0]):
        for j, b in enumerate(table):
            pool[layer, int(b), :] = staging[layer, j, :]
    return pool


def kv_migrate(src_pool, src_table, dst_pool, dst_table):
    """Returns a copy of dst_pool with dst[l][dst_table[j]] = src[l][src_table[j]]."""
    dst = np.array(dst_pool, copy=True)
    for layer in range(dst.shape[0]):
        for j in range(len(src_table)):
            dst[layer, int(dst_table[j]), :] = src_pool[layer, int(src_table[j]), :]
    return dst
