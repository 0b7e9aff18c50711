"""ctypes binding to libstar.so (include/star.h).  Argument marshalling only: every step of
the path runs in the library's CUDA kernels.  There is no CPU fallback: if the library is
missing or the device is not sm_100a, every call raises."""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstar.so")

STAR_F32, STAR_BF16 = 0, 1
STRICT_MEM, CURRENT_ONLY = 1, 2
L_CTX = 32768

P = C.c_void_p
I = C.c_int
I32 = C.c_int32
I64 = C.c_int64


class StarError(RuntimeError):
    pass


class PlanParamsC(C.Structure):
    _fields_ = [("n_inst", I), ("H", I), ("max_moves", I), ("theta_num", I32), ("theta_den", I32),
                ("beta_q", P), ("c_mem", P), ("reserved", P), ("t_exec_a_ps", I64), ("t_exec_b_ps", I64),
                ("mig_c0_ps", I64), ("mig_c1_ps", I64), ("flags", C.c_uint32)]


class PlanSegmentsC(C.Structure):
    _fields_ = [("world", I), ("n_loc", I), ("r_cap", I), ("seg_stride", I64), ("L", P), ("r_count", P),
                ("req_id", P), ("inst", P), ("n_tok", P), ("n_hat", P), ("pinned", P)]


class KvPoolC(C.Structure):
    _fields_ = [("base", P), ("n_layers", I), ("layer_stride", I64), ("n_blocks", I64), ("block_bytes", I64)]


MOVE_DTYPE = np.dtype([("req_id", "<i4"), ("src", "<i4"), ("dst", "<i4"), ("round", "<i4"),
                       ("gain_hi", "<i8"), ("gain_lo", "<u8")])
MOVE_BYTES = 32

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise StarError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    sig = {
        "star_last_error": ([], C.c_char_p),
        "star_version": ([], C.c_char_p),
        "star_predictor_create": ([C.POINTER(P), I, I, I, I, I, P, P, P, P, P, P, P, P, I, P], I),
        "star_predictor_destroy": ([P], I),
        "star_predictor_layer1_timing": ([P, I], I),
        "star_predictor_layer1_ms": ([P, C.POINTER(C.c_float)], I),
        "star_predictor_path": ([P, I, C.POINTER(I)], I),
        "star_predictor_timeline": ([P, I, P, I, C.POINTER(I)], I),
        "lenpred_forward": ([P, P, I64, I, P, I32, P, P, P], I),
        "lenpred_quantize": ([P, P, I, I32, P, P], I),
        "lenpred_forward_project": ([P, P, I64, I, P, I32, P, P, I, I, I, P, P, P, P, P, P, P, P, P, P], I),
        "lenpred_forward_refresh": ([P, P, I64, I, P, I32, P, P, P, I32, P, P, P], I),
        "lenpred_forward_refresh_project": ([P, P, I64, I, P, I32, P, P, P, I32, P, P, I, I, I, P, P, P, P, P, P, P,
                                             P, P, P], I),
        "star_project_workspace_bytes": ([I, I], C.c_size_t),
        "star_project_single_cta_max_rows": ([], I),
        "project_instance_load": ([I, I, I, I, P, P, P, P, P, P, P, P, P, P, P, P], I),
        "plan_reschedule": ([C.POINTER(PlanParamsC), P, I, P, P, P, P, P, P, P, P, P], I),
        "plan_reschedule_segmented": ([C.POINTER(PlanParamsC), C.POINTER(PlanSegmentsC), P, P, P, P], I),
        "lenpred_forward_project_plan": ([P, P, I64, I, P, I32, P, P, I, I, P, P, P, P, P, P, P, P,
                                          C.POINTER(PlanParamsC), C.POINTER(PlanSegmentsC), P, P, P, P], I),
        "star_dispatch_workspace_bytes": ([I, I], C.c_size_t),
        "star_plan_workspace_bytes": ([I, I, I64], C.c_size_t),
        "star_plan_timeline": ([P], I),
        "plan_reschedule_segmented_ws": ([C.POINTER(PlanParamsC), C.POINTER(PlanSegmentsC), P, P, P, P, P], I),
        "dispatch_requests": ([I, I, I, P, P, P, P, I, P, P, I32, P, P, P], I),
        "kv_pack": ([C.POINTER(KvPoolC), P, I, P, P, P], I),
        "kv_unpack": ([P, C.POINTER(KvPoolC), P, I, P, P], I),
        "kv_migrate": ([C.POINTER(KvPoolC), P, C.POINTER(KvPoolC), P, I, P, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().star_last_error().decode(errors="replace")
        raise StarError(f"{what} failed (status {rc}): {msg}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise StarError("expected a CUDA tensor (the library takes device pointers)")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _req(t: torch.Tensor, dtype: torch.dtype, name: str):
    if t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
        raise StarError(f"{name} must be a contiguous CUDA {dtype} tensor (got {t.dtype}, {t.device})")
    return t


def version() -> str:
    return lib().star_version().decode()


# ================================================================ predictor (Eq. 2)
class Predictor:
    """Handle over star_predictor_create; keeps references to the weights it was built on."""

    def __init__(self, W1, W2, W3, w4, b1=None, b2=None, b3=None, b4=None, max_rows=4096, stream=None):
        dt = W1.dtype
        if dt == torch.bfloat16:
            self.dt = STAR_BF16
        elif dt == torch.float32:
            self.dt = STAR_F32
        else:
            raise StarError("weights must be bf16 or fp32")
        for n_, t in (("W2", W2), ("W3", W3)):
            _req(t, dt, n_)
        _req(W1, dt, "W1")
        _req(w4, torch.float32, "w4")
        for n_, t in (("b1", b1), ("b2", b2), ("b3", b3), ("b4", b4)):
            if t is not None:
                _req(t, torch.float32, n_)
        self.m1, self.d = W1.shape
        self.m2 = W2.shape[0]
        self.m3 = W3.shape[0]
        self.max_rows = max_rows
        self._keep = (W1, W2, W3, w4, b1, b2, b3, b4)
        h = P()
        _check(lib().star_predictor_create(C.byref(h), self.d, self.m1, self.m2, self.m3, self.dt,
                                           _ptr(W1), _ptr(W2), _ptr(W3), _ptr(w4), _ptr(b1), _ptr(b2),
                                           _ptr(b3), _ptr(b4), max_rows, _stream(stream)),
               "star_predictor_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().star_predictor_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layer1_timing(self, enable: bool = True):
        """Library-owned CUDA events around every layer-1 GEMM launch (see star.h)."""
        _check(lib().star_predictor_layer1_timing(self.handle, int(enable)), "layer1_timing")

    def timeline(self, enable: bool = True, fetch: bool = False, layer1: bool = False, raw: bool = False):
        """Diagnostics: per-CTA phase stamps of the fused tail / layer-1 GEMM (star_predictor_timeline)."""
        if not fetch:
            _check(lib().star_predictor_timeline(self.handle, (2 if layer1 else 1) if enable else 0, None, 0, None),
                   "timeline")
            return None
        buf = np.zeros((4 * 148, 16 if layer1 else 32), dtype=np.uint64)
        n = I()
        _check(lib().star_predictor_timeline(self.handle, 2 if layer1 else 1, buf.ctypes.data_as(P), buf.shape[0],
                                             C.byref(n)), "timeline")
        return buf if raw else buf[: n.value]

    def layer1_ms(self) -> float:
        ms = C.c_float()
        _check(lib().star_predictor_layer1_ms(self.handle, C.byref(ms)), "layer1_ms")
        return float(ms.value)

    def path(self, R: int) -> int:
        """1 if a forward of R rows runs the one-launch small-batch (bf16) kernel, 2 the one-launch fp32
        kernel, else 0 (star.h)."""
        v = C.c_int()
        _check(lib().star_predictor_path(self.handle, int(R), C.byref(v)), "star_predictor_path")
        return int(v.value)


def _h_ld(h: torch.Tensor, pred: "Predictor") -> int:
    """Row stride (elements) of the hidden-state matrix: rows contiguous, unit column stride.  An
    empty batch (R = 0) carries no data, whatever strides torch gave the empty view."""
    if h.dim() != 2:
        raise StarError("h must be 2-D")
    if h.shape[0] == 0:
        return pred.d
    if h.stride(1) != 1:
        raise StarError("h must be 2-D with unit column stride")
    return h.stride(0)


def lenpred_forward(pred: Predictor, h: torch.Tensor, n_tok: Optional[torch.Tensor] = None,
                    max_ctx_len: int = L_CTX, y_hat: Optional[torch.Tensor] = None,
                    n_hat: Optional[torch.Tensor] = None, want_y: bool = True, want_n: bool = True,
                    stream=None):
    """Eq. 2 forward on the rows of h ([R, ld_h >= d], dtype of the predictor)."""
    R = h.shape[0]
    ld_h = _h_ld(h, pred)
    exp = torch.bfloat16 if pred.dt == STAR_BF16 else torch.float32
    if h.dtype != exp or not h.is_cuda:
        raise StarError(f"h must be a CUDA {exp} tensor")
    dev = h.device
    if y_hat is None and want_y:
        y_hat = torch.empty(R, dtype=torch.float32, device=dev)
    if n_hat is None and want_n:
        n_hat = torch.empty(R, dtype=torch.int32, device=dev)
    if n_tok is not None:
        _req(n_tok, torch.int32, "n_tok")
    _check(lib().lenpred_forward(pred.handle, _ptr(h), ld_h, R, _ptr(n_tok), max_ctx_len,
                                 _ptr(y_hat), _ptr(n_hat), _stream(stream)), "lenpred_forward")
    return y_hat, n_hat


def lenpred_forward_project(pred: Predictor, h: torch.Tensor, n_tok: torch.Tensor, inst: torch.Tensor, n_inst: int,
                            H: int, beta_q: torch.Tensor, workspace: torch.Tensor, inst_base: int = 0,
                            max_ctx_len: int = L_CTX, y_hat: Optional[torch.Tensor] = None,
                            n_hat: Optional[torch.Tensor] = None, out: Optional["ProjectOut"] = None,
                            err_flag: Optional[torch.Tensor] = None, want_y: bool = True, stream=None):
    """Eq. 2 forward fused with the projection of its N_hat (star.h lenpred_forward_project)."""
    R = h.shape[0]
    ld_h = _h_ld(h, pred)
    exp = torch.bfloat16 if pred.dt == STAR_BF16 else torch.float32
    if h.dtype != exp or not h.is_cuda:
        raise StarError(f"h must be a CUDA {exp} tensor")
    for n_, t in (("n_tok", n_tok), ("inst", inst), ("beta_q", beta_q)):
        _req(t, torch.int32, n_)
    dev = h.device
    if y_hat is None and want_y:
        y_hat = torch.empty(R, dtype=torch.float32, device=dev)
    if n_hat is None:
        n_hat = torch.empty(max(R, 1), dtype=torch.int32, device=dev)
    if out is None:
        out = ProjectOut(n_inst, H, dev)
    _check(lib().lenpred_forward_project(pred.handle, _ptr(h), ld_h, R, _ptr(n_tok), max_ctx_len,
                                         _ptr(y_hat), _ptr(n_hat), n_inst, inst_base, H, _ptr(inst), _ptr(beta_q),
                                         _ptr(out.L), _ptr(out.W), _ptr(out.peak), _ptr(out.growth),
                                         _ptr(out.count), _ptr(workspace), _ptr(err_flag), _stream(stream)),
           "lenpred_forward_project")
    return y_hat, n_hat, out


def lenpred_forward_project_plan(pred: Predictor, h: torch.Tensor, n_tok: torch.Tensor, inst: torch.Tensor,
                                 n_inst: int, H: int, beta_q: torch.Tensor, workspace: torch.Tensor,
                                 params: "PlanParams", seg: "PlanSegmentsC", moves: torch.Tensor,
                                 n_moves: torch.Tensor, n_hat: torch.Tensor, out: "ProjectOut",
                                 max_ctx_len: int = L_CTX, y_hat: Optional[torch.Tensor] = None,
                                 err_flag: Optional[torch.Tensor] = None, stream=None):
    """One-rank step: forward + projection + Alg. 1 (star.h lenpred_forward_project_plan)."""
    R = h.shape[0]
    ld_h = _h_ld(h, pred)
    exp = torch.bfloat16 if pred.dt == STAR_BF16 else torch.float32
    if h.dtype != exp or not h.is_cuda:
        raise StarError(f"h must be a CUDA {exp} tensor")
    for n_, t in (("n_tok", n_tok), ("inst", inst), ("beta_q", beta_q), ("n_hat", n_hat)):
        _req(t, torch.int32, n_)
    _check(lib().lenpred_forward_project_plan(pred.handle, _ptr(h), ld_h, R, _ptr(n_tok), max_ctx_len,
                                              _ptr(y_hat), _ptr(n_hat), n_inst, H, _ptr(inst), _ptr(beta_q),
                                              _ptr(out.L), _ptr(out.W), _ptr(out.peak), _ptr(out.growth),
                                              _ptr(out.count), _ptr(workspace), C.byref(params.c), C.byref(seg),
                                              _ptr(moves), _ptr(n_moves), _ptr(err_flag), _stream(stream)),
           "lenpred_forward_project_plan")
    return moves, n_moves


def lenpred_forward_refresh(pred: Predictor, h: torch.Tensor, n_tok: torch.Tensor, gen: torch.Tensor,
                            g_last: torch.Tensor, nhat_last: torch.Tensor, k: int, max_ctx_len: int = L_CTX,
                            n_hat: Optional[torch.Tensor] = None, n_refreshed: Optional[torch.Tensor] = None,
                            stream=None):
    """Prediction cadence k (star.h lenpred_forward_refresh); g_last / nhat_last are updated in place."""
    R = h.shape[0]
    ld_h = _h_ld(h, pred)
    if h.dtype != torch.bfloat16 or not h.is_cuda:
        raise StarError("h must be a 2-D CUDA bf16 tensor with unit column stride")
    for n_, t in (("n_tok", n_tok), ("gen", gen), ("g_last", g_last), ("nhat_last", nhat_last)):
        _req(t, torch.int32, n_)
    if n_hat is None:
        n_hat = torch.empty(max(R, 1), dtype=torch.int32, device=h.device)
    _check(lib().lenpred_forward_refresh(pred.handle, _ptr(h), ld_h, R, _ptr(n_tok), max_ctx_len, _ptr(gen),
                                         _ptr(g_last), _ptr(nhat_last), int(k), _ptr(n_hat), _ptr(n_refreshed),
                                         _stream(stream)), "lenpred_forward_refresh")
    return n_hat[:R]


def lenpred_forward_refresh_project(pred: Predictor, h: torch.Tensor, n_tok: torch.Tensor, gen: torch.Tensor,
                                    g_last: torch.Tensor, nhat_last: torch.Tensor, k: int, inst: torch.Tensor,
                                    n_inst: int, H: int, beta_q: torch.Tensor, workspace: torch.Tensor,
                                    inst_base: int = 0, max_ctx_len: int = L_CTX,
                                    n_hat: Optional[torch.Tensor] = None, n_refreshed: Optional[torch.Tensor] = None,
                                    out: Optional["ProjectOut"] = None, err_flag: Optional[torch.Tensor] = None,
                                    R: Optional[int] = None, stream=None):
    """Cadence-k step of one worker (star.h lenpred_forward_refresh_project): refresh + projection."""
    R = h.shape[0] if R is None else R
    ld_h = _h_ld(h, pred)
    if h.dtype != torch.bfloat16 or not h.is_cuda:
        raise StarError("h must be a 2-D CUDA bf16 tensor with unit column stride")
    for n_, t in (("n_tok", n_tok), ("gen", gen), ("g_last", g_last), ("nhat_last", nhat_last), ("inst", inst),
                  ("beta_q", beta_q)):
        _req(t, torch.int32, n_)
    if n_hat is None:
        n_hat = torch.empty(max(R, 1), dtype=torch.int32, device=h.device)
    if out is None:
        out = ProjectOut(n_inst, H, h.device)
    _check(lib().lenpred_forward_refresh_project(
        pred.handle, _ptr(h), ld_h, R, _ptr(n_tok), max_ctx_len, _ptr(gen), _ptr(g_last), _ptr(nhat_last),
        int(k), _ptr(n_hat), _ptr(n_refreshed), n_inst, inst_base, H, _ptr(inst), _ptr(beta_q), _ptr(out.L),
        _ptr(out.W), _ptr(out.peak), _ptr(out.growth), _ptr(out.count), _ptr(workspace), _ptr(err_flag),
        _stream(stream)), "lenpred_forward_refresh_project")
    return n_hat[:R], out


def lenpred_quantize(y_hat: torch.Tensor, n_tok: Optional[torch.Tensor] = None, max_ctx_len: int = L_CTX,
                     n_hat: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    _req(y_hat, torch.float32, "y_hat")
    if n_tok is not None:
        _req(n_tok, torch.int32, "n_tok")
    R = y_hat.shape[0]
    if n_hat is None:
        n_hat = torch.empty(R, dtype=torch.int32, device=y_hat.device)
    _check(lib().lenpred_quantize(_ptr(y_hat), _ptr(n_tok), R, max_ctx_len, _ptr(n_hat), _stream(stream)),
           "lenpred_quantize")
    return n_hat


# ================================================================ projection
def project_workspace_bytes(n_inst: int, H: int) -> int:
    return int(lib().star_project_workspace_bytes(n_inst, H))


class ProjectOut:
    def __init__(self, n_inst: int, H: int, device, L: Optional[torch.Tensor] = None):
        self.L = L if L is not None else torch.empty((n_inst, H + 1), dtype=torch.int64, device=device)
        self.W = torch.empty(n_inst, dtype=torch.int64, device=device)
        self.peak = torch.empty(n_inst, dtype=torch.int64, device=device)
        self.growth = torch.empty(n_inst, dtype=torch.int64, device=device)
        self.count = torch.empty(n_inst, dtype=torch.int32, device=device)


def project_instance_load(inst: torch.Tensor, n_tok: torch.Tensor, n_hat: torch.Tensor, n_inst: int, H: int,
                          beta_q: torch.Tensor, inst_base: int = 0, out: Optional[ProjectOut] = None,
                          workspace: Optional[torch.Tensor] = None, err_flag: Optional[torch.Tensor] = None,
                          R: Optional[int] = None, stream=None) -> ProjectOut:
    for n_, t in (("inst", inst), ("n_tok", n_tok), ("n_hat", n_hat), ("beta_q", beta_q)):
        _req(t, torch.int32, n_)
    R = inst.shape[0] if R is None else R
    if out is None:
        out = ProjectOut(n_inst, H, inst.device)
    _check(lib().project_instance_load(R, n_inst, inst_base, H, _ptr(inst), _ptr(n_tok), _ptr(n_hat), _ptr(beta_q),
                                       _ptr(out.L), _ptr(out.W), _ptr(out.peak), _ptr(out.growth),
                                       _ptr(out.count), _ptr(workspace), _ptr(err_flag), _stream(stream)),
           "project_instance_load")
    return out


# ================================================================ plan
class PlanParams:
    """Device-resident star_plan_params (beta_q / c_mem / reserved live in CUDA tensors)."""

    def __init__(self, n_inst, H, beta_q, theta_num=1, theta_den=10, max_moves=1, c_mem=None, reserved=None,
                 t_exec_a_ps=5_000_000_000, t_exec_b_ps=10_000, mig_c0_ps=0, mig_c1_ps=145_636, flags=0,
                 device="cuda"):
        self.beta_q = torch.as_tensor(np.asarray(beta_q, dtype=np.int64).astype(np.int32), device=device)
        self.c_mem = None if c_mem is None else torch.as_tensor(np.asarray(c_mem, dtype=np.int64), device=device)
        self.reserved = None if reserved is None else torch.as_tensor(np.asarray(reserved, dtype=np.int64),
                                                                        device=device)
        self.n_inst, self.H, self.max_moves = int(n_inst), int(H), int(max_moves)
        self.c = PlanParamsC(self.n_inst, self.H, self.max_moves, int(theta_num), int(theta_den),
                             _ptr(self.beta_q), _ptr(self.c_mem), _ptr(self.reserved), int(t_exec_a_ps),
                             int(t_exec_b_ps), int(mig_c0_ps), int(mig_c1_ps), int(flags))

    @classmethod
    def from_host(cls, hp, device="cuda"):
        """From a datagen.PlanParams-like object (duck-typed; no import of datagen here)."""
        return cls(hp.n_inst, hp.H, hp.beta_q, hp.theta_num, hp.theta_den, hp.max_moves, hp.c_mem, hp.reserved,
                   hp.t_exec_a_ps, hp.t_exec_b_ps, hp.mig_c0_ps, hp.mig_c1_ps, hp.flags, device)


def alloc_moves(max_moves: int, device="cuda"):
    return (torch.zeros(max(max_moves, 1) * MOVE_BYTES, dtype=torch.uint8, device=device),
            torch.zeros(1, dtype=torch.int32, device=device))


def decode_moves(moves_buf: torch.Tensor, n_moves) -> list:
    """Host decode: [(req_id, src, dst, round, gain_int)]."""
    n = int(n_moves.item() if torch.is_tensor(n_moves) else n_moves)
    raw = moves_buf.detach().cpu().numpy()[: n * MOVE_BYTES].view(MOVE_DTYPE)
    return [(int(m["req_id"]), int(m["src"]), int(m["dst"]), int(m["round"]),
             (int(m["gain_hi"]) << 64) | int(m["gain_lo"])) for m in raw]


def plan_reschedule(params: PlanParams, L: torch.Tensor, req_id, inst, n_tok, n_hat, pinned=None,
                    moves=None, n_moves=None, err_flag=None, R_total: Optional[int] = None, stream=None):
    _req(L, torch.int64, "L")
    for n_, t in (("req_id", req_id), ("inst", inst), ("n_tok", n_tok), ("n_hat", n_hat)):
        _req(t, torch.int32, n_)
    if pinned is not None:
        _req(pinned, torch.uint8, "pinned")
    if moves is None:
        moves, n_moves = alloc_moves(params.max_moves, L.device)
    R = req_id.shape[0] if R_total is None else R_total
    _check(lib().plan_reschedule(C.byref(params.c), _ptr(L), R, _ptr(req_id), _ptr(inst), _ptr(n_tok), _ptr(n_hat),
                                 _ptr(pinned), _ptr(moves), _ptr(n_moves), _ptr(err_flag), _stream(stream)),
           "plan_reschedule")
    return moves, n_moves


def plan_workspace_bytes(n_inst: int, H: int, request_slots: int) -> int:
    return int(lib().star_plan_workspace_bytes(n_inst, H, request_slots))


def plan_reschedule_large(params: PlanParams, L: torch.Tensor, req_id, inst, n_tok, n_hat, pinned=None,
                          moves=None, n_moves=None, err_flag=None, workspace=None, R_total: Optional[int] = None,
                          stream=None):
    """Cluster-scale multi-CTA plan (star.h plan_reschedule_segmented_ws) on a contiguous state."""
    _req(L, torch.int64, "L")
    for n_, t in (("req_id", req_id), ("inst", inst), ("n_tok", n_tok), ("n_hat", n_hat)):
        _req(t, torch.int32, n_)
    if pinned is not None:
        _req(pinned, torch.uint8, "pinned")
    if moves is None:
        moves, n_moves = alloc_moves(params.max_moves, L.device)
    R = req_id.shape[0] if R_total is None else R_total
    if workspace is None:
        workspace = torch.empty(plan_workspace_bytes(params.n_inst, params.H, R), dtype=torch.uint8, device=L.device)
    seg = PlanSegmentsC(1, params.n_inst, R, 0, _ptr(L), None, _ptr(req_id), _ptr(inst), _ptr(n_tok), _ptr(n_hat),
                        _ptr(pinned))
    _check(lib().plan_reschedule_segmented_ws(C.byref(params.c), C.byref(seg), _ptr(moves), _ptr(n_moves),
                                              _ptr(err_flag), _ptr(workspace), _stream(stream)),
           "plan_reschedule_segmented_ws")
    return moves, n_moves


def plan_reschedule_segmented_ws(params: PlanParams, seg: PlanSegmentsC, workspace: torch.Tensor, moves=None,
                                 n_moves=None, err_flag=None, stream=None):
    if moves is None:
        moves, n_moves = alloc_moves(params.max_moves, "cuda")
    _check(lib().plan_reschedule_segmented_ws(C.byref(params.c), C.byref(seg), _ptr(moves), _ptr(n_moves),
                                              _ptr(err_flag), _ptr(workspace), _stream(stream)),
           "plan_reschedule_segmented_ws")
    return moves, n_moves


def plan_reschedule_segmented(params: PlanParams, seg: PlanSegmentsC, moves=None, n_moves=None, err_flag=None,
                              stream=None):
    if moves is None:
        moves, n_moves = alloc_moves(params.max_moves, "cuda")
    _check(lib().plan_reschedule_segmented(C.byref(params.c), C.byref(seg), _ptr(moves), _ptr(n_moves),
                                           _ptr(err_flag), _stream(stream)), "plan_reschedule_segmented")
    return moves, n_moves


# ================================================================ P -> D dispatch (NEXT-2)
DISPATCH_ROUND_ROBIN, DISPATCH_CURRENT_LOAD, DISPATCH_PROJECTED = 0, 1, 2


def dispatch_requests(policy: int, L: torch.Tensor, beta_q: torch.Tensor, n_tok: torch.Tensor, n_hat: torch.Tensor,
                      c_mem: Optional[torch.Tensor] = None, reserved: Optional[torch.Tensor] = None,
                      counter: int = 0, assign: Optional[torch.Tensor] = None,
                      workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Places the arrivals in order (star.h dispatch_requests); L is updated in place."""
    _req(L, torch.int64, "L")
    for n_, t in (("beta_q", beta_q), ("n_tok", n_tok), ("n_hat", n_hat)):
        _req(t, torch.int32, n_)
    n_inst, H1 = L.shape
    A = int(n_tok.shape[0])
    if assign is None:
        assign = torch.empty(max(A, 1), dtype=torch.int32, device=L.device)
    if workspace is None and policy == DISPATCH_PROJECTED:
        workspace = torch.empty(int(lib().star_dispatch_workspace_bytes(n_inst, H1 - 1)), dtype=torch.uint8,
                                device=L.device)
    _check(lib().dispatch_requests(int(policy), n_inst, H1 - 1, _ptr(beta_q), _ptr(L), _ptr(c_mem), _ptr(reserved),
                                   A, _ptr(n_tok), _ptr(n_hat), int(counter), _ptr(assign), _ptr(workspace),
                                   _stream(stream)), "dispatch_requests")
    return assign[:A]


def plan_timeline():
    """Diagnostics: phase stamps (ns) of the most recent single-CTA plan (star_plan_timeline)."""
    buf = np.zeros(128, dtype=np.uint64)
    _check(lib().star_plan_timeline(buf.ctypes.data_as(P)), "star_plan_timeline")
    return buf


# ================================================================ KV migration (NEXT-4)
def kv_pool(pool: torch.Tensor) -> KvPoolC:
    """Describes a paged KV pool tensor [n_layers, n_blocks, block_bytes] (any dtype; the last
    dimension is taken in bytes).  Layers may be strided (a view into a larger allocation)."""
    if not pool.is_cuda or pool.dim() != 3 or pool.stride(2) != 1 or pool.stride(1) != pool.shape[2]:
        raise StarError("pool must be a CUDA tensor [n_layers, n_blocks, block] with contiguous blocks")
    es = pool.element_size()
    return KvPoolC(pool.data_ptr(), pool.shape[0], pool.stride(0) * es, pool.shape[1], pool.shape[2] * es)


def kv_pack(pool: torch.Tensor, table: torch.Tensor, staging: Optional[torch.Tensor] = None,
            err_flag: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """staging[l, j] = pool[l, table[j]] (star.h kv_pack)."""
    _req(table, torch.int32, "table")
    n = int(table.shape[0])
    if staging is None:
        staging = torch.empty((pool.shape[0], n, pool.shape[2]), dtype=pool.dtype, device=pool.device)
    d = kv_pool(pool)
    _check(lib().kv_pack(C.byref(d), _ptr(table), n, _ptr(staging), _ptr(err_flag), _stream(stream)), "kv_pack")
    return staging


def kv_unpack(staging: torch.Tensor, pool: torch.Tensor, table: torch.Tensor, err_flag: Optional[torch.Tensor] = None,
              stream=None) -> None:
    """pool[l, table[j]] = staging[l, j] (star.h kv_unpack)."""
    _req(table, torch.int32, "table")
    d = kv_pool(pool)
    _check(lib().kv_unpack(_ptr(staging), C.byref(d), _ptr(table), int(table.shape[0]), _ptr(err_flag),
                           _stream(stream)), "kv_unpack")


def kv_migrate(src_pool: torch.Tensor, src_table: torch.Tensor, dst_pool: torch.Tensor, dst_table: torch.Tensor,
               err_flag: Optional[torch.Tensor] = None, stream=None) -> None:
    """dst_pool[l, dst_table[j]] = src_pool[l, src_table[j]] (star.h kv_migrate)."""
    _req(src_table, torch.int32, "src_table")
    _req(dst_table, torch.int32, "dst_table")
    if src_table.shape[0] != dst_table.shape[0]:
        raise StarError("src_table and dst_table must have the same length")
    s, d = kv_pool(src_pool), kv_pool(dst_pool)
    _check(lib().kv_migrate(C.byref(s), _ptr(src_table), C.byref(d), _ptr(dst_table), int(src_table.shape[0]),
                            _ptr(err_flag), _stream(stream)), "kv_migrate")
