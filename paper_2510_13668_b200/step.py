"""One decode-step pass of the STAR hot path on one rank (one process per GPU).

    lenpred_forward_project (predictor fused with project_instance_load) -> all-gather(records)
    -> plan_reschedule_segmented
    (one rank: lenpred_forward_project_plan, the plan run by the fused tail's last CTA)

Sharding follows the paper's deployment unit (one decode instance per GPU, PAPER.md:488;
SURVEY.md §8(e)): the n decode instances are split into contiguous blocks of n_loc = n/W per
rank; each rank predicts and projects only its own requests ("workers ... perform local future
state simulation and proactively report").  The rank's whole state lives in one
fixed-size byte record that is also the exchange buffer (zero-copy packing):

    [count i32 | pad] [L n_loc*(H+1) i64] [W | peak | growth n_loc i64] [count n_loc i32]
    [req_id | inst | n_tok | n_hat  r_cap i32 each] [pinned r_cap u8]      (16-byte aligned sections)

The predictor writes N_hat straight into the record, the projection writes L/W/peak/growth
into it, one NCCL all-gather (torch.distributed, NVLink) concatenates the W records, and every
rank runs the identical integer plan directly on the gathered buffer (plan_reschedule_segmented
reads the W segments in place).  Plans agree across ranks by construction (same bytes in, same
bytes out).  PyTorch is used for device memory, streams, CUDA graphs and the process group only.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib


def _align(x: int, a: int = 16) -> int:
    return (x + a - 1) // a * a


@dataclasses.dataclass
class RecordLayout:
    n_loc: int
    H: int
    r_cap: int

    def __post_init__(self):
        o = 0
        self.off_count = o; o += 16
        self.off_L = o; o = _align(o + 8 * self.n_loc * (self.H + 1))
        self.off_W = o; o = _align(o + 8 * self.n_loc)
        self.off_peak = o; o = _align(o + 8 * self.n_loc)
        self.off_growth = o; o = _align(o + 8 * self.n_loc)
        self.off_icount = o; o = _align(o + 4 * self.n_loc)
        self.off_req_id = o; o = _align(o + 4 * self.r_cap)
        self.off_inst = o; o = _align(o + 4 * self.r_cap)
        self.off_n_tok = o; o = _align(o + 4 * self.r_cap)
        self.off_n_hat = o; o = _align(o + 4 * self.r_cap)
        self.off_pinned = o; o = _align(o + self.r_cap)
        self.nbytes = o

    def views(self, buf: torch.Tensor) -> dict:
        """Typed views into one record (a uint8 tensor of nbytes; works on CPU or CUDA)."""
        assert buf.dtype == torch.uint8 and buf.numel() == self.nbytes

        def v(off, n, dt, shape=None):
            t = buf[off:off + n * torch.empty((), dtype=dt).element_size()].view(dt)
            return t.view(shape) if shape is not None else t

        return dict(
            count=v(self.off_count, 1, torch.int32),
            L=v(self.off_L, self.n_loc * (self.H + 1), torch.int64, (self.n_loc, self.H + 1)),
            W=v(self.off_W, self.n_loc, torch.int64),
            peak=v(self.off_peak, self.n_loc, torch.int64),
            growth=v(self.off_growth, self.n_loc, torch.int64),
            icount=v(self.off_icount, self.n_loc, torch.int32),
            req_id=v(self.off_req_id, self.r_cap, torch.int32),
            inst=v(self.off_inst, self.r_cap, torch.int32),
            n_tok=v(self.off_n_tok, self.r_cap, torch.int32),
            n_hat=v(self.off_n_hat, self.r_cap, torch.int32),
            pinned=v(self.off_pinned, self.r_cap, torch.uint8),
        )

    def segments(self, base_ptr: int, world: int) -> "_lib.PlanSegmentsC":
        return _lib.PlanSegmentsC(world, self.n_loc, self.r_cap, self.nbytes, base_ptr + self.off_L,
                                  base_ptr + self.off_count, base_ptr + self.off_req_id, base_ptr + self.off_inst,
                                  base_ptr + self.off_n_tok, base_ptr + self.off_n_hat, base_ptr + self.off_pinned)


def exchange(send: torch.Tensor, recv: torch.Tensor, group=None):
    """All-gather of the fixed-size records: recv[k*nbytes:(k+1)*nbytes] = rank k's record.
    One NCCL collective over NVLink on GPU; the same call runs over gloo on CPU (tests)."""
    import torch.distributed as dist
    if send.is_cuda:
        dist.all_gather_into_tensor(recv, send, group=group)
    else:   # gloo: list form
        world = recv.numel() // send.numel()
        outs = list(recv.view(world, send.numel()).unbind(0))
        dist.all_gather(outs, send, group=group)


class Step:
    """Per-rank decode-step pass.  `rank`/`world` describe the instance sharding; `group` is
    the torch.distributed process group (None when world == 1)."""

    def __init__(self, predictor: _lib.Predictor, params: _lib.PlanParams, n_inst: int, r_cap: int,
                 rank: int = 0, world: int = 1, group=None, device: Optional[torch.device] = None,
                 max_ctx_len: int = _lib.L_CTX, refresh_k: Optional[int] = None,
                 gathered: Optional[torch.Tensor] = None, force_collective: bool = False):
        """gathered: (single-GPU measurement of one rank of a W-rank job) a caller-owned buffer of
        world * nbytes holding the OTHER ranks' records as the all-gather would deliver them; this
        rank's record is written in place at slot `rank` and no collective is issued."""
        if n_inst % world:
            raise ValueError(f"n_inst={n_inst} must be divisible by world={world}")
        # force_collective: take the W > 1 path (separate plan launch after an all-gather over
        # `group`) even at world 1 -- exercises the exchange on a one-GPU box
        self.force_collective = bool(force_collective) and group is not None
        self.pred, self.params = predictor, params
        self.n_inst, self.world, self.rank, self.group = n_inst, world, rank, group
        self.n_loc = n_inst // world
        self.H = params.H
        self.r_cap = r_cap
        self.max_ctx_len = max_ctx_len
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.layout = RecordLayout(self.n_loc, self.H, r_cap)
        self.emulated = gathered is not None
        if self.emulated:
            nb = self.layout.nbytes
            if gathered.dtype != torch.uint8 or gathered.numel() != world * nb:
                raise ValueError(f"gathered must be a uint8 buffer of world*nbytes = {world * nb}")
            self.recv = gathered
            self.send = gathered[rank * nb:(rank + 1) * nb]
        else:
            self.send = torch.zeros(self.layout.nbytes, dtype=torch.uint8, device=self.device)
            self.recv = (torch.zeros(world * self.layout.nbytes, dtype=torch.uint8, device=self.device)
                         if world > 1 or self.force_collective else self.send)
        self.v = self.layout.views(self.send)
        self.seg = self.layout.segments(self.recv.data_ptr(), world)
        self.ws = torch.zeros(_lib.project_workspace_bytes(self.n_loc, self.H), dtype=torch.uint8, device=self.device)
        self.moves, self.n_moves = _lib.alloc_moves(params.max_moves, self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.proj_out = _lib.ProjectOut(self.n_loc, self.H, self.device, L=self.v["L"])
        self.proj_out.W, self.proj_out.peak, self.proj_out.growth = self.v["W"], self.v["peak"], self.v["growth"]
        self.proj_out.count = self.v["icount"]
        self.R = 0
        self.graph = None
        self._graph_R = -1
        # prediction cadence (NEXT-1): re-predict a request every refresh_k generated tokens, age
        # its prediction in between; None = predict every request every step
        self.refresh_k = refresh_k
        if refresh_k is not None:
            self.gen = torch.zeros(r_cap, dtype=torch.int32, device=self.device)
            self.g_last = torch.full((r_cap,), -1, dtype=torch.int32, device=self.device)
            self.nhat_last = torch.zeros(r_cap, dtype=torch.int32, device=self.device)
            self.n_refreshed = torch.zeros(1, dtype=torch.int32, device=self.device)

    # ---------------------------------------------------------------- state
    def load_requests(self, req_id, inst, n_tok, pinned=None, non_blocking=False):
        """Installs this rank's running requests (global instance ids in this rank's block)."""
        R = int(req_id.shape[0])
        if R > self.r_cap:
            raise ValueError(f"{R} requests exceed r_cap={self.r_cap}")
        v = self.v
        for name, src in (("req_id", req_id), ("inst", inst), ("n_tok", n_tok)):
            v[name][:R].copy_(torch.as_tensor(src), non_blocking=non_blocking)
        if pinned is not None:
            v["pinned"][:R].copy_(torch.as_tensor(pinned), non_blocking=non_blocking)
        else:
            v["pinned"][:R].zero_()
        v["count"].fill_(R)
        self.R = R
        if self.refresh_k is not None:
            # new occupants: no prediction yet (a slot must not inherit the previous request's
            # cadence state, reading A27); set_generation() may install an explicit state after
            self.g_last[:R].fill_(-1)
            self.nhat_last[:R].zero_()

    def set_generation(self, gen, g_last=None, nhat_last=None, non_blocking=False):
        """Refresh mode: tokens generated so far per slot (and optionally the cadence state)."""
        R = int(torch.as_tensor(gen).shape[0])
        self.gen[:R].copy_(torch.as_tensor(gen), non_blocking=non_blocking)
        if g_last is not None:
            self.g_last[:R].copy_(torch.as_tensor(g_last), non_blocking=non_blocking)
        if nhat_last is not None:
            self.nhat_last[:R].copy_(torch.as_tensor(nhat_last), non_blocking=non_blocking)

    # ---------------------------------------------------------------- the pass
    def run(self, h: torch.Tensor, stream=None):
        """h: [R, d] hidden states of this rank's running requests (row r <-> request slot r)."""
        v, R = self.v, self.R
        if self.refresh_k is not None:
            # cadence k: re-predict only the due rows, age the rest, then project all of them
            _lib.lenpred_forward_refresh_project(self.pred, h[:R], v["n_tok"][:R], self.gen[:R], self.g_last[:R],
                                                 self.nhat_last[:R], self.refresh_k, v["inst"][:R], self.n_loc,
                                                 self.H, self.params.beta_q, self.ws,
                                                 inst_base=self.rank * self.n_loc, max_ctx_len=self.max_ctx_len,
                                                 n_hat=v["n_hat"][:max(R, 1)], n_refreshed=self.n_refreshed,
                                                 out=self.proj_out, err_flag=self.err, R=R, stream=stream)
            self._exchange(stream)
            _lib.plan_reschedule_segmented(self.params, self.seg, self.moves, self.n_moves, self.err, stream=stream)
            return self.moves, self.n_moves
        if self.world == 1 and not self.force_collective:
            # one rank: forward + projection + Alg. 1 (the plan runs in the fused tail's last CTA)
            _lib.lenpred_forward_project_plan(self.pred, h[:R], v["n_tok"][:R], v["inst"][:R], self.n_loc, self.H,
                                              self.params.beta_q, self.ws, self.params, self.seg, self.moves,
                                              self.n_moves, v["n_hat"][:max(R, 1)], self.proj_out,
                                              max_ctx_len=self.max_ctx_len, err_flag=self.err, stream=stream)
            return self.moves, self.n_moves
        # predictor fused with the projection of its own N_hat (2 launches for bf16 predictors)
        _lib.lenpred_forward_project(self.pred, h[:R], v["n_tok"][:R], v["inst"][:R], self.n_loc, self.H,
                                     self.params.beta_q, self.ws, inst_base=self.rank * self.n_loc,
                                     max_ctx_len=self.max_ctx_len, n_hat=v["n_hat"][:max(R, 1)],
                                     out=self.proj_out, err_flag=self.err, want_y=False, stream=stream)
        self._exchange(stream)
        _lib.plan_reschedule_segmented(self.params, self.seg, self.moves, self.n_moves, self.err, stream=stream)
        return self.moves, self.n_moves

    def _exchange(self, stream=None):
        """The all-gather, ordered on the SAME stream as the kernels around it: the NCCL collective
        is enqueued on `stream` (torch.distributed uses the current stream), so it reads the record
        only after the predictor/projection wrote it and the plan reads `recv` only after it landed."""
        if (self.world == 1 and not self.force_collective) or self.emulated:
            return
        if stream is None:
            exchange(self.send, self.recv, self.group)
        else:
            with torch.cuda.stream(stream):
                exchange(self.send, self.recv, self.group)

    def capture(self, h: torch.Tensor):
        """Captures run(h) into a CUDA graph (one launch per step)."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.run(h)   # warm-up (sets function attributes, TMA maps)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(h)
        self.graph = g
        self._graph_R = self.R   # the request count (and h's address) are baked into the graph
        return g

    def replay(self):
        """One launch of the captured step.  The request arrays and h may change in place; the
        request COUNT may not (it is baked into the kernels' grids): recapture after a
        load_requests() that changed it."""
        if self.graph is None:
            raise RuntimeError("Step.replay() before Step.capture()")
        if self.R != self._graph_R:
            raise RuntimeError(f"request count changed since capture ({self._graph_R} -> {self.R}): capture again")
        self.graph.replay()
        return self.moves, self.n_moves

    def result(self):
        return _lib.decode_moves(self.moves, self.n_moves)

    def gathered_views(self):
        """Typed views of every rank's record in the gathered buffer (for reporting/tests)."""
        nb = self.layout.nbytes
        return [self.layout.views(self.recv[k * nb:(k + 1) * nb]) for k in range(self.world)]


def split_snapshot_by_rank(inst: np.ndarray, n_inst: int, world: int, rank: int) -> np.ndarray:
    """Indices of the requests owned by `rank` (instances [rank*n_loc, (rank+1)*n_loc))."""
    n_loc = n_inst // world
    return np.nonzero((inst >= rank * n_loc) & (inst < (rank + 1) * n_loc))[0]
