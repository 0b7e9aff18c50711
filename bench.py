#!/usr/bin/env python
"""bench.py -- requests predicted+planned per second for the STAR hot path on B200.

One "step" = one pass of the whole hot path over one batch of synthetic
input: Eq. 2 predictor on every running request's hidden state -> integer projection of the
per-instance loads -> (NCCL all-gather of the per-rank records when N > 1) -> Alg. 1 plan.

    python bench.py [--gpus N --steps K --warmup W] [--config C2] [--impl star|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Defaults: N=1, workload TGT, the north-star point (8 instances x 512 requests, hidden 4096, bf16,
long-tailed CoT lengths, instance 0 overloaded so Alg. 1 moves a request every step).  Sharding:
the 8 instances are split in contiguous blocks over the N ranks (one decode instance per GPU at
N = 8; total work fixed).  The step is one CUDA graph
[L2 flush (256 MB write) -> event -> step -> event]: the events are graph nodes on the step's
stream, so the timed span excludes the flush and host launch latency; the reported time is the
max over ranks of the summed per-step times.  Prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "requests predicted+planned/sec and µs per decode step at 1/2/4/8 B200"
UNIT = "requests/s"
CONFIG_ORDER = ["C1", "C2", "C3", "C4", "TGT"]


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults per arm (None = not given): the GPU arm 500 / 20; the reference arm (the CPU oracle,
    # ~1.3 s per whole TGT step on 16 cores) 10 / 2, so that a bare run of either ends within minutes
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", choices=["star", "reference"], default="star")
    ap.add_argument("--config", default="TGT", choices=CONFIG_ORDER)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the projection bandwidth sweep")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU budget of the cpu_baseline sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no clocks/e2e/cpu legs")
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 10 if args.impl == "reference" else 500
    if args.warmup is None:
        args.warmup = 2 if args.impl == "reference" else 20
    return args


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm_gbs=d["hbm_gbs"], bf16_tflops=d["bf16_tflops"],
                    bf16_tflops_sustained=d.get("bf16_tflops_sustained"), source="MEASURED_PEAKS.json")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0,
                source="fallback (B200_PROFILING.md)")


# ------------------------------------------------------------------------------ workload
def make_workload(cfg_name, world, rank, seed, r_per=None):
    import datagen
    from paper_2510_13668_b200.step import split_snapshot_by_rank
    c = dict(datagen.CONFIGS[cfg_name])
    if r_per is not None:
        c["r_per_inst"] = r_per
    n_inst, r_per = c["n_inst"], c["r_per_inst"]
    if n_inst % world:
        raise SystemExit(f"config {cfg_name} has {n_inst} instances; --gpus {world} must divide it")
    snap = datagen.make_snapshot(seed, n_inst, r_per, skewed=c.get("skewed", False))
    params = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10), max_moves=c["max_moves"])
    idx = split_snapshot_by_rank(snap.inst, n_inst, world, rank)
    pw = datagen.make_predictor_weights(seed, c["d"], c["dtype"])
    h = datagen.make_hidden(seed * 1000 + rank, len(idx), c["d"], c["dtype"])
    return c, snap, params, idx, pw, h


def config_block(cfg_name, c, world):
    """The workload (identical in both arms; timing details are separate keys of the line)."""
    return {"workload": f"{cfg_name}: {c['desc']}", "n_inst": c["n_inst"], "requests_per_instance": c["r_per_inst"],
            "total_requests": c["n_inst"] * c["r_per_inst"], "hidden": c["d"], "m1_m2_m3": [2048, 512, 64],
            "dtype": c["dtype"], "H": 50, "max_moves": c["max_moves"], "skewed": bool(c.get("skewed", False)),
            "instances_per_gpu": c["n_inst"] // world,
            "parallelism": f"instance-sharded x{world} (one NCCL all-gather of per-rank records)",
            "l2": "GPU arm: flushed before every timed step (256 MB write, outside the timed span)",
            "n_hat_source": "the arm's own predictor (hidden rows scaled so predictions are long-tailed)"}


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index):
        self.samples, self.reasons, self.stop_ev = [], 0, threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            pass

    def _run(self):
        while not self.stop_ev.is_set():
            self.sample()
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_ev.set()
        self.t.join()
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------------ oracle timing
def oracle_full_step(snap, params, pw, h_all, nthreads):
    """One whole step of the oracle (as it stands) on the whole workload: Eq. 2 over EVERY
    running request's hidden row (fp64 loops, OpenMP over rows), the quantizer, the projection
    and Alg. 1 over the whole snapshot.  Returns (t_pred, t_proj, t_plan, n_moves) in seconds."""
    import oracle
    t0 = time.perf_counter()
    y = oracle.lenpred_weights(h_all, pw, nthreads=nthreads)
    n_hat = oracle.quantize(y.astype(np.float32), snap.n_tok)
    t1 = time.perf_counter()
    P = oracle.project(snap.inst, snap.n_tok, n_hat, snap.n_inst, params.H, params.beta_q)
    t2 = time.perf_counter()
    moves = oracle.plan(params, P["L"], snap.req_id, snap.inst, snap.n_tok, n_hat, snap.pinned)
    t3 = time.perf_counter()
    return t1 - t0, t2 - t1, t3 - t2, len(moves)


def oracle_workload(cfg_name, seed):
    """The GPU arm's workload at N = 1 (all ranks' hidden rows in instance-rank order)."""
    import datagen   # (no product import on this path)
    c = datagen.CONFIGS[cfg_name]
    snap = datagen.make_snapshot(seed, c["n_inst"], c["r_per_inst"], skewed=c.get("skewed", False))
    params = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10), max_moves=c["max_moves"])
    idx = np.arange(snap.R)   # N = 1: one rank owns every instance
    pw = datagen.make_predictor_weights(seed, c["d"], c["dtype"])
    h = datagen.make_hidden(seed * 1000, len(idx), c["d"], c["dtype"])
    # long-tailed self-predictions, as in the GPU arm: rows scaled by true_rem / median(y_hat),
    # the median taken from this arm's own predictor (untimed setup)
    import oracle
    y0 = oracle.lenpred_weights(h, pw)
    scale = np.maximum(snap.true_rem[idx], 1).astype(np.float32) / max(float(np.median(y0)), 1e-3)
    h = datagen.round_to_dtype(h * scale[:, None], c["dtype"])
    return c, snap, params, pw, h


def cpu_baseline(cfg_name, seed, budget_s):
    """The oracle timed on the host cores: whole steps of the bench workload (no extrapolation),
    as many as fit in the budget (at least one)."""
    import oracle
    oracle.build()
    c, snap, params, pw, h = oracle_workload(cfg_name, seed)
    cores = os.cpu_count() or 1
    ts = []
    t_beg = time.perf_counter()
    while not ts or (time.perf_counter() - t_beg + ts[-1] <= budget_s and len(ts) < 20):
        tp, tj, tl, nm = oracle_full_step(snap, params, pw, h, cores)
        ts.append(tp + tj + tl)
    t_step = float(np.mean(ts))
    return {"value": snap.R / t_step, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"{len(ts)} whole step(s) of the bench workload ({snap.R} requests): oracle Eq. 2 on every "
                       f"hidden row (fp64 loops, OpenMP {cores} threads, {tp:.2f} s), quantizer, projection "
                       f"({tj * 1e3:.1f} ms) and Alg. 1 ({tl * 1e3:.1f} ms, {nm} move(s)) single-threaded"),
            "s_per_step": t_step}


# ------------------------------------------------------------------------------ reference arm
def run_reference(args):
    """Reference arm: the plain CPU oracle (the paper ships no code) timed as it stands on the
    host cores; every step is a WHOLE step of the same workload (no sampling, no extrapolation)."""
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    c, snap, params, pw, h = oracle_workload(args.config, args.seed)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_full_step(snap, params, pw, h, cores)
    ts, parts = [], np.zeros(3)
    nm = 0
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        tp, tj, tl, nm = oracle_full_step(snap, params, pw, h, cores)
        ts.append(tp + tj + tl)
        parts += (tp, tj, tl)
    wall = time.perf_counter() - t_wall0
    t_step = wall / max(args.steps, 1)
    value = snap.R / t_step
    sample = (f"every step is the whole workload ({snap.R} requests): oracle Eq. 2 on every hidden row (fp64 "
              f"loops, OpenMP {cores} threads), quantizer, projection and Alg. 1 single-threaded "
              f"({nm} move(s) per step)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args.config, c, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "stage_ms": {"predict": round(parts[0] / args.steps * 1e3, 2),
                         "project": round(parts[1] / args.steps * 1e3, 3),
                         "plan": round(parts[2] / args.steps * 1e3, 3)},
            "wall_s_timed": wall,
            "note": "The paper ships no code; the reference arm is the plain CPU oracle written from the paper, "
                    "timed over whole steps (wall clock of the K timed steps / K)."}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------------------ product arm
def count_kernel_nodes(graph) -> int:
    """Kernel nodes in a captured CUDA graph (our launches per step; events/memcpys excluded)."""
    from cuda.bindings import runtime as rt
    g = graph.raw_cuda_graph()
    err, _, n = rt.cudaGraphGetNodes(g, 0)
    err, nodes, n = rt.cudaGraphGetNodes(g, n)
    k = 0
    for nd in nodes[:n]:
        err, t = rt.cudaGraphNodeGetType(nd)
        if t == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel:
            k += 1
    return k


def _ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            return json.load(f).get(key)
    return None


def _projection_point(star, snap, params, dev, R, reps=10, grouped=True):
    """Per-launch time of the standalone projection over R requests of R / 65536 instances (the
    documented per-instance bound; the C2 snapshot tiled), 10 launches back to back per event span
    (no host latency in the span); inputs beyond L2 stream from HBM.  grouped: requests sorted by
    instance (a worker's running batch); otherwise shuffled (every instance interleaved)."""
    import torch
    reps_tile = (R + snap.R - 1) // snap.R
    per = max(R // 65536 // snap.n_inst, 1)   # tiles per instance group: tile k -> instances 8*(k % per) + inst
    n = snap.n_inst * per
    shift = (np.arange(reps_tile, dtype=np.int64) % per * snap.n_inst).repeat(snap.R)[:R]
    inst_h = (np.tile(snap.inst, reps_tile)[:R] + shift).astype(np.int32)
    order = np.argsort(inst_h, kind="stable") if grouped else np.random.default_rng(1).permutation(R)
    inst = torch.from_numpy(inst_h[order]).to(dev)
    ntok = torch.from_numpy(np.tile(snap.n_tok, reps_tile)[:R][order]).to(dev)
    nhat = torch.from_numpy(np.tile(snap.true_rem.astype(np.int32), reps_tile)[:R][order]).to(dev)
    H = params.H
    out = star.ProjectOut(n, H, dev)
    ws = torch.zeros(star.project_workspace_bytes(n, H), dtype=torch.uint8, device=dev)
    fn = lambda: star.project_instance_load(inst, ntok, nhat, n, H, params.beta_q, out=out, workspace=ws)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    K = 10
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3 / K)
    del inst, ntok, nhat, ws
    return float(np.median(ts)), n, 12.0 * R + n * (H + 5) * 8.0


def projection_sweep(star, snap, params, dev, peaks, R=1 << 24):
    """Bandwidth-scale evidence for the projection kernel: the standalone
    project_instance_load over R = 2^20 ... 2^26 requests (12.6 MB ... 805 MB), instance-grouped
    and shuffled; algorithmic bytes = 12 B x R (+ outputs).  Headline point: 2^24 grouped."""
    sweep = []
    head = None
    for lg in (20, 22, 24, 25, 26):
        for grouped in (True, False):
            Rk = 1 << lg
            t, n, algo = _projection_point(star, snap, params, dev, Rk, grouped=grouped)
            gbs = algo / t / 1e9
            pt = {"requests": Rk, "instances": n, "order": "grouped" if grouped else "shuffled",
                  "bins": n * (params.H + 2), "us": round(t * 1e6, 2), "GBps": round(gbs, 1),
                  "frac": round(gbs / peaks["hbm_gbs"], 4)}
            sweep.append(pt)
            if Rk == R and grouped:
                head = (t, n, algo, gbs)
    t_med, n, algo, gbs = head
    return {"kernel": "project_ldg_kernel (standalone, windowed histogram, 2 CTAs/SM)", "bound": "hbm", "requests": R,
            "algorithmic_bytes": algo, "avg_launch_us": t_med * 1e6, "achieved": gbs, "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"], "traffic": _ncu_traffic("sweep/project"),
            "instances": n, "sweep": sweep,
            "note": "headline: 2^24 requests (201 MB, beyond L2), the C2 snapshot tiled over 256 instances x 65536 "
                    "requests, instance-grouped as a worker's batch is; 'shuffled' = every instance interleaved "
                    "(beyond the 3072-bin shared-memory window the kernel falls back to global 64-bit atomics); "
                    "the in-step projection is fused into the predictor tail"}


def longtail_hidden(star, pred, h_np, snap, idx, tdt, dev):
    """Long-tailed self-predictions: scale h rows so the GPU's y_hat tracks the snapshot's true
    remaining lengths (positive homogeneity of the bias-free Eq. 2)."""
    import torch
    h0 = torch.from_numpy(h_np).to(tdt).to(dev)
    y0, _ = star.lenpred_forward(pred, h0)
    med = float(torch.median(y0.float()).item())
    target = np.maximum(snap.true_rem[idx], 1).astype(np.float32)
    scale = target / max(med, 1e-3)
    return torch.from_numpy((h_np * scale[:, None]).astype(np.float32)).to(tdt).to(dev)


def tgt_rank_timing(star, Step, dev, flush, seed=0, reps=200, world=8, cfg="TGT", r_per=None, stages=True):
    """North-star target point, one rank of the W = 8 job (8 instances x 512 requests, d = 4096,
    bf16; one instance per GPU): this rank's predictor + fused projection over its 512 requests,
    then Alg. 1 over the 8 gathered records (4096 requests).  Measured on ONE GPU: the other 7
    ranks' records are computed first with the same library calls and sit in the gathered buffer
    as the all-gather would deliver them; the NCCL all-gather itself is not in the timed span.
    (cfg="C5", r_per=R: the same per-rank measurement at R requests per instance.)"""
    import torch
    from paper_2510_13668_b200.step import RecordLayout
    steps, hs = [], []
    buf = pred = params = None
    for k in range(world):
        c, snap, params_h, idx, pw, h_np = make_workload(cfg, world, k, seed, r_per=r_per)
        tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
        if pred is None:
            W = [torch.from_numpy(x).to(tdt).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
            pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=c["r_per_inst"])
            params = star.PlanParams.from_host(params_h, device=dev)
            nb = RecordLayout(c["n_inst"] // world, params_h.H, c["r_per_inst"]).nbytes
            buf = torch.zeros(world * nb, dtype=torch.uint8, device=dev)
        st = Step(pred, params, c["n_inst"], r_cap=c["r_per_inst"], rank=k, world=world, device=dev, gathered=buf)
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                      snap.n_tok)),
                         pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
        h = longtail_hidden(star, pred, h_np, snap, idx, tdt, dev)
        st.run(h)
        steps.append(st)
        hs.append(h)
    torch.cuda.synchronize()
    st, h = steps[0], hs[0]
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g):
        st.run(h)
    try:
        launches = count_kernel_nodes(g)
    except Exception:
        launches = None
    g.instantiate()
    stream = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 10):
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        e1.synchronize()
        if i >= 10:
            ts.append(e0.elapsed_time(e1) * 1e3)
    n_moves = int(st.n_moves.item())
    if not stages:
        pred.close()
        return {"requests_per_instance": c["r_per_inst"], "us_per_step_p50": round(float(np.median(ts)), 2),
                "us_per_step_mean": round(float(np.mean(ts)), 2), "us_per_step_min": round(float(np.min(ts)), 2), "launches_per_step": launches, "moves": n_moves,
                "rank_requests_per_s": round(c["r_per_inst"] / (float(np.median(ts)) * 1e-6), 1)}
    # stage split (event nodes between the stages: each costs ~2 us and blocks the PDL overlap, so
    # the stages sum to more than the step)
    es = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
    v = st.v
    gs = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gs):
        if flush is not None:
            flush.fill_(1.0)
        es[0].record()
        star.lenpred_forward_project(pred, h, v["n_tok"][:st.R], v["inst"][:st.R], st.n_loc, st.H, params.beta_q,
                                     st.ws, inst_base=0, n_hat=v["n_hat"][:st.R], out=st.proj_out, err_flag=st.err,
                                     want_y=False)
        es[1].record()
        star.plan_reschedule_segmented(params, st.seg, st.moves, st.n_moves, st.err)
        es[2].record()
    acc = np.zeros(2)
    for _ in range(50):
        gs.replay()
        es[2].synchronize()
        acc += [es[k].elapsed_time(es[k + 1]) * 1e3 / 50 for k in range(2)]
    pred.close()
    return {"workload": "TGT, one rank of W=8: 1 instance x 512 requests, d=4096 bf16; Alg. 1 over the 8 gathered "
                        "records (4096 requests)",
            "us_per_step_p50": round(float(np.median(ts)), 2), "us_per_step_p99": round(float(np.percentile(ts, 99)), 2),
            "us_per_step_mean": round(float(np.mean(ts)), 2),
            "us_per_step_min": round(float(np.min(ts)), 2), "us_per_step_p10": round(float(np.percentile(ts, 10)), 2),
            "target_us": 50.0, "launches_per_step": launches, "moves": n_moves,
            "exchange_budget_us": round(50.0 - float(np.median(ts)), 2),
            "exchange_estimate_us": "5-15 (SURVEY.md 8(d): NCCL all-gather of 8 x %d B over NVLink; unmeasured here, "
                                    "one GPU)" % (buf.numel() // world),
            "stage_us": {"predict+project": round(acc[0], 2), "plan_4096_gathered": round(acc[1], 2)},
            "l2": "flushed before every step" if flush is not None else "warm",
            "note": "one GPU: the other 7 ranks' records are pre-computed into the gathered buffer; the NCCL "
                    "all-gather (8 x %d B) is NOT in the timed span: the span plus the all-gather must fit "
                    "50 us, i.e. the all-gather has exchange_budget_us" % (buf.numel() // world)}


def run_star(args):
    import torch
    rank, local_rank, world = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    import paper_2510_13668_b200 as star
    from paper_2510_13668_b200.step import Step

    c, snap, params_h, idx, pw, h_np = make_workload(args.config, world, rank, args.seed)
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    R = len(idx)
    W = [torch.from_numpy(x).to(tdt).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
    w4 = torch.from_numpy(pw.w4).to(dev)
    pred = star.Predictor(*W, w4, max_rows=max(R, 1))
    params = star.PlanParams.from_host(params_h, device=dev)

    h_dev = longtail_hidden(star, pred, h_np, snap, idx, tdt, dev)
    h_pin = h_dev.cpu().pin_memory()

    step = Step(pred, params, c["n_inst"], r_cap=max(R, 1), rank=rank, world=world, group=group, device=dev)
    req_np = [snap.req_id[idx], snap.inst[idx], snap.n_tok[idx], snap.pinned[idx]]
    step.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in req_np[:3]),
                       pinned=torch.from_numpy(np.ascontiguousarray(req_np[3])))
    req_pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in req_np]

    ev = lambda ext=False: torch.cuda.Event(enable_timing=True, external=ext)
    pred.layer1_timing(True)
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    # warm-up outside capture (function attributes, TMA descriptors, NCCL communicator)
    s_ = torch.cuda.Stream(device=dev)
    s_.wait_stream(stream)
    with torch.cuda.stream(s_):
        step.run(h_dev)
    stream.wait_stream(s_)
    torch.cuda.synchronize()

    # Timed step: the step is one CUDA graph WITHOUT event nodes (an event node inside the graph
    # breaks the programmatic-dependent-launch chain and costs several us); each step is
    # [L2 flush kernel] -> stream event -> graph launch -> stream event.  The ~40 us flush keeps
    # the GPU busy while the host enqueues the event and the graph, so the timed span contains
    # the step's device time (plus the graph's own launch latency), not host latency.
    use_graph = not args.no_graph
    launches = None
    g = g_l1 = None
    graph_error = None
    if use_graph:
        try:
            pred.layer1_timing(False)
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g):
                step.run(h_dev)
            try:
                launches = count_kernel_nodes(g)
            except Exception:
                launches = None
            g.instantiate()
            # a second graph of the same step with the library's layer-1 event pair (roofline pass)
            pred.layer1_timing(True)
            g_l1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_l1):
                step.run(h_dev)
        except Exception as ex:   # e.g. a collective that cannot be captured: time the eager step instead
            graph_error = f"{type(ex).__name__}: {ex}"
            torch.cuda.synchronize()
            g = g_l1 = None
            use_graph = False
            launches = None

    def timed(graph, store, l1):
        if flush is not None:
            flush.fill_(1.0)
        e_beg, e_end = ev(), ev()
        e_beg.record(stream)
        if graph is not None:
            graph.replay()
        else:
            step.run(h_dev)
        e_end.record(stream)
        e_end.synchronize()
        if store is not None:
            store.append(e_beg.elapsed_time(e_end))
            if l1 is not None:
                l1.append(pred.layer1_ms())

    for _ in range(max(args.warmup, 3)):
        timed(g, None, None)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank) if not args.profile else None
    if clk:
        clk.start()
    t0 = time.perf_counter()
    step_ms = []
    for i in range(args.steps):
        timed(g, step_ms, None)
        if clk and i % 25 == 0:   # also sample from this thread (between steps, outside the event span)
            clk.sample()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    wall = time.perf_counter() - t0
    clocks = clk.stop() if clk else None

    # warm-L2 mode: the same graph without the flush, back to back; the GPU is kept
    # busy by the previous replay, so the span is device time (median per step over 5 spans of 20)
    warm_us = None
    if g is not None and not args.profile:
        spans = []
        for _ in range(5):
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(20):
                g.replay()
            e1.record(stream)
            e1.synchronize()
            spans.append(e0.elapsed_time(e1) * 1e3 / 20)
        warm_us = round(float(np.median(spans)), 2)

    # roofline pass: the same timed loop on the graph carrying the layer-1 events
    l1_ms, step_l1_ms = [], []
    if g_l1 is not None:
        for _ in range(3):
            timed(g_l1, None, None)
        for _ in range(args.steps):
            timed(g_l1, step_l1_ms, l1_ms)
    else:
        pred.layer1_timing(True)
        for _ in range(args.steps):
            timed(None, step_l1_ms, l1_ms)

    tot = torch.tensor([sum(step_ms), sum(l1_ms), sum(step_l1_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    ms_per_step = float(tot[0].item()) / args.steps
    l1_avg_ms = float(tot[1].item()) / max(len(l1_ms), 1)
    step_l1_avg_ms = float(tot[2].item()) / max(len(step_l1_ms), 1)
    R_total = c["n_inst"] * c["r_per_inst"]
    value = R_total / (ms_per_step / 1e3)

    # ---- per-stage breakdown: the same step with event nodes between the stages ----
    stage = {}
    if not args.profile and use_graph:
        pred.layer1_timing(True)
        es = [ev(True) for _ in range(4)]
        gs = torch.cuda.CUDAGraph()
        v = step.v
        from paper_2510_13668_b200.step import exchange
        with torch.cuda.graph(gs):
            if flush is not None:
                flush.fill_(1.0)
            es[0].record()
            star.lenpred_forward_project(pred, h_dev[:R], v["n_tok"][:R], v["inst"][:R], step.n_loc, step.H,
                                         params.beta_q, step.ws, inst_base=rank * step.n_loc,
                                         n_hat=v["n_hat"][:max(R, 1)], out=step.proj_out, err_flag=step.err,
                                         want_y=False)
            es[1].record()
            if world > 1:
                exchange(step.send, step.recv, group)
            es[2].record()
            star.plan_reschedule_segmented(params, step.seg, step.moves, step.n_moves, step.err)
            es[3].record()
        acc = np.zeros(3)
        nrep = 50
        for _ in range(nrep):
            gs.replay()
            es[3].synchronize()
            acc += [es[k].elapsed_time(es[k + 1]) * 1e3 / nrep for k in range(3)]
        stage = {"predict+project": round(acc[0], 2), "allgather": round(acc[1], 2), "plan": round(acc[2], 2),
                 ("predictor_launch" if pred.path(R) else "layer1_gemm"): round(l1_avg_ms * 1e3, 2),
                 "note": "event nodes between stages (each costs a few us and blocks PDL overlap); "
                         "the sum exceeds us_per_step"}

    # ---- e2e: pinned host inputs -> device, step, moves -> host, every step ----
    e2e = None
    if not args.no_e2e and not args.profile:
        moves_h = torch.empty_like(step.moves, device="cpu").pin_memory()
        nm_h = torch.empty(1, dtype=torch.int32).pin_memory()
        v = step.v
        pred.layer1_timing(False)
        if use_graph:
            step.capture(h_dev)   # public API: Step.capture / Step.replay (one graph launch per step)
        else:
            step.replay = lambda: step.run(h_dev)   # eager fallback (graph capture failed above)
        # Pipelined serving loop: step i+1's hidden states travel host -> device (PCIe, the e2e
        # bottleneck: 16.8 MB per C2 step) on copy streams into one of two staging buffers while
        # step i computes; the compute stream then moves the staged rows into the step's input
        # (device-to-device) and copies the small request arrays and the moves itself.  The
        # whole K-step loop is timed between two events (per-step = total / K); the L2 flush
        # stays in every step (it overlaps the next step's host copy).
        NCS = 2   # h split in row blocks over 2 copy streams (measured: 1 -> 386 us, 2 -> 341 us, 4 -> 348 us per C2 step)
        cstreams = [torch.cuda.Stream(device=dev) for _ in range(NCS)]
        hstage = [torch.empty_like(h_dev), torch.empty_like(h_dev)]
        copied = [[torch.cuda.Event() for _ in range(NCS)] for _ in range(2)]
        rows = [(R * k // NCS, R * (k + 1) // NCS) for k in range(NCS)]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]
        moves_h = [torch.empty_like(step.moves, device="cpu").pin_memory() for _ in range(2)]
        nm_h = [torch.empty(1, dtype=torch.int32).pin_memory() for _ in range(2)]

        def e2e_loop(n):
            s, e = ev(), ev()
            s.record(stream)
            for cs in cstreams:
                cs.wait_event(s)
            for i in range(n):
                b = i & 1
                for k, cs in enumerate(cstreams):
                    if i >= 2:
                        cs.wait_event(consumed[b])   # step i-2 has moved its rows out of hstage[b]
                    with torch.cuda.stream(cs):
                        hstage[b][rows[k][0]:rows[k][1]].copy_(h_pin[rows[k][0]:rows[k][1]], non_blocking=True)
                        copied[b][k].record(cs)
                if flush is not None:
                    flush.fill_(1.0)
                for k in range(NCS):
                    stream.wait_event(copied[b][k])
                h_dev.copy_(hstage[b])
                consumed[b].record(stream)
                v["req_id"][:R].copy_(req_pin[0], non_blocking=True)
                v["inst"][:R].copy_(req_pin[1], non_blocking=True)
                v["n_tok"][:R].copy_(req_pin[2], non_blocking=True)
                v["pinned"][:R].copy_(req_pin[3], non_blocking=True)
                step.replay()
                moves_h[b].copy_(step.moves, non_blocking=True)
                nm_h[b].copy_(step.n_moves, non_blocking=True)
            e.record(stream)
            e.synchronize()
            return s.elapsed_time(e)

        e2e_loop(max(args.warmup, 3))
        e2e_ms = [e2e_loop(args.steps)]
        te = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e_ms_step = float(te.item()) / args.steps
        h2d = h_pin.numel() * h_pin.element_size() + sum(t.numel() * t.element_size() for t in req_pin)
        d2h = moves_h[0].numel() + 4
        e2e = {"value": R_total / (e2e_ms_step / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms_step,
               "path": "Step public API (Step.capture/replay of the step through the C ABI): every step "
                       "pinned-host h + request arrays -> device and moves -> pinned host; the next step's "
                       "h copy (copy stream, double-buffered) overlaps the current step's compute"}

    # ---- roofline: the layer-1 tcgen05 GEMM (dominant kernel), timed live inside the step ----
    peaks = load_peaks()
    path = pred.path(R) if R >= 1 else 0
    small_path = path in (1, 2)   # one-launch predictor (bf16 <= 512 rows / fp32 <= 128 rows)
    # the timed launch: layer 1 alone (2 R d m1), or the whole one-launch predictor (2 R (d m1 + m1 m2 + m2 m3 + m3))
    flops_l1 = 2.0 * R * (c["d"] * 2048 + (2048 * 512 + 512 * 64 + 64 if small_path else 0))
    achieved = flops_l1 / (l1_avg_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{args.config}/w{world}/" + ("small" if small_path else "layer1"))
    m_tiles = (R + 127) // 128
    pair = c["dtype"] == "bf16" and (m_tiles == 2 or (m_tiles + 1) // 2 * 2 * 8 >= 148 * 5 // 8)
    # the contraction's own dtype: bf16 at its measured peak; fp32 runs as 3xTF32 (three tcgen05 kind::tf32
    # MMAs per product) against the TF32 peak = measured bf16 x 0.5 (the nominal dense TF32 : BF16 ratio)
    f32 = c["dtype"] == "f32"
    peak = peaks["bf16_tflops"] * (0.5 if f32 else 1.0)
    small = small_path
    # which layer-1 kernel the library picks (mirrors forward_impl in star_api.cu): 9 non-uniform
    # column tiles when they need no more waves than 8, and the persistent two-tile form when
    # those tiles would take two waves but two tiles per pair fit one
    npairs, slots = (m_tiles + 1) // 2, (148 // 2) * 2
    w8, w9 = -(-npairs * 16 // slots), -(-npairs * 18 // slots)
    nu = pair and w9 * 240 < w8 * 256
    nu2 = nu and npairs * 9 * 2 > slots and (npairs * 9 + 1) // 2 * 2 <= slots and \
        os.environ.get("STAR_L1_PERSIST", "1") != "0"
    kname = ("lenpred_f32_kernel (one launch: 3xTF32 layers 1-3 with the A operand split into TMEM, head, "
             "quantizer, projection; events around the whole launch)" if path == 2 else
             "lenpred_small_kernel (one launch: layers 1-3, head, projection; events around the whole launch)"
             if small else ("umma_pair_nu2_kernel<256> (persistent tcgen05 cta_group::2 pairs + TMA, two "
                            "9-column tiles per pair, one wave)" if nu2 else
                            "umma_pair_gemm_kernel<256> (tcgen05 cta_group::2 + TMA" +
                            (", 9 column tiles)" if nu else ")") if pair else
                            "umma_gemm_kernel (tcgen05 + TMA, cluster split-K)") + " = predictor layer 1")
    roofline = {"kernel": kname,
                "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "algorithmic_flop_per_launch": flops_l1, "flop_per_request": flops_l1 / max(R, 1),
                "avg_launch_us": l1_avg_ms * 1e3, "share_of_step": l1_avg_ms / step_l1_avg_ms,
                "timing": "CUDA events recorded on the step's stream around the layer-1 launch inside the "
                          "captured step, over a second timed loop of the same K steps (the event pair "
                          "itself costs a few us, so the headline step time is taken without it)",
                "peak_source": peaks["source"] + " bf16_tflops (burst figure: the kernel runs inside a ~60 us step)"
                               + (" x 0.5 = TF32 (3xTF32: the tensor pipe does 3 MMAs per algorithmic product, so "
                                  "frac_3xtf32 = achieved / (peak / 3) is the fraction of what 3xTF32 can reach)"
                                  if f32 else "")}
    if f32:
        roofline["frac_3xtf32"] = achieved / (peak / 3.0)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "us_per_step": ms_per_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": c["dtype"],
            "data": "synthetic (seeded datagen: N(0,1) hidden states, He-normal weights, long-tailed CoT lengths)",
            "config": config_block(args.config, c, world), "cuda_graph": use_graph,
            "l2_flushed": flush is not None,
            "roofline": roofline, "stage_us": stage,
            "gpu_launches": (launches if launches is not None else 3 + (world > 1)) * args.steps,
            "launches_per_step": launches,
            "clocks": clocks, "e2e": e2e, "wall_s_timed": wall,
            "step_us_p50": float(np.median(step_ms)) * 1e3, "step_us_p99": float(np.percentile(step_ms, 99)) * 1e3,
            "step_us_warm_l2": warm_us, "requests_per_s_per_gpu": value / world}
    if graph_error:
        line["graph_error"] = graph_error
    # the paper's own figures (other hardware, context only), next to this run's
    line["paper_context"] = {
        "predictor_latency_ms": {"batch1": 1.33, "batch10": 1.40, "hw": "RTX 4090D (PAPER.md:306, 466)"},
        "decode_iteration_ms": {"value": 18.23, "hw": "RTX 4090D, R1-Distill-Qwen-7B W8A8 (PAPER.md:466)"},
        "overhead_pct": {"k1": 7.68, "k20": 0.38, "source": "PAPER.md:466-469"},
        "mae_tokens": {"value": 3873.21, "source": "PAPER.md:280-287, 305 (trained weights not available here)"},
        "p99_tpot_ms_sharegpt": {"vllm": 96.3, "vllm_rescheduling": 28.3, "star": 24.3,
                                 "hw": "4x RTX 4090D (PAPER.md:488, 577)"},
        "goodput_x_vs_vllm": {"sharegpt": 1.93, "max": 2.24, "source": "PAPER.md:15, 571, 652"},
        "this_run_step_ms": ms_per_step}
    try:
        line["plan_stats"] = {"moves_per_step": len(step.result()), "max_moves": c["max_moves"]}
    except Exception as ex:
        line["plan_stats"] = {"error": str(ex)}
    if world > 1 and not args.profile:
        try:   # NCCL floor: a 1-byte-per-rank all-gather on the same process group, device-timed
            one = torch.zeros(1, dtype=torch.uint8, device=dev)
            allb = torch.zeros(world, dtype=torch.uint8, device=dev)
            for _ in range(5):
                torch.distributed.all_gather_into_tensor(allb, one, group=group)
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(50):
                torch.distributed.all_gather_into_tensor(allb, one, group=group)
            e1.record(stream)
            e1.synchronize()
            tf = torch.tensor([e0.elapsed_time(e1) / 50 * 1e3], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(tf, op=torch.distributed.ReduceOp.MAX)
            line["nccl_floor_us"] = round(float(tf.item()), 2)
        except Exception as ex:
            line["nccl_floor_us"] = {"error": str(ex)}
    if rank == 0 and not args.profile and not args.no_sweep:
        try:
            line["roofline_projection"] = projection_sweep(star, snap, params_h_dev(star, params_h, dev), dev, peaks)
        except Exception as ex:  # keep the bench line
            line["roofline_projection"] = {"error": str(ex)}
    if world == 1 and not args.profile and not args.no_sweep and c["dtype"] == "bf16":
        try:
            line["refresh_k20"] = refresh_step_timing(star, Step, pred, params, c, snap, idx, h_dev, dev, flush)
        except Exception as ex:
            line["refresh_k20"] = {"error": str(ex)}
    if world == 1 and not args.profile and not args.no_sweep:
        try:
            line["tgt_rank"] = tgt_rank_timing(star, Step, dev, flush, seed=args.seed)
        except Exception as ex:
            line["tgt_rank"] = {"error": str(ex)}
    if world == 1 and not args.profile and not args.no_sweep:
        try:   # C5 (BASELINE.json configs[4]) at N = 1: the per-rank step of a W = 8 job vs R per instance
            import datagen
            line["c5_rank_sweep"] = {
                "workload": "C5: one rank of W = 8 (one instance per GPU), R requests per instance, d = 4096 bf16, "
                            "skewed; predictor + fused projection over this rank's R rows, Alg. 1 over the 8 "
                            "gathered records (8R requests); L2 flushed before every step; the NCCL all-gather "
                            "is not in the span",
                "points": [tgt_rank_timing(star, Step, dev, flush, seed=args.seed, reps=60, cfg="C5", r_per=r,
                                           stages=False) for r in datagen.CONFIGS["C5"]["r_sweep"]]}
        except Exception as ex:
            line["c5_rank_sweep"] = {"error": str(ex)}
        try:
            import episode
            line["c4_episode"] = episode.run_episode(star, Step, steps=200, dev=dev)
        except Exception as ex:
            line["c4_episode"] = {"error": str(ex)}
    if rank == 0 and not args.profile and not args.no_sweep:
        try:
            line["next_rows"] = next_rows_timing(star, dev)
        except Exception as ex:
            line["next_rows"] = {"error": str(ex)}
    if world == 1 and not args.no_cpu_baseline and not args.profile and rank == 0:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, args.seed, args.cpu_seconds)
        except Exception as ex:  # keep the bench line even if the oracle cannot be built
            line["cpu_baseline"] = {"value": None, "error": str(ex)}
    if rank == 0:
        print(json.dumps(line))
        if args.json_out:
            with open(args.json_out, "w") as f:
                json.dump(line, f, indent=1)
    if world > 1:
        torch.distributed.destroy_process_group()
    pred.close()
    return 0


def next_rows_timing(star, dev, seed=0):
    """NEXT rows at the paper's cluster scale, timed with CUDA events (warm, median of 20):
    the multi-CTA plan over 256 instances x 64 requests (H = 50; the paper budgets <= 300 ms at
    256 instances) and the projected P->D dispatch of 64 arrivals onto them."""
    import torch
    import datagen
    n, r_per = 256, 64
    snap = datagen.make_snapshot(seed + 77, n, r_per)
    out = {}
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    beta = datagen.beta_schedule_q16(50)
    proj = star.project_instance_load(d(snap.inst), d(snap.n_tok), d(snap.true_rem.astype(np.int32)), n, 50,
                                      d(beta.astype(np.int32)),
                                      workspace=torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8,
                                                            device=dev))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def device_us(fn, reps=20):
        """Device time of fn: captured in a CUDA graph, replayed after an L2 flush that keeps the
        GPU busy while the host enqueues (the span holds no host launch latency)."""
        s_ = torch.cuda.Stream(device=dev)
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            fn()
        torch.cuda.current_stream().wait_stream(s_)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        ts = []
        for i in range(reps + 3):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            e1.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        return round(float(np.median(ts)), 2)

    for mm in (1, 4):
        ph = datagen.make_plan_params(snap, max_moves=mm)
        pp = star.PlanParams.from_host(ph, device=dev)
        ws = torch.empty(star.plan_workspace_bytes(n, 50, snap.R), dtype=torch.uint8, device=dev)
        moves, nm = star.alloc_moves(mm, dev)
        args = (pp, proj.L, d(snap.req_id), d(snap.inst), d(snap.n_tok), d(snap.true_rem.astype(np.int32)))
        out[f"plan_256x64_max_moves_{mm}_us"] = device_us(
            lambda: star.plan_reschedule_large(*args, moves=moves, n_moves=nm, workspace=ws))
        out[f"plan_256x64_max_moves_{mm}_moves"] = int(nm.item())
    arr = datagen.make_snapshot(seed + 78, 1, 64)
    L0 = proj.L.clone()
    L1 = L0.clone()
    beta_d, ntok_d, nhat_d = d(beta.astype(np.int32)), d(arr.n_tok), d(arr.true_rem.astype(np.int32))
    assign = torch.empty(64, dtype=torch.int32, device=dev)
    from paper_2510_13668_b200 import _lib
    dws = torch.empty(int(_lib.lib().star_dispatch_workspace_bytes(n, 50)), dtype=torch.uint8, device=dev)

    def disp():
        L1.copy_(L0)   # same starting loads every replay (a 5.6 KB device copy)
        star.dispatch_requests(star.DISPATCH_PROJECTED, L1, beta_d, ntok_d, nhat_d, assign=assign, workspace=dws)
    out["dispatch_projected_64_arrivals_onto_256_us"] = device_us(disp)
    del flush
    out["kv_migration"] = kv_migration_timing(star, dev)
    out["note"] = ("paper: scheduler <= 300 ms at 256 instances (PAPER.md:460); NEXT rows of SURVEY 8(f), "
                   "bit-exact vs the oracle in tests/test_gpu_parity.py, tests/test_gpu_migrate.py")
    return out


def kv_migration_timing(star, dev, layers=32, blocks_per_layer=1024, n_tok=13_700, reps=5):
    """NEXT-4 (ExecuteMigration's KV copy): one request of the snapshot's mean
    running length (~13.7K tokens) in a Llama-3-8B-shaped paged pool (32 layers; block = 16 tokens
    x 8 KV heads x 128 x K,V x bf16 = 64 KB per layer), fragmented block tables.  Pack (pool ->
    staging), unpack (staging -> pool) and direct block-to-block migrate on ONE GPU; HBM GB/s =
    (read + write bytes) / CUDA-event time, against the measured copy peak (read + write).  The
    NVLink hop needs two GPUs: unmeasured here."""
    import torch
    bb = 16 * 8 * 128 * 2 * 2
    n = (n_tok + 15) // 16
    g = np.random.default_rng(3)
    src = torch.empty((layers, blocks_per_layer, bb), dtype=torch.uint8, device=dev)
    dst = torch.empty_like(src)
    st = torch.from_numpy(g.permutation(blocks_per_layer)[:n].astype(np.int32)).to(dev)
    dt = torch.from_numpy(g.permutation(blocks_per_layer)[:n].astype(np.int32)).to(dev)
    stg = torch.empty((layers, n, bb), dtype=torch.uint8, device=dev)
    moved = layers * n * bb
    peak = load_peaks()["hbm_gbs"]
    res = {"request_tokens": n_tok, "blocks": n, "layers": layers, "block_bytes": bb, "bytes_moved": moved}
    for name, fn in (("pack", lambda: star.kv_pack(src, st, staging=stg)),
                     ("unpack", lambda: star.kv_unpack(stg, dst, dt)),
                     ("migrate", lambda: star.kv_migrate(src, st, dst, dt))):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(ts))
        res[name] = {"us": round(t * 1e6, 1), "GBps": round(2 * moved / t / 1e9, 1),
                     "frac_hbm": round(2 * moved / t / 1e9 / peak, 4)}
    res["nvlink"] = ("unmeasured (one GPU); at NVLink 5's 900 GB/s per direction the transfer of this request "
                     "takes %.2f ms, at the paper's 25 Gbps %.0f ms (PAPER.md:647)" % (moved / 900e9 * 1e3,
                                                                                     moved * 8 / 25e9 * 1e3))
    del src, dst, stg
    return res


def refresh_step_timing(star, Step, pred, params, c, snap, idx, h_dev, dev, flush, k=20, reps=50):
    """Steady-state step in the paper's deployment mode (prediction cadence k = 20):
    1/k of the requests are due each step (slot r last predicted r mod k tokens ago), the rest
    age.  One CUDA graph per step, L2 flushed before each, CUDA events around the graph launch."""
    import torch
    R = len(idx)
    st = Step(pred, params, c["n_inst"], r_cap=max(R, 1), device=dev, refresh_k=k)
    req = [snap.req_id[idx], snap.inst[idx], snap.n_tok[idx]]
    st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in req))
    gen = (snap.n_tok[idx] - np.minimum(snap.n_tok[idx] - 1, 36)).astype(np.int32) + 100
    g_last = (gen - (np.arange(R) % k) - 1).astype(np.int32)   # slot r due when (r + 1) % k == 0 ...
    nhat_last = np.maximum(snap.true_rem[idx], 1).astype(np.int32)
    st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last), torch.from_numpy(nhat_last))
    s_ = torch.cuda.Stream(device=dev)
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        st.run(h_dev)
    torch.cuda.current_stream().wait_stream(s_)
    torch.cuda.synchronize()
    st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last), torch.from_numpy(nhat_last))
    g = torch.cuda.CUDAGraph(keep_graph=True)
    with torch.cuda.graph(g):
        st.run(h_dev)
    try:
        launches = count_kernel_nodes(g)
    except Exception:
        launches = None
    g.instantiate()
    ts, nref = [], []
    for i in range(reps + 5):
        st.set_generation(torch.from_numpy(gen + i))   # one token per step; the cadence state evolves
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
            nref.append(int(st.n_refreshed.item()))
    t = float(np.median(ts))
    return {"k": k, "us_per_step": round(t, 2), "us_per_step_mean": round(float(np.mean(ts)), 2),
            "requests_per_s": R / (t * 1e-6),
            "rows_repredicted_per_step": float(np.mean(nref)), "launches_per_step": launches,
            "note": "paper's deployment mode (k = 20, PAPER.md:463-469): due rows re-predicted, the rest "
                    "aged; projection + plan over all requests every step"}


def params_h_dev(star, params_h, dev):
    """PlanParams-like object for the sweep: H and a device beta_q."""
    class _P:
        pass
    p = _P()
    p.H = params_h.H
    p.beta_q = star.PlanParams.from_host(params_h, device=dev).beta_q
    return p


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_star(args)


if __name__ == "__main__":
    sys.exit(main())
