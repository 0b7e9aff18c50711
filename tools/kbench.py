"""Per-stage in-graph timings of the hot path (development tool, not the bench contract).

Captures one CUDA graph per stage (predictor forward, projection, plan, whole step) for a
BASELINE config on one GPU and replays each with CUDA events, with the L2 flushed before every
replay (outside the timed span) and warm.  Prints one JSON object.

    python tools/kbench.py [--config C2] [--reps 200]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--rows", type=int, default=None, help="override total rows (all on one GPU)")
    args = ap.parse_args()
    c = datagen.CONFIGS[args.config]
    n_inst, r_per = c["n_inst"], c["r_per_inst"]
    if args.rows:
        r_per = args.rows // n_inst
    snap = datagen.make_snapshot(0, n_inst, r_per, skewed=c.get("skewed", False))
    params_h = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10), max_moves=c["max_moves"])
    pw = datagen.make_predictor_weights(0, c["d"], c["dtype"])
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    R = snap.R
    dev = torch.device("cuda", 0)
    W = [torch.from_numpy(x).to(tdt).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
    pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=R)
    h = torch.from_numpy(datagen.make_hidden(0, R, c["d"], c["dtype"])).to(tdt).to(dev)
    d32 = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    inst, n_tok, ids = d32(snap.inst), d32(snap.n_tok), d32(snap.req_id)
    n_hat = d32(snap.true_rem.astype(np.int32))
    y = torch.empty(R, dtype=torch.float32, device=dev)
    nh_pred = torch.empty(R, dtype=torch.int32, device=dev)
    params = star.PlanParams.from_host(params_h, device=dev)
    out = star.ProjectOut(n_inst, params_h.H, dev)
    ws = torch.zeros(star.project_workspace_bytes(n_inst, params_h.H), dtype=torch.uint8, device=dev)
    moves, nm = star.alloc_moves(params_h.max_moves, dev)
    pred.layer1_timing(True)

    def fwd():
        star.lenpred_forward(pred, h, n_tok=n_tok, y_hat=y, n_hat=nh_pred)

    def proj():
        star.project_instance_load(inst, n_tok, n_hat, n_inst, params_h.H, params.beta_q, out=out, workspace=ws)

    def plan():
        star.plan_reschedule(params, out.L, ids, inst, n_tok, n_hat, moves=moves, n_moves=nm)

    def step():
        fwd()
        proj()
        plan()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    res = {"config": args.config, "R": R, "d": c["d"]}
    for name, fn in (("forward", fwd), ("projection", proj), ("plan", plan), ("step", step)):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.synchronize()
        for mode in ("cold", "warm"):
            # events are graph nodes: the timed span starts when the GPU reaches it (after the
            # in-graph L2 flush), independent of host launch latency
            e0 = torch.cuda.Event(enable_timing=True, external=True)
            e1 = torch.cuda.Event(enable_timing=True, external=True)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                if mode == "cold":
                    flush.fill_(1.0)
                e0.record()
                fn()
                e1.record()
            ts, l1 = [], []
            for it in range(args.reps + 10):
                g.replay()
                e1.synchronize()
                if it >= 10:
                    ts.append(e0.elapsed_time(e1) * 1e3)
                    if name in ("forward", "step"):
                        l1.append(pred.layer1_ms() * 1e3)
            res[f"{name}_{mode}_us"] = round(statistics.median(ts), 2)
            if l1:
                res[f"{name}_{mode}_layer1_us"] = round(statistics.median(l1), 2)
        # marginal device time per stage: K back-to-back copies in one graph (warm L2)
        K = 10
        e0 = torch.cuda.Event(enable_timing=True, external=True)
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            e0.record()
            for _ in range(K):
                fn()
            e1.record()
        ts = []
        for it in range(30):
            g.replay()
            e1.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3 / K)
        res[f"{name}_marginal_us"] = round(statistics.median(ts), 2)
    # cost of the layer-1 timing events inside the graph: marginal step time without them
    pred.layer1_timing(False)
    e0 = torch.cuda.Event(enable_timing=True, external=True)
    e1 = torch.cuda.Event(enable_timing=True, external=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        e0.record()
        for _ in range(10):
            step()
        e1.record()
    ts = []
    for it in range(30):
        g.replay()
        e1.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3 / 10)
    res["step_marginal_no_l1_events_us"] = round(statistics.median(ts), 2)
    for name, fn in (("forward", fwd), ("plan", plan), ("proj", proj)):
        e0 = torch.cuda.Event(enable_timing=True, external=True)
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg):
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
        ts = []
        for it in range(30):
            gg.replay()
            e1.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3 / 10)
        res[f"{name}_marginal_no_l1_events_us"] = round(statistics.median(ts), 2)
    # (B) step graph without event nodes; stream events around its launch, flush kernel before
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        step()
    for mode in ("cold", "warm"):
        ts = []
        for it in range(110):
            if mode == "cold":
                flush.fill_(1.0)
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            g2.replay()
            a1.record()
            a1.synchronize()
            if it >= 10:
                ts.append(a0.elapsed_time(a1) * 1e3)
        res[f"step_streamevents_{mode}_us"] = round(statistics.median(ts), 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
