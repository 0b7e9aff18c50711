"""Where the per-rank step's span goes besides the two kernels (development tool): the bench's
timing (flush; event; graph replay; event) against the same with the GPU kept busy by a sleep
kernel between the flush and the first event (so no host launch latency can sit inside the span),
and graphs of 1 / 2 empty kernels timed the same two ways.

    python tools/rank_gap.py [--config TGT] [--r-per R]"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200.step import RecordLayout, Step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="TGT")
ap.add_argument("--r-per", type=int, default=None)
args = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
world = 8
steps, hs = [], []
buf = pred = params = None
for k in range(world):
    c, snap, params_h, idx, pw, h_np = bench.make_workload(args.config, world, k, 0, r_per=args.r_per)
    if pred is None:
        W = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
        pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=c["r_per_inst"])
        params = star.PlanParams.from_host(params_h, device=dev)
        nb = RecordLayout(c["n_inst"] // world, params_h.H, c["r_per_inst"]).nbytes
        buf = torch.zeros(world * nb, dtype=torch.uint8, device=dev)
    st = Step(pred, params, c["n_inst"], r_cap=c["r_per_inst"], rank=k, world=world, device=dev, gathered=buf)
    st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                  snap.n_tok)),
                     pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
    h = bench.longtail_hidden(star, pred, h_np, snap, idx, torch.bfloat16, dev)
    st.run(h)
    steps.append(st)
    hs.append(h)
torch.cuda.synchronize()
st, h = steps[0], hs[0]


def graph_of(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def timed(g, do_flush, sleep_cycles, reps=200, eager=None):
    ts = []
    for i in range(reps + 10):
        if do_flush:
            flush.fill_(1.0)
        if sleep_cycles:
            torch.cuda._sleep(sleep_cycles)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if eager is not None:
            eager()
        else:
            g.replay()
        e1.record()
        e1.synchronize()
        if i >= 10:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts), np.min(ts)


x = torch.zeros(1, device=dev)
variants = {"rank step": graph_of(lambda: st.run(h)),
            "1 empty kernel": graph_of(lambda: x.add_(1)),
            "2 empty kernels": graph_of(lambda: (x.add_(1), x.add_(1)))}
for name, g in variants.items():
    for do_flush in (True, False):
        for sl in (0, 200000):
            med, mn = timed(g, do_flush, sl)
            print(f"{name:16s} flush={int(do_flush)} sleep={sl:6d}: median {med:7.2f} us  min {mn:7.2f}")
eagers = {"rank step": lambda: st.run(h), "1 empty kernel": lambda: x.add_(1),
          "2 empty kernels": lambda: (x.add_(1), x.add_(1))}
for name, fn in eagers.items():
    for do_flush in (True, False):
        med, mn = timed(None, do_flush, 200000, eager=fn)
        print(f"{name:16s} EAGER flush={int(do_flush)} sleep=200000: median {med:7.2f} us  min {mn:7.2f}")
print("moves", int(st.n_moves.item()))
pred.close()
