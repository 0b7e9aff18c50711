"""Marginal cost (10 back-to-back steps in one graph, no inner events) of the fused single-rank
step vs forward_project + plan_reschedule (development tool)."""
import os, sys, statistics
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = datagen.CONFIGS[cfg]
n = c["n_inst"]
snap = datagen.make_snapshot(0, n, c["r_per_inst"])
R = snap.R
pw = datagen.make_predictor_weights(0, c["d"], "bf16")
h = datagen.make_hidden(0, R, c["d"], "bf16", scale=(np.maximum(snap.true_rem, 1) / 1500.0).astype(np.float32))
d = lambda a, dt=None: (torch.from_numpy(np.ascontiguousarray(a)).to(dt) if dt else torch.from_numpy(np.ascontiguousarray(a))).cuda()
W = [d(x, torch.bfloat16) for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, d(pw.w4), max_rows=R)
pp = star.PlanParams.from_host(datagen.make_plan_params(snap, max_moves=c["max_moves"]))
hd, ntd, ind, idd = d(h, torch.bfloat16), d(snap.n_tok), d(snap.inst), d(snap.req_id)
ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
nh = torch.empty(R, dtype=torch.int32, device="cuda")
out = star.ProjectOut(n, 50, "cuda")
mv, nm = star.alloc_moves(pp.max_moves, "cuda")

def fused():
    star.lenpred_forward_project_plan(pred, hd, ntd, ind, idd, pp, ws, n_hat=nh, out=out, moves=mv, n_moves=nm)

def sep():
    star.lenpred_forward_project(pred, hd, ntd, ind, n, 50, pp.beta_q, ws, n_hat=nh, out=out, want_y=False)
    star.plan_reschedule(pp, out.L, idd, ind, ntd, nh, moves=mv, n_moves=nm)

def fwd_only():
    star.lenpred_forward_project(pred, hd, ntd, ind, n, 50, pp.beta_q, ws, n_hat=nh, out=out, want_y=False)

res = {}
for name, fn in (("fused", fused), ("separate", sep), ("forward_project_only", fwd_only)):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True, external=True)
    e1 = torch.cuda.Event(enable_timing=True, external=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
    ts = []
    for it in range(25):
        g.replay()
        e1.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1) * 100)
    res[name] = round(statistics.median(ts), 2)
print(cfg, res, "moves", int(nm.item()))
