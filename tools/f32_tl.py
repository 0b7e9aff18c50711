"""Phase timeline of the one-launch fp32 predictor (development tool): per-CTA %globaltimer stamps
as offsets from the CTA's own entry.   python tools/f32_tl.py [R] [d] [--cold]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

args = [a for a in sys.argv[1:] if a.isdigit()]
R = int(args[0]) if args else 128
d = int(args[1]) if len(args) > 1 else 896
cold = "--cold" in sys.argv
pw = datagen.make_predictor_weights(0, d, "f32")
W = [torch.from_numpy(x).cuda() for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=R)
assert pred.path(R) == 2
h = torch.from_numpy(datagen.make_hidden(0, R, d, "f32")).cuda()
snap = datagen.make_snapshot(0, 2, (R + 1) // 2)
nt, ins = torch.from_numpy(snap.n_tok[:R]).cuda(), torch.from_numpy(snap.inst[:R]).cuda()
beta = torch.from_numpy(datagen.beta_schedule_q16(50).astype(np.int32)).cuda()
ws = torch.zeros(star.project_workspace_bytes(2, 50), dtype=torch.uint8, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
pred.timeline(True)
for _ in range(5):
    star.lenpred_forward_project(pred, h, nt, ins, 2, 50, beta, ws)
if cold:
    flush.fill_(1.0)
star.lenpred_forward_project(pred, h, nt, ins, 2, 50, beta, ws)
torch.cuda.synchronize()
tl = pred.timeline(fetch=True).astype(np.int64)
names = {1: "prod pdl_wait", 2: "L1 acc ready", 3: "L1 partials in", 4: "Z1 published", 5: "L2 z1 ready",
         6: "L2 acc ready", 7: "L2 partials in", 8: "Z2 published", 9: "L3 acc ready", 10: "y partial out",
         11: "finalized"}
print(f"R={R} d={d} ctas={tl.shape[0]} cold={cold}")
for k, nm in sorted(names.items(), key=lambda kv: np.median(tl[tl[:, kv[0]] > 0, kv[0]] - tl[tl[:, kv[0]] > 0, 0]) if (tl[:, kv[0]] > 0).any() else 0):
    v = tl[:, k]
    ok = (v > 0) & (tl[:, 0] > 0)
    if not ok.any():
        continue
    off = (v[ok] - tl[ok, 0]) / 1e3
    print(f"{k:2d} {nm:16s} n={ok.sum():3d}  min {off.min():7.2f}  med {np.median(off):7.2f}  max {off.max():7.2f} us")
for k, nm in ((24, "conv wait L1"), (25, "conv split L1"), (26, "conv wait L2"), (27, "conv split L2"),
              (20, "mma wait L1"), (21, "mma wait L2"), (23, "mma span L1")):
    v = tl[:, k].astype(np.float64)
    print(f"   {nm:14s} cycles: med {np.median(v):9.0f}  max {v.max():9.0f}")
v = tl[:4, 28].astype(np.float64), tl[:4, 29].astype(np.float64), tl[:4, 22].astype(np.float64)
print(f"   L3 conv wait {v[0]}  split {v[1]}  mma wait {v[2]}")
e0 = tl[tl[:, 0] > 0, 0]
print(f"entry spread: {(e0.max() - e0.min()) / 1e3:.2f} us")
pred.timeline(False)
g = torch.cuda.CUDAGraph()
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_):
    star.lenpred_forward_project(pred, h, nt, ins, 2, 50, beta, ws)
torch.cuda.current_stream().wait_stream(s_)
with torch.cuda.graph(g):
    star.lenpred_forward_project(pred, h, nt, ins, 2, 50, beta, ws)
for mode in ("warm", "cold"):
    ts = []
    for i in range(30):
        if mode == "cold":
            flush.fill_(1.0)
        e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0_.record()
        for _ in range(1 if mode == "cold" else 10):
            g.replay()
        e1_.record()
        e1_.synchronize()
        ts.append(e0_.elapsed_time(e1_) * 1e3 / (1 if mode == "cold" else 10))
    print(f"{mode}: median {np.median(ts):.2f} us  min {np.min(ts):.2f}")
