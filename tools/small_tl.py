"""Phase timeline of the one-launch small-batch predictor (development tool): per-CTA %globaltimer
stamps, reported as offsets from the CTA's own entry (robust to the per-GPC timer offsets).
    python tools/small_tl.py [R] [--cold]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 512
cold = "--cold" in sys.argv
d = 4096
pw = datagen.make_predictor_weights(0, d, "bf16")
W = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=R)
assert pred.path(R) == 1
h = torch.from_numpy(datagen.make_hidden(0, R, d, "bf16")).to(torch.bfloat16).cuda()
snap = datagen.make_snapshot(0, 1, R)
nt, ins = torch.from_numpy(snap.n_tok).cuda(), torch.from_numpy(snap.inst).cuda()
beta = torch.from_numpy(datagen.beta_schedule_q16(50).astype(np.int32)).cuda()
ws = torch.zeros(star.project_workspace_bytes(1, 50), dtype=torch.uint8, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
pred.timeline(True)
for _ in range(5):
    star.lenpred_forward_project(pred, h, nt, ins, 1, 50, beta, ws)
if cold:
    flush.fill_(1.0)
star.lenpred_forward_project(pred, h, nt, ins, 1, 50, beta, ws)
torch.cuda.synchronize()
tl = pred.timeline(fetch=True).astype(np.int64)
names = {0: "entry", 1: "setup+csync", 2: "prod pdl_wait", 3: "L1 acc ready", 4: "L1 csync (push)",
         5: "L2 z1 ready", 6: "Z1 published", 7: "L2 acc ready", 8: "Z2 published", 9: "L3 acc ready",
         10: "head+proj", 11: "finalized", 12: "L1 recv landed", 13: "L1 reduced+stored", 14: "L2 recv landed",
         16: "L3 recv landed"}
print(f"R={R} ctas={tl.shape[0]} SMs={len(set(tl[:, 15]))} cold={cold}")
for k, nm in sorted(names.items(), key=lambda kv: np.median(tl[tl[:, kv[0]] > 0, kv[0]] - tl[tl[:, kv[0]] > 0, 0]) if (tl[:, kv[0]] > 0).any() else 0):
    v = tl[:, k]
    ok = v > 0
    if k == 0 or not ok.any():
        continue
    off = (v[ok] - tl[ok, 0]) / 1e3
    print(f"{k:2d} {nm:16s} n={ok.sum():3d}  min {off.min():7.2f}  med {np.median(off):7.2f}  max {off.max():7.2f} us")
# whole-launch time, warm (back to back) and cold (L2 flushed before each), CUDA graph + events
pred.timeline(False)
g = torch.cuda.CUDAGraph()
s_ = torch.cuda.Stream()
s_.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s_):
    star.lenpred_forward_project(pred, h, nt, ins, 1, 50, beta, ws)
torch.cuda.current_stream().wait_stream(s_)
with torch.cuda.graph(g):
    star.lenpred_forward_project(pred, h, nt, ins, 1, 50, beta, ws)
for mode in ("warm", "cold"):
    ts = []
    for i in range(30):
        if mode == "cold":
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(1 if mode == "cold" else 10):
            g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / (1 if mode == "cold" else 10))
    print(f"{mode}: median {np.median(ts):.2f} us  min {np.min(ts):.2f}")
