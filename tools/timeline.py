"""Fused-tail phase timeline (diagnostics): per-phase median/max offsets across CTAs."""
import os
import sys
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
pw = datagen.make_predictor_weights(0, d, "bf16")
W = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=R)
h = torch.from_numpy(datagen.make_hidden(0, R, d, "bf16")).to(torch.bfloat16).cuda()
snap = datagen.make_snapshot(0, 8, R // 8)
nt, ins = torch.from_numpy(snap.n_tok).cuda(), torch.from_numpy(snap.inst).cuda()
beta = torch.from_numpy(datagen.beta_schedule_q16(50).astype(np.int32)).cuda()
ws = torch.zeros(star.project_workspace_bytes(8, 50), dtype=torch.uint8, device="cuda")
pred.timeline(True, layer1=True)
for _ in range(5):
    star.lenpred_forward_project(pred, h, nt, ins, 8, 50, beta, ws)
torch.cuda.synchronize()
tl = pred.timeline(fetch=True).astype(np.int64)
names = ["entry", "prologue", "prod pdl_wait", "prod issued", "mma done", "epi consts", "accum ready",
         "publish L2", "csync1", "A3 done", "l3 ready", "publish Z3", "csync2", "stageA+ctr", "end"]
t0 = tl[:, 0].min()
print(f"R={R} ctas={tl.shape[0]} SMs used={len(set(tl[:, 15]))}")
for k, nm in enumerate(names):
    v = tl[:, k]
    v = v[v > 0] - t0
    if len(v):
        print(f"{k:2d} {nm:14s} min {v.min()/1e3:7.2f}  med {np.median(v)/1e3:7.2f}  max {v.max()/1e3:7.2f} us")

last = tl[tl[:, 16] > 0]
if len(last):
    r = last[0]
    print("last finisher (us after its arrival): staged", round((r[17] - r[16]) / 1e3, 2), "finalized",
          round((r[18] - r[16]) / 1e3, 2), "zeroed", round((r[19] - r[16]) / 1e3, 2), "end", round((r[14] - r[16]) / 1e3, 2),
          "| arrival at", round((r[16] - t0) / 1e3, 2))
tl1 = pred.timeline(fetch=True, layer1=True).astype(np.int64)
names1 = ["entry", "prologue", "prod pdl_wait", "mma kb0", "mma kb16", "mma kb32", "mma kb48", "splitK published",
          "splitK met", "mma done",
          "accum ready", "epilogue end", "exit sync"]
t0 = tl1[:, 0].min()
print(f"layer 1: ctas={tl1.shape[0]}")
for k, nm in enumerate(names1):
    if not nm:
        continue
    v = tl1[:, k]
    v = v[v > 0] - t0
    if len(v):
        print(f"{k:2d} {nm:14s} min {v.min()/1e3:7.2f}  med {np.median(v)/1e3:7.2f}  max {v.max()/1e3:7.2f} us")
print("same-CTA phase offsets from the CTA's own entry (robust to the per-GPC timer offset):")
for k, nm in enumerate(names1):
    if not nm or k == 0:
        continue
    ok = (tl1[:, k] > 0) & (tl1[:, 0] > 0)
    if ok.any():
        v = (tl1[ok, k] - tl1[ok, 0]) / 1e3
        print(f"{k:2d} {nm:16s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us (n={ok.sum()})")
print("per-CTA (us from own prologue), leader CTAs 0,2,64:")
for cta in (0, 2, 64):
    r = tl1[cta].astype(np.int64)
    print(cta, [round((r[k] - r[1]) / 1e3, 2) if r[k] else None for k in (2, 3, 4, 5, 6, 9, 10, 11, 12)])

# same-SM deltas (the globaltimer offset differs between SMs): tail griddepcontrol.wait release
# minus the layer-1 CTA exit on that SM; the smallest delta ~ the gap after the last layer-1 exit
l1_exit = {int(r[15]): int(r[12]) for r in tl1 if r[12]}
d = [int(r[2]) - l1_exit[int(r[15])] for r in tl if r[2] and int(r[15]) in l1_exit]
if d:
    d = np.array(d) / 1e3
    print(f"tail wait release - layer-1 exit on the same SM: min {d.min():.2f} med {np.median(d):.2f} max {d.max():.2f} us (n={len(d)})")
