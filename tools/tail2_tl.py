"""Phase timeline of tail2 (the large-batch tail) after the layer-1 GEMM (development tool).
    python tools/tail2_tl.py [R]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = 4096
pw = datagen.make_predictor_weights(0, d, "bf16")
W = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=R)
h = torch.from_numpy(datagen.make_hidden(0, R, d, "bf16")).to(torch.bfloat16).cuda()
snap = datagen.make_snapshot(0, 8, R // 8)
nt, ins = torch.from_numpy(snap.n_tok).cuda(), torch.from_numpy(snap.inst).cuda()
beta = torch.from_numpy(datagen.beta_schedule_q16(50).astype(np.int32)).cuda()
ws = torch.zeros(star.project_workspace_bytes(8, 50), dtype=torch.uint8, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
pred.timeline(True)
for _ in range(5):
    flush.fill_(1.0)
    star.lenpred_forward_project(pred, h, nt, ins, 8, 50, beta, ws)
torch.cuda.synchronize()
tl = pred.timeline(fetch=True).astype(np.int64)
names = {1: "setup", 2: "prod pdl_wait", 3: "L2 acc ready", 4: "L3 acc ready (staged)", 5: "cluster sync",
         6: "head+proj (CTA0)", 7: "finalized"}
print(f"R={R} ctas={tl.shape[0]} SMs={len(set(tl[:, 15]))}")
for k, nm in names.items():
    v = tl[:, k]
    ok = v > 0
    if not ok.any():
        continue
    off = (v[ok] - tl[ok, 0]) / 1e3
    print(f"{k:2d} {nm:22s} n={ok.sum():3d}  min {off.min():7.2f}  med {np.median(off):7.2f}  max {off.max():7.2f} us")
