"""Projection at bandwidth scale (development tool): timing + optional ncu target."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

R = 1 << (int(sys.argv[4]) if len(sys.argv) > 4 else 24)
n_per = int(sys.argv[1]) if len(sys.argv) > 1 else 32   # instance multiplier: n_inst = 8 * n_per
snap = datagen.make_snapshot(0, 8, 256)
reps = R // snap.R
shift = (np.arange(reps, dtype=np.int64) % n_per * 8).repeat(snap.R)
inst = torch.from_numpy((np.tile(snap.inst, reps) + shift).astype(np.int32)).cuda()
ntok = torch.from_numpy(np.tile(snap.n_tok, reps)).cuda()
nhat = torch.from_numpy(np.tile(snap.true_rem.astype(np.int32), reps)).cuda()
n = 8 * n_per
dist = sys.argv[3] if len(sys.argv) > 3 else "real"
if dist == "hot":
    nhat = torch.full_like(nhat, 1000)
elif dist == "cold":
    nhat = torch.randint(0, 51, nhat.shape, dtype=torch.int32, device=nhat.device)
if len(sys.argv) > 2 and sys.argv[2] == "grouped":   # instance-major layout (each instance's batch contiguous)
    order = torch.argsort(inst, stable=True)
    inst, ntok, nhat = inst[order].contiguous(), ntok[order].contiguous(), nhat[order].contiguous()
beta = torch.from_numpy(datagen.beta_schedule_q16(50).astype(np.int32)).cuda()
ws = torch.zeros(star.project_workspace_bytes(n, 50), dtype=torch.uint8, device="cuda")
out = star.ProjectOut(n, 50, "cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
fn = lambda: star.project_instance_load(inst, ntok, nhat, n, 50, beta, out=out, workspace=ws, err_flag=err)
for _ in range(3):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(10):   # 10 launches back to back per span: device time (inputs beyond L2 stream from HBM)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 10)
t = float(np.median(ts)) * 1e-3
print(f"n_inst={n} R=2^{R.bit_length()-1} {sys.argv[2:3]}: {t*1e6:.1f} us, {12*R/t/1e9:.0f} GB/s, err={err.item()}")
