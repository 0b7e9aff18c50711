"""Isolated-launch durations from %globaltimer stamps (first CTA entry -> last CTA exit)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pw = datagen.make_predictor_weights(0, 4096, "bf16")
W = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).cuda(), max_rows=R)
h = torch.from_numpy(datagen.make_hidden(0, R, 4096, "bf16")).to(torch.bfloat16).cuda()
snap = datagen.make_snapshot(0, 8, R // 8)
nt, ins = torch.from_numpy(snap.n_tok).cuda(), torch.from_numpy(snap.inst).cuda()
beta = torch.from_numpy(datagen.beta_schedule_q16(50).astype(np.int32)).cuda()
ws = torch.zeros(star.project_workspace_bytes(8, 50), dtype=torch.uint8, device="cuda")
pred.timeline(True)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for it in range(6):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    star.lenpred_forward_project(pred, h, nt, ins, 8, 50, beta, ws)
    torch.cuda.synchronize()
t1 = pred.timeline(fetch=True, layer1=True).astype(np.int64)
tt = pred.timeline(fetch=True).astype(np.int64)
l1_beg, l1_end = t1[:, 0].min(), t1[:, 12].max()
ta_beg, ta_end = tt[:, 0].min(), tt[:, 14].max()
print(f"R={R}: layer1 {(l1_end - l1_beg)/1e3:.2f} us (pdl_wait med {np.median(t1[:,2]-l1_beg)/1e3:.2f}, "
      f"mma done med {np.median(t1[t1[:,9]>0,9]-l1_beg)/1e3:.2f}); gap {(ta_beg - l1_end)/1e3:.2f}; "
      f"tail {(ta_end - ta_beg)/1e3:.2f} us; layer1 start -> tail end {(ta_end - l1_beg)/1e3:.2f} us")
e = t1[:, 0] - l1_beg
print("layer1 entry spread: min %.2f med %.2f max %.2f us" % (e.min()/1e3, np.median(e)/1e3, e.max()/1e3))
w = (t1[:, 2] - t1[:, 0])
w = w[t1[:, 2] > 0]
print("layer1 pdl_wait - entry (producer CTAs): min %.2f med %.2f max %.2f us" % (w.min()/1e3, np.median(w)/1e3, w.max()/1e3))
m = t1[:, 9] - t1[:, 2]
m = m[t1[:, 9] > 0]
print("layer1 mma done - pdl_wait (leaders): min %.2f med %.2f max %.2f us" % (m.min()/1e3, np.median(m)/1e3, m.max()/1e3))
x = t1[:, 12] - t1[:, 9]
x = x[t1[:, 9] > 0]
print("layer1 exit - mma done: med %.2f us" % (np.median(x)/1e3))
order = np.argsort(e)
print("entry offsets (us) sorted, with smid:", [(round(e[i] / 1e3, 2), int(t1[i, 15])) for i in order[:12]], "...",
      [(round(e[i] / 1e3, 2), int(t1[i, 15])) for i in order[-4:]])
early = e < 5000
print("early CTAs:", int(early.sum()), "SMs", sorted(int(x) for x in t1[early, 15]))
print("early CTAs' exit (us):", np.round((t1[early, 12] - l1_beg) / 1e3, 1)[:10])
print("late CTAs:", int((~early).sum()))
te_ = tt[:, 0] - l1_beg
print("tail entry rel. layer1 start: min %.2f med %.2f max %.2f; tail pdl_wait(producer) med %.2f; tail end max %.2f" % (
    te_.min()/1e3, np.median(te_)/1e3, te_.max()/1e3, np.median(tt[:, 2] - l1_beg)/1e3, (tt[:, 14].max() - l1_beg)/1e3))
print("tail CTAs entering before 5 us:", int((te_ < 5000).sum()))
