"""Phase stamps of the plan run inside the fused tail's last CTA (Step at world 1), C2 or C4."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
c, snap, params_h, idx, pw, h_np = bench.make_workload(cfg, 1, 0, 0)
dev = torch.device("cuda:0")
R = len(idx)
W = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=R)
y0, _ = star.lenpred_forward(pred, torch.from_numpy(h_np).to(torch.bfloat16).to(dev))
scale = np.maximum(snap.true_rem[idx], 1).astype(np.float32) / max(float(torch.median(y0.float()).item()), 1e-3)
h = torch.from_numpy(h_np * scale[:, None]).to(torch.bfloat16).to(dev)
params = star.PlanParams.from_host(params_h, device=dev)
st = Step(pred, params, c["n_inst"], r_cap=R, device=dev)
st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in (snap.req_id[idx], snap.inst[idx], snap.n_tok[idx])),
                 pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
pred.timeline(True)
for _ in range(5):
    st.run(h)
torch.cuda.synchronize()
raw = pred.timeline(fetch=True, raw=True).astype(np.int64).reshape(-1)
pt = raw[590 * 32: 592 * 32]
tl = pred.timeline(fetch=True).astype(np.int64)
last = tl[tl[:, 16] > 0]
print(cfg, "moves", st.result())
cl = pt[32:64]
names = {12: "static+L issued", 15: "loads done", 2: "barrier", 3: "W pass", 4: "classify", 9: "compact", 5: "eval",
         6: "apply", 7: "end"}
prev = None
for k in (12, 15, 2, 3, 4, 9, 5, 6, 7):
    if cl[k]:
        print(f"{names[k]:16s} clock {(cl[k] - cl[12]) / 1965.0:7.2f} us")
if len(last):
    r = last[0]
    print("last finisher: finalize staged", round((r[17] - r[16]) / 1e3, 2), "finalized", round((r[18] - r[16]) / 1e3, 2),
          "zeroed", round((r[19] - r[16]) / 1e3, 2), "| plan start (globaltimer, same CTA) +",
          round((pt[12] - r[19]) / 1e3, 2), "plan end +", round((pt[7] - r[19]) / 1e3, 2))
print("W pass detail (us from barrier): start", round((cl[20] - cl[2]) / 1965, 2), "dot", round((cl[21] - cl[2]) / 1965, 2),
      "reduce", round((cl[22] - cl[2]) / 1965, 2), "warp0 done", round((cl[23] - cl[2]) / 1965, 2), "all", round((cl[3] - cl[2]) / 1965, 2))
