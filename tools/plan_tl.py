"""Single-CTA plan phase timeline inside the real step (C2), development tool."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200 import _lib  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
import bench  # noqa: E402
c, snap, params, idx, pw, h = bench.make_workload(cfg, 1, 0, 0)
R = len(idx)
d = lambda a, dt=None: (torch.from_numpy(np.ascontiguousarray(a)).to(dt) if dt else torch.from_numpy(np.ascontiguousarray(a))).cuda()
pred = star.Predictor(*[d(x, torch.bfloat16) for x in (pw.W1, pw.W2, pw.W3)], d(pw.w4), max_rows=R)
y0, _ = star.lenpred_forward(pred, d(h, torch.bfloat16))
scale = np.maximum(snap.true_rem[idx], 1).astype(np.float32) / max(float(torch.median(y0.float()).item()), 1e-3)
h = (h * scale[:, None]).astype(np.float32)
pp = star.PlanParams.from_host(params)
st = Step(pred, pp, c["n_inst"], r_cap=R)
st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in (snap.req_id[idx], snap.inst[idx], snap.n_tok[idx])),
                 pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
hd = d(h, torch.bfloat16)
for _ in range(5):
    st.run(hd)
torch.cuda.synchronize()
tl = _lib.plan_timeline().astype(np.int64)
names = ["entry", "launch", "staged", "W pass", "classify", "argmax", "apply", "end"]
print(cfg, "moves", st.result())
for k in range(1, 8):
    print(f"{names[k]:9s} +{(tl[k] - tl[k-1]) / 1e3:6.2f} us   (t={(tl[k] - tl[0]) / 1e3:6.2f})")

extra = {"scan start": 11, "scan end": 12, "warp argmax": 13, "blk argmax": 8, "apply loop": 9, "move write": 10}
for nm, k in extra.items():
    print(f"{nm:12s} t={(tl[k] - tl[0]) / 1e3:8.2f}")

cl = tl[32:48]
print("clock64 deltas (us at 1.965 GHz):", [(names[k], round((cl[k] - cl[k-1]) / 1965.0, 2)) for k in range(3, 8)],
      "blk argmax", round((cl[8] - cl[5]) / 1965.0, 2))

print("blk argmax detail (us): read", round((cl[9] - cl[5]) / 1965.0, 2), "reps", [round((cl[10 + r] - cl[9 + r]) / 1965.0, 3) for r in range(3)])

print("staging detail (us): static (pre-wait)", round((cl[12] - cl[1]) / 1965.0, 2), "pdl wait", round((cl[13] - cl[12]) / 1965.0, 2),
      "post-wait loads", round((cl[15] - cl[13]) / 1965.0, 2), "barrier+B", round((cl[2] - cl[15]) / 1965.0, 2))

print("round detail (us): compaction", round((cl[9] - cl[4]) / 1965.0, 2), "eval(t0)", round((cl[10] - cl[9]) / 1965.0, 2),
      "warp argmax", round((cl[11] - cl[10]) / 1965.0, 2), "to barrier", round((cl[5] - cl[11]) / 1965.0, 2))
