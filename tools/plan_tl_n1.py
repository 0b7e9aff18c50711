"""Plan phase timeline of the bench's N = 1 TGT step (development tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200 import _lib  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402

dev = torch.device("cuda", 0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "TGT"
c, snap, params_h, idx, pw, h_np = bench.make_workload(cfg, 1, 0, 0)
W = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=len(idx))
params = star.PlanParams.from_host(params_h, device=dev)
st = Step(pred, params, c["n_inst"], r_cap=len(idx), device=dev)
st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst, snap.n_tok)),
                 pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
h = bench.longtail_hidden(star, pred, h_np, snap, idx, torch.bfloat16, dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for _ in range(5):
    flush.fill_(1.0)
    st.run(h)
torch.cuda.synchronize()
print("moves", st.result())
tl = _lib.plan_timeline().astype(np.int64)
order = [1, 12, 13, 15, 2, 3, 4, 9, 10, 11, 5, 8, 6, 7]
lbl = {1: "launch", 12: "static staged", 13: "pdl_wait", 15: "dyn loads", 2: "staged", 3: "W pass", 4: "classify",
       9: "compaction", 10: "evaluate", 11: "warp argmax", 5: "block bar", 8: "final argmax", 6: "apply", 7: "end"}
prev = None
for k in order:
    cv = tl[32 + k]
    if cv:
        print(f"  clk {lbl[k]:14s} {(cv - tl[33]) / 1965.0:7.2f} us" + ("" if prev is None else f"  (+{(cv - prev) / 1965.0:.2f})"))
        prev = cv
cl = tl[64:128].reshape(8, 8)
t0 = cl[:, 0].min()
print("per-CTA (us from the earliest entry): entry, pdl_wait, pre-sync, post-sync (round-parity 0)")
for r in range(8):
    print(r, [round((cl[r, j] - t0) / 1e3, 2) if cl[r, j] else None for j in (0, 1, 2, 3)])
print("per-CTA slowest-thread evaluation (cycles), candidates, targets:")
for r in range(8):
    v = int(cl[r, 7])
    print(r, int(cl[r, 6]), v >> 32, v & 0xFFFFFFFF)
