"""Phase stamps of the refresh select kernel (development tool): the bench's cadence-k step (k = 20)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
dev = torch.device("cuda", 0)
c, snap, params_h, idx, pw, h_np = bench.make_workload(cfg, 1, 0, 0)
W = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=len(idx))
params = star.PlanParams.from_host(params_h, device=dev)
h = bench.longtail_hidden(star, pred, h_np, snap, idx, torch.bfloat16, dev)
R, k = len(idx), 20
st = Step(pred, params, c["n_inst"], r_cap=R, device=dev, refresh_k=k)
st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst, snap.n_tok)))
gen = (snap.n_tok[idx] - np.minimum(snap.n_tok[idx] - 1, 36)).astype(np.int32) + 100
g_last = (gen - (np.arange(R) % k) - 1).astype(np.int32)
st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last), torch.from_numpy(np.maximum(snap.true_rem[idx], 1).astype(np.int32)))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
pred.timeline(True)
for i in range(4):
    st.set_generation(torch.from_numpy(gen + i))
    flush.fill_(1.0)
    st.run(h)
torch.cuda.synchronize()
tl = pred.timeline(fetch=True, raw=True).astype(np.int64)
G = (R + 127) // 128
sel = tl[400:400 + G, :6]
t0 = sel[:, 0].min()
print(f"{cfg}: R={R} select CTAs={G}; stamps (us from the earliest entry): entry, after pdl_wait, flags+scan, aged+projected, counts met, gathered")
for b in range(G):
    print(b, [round((v - t0) / 1e3, 2) for v in sel[b]])
