"""Refresh-mode (k = 20) step on C2 run a few times without a graph, for an ncu launch list
(development tool):  ncu --metrics gpu__time_duration.sum python tools/refresh_prof.py"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
k = 20
c, snap, params_h, idx, pw, h_np = bench.make_workload(cfg, 1, 0, 0)
dev = torch.device("cuda:0")
R = len(idx)
W = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=R)
params = star.PlanParams.from_host(params_h, device=dev)
h_dev = torch.from_numpy(h_np).to(torch.bfloat16).to(dev)
st = Step(pred, params, c["n_inst"], r_cap=R, device=dev, refresh_k=k)
st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in (snap.req_id[idx], snap.inst[idx], snap.n_tok[idx])))
gen = (snap.n_tok[idx] - np.minimum(snap.n_tok[idx] - 1, 36)).astype(np.int32) + 100
g_last = (gen - (np.arange(R) % k) - 1).astype(np.int32)
nhat_last = np.maximum(snap.true_rem[idx], 1).astype(np.int32)
st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last), torch.from_numpy(nhat_last))
for i in range(4):
    st.set_generation(torch.from_numpy(gen + i))
    st.run(h_dev)
torch.cuda.synchronize()
print("refreshed rows last step:", int(st.n_refreshed.item()))
