"""NEXT-2/3 at cluster scale (256 instances x 64 requests, bench.py next_rows_timing's workload):
runs the multi-CTA plan (max_moves 4) and the projected dispatch a few times so an ncu launch
list shows the per-kernel split; prints the workload's candidate counts."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
n, r_per, H = 256, 64, 50
snap = datagen.make_snapshot(77, n, r_per)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
beta = datagen.beta_schedule_q16(H)
proj = star.project_instance_load(d(snap.inst), d(snap.n_tok), d(snap.true_rem.astype(np.int32)), n, H,
                                  d(beta.astype(np.int32)),
                                  workspace=torch.zeros(star.project_workspace_bytes(n, H), dtype=torch.uint8, device=dev))
mm = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ph = datagen.make_plan_params(snap, max_moves=mm)
pp = star.PlanParams.from_host(ph, device=dev)
ws = torch.empty(star.plan_workspace_bytes(n, H, snap.R), dtype=torch.uint8, device=dev)
moves, nm = star.alloc_moves(mm, dev)
args = (pp, proj.L, d(snap.req_id), d(snap.inst), d(snap.n_tok), d(snap.true_rem.astype(np.int32)))
for _ in range(3):
    star.plan_reschedule_large(*args, moves=moves, n_moves=nm, workspace=ws)
torch.cuda.synchronize()
print("moves", int(nm.item()))
arr = datagen.make_snapshot(78, 1, 64)
L1 = proj.L.clone()
assign = torch.empty(64, dtype=torch.int32, device=dev)
dws = torch.empty(int(_lib.lib().star_dispatch_workspace_bytes(n, H)), dtype=torch.uint8, device=dev)
for _ in range(3):
    star.dispatch_requests(star.DISPATCH_PROJECTED, L1, d(beta.astype(np.int32)), d(arr.n_tok),
                           d(arr.true_rem.astype(np.int32)), assign=assign, workspace=dws)
torch.cuda.synchronize()
print("ok")
