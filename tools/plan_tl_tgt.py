"""Standalone plan kernel phase timeline at the per-rank north-star point (development tool):
one rank of W=8 at TGT on one GPU (bench.tgt_rank_timing), then star_plan_timeline."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200 import _lib  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402

r = bench.tgt_rank_timing(star, Step, torch.device("cuda", 0), None, reps=20)
print({k: r[k] for k in ("us_per_step_p50", "stage_us", "moves")})
tl = _lib.plan_timeline().astype(np.int64)
names = ["entry", "launch", "staged", "W pass", "classify", "argmax", "apply", "end"]
for k in range(1, 8):
    if tl[k]:
        print(f"{names[k]:9s} t={(tl[k] - tl[0]) / 1e3:6.2f} us")
cl = tl[32:48]
print("staging detail (us): static (pre-wait)", round((cl[12] - cl[1]) / 1965.0, 2), "pdl wait",
      round((cl[13] - cl[12]) / 1965.0, 2), "post-wait loads", round((cl[15] - cl[13]) / 1965.0, 2),
      "barrier", round((cl[2] - cl[15]) / 1965.0, 2))
print("raw globaltimer offsets (us):", [(k, round((tl[k] - tl[0]) / 1e3, 2)) for k in range(16) if tl[k]])
order = [1, 12, 13, 15, 2, 3, 4, 9, 10, 11, 5, 8, 6, 7]
lbl = {1: "launch", 12: "static staged", 13: "pdl_wait", 15: "dyn loads", 2: "staged", 3: "W pass", 4: "classify",
       9: "compaction", 10: "evaluate", 11: "warp argmax", 5: "block bar", 8: "final argmax", 6: "apply", 7: "end"}
prev = None
for k in order:
    if cl[k - 0 if k < 16 else k]:
        pass
for k in order:
    c = tl[32 + k]
    if c:
        print(f"  clk {lbl[k]:14s} {(c - tl[33]) / 1965.0:7.2f} us" + ("" if prev is None else f"  (+{(c - prev) / 1965.0:.2f})"))
        prev = c
print("per-CTA: eval cycles of the slowest thread (round 0), candidates, targets")
for r_ in range(8):
    v7 = int(tl[64 + 8 * r_ + 7])
    print(f"  cta {r_}: eval {int(tl[64 + 8 * r_ + 6]):6d} cyc  ncand {v7 >> 32}  nU {v7 & 0xffffffff}")
