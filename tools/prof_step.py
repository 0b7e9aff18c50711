"""A few eager steps of the hot path for ncu (development tool; never a bench number).

    python tools/prof_step.py [--mode n1|rank|kv|proj] [--steps 3]

n1    the bench's N = 1 step of --config (TGT: 8 x 512 requests on one GPU, d = 4096 bf16: layer-1
      GEMM, fused tail (+ projection), cluster plan; C1: the one-launch fp32 predictor, cluster plan)
rank  one rank of the W = 8 TGT job: the one-launch small-batch predictor over 512 rows, then
      the cluster plan over the 8 gathered records (4096 requests)
kv    one KV-migration pack / unpack / migrate (NEXT-4) of a 13.7K-token request
proj  the standalone projection over 2^24 instance-grouped requests
The L2 is flushed (256 MB write) before every step, as in bench.py."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200.step import RecordLayout, Step  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="n1", choices=["n1", "rank", "kv", "proj", "refresh"])
ap.add_argument("--config", default="TGT")
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

if args.mode in ("n1", "rank"):
    world = 1 if args.mode == "n1" else 8
    steps, hs = [], []
    buf = pred = params = None
    for k in range(world):
        c, snap, params_h, idx, pw, h_np = bench.make_workload(args.config, world, k, 0)
        tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
        if pred is None:
            W = [torch.from_numpy(x).to(tdt).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
            pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=len(idx))
            params = star.PlanParams.from_host(params_h, device=dev)
            if world > 1:
                nb = RecordLayout(c["n_inst"] // world, params_h.H, len(idx)).nbytes
                buf = torch.zeros(world * nb, dtype=torch.uint8, device=dev)
        st = Step(pred, params, c["n_inst"], r_cap=len(idx), rank=k, world=world, device=dev, gathered=buf)
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                     snap.n_tok)),
                         pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
        h = bench.longtail_hidden(star, pred, h_np, snap, idx, tdt, dev)
        st.run(h)
        steps.append(st)
        hs.append(h)
    torch.cuda.synchronize()
    st, h = steps[0], hs[0]
    for _ in range(args.steps):
        flush.fill_(1.0)
        st.run(h)
    torch.cuda.synchronize()
    print("moves", st.result())
elif args.mode == "refresh":   # the bench's cadence-k step (k = 20, ~1/20 of the rows due)
    c, snap, params_h, idx, pw, h_np = bench.make_workload(args.config, 1, 0, 0)
    W = [torch.from_numpy(x).to(torch.bfloat16).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
    pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=len(idx))
    params = star.PlanParams.from_host(params_h, device=dev)
    h = bench.longtail_hidden(star, pred, h_np, snap, idx, torch.bfloat16, dev)
    R, k = len(idx), 20
    st = Step(pred, params, c["n_inst"], r_cap=R, device=dev, refresh_k=k)
    st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst, snap.n_tok)))
    gen = (snap.n_tok[idx] - np.minimum(snap.n_tok[idx] - 1, 36)).astype(np.int32) + 100
    g_last = (gen - (np.arange(R) % k) - 1).astype(np.int32)
    st.set_generation(torch.from_numpy(gen), torch.from_numpy(g_last),
                      torch.from_numpy(np.maximum(snap.true_rem[idx], 1).astype(np.int32)))
    for i in range(args.steps + 1):
        st.set_generation(torch.from_numpy(gen + i))
        flush.fill_(1.0)
        st.run(h)
    torch.cuda.synchronize()
    print("refreshed", int(st.n_refreshed.item()), "moves", st.result())
elif args.mode == "kv":
    r = bench.kv_migration_timing(star, dev, reps=1)
    print({k: r[k] for k in ("pack", "unpack", "migrate")})
else:
    import datagen
    c, snap, params_h, idx, pw, h_np = bench.make_workload("C2", 1, 0, 0)
    t, n, algo = bench._projection_point(star, snap, bench.params_h_dev(star, params_h, dev), dev, 1 << 24, reps=1)
    print("projection us", t * 1e6, "instances", n)
