"""A serving loop around the public API (development example; synthetic inputs):

    python examples/decode_loop.py [--steps 50] [--k 20] [--kv]

Per decode iteration of one decode instance block (one rank, world 1 here): the running requests'
last-layer hidden states go through the length predictor (Eq. 2), the projection of every
instance's future token load, and Alg. 1, all captured in one CUDA graph (`Step.capture` /
`Step.replay`: one launch per step).  Every request generates one token per step; a request
that finishes leaves and a new one takes its slot (the request COUNT stays fixed, so the graph
stays valid; a changed count needs `Step.capture` again).  With --kv every planned move is also
executed: the request's paged KV blocks move between per-instance pools with `kv_migrate`.  With
--k the predictor re-predicts a request every k generated tokens and ages its prediction in
between (the paper's deployment mode).  The moves are what the engine hands to ExecuteMigration (Alg. 1 line 10,
PAPER.md:418)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2510_13668_b200 as star  # noqa: E402
from paper_2510_13668_b200.step import Step  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--k", type=int, default=0, help="prediction cadence (0: predict every request every step)")
    ap.add_argument("--instances", type=int, default=8)
    ap.add_argument("--requests", type=int, default=128, help="running requests per instance")
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--kv", action="store_true",
                    help="also run ExecuteMigration: per-instance paged KV pools (one GPU), kv_migrate per move")
    args = ap.parse_args(argv)
    dev = torch.device("cuda", 0)
    n, r_per, d = args.instances, args.requests, args.d
    snap = datagen.make_snapshot(0, n, r_per, skewed=True)
    R = snap.R
    # the predictor's weights (random here; a deployment loads the trained MLP) and the plan's knobs
    pw = datagen.make_predictor_weights(0, d, "bf16")
    pred = star.Predictor(*(torch.from_numpy(w).to(torch.bfloat16).to(dev) for w in (pw.W1, pw.W2, pw.W3)),
                          torch.from_numpy(pw.w4).to(dev), max_rows=R)
    params = star.PlanParams.from_host(datagen.make_plan_params(snap, H=50, max_moves=1), device=dev)
    step = Step(pred, params, n, r_cap=R, device=dev, refresh_k=args.k or None)
    req_id, inst, n_tok = snap.req_id.copy(), snap.inst.copy(), snap.n_tok.copy()
    remaining = np.maximum(snap.true_rem, 1).copy()
    step.load_requests(*(torch.from_numpy(a) for a in (req_id, inst, n_tok)))
    gen = np.zeros(R, np.int32)
    if args.k:
        step.set_generation(torch.from_numpy(gen))
    # the engine's buffer of last-layer hidden states (synthetic, scaled so predictions are long-tailed)
    h = torch.from_numpy(datagen.make_hidden(0, R, d, "bf16", scale=remaining.astype(np.float32) / 60.0)).to(
        torch.bfloat16).to(dev)
    step.capture(h)
    next_id = int(req_id.max()) + 1
    # ExecuteMigration's data: every instance owns a paged KV pool [layers, blocks, block bytes]; a
    # request owns ceil(tokens / 256) blocks of its instance's pool (a small synthetic model: 4
    # layers x 2 KB per block-layer)
    if args.kv:
        LAYERS, BLK_TOK, BLK_BYTES = 4, 256, 2048
        per_inst = int(np.ceil((n_tok.max() + args.steps) / BLK_TOK)) * (R // n) * 3
        pools = [torch.randint(0, 256, (LAYERS, per_inst, BLK_BYTES), dtype=torch.uint8, device=dev) for _ in range(n)]
        free = [list(range(per_inst)) for _ in range(n)]
        blocks = {}
        for r in range(R):
            nb = int(np.ceil(n_tok[r] / BLK_TOK))
            blocks[int(req_id[r])] = [free[inst[r]].pop() for _ in range(nb)]
        kv_bytes = 0
    moved = 0
    t0 = time.perf_counter()
    for it in range(args.steps):
        step.replay()
        moves = step.result()   # [(req_id, src, dst, round, gain)] -> ExecuteMigration
        moved += len(moves)
        for rid, src, dst, _, _ in moves:   # the engine migrates the request: its slot's instance changes
            inst[req_id == rid] = dst
            if args.kv:   # ExecuteMigration: the request's KV blocks into blocks the destination allocates
                src_tab = blocks[rid]
                dst_tab = [free[dst].pop() for _ in src_tab]
                expect = pools[src][:, src_tab].clone()
                star.kv_migrate(pools[src], torch.tensor(src_tab, dtype=torch.int32, device=dev), pools[dst],
                                torch.tensor(dst_tab, dtype=torch.int32, device=dev))
                assert torch.equal(pools[dst][:, dst_tab], expect), "KV migration mismatch"
                free[src].extend(src_tab)
                blocks[rid] = dst_tab
                kv_bytes += LAYERS * len(src_tab) * BLK_BYTES
        # one decode iteration: every request generates a token; finished ones are replaced in place
        remaining -= 1
        n_tok += 1
        gen += 1
        done = remaining <= 0
        if args.kv:   # requests growing into a new block
            for r in np.nonzero((n_tok % BLK_TOK == 1) & ~done)[0]:
                blocks[int(req_id[r])].append(free[inst[r]].pop())
            for r in np.nonzero(done)[0]:   # finished requests free their blocks
                free[inst[r]].extend(blocks.pop(int(req_id[r])))
        if done.any():
            req_id[done] = np.arange(next_id, next_id + int(done.sum()), dtype=req_id.dtype)
            next_id += int(done.sum())
            n_tok[done] = np.random.default_rng(it).integers(64, 2048, int(done.sum()))
            remaining[done] = np.random.default_rng(it + 1).integers(16, 4000, int(done.sum()))
            gen[done] = 0
            if args.kv:
                for r in np.nonzero(done)[0]:
                    blocks[int(req_id[r])] = [free[inst[r]].pop() for _ in range(int(np.ceil(n_tok[r] / BLK_TOK)))]
        step.v["req_id"][:R].copy_(torch.from_numpy(req_id))
        step.v["inst"][:R].copy_(torch.from_numpy(inst))
        step.v["n_tok"][:R].copy_(torch.from_numpy(n_tok))
        if args.k:
            step.gen[:R].copy_(torch.from_numpy(gen))
            if done.any():   # new occupants: no prediction yet
                idx = torch.from_numpy(np.nonzero(done)[0]).to(dev)
                step.g_last.index_fill_(0, idx, -1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{args.steps} steps of {R} requests ({n} instances, d = {d}): {moved} migrations planned"
          + (f" and executed ({kv_bytes / 1e6:.1f} MB of KV blocks moved, byte-exact)" if args.kv else "")
          + f"; host loop {dt / args.steps * 1e3:.2f} ms per step (synthetic inputs, host bookkeeping included)")
    assert step.err.item() == 0
    pred.close()
    return moved


if __name__ == "__main__":
    main()
