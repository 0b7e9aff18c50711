"""C4 episode harness (SURVEY.md §8(d) "C4 episode"; BASELINE.json configs[3]: "4 instances x
1024 requests, hidden 4096, skewed arrivals forcing repeated migrations near KV-OOM").

A closed loop AROUND the hot path (the harness is not on it): every episode step runs the
product's Step (predictor -> fused projection -> Alg. 1, through the C ABI) on the current
running batch, then the harness plays the decode engine between two planning rounds:

  1. the planned moves are applied (the request's instance is rewritten, and it stays pinned --
     "migrating" -- for the next round, reading A22);
  2. every unpinned request generates `tokens_per_step` tokens (N += t, remaining -= t);
  3. finished requests leave;
  4. Poisson arrivals (mean = the departures, so the batch size stays level) land on instance 0
     with probability `p_inst0`, otherwise uniformly (the skew a length-unaware dispatcher
     produces), each a fresh long-tailed request (datagen.sample_lengths).

A round of Alg. 1 per scheduling interval ("every 1 second"; at the paper's
18.23 ms decode iteration, that is ~50 iterations, hence tokens_per_step = 50).
Reported: moves per step, how many steps had an instance over its C_mem, batch size range, and
the eager step time.  Hidden states: each request keeps one N(0,1) base row, scaled every step
by its current true remaining length / median(y_hat) -- positive homogeneity of bias-free Eq. 2
keeps the predictions tracking the remaining lengths as they shrink.

This module holds none of the method's arithmetic and never imports the oracle; a test passes
`check(step_index, state, st)` to compare each step against it."""
from __future__ import annotations

import numpy as np
import torch

import datagen


def run_episode(star, Step, cfg="C4", steps=200, tokens_per_step=50, p_inst0=0.5, seed=0, dev=None,
                check=None, r_slack=1024):
    dev = dev or torch.device("cuda", torch.cuda.current_device())
    c = datagen.CONFIGS[cfg]
    n, d = c["n_inst"], c["d"]
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    snap = datagen.make_snapshot(seed, n, c["r_per_inst"], skewed=c.get("skewed", False))
    params_h = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10), max_moves=c["max_moves"])
    params = star.PlanParams.from_host(params_h, device=dev)
    pw = datagen.make_predictor_weights(seed, d, c["dtype"])
    r_cap = snap.R + r_slack
    W = [torch.from_numpy(x).to(tdt).to(dev) for x in (pw.W1, pw.W2, pw.W3)]
    pred = star.Predictor(*W, torch.from_numpy(pw.w4).to(dev), max_rows=r_cap)
    st = Step(pred, params, n, r_cap=r_cap, device=dev)
    g = datagen.rng(seed + 555)

    # hidden base rows: one per request slot ever used (recycled ring of r_cap + arrivals)
    pool = r_cap + 2048
    h_base = torch.from_numpy(datagen.make_hidden(seed + 1, pool, d, c["dtype"])).to(dev)
    y0, _ = star.lenpred_forward(pred, h_base[:min(pool, r_cap)].to(tdt))
    med = max(float(torch.median(y0.float()).item()), 1e-3)

    req_id = snap.req_id.astype(np.int64)
    inst = snap.inst.astype(np.int64)
    n_tok = snap.n_tok.astype(np.int64)
    rem = snap.true_rem.astype(np.int64)
    row = np.arange(snap.R, dtype=np.int64)
    pinned = np.zeros(snap.R, np.uint8)
    next_id = int(req_id.max()) + 1
    next_row = snap.R
    c_mem = params_h.c_mem
    reserved = params_h.reserved if params_h.reserved is not None else np.zeros(n, np.int64)

    out = dict(moves=[], over=[], R=[], step_us=[], arrivals=0, departures=0, dropped_arrivals=0,
               inst0_share=[], max_over_tokens=[])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(steps):
        R = req_id.shape[0]
        st.load_requests(torch.from_numpy(req_id.astype(np.int32)), torch.from_numpy(inst.astype(np.int32)),
                         torch.from_numpy(n_tok.astype(np.int32)), pinned=torch.from_numpy(pinned))
        scale = torch.from_numpy((np.maximum(rem, 1) / med).astype(np.float32)).to(dev)
        h = (h_base[torch.from_numpy(row % pool).to(dev)] * scale[:, None]).to(tdt)
        torch.cuda.synchronize()
        e0.record()
        st.run(h)
        e1.record()
        e1.synchronize()
        out["step_us"].append(e0.elapsed_time(e1) * 1e3)
        moves = st.result()
        L0 = st.v["L"][:, 0].cpu().numpy()
        if check is not None:
            check(k, dict(req_id=req_id, inst=inst, n_tok=n_tok, pinned=pinned, params=params_h), st)
        over = L0 + reserved > c_mem
        out["over"].append(int(over.sum()))
        out["max_over_tokens"].append(int(np.max(L0 + reserved - c_mem)))
        out["moves"].append(len(moves))
        out["R"].append(R)
        out["inst0_share"].append(float(np.mean(inst == 0)))
        # 1. apply the moves; the moved request is pinned (migrating) for the next round
        pinned[:] = 0
        pos = {int(r): i for i, r in enumerate(req_id)}
        for (rid, src, dst, _rnd, _gain) in moves:
            i = pos[int(rid)]
            assert inst[i] == src
            inst[i] = dst
            pinned[i] = 1
        # 2. decode tokens_per_step iterations (pinned requests are in flight and do not decode)
        adv = np.where(pinned == 1, 0, np.minimum(tokens_per_step, rem))
        n_tok += adv
        rem -= adv
        # 3. finished requests leave
        keep = rem > 0
        dep = int((~keep).sum())
        out["departures"] += dep
        req_id, inst, n_tok, rem, row, pinned = (a[keep] for a in (req_id, inst, n_tok, rem, row, pinned))
        # 4. skewed Poisson arrivals
        A = int(g.poisson(max(dep, 1)))
        A_ok = min(A, r_cap - req_id.shape[0])
        out["dropped_arrivals"] += A - A_ok
        if A_ok > 0:
            p, lout, _ = datagen.sample_lengths(g, A_ok)
            to0 = g.random(A_ok) < p_inst0
            dst = np.where(to0, 0, g.integers(0, n, A_ok))
            req_id = np.concatenate([req_id, np.arange(next_id, next_id + A_ok)])
            inst = np.concatenate([inst, dst])
            n_tok = np.concatenate([n_tok, p])
            rem = np.concatenate([rem, lout])
            row = np.concatenate([row, np.arange(next_row, next_row + A_ok)])
            pinned = np.concatenate([pinned, np.zeros(A_ok, np.uint8)])
            next_id += A_ok
            next_row += A_ok
            out["arrivals"] += A_ok
    pred.close()
    mv = np.array(out["moves"])
    return {"config": cfg, "steps": steps, "tokens_per_step": tokens_per_step, "p_inst0": p_inst0,
            "moves_per_step": float(mv.mean()), "steps_with_moves": int((mv > 0).sum()),
            "total_moves": int(mv.sum()), "steps_over_c_mem": int(np.sum(np.array(out["over"]) > 0)),
            "instance_steps_over_c_mem": int(np.sum(out["over"])),
            "over_c_mem_first_last": [out["over"][0], out["over"][-1]],
            "R_min_max": [int(min(out["R"])), int(max(out["R"]))], "arrivals": out["arrivals"],
            "departures": out["departures"], "dropped_arrivals": out["dropped_arrivals"],
            "inst0_share_first_last": [round(out["inst0_share"][0], 4), round(out["inst0_share"][-1], 4)],
            "step_us_eager_median": round(float(np.median(out["step_us"])), 2),
            "note": "one Alg. 1 round per scheduling interval (PAPER.md:411, ~50 decode iterations); eager "
                    "steps (the batch changes every step), host harness between steps not timed"}
