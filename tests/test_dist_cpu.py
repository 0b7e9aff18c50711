"""Multi-process host logic of the distributed step (CPU, gloo, world size 2 and 4).

Every rank packs its own decode instances' state into the fixed-size exchange record
(step.RecordLayout), the records are all-gathered with step.exchange (the same call that runs
over NCCL on the GPU box), and every rank decodes the gathered bytes back into the
concatenated cluster state.  The oracle plan on that state must equal the oracle plan on the
undivided snapshot and be byte-identical on every rank (hash all-gather).
The projection here is the oracle's (the CUDA kernels need a GPU); the GPU test
test_plan_segmented_equals_contiguous covers the kernel reading the same layout in place."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_inst, r_per, seed, q):
    import oracle
    from paper_2510_13668_b200.step import RecordLayout, exchange, split_snapshot_by_rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        snap = datagen.make_snapshot(seed, n_inst, r_per, pinned_frac=0.05)
        params = datagen.make_plan_params(snap, max_moves=3, reserved_seed=seed)
        n_hat = snap.true_rem.astype(np.int32)
        H, n_loc = params.H, n_inst // world
        idx = split_snapshot_by_rank(snap.inst, n_inst, world, rank)
        r_cap = r_per * n_loc + 3
        lay = RecordLayout(n_loc, H, r_cap)
        send = torch.zeros(lay.nbytes, dtype=torch.uint8)
        v = lay.views(send)
        R = len(idx)
        proj = oracle.project(snap.inst[idx], snap.n_tok[idx], n_hat[idx], n_loc, H, params.beta_q,
                              inst_base=rank * n_loc)
        v["L"].copy_(torch.from_numpy(proj["L"]))
        v["W"].copy_(torch.from_numpy(proj["W"]))
        v["count"].fill_(R)
        for name, arr in (("req_id", snap.req_id), ("inst", snap.inst), ("n_tok", snap.n_tok), ("n_hat", n_hat)):
            v[name][:R].copy_(torch.from_numpy(np.ascontiguousarray(arr[idx])))
        v["pinned"][:R].copy_(torch.from_numpy(np.ascontiguousarray(snap.pinned[idx])))
        recv = torch.zeros(world * lay.nbytes, dtype=torch.uint8)
        exchange(send, recv)
        # decode the gathered records into the concatenated state
        Ls, cols = [], {k: [] for k in ("req_id", "inst", "n_tok", "n_hat", "pinned")}
        for k in range(world):
            g = lay.views(recv[k * lay.nbytes:(k + 1) * lay.nbytes])
            cnt = int(g["count"].item())
            Ls.append(g["L"].numpy().copy())
            for name in cols:
                cols[name].append(g[name][:cnt].numpy().copy())
        L = np.concatenate(Ls, 0)
        st = {k: np.concatenate(v_) for k, v_ in cols.items()}
        plan = oracle.plan(params, L, st["req_id"], st["inst"], st["n_tok"], st["n_hat"], st["pinned"])
        # whole-cluster references (on the undivided snapshot)
        L_ref = oracle.project(snap.inst, snap.n_tok, n_hat, n_inst, H, params.beta_q)["L"]
        order = np.argsort(snap.inst, kind="stable")
        ref = oracle.plan(params, L_ref, *(a[order] for a in (snap.req_id, snap.inst, snap.n_tok, n_hat)),
                          snap.pinned[order])
        h = hashlib.sha256(repr(plan).encode()).digest()[:8]
        ht = torch.frombuffer(bytearray(h), dtype=torch.uint8)
        hs = [torch.zeros(8, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(hs, ht)
        q.put((rank, np.array_equal(L, L_ref), plan == ref, all(torch.equal(x, hs[0]) for x in hs), len(plan)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_inst,r_per,seed", [(2, 8, 40, 0), (2, 2, 64, 1), (4, 8, 24, 2)])
def test_gathered_records_give_the_cluster_plan(world, n_inst, r_per, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_inst, r_per, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert any(r[4] > 0 for r in res) or seed == 1, "fixture should produce moves"
    for rank, loads_ok, plan_ok, hash_ok, nmoves in res:
        assert loads_ok, f"rank {rank}: gathered loads != cluster projection"
        assert plan_ok, f"rank {rank}: plan on gathered records != cluster plan"
        assert hash_ok, f"rank {rank}: plans differ across ranks"


def test_step_gathered_buffer_layout():
    """Step(gathered=...) (one rank of a W-rank job measured on one GPU): rank k's record is a
    view of slot k of the caller's gathered buffer -- exactly where the all-gather would put it --
    so load_requests writes the bytes the exchange would deliver; a wrong-sized buffer is rejected."""
    from paper_2510_13668_b200.step import RecordLayout, Step

    class _P:   # the layout needs H / max_moves / beta_q only
        pass
    snap = datagen.make_snapshot(4, 8, 16)
    params_h = datagen.make_plan_params(snap)
    pp = _P()
    pp.H, pp.max_moves = params_h.H, 1
    pp.beta_q = torch.zeros(params_h.H + 1, dtype=torch.int32)
    world, r_cap = 8, 32
    lay = RecordLayout(1, params_h.H, r_cap)
    buf = torch.zeros(world * lay.nbytes, dtype=torch.uint8)
    cpu = torch.device("cpu")
    for k in range(world):
        st = Step(None, pp, 8, r_cap=r_cap, rank=k, world=world, device=cpu, gathered=buf)
        assert st.recv is buf and st.send.data_ptr() == buf.data_ptr() + k * lay.nbytes
        idx = np.nonzero(snap.inst == k)[0]
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a[idx])) for a in (snap.req_id, snap.inst,
                                                                                      snap.n_tok)))
    # the gathered buffer now decodes to every rank's requests in rank order
    for k in range(world):
        v = lay.views(buf[k * lay.nbytes:(k + 1) * lay.nbytes])
        idx = np.nonzero(snap.inst == k)[0]
        assert int(v["count"].item()) == len(idx)
        assert np.array_equal(v["req_id"][:len(idx)].numpy(), snap.req_id[idx])
        assert np.array_equal(v["inst"][:len(idx)].numpy(), snap.inst[idx])
    with pytest.raises(ValueError):
        Step(None, pp, 8, r_cap=r_cap, rank=0, world=world, device=cpu, gathered=buf[:-1])
