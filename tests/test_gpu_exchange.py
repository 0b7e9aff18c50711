"""Exchange readiness on one GPU (`-m gpu`): the W > 1 code path of Step -- predictor + fused
projection, the NCCL all-gather of the per-rank records ("collect states"),
then plan_reschedule_segmented on the gathered buffer -- driven over a world-size-1 NCCL
process group, eagerly on a NON-current stream and captured in a CUDA graph next to the
PDL-launched kernels.  Checked bit for bit against the oracle."""
import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def star():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2510_13668_b200 as star
    star.version()
    return star


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    assert not dist.is_initialized()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1, device_id=dev)
    yield dist.group.WORLD
    dist.destroy_process_group()


def _dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return (t.to(dtype) if dtype is not None else t).cuda()


@pytest.mark.parametrize("cfg,r_per,seed,refresh", [("TGT", 128, 0, None), ("C4", 200, 1, None),
                                                    ("TGT", 64, 2, 20)])
def test_step_nccl_world1_exchange(star, oracle_mod, nccl_world1, cfg, r_per, seed, refresh):
    from paper_2510_13668_b200.step import Step
    c = datagen.CONFIGS[cfg]
    n = c["n_inst"]
    snap = datagen.make_snapshot(seed, n, r_per, skewed=c.get("skewed", False), pinned_frac=0.05)
    R = snap.R
    pw = datagen.make_predictor_weights(seed, c["d"], c["dtype"])
    scale = np.maximum(snap.true_rem, 1).astype(np.float32) / 60.0
    h = _dev(datagen.make_hidden(seed, R, c["d"], c["dtype"], scale=scale), torch.bfloat16)
    W = [_dev(pw.W1, torch.bfloat16), _dev(pw.W2, torch.bfloat16), _dev(pw.W3, torch.bfloat16), _dev(pw.w4)]
    pred = star.Predictor(*W, max_rows=R)
    params_h = datagen.make_plan_params(snap, H=50, mem_factor=c.get("mem_factor", 1.10),
                                        max_moves=max(c["max_moves"], 2))
    params = star.PlanParams.from_host(params_h)
    st = Step(pred, params, n, r_cap=R, world=1, group=nccl_world1, force_collective=True, refresh_k=refresh)
    assert st.recv.data_ptr() != st.send.data_ptr()   # a real gathered buffer, filled by NCCL
    st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in (snap.req_id, snap.inst, snap.n_tok)),
                     pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned)))

    def check():
        nh = st.v["n_hat"][:R].cpu().numpy()
        ref_p = oracle_mod.project(snap.inst, snap.n_tok, nh, n, 50, params_h.beta_q)
        assert st.err.item() == 0
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"])
        # the plan ran on the all-gathered copy of the record
        assert torch.equal(st.recv, st.send)
        ref = oracle_mod.plan(params_h, ref_p["L"], snap.req_id, snap.inst, snap.n_tok, nh, snap.pinned)
        assert st.result() == ref
        return ref

    # eager, on a side stream that is NOT torch's current stream (the all-gather must be ordered
    # on it: it reads the record the predictor just wrote, the plan reads what it delivered)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    st.recv.zero_()
    st.run(h, stream=s)
    s.synchronize()
    ref = check()
    if refresh is None:
        assert len(ref) >= 1   # skewed snapshot: Phases 2-3 reached
    # captured in one CUDA graph (kernels + the NCCL collective), replayed from a cleared state
    if refresh is not None:
        st.load_requests(*(torch.from_numpy(np.ascontiguousarray(a)) for a in (snap.req_id, snap.inst,
                                                                                 snap.n_tok)),
                         pinned=torch.from_numpy(np.ascontiguousarray(snap.pinned)))
    st.capture(h)
    for _ in range(2):
        st.recv.zero_()
        st.moves.zero_()
        st.n_moves.zero_()
        if refresh is not None:   # every row due again: the refreshed N_hat must equal the first pass
            st.g_last.fill_(-1)
        st.replay()
        torch.cuda.synchronize()
        assert check() == ref
    pred.close()
