"""C4 episode (BASELINE.json configs[3]) on the GPU path, every step checked
against the oracle: the fused projection of the GPU's own N_hat == oracle.project, and the
plan == oracle.plan on that state, bit for bit, while moves are applied, requests finish and
skewed arrivals land between steps (`-m gpu`)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_c4_episode_steps_equal_oracle(oracle_mod):
    import episode
    import paper_2510_13668_b200 as star
    from paper_2510_13668_b200.step import Step
    seen = []

    def check(k, s, st):
        R = s["req_id"].shape[0]
        nh = st.v["n_hat"][:R].cpu().numpy()
        p = s["params"]
        ref_p = oracle_mod.project(s["inst"], s["n_tok"], nh, p.n_inst, p.H, p.beta_q)
        assert np.array_equal(st.v["L"].cpu().numpy(), ref_p["L"]), k
        ref = oracle_mod.plan(p, ref_p["L"], s["req_id"], s["inst"], s["n_tok"], nh, s["pinned"])
        assert st.result() == ref, k
        seen.append(len(ref))

    res = episode.run_episode(star, Step, steps=10, check=check, tokens_per_step=200)
    assert len(seen) == 10
    assert res["total_moves"] >= 1 and res["arrivals"] > 0 and res["departures"] > 0
