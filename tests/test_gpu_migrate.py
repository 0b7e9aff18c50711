"""KV migration (NEXT-4: ExecuteMigration's paged-KV copy) through the C
ABI on one GPU -- source and destination pools on the same device -- byte-exact against the
oracle (`-m gpu`)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def star():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2510_13668_b200 as star
    star.version()
    return star


def _pool(g, layers, blocks, bb):
    return g.integers(0, 256, (layers, blocks, bb), dtype=np.uint8)


@pytest.mark.parametrize("layers,blocks,bb,n,seed", [(1, 4, 16, 1, 0), (2, 16, 48, 7, 1), (32, 64, 1024, 33, 2),
                                                     (4, 300, 65536, 97, 3), (3, 9, 8208, 9, 4), (5, 20, 256, 0, 5),
                                                     (32, 40, 65536, 40, 6)])
def test_kv_pack_unpack_migrate_bitexact(star, oracle_mod, layers, blocks, bb, n, seed):
    g = np.random.default_rng(seed)
    src = _pool(g, layers, blocks, bb)
    dst = _pool(g, layers, blocks, bb)
    st_tab = g.permutation(blocks)[:n].astype(np.int32)     # fragmented source blocks
    dt_tab = g.permutation(blocks)[:n].astype(np.int32)     # blocks the destination allocated
    src_d, dst_d = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    st_d, dt_d = torch.from_numpy(st_tab).cuda(), torch.from_numpy(dt_tab).cuda()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    stg = star.kv_pack(src_d, st_d, err_flag=err)
    torch.cuda.synchronize()
    ref_stg = oracle_mod.kv_pack(src, st_tab)
    assert np.array_equal(stg.cpu().numpy(), ref_stg)
    d1 = dst_d.clone()
    star.kv_unpack(stg, d1, dt_d, err_flag=err)
    d2 = dst_d.clone()
    star.kv_migrate(src_d, st_d, d2, dt_d, err_flag=err)
    torch.cuda.synchronize()
    ref = oracle_mod.kv_migrate(src, st_tab, dst, dt_tab)
    assert np.array_equal(d1.cpu().numpy(), ref)
    assert np.array_equal(d2.cpu().numpy(), oracle_mod.kv_unpack(ref_stg, dst, dt_tab))
    assert np.array_equal(d2.cpu().numpy(), ref)
    assert err.item() == 0


def test_kv_strided_layers_and_bad_block(star, oracle_mod):
    """Layers as a strided view into a larger allocation (per-layer pools of one engine); a block
    id outside the pool sets STAR_ERRF_BLOCK and only that copy is skipped."""
    g = np.random.default_rng(7)
    big = _pool(g, 6, 50, 512)
    src = big[::2, 5:45]                                     # 3 layers, 40 blocks, stride 2 layers
    big_d = torch.from_numpy(big).cuda()
    src_d = big_d[::2, 5:45]
    tab = np.array([39, 0, 17, 40, 3], np.int32)             # 40 is outside the 40-block pool
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    stg = torch.zeros((3, 5, 512), dtype=torch.uint8, device="cuda")
    star.kv_pack(src_d, torch.from_numpy(tab).cuda(), staging=stg, err_flag=err)
    torch.cuda.synchronize()
    assert err.item() == 4
    ok = [0, 1, 2, 4]
    ref = oracle_mod.kv_pack(np.ascontiguousarray(src), tab[ok])
    got = stg.cpu().numpy()
    assert np.array_equal(got[:, ok], ref)
    assert not got[:, 3].any()


def test_kv_host_validation(star):
    pool = torch.zeros((2, 4, 24), dtype=torch.uint8, device="cuda")   # block_bytes not a multiple of 16
    with pytest.raises(star.StarError):
        star.kv_pack(pool, torch.zeros(1, dtype=torch.int32, device="cuda"))
