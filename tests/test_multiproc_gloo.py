"""world_size-2 (and 3) gloo tests of the N>1 host path on CPU: shard
partitioning by first-level subtree, per-shard index build (host C++), the
all-gather of per-shard top-k lists, and the merge -- checked against the
unsharded oracle result.  (The per-shard scan and the merge kernel are GPU
code; here the per-shard lists come from the oracle, and the merged result
must equal the single-index top-k.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import pq, topk
    from paper_1509_05186_b200 import api, shard, synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, M, K, s, Q, k = 20_000, 8, 32, 4, 12, 50
    codes = synth.random_codes(31, N, M, K, n_distinct=3000)
    cb = synth.random_floats(32, (M, K, s), 0, 5)
    qx = synth.random_floats(33, (Q, M * s), 0, 5)
    mine, ids = shard.shard_select(codes, rank, world, K)
    # host-side build of this rank's index (no GPU): leaves never cross shards
    st = api.et_build_stats(mine, ids=ids, K=K)[0] if len(mine) else {"L1": 0, "L2": 0, "N": 0}
    table = pq.lut64(cb, qx)
    D, I = topk.topk(pq.adc(table, mine), ids, k)
    gd, gi = shard.gather_lists(torch.from_numpy(D), torch.from_numpy(I))
    t = torch.tensor([st["L1"], st["L2"], st["N"]], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        mD, mI = topk.merge(list(gd.numpy()), list(gi.numpy()), k)
        gD, gI = topk.topk(pq.adc(table, codes), np.arange(N), k)
        glob = api.et_build_stats(codes, K=K)[0]
        np.save(os.path.join(outdir, "ok.npy"), np.array([
            np.array_equal(mI, gI), np.array_equal(mD, gD),
            int(t[0]) == glob["L1"], int(t[1]) == glob["L2"], int(t[2]) == N]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_topk_over_gloo(tmp_path, world):
    from paper_1509_05186_b200 import build
    build.build()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    ok = np.load(tmp_path / "ok.npy")
    assert ok.all(), ok.tolist()


def test_shard_bounds_match_oracle_rule():
    """The product's C++ cut (et_shard_bounds) against the oracle's rule as
    written (a plain loop over byte values), incl. skewed and empty shards."""
    from oracle import shard as oshard
    from paper_1509_05186_b200 import api, build, synth
    build.build()
    for G in (1, 2, 3, 4, 8):
        for codes in (synth.random_codes(40 + G, 3000, 2, 256),
                      synth.random_codes(50 + G, 700, 3, 16),
                      np.repeat(synth.random_codes(60 + G, 3, 2, 256), 200, axis=0)):   # 3 first bytes
            K = 16 if codes.max() < 16 else 256
            got = api.et_shard_bounds(codes, G, K)
            assert np.array_equal(got, oshard.shard_bounds(codes[:, 0], G, K)), (G, K)


def test_ivf_list_shard_plan_is_a_balanced_partition():
    """LPT plan (et_shard_lists): every list owned by exactly one rank; the
    load spread is at most the largest list (the greedy bound)."""
    from paper_1509_05186_b200 import api, build
    build.build()
    r = np.random.default_rng(9)
    for G in (1, 2, 3, 8):
        sizes = r.integers(0, 40000, size=1024)
        sizes[:4] = 0
        owner = api.et_shard_lists(sizes, G)
        assert owner.min() >= 0 and owner.max() < G
        load = np.bincount(owner, weights=sizes, minlength=G)
        assert load.sum() == sizes.sum()
        assert load.max() - load.min() <= sizes.max()
