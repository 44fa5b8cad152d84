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


def _bench_dry(config, gpus, n=20_000, q=6):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    for v in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(v, None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", str(gpus), "--config", config,
                        "--dry-run", "bench_dry_backend:Backend", "--dry-n", str(n), "--dry-q", str(q)],
                       capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("config,mode", [("c5", "db"), ("c4", "lists")])
def test_bench_dry_run_two_ranks_equals_oracle_global_topk(config, mode):
    """bench.py --gpus 2 (self-launched under torchrun, gloo): each rank
    generates half the base, the rows are exchanged by first byte (db) or by
    list owner (lists), per-shard top-k lists are all-gathered and merged --
    and the merged lists equal the oracle's global top-k on the whole base."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from bench_dry_backend import Backend
    from paper_1509_05186_b200 import synth
    out2 = _bench_dry(config, 2)
    assert out2["world"] == 2 and out2["mode"] == mode
    # the single-process reference: the same recipe on one rank (no sharding)
    be = Backend()
    over = dict(N=20_000, Q=6, n_train=2000, lloyd_iters=3)
    cfg = synth.scaled(synth.CONFIGS[config], **over)
    if cfg.ivf_nlist:
        cfg = synth.scaled(cfg, ivf_nlist=16, n_coarse_train=2000)
    means = synth.mixture_means(cfg)
    st = {"qx": synth.queries(cfg, means=means), "ids": np.arange(cfg.N)}
    if cfg.ivf_nlist:
        co = be.train_coarse(synth.coarse_train(cfg, means=means), cfg.ivf_nlist, cfg.lloyd_iters,
                             synth.kmeanspp_seed(cfg, 1))
        rt = synth.resid_train(cfg, means=means)
        a = be.assign(co, rt)
        cb = be.train_codebooks((rt - co[a]).astype(np.float32), cfg.M, cfg.K, cfg.lloyd_iters,
                                synth.kmeanspp_seed(cfg, 2))
        st["codes"], st["cells"] = be.encode(cb, synth.base(cfg, means=means), co)
        st["coarse"] = co
    else:
        cb = be.train_codebooks(synth.train(cfg, means=means), cfg.M, cfg.K, cfg.lloyd_iters,
                                synth.kmeanspp_seed(cfg))
        st["codes"], _ = be.encode(cb, synth.base(cfg, means=means))
    st["cb"] = cb
    D, I = be.topk(cfg, st)
    assert out2["n_local"] < cfg.N
    assert np.array_equal(np.array(out2["ids"]), I)
    assert np.array_equal(np.array(out2["dist"]), D)
