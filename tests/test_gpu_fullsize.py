"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times, on sampled outputs:

* c3 -- E-Forest at d = 960 (N = 10^6, Q = 10^3, T = 2, top-100): oracle
  codebooks (shortened training) and codes; 24 sampled queries against the oracle's exact top-k.
* c5 -- E-Forest at N = 10^8 (T = 2 over bytes 0-3 | 4-7, Q = 10^4, top-100):
  the oracle cannot encode 10^8 vectors in test time, so the codes come from
  et_encode (reading C4b in DESIGN.md §3) -- pinned here against the oracle's
  encode on four random 65,536-vector blocks -- and the oracle computes the
  exact top-k over all 10^8 codes for three sampled queries; every query's
  returned pairs and a 4096-code sample bound against ADC64.

Slow (minutes): generation of the 10^8 base vectors dominates.
"""
import os
import sys

import numpy as np
import pytest

from oracle import pq
from oracle import topk as otopk
from paper_1509_05186_b200 import api, build, synth

from gpu_common import RTOL, check_topk, pq_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build.build()
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    api._lib.load()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_c3_full_size_topk_sampled():
    # (the oracle's k-means on 20,000 training vectors x 10 Lloyd iterations: the
    # full 100,000 x 25 training is 4 of this test's 5 minutes and changes
    # neither the shapes nor the launch configuration)
    cfg, cb, codes, qx, X = pq_inputs("c3", n_train=20_000, iters=10)
    assert (cfg.N, cfg.Q, cfg.d, cfg.M) == (1_000_000, 1_000, 960, 16)
    ix = api.Index.et_build_eforest(codes, split=list(cfg.forest_split))
    d, i = ix.et_etree_topk(cfg.topk, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    sample = sorted(set([0, cfg.Q - 1] + rng.choice(cfg.Q, 22, replace=False).tolist()))
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, cfg.topk, sample)


def _adc64_chunked(cb, qrow, codes, chunk=1 << 24):
    """Oracle ADC64 of one query to every code, in chunks (10^8 codes)."""
    table = pq.lut64(cb, qrow[None, :])
    out = np.empty(len(codes), dtype=np.float64)
    for s in range(0, len(codes), chunk):
        out[s:s + chunk] = pq.adc(table, codes[s:s + chunk])[0]
    return out


@pytest.fixture(scope="module")
def c5_full():
    cfg = synth.CONFIGS["c5"]
    means = synth.mixture_means(cfg)
    cb, _ = pq.train_pq(synth.train(cfg, means=means), cfg.M, cfg.K, cfg.lloyd_iters,
                        synth.kmeanspp_seed(cfg))
    sys.path.insert(0, ROOT)
    import bench   # the bench's generator + et_encode pipeline (process pool)
    codes, _ = bench.gen_encode_range(cfg, {}, bench.CudaBackend(torch.device("cuda", 0)), cb, means, 0, cfg.N)
    qx = synth.queries(cfg, means=means)
    return cfg, cb, codes, qx, means


def test_c5_encode_matches_oracle_on_sampled_blocks(c5_full):
    cfg, cb, codes, qx, means = c5_full
    rng = np.random.default_rng(5)
    nblk = cfg.N // synth.BLOCK
    s = cfg.d // cfg.M
    for b in rng.choice(nblk, 4, replace=False):
        X = synth.base(cfg, int(b) * synth.BLOCK, synth.BLOCK, means=means)
        ref = pq.encode(cb, X)
        got = codes[int(b) * synth.BLOCK:(int(b) + 1) * synth.BLOCK]
        diff = np.argwhere(got != ref)
        for (r, m) in diff:   # only near ties may differ
            dd = pq.sqdist_direct(X[r:r + 1, m * s:(m + 1) * s], cb[m])[0]
            a, c = dd[got[r, m]], dd[ref[r, m]]
            assert abs(a - c) <= 1e-5 * max(a, c)
        assert len(diff) <= 64


def test_c5_full_size_topk_sampled(c5_full):
    cfg, cb, codes, qx, means = c5_full
    ix = api.Index.et_build_eforest(codes, split=list(cfg.forest_split))
    d, i = ix.et_etree_topk(cfg.topk, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    gd, gi = d.cpu().numpy(), i.cpu().numpy()
    assert np.all(np.diff(gd.astype(np.float64), axis=1) >= 0)
    assert gi.min() >= 0 and gi.max() < cfg.N
    ids_all = np.arange(cfg.N)
    for q in (0, 4321, cfg.Q - 1):
        full = _adc64_chunked(cb, qx[q], codes)
        # the oracle's full-sort top-k on the ids whose distance is <= the k-th
        # smallest (np.partition, exact): a superset of the top-k incl. ties
        kth = np.partition(full, cfg.topk - 1)[cfg.topk - 1]
        sel = np.flatnonzero(full <= kth)
        od, oi = otopk.topk(full[sel][None, :], ids_all[sel], cfg.topk)
        od, oi = od[0], oi[0]
        g_d = gd[q].astype(np.float64)
        g_i = gi[q].astype(np.int64)
        assert len(np.unique(g_i)) == cfg.topk
        truth = full[g_i]
        assert np.all(np.abs(g_d - truth) <= RTOL * np.maximum(truth, 1e-30)), q
        assert np.all(np.abs(g_d - od) <= RTOL * np.maximum(od, 1e-30)), q
        mism = g_i != oi
        if mism.any():
            assert np.all(np.abs(truth[mism] - od[mism]) <= RTOL * od[mism]), q
    # every query (properties that hold at any size): each returned distance is
    # the oracle's ADC64 of (query, codes[returned id]), ids are distinct, and
    # no code of a random 4096-code sample beats the k-th returned distance
    # unless it is in the list (it would belong to the exact top-k).
    table = pq.lut64(cb, qx)
    rng = np.random.default_rng(55)
    samp = np.sort(rng.choice(cfg.N, 4096, replace=False))
    dsamp = pq.adc(table, codes[samp])                      # [Q, 4096] fp64
    for q in range(cfg.Q):
        g_i = gi[q].astype(np.int64)
        assert len(np.unique(g_i)) == cfg.topk, q
        truth = pq.adc(table[q:q + 1], codes[g_i])[0]
        g_d = gd[q].astype(np.float64)
        assert np.all(np.abs(g_d - truth) <= RTOL * np.maximum(truth, 1e-30)), q
        better = samp[dsamp[q] < g_d[-1] * (1 - RTOL)]
        assert np.isin(better, g_i).all(), q


# --------------------------------------------------------------------------- c4 at full size

@pytest.fixture(scope="module")
def c4_full():
    """BASELINE config 4 at full size: coarse quantizer (K' = 1024) and the
    residual codebook trained by the ORACLE (k-means++ + 25 Lloyd); the 10^7
    base vectors assigned and encoded by et_assign / et_encode (reading C4b:
    the oracle cannot encode 10^7 x 1024 in test time) -- pinned below on
    sampled blocks against oracle assign + encode."""
    cfg = synth.CONFIGS["c4"]
    means = synth.mixture_means(cfg)
    coarse, _ = pq.kmeans(synth.coarse_train(cfg, means=means), cfg.ivf_nlist, cfg.lloyd_iters,
                          synth.kmeanspp_seed(cfg, 1))
    coarse = coarse.astype(np.float32)
    rt = synth.resid_train(cfg, means=means)
    a = pq.assign(rt, coarse)
    cb, _ = pq.train_pq((rt.astype(np.float64) - coarse[a]).astype(np.float32), cfg.M, cfg.K, cfg.lloyd_iters,
                        synth.kmeanspp_seed(cfg, 2))
    cd, cbd = dev(coarse), dev(cb)
    codes = np.empty((cfg.N, cfg.M), np.uint8)
    cells = np.empty(cfg.N, np.int32)
    sys.path.insert(0, ROOT)
    import bench
    import multiprocessing as mp
    jobs = [("c4", {}, s, min(1 << 18, cfg.N - s)) for s in range(0, cfg.N, 1 << 18)]
    with mp.get_context("spawn").Pool(max(1, min(32, (os.cpu_count() or 2) - 1)), initializer=bench._gen_init,
                                      initargs=("c4", {})) as pool:
        for s, x in pool.imap(bench._gen_chunk, jobs, chunksize=1):
            xd = dev(x)
            asg = api.et_assign(cd, xd)
            codes[s:s + len(x)] = api.et_encode(cbd, xd, centroids=cd, assign=asg).cpu().numpy()
            cells[s:s + len(x)] = asg.cpu().numpy()
    return cfg, coarse, cb, codes, cells, synth.queries(cfg, means=means), means


def test_c4_assign_encode_match_oracle_on_sampled_blocks(c4_full):
    cfg, coarse, cb, codes, cells, qx, means = c4_full
    rng = np.random.default_rng(4)
    s = cfg.d // cfg.M
    for b in rng.choice(cfg.N // synth.BLOCK, 2, replace=False):
        lo = int(b) * synth.BLOCK
        X = synth.base(cfg, lo, synth.BLOCK, means=means)
        oa = pq.assign(X, coarse)
        diff = np.flatnonzero(oa != cells[lo:lo + synth.BLOCK])
        for r in diff:   # coarse near ties only
            dd = pq.sqdist_direct(X[r:r + 1], coarse)[0]
            x1, x2 = dd[oa[r]], dd[cells[lo + r]]
            assert abs(x1 - x2) <= 1e-5 * max(x1, x2)
        R = X.astype(np.float64) - coarse[cells[lo:lo + synth.BLOCK]].astype(np.float64)
        ref = pq.encode(cb, R)
        got = codes[lo:lo + synth.BLOCK]
        bad = np.argwhere(got != ref)
        for (r, m) in bad:
            dd = pq.sqdist_direct(R[r:r + 1, m * s:(m + 1) * s], cb[m])[0]
            x1, x2 = dd[got[r, m]], dd[ref[r, m]]
            assert abs(x1 - x2) <= 1e-5 * max(x1, x2)
        assert len(diff) <= 64 and len(bad) <= 64


def test_c4_full_size_ivf_topk_sampled(c4_full):
    """N = 10^7, K' = 1024, w = 8, Q = 10^4, top-100 in the launch bench.py
    times; 24 sampled queries vs the oracle's probe (fp64) and exact residual
    ADC64 top-k over the probed lists (C6 near-tie rule for the probes)."""
    from oracle import ivf as oivf
    cfg, coarse, cb, codes, cells, qx, means = c4_full
    ix = api.Index.et_build_ivf(codes, cells, coarse, cb)
    d, i, pr = ix.et_ivf_topk(dev(qx), nprobe=cfg.ivf_nprobe, k=cfg.topk, return_probes=True)
    torch.cuda.synchronize()
    d, i, pr = d.cpu().numpy(), i.cpu().numpy(), pr.cpu().numpy()
    order = np.argsort(cells, kind="stable")
    starts = np.searchsorted(cells[order], np.arange(cfg.ivf_nlist + 1))
    rng = np.random.default_rng(44)
    sample = sorted(set([0, cfg.Q - 1] + rng.choice(cfg.Q, 22, replace=False).tolist()))
    oprobe = oivf.probe(qx[sample], coarse, cfg.ivf_nprobe)
    for j, q in enumerate(sample):
        if not np.array_equal(np.sort(pr[q]), np.sort(oprobe[j])):
            cd = pq.sqdist_direct(qx[q:q + 1], coarse)[0]
            kth = np.sort(cd)[cfg.ivf_nprobe - 1]
            for c in set(pr[q]) ^ set(oprobe[j]):
                assert abs(cd[c] - kth) <= 1e-5 * kth, (q, c)
        members, dists = [], []
        for c in pr[q]:
            m = order[starts[c]:starts[c + 1]]
            if len(m):
                r = qx[q].astype(np.float64) - coarse[c].astype(np.float64)
                dists.append(pq.adc(pq.lut64(cb, r[None]), codes[m])[0])
                members.append(m)
        full, ids = np.concatenate(dists), np.concatenate(members)
        od, oi = otopk.topk(full[None], ids, cfg.topk)
        od, oi = od[0], oi[0]
        nv = int((oi >= 0).sum())
        g_d, g_i = d[q].astype(np.float64), i[q].astype(np.int64)
        assert int((g_i >= 0).sum()) == nv and len(np.unique(g_i[:nv])) == nv
        pos = {int(x): t for t, x in enumerate(ids)}
        truth = full[[pos[int(x)] for x in g_i[:nv]]]
        assert np.all(np.abs(g_d[:nv] - truth) <= RTOL * np.maximum(truth, 1e-30)), q
        assert np.all(np.abs(g_d[:nv] - od[:nv]) <= RTOL * np.maximum(od[:nv], 1e-30)), q
        mism = g_i[:nv] != oi[:nv]
        if mism.any():
            assert np.all(np.abs(truth[mism] - od[:nv][mism]) <= RTOL * od[:nv][mism]), q
