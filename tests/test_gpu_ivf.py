"""GPU parity for the IVF application: probe + residual tables +
per-list E-Tree scan + fused top-k, against oracle/ivf.py."""
import numpy as np
import pytest

from oracle import etree as oetree
from oracle import ivf as oivf
from oracle import pq
from paper_1509_05186_b200 import api, build, synth

from gpu_common import RTOL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build.build()
    assert torch.cuda.is_available()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def c4s():
    # BASELINE config 4's generator (integer mixture, d=128, M=8, K=256), scaled:
    # N=2e5, K'=64 lists, 64 queries.
    cfg = synth.scaled(synth.CONFIGS["c4"], N=200_000, Q=64, n_train=20_000, n_coarse_train=20_000,
                       ivf_nlist=64, lloyd_iters=8)
    means = synth.mixture_means(cfg)
    coarse, _ = pq.kmeans(synth.coarse_train(cfg, means=means), cfg.ivf_nlist, 8, synth.kmeanspp_seed(cfg, 1))
    rt = synth.resid_train(cfg, means=means)
    a = pq.assign(rt, coarse)
    R = (rt.astype(np.float64) - coarse[a]).astype(np.float32)
    cb, _ = pq.train_pq(R, cfg.M, cfg.K, cfg.lloyd_iters, synth.kmeanspp_seed(cfg, 2))
    index = oivf.encode_ivf(synth.base(cfg, means=means), coarse.astype(np.float32), cb)
    return cfg, index, synth.queries(cfg, means=means)


def _truth(index, q, ids):
    out = np.empty(len(ids))
    for j, i in enumerate(ids):
        r = q.astype(np.float64) - index.coarse[index.assign[i]].astype(np.float64)
        out[j] = pq.adc(pq.lut64(index.codebooks, r[None]), index.codes[i:i + 1])[0, 0]
    return out


@pytest.mark.parametrize("w,k", [(8, 100), (1, 10), (64, 50)])
def test_ivf_topk_vs_oracle(c4s, w, k):
    cfg, index, qx = c4s
    ix = api.Index.et_build_ivf(index.codes, index.assign.astype(np.int32), index.coarse, index.codebooks)
    st = ix.et_index_stats(0)
    L1 = L2 = 0
    for m in index.lists:
        if len(m):
            s = oetree.tree_stats_def(oetree.sort_codes(index.codes[m])[0])
            L1 += s.L1
            L2 += s.L2
    assert (st["L1"], st["L2"]) == (L1, L2)
    d, i, pr = ix.et_ivf_topk(dev(qx), nprobe=w, k=k, return_probes=True)
    torch.cuda.synchronize()
    d, i, pr = d.cpu().numpy(), i.cpu().numpy(), pr.cpu().numpy()
    oprobe = oivf.probe(qx, index.coarse, w)
    cd = pq.sqdist_direct(qx, index.coarse)
    for q in range(cfg.Q):
        if not np.array_equal(np.sort(pr[q]), np.sort(oprobe[q])):   # C6: only near ties may swap
            a = set(pr[q]) ^ set(oprobe[q])
            kth = np.sort(cd[q])[w - 1]
            for c in a:
                assert abs(cd[q, c] - kth) <= 1e-5 * kth
    D, I, _ = oivf.search(index, qx, w, k, probes=pr)
    for q in range(cfg.Q):
        nv = int((I[q] >= 0).sum())
        assert int((i[q] >= 0).sum()) == nv
        g = i[q][:nv]
        assert len(np.unique(g)) == nv
        tg = _truth(index, qx[q], g)
        assert np.all(np.abs(d[q][:nv] - tg) <= RTOL * np.maximum(tg, 1e-30))
        assert np.all(np.abs(d[q][:nv] - D[q][:nv]) <= RTOL * np.maximum(D[q][:nv], 1e-30))
        mism = g != I[q][:nv]
        if mism.any():
            assert np.all(np.abs(tg[mism] - D[q][:nv][mism]) <= RTOL * D[q][:nv][mism])


def test_ivf_full_probe_equals_exhaustive(c4s):
    """w = K': the IVF search equals exhaustive residual ADC."""
    cfg, index, qx = c4s
    ix = api.Index.et_build_ivf(index.codes, index.assign.astype(np.int32), index.coarse, index.codebooks)
    d, i = ix.et_ivf_topk(dev(qx[:8]), nprobe=cfg.ivf_nlist, k=20)
    torch.cuda.synchronize()
    D, I, _ = oivf.search(index, qx[:8], cfg.ivf_nlist, 20)
    dd = d.cpu().numpy()
    assert np.all(np.abs(dd - D) <= RTOL * D)
