"""GPU: et_etree_topk_host (include/etree.h) -- the end-to-end call with host
buffers, the queries' upload and the results' read-back pipelined with the
search in batches.  Its results must equal et_etree_topk's bit for bit (the
per-query arithmetic does not depend on the batch) and the oracle's top-k
under the comparison protocol."""
import numpy as np
import pytest

from paper_1509_05186_b200 import api, build, synth

from gpu_common import check_topk, pq_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build.build()
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    api._lib.load()


@pytest.fixture(scope="module")
def c1():
    return pq_inputs("c1")


@pytest.mark.parametrize("n_batches", [0, 1, 3, 7])
def test_host_topk_equals_device_topk_and_oracle(c1, n_batches):
    cfg, cb, codes, qx, X = c1                     # Q = 100: batches of 100, 34/33/33, 14/15/...
    ix = api.Index.et_build_etree(codes)
    cbd = torch.from_numpy(cb).cuda()
    qh = torch.from_numpy(np.ascontiguousarray(qx)).pin_memory()
    dd, di = ix.et_etree_topk(100, queries=qh.cuda(), codebooks=cbd)
    hd, hi = ix.et_etree_topk_host(100, qh, cbd, n_batches=n_batches)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(hd, dd.cpu()) and torch.equal(hi, di.cpu())
    check_topk(hd.numpy(), hi.numpy(), cb, qx, codes, 100, range(cfg.Q))


def test_host_topk_c2_full_size_batches():
    """c2 (BASELINE configs[1]) in bench.py's e2e configuration (default batches):
    equal to the device call on all 10^4 queries, and the oracle on a sample."""
    cfg, cb, codes, qx, X = pq_inputs("c2")
    ix = api.Index.et_build_etree(codes)
    cbd = torch.from_numpy(cb).cuda()
    qh = torch.from_numpy(np.ascontiguousarray(qx)).pin_memory()
    dd, di = ix.et_etree_topk(100, queries=qh.cuda(), codebooks=cbd)
    out = (torch.empty((cfg.Q, 100), dtype=torch.float32).pin_memory(),
           torch.empty((cfg.Q, 100), dtype=torch.int32).pin_memory())
    for _ in range(2):   # the second call reuses the cached staging, streams and events
        out[0].fill_(-1.0)
        hd, hi = ix.et_etree_topk_host(100, qh, cbd, out=out)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(hd, dd.cpu()) and torch.equal(hi, di.cpu())
    rng = np.random.default_rng(11)
    sample = sorted(set([0, cfg.Q - 1] + rng.choice(cfg.Q, 30, replace=False).tolist()))
    check_topk(hd.numpy(), hi.numpy(), cb, qx, codes, 100, sample)


def test_host_topk_forest_and_ragged_q():
    """A two-tree E-Forest (c5's split shape) with Q not a multiple of anything."""
    cfg, cb, codes, qx, X = pq_inputs("c1", Q=37)
    ix = api.Index.et_build_eforest(codes, [0, 4, 8])
    cbd = torch.from_numpy(cb).cuda()
    qh = torch.from_numpy(np.ascontiguousarray(qx))        # pageable host memory: still correct
    dd, di = ix.et_etree_topk(10, queries=qh.cuda(), codebooks=cbd)
    hd, hi = ix.et_etree_topk_host(10, qh, cbd, n_batches=5)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(hd, dd.cpu()) and torch.equal(hi, di.cpu())


def test_host_topk_errors():
    cfg, cb, codes, qx, X = pq_inputs("c1", Q=8)
    ix = api.Index.et_build_etree(codes)
    cbd = torch.from_numpy(cb).cuda()
    with pytest.raises(ValueError):
        ix.et_etree_topk_host(10, torch.from_numpy(qx).cuda(), cbd)     # device queries
    with pytest.raises(Exception):
        ix.et_etree_topk_host(0, torch.from_numpy(qx), cbd)             # k out of range


def test_host_topk_graph_replay_equals_eager_and_survives_index_reuse(monkeypatch):
    """Page-locked buffers: the call is captured into a CUDA graph once per
    argument set and replayed; the replay must equal the eager enqueue
    (ET_HOST_EAGER=1), and freeing an index drops its graphs (a new index at
    the same address must not replay the old one's)."""
    cfg, cb, codes, qx, X = pq_inputs("c1")
    cbd = torch.from_numpy(cb).cuda()
    qh = torch.from_numpy(np.ascontiguousarray(qx)).pin_memory()
    out = (torch.empty((cfg.Q, 20), dtype=torch.float32).pin_memory(),
           torch.empty((cfg.Q, 20), dtype=torch.int32).pin_memory())
    ix = api.Index.et_build_etree(codes)
    ref = ix.et_etree_topk(20, queries=qh.cuda(), codebooks=cbd)
    for _ in range(3):   # capture, then replays
        out[0].zero_()
        ix.et_etree_topk_host(20, qh, cbd, out=out, n_batches=3)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(out[0], ref[0].cpu()) and torch.equal(out[1], ref[1].cpu())
    monkeypatch.setenv("ET_HOST_EAGER", "1")
    out[0].zero_()
    ix.et_etree_topk_host(20, qh, cbd, out=out, n_batches=3)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(out[0], ref[0].cpu()) and torch.equal(out[1], ref[1].cpu())
    monkeypatch.delenv("ET_HOST_EAGER")
    ix.free()
    codes2 = np.ascontiguousarray(codes[::-1][: len(codes) // 2])
    ix2 = api.Index.et_build_etree(codes2)
    ref2 = ix2.et_etree_topk(20, queries=qh.cuda(), codebooks=cbd)
    ix2._ws = ix._ws     # the same workspace and staging pointers as the freed index's graph
    ix2.et_etree_topk_host(20, qh, cbd, out=out, n_batches=3)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(out[0], ref2[0].cpu()) and torch.equal(out[1], ref2[1].cpu())
