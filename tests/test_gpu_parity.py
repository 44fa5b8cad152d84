"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Every test here calls libetree.so kernels; the oracle supplies inputs
(codebooks/codes) and expected values only.  Tolerance: 1e-5 relative on every
fp32 distance vs the fp64 truth (north_star); top-k ids identical up to swaps
among distances tied within that tolerance.
"""
import numpy as np
import pytest

from oracle import eforest as oforest
from oracle import etree as oetree
from oracle import pq, topk as otopk
from paper_1509_05186_b200 import api, build, synth

from gpu_common import RTOL, check_topk, oracle_dist, pq_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build.build()
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    api._lib.load()


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-30)


# --------------------------------------------------------------------------- c1

@pytest.fixture(scope="module")
def c1():
    return pq_inputs("c1")


def test_c1_stats_match_oracle(c1):
    cfg, cb, codes, qx, X = c1
    ix = api.Index.et_build_etree(codes)
    st = ix.et_index_stats(0)
    sc, _ = oetree.sort_codes(codes)
    ref = oetree.tree_stats_def(sc)
    assert (st["L1"], st["L2"], st["total_postfix"], st["lookups"], st["paper_bytes"]) == \
           (ref.L1, ref.L2, ref.total_postfix, ref.lookups, ref.paper_bytes)


def test_c1_luts_vs_oracle(c1):
    cfg, cb, codes, qx, X = c1
    luts = api.et_compute_luts(dev(cb), dev(qx)).cpu().numpy()
    ref = pq.lut64(cb, qx)
    s = cfg.d // cfg.M
    assert rel_err(luts, ref).max() <= (2 * s + 2) * 2.0 ** -24


def test_c1_full_output_every_entry(c1):
    """BASELINE config 1: the full fp32 Q x N matrix, every entry vs ADC64."""
    cfg, cb, codes, qx, X = c1
    ix = api.Index.et_build_etree(codes)
    out = ix.et_etree_distances(queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = pq.adc(pq.lut64(cb, qx), codes)
    assert got.shape == (cfg.Q, cfg.N)
    assert rel_err(got, ref).max() <= RTOL


def test_tree_equals_flat_adc_bitwise(c1):
    """Same tables, same order: E-Tree scan == naive ADC bit for bit (north_star);
    fused tables == materialised tables bit for bit."""
    cfg, cb, codes, qx, X = c1
    ix = api.Index.et_build_etree(codes)
    luts = api.et_compute_luts(dev(cb), dev(qx))
    tree_l = ix.et_etree_distances(luts=luts)
    tree_q = ix.et_etree_distances(queries=dev(qx), codebooks=dev(cb))
    flat = api.et_flat_adc(luts, dev(codes))
    flat_ix = api.Index.et_build_flat(codes)
    flat2 = flat_ix.et_etree_distances(luts=luts)
    torch.cuda.synchronize()
    assert torch.equal(tree_l, flat)
    assert torch.equal(tree_q, flat)
    assert torch.equal(flat2, flat)


def test_c1_topk(c1):
    cfg, cb, codes, qx, X = c1
    ix = api.Index.et_build_etree(codes)
    d, i = ix.et_etree_topk(100, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 100, range(cfg.Q))


# --------------------------------------------------------------------------- c2 (headline)

@pytest.fixture(scope="module")
def c2():
    return pq_inputs("c2")


def test_c2_topk_full_size_sampled(c2):
    """BASELINE config 2 at full size (N=1e6, Q=1e4, top-100), in the launch
    configuration bench.py times; 200 sampled queries vs the oracle."""
    cfg, cb, codes, qx, X = c2
    ix = api.Index.et_build_etree(codes)
    d, i = ix.et_etree_topk(100, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    sample = sorted(set([0, cfg.Q - 1] + rng.choice(cfg.Q, 198, replace=False).tolist()))
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 100, sample)
    # property at any size: rows sorted by (dist, id), ids in range, distances
    # equal the oracle ADC64 of the returned ids for every query
    dn = d.cpu().numpy().astype(np.float64)
    inn = i.cpu().numpy()
    assert np.all(np.diff(dn, axis=1) >= 0)
    assert inn.min() >= 0 and inn.max() < cfg.N
    luts = api.et_compute_luts(dev(cb), dev(qx))
    g = torch.gather(luts.view(cfg.Q, -1), 1,
                     (torch.arange(cfg.M, device="cuda").view(1, 1, -1) * cfg.K +
                      dev(codes).long()[i.long()]).view(cfg.Q, -1)).view(cfg.Q, 100, cfg.M)
    # recompute sums in m order with torch on the GPU tables (consistency of ids vs distances)
    s = g[:, :, 0].clone()
    for m in range(1, cfg.M):
        s = s + g[:, :, m]
    assert torch.equal(s, d)


def test_uniform_codes_topk_refresh_path():
    """U1M companion shape (iid uniform codes: every leaf has multiplicity 1, the
    candidate buffers overflow and are pruned repeatedly)."""
    cfg, cb, _, qx, _ = pq_inputs("c1")
    N = 300_000
    codes = synth.uniform_codes(synth.CONFIGS["u1m"], N)
    ix = api.Index.et_build_etree(codes)
    Q = 64
    d, i = ix.et_etree_topk(100, queries=dev(qx[:Q]), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx[:Q], codes, 100, range(0, Q, 3))


# --------------------------------------------------------------------------- edge cases

def _small(seed, N, M, K, s, Q, nd=None, lo=0.0, hi=10.0):
    codes = synth.random_codes(seed, N, M, K, nd)
    cb = synth.random_floats(seed + 1, (M, K, s), lo, hi)
    qx = synth.random_floats(seed + 2, (Q, M * s), lo, hi)
    return cb, codes, qx


@pytest.mark.parametrize("seed,N,M,K,s,Q,nd,k", [
    (1, 50, 8, 256, 16, 5, None, 100),       # k > N: padding
    (2, 5000, 4, 16, 4, 33, None, 10),       # all levels in smem, K < 256, ragged Q
    (3, 20000, 8, 256, 3, 1, None, 64),      # generic s (d = 24), Q = 1
    (4, 8000, 8, 64, 8, 257, 300, 100),      # duplicate heavy, Q spans many chunks
    (5, 3000, 6, 256, 16, 40, None, 256),    # M = 6, k = 256 (max)
    (6, 1, 8, 256, 16, 3, None, 5),          # N = 1
    (7, 40000, 2, 256, 16, 70, None, 7),     # shallow tree, many leaves per level
])
def test_edge_topk_and_full(seed, N, M, K, s, Q, nd, k):
    cb, codes, qx = _small(seed, N, M, K, s, Q, nd)
    ix = api.Index.et_build_etree(codes, K=K)
    d, i = ix.et_etree_topk(k, queries=dev(qx), codebooks=dev(cb))
    full = ix.et_etree_distances(queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, k, range(Q))
    ref = pq.adc(pq.lut64(cb, qx), codes)
    assert rel_err(full.cpu().numpy(), ref).max() <= RTOL


def test_all_identical_codes_single_leaf():
    cb, _, qx = _small(8, 10, 8, 256, 16, 4)
    codes = np.tile(np.arange(8, dtype=np.uint8), (1000, 1))
    ix = api.Index.et_build_etree(codes)
    d, i = ix.et_etree_topk(10, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    assert i.cpu().numpy().tolist() == [list(range(10))] * 4
    dd = d.cpu().numpy()
    assert np.all(dd == dd[:, :1])


def test_all_zero_distances_ties_resolve_by_id():
    """All-zero tables: every code ties at 0; the top-k must be the k
    smallest ids.  Exercises the tie rule of the pruning and finalize."""
    N, M, K = 20000, 8, 16
    codes = synth.random_codes(9, N, M, K)
    ids = np.random.default_rng(3).permutation(N * 3)[:N].astype(np.int32)
    cb = np.zeros((M, K, 4), np.float32)
    qx = np.zeros((6, M * 4), np.float32)
    ix = api.Index.et_build_etree(codes, ids=ids, K=K)
    d, i = ix.et_etree_topk(100, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    exp = np.sort(ids)[:100]
    for q in range(6):
        assert i.cpu().numpy()[q].tolist() == exp.tolist()
    assert np.all(d.cpu().numpy() == 0)


def test_user_ids_and_byte_perm(c1):
    cfg, cb, codes, qx, X = c1
    ids = np.random.default_rng(5).permutation(cfg.N).astype(np.int32) * 2 + 1
    perm = np.array([3, 1, 7, 0, 5, 2, 6, 4], np.int32)
    ix = api.Index.et_build_etree(codes, ids=ids, byte_perm=perm)
    d, i = ix.et_etree_topk(50, queries=dev(qx[:20]), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx[:20], codes, 50, range(20), ids_map=ids)


# --------------------------------------------------------------------------- forest

@pytest.fixture(scope="module")
def c3s():
    # BASELINE config 3's generator and PQ shape (d=960, M=16, s=60), scaled
    return pq_inputs("c3", N=100_000, Q=48, n_train=20_000, iters=8)


def test_forest_c3_shape_topk_and_full(c3s):
    cfg, cb, codes, qx, X = c3s
    ix = api.Index.et_build_eforest(codes, split=[0, 8, 16])
    st = ix.stats()
    for t, (a, b) in enumerate([(0, 8), (8, 16)]):
        sc, _ = oetree.sort_codes(codes[:, a:b])
        ref = oetree.tree_stats_def(sc)
        assert (st[t]["L1"], st[t]["L2"], st[t]["total_postfix"]) == (ref.L1, ref.L2, ref.total_postfix)
    d, i = ix.et_etree_topk(100, queries=dev(qx), codebooks=dev(cb))
    full = ix.et_etree_distances(queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 100, range(cfg.Q))
    ref = pq.adc(pq.lut64(cb, qx), codes)
    assert rel_err(full.cpu().numpy(), ref).max() <= RTOL
    # tables built inside the scan CTAs (s = 60 wide build) == lut_kernel's
    # materialised tables, bit for bit: the same j-ascending FMA chains
    luts = api.et_compute_luts(dev(cb), dev(qx))
    full_m = ix.et_etree_distances(luts=luts)
    torch.cuda.synchronize()
    assert torch.equal(full, full_m)
    # chunk sizes 1..8 queries per CTA (odd and even pair counts): 1181 queries
    # over the SMs; fused top-k == materialised top-k exactly
    qb = np.concatenate([qx] * 25)[:1181]
    df, if_ = ix.et_etree_topk(100, queries=dev(qb), codebooks=dev(cb))
    dm, im = ix.et_etree_topk(100, luts=api.et_compute_luts(dev(cb), dev(qb)))
    torch.cuda.synchronize()
    assert torch.equal(df, dm) and torch.equal(if_, im)


def test_forest_T1_equals_tree_and_split_invariance(c1):
    cfg, cb, codes, qx, X = c1
    luts = api.et_compute_luts(dev(cb), dev(qx))
    a = api.Index.et_build_etree(codes).et_etree_distances(luts=luts)
    b = api.Index.et_build_eforest(codes, split=[0, 8]).et_etree_distances(luts=luts)
    c = api.Index.et_build_eforest(codes, split=[0, 4, 8]).et_etree_distances(luts=luts)
    e = api.Index.et_build_eforest(codes, split=[0, 3, 5, 8]).et_etree_distances(luts=luts)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    ref = pq.adc(pq.lut64(cb, qx), codes)
    for x in (c, e):
        assert rel_err(x.cpu().numpy(), ref).max() <= RTOL
    # forest partial sums in tree order (A13): p0 + p1 exactly, from the GPU tables
    L = luts.cpu().numpy()
    exp = oforest.forest_sum_adc(L, codes, (0, 4, 8))
    assert np.array_equal(c.cpu().numpy(), exp)


# --------------------------------------------------------------------------- sharding

def test_logical_shards_merge_equals_single(c1):
    """shards of first-level subtrees; per-shard top-k merged with
    K7 equals the single-index top-k exactly (same sums, same order)."""
    cfg, cb, codes, qx, X = c1
    k = 100
    one = api.Index.et_build_etree(codes)
    d1, i1 = one.et_etree_topk(k, queries=dev(qx), codebooks=dev(cb))
    for G in (2, 3, 8):
        b = api.et_shard_bounds(codes, G)   # the product's cut (host C++)
        ds, is_ = [], []
        for r in range(G):
            m = np.flatnonzero((codes[:, 0] >= b[r]) & (codes[:, 0] < b[r + 1]))
            if len(m) == 0:
                ds.append(torch.full((cfg.Q, k), float("inf"), device="cuda"))
                is_.append(torch.full((cfg.Q, k), -1, dtype=torch.int32, device="cuda"))
                continue
            ix = api.Index.et_build_etree(codes[m], ids=m.astype(np.int32))
            d, i = ix.et_etree_topk(k, queries=dev(qx), codebooks=dev(cb))
            ds.append(d)
            is_.append(i)
        md, mi = api.et_merge_topk(torch.stack(ds), torch.stack(is_))
        torch.cuda.synchronize()
        assert torch.equal(mi, i1) and torch.equal(md, d1), G
        # and against the oracle's global top-k (not only the single GPU index)
        check_topk(md.cpu().numpy(), mi.cpu().numpy(), cb, qx, codes, k, range(cfg.Q))


# --------------------------------------------------------------------------- PQ support kernels

def test_encode_matches_oracle_up_to_near_ties(c1):
    cfg, cb, codes, qx, X = c1
    g = api.et_encode(dev(cb), dev(X[:20000])).cpu().numpy()
    ref = codes[:20000]
    diff = np.argwhere(g != ref)
    s = cfg.d // cfg.M
    for (r, m) in diff:   # only near ties may differ
        dd = pq.sqdist_direct(X[r:r + 1, m * s:(m + 1) * s], cb[m])[0]
        a, b = dd[g[r, m]], dd[ref[r, m]]
        assert abs(a - b) <= 1e-5 * max(a, b)
    assert len(diff) <= 20


def test_build_codebooks_monotone_and_close_to_oracle():
    cfg = synth.scaled(synth.CONFIGS["c1"], n_train=20_000)
    tr = synth.train(cfg)
    cb, hist = api.et_build_codebooks(tr, cfg.M, cfg.K, 10, seed=11)
    assert cb.shape == (8, 256, 16)
    for m in range(cfg.M):
        h = hist[m]
        assert np.all(np.diff(h) <= 1e-6 * h[:-1]), h
    ocb, ohist = pq.train_pq(tr, cfg.M, cfg.K, 10, seed=11)
    ours = sum(h[-1] for h in hist)
    theirs = sum(h[-1] for h in ohist)
    assert abs(ours - theirs) / theirs < 0.05


# --------------------------------------------------------------------------- GPU-native build (f1)

@pytest.mark.parametrize("seed,N,M,K,nd,split,user_ids", [
    (1, 30000, 8, 256, None, (0, 8), False),
    (3, 40000, 8, 256, 500, (0, 8), True),        # duplicate heavy, user ids
    (4, 20000, 16, 16, None, (0, 8, 16), False),  # joined forest (M = 16)
    (5, 20000, 8, 4, None, (0, 4, 8), True),      # fused forest
    (7, 25000, 6, 3, None, (0, 2, 5, 6), False),
])
def test_gpu_build_stats_equal_host_and_oracle(seed, N, M, K, nd, split, user_ids):
    """The GPU grouping step (radix sort + flag scan, build_gpu.cu) yields the
    same trees as the host build and the oracle's plain definition."""
    from test_lib_cpu import _oracle_stats
    codes = synth.random_codes(seed, N, M, K, nd)
    ids = (np.random.default_rng(seed).permutation(3 * N)[:N].astype(np.int32) if user_ids else None)
    if len(split) == 2:
        ix = api.Index.et_build_etree(codes, ids=ids, K=K)
    else:
        ix = api.Index.et_build_eforest(codes, split=list(split), ids=ids, K=K)
    got = ix.stats()
    host = api.et_build_stats(codes, split=list(split), ids=ids, K=K)
    ref = _oracle_stats(codes, split)
    keys = ("L1", "L2", "total_postfix", "lookups", "L2_records", "paper_bytes", "groups", "scan_lookups")
    for g, h, r in zip(got, host, ref):
        assert all(g[k_] == h[k_] for k_ in keys), (g, h)
        assert (g["L1"], g["L2"], g["total_postfix"]) == (r.L1, r.L2, r.total_postfix)
    # the device id order (ascending within a group) through a query: top-k vs oracle
    cb = synth.random_floats(seed + 9, (M, K, 4), 0, 5)
    qx = synth.random_floats(seed + 10, (6, M * 4), 0, 5)
    d, i = ix.et_etree_topk(30, queries=dev(qx), codebooks=dev(cb))
    full = ix.et_etree_distances(queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 30, range(6), ids_map=ids)
    ref_full = pq.adc(pq.lut64(cb, qx), codes)
    assert rel_err(full.cpu().numpy(), ref_full).max() <= RTOL
