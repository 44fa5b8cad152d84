"""Pins for oracle/eforest.py, topk.py, ivf.py, shard.py and the synth module."""
import os

import numpy as np
import pytest

from oracle import eforest, etree, ivf, pq, shard, topk
from paper_1509_05186_b200 import synth


def _setup(seed, N, M, K, s=3, nd=None, Q=4):
    codes = synth.random_codes(seed, N, M, K, nd)
    cb = synth.random_floats(seed + 1, (M, K, s), 0, 5)
    qx = synth.random_floats(seed + 2, (Q, M * s), 0, 5)
    return codes, cb, qx


# ------------------------------------------------------------------ forest

def test_forest_T1_is_the_etree_bitwise():
    codes, cb, qx = _setup(1, 600, 8, 16)
    t = pq.lut32(cb, qx)
    f = eforest.build_forest(codes, None, (0, 8))
    tree_out, _ = etree.traverse(etree.build(codes)[1], 8, t, 600)
    assert np.array_equal(eforest.forest_distances(f, t, 600), tree_out)


@pytest.mark.parametrize("split", [(0, 4, 8), (0, 3, 8), (0, 2, 5, 8), tuple(range(9))])
def test_forest_split_invariance_and_partials(split):
    codes, cb, qx = _setup(2, 900, 8, 8, nd=300)
    t32 = pq.lut32(cb, qx)
    t64 = pq.lut64(cb, qx)
    f = eforest.build_forest(codes, None, split)
    got = eforest.forest_distances(f, t32, 900)
    assert np.array_equal(got, eforest.forest_sum_adc(t32, codes, split))
    # each partial = ADC on the projected codes with the projected table
    for (a, Mt, buf, _), p in zip(f.trees, eforest.forest_partials(f, t32, 900)):
        assert np.array_equal(p, pq.adc(t32[:, a:a + Mt], codes[:, a:a + Mt]))
    ref = pq.adc(t64, codes)
    assert (np.abs(got - ref) / ref).max() < 1e-5
    # memory accounting: sum of per-tree formula values
    total = sum(len(buf) for (_, _, buf, _) in f.trees)
    assert total == sum(s.paper_bytes for s in f.stats())
    if len(split) == 9:          # T = M: depth-0 leaves only, <= K leaves per tree
        for s in f.stats():
            assert s.L1 == 0 and s.L2 <= 8


def test_forest_bad_split():
    with pytest.raises(ValueError, match="config"):
        eforest.build_forest(np.zeros((3, 4), np.uint8), None, (0, 2, 2, 4))


# ------------------------------------------------------------------ top-k

def test_topk_ties_by_id_and_padding():
    d = np.array([[3.0, 1.0, 2.0, 1.0]])
    ids = np.array([10, 7, 5, 3])
    D, I = topk.topk(d, ids, 3)
    assert I.tolist() == [[3, 7, 5]] and D.tolist() == [[1.0, 1.0, 2.0]]
    D, I = topk.topk(d, ids, 6)
    assert I.tolist() == [[3, 7, 5, 10, -1, -1]] and np.isinf(D[0, 4:]).all()


def test_topk_merge_equals_global():
    r = np.random.default_rng(3)
    d = r.integers(0, 20, size=(5, 300)).astype(np.float64)   # many exact ties
    ids = r.permutation(1000)[:300]
    D, I = topk.topk(d, ids, 17)
    parts = np.array_split(np.arange(300), 4)
    Ds, Is = zip(*[topk.topk(d[:, p], ids[p], 17) for p in parts])
    D2, I2 = topk.merge(Ds, Is, 17)
    assert np.array_equal(I, I2) and np.array_equal(D, D2)


# ------------------------------------------------------------------ shard

@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_shard_merge_equals_single(G):
    codes, cb, qx = _setup(4, 2000, 8, 32)
    dist = pq.adc(pq.lut64(cb, qx), codes)
    ids = np.arange(2000)
    D, I = topk.topk(dist, ids, 50)
    D2, I2 = shard.sharded_topk(dist, ids, codes[:, 0], G, 50)
    assert np.array_equal(I, I2) and np.array_equal(D, D2)
    b = shard.shard_bounds(codes[:, 0], G)
    assert b[0] == 0 and b[-1] == 256 and np.all(np.diff(b) >= 0)


def test_concatenated_shard_trees_are_the_tree():
    """subtrees built separately and concatenated form the whole
    structure -- byte for byte, when cut at first-level boundaries."""
    codes = synth.random_codes(5, 3000, 6, 12)
    _, buf, sc, sid = etree.build(codes)
    b = shard.shard_bounds(codes[:, 0], 3, K=12)
    parts = []
    for r in range(3):
        m = (sc[:, 0] >= b[r]) & (sc[:, 0] < b[r + 1])
        if m.any():
            parts.append(etree.serialize(etree.build_alg1(sc[m], sid[m])))
    assert b"".join(parts) == buf


# ------------------------------------------------------------------ ivf

def _ivf_small(seed=6):
    cfg = synth.scaled(synth.CONFIGS["c4"], N=3000, d=16, M=4, K=16, n_comp=20, n_train=2000)
    X = synth.base(cfg)
    coarse, _ = pq.kmeans(synth.coarse_train(cfg, 2000), 8, 5, seed)
    a = pq.assign(synth.resid_train(cfg, 2000), coarse)
    R = synth.resid_train(cfg, 2000) - coarse[a]
    cbs, _ = pq.train_pq(R.astype(np.float32), 4, 16, 5, seed)
    return ivf.encode_ivf(X, coarse.astype(np.float32), cbs), synth.queries(cfg, 6)


def test_ivf_full_probe_equals_exhaustive_residual_adc():
    index, qx = _ivf_small()
    D, I, _ = ivf.search(index, qx, w=8, k=30)
    N = len(index.codes)
    # exhaustive: residual ADC of every vector w.r.t. its own cell
    full = np.empty((len(qx), N))
    for q in range(len(qx)):
        for c in range(8):
            m = index.lists[c]
            r = qx[q].astype(np.float64) - index.coarse[c].astype(np.float64)
            full[q, m] = pq.adc(pq.lut64(index.codebooks, r[None]), index.codes[m])[0]
    D2, I2 = topk.topk(full, np.arange(N), 30)
    assert np.array_equal(I, I2) and np.allclose(D, D2, rtol=1e-12)


def test_ivf_tree_substitution_changes_nothing():
    index, qx = _ivf_small()
    D, I, p = ivf.search(index, qx, w=3, k=20)
    D2, I2, _ = ivf.search(index, qx, w=3, k=20, probes=p, use_tree=True)
    assert np.array_equal(I, I2) and np.array_equal(D, D2)
    assert sorted(np.concatenate(index.lists).tolist()) == list(range(len(index.codes)))


# ------------------------------------------------------------------ synth

def test_synth_deterministic_and_random_access():
    cfg = synth.scaled(synth.CONFIGS["c1"], N=200_000)
    a = synth.base(cfg, 65_000, 2_000)
    b = synth.base(cfg, 0, 70_000)
    assert np.array_equal(a, b[65_000:67_000])
    assert np.array_equal(synth.queries(cfg, 10), synth.queries(cfg, 10))
    assert a.dtype == np.float32 and a.min() >= 0 and a.max() <= 255
    assert np.array_equal(a, np.rint(a))
    c3 = synth.scaled(synth.CONFIGS["c3"], N=10)
    x = synth.base(c3)
    assert x.shape == (10, 960) and x.min() >= 0 and not np.array_equal(x, np.rint(x))


# ------------------------------------------------------------------ ivf probe / assignment pins

def _golden_probe():
    cent, qv, exp = None, None, {}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ivf_probe.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if not line:
                continue
            if line[0] == "centroids":
                cent = np.array([[float(t)] for t in line[1:]], np.float32)
            elif line[0] == "query":
                qv = np.array([[float(line[1])]], np.float32)
            elif line[0] == "expect":
                exp[int(line[1][1:])] = [int(t) for t in line[2:]]
    return cent, qv, exp


def test_ivf_probe_golden_ties_to_lower_cell():
    """Hand example (tests/golden/ivf_probe.txt): w < K' with exact distance
    ties (cells 1/2 at 1, 3/4 at 4) resolving to the lower cell."""
    cent, qv, exp = _golden_probe()
    for w, cells in exp.items():
        assert ivf.probe(qv, cent, w)[0].tolist() == cells, w


def _brute_probe(qx, coarse, w):
    """Pure-Python brute force: every distance by an explicit loop, then
    Python's sort on (distance, cell) tuples."""
    out = []
    for q in qx:
        d = []
        for c, cc in enumerate(coarse):
            s = 0.0
            for a, b in zip(q.tolist(), cc.tolist()):
                s += (a - b) * (a - b)
            d.append((s, c))
        out.append([c for _, c in sorted(d)[:w]])
    return np.array(out)


@pytest.mark.parametrize("seed,w", [(1, 1), (2, 3), (3, 7), (4, 16)])
def test_ivf_probe_brute_force_and_nesting(seed, w):
    r = np.random.default_rng(seed)
    coarse = r.integers(0, 4, size=(16, 3)).astype(np.float32)   # small integers: many exact ties
    qx = r.integers(0, 4, size=(9, 3)).astype(np.float32)
    got = ivf.probe(qx, coarse, w)
    assert np.array_equal(got, _brute_probe(qx, coarse, w))
    # nesting: the w nearest are the first w of the w+1 nearest; w = K' is a permutation
    if w < 16:
        assert np.array_equal(ivf.probe(qx, coarse, w + 1)[:, :w], got)
    allp = ivf.probe(qx, coarse, 16)
    assert all(sorted(row) == list(range(16)) for row in allp.tolist())


def test_encode_ivf_assignment_and_residual_codes_pinned():
    """encode_ivf: (a) vectors built as coarse centroid + a codeword
    concatenation, with well-separated centroids, get exactly that cell and
    re-encode to exactly those codewords (SPEC.md:369 'each residual code
    re-encodes to itself'); (b) K' = 1 degenerates to PQ of x - centroid
    (SPEC.md:367); (c) ties in the coarse assignment go to the lower cell."""
    r = np.random.default_rng(11)
    M, K, s, nl = 4, 8, 2, 5
    coarse = (np.arange(nl, dtype=np.float32)[:, None] * 1000.0) * np.ones((1, M * s), np.float32)
    cbs = r.integers(-3, 4, size=(M, K, s)).astype(np.float32)
    # make the codewords of each subspace distinct so the re-encode is unique
    cbs[:, :, 0] = np.arange(K, dtype=np.float32)[None, :] * 10.0
    cell = r.integers(0, nl, size=40)
    code = r.integers(0, K, size=(40, M))
    X = coarse[cell] + np.concatenate([cbs[m][code[:, m]] for m in range(M)], axis=1)
    ix = ivf.encode_ivf(X.astype(np.float32), coarse, cbs)
    assert ix.assign.tolist() == cell.tolist()
    assert np.array_equal(ix.codes, code.astype(np.uint8))
    # (b) one cell
    c1 = X.mean(0, keepdims=True).astype(np.float32)
    ix1 = ivf.encode_ivf(X.astype(np.float32), c1, cbs)
    assert np.all(ix1.assign == 0)
    assert np.array_equal(ix1.codes, pq.encode(cbs, X.astype(np.float64) - c1.astype(np.float64)))
    # (c) a point equidistant from cells 1 and 2 -> cell 1
    mid = ((coarse[1] + coarse[2]) / 2)[None, :]
    assert ivf.encode_ivf(mid, coarse, cbs).assign.tolist() == [1]
