"""Pins for oracle/etree.py against what the paper and mathematics fix.

Pins: the SPEC worked example (golden), degenerate trees, plain definition vs
Algorithm 1, the memory identity P:223, HMS round trip, the A7 decodability
reading (golden), traversal == naive ADC bit for bit (the north_star's "E-Tree
traversal equals naive ADC for every code when both sum in subspace order"),
the lookup-count identity, and the iid-uniform closed form.
"""
import math

from scipy.stats import binom

import numpy as np
import pytest

from oracle import etree, pq
from paper_1509_05186_b200 import synth
from golden_io import load


def _tree(codes, ids=None, chain=127):
    tree, buf, sc, sid = etree.build(codes, ids, chain=chain)
    return tree, buf, sc, sid


def test_spec_worked_example():
    M, codes, exp = load("spec_example.txt")
    tree, buf, sc, sid = _tree(codes)
    st = tree.stats()
    sd = etree.tree_stats_def(sc)
    for s in (st, sd):
        assert s.L1 == int(exp["L1"][0])
        assert s.L2 == int(exp["L2"][0])
        assert s.total_postfix == int(exp["total_postfix"][0])
        assert s.lookups == int(exp["lookups"][0])
    posts = sorted(len(n.postfix) for n in tree.nodes() if n.is_leaf)
    assert posts == [int(x) for x in exp["postfix_sorted"]]
    assert len(buf) == int(exp["bytes"][0]) == st.paper_bytes


def _records(buf, M):
    out = []
    cur = -1
    pos = 0
    while pos < len(buf):
        K, u = buf[pos], buf[pos + 1]
        if u & 1:
            l = cur + 1
            out.append(f"L:{K}")
            pos += 2 + (M - 1 - l) + 4 * (u >> 1)
        else:
            cur = u >> 1
            out.append(f"I{cur}:{K}")
            pos += 2
    return out


def test_f4_leaves_first_is_decodable():
    M, codes, exp = load("f4_ambiguity.txt")
    tree, buf, sc, sid = _tree(codes)
    assert _records(buf, M) == exp["leaves_first_records"]
    pc, pid = etree.sort_codes(*etree.parse(buf, M))
    assert np.array_equal(pc, sc) and np.array_equal(pid, sid)
    # plain lexicographic child order cannot be decoded by the same rule
    lex = etree.serialize(tree, leaves_first=False)
    try:
        pc2, pid2 = etree.sort_codes(*etree.parse(lex, M))
        ok = np.array_equal(pc2, sc)
    except ValueError:
        ok = False
    assert not ok


@pytest.mark.parametrize("N,M", [(1, 4), (50, 8), (127, 8), (128, 8), (1000, 4)])
def test_identical_codes_single_leaf(N, M):
    codes = np.tile(np.arange(M, dtype=np.uint8) + 3, (N, 1))
    tree, buf, sc, sid = _tree(codes)
    st = tree.stats()
    assert (st.L1, st.L2, st.total_postfix) == (0, 1, M - 1)
    recs = math.ceil(N / 127)
    assert st.L2_records == recs
    assert len(buf) == 4 * N + 2 * recs + recs * (M - 1)
    leaf = next(iter(tree.nodes()))
    assert leaf.ids == list(range(N))


def test_distinct_first_bytes_no_sharing():
    M = 8
    N = 200
    r = np.random.default_rng(1)
    codes = r.integers(0, 256, size=(N, M)).astype(np.uint8)
    codes[:, 0] = np.arange(N)
    tree, buf, sc, sid = _tree(codes)
    st = tree.stats()
    assert (st.L1, st.L2, st.total_postfix) == (0, N, N * (M - 1))
    assert st.lookups == N * M
    assert len(buf) == 4 * N + 2 * N + N * (M - 1)


CASES = [
    # (seed, N, M, K, n_distinct)
    (1, 300, 4, 256, None),
    (2, 500, 8, 16, None),
    (3, 1000, 8, 4, None),
    (4, 2000, 8, 256, 40),     # duplicate heavy: chained leaves (n' > 127)
    (5, 400, 16, 16, None),
    (6, 3000, 4, 8, None),
    (7, 1, 8, 256, None),
    (8, 700, 2, 256, None),
    (9, 1500, 8, 2, None),
]


@pytest.mark.parametrize("seed,N,M,K,nd", CASES)
def test_definition_matches_algorithm1_and_roundtrip(seed, N, M, K, nd):
    codes = synth.random_codes(seed, N, M, K, nd)
    tree, buf, sc, sid = _tree(codes)
    st = tree.stats()
    sd = etree.tree_stats_def(sc)
    assert (st.L1, st.L2, st.total_postfix, st.L2_records, st.total_postfix_records) == \
           (sd.L1, sd.L2, sd.total_postfix, sd.L2_records, sd.total_postfix_records)
    assert st.depth_hist == sd.depth_hist
    # memory identity holds byte-exactly on the serialised buffer
    assert len(buf) == st.paper_bytes == 4 * N + 2 * (st.L1 + st.L2_records) + st.total_postfix_records
    # round trip: leaf enumeration reproduces the sorted input (the
    # leaves-first buffer order is re-sorted; the sort is stable)
    pc, pid = etree.sort_codes(*etree.parse(buf, M))
    assert np.array_equal(pc, sc) and np.array_equal(pid, sid)
    # every internal node has >= 1 child; every leaf's postfix has M-1-depth bytes
    for n in tree.nodes():
        if n.is_leaf:
            assert len(n.postfix) == M - 1 - n.depth and len(n.ids) >= 1
        else:
            assert len(n.children) >= 1 and n.depth <= M - 2
    # lookup identity: sum over distinct codes of (M - LCP with predecessor)
    U, _ = etree.distinct(sc)
    lp = etree.adjacent_lcp(U)
    assert int((M - lp).sum()) == st.lookups


@pytest.mark.parametrize("seed,N,M,K,nd", CASES)
def test_traversal_equals_naive_adc_bitwise(seed, N, M, K, nd):
    codes = synth.random_codes(seed, N, M, K, nd)
    s = 4
    cb = synth.random_floats(seed + 100, (M, K, s), 0.0, 4.0)
    qx = synth.random_floats(seed + 200, (5, M * s), 0.0, 4.0)
    tree, buf, sc, sid = _tree(codes)
    st = tree.stats()
    for table in (pq.lut32(cb, qx), pq.lut64(cb, qx)):
        out, lookups = etree.traverse(buf, M, table, N)
        ref = pq.adc(table, codes)
        assert out.dtype == ref.dtype
        assert np.array_equal(out, ref)          # bit for bit, same summation order
        assert lookups == st.lookups_records


def test_all_zero_table_gives_zero():
    codes = synth.random_codes(11, 300, 8, 16)
    tree, buf, sc, sid = _tree(codes)
    out, _ = etree.traverse(buf, 8, np.zeros((2, 8, 16), np.float32), 300)
    assert np.all(out == 0)


def test_chunk_order_changes_speed_not_values():
    codes = synth.random_codes(12, 800, 8, 8)
    cb = synth.random_floats(13, (8, 8, 2))
    qx = synth.random_floats(14, (3, 16))
    table = pq.lut64(cb, qx)
    order = np.array([3, 1, 7, 0, 5, 2, 6, 4])
    base_out, _ = etree.traverse(_tree(codes)[1], 8, table, 800)
    sc, sid = etree.sort_codes(codes, None, order)
    buf = etree.serialize(etree.build_alg1(sc, sid))
    perm_out, _ = etree.traverse(buf, 8, table[:, order, :], 800)
    np.testing.assert_allclose(perm_out, base_out, rtol=1e-12)


def test_errors():
    with pytest.raises(ValueError, match="empty"):
        etree.build_alg1(np.zeros((0, 4), np.uint8), np.zeros(0))
    bad = np.array([[2, 0], [1, 0]], np.uint8)
    with pytest.raises(ValueError, match="precondition"):
        etree.build_alg1(bad, np.arange(2))
    with pytest.raises(ValueError, match="config"):
        etree.sort_codes(bad, None, np.array([0, 0]))
    buf = _tree(synth.random_codes(3, 50, 4, 8))[1]
    with pytest.raises(ValueError, match="corrupt"):
        etree.parse(buf[:-3], 4)


def test_sort_spec_examples():
    sc, sid = etree.sort_codes(np.array([[2, 1], [1, 2]], np.uint8))
    assert sc.tolist() == [[1, 2], [2, 1]] and sid.tolist() == [1, 0]
    # stability: equal codes keep input id order
    c = np.array([[1, 1], [0, 0], [1, 1], [0, 0]], np.uint8)
    sc, sid = etree.sort_codes(c, np.array([10, 20, 30, 40]))
    assert sid.tolist() == [20, 40, 10, 30]


def _uniform_expectations(N, M, B=256):
    EL1 = 0.0
    Ed = 0.0
    for l in range(1, M):
        p = float(B) ** (-l)
        EL1 += float(B) ** l * binom.sf(1, N, p)          # P(Bin(N, p) >= 2)
        Ed += -np.expm1((N - 1) * np.log1p(-p))            # 1 - (1-p)^(N-1)
    return EL1, Ed


def test_uniform_code_closed_form():
    """for iid uniform byte codes the expected internal-node
    count and leaf depth have a closed form (N=1e5, M=8: E[L1]~30.1k, mean
    postfix ~5.21)."""
    N, M = 100_000, 8
    codes = synth.random_codes(21, N, M, 256)
    sc, _ = etree.sort_codes(codes)
    st = etree.tree_stats_def(sc)
    EL1, Ed = _uniform_expectations(N, M)
    assert EL1 > 0 and abs(st.L1 - EL1) / EL1 < 0.02
    assert abs(st.avg_postfix - (M - 1 - Ed)) < 0.02
    assert st.L2 == len(etree.distinct(sc)[0])
    ratio = st.lookups / (N * M)
    assert abs(ratio - (EL1 + N + N * (M - 1 - Ed)) / (N * M)) < 0.005
