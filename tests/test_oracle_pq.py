"""Pins for oracle/pq.py: exact-L2 special case, Eq. 1 with reading A1, SPEC
table/encode/k-means examples, fp32-vs-fp64 error bounds."""
import numpy as np
import pytest

from oracle import pq
from paper_1509_05186_b200 import synth


def _cb(seed, M, K, s, lo=0.0, hi=10.0):
    return synth.random_floats(seed, (M, K, s), lo, hi)


def test_adc_equals_exact_l2_on_codeword_concatenations():
    """north_star: on inputs where every database vector is itself a codeword
    concatenation, ADC equals brute-force exact squared L2."""
    M, K, s = 4, 16, 3
    cb = _cb(1, M, K, s)
    codes = synth.random_codes(2, 200, M, K)
    X = pq.decode(cb, codes)
    qx = synth.random_floats(3, (7, M * s), 0.0, 10.0)
    got = pq.adc(pq.lut64(cb, qx), codes)
    ref = pq.exact_sqdist(qx, X)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)
    # q == decode(c) => 0
    z = pq.adc(pq.lut64(cb, X[:3]), codes[:3])
    assert np.allclose(np.diag(z), 0.0, atol=1e-12)


def test_eq1_with_M_minus_1_reading():
    """P:92-99 Eq. 1: ||q - sum_m c~_m||^2 = sum_m ||q - c~_m||^2 - (M-1)||q||^2 +
    sum_{i != j} c~_i . c~_j with zero-padded codewords c~_m.  The printed
    '(m-1)' only balances with m = M (reading A1); the cross term vanishes for
    PQ's disjoint supports, leaving the table sum."""
    M, K, s = 4, 8, 2
    cb = _cb(5, M, K, s)
    code = [1, 5, 0, 7]
    q = synth.random_floats(6, (M * s,), 0.0, 10.0).astype(np.float64)
    pads = []
    for m in range(M):
        c = np.zeros(M * s)
        c[m * s:(m + 1) * s] = cb[m, code[m]]
        pads.append(c)
    lhs = np.sum((q - np.sum(pads, 0)) ** 2)
    first = sum(np.sum((q - c) ** 2) for c in pads)
    cross = sum(pads[i] @ pads[j] for i in range(M) for j in range(M) if i != j)
    assert cross == 0.0
    assert np.isclose(lhs, first - (M - 1) * (q @ q) + cross, rtol=1e-12)
    assert not np.isclose(lhs, first - (0) * (q @ q))  # the constant matters
    tab = pq.lut64(cb, q[None])[0]
    assert np.isclose(lhs, pq.adc_one(tab, code), rtol=1e-12)


def test_lut_spec_examples():
    M, K, s = 3, 5, 4
    cb = _cb(7, M, K, s)
    q0 = np.concatenate([cb[m, 0] for m in range(M)])[None]
    for t in (pq.lut64(cb, q0), pq.lut32(cb, q0)):
        assert np.all(t[0, :, 0] == 0.0)
        assert np.all(t >= 0)
    zero = pq.lut64(np.zeros((M, K, s), np.float32), np.zeros((1, M * s)))
    assert np.all(zero == 0)
    # permutation covariance
    qx = synth.random_floats(8, (4, M * s), 0, 10)
    perm = np.array([3, 0, 4, 1, 2])
    t0 = pq.lut64(cb, qx)
    t1 = pq.lut64(cb[:, perm, :], qx)
    assert np.array_equal(t1, t0[:, :, perm])
    with pytest.raises(ValueError, match="dimension"):
        pq.lut64(cb, np.zeros((1, 5)))


def test_lut32_error_bound_vs_lut64():
    """fp32 table entries are sums of s positive terms: relative error <= ~s*2^-24."""
    M, K, s = 8, 256, 16
    cb = _cb(9, M, K, s, 0.0, 255.0)
    qx = np.rint(synth.random_floats(10, (6, M * s), 0.0, 255.0))
    t32 = pq.lut32(cb, qx).astype(np.float64)
    t64 = pq.lut64(cb, qx)
    rel = np.abs(t32 - t64) / np.maximum(t64, 1e-30)
    assert rel.max() <= (2 * s + 2) * 2.0 ** -24
    codes = synth.random_codes(11, 1000, M, K)
    a32 = pq.adc(pq.lut32(cb, qx), codes).astype(np.float64)
    a64 = pq.adc(t64, codes)
    assert (np.abs(a32 - a64) / a64).max() < 1e-5


def test_adc_small_cases():
    t = synth.random_floats(12, (2, 1, 9), 0, 1)
    codes = np.array([[4], [0]], np.uint8)
    assert np.array_equal(pq.adc(t, codes), t[:, 0, [4, 0]])     # M=1
    assert pq.adc(synth.random_floats(1, (2, 3, 4)), np.zeros((0, 3), np.uint8)).shape == (2, 0)
    with pytest.raises(ValueError, match="config"):
        pq.adc(t, np.zeros((2, 2), np.uint8))


def test_encode_examples():
    cb = np.array([[[0.0], [1.0]], [[0.0], [1.0]]], np.float32)   # d=2, M=2, K=2
    assert pq.encode(cb, np.array([[0.9, 0.1]], np.float32)).tolist() == [[1, 0]]
    M, K, s = 4, 32, 3
    cbr = _cb(13, M, K, s)
    X = synth.random_floats(14, (300, M * s), 0, 10)
    codes = pq.encode(cbr, X)
    for m in range(M):
        d = pq.sqdist_direct(X[:, m * s:(m + 1) * s], cbr[m])
        assert np.array_equal(codes[:, m], np.argmin(d, 1))       # brute force
    # codeword concatenations encode to themselves and decode back
    c = synth.random_codes(15, 50, M, K)
    assert np.array_equal(pq.encode(cbr, pq.decode(cbr, c)), c)
    # ties -> lowest index
    cbt = cbr.copy()
    cbt[:, 7] = cbt[:, 3]
    xt = pq.decode(cbt, np.full((1, M), 7, np.uint8))
    assert pq.encode(cbt, xt).tolist() == [[3] * M]
    with pytest.raises(ValueError, match="dimension"):
        pq.encode(cbr, np.zeros((1, 5)))
    with pytest.raises(ValueError, match="invalid code"):
        pq.decode(cbr, np.full((1, M), 40, np.uint8))


def test_fast_sqdist_matches_direct():
    X = synth.random_floats(16, (100, 16), 0, 255)
    C = synth.random_floats(17, (50, 16), 0, 255)
    np.testing.assert_allclose(pq._sqdist_f64(X, C), pq.sqdist_direct(X, C), rtol=1e-9, atol=1e-6)


def test_kmeans_monotone_and_examples():
    X = synth.random_floats(18, (2000, 8), 0, 10)
    C, hist = pq.kmeans(X, 16, 10, seed=3)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))
    C2, hist2 = pq.kmeans(X, 16, 10, seed=3)
    assert np.array_equal(C, C2)                                          # determinism
    # K = N -> zero quantisation error
    Y = synth.random_floats(19, (20, 4), 0, 10)
    Cy, hy = pq.kmeans(Y, 20, 3, seed=1)
    assert pq.objective(Y, Cy, pq.assign(Y, Cy)) == 0.0
    # two well separated clusters, K=2 -> the cluster means
    A = synth.random_floats(20, (100, 3), 0, 1)
    B = synth.random_floats(21, (150, 3), 100, 101)
    Cab, _ = pq.kmeans(np.concatenate([A, B]), 2, 3, seed=5)
    Cab = Cab[np.argsort(Cab[:, 0])]
    np.testing.assert_allclose(Cab[0], A.astype(np.float64).mean(0), rtol=1e-12)
    np.testing.assert_allclose(Cab[1], B.astype(np.float64).mean(0), rtol=1e-12)
    with pytest.raises(ValueError, match="insufficient"):
        pq.kmeans(Y[:3], 4, 1, seed=0)


def test_train_pq_errors():
    with pytest.raises(ValueError, match="invalid subspace"):
        pq.train_pq(np.zeros((10, 5), np.float32), 2, 2, 1, 0)
    bad = np.zeros((10, 4), np.float32)
    bad[0, 0] = np.nan
    with pytest.raises(ValueError, match="invalid vector"):
        pq.train_pq(bad, 2, 2, 1, 0)
