"""Pins of oracle/leafextra.py (Eq. 1) against the
mathematics, not against its own formula."""
import numpy as np
import pytest

from oracle import leafextra as lx
from oracle import pq, topk


def _aq_case(seed=0, M=3, K=5, d=6, n=40, Q=4):
    r = np.random.default_rng(seed)
    cb = r.normal(size=(M, K, d))
    codes = r.integers(0, K, size=(n, M)).astype(np.uint8)
    q = r.normal(size=(Q, d))
    return cb, codes, q


def test_eq1_identity_with_exact_cross_term():
    """Eq. 1 (A1: (M-1)): sum_m ||q - c_m||^2 + cross = ||q - x_hat||^2 + (M-1)||q||^2,
    brute force on the decoded vectors."""
    cb, codes, q = _aq_case()
    M = cb.shape[0]
    # one extra byte per distinct code, its exact cross term in the table
    uniq, inv = np.unique(codes, axis=0, return_inverse=True)
    E = np.zeros(256)
    E[: len(uniq)] = lx.aq_cross(cb, uniq)
    got = lx.adc_extra(lx.aq_tables(cb, q), codes, inv.astype(np.uint8), E)
    xh = lx.aq_decode(cb, codes)
    want = ((q[:, None, :] - xh[None, :, :]) ** 2).sum(-1) + (M - 1) * (q ** 2).sum(-1)[:, None]
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_aq_decode_brute_force():
    cb, codes, _ = _aq_case(seed=1)
    xh = lx.aq_decode(cb, codes)
    for i in range(len(codes)):
        ref = sum(cb[m][codes[i, m]] for m in range(cb.shape[0]))
        assert np.allclose(xh[i], ref)


def test_zero_table_is_plain_adc():
    r = np.random.default_rng(2)
    T = r.random((3, 4, 16))
    codes = r.integers(0, 16, size=(50, 4)).astype(np.uint8)
    e = r.integers(0, 256, size=50).astype(np.uint8)
    assert np.array_equal(lx.adc_extra(T, codes, e, np.zeros(256)), pq.adc(T, codes))


def test_constant_table_keeps_the_ranking():
    """E[e] = kappa for every byte: distances shift by kappa, top-k ids unchanged."""
    r = np.random.default_rng(3)
    T = r.random((2, 4, 16))
    codes = r.integers(0, 16, size=(300, 4)).astype(np.uint8)
    e = r.integers(0, 256, size=300).astype(np.uint8)
    D0 = pq.adc(T, codes)
    D1 = lx.adc_extra(T, codes, e, np.full(256, 7.25))
    assert np.allclose(D1 - D0, 7.25, rtol=0, atol=1e-12)
    ids = np.arange(300)
    for q in range(2):
        a = topk.topk(D0[q][None], ids, 20)[1]
        b = topk.topk(D1[q][None], ids, 20)[1]
        assert np.array_equal(a, b)


def test_extra_changes_the_ranking_by_its_term():
    """Two codes with equal table sums: the smaller decoded extra ranks first."""
    T = np.zeros((1, 2, 4))
    codes = np.array([[1, 2], [2, 1]], dtype=np.uint8)
    E = np.zeros(256)
    E[9], E[3] = 5.0, 1.0
    D = lx.adc_extra(T, codes, np.array([9, 3], dtype=np.uint8), E)
    assert D.tolist() == [[5.0, 1.0]]


def test_leaf_extra_is_a_function_of_the_code():
    codes = np.array([[1, 2], [1, 2], [3, 4]], dtype=np.uint8)
    assert lx.leaf_extra(codes, np.array([7, 7, 9], dtype=np.uint8)) == {bytes([1, 2]): 7, bytes([3, 4]): 9}
    with pytest.raises(ValueError):
        lx.leaf_extra(codes, np.array([7, 8, 9], dtype=np.uint8))


def test_quantize_extra_error_bound_and_range():
    v = np.random.default_rng(4).normal(size=1000) * 30.0
    e, E, shift = lx.quantize_extra(v)
    step = E[1] - E[0]
    assert E[0] == 0.0 and e.min() == 0 and e.max() == 255
    assert np.abs(E[e] + shift - v).max() <= step / 2 + 1e-9


# ---------------------------------------------------------------- inner product (oracle/ip.py)

from oracle import ip as oip  # noqa: E402


def test_ip_tables_shift_identity_and_ranking():
    """sum_m T = off - <q, x_hat> (brute force on decoded vectors); entries >= 0
    with a zero per row; smallest sums = largest inner products."""
    r = np.random.default_rng(7)
    M, K, s = 4, 8, 3
    cb = r.normal(size=(M, K, s))
    codes = r.integers(0, K, size=(200, M)).astype(np.uint8)
    q = r.normal(size=(5, M * s))
    T, off = oip.ip_tables(cb, q)
    assert T.min() >= 0 and np.all(T.min(axis=2) == 0)
    S = pq.adc(T, codes)
    IP = oip.inner_products(cb, q, codes)
    assert np.allclose(off[:, None] - S, IP, rtol=0, atol=1e-12)
    for i in range(5):
        assert np.array_equal(np.argsort(S[i], kind="stable")[:10], np.argsort(-IP[i], kind="stable")[:10])


def test_ip_of_codeword_concatenation_brute_force():
    r = np.random.default_rng(8)
    cb = r.normal(size=(2, 3, 2))
    codes = np.array([[0, 2], [1, 1]], dtype=np.uint8)
    q = np.array([[1.0, -2.0, 0.5, 3.0]])
    want = [q[0] @ np.r_[cb[0][0], cb[1][2]], q[0] @ np.r_[cb[0][1], cb[1][1]]]
    assert np.allclose(oip.inner_products(cb, q, codes)[0], want)
