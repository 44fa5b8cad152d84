"""Leaf extra byte on the GPU vs oracle/leafextra.py: the E-Tree
top-k with dist = table sum + E[e] (C1/C2 protocol, DESIGN.md 3.C)."""
import numpy as np
import pytest
import torch

from oracle import leafextra as lx
from oracle import pq
from paper_1509_05186_b200 import api
from paper_1509_05186_b200._lib import EtError
from gpu_common import check_topk, pq_inputs

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _extra_of(codes):
    # a deterministic function of the code (the byte is stored on the leaf)
    w = np.array([37, 11, 101, 7, 53, 29, 3, 71], dtype=np.int64)[: codes.shape[1]]
    return ((codes.astype(np.int64) * w).sum(1) % 256).astype(np.uint8)


def test_pq_codes_with_leaf_extra_topk():
    cfg, cb, codes, qx, X = pq_inputs("c1", N=40_000, Q=32, n_train=8_000, iters=6)
    extra = _extra_of(codes)
    E = np.random.default_rng(5).uniform(0, 3000.0, 256).astype(np.float32)
    ix = api.Index.et_build_etree(codes)
    ix.et_index_set_extra(extra)
    d, i = ix.et_etree_topk(50, queries=dev(qx), codebooks=dev(cb), extra_table=dev(E))
    torch.cuda.synchronize()
    T = pq.lut64(cb, qx)
    E64 = E.astype(np.float64)
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 50, range(cfg.Q),
               full_fn=lambda q: lx.adc_extra(T[q:q + 1], codes, extra, E64)[0])
    # E == 0 reproduces the plain E-Tree top-k bit for bit
    d0, i0 = ix.et_etree_topk(50, queries=dev(qx), codebooks=dev(cb), extra_table=dev(np.zeros(256, np.float32)))
    d1, i1 = ix.et_etree_topk(50, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    assert torch.equal(d0, d1) and torch.equal(i0, i1)


def test_aq_tables_with_quantized_cross_term():
    """Additive quantization: full-dimensional codebooks, tables
    ||q - c_m(k)||^2 given as luts, the Eq. 1 cross term quantized to one byte
    on the leaf."""
    r = np.random.default_rng(6)
    M, K, d, N, Q = 8, 16, 32, 6000, 24
    cb = r.normal(size=(M, K, d)) * 0.5
    codes = r.integers(0, K, size=(N, M)).astype(np.uint8)
    qx = r.normal(size=(Q, d))
    e, E, _ = lx.quantize_extra(lx.aq_cross(cb, codes))
    T32 = lx.aq_tables(cb, qx).astype(np.float32)
    E32 = E.astype(np.float32)
    ix = api.Index.et_build_etree(codes, K=K)
    ix.et_index_set_extra(e)
    dg, ig = ix.et_etree_topk(40, luts=dev(T32), extra_table=dev(E32))
    torch.cuda.synchronize()
    T64, E64 = T32.astype(np.float64), E32.astype(np.float64)
    check_topk(dg.cpu().numpy(), ig.cpu().numpy(), None, qx, codes, 40, range(Q),
               full_fn=lambda q: lx.adc_extra(T64[q:q + 1], codes, e, E64)[0])


def test_extra_byte_must_be_a_function_of_the_code():
    codes = np.array([[1, 2, 3, 4, 5, 6, 7, 8]] * 3 + [[9, 9, 9, 9, 9, 9, 9, 9]], dtype=np.uint8)
    ix = api.Index.et_build_etree(codes)
    with pytest.raises(EtError) as ei:
        ix.et_index_set_extra(np.array([1, 1, 2, 0], dtype=np.uint8))
    assert ei.value.status == 5   # ET_ERR_INVALID_CODE
    ix.et_index_set_extra(np.array([1, 1, 1, 0], dtype=np.uint8))


# ---------------------------------------------------------------- inner product (reading A26)

def test_inner_product_tables_and_topk():
    """Shifted inner-product tables (oracle/ip.py) and the E-Tree top-k over
    them = the largest inner products <q, x_hat>."""
    from oracle import ip as oip
    cfg, cb, codes, qx, X = pq_inputs("c1", N=30_000, Q=24, n_train=6_000, iters=4)
    luts, off = api.et_compute_ip_luts(dev(cb), dev(qx))
    torch.cuda.synchronize()
    L, O = luts.cpu().numpy().astype(np.float64), off.cpu().numpy().astype(np.float64)
    T, off64 = oip.ip_tables(cb, qx)
    # fp32 error bound of B - <q_m, c>: the two dot products' FMA chains
    # (<= (s + 2) 2^-24 sum_j |q_j c_j| each) plus the subtraction's rounding
    M, K, s = cb.shape
    A = np.stack([np.abs(qx[:, m * s:(m + 1) * s]) @ np.abs(cb[m]).T for m in range(M)], axis=1)   # [Q, M, K]
    tol = (s + 2) * 2.0 ** -24 * (A + A.max(axis=2, keepdims=True)) + 2.0 ** -23 * np.abs(T)
    assert np.all(np.abs(L - T) <= tol)
    assert L.min() >= 0 and np.all(L.min(axis=2) == 0)
    assert np.allclose(O, off64, rtol=1e-5)
    ix = api.Index.et_build_etree(codes)
    d, i = ix.et_etree_topk(30, luts=luts)
    torch.cuda.synchronize()
    # the scan over the GPU's own tables: C1/C2 protocol (non-negative sums)
    check_topk(d.cpu().numpy(), i.cpu().numpy(), None, qx, codes, 30, range(cfg.Q),
               full_fn=lambda q: pq.adc(L[q:q + 1], codes)[0])
    # and the ranking is the inner product's: the returned codes' exact <q, x_hat>
    # are the largest, within the tables' error bound
    IP = oip.inner_products(cb, qx, codes)
    gi = i.cpu().numpy()
    for q in range(cfg.Q):
        best = np.sort(IP[q])[::-1][:30]
        got = IP[q][gi[q]]
        slack = (tol[q].max(axis=1).sum()) * 2
        assert np.all(np.abs(np.sort(got)[::-1] - best) <= slack)
