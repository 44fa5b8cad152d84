"""Shared helpers for the -m gpu parity tests: oracle-side inputs (codebooks,
codes) for the BASELINE configs and the comparison protocol of DESIGN.md §3.C
(tolerance 1e-5 relative on every fp32 distance; top-k ids may differ only by
swaps among distances tied within that tolerance)."""
import functools

import numpy as np

from oracle import pq, topk as otopk
from paper_1509_05186_b200 import synth

RTOL = 1e-5


@functools.lru_cache(maxsize=None)
def pq_inputs(name: str, N: int = None, Q: int = None, n_train: int = None, iters: int = None):
    """Oracle-trained codebooks + oracle-encoded codes for config ``name``
    (optionally scaled down).  Returns (cfg, codebooks f32, codes u8, queries f32, base f32)."""
    cfg = synth.CONFIGS[name]
    over = {}
    if N is not None:
        over["N"] = N
    if Q is not None:
        over["Q"] = Q
    if n_train is not None:
        over["n_train"] = n_train
    if iters is not None:
        over["lloyd_iters"] = iters
    cfg = synth.scaled(cfg, **over)
    means = synth.mixture_means(cfg)
    tr = synth.train(cfg, means=means)
    cb, _ = pq.train_pq(tr, cfg.M, cfg.K, cfg.lloyd_iters, synth.kmeanspp_seed(cfg))
    X = synth.base(cfg, means=means)
    codes = pq.encode(cb, X)
    qx = synth.queries(cfg, means=means)
    return cfg, cb, codes, qx, X


def oracle_dist(cb, qx_row, codes_sel):
    """ADC64 distances of one query to the selected codes (the truth)."""
    return pq.adc(pq.lut64(cb, qx_row[None, :]), codes_sel)[0]


def check_topk(gd, gi, cb, qx, codes, k, qidx, ids_map=None, rtol=RTOL, full_fn=None):
    """Compare GPU top-k (gd, gi: numpy [Q, k]) with the oracle for queries qidx.

    ``ids_map``: slot -> id array when ids are not the slots (None = identity).
    ``full_fn(q)``: the oracle's distances of query q to every slot (default:
    ADC64 of the PQ codes).
    """
    N = len(codes)
    ids_all = np.arange(N) if ids_map is None else np.asarray(ids_map)
    inv = None
    if ids_map is not None:
        inv = np.empty(ids_all.max() + 1, dtype=np.int64)
        inv[ids_all] = np.arange(N)
    for q in qidx:
        full = full_fn(q) if full_fn is not None else oracle_dist(cb, qx[q], codes)
        # the oracle's full sort on the exact superset {distance <= k-th smallest}
        kk = min(k, N)
        kth = np.partition(full, kk - 1)[kk - 1]
        sel = np.flatnonzero(full <= kth)
        od, oi = otopk.topk(full[sel][None, :], ids_all[sel], k)
        od, oi = od[0], oi[0]
        g_d = gd[q].astype(np.float64)
        g_i = gi[q].astype(np.int64)
        nvalid = int((oi >= 0).sum())
        assert int((g_i >= 0).sum()) == nvalid, (q, g_i, oi)
        assert np.all(g_i[nvalid:] == -1) and np.all(np.isinf(g_d[nvalid:]))
        gv = g_i[:nvalid]
        assert len(np.unique(gv)) == nvalid, "duplicate ids"
        slots = gv if inv is None else inv[gv]
        truth_of_gpu = full[slots]
        ref = od[:nvalid]
        tol = rtol * np.maximum(ref, 1e-30)
        assert np.all(np.abs(g_d[:nvalid] - truth_of_gpu) <= rtol * np.maximum(truth_of_gpu, 1e-30)), q
        assert np.all(np.abs(g_d[:nvalid] - ref) <= tol), q
        mism = gv != oi[:nvalid]
        if mism.any():
            assert np.all(np.abs(truth_of_gpu[mism] - ref[mism]) <= tol[mism]), (q, np.flatnonzero(mism))
