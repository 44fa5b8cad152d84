"""Exact top-k (not in the paper; BASELINE north_star item 4, reading A14).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Per query, the k smallest (distance, id) pairs in lexicographic order: distance
ascending, ties by smaller id.  If fewer than k vectors exist the
list is padded with (+inf, -1).  Implemented as a full sort -- the definition.
"""
from __future__ import annotations

import numpy as np


def topk(dist: np.ndarray, ids: np.ndarray, k: int):
    """dist [Q, N] (any float dtype), ids [N] -> (D [Q, k] float64, I [Q, k] int64)."""
    dist = np.asarray(dist)
    ids = np.asarray(ids, dtype=np.int64)
    Q, N = dist.shape
    D = np.full((Q, k), np.inf, dtype=np.float64)
    I = np.full((Q, k), -1, dtype=np.int64)
    n = min(k, N)
    for q in range(Q):
        order = np.lexsort((ids, dist[q]))[:n]
        D[q, :n] = dist[q][order]
        I[q, :n] = ids[order]
    return D, I


def merge(lists_D, lists_I, k: int):
    """Merge several per-query top-k lists (same Q) into one, by (dist, id)."""
    D = np.concatenate(lists_D, axis=1)
    I = np.concatenate(lists_I, axis=1)
    Q = D.shape[0]
    outD = np.full((Q, k), np.inf)
    outI = np.full((Q, k), -1, dtype=np.int64)
    for q in range(Q):
        valid = I[q] >= 0
        d, i = D[q][valid], I[q][valid]
        order = np.lexsort((i, d))[:k]
        outD[q, :len(order)] = d[order]
        outI[q, :len(order)] = i[order]
    return outD, outI
