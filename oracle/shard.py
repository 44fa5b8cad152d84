"""Sharding by first-level subtrees and top-k merge.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:217-218: "Hierarchical Memory Structure can be separately constructed in
different memory chunks, and concatenate them to form the whole structure" --
so cutting the sorted codes between first-level subtrees (first code byte)
gives G valid sub-trees whose concatenation is the whole tree.  The cut rule
(SURVEY.md §8e): histogram of the first byte, boundary r = the smallest byte
value v with (#codes whose first byte < v) >= r*N/G.
"""
from __future__ import annotations

import numpy as np

from . import topk as _topk


def shard_bounds(first_byte: np.ndarray, G: int, K: int = 256) -> np.ndarray:
    """G+1 byte boundaries b_0=0 <= ... <= b_G=K; shard r holds first bytes in
    [b_r, b_{r+1}).  Written as the rule reads: for each r, walk v up from
    0 until the number of codes whose first byte is < v reaches r*N/G."""
    fb = [int(x) for x in np.asarray(first_byte).ravel()]
    N = len(fb)
    b = [0]
    for r in range(1, G):
        v = 0
        while v < K and sum(1 for x in fb if x < v) < r * N / G:
            v += 1
        b.append(max(b[-1], v))
    b.append(K)
    return np.array(b, dtype=np.int64)


def shard_of(first_byte: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    return np.searchsorted(bounds, np.asarray(first_byte), side="right") - 1


def sharded_topk(dist: np.ndarray, ids: np.ndarray, first_byte: np.ndarray, G: int, k: int):
    """Per-shard exact top-k, then merge; equals the unsharded top-k."""
    bounds = shard_bounds(first_byte, G)
    s = shard_of(first_byte, bounds)
    Ds, Is = [], []
    for r in range(G):
        m = np.flatnonzero(s == r)
        D, I = _topk.topk(dist[:, m], np.asarray(ids)[m], k)
        Ds.append(D)
        Is.append(I)
    return _topk.merge(Ds, Is, k)
