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
    [b_r, b_{r+1})."""
    hist = np.bincount(np.asarray(first_byte, dtype=np.int64), minlength=K)
    below = np.concatenate(([0], np.cumsum(hist)))      # below[v] = #codes with byte < v
    N = int(below[-1])
    b = [0]
    for r in range(1, G):
        target = r * N / G
        v = int(np.searchsorted(below, target, side="left"))
        b.append(max(b[-1], min(v, K)))
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
