"""IVFADC with per-list E-Trees (Table 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The application the paper accelerates: a coarse quantizer with K' centroids,
residuals r = x - cc(x) PQ-encoded with ONE shared residual codebook, one
inverted list (here: one E-Tree) per coarse cell.  A query probes the w nearest
cells (ties -> lower cell index), builds the residual distance table on
(q - cc) for each probed cell, scans that cell's codes and merges everything into
a top-k by (distance, id).  fp64 throughout (reading A17).
"""
from __future__ import annotations

from typing import List

import numpy as np

from . import pq, etree, topk as _topk


class IVF:
    def __init__(self, coarse: np.ndarray, codebooks: np.ndarray, assign: np.ndarray,
                 codes: np.ndarray):
        self.coarse = coarse              # [K', d] float32
        self.codebooks = codebooks        # [M, K, d/M] float32 (residual space)
        self.assign = assign              # [N] cell of each vector
        self.codes = codes                # [N, M] residual codes
        nlist = len(coarse)
        self.lists: List[np.ndarray] = [np.flatnonzero(assign == c) for c in range(nlist)]


def encode_ivf(X: np.ndarray, coarse: np.ndarray, codebooks: np.ndarray) -> IVF:
    """Assign to the nearest coarse centroid and PQ-encode the residual."""
    a = pq.assign(X, coarse)
    R = X.astype(np.float64) - coarse.astype(np.float64)[a]
    return IVF(coarse, codebooks, a, pq.encode(codebooks, R))


def probe(Qx: np.ndarray, coarse: np.ndarray, w: int) -> np.ndarray:
    """The w nearest coarse cells per query by (fp64 distance, cell index)."""
    d = pq.sqdist_direct(Qx, coarse)
    cells = np.arange(len(coarse))
    return np.stack([np.lexsort((cells, d[q]))[:w] for q in range(len(Qx))])


def search(index: IVF, Qx: np.ndarray, w: int, k: int, probes: np.ndarray = None,
           use_tree: bool = False):
    """Top-k over the probed lists.  ``use_tree`` runs each list through its own
    E-Tree traversal instead of naive ADC (the substitution of P:388)."""
    if probes is None:
        probes = probe(Qx, index.coarse, w)
    Q = len(Qx)
    D = np.full((Q, k), np.inf)
    I = np.full((Q, k), -1, dtype=np.int64)
    for q in range(Q):
        ds, ids = [], []
        for c in probes[q]:
            members = index.lists[int(c)]
            if len(members) == 0:
                continue
            r = Qx[q].astype(np.float64) - index.coarse[int(c)].astype(np.float64)
            table = pq.lut64(index.codebooks, r[None, :])
            if use_tree:
                M = index.codes.shape[1]
                sc, sid = etree.sort_codes(index.codes[members], members)
                buf = etree.serialize(etree.build_alg1(sc, sid))
                full, _ = etree.traverse(buf, M, table, int(members.max()) + 1)
                ds.append(full[0, members])
            else:
                ds.append(pq.adc(table, index.codes[members])[0])
            ids.append(members)
        if ds:
            d1, i1 = _topk.topk(np.concatenate(ds)[None, :], np.concatenate(ids), k)
            D[q], I[q] = d1[0], i1[0]
    return D, I, probes
