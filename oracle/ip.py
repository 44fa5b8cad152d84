"""Inner-product tables for the E-Tree (maximum inner product search).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper passages followed:
* "One can also easily extend ADC to perform efficient scalar
  product"; P:135 (footnote) -- "It can also easily extended to compute inner
  product ... We omit the discussion"; P:389-391 -- "One can also extend
  E-Tree to allow fast scalar product".

Reading (A26): the E-Tree sums table entries; a top-k by the
smallest sum with non-negative entries is what the scan computes.  The inner
product <q, x_hat> = sum_m <q_m, c_m(k_m)> (PQ: x_hat = concatenated
codewords) becomes such a sum with the shifted table
    T[q][m][k] = B[q][m] - <q_m, c_m(k)>,   B[q][m] = max_k <q_m, c_m(k)>
(every entry >= 0, each row has a 0), so
    sum_m T[q][m][code[m]] = off[q] - <q, x_hat>,   off[q] = sum_m B[q][m],
and the k smallest sums are the k largest inner products.
"""
from __future__ import annotations

import numpy as np


def ip_tables(codebooks: np.ndarray, Qx: np.ndarray):
    """(T [Q][M][K], off [Q]) in fp64; codebooks [M][K][s], queries [Q][M*s]."""
    cb = np.asarray(codebooks, dtype=np.float64)
    q = np.asarray(Qx, dtype=np.float64)
    M, K, s = cb.shape
    T = np.empty((q.shape[0], M, K))
    off = np.zeros(q.shape[0])
    for m in range(M):
        ip = q[:, m * s:(m + 1) * s] @ cb[m].T           # [Q, K] = <q_m, c_m(k)>
        B = ip.max(axis=1)
        T[:, m, :] = B[:, None] - ip
        off += B
    return T, off


def inner_products(codebooks: np.ndarray, Qx: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """<q, x_hat> of every (query, code), by decoding x_hat (fp64) -- brute force."""
    cb = np.asarray(codebooks, dtype=np.float64)
    M, K, s = cb.shape
    xh = np.concatenate([cb[m][codes[:, m]] for m in range(M)], axis=1)
    return np.asarray(Qx, dtype=np.float64) @ xh.T
