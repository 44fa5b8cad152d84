"""Leaf extra byte: extra information stored on the
E-Tree's leaf nodes and added to the distance.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper passages followed:
* Additive Quantization "doesn't decompose data space into
  orthogonal subspaces ... it makes the third term in equation 1 non-zero,
  requiring additional information to be stored along with the encoded
  dataset".
* "For Additive Quantization we quantized on the extra
  information to 1 Byte ... and store the extra information on the leaf node."
* P:92-96 (Eq. 1, reading A1 with (M-1)):
      ||q - x_hat||^2 = sum_m ||q - c_m(i_m)||^2 - (M-1)||q||^2
                        + sum_{i != j} c_i^T c_j ,   x_hat = sum_m c_m(i_m).

Operation: a vector carries one extra byte e next to its M-byte code; a decode
table E[256] turns it into an additive term, and the distance of a code is the
table sum plus that term,
      D(q, i) = sum_m T[q][m][code_i[m]] + E[e_i]                       (1)
(the sum over m in order, then + E).  Stored on the leaf, the byte is shared
by the leaf's vectors: it must be a function of the code (`leaf_extra`).
With AQ tables T[q][m][k] = ||q - c_m(k)||^2 over all d dimensions and E = the
cross term of Eq. 1, (1) equals ||q - x_hat||^2 + (M-1)||q||^2 (a per-query
constant): the ranking is the exact AQ one.
"""
from __future__ import annotations

import numpy as np

from . import pq


def adc_extra(table: np.ndarray, codes: np.ndarray, extra: np.ndarray, etab: np.ndarray) -> np.ndarray:
    """(1): naive ADC (m ascending) plus the decoded extra byte, [Q, n]."""
    return pq.adc(table, codes) + np.asarray(etab, dtype=table.dtype)[np.asarray(extra, dtype=np.int64)][None, :]


def leaf_extra(codes: np.ndarray, extra: np.ndarray) -> dict:
    """The extra byte of every distinct code; raises ValueError if two vectors
    with the same code carry different bytes (the leaf holds one byte)."""
    out: dict = {}
    for row, e in zip(map(bytes, np.asarray(codes, dtype=np.uint8)), np.asarray(extra, dtype=np.uint8)):
        if out.setdefault(row, int(e)) != int(e):
            raise ValueError("extra byte differs among vectors with the same code")
    return out


# ---------------------------------------------------------------------------
# Additive quantization pieces: full-dimensional codebooks
# ---------------------------------------------------------------------------

def aq_decode(codebooks: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """x_hat = sum_m c_m(code[m]) (codebooks [M][K][d], fp64)."""
    cb = np.asarray(codebooks, dtype=np.float64)
    out = np.zeros((codes.shape[0], cb.shape[2]))
    for m in range(cb.shape[0]):
        out += cb[m][codes[:, m]]
    return out


def aq_tables(codebooks: np.ndarray, Qx: np.ndarray) -> np.ndarray:
    """T[q][m][k] = ||q - c_m(k)||^2 over all d dimensions (fp64), by direct
    differences."""
    cb = np.asarray(codebooks, dtype=np.float64)
    q = np.asarray(Qx, dtype=np.float64)
    M, K, _ = cb.shape
    T = np.empty((q.shape[0], M, K))
    for m in range(M):
        diff = q[:, None, :] - cb[m][None, :, :]
        T[:, m, :] = np.einsum("qkd,qkd->qk", diff, diff)
    return T


def aq_cross(codebooks: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Eq. 1's third term sum_{i != j} c_i^T c_j of every code (fp64)."""
    cb = np.asarray(codebooks, dtype=np.float64)
    M = cb.shape[0]
    out = np.zeros(codes.shape[0])
    for i in range(M):
        for j in range(M):
            if i != j:
                out += np.einsum("nd,nd->n", cb[i][codes[:, i]], cb[j][codes[:, j]])
    return out


def quantize_extra(values: np.ndarray, levels: int = 256):
    """1-byte scalar quantization of the extra information: uniform
    levels over [min, max] shifted to start at 0 -- bytes e and the decode
    table E (E[0] = 0, so every decoded term is >= 0; the shift min(values) is
    a per-dataset constant that leaves every ranking unchanged).  Returns
    (e uint8 [n], E float64 [256], shift)."""
    v = np.asarray(values, dtype=np.float64)
    lo, hi = float(v.min()), float(v.max())
    step = (hi - lo) / (levels - 1) if hi > lo else 1.0
    e = np.clip(np.rint((v - lo) / step), 0, levels - 1).astype(np.uint8)
    E = np.arange(256, dtype=np.float64) * step
    return e, E, lo
