"""Product quantization: training, encoding, distance tables and naive ADC.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper passages followed:
* split d dims into M groups, quantize each group with its
  own codebook of K codewords (d/M dims each); encode = one codeword index per
  group; reconstruction = concatenation (zero-padded sum) of the codewords.
* P:92-106 (Eq. 1) -- ADC: the first term, the per-subspace squared distances
  ||q_m - c_m(k)||^2, is "computed only once for all vectors" into the
  "precomputed distance table"; a code's distance is then "M table lookups and
  M-1 addition".  Reading A1: the table is the *subspace* distance, so the sum
  is exactly ||q - x_hat||^2 with no constant term.
* k-means details are not in the paper (reading A15): k-means++ seeding, Lloyd
  iterations, empty cluster -> farthest point, argmin ties -> lowest index.
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------
# k-means (codebook training, P:35-37 / P:80-81; reading A15)
# ----------------------------------------------------------------------------

def _sqdist_f64(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    """All squared distances ||x_i - c_k||^2 in fp64, [n, K].

    Uses the library matmul for speed (||x||^2 - 2 x.c + ||c||^2 in fp64); its
    rounding (~1e-16 relative) only matters for exact ties, which
    ``tests/test_oracle_pq.py`` pins against the direct difference.
    """
    X = X.astype(np.float64)
    C = C.astype(np.float64)
    d = (X * X).sum(1)[:, None] - 2.0 * (X @ C.T) + (C * C).sum(1)[None, :]
    return np.maximum(d, 0.0)


def sqdist_direct(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Direct-difference squared distances sum_j (x_j - c_j)^2, fp64, [n, K]."""
    X = X.astype(np.float64)
    C = C.astype(np.float64)
    return ((X[:, None, :] - C[None, :, :]) ** 2).sum(-1)


def assign(X: np.ndarray, C: np.ndarray, chunk: int = 65536) -> np.ndarray:
    """argmin_k ||x - c_k||^2, ties -> lowest index (np.argmin returns the first)."""
    out = np.empty(len(X), dtype=np.int64)
    for s in range(0, len(X), chunk):
        out[s:s + chunk] = np.argmin(_sqdist_f64(X[s:s + chunk], C), axis=1)
    return out


def objective(X: np.ndarray, C: np.ndarray, a: np.ndarray) -> float:
    """Sum of squared distances to the assigned centroid (direct, fp64)."""
    diff = X.astype(np.float64) - C.astype(np.float64)[a]
    return float((diff * diff).sum())


def kmeans_pp(X: np.ndarray, K: int, seed: int) -> np.ndarray:
    """k-means++ seeding: first centre uniform, then each next centre drawn with
    probability proportional to D(x)^2 (distance to the nearest chosen centre)."""
    rng = np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, 4]))
    X = X.astype(np.float64)
    n = len(X)
    C = np.empty((K, X.shape[1]), dtype=np.float64)
    i0 = int(rng.integers(0, n))
    C[0] = X[i0]
    D = ((X - C[0]) ** 2).sum(1)
    for k in range(1, K):
        tot = D.sum()
        if tot <= 0.0:  # fewer distinct points than K: take any remaining point
            i = int(rng.integers(0, n))
        else:
            u = rng.random() * tot
            i = int(np.searchsorted(np.cumsum(D), u, side="right"))
            i = min(i, n - 1)
        C[k] = X[i]
        D = np.minimum(D, ((X - C[k]) ** 2).sum(1))
    return C


def lloyd(X: np.ndarray, C0: np.ndarray, iters: int):
    """Lloyd iterations.  Returns (C, history) where history[t] is the
    objective after the assignment step of iteration t (non-increasing).

    Empty cluster -> the point farthest from its assigned centroid.
    """
    X = X.astype(np.float64)
    C = C0.astype(np.float64).copy()
    K = len(C)
    hist = []
    for _ in range(iters):
        a = assign(X, C)
        hist.append(objective(X, C, a))
        counts = np.bincount(a, minlength=K)
        sums = np.zeros_like(C)
        np.add.at(sums, a, X)
        newC = C.copy()
        nz = counts > 0
        newC[nz] = sums[nz] / counts[nz][:, None]
        empty = np.flatnonzero(~nz)
        if len(empty):
            far = ((X - C[a]) ** 2).sum(1)
            order = np.argsort(-far, kind="stable")
            for j, e in enumerate(empty):
                newC[e] = X[order[j]]
        C = newC
    return C, hist


def kmeans(X: np.ndarray, K: int, iters: int, seed: int):
    """k-means++ + ``iters`` Lloyd iterations (BASELINE config 1's recipe)."""
    if len(X) < K:
        raise ValueError("insufficient data")
    C0 = kmeans_pp(X, K, seed)
    return lloyd(X, C0, iters)


def train_pq(X: np.ndarray, M: int, K: int, iters: int, seed: int):
    """M independent k-means, one per subspace.

    Returns (codebooks [M, K, d/M] float32, per-subspace objective histories).
    Subspace m uses seed ``seed + m``.
    """
    n, d = X.shape
    if d % M:
        raise ValueError("invalid subspace split")
    if not np.all(np.isfinite(X)):
        raise ValueError("invalid vector")
    s = d // M
    cbs = np.empty((M, K, s), dtype=np.float32)
    hists = []
    for m in range(M):
        C, h = kmeans(X[:, m * s:(m + 1) * s], K, iters, seed + m)
        cbs[m] = C.astype(np.float32)
        hists.append(h)
    return cbs, hists


# ----------------------------------------------------------------------------
# encode / decode
# ----------------------------------------------------------------------------

def encode(codebooks: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Code byte m = argmin_k ||x_m - c_m(k)||^2 (ties -> lowest k), uint8 [n, M]."""
    M, K, s = codebooks.shape
    if X.shape[1] != M * s:
        raise ValueError("dimension error")
    codes = np.empty((len(X), M), dtype=np.uint8)
    for m in range(M):
        codes[:, m] = assign(X[:, m * s:(m + 1) * s], codebooks[m]).astype(np.uint8)
    return codes


def decode(codebooks: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Concatenation of the selected codewords, float32 [n, d]."""
    M, K, s = codebooks.shape
    codes = np.asarray(codes)
    if codes.size and codes.max() >= K:
        raise ValueError("invalid code")
    return np.concatenate([codebooks[m][codes[:, m].astype(np.int64)] for m in range(M)], axis=1)


# ----------------------------------------------------------------------------
# precomputed distance table and naive ADC
# ----------------------------------------------------------------------------

def lut64(codebooks: np.ndarray, Qx: np.ndarray) -> np.ndarray:
    """T[q][m][k] = sum_j (q[m*s+j] - c_m(k)[j])^2 in fp64, [Q, M, K] (the truth)."""
    M, K, s = codebooks.shape
    Qx = np.asarray(Qx, dtype=np.float64)
    if Qx.shape[1] != M * s:
        raise ValueError("dimension error")
    out = np.empty((len(Qx), M, K), dtype=np.float64)
    C = codebooks.astype(np.float64)
    for m in range(M):
        qm = Qx[:, m * s:(m + 1) * s]
        for q0 in range(0, len(Qx), 256):
            diff = qm[q0:q0 + 256, None, :] - C[m][None, :, :]
            out[q0:q0 + 256, m] = (diff * diff).sum(-1)
    return out


def lut32(codebooks: np.ndarray, Qx: np.ndarray) -> np.ndarray:
    """Paper-faithful fp32 table (P:234 declares ``float``): for j ascending,
    ``t = q_j - c_j; acc = acc + t*t`` with each operation rounded to fp32 (no
    fused multiply-add), [Q, M, K] float32."""
    M, K, s = codebooks.shape
    Qx = np.asarray(Qx, dtype=np.float32)
    C = codebooks.astype(np.float32)
    out = np.zeros((len(Qx), M, K), dtype=np.float32)
    for m in range(M):
        acc = np.zeros((len(Qx), K), dtype=np.float32)
        for j in range(s):
            t = Qx[:, m * s + j][:, None] - C[m][None, :, j]
            acc = acc + t * t
        out[:, m] = acc
    return out


def adc(table: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Naive ADC scan: out[q][i] = sum_{m=0..M-1} T[q][m][code_i[m]],
    summed left to right (m ascending) in the table's dtype.  [Q, N]."""
    table = np.asarray(table)
    codes = np.asarray(codes).astype(np.int64)
    Q, M, K = table.shape
    if codes.shape[1] != M:
        raise ValueError("config error")
    out = table[:, 0, :][:, codes[:, 0]]
    for m in range(1, M):
        out = out + table[:, m, :][:, codes[:, m]]
    return out


def adc_one(table_q: np.ndarray, code) -> float:
    """One code's ADC distance (M lookups, M-1 additions), table_q [M, K]."""
    acc = table_q[0, int(code[0])]
    for m in range(1, len(code)):
        acc = acc + table_q[m, int(code[m])]
    return acc


def exact_sqdist(Qx: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Brute-force ||q - x||^2 in fp64, [Q, N] (used by the exact-L2 pin)."""
    Qx = np.asarray(Qx, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    return ((Qx[:, None, :] - X[None, :, :]) ** 2).sum(-1)
