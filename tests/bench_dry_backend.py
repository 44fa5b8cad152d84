"""CPU stand-in for the GPU kernels in ``bench.py --dry-run`` (test
infrastructure: the oracle computes, bench.py's multi-rank plumbing --
self-launch under torchrun, distributed generation, the first-byte / list
exchange, the list all-gather -- is what the test exercises)."""
import numpy as np

from oracle import ivf as oivf
from oracle import pq, topk


class Backend:
    name = "oracle"

    def train_codebooks(self, X, M, K, iters, seed):
        return pq.train_pq(X, M, K, iters, seed)[0]

    def train_coarse(self, X, nlist, iters, seed):
        return pq.kmeans(X, nlist, iters, seed)[0].astype(np.float32)

    def assign(self, coarse, X):
        return pq.assign(X, coarse)

    def encode(self, cb, X, coarse=None):
        if coarse is None:
            return pq.encode(cb, X), None
        a = pq.assign(X, coarse)
        return pq.encode(cb, X.astype(np.float64) - coarse.astype(np.float64)[a]), a.astype(np.int32)

    def topk(self, cfg, st):
        """Exact top-k of every query over this rank's codes."""
        codes, ids, k = st["codes"], st["ids"], cfg.topk
        Q = len(st["qx"])
        if len(codes) == 0:
            return np.full((Q, k), np.inf), np.full((Q, k), -1, np.int64)
        if not cfg.ivf_nlist:
            return topk.topk(pq.adc(pq.lut64(st["cb"], st["qx"]), codes), ids, k)
        probes = oivf.probe(st["qx"], st["coarse"], cfg.ivf_nprobe)
        D = np.full((Q, k), np.inf)
        I = np.full((Q, k), -1, np.int64)
        for q in range(Q):
            full = np.full(len(codes), np.inf)
            for c in probes[q]:
                m = np.flatnonzero(st["cells"] == c)
                if len(m):
                    r = st["qx"][q].astype(np.float64) - st["coarse"][c].astype(np.float64)
                    full[m] = pq.adc(pq.lut64(st["cb"], r[None]), codes[m])[0]
            fin = np.flatnonzero(np.isfinite(full))
            D[q:q + 1], I[q:q + 1] = topk.topk(full[fin][None], ids[fin], k)
        return D, I

    def merge(self, gd, gi, k):
        return topk.merge(list(gd), list(gi), k)
