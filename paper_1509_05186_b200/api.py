"""Thin PyTorch-facing binding of libetree (same names as the C ABI).

Only argument marshalling happens here: torch tensors provide device memory
and the current CUDA stream; every step of the hot path runs in the CUDA
kernels of libetree.so.  Builds take host (numpy) arrays -- the index build is
an offline C++ step (include/etree.h).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check

_torch = None


def _t():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream(stream=None) -> Optional[int]:
    torch = _t()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _dev(x, dtype):
    if not (x.is_cuda and x.is_contiguous() and x.dtype == dtype):
        raise ValueError(f"expected a contiguous CUDA {dtype} tensor, got {x.dtype} on {x.device} "
                         f"(contiguous={x.is_contiguous()})")
    return x


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def version() -> str:
    return _lib.load().et_version().decode()


def et_host_batches(Q: int, n_batches: int = 0) -> int:
    """Batches et_etree_topk_host uses for Q queries (n_batches <= 0: the default)."""
    out = C.c_int32()
    check(_lib.load().et_host_batches(Q, n_batches, C.byref(out)))
    return out.value


def et_launch_count() -> int:
    return int(_lib.load().et_launch_count())


def et_timing_enable(on: bool = True):
    _lib.load().et_timing_enable(1 if on else 0)


def et_timing_reset():
    _lib.load().et_timing_reset()


def et_timing_get(name: str):
    """(total ms, launches) of kernel ``name`` since the last reset."""
    ms, n = C.c_double(), C.c_int64()
    _lib.load().et_timing_get(name.encode(), C.byref(ms), C.byref(n))
    return ms.value, n.value


class Index:
    """An E-Tree / E-Forest / flat / IVF index owned by libetree (device memory)."""

    def __init__(self, handle: int, kind: str, keep=()):
        self._h = C.c_void_p(handle)
        self.kind = kind
        self._keep = keep
        T, n, M, K, G, nl = C.c_int32(), C.c_int64(), C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
        check(_lib.load().et_index_info(self._h, C.byref(T), C.byref(n), C.byref(M), C.byref(K),
                                        C.byref(G), C.byref(nl)))
        self.T, self.N, self.M, self.K = T.value, n.value, M.value, K.value
        self.groups, self.nlist = G.value, nl.value
        self._ws = {}   # one workspace per (device, stream): a call in flight owns its workspace

    # ---------------------------------------------------------------- builds
    @staticmethod
    def _codes(codes, ids):
        codes = _host(codes, np.uint8)
        n, M = codes.shape
        ids_a = None if ids is None else _host(ids, np.int32)
        if ids_a is not None and len(ids_a) != n:
            raise ValueError("ids length")
        return codes, ids_a, n, M

    @classmethod
    def et_build_etree(cls, codes, ids=None, K: int = 256, byte_perm=None) -> "Index":
        codes, ids_a, n, M = cls._codes(codes, ids)
        perm = None if byte_perm is None else _host(byte_perm, np.int32)
        h = C.c_void_p()
        check(_lib.load().et_build_etree(_ptr(codes), _ptr(ids_a), n, M, K, _ptr(perm), C.byref(h)))
        return cls(h.value, "etree")

    @classmethod
    def et_build_eforest(cls, codes, split: Sequence[int], ids=None, K: int = 256, byte_perm=None) -> "Index":
        codes, ids_a, n, M = cls._codes(codes, ids)
        sp = _host(split, np.int32)
        perm = None if byte_perm is None else _host(byte_perm, np.int32)
        h = C.c_void_p()
        check(_lib.load().et_build_eforest(_ptr(codes), _ptr(ids_a), n, M, K, _ptr(perm),
                                           len(sp) - 1, _ptr(sp), C.byref(h)))
        return cls(h.value, "eforest")

    @classmethod
    def et_build_flat(cls, codes, ids=None, K: int = 256) -> "Index":
        codes, ids_a, n, M = cls._codes(codes, ids)
        h = C.c_void_p()
        check(_lib.load().et_build_flat(_ptr(codes), _ptr(ids_a), n, M, K, C.byref(h)))
        return cls(h.value, "flat")

    @classmethod
    def et_build_ivf(cls, codes, list_of, coarse, codebooks, ids=None, K: int = 256) -> "Index":
        codes, ids_a, n, M = cls._codes(codes, ids)
        lo = _host(list_of, np.int32)
        co = _host(coarse, np.float32)
        cb = _host(codebooks, np.float32)
        h = C.c_void_p()
        check(_lib.load().et_build_ivf(_ptr(codes), _ptr(ids_a), n, M, K, _ptr(lo), co.shape[0],
                                       _ptr(co), co.shape[1], _ptr(cb), C.byref(h)))
        return cls(h.value, "ivf")

    def free(self):
        if self._h is not None and self._h.value:
            _lib.load().et_index_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # ---------------------------------------------------------------- info
    def et_index_stats(self, tree: int = 0) -> dict:
        st = _lib.TreeStats()
        check(_lib.load().et_index_stats(self._h, tree, C.byref(st)))
        return st.as_dict()

    def stats(self):
        return [self.et_index_stats(t) for t in range(self.T)]

    def et_plan_info(self, Q: int, k: int) -> dict:
        """The launch plan of et_etree_topk (k > 0) / et_etree_distances (k <= 0)."""
        c, s, ns = C.c_int32(), C.c_int32(), C.c_int32()
        check(_lib.load().et_plan_info(self._h, Q, k, C.byref(c), C.byref(s), C.byref(ns)))
        return {"chunks": c.value, "S": s.value, "streams": ns.value}

    def et_workspace_size(self, Q: int, k: int, nprobe: int = 0) -> int:
        b = C.c_size_t()
        check(_lib.load().et_workspace_size(self._h, Q, k, nprobe, C.byref(b)))
        return b.value

    def _workspace(self, nbytes: int, device, stream=None):
        """Workspace for a call on ``stream`` (etree.h: one workspace per call
        in flight).  Cached per (device, stream); when it grows, the old block
        is released with record_stream so the caching allocator cannot hand
        it out while a kernel on that stream may still read it."""
        torch = _t()
        s = torch.cuda.current_stream(device) if stream is None else stream
        key = (device, s.cuda_stream)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            if ws is not None:
                ws.record_stream(s)
            with torch.cuda.stream(s):
                ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._ws[key] = ws
        return ws

    # ---------------------------------------------------------------- queries
    def et_index_set_extra(self, extra) -> None:
        """Leaf extra byte per database vector: uint8 [N] (host)."""
        e = np.ascontiguousarray(extra, dtype=np.uint8)
        check(_lib.load().et_index_set_extra(self._h, e.ctypes.data, int(e.shape[0])))

    def et_etree_topk(self, k: int, queries=None, codebooks=None, luts=None, out=None, stream=None,
                      extra_table=None):
        """(dist [Q,k] fp32, ids [Q,k] int32) on the queries' device.  extra_table:
        the leaf extra byte's decode table (device fp32 [256]; et_etree_topk_extra)."""
        torch = _t()
        ref = luts if luts is not None else queries
        Q = ref.shape[0]
        d = 0 if queries is None else queries.shape[1]
        if queries is not None:
            _dev(queries, torch.float32)
            _dev(codebooks, torch.float32)
        if luts is not None:
            _dev(luts, torch.float32)
        if out is None:
            dist = torch.empty((Q, k), dtype=torch.float32, device=ref.device)
            ids = torch.empty((Q, k), dtype=torch.int32, device=ref.device)
        else:
            dist, ids = out
        nb = self.et_workspace_size(Q, k)
        ws = self._workspace(nb, ref.device, stream)
        if extra_table is not None:
            _dev(extra_table, torch.float32)
            if extra_table.numel() != 256:
                raise ValueError("extra_table must hold 256 entries")
            check(_lib.load().et_etree_topk_extra(self._h, _ptr(codebooks), d, _ptr(luts), _ptr(queries), Q, k,
                                                  _ptr(extra_table), _ptr(dist), _ptr(ids), _ptr(ws), ws.numel(),
                                                  _stream(stream)))
            return dist, ids
        check(_lib.load().et_etree_topk(self._h, _ptr(codebooks), d, _ptr(luts), _ptr(queries), Q, k,
                                        _ptr(dist), _ptr(ids), _ptr(ws), ws.numel(), _stream(stream)))
        return dist, ids

    def et_etree_topk_host(self, k: int, queries_host, codebooks, out=None, n_batches: int = 0, stream=None):
        """et_etree_topk from host buffers (etree.h et_etree_topk_host): queries_host
        is a CPU fp32 [Q, d] tensor (pinned for the copies to overlap the search);
        returns host (dist [Q,k] fp32, ids [Q,k] int32), complete once ``stream``
        (default: the current stream) passes the call.  Device staging buffers
        are cached per (device, stream, shape)."""
        torch = _t()
        if queries_host.is_cuda or not queries_host.is_contiguous() or queries_host.dtype != torch.float32:
            raise ValueError("queries_host must be a contiguous CPU float32 tensor")
        _dev(codebooks, torch.float32)
        Q, d = queries_host.shape
        dev = codebooks.device
        if out is None:
            dist_h = torch.empty((Q, k), dtype=torch.float32).pin_memory()
            ids_h = torch.empty((Q, k), dtype=torch.int32).pin_memory()
        else:
            dist_h, ids_h = out
            for t, dt in ((dist_h, torch.float32), (ids_h, torch.int32)):
                if t.is_cuda or not t.is_contiguous() or t.dtype != dt or tuple(t.shape) != (Q, k):
                    raise ValueError(f"host outputs must be contiguous CPU {dt} tensors of shape {(Q, k)}")
        nbat = C.c_int32()
        check(_lib.load().et_host_batches(Q, n_batches, C.byref(nbat)))
        qmax = -(-Q // max(1, nbat.value))
        nb = self.et_workspace_size(qmax, k)
        ws = self._workspace(nb, dev, stream)
        s = torch.cuda.current_stream(dev) if stream is None else stream
        key = ("host", dev, s.cuda_stream, Q, d, k)
        stg = self._ws.get(key)
        if stg is None:
            with torch.cuda.stream(s):
                stg = (torch.empty((Q, d), dtype=torch.float32, device=dev),
                       torch.empty((Q, k), dtype=torch.float32, device=dev),
                       torch.empty((Q, k), dtype=torch.int32, device=dev))
            self._ws[key] = stg
        qd, dd, idd = stg
        check(_lib.load().et_etree_topk_host(self._h, _ptr(codebooks), d, _ptr(queries_host), Q, k, _ptr(dist_h),
                                             _ptr(ids_h), nbat.value, _ptr(qd), _ptr(dd), _ptr(idd), _ptr(ws),
                                             ws.numel(), _stream(stream)))
        return dist_h, ids_h

    def et_etree_distances(self, queries=None, codebooks=None, luts=None, out=None, stream=None):
        """Full output [Q, N] fp32 indexed by slot."""
        torch = _t()
        ref = luts if luts is not None else queries
        Q = ref.shape[0]
        d = 0 if queries is None else queries.shape[1]
        if out is None:
            out = torch.empty((Q, self.N), dtype=torch.float32, device=ref.device)
        nb = self.et_workspace_size(Q, 0)
        ws = self._workspace(nb, ref.device, stream)
        check(_lib.load().et_etree_distances(self._h, _ptr(codebooks), d, _ptr(luts), _ptr(queries), Q,
                                             _ptr(out), _ptr(ws), ws.numel(), _stream(stream)))
        return out

    def et_ivf_topk(self, queries, nprobe: int, k: int, stream=None, return_probes=False):
        torch = _t()
        _dev(queries, torch.float32)
        Q = queries.shape[0]
        dist = torch.empty((Q, k), dtype=torch.float32, device=queries.device)
        ids = torch.empty((Q, k), dtype=torch.int32, device=queries.device)
        probes = torch.empty((Q, nprobe), dtype=torch.int32, device=queries.device)
        nb = self.et_workspace_size(Q, k, nprobe)
        ws = self._workspace(nb, queries.device, stream)
        check(_lib.load().et_ivf_topk(self._h, _ptr(queries), Q, nprobe, k, _ptr(dist), _ptr(ids),
                                      _ptr(probes), _ptr(ws), ws.numel(), _stream(stream)))
        return (dist, ids, probes) if return_probes else (dist, ids)


# -------------------------------------------------------------------- free functions

def et_compute_luts(codebooks, queries, stream=None):
    torch = _t()
    _dev(codebooks, torch.float32)
    _dev(queries, torch.float32)
    M, K, s = codebooks.shape
    Q, d = queries.shape
    luts = torch.empty((Q, M, K), dtype=torch.float32, device=queries.device)
    check(_lib.load().et_compute_luts(_ptr(codebooks), d, M, K, _ptr(queries), Q, _ptr(luts), _stream(stream)))
    return luts


def et_compute_ip_luts(codebooks, queries, stream=None):
    """(luts [Q,M,K], offsets [Q]): shifted inner-product tables (reading A26);
    et_etree_topk(luts=luts) then ranks by largest <q, x_hat> = offsets - dist."""
    torch = _t()
    _dev(codebooks, torch.float32)
    _dev(queries, torch.float32)
    M, K, s = codebooks.shape
    Q, d = queries.shape
    luts = torch.empty((Q, M, K), dtype=torch.float32, device=queries.device)
    off = torch.empty((Q,), dtype=torch.float32, device=queries.device)
    check(_lib.load().et_compute_ip_luts(_ptr(codebooks), d, M, K, _ptr(queries), Q, _ptr(luts), _ptr(off),
                                         _stream(stream)))
    return luts, off


def et_encode(codebooks, x, centroids=None, assign=None, stream=None):
    torch = _t()
    _dev(codebooks, torch.float32)
    _dev(x, torch.float32)
    M, K, s = codebooks.shape
    n, d = x.shape
    codes = torch.empty((n, M), dtype=torch.uint8, device=x.device)
    check(_lib.load().et_encode(_ptr(codebooks), d, M, K, _ptr(x), n, _ptr(centroids), _ptr(assign),
                                _ptr(codes), _stream(stream)))
    return codes


def et_assign(centroids, x, stream=None):
    torch = _t()
    _dev(centroids, torch.float32)
    _dev(x, torch.float32)
    n, d = x.shape
    a = torch.empty((n,), dtype=torch.int32, device=x.device)
    check(_lib.load().et_assign(_ptr(centroids), centroids.shape[0], d, _ptr(x), n, _ptr(a), _stream(stream)))
    return a


def et_build_codebooks(train, M: int, K: int, lloyd_iters: int, seed: int):
    """Host fp32 [n, d] -> (codebooks [M, K, d/M] float32, objective history [M, iters])."""
    train = _host(train, np.float32)
    n, d = train.shape
    cb = np.empty((M, K, d // M if M else 0), dtype=np.float32)
    hist = np.empty((M, lloyd_iters), dtype=np.float64)
    check(_lib.load().et_build_codebooks(_ptr(train), n, d, M, K, lloyd_iters, seed & (2**64 - 1),
                                         _ptr(cb), _ptr(hist)))
    return cb, hist


def et_build_stats(codes, split=None, ids=None, K: int = 256, byte_perm=None):
    """Host-only build statistics (no GPU): list of per-tree dicts."""
    codes = _host(codes, np.uint8)
    n, M = codes.shape
    sp = _host([0, M] if split is None else split, np.int32)
    T = len(sp) - 1
    ids_a = None if ids is None else _host(ids, np.int32)
    perm = None if byte_perm is None else _host(byte_perm, np.int32)
    out = (_lib.TreeStats * T)()
    check(_lib.load().et_build_stats(_ptr(codes), _ptr(ids_a), n, M, K, _ptr(perm), T, _ptr(sp), out))
    return [out[t].as_dict() for t in range(T)]


def et_build_coarse(train, nlist: int, lloyd_iters: int, seed: int):
    """Host fp32 [n, d] -> (centroids [nlist, d] float32, objective history [iters])."""
    train = _host(train, np.float32)
    n, d = train.shape
    c = np.empty((nlist, d), dtype=np.float32)
    hist = np.empty((lloyd_iters,), dtype=np.float64)
    check(_lib.load().et_build_coarse(_ptr(train), n, d, nlist, lloyd_iters, seed & (2**64 - 1),
                                      _ptr(c), _ptr(hist)))
    return c, hist


def et_merge_topk(dist, ids, stream=None):
    """dist/ids [G, Q, k] (e.g. all-gathered shards) -> merged [Q, k].

    float32 distances and int32 ids on one CUDA device; non-contiguous inputs
    are copied to locals that stay alive until the launch has been enqueued
    on ``stream`` (the caching allocator then orders any reuse after it)."""
    torch = _t()
    if dist.dim() != 3 or ids.shape != dist.shape:
        raise ValueError(f"et_merge_topk: need dist/ids of equal shape [G, Q, k], got {tuple(dist.shape)} / {tuple(ids.shape)}")
    if dist.device != ids.device or not dist.is_cuda:
        raise ValueError("et_merge_topk: dist and ids must be on the same CUDA device")
    dc = _dev(dist.contiguous(), torch.float32)
    ic = _dev(ids.contiguous(), torch.int32)
    G, Q, k = dc.shape
    od = torch.empty((Q, k), dtype=torch.float32, device=dc.device)
    oi = torch.empty((Q, k), dtype=torch.int32, device=dc.device)
    st = _stream(stream)
    check(_lib.load().et_merge_topk(_ptr(dc), _ptr(ic), G, Q, k, _ptr(od), _ptr(oi), st))
    if stream is not None:   # temporaries used on a side stream: keep them alive there
        dc.record_stream(stream)
        ic.record_stream(stream)
    return od, oi


def et_flat_adc(luts, codes, stream=None):
    torch = _t()
    Q, M, K = luts.shape
    n = codes.shape[0]
    out = torch.empty((Q, n), dtype=torch.float32, device=luts.device)
    check(_lib.load().et_flat_adc(_ptr(luts), Q, M, K, _ptr(codes), n, _ptr(out), _stream(stream)))
    return out


def et_shard_bounds(codes, G: int, K: int = 256) -> np.ndarray:
    """Host shard plan by first-level subtree: int32 [G+1] byte bounds."""
    codes = _host(codes, np.uint8)
    n, M = codes.shape if codes.ndim == 2 else (codes.shape[0], 1)
    b = np.empty(G + 1, dtype=np.int32)
    check(_lib.load().et_shard_bounds(_ptr(codes), n, M, G, K, _ptr(b)))
    return b


def et_shard_lists(list_sizes, G: int) -> np.ndarray:
    """Host IVF shard plan (LPT on list size): int32 [nlist] owner rank."""
    ls = _host(list_sizes, np.int64)
    owner = np.empty(len(ls), dtype=np.int32)
    check(_lib.load().et_shard_lists(_ptr(ls), len(ls), G, _ptr(owner)))
    return owner


def et_shard_bounds_hist(hist, G: int) -> np.ndarray:
    """Shard bounds from a first-byte histogram (int64 [K])."""
    h = _host(hist, np.int64)
    b = np.empty(G + 1, dtype=np.int32)
    check(_lib.load().et_shard_bounds_hist(_ptr(h), len(h), G, _ptr(b)))
    return b
