"""ctypes binding of libetree.so (include/etree.h): argument marshalling only.

Loading fails loudly if the library was not built -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ET_LIB_PATH") or os.path.join(HERE, "_build", "libetree.so")  # override: experiment builds

ET_STATUS = {
    0: "ET_OK", 1: "ET_ERR_INSUFFICIENT_DATA", 2: "ET_ERR_SUBSPACE_SPLIT",
    3: "ET_ERR_INVALID_VECTOR", 4: "ET_ERR_DIMENSION", 5: "ET_ERR_INVALID_CODE",
    6: "ET_ERR_CONFIG", 7: "ET_ERR_PRECONDITION", 8: "ET_ERR_EMPTY", 9: "ET_ERR_CORRUPT",
    10: "ET_ERR_CUDA", 11: "ET_ERR_OOM", 12: "ET_ERR_WORKSPACE",
}


class EtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{ET_STATUS.get(status, status)}: {msg}")
        self.status = status


class TreeStats(C.Structure):
    _fields_ = [
        ("N", C.c_int64), ("M", C.c_int32), ("layer0", C.c_int32),
        ("L1", C.c_int64), ("L2", C.c_int64), ("total_postfix", C.c_int64),
        ("lookups", C.c_int64), ("L2_records", C.c_int64), ("paper_bytes", C.c_int64),
        ("device_bytes", C.c_int64), ("groups", C.c_int64), ("scan_lookups", C.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
U64 = C.c_uint64
SZ = C.c_size_t

# (name, restype, argtypes) -- mirrors include/etree.h
SIGNATURES = [
    ("et_last_error", C.c_char_p, []),
    ("et_version", C.c_char_p, []),
    ("et_launch_count", I64, []),
    ("et_timing_enable", None, [C.c_int]),
    ("et_timing_reset", None, []),
    ("et_timing_get", C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(I64)]),
    ("et_build_codebooks", C.c_int, [P, I64, I32, I32, I32, I32, U64, P, P]),
    ("et_build_coarse", C.c_int, [P, I64, I32, I32, I32, U64, P, P]),
    ("et_encode", C.c_int, [P, I32, I32, I32, P, I64, P, P, P, P]),
    ("et_assign", C.c_int, [P, I32, I32, P, I64, P, P]),
    ("et_build_etree", C.c_int, [P, P, I64, I32, I32, P, C.POINTER(P)]),
    ("et_build_eforest", C.c_int, [P, P, I64, I32, I32, P, I32, P, C.POINTER(P)]),
    ("et_build_flat", C.c_int, [P, P, I64, I32, I32, C.POINTER(P)]),
    ("et_build_ivf", C.c_int, [P, P, I64, I32, I32, P, I32, P, I32, P, C.POINTER(P)]),
    ("et_index_stats", C.c_int, [P, I32, C.POINTER(TreeStats)]),
    ("et_build_stats", C.c_int, [P, P, I64, I32, I32, P, I32, P, C.POINTER(TreeStats)]),
    ("et_index_info", C.c_int, [P, C.POINTER(I32), C.POINTER(I64), C.POINTER(I32),
                                C.POINTER(I32), C.POINTER(I64), C.POINTER(I32)]),
    ("et_index_free", None, [P]),
    ("et_compute_luts", C.c_int, [P, I32, I32, I32, P, I64, P, P]),
    ("et_workspace_size", C.c_int, [P, I64, I32, I32, C.POINTER(SZ)]),
    ("et_plan_info", C.c_int, [P, I64, I32, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32)]),
    ("et_index_set_extra", C.c_int, [P, P, I64]),
    ("et_compute_ip_luts", C.c_int, [P, I32, I32, I32, P, I64, P, P, P]),
    ("et_etree_topk_extra", C.c_int, [P, P, I32, P, P, I64, I32, P, P, P, P, SZ, P]),
    ("et_etree_distances", C.c_int, [P, P, I32, P, P, I64, P, P, SZ, P]),
    ("et_etree_topk", C.c_int, [P, P, I32, P, P, I64, I32, P, P, P, SZ, P]),
    ("et_host_batches", C.c_int, [I64, I32, C.POINTER(I32)]),
    ("et_etree_topk_host", C.c_int, [P, P, I32, P, I64, I32, P, P, I32, P, P, P, P, SZ, P]),
    ("et_ivf_topk", C.c_int, [P, P, I64, I32, I32, P, P, P, P, SZ, P]),
    ("et_merge_topk", C.c_int, [P, P, I32, I64, I32, P, P, P]),
    ("et_flat_adc", C.c_int, [P, I64, I32, I32, P, I64, P, P]),
    ("et_shard_bounds", C.c_int, [P, I64, I32, I32, I32, P]),
    ("et_shard_lists", C.c_int, [P, I32, I32, P]),
    ("et_shard_bounds_hist", C.c_int, [P, I32, I32, P]),
]

EXPORTED = [s[0] for s in SIGNATURES]

_lib = None


def load(path: str = LIB_PATH):
    """Load libetree.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libetree.so not found at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != 0:
        raise EtError(status, load().et_last_error().decode())
