"""CPU-only checks of the C ABI library: it loads, exports every symbol that
include/etree.h declares, and its host-side build (independent C++) reproduces
the oracle's tree statistics exactly."""
import os
import re

import numpy as np
import pytest

from oracle import etree as oetree
from paper_1509_05186_b200 import _lib, api, build, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "etree.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(et_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED, f"{name} missing from the ctypes binding"
    assert set(_lib.EXPORTED) <= set(decl)


def test_version_and_errors(lib):
    assert b"sm_100a" in lib.et_version()
    with pytest.raises(_lib.EtError, match="EMPTY"):
        api.et_build_stats(np.zeros((0, 8), np.uint8))
    with pytest.raises(_lib.EtError, match="CONFIG"):
        api.et_build_stats(np.zeros((4, 12), np.uint8))          # single tree deeper than 8
    with pytest.raises(_lib.EtError, match="INVALID_CODE"):
        api.et_build_stats(np.full((3, 4), 20, np.uint8), K=16)
    with pytest.raises(_lib.EtError, match="CONFIG"):
        api.et_build_stats(np.zeros((3, 4), np.uint8), split=[0, 2, 2, 4])
    with pytest.raises(_lib.EtError, match="CONFIG"):
        api.et_build_stats(np.zeros((3, 4), np.uint8), ids=[1, -1, 2])


def _oracle_stats(codes, split):
    out = []
    for a, b in zip(split, split[1:]):
        sc, _ = oetree.sort_codes(codes[:, a:b])
        out.append(oetree.tree_stats_def(sc))
    return out


CASES = [
    (1, 3000, 8, 256, None, (0, 8)),
    (2, 5000, 8, 8, None, (0, 8)),
    (3, 4000, 8, 256, 50, (0, 8)),           # duplicate heavy, chained records
    (4, 3000, 16, 16, None, (0, 8, 16)),     # forest of two 8-byte trees
    (5, 2000, 8, 4, None, (0, 4, 8)),
    (6, 1, 4, 256, None, (0, 4)),
    (7, 2500, 6, 3, None, (0, 2, 5, 6)),
]


@pytest.mark.parametrize("seed,N,M,K,nd,split", CASES)
def test_host_build_stats_match_oracle(lib, seed, N, M, K, nd, split):
    codes = synth.random_codes(seed, N, M, K, nd)
    got = api.et_build_stats(codes, split=list(split), K=K)
    ref = _oracle_stats(codes, split)
    for g, r in zip(got, ref):
        assert (g["N"], g["L1"], g["L2"], g["total_postfix"], g["lookups"], g["L2_records"], g["paper_bytes"]) == \
               (N, r.L1, r.L2, r.total_postfix, r.lookups, r.L2_records, r.paper_bytes)


def test_host_build_spec_example(lib):
    from golden_io import load
    M, codes, exp = load("spec_example.txt")
    st = api.et_build_stats(codes)[0]
    assert st["L1"] == 3 and st["L2"] == 4 and st["total_postfix"] == 4 and st["paper_bytes"] == 34


def test_host_build_uniform_u1m_scale(lib):
    """U1M companion at 1/5 scale: stats equal the oracle's plain definition."""
    codes = synth.uniform_codes(synth.CONFIGS["u1m"], 200_000)
    g = api.et_build_stats(codes)[0]
    sc, _ = oetree.sort_codes(codes)
    r = oetree.tree_stats_def(sc)
    assert (g["L1"], g["L2"], g["total_postfix"]) == (r.L1, r.L2, r.total_postfix)


@pytest.mark.parametrize("seed,N,M,K,nd,split", [c for c in CASES if len(c[5]) > 2 and c[5][-1] <= 8])
def test_fused_forest_scan_lookups(lib, seed, N, M, K, nd, split):
    """Fused E-Forest (M <= 8): the scan's lookups per query
    are each tree's Distance Context run along the distinct full codes in
    lexicographic order -- sum over tuples of sum over trees of
    (tree width - LCP with the previous tuple over that tree's bytes).  For
    T = 1 this is exactly L1 + L2 + postfix."""
    codes = synth.random_codes(seed, N, M, K, nd)
    U = np.unique(codes, axis=0)          # distinct full codes, lexicographic
    exp = 0
    for i in range(len(U)):
        for a, b in zip(split, split[1:]):
            l = 0
            if i:
                while a + l < b and U[i, a + l] == U[i - 1, a + l]:
                    l += 1
            exp += (b - a) - l
    got = api.et_build_stats(codes, split=list(split), K=K)
    assert all(g["scan_lookups"] == exp for g in got)
    t1 = api.et_build_stats(codes, K=K)[0]
    assert t1["scan_lookups"] == t1["lookups"]


@pytest.mark.parametrize("split", [(0, 8), (0, 3, 8)])
def test_byte_perm_stats_match_oracle_on_permuted_codes(lib, split):
    """Encoding ordering (A21): building over a chunk permutation
    equals building over the codes with their columns permuted first."""
    codes = synth.random_codes(11, 4000, 8, 16, 300)
    perm = np.random.default_rng(5).permutation(8).astype(np.int32)
    got = api.et_build_stats(codes, split=list(split), K=16, byte_perm=perm)
    ref = _oracle_stats(np.ascontiguousarray(codes[:, perm]), split)
    for g, r in zip(got, ref):
        assert (g["L1"], g["L2"], g["total_postfix"], g["lookups"]) == (r.L1, r.L2, r.total_postfix, r.lookups)
