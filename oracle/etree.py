"""Encoding Tree: construction, Hierarchical Memory Structure, traversal.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Two independent constructions of the same tree are kept so each checks the
other:

* ``tree_stats_def`` -- the plain definition (reading A4): a node of depth l
  (0-based; it consumes code byte l) is *internal* iff the length-(l+1) prefix
  is shared by >= 2 distinct codes; every distinct code is one leaf whose depth
  is the length of its longest common prefix with a neighbour in sorted order;
  its postfix holds the remaining M-1-depth bytes.
* ``build_alg1`` -- Algorithm 1 step by step: per sorted code,
  LCP with ``lastPath``, "Merge lastPath{l+1..M}", create nodes, associate the
  vector with ``lastPath{M}``; the merge compresses every node whose subtree
  holds exactly one distinct code into a leaf (A4).

``serialize`` writes the Hierarchical Memory Structure (Fig. 1
caption P:123): records in depth-first order, internal record
``[K][depth<<1 | 0]`` (2 bytes), leaf record ``[K][n'<<1 | 1][postfix][n' x
u32 ids]``.  Readings: A7 children are emitted *leaves first* so a leaf's depth
is always (depth of the last internal record) + 1 -- the format as printed is
otherwise undecodable; A8 ids are 4-byte little-endian (the text's 4N bytes,
P:222); A9 a leaf holding more than 127 ids is chained into consecutive records
with the same K/postfix.  Memory identity: ``len == 4N + 2(L1 + L2) + sum
postfix`` (L2 and postfix counted per record).

``traverse`` is the Distance-Context pseudocode with readings A2
(table indexed by layer), A3 (a leaf at depth l reads K at layer l and a
postfix of M-1-l bytes at layers l+1..M-1), A5 (virtual root, ctx[-1] = 0),
A10 (advance 2 + postfix + 4 n' bytes) and A11 (stop at end of buffer).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


# ----------------------------------------------------------------------------
# sorting (Algorithm 1 input "in lexicographic order")
# ----------------------------------------------------------------------------

def sort_codes(codes: np.ndarray, ids: Optional[np.ndarray] = None,
               order: Optional[np.ndarray] = None):
    """Permute code bytes by ``order`` (identity default; P:358-371 chunk
    ordering), then sort lexicographically, stable in input position (equal
    codes keep input id order).  Returns (sorted codes uint8 [N, M], ids int64)."""
    codes = np.asarray(codes, dtype=np.uint8)
    N, M = codes.shape
    if ids is None:
        ids = np.arange(N, dtype=np.int64)
    ids = np.asarray(ids, dtype=np.int64)
    if order is not None:
        order = np.asarray(order)
        if sorted(order.tolist()) != list(range(M)):
            raise ValueError("config error")
        codes = codes[:, order]
    # np.lexsort sorts by the last key first; it is stable.
    perm = np.lexsort(tuple(codes[:, m] for m in range(M - 1, -1, -1)))
    return codes[perm], ids[perm]


def lcp(a, b) -> int:
    """Longest common prefix length of two codes, in bytes."""
    n = 0
    for x, y in zip(a, b):
        if x != y:
            break
        n += 1
    return n


# ----------------------------------------------------------------------------
# plain-definition statistics (reading A4)
# ----------------------------------------------------------------------------

@dataclass
class TreeStats:
    N: int
    M: int
    L1: int                 # internal nodes
    L2: int                 # leaves = distinct codes (no chaining)
    total_postfix: int      # sum over leaves of M-1-depth
    L2_records: int         # leaf records after n' <= 127 chaining (A9)
    total_postfix_records: int
    lookups: int            # L1 + L2 + total_postfix (one evaluation per leaf)
    lookups_records: int    # L1 + L2_records + total_postfix_records
    paper_bytes: int        # 4N + 2(L1 + L2_records) + total_postfix_records
    depth_hist: List[int] = field(default_factory=list)

    @property
    def avg_postfix(self) -> float:
        return self.total_postfix / self.L2 if self.L2 else 0.0

    @property
    def n_nodes(self) -> int:
        return self.L1 + self.L2


def distinct(sorted_codes: np.ndarray):
    """Distinct codes of a sorted array and their run lengths."""
    sc = np.asarray(sorted_codes, dtype=np.uint8)
    if len(sc) == 0:
        return sc, np.zeros(0, dtype=np.int64)
    new = np.ones(len(sc), dtype=bool)
    new[1:] = np.any(sc[1:] != sc[:-1], axis=1)
    starts = np.flatnonzero(new)
    counts = np.diff(np.append(starts, len(sc)))
    return sc[starts], counts


def adjacent_lcp(U: np.ndarray) -> np.ndarray:
    """lcp[i] = LCP(U[i-1], U[i]) for i >= 1 (lcp[0] = 0), vectorised."""
    n, M = U.shape
    out = np.zeros(n, dtype=np.int64)
    if n > 1:
        eq = U[1:] == U[:-1]
        # number of leading True per row
        first_diff = np.where(~eq.all(1), np.argmin(eq, axis=1), M)
        out[1:] = first_diff
    return out


def leaf_depths(U: np.ndarray) -> np.ndarray:
    """Depth of each distinct code's leaf: max LCP with its sorted neighbours,
    capped at M-1 (a node whose subtree holds one code becomes the leaf)."""
    n, M = U.shape
    lp = adjacent_lcp(U)
    nxt = np.zeros(n, dtype=np.int64)
    nxt[:-1] = lp[1:]
    return np.minimum(M - 1, np.maximum(lp, nxt))


def internal_count(U: np.ndarray) -> np.ndarray:
    """Per depth l in 0..M-2: number of length-(l+1) prefixes shared by >= 2
    distinct codes (= internal nodes at depth l)."""
    n, M = U.shape
    lp = adjacent_lcp(U)
    per = np.zeros(max(M - 1, 0), dtype=np.int64)
    for l in range(M - 1):
        ok = lp[1:] >= l + 1             # U[i-1], U[i] share the length-(l+1) prefix
        # maximal runs of True = groups of >= 2 codes sharing that prefix
        starts = ok & np.concatenate(([True], ~ok[:-1])) if len(ok) else ok
        per[l] = int(starts.sum())
    return per


def tree_stats_def(sorted_codes: np.ndarray, chain: int = 127) -> TreeStats:
    """Statistics of the E-Tree of ``sorted_codes`` from the plain definition."""
    sc = np.asarray(sorted_codes, dtype=np.uint8)
    N, M = sc.shape
    if N == 0:
        raise ValueError("empty dataset")
    U, cnt = distinct(sc)
    depth = leaf_depths(U)
    post = (M - 1) - depth
    per = internal_count(U)
    L1 = int(per.sum())
    L2 = len(U)
    recs = (cnt + chain - 1) // chain
    tp = int(post.sum())
    tpr = int((post * recs).sum())
    L2r = int(recs.sum())
    return TreeStats(N=N, M=M, L1=L1, L2=L2, total_postfix=tp, L2_records=L2r,
                     total_postfix_records=tpr, lookups=L1 + L2 + tp,
                     lookups_records=L1 + L2r + tpr,
                     paper_bytes=4 * N + 2 * (L1 + L2r) + tpr,
                     depth_hist=np.bincount(depth, minlength=M).tolist())


# ----------------------------------------------------------------------------
# Algorithm 1
# ----------------------------------------------------------------------------

class Node:
    __slots__ = ("K", "depth", "children", "ids", "postfix", "is_leaf")

    def __init__(self, K: int, depth: int):
        self.K = K
        self.depth = depth
        self.children: List["Node"] = []
        self.ids: List[int] = []
        self.postfix: bytes = b""
        self.is_leaf = False

    def n_codes(self) -> int:
        """Distinct full codes in this (still uncompressed or merged) subtree."""
        if self.is_leaf:
            return 1
        if not self.children:          # a full-depth node (depth M-1) = one code
            return 1
        return sum(c.n_codes() for c in self.children)


def _merge(node: Node, M: int) -> None:
    """'Merge' (reading A4): a finished subtree with exactly one distinct
    code collapses into a leaf at its top node; otherwise recurse."""
    if node.is_leaf:
        return
    if node.n_codes() == 1:
        post: List[int] = []
        cur = node
        while cur.children:                 # walk the single-child chain down
            cur = cur.children[0]
            post.append(cur.K)
        if cur.is_leaf:                     # (defensive) an already-merged tail
            post += list(cur.postfix)
        ids = cur.ids
        node.children = []
        node.postfix = bytes(post)
        node.ids = list(ids)
        node.is_leaf = True
        assert len(node.postfix) == M - 1 - node.depth
        return
    for c in node.children:
        _merge(c, M)


class Tree:
    """Explicit E-Tree: the virtual root's children are the depth-0 nodes (A5)."""

    def __init__(self, M: int, N: int):
        self.M = M
        self.N = N
        self.roots: List[Node] = []

    def nodes(self):
        stack = list(reversed(self.roots))
        while stack:
            n = stack.pop()
            yield n
            stack.extend(reversed(n.children))

    def stats(self, chain: int = 127) -> TreeStats:
        L1 = L2 = tp = L2r = tpr = 0
        depth_hist = [0] * self.M
        for n in self.nodes():
            if n.is_leaf:
                L2 += 1
                r = (len(n.ids) + chain - 1) // chain
                L2r += r
                tp += len(n.postfix)
                tpr += r * len(n.postfix)
                depth_hist[n.depth] += 1
            else:
                L1 += 1
        return TreeStats(N=self.N, M=self.M, L1=L1, L2=L2, total_postfix=tp,
                         L2_records=L2r, total_postfix_records=tpr,
                         lookups=L1 + L2 + tp, lookups_records=L1 + L2r + tpr,
                         paper_bytes=4 * self.N + 2 * (L1 + L2r) + tpr,
                         depth_hist=depth_hist)


def build_alg1(sorted_codes: np.ndarray, ids: np.ndarray) -> Tree:
    """Algorithm 1, line by line, on lexicographically sorted codes.

    ``root <- P_1`` is the virtual root (A5); lastPath holds the open node at
    each depth 0..M-1; identical codes attach to the same leaf (A6).
    """
    sc = np.asarray(sorted_codes, dtype=np.uint8)
    N, M = sc.shape
    if N == 0:
        raise ValueError("empty dataset")
    tree = Tree(M, N)
    last: List[Node] = []
    last_code = None
    for i in range(N):
        P = sc[i]
        if last_code is None:
            l = 0
        else:
            l = lcp(last_code, P)
            if l < M and P[l] < last_code[l]:
                raise ValueError("precondition violation")
        if l == M:                                  # identical code (A6)
            last[M - 1].ids.append(int(ids[i]))
            continue
        if last:                                    # Merge lastPath{l+1..M}
            _merge(last[l], M)
        parent_children = tree.roots if l == 0 else last[l - 1].children
        new = []
        for dpt in range(l, M):                     # create nodes P{l+1} .. P{M}
            nd = Node(int(P[dpt]), dpt)
            (parent_children if dpt == l else new[-1].children).append(nd)
            new.append(nd)
        last = last[:l] + new                       # lastPath{l+1~M} := P{l+1~M}
        last[M - 1].ids.append(int(ids[i]))         # associate i-th vector
        last_code = P
    _merge(last[0], M)                              # close the final path
    return tree


# ----------------------------------------------------------------------------
# Hierarchical Memory Structure
# ----------------------------------------------------------------------------

def serialize(tree: Tree, chain: int = 127, leaves_first: bool = True) -> bytes:
    """DFS byte buffer.  ``leaves_first=False`` gives plain lexicographic child
    order (kept only to demonstrate the A7 ambiguity in the tests)."""
    out = bytearray()

    def children(n_list):
        if leaves_first:
            return sorted(n_list, key=lambda c: (not c.is_leaf, c.K))
        return sorted(n_list, key=lambda c: c.K)

    def emit(n: Node):
        if n.is_leaf:
            ids = n.ids
            for s in range(0, len(ids), chain):
                grp = ids[s:s + chain]
                out.append(n.K)
                out.append((len(grp) << 1) | 1)
                out.extend(n.postfix)
                for v in grp:
                    out.extend(int(v).to_bytes(4, "little"))
        else:
            out.append(n.K)
            out.append((n.depth << 1) | 0)
            for c in children(n.children):
                emit(c)

    for r in children(tree.roots):
        emit(r)
    return bytes(out)


def parse(buf: bytes, M: int):
    """Decode a leaves-first HMS buffer back to its leaf list.

    Returns (codes uint8 [N, M], ids int64 [N]) in buffer (leaves-first DFS)
    order; re-sorting them reproduces the sorted input of ``serialize``.  Raises
    ValueError("corrupt buffer") on malformed input.
    """
    codes: List[List[int]] = []
    ids: List[int] = []
    path = [0] * M
    cur = -1                                 # depth of the last internal record
    pos = 0
    n = len(buf)
    while pos < n:
        if pos + 2 > n:
            raise ValueError("corrupt buffer")
        K, u = buf[pos], buf[pos + 1]
        if u & 1:
            l = cur + 1
            if l > M - 1:
                raise ValueError("corrupt buffer")
            plen = M - 1 - l
            cnt = u >> 1
            end = pos + 2 + plen + 4 * cnt
            if cnt == 0 or end > n:
                raise ValueError("corrupt buffer")
            code = path[:l] + [K] + list(buf[pos + 2:pos + 2 + plen])
            for j in range(cnt):
                o = pos + 2 + plen + 4 * j
                codes.append(code)
                ids.append(int.from_bytes(buf[o:o + 4], "little"))
            pos = end
        else:
            l = u >> 1
            if l > M - 2 or l > cur + 1:
                raise ValueError("corrupt buffer")
            path[l] = K
            cur = l
            pos += 2
    return np.array(codes, dtype=np.uint8).reshape(-1, M), np.array(ids, dtype=np.int64)


def traverse(buf: bytes, M: int, table: np.ndarray, n_out: int, layer0: int = 0):
    """Distance-Context traversal (readings A2/A3/A5/A10/A11).

    ``table`` is [Q, M_total, K] (any float dtype; the arithmetic happens in that
    dtype, vectorised over the Q queries); this tree's layer l reads table layer
    ``layer0 + l`` (forest use).  Output ``out[q][id]`` ([Q, n_out]; ids index
    the output) and the number of table lookups performed per query.
    """
    table = np.asarray(table)
    Q = table.shape[0]
    dt = table.dtype
    out = np.full((Q, n_out), np.nan, dtype=dt)
    ctx = [np.zeros(Q, dtype=dt) for _ in range(M)]
    zero = np.zeros(Q, dtype=dt)                     # ctx[-1] = 0 (virtual root)
    cur = -1
    pos = 0
    lookups = 0
    n = len(buf)
    while pos < n:                                   # A11: stop at end of buffer
        K, u = buf[pos], buf[pos + 1]
        if u & 1:                                    # leaf
            l = cur + 1
            dist = (ctx[l - 1] if l > 0 else zero) + table[:, layer0 + l, K]
            lookups += 1
            plen = M - 1 - l                         # A3
            for i in range(plen):
                dist = dist + table[:, layer0 + l + 1 + i, buf[pos + 2 + i]]
                lookups += 1
            cnt = u >> 1
            for j in range(cnt):                     # OutputResult()
                o = pos + 2 + plen + 4 * j
                out[:, int.from_bytes(buf[o:o + 4], "little")] = dist
            pos += 2 + plen + 4 * cnt                # A10
        else:                                        # internal
            cur = u >> 1
            ctx[cur] = (ctx[cur - 1] if cur > 0 else zero) + table[:, layer0 + cur, K]
            lookups += 1
            pos += 2
    return out, lookups


def build(codes: np.ndarray, ids: Optional[np.ndarray] = None, order=None, chain: int = 127):
    """Convenience: sort, Algorithm 1, serialise.  Returns (tree, buffer, sorted
    codes, sorted ids)."""
    sc, sid = sort_codes(codes, ids, order)
    tree = build_alg1(sc, sid)
    return tree, serialize(tree, chain), sc, sid
