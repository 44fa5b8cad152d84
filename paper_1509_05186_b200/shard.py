"""Multi-GPU plumbing: shard the database by first-level subtrees, gather the
per-shard top-k lists.

Cutting the lexicographically sorted codes between first-level subtrees (first
code byte) gives G sub-trees whose concatenation is the whole tree, so each
rank can build its own index with global ids and the per-id sums stay
bit-identical to the single-GPU path.  The merge itself runs on the GPU
(``api.et_merge_topk``); this module only partitions and moves lists.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(first_byte: np.ndarray, G: int, K: int = 256) -> np.ndarray:
    """G+1 byte boundaries: shard r holds codes whose first byte is in
    [b_r, b_{r+1}); b_r = smallest byte value v with #(first byte < v) >= r*N/G."""
    hist = np.bincount(np.asarray(first_byte, dtype=np.int64), minlength=K)
    below = np.concatenate(([0], np.cumsum(hist)))
    N = int(below[-1])
    b = [0]
    for r in range(1, G):
        v = int(np.searchsorted(below, r * N / G, side="left"))
        b.append(max(b[-1], min(v, K)))
    b.append(K)
    return np.asarray(b, dtype=np.int64)


def shard_select(codes: np.ndarray, rank: int, world: int, K: int = 256):
    """Rows (codes, global slot ids int32) of shard ``rank``."""
    b = shard_bounds(codes[:, 0], world, K)
    m = (codes[:, 0] >= b[rank]) & (codes[:, 0] < b[rank + 1])
    return codes[m], np.flatnonzero(m).astype(np.int32)


def gather_lists(dist, ids, group=None):
    """All-gather per-rank [Q, k] (dist, ids) into [G, Q, k] tensors.

    NCCL: one ``all_gather_into_tensor`` per array; other backends (gloo, for
    the CPU tests) fall back to ``all_gather`` into a list."""
    import torch
    import torch.distributed as dist_
    G = dist_.get_world_size(group)
    if dist_.get_backend(group) == "nccl":
        gd = torch.empty((G, *dist.shape), dtype=dist.dtype, device=dist.device)
        gi = torch.empty((G, *ids.shape), dtype=ids.dtype, device=ids.device)
        dist_.all_gather_into_tensor(gd, dist.contiguous(), group=group)
        dist_.all_gather_into_tensor(gi, ids.contiguous(), group=group)
        return gd, gi
    ld = [torch.empty_like(dist) for _ in range(G)]
    li = [torch.empty_like(ids) for _ in range(G)]
    dist_.all_gather(ld, dist.contiguous(), group=group)
    dist_.all_gather(li, ids.contiguous(), group=group)
    return torch.stack(ld), torch.stack(li)
