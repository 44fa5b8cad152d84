"""Multi-GPU plumbing: shard the database by first-level subtrees, gather the
per-shard top-k lists.

Cutting the lexicographically sorted codes between first-level subtrees (first
code byte) gives G sub-trees whose concatenation is the whole tree, so each
rank can build its own index with global ids and the per-id sums stay
bit-identical to the single-GPU path.  The cut itself (``et_shard_bounds``) and
the IVF list assignment (``et_shard_lists``) are host C++ in libetree; the
merge runs on the GPU (``api.et_merge_topk``).  This module only selects rows
and moves lists.
"""
from __future__ import annotations

import numpy as np

from . import api


def shard_select(codes: np.ndarray, rank: int, world: int, K: int = 256, ids=None):
    """Rows of shard ``rank``: (codes, ids int32).  ``ids`` are the global ids
    of the rows (default: their positions)."""
    b = api.et_shard_bounds(codes, world, K)
    m = (codes[:, 0] >= b[rank]) & (codes[:, 0] < b[rank + 1])
    sel = np.flatnonzero(m)
    gid = sel.astype(np.int32) if ids is None else np.asarray(ids, dtype=np.int32)[sel]
    return codes[m], gid


def ivf_select(list_sizes: np.ndarray, list_of: np.ndarray, rank: int, world: int):
    """Boolean row mask of the vectors whose inverted list rank ``rank`` owns."""
    owner = api.et_shard_lists(list_sizes, world)
    return owner[np.asarray(list_of)] == rank


def gather_lists(dist, ids, group=None):
    """All-gather per-rank [Q, k] (dist, ids) into [G, Q, k] tensors.

    NCCL: one ``all_gather_into_tensor`` per array; other backends (gloo, for
    the CPU tests) use ``all_gather`` into a list."""
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
