"""Multi-GPU sharding and the top-k exchange (DESIGN.md §"Multi-GPU").

The paper distributes work as one host thread per coprocessor pulling chunks
of the length-sorted database.  Here every rank computes the
same deterministic residue-balanced partition from the global lengths (no
communication), builds its own sw_db over its shard, searches it, and the
per-rank top-k lists are exchanged with one all_gather (NCCL over NVLink on
GPUs, gloo on CPU) and merged by (score desc, global id asc) with
sw_merge_topk.  No other collective is on the path.
"""
from __future__ import annotations

import numpy as np


def snake_shard(lengths: np.ndarray, world: int, rank: int) -> np.ndarray:
    """Ascending global ids of `rank`'s shard.  Stable sort by (length, id); the
    r-th sorted id goes to r mod 2P if that is < P, else to 2P-1-(r mod 2P).
    Every shard then has the same length histogram; shard residue totals
    differ by at most twice the longest sequence (each round of 2P sorted ids
    adds at most that round's length spread; the spreads telescope to <= max,
    and the last partial round adds <= max)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    order = np.argsort(np.asarray(lengths), kind="stable")
    r = np.arange(order.size) % (2 * world)
    owner = np.where(r < world, r, 2 * world - 1 - r)
    return np.sort(order[owner == rank]).astype(np.int64)


def gather_topk(ids_local, scores_local, k: int, group=None):
    """All-gather each rank's top-k (torch tensors, any device) and merge on the
    host with sw_merge_topk.  Returns (ids int64[k], scores int32[k]) on every rank."""
    import torch
    import torch.distributed as dist

    from . import merge_topk
    world = dist.get_world_size(group)
    gi = torch.empty(world * k, dtype=torch.int64, device=ids_local.device)
    gs = torch.empty(world * k, dtype=torch.int32, device=scores_local.device)
    dist.all_gather_into_tensor(gi, ids_local.contiguous(), group=group)
    dist.all_gather_into_tensor(gs, scores_local.contiguous(), group=group)
    return merge_topk(gi.view(world, k).cpu().numpy(), gs.view(world, k).cpu().numpy(), k)
