"""Multi-GPU sharding and the top-k exchange.

The paper distributes the database over coprocessors, one host thread per
device, each searching its part; only the final ranking is shared (PAPER.md:55,
65, §III; 1.95x on 2 and 3.66x on 4 devices).  Here: one process
per GPU.  Every rank computes the same deterministic residue-balanced partition
from the global lengths (no communication), builds its own sw_db over its shard
(with global ids), searches it, and the per-rank top-k lists are exchanged with
one all_gather -- NCCL over NVLink on GPUs, gloo on CPU tensors -- and merged by
(score desc, global id asc) with sw_merge_topk.  No other collective is on the
path: the scores of a subject never leave its rank.
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
    """All-gather each rank's top-k (torch tensors; CUDA with NCCL, CPU with
    gloo) and merge on the host with sw_merge_topk.  Returns (ids int64[k],
    scores int32[k]) on every rank."""
    import torch
    import torch.distributed as dist

    from . import merge_topk
    world = dist.get_world_size(group)
    gi = torch.empty(world * k, dtype=torch.int64, device=ids_local.device)
    gs = torch.empty(world * k, dtype=torch.int32, device=scores_local.device)
    dist.all_gather_into_tensor(gi, ids_local.contiguous(), group=group)
    dist.all_gather_into_tensor(gs, scores_local.contiguous(), group=group)
    return merge_topk(gi.view(world, k).cpu().numpy(), gs.view(world, k).cpu().numpy(), k)


class ShardedSearch:
    """The rank step of a multi-GPU search: this rank's shard as an sw_db
    (global ids kept for the top-k), its search, and the top-k exchange.

        ss = ShardedSearch(shard_db, k, device)        # shard_db: SynthDB-like
        ss.enqueue(q, M, alpha, beta, stream)          # local search + all_gather, no host sync
        ids, scores = ss.merged_topk()                 # host merge (after the stream)
        ids, scores, local_scores = ss.search(q, M, alpha, beta)   # blocking, host buffers

    With NCCL the exchange runs on `stream` right after the search kernels; with
    gloo (CPU-only collectives, e.g. several ranks sharing one GPU in tests) the
    top-k is copied to the host first.
    """

    def __init__(self, shard, k: int, device: int, group=None, db_kwargs: dict | None = None):
        import torch
        import torch.distributed as dist

        from . import Database
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
        self.k = k
        self.device = device
        self.db = Database(shard.residues, shard.offsets, shard.lengths, global_ids=shard.global_ids,
                           device=device, **(db_kwargs or {}))
        self.n = int(shard.lengths.size)
        self.global_ids = np.asarray(shard.global_ids, dtype=np.int64)
        dev = torch.device("cuda", device)
        self.d_scores = torch.empty(max(self.n, 1), dtype=torch.int32, device=dev)
        self.d_ti = torch.empty(k, dtype=torch.int64, device=dev)
        self.d_ts = torch.empty(k, dtype=torch.int32, device=dev)
        xdev = dev if self.nccl else torch.device("cpu")
        self.g_ti = torch.empty(self.world * k, dtype=torch.int64, device=xdev)
        self.g_ts = torch.empty(self.world * k, dtype=torch.int32, device=xdev)

    def enqueue(self, q, M, alpha: int, beta: int, stream=None):
        """Local search on `stream` (device outputs) followed by the top-k all-gather."""
        torch, dist = self.torch, self.dist
        self.db.search_async(q, M, alpha, beta, self.k, self.d_scores if self.n else None, self.d_ti, self.d_ts,
                             stream=stream)
        if self.world == 1:
            return
        if self.nccl:
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                dist.all_gather_into_tensor(self.g_ti, self.d_ti, group=self.group)
                dist.all_gather_into_tensor(self.g_ts, self.d_ts, group=self.group)
        else:
            if stream is not None:
                stream.synchronize()
            else:
                torch.cuda.synchronize(self.device)
            dist.all_gather_into_tensor(self.g_ti, self.d_ti.cpu(), group=self.group)
            dist.all_gather_into_tensor(self.g_ts, self.d_ts.cpu(), group=self.group)

    def merged_topk(self):
        """(ids, scores) of the global top-k (call after the enqueue's stream)."""
        from . import merge_topk
        if self.world == 1:
            return self.d_ti.cpu().numpy(), self.d_ts.cpu().numpy()
        return merge_topk(self.g_ti.view(self.world, self.k).cpu().numpy(),
                          self.g_ts.view(self.world, self.k).cpu().numpy(), self.k)

    def search(self, q, M, alpha: int, beta: int, scores=None):
        """Blocking search through sw_search with host buffers, then the exchange:
        returns (global top-k ids, scores, this shard's scores in shard order)."""
        torch = self.torch
        r = self.db.search(q, M, alpha, beta, k=self.k, scores=True if scores is None else scores)
        if self.world == 1:
            return r.topk_ids, r.topk_scores, r.scores
        dev = self.g_ti.device
        ti = torch.from_numpy(np.ascontiguousarray(r.topk_ids)).to(dev)
        ts = torch.from_numpy(np.ascontiguousarray(r.topk_scores)).to(dev)
        self.dist.all_gather_into_tensor(self.g_ti, ti, group=self.group)
        self.dist.all_gather_into_tensor(self.g_ts, ts, group=self.group)
        ids, sc = self.merged_topk()
        return ids, sc, r.scores

    def close(self):
        self.db.close()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
