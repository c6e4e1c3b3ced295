"""Multi-rank host logic on CPU (gloo, world_size 2): the residue-balanced
partition and the top-k exchange + merge, checked against the oracle ranking
of the whole (unsharded) score vector."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_1404_4152_b200.dist import snake_shard
from swdata import db_lengths


def test_snake_partition_balance_and_coverage():
    L, _ = db_lengths("C1")
    for world in (1, 2, 3, 4, 8):
        shards = [snake_shard(L, world, r) for r in range(world)]
        allids = np.concatenate(shards)
        assert np.array_equal(np.sort(allids), np.arange(L.size))      # disjoint cover
        tot = np.array([L[s].sum() for s in shards])
        assert tot.max() - tot.min() <= 2 * L.max()                    # residue balance (snake bound)
        assert all(np.all(np.diff(s) > 0) for s in shards)             # ascending ids
        assert [snake_shard(L, world, r).tolist() for r in range(world)] == [s.tolist() for s in shards]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scores, k, out):
    import torch
    import torch.distributed as dist
    from paper_1404_4152_b200.dist import gather_topk, snake_shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lens = np.arange(scores.size) % 97
    ids = snake_shard(lens, world, rank)
    ti, ts = oracle.topk(scores[ids], k, ids)          # stands in for the rank's device top-k
    mi, ms = gather_topk(torch.from_numpy(ti), torch.from_numpy(ts), k)
    out[rank] = (mi.tolist(), ms.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_topk_exchange_matches_global_ranking(world):
    rng = np.random.default_rng(0)
    scores = rng.integers(0, 40, size=5000).astype(np.int32)      # heavy ties
    k = 25
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, scores, k, out), nprocs=world, join=True)
    ri, rs = oracle.topk(scores, k)
    for r in range(world):
        assert out[r][0] == ri.tolist() and out[r][1] == rs.tolist()
