"""Multi-rank path on real hardware: N
processes each build their snake shard of the database as an sw_db with global
ids, search it on the GPU, exchange their top-k with an all_gather and merge it
with sw_merge_topk (paper_1404_4152_b200.dist.ShardedSearch, the step bench.py
runs at N > 1).  Only one GPU is available to the tests, so the N ranks share
device 0 and talk over gloo (NCCL refuses two ranks on one device); their
kernels never wait on one another, only the host-side exchange is collective.

Sharding invariance: for N in {1, 2, 3} the union of the shard
scores equals the oracle's scores of the whole database -- and, for C1, the
stored full-config oracle digest -- and the merged top-k equals oracle.topk.
"""
import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from swdata import CONFIGS, make_db, make_query
from swdata.synth import Config, db_lengths

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(name, n):
    base = CONFIGS[name]
    return base if n is None else Config(**{**base.__dict__, "n_seqs": n})


def _rank(rank, world, port, name, n, k, out):
    import torch
    import torch.distributed as dist
    from paper_1404_4152_b200.dist import ShardedSearch, snake_shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = _cfg(name, n)
    lk = db_lengths(cfg)
    ids = snake_shard(lk[0], world, rank)
    shard = make_db(cfg, ids=ids, lengths_kind=lk)
    q, M = make_query(cfg), cfg.matrix32()
    ss = ShardedSearch(shard, k, device=0)
    stream = torch.cuda.Stream()
    ss.enqueue(q, M, cfg.alpha, cfg.beta, stream)                # async path (device outputs)
    stream.synchronize()
    ai, asc = ss.merged_topk()
    local = ss.d_scores[:shard.n_seqs].cpu().numpy()
    bi, bsc, blocal = ss.search(q, M, cfg.alpha, cfg.beta)       # blocking path (host buffers)
    out[rank] = (ids, local, blocal, ai.tolist(), asc.tolist(), bi.tolist(), bsc.tolist())
    ss.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("name,n", [("C1", None), ("C2", 40_000)])
def test_sharded_search_equals_whole_database_oracle(world, name, n):
    cfg = _cfg(name, n)
    k = cfg.k
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _free_port(), name, n, k, out), nprocs=world, join=True)
    full = make_db(cfg)
    ref = oracle.db_scores(make_query(cfg), full, cfg.matrix32(), cfg.alpha, cfg.beta)
    got = np.full(full.n_seqs, -1, dtype=np.int64)
    for r in range(world):
        ids, local, blocal, *_ = out[r]
        assert np.array_equal(local, blocal)
        assert np.all(got[ids] == -1)                               # shards are disjoint
        got[ids] = local
    assert np.array_equal(got, ref)                                  # and cover every subject exactly
    ti, ts = oracle.topk(ref, k)
    for r in range(world):
        assert out[r][3] == ti.tolist() and out[r][4] == ts.tolist()   # async path, every rank
        assert out[r][5] == ti.tolist() and out[r][6] == ts.tolist()   # blocking path
    if name == "C1":                                                 # and the stored full-config digest
        rec = json.load(open(os.path.join(HERE, "golden", "digests", "C1_m144.json")))
        B = rec["block"]
        digs = [hashlib.sha256(got[b:b + B].astype("<i4").tobytes()).hexdigest() for b in range(0, got.size, B)]
        assert digs == rec["block_sha256"] and rec["topk_ids"] == ti.tolist()[:len(rec["topk_ids"])]


@pytest.mark.parametrize("world", [2, 3])
def test_bench_multi_rank_branch_on_one_gpu(world):
    """bench.py's N > 1 path (never executed): torchrun N ranks on the one GPU with
    the gloo backend -- each rank generates and searches its snake shard of C1, the top-k goes
    through all_gather + sw_merge_topk, the device times are reduced with MAX, and rank 0's parity gate
    checks every subject against the stored C1 oracle digest.  One JSON line, n_gpus = N, strong scaling."""
    import subprocess
    import sys
    root = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(world),
           "--steps", "3", "--warmup", "3", "--config", "C1", "--backend", "gloo", "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["seqs_total"] == CONFIGS["C1"].n_seqs and d["config"]["seqs_rank0"] < CONFIGS["C1"].n_seqs
    assert d["parity"]["ok"] and d["parity"]["blocks_ok"] == d["parity"]["blocks"]
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
