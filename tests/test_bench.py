"""bench.py host logic (no GPU): the analytic DRAM traffic model, the snake
partition used for the multi-GPU shards, and the reference arm's JSON contract."""
import numpy as np

import bench


def test_traffic_model_small_case():
    # one group of 64 subjects of 10 residues, m = 96: two 48-row tiles, one internal edge
    t = bench.traffic_model(np.full(64, 10), 96, n_warps=1776)
    assert t["db_bytes"] == 2 * 32 * 8                     # ceil(10/6) = 2 words x 32 lanes x 8 B
    assert t["boundary_bytes"] == 10 * 32 * 8 * 2 * 1      # cols x lanes x 8 B x (write+read) x 1 edge
    assert t["total"] == t["db_bytes"] + t["boundary_bytes"]


def test_traffic_model_intra_groups_have_pass_edges_only():
    # a single group wider than the split floor goes intra-task: m = 600 -> TR 16, 2 passes
    t = bench.traffic_model(np.full(64, 5000), 600, n_warps=1776)
    assert t["boundary_bytes"] == 5000 * 32 * 8 * 2 * 1


def test_snake_partition_covers_and_balances():
    rng = np.random.default_rng(0)
    lens = rng.integers(10, 5000, 10001)
    parts = [bench.snake_partition(lens, 4, r) for r in range(4)]
    allids = np.sort(np.concatenate(parts))
    assert np.array_equal(allids, np.arange(lens.size))
    tot = [int(lens[p].sum()) for p in parts]
    assert max(tot) - min(tot) <= 2 * int(lens.max())


def test_reference_arm_contract_under_torchrun():
    """`bench.py --impl reference` under torchrun (N=2): rank 0 alone prints ONE JSON line with the
    contract's keys; every rank exits 0 (the oracle is the reference arm for this tier)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = 29500 + os.getpid() % 1000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", "C1", "--ref-sample", "300"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
