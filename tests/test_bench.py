"""bench.py host logic (no GPU): the analytic DRAM traffic model and the snake
partition used for the multi-GPU shards."""
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
