"""The pipelined first pass (sw_tuning.pipeline = 1, k_inter16_pipe in
csrc/sw_pipe.cuh): query tiles of a group run on consecutive warps, tile-edge
rows go through shared-memory rings between them and through a per-chain
global slab across rounds.  Every score and the top-k equal the oracle's,
across the shapes that exercise its protocol: groups of zero columns and
shorter than a ring chunk, one tile per group (no rings), tile counts below,
at and above the chain length, ragged last tiles, the ring-slot counts chosen
for short and long queries, queries too long for the rings (slab fallback),
int16 saturation and int32 reruns, wide groups with no slab limit, streamed
chunks, and chains of 1, 3 (production), 6 and 12 warps (ablation build)."""
import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues

pytestmark = pytest.mark.gpu
B62 = matrix32(blosum62())


def _query(m, seed=0):
    return gen_residues(stream_key(seed, "pipe-query", m), 0, m)


def _check(db, q, M=B62, alpha=2, beta=12, k=10, chain=0, **kw):
    with sw.Database.from_synth(db, device=0, tuning={"pipeline": 1, "pipe_chain": chain}, **kw) as g:
        r = g.search(q, M, alpha, beta, k=k)
    ref = oracle.db_scores(q, db, M, alpha, beta)
    bad = np.nonzero(r.scores != ref)[0]
    assert bad.size == 0, (f"chain={chain} m={q.size}: {bad.size} differ, first {bad[:4]} "
                           f"gpu {r.scores[bad[:4]]} oracle {ref[bad[:4]]}")
    ti, ts = oracle.topk(ref, k)
    assert np.array_equal(r.topk_ids, ti) and np.array_equal(r.topk_scores, ts)


@pytest.mark.parametrize("chain", [0, 1, 6, 12])
@pytest.mark.parametrize("m", [1, 40, 48, 49, 96, 144, 464, 575, 576, 577, 1000, 1500])
def test_pipeline_tile_counts_and_chains(chain, m):
    """n_tiles = ceil(m/48) from 1 to 32 against chains of 1..12 warps; lengths 0..900 incl. groups
    of zero columns and of fewer columns than a ring chunk (8)."""
    rng = np.random.default_rng(m * 7 + chain)
    lens = np.concatenate([np.zeros(70, int), rng.integers(1, 9, 90), rng.integers(0, 900, 1300)])
    _check(random_db(900 + m, lens), _query(m, 1), chain=chain)


@pytest.mark.parametrize("m", [2000, 4000, 4500, 6500, 9000])
def test_pipeline_ring_slots_and_fallback(m):
    """Long queries: fewer ring slots (8 -> 4 -> 2) as the profile grows, then the slab kernel
    when profile + rings exceed shared memory (and the global-memory profile past 200 KB)."""
    rng = np.random.default_rng(m)
    _check(random_db(77 + m, rng.integers(0, 400, 300)), _query(m, 2), max_qlen=max(m, 8192))


def test_pipeline_saturation_and_reruns():
    m = 1200
    q = _query(m, 3)
    M = B62.copy()
    for c in range(20):
        M[c, c] = 60                                   # planted copies score > LIMIT16 -> int32 reruns
    rng = np.random.default_rng(5)
    lens = np.concatenate([rng.integers(0, 600, 700), [m, m + 50, 3 * m]])
    db = random_db(31, lens)
    for i in (700, 701, 702):
        db.residues[db.offsets[i]:db.offsets[i] + m] = q
    _check(db, q, M=M)


def test_pipeline_wide_groups_without_slab_limit():
    """long_threshold -1: every group stays inter-task, including groups far wider than a warp's
    boundary slab (the pipeline needs none; its round-crossing slab spans the widest group)."""
    rng = np.random.default_rng(8)
    lens = np.concatenate([rng.integers(1, 400, 600), rng.integers(6200, 15000, 200)])
    db = random_db(8, lens)
    q = _query(300, 8)
    for t in (600, 650, 799):
        db.residues[db.offsets[t] + 5000:db.offsets[t] + 5300] = q
    _check(db, q, long_threshold=-1)


def test_pipeline_streamed_chunks():
    rng = np.random.default_rng(9)
    db = random_db(9, rng.integers(0, 2500, 3000))
    for chunk_mb in (1, 2):
        _check(db, _query(700, 9), residency=1, chunk_mb=chunk_mb)


def test_pipeline_alpha_beta_extremes():
    rng = np.random.default_rng(10)
    db = random_db(10, rng.integers(0, 700, 800))
    q = _query(333, 10)
    for a, b in ((0, 0), (0, 3), (5, 5), (1, 32767)):
        _check(db, q, alpha=a, beta=b)
