"""f4: the paper's kernel variants rebuilt as ablations (sw_tuning.variant, the
ablation build libswsearch_ablation.so) compute the
same Eq. 1 scores as the oracle, bit-exactly, including tails, long subjects
(intra-task path beside them) and int32 reruns."""
import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum50, blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues

pytestmark = pytest.mark.gpu
B62 = matrix32(blosum62())
B50 = matrix32(blosum50())


def _query(m, seed=0):
    return gen_residues(stream_key(seed, "ablation-query", m), 0, m)


@pytest.mark.parametrize("variant", ["intersp", "intraqp", "static"])
@pytest.mark.parametrize("m", [1, 8, 31, 33, 100, 464, 1100])
def test_variant_equals_oracle(variant, m):
    # intraqp: every group through the (striped) intra-task path
    kw = dict(tuning={"variant": variant}, long_threshold=1 if variant == "intraqp" else 0)
    rng = np.random.default_rng(m)
    lens = np.concatenate([rng.integers(0, 700, 1500), [3000, 4000, 1, 0]])
    db = random_db(400 + m, lens)
    q = _query(m, 1)
    for M, a, b in ((B62, 2, 12), (B50, 0, 3)):
        with sw.Database.from_synth(db, device=0, **kw) as g:
            r = g.search(q, M, a, b, k=10)
        ref = oracle.db_scores(q, db, M, a, b)
        bad = np.nonzero(r.scores != ref)[0]
        assert bad.size == 0, (variant, m, bad[:5], r.scores[bad[:5]], ref[bad[:5]])


@pytest.mark.parametrize("variant,m", [("intersp", 8000), ("intraqp", 2000)])
def test_variant_saturation(variant, m):
    """Planted copies whose self-score exceeds int16: flagged, rerun in int32, exact."""
    q = _query(m, 3)
    M = B62.copy()
    for c in range(20):
        M[c, c] = 100                                     # self-score ~ 100 m > 32767 at m = 2000
    lens = np.array([m, 300, m // 2, 50])
    db = random_db(9, lens)
    db.residues[db.offsets[0]:db.offsets[0] + m] = q
    db.residues[db.offsets[2]:db.offsets[2] + m // 2] = q[m // 8:m // 8 + m // 2]
    with sw.Database.from_synth(db, device=0, long_threshold=1, tuning={"variant": variant}) as g:
        r = g.search(q, M, 2, 12, k=3)
    ref = oracle.db_scores(q, db, M, 2, 12)
    assert np.array_equal(r.scores, ref) and r.stats["n_rerun32"] >= 1


@pytest.mark.parametrize("nc", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 8, 129, 144, 300, 600, 1100])
def test_intra_columns_per_step(nc, m):
    """The intra-task wavefront with 2 (previous design, ablation build), 4 (throughput) or 8 (latency-bound
    small databases) columns per step,
    every group forced through it: exact, across rows-per-lane shapes, multi-pass queries, ragged
    column counts (every ncols mod 4) and int32 reruns of planted copies."""
    rng = np.random.default_rng(50 + m)
    lens = np.concatenate([rng.integers(0, 400, 300), [1, 2, 3, 4, 5, 2999, 3000, 3001, 3002]])
    db = random_db(500 + m, lens)
    q = _query(m, 5)
    M = B62.copy()
    if m >= 600:
        for c in range(20):
            M[c, c] = 60                                  # planted copies score > LIMIT16
        db.residues[db.offsets[-1]:db.offsets[-1] + m] = q
    for first_stage in (16, 32):
        with sw.Database.from_synth(db, device=0, first_stage=first_stage, long_threshold=1,
                                    tuning={"intra_cols": nc}) as g:
            r = g.search(q, M, 2, 12, k=10)
        ref = oracle.db_scores(q, db, M, 2, 12)
        bad = np.nonzero(r.scores != ref)[0]
        assert bad.size == 0, (nc, m, first_stage, bad[:5], r.scores[bad[:5]], ref[bad[:5]])
