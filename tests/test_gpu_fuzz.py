"""Randomised differential test: many seeded cases that combine the options the other parity tests vary
one at a time (first stage, residency and chunking, long-subject split, gap parameters, matrices with
large or asymmetric scores, empty / tiny / very long subjects, k, batched queries, traceback) and compare
every score and the top-k with the oracle.  Each case prints its seed; a failure names the options."""
import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum50, blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues

pytestmark = pytest.mark.gpu

N_CASES = 240


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([0, 1, 7, 64, 65, 200, 700]))
    kind = rng.integers(0, 4)
    if kind == 0:
        lens = rng.integers(0, 40, size=n)
    elif kind == 1:
        lens = rng.integers(0, 700, size=n)
    elif kind == 2:
        lens = np.clip(rng.lognormal(np.log(300), 0.65, size=n), 0, 5000).astype(int)
    else:   # a few very long subjects among short ones
        lens = rng.integers(1, 300, size=n)
        if n:
            lens[rng.integers(0, n, size=min(3, n))] = rng.integers(2000, 9000, size=min(3, n))
    db = random_db(2000 + seed, lens, alphabet=int(rng.choice([4, 20])))
    mk = rng.integers(0, 4)
    if mk == 0:
        M = matrix32(blosum62())
    elif mk == 1:
        M = matrix32(blosum50())
    elif mk == 2:   # random asymmetric scores
        M = np.zeros((32, 32), dtype=np.int8)
        M[:24, :24] = rng.integers(-20, 21, size=(24, 24))
    else:           # large positive diagonal: int16 saturation and int32 reruns for long matches
        M = np.zeros((32, 32), dtype=np.int8)
        M[:24, :24] = rng.integers(-30, 5, size=(24, 24))
        np.fill_diagonal(M[:24, :24], 120)
    alpha = int(rng.integers(0, 12))
    beta = int(alpha + rng.integers(0, 30))
    m = int(rng.choice([1, 2, 17, 96, 144, 300, 700, 1500]))
    q = gen_residues(stream_key(seed, "fuzz-query", m), 0, m)
    if mk == 3:   # plant the query into the longest subjects so the diagonal run can saturate int16
        for i in np.argsort(-db.lengths, kind="stable")[:2]:
            if db.lengths[i] >= m:
                o = int(db.offsets[i]) + int(rng.integers(0, db.lengths[i] - m + 1))
                db.residues[o:o + m] = q
    stage = int(rng.choice([8, 16, 32]))
    residency = int(rng.integers(0, 2)) if stage != 8 else 0
    opts = dict(first_stage=stage, residency=residency, chunk_mb=int(rng.choice([0, 1, 2])),
                long_threshold=int(rng.choice([0, -1, 64, 300])))
    if seed % 5 == 2:                    # the pipelined first pass (sw_tuning.pipeline)
        opts["tuning"] = {"pipeline": 1}
    k = int(rng.integers(1, 40))
    return db, q, M, alpha, beta, k, opts


@pytest.mark.parametrize("seed", range(N_CASES))
def test_fuzz_search_matches_oracle(seed):
    db, q, M, alpha, beta, k, opts = _case(seed)
    desc = f"seed={seed} n={db.n_seqs} m={q.size} alpha={alpha} beta={beta} k={k} {opts}"
    ref = oracle.db_scores(q, db, M, alpha, beta)
    gids = (np.arange(db.n_seqs, dtype=np.int64) * 7 + 3) if seed % 2 else None
    with sw.Database(db.residues, db.offsets, db.lengths, global_ids=gids, device=0, **opts) as g:
        r = g.search(q, M, alpha, beta, k=k)
        assert np.array_equal(r.scores, ref), desc
        ti, ts = oracle.topk(ref, k, gids)
        assert np.array_equal(r.topk_ids, ti) and np.array_equal(r.topk_scores, ts), desc
        if opts["residency"] == 0 and db.n_seqs and seed % 3 == 0:
            q2 = gen_residues(stream_key(seed, "fuzz-query-2", q.size + 5), 0, q.size + 5)
            rb = g.search_batch([q, q2], M, alpha, beta, k=k)
            assert np.array_equal(rb.scores[0], ref), desc + " batch[0]"
            assert np.array_equal(rb.scores[1], oracle.db_scores(q2, db, M, alpha, beta)), desc + " batch[1]"
        if db.n_seqs and seed % 4 == 1:
            hits = np.argsort(-ref, kind="stable")[:3].astype(np.int64)
            al = g.align(q, M, alpha, beta, hits)
            assert [a["score"] for a in al] == ref[hits].tolist(), desc + " align"
