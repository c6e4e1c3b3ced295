"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (default options): every score where the oracle can afford it (C1, S16),
else sampled subjects the oracle computes one by one (C2, C3, C4, C5) plus
properties that hold at any size (bounds, top-k consistency)."""
import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query
from swdata.synth import db_lengths

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _search(cfg, m=None, **kw):
    db = make_db(cfg)
    q = make_query(cfg, m)
    M = cfg.matrix32()
    with sw.Database.from_synth(db, device=0, **kw) as g:
        res = g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)
    return db, q, M, res


def _properties(cfg, db, q, M, res):
    sc = res.scores
    smax = int(M.max())
    assert sc.min() >= 0
    assert np.all(sc <= np.minimum(db.lengths, q.size) * smax)
    # top-k is the (score desc, id asc) head of the returned score vector ...
    order = np.lexsort((np.arange(sc.size), -sc.astype(np.int64)))[:cfg.k]
    assert np.array_equal(res.topk_ids, order)
    assert np.array_equal(res.topk_scores, sc[order])
    # ... and each top-k score is exact
    ref = oracle.db_scores(q, db, M, cfg.alpha, cfg.beta, sample=res.topk_ids)
    assert np.array_equal(ref, res.topk_scores)


def _sampled(cfg, db, q, M, res, n_random=2000, n_longest=200, extra=None, seed=0):
    rng = np.random.default_rng(seed)
    idx = [rng.choice(db.n_seqs, size=min(n_random, db.n_seqs), replace=False),
           np.argsort(db.lengths, kind="stable")[-n_longest:]]
    if extra is not None:
        idx.append(extra)
    idx = np.unique(np.concatenate(idx))
    ref = oracle.db_scores(q, db, M, cfg.alpha, cfg.beta, sample=idx)
    bad = np.nonzero(ref != res.scores[idx])[0]
    assert bad.size == 0, f"{bad.size} of {idx.size} sampled differ, e.g. id {idx[bad[0]]}"


def test_c1_full_parity():
    cfg = CONFIGS["C1"]
    db, q, M, res = _search(cfg)
    ref = oracle.db_scores(q, db, M, cfg.alpha, cfg.beta)
    assert np.array_equal(ref, res.scores)
    ti, ts = oracle.topk(ref, cfg.k)
    assert np.array_equal(ti, res.topk_ids) and np.array_equal(ts, res.topk_scores)


def test_c2_fullsize_sampled():
    cfg = CONFIGS["C2"]
    db, q, M, res = _search(cfg)
    _properties(cfg, db, q, M, res)
    _sampled(cfg, db, q, M, res)


@pytest.mark.parametrize("first_stage", [16, 8])
def test_c4_fullsize_planted(first_stage):
    """C4 is the overflow stress config: with the int8 first stage every planted
    copy saturates and is re-aligned at int16 (R14: int16 cannot saturate here)."""
    cfg = CONFIGS["C4"]
    db, q, M, res = _search(cfg, first_stage=first_stage)
    if first_stage == 8:
        assert res.stats["n_rerun16"] >= 90_000 and res.stats["n_rerun32"] == 0
    _, kind = db_lengths(cfg)
    planted = np.nonzero(kind == 2)[0]
    _properties(cfg, db, q, M, res)
    assert np.all(kind[res.topk_ids] == 2)            # the top hits are planted copies
    rng = np.random.default_rng(1)
    _sampled(cfg, db, q, M, res, n_random=1500, n_longest=50, extra=rng.choice(planted, 150, replace=False))


def test_s16_full_parity_int32_reruns():
    cfg = CONFIGS["S16"]
    db, q, M, res = _search(cfg)
    ref = oracle.db_scores(q, db, M, cfg.alpha, cfg.beta)
    assert np.array_equal(ref, res.scores)
    assert res.stats["n_rerun32"] == int((ref > 32767 - int(M.max())).sum()) >= 200


@pytest.mark.parametrize("m", [144, 5478])
def test_c3_fullsize_sampled(m):
    cfg = CONFIGS["C3"]
    db, q, M, res = _search(cfg, m)
    _properties(cfg, db, q, M, res)
    _sampled(cfg, db, q, M, res, n_random=1000, n_longest=100)


def test_c5_fullsize_sampled():
    cfg = CONFIGS["C5"]
    db, q, M, res = _search(cfg)
    _properties(cfg, db, q, M, res)
    _sampled(cfg, db, q, M, res, n_random=1500, n_longest=100)
