"""GPU parity of f2 (host-resident, streamed database):
with residency 1 the packed words stay in pinned host memory and every search
copies them chunk by chunk (double-buffered, copy stream) while the previous
chunk is aligned.  Scores and top-k must equal the oracle bit-exactly and
the device-resident database exactly, whatever the chunking.
"""
import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues

pytestmark = pytest.mark.gpu
B62 = matrix32(blosum62())


def _query(m, seed=0):
    return gen_residues(stream_key(seed, "stream-query", m), 0, m)


def _db(seed, n=3000, long_tail=True):
    rng = np.random.default_rng(seed)
    lens = rng.lognormal(np.log(350) - 0.65 ** 2 / 2, 0.65, n).round().clip(10, 5000).astype(np.int64)
    if long_tail:
        lens = np.concatenate([lens, [9000, 12000, 0, 1]])
    return random_db(seed, lens)


@pytest.mark.parametrize("chunk_mb", [1, 3, 0])
@pytest.mark.parametrize("m", [64, 464, 1100])
def test_streamed_equals_oracle_and_resident(chunk_mb, m):
    db = _db(100 + m)
    q = _query(m, 1)
    ref = oracle.db_scores(q, db, B62, 2, 12)
    with sw.Database.from_synth(db, device=0, residency=1, chunk_mb=chunk_mb) as g:
        info = g.info()
        assert info["residency"] == 1 and info["n_chunks"] >= (2 if chunk_mb == 1 else 1)
        r = g.search(q, B62, 2, 12, k=25)
    bad = np.nonzero(r.scores != ref)[0]
    assert bad.size == 0, (bad[:5], r.scores[bad[:5]], ref[bad[:5]])
    ti, ts = oracle.topk(ref, 25)
    assert np.array_equal(r.topk_ids, ti) and np.array_equal(r.topk_scores, ts)
    with sw.Database.from_synth(db, device=0) as g:
        r2 = g.search(q, B62, 2, 12, k=25)
    assert np.array_equal(r.scores, r2.scores)


def test_streamed_saturation_reruns_and_first_stage_32():
    """Exact copies of an 8,000-residue query (self-score > 32767) in different
    chunks: each chunk's int32 rerun sees its own flagged subjects."""
    q = _query(8000, 2)
    rng = np.random.default_rng(3)
    lens = np.concatenate([rng.integers(50, 800, 2500), [8000], rng.integers(50, 800, 2500), [8000]])
    db = random_db(17, lens)
    for t in (2500, 5001):
        db.residues[db.offsets[t]:db.offsets[t] + 8000] = q
    ref = oracle.db_scores(q, db, B62, 2, 12)
    for fs in (16, 32):
        with sw.Database.from_synth(db, device=0, residency=1, chunk_mb=1, first_stage=fs) as g:
            r = g.search(q, B62, 2, 12, k=5)
        assert np.array_equal(r.scores, ref)
        if fs == 16:
            assert r.stats["n_rerun32"] == int((ref > 32767 - 11).sum()) >= 2


def test_streamed_async_repeated_searches():
    import torch
    db = _db(7, n=2000)
    qs = [_query(m, 9) for m in (100, 300, 700)]
    with sw.Database.from_synth(db, device=0, residency=1, chunk_mb=1) as g:
        st = torch.cuda.Stream()
        outs = []
        for q in qs * 2:                         # back-to-back: buffers reused across searches
            d = torch.empty(db.n_seqs, dtype=torch.int32, device="cuda")
            g.search_async(q, B62, 2, 12, 5, d, None, None, stream=st)
            outs.append(d)
        st.synchronize()
    for t, q in enumerate(qs * 2):
        assert np.array_equal(outs[t].cpu().numpy(), oracle.db_scores(q, db, B62, 2, 12)), t


def test_streamed_save_load_align_and_batch(tmp_path):
    db = _db(11, n=800)
    q = _query(250, 4)
    path = str(tmp_path / "db.swdb")
    with sw.Database.from_synth(db, device=0, residency=1, chunk_mb=1) as g:
        g.save(path)
        r = g.search(q, B62, 2, 12, k=10)
        al = g.align(q, B62, 2, 12, r.topk_ids)
        with pytest.raises(sw.SwError) as e:
            g.search_batch([q, q], B62, 2, 12)
        assert e.value.code == sw.SW_EINVAL
    for a in al:
        assert {k: a[k] for k in ("score", "q_begin", "q_end", "s_begin", "s_end", "ops")} == \
            oracle.sw_align(q, db.seq(a["subject"]), B62, 2, 12)
    for residency in (0, 1):
        with sw.Database.load(path, device=0, residency=residency, chunk_mb=1) as g:
            r2 = g.search(q, B62, 2, 12, k=10)
        assert np.array_equal(r2.scores, r.scores)
