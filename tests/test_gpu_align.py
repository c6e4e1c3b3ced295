"""GPU parity of f3 (sw_align): every alignment returned through the C ABI
equals the oracle's full-matrix traceback (oracle.sw_align) exactly -- score,
end cell, start cell and op string -- because both implement the same
deterministic readings (R17-R19).  Independently, each alignment
re-scores (from its ops) to the score sw_search returns for that subject.
"""
import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum50, blosum62, matrix32, random_db, stream_key
from swdata.synth import SynthDB, _mutate, gen_residues

pytestmark = pytest.mark.gpu

B62 = matrix32(blosum62())
B50 = matrix32(blosum50())


def _query(m, seed=0):
    return gen_residues(stream_key(seed, "align-query", m), 0, m)


def _db_from(seqs):
    lens = np.array([s.size for s in seqs], dtype=np.int32)
    offs = np.zeros(lens.size, dtype=np.int64)
    if lens.size > 1:
        np.cumsum(lens[:-1], out=offs[1:])
    res = np.concatenate(seqs).astype(np.uint8) if lens.sum() else np.zeros(0, np.uint8)
    return SynthDB(res, offs, lens, np.arange(lens.size, dtype=np.int64), "align")


def _rescore(q, s, M, alpha, beta, a):
    i, j, total, last = a["q_begin"], a["s_begin"], 0, ""
    for op in a["ops"]:
        if op == "M":
            total += int(M[q[i]][s[j]])
            i, j = i + 1, j + 1
        elif op == "I":
            total -= alpha if last == "I" else beta
            i += 1
        else:
            total -= alpha if last == "D" else beta
            j += 1
        last = op
    assert (i, j) == (a["q_end"], a["s_end"])
    return total


def _check(db, q, M, alpha, beta, subjects=None, **kw):
    subjects = np.arange(db.n_seqs) if subjects is None else np.asarray(subjects)
    with sw.Database(db.residues, db.offsets, db.lengths, device=0, **kw) as g:
        res = g.search(q, M, alpha, beta, k=1)
        al = g.align(q, M, alpha, beta, subjects)
    assert len(al) == len(subjects)
    for a, t in zip(al, subjects):
        s = db.residues[db.offsets[t]:db.offsets[t] + db.lengths[t]]
        ref = oracle.sw_align(q, s, M, alpha, beta)
        got = {k: a[k] for k in ref}
        assert got == ref, (int(t), int(s.size), got, ref)
        assert a["subject"] == t and a["score"] == res.scores[t]
        if a["score"]:
            assert _rescore(q, s, M, alpha, beta, a) == a["score"]
    return al


def test_random_lengths_every_subject():
    rng = np.random.default_rng(5)
    db = random_db(31, np.concatenate([rng.integers(0, 400, 120), [0, 1, 2, 7, 8, 9]]))
    for m in (1, 7, 8, 9, 64, 255, 256, 257):
        _check(db, _query(m), B62, 2, 12)


@pytest.mark.parametrize("m", [100, 464, 513, 1000, 2100, 4200])
def test_planted_near_copies(m):
    """Near-copies of the query (80% identity, indels: the C4 planting model)
    give long gapped alignments crossing lane, pass and row-block edges."""
    q = _query(m, 3)
    seqs = [_mutate(q, stream_key(9, "align-plant", m, t)) for t in range(12)]
    rng = np.random.default_rng(m)
    bg = random_db(77 + m, rng.integers(50, 900, 20))
    seqs += [bg.residues[o:o + n] for o, n in zip(bg.offsets, bg.lengths)]
    pieces = []
    for t in range(6):                                    # query fragments embedded in background
        a = int(rng.integers(0, m // 2))
        pieces.append(np.concatenate([gen_residues(stream_key(t, "pad", m), 0, 40), q[a:a + m // 3],
                                      gen_residues(stream_key(t, "pad2", m), 0, 55)]))
    db = _db_from(seqs + pieces)
    al = _check(db, q, B62, 2, 12)
    assert max(a["ops"].count("I") + a["ops"].count("D") for a in al) > 0      # gapped paths exercised


@pytest.mark.parametrize("alpha,beta", [(0, 0), (0, 1), (1, 1), (3, 7), (10, 40)])
def test_gap_parameters_and_ties(alpha, beta):
    rng = np.random.default_rng(alpha * 100 + beta)
    q = _query(150, 4)
    seqs = [_mutate(q, stream_key(1, "tie", alpha, beta, t)) for t in range(5)]
    db4 = random_db(5 + beta, rng.integers(1, 300, 25), alphabet=4)   # 4 letters: many ties
    seqs += [db4.residues[o:o + n] for o, n in zip(db4.offsets, db4.lengths)]
    db = _db_from(seqs)
    _check(db, q, B50, alpha, beta)
    q4 = (q % 4).astype(np.uint8)
    _check(db, q4, B62, alpha, beta)


def test_asymmetric_matrix():
    rng = np.random.default_rng(11)
    M = np.zeros((32, 32), dtype=np.int8)
    M[:24, :24] = rng.integers(-7, 10, size=(24, 24))
    db = random_db(12, rng.integers(0, 250, 60))
    _check(db, _query(90, 5), M, 1, 5)


def test_repeats_subset_and_batching():
    rng = np.random.default_rng(13)
    db = random_db(14, np.concatenate([rng.integers(0, 600, 80), [3000, 0]]))
    q = _query(300, 6)
    subjects = np.array([80, 3, 3, 81, 0, 79, 80])
    _check(db, q, B62, 2, 12, subjects)
    _check(db, q, B62, 2, 12, np.arange(db.n_seqs), tuning={"align_ws_kb": 64})   # many small batches


def test_errors():
    db = random_db(15, [10, 20, 30])
    q = _query(20, 7)
    with sw.Database(db.residues, db.offsets, db.lengths, device=0) as g:
        with pytest.raises(sw.SwError) as e:
            g.align(q, B62, 2, 12, [3])
        assert e.value.code == sw.SW_EINVAL
        with pytest.raises(sw.SwError):
            g.align(q, B62, 13, 12, [0])
        out = (sw.sw_alignment * 1)()
        import ctypes
        buf = ctypes.create_string_buffer(8)
        idx = np.array([2], dtype=np.int64)
        M = np.ascontiguousarray(B62)
        rc = sw.lib().sw_align(g._h, q.ctypes.data, q.size, M.ctypes.data, 2, 12, idx.ctypes.data, 1, out, buf, 8)
        assert rc == sw.SW_EINVAL and b"need 50" in sw.lib().sw_last_error()
        assert g.align(q, B62, 2, 12, []) == []
