"""The synthetic input generators: determinism, C == numpy reference,
shard/subset independence, and the distribution shape of the recipe."""
import numpy as np

from swdata import CONFIGS, db_lengths, gen_residues, make_db, make_query, manifest_hash, stream_key
from swdata import synth


def test_c_generator_matches_numpy_reference():
    if synth._clib() is None:
        return
    for key, start, n in [(1, 0, 1000), (stream_key(0, "C2", "res"), 10**9, 200_000)]:
        assert np.array_equal(gen_residues(key, start, n), gen_residues(key, start, n, use_c=False))
    q = make_query("C4")
    for i in range(10):
        k = stream_key(0, "C4", "plant", i)
        assert np.array_equal(synth._mutate(q, k), synth._mutate(q, k, use_c=False))


def test_subset_generation_is_shard_independent():
    full = make_db("C1")
    ids = np.array([5, 6, 7, 100, 9999, 0], dtype=np.int64)
    sub = make_db("C1", ids=ids)
    for j, i in enumerate(ids):
        assert np.array_equal(sub.seq(j), full.seq(int(i)))
    assert manifest_hash(make_db("C1")) == manifest_hash(full)


def test_length_distribution():
    L, kind = db_lengths("C2")
    assert L.min() >= 10 and L.max() <= 5000
    assert abs(L.mean() - 350) < 3
    assert (kind == 0).all()


def test_residue_composition():
    r = gen_residues(stream_key(0, "t"), 0, 2_000_000)
    assert r.max() < 20
    f = np.bincount(r, minlength=20) / r.size
    p = np.array([synth.BACKGROUND[c] for c in "ARNDCQEGHILKMFPSTWYV"])
    assert np.abs(f - p / p.sum()).max() < 2e-3


def test_planted_copies_c4_shape():
    cfg = CONFIGS["C4"]
    q = make_query(cfg)
    ident = []
    for i in range(20):
        s = synth._mutate(q, stream_key(0, "C4", "plant", i))
        assert abs(s.size - q.size) < 120
        ident.append(np.mean(s[:10] == q[:10]))
    assert 0.6 < np.mean(ident) <= 0.95   # ~80% identity before the first indel


def test_s16_layout():
    L, kind = db_lengths("S16")
    assert (kind == 3).sum() == 200 and (kind == 2).sum() == 200
    assert (L[kind == 3] == 8000).all()
