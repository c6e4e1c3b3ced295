"""GPU parity: every score from the CUDA path (through the C ABI) equals the
oracle bit-exactly; the top-k equals the oracle's full-sort ranking.

Small cases cover every subject exhaustively (several query tiles, ragged
tails, word/tile boundaries, degenerate parameters, saturation limits).
"""
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
    return gen_residues(stream_key(seed, "test-query", m), 0, m)


def _check(db, q, M, alpha, beta, k=10, first_stage=16, gids=None, **kw):
    with sw.Database(db.residues, db.offsets, db.lengths, global_ids=gids, device=0,
                     first_stage=first_stage, **kw) as g:
        res = g.search(q, M, alpha, beta, k=k)
    ref = oracle.db_scores(q, db, M, alpha, beta)
    bad = np.nonzero(res.scores != ref)[0]
    assert bad.size == 0, (f"{bad.size}/{ref.size} differ; first id {bad[0]} len {db.lengths[bad[0]]}: "
                           f"gpu {res.scores[bad[0]]} oracle {ref[bad[0]]}")
    ti, ts = oracle.topk(ref, k, gids)
    assert np.array_equal(res.topk_scores, ts)
    assert np.array_equal(res.topk_ids, ti)
    return res


def test_lengths_0_to_300_exhaustive():
    db = random_db(1, np.arange(0, 301))
    for m in (1, 7, 8, 9, 63, 64, 65, 144):
        _check(db, _query(m), B62, 2, 12)


@pytest.mark.parametrize("m", [127, 128, 129, 191, 200, 464, 1000])
@pytest.mark.parametrize("long_threshold", [-1, 0, 64])
def test_query_tiles_and_ragged_tail(m, long_threshold):
    """long_threshold -1: all inter-task; 0: auto; 64: every group longer than 64
    columns goes pair-wise through the intra-task wavefront (multi-pass for m > 512)."""
    rng = np.random.default_rng(m)
    lens = np.concatenate([rng.integers(0, 700, size=900), [5, 6, 7, 11, 12, 13, 1, 0]])
    _check(random_db(m, lens), _query(m, 1), B62, 2, 12, long_threshold=long_threshold)


@pytest.mark.parametrize("m", [1, 9, 16, 17, 511, 512, 513, 1100])
def test_intra_wavefront_pass_boundaries(m):
    """Intra-task path: 16 rows per lane, 512 rows per pass; lane/pass edges."""
    rng = np.random.default_rng(1000 + m)
    lens = np.concatenate([rng.integers(100, 1500, size=150), [1, 2, 33]])
    _check(random_db(2000 + m, lens), _query(m, 2), B62, 2, 12, long_threshold=1)


@pytest.mark.parametrize("m", [1, 8, 100, 144, 300, 512])
@pytest.mark.parametrize("tuning", [{}, {"intra_chain": -1}, {"intra_isolate": 1}, {"intra_isolate": -1}])
def test_chained_intra_stream(m, tuning):
    """Single-pass queries: a warp's pair items run as one chained stream through the
    lanes (items of 1..60 steps, i.e. shorter and longer than the lane lag, empty
    slots of partial groups, the last pairs of the queue).  Chained, per-item
    (intra_chain -1) and isolated-warp runs all give the oracle's scores."""
    rng = np.random.default_rng(31 + m)
    lens = np.concatenate([rng.integers(0, 12, size=300), rng.integers(0, 240, size=700),
                           rng.integers(200, 900, size=60), [0, 1, 2, 3, 5]])
    rng.shuffle(lens)
    db = random_db(3100 + m, lens)
    _check(db, _query(m, 31), B62, 2, 12, k=12, long_threshold=1, tuning=tuning)


@pytest.mark.parametrize("m", [40, 144, 300, 512])
@pytest.mark.parametrize("tuning", [{"intra_isolate": 1}, {"intra_isolate": 1, "intra_split": -1}])
def test_split_critical_pairs(m, tuning):
    """The isolated warps' longest pairs (>= 1,024 columns) are cut into two column
    segments, the second run speculatively from a zero boundary and repaired from
    the first's final rows.  Random pairs (the repair meets the speculative rows
    within a checkpoint or two), planted query copies straddling the cut (it meets
    them only past the copy) and a long run of copies (it never meets them before
    the end): every score equals the oracle's, with and without the split."""
    rng = np.random.default_rng(700 + m)
    q = _query(m, 70)
    lens = np.concatenate([rng.integers(1024, 3200, size=70), rng.integers(0, 300, size=400)])
    db = random_db(7000 + m, lens)
    for t in range(0, 20, 3):                    # copies around the middle of the pair's columns
        n = int(lens[t])
        at = max(0, min(n - m, (n + 64) // 2 - m // 2 + int(rng.integers(-40, 40))))
        db.residues[db.offsets[t] + at:db.offsets[t] + at + min(m, n)] = q[:min(m, n - at)]
    n = int(lens[1])
    for at in range(0, n - m, m):                # back-to-back copies over the whole subject
        db.residues[db.offsets[1] + at:db.offsets[1] + at + m] = q
    _check(db, q, B62, 2, 12, k=15, long_threshold=1, tuning=tuning)


@pytest.mark.parametrize("alpha,beta", [(0, 0), (1, 1), (2, 12), (1, 12), (5, 40), (0, 30), (3, 32767)])
def test_gap_parameters(alpha, beta):
    rng = np.random.default_rng(alpha * 100 + beta)
    db = random_db(7, rng.integers(1, 400, size=700))
    _check(db, _query(300, 2), B62, alpha, beta)


@pytest.mark.parametrize("path", ["auto", "inter_big", "intra"])
def test_fixed_gap_instances_equal_generic(path):
    """The paper's 10-2k penalties (alpha 2, beta 12) run first-pass instances (inter-task,
    intra-task wavefront, paired queries) with them as immediates; sw_tuning.generic_gaps = 1
    forces the register instances.  Both give the oracle's scores on tiles, ragged tails,
    wide groups (own slabs), the wavefront and planted copies past LIMIT16 (int32 reruns);
    neighbouring penalties take the generic instances."""
    big = path == "inter_big"
    lt = {"auto": 0, "inter_big": -1, "intra": 1}[path]
    rng = np.random.default_rng(4212 + big)
    lens = np.concatenate([rng.integers(0, 700, size=800), [6400, 6400, 0, 1]])
    if big:
        lens = np.concatenate([lens, rng.integers(6200, 7000, size=70)])
    db = random_db(4212 + big, lens)
    q = _query(6600, 42)
    db.residues[db.offsets[800]:db.offsets[800] + 6400] = q[:6400]          # self-score > LIMIT16
    db.residues[db.offsets[801]:db.offsets[801] + 6400] = q[100:6500]
    for m in (100, 6600):
        for tuning in ({}, {"generic_gaps": 1}):
            r = _check(db, q[:m], B62, 2, 12, k=6, long_threshold=lt, tuning=tuning)
            if m == 6600:
                assert r.stats["n_rerun32"] >= 1
        _check(db, q[:m], B62, 2, 13, long_threshold=lt)
        _check(db, q[:m], B62, 3, 12, long_threshold=lt)
    qs = [q[:300], q[1000:1290]]                                             # paired into one int16x2 pass
    for tuning in ({}, {"generic_gaps": 1}):
        with sw.Database.from_synth(db, device=0, long_threshold=lt, tuning=tuning) as g:
            r = g.search_batch(qs, B62, 2, 12, k=5)
        for i, qq in enumerate(qs):
            assert np.array_equal(r.scores[i], oracle.db_scores(qq, db, B62, 2, 12))


def test_blosum50_and_random_asymmetric_matrices():
    rng = np.random.default_rng(3)
    db = random_db(8, rng.integers(1, 500, size=600))
    _check(db, _query(250, 3), B50, 2, 12)
    for t in range(3):
        M = np.zeros((32, 32), dtype=np.int8)
        M[:24, :24] = rng.integers(-128 if t == 0 else -10, 128 if t == 0 else 12, size=(24, 24))
        _check(db, _query(180, 4 + t), M, 1 + t, 10 + 3 * t)


def test_first_stage_32_equals_oracle():
    rng = np.random.default_rng(4)
    db = random_db(9, rng.integers(0, 600, size=800))
    _check(db, _query(333, 5), B62, 2, 12, first_stage=32)


@pytest.mark.parametrize("first_stage", [8, 32])
@pytest.mark.parametrize("m", [1, 100, 333, 1000])
def test_first_stage_8_and_32(first_stage, m):
    rng = np.random.default_rng(400 + m)
    db = random_db(40 + m, rng.integers(0, 700, size=1200))
    r = _check(db, _query(m, 16), B62, 2, 12, first_stage=first_stage)
    assert r.stats["first_stage"] == first_stage


def test_int8_stage_falls_back_when_bytes_do_not_fit():
    db = random_db(41, np.random.default_rng(1).integers(1, 300, size=300))
    r = _check(db, _query(200, 17), B62, 2, 300, first_stage=8)       # beta > 255
    assert r.stats["first_stage"] == 16


def test_escalation_chain_8_16_32_exact():
    """Planted copies whose self-scores straddle LIMIT8 = 255-(s_max+B) = 240 and
    LIMIT16 = 32756 (BLOSUM62): every score exact, and exactly the subjects above
    each limit are re-aligned at the next width."""
    M24 = blosum62()
    limit8, limit16 = 255 - (11 + 4), 32767 - 11
    targets = [limit8 - 1, limit8, limit8 + 1, 300, 1000, limit16 - 1, limit16, limit16 + 1, 40000]
    seqs = [_seq_with_self_score(t, M24) for t in targets]
    rng = np.random.default_rng(9)
    lens = np.concatenate([[x.size for x in seqs], rng.integers(1, 400, size=500)])
    db = random_db(42, lens)
    for i, x in enumerate(seqs):
        db.residues[db.offsets[i]:db.offsets[i] + x.size] = x
    for qi, q in enumerate((seqs[4], seqs[-1])):      # query = one of the planted sequences
        r = _check(db, q, B62, 2, 12, first_stage=8)
        ref = oracle.db_scores(q, db, B62, 2, 12)
        assert r.stats["n_rerun16"] == int((ref > limit8).sum())
        assert r.stats["n_rerun32"] == int((ref > limit16).sum())


@pytest.mark.parametrize("n", [1, 33, 12288, 12289, 65536, 65537])
def test_ranking_paths_and_sizes(n):
    """The ranking paths by database size: n <= 12,288 one fused launch (scatter +
    keys in shared memory + top-k), n <= 65,536 one CTA over global keys, larger the
    multi-CTA radix select; k <= 32 by block-wide argmax rounds, larger k by radix
    select + bitonic sort.  Heavy score ties (4-letter alphabet, short subjects) with
    permuted global ids: the top-k equals the oracle's (score desc, id asc) order."""
    rng = np.random.default_rng(n)
    db = random_db(700 + n % 97, rng.integers(0, 24, size=n), alphabet=4)
    gids = rng.permutation(np.arange(3 * n, dtype=np.int64))[:n]
    q = _query(17, 3)
    ref = oracle.db_scores(q, db, B62, 2, 12)
    with sw.Database(db.residues, db.offsets, db.lengths, global_ids=gids, device=0) as g:
        for k in (1, 10, 32, 33, 100):
            r = g.search(q, B62, 2, 12, k=k)
            assert np.array_equal(r.scores, ref)
            ti, ts = oracle.topk(ref, k, gids)
            assert np.array_equal(r.topk_ids, ti) and np.array_equal(r.topk_scores, ts), k


def test_rerun_compaction_above_one_cta():
    """More than 65,536 subjects with int16-saturating planted copies scattered over
    the sorted order: the multi-CTA flag compaction gives the same int32 reruns as the
    one-CTA path (exact scores, exact rerun count)."""
    rng = np.random.default_rng(65)
    q = _query(6500, 65)
    n = 70000
    lens = rng.integers(1, 60, size=n)
    hot = rng.choice(n, size=12, replace=False)
    lens[hot] = 6400 + rng.integers(0, 100, size=hot.size)
    db = random_db(65, lens)
    for t in hot:
        db.residues[db.offsets[t]:db.offsets[t] + 6400] = q[:6400]
    r = _check(db, q, B62, 2, 12, k=20)
    ref = oracle.db_scores(q, db, B62, 2, 12)
    assert r.stats["n_rerun32"] == int((ref > 32767 - 11).sum()) == hot.size


@pytest.mark.parametrize("tile_rows,threads", [(32, 0), (32, 384), (48, 0), (48, 512), (64, 0)])
def test_tile_rows_invariance(tile_rows, threads):
    """Scores do not depend on the register-tile height or CTA size (SPEC.md:252-255,
    T-invariance; the non-48 / non-384 instances live in the ablation build)."""
    rng = np.random.default_rng(44)
    db = random_db(19, rng.integers(0, 900, size=1500))
    _check(db, _query(377, 15), B62, 2, 12, long_threshold=-1, tuning={"tile_rows": tile_rows, "threads": threads})


def test_ties_and_global_ids():
    one = _query(120, 6)
    lens = np.full(300, 120)
    db = random_db(10, lens)
    for i in range(0, 300, 3):             # many identical subjects -> ties
        db.residues[db.offsets[i]:db.offsets[i] + 120] = one
    gids = np.random.default_rng(0).permutation(10_000)[:300].astype(np.int64) * 7
    _check(db, _query(100, 7), B62, 2, 12, k=37, gids=gids)
    _check(db, one, B62, 2, 12, k=50, gids=gids)


def test_k_larger_than_n_and_tiny_dbs():
    db = random_db(11, [5, 0, 17])
    r = _check(db, _query(40, 8), B62, 2, 12, k=6)
    assert r.topk_ids[3:].tolist() == [-1, -1, -1]
    _check(random_db(12, [0]), _query(3, 9), B62, 2, 12, k=1)
    _check(random_db(13, [1]), _query(1, 9), B62, 2, 12, k=1)


def test_large_k_uses_full_sort_path():
    rng = np.random.default_rng(5)
    db = random_db(14, rng.integers(1, 100, size=6000))
    _check(db, _query(50, 10), B62, 2, 12, k=5000)


def _seq_with_self_score(target, M24):
    """A sequence of standard residues whose diagonal sum is exactly `target`
    (closed form: self-score = sum of diagonal under row dominance, reading R13)."""
    import itertools
    diag = {int(M24[c, c]): c for c in range(20)}
    w = max(diag)
    out = []
    t = target
    while t > 4 * w:
        out.append(diag[w])
        t -= w
    for n in range(1, 6):
        for combo in itertools.combinations_with_replacement(sorted(diag), n):
            if sum(combo) == t:
                return np.array(out + [diag[v] for v in combo], dtype=np.uint8)
    raise AssertionError(t)


def test_int16_saturation_limits_exact():
    """Planted exact copies whose self-score sits at LIMIT16-1, LIMIT16, LIMIT16+1
    (LIMIT16 = 32767 - s_max): scores stay exact and exactly the subjects above
    the limit are re-aligned in int32 (DESIGN.md §"Saturation")."""
    M24 = blosum62()
    limit = 32767 - 11
    for target in (limit - 1, limit, limit + 1, 32767, 32768, 40000):
        q = _seq_with_self_score(target, M24)
        assert sum(int(M24[c, c]) for c in q) == target
        lens = np.array([q.size, 50, q.size, 300, 0])
        db = random_db(15, lens)
        db.residues[db.offsets[0]:db.offsets[0] + q.size] = q
        db.residues[db.offsets[2]:db.offsets[2] + q.size] = q[::-1]
        with sw.Database(db.residues, db.offsets, db.lengths, device=0) as g:
            res = g.search(q, B62, 2, 12, k=3)
        ref = oracle.db_scores(q, db, B62, 2, 12)
        assert ref[0] == target
        assert np.array_equal(res.scores, ref), (target, res.scores, ref)
        assert res.stats["n_rerun32"] == int((ref > limit).sum())


def test_flags_reset_between_searches_on_one_handle():
    """The int16 saturation flags are zeroed per search -- for small databases
    inside k_profiles, with the intra-task pass launched as its programmatic
    dependent: a saturating search, a clean one and the saturating one again on
    one handle each re-align exactly the subjects above LIMIT16."""
    M24 = blosum62()
    limit = 32767 - 11
    q_hot = _seq_with_self_score(40000, M24)
    lens = np.concatenate([[q_hot.size, 50, q_hot.size], np.arange(1, 400, 7), [5000, 0]])
    db = random_db(16, lens)
    db.residues[db.offsets[0]:db.offsets[0] + q_hot.size] = q_hot
    db.residues[db.offsets[2]:db.offsets[2] + q_hot.size] = q_hot[::-1]
    q_cold = _query(700, seed=5)
    with sw.Database(db.residues, db.offsets, db.lengths, device=0) as g:
        for q in (q_hot, q_cold, q_hot, q_cold):
            res = g.search(q, B62, 2, 12, k=5)
            ref = oracle.db_scores(q, db, B62, 2, 12)
            assert np.array_equal(res.scores, ref), q.size
            assert res.stats["n_rerun32"] == int((ref > limit).sum()), q.size


def test_s16_style_long_query_reruns():
    """8,000-residue query vs exact and near copies: self-scores ~42k exceed
    int16, forcing the int32 rerun (stress case S16)."""
    q = _query(8000, 11)
    rng = np.random.default_rng(6)
    lens = np.concatenate([rng.integers(50, 800, size=300), [8000, 8000, 4000]])
    db = random_db(16, lens)
    db.residues[db.offsets[300]:db.offsets[300] + 8000] = q
    mut = q.copy()
    pos = rng.choice(8000, size=1600, replace=False)
    mut[pos] = (mut[pos] + 1 + rng.integers(0, 19, size=pos.size)) % 20
    db.residues[db.offsets[301]:db.offsets[301] + 8000] = mut
    db.residues[db.offsets[302]:db.offsets[302] + 4000] = q[2000:6000]
    r = _check(db, q, B62, 2, 12, k=5)
    _check(db, q, B62, 2, 12, k=5, long_threshold=1000)     # long copies via the intra path
    ref = oracle.db_scores(q, db, B62, 2, 12)
    assert ref[300] > 40000 and r.stats["n_rerun32"] == int((ref > 32767 - 11).sum()) >= 1


def test_async_api_with_torch_stream():
    import torch
    rng = np.random.default_rng(8)
    db = random_db(17, rng.integers(0, 500, size=2000))
    q = _query(200, 12)
    ref = oracle.db_scores(q, db, B62, 2, 12)
    ti, ts = oracle.topk(ref, 10)
    with sw.Database.from_synth(db, device=0) as g:
        s = torch.cuda.Stream()
        d_sc = torch.empty(db.n_seqs, dtype=torch.int32, device="cuda")
        d_ti = torch.empty(10, dtype=torch.int64, device="cuda")
        d_ts = torch.empty(10, dtype=torch.int32, device="cuda")
        for _ in range(2):      # back-to-back searches on one handle serialise
            g.search_async(q, B62, 2, 12, 10, d_sc, d_ti, d_ts, stream=s)
        s.synchronize()
    assert np.array_equal(d_sc.cpu().numpy(), ref)
    assert np.array_equal(d_ti.cpu().numpy(), ti) and np.array_equal(d_ts.cpu().numpy(), ts)


def test_search_validation_errors():
    db = random_db(18, [10, 20])
    with sw.Database.from_synth(db, device=0) as g:
        q = _query(10, 13)
        for args, code in [((q, B62, 3, 2, 5), sw.SW_EINVAL),          # beta < alpha
                           ((q, B62, 2, 12, 0), sw.SW_EINVAL),         # k < 1
                           ((np.array([], np.uint8), B62, 2, 12, 5), sw.SW_EINVAL),
                           ((np.array([1, 30], np.uint8), B62, 2, 12, 5), sw.SW_EINVAL)]:
            with pytest.raises(sw.SwError) as ei:
                g.search(*args[:4], k=args[4])
            assert ei.value.code == code
        Mbad = B62.copy()
        Mbad[30, 1] = 2
        with pytest.raises(sw.SwError):
            g.search(q, Mbad, 2, 12, k=2)
        Mbig = np.zeros((32, 32), np.int8)
        Mbig[:24, :24] = 127
        qbig = np.zeros((1 << 31) // 127 + 1, dtype=np.uint8)
        with pytest.raises(sw.SwError) as ei:
            g.search(qbig, Mbig, 2, 12, k=2)
        assert ei.value.code == sw.SW_ERANGE


@pytest.mark.parametrize("long_threshold", [0, 64, -1])
def test_batched_queries_equal_single_searches(long_threshold):
    """f1: queries paired in one int16x2 pass give exactly the per-query oracle
    scores and top-k (odd count, unequal lengths, lengths too far apart to pair,
    one query too long to pair).  long_threshold 64 sends most groups pair by
    pair through the two intra-task passes that run beside the joint pass."""
    rng = np.random.default_rng(77)
    db = random_db(77, np.concatenate([rng.integers(0, 900, size=1500), [0, 1, 5000]]))
    qs = [_query(m, 30 + i) for i, m in enumerate([1, 100, 333, 464, 420, 47, 2600, 129, 120])]
    with sw.Database.from_synth(db, device=0, long_threshold=long_threshold) as g:
        r = g.search_batch(qs, B62, 2, 12, k=12)
    assert r.stats["pairs"] == 2                       # (464, 420) and (129, 120): min/max >= 0.85
    for i, q in enumerate(qs):
        ref = oracle.db_scores(q, db, B62, 2, 12)
        assert np.array_equal(r.scores[i], ref), i
        ti, ts = oracle.topk(ref, 12)
        assert np.array_equal(r.topk_ids[i], ti) and np.array_equal(r.topk_scores[i], ts)


def test_batched_queries_saturation_reruns():
    """Both halves of a query pair saturate independently and are rerun exactly
    (matrix with diagonal 30 so that ~1,100-residue self-alignments pass LIMIT16)."""
    M = B62.copy()
    for c in range(20):
        M[c, c] = 30
    qa, qb = _query(1200, 50), _query(1050, 51)       # self-scores 36,000 and 31,500 (row dominance)
    lens = np.array([qa.size, qb.size, 100, 200, 0])
    db = random_db(78, lens)
    db.residues[db.offsets[0]:db.offsets[0] + qa.size] = qa
    db.residues[db.offsets[1]:db.offsets[1] + qb.size] = qb
    with sw.Database.from_synth(db, device=0) as g:
        r = g.search_batch([qa, qb], M, 2, 12, k=2)
    assert r.stats["pairs"] == 1
    refs = [oracle.db_scores(q, db, M, 2, 12) for q in (qa, qb)]
    assert refs[0][0] == 36000 and refs[1][1] == 31500
    for i in range(2):
        assert np.array_equal(r.scores[i], refs[i])
    assert r.stats["n_rerun32"] == sum(int((x > 32767 - 30).sum()) for x in refs)


def test_persistent_index_roundtrip(tmp_path):
    """f2: save the packed index, load it (mmap, no re-pack): identical results."""
    rng = np.random.default_rng(90)
    db = random_db(90, rng.integers(0, 800, size=3000))
    gids = rng.permutation(100_000)[:3000].astype(np.int64)
    q = _query(250, 90)
    path = str(tmp_path / "db.swb")
    with sw.Database.from_synth(db, global_ids=gids, device=0) as g:
        r0 = g.search(q, B62, 2, 12, k=25)
        g.save(path)
        info0 = g.info()
    for fs in (16, 8):
        with sw.Database.load(path, device=0, first_stage=fs) as h:
            info1 = h.info()
            r1 = h.search(q, B62, 2, 12, k=25)
        assert info1["n_seqs"] == info0["n_seqs"] and info1["packed_bytes"] == info0["packed_bytes"]
        assert np.array_equal(r0.scores, r1.scores)
        assert np.array_equal(r0.topk_ids, r1.topk_ids) and np.array_equal(r0.topk_scores, r1.topk_scores)
    ref = oracle.db_scores(q, db, B62, 2, 12)
    assert np.array_equal(r1.scores, ref)


def test_index_file_matches_layout_definition(tmp_path):
    """f2: sw_db_save writes byte-for-byte the file tests/index_file.py builds from the layout's definition,
    and a hand-written file loads and searches equal to the oracle."""
    import index_file
    rng = np.random.default_rng(92)
    db = random_db(92, rng.integers(0, 400, size=700))
    gids = rng.permutation(50_000)[:700].astype(np.int64)
    crafted = str(tmp_path / "crafted.swb")
    saved = str(tmp_path / "saved.swb")
    index_file.write(crafted, index_file.build(db.residues, db.offsets, db.lengths, gids))
    with sw.Database(db.residues, db.offsets, db.lengths, global_ids=gids, device=0) as g:
        g.save(saved)
    assert open(saved, "rb").read() == open(crafted, "rb").read()
    q = _query(300, 92)
    with sw.Database.load(crafted, device=0) as h:
        r = h.search(q, B62, 2, 12, k=15)
    ref = oracle.db_scores(q, db, B62, 2, 12)
    assert np.array_equal(r.scores, ref)
    ti, ts = oracle.topk(ref, 15, gids)
    assert np.array_equal(r.topk_ids, ti) and np.array_equal(r.topk_scores, ts)


@pytest.mark.parametrize("first_stage", [16, 8, 32])
def test_very_long_subjects_exceeding_boundary_slab(first_stage):
    """Subjects longer than the per-warp boundary slab (6,144 columns): inter-task
    with slabs of their own (first pass), intra-task or rerun elsewhere, in every
    stage; scores stay exact."""
    rng = np.random.default_rng(91)
    lens = np.concatenate([rng.integers(1, 300, size=200), [7000, 9000, 20000, 6145, 6144]])
    db = random_db(91, lens)
    q = _query(700, 91)
    db.residues[db.offsets[202]:db.offsets[202] + 700] = q          # one strong hit inside the 20,000-long subject
    _check(db, q, B62, 2, 12, first_stage=first_stage, long_threshold=-1)
    with sw.Database.from_synth(db, device=0) as g:
        r = g.search_batch([q, _query(300, 92)], B62, 2, 12, k=5)
    for i, qq in enumerate([q, _query(300, 92)]):
        assert np.array_equal(r.scores[i], oracle.db_scores(qq, db, B62, 2, 12))


@pytest.mark.parametrize("max_big", [-1, 2, 1000])
def test_wide_groups_big_slabs_and_fallback(max_big):
    """Groups wider than a warp's slab take per-item slabs (the first items of the
    longest-first queue); with sw_tuning.max_big below their number (-1: none) the
    widest fall back to the intra-task wavefront.  Every split gives the oracle's scores."""
    rng = np.random.default_rng(77)
    lens = np.concatenate([rng.integers(1, 400, size=600), rng.integers(6200, 9000, size=320)])
    db = random_db(77, lens)
    q = _query(150, 77)
    for t in (600, 700, 919):                                  # strong hits inside wide subjects
        db.residues[db.offsets[t] + 3000:db.offsets[t] + 3150] = q
    _check(db, q, B62, 2, 12, k=8, long_threshold=-1, tuning={"max_big": max_big})


def test_empty_database():
    empty = random_db(3, np.zeros(0, dtype=np.int64))
    with sw.Database(empty.residues, empty.offsets, empty.lengths, device=0) as g:
        r = g.search(_query(50, 3), B62, 2, 12, k=4)
        assert r.scores.size == 0
        assert r.topk_ids.tolist() == [-1] * 4 and r.topk_scores.tolist() == [-1] * 4
        assert g.align(_query(50, 3), B62, 2, 12, []) == []


def test_destroy_releases_device_memory():
    """Every buffer a handle allocates (search, batch, traceback, streaming,
    wide-group slabs) is released by sw_db_destroy: free device memory comes back."""
    import torch
    rng = np.random.default_rng(99)
    db = random_db(99, np.concatenate([rng.integers(1, 900, 3000), [7000, 9000]]))
    qs = [_query(m, 99) for m in (300, 290, 120)]

    def cycle(residency):
        with sw.Database.from_synth(db, device=0, residency=residency, chunk_mb=1, long_threshold=64) as g:
            g.search(qs[0], B62, 2, 12, k=5)
            if residency == 0:
                g.search_batch(qs, B62, 2, 12, k=5)
            r = g.search(qs[2], B62, 2, 12, k=3)
            g.align(qs[2], B62, 2, 12, r.topk_ids)
        torch.cuda.synchronize()

    cycle(0)
    cycle(1)                                           # warm up the CUDA context and allocator
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(4):
        cycle(0)
        cycle(1)
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20, f"{(free0 - free1) >> 20} MiB not released"


def test_concurrent_handles_and_threads():
    """Two handles searched from four host threads at once (the C ABI serialises
    each handle, distinct handles run independently): every result exact."""
    import threading
    rng = np.random.default_rng(123)
    dbs = [random_db(123 + t, rng.integers(1, 800, 1500)) for t in range(2)]
    qs = [_query(m, 123) for m in (150, 400)]
    refs = {(d, i): oracle.db_scores(q, dbs[d], B62, 2, 12) for d in range(2) for i, q in enumerate(qs)}
    handles = [sw.Database.from_synth(d, device=0) for d in dbs]
    errors = []

    def worker(d, i):
        try:
            for _ in range(5):
                r = handles[d].search(qs[i], B62, 2, 12, k=5)
                if not np.array_equal(r.scores, refs[(d, i)]):
                    errors.append((d, i))
        except Exception as e:                          # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(d, i)) for d in range(2) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for h in handles:
        h.close()
    assert not errors, errors
