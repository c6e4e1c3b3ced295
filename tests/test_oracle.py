"""Pins for oracle/ against things other than itself (CPU only, -m "not gpu").

Every check here is fixed by the paper, by mathematics, or by an independent
formulation: brute-force enumeration of alignments, Gotoh's -inf boundary full
matrix, textbook special cases (Kadane, linear-gap SW), closed forms, and
invariants.  A plausible slip in sw_oracle.c (dropped term, wrong sign,
swapped operand or index, wrong boundary) fails at least one of them.
"""
import os

import numpy as np
import pytest

import oracle
from oracle.brute import brute_force
from swdata import blosum50, blosum62, encode, matrix32, random_db

HERE = os.path.dirname(os.path.abspath(__file__))
B62 = matrix32(blosum62())
B50 = matrix32(blosum50())


def _golden():
    rows = []
    with open(os.path.join(HERE, "golden", "spec_examples.txt")) as f:
        for ln in f:
            if ln.startswith("#") or not ln.strip():
                continue
            q, s, mat, a, b, e = ln.split()
            rows.append((q, s, mat, int(a), int(b), int(e)))
    return rows


@pytest.mark.parametrize("q,s,mat,alpha,beta,expected", _golden())
def test_spec_worked_examples(q, s, mat, alpha, beta, expected):
    M = B62 if mat == "blosum62" else B50
    assert oracle.sw_score(encode(q), encode(s), M, alpha, beta) == expected
    assert brute_force(encode(q), encode(s), M, alpha, beta) == expected


def _rand_case(rng, maxlen=6):
    a = int(rng.integers(2, 5))                        # small alphabets: repeats and ties
    M = rng.integers(-6, 8, size=(a, a))               # asymmetric, off-diagonals can beat the diagonal
    alpha = int(rng.integers(0, 5))
    beta = alpha + int(rng.integers(0, 7))
    if rng.random() < 0.1:
        alpha = beta = 0
    q = rng.integers(0, a, size=int(rng.integers(1, maxlen + 1)))
    s = rng.integers(0, a, size=int(rng.integers(1, maxlen + 1)))
    return q, s, M, alpha, beta


def test_brute_force_equals_eq1():
    """Enumeration of all local alignments (|Q|,|S| <= 6) == Eq. 1 (pins recurrence,
    boundary, gap-run charging and fsbt orientation via asymmetric matrices)."""
    rng = np.random.default_rng(2024)
    for _ in range(600):
        q, s, M, a, b = _rand_case(rng)
        assert oracle.sw_score(q, s, M, a, b) == brute_force(q, s, M, a, b), (q, s, M, a, b)


def test_brute_force_full_6x6():
    rng = np.random.default_rng(7)
    for _ in range(25):
        a = 3
        M = rng.integers(-4, 6, size=(a, a))
        q = rng.integers(0, a, size=6)
        s = rng.integers(0, a, size=6)
        for (al, be) in [(0, 0), (1, 3), (2, 12), (3, 3)]:
            assert oracle.sw_score(q, s, M, al, be) == brute_force(q, s, M, al, be)


def test_orientation_row_is_query():
    """fsbt(S1[i], S2[j]) with S1 = query (reading R1): an asymmetric matrix
    distinguishes M[q][s] from M[s][q]."""
    M = np.zeros((32, 32), dtype=np.int8)
    M[0, 1] = 7      # query residue 0 vs subject residue 1
    M[1, 0] = 3
    assert oracle.sw_score([0], [1], M, 1, 1) == 7
    assert oracle.sw_score([1], [0], M, 1, 1) == 3


def test_gotoh_minus_inf_boundary_equivalence():
    """Printed 0 boundary (E(0,j)=F(i,0)=0) == Gotoh -inf boundary (reading R2),
    on inputs up to 40x40."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        m, n = int(rng.integers(1, 41)), int(rng.integers(1, 41))
        q = rng.integers(0, 20, size=m)
        s = rng.integers(0, 20, size=n)
        a = int(rng.integers(0, 6))
        b = a + int(rng.integers(0, 14))
        M = B62 if rng.random() < 0.5 else matrix32(rng.integers(-8, 9, size=(24, 24)))
        assert oracle.sw_score(q, s, M, a, b) == oracle.sw_full(q, s, M, a, b)


def test_closed_form_self_alignment():
    """Self-score == sum of diagonal when M[a][a] > 0 and M[a][b] <= M[a][a]
    (row dominance; reading R13)."""
    rng = np.random.default_rng(3)
    for M24 in (blosum62(), blosum50()):
        sub = M24[:20, :20].astype(int)
        assert all(sub[a, a] > 0 for a in range(20))
        assert all(sub[a, b] <= sub[a, a] for a in range(20) for b in range(20))   # precondition
        M = matrix32(M24)
        for _ in range(30):
            s = rng.integers(0, 20, size=int(rng.integers(1, 400)))
            assert oracle.sw_score(s, s, M, 2, 12) == int(sum(int(M24[c, c]) for c in s))


def test_closed_form_needs_row_dominance():
    """The c13 counterexample: positive diagonal without row dominance."""
    M = np.zeros((32, 32), dtype=np.int8)
    M[0, 0] = M[1, 1] = 1
    M[0, 1] = M[1, 0] = 10
    s = [0, 1]
    assert brute_force(s, s, M, 1, 1) == 10
    assert oracle.sw_score(s, s, M, 1, 1) == 10      # not 1 + 1


def test_single_residue_query():
    """m = 1: H(1,j) = max(0, fsbt(q1, s_j)) since E, F < H-values of zero rows."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        q = rng.integers(0, 24, size=1)
        s = rng.integers(0, 24, size=int(rng.integers(1, 60)))
        a = int(rng.integers(0, 4))
        b = a + int(rng.integers(0, 5))
        assert oracle.sw_score(q, s, B62, a, b) == max(0, max(int(B62[q[0], c]) for c in s))


def test_all_nonpositive_matrix_scores_zero():
    rng = np.random.default_rng(6)
    M = -np.abs(rng.integers(0, 6, size=(32, 32))).astype(np.int8)
    for _ in range(50):
        q = rng.integers(0, 24, size=int(rng.integers(1, 50)))
        s = rng.integers(0, 24, size=int(rng.integers(1, 50)))
        assert oracle.sw_score(q, s, M, 0, 0) == 0


def _kadane_diagonals(q, s, M):
    """Textbook ungapped local alignment: best max-subarray over every diagonal."""
    best = 0
    m, n = len(q), len(s)
    for d in range(-(m - 1), n):
        cur = 0
        for i in range(m):
            j = i + d
            if 0 <= j < n:
                cur = max(0, cur + int(M[q[i], s[j]]))
                best = max(best, cur)
    return best


def test_ungapped_limit_is_kadane():
    """beta above every attainable H -> no gap can open."""
    rng = np.random.default_rng(8)
    for _ in range(150):
        m, n = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        q = rng.integers(0, 20, size=m)
        s = rng.integers(0, 20, size=n)
        beta = min(m, n) * 11 + 1
        alpha = int(rng.integers(0, beta + 1))
        assert oracle.sw_score(q, s, B62, alpha, beta) == _kadane_diagonals(q, s, B62)


def _linear_gap_sw(q, s, M, g):
    """Textbook Smith-Waterman with linear gap penalty g (full matrix)."""
    m, n = len(q), len(s)
    H = np.zeros((m + 1, n + 1), dtype=np.int64)
    for i in range(1, m + 1):
        for j in range(1, n + 1):
            H[i, j] = max(0, H[i - 1, j - 1] + int(M[q[i - 1], s[j - 1]]), H[i - 1, j] - g, H[i, j - 1] - g)
    return int(H.max())


def test_alpha_equals_beta_is_linear_gap():
    rng = np.random.default_rng(9)
    for _ in range(150):
        m, n = int(rng.integers(1, 35)), int(rng.integers(1, 35))
        q = rng.integers(0, 20, size=m)
        s = rng.integers(0, 20, size=n)
        g = int(rng.integers(0, 10))
        assert oracle.sw_score(q, s, B62, g, g) == _linear_gap_sw(q, s, B62, g)


def test_invariants():
    rng = np.random.default_rng(10)
    for _ in range(200):
        m, n = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        q = rng.integers(0, 20, size=m)
        s = rng.integers(0, 20, size=n)
        a = int(rng.integers(0, 4))
        b = a + int(rng.integers(0, 12))
        sc = oracle.sw_score(q, s, B62, a, b)
        assert sc >= 0
        assert sc <= min(m, n) * 11                                    # min(m,n) * s_max
        assert sc == oracle.sw_score(s, q, B62, a, b)                   # symmetric matrix
        assert oracle.sw_score(q, s, B62, a + 1, b + 1) <= sc           # monotone in alpha, beta
        assert oracle.sw_score(q, s, B62, a, b + 3) <= sc
        ext = np.concatenate([s, rng.integers(0, 20, size=5)])
        assert oracle.sw_score(q, ext, B62, a, b) >= sc                # appending residues
        M2 = B62.copy()
        M2[q[0], s[0]] += 3
        assert oracle.sw_score(q, s, M2, a, b) >= sc                   # raising one entry
        # DUMMY (24) padding anywhere before/after either sequence is score-neutral (R9)
        pad = lambda x, k1, k2: np.concatenate([np.full(k1, 24), x, np.full(k2, 24)])
        assert oracle.sw_score(pad(q, 3, 7), pad(s, 5, 2), B62, a, b) == sc


def test_zero_length_subject_scores_zero():
    assert oracle.sw_score([1, 2, 3], [], B62, 2, 12) == 0


def test_db_scores_threading_invariant():
    db = random_db(1, np.random.default_rng(0).integers(0, 300, size=500))
    q = random_db(2, [200]).residues
    ref = np.array([oracle.sw_score(q, db.seq(i), B62, 2, 12) for i in range(db.n_seqs)], dtype=np.int32)
    for t in (1, 3, 8):
        assert np.array_equal(oracle.db_scores(q, db, B62, 2, 12, nthreads=t), ref)
    samp = np.array([5, 17, 499, 0])
    assert np.array_equal(oracle.db_scores(q, db, B62, 2, 12, sample=samp), ref[samp])


def test_topk_is_full_sort_with_id_tiebreak():
    rng = np.random.default_rng(12)
    sc = rng.integers(0, 6, size=300).astype(np.int32)     # many ties
    ids = rng.permutation(300).astype(np.int64) * 3
    ki, ks = oracle.topk(sc, 50, ids)
    ref = sorted(zip((-sc).tolist(), ids.tolist()))[:50]
    assert ks.tolist() == [-x for x, _ in ref]
    assert ki.tolist() == [i for _, i in ref]
    ki, ks = oracle.topk(sc[:4], 6)
    assert ki[4:].tolist() == [-1, -1] and ks[4:].tolist() == [-1, -1]
