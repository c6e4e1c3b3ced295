"""Transcription checks for the embedded BLOSUM matrices (the
matrices are not in the container, so they are verified by properties)."""
import numpy as np

from swdata import ALPHABET, blosum50, blosum62, matrix32
from swdata.synth import BACKGROUND


def _check_common(M, lo, hi, star_self):
    M = M.astype(int)
    assert M.shape == (24, 24)
    assert (M == M.T).all()                                       # symmetric
    assert M.min() == lo and M.max() == hi                        # published ranges
    w = ALPHABET.index("W")
    assert M[w, w] == hi and (M[:20, :20] == hi).sum() == 1       # W-W is the unique maximum
    assert (np.diag(M)[:20] > 0).all()
    assert M[23, 23] == star_self and (M[23, :23] == lo).all()    # '*' row
    p = np.array([BACKGROUND[c] for c in ALPHABET[:20]])
    p = p / p.sum()
    assert float(p @ M[:20, :20] @ p) < 0                         # local-alignment regime
    # B (D/N) and Z (E/Q) are ambiguity codes: never above both parents' self-scores
    b, z = ALPHABET.index("B"), ALPHABET.index("Z")
    assert M[b, b] <= max(M[2, 2], M[3, 3]) and M[z, z] <= max(M[5, 5], M[6, 6])


def test_blosum62():
    M = blosum62()
    _check_common(M, -4, 11, 1)
    A, P = ALPHABET.index("A"), ALPHABET.index("P")
    assert M[A, A] == 4 and M[A, P] == -1
    assert M[ALPHABET.index("C"), ALPHABET.index("C")] == 9
    assert M[22, 22] == -1                                         # X-X negative (reading R13)


# A second transcription, typed independently of the tables in swdata/matrices.py.
B62_DIAG = dict(A=4, R=5, N=6, D=6, C=9, Q=5, E=5, G=6, H=8, I=4, L=4, K=5, M=5, F=6, P=7, S=4, T=5, W=11,
                Y=7, V=4, B=4, Z=4, X=-1)
B50_DIAG = dict(A=5, R=7, N=7, D=8, C=13, Q=7, E=6, G=8, H=10, I=5, L=5, K=6, M=7, F=8, P=10, S=5, T=5, W=15,
                Y=8, V=5, B=5, Z=5, X=-1)
B62_PAIRS = dict(WC=-2, WY=2, FY=3, IV=3, LI=2, KR=2, ED=2, HY=2, ST=1, NB=3, DB=4, EZ=4, QZ=3, LM=2, IM=1,
                 VM=1, FW=1, HN=1, RQ=1, AP=-1)


def test_second_transcription_diagonals_and_pairs():
    for M, diag in ((blosum62(), B62_DIAG), (blosum50(), B50_DIAG)):
        for c, v in diag.items():
            assert M[ALPHABET.index(c), ALPHABET.index(c)] == v, c
    M = blosum62()
    for pair, v in B62_PAIRS.items():
        i, j = ALPHABET.index(pair[0]), ALPHABET.index(pair[1])
        assert M[i, j] == v and M[j, i] == v, pair


def test_blosum50():
    M = blosum50()
    _check_common(M, -5, 15, 1)
    assert M[ALPHABET.index("C"), ALPHABET.index("C")] == 13


def test_matrix32_padding():
    for M in (blosum62(), blosum50()):
        P = matrix32(M)
        assert P.dtype == np.int8 and P.shape == (32, 32)
        assert (P[24:, :] == 0).all() and (P[:, 24:] == 0).all()   # DUMMY scores 0
        assert (P[:24, :24] == M).all()
