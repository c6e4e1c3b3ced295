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
