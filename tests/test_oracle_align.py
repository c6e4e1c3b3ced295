"""Pins for the oracle's traceback (oracle.sw_align, f3) against things other
than itself (CPU only, -m "not gpu").

* brute force: on tiny inputs the returned alignment is one of the optimal
  local alignments found by enumerating every alignment (oracle/brute.py);
* independent re-scoring: the ops re-scored column by column (fsbt for 'M',
  beta + (len-1)*alpha per maximal gap run, PAPER.md:35 / reading R4) equal
  the returned score, which equals the pinned linear-space score;
* closed form: self-alignment under row dominance is the full diagonal;
* structure: ops consume exactly the returned query/subject ranges, never
  start or end with a gap when beta > 0, and score 0 gives the empty alignment.
"""
import numpy as np
import pytest

import oracle
from oracle.brute import optimal_alignments
from swdata import blosum50, blosum62, matrix32

B62 = matrix32(blosum62())
B50 = matrix32(blosum50())


def rescore(q, s, M, alpha, beta, a):
    """Score of alignment `a` computed from its ops (independent of Eq. 1)."""
    i, j, total, last = a["q_begin"], a["s_begin"], 0, ""
    for op in a["ops"]:
        if op == "M":
            total += int(M[q[i]][s[j]])
            i += 1
            j += 1
        elif op == "I":
            total -= alpha if last == "I" else beta
            i += 1
        else:
            total -= alpha if last == "D" else beta
            j += 1
        last = op
    assert i == a["q_end"] and j == a["s_end"], "ops do not consume the returned ranges"
    return total


def _rand_matrix(rng):
    M = np.zeros((32, 32), dtype=np.int8)
    M[:24, :24] = rng.integers(-6, 9, size=(24, 24))
    return M


def test_brute_force_membership():
    rng = np.random.default_rng(1404)
    checked = 0
    for t in range(400):
        m, n = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        alph = int(rng.integers(2, 6))                     # small alphabets: many ties
        q = rng.integers(0, alph, m).astype(np.uint8)
        s = rng.integers(0, alph, n).astype(np.uint8)
        M = B62 if t % 3 == 0 else _rand_matrix(rng)
        alpha = int(rng.integers(0, 5))
        beta = alpha + int(rng.integers(1, 8))
        a = oracle.sw_align(q, s, M, alpha, beta)
        best, found = optimal_alignments(q, s, M, alpha, beta)
        assert a["score"] == best
        if best > 0:
            key = (a["q_begin"], a["q_end"], a["s_begin"], a["s_end"], a["ops"])
            assert key in found, (q, s, alpha, beta, a, sorted(found)[:5])
            checked += 1
        else:
            assert a["ops"] == "" and a["q_end"] == 0 and a["s_end"] == 0
    assert checked > 200


@pytest.mark.parametrize("mat", ["b62", "b50", "rand"])
def test_rescore_equals_score(mat):
    rng = np.random.default_rng(7)
    for t in range(120):
        m, n = int(rng.integers(1, 70)), int(rng.integers(1, 90))
        q = rng.integers(0, 20, m).astype(np.uint8)
        s = rng.integers(0, 20, n).astype(np.uint8)
        if t % 2:                                           # plant a shared segment with a gap
            seg = rng.integers(0, 20, 25).astype(np.uint8)
            q = np.concatenate([q[: m // 2], seg, q[m // 2:]]).astype(np.uint8)
            cut = int(rng.integers(3, 20))
            s = np.concatenate([s[: n // 3], seg[:cut], seg[cut + int(rng.integers(1, 4)):], s[n // 3:]])
            s = s.astype(np.uint8)
        M = {"b62": B62, "b50": B50}.get(mat)
        if M is None:
            M = _rand_matrix(rng)
        alpha = int(rng.integers(0, 4))
        beta = alpha + int(rng.integers(1, 14))
        a = oracle.sw_align(q, s, M, alpha, beta)
        assert a["score"] == oracle.sw_score(q, s, M, alpha, beta)
        if a["score"] > 0:
            assert rescore(q, s, M, alpha, beta, a) == a["score"]
            assert a["ops"][0] == "M" and a["ops"][-1] == "M"
            assert a["ops"].count("M") + a["ops"].count("I") == a["q_end"] - a["q_begin"]


def test_self_alignment_is_full_diagonal():
    rng = np.random.default_rng(3)
    for M in (B62, B50):
        for n in (1, 2, 17, 150):
            q = rng.integers(0, 20, n).astype(np.uint8)
            a = oracle.sw_align(q, q, M, 2, 12)
            assert a["score"] == int(sum(int(M[x][x]) for x in q))
            assert (a["q_begin"], a["q_end"], a["s_begin"], a["s_end"]) == (0, n, 0, n)
            assert a["ops"] == "M" * n


def test_gap_run_reconstructed():
    # subject = query with 5 residues removed from the middle; the unique
    # best alignment bridges them with one 'I' run of length 5
    q = np.array([17, 4, 18, 13, 5, 8, 9, 10, 11, 12, 14, 15, 16, 7, 6, 3, 2, 1, 19, 0, 4, 17, 18, 13],
                 dtype=np.uint8)
    s = np.concatenate([q[:10], q[15:]]).astype(np.uint8)
    a = oracle.sw_align(q, s, B62, 1, 6)
    assert a["ops"] == "M" * 10 + "I" * 5 + "M" * 9
    assert (a["q_begin"], a["q_end"], a["s_begin"], a["s_end"]) == (0, 24, 0, 19)
    assert a["score"] == int(sum(int(B62[x][x]) for x in s)) - (6 + 4 * 1)
    # and the mirrored case gives a 'D' run
    b = oracle.sw_align(s, q, B62, 1, 6)
    assert b["ops"] == "M" * 10 + "D" * 5 + "M" * 9 and b["score"] == a["score"]


def test_empty_and_zero():
    M = np.zeros((32, 32), dtype=np.int8)
    M[:24, :24] = -1
    a = oracle.sw_align(np.array([1, 2, 3], np.uint8), np.array([4, 5], np.uint8), M, 1, 2)
    assert a == {"score": 0, "q_begin": 0, "q_end": 0, "s_begin": 0, "s_end": 0, "ops": ""}
    a = oracle.sw_align(np.array([1], np.uint8), np.array([], np.uint8), B62, 1, 2)
    assert a["score"] == 0 and a["ops"] == ""
