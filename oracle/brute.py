"""Brute-force enumeration of all local alignments — TEST INFRASTRUCTURE ONLY.

Independent of Eq. 1's recurrence: the optimal local score is the maximum,
over every pair of substrings and every column string over {M, D, I}, of
  sum of fsbt over M columns  -  sum over maximal D-runs and I-runs of
  (beta + (len - 1) * alpha),
with the empty alignment scoring 0 (alpha = gap extension,
beta = gap open + extension; a gap of k residues costs beta + (k-1) alpha).
A D-run directly followed by an I-run is two runs, each charged separately.
Exponential: use for |Q|, |S| <= 6 only.
"""


def brute_force(q, s, M, alpha: int, beta: int) -> int:
    q = [int(x) for x in q]
    s = [int(x) for x in s]
    m, n = len(q), len(s)
    best = 0

    # DFS over alignments starting at (i0, j0); state = (i, j, last column type, score)
    def walk(i, j, last, score):
        nonlocal best
        if score > best:
            best = score
        if i < m and j < n:                                   # M column
            walk(i + 1, j + 1, "M", score + int(M[q[i]][s[j]]))
        if i < m:                                             # D: query residue vs gap
            walk(i + 1, j, "D", score - (alpha if last == "D" else beta))
        if j < n:                                             # I: subject residue vs gap
            walk(i, j + 1, "I", score - (alpha if last == "I" else beta))

    for i0 in range(m):
        for j0 in range(n):
            walk(i0, j0, "", 0)
    return best


def optimal_alignments(q, s, M, alpha: int, beta: int):
    """(best, set of (q_begin, q_end, s_begin, s_end, ops)) over every non-empty
    local alignment, ops in SAM form with the query as the read: 'M' query
    residue vs subject residue, 'I' query residue vs gap, 'D' subject residue
    vs gap.  Same scoring as brute_force; exponential, |Q|, |S| <= 5."""
    q = [int(x) for x in q]
    s = [int(x) for x in s]
    m, n = len(q), len(s)
    best, found = 0, set()

    def walk(i0, j0, i, j, last, score, ops):
        nonlocal best, found
        if ops:
            if score > best:
                best, found = score, set()
            if score == best:
                found.add((i0, i, j0, j, "".join(ops)))
        if i < m and j < n:
            ops.append("M")
            walk(i0, j0, i + 1, j + 1, "M", score + int(M[q[i]][s[j]]), ops)
            ops.pop()
        if i < m:
            ops.append("I")
            walk(i0, j0, i + 1, j, "I", score - (alpha if last == "I" else beta), ops)
            ops.pop()
        if j < n:
            ops.append("D")
            walk(i0, j0, i, j + 1, "D", score - (alpha if last == "D" else beta), ops)
            ops.pop()

    for i0 in range(m + 1):
        for j0 in range(n + 1):
            walk(i0, j0, i0, j0, "", 0, [])
    return best, found
