"""Test helper: writes the persistent index format of sw_db_save (include/swsearch.h, DESIGN.md §9 f2)
from the layout's definition, independently of the library, so the loader's validation can be tested
on crafted and corrupted files (CPU) and a hand-written file can be searched (GPU).

Layout (little endian): a 112-byte header, then at 64-byte aligned offsets the group table
(int64 base, int32 ncols, int32 count per group of 64 length-sorted subjects), the permutation
(int32, sorted position -> input index), the sorted lengths (int32), the global ids (int64, input
order, optional) and the packed words (per group: ceil(ncols/6) rows of 32 uint2; subject l of the
group sits in word row w at lane l>>1, .x for even l, .y for odd; 6 five-bit codes per uint32,
padding code 24)."""
import struct

import numpy as np

GROUP, PER_WORD, DUMMY = 64, 6, 24
HEADER = struct.Struct("<8sII5q2i6q")


def _align64(x):
    return (x + 63) // 64 * 64


def build(residues, offsets, lengths, gids=None):
    """Returns dict of the sections for subjects given in input order."""
    lengths = np.asarray(lengths, dtype=np.int32)
    n = lengths.size
    perm = np.argsort(lengths, kind="stable").astype(np.int32)
    len_sorted = lengths[perm]
    n_groups = (n + GROUP - 1) // GROUP
    groups, words, base = [], [], 0
    for g in range(n_groups):
        members = perm[g * GROUP:(g + 1) * GROUP]
        ncols = int(len_sorted[min((g + 1) * GROUP, n) - 1])
        nw = (ncols + PER_WORD - 1) // PER_WORD
        block = np.zeros((nw, 32, 2), dtype=np.uint32)
        for l in range(GROUP):
            codes = np.full(nw * PER_WORD, DUMMY, dtype=np.uint32)
            if l < members.size:
                i = members[l]
                codes[:lengths[i]] = residues[offsets[i]:offsets[i] + lengths[i]]
            packed = (codes.reshape(nw, PER_WORD) << (5 * np.arange(PER_WORD, dtype=np.uint32))).sum(axis=1)
            block[:, l >> 1, l & 1] = packed
        groups.append((base, ncols, members.size))
        words.append(block.reshape(-1))
        base += nw * 32
    return {
        "groups": groups, "perm": perm, "len_sorted": len_sorted,
        "gids": None if gids is None else np.asarray(gids, dtype=np.int64),
        "words": np.concatenate(words) if words else np.zeros(0, dtype=np.uint32),
        "n_residues": int(len(residues)),
    }


def write(path, sec, header_overrides=None):
    n = sec["len_sorted"].size
    n_groups = len(sec["groups"])
    n_words = sec["words"].size // 2
    has_gid = sec["gids"] is not None
    off_groups = _align64(HEADER.size)
    off_perm = _align64(off_groups + 16 * n_groups)
    off_len = _align64(off_perm + 4 * n)
    off_gid = _align64(off_len + 4 * n)
    off_words = _align64(off_gid + (8 * n if has_gid else 0))
    file_bytes = off_words + 8 * n_words
    h = dict(magic=b"SWB200DB", version=1, header_bytes=HEADER.size, n_seqs=n, n_residues=sec["n_residues"],
             sum_len=int(sec["len_sorted"].astype(np.int64).sum()), n_groups=n_groups, n_words=n_words,
             max_len=int(sec["len_sorted"][-1]) if n else 0, has_gid=int(has_gid), off_groups=off_groups,
             off_perm=off_perm, off_len=off_len, off_gid=off_gid, off_words=off_words, file_bytes=file_bytes)
    h.update(header_overrides or {})
    buf = bytearray(file_bytes)
    buf[:HEADER.size] = HEADER.pack(*h.values())
    gt = b"".join(struct.pack("<qii", *g) for g in sec["groups"])
    buf[off_groups:off_groups + len(gt)] = gt
    buf[off_perm:off_perm + 4 * n] = sec["perm"].astype("<i4").tobytes()
    buf[off_len:off_len + 4 * n] = sec["len_sorted"].astype("<i4").tobytes()
    if has_gid:
        buf[off_gid:off_gid + 8 * n] = sec["gids"].astype("<i8").tobytes()
    buf[off_words:] = sec["words"].astype("<u4").tobytes()
    with open(path, "wb") as f:
        f.write(bytes(buf))
