"""oracle/ — TEST INFRASTRUCTURE ONLY (never imported by the product path).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It shares no code with
paper_1404_4152_b200/ and neither imports the other; both read inputs from
swdata/ only.

* `sw_score`, `scores`: Eq. 1 as printed, scalar int32,
  linear space (sw_oracle.c), threaded over subjects for whole databases.
* `sw_full`: Gotoh full matrix with -inf boundaries (pins reading R2).
* `topk`: stage (iv) "sort all alignment scores in descending order"
   by a full sort, tie-break id ascending (reading R7).
* `sw_align`: one optimal local alignment by full-matrix traceback with the
  deterministic tie rules of DESIGN.md R17-R19 (f3).
* `brute.brute_force`: enumeration of every local alignment (tiny inputs);
  `brute.optimal_alignments`: the set of all optimal ones.

Pinned by tests/test_oracle.py (-m "not gpu"); no function is parity-unpinned.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sw_oracle.c")
_lib = None

# BASELINE.md's CPU-baseline plan: plain scalar C, -O3 -march=native, no
# intrinsics, flags recorded.  -march=native ties the binary to the host CPU,
# so the library is built per CPU model (the GPU box builds its own on first use).
CFLAGS = ["-O3", "-march=native", "-shared", "-fPIC", "-pthread"]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _so_path() -> str:
    import hashlib
    tag = hashlib.sha1((cpu_model() + " ".join(CFLAGS)).encode()).hexdigest()[:10]
    return os.path.join(_HERE, f"_liboracle_{tag}.so")


def build(force: bool = False) -> str:
    so = _so_path()
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
        tmp = f"{so}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, so)
    return so


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.oracle_sw_score.argtypes = [P, i32, P, i32, P, i32, i32]
        L.oracle_sw_score.restype = i32
        L.oracle_sw_full.argtypes = [P, i32, P, i32, P, i32, i32]
        L.oracle_sw_full.restype = i32
        L.oracle_scores.argtypes = [P, i32, P, P, P, i64, P, i32, i32, ctypes.c_int, P]
        L.oracle_scores.restype = ctypes.c_int
        L.oracle_topk.argtypes = [P, P, i64, i32, P, P]
        L.oracle_topk.restype = ctypes.c_int
        L.oracle_sw_align.argtypes = [P, i32, P, i32, P, i32, i32, P, ctypes.c_char_p]
        L.oracle_sw_align.restype = ctypes.c_int
        _lib = L
    return _lib


def _u8(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def _m32(M):
    M = np.asarray(M)
    if M.shape != (32, 32):
        out = np.zeros((32, 32), dtype=np.int8)
        out[:M.shape[0], :M.shape[1]] = M
        M = out
    return np.ascontiguousarray(M, dtype=np.int8)


def sw_score(q, s, M, alpha: int, beta: int) -> int:
    q, s, M = _u8(q), _u8(s), _m32(M)
    r = lib().oracle_sw_score(q.ctypes.data, q.size, s.ctypes.data, s.size, M.ctypes.data, alpha, beta)
    if r < 0:
        raise MemoryError("oracle_sw_score")
    return int(r)


def sw_full(q, s, M, alpha: int, beta: int) -> int:
    q, s, M = _u8(q), _u8(s), _m32(M)
    r = lib().oracle_sw_full(q.ctypes.data, q.size, s.ctypes.data, s.size, M.ctypes.data, alpha, beta)
    if r < 0:
        raise MemoryError("oracle_sw_full")
    return int(r)


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def scores(query, residues, offsets, lengths, M, alpha: int, beta: int, nthreads: int | None = None) -> np.ndarray:
    """Eq. 1 score of `query` against every subject (input order), int32."""
    q, res, M = _u8(query), _u8(residues), _m32(M)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    lens = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.empty(lens.size, dtype=np.int32)
    rc = lib().oracle_scores(q.ctypes.data, q.size, res.ctypes.data if res.size else None,
                             offs.ctypes.data, lens.ctypes.data, lens.size, M.ctypes.data,
                             alpha, beta, nthreads or default_threads(), out.ctypes.data)
    if rc != 0:
        raise MemoryError("oracle_scores")
    return out


def db_scores(query, db, M, alpha, beta, nthreads=None, sample=None):
    """`scores` over a swdata.SynthDB, optionally on the index subset `sample`."""
    if sample is None:
        return scores(query, db.residues, db.offsets, db.lengths, M, alpha, beta, nthreads)
    sample = np.asarray(sample, dtype=np.int64)
    return scores(query, db.residues, db.offsets[sample], db.lengths[sample], M, alpha, beta, nthreads)


def topk(scores_, k: int, ids=None):
    """(ids int64[k], scores int32[k]) by (score desc, id asc); (-1,-1) past n."""
    sc = np.ascontiguousarray(scores_, dtype=np.int32)
    idp = None
    if ids is not None:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        idp = ids.ctypes.data
    oi = np.empty(k, dtype=np.int64)
    os_ = np.empty(k, dtype=np.int32)
    if lib().oracle_topk(sc.ctypes.data, idp, sc.size, k, oi.ctypes.data, os_.ctypes.data) != 0:
        raise MemoryError("oracle_topk")
    return oi, os_


def sw_align(q, s, M, alpha: int, beta: int) -> dict:
    """One optimal local alignment (full-matrix traceback, sw_oracle.c).
    Returns {score, q_begin, q_end, s_begin, s_end, ops} (0-based, half-open;
    ops over 'M' / 'I' (query residue vs gap) / 'D' (subject residue vs gap))."""
    q, s, M = _u8(q), _u8(s), _m32(M)
    out = np.zeros(6, dtype=np.int32)
    buf = ctypes.create_string_buffer(q.size + s.size + 1)
    rc = lib().oracle_sw_align(q.ctypes.data, q.size, s.ctypes.data, s.size, M.ctypes.data, alpha, beta,
                               out.ctypes.data, buf)
    if rc != 0:
        raise MemoryError("oracle_sw_align")
    return {"score": int(out[0]), "q_begin": int(out[1]), "q_end": int(out[2]), "s_begin": int(out[3]),
            "s_end": int(out[4]), "ops": buf.raw[:int(out[5])].decode()}
