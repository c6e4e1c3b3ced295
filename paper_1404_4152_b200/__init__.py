"""paper_1404_4152_b200 — B200-native Smith-Waterman protein database search.

Thin ctypes binding over the C ABI in include/swsearch.h (libswsearch.so,
built in-tree for sm_100a).  Argument marshalling only: every step of the
search runs in the library's CUDA kernels.  There is no CPU fallback: if the
shared library is missing, importing this package raises.

    db = Database(residues, offsets, lengths)            # sw_db_create
    res = db.search(query, matrix, alpha=2, beta=12, k=10)   # sw_search
    res.scores, res.topk_ids, res.topk_scores, res.stats
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libswsearch.so")
# Same source built with -DSW_ABLATION: the f4 ablation kernels and the
# tile/CTA-size instances selected by sw_tuning (measurement only).
ABLATION_LIB_PATH = os.path.join(_HERE, "libswsearch_ablation.so")

SW_OK, SW_EINVAL, SW_ENOMEM, SW_ECUDA, SW_ERANGE, SW_EINTERNAL = 0, -1, -2, -3, -4, -5


class SwError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class sw_tuning(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("tile_rows", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("intra_cols", ctypes.c_int32), ("max_big", ctypes.c_int32), ("align_ws_kb", ctypes.c_int32),
                ("pipeline", ctypes.c_int32), ("pipe_chain", ctypes.c_int32),
                ("intra_isolate", ctypes.c_int32), ("generic_gaps", ctypes.c_int32),
                ("intra_chain", ctypes.c_int32), ("intra_split", ctypes.c_int32),
                ("launch_chain", ctypes.c_int32)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class sw_opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("first_stage", ctypes.c_int32),
                ("long_threshold", ctypes.c_int32), ("verbose", ctypes.c_int32),
                ("residency", ctypes.c_int32), ("chunk_mb", ctypes.c_int32),
                ("max_qlen", ctypes.c_int32), ("max_k", ctypes.c_int32),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", ctypes.c_void_p),
                ("tuning", sw_tuning), ("reserved", ctypes.c_int32 * 4)]

# variant names of sw_tuning.variant (f4 ablations)
VARIANTS = {"production": 0, "intersp": 1, "intraqp": 2, "static": 3}


class sw_stats(ctypes.Structure):
    _fields_ = [("cells", ctypes.c_int64), ("n_seqs", ctypes.c_int64), ("n_inter", ctypes.c_int64),
                ("n_intra", ctypes.c_int64), ("n_rerun16", ctypes.c_int64), ("n_rerun32", ctypes.c_int64),
                ("seconds", ctypes.c_double), ("gcups", ctypes.c_double),
                ("ms_profile", ctypes.c_float), ("ms_inter", ctypes.c_float),
                ("ms_rerun", ctypes.c_float), ("ms_finalize", ctypes.c_float),
                ("first_stage", ctypes.c_int32), ("reserved", ctypes.c_int32 * 7)]

    def as_dict(self) -> dict:
        return {f: (getattr(self, f) if f != "reserved" else None) for f, _ in self._fields_ if f != "reserved"}


class sw_db_info(ctypes.Structure):
    _fields_ = [("n_seqs", ctypes.c_int64), ("n_residues", ctypes.c_int64), ("n_inter", ctypes.c_int64),
                ("n_intra", ctypes.c_int64), ("n_groups", ctypes.c_int64), ("packed_bytes", ctypes.c_int64),
                ("scratch_bytes", ctypes.c_int64), ("launches", ctypes.c_int64), ("n_searches", ctypes.c_int64),
                ("n_device_allocs", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("max_len", ctypes.c_int32), ("device", ctypes.c_int32),
                ("long_threshold", ctypes.c_int32), ("residency", ctypes.c_int32), ("n_chunks", ctypes.c_int32),
                ("max_qlen", ctypes.c_int32), ("max_k", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1)]


class sw_alignment(ctypes.Structure):
    _fields_ = [("subject", ctypes.c_int64), ("score", ctypes.c_int32), ("q_begin", ctypes.c_int32),
                ("q_end", ctypes.c_int32), ("s_begin", ctypes.c_int32), ("s_end", ctypes.c_int32),
                ("n_ops", ctypes.c_int32), ("reserved", ctypes.c_int32), ("ops_offset", ctypes.c_int64)]


# Every symbol include/swsearch.h declares (tests check the .so exports all of them).
EXPORTS = ("sw_opts_default", "sw_db_create", "sw_search", "sw_search_async", "sw_search_batch", "sw_merge_topk",
           "sw_db_get_info", "sw_db_stage_times", "sw_db_reserve", "sw_align", "sw_encode", "sw_db_save",
           "sw_db_load", "sw_db_destroy", "sw_strerror", "sw_last_error")

_libs = {}


def lib(ablation: bool = False) -> ctypes.CDLL:
    """Load libswsearch.so (or the ablation build); raises (no fallback) when
    it has not been built."""
    path = ABLATION_LIB_PATH if ablation else LIB_PATH
    if path not in _libs:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(path)
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.sw_opts_default.argtypes = [ctypes.POINTER(sw_opts)]
        L.sw_opts_default.restype = None
        L.sw_db_create.argtypes = [P, i64, P, P, i64, P, ctypes.POINTER(sw_opts), ctypes.POINTER(P)]
        L.sw_db_create.restype = ctypes.c_int
        L.sw_search.argtypes = [P, P, i32, P, i32, i32, i32, P, P, P, ctypes.POINTER(sw_stats)]
        L.sw_search.restype = ctypes.c_int
        L.sw_search_async.argtypes = [P, P, i32, P, i32, i32, i32, P, P, P, P]
        L.sw_search_async.restype = ctypes.c_int
        L.sw_search_batch.argtypes = [P, P, P, P, i32, P, i32, i32, i32, P, P, P, ctypes.POINTER(sw_stats)]
        L.sw_search_batch.restype = ctypes.c_int
        L.sw_align.argtypes = [P, P, i32, P, i32, i32, P, i32, ctypes.POINTER(sw_alignment), P, i64]
        L.sw_align.restype = ctypes.c_int
        L.sw_encode.argtypes = [ctypes.c_char_p, i64, P]
        L.sw_encode.restype = ctypes.c_int
        L.sw_merge_topk.argtypes = [P, P, i32, i32, i32, P, P]
        L.sw_merge_topk.restype = ctypes.c_int
        L.sw_db_get_info.argtypes = [P, ctypes.POINTER(sw_db_info)]
        L.sw_db_get_info.restype = ctypes.c_int
        L.sw_db_stage_times.argtypes = [P, i32, ctypes.POINTER(ctypes.c_float)]
        L.sw_db_stage_times.restype = ctypes.c_int
        L.sw_db_reserve.argtypes = [P, i32, i32]
        L.sw_db_reserve.restype = ctypes.c_int
        L.sw_db_save.argtypes = [P, ctypes.c_char_p]
        L.sw_db_save.restype = ctypes.c_int
        L.sw_db_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(sw_opts), ctypes.POINTER(P)]
        L.sw_db_load.restype = ctypes.c_int
        L.sw_db_destroy.argtypes = [P]
        L.sw_db_destroy.restype = None
        L.sw_strerror.argtypes = [ctypes.c_int]
        L.sw_strerror.restype = ctypes.c_char_p
        L.sw_last_error.argtypes = []
        L.sw_last_error.restype = ctypes.c_char_p
        _libs[path] = L
    return _libs[path]


def _check(rc: int, L=None):
    if rc != SW_OK:
        L = L or lib()
        raise SwError(rc, f"{L.sw_strerror(rc).decode()}: {L.sw_last_error().decode()}")


class TorchAllocator:
    """sw_opts.alloc / free backed by torch's CUDA caching allocator (SURVEY.md
    §8(b)): the library's device buffers then come from torch's pool.  Counts
    the calls (tests check that searches allocate nothing)."""

    def __init__(self, device: int):
        import torch
        self.torch = torch
        self.device = device
        self.n_alloc = 0
        self.n_free = 0
        self.live = {}

        def _alloc(nbytes, ctx):
            try:
                ptr = torch.cuda.caching_allocator_alloc(int(nbytes), device=self.device)
            except Exception:
                return None
            self.n_alloc += 1
            self.live[int(ptr)] = int(nbytes)
            return int(ptr)

        def _free(ptr, ctx):
            if ptr:
                self.n_free += 1
                self.live.pop(int(ptr), None)
                torch.cuda.caching_allocator_delete(int(ptr))

        self.alloc_fn = ALLOC_FN(_alloc)     # kept alive with the Database
        self.free_fn = FREE_FN(_free)


def _make_opts(L, device, first_stage, long_threshold, residency, chunk_mb, max_qlen, max_k, allocator,
               tuning) -> sw_opts:
    o = sw_opts()
    L.sw_opts_default(ctypes.byref(o))
    o.device, o.first_stage, o.long_threshold = device, first_stage, long_threshold
    o.residency, o.chunk_mb = residency, chunk_mb
    if max_qlen:
        o.max_qlen = max_qlen
    if max_k:
        o.max_k = max_k
    if allocator is not None:
        o.alloc, o.free = allocator.alloc_fn, allocator.free_fn
    for key, val in (tuning or {}).items():
        if key == "variant" and isinstance(val, str):
            val = VARIANTS[val]
        setattr(o.tuning, key, int(val))
    return o


def _needs_ablation(tuning) -> bool:
    t = tuning or {}
    v = t.get("variant", 0)
    v = VARIANTS[v] if isinstance(v, str) else v
    return bool(v) or t.get("tile_rows", 0) not in (0, 48) or t.get("threads", 0) not in (0, 384) \
        or t.get("intra_cols", 0) == 2 or t.get("pipe_chain", 0) not in (0, 3)


def _ptr(a) -> int | None:
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


@dataclass
class SearchResult:
    scores: np.ndarray | None
    topk_ids: np.ndarray
    topk_scores: np.ndarray
    stats: dict


class Database:
    """sw_db_create / sw_db_destroy.  Arrays are copied (and packed) by the library."""

    def __init__(self, residues, offsets, lengths, global_ids=None, device: int = -1,
                 first_stage: int = 16, long_threshold: int = 0, residency: int = 0, chunk_mb: int = 0,
                 max_qlen: int = 0, max_k: int = 0, allocator=None, tuning: dict | None = None):
        """allocator: None (cudaMalloc), "torch" (torch's caching allocator) or a
        TorchAllocator-like object with alloc_fn / free_fn ctypes callbacks.
        tuning: sw_tuning fields (measurement switches; the non-production ones
        load the ablation build)."""
        L = lib(_needs_ablation(tuning))
        res = np.ascontiguousarray(residues, dtype=np.uint8)
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        lens = np.ascontiguousarray(lengths, dtype=np.int32)
        gids = None if global_ids is None else np.ascontiguousarray(global_ids, dtype=np.int64)
        if offs.shape != lens.shape:
            raise ValueError("offsets and lengths must have the same shape")
        if allocator == "torch":
            import torch
            allocator = TorchAllocator(device if device >= 0 else torch.cuda.current_device())
        o = _make_opts(L, device, first_stage, long_threshold, residency, chunk_mb, max_qlen, max_k, allocator,
                       tuning)
        h = ctypes.c_void_p()
        _check(L.sw_db_create(_ptr(res) if res.size else None, res.size, _ptr(offs) if offs.size else None,
                              _ptr(lens) if lens.size else None, lens.size,
                              None if gids is None else _ptr(gids), ctypes.byref(o), ctypes.byref(h)), L)
        self._L = L
        self._h = h
        self.allocator = allocator          # the callbacks must outlive the handle
        self.n_seqs = int(lens.size)
        self._lengths = lens.copy()        # sizes the ops buffer of align()

    def _call(self, name, *args):
        _check(getattr(self._L, name)(*args), self._L)

    def reserve(self, max_qlen: int, max_k: int):
        """sw_db_reserve: size the per-search buffers (sw_search_async never allocates)."""
        self._call("sw_db_reserve", self._h, max_qlen, max_k)

    @classmethod
    def from_synth(cls, db, **kw) -> "Database":
        return cls(db.residues, db.offsets, db.lengths, **kw)

    @classmethod
    def load(cls, path: str, device: int = -1, first_stage: int = 16, long_threshold: int = 0,
             residency: int = 0, chunk_mb: int = 0, max_qlen: int = 0, max_k: int = 0, allocator=None,
             tuning: dict | None = None) -> "Database":
        """sw_db_load: map a file written by save() and upload it (no re-sort / re-pack)."""
        L = lib(_needs_ablation(tuning))
        if allocator == "torch":
            import torch
            allocator = TorchAllocator(device if device >= 0 else torch.cuda.current_device())
        o = _make_opts(L, device, first_stage, long_threshold, residency, chunk_mb, max_qlen, max_k, allocator,
                       tuning)
        h = ctypes.c_void_p()
        _check(L.sw_db_load(os.fsencode(path), ctypes.byref(o), ctypes.byref(h)), L)
        self = cls.__new__(cls)
        self._L = L
        self._h = h
        self.allocator = allocator
        self._lengths = None
        self.n_seqs = self.info()["n_seqs"]
        return self

    def save(self, path: str):
        """sw_db_save: write the packed, length-sorted layout to `path`."""
        self._call("sw_db_save", self._h, os.fsencode(path))

    def info(self) -> dict:
        i = sw_db_info()
        self._call("sw_db_get_info", self._h, ctypes.byref(i))
        return {f: getattr(i, f) for f, _ in i._fields_ if f != "reserved"}

    def stage_times(self, back: int = 1) -> list:
        """[profile, first pass, rerun, ranking] device ms of the search `back` calls ago."""
        ms = (ctypes.c_float * 4)()
        self._call("sw_db_stage_times", self._h, back, ms)
        return list(ms)

    def search(self, query, matrix, alpha: int, beta: int, k: int = 10, scores: bool | np.ndarray = True,
               topk_ids=None, topk_scores=None) -> SearchResult:
        """Blocking search with host buffers (sw_search).  `scores` may be a
        preallocated (e.g. pinned) int32 host array, True (allocate) or False."""
        q = np.ascontiguousarray(query, dtype=np.uint8)
        M = np.ascontiguousarray(matrix, dtype=np.int8)
        if M.shape != (32, 32):
            raise ValueError("matrix must be 32x32 int8 (see swdata.matrix32)")
        if scores is True:
            sc = np.empty(self.n_seqs, dtype=np.int32)
        elif scores is False or scores is None:
            sc = None
        else:
            sc = scores
        ti = np.empty(k, dtype=np.int64) if topk_ids is None else topk_ids
        ts = np.empty(k, dtype=np.int32) if topk_scores is None else topk_scores
        st = sw_stats()
        self._call("sw_search", self._h, _ptr(q), q.size, _ptr(M), alpha, beta, k, _ptr(sc), _ptr(ti),
                               _ptr(ts), ctypes.byref(st))
        return SearchResult(sc, ti, ts, st.as_dict())

    def search_batch(self, queries, matrix, alpha: int, beta: int, k: int = 10, scores: bool = True):
        """sw_search_batch: a list of query code arrays -> SearchResult with
        scores (n_queries, n_seqs), topk_ids/topk_scores (n_queries, k)."""
        qs = [np.ascontiguousarray(q, dtype=np.uint8) for q in queries]
        cat = np.concatenate(qs) if qs else np.zeros(0, np.uint8)
        lens = np.array([q.size for q in qs], dtype=np.int32)
        offs = np.zeros(len(qs), dtype=np.int64)
        if len(qs) > 1:
            np.cumsum(lens[:-1], out=offs[1:])
        M = np.ascontiguousarray(matrix, dtype=np.int8)
        sc = np.empty((len(qs), self.n_seqs), dtype=np.int32) if scores else None
        ti = np.empty((len(qs), k), dtype=np.int64)
        ts = np.empty((len(qs), k), dtype=np.int32)
        st = sw_stats()
        self._call("sw_search_batch", self._h, _ptr(cat) if cat.size else None, _ptr(offs), _ptr(lens), len(qs),
                                     _ptr(M), alpha, beta, k, _ptr(sc), _ptr(ti), _ptr(ts), ctypes.byref(st))
        d = st.as_dict()
        d["pairs"] = st.reserved[0]
        return SearchResult(sc, ti, ts, d)

    def align(self, query, matrix, alpha: int, beta: int, subjects) -> list:
        """sw_align: one optimal local alignment per subject (input indices).
        Returns dicts {subject, score, q_begin, q_end, s_begin, s_end, ops}
        (0-based half-open ranges; ops over 'M', 'I' = query residue vs gap,
        'D' = subject residue vs gap)."""
        q = np.ascontiguousarray(query, dtype=np.uint8)
        M = np.ascontiguousarray(matrix, dtype=np.int8)
        idx = np.ascontiguousarray(np.atleast_1d(subjects), dtype=np.int64)
        n = idx.size
        if n == 0:
            return []
        ok = getattr(self, "_lengths", None) is not None and idx.min() >= 0 and idx.max() < self.n_seqs
        lens = self._lengths[idx] if ok else None      # out-of-range ids: the library reports them
        cap = int(n * q.size + (lens.sum() if lens is not None else n * (self.info()["max_len"])))
        out = (sw_alignment * n)()
        buf = ctypes.create_string_buffer(max(cap, 1))
        self._call("sw_align", self._h, _ptr(q), q.size, _ptr(M), alpha, beta, _ptr(idx), n, out, buf, cap)
        raw = buf.raw
        res = []
        for a in out:
            res.append({"subject": a.subject, "score": a.score, "q_begin": a.q_begin, "q_end": a.q_end,
                        "s_begin": a.s_begin, "s_end": a.s_end,
                        "ops": raw[a.ops_offset:a.ops_offset + a.n_ops].decode()})
        return res

    def search_async(self, query, matrix, alpha: int, beta: int, k: int, d_scores=None, d_topk_ids=None,
                     d_topk_scores=None, stream=None):
        """Enqueue on a CUDA stream (torch.cuda.Stream or raw handle) with device
        outputs (torch tensors: int32[n], int64[k], int32[k]); no host sync."""
        q = np.ascontiguousarray(query, dtype=np.uint8)
        M = np.ascontiguousarray(matrix, dtype=np.int8)
        if stream is None:
            h = None
        elif hasattr(stream, "cuda_stream"):
            h = stream.cuda_stream
        else:
            h = int(stream)
        self._call("sw_search_async", self._h, _ptr(q), q.size, _ptr(M), alpha, beta, k, _ptr(d_scores),
                                     _ptr(d_topk_ids), _ptr(d_topk_scores), h)

    def close(self):
        if getattr(self, "_h", None):
            self._L.sw_db_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def encode(text) -> np.ndarray:
    """sw_encode: protein letters (str or bytes) -> residue codes uint8 (J, O, U -> X)."""
    raw = text.encode("ascii") if isinstance(text, str) else bytes(text)
    out = np.empty(len(raw), dtype=np.uint8)
    _check(lib().sw_encode(raw, len(raw), out.ctypes.data if out.size else None))
    return out


def merge_topk(ids: np.ndarray, scores: np.ndarray, k_out: int):
    """sw_merge_topk over a (n_lists, k_in) stack of per-device top-k lists."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    scores = np.ascontiguousarray(scores, dtype=np.int32)
    n_lists, k_in = ids.shape if ids.ndim == 2 else (1, ids.size)
    oi = np.empty(k_out, dtype=np.int64)
    os_ = np.empty(k_out, dtype=np.int32)
    _check(lib().sw_merge_topk(_ptr(ids), _ptr(scores), n_lists, k_in, k_out, _ptr(oi), _ptr(os_)))
    return oi, os_
