"""Counter-based synthetic workloads (inputs only; no method arithmetic).

Every random draw is `splitmix64(key + (index + 1) * GOLDEN)` with a key
derived from (seed, config, stream label, ...), so any subset of sequences can
be generated independently of order, thread count or sharding (SURVEY.md
§8(d) "RNG").  Recipe (DESIGN.md §"Input recipe"):

* residues: iid over the 20 standard amino acids with the Robinson & Robinson
  background frequencies, quantised to a 2^16-entry lookup table;
* lengths: lognormal, sigma = 0.65, mu = ln 350 - sigma^2/2 (mean 350),
  rounded and clipped to [10, 5000] (BASELINE.json configs; TrEMBL mean 318,
  PAPER.md:168);
* C3 long tail: each sequence independently with p = 0.001 gets a uniform
  integer length in [5000, 35000] (TrEMBL longest 36,805);
* C4 planting: each sequence independently with p = 0.05 is a near-copy of the
  query: per query residue keep 0.80 / substitute 0.18 / delete 0.01 /
  insert 1+Geometric(0.5) background residues before it 0.01;
* queries: iid background residues of the stated length.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .alphabet import ALPHABET, DUMMY  # noqa: F401
from .matrices import blosum50, blosum62, matrix32

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1

# Robinson & Robinson (1991) background composition, alphabet order A..V.
BACKGROUND = {
    "A": 0.078, "R": 0.051, "N": 0.045, "D": 0.054, "C": 0.019, "Q": 0.043, "E": 0.063,
    "G": 0.074, "H": 0.022, "I": 0.051, "L": 0.090, "K": 0.057, "M": 0.022, "F": 0.039,
    "P": 0.052, "S": 0.071, "T": 0.058, "W": 0.013, "Y": 0.032, "V": 0.064,
}


def _quantised_lut() -> np.ndarray:
    p = np.array([BACKGROUND[c] for c in ALPHABET[:20]], dtype=np.float64)
    p = p / p.sum()
    raw = p * 65536.0
    cnt = np.floor(raw).astype(np.int64)
    rem = 65536 - int(cnt.sum())
    order = np.argsort(-(raw - cnt), kind="stable")       # largest remainder
    cnt[order[:rem]] += 1
    return np.repeat(np.arange(20, dtype=np.uint8), cnt)


RESIDUE_LUT = _quantised_lut()      # 65536 entries, codes 0..19


def _mix_int(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = z ^ (z >> np.uint64(30))
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def stream_key(seed: int, *labels) -> int:
    """Fold (seed, labels...) into one 64-bit stream key.  Labels: ints or str."""
    k = _mix_int(seed * GOLDEN + 0x1234567)
    for lab in labels:
        if isinstance(lab, str):
            v = 0
            for ch in lab.encode():
                v = (v * 131 + ch) & M64
            lab = v
        k = _mix_int(k ^ _mix_int((int(lab) + 1) * GOLDEN))
    return k


def uniform_u64(key: int, idx) -> np.ndarray:
    """The idx-th draw of stream `key` (idx: int array), as uint64."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (idx + np.uint64(1)) * np.uint64(GOLDEN)
    return splitmix64(z)


def _unit(u: np.ndarray) -> np.ndarray:
    """uint64 -> float64 in (0, 1)."""
    return ((u >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


_CLIB = None


def _clib():
    """ctypes handle on swdata/_libswgen.so (built by __graft_entry__.build());
    None -> the numpy reference implementation is used (bit-identical)."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(__file__), "_libswgen.so")
        if not os.path.exists(path):
            _CLIB = False
            return None
        lib = ctypes.CDLL(path)
        lib.swgen_residues.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.swgen_residues_runs.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.swgen_mutate.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        lib.swgen_mutate.restype = ctypes.c_int64
        _CLIB = lib
    return _CLIB or None


def _nthreads() -> int:
    import os
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return os.cpu_count() or 1


def gen_residues(key: int, start: int, n: int, use_c: bool = True) -> np.ndarray:
    """Residues [start, start+n) of background stream `key` (uint8 codes 0..19)."""
    lib = _clib() if use_c else None
    if lib is not None:
        out = np.empty(n, dtype=np.uint8)
        if n:
            lib.swgen_residues(key, start, n, RESIDUE_LUT.ctypes.data, out.ctypes.data, _nthreads())
        return out
    out = np.empty(n, dtype=np.uint8)
    chunk = 1 << 24
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        u = uniform_u64(key, np.arange(start + a, start + b, dtype=np.uint64))
        out[a:b] = RESIDUE_LUT[(u >> np.uint64(48)).astype(np.int64)]
    return out


def lognormal_lengths(key: int, ids: np.ndarray, mean: float = 350.0, sigma: float = 0.65,
                      lo: int = 10, hi: int = 5000) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.uint64)
    u1 = _unit(uniform_u64(key, ids * np.uint64(2)))
    u2 = _unit(uniform_u64(key, ids * np.uint64(2) + np.uint64(1)))
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    mu = math.log(mean) - 0.5 * sigma * sigma
    ln = np.floor(np.exp(mu + sigma * z) + 0.5)
    return np.clip(ln, lo, hi).astype(np.int32)


@dataclass
class Config:
    name: str
    n_seqs: int
    qlens: tuple
    matrix: str = "blosum62"
    alpha: int = 2
    beta: int = 12
    k: int = 10
    long_p: float = 0.0            # C3 long tail
    long_range: tuple = (5000, 35000)
    plant_p: float = 0.0           # C4 planted near-copies
    exact_copies: int = 0          # S16
    near_copies: int = 0           # S16
    note: str = ""

    def matrix32(self) -> np.ndarray:
        return matrix32(blosum62() if self.matrix == "blosum62" else blosum50())


CONFIGS = {
    "C1": Config("C1", 10_000, (144,), note="BASELINE.json configs[0]"),
    "C2": Config("C2", 1_000_000, (464,), note="BASELINE.json configs[1]; all scores + top-10"),
    "C3": Config("C3", 20_000_000, (144, 375, 729, 1500, 2005, 5478), long_p=0.001,
                 note="BASELINE.json configs[2]; query-length sweep with 0.1% 5k-35k tail"),
    "C4": Config("C4", 2_000_000, (2000,), plant_p=0.05,
                 note="BASELINE.json configs[3]; 5% planted near-copies (80% identity)"),
    "C5": Config("C5", 50_000_000, (1000,), matrix="blosum50", k=100,
                 note="BASELINE.json configs[4]; scaling run, BLOSUM50, top-100"),
    "S16": Config("S16", 10_400, (8000,), exact_copies=200, near_copies=200,
                  note="added stress case: int16 -> int32 escalation (SURVEY.md §8(d))"),
}


def make_query(cfg: Config | str, m: int | None = None, seed: int = 0) -> np.ndarray:
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    m = cfg.qlens[0] if m is None else m
    return gen_residues(stream_key(seed, cfg.name, "query", m), 0, m)


def _mutate(query: np.ndarray, key: int, use_c: bool = True) -> np.ndarray:
    """C4 planting model: one near-copy of `query` (80% identity, random indels)."""
    lib = _clib() if use_c else None
    if lib is not None:
        q = np.ascontiguousarray(query, dtype=np.uint8)
        cap = 2 * q.size + 64
        out = np.empty(cap, dtype=np.uint8)
        n = lib.swgen_mutate(q.ctypes.data, q.size, key, RESIDUE_LUT.ctypes.data, out.ctypes.data, cap)
        if n > cap:
            out = np.empty(n, dtype=np.uint8)
            lib.swgen_mutate(q.ctypes.data, q.size, key, RESIDUE_LUT.ctypes.data, out.ctypes.data, n)
        return out[:n].copy()
    m = query.size
    pos = np.arange(m, dtype=np.uint64)
    act = _unit(uniform_u64(key, pos * np.uint64(8)))
    sub = query.copy()
    # substitution: background draw, redrawn until different (up to 4 draws, then +1 mod 20)
    todo = np.ones(m, dtype=bool)
    for t in range(4):
        d = RESIDUE_LUT[(uniform_u64(key, pos * np.uint64(8) + np.uint64(1 + t)) >> np.uint64(48)).astype(np.int64)]
        take = todo & (d != query)
        sub[take] = d[take]
        todo &= ~take
    sub[todo] = (query[todo] + 1) % 20
    geo = uniform_u64(key, pos * np.uint64(8) + np.uint64(5))
    # 1 + Geometric(0.5): 1 + number of trailing one-bits (capped at 16)
    nins = np.ones(m, dtype=np.int64)
    g = geo.copy()
    for _ in range(15):
        one = (g & np.uint64(1)).astype(bool)
        nins += one
        g = np.where(one, g >> np.uint64(1), np.uint64(0))
    keep = act < 0.80
    subst = (act >= 0.80) & (act < 0.98)
    delete = (act >= 0.98) & (act < 0.99)
    insert = act >= 0.99
    out_res = np.where(subst, sub, query)
    emit = (~delete).astype(np.int64)
    ins_cnt = np.where(insert, nins, 0)
    total = int((emit + ins_cnt).sum())
    out = np.empty(total, dtype=np.uint8)
    ins_key = key ^ 0x5DEECE66D
    w = 0
    # emission order per position: inserted residues, then the (kept/substituted) residue
    starts = np.concatenate([[0], np.cumsum(emit + ins_cnt)[:-1]])
    ipos = np.nonzero(ins_cnt)[0]
    for p in ipos:                       # rare (1%): small python loop is fine
        c = int(ins_cnt[p])
        s = int(starts[p])
        out[s:s + c] = gen_residues(ins_key, int(p) * 32, c, use_c=False)
    kpos = np.nonzero(emit)[0]
    out[starts[kpos] + ins_cnt[kpos]] = out_res[kpos]
    del keep, w
    return out


@dataclass
class SynthDB:
    """A (sub)database in the ABI layout: concatenated codes + offsets + lengths."""
    residues: np.ndarray
    offsets: np.ndarray
    lengths: np.ndarray
    global_ids: np.ndarray
    config: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_seqs(self) -> int:
        return int(self.lengths.size)

    def seq(self, i: int) -> np.ndarray:
        o = int(self.offsets[i])
        return self.residues[o:o + int(self.lengths[i])]


def db_lengths(cfg: Config | str, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """(lengths int32[N], kind int8[N]) for the whole config: kind 0 background,
    1 long-tail, 2 planted near-copy, 3 exact copy."""
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    n = cfg.n_seqs
    ids = np.arange(n, dtype=np.uint64)
    lengths = lognormal_lengths(stream_key(seed, cfg.name, "len"), ids)
    kind = np.zeros(n, dtype=np.int8)
    if cfg.long_p > 0:
        u = _unit(uniform_u64(stream_key(seed, cfg.name, "longsel"), ids))
        sel = u < cfg.long_p
        lo, hi = cfg.long_range
        ul = uniform_u64(stream_key(seed, cfg.name, "longlen"), ids[sel])
        lengths[sel] = (lo + (ul % np.uint64(hi - lo + 1))).astype(np.int32)
        kind[sel] = 1
    if cfg.plant_p > 0 or cfg.exact_copies or cfg.near_copies:
        q = make_query(cfg, seed=seed)
        if cfg.plant_p > 0:
            u = _unit(uniform_u64(stream_key(seed, cfg.name, "plantsel"), ids))
            sel = np.nonzero(u < cfg.plant_p)[0]
        else:
            period = n // (cfg.exact_copies + cfg.near_copies)
            sel_exact = np.arange(cfg.exact_copies) * period + 7
            sel_near = np.arange(cfg.near_copies) * period + 7 + cfg.exact_copies * period
            kind[sel_exact] = 3
            lengths[sel_exact] = q.size
            sel = sel_near
        kind[sel] = 2
        for i in sel:
            lengths[i] = _mutate(q, stream_key(seed, cfg.name, "plant", int(i))).size
    return lengths, kind


def make_db(cfg: Config | str, seed: int = 0, ids=None, lengths_kind=None) -> SynthDB:
    """Generate the database of `cfg` (or the subset `ids`, in that order)."""
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    lengths_all, kind = db_lengths(cfg, seed) if lengths_kind is None else lengths_kind
    goff = np.zeros(lengths_all.size + 1, dtype=np.int64)
    np.cumsum(lengths_all, out=goff[1:])
    ids = np.arange(cfg.n_seqs, dtype=np.int64) if ids is None else np.asarray(ids, dtype=np.int64)
    lens = lengths_all[ids]
    offs = np.zeros(ids.size, dtype=np.int64)
    if ids.size > 1:
        np.cumsum(lens[:-1], out=offs[1:])
    res = np.empty(int(lens.sum()), dtype=np.uint8)
    rkey = stream_key(seed, cfg.name, "res")
    # contiguous runs of ids -> one bulk draw each
    k = ids.size
    if k:
        brk = np.nonzero(np.diff(ids) != 1)[0] + 1
        first = np.concatenate([[0], brk]).astype(np.int64)          # first position of each run of ids
        last = np.concatenate([brk, [k]]).astype(np.int64)           # one past its last position
        g0 = goff[ids[first]]
        rl = goff[ids[last - 1] + 1] - g0
        lib = _clib()
        if lib is not None and first.size > 64:                       # a scattered shard: one C call
            g0 = np.ascontiguousarray(g0, dtype=np.int64)
            rl = np.ascontiguousarray(rl, dtype=np.int64)
            oo = np.ascontiguousarray(offs[first], dtype=np.int64)
            lib.swgen_residues_runs(rkey, g0.ctypes.data, rl.ctypes.data, oo.ctypes.data, first.size,
                                    RESIDUE_LUT.ctypes.data, res.ctypes.data, _nthreads())
        else:
            for a, s0, n in zip(first.tolist(), g0.tolist(), rl.tolist()):
                res[offs[a]:offs[a] + n] = gen_residues(rkey, s0, n)
    special = np.nonzero(kind[ids] >= 2)[0]
    if special.size:
        q = make_query(cfg, seed=seed)
        for j in special:
            gid = int(ids[j])
            s = q if kind[gid] == 3 else _mutate(q, stream_key(seed, cfg.name, "plant", gid))
            res[offs[j]:offs[j] + s.size] = s
    return SynthDB(res, offs, lens.astype(np.int32), ids, cfg.name,
                   {"n_total": cfg.n_seqs, "kinds": np.bincount(kind[ids], minlength=4).tolist()})


def random_db(seed: int, lengths, alphabet: int = 20, label: str = "adhoc") -> SynthDB:
    """Small ad-hoc database with given lengths (tests: edge cases, ragged tails)."""
    lengths = np.asarray(lengths, dtype=np.int32)
    offs = np.zeros(lengths.size, dtype=np.int64)
    if lengths.size > 1:
        np.cumsum(lengths[:-1], out=offs[1:])
    n = int(lengths.sum())
    u = uniform_u64(stream_key(seed, label, "res"), np.arange(n, dtype=np.uint64))
    if alphabet == 20:
        res = RESIDUE_LUT[(u >> np.uint64(48)).astype(np.int64)]
    else:
        res = (u % np.uint64(alphabet)).astype(np.uint8)
    return SynthDB(res.astype(np.uint8), offs, lengths, np.arange(lengths.size, dtype=np.int64), label)


def manifest_hash(db: SynthDB) -> str:
    import hashlib
    h = hashlib.sha256()
    h.update(db.lengths.astype("<i4").tobytes())
    h.update(db.residues.tobytes())
    return h.hexdigest()
