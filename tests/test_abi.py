"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/swsearch.h declares, rejects invalid inputs before touching
the device, and merges top-k lists (host function) as the oracle ranks."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "swsearch.h")).read()
    return set(re.findall(r"^\S[^\n(]*?\b(sw_\w+)\s*\(", txt, flags=re.M))


def test_header_and_binding_agree():
    assert _declared() == set(sw.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = sw.lib()
    for name in _declared():
        assert hasattr(L, name), name
    out = os.popen(f"nm -D --defined-only {sw.LIB_PATH}").read()
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported"


def test_strerror():
    L = sw.lib()
    assert L.sw_strerror(0) == b"ok"
    assert L.sw_strerror(-1) == b"invalid argument"
    assert L.sw_strerror(-4).startswith(b"score range")


def _create(res, offs, lens, gids=None, **kw):
    return sw.Database(res, offs, lens, global_ids=gids, **kw)


@pytest.mark.parametrize("case", ["bad_code", "overrun", "neg_len", "bad_gid", "dup_gid", "bad_stage",
                                  "bad_residency", "stream_int8", "bad_chunk", "bad_tuning", "neg_cap"])
def test_db_create_validation(case):
    res = np.array([0, 1, 2, 3, 4, 5], dtype=np.uint8)
    offs = np.array([0, 3], dtype=np.int64)
    lens = np.array([3, 3], dtype=np.int32)
    gids = None
    kw = {}
    if case == "bad_code":
        res[4] = 24
    elif case == "overrun":
        lens[1] = 4
    elif case == "neg_len":
        lens[0] = -1
    elif case == "bad_gid":
        gids = np.array([0, 1 << 33], dtype=np.int64)
    elif case == "dup_gid":            # ranking keys (score<<32 | ~id) must be unique
        gids = np.array([7, 7], dtype=np.int64)
    elif case == "bad_tuning":
        kw["tuning"] = {"tile_rows": 40}
    elif case == "neg_cap":
        kw["max_qlen"] = -3
    elif case == "bad_stage":
        kw["first_stage"] = 12
    elif case == "bad_residency":
        kw["residency"] = 2
    elif case == "stream_int8":
        kw["residency"], kw["first_stage"] = 1, 8
    elif case == "bad_chunk":
        kw["residency"], kw["chunk_mb"] = 1, -5
    with pytest.raises(sw.SwError) as ei:
        _create(res, offs, lens, gids, **kw)
    assert ei.value.code == sw.SW_EINVAL


def test_distinct_ids_checked_at_any_position():
    """The duplicate-id check covers large, sparse ids (bitmap up to the max id)."""
    n = 5000
    res = np.zeros(n, dtype=np.uint8)
    offs = np.arange(n, dtype=np.int64)
    lens = np.ones(n, dtype=np.int32)
    gids = np.arange(n, dtype=np.int64) * 800_000 + 17          # up to ~4e9 < 2^32 - 1
    gids[-1] = gids[1234]
    with pytest.raises(sw.SwError) as ei:
        _create(res, offs, lens, gids)
    assert ei.value.code == sw.SW_EINVAL and "repeats" in str(ei.value)


def _raw_create(L, **fields):
    """sw_db_create through the production library with raw sw_opts fields."""
    res = np.array([0, 1, 2], dtype=np.uint8)
    offs = np.array([0], dtype=np.int64)
    lens = np.array([3], dtype=np.int32)
    o = sw.sw_opts()
    L.sw_opts_default(ctypes.byref(o))
    for k, v in fields.items():
        if k.startswith("tuning."):
            setattr(o.tuning, k[7:], v)
        else:
            setattr(o, k, v)
    h = ctypes.c_void_p()
    rc = L.sw_db_create(res.ctypes.data, 3, offs.ctypes.data, lens.ctypes.data, 1, None, ctypes.byref(o),
                        ctypes.byref(h))
    return rc, h


@pytest.mark.parametrize("fields", [{"tuning.variant": 1}, {"tuning.tile_rows": 64}, {"tuning.threads": 512},
                                    {"tuning.intra_cols": 2}, {"tuning.pipe_chain": 12}, {"tuning.pipe_chain": 5},
                                    {"tuning.intra_isolate": 2}, {"tuning.launch_chain": 1}, {"tuning.intra_chain": 1}, {"tuning.intra_split": 2},
                                    {"tuning.generic_gaps": 2},
                                    {"reserved": (ctypes.c_int32 * 4)(0, 1, 0, 0)},
                                    {"alloc": sw.ALLOC_FN(lambda n, c: None)}])
def test_production_library_rejects_ablation_switches_and_bad_opts(fields):
    """Measurement switches are create-time options (never environment variables);
    the production build accepts only the shipped design; hooks come in pairs."""
    L = sw.lib()
    rc, h = _raw_create(L, **fields)
    assert rc == sw.SW_EINVAL and not h.value, L.sw_last_error()
    msg = L.sw_last_error().decode()
    if "tuning.variant" in fields:
        assert "ablation build" in msg


def test_opts_default_capacity():
    o = sw.sw_opts()
    sw.lib().sw_opts_default(ctypes.byref(o))
    assert (o.max_qlen, o.max_k, o.device, o.first_stage) == (8192, 4096, -1, 16)
    assert not o.alloc and not o.free and o.tuning.variant == 0


def test_no_environment_knobs_in_the_library():
    """No search path reads the environment (getenv per search)."""
    src = os.path.join(ROOT, "paper_1404_4152_b200", "csrc")
    for f in os.listdir(src):
        assert "getenv" not in open(os.path.join(src, f)).read(), f


def test_merge_topk_matches_oracle_ranking():
    rng = np.random.default_rng(0)
    lists_ids, lists_sc = [], []
    all_ids, all_sc = [], []
    for r in range(4):
        ids = np.arange(r, 400, 4)
        sc = rng.integers(0, 30, size=ids.size).astype(np.int32)
        all_ids.append(ids)
        all_sc.append(sc)
        ti, ts = oracle.topk(sc, 12, ids)
        lists_ids.append(ti)
        lists_sc.append(ts)
    mi, ms = sw.merge_topk(np.stack(lists_ids), np.stack(lists_sc), 12)
    ri, rs = oracle.topk(np.concatenate(all_sc), 12, np.concatenate(all_ids))
    assert np.array_equal(mi, ri) and np.array_equal(ms, rs)
    mi, ms = sw.merge_topk(np.array([[3, -1]]), np.array([[7, -1]]), 3)
    assert mi.tolist() == [3, -1, -1] and ms.tolist() == [7, -1, -1]


@pytest.mark.parametrize("content", [None, b"", b"not a database" * 20, b"SWB200DB" + b"\x01\x00\x00\x00" + b"\x00" * 200])
def test_db_load_rejects_bad_files(tmp_path, content):
    path = tmp_path / "db.swb"
    if content is not None:
        path.write_bytes(content)
    with pytest.raises(sw.SwError) as ei:
        sw.Database.load(str(path))
    assert ei.value.code == sw.SW_EINVAL


def test_encode_matches_alphabet_table():
    from swdata import encode as ref_encode
    rng = np.random.default_rng(5)
    letters = "ARNDCQEGHILKMFPSTWYVBZX*JOUarndcqeghilkmfpstwyvbzxjou"
    for n in (0, 1, 7, 1000):
        text = "".join(rng.choice(list(letters), size=n))
        assert np.array_equal(sw.encode(text), ref_encode(text)), text[:20]
    assert sw.encode("ARNDJ*").tolist() == [0, 1, 2, 3, 22, 23]
    with pytest.raises(sw.SwError) as e:
        sw.encode("AR1N")
    assert e.value.code == sw.SW_EINVAL and b"position 2" in sw.lib().sw_last_error()


def _crafted_index(seed=11, n=150):
    import index_file
    rng = np.random.default_rng(seed)
    lengths = rng.integers(0, 90, size=n).astype(np.int32)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    residues = rng.integers(0, 24, size=int(lengths.sum())).astype(np.uint8)
    gids = rng.permutation(10 * n)[:n].astype(np.int64)
    return index_file, index_file.build(residues, offsets, lengths, gids)


@pytest.mark.parametrize("corrupt", ["none", "perm_dup", "perm_range", "len_order", "group_count", "group_ncols",
                                     "code_25", "top_bits", "gid_range", "sum_len", "max_len"])
def test_db_load_validates_index_contents(tmp_path, corrupt):
    """A file written from the layout's definition passes the loader's host-side checks (on CPU the load then
    stops at the device: SW_ECUDA); each corruption of its contents is SW_EINVAL before any device work."""
    index_file, sec = _crafted_index()
    hdr = {}
    if corrupt == "perm_dup":
        sec["perm"][5] = sec["perm"][6]
    elif corrupt == "perm_range":
        sec["perm"][0] = sec["len_sorted"].size
    elif corrupt == "len_order":
        sec["len_sorted"][[3, 140]] = sec["len_sorted"][[140, 3]]
    elif corrupt == "group_count":
        b, c, k = sec["groups"][0]
        sec["groups"][0] = (b, c, k - 1)
    elif corrupt == "group_ncols":
        b, c, k = sec["groups"][1]
        sec["groups"][1] = (b, c - 1, k)
    elif corrupt == "code_25":
        sec["words"][7] = (sec["words"][7] & ~np.uint32(31 << 10)) | np.uint32(25 << 10)
    elif corrupt == "top_bits":
        sec["words"][9] |= np.uint32(1 << 31)
    elif corrupt == "gid_range":
        sec["gids"][4] = -3
    elif corrupt == "sum_len":
        hdr["sum_len"] = int(sec["len_sorted"].sum()) + 1
    elif corrupt == "max_len":
        hdr["max_len"] = int(sec["len_sorted"][-1]) + 1
    path = str(tmp_path / "crafted.swb")
    index_file.write(path, sec, hdr)
    if corrupt == "none" and __import__("torch").cuda.is_available():
        pytest.skip("loads for real on a GPU box (tests/test_gpu_parity.py)")
    with pytest.raises(sw.SwError) as ei:
        sw.Database.load(path)
    assert ei.value.code == (sw.SW_ECUDA if corrupt == "none" else sw.SW_EINVAL), sw.lib().sw_last_error()
