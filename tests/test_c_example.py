"""The C ABI from plain C: examples/swsearch_cli.c compiles as strict C99 against include/swsearch.h
and links libswsearch.so (CPU); on a GPU its scores, top-k and traceback equal the oracle's."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum62, decode, matrix32, random_db, stream_key
from swdata.synth import gen_residues

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1404_4152_b200")


def _build(tmp_path):
    sw.lib()                                   # the library must exist (built by __graft_entry__.build)
    exe = str(tmp_path / "swsearch_cli")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "swsearch_cli.c"), "-L", PKG, "-lswsearch",
                    f"-Wl,-rpath,{PKG}", "-o", exe], check=True, capture_output=True, text=True)
    return exe


def _inputs(tmp_path, n=300, m=120):
    db = random_db(33, np.random.default_rng(33).integers(0, 500, size=n))
    q = gen_residues(stream_key(33, "c-example-query", m), 0, m)
    mpath, dpath = tmp_path / "blosum62.txt", tmp_path / "db.txt"
    mpath.write_text("\n".join(" ".join(str(int(v)) for v in row) for row in blosum62()) + "\n")
    dpath.write_text("".join(decode(db.residues[o:o + ln]) + "\n" for o, ln in zip(db.offsets, db.lengths)))
    return db, q, str(mpath), str(dpath)


def test_c_example_compiles_and_fails_loudly_without_gpu(tmp_path):
    exe = _build(tmp_path)
    _, q, mpath, dpath = _inputs(tmp_path, n=20)
    if __import__("torch").cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    p = subprocess.run([exe, mpath, dpath, decode(q)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 2 and "sw_db_create" in p.stderr and "CUDA error" in p.stderr, p.stderr


@pytest.mark.gpu
def test_c_example_matches_oracle(tmp_path):
    exe = _build(tmp_path)
    db, q, mpath, dpath = _inputs(tmp_path)
    k = 7
    p = subprocess.run([exe, mpath, dpath, decode(q), str(k), "2", "12"], capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr
    lines = [ln.split() for ln in p.stdout.splitlines()]
    got = np.array([int(x[2]) for x in lines if x[0] == "score"], dtype=np.int32)
    M = matrix32(blosum62())
    ref = oracle.db_scores(q, db, M, 2, 12)
    assert np.array_equal(got, ref)
    ti, ts = oracle.topk(ref, k)
    top = [(int(x[2]), int(x[3])) for x in lines if x[0] == "top"]
    assert top == list(zip(ti.tolist(), ts.tolist()))
    al = [x for x in lines if x[0] == "align"][0]
    best = int(ti[0])
    o = oracle.sw_align(q, db.residues[db.offsets[best]:db.offsets[best] + db.lengths[best]], M, 2, 12)
    want = [str(best), str(o["score"]), str(o["q_begin"]), str(o["q_end"]), str(o["s_begin"]), str(o["s_end"])]
    assert al[1:7] == want and (al[7] if len(al) > 7 else "") == o["ops"]
