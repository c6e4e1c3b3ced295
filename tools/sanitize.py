"""Small invocation of every device entry point, for compute-sanitizer (memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize.py [--case all|search|stream|batch|align]
Each case checks its scores against the oracle too, so a sanitizer-clean run is also a correct one.
Sizes are small (the sanitizers slow kernels down 10-100x) but still cover every kernel: int8/16/32
first stages, saturation reruns, long subjects (intra-task wavefront and big boundary slabs),
streamed chunks (first chunk in pieces), paired batch queries, the traceback and the pipelined first
pass (shared-memory rings with mbarriers)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import blosum62, matrix32, random_db, stream_key  # noqa: E402
from swdata.synth import gen_residues  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="all")
a = ap.parse_args()

M = matrix32(blosum62())
rng = np.random.default_rng(7)
lens = np.concatenate([rng.integers(0, 400, size=700), [1, 2, 6, 7, 64, 65, 2500, 4100, 7000]])
db = random_db(7, lens)
q = gen_residues(stream_key(7, "sanitize-query", 200), 0, 200)
ref = oracle.db_scores(q, db, M, 2, 12)
cases = a.case.split(",") if a.case != "all" else ["search", "intra", "stream", "batch", "align", "pipeline"]


def check(name, scores, want=ref):
    ok = np.array_equal(scores, want)
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


if "search" in cases:
    for fs in (8, 16, 32):
        with sw.Database(db.residues, db.offsets, db.lengths, device=0, first_stage=fs) as g:
            check(f"search first_stage={fs}", g.search(q, M, 2, 12, k=10).scores)
    # saturation: large scores force int16 -> int32 reruns
    big = np.zeros((32, 32), dtype=np.int8)
    big[:24, :24] = 127
    ql = gen_residues(stream_key(9, "sanitize-query", 400), 0, 400)
    with sw.Database(db.residues, db.offsets, db.lengths, device=0) as g:
        r = g.search(ql, big, 2, 12, k=10)
    print("int32 reruns:", r.stats["n_rerun32"])
    check("search saturating", r.scores, oracle.db_scores(ql, db, big, 2, 12))
if "intra" in cases:   # every long group pair-wise: chained streams, isolated warps, 10-2k and register instances
    for tuning in ({}, {"intra_isolate": 1}, {"intra_chain": -1}, {"generic_gaps": 1}):
        with sw.Database(db.residues, db.offsets, db.lengths, device=0, long_threshold=1, tuning=tuning) as g:
            check(f"search all-intra {tuning}", g.search(q, M, 2, 12, k=10).scores)
    with sw.Database(db.residues, db.offsets, db.lengths, device=0, long_threshold=1) as g:
        check("search all-intra k=40 (radix top-k)", g.search(q, M, 2, 12, k=40).scores)
if "stream" in cases:
    with sw.Database(db.residues, db.offsets, db.lengths, device=0, residency=1, chunk_mb=1) as g:
        check("search streamed", g.search(q, M, 2, 12, k=10).scores)
if "batch" in cases:
    q2 = gen_residues(stream_key(8, "sanitize-query", 150), 0, 150)
    with sw.Database(db.residues, db.offsets, db.lengths, device=0) as g:
        r = g.search_batch([q, q2], M, 2, 12, k=10)
    check("batch q0", r.scores[0])
    check("batch q1", r.scores[1], oracle.db_scores(q2, db, M, 2, 12))
if "align" in cases:
    with sw.Database(db.residues, db.offsets, db.lengths, device=0) as g:
        hits = np.argsort(-ref, kind="stable")[:6].astype(np.int64)
        hits = np.concatenate([hits, [len(lens) - 1, len(lens) - 2]])
        al = g.align(q, M, 2, 12, hits)
    got = np.array([x["score"] for x in al])
    check("align scores", got, ref[hits])
if "pipeline" in cases:   # the pipelined first pass: rings, mbarriers, slabs, cp.async staging
    for chain in (0, 12):
        with sw.Database(db.residues, db.offsets, db.lengths, device=0,
                         tuning={"pipeline": 1, "pipe_chain": chain}) as g:
            check(f"search pipeline chain={chain or 3}", g.search(q, M, 2, 12, k=10).scores)
print("sanitize cases done", flush=True)
