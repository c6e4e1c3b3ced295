"""f3 measurement: traceback of the top-k hits after a search (sw_search -> sw_align).
    python tools/run_align.py [--configs C2,C4] [--k 10] [--reps 3] [--json out.json]
Reports the align call's wall time, its DP cells (qlen x subject length per hit),
Gcell/s, and the oracle's full-matrix traceback time on the same hits (host cores)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C4")
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()
rows = []
for name in a.configs.split(","):
    cfg = CONFIGS[name]
    sdb = make_db(cfg)
    q = make_query(cfg)
    M = cfg.matrix32()
    with sw.Database.from_synth(sdb, device=0) as g:
        r = g.search(q, M, cfg.alpha, cfg.beta, k=a.k)
        hits = r.topk_ids.astype(np.int64)        # global ids == input indices here (1 GPU)
        g.align(q, M, cfg.alpha, cfg.beta, hits)   # warm-up
        best = 1e30
        for _ in range(a.reps):
            t = time.perf_counter()
            al = g.align(q, M, cfg.alpha, cfg.beta, hits)
            best = min(best, time.perf_counter() - t)
    cells = int(q.size * sdb.lengths[hits].sum())
    t = time.perf_counter()
    ref = [oracle.sw_align(q, sdb.seq(int(h)), M, cfg.alpha, cfg.beta) for h in hits]
    t_or = time.perf_counter() - t
    same = all({k: x[k] for k in y} == y for x, y in zip(al, ref))
    row = {"config": name, "qlen": int(q.size), "hits": int(hits.size), "cells": cells,
           "align_ms": round(best * 1e3, 3), "gcups": round(cells / best / 1e9, 2),
           "oracle_ms": round(t_or * 1e3, 1), "oracle_gcups": round(cells / t_or / 1e9, 3),
           "identical_to_oracle": same, "top_score": int(al[0]["score"]),
           "ops_lengths": [len(x["ops"]) for x in al][:5]}
    rows.append(row)
    print(json.dumps(row), flush=True)
if a.json:
    with open(a.json, "w") as f:
        json.dump(rows, f, indent=1)
