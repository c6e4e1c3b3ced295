"""f1 measurement: the paper's 20-query protocol as one sw_search_batch call
against a C2-shaped database, vs 20 single searches.  Query lengths: 20 synthetic lengths
spaced geometrically from 144 to 5,478 (the paper's range; its queries are not reproduced).
    python tools/run_batch.py [--config C2] [--n 20]
Both arms are warmed up on the full query set first (the first call of a process loads every kernel
instance it uses) and timed best of 3."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--lengths", default=None, help="comma-separated query lengths (default: geometric 144..5478)")
ap.add_argument("--json", default=None)
a = ap.parse_args()
cfg = CONFIGS[a.config]
sdb = make_db(cfg)
M = cfg.matrix32()
lens = (np.array([int(x) for x in a.lengths.split(",")]) if a.lengths
        else np.unique(np.round(np.geomspace(144, 5478, a.n)).astype(int)))
qs = [make_query(cfg, int(m), seed=7) for m in lens]
cells = int(sdb.lengths.sum()) * int(lens.sum())
with sw.Database.from_synth(sdb, device=0) as g:
    g.search_batch(qs, M, cfg.alpha, cfg.beta, k=10, scores=False)   # warm-up: first use of every kernel instance
    for q in qs:
        g.search(q, M, cfg.alpha, cfg.beta, k=10)
    t_batch = t_single = 1e30
    for _ in range(3):                                                # best of 3, warm
        t = time.perf_counter()
        rb = g.search_batch(qs, M, cfg.alpha, cfg.beta, k=10, scores=True)
        t_batch = min(t_batch, time.perf_counter() - t)
        t = time.perf_counter()
        singles = [g.search(q, M, cfg.alpha, cfg.beta, k=10) for q in qs]
        t_single = min(t_single, time.perf_counter() - t)
same = all(np.array_equal(rb.scores[i], singles[i].scores) and np.array_equal(rb.topk_ids[i], singles[i].topk_ids)
           for i in range(len(qs)))
row = {"config": a.config, "queries": len(qs), "qlens": lens.tolist(), "cells": cells,
       "batch_s": round(t_batch, 3), "batch_gcups": round(cells / t_batch / 1e9, 1),
       "pairs_joint": rb.stats.get("pairs"), "singles_s": round(t_single, 3),
       "singles_gcups": round(cells / t_single / 1e9, 1), "identical": bool(same)}
print(json.dumps(row), flush=True)
if a.json:
    json.dump(row, open(a.json, "w"), indent=1)
