"""f2 measurement: the same searches on a device-resident and on a host-resident
(streamed, residency 1) database.  python tools/run_stream.py [--configs C2,C5] [--chunk-mb 512]"""
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
ap.add_argument("--configs", default="C2,C5")
ap.add_argument("--chunk-mb", type=int, default=512)
ap.add_argument("--searches", type=int, default=3)
ap.add_argument("--json", default=None)
a = ap.parse_args()
rows = []
for name in a.configs.split(","):
    cfg = CONFIGS[name]
    sdb = make_db(cfg)
    M = cfg.matrix32()
    for m in cfg.qlens:
        q = make_query(cfg, m)
        res = {}
        for residency in (0, 1):
            t = time.perf_counter()
            g = sw.Database.from_synth(sdb, device=0, residency=residency, chunk_mb=a.chunk_mb)
            tc = time.perf_counter() - t
            g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)
            best = None
            for _ in range(a.searches):
                r = g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)
                if best is None or r.stats["seconds"] < best.stats["seconds"]:
                    best = r
            info = g.info()
            g.close()
            res[residency] = (best, info, tc)
        r0, r1 = res[0][0], res[1][0]
        row = {"config": name, "m": int(m), "cells": int(r0.stats["cells"]),
               "packed_gb": round(res[1][1]["packed_bytes"] / 1e9, 2), "chunks": res[1][1]["n_chunks"],
               "chunk_mb": a.chunk_mb,
               "resident_gcups": round(r0.stats["gcups"], 1), "streamed_gcups": round(r1.stats["gcups"], 1),
               "streamed_over_resident": round(r1.stats["gcups"] / r0.stats["gcups"], 3),
               "streamed_h2d_gb_per_s": round(res[1][1]["packed_bytes"] / r1.stats["seconds"] / 1e9, 1),
               "identical": bool(np.array_equal(r0.scores, r1.scores) and np.array_equal(r0.topk_ids, r1.topk_ids)),
               "create_s": [round(res[0][2], 1), round(res[1][2], 1)]}
        rows.append(row)
        print(json.dumps(row), flush=True)
if a.json:
    with open(a.json, "w") as f:
        json.dump(rows, f, indent=1)
