"""A/B of first-pass variants on one config: first-pass device time (median of
5 after 2 warm-ups) and identical scores.  Default variants: per-warp global
slabs (production), the shared-memory pipeline (sw_tuning.pipeline = 1) with
chains of 3 (one SM sub-partition), 1, 6 and 12 warps (ablation build).
    python tools/ab_pipe.py [C2] [m|-] ['[{"pipeline": 1}, ...]']"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
m = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else cfg.qlens[0]
variants = json.loads(sys.argv[3]) if len(sys.argv) > 3 else [{}, {"pipeline": 1}, {"pipeline": 1, "pipe_chain": 1},
                                                           {"pipeline": 1, "pipe_chain": 6},
                                                           {"pipeline": 1, "pipe_chain": 12}]
sdb = make_db(cfg)
q = make_query(cfg, m)
M = cfg.matrix32()
cells = m * int(sdb.lengths.astype(np.int64).sum())
out = []
ref = None
for tun in variants:
    with sw.Database.from_synth(sdb, device=0, tuning=tun) as g:
        for _ in range(2):
            g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)
        rs = [g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k) for _ in range(5)]
    t = statistics.median(r.stats["ms_inter"] for r in rs)
    if ref is None:
        ref = rs[0].scores
    out.append({"tuning": tun, "ms_first_pass": round(t, 3), "gcups": round(cells / t / 1e6, 1),
                "same_scores": bool(np.array_equal(rs[0].scores, ref))})
print(json.dumps({"config": name, "m": m, "variants": out}), flush=True)
