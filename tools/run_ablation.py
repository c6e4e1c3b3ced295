"""f4 measurement: first-pass device time of each kernel variant (sw_tuning.variant, ablation build) on C2 (and C4).
    python tools/run_ablation.py [--configs C2,C4] [--variants base,intersp]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json
sys.path.insert(0, %r)
import numpy as np
import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query
cfg = CONFIGS[sys.argv[1]]; sdb = make_db(cfg); q = make_query(cfg); M = cfg.matrix32()
g = sw.Database.from_synth(sdb, device=0, **json.loads(sys.argv[2]))
for _ in range(2): g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)
rs = [g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k) for _ in range(3)]
t = min(r.stats["ms_inter"] for r in rs)
cells = q.size * int(sdb.lengths.sum())
h = int(np.bitwise_xor.reduce(rs[0].scores.astype(np.int64) * 2654435761 %% 1000003))
print(json.dumps({"ms_first_pass": round(t, 3), "gcups_first_pass": round(cells / t / 1e6, 1), "score_hash": h}))
''' % ROOT
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2,C4")
ap.add_argument("--variants", default="base,intersp,intra,intraqp,static")
ap.add_argument("--json", default=None)
a = ap.parse_args()
rows = []
for cfgname in a.configs.split(","):
    for v in a.variants.split(","):
        kw = {}
        if v in ("intersp", "intraqp", "static"):
            kw["tuning"] = {"variant": v}
        if v in ("intra", "intraqp"):                    # every group through the intra-task path
            kw["long_threshold"] = 1
        out = subprocess.run([sys.executable, "-c", code, cfgname, json.dumps(kw)], capture_output=True, text=True)
        try:
            res = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            res = {"error": out.stderr[-400:]}
        row = {"config": cfgname, "variant": v, **res}
        rows.append(row)
        print(json.dumps(row), flush=True)
if a.json:
    json.dump(rows, open(a.json, "w"), indent=1)
