"""Small-database (C1) sweep of the inter/intra split (sw_opts.long_threshold).  python tools/c1_sweep.py"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json
sys.path.insert(0, %r)
import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query
cfg = CONFIGS[sys.argv[1]]; sdb = make_db(cfg); q = make_query(cfg); M = cfg.matrix32()
g = sw.Database.from_synth(sdb, device=0, long_threshold=int(sys.argv[2]))
for _ in range(3): g.search(q, M, 2, 12, k=10)
rs = [g.search(q, M, 2, 12, k=10).stats for _ in range(5)]
b = min(rs, key=lambda r: r["ms_inter"])
print(json.dumps({"ms_first_pass": round(b["ms_inter"], 3), "ms_total_dev": round(b["ms_profile"] + b["ms_inter"] + b["ms_rerun"] + b["ms_finalize"], 3), "n_intra": b["n_intra"], "max_len": int(sdb.lengths.max())}))
''' % ROOT
for cols in (sys.argv[2].split(",") if len(sys.argv) > 2 else (None, "128", "512", "1000", "2000", "100000")):
    lt = cols if cols and cols != "default" else "0"
    out = subprocess.run([sys.executable, "-c", code, sys.argv[1] if len(sys.argv) > 1 else "C1", lt],
                         capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    print(json.dumps({"long_threshold": cols or "default", "result": line}), flush=True)
