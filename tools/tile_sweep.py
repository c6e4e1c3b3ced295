"""Sweep register-tile height / CTA size of the int16x2 first pass (sw_tuning.tile_rows / threads, ablation build) on C2.
    python tools/tile_sweep.py"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json, statistics
sys.path.insert(0, %r)
import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query
cfg = CONFIGS["C2"]; sdb = make_db(cfg); q = make_query(cfg); M = cfg.matrix32()
g = sw.Database.from_synth(sdb, device=0, tuning=json.loads(sys.argv[1]))
for _ in range(2): g.search(q, M, 2, 12, k=10)
t = [g.search(q, M, 2, 12, k=10).stats["ms_inter"] for _ in range(4)]
print(json.dumps({"ms_first_pass": min(t), "tcups": cfg.qlens[0] * int(sdb.lengths.sum()) / min(t) / 1e9}))
''' % ROOT
for T, NT in ((48, 384), (32, 384), (32, 512), (64, 384)):
    out = subprocess.run([sys.executable, "-c", code, json.dumps({"tile_rows": T, "threads": NT})],
                         capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    print(json.dumps({"tile_rows": T, "threads": NT, "result": line}), flush=True)
