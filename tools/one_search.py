"""One warm search of a config (for ncu captures): python tools/one_search.py C2 [tuning-json] [m]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
tuning = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
m = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.qlens[0]
sdb = make_db(cfg)
q = make_query(cfg, m)
with sw.Database.from_synth(sdb, device=0, tuning=tuning) as g:
    for _ in range(2):
        r = g.search(q, cfg.matrix32(), cfg.alpha, cfg.beta, k=cfg.k)
print(json.dumps({"config": cfg.name, "m": m, "tuning": tuning, "ms_first_pass": r.stats["ms_inter"],
                  "top": int(r.topk_scores[0])}))
