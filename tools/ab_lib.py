"""A/B: first-pass time with the in-tree library and an alternative build (path in argv[1]);
AB_TUNING (JSON) passes sw_tuning fields, e.g. AB_TUNING='{"generic_gaps": 1}'; AB_LT sets long_threshold."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1404_4152_b200 as sw  # noqa: E402

if len(sys.argv) > 1:
    sw.LIB_PATH = sys.argv[1]
from swdata import CONFIGS, make_db, make_query  # noqa: E402

cfg = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "C2"]
sdb = make_db(cfg)
q = make_query(cfg)
M = cfg.matrix32()
tuning = json.loads(os.environ.get("AB_TUNING", "{}"))
g = sw.Database.from_synth(sdb, device=0, tuning=tuning or None, long_threshold=int(os.environ.get("AB_LT", "0")))
for _ in range(3):
    g.search(q, M, cfg.alpha, cfg.beta, k=10)
n = int(os.environ.get("AB_N", "6"))
t = sorted(g.search(q, M, cfg.alpha, cfg.beta, k=10).stats["ms_inter"] for _ in range(n))
print(os.path.basename(sw.LIB_PATH), tuning, cfg.name, "first pass ms min/median", round(t[0], 3), round(t[n // 2], 3), flush=True)
