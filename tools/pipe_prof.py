"""Per-warp-position wait profile of the pipelined first pass (debug build
libswsearch_prof.so, -DSW_PIPE_PROF): python tools/pipe_prof.py C2"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query

sw.LIB_PATH = os.path.join(ROOT, "paper_1404_4152_b200", "libswsearch_prof.so")
L = sw.lib()
L.sw_debug_pipe_counters.argtypes = [ctypes.c_void_p]
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
sdb = make_db(cfg)
q = make_query(cfg)
buf = np.zeros((16, 8), dtype=np.uint64)
with sw.Database.from_synth(sdb, device=0, tuning={"pipeline": 1}) as g:
    g.search(q, cfg.matrix32(), cfg.alpha, cfg.beta, k=cfg.k)
    L.sw_debug_pipe_counters(buf.ctypes.data)
    r = g.search(q, cfg.matrix32(), cfg.alpha, cfg.beta, k=cfg.k)
    L.sw_debug_pipe_counters(buf.ctypes.data)
tot = buf[:12, 3].astype(float)
for w in range(12):
    print(json.dumps({"warp": w, "item_wait": round(buf[w, 0] / tot[w], 4), "in_wait": round(buf[w, 1] / tot[w], 4),
                      "out_wait": round(buf[w, 2] / tot[w], 4), "items": int(buf[w, 4]) , "chunks": int(buf[w, 5]),
                      "mcycles": round(tot[w] / 148 / 1e6, 2)}))
print(json.dumps({"ms_first_pass": r.stats["ms_inter"]}))
