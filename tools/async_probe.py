"""Probe: first-pass device time of back-to-back async searches vs blocking searches (C2).
    python tools/async_probe.py"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402

cfg = CONFIGS["C2"]
sdb = make_db(cfg)
q = make_query(cfg, None)
M = cfg.matrix32()
for lt in (0, -1):
    db = sw.Database.from_synth(sdb, device=0, long_threshold=lt)
    st = torch.cuda.Stream()
    d_s = torch.empty(sdb.n_seqs, dtype=torch.int32, device="cuda")
    d_i = torch.empty(10, dtype=torch.int64, device="cuda")
    d_v = torch.empty(10, dtype=torch.int32, device="cuda")
    for mode in ("async", "async_sync_each", "sync"):
        for _ in range(3):
            db.search_async(q, M, 2, 12, 10, d_s, d_i, d_v, stream=st)
        st.synchronize()
        for _ in range(8):
            if mode == "sync":
                db.search(q, M, 2, 12, 10)
            else:
                db.search_async(q, M, 2, 12, 10, d_s, d_i, d_v, stream=st)
                if mode == "async_sync_each":
                    st.synchronize()
        st.synchronize()
        t = [db.stage_times(b) for b in range(1, 9)]
        print(f"long_threshold={lt:3d} {mode:16s} first-pass ms: mean {statistics.mean(x[1] for x in t):.3f} "
              f"min {min(x[1] for x in t):.3f} max {max(x[1] for x in t):.3f}", flush=True)
    db.close()
