"""Per-config GPU throughput table (device stage times via CUDA events inside the library).
    python tools/run_configs.py [--configs C1,C2,C3,C4,C5] [--searches 5] [--first-stage 16] [--ncu]
SURVEY.md §8(d)'s protocol: per config and per query, the median of 5 timed sw_search calls after 1
warm-up, SM clocks sampled (nvidia-smi) during the timed calls, and the roofline fraction at the max
clock and at the sampled clock.  --ncu: one search per query and no warm-up (for an ncu metric pass)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import statistics  # noqa: E402

import paper_1404_4152_b200 as sw  # noqa: E402
from bench import ClockSampler  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402

PEAK = 148 * 1965e6 * 64 / 1.75 / 1e9   # DPX roofline, Gcell/s at max clock

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
ap.add_argument("--searches", type=int, default=5)
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--first-stage", type=int, default=16)
ap.add_argument("--json", default=None)
a = ap.parse_args()
rows = []
for name in a.configs.split(","):
    cfg = CONFIGS[name]
    t = time.time()
    db = make_db(cfg)
    tg = time.time() - t
    t = time.time()
    g = sw.Database.from_synth(db, device=0, first_stage=a.first_stage)
    tc = time.time() - t
    M = cfg.matrix32()
    for m in cfg.qlens:
        q = make_query(cfg, m)
        if a.ncu:
            g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)
            print(json.dumps({"config": name, "m": m, "ncu": "one search"}), flush=True)
            continue
        g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k)      # warm-up
        clocks = ClockSampler(0)
        clocks.start()
        sts = [g.search(q, M, cfg.alpha, cfg.beta, k=cfg.k).stats for _ in range(a.searches)]
        clk = clocks.stop()

        def med(key):
            return statistics.median(x[key] for x in sts)
        cells = sts[0]["cells"]
        dev = [x["ms_profile"] + x["ms_inter"] + x["ms_rerun"] + x["ms_finalize"] for x in sts]
        dev_ms, ms_inter = statistics.median(dev), med("ms_inter")
        f_run = (clk.get("sm_mhz") or 1965.0) / 1965.0
        row = {"config": name, "m": m, "n_seqs": db.n_seqs, "cells": cells, "searches": a.searches,
               "stat": "median", "wall_ms": round(med("seconds") * 1e3, 3),
               "wall_ms_min": round(min(x["seconds"] for x in sts) * 1e3, 3), "device_ms": round(dev_ms, 3),
               "gcups_wall": round(cells / med("seconds") / 1e9, 1), "gcups_device": round(cells / dev_ms / 1e6, 1),
               "gcups_first_pass": round(cells / ms_inter / 1e6, 1),
               "frac_dpx_roofline": round(cells / ms_inter / 1e6 / PEAK, 4),
               "frac_dpx_roofline_at_run_clock": round(cells / ms_inter / 1e6 / (PEAK * f_run), 4),
               "ms_first_pass": round(ms_inter, 3), "ms_rerun": round(med("ms_rerun"), 3),
               "ms_rank": round(med("ms_finalize"), 3), "rerun_share": round(med("ms_rerun") / dev_ms, 5),
               "n_rerun32": sts[0]["n_rerun32"], "n_intra": sts[0]["n_intra"], "clocks": clk,
               "gen_s": round(tg, 1), "create_s": round(tc, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    g.close()
    del db
if a.json:
    with open(a.json, "w") as f:
        json.dump(rows, f, indent=1)
