"""Run a few searches of one config (for ncu / quick timing).  Not part of the product.
    python tools/profile_search.py [--config C2] [--searches 3] [--n N] [--first-stage 16]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402
from swdata.synth import Config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--searches", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--first-stage", type=int, default=16)
a = ap.parse_args()
base = CONFIGS[a.config]
cfg = Config(**{**base.__dict__, "n_seqs": a.n}) if a.n else base
t = time.time()
db = make_db(cfg)
q = make_query(base, a.m)
print(f"data {time.time() - t:.1f}s  n={db.n_seqs} residues={db.residues.size} m={q.size}", flush=True)
M = base.matrix32()
g = sw.Database.from_synth(db, device=0, first_stage=a.first_stage)
for i in range(a.searches):
    r = g.search(q, M, base.alpha, base.beta, k=base.k)
    st = r.stats
    print(f"search {i}: {st['seconds']*1e3:.2f} ms wall  {st['gcups']:.1f} GCUPS  profile {st['ms_profile']:.3f} "
          f"inter {st['ms_inter']:.3f} rerun {st['ms_rerun']:.3f} final {st['ms_finalize']:.3f} ms  "
          f"kernel GCUPS {st['cells']/st['ms_inter']/1e6:.1f}  reruns {st['n_rerun32']}", flush=True)
g.close()
if os.environ.get("SW_BATCH"):
    qs = [make_query(base, a.m, seed=s) for s in range(int(os.environ["SW_BATCH"]))]
    g = sw.Database.from_synth(db, device=0, first_stage=a.first_stage)
    for i in range(a.searches):
        r = g.search_batch(qs, M, base.alpha, base.beta, k=base.k, scores=False)
        st = r.stats
        print(f"batch {len(qs)} queries: {st['seconds']*1e3:.2f} ms wall  {st['gcups']:.1f} GCUPS  pairs {st['pairs']}", flush=True)
    g.close()
