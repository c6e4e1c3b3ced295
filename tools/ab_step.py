"""A/B of the whole search step on a small database, timed as bench.py times C1:
one 512 MB L2 flush before each step (outside the timed interval), CUDA events
around each step on the search stream, sw_search_async with device outputs.

  python tools/ab_step.py C1 '{}' '{"launch_chain": -1}' [rounds] [steps]

Each arm (JSON sw_tuning fields, plus "long_threshold" for sw_opts) gets its own handle; the arms alternate
`rounds` times and every round prints the median and mean ms per step.
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
    tunings = [json.loads(a) for a in sys.argv[2:4]] if len(sys.argv) > 3 else [{}, {"launch_chain": -1}]
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
    torch.cuda.set_device(0)
    sdb = make_db(cfg)
    q = make_query(cfg)
    M = cfg.matrix32()
    n = sdb.n_seqs
    # an arm's "long_threshold" key goes to sw_opts, the rest to sw_tuning
    dbs = [sw.Database.from_synth(sdb, device=0, long_threshold=int(t.get("long_threshold", 0)),
                                  tuning={a: v for a, v in t.items() if a != "long_threshold"} or None)
           for t in tunings]
    for db in dbs:
        db.reserve(q.size, cfg.k)
    stream = torch.cuda.Stream()
    d_scores = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    d_ids = torch.empty(cfg.k, dtype=torch.int64, device="cuda")
    d_ts = torch.empty(cfg.k, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ref = None
    for db in dbs:                                   # same results on every arm
        db.search_async(q, M, cfg.alpha, cfg.beta, cfg.k, d_scores, d_ids, d_ts, stream)
        stream.synchronize()
        got = d_scores[:n].cpu().numpy().copy()
        if ref is None:
            ref = got
        assert np.array_equal(ref, got), "arms differ"
    for r in range(rounds):
        for t, db in zip(tunings, dbs):
            for _ in range(5):
                db.search_async(q, M, cfg.alpha, cfg.beta, cfg.k, d_scores, d_ids, d_ts, stream)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for a, b in ev:
                with torch.cuda.stream(stream):
                    flush.fill_(1)
                a.record(stream)
                db.search_async(q, M, cfg.alpha, cfg.beta, cfg.k, d_scores, d_ids, d_ts, stream)
                b.record(stream)
            stream.synchronize()
            ms = [a.elapsed_time(b) for a, b in ev]
            print(json.dumps({"round": r, "tuning": t, "config": cfg.name, "median_ms": round(statistics.median(ms), 4),
                              "mean_ms": round(statistics.mean(ms), 4), "min_ms": round(min(ms), 4)}), flush=True)


if __name__ == "__main__":
    main()
