"""Full-size oracle references as digests (SURVEY.md §8(d) plan): for one
config and query length, the oracle (oracle/ only) scores every subject in
blocks of 65,536 input-order sequences; each block's int32 scores are hashed
(SHA-256, little-endian) and the exact top-k is kept.  Output: one small JSON
file under tests/golden/digests/, checked against the GPU by
tests/test_gpu_digests.py.  CPU only; run in the background:
    python tools/make_digests.py C2 [--m 464] [--threads N]"""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402
from swdata.synth import db_lengths, manifest_hash  # noqa: E402

BLOCK = 65536

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--m", type=int, default=None)
ap.add_argument("--threads", type=int, default=None)
ap.add_argument("--out", default=None, help="output directory (default tests/golden/digests)")
ap.add_argument("--blocks", default=None, help="a:b -- only blocks [a, b) (a part file, merged with --merge)")
ap.add_argument("--merge", nargs="*", default=None, help="part files to merge into the full digest file")
a = ap.parse_args()
cfg = CONFIGS[a.config]
m = a.m or cfg.qlens[0]
q = make_query(cfg, m)
M = cfg.matrix32()
lk = db_lengths(cfg)
n = cfg.n_seqs
out = os.path.join(a.out or os.path.join(ROOT, "tests", "golden", "digests"), f"{cfg.name}_m{m}.json")
os.makedirs(os.path.dirname(out), exist_ok=True)
if a.merge:                                            # combine part files written with --blocks
    parts = sorted((json.load(open(f)) for f in a.merge), key=lambda r: r["blocks"][0])
    assert parts[0]["blocks"][0] == 0 and all(p["blocks"][1] == q["blocks"][0] for p, q in zip(parts, parts[1:]))
    ci = np.concatenate([np.array(p["topk_ids"], np.int64) for p in parts])
    cs = np.concatenate([np.array(p["topk_scores"], np.int32) for p in parts])
    order = np.lexsort((ci, -cs.astype(np.int64)))[:cfg.k]
    rec = {k: v for k, v in parts[0].items() if k != "blocks"}
    rec["block_sha256"] = [d for p in parts for d in p["block_sha256"]]
    rec["block_manifest16"] = [d for p in parts for d in p["block_manifest16"]]
    assert len(rec["block_sha256"]) == (n + BLOCK - 1) // BLOCK
    rec["topk_ids"], rec["topk_scores"] = ci[order].tolist(), cs[order].tolist()
    rec["oracle_seconds"] = round(sum(p["oracle_seconds"] for p in parts), 1)
    with open(out, "w") as f:
        json.dump(rec, f)
    print(f"merged {len(parts)} parts into {out}")
    sys.exit(0)
blk = range(0, n, BLOCK)
if a.blocks:
    lo, hi = (int(x) for x in a.blocks.split(":"))
    blk = range(lo * BLOCK, min(n, hi * BLOCK), BLOCK)
    out = out[:-5] + f".part{lo}.json"
t0 = time.time()
digests, top_ids, top_scores, manifests = [], np.zeros(0, np.int64), np.zeros(0, np.int32), []
for b0 in blk:
    ids = np.arange(b0, min(n, b0 + BLOCK), dtype=np.int64)
    db = make_db(cfg, ids=ids, lengths_kind=lk)
    s = oracle.db_scores(q, db, M, cfg.alpha, cfg.beta, nthreads=a.threads)
    digests.append(hashlib.sha256(s.astype("<i4").tobytes()).hexdigest())
    manifests.append(manifest_hash(db)[:16])
    # running exact top-k by (score desc, id asc)
    ci = np.concatenate([top_ids, ids])
    cs = np.concatenate([top_scores, s])
    order = np.lexsort((ci, -cs.astype(np.int64)))[:cfg.k]
    top_ids, top_scores = ci[order], cs[order]
    if (b0 // BLOCK) % 20 == 0:
        print(f"{cfg.name} m={m}: {b0 + ids.size}/{n} seqs, {time.time() - t0:.0f}s", flush=True)
rec = {"config": cfg.name, "m": m, "n_seqs": n, "block": BLOCK, "alpha": cfg.alpha, "beta": cfg.beta,
       "blocks": [blk.start // BLOCK, (blk.stop + BLOCK - 1) // BLOCK],
       "matrix": cfg.matrix, "k": cfg.k, "block_sha256": digests, "block_manifest16": manifests,
       "topk_ids": top_ids.tolist(), "topk_scores": top_scores.tolist(),
       "oracle_seconds": round(time.time() - t0, 1), "written_by": "tools/make_digests.py (oracle/ only)"}
with open(out, "w") as f:
    json.dump(rec, f)
print(f"wrote {out} in {time.time() - t0:.0f}s", flush=True)
