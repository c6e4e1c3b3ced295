"""Full-size, every-subject parity against stored oracle digests (SURVEY.md
§8(d) plan).  tools/make_digests.py (oracle/ only, run on CPU) stored, per
65,536-sequence block of each full BASELINE config, the SHA-256 of the
oracle's int32 scores and the exact top-k.  Here the GPU searches the same
regenerated database (the per-block data manifest is checked first) and every
block digest and the top-k must match: bit-exactness for all N subjects."""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1404_4152_b200 as sw
from swdata import CONFIGS, make_db, make_query
from swdata.synth import manifest_hash

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "digests", "*.json")))


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f)[:-5] for f in FILES])
def test_full_config_matches_oracle_digests(path):
    rec = json.load(open(path))
    cfg = CONFIGS[rec["config"]]
    q = make_query(cfg, rec["m"])
    db = make_db(cfg)
    B = rec["block"]
    assert db.n_seqs == rec["n_seqs"]
    for b, man in zip(range(0, db.n_seqs, B), rec["block_manifest16"][:3]):   # same input bytes
        lens = db.lengths[b:b + B]
        o0 = int(db.offsets[b])
        sub = type(db)(db.residues[o0:o0 + int(lens.sum())], db.offsets[b:b + B] - o0, lens,
                       db.global_ids[b:b + B], db.config)
        assert manifest_hash(sub)[:16] == man
    with sw.Database.from_synth(db, device=0) as g:
        r = g.search(q, cfg.matrix32(), rec["alpha"], rec["beta"], k=rec["k"])
    bad = [i for i, b in enumerate(range(0, db.n_seqs, B))
           if hashlib.sha256(r.scores[b:b + B].astype("<i4").tobytes()).hexdigest() != rec["block_sha256"][i]]
    assert not bad, f"{len(bad)} of {len(rec['block_sha256'])} blocks differ, first block {bad[0]}"
    assert r.topk_ids.tolist() == rec["topk_ids"] and r.topk_scores.tolist() == rec["topk_scores"]
