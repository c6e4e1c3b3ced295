"""Uncontended intra-task wavefront: one database of two 3,303-residue subjects
(one pair item), query lengths 144 / 464; first-pass time per wavefront step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import blosum62, matrix32, random_db, stream_key  # noqa: E402
from swdata.synth import gen_residues  # noqa: E402

M = matrix32(blosum62())
for n in (3303,):
    db = random_db(1, np.array([n, n]))
    for m in (144, 464, 1000):
        q = gen_residues(stream_key(0, "q", m), 0, m)
        with sw.Database.from_synth(db, device=0, long_threshold=1) as g:
            for _ in range(3):
                g.search(q, M, 2, 12, k=1)
            t = min(g.search(q, M, 2, 12, k=1).stats["ms_inter"] for _ in range(5))
        tr = {144: 6, 464: 16, 1000: 16}[m]
        lanes = min(32, -(-((m + 7) // 8 * 8) // tr))
        passes = -(-((m + 7) // 8 * 8) // (32 * tr))
        steps = passes * (n + lanes)
        print(f"n={n} m={m}: first pass {t * 1e3:.1f} us, {steps} steps, {t * 1e6 / steps:.1f} ns/step "
              f"= {t * 1e-3 / steps * 1.965e9:.0f} cycles/step", flush=True)
