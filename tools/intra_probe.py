"""Uncontended intra-task wavefront: one pair of 3,303-residue subjects, query lengths 8..512 (rows per
lane TR = 4..16); first-pass time per subject column and per column-row.  `python tools/intra_probe.py [2|4]` selects the
columns per wavefront step (sw_tuning.intra_cols; 2 needs the ablation build)."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1404_4152_b200 as sw
from swdata import blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues
M = matrix32(blosum62())
n = 3303
db = random_db(1, np.array([n, n]))
for m in (8, 32, 64, 128, 144, 256, 512):
    q = gen_residues(stream_key(0, "q", m), 0, m)
    with sw.Database.from_synth(db, device=0, long_threshold=1,
                                tuning={"intra_cols": int(sys.argv[1]) if len(sys.argv) > 1 else 0}) as g:
        for _ in range(3):
            g.search(q, M, 2, 12, k=1)
        t = min(g.search(q, M, 2, 12, k=1).stats["ms_inter"] for _ in range(5))
    m_pad = (m + 7) // 8 * 8
    need = (m_pad + 31) // 32
    tr = 4 if need <= 4 else need if need <= 8 else 10 if need <= 10 else 12 if need <= 12 else 14 if need <= 14 else 16
    lanes = min(32, -(-m_pad // tr))
    passes = -(-m_pad // (32 * tr))
    cols = passes * n
    cyc = t * 1e-3 / cols * 1.965e9
    print(f"m={m} TR={tr} lanes={lanes} passes={passes}: {t*1e3:.1f} us, {t*1e6/cols:.1f} ns/column = "
          f"{cyc:.0f} cycles/column, {cyc/tr:.1f} cycles/column-row", flush=True)
