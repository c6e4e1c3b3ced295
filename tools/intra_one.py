"""One intra-task pair item (two 3,303-residue subjects, m = 144): for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1404_4152_b200 as sw
from swdata import blosum62, matrix32, random_db, stream_key
from swdata.synth import gen_residues
M = matrix32(blosum62())
db = random_db(1, np.array([3303, 3303]))
q = gen_residues(stream_key(0, "q", 144), 0, 144)
with sw.Database.from_synth(db, device=0, long_threshold=1) as g:
    for _ in range(2):
        g.search(q, M, 2, 12, k=1)
