import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle, paper_1404_4152_b200 as sw
from swdata import random_db, blosum62, matrix32
from test_gpu_parity import _query
B62 = matrix32(blosum62())
rng = np.random.default_rng(77)
db = random_db(77, np.concatenate([rng.integers(0, 900, size=1500), [0, 1, 5000]]))
qs = [_query(m, 30 + i) for i, m in enumerate([1, 100, 333, 464, 47, 2600, 129])]
g = sw.Database.from_synth(db, device=0)
ref = oracle.db_scores(qs[5], db, B62, 2, 12)
r1 = g.search(qs[5], B62, 2, 12, k=12)
print("single ok", np.array_equal(r1.scores, ref), r1.stats["n_intra"])
r = g.search_batch(qs, B62, 2, 12, k=12)
bad = np.nonzero(r.scores[5] != ref)[0]
print("batch bad", bad.size, bad[:10], db.lengths[bad[:10]], r.scores[5][bad[:5]], ref[bad[:5]])
r2 = g.search_batch([qs[5]], B62, 2, 12, k=12)
print("batch-of-1 ok", np.array_equal(r2.scores[0], ref))
r3 = g.search_batch([qs[0], qs[5]], B62, 2, 12, k=12)
print("batch (1, 2600) ok", np.array_equal(r3.scores[1], ref))
