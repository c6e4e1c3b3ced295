"""Profile the f1 pair kernel alone: one sw_search_batch of 2 C2 queries."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1404_4152_b200 as sw  # noqa: E402
from swdata import CONFIGS, make_db, make_query  # noqa: E402
base = CONFIGS["C2"]
db = make_db(base)
qs = [make_query(base, None, seed=s) for s in range(2)]
g = sw.Database.from_synth(db, device=0)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    r = g.search_batch(qs, base.matrix32(), base.alpha, base.beta, k=10, scores=False)
    print(r.stats["seconds"], r.stats["gcups"], flush=True)
g.close()
