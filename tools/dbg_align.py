"""Debug: one planted near-copy at query length m; GPU traceback vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1404_4152_b200 as sw
from swdata import blosum62, matrix32, stream_key
from swdata.synth import SynthDB, _mutate, gen_residues
B62 = matrix32(blosum62())
for m in [int(x) for x in sys.argv[1:]]:
    q = gen_residues(stream_key(3, "align-query", m), 0, m)
    s = _mutate(q, stream_key(9, "plant", m))
    db = SynthDB(s, np.array([0]), np.array([s.size], np.int32), np.array([0]), "dbg")
    with sw.Database.from_synth(db, device=0) as g:
        r = g.search(q, B62, 2, 12, k=1)
        try:
            a = g.align(q, B62, 2, 12, [0])[0]
        except Exception as e:
            a = {"error": str(e)}
    ref = oracle.sw_align(q, s, B62, 2, 12)
    print(m, s.size, "search", r.scores[0], "gpu", {k: a.get(k) for k in ("score", "q_begin", "q_end", "s_begin", "s_end")},
          "ref", {k: ref[k] for k in ("score", "q_begin", "q_end", "s_begin", "s_end")},
          "ops_equal", a.get("ops") == ref["ops"], a.get("error", ""), flush=True)
