"""The unmodified reference closest_pair (oracle/_ref) on the FULL C2 config
(n = 2^20, d = 128, the same seeded recipe as bench.py), single thread, timed.
Test infrastructure / measurement only.  Writes one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1407_5609_b200 as psg

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n, d = 1 << logn, 128
pts, planted = psg.gen.gauss_planted(2, n, d)
ref = oracle.reference()
t0 = time.perf_counter()
r = ref.closest_pair(pts.astype(np.float64), 10, 10.0, 1, 0)
t = time.perf_counter() - t0
print(json.dumps({"n": n, "d": d, "seconds": t, "threads": 1, "answer": [r.index_i, r.index_j, r.distance],
                  "planted": sorted(planted), "pairs_examined": r.pairs_examined,
                  "host": os.uname().nodename, "nproc": os.cpu_count()}))
