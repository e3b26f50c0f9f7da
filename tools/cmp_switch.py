import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
rng = np.random.default_rng(5)
for n, d in [(65536, 100), (65536, 128), (65536, 256), (4096, 100), (524288, 100)]:
    for fam in ("clusters", "gauss"):
        if fam == "gauss":
            x = rng.standard_normal((n, d)).astype(np.float32)
        else:
            x = (rng.uniform(-1, 1, (n // 64, d))[rng.integers(0, n // 64, n)] + rng.normal(0, 0.02, (n, d))).astype(np.float32)
        ps = psg.PointSet.from_flat(x, d)
        psg.closest_pair(ps, 10, 10.0, 1, 0)
        ts = []
        for _ in range(2):
            t0 = time.perf_counter(); psg.closest_pair(ps, 10, 10.0, 1, 0); ts.append(time.perf_counter() - t0)
        print(os.environ.get("PSG_NO_BRUTE_SWITCH", "switch"), n, d, fam, "%.2f ms" % (min(ts) * 1e3), flush=True)
        ps.release()
