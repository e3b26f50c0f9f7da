"""Resident closest-pair solve times over shapes and data families (second
and third solves; the first learns), to spot pathological engine choices."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
rng = np.random.default_rng(5)
fams = {
    "gauss": lambda n, d: rng.standard_normal((n, d)).astype(np.float32),
    "uniform": lambda n, d: rng.random((n, d), dtype=np.float32),
    "clusters": lambda n, d: (rng.uniform(-1, 1, (max(1, n // 64), d))[rng.integers(0, max(1, n // 64), n)]
                              + rng.normal(0, 0.02, (n, d))).astype(np.float32),
}
for n in (1 << 12, 1 << 16, 1 << 19):
    for d in (2, 3, 8, 16, 32, 64, 100, 128, 256):
        if n * d > (1 << 26):
            continue
        for fam, gen in fams.items():
            x = gen(n, d)
            ps = psg.PointSet.from_flat(x, d)
            t0 = time.perf_counter(); r = psg.closest_pair(ps, 10, 10.0, 1, 0); t1 = time.perf_counter() - t0
            ts = []
            for _ in range(2):
                t0 = time.perf_counter(); r = psg.closest_pair(ps, 10, 10.0, 1, 0); ts.append(time.perf_counter() - t0)
            print(f"n={n:7d} d={d:3d} {fam:8s} first {t1*1e3:8.2f} ms  resident {min(ts)*1e3:8.3f} ms", flush=True)
            ps.release()
