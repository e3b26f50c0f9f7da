"""C5 at full size (n = 2^24, d = 64, 1024-cluster mixture) pinned by an
independent exhaustive search: the scan's answer, its FP64 distance
recomputed by the oracle, and the one-pass device brute force over the FP64
band of that distance (every pair at distance <= it; refscan.cpp:134-157).
Writes one JSON object (argv[1], default gpurun_out/c5_fullsize.json)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_1407_5609_b200 as psg  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5_fullsize.json"
logn = int(sys.argv[2]) if len(sys.argv) > 2 else 24
n = 1 << logn
t0 = time.time()
pts = psg.gen.mixture(5, n, 64, 1024, 0.05)
gen_s = time.time() - t0
ps = psg.PointSet.from_flat(pts, 64)
solves = []
for _ in range(3):
    t = time.time()
    got = psg.closest_pair(ps, 10, 10.0, 1, 0)
    solves.append({"wall_s": time.time() - t, "profile": {k: v for k, v in psg.last_profile().items()
                                                          if k not in ("stages",)}})
orc = oracle.port()
d_oracle = orc.euclidean(pts[got.index_i].astype(np.float64), pts[got.index_j].astype(np.float64))
t = time.time()
bf = psg.brute_force_bounded(ps, 0, got.distance)
brute_s = time.time() - t
res = {
    "config": f"C5 recipe n=2^{logn} d=64, 1024 clusters sigma=0.05, master seed 5; q=10 f=10 seed=1 zone=0",
    "n": n,
    "answer": [got.index_i, got.index_j, got.distance],
    "oracle_fp64_distance_of_answer": d_oracle,
    "brute_force": [bf.index_i, bf.index_j, bf.distance],
    "brute_force_s": brute_s,
    "brute_pairs": n * (n - 1) // 2,
    "agree": (bf.index_i, bf.index_j, bf.distance) == (got.index_i, got.index_j, got.distance)
    and d_oracle == got.distance,
    "gen_s": gen_s,
    "solves": solves,
}
os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
with open(out_path, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "solves"}))
print("solve wall s:", [round(x["wall_s"], 4) for x in solves])
