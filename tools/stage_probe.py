"""Per-stage device times of one config: graph replays carry event nodes at
level PSG_GRAPH_PROF (default 2; 0 gives the graph's own total only).  python tools/stage_probe.py c2|c5|c3|c1 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_5609_b200 as psg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
zone = 0
if which == "c2":
    pts, _ = psg.gen.gauss_planted(2, 1 << 20, 128)
    ps = psg.PointSet.from_flat(pts, 128)
elif which == "c1":
    ps = psg.PointSet.from_flat(psg.gen.uniform(1, 16384, 2), 2)
elif which == "c3":
    s, _ = psg.gen.walk_motif(3, 1 << 20, 256)
    ps = psg.PointSet.windows_of(s.astype(np.float64), 256, znorm=True)
    zone = 256
else:
    ps = psg.PointSet.from_flat(psg.gen.mixture(5, 1 << 24, 64, 1024, 0.05), 64)
psg.set_graph_profiling(int(os.environ.get("PSG_GRAPH_PROF", "2")))
out = []
for k in range(reps + 1):
    r = psg.closest_pair(ps, 10, 10.0, 1, zone)
    p = psg.last_profile()
    if k:
        out.append({"total_ms": p["total_ms"], "stages": p["stage_list"], "project_ms": p["project_kernel_ms"],
                    "bootstrap_ms": p["bootstrap_kernel_ms"], "scan_ms": p["scan_kernel_ms"],
                    "window_pairs": p["window_pairs"], "lb_survivors": p["lb_survivors"],
                    "dense_tiles": p["dense_tiles"], "launches": p["launches"]})
print(json.dumps({"config": which, "graph": os.environ.get("PSG_NO_GRAPH") is None,
                  "boot_evals": os.environ.get("PSG_BOOT_EVALS"), "answer": [r.index_i, r.index_j, r.distance],
                  "runs": out}))
