"""C5 recipe at a given n: stage list and counters (profiling aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
pts = psg.gen.mixture(5, n, 64, 1024, 0.05)
ps = psg.PointSet.from_flat(pts, 64)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    r = psg.closest_pair(ps, 10, 10.0, 1, 0)
    p = psg.last_profile()
    print(r.index_i, r.index_j, r.distance, p["total_ms"], p["stage_list"], p["window_pairs"], p["lb_survivors"], p["launches"])
