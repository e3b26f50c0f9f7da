"""One (or a few) C3 solves (z-normalised motif), for profiling under ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s, (a, b) = psg.gen.walk_motif(3, 1 << 20, 256)
ps = psg.PointSet.windows_of(s.astype(np.float64), 256, znorm=True)
for _ in range(reps):
    r = psg.closest_pair(ps, 10, 10.0, 1, 256)
p = psg.last_profile()
print(r, sorted((a, b)), p["stage_list"], p["launches"], p["window_pairs"], p["lb_survivors"], p["candidates"])
