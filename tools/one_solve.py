"""One (or a few) C2 solves, for profiling under ncu."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
logn = int(sys.argv[1]) if len(sys.argv) > 1 else 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pts, planted = psg.gen.gauss_planted(2, 1 << logn, 128)
ps = psg.PointSet.from_flat(pts, 128)
for _ in range(reps):
    r = psg.closest_pair(ps, 10, 10.0, 1, 0)
p = psg.last_profile()
print(r, sorted(planted), p["stage_list"], p["launches"])
assert (r.index_i, r.index_j) == tuple(sorted(planted))
