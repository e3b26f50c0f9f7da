import sys, os
sys.path.insert(0, os.getcwd())
import paper_1407_5609_b200 as psg
pts, planted = psg.gen.gauss_planted(2, 5000, 16)
ps = psg.PointSet.from_flat(pts, 16)
r = psg.closest_pair(ps, 10, 10.0, 1, 0)
print(r.index_i, r.index_j, sorted(planted))
