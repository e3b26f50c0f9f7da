import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
for n, d in [(16384, 2), (4096, 128), (32768, 2), (65536, 2), (16384, 16)]:
    pts = psg.gen.uniform(1, n, d)
    ps = psg.PointSet.from_flat(pts, d)
    for _ in range(2):
        a = psg.closest_pair(ps, 10, 10.0, 1, 0)
        b = psg.brute_force_closest_pair(ps, 0)
    ta, tb = [], []
    for _ in range(5):
        t0 = time.perf_counter(); a = psg.closest_pair(ps, 10, 10.0, 1, 0); ta.append(time.perf_counter() - t0)
        t0 = time.perf_counter(); b = psg.brute_force_closest_pair(ps, 0); tb.append(time.perf_counter() - t0)
    print(n, d, "grid %.3f ms" % (min(ta) * 1e3), "brute %.3f ms" % (min(tb) * 1e3), (a.index_i, a.index_j) == (b.index_i, b.index_j))
