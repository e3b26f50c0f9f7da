"""Per-call wall time of resident C2 solves (ctypes straight into the C ABI)
against the graph's device total, to size the host overhead per call."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
L = psg.lib()
pts, _ = psg.gen.gauss_planted(2, 1 << 20, 128)
ps = psg.PointSet.from_flat(pts, 128)
dev = ps._device()
out = psg._Pair()
psg.set_graph_profiling(0)
for _ in range(5):
    psg._check(L.psg_closest_pair_ps(dev, 10, 10.0, 1, 0, C.byref(out)))
tot = []
t0 = time.perf_counter()
for _ in range(200):
    L.psg_closest_pair_ps(dev, 10, 10.0, 1, 0, C.byref(out))
    tot.append(psg.last_profile()["total_ms"])
wall = (time.perf_counter() - t0) / 200
tot.sort()
print("wall per call %.1f us, device span median %.1f us" % (wall * 1e6, tot[len(tot) // 2] * 1e3))
