"""C3 one-shot breakdown: window point set creation, first solve, later solves."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
s, (a, b) = psg.gen.walk_motif(3, 1 << 20, 256)
s64 = s.astype(np.float64)
psg.motif(s64, 256)  # warm-up (context, directions cache)
out = {}
for rep in range(2):
    t0 = time.perf_counter()
    ps = psg.PointSet.windows_of(s64, 256, znorm=True)
    ps._device()
    t1 = time.perf_counter()
    r = psg.closest_pair(ps, 10, 10.0, 1, 256)
    p1 = psg.last_profile()
    t2 = time.perf_counter()
    r2 = psg.closest_pair(ps, 10, 10.0, 1, 256)
    t3 = time.perf_counter()
    r3 = psg.closest_pair(ps, 10, 10.0, 1, 256)
    t4 = time.perf_counter()
    out[rep] = {"create_s": t1 - t0, "first_solve_s": t2 - t1, "second_s": t3 - t2, "third_s": t4 - t3,
                "first_stages": p1["stage_list"], "first_launches": p1["launches"]}
    ps.release()
t0 = time.perf_counter(); m = psg.motif(s64, 256); t1 = time.perf_counter()
out["one_shot_s"] = t1 - t0
out["one_shot_stages"] = psg.last_profile()["stage_list"]
print(json.dumps(out))
