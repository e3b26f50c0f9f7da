"""SURVEY §8(f)4 measurement: series text parsing (reference io.cpp vs the
parallel reader) and device point-set creation from a .psgb file vs from a
pageable numpy array.  Prints JSON lines."""
import json, os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1407_5609_b200 as psg


def best(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return out, min(ts)


tmp = tempfile.mkdtemp()
ref = oracle.reference()
s, _ = psg.gen.walk_motif(3, 1 << 20, 256)
series = s.astype(np.float64)
txt = os.path.join(tmp, "walk.txt")
psg.save_series_text(series, txt)
mine, t_mine = best(lambda: psg.load_series_text(txt))
line = {"io": "load_series text, 2^20 lines", "ours_s": t_mine, "threads": min(os.cpu_count() or 1, 16)}
if ref is not None:
    (theirs, rc, _), t_ref = best(lambda: ref.load_series(txt))
    line.update({"reference_s": t_ref, "identical": bool(rc == 0 and np.array_equal(theirs.view(np.uint64), mine.view(np.uint64)))})
print(json.dumps(line), flush=True)

pts, _ = psg.gen.gauss_planted(2, 1 << 20, 128)
bin_path = os.path.join(tmp, "c2.psgb")
psg.save_binary(pts, bin_path)
os.system(f"cat {bin_path} > /dev/null")  # page cache warm for both paths
_, t_file = best(lambda: psg.FilePointSet(bin_path))
def from_numpy():
    p = psg.PointSet.from_flat(pts, 128)
    p._device()
    return p
_, t_np = best(from_numpy)
print(json.dumps({"io": "C2 points (512 MiB) -> device point set", "psgb_file_s": t_file, "pageable_numpy_s": t_np}))
