"""Point-set creation from pageable host memory through the C ABI
(psg_pointset_from_f32/_f64: upload + validation pass): C4 (50 MB f32) and C2
(1 GiB f64); best of 3 after one warm-up."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
L = psg.lib()
cube = np.ascontiguousarray(psg.gen.uniform(4, 1 << 22, 3), dtype=np.float32)
big = np.random.default_rng(1).standard_normal((1 << 20, 128))
for name, arr, fn in [("c4 f32 50MB", cube, L.psg_pointset_from_f32), ("c2 f64 1GiB", big, L.psg_pointset_from_f64)]:
    ts = []
    for k in range(4):
        out = C.c_void_p()
        t0 = time.perf_counter()
        psg._check(fn(arr.ctypes.data, arr.shape[0], arr.shape[1], 0, C.byref(out)))
        ts.append(time.perf_counter() - t0)
        L.psg_pointset_free(out)
    print(name, "%.2f ms" % (min(ts[1:]) * 1e3), [round(t * 1e3, 2) for t in ts], flush=True)
