"""Back-to-back vs idle-separated 50 MB pageable uploads (is the first transfer
after idle slow?)."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
L = psg.lib()
cube = np.ascontiguousarray(psg.gen.uniform(4, 1 << 22, 3), dtype=np.float32)
def once():
    out = C.c_void_p()
    t0 = time.perf_counter()
    psg._check(L.psg_pointset_from_f32(cube.ctypes.data, cube.shape[0], 3, 0, C.byref(out)))
    t = time.perf_counter() - t0
    L.psg_pointset_free(out)
    return round(t * 1e3, 2)
once()
print("back-to-back", [once() for _ in range(6)])
r = []
for _ in range(4):
    time.sleep(0.2)
    r.append(once())
print("after 200 ms idle", r)
