"""Trace one end-to-end C2 solve from pinned host memory (psg_closest_pair_f32)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
L = psg.lib()
n, d = 1 << 20, 128
hp = C.c_void_p()
psg._check(L.psg_host_alloc(n * d * 4, C.byref(hp)))
pi, pj = C.c_uint64(), C.c_uint64()
L.psg_gen_gauss_planted(2, n, d, 1e-3, hp.value, C.byref(pi), C.byref(pj))
for rep in range(4):
    out = psg._Pair()
    t0 = time.perf_counter()
    psg._check(L.psg_closest_pair_f32(hp.value, n, d, 10, 10.0, 1, 0, C.byref(out)))
    t1 = time.perf_counter()
    p = psg.last_profile()
    print(f"rep {rep}: wall {1e3*(t1-t0):.2f} ms, device span {p['total_ms']:.2f} ms, stages {p['stage_list']}", flush=True)
