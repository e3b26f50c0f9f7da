"""C4 list outputs one-shot from pageable points: the packed pair list vs the
upper-triangular CSR, best of 3 after a warm-up, with the stage times."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg
R = float.fromhex("0x1.902ce9269f6dp-7")
n = 1 << 22
cube = psg.gen.uniform(4, n, 3)
pin = psg.PinnedBuffer(20 * n)
poff, pcols = psg.PinnedBuffer(n + 1), psg.PinnedBuffer(20 * n, np.uint32)
for name, fn in [("list", lambda: psg.frnn_pairs(cube, R, out=pin.array)),
                 ("csr", lambda: psg.frnn_pairs_csr(cube, R, offsets=poff.array, cols=pcols.array)),
                 ("count", lambda: psg.frnn_pairs(cube, R, want_pairs=False))]:
    ts = []
    for k in range(4):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(name, round(min(ts[1:]) * 1e3, 3), "ms", psg.last_profile()["stage_list"], flush=True)
