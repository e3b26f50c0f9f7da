"""Step through the sharded plan API on the C2 recipe at several n (diagnostics)."""
import ctypes as C, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg
from paper_1407_5609_b200 import sharded
L = psg.lib()
for logn in [int(a) for a in sys.argv[1:]] or [16, 18, 20]:
    n = 1 << logn
    pts, planted = psg.gen.gauss_planted(2, n, 128)
    ps = psg.PointSet.from_flat(pts, 128)
    plan = sharded.DevicePlan(ps._device(), 10, 10.0, 1, 0)
    b = plan.bootstrap(0, 1)
    prof = psg.last_profile()
    print(f"n=2^{logn} planted={sorted(planted)} bound_s32={b:.6g} width={prof['bootstrap_width']} "
          f"boot_ms={prof['bootstrap_kernel_ms']:.3f}", flush=True)
    try:
        r = plan.scan(0, 1, b)
        prof = psg.last_profile()
        print("  result", r, flush=True)
        print("  prof", {k: v for k, v in prof.items() if k != 'stage_list'}, flush=True)
    except Exception as e:
        print("  FAILED", e, flush=True)
    plan.close()
