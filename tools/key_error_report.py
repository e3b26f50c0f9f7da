"""Realised projection-key error vs the charged bound E (profiles/ evidence)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1407_5609_b200 as psg

rng = np.random.default_rng(5)
for d in (32, 64, 128, 256, 3, 16):
    for name, x in (("gauss", rng.standard_normal((20000, d))), ("offset", rng.standard_normal((20000, d)) * 1e3 + 5e3)):
        x = x.astype(np.float32)
        keys, dirs, E, scale = psg.debug_projection(psg.PointSet.from_flat(x, d), q=10, seed=7)
        exact = (x.astype(np.float64) * scale) @ dirs.astype(np.float64).T
        err = np.abs(keys - exact)
        print(f"d={d:4d} {name:7s} engine={'tcgen05' if d in (32,64,128,256) else 'cuda-core'} "
              f"E={E:.3e} max_err={err.max():.3e} ratio={err.max()/E:.4f} rms_err={np.sqrt((err**2).mean()):.3e}")
