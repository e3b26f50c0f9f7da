"""Time every BASELINE.json config once at full size (after one warm-up solve).

    python tools/bench_configs.py [c1 c2 c3 c4 c5] > gpurun_out/configs.jsonl

Prints one JSON line per config: device-resident solve time (CUDA events on
the library stream), the answer, and the profile counters.
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1407_5609_b200 as psg  # noqa: E402

R_C4 = float.fromhex("0x1.902ce9269f6dp-7")


def timed(fn, reps=3):
    fn()  # warm-up (allocations, graph capture)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return out, min(ts), psg.last_profile()


def main(which):
    res = []
    if "c1" in which:
        pts = psg.gen.uniform(1, 16384, 2)
        ps = psg.PointSet.from_flat(pts, 2)
        r, t, p = timed(lambda: psg.closest_pair(ps, 10, 10.0, 1, 0))
        res.append({"config": "C1 CPP n=16384 d=2", "solve_s": t, "answer": [r.index_i, r.index_j, r.distance],
                    "device_ms": p["total_ms"], "window_pairs": p["window_pairs"]})
    if "c2" in which:
        pts, planted = psg.gen.gauss_planted(2, 1 << 20, 128)
        ps = psg.PointSet.from_flat(pts, 128)
        r, t, p = timed(lambda: psg.closest_pair(ps, 10, 10.0, 1, 0))
        res.append({"config": "C2 CPP n=2^20 d=128", "solve_s": t, "answer": [r.index_i, r.index_j, r.distance],
                    "planted": sorted(planted), "device_ms": p["total_ms"], "window_pairs": p["window_pairs"]})
    if "c3" in which:
        s, (a, b) = psg.gen.walk_motif(3, 1 << 20, 256)
        ps = psg.PointSet.windows_of(s.astype(np.float64), 256, znorm=True)
        r, t, p = timed(lambda: psg.closest_pair(ps, 10, 10.0, 1, 256))
        res.append({"config": "C3 TSMM N=2^20 l=256 znorm zone=256", "solve_s": t,
                    "answer": [r.index_i, r.index_j, r.distance], "planted": sorted((a, b)),
                    "device_ms": p["total_ms"], "window_pairs": p["window_pairs"]})
    if "c4" in which:
        cube = psg.gen.uniform(4, 1 << 22, 3)
        pc = psg.PointSet.from_flat(cube, 3)
        nr, t, p = timed(lambda: psg.fixed_radius_neighbors(pc, R_C4, 10, 10.0, 1, 0, want_lists=False))
        cnt, h = nr.pair_count, nr.pair_hash
        res.append({"config": "C4 FRNN n=2^22 d=3 R=cbrt(3*32/(4 pi n)) (resident, count+hash)", "solve_s": t,
                    "pairs": cnt, "hash": h, "device_ms": p["total_ms"], "candidates": p["window_pairs"],
                    "stages": p["stage_list"]})
        (pairs, cnt1, h1), t1, p1 = timed(lambda: psg.frnn_pairs(cube, R_C4, want_pairs=False))
        res.append({"config": "C4 FRNN one-shot from host (H2D of pageable points included)", "solve_s": t1,
                    "pairs": cnt1, "hash": h1})
        pinned = psg.PinnedBuffer(20 * len(cube))
        (pairs, cnt2, h2), t2, p2 = timed(lambda: psg.frnn_pairs(cube, R_C4, want_pairs=True, out=pinned.array), reps=2)
        ok = bool(np.all(pairs[1:] > pairs[:-1])) and cnt2 == cnt
        res.append({"config": "C4 FRNN sorted pair list -> pinned host", "solve_s": t2, "pairs": cnt2,
                    "device_ms": p2["total_ms"], "sorted_unique": ok, "stages": p2["stage_list"]})
    if "c5" in which:
        n = int(os.environ.get("C5_N", 1 << 24))
        pts = psg.gen.mixture(5, n, 64, 1024, 0.05)
        ps = psg.PointSet.from_flat(pts, 64)
        r, t, p = timed(lambda: psg.closest_pair(ps, 10, 10.0, 1, 0), reps=1)
        res.append({"config": f"C5 CPP n={n} d=64 mixture", "solve_s": t, "answer": [r.index_i, r.index_j, r.distance],
                    "device_ms": p["total_ms"], "window_pairs": p["window_pairs"], "lb_survivors": p["lb_survivors"]})
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"c1", "c2", "c3", "c4", "c5"})
