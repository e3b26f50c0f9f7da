"""Per-rank work of the sharded closest-pair solve, measured part by part on ONE GPU.

    python tools/parts_c5.py [n] [W...]  > gpurun_out/parts_c5.jsonl

A rank of `closest_pair_sharded` (paper_1407_5609_b200/sharded.py) runs
plan_create (projection + grid, replicated on every rank), bootstrap(part),
one all-reduce MIN, scan(part, W, bound), one all-gather.  The parts never
wait on one another, so each part's device work can be timed alone here; the
W-rank wall time is bounded below by max over parts of (create + bootstrap +
scan) plus the two collectives (not measured: one GPU).  This is a work-balance
measurement, NOT a multi-GPU scaling measurement.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg  # noqa: E402
from paper_1407_5609_b200 import sharded  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
    worlds = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
    pts = psg.gen.mixture(5, n, 64, 1024, 0.05)
    ps = psg.PointSet.from_flat(pts, 64)
    adm = sharded.admissible_pairs(n, 0)
    psg.closest_pair(ps, 10, 10.0, 1, 0)  # warm-up (allocations, learned engine choice)
    for W in worlds:
        t0 = time.perf_counter()
        plan = sharded.DevicePlan(ps._device(), 10, 10.0, 1, 0)
        t_create = time.perf_counter() - t0
        boots, t_boot = [], []
        for part in range(W):
            t0 = time.perf_counter()
            boots.append(plan.bootstrap(part, W))
            t_boot.append(time.perf_counter() - t0)
        bound = min(boots)
        res, t_scan = [], []
        for part in range(W):
            t0 = time.perf_counter()
            res.append(plan.scan(part, W, bound))
            t_scan.append(time.perf_counter() - t0)
        plan.close()
        r = sharded.combine(res, adm)
        per_rank = [t_create + b + s for b, s in zip(t_boot, t_scan)]
        print(json.dumps({"n": n, "W": W, "create_s": t_create, "bootstrap_s": t_boot, "scan_s": t_scan,
                          "per_rank_s": per_rank, "max_rank_s": max(per_rank),
                          "answer": [r.index_i, r.index_j, r.distance]}), flush=True)


if __name__ == "__main__":
    main()
