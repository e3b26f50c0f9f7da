"""C2 device solve time under one grid setting (PSG_BOXSD / PSG_OCC from the env).

    for b in 3 2.5 2; do PSG_BOXSD=$b python tools/sweep_grid.py; done
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_5609_b200 as psg  # noqa: E402

pts, planted = psg.gen.gauss_planted(2, 1 << 20, 128)
ps = psg.PointSet.from_flat(pts, 128)
best = None
for _ in range(6):
    r = psg.closest_pair(ps, 10, 10.0, 1, 0)
    p = psg.last_profile()
    if best is None or p["total_ms"] < best["total_ms"]:
        best = p
assert (r.index_i, r.index_j) == tuple(sorted(planted))
keep = {k: best[k] for k in ("total_ms", "scan_kernel_ms", "bootstrap_kernel_ms", "project_kernel_ms",
                             "window_pairs", "lb_survivors") if k in best}
print(json.dumps({"box_sd": os.environ.get("PSG_BOXSD"), "occ": os.environ.get("PSG_OCC"), **keep}))
