"""Generate tests/golden/reference_golden.json from the UNMODIFIED reference.

Runs in the dev container only (needs oracle/_ref/libpairscan_ref.so, built by
oracle/Makefile from /root/reference/proj/core/src).  The JSON is committed so
tests on any machine can pin the oracle restatement without the reference.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def gauss(ref, seed, n, d):
    return ref.gaussian_stream(seed, 0.0, 1.0, n * d).reshape(n, d)


def main():
    oracle.build()
    ref = oracle.reference()
    assert ref is not None, "oracle/_ref not built"
    g = {"source": "unmodified reference core (/root/reference/proj/core/src) via oracle/ref_capi.cpp"}
    # rng.cpp
    g["rng_stream"] = {str(s): [str(v) for v in ref.rng_stream(s, 16)] for s in (0, 1, 5489, 12345)}
    g["gaussian_stream"] = {str(s): ref.gaussian_stream(s, 0.0, 1.0, 16).tolist() for s in (1, 7, 77)}
    g["uniform_below"] = {f"{s}:{b}": [int(v) for v in ref.uniform_below_stream(s, b, 16)]
                          for s, b in ((1, 10), (2, 1000), (3, 1 << 40), (4, 7))}
    g["sample_without_replacement"] = {f"{s}:{n}:{k}": [int(v) for v in ref.sample_without_replacement(s, n, k)]
                                       for s, n, k in ((1, 100, 10), (3, 60, 7), (9, 5, 5))}
    g["mix_seed"] = {str(x): str(ref.mix_seed(x)) for x in (0, 1, 42, (1 << 63) + 5)}
    g["derive_seed"] = {f"{b}:{s}": str(ref.derive_seed(b, s)) for b, s in ((1, 0), (2, 1), (3, 1000), (5, 1001))}
    # datagen.cpp
    g["random_walk"] = {f"{n}:{s}": ref.gen_random_walk(n, s).tolist() for n, s in ((5, 7), (12, 1))}
    # refscan.cpp closest pair (brute force and the MPR engine itself)
    cases = {}
    for name, (kind, args) in {
        "walk400_11_l24": ("windows", (400, 11, 24)),
        "walk2000_1_l64": ("windows", (2000, 1, 64)),
        "walk240_5_l8": ("windows", (240, 5, 8)),
        "gauss77_150x4": ("gauss", (77, 150, 4)),
        "gauss7_1000x16": ("gauss", (7, 1000, 16)),
    }.items():
        if kind == "windows":
            n, s, l = args
            w = ref.gen_random_walk(n, s)
            pts = np.ascontiguousarray(np.lib.stride_tricks.sliding_window_view(w, l))
            zone = l
        else:
            s, n, d = args
            pts = gauss(ref, s, n, d)
            zone = 0
        b = ref.brute_force_closest_pair(pts, zone)
        m = ref.closest_pair(pts, 10, 10.0, 1, zone)
        cases[name] = {"zone": zone, "brute": [b.index_i, b.index_j, b.distance, b.pairs_examined],
                       "mpr": [m.index_i, m.index_j, m.distance]}
    g["closest_pair"] = cases
    # C1 at full size (16384 x 2, SURVEY §8(d) recipe)
    orc = oracle.port()
    c1 = orc.gen_uniform(1, 16384, 2).astype(np.float64)
    b = ref.brute_force_closest_pair(c1, 0)
    g["c1_full"] = [b.index_i, b.index_j, b.distance]
    # FRNN: count + hash + the pair list for small sets; boundary fixture
    fr = {}
    for s, n, d in ((31, 120, 3), (11, 200, 5)):
        pts = gauss(ref, s, n, d)
        for R in (0.35, 1.2):
            for zone in (0, 2):
                cnt, h, pairs = ref.brute_force_neighbors(pts, R, zone, lists=True)
                mp = ref.fixed_radius_neighbors(pts, R, 8, 10.0, 9, zone)
                fr[f"{s}:{n}x{d}:{R}:{zone}"] = {"count": cnt, "hash": str(h), "pairs": [str(int(v)) for v in pairs],
                                                  "mpr_count": mp["count"], "mpr_hash": str(mp["hash"])}
    g["frnn"] = fr
    # build_reference_set (test_refscan.cpp:42-69 shape)
    pts = gauss(ref, 11, 60, 5)
    ri, refs, table, order = ref.build_reference_set(pts, 7, 10.0, 3)
    g["reference_set_11_60x5_q7_f10_s3"] = {"ref_indices": [int(v) for v in ri], "references": refs.ravel().tolist(),
                                             "dist_table": table.ravel().tolist(), "order": [int(v) for v in order]}
    # metrics
    x, y = ref.gaussian_stream(23, 0, 1, 16), ref.gaussian_stream(24, 0, 1, 16)
    dfull = ref.euclidean(x, y)
    g["metrics"] = {"x": x.tolist(), "y": y.tolist(), "euclidean": dfull,
                    "early_abandon": {str(t): ref.early_abandon(x, y, t) for t in (0.0, dfull * 0.5, dfull, dfull * 1.5)},
                    "three_four_five": [ref.early_abandon([0, 0], [3, 4], 5.0), ref.early_abandon([0, 0], [3, 4], 4.999)]}
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")
    with open(out, "w") as fh:
        json.dump(g, fh, indent=1)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
