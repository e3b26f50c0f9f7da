"""CPU: pin the oracle restatement (oracle/oracle.c) to the reference.

Against (a) golden vectors produced by the unmodified reference
(tests/golden/reference_golden.json, made by tests/golden/make_golden.py),
(b) the reference library itself when oracle/_ref is built (dev container),
(c) the reference's own unit-test identities re-expressed (test_metrics.cpp,
test_refscan.cpp, test_datagen.cpp) and the C++ standard's mt19937_64 check.
"""
import json
import os

import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def windows(series, length):
    return np.ascontiguousarray(sliding_window_view(np.asarray(series, dtype=np.float64), length))


def gauss(orc, seed, n, d):
    return orc.gaussian_stream(seed, 0.0, 1.0, n * d).reshape(n, d)


# --- rng.cpp ---------------------------------------------------------------------
def test_mt19937_64_standard_check_value(orc):
    # [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert int(orc.rng_stream(5489, 10000)[-1]) == 9981545732273789042


def test_rng_streams_match_reference_golden(orc):
    for seed, vals in GOLD["rng_stream"].items():
        assert [str(v) for v in orc.rng_stream(int(seed), 16)] == vals
    for seed, vals in GOLD["gaussian_stream"].items():
        assert orc.gaussian_stream(int(seed), 0.0, 1.0, 16).tolist() == vals  # bit-exact
    for key, vals in GOLD["uniform_below"].items():
        s, b = map(int, key.split(":"))
        assert orc.uniform_below_stream(s, b, 16).tolist() == vals
    for key, vals in GOLD["sample_without_replacement"].items():
        s, n, k = map(int, key.split(":"))
        assert orc.sample_without_replacement(s, n, k).tolist() == vals
    for x, v in GOLD["mix_seed"].items():
        assert str(orc.mix_seed(int(x))) == v
    for key, v in GOLD["derive_seed"].items():
        b, s = map(int, key.split(":"))
        assert str(orc.derive_seed(b, s)) == v


def test_sample_without_replacement_rejects_k_over_n(orc):
    with pytest.raises(ValueError):
        orc.sample_without_replacement(1, 3, 4)


# --- datagen.cpp / test_datagen.cpp -------------------------------------------------
def test_random_walk_golden_and_identities(orc):
    for key, vals in GOLD["random_walk"].items():
        n, s = map(int, key.split(":"))
        assert orc.gen_random_walk(n, s).tolist() == vals
    w = orc.gen_random_walk(1000, 3)
    assert w[0] == 0.0 and np.array_equal(w, orc.gen_random_walk(1000, 3))  # test_datagen.cpp:30-38
    # stddev linearity (test_datagen.cpp:40-48): steps scale exactly with sd
    a, b = orc.gen_random_walk(50, 9, 1.0), orc.gen_random_walk(50, 9, 2.0)
    assert np.allclose(np.diff(b), 2.0 * np.diff(a), rtol=0, atol=1e-12)
    with pytest.raises(ValueError):
        orc.gen_random_walk(0, 1)


# --- metrics.cpp / test_metrics.cpp -----------------------------------------------------
def test_euclidean_and_early_abandon_golden(orc):
    m = GOLD["metrics"]
    x, y = np.array(m["x"]), np.array(m["y"])
    assert orc.euclidean(x, y) == m["euclidean"]
    for t, want in m["early_abandon"].items():
        assert orc.early_abandon(x, y, float(t)) == want
    assert [orc.early_abandon([0, 0], [3, 4], 5.0), orc.early_abandon([0, 0], [3, 4], 4.999)] == m["three_four_five"]


def test_early_abandon_bitwise_consistent(orc):
    # test_metrics.cpp:65-80
    for t in range(300):
        x, y = gauss(orc, 1000 + t, 2, 16)
        d = orc.euclidean(x, y)
        for thr in (0.0, d * 0.5, d, d * 1.5):
            r = orc.early_abandon(x, y, thr)
            if d <= thr:
                assert r == d
            if r is None:
                assert d > thr


def test_triangle_lower_bound(orc):
    # test_metrics.cpp:53-63 and refscan reference_bound sign (test_refscan.cpp:71-83)
    for t in range(200):
        r, x, y = gauss(orc, 5000 + t, 3, 8)
        b = orc.reference_bound(r, x, y)
        assert b == orc.euclidean(r, x) - orc.euclidean(r, y)
        assert b == -orc.reference_bound(r, y, x)
        assert abs(b) <= orc.euclidean(x, y) + 1e-9


# --- refscan.cpp ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", sorted(GOLD["closest_pair"]))
def test_brute_force_closest_pair_matches_reference(orc, name):
    case = GOLD["closest_pair"][name]
    if name.startswith("walk"):
        parts = name.split("_")
        n, s, l = int(parts[0][4:]), int(parts[1]), int(parts[2][1:])
        pts = windows(orc.gen_random_walk(n, s), l)
    else:
        parts = name.split("_")
        s = int(parts[0][5:])
        n, d = map(int, parts[1].split("x"))
        pts = gauss(orc, s, n, d)
    got = orc.brute_force_closest_pair(pts, case["zone"])
    assert [got.index_i, got.index_j, got.distance, got.pairs_examined] == case["brute"]
    assert case["mpr"] == case["brute"][:3]  # the reference's own engine agrees


def test_c1_full_size_matches_reference(orc):
    pts = orc.gen_uniform(1, 16384, 2)
    got = orc.brute_force_closest_pair(pts, 0)
    assert [got.index_i, got.index_j, got.distance] == GOLD["c1_full"]


def test_exclusion_zone_fixture(orc):
    # test_refscan.cpp:143-157
    pts = np.array([0.0, 0.0005, 10.0, 30.0, 50.0, 10.1]).reshape(-1, 1)
    for zone in (0, 1):
        r = orc.brute_force_closest_pair(pts, zone)
        assert (r.index_i, r.index_j) == (0, 1)
    r = orc.brute_force_closest_pair(pts, 2)
    assert (r.index_i, r.index_j) == (2, 5) and r.distance == pytest.approx(0.1)
    with pytest.raises(ValueError, match="no admissible pair"):
        orc.brute_force_closest_pair(pts, 6)
    with pytest.raises(ValueError, match="at least 2 points"):
        orc.brute_force_closest_pair(pts[:1], 0)


@pytest.mark.parametrize("key", sorted(GOLD["frnn"]))
def test_brute_force_neighbors_match_reference(orc, key):
    s, nd, R, zone = key.split(":")
    n, d = map(int, nd.split("x"))
    pts = gauss(orc, int(s), n, d)
    cnt, h, pairs = orc.brute_force_neighbors(pts, float(R), int(zone), lists=True)
    want = GOLD["frnn"][key]
    assert (cnt, str(h)) == (want["count"], want["hash"])
    assert [str(int(v)) for v in pairs] == want["pairs"]
    assert (want["mpr_count"], want["mpr_hash"]) == (want["count"], want["hash"])  # reference MPR == brute


def test_frnn_boundary_fixture(orc):
    # test_refscan.cpp:159-167: {0,1,2,3.5}, R=1 -> (0,1), (1,2)
    pts = np.array([0.0, 1.0, 2.0, 3.5]).reshape(-1, 1)
    cnt, h, pairs = orc.brute_force_neighbors(pts, 1.0, 0, lists=True)
    assert cnt == 2 and [int(v) for v in pairs] == [(0 << 32) | 1, (1 << 32) | 2]


@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_frnn_grid_restatement_equals_brute_force(orc, d):
    pts = orc.gen_uniform(40 + d, 3000, d)
    R = 0.08 if d <= 3 else 0.3
    for zone in (0, 3):
        assert orc.frnn_grid(pts, R, zone) == orc.brute_force_neighbors(pts.astype(np.float64), R, zone)


def test_build_reference_set_matches_reference(orc):
    g = GOLD["reference_set_11_60x5_q7_f10_s3"]
    pts = gauss(orc, 11, 60, 5)
    ri, refs, table, order = orc.build_reference_set(pts, 7, 10.0, 3)
    assert ri.tolist() == g["ref_indices"]
    assert refs.ravel().tolist() == g["references"]
    assert table.ravel().tolist() == g["dist_table"]
    assert order.tolist() == g["order"]


def test_znorm_windows_definition(orc):
    s = orc.gen_random_walk(300, 4)
    z = orc.znorm_windows(s, 16)
    w = windows(s, 16)
    mu = w.mean(axis=1, keepdims=True)
    sd = w.std(axis=1, keepdims=True)
    assert np.allclose(z, (w - mu) / sd, atol=1e-12)
    flat = np.concatenate([np.full(20, 3.0), s[:50]])
    zf = orc.znorm_windows(flat, 8)
    assert np.all(zf[0] == 0.0)  # sigma == 0 -> zeros
    a = orc.motif_brute_znorm(s, 16, 16)
    b = orc.brute_force_closest_pair(z, 16)
    assert (a.index_i, a.index_j, a.distance) == (b.index_i, b.index_j, b.distance)


# --- live cross-check against the reference build (dev container only) --------------------
def test_port_matches_live_reference_on_random_cases(orc, ref):
    rng = np.random.default_rng(0)
    for t in range(20):
        n, d = int(rng.integers(2, 80)), int(rng.integers(1, 6))
        pts = rng.normal(size=(n, d))
        zone = int(rng.integers(0, 4)) if n > 4 else 0
        try:
            want = ref.brute_force_closest_pair(pts, zone)
        except Exception:
            with pytest.raises(ValueError):
                orc.brute_force_closest_pair(pts, zone)
            continue
        got = orc.brute_force_closest_pair(pts, zone)
        assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)
        R = float(rng.uniform(0.2, 2.0))
        assert orc.brute_force_neighbors(pts, R, zone) == ref.brute_force_neighbors(pts, R, zone)
