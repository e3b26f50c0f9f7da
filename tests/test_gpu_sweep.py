"""Seeded sweep of shapes and data families: every engine path (CUDA-core and
tcgen05 projections, sparse grid, window-free dense cell pairs with tensor-core
Gram tiles, regrids, exclusion zones) against the C oracle's FP64 brute force
(refscan.cpp:134-157): indices and distance must be identical.

Dimensions cover both projection engines (d < 32 and d in {32, 64, 128, 256},
plus irregular d), n covers tiny sets (n = 2, 3) through a few thousand, and
the data families include exact duplicates, integer lattices full of exact
ties, tight clusters (the dense engine), wildly different row scales and
FP64 values that are not float-representable.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def family(name, rng, n, d):
    if name == "gauss":
        return rng.standard_normal((n, d))
    if name == "uniform_f32":
        return rng.random((n, d), dtype=np.float32)
    if name == "clusters":
        c = rng.uniform(-1, 1, (max(1, n // 50), d))
        return c[rng.integers(0, len(c), n)] + rng.normal(0, 0.01, (n, d))
    if name == "lattice_ties":
        return rng.integers(0, 4, (n, d)).astype(np.float64)
    if name == "duplicates":
        x = rng.standard_normal((n, d))
        k = max(1, n // 10)
        x[rng.integers(0, n, k)] = x[rng.integers(0, n, k)]
        return x
    if name == "row_scales":
        return rng.standard_normal((n, d)) * np.exp(rng.uniform(-8, 8, (n, 1)))
    if name == "not_float":
        return rng.standard_normal((n, d)) * (1 + 1e-12)
    raise ValueError(name)


CASES = []
_rng = np.random.default_rng(20261019)
for d in (1, 2, 3, 5, 16, 31, 32, 33, 64, 100, 128, 200, 256):
    for fam in ("gauss", "uniform_f32", "clusters", "lattice_ties", "duplicates", "row_scales", "not_float"):
        n = int(_rng.choice([2, 3, 17, 400, 2500]))
        zone = int(_rng.choice([0, 0, 1, 3]))
        CASES.append((d, fam, n, zone, int(_rng.integers(1, 1 << 30)), int(_rng.choice([1, 4, 10]))))


@pytest.mark.parametrize("d,fam,n,zone,seed,q", CASES, ids=[f"d{c[0]}-{c[1]}-n{c[2]}-z{c[3]}-q{c[5]}" for c in CASES])
def test_closest_pair_matches_oracle(psg, orc, d, fam, n, zone, seed, q):
    rng = np.random.default_rng(seed)
    pts = family(fam, rng, n, d)
    if zone >= n:
        zone = 0
    q = min(q, n)  # refscan.cpp:34: q > n is the reference's invalid_argument
    want = orc.brute_force_closest_pair(np.asarray(pts, dtype=np.float64), zone)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, d), q, 10.0, seed, zone)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


# Larger sets: the grid's regrid path, the dense engine (tensor-core Gram tiles
# for d in {32, 64}, CUDA-core tiles otherwise) and the FRNN engine, against
# the device all-pairs engine (itself pinned to the oracle above and in
# test_gpu_parity.py).
BIG = [(d, fam, n) for d in (3, 16, 32, 64, 128) for fam in ("clusters", "gauss", "lattice_ties") for n in (30_000,)]


@pytest.mark.parametrize("d,fam,n", BIG, ids=[f"d{d}-{fam}-n{n}" for d, fam, n in BIG])
def test_closest_pair_large_matches_device_brute_force(psg, d, fam, n):
    rng = np.random.default_rng(d * 1000 + n + len(fam))
    pts = family(fam, rng, n, d).astype(np.float32)
    ps = psg.PointSet.from_flat(pts, d)
    got = psg.closest_pair(ps, 10, 10.0, 7, 0)
    bf = psg.brute_force_closest_pair(ps, 0)
    assert (got.index_i, got.index_j, got.distance) == (bf.index_i, bf.index_j, bf.distance)


@pytest.mark.parametrize("d,fam", [(2, "clusters"), (3, "gauss"), (7, "uniform_f32"), (32, "clusters")])
def test_fixed_radius_large_matches_device_brute_force(psg, d, fam):
    rng = np.random.default_rng(d + 99)
    pts = family(fam, rng, 20_000, d).astype(np.float32)
    ps = psg.PointSet.from_flat(pts, d)
    bf = psg.brute_force_closest_pair(ps, 0)
    radius = bf.distance * 40.0 if bf.distance > 0 else 1e-3
    got = psg.fixed_radius_neighbors(ps, radius, 10, 10.0, 3, 0, want_lists=False)
    want = psg.brute_force_neighbors(ps, radius, 0)
    cnt = sum(len(l) for l in want) // 2
    assert got.pair_count == cnt


# The d <= 4 cell scan's variants (list / count, d = 4, exclusion zone): the
# count, hash and sorted pair list against the device brute force (a13), and
# the count + hash run against the list run.
@pytest.mark.parametrize("d,zone", [(1, 0), (2, 7), (3, 0), (3, 5), (4, 0), (4, 9)])
def test_fixed_radius_cell_scan_variants(psg, d, zone):
    rng = np.random.default_rng(100 + 10 * d + zone)
    n = 30_000
    pts = rng.random((n, d)).astype(np.float32)
    ps = psg.PointSet.from_flat(pts, d)
    radius = float((24.0 / n) ** (1.0 / d)) * 0.6  # tens of neighbours per point
    want = psg.brute_force_neighbors(ps, radius, zone)
    lists = psg.fixed_radius_neighbors(ps, radius, 10, 10.0, 3, zone)
    assert [list(map(int, l)) for l in lists.neighbors] == [list(map(int, l)) for l in want]
    counted = psg.fixed_radius_neighbors(ps, radius, 10, 10.0, 3, zone, want_lists=False)
    assert (counted.pair_count, counted.pair_hash) == (lists.pair_count, lists.pair_hash)
    assert counted.pair_count == sum(len(l) for l in want) // 2 > 0
