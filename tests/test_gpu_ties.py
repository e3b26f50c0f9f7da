"""Exact ties at scale and repeated solves on one point set.

The reference breaks distance ties by the lexicographically smallest (i, j)
(refscan.cpp:118-126) and returns an answer for any input with an admissible
pair.  Runs of identical points put every pair of the run inside the FP64
recheck band at once (a flat-lined series, zero padding, lattice data):
these cases hold far more band pairs than the candidate list, so they go
through the inline 128-bit (distance, i, j) minimum of record()
(psg_scan.cuh).  The expected answer is computed directly: among duplicate
points the distance is exactly 0 and the winner is the smallest admissible
(i, j) over the duplicate indices.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def first_admissible(idx, zone):
    """Lexicographically smallest (i, j), i < j from sorted idx with j - i >= zone."""
    z = max(zone, 1)
    for i in idx:
        k = np.searchsorted(idx, i + z)
        if k < len(idx):
            return int(i), int(idx[k])
    return None


def planted_duplicates(n, dup, d, seed):
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, d)).astype(np.float32)
    idx = np.sort(rng.choice(n, dup, replace=False))
    pts[idx] = pts[idx[0]]
    return pts, idx


@pytest.mark.parametrize("zone", [0, 5])
def test_hundred_thousand_duplicates(psg, zone):
    """100k copies of one point among 120k: about 5e9 band pairs (the advisor's
    ~92k-duplicate counter wrap and the ~23k overflow both sit below this)."""
    pts, idx = planted_duplicates(120_000, 100_000, 8, 11)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 8), 10, 10.0, 1, zone)
    assert (got.index_i, got.index_j) == first_admissible(idx, zone)
    assert got.distance == 0.0


def test_all_points_identical(psg):
    n = 30_000
    pts = np.full((n, 4), 0.25, dtype=np.float32)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 4), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (0, 1, 0.0)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 4), 10, 10.0, 1, 7)
    assert (got.index_i, got.index_j, got.distance) == (0, 7, 0.0)


def test_flat_series_motif(psg):
    """A z-normalised series with a constant stretch: every window inside the
    stretch normalises to the zero vector (sigma == 0 guard), so they all tie."""
    rng = np.random.default_rng(5)
    s = np.cumsum(rng.standard_normal(40_000))
    s[10_000:22_000] = 3.0
    got = psg.motif(s, 64, znorm=True)
    # windows fully inside [10000, 22000): start 10000 .. 21936; zone = 64
    assert (got.index_i, got.index_j, got.distance) == (10_000, 10_064, 0.0)


@pytest.mark.parametrize("q", [1, 10])
def test_repeated_solves_one_pointset_past_list_capacity(psg, orc, q):
    """Solves 2 and 3 run on the same PointSet after solve 1 outgrew the
    candidate list (the list is reallocated and a captured graph holding the
    old buffers must not be replayed); all three answers are the oracle's."""
    pts, idx = planted_duplicates(50_000, 2_000, 16, 3)  # ~2e6 band pairs > 65536
    ps = psg.PointSet.from_flat(pts, 16)
    want = first_admissible(idx, 0)
    for _ in range(3):
        got = psg.closest_pair(ps, q, 10.0, 1, 0)
        assert (got.index_i, got.index_j, got.distance) == (*want, 0.0)
    # another point set created after the growth must not be written by a
    # stale replay of the first one's graph
    other = planted_duplicates(50_000, 2, 16, 4)
    ps2 = psg.PointSet.from_flat(other[0], 16)
    got = psg.closest_pair(ps, q, 10.0, 1, 0)
    assert (got.index_i, got.index_j) == want
    bf = psg.brute_force_closest_pair(ps2, 0)
    assert (bf.index_i, bf.index_j) == tuple(int(x) for x in other[1])


def test_duplicates_near_not_exact(psg, orc):
    """3000 points on a small lattice around one point: hundreds of exact
    duplicate pairs and many equal nonzero distances; the oracle's brute force
    over those 3000 points (every other point is far away) is the answer."""
    rng = np.random.default_rng(9)
    n, d = 40_000, 8
    pts = rng.standard_normal((n, d)).astype(np.float32)
    idx = np.sort(rng.choice(n, 3000, replace=False))
    base = pts[idx[0]].copy()
    # quantised offsets: many exact distance ties between different pairs
    pts[idx] = base + (rng.integers(0, 3, (3000, d)) * np.float32(2.0 ** -10)).astype(np.float32)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, d), 10, 10.0, 1, 0)
    sub = pts[idx].astype(np.float64)
    want = orc.brute_force_closest_pair(sub, 0)
    assert got.distance == want.distance
    assert (got.index_i, got.index_j) == (int(idx[want.index_i]), int(idx[want.index_j]))


@pytest.mark.parametrize("q", [1, 10])
def test_sparse_engine_exact_rescan(psg, q):
    """10k duplicates among 120k points: ~5e7 band pairs, more than the
    sparse engines' longest candidate list (2^24), so the scan is redone with
    every band pair evaluated inline in FP64 (k_grid_scan2 / k_scan <kExact>)."""
    pts, idx = planted_duplicates(120_000, 10_000, 8, 21)
    ps = psg.PointSet.from_flat(pts, 8)
    for _ in range(2):
        got = psg.closest_pair(ps, q, 10.0, 1, 3)
        assert (got.index_i, got.index_j, got.distance) == (*first_admissible(idx, 3), 0.0)
        assert psg.last_profile()["inline_fp64"] > 1 << 24
