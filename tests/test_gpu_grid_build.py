"""The counting grid build (psg_grid.cu: per-cell atomic counts, one scan,
atomic placement, deterministic per-cell ranking by original index): cells of
every size class — one point, up to 64 (per-position ranking), up to 8192
(one shared-memory bitonic run) and beyond (several sorted runs) — must give
the reference's answer, and key-range parts (which split SORTED POSITIONS)
must agree with the single solve, which only holds if the order inside every
cell is the deterministic (cell, index) order."""
import numpy as np
import pytest

from paper_1407_5609_b200 import sharded

pytestmark = pytest.mark.gpu


def big_cells(n, d, dup, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32)
    # `dup` copies of one point scattered through the index range, plus a
    # second, smaller group of 100 copies of another
    idx = rng.choice(n, dup + 100, replace=False)
    x[idx[:dup]] = x[idx[0]]
    x[idx[dup:]] = x[idx[dup]]
    return x, np.sort(idx[:dup]), np.sort(idx[dup:])


@pytest.mark.parametrize("n,d,dup", [(5000, 3, 70), (20000, 16, 3000), (40000, 3, 20000), (30000, 64, 9000)])
def test_big_cells_closest_pair(psg, n, d, dup):
    x, g1, g2 = big_cells(n, d, dup, n + d)
    got = psg.closest_pair(psg.PointSet.from_flat(x, d), 10, 10.0, 1, 0)
    first = min((g1[0], g1[1]), (g2[0], g2[1]))  # every duplicate pair has distance 0: lexicographic minimum
    assert (got.index_i, got.index_j, got.distance) == (first[0], first[1], 0.0)


@pytest.mark.parametrize("world", [2, 3])
def test_big_cells_parts_agree(psg, world):
    n, d = 40000, 3
    x, g1, g2 = big_cells(n, d, 12000, 7)
    x[g1[0]] += 1e-3  # no exact tie at the top: the minimum is a unique duplicate pair
    sets = [psg.PointSet.from_flat(x, d) for _ in range(world)]
    plans = [sharded.DevicePlan(s._device(), 10, 10.0, 1, 0) for s in sets]
    bound = min(plans[r].bootstrap(r, world) for r in range(world))
    parts = [plans[r].scan(r, world, bound) for r in range(world)]
    got = sharded.combine(parts, sharded.admissible_pairs(n, 0))
    one = psg.closest_pair(psg.PointSet.from_flat(x, d), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (one.index_i, one.index_j, one.distance)
    assert got.stats.admissible_pairs() == n * (n - 1) // 2


def test_big_cells_frnn_counts(psg, orc):
    n, d = 6000, 3
    x, _, _ = big_cells(n, d, 2000, 11)
    ps = psg.PointSet.from_flat(x, d)
    want = orc.brute_force_neighbors(x.astype(np.float64), 0.05, 0)
    got = psg.fixed_radius_neighbors(ps, 0.05, 10, 10.0, 1, 0, want_lists=False)
    assert (got.pair_count, got.pair_hash) == want


def test_repeated_solves_identical_stats(psg):
    # deterministic order => identical work and stats on every call
    x, _, _ = big_cells(50000, 8, 5000, 3)
    ps = psg.PointSet.from_flat(x, 8)
    a = psg.closest_pair(ps, 10, 10.0, 1, 0)
    b = psg.closest_pair(psg.PointSet.from_flat(x, 8), 10, 10.0, 1, 0)
    assert (a.index_i, a.index_j, a.distance, a.stats) == (b.index_i, b.index_j, b.distance, b.stats)
