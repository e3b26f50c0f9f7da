"""GPU: the key-range sharded solve (psg_cpp_plan_*, paper_1407_5609_b200/
sharded.py) with W parts run on one device, one point set per emulated rank
(every rank of a real run owns its copy), combined exactly as the NCCL path
combines them: the bound is the MIN over parts' bootstraps, the answer the
lexicographic minimum of the parts' results.  Must equal the single solve and
the brute force, for the grid engine, the window-z-norm motif and the dense
cell-pair engine (clustered data, tensor-core Gram tiles, strips round-robin
over parts)."""
import numpy as np
import pytest

from paper_1407_5609_b200 import sharded

pytestmark = pytest.mark.gpu


def run_parts(psg, make_points, world, q=10, f=10.0, seed=1, zone=0):
    sets = [make_points() for _ in range(world)]
    plans = [sharded.DevicePlan(ps._device(), q, f, seed, zone) for ps in sets]
    bound = min(plans[r].bootstrap(r, world) for r in range(world))
    parts = [plans[r].scan(r, world, bound) for r in range(world)]
    n = sets[0].size()
    return sharded.combine(parts, sharded.admissible_pairs(n, zone))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gauss_planted(psg, world):
    pts, planted = psg.gen.gauss_planted(2, 60_000, 128)
    got = run_parts(psg, lambda: psg.PointSet.from_flat(pts, 128), world)
    one = psg.closest_pair(psg.PointSet.from_flat(pts, 128), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (one.index_i, one.index_j, one.distance)
    assert (got.index_i, got.index_j) == tuple(sorted(planted))
    assert got.stats.admissible_pairs() == 60_000 * 59_999 // 2


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_dense_engine(psg, world):
    pts = psg.gen.mixture(5, 1 << 17, 64, 1024, 0.05)
    got = run_parts(psg, lambda: psg.PointSet.from_flat(pts, 64), world)
    ps = psg.PointSet.from_flat(pts, 64)
    bf = psg.brute_force_closest_pair(ps, 0)
    assert (got.index_i, got.index_j, got.distance) == (bf.index_i, bf.index_j, bf.distance)


@pytest.mark.parametrize("d,clusters", [(16, 16), (128, 64)])
def test_sharded_dense_cuda_core_tiles(psg, d, clusters):
    # d outside {32, 64}: the dense engine's CUDA-core tiles, tiles round-robin over parts
    pts = psg.gen.mixture(6, 1 << 17, d, clusters, 0.05)
    got = run_parts(psg, lambda: psg.PointSet.from_flat(pts, d), 3)
    assert "dense grid" in psg.last_profile()["stages"]  # the last part went through the dense engine
    bf = psg.brute_force_closest_pair(psg.PointSet.from_flat(pts, d), 0)
    assert (got.index_i, got.index_j, got.distance) == (bf.index_i, bf.index_j, bf.distance)


def test_sharded_motif_windows(psg):
    s, (a, b) = psg.gen.walk_motif(3, 50_000, 64)
    series = s.astype(np.float64)
    got = run_parts(psg, lambda: psg.PointSet.windows_of(series, 64, znorm=True), 2, zone=64)
    one = psg.closest_pair(psg.PointSet.windows_of(series, 64, znorm=True), 10, 10.0, 1, 64)
    assert (got.index_i, got.index_j, got.distance) == (one.index_i, one.index_j, one.distance)


# --- sharded FRNN (psg_frnn_plan_*): W parts on one device ----------------------
def frnn_parts(psg, pts, radius, world, zone=0):
    d = pts.shape[1]
    # one point set per emulated rank, alive as long as its plan
    sets = [psg.PointSet.from_flat(pts, d) for _ in range(world)]
    plans = [sharded.DeviceFrnnPlan(ps._device(), radius, 10, 10.0, 1, zone) for ps in sets]
    outs = [plans[r].scan(r, world, keep_pairs=True) for r in range(world)]
    runs = [plans[r].pairs(world) for r in range(world)]
    # the all-to-all: rank b receives bucket b of every part
    lists = []
    for b in range(world):
        recv = []
        for keys, counts in runs:
            off = int(np.sum(counts[:b]))
            recv.append(keys[off:off + int(counts[b])])
        lists.append(sharded.merge_sorted_runs(recv))
    cnt = sum(o[0] for o in outs)
    h = sum(o[1] for o in outs) & sharded.MASK64
    for p in plans:
        p.close()
    return cnt, h, np.concatenate(lists)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_frnn_c4_shape(psg, orc, world):
    n = 1 << 20
    cube = psg.gen.uniform(4, n, 3)
    R = (3 * 32 / (4 * np.pi * n)) ** (1 / 3)
    cnt, h, pairs = frnn_parts(psg, cube, R, world)
    one, c1, h1 = psg.frnn_pairs(cube, R)
    assert (cnt, h) == (c1, h1) == orc.frnn_grid(cube, R)
    assert np.array_equal(pairs, one)


@pytest.mark.parametrize("d,zone", [(5, 0), (3, 7)])
def test_sharded_frnn_scan_and_zone(psg, orc, d, zone):
    rng = np.random.default_rng(d + zone)
    pts = rng.random((30_000, d)).astype(np.float32)
    R = 0.1 if d == 5 else 0.02
    cnt, h, pairs = frnn_parts(psg, pts, R, 3, zone)
    want = orc.brute_force_neighbors(pts.astype(np.float64), R, zone, lists=True)
    assert (cnt, h) == want[:2]
    assert np.array_equal(pairs, np.sort(want[2]))


@pytest.mark.parametrize("recipe", ["mixture", "motif"])
def test_sharded_ranks_with_different_histories(psg, recipe):
    """Rank 0's point set has been solved before (it learned a cell width /
    engine / bootstrap mode), rank 1's has not: the part plans must still
    build the same grid on both (learned hints are not used by part plans),
    or pairs fall between the ranks' work lists."""
    if recipe == "mixture":
        pts = psg.gen.mixture(5, 1 << 18, 64, 1024, 0.05)
        make = lambda: psg.PointSet.from_flat(pts, 64)  # noqa: E731
        zone = 0
    else:
        s, _ = psg.gen.walk_motif(3, 1 << 18, 128)
        series = s.astype(np.float64)
        make = lambda: psg.PointSet.windows_of(series, 128, znorm=True)  # noqa: E731
        zone = 128
    sets = [make() for _ in range(2)]
    for _ in range(2):
        psg.closest_pair(sets[0], 10, 10.0, 1, zone)  # history on rank 0 only
    plans = [sharded.DevicePlan(ps._device(), 10, 10.0, 1, zone) for ps in sets]
    bound = min(plans[r].bootstrap(r, 2) for r in range(2))
    parts = [plans[r].scan(r, 2, bound) for r in range(2)]
    got = sharded.combine(parts, sharded.admissible_pairs(sets[0].size(), zone))
    one = psg.closest_pair(make(), 10, 10.0, 1, zone)
    assert (got.index_i, got.index_j, got.distance) == (one.index_i, one.index_j, one.distance)
