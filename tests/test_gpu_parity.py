"""GPU parity: the sm_100a engines through the C ABI versus the oracle.

Re-expresses the reference's hot-path tests (paths relative to
/root/reference/proj): tests/test_refscan.cpp, tests/test_metrics.cpp and the
hot-path acceptance criteria in tests/acceptance.cpp, plus the BASELINE
configs at oracle-sized n.  Integer results (indices, counts, hashes) must be
bit-exact; distances must equal the oracle's FP64 value exactly (the engines
recheck in the reference's FP64 order), which is stricter than north_star's
1e-5 relative tolerance.
"""
import ctypes

import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view

pytestmark = pytest.mark.gpu


def gauss_points(orc, seed, n, dim):
    r = orc.rng(seed)
    return np.array([orc.lib.orc_gaussian(r, 0.0, 1.0) for _ in range(n * dim)]).reshape(n, dim)


def windows(series, length):
    return np.ascontiguousarray(sliding_window_view(np.asarray(series, dtype=np.float64), length))


def admissible(n, zone):
    return sum(max(0, n - i - max(zone, 1)) for i in range(n)) if zone > 1 else n * (n - 1) // 2


# --- test_refscan.cpp:101-118 ---------------------------------------------------
def test_projected_scan_equals_brute_force_on_walk_windows(psg, orc):
    walk = orc.gen_random_walk(240, 5)
    pts = psg.PointSet.windows_of(walk, 8)
    want = orc.brute_force_closest_pair(windows(walk, 8), 8)
    assert want.pairs_examined == admissible(pts.size(), 8)
    for seed in (1, 2, 3):
        for q in (1, 3, 10):
            for f in (1.0, 10.0):
                got = psg.closest_pair(pts, q, f, seed, 8)
                assert (got.index_i, got.index_j) == (want.index_i, want.index_j)
                assert got.distance == want.distance
                assert got.stats.admissible_pairs() == want.pairs_examined


# --- test_refscan.cpp:120-129 ---------------------------------------------------
def test_scan_equals_brute_force_on_point_cloud(psg, orc):
    g = gauss_points(orc, 77, 150, 4)
    got = psg.closest_pair(psg.PointSet.from_flat(g, 4), 10, 10.0, 4, 0)
    assert (got.index_i, got.index_j) == (61, 102)  # SURVEY §8(c) known answer
    assert got.distance == 0.19603678271520741
    assert got.stats.admissible_pairs() == 150 * 149 // 2
    bf = psg.brute_force_closest_pair(psg.PointSet.from_flat(g, 4), 0)
    assert (bf.index_i, bf.index_j, bf.distance) == (61, 102, got.distance)


# --- test_refscan.cpp:131-141 ---------------------------------------------------
def test_stats_partition_admissible_pairs(psg, orc):
    walk = orc.gen_random_walk(180, 13)
    pts = psg.PointSet.windows_of(walk, 6)
    for zone in (0, 1, 6, 50):
        s = psg.closest_pair(pts, 5, 10.0, 2, zone).stats
        assert s.pairs_examined + s.pairs_pruned_by_reference + s.pairs_skipped_by_exit == admissible(pts.size(), zone)
        assert s.pairs_examined >= 1


# --- test_refscan.cpp:143-157 ---------------------------------------------------
def test_exclusion_zone_hides_adjacent_duplicates(psg):
    pts = psg.PointSet.from_flat([0.0, 0.0005, 10.0, 30.0, 50.0, 10.1], 1)
    for zone in (0, 1):
        r = psg.closest_pair(pts, 2, 10.0, 1, zone)
        assert (r.index_i, r.index_j) == (0, 1)
    wide = psg.closest_pair(pts, 2, 10.0, 1, 2)
    assert (wide.index_i, wide.index_j) == (2, 5)
    assert wide.distance == pytest.approx(0.1)
    brute = psg.brute_force_closest_pair(pts, 2)
    assert (brute.index_i, brute.index_j) == (2, 5)


# --- test_refscan.cpp:159-167 ---------------------------------------------------
def test_fixed_radius_boundary_inclusive(psg):
    pts = psg.PointSet.from_flat([0.0, 1.0, 2.0, 3.5], 1)
    got = psg.fixed_radius_neighbors(pts, 1.0, 2, 10.0, 1)
    assert [list(map(int, l)) for l in got.neighbors] == [[1], [0, 2], [1], []]


# --- test_refscan.cpp:169-182 ---------------------------------------------------
def test_fixed_radius_matches_brute_force(psg, orc):
    g = gauss_points(orc, 31, 120, 3)
    pts = psg.PointSet.from_flat(g, 3)
    for radius in (0.35, 1.2, 2.5):
        for zone in (0, 2):
            got = psg.fixed_radius_neighbors(pts, radius, 8, 10.0, 9, zone)
            cnt, h, pairs = orc.brute_force_neighbors(g, radius, zone, lists=True)
            assert (got.pair_count, got.pair_hash) == (cnt, h)
            want = [[] for _ in range(120)]
            for key in pairs.tolist():
                i, j = key >> 32, key & 0xFFFFFFFF
                want[i].append(j)
                want[j].append(i)
            assert [sorted(map(int, l)) for l in got.neighbors] == [sorted(w) for w in want]
            assert [list(map(int, l)) for l in got.neighbors] == [sorted(w) for w in want]
            s = got.stats
            assert s.pairs_examined + s.pairs_pruned_by_reference + s.pairs_skipped_by_exit == admissible(120, zone)
            bf = psg.brute_force_neighbors(pts, radius, zone)
            assert [list(map(int, l)) for l in bf] == [sorted(w) for w in want]


# --- test_refscan.cpp:184-194 ---------------------------------------------------
def test_results_do_not_depend_on_seed(psg, orc):
    walk = orc.gen_random_walk(300, 17)
    pts = psg.PointSet.windows_of(walk, 12)
    want = orc.brute_force_closest_pair(windows(walk, 12), 12)
    for seed in range(1, 11):
        got = psg.closest_pair(pts, 10, 10.0, seed, 12)
        assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


# --- test_refscan.cpp:196-206 ---------------------------------------------------
def test_degenerate_arguments_rejected(psg, orc):
    pts = psg.PointSet.from_flat(gauss_points(orc, 1, 5, 2), 2)
    with pytest.raises(psg.InvalidArgument, match="reference count must be positive"):
        psg.build_reference_set(pts, 0, 10.0, 1)
    with pytest.raises(psg.InvalidArgument, match="reference count exceeds point count"):
        psg.build_reference_set(pts, 6, 10.0, 1)
    with pytest.raises(psg.InvalidArgument, match="projection factor must be positive"):
        psg.build_reference_set(pts, 2, 0.0, 1)
    with pytest.raises(psg.InvalidArgument, match="no admissible pair"):
        psg.closest_pair(pts, 2, 10.0, 1, 5)
    with pytest.raises(psg.InvalidArgument, match="radius must be positive"):
        psg.fixed_radius_neighbors(pts, 0.0, 2, 10.0, 1)
    one = psg.PointSet.from_flat([1.0, 2.0], 2)
    with pytest.raises(psg.InvalidArgument, match="closest_pair needs at least 2 points"):
        psg.closest_pair(one, 1, 1.0, 1, 0)
    with pytest.raises(psg.InvalidArgument, match="closest_pair needs at least 2 points"):
        psg.brute_force_closest_pair(one, 0)


# --- test_refscan.cpp:42-69: reference set, bit-exact ------------------------------
def test_build_reference_set_bit_exact(psg, orc):
    g = gauss_points(orc, 11, 60, 5)
    rs = psg.build_reference_set(psg.PointSet.from_flat(g, 5), 7, 10.0, 3)
    ri, refs, table, order = orc.build_reference_set(g, 7, 10.0, 3)
    assert rs.ref_indices.tolist() == ri.tolist()
    assert np.array_equal(rs.references, refs)
    assert np.array_equal(rs.dist_table, table)
    assert rs.order.tolist() == order.tolist()
    for k in range(7):
        assert np.array_equal(rs.references[k], g[int(ri[k])] * 10.0)


# --- acceptance.cpp:201-231 (criterion 5 anchors) -------------------------------------
def test_reference_bound_anchors(psg, orc):
    r2 = np.sqrt(2.0)
    c30, s30 = np.cos(np.pi / 6), np.sin(np.pi / 6)
    c45, s45 = np.cos(np.pi / 4), np.sin(np.pi / 4)
    anchors = [([1.0, 1.0], 0.414), ([r2 * c30, r2 * s30], 0.6722), ([10 * c45, 10 * s45], 0.6803),
               ([10 * c30, 10 * s30], 0.8526), ([1000 * c45, 1000 * s45], 0.7071)]
    for r, want in anchors:
        got = psg.reference_bound(r, [0.0, 0.0], [1.0, 0.0])
        assert abs(got - want) <= 1e-3
        assert got == orc.reference_bound(r, [0.0, 0.0], [1.0, 0.0])


# --- acceptance.cpp:57-75 (criterion 1, exact on 100 walks) ---------------------------
def test_acceptance_c1_exact_on_100_walks(psg, orc):
    for seed in range(1, 101):
        walk = orc.gen_random_walk(2000, seed)
        got = psg.closest_pair(psg.PointSet.windows_of(walk, 64), 10, 10.0, seed, 64)
        want = orc.brute_force_closest_pair(windows(walk, 64), 64)
        assert got.distance == want.distance, seed
        assert (got.index_i, got.index_j) == (want.index_i, want.index_j), seed


# --- acceptance.cpp:152-196 (criterion 4: radius at a realised distance) --------------
def test_acceptance_c4_frnn_boundary_pair(psg, orc):
    g = gauss_points(orc, 7, 1000, 16)
    i, j = np.triu_indices(1000, 1)
    d = np.sqrt(((g[i] - g[j]) ** 2).sum(axis=1))
    k = d.size * 5 // 1000
    approx_r = np.partition(d, k)[k]
    # exact realised distance of that pair in the reference's FP64 order
    idx = int(np.argmin(np.abs(d - approx_r)))
    radius = orc.euclidean(g[i[idx]], g[j[idx]])
    got = psg.fixed_radius_neighbors(psg.PointSet.from_flat(g, 16), radius, 10, 10.0, 7)
    cnt, h = orc.brute_force_neighbors(g, radius)
    assert (got.pair_count, got.pair_hash) == (cnt, h)
    assert int(j[idx]) in set(map(int, got.neighbors[int(i[idx])]))  # boundary pair listed


# --- BASELINE configs at oracle-sized n ----------------------------------------------------
def test_c1_full_size(psg, orc):
    pts = orc.gen_uniform(1, 16384, 2)
    want = orc.brute_force_closest_pair(pts, 0)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 2), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


def test_c2_recipe_small(psg, orc):
    pts, planted = orc.gen_gauss_planted(2, 1 << 14, 128)
    want = orc.brute_force_closest_pair(pts, 0)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 128), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)
    assert (got.index_i, got.index_j) == tuple(sorted(planted))


def test_c3_recipe_small(psg, orc):
    s, (a, b) = orc.gen_walk_motif(3, 4096, 256)
    want = orc.motif_brute_znorm(s, 256, 256)
    got = psg.motif(s, 256, znorm=True)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)
    assert (got.index_i, got.index_j) == (min(a, b), max(a, b))


def test_c4_recipe_small(psg, orc):
    n = 1 << 16
    cube = orc.gen_uniform(4, n, 3)
    R = (3 * 32 / (4 * np.pi * n)) ** (1 / 3)
    pairs, cnt, h = psg.frnn_pairs(cube, R)
    assert (cnt, h) == orc.frnn_grid(cube, R)
    assert np.all(pairs[1:] > pairs[:-1])  # sorted lexicographically, unique
    i, j = pairs >> np.uint64(32), pairs & np.uint64(0xFFFFFFFF)
    assert np.all(i < j)


def _csr_from_pairs(pairs, n):
    i = (pairs >> np.uint64(32)).astype(np.int64)
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(np.bincount(i, minlength=n), out=off[1:])
    return off, (pairs & np.uint64(0xFFFFFFFF)).astype(np.uint32)


@pytest.mark.parametrize("n,k", [(1 << 12, 32), (1 << 16, 32), (1 << 16, 0.01), (3000, 200)])
def test_frnn_csr_matches_sorted_pairs(psg, orc, n, k):
    """The upper-triangular CSR output (psg_frnn_pairs_csr_f32) is the sorted
    pair list re-encoded: same count and hash, offsets = row starts, columns =
    the j's in order (one bucket, several buckets, almost no pairs, dense rows)."""
    cube = orc.gen_uniform(6, n, 3)
    R = (3 * k / (4 * np.pi * n)) ** (1 / 3)
    pairs, cnt, h = psg.frnn_pairs(cube, R)
    off, cols, c2, h2 = psg.frnn_pairs_csr(cube, R)
    assert (c2, h2) == (cnt, h)
    woff, wcols = _csr_from_pairs(pairs, n)
    assert np.array_equal(off, woff)
    assert np.array_equal(cols, wcols)
    if cnt > 10:  # a short column buffer: offsets complete, columns cut at capacity
        short = np.zeros(cnt // 3, np.uint32)
        off2, cols2, c3, _ = psg.frnn_pairs_csr(cube, R, cols=short)
        assert c3 == cnt and cols2 is None
        assert np.array_equal(off2, woff)
        assert np.array_equal(short, wcols[: short.size])


def test_frnn_csr_long_row(psg):
    """A row of 1100 columns inside a row group under the group capacity: the
    block-wide sort path of the group CSR kernel."""
    rng = np.random.default_rng(7)
    R = 1.0
    pts = np.zeros((1356, 64), np.float32)
    far = rng.normal(size=(255, 64)).astype(np.float32)
    pts[1:256] = 50.0 * far / np.linalg.norm(far, axis=1, keepdims=True) * (1 + np.arange(255)[:, None])
    ring = rng.normal(size=(1100, 64))
    pts[256:] = (0.9 * R * ring / np.linalg.norm(ring, axis=1, keepdims=True)).astype(np.float32)
    pairs, cnt, h = psg.frnn_pairs(pts, R)
    off, cols, c2, h2 = psg.frnn_pairs_csr(pts, R)
    assert (c2, h2) == (cnt, h)
    assert int(off[1] - off[0]) >= 1100
    woff, wcols = _csr_from_pairs(pairs, pts.shape[0])
    assert np.array_equal(off, woff) and np.array_equal(cols, wcols)


def test_frnn_csr_edge_cases(psg, orc):
    """No pairs at all, two points, an exclusion zone, and the empty input
    (the reference's message)."""
    far = np.arange(40, dtype=np.float32).reshape(20, 2) * 100
    off, cols, cnt, h = psg.frnn_pairs_csr(far, 1.0)
    assert cnt == 0 and h == 0 and np.all(off == 0) and cols.size == 0
    two = np.array([[0, 0], [0.5, 0]], np.float32)
    off, cols, cnt, _ = psg.frnn_pairs_csr(two, 1.0)
    assert cnt == 1 and list(off) == [0, 1, 1] and list(cols) == [1]
    walk = orc.gen_random_walk(3000, 5)
    win = np.lib.stride_tricks.sliding_window_view(walk, 8).astype(np.float32)
    for zone in (0, 8):
        pairs, c1, h1 = psg.frnn_pairs(win, 2.0, exclusion_zone=zone)
        off, cols, c2, h2 = psg.frnn_pairs_csr(win, 2.0, exclusion_zone=zone)
        assert (c2, h2) == (c1, h1)
        woff, wcols = _csr_from_pairs(pairs, win.shape[0])
        assert np.array_equal(off, woff) and np.array_equal(cols, wcols)
    with pytest.raises(psg.InvalidArgument, match="empty input"):
        psg.frnn_pairs_csr(np.zeros((0, 3), np.float32), 1.0)


@pytest.mark.parametrize("d", [16, 100])
def test_unseparable_sets_take_the_all_pairs_engine(psg, orc, d):
    """Uniform data in mid/high dimensions at a small n: the grid cannot
    separate the pairs (the estimate is a large share of all pairs) and the
    set is small enough for the all-pairs engine to beat the dense engine's
    set-up, so the solve goes there — learned for later solves.  Same answer
    as the oracle every time."""
    x = orc.gen_uniform(9, 6000, d)
    want = orc.brute_force_closest_pair(x, 0)
    ps = psg.PointSet.from_flat(x, d)
    for _ in range(3):  # first solve (grid, then the switch), then the learned path
        got = psg.closest_pair(ps, 10, 10.0, 1, 0)
        assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


def test_c5_recipe_small(psg, orc):
    pts = orc.gen_mixture(5, 8192, 64, 1024, 0.05)
    want = orc.brute_force_closest_pair(pts, 0)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 64), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


# --- numeric edge cases -------------------------------------------------------------------
def test_double_inputs_not_float_representable(psg, orc):
    g = gauss_points(orc, 123, 3000, 7)  # FP64 values: the FP32 filter narrows them
    want = orc.brute_force_closest_pair(g, 0)
    got = psg.closest_pair(psg.PointSet.from_flat(g, 7), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


def test_huge_and_tiny_magnitudes_rescaled(psg, orc):
    g = gauss_points(orc, 5, 2000, 3)
    for scale in (1e30, 1e-30):
        h = g * scale
        want = orc.brute_force_closest_pair(h, 0)
        got = psg.closest_pair(psg.PointSet.from_flat(h, 3), 10, 10.0, 1, 0)
        assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)


def test_exact_ties_break_to_lowest_pair(psg, orc):
    # integer lattice: many pairs at distance exactly 1; duplicates at 0
    grid = np.array([[x, y] for x in range(40) for y in range(40)], dtype=np.float64)
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(grid))
    pts = grid[perm]
    want = orc.brute_force_closest_pair(pts, 0)
    got = psg.closest_pair(psg.PointSet.from_flat(pts, 2), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)
    dup = np.vstack([pts, pts[[17, 900, 17]]])
    want = orc.brute_force_closest_pair(dup, 0)
    got = psg.closest_pair(psg.PointSet.from_flat(dup, 2), 10, 10.0, 1, 0)
    assert (got.index_i, got.index_j, got.distance) == (want.index_i, want.index_j, want.distance)
    assert got.distance == 0.0


def test_repeated_runs_are_identical(psg, orc):
    pts, _ = orc.gen_gauss_planted(2, 1 << 13, 128)
    ps = psg.PointSet.from_flat(pts, 128)
    a = psg.closest_pair(ps, 10, 10.0, 1, 0)
    b = psg.closest_pair(ps, 10, 10.0, 1, 0)
    assert a == b


def test_float32_and_float64_entry_points_agree(psg, orc):
    pts = orc.gen_uniform(1, 5000, 3)
    a = psg.closest_pair(psg.PointSet.from_flat(pts, 3), 10, 10.0, 1, 0)
    b = psg.closest_pair(psg.PointSet.from_flat(pts.astype(np.float64), 3), 10, 10.0, 1, 0)
    assert (a.index_i, a.index_j, a.distance) == (b.index_i, b.index_j, b.distance)


@pytest.mark.parametrize("length,znorm", [(8192, True), (8192, False), (3, True)])
def test_window_projection_shapes(psg, orc, length, znorm):
    """Window sets whose directions do not fit shared memory (len 8192: the
    projection reads U from global memory) and tiny windows: the motif equals
    the device brute force over the same virtual rows."""
    walk = orc.gen_random_walk(12000 if length > 100 else 4000, 21)
    zone = 64  # admissible pairs among the 3809 windows of length 8192
    got = psg.motif(walk, length, znorm=znorm, exclusion_zone=zone)
    out = psg._Pair()
    psg._check(psg.lib().psg_brute_force_motif_f64(walk.ctypes.data, walk.size, length, int(znorm), zone,
                                                   ctypes.byref(out)))
    assert (got.index_i, got.index_j, got.distance) == (out.index_i, out.index_j, out.distance)


def test_raw_windows_motif_matches_reference_engine(psg, orc):
    walk = orc.gen_random_walk(400, 11)
    got = psg.motif(walk, 24, znorm=False)
    assert (got.index_i, got.index_j) == (100, 208)  # SURVEY §8(c) known answer
    assert got.distance == 5.282423415841313


# --- CSR list building: every row-size class of the warp bitonic sort (1..1024)
# and the global-sort fallback for rows longer than 1024 -------------------------
@pytest.mark.parametrize("radius", [0.12, 0.5, 0.8])
def test_fixed_radius_lists_all_row_sizes(psg, orc, radius):
    g = gauss_points(orc, 77, 4000, 2)
    got = psg.fixed_radius_neighbors(psg.PointSet.from_flat(g, 2), radius, 8, 10.0, 3)
    cnt, h, pairs = orc.brute_force_neighbors(g, radius, 0, lists=True)
    assert (got.pair_count, got.pair_hash) == (cnt, h)
    want = [[] for _ in range(4000)]
    for key in pairs.tolist():
        i, j = key >> 32, key & 0xFFFFFFFF
        want[i].append(j)
        want[j].append(i)
    lens = [len(w) for w in want]
    if radius == 0.8:
        assert max(lens) > 1024  # exercises the fallback
    assert [list(map(int, l)) for l in got.neighbors] == [sorted(w) for w in want]
    plist, pc, ph = psg.frnn_pairs(g.astype(np.float32), radius)
    cnt32, h32, pairs32 = orc.brute_force_neighbors(g.astype(np.float32).astype(np.float64), radius, 0, lists=True)
    assert (pc, ph) == (cnt32, h32)
    assert np.array_equal(plist, np.sort(np.asarray(pairs32, dtype=np.uint64)))
