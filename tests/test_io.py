"""Data formats on either side of the path.

The text series format is the reference's own (io.cpp:44-60 load_series,
62-70 save_series).  CPU tests compare the library's parallel parser with the
UNMODIFIED reference io.cpp (compiled into oracle/_ref) on the same files:
values bit-identical, error class and message identical.  The GPU tests load
.psgb files straight into device point sets and solve them.
"""
import numpy as np
import pytest

GOOD = {
    "plain": "1\n2.5\n-3\n",
    "exponents_hex_signed_zero": "1e-300\n-0.0\n0x1.8p3\n+7\n.5\n5.\n",
    "crlf_and_spaces": "  1.25 \r\n\t-2\r\n3\r\n",
    "no_final_newline": "4\n5\n6",
    "smallest_normal": "2.2250738585072014e-308\n",
}
BAD = {
    "empty_line_middle": "1\n\n2\n",
    "empty_line_end": "1\n2\n\n",
    "two_values": "1\n2 3\n",
    "not_a_number": "1\nabc\n",
    "trailing_garbage": "1\n2x\n",
    "overflow": "1\n1e999\n",
    "subnormal_is_erange": "4.9e-324\n",  # glibc strtod sets ERANGE: the reference rejects it
    "nan": "1\nnan\n",
    "inf": "inf\n",
    "empty_file": "",
    "only_spaces": "   \n",
}


def _write(tmp_path, name, text):
    p = tmp_path / (name + ".txt")
    p.write_bytes(text.encode())
    return str(p)


@pytest.mark.parametrize("name", sorted(GOOD))
def test_series_text_values_match_reference(psg, ref, tmp_path, name):
    path = _write(tmp_path, name, GOOD[name])
    want, rc, msg = ref.load_series(path)
    assert rc == 0, msg
    got = psg.load_series_text(path)
    assert got.dtype == np.float64 and got.view(np.uint64).tolist() == want.view(np.uint64).tolist()


@pytest.mark.parametrize("name", sorted(BAD))
def test_series_text_errors_match_reference(psg, ref, tmp_path, name):
    path = _write(tmp_path, name, BAD[name])
    _, rc, msg = ref.load_series(path)
    assert rc != 0
    exc = psg.InvalidArgument if rc == -1 else psg.SeriesFileError
    with pytest.raises(exc) as e:
        psg.load_series_text(path)
    assert str(e.value) == msg


def test_missing_file_message(psg, ref, tmp_path):
    path = str(tmp_path / "absent.txt")
    _, rc, msg = ref.load_series(path)
    with pytest.raises(psg.SeriesFileError) as e:
        psg.load_series_text(path)
    assert rc == -2 and str(e.value) == msg


def test_large_file_parallel_chunks_and_line_numbers(psg, ref, tmp_path):
    # 300k lines: several parser chunks; an error deep inside must name its line
    rng = np.random.default_rng(7)
    vals = rng.standard_normal(300_000) * 10.0 ** rng.integers(-30, 30, 300_000)
    path = str(tmp_path / "big.txt")
    ref.save_series(vals, path)
    got = psg.load_series_text(path)
    want, rc, _ = ref.load_series(path)
    assert rc == 0 and np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(got, vals)  # %.17g round-trips exactly
    lines = open(path).read().split("\n")
    lines[234_567] = "oops"
    bad = str(tmp_path / "bad.txt")
    open(bad, "w").write("\n".join(lines))
    _, rc, msg = ref.load_series(bad)
    with pytest.raises(psg.SeriesFileError) as e:
        psg.load_series_text(bad)
    assert rc == -2 and str(e.value) == msg and ":234568:" in msg


def test_save_series_text_bytes_match_reference(psg, ref, tmp_path):
    vals = np.array([0.1, -2.0, 1e-310, 3.141592653589793, 1e300, -0.0])
    a, b = str(tmp_path / "a.txt"), str(tmp_path / "b.txt")
    psg.save_series_text(vals, a)
    ref.save_series(vals, b)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_binary_header_layout(psg, tmp_path):
    x = np.arange(12, dtype=np.float32).reshape(4, 3)
    p = str(tmp_path / "x.psgb")
    psg.save_binary(x, p)
    raw = open(p, "rb").read()
    assert raw[:4] == b"PSGB" and len(raw) == 32 + x.nbytes
    version, dtype, reserved = np.frombuffer(raw[4:16], dtype="<u4")
    rows, cols = np.frombuffer(raw[16:32], dtype="<u8")
    assert (version, dtype, reserved, rows, cols) == (1, 2, 0, 4, 3)
    assert np.array_equal(np.frombuffer(raw[32:], dtype="<f4").reshape(4, 3), x)


@pytest.mark.gpu
def test_pointset_from_binary_file_solves_like_from_flat(psg, tmp_path):
    pts, planted = psg.gen.gauss_planted(2, 50_000, 64)
    p = str(tmp_path / "pts.psgb")
    psg.save_binary(pts, p)
    fs = psg.FilePointSet(p)
    assert (fs.size(), fs.dim()) == (50_000, 64)
    a = psg.closest_pair(fs, 10, 10.0, 1, 0)
    b = psg.closest_pair(psg.PointSet.from_flat(pts, 64), 10, 10.0, 1, 0)
    assert (a.index_i, a.index_j, a.distance) == (b.index_i, b.index_j, b.distance)
    assert (a.index_i, a.index_j) == tuple(sorted(planted))
    # f64 rows too (the recheck reads the original doubles)
    p64 = str(tmp_path / "pts64.psgb")
    psg.save_binary(pts.astype(np.float64) / 3.0, p64)
    c = psg.closest_pair(psg.FilePointSet(p64), 10, 10.0, 1, 0)
    d = psg.closest_pair(psg.PointSet.from_flat(pts.astype(np.float64) / 3.0, 64), 10, 10.0, 1, 0)
    assert (c.index_i, c.index_j, c.distance) == (d.index_i, d.index_j, d.distance)


@pytest.mark.gpu
def test_windows_from_binary_series_file(psg, tmp_path):
    s, _ = psg.gen.walk_motif(3, 40_000, 64)
    walk = s.astype(np.float64)
    p = str(tmp_path / "walk.psgb")
    psg.save_binary(np.asarray(walk, dtype=np.float64), p)
    fs = psg.FilePointSet(p, window=64, znorm=True)
    a = psg.closest_pair(fs, 10, 10.0, 1, 64)
    b = psg.closest_pair(psg.PointSet.windows_of(np.asarray(walk, dtype=np.float64), 64, znorm=True), 10, 10.0, 1, 64)
    assert (a.index_i, a.index_j, a.distance) == (b.index_i, b.index_j, b.distance)
