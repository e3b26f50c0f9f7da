"""pairscan-gpu, the reference front end's motif / frnn / sweep / verify over
the B200 library (tools/src/main.cpp).

Brute-engine reports must be byte-identical to what the reference CLI prints
for the same command: the test rebuilds the reference's Report from the
UNMODIFIED reference library (oracle/_ref: datagen, brute-force scans and the
io.cpp JSON/CSV writers) with the params line main.cpp would record.  The
mpr / mk engines must return the reference's pair and distance (their
pairs_examined counts the GPU engine's work) and replay through
`verify`.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1407_5609_b200", "bin", "pairscan-gpu")


def run(*args, cwd=None):
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=600)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not os.path.exists(CLI):
        pytest.fail("paper_1407_5609_b200/bin/pairscan-gpu not built (run __graft_entry__.build())")


def fmt(v: float) -> str:
    """fmt_num (main.cpp:44-46): nlohmann's shortest round-trip, '.0' on integers."""
    s = json.dumps(float(v))
    return s


def admissible(n, zone):  # main.cpp:384-393
    if zone == 0:
        return n * (n - 1) // 2
    return sum(n - i - zone for i in range(n) if n > i + zone)


# --------------------------------------------------------------------- CPU


def test_gen_walk_file_matches_reference(ref, tmp_path):
    out = tmp_path / "w.txt"
    rc, so, _ = run("gen-walk", "--n", 5000, "--seed", 7, "--stddev", 0.5, "--out", out)
    assert rc == 0 and so == f"wrote 5000 values to {out}\n"
    want = tmp_path / "r.txt"
    ref.save_series(ref.gen_random_walk(5000, 7, 0.5), str(want))
    assert out.read_bytes() == want.read_bytes()


@pytest.mark.parametrize("args,msg", [
    ((), "a subcommand is required"),
    (("motif", "--gen-walk", "100"), "--len is required"),
    (("motif", "--gen-walk", "100", "--len", "8", "--engine", "fast"), "--engine: fast not in"),
    (("motif", "--len", "8"), "pass a series file or --gen-walk, not both"),
    (("motif", "--gen-walk", "100", "--len", "-3"), "--len: expected a non-negative integer"),
    (("motif", "--gen-walk", "100", "--len", "8", "--bogus", "1"), "not expected: --bogus"),
    (("frnn", "--gen-walk", "100", "--len", "8"), "--radius is required"),
    (("sweep", "--n-list", "100"), "--len-list is required"),
    (("closest",), "points is required"),
    (("gen-walk", "--n", "10"), "--out is required"),
    (("frobnicate",), "unknown subcommand: frobnicate"),
])
def test_usage_errors(args, msg):
    rc, so, se = run(*args)
    assert rc == 2 and so == "" and msg in se, se


def test_missing_series_file_message(ref, tmp_path):
    # io.cpp's message through the library's parser (no device needed to fail)
    path = str(tmp_path / "absent.txt")
    _, _, want = ref.load_series(path)
    rc, _, se = run("motif", path, "--len", 8)
    assert rc == 2 and se == f"error: {want}\n"


def test_version_and_help():
    assert run("--version") == (0, "0.1.0\n", "")
    rc, so, _ = run("--help")
    assert rc == 0 and "motif" in so and "verify" in so


def test_no_device_fails_loudly(psg):
    if psg.lib().psg_device_ok(0) == 1:
        pytest.skip("a B200 is present")
    rc, so, se = run("motif", "--gen-walk", 200, "--len", 8)
    assert rc == 2 and so == "" and se.startswith("error: ")


# --------------------------------------------------------------------- GPU

gpu = pytest.mark.gpu


def windows(series, l):
    return np.lib.stride_tricks.sliding_window_view(np.asarray(series, np.float64), l)


@gpu
def test_motif_brute_report_is_the_reference_report(ref, tmp_path):
    n, l, seed = 3000, 32, 5
    rc, so, se = run("motif", "--gen-walk", n, "--len", l, "--seed", seed, "--engine", "brute", "--deterministic",
                     "--out", tmp_path / "m.json")
    assert rc == 0, se
    walk = ref.gen_random_walk(n, seed, 1.0)
    bf = ref.brute_force_closest_pair(windows(walk, l), l)
    params = (f"motif --gen-walk {n} --walk-stddev 1.0 --len {l} --refs 10 --factor 10.0 --seed {seed} "
              f"--exclusion {l} --engine brute --version-tag 0.1.0 --deterministic")
    want_json, want_csv = ref.report("brute", params, f"gen-walk:n={n},seed={seed},stddev=1.0", bf.index_i + 1,
                                     bf.index_j + 1, bf.distance, bf.pairs_examined, 0, 0.0, seed)
    assert bf.pairs_examined == admissible(n - l + 1, l)
    assert so == want_json
    assert (tmp_path / "m.json").read_text() == want_json
    assert (tmp_path / "m.csv").read_text() == want_csv


@gpu
@pytest.mark.parametrize("engine,f", [("mpr", 10.0), ("mk", 1.0), ("gpu", 3.0)])
def test_motif_engines_match_reference_and_replay(ref, tmp_path, engine, f):
    n, l, seed = 20_000, 64, 3
    series = tmp_path / "s.txt"
    assert run("gen-walk", "--n", n, "--seed", 11, "--out", series)[0] == 0
    out = tmp_path / "r.json"
    rc, so, se = run("motif", series, "--len", l, "--seed", seed, "--factor", f, "--engine", engine,
                     "--verify", "brute", "--out", out)
    assert rc == 0, se
    r = json.loads(so)
    walk = ref.gen_random_walk(n, 11, 1.0)
    want = ref.closest_pair_windows(walk, l, 10, 1.0 if engine == "mk" else f, seed, l)
    assert (r["pair_index_1"], r["pair_index_2"], r["distance_or_matches"]) == (want.index_i + 1, want.index_j + 1,
                                                                              want.distance)
    assert r["algorithm"] == engine and r["dataset"] == str(series) and r["seed"] == seed
    assert f"--factor {fmt(1.0 if engine == 'mk' else f)}" in r["params"]
    assert se.startswith(f"verify: brute agrees, distance {fmt(want.distance)}")
    rc, so, se = run("verify", out)
    assert rc == 0 and so == f"verify: OK {r['params']}\n", (so, se)


@gpu
def test_verify_detects_a_tampered_report(tmp_path):
    out = tmp_path / "r.json"
    assert run("motif", "--gen-walk", 4000, "--len", 16, "--deterministic", "--out", out)[0] == 0
    doc = json.loads(out.read_text())
    doc["pair_index_2"] += 1
    out.write_text(json.dumps(doc))
    rc, so, _ = run("verify", out)
    assert rc == 3 and so.startswith("verify: MISMATCH row 1: pair_index_2 expected")


@gpu
def test_frnn_brute_report_and_pairs_match_reference(ref, tmp_path):
    n, l, seed = 2500, 16, 9
    walk = ref.gen_random_walk(n, seed, 1.0)
    W = windows(walk, l)
    cnt, _, pairs = ref.brute_force_neighbors(W, 4.0, l, lists=True)
    assert cnt > 10
    rc, so, se = run("frnn", "--gen-walk", n, "--len", l, "--seed", seed, "--radius", 4.0, "--engine", "brute",
                     "--deterministic", "--pairs-out", tmp_path / "p.csv")
    assert rc == 0, se
    first = (int(pairs[0] >> 32) + 1, int(pairs[0] & 0xFFFFFFFF) + 1)
    params = (f"frnn --gen-walk {n} --walk-stddev 1.0 --len {l} --refs 10 --factor 10.0 --seed {seed} "
              f"--exclusion {l} --engine brute --radius 4.0 --version-tag 0.1.0 --deterministic")
    want_json, _ = ref.report("brute", params, f"gen-walk:n={n},seed={seed},stddev=1.0", first[0], first[1],
                              float(cnt), admissible(n - l + 1, l), 0, 0.0, seed)
    assert so == want_json
    lines = "".join(f"{int(k >> 32) + 1},{int(k & 0xFFFFFFFF) + 1}\n" for k in pairs)
    assert (tmp_path / "p.csv").read_text() == lines


@gpu
def test_frnn_mpr_agrees_with_brute_and_replays(ref, tmp_path):
    n, l = 30_000, 32
    out = tmp_path / "f.json"
    rc, so, se = run("frnn", "--gen-walk", n, "--len", l, "--radius", 6.0, "--verify", "brute", "--out", out)
    assert rc == 0 and "verify: brute agrees" in se, se
    walk = ref.gen_random_walk(n, 1, 1.0)
    cnt = ref.fixed_radius_neighbors(windows(walk, l), 6.0, 10, 10.0, 1, l)["count"]
    assert cnt > 1000
    assert json.loads(so)["distance_or_matches"] == float(cnt)
    rc, so, _ = run("verify", out)
    assert rc == 0 and so.startswith("verify: OK frnn ")


@gpu
def test_point_cloud_commands(psg, orc, tmp_path):
    pts, planted = psg.gen.gauss_planted(4, 40_000, 64)
    p = tmp_path / "cloud.psgb"
    psg.save_binary(pts, str(p))
    rc, so, se = run("closest", p, "--engine", "mpr", "--verify", "brute", "--deterministic", "--out",
                     tmp_path / "c.json")
    assert rc == 0 and "verify: brute agrees" in se, se
    r = json.loads(so)
    assert (r["pair_index_1"] - 1, r["pair_index_2"] - 1) == tuple(sorted(planted))
    small = pts[:3000].astype(np.float64)
    q = tmp_path / "small.psgb"
    psg.save_binary(small, str(q))
    want = orc.brute_force_closest_pair(small, 0)
    r = json.loads(run("closest", q, "--engine", "brute")[1])
    assert (r["pair_index_1"], r["pair_index_2"], r["distance_or_matches"]) == (want.index_i + 1, want.index_j + 1,
                                                                              want.distance)
    radius = want.distance * 1.5
    cnt, _ = orc.brute_force_neighbors(small, radius, 0)
    rc, so, se = run("neighbors", q, "--radius", radius, "--verify", "brute")
    assert rc == 0 and json.loads(so)["distance_or_matches"] == float(cnt) and "agrees" in se
    assert run("verify", tmp_path / "c.json")[0] == 0


@gpu
def test_sweep_rows_match_reference(ref, tmp_path):
    rc, so, se = run("sweep", "--n-list", "1500,2500", "--len-list", "16,32", "--reps", 2, "--engines",
                     "mk,mpr,brute", "--q-list", "4,10", "--f-list", "1.5,10", "--seed", 3, "--deterministic",
                     "--out", tmp_path / "s.csv")
    assert rc == 0, se
    raw = (tmp_path / "s.raw.csv").read_text().splitlines()
    assert raw[0] == "n,len,q,f,engine,rep,seed,pair_index_1,pair_index_2,distance,pairs_examined,wall_seconds"
    rows = [r.split(",") for r in raw[1:]]
    # per cell: mk (q-list x f=1), mpr (q-list x f-list), brute once
    assert len(rows) == 2 * 2 * 2 * (2 + 4 + 1)
    for r in rows:
        n, l, q, f, eng, rep, dseed = int(r[0]), int(r[1]), int(r[2]), float(r[3]), r[4], int(r[5]), int(r[6])
        cell = [1500, 2500].index(n) * 2 + [16, 32].index(l)
        assert dseed == ref.derive_seed3(3, cell, rep - 1)
        walk = ref.gen_random_walk(n, dseed, 1.0)
        want = (ref.brute_force_closest_pair(windows(walk, l), l) if eng == "brute"
                else ref.closest_pair_windows(walk, l, q, f, dseed, l))
        assert (int(r[7]), int(r[8]), r[9]) == (want.index_i + 1, want.index_j + 1, fmt(want.distance))
        if eng == "brute":
            assert int(r[10]) == admissible(n - l + 1, l)
        assert r[11] == "0.0"
    table = (tmp_path / "s.csv").read_text()
    assert table == so and table.startswith("n,len,q,f,engine,reps,mean_pairs_examined,mean_wall_seconds\n")
