"""CPU: the C-ABI library loads, exports every symbol include/*.h declares,
its host-side pieces (seeded generators, validation) agree with the oracle,
and compute entries fail loudly (no CPU fallback) when no sm_100 GPU exists."""
import ctypes as C
import glob
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(psg_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol(psg):
    syms = declared_symbols()
    assert len(syms) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", psg.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = syms - exported
    assert not missing, missing
    for name in syms:  # and ctypes can bind each one
        getattr(psg.lib(), name)


def test_library_is_sm100a_only(psg):
    out = subprocess.run(["cuobjdump", "--list-elf", psg.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_device_probe(psg):
    assert b"sm_100a" in psg.lib().psg_version()
    assert psg.lib().psg_device_ok(0) in (0, 1)


def test_compute_without_gpu_fails_loudly(psg):
    if psg.lib().psg_device_ok(0):
        pytest.skip("a GPU is present")
    pts = np.random.default_rng(0).normal(size=(64, 4))
    with pytest.raises(psg.DeviceError):
        psg.closest_pair(psg.PointSet.from_flat(pts, 4), 10, 10.0, 1, 0)
    out = psg._Pair()
    rc = psg.lib().psg_closest_pair_f64(pts.ctypes.data, 64, 4, 10, 10.0, 1, 0, C.byref(out))
    assert rc == psg.PSG_ERR_CUDA


def test_pointset_validation_matches_reference_messages(psg):
    # series.cpp:19-32 and :8-11
    with pytest.raises(psg.InvalidArgument, match="point dimension must be positive"):
        psg.PointSet.from_flat([1.0, 2.0], 0)
    with pytest.raises(psg.InvalidArgument, match="flat buffer not a multiple of dim"):
        psg.PointSet.from_flat([1.0, 2.0, 3.0], 2)
    with pytest.raises(psg.InvalidArgument, match="point coordinate must be finite"):
        psg.PointSet.from_flat([1.0, np.nan], 1)
    with pytest.raises(psg.InvalidArgument, match="window length out of range"):
        psg.PointSet.windows_of(np.arange(5.0), 6)
    with pytest.raises(psg.InvalidArgument, match="window length out of range"):
        psg.TimeSeries(np.arange(5.0)).window_count(0)
    ps = psg.PointSet.windows_of(np.arange(10.0), 4)
    assert (ps.size(), ps.dim()) == (7, 4)
    assert ps.point(2).tolist() == [2.0, 3.0, 4.0, 5.0]


def test_host_generators_match_oracle(psg, orc):
    # product host datagen == oracle restatement, bit for bit
    assert np.array_equal(psg.gen.random_walk(1000, 7), orc.gen_random_walk(1000, 7))
    assert np.array_equal(psg.gen.uniform(1, 70000, 2), orc.gen_uniform(1, 70000, 2))
    a, pa = psg.gen.gauss_planted(2, 70000, 8)
    b, pb = orc.gen_gauss_planted(2, 70000, 8)
    assert pa == pb and np.array_equal(a, b)
    a, pa = psg.gen.walk_motif(3, 5000, 64)
    b, pb = orc.gen_walk_motif(3, 5000, 64)
    assert pa == pb and np.array_equal(a, b)
    assert np.array_equal(psg.gen.mixture(5, 70000, 4, 16, 0.05), orc.gen_mixture(5, 70000, 4, 16, 0.05))
    for x in (0, 1, 12345, (1 << 64) - 1):
        assert psg.gen.mix_seed(x) == orc.mix_seed(x)
        assert psg.gen.derive_seed(x, 3) == orc.derive_seed(x, 3)


def test_c4_radius_literal():
    import oracle

    # R pinned as the cbrt value, one ulp below pow(x, 1/3)
    assert oracle.R_C4 == float.fromhex("0x1.902ce9269f6dp-7")
    x = 3 * 32 / (4 * np.pi * 4194304)
    assert abs(oracle.R_C4 - x ** (1 / 3)) <= 2 * np.spacing(oracle.R_C4)
