"""The C++ drop-in header (include/pairscan_b200.hpp): compiles here against
the C ABI (CPU), and runs the reference's refscan tests re-expressed in C++ on
the GPU (tests/cxx/test_shim.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cxx", "test_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_1407_5609_b200")


def build(out):
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), SRC, "-o", out,
                    "-L", LIBDIR, "-lpairscan_b200", f"-Wl,-rpath,{LIBDIR}"], check=True,
                   stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    # the library's soname is its file name; link against it directly


def test_shim_compiles_and_links(tmp_path, psg):
    if not os.path.exists(os.path.join(LIBDIR, "libpairscan_b200.so")):
        pytest.fail("product library not built")
    build(str(tmp_path / "test_shim"))


@pytest.mark.gpu
def test_shim_reference_tests_pass_on_gpu(tmp_path, psg):
    exe = str(tmp_path / "test_shim")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
