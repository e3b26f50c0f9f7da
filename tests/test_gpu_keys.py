"""The projection keys stay inside the error bound E the filters charge.

Every FP32 filter (grid cells, key lower bound) assumes |key - <U_k, x>| <= E
(psg_internal.cuh key_gamma).  For the tensor-core shapes
(d in {32, 64, 128, 256}: tcgen05 kind::tf32 on an exact hi/lo split of x,
psg_project_tc.cu) E is a charged model of the tensor core's FP32
accumulation, so it is checked here against FP64 projections of the same
FP32 directions on several data families; the realised error must stay well
inside it.  The CUDA-core shapes are checked the same way.
"""
import numpy as np
import pytest

import paper_1407_5609_b200 as psg

pytestmark = pytest.mark.gpu


def _families(rng, n, d):
    yield "gauss", rng.standard_normal((n, d)).astype(np.float32)
    yield "uniform", rng.random((n, d), dtype=np.float32)
    big = rng.standard_normal((n, d)) * 1e3 + 5e3  # large offset: cancellation inside the dot products
    yield "offset", big.astype(np.float32)
    tiny = rng.standard_normal((n, d)) * 1e-20
    yield "tiny", tiny.astype(np.float32)
    mixed = rng.standard_normal((n, d)) * np.exp(rng.uniform(-20, 20, (n, 1)))  # rows of very different scale
    yield "mixed", mixed.astype(np.float32)


@pytest.mark.parametrize("d", [32, 64, 128, 256, 3, 16])
@pytest.mark.parametrize("q", [4, 10])
def test_keys_within_charged_error(d, q):
    rng = np.random.default_rng(1000 + d + q)
    n = 4099  # not a multiple of the 128-row tile: exercises the zero-filled tail
    for name, x in _families(rng, n, d):
        ps = psg.PointSet.from_flat(x, d)
        keys, dirs, E, scale = psg.debug_projection(ps, q=q, seed=7)
        xw = (x.astype(np.float64) * scale).astype(np.float32).astype(np.float64)  # the FP32 working rows
        exact = xw @ dirs.astype(np.float64).T
        err = np.abs(keys.astype(np.float64) - exact).max()
        assert err <= E, f"{name}: key error {err:.3e} exceeds the charged bound {E:.3e}"
        # the bound is not vacuous for the tensor-core shapes: realised error well inside it
        if d in (32, 64, 128, 256) and name in ("gauss", "offset"):
            assert err <= 0.25 * E, f"{name}: key error {err:.3e} uses more than a quarter of E = {E:.3e}"


def test_tensor_core_directions_are_tf32():
    x = np.random.default_rng(3).standard_normal((300, 128)).astype(np.float32)
    _, dirs, _, _ = psg.debug_projection(psg.PointSet.from_flat(x, 128), q=10, seed=1)
    bits = dirs.view(np.uint32)
    assert np.all(bits & 0x1FFF == 0), "tensor-core directions must be exact TF32 operands"


def _window_rows(series, length, znorm):
    """The FP32 virtual window rows the device filters read (psg_points.cuh
    Rows): fl(fl(s32[i+t] - m32[i]) * r32[i]) with the FP64 two-pass window
    statistics (sequential sums, like k_window_stats), or s32[i+t] raw."""
    s64 = np.asarray(series, dtype=np.float64)
    nw = s64.size - length + 1
    w = np.lib.stride_tricks.sliding_window_view(s64, length)
    s32 = s64.astype(np.float32)
    ws = np.lib.stride_tricks.sliding_window_view(s32, length)
    if not znorm:
        return ws.astype(np.float64)
    mu = np.zeros(nw)
    for t in range(length):  # sequential, as the device sums
        mu = mu + w[:, t]
    mu = mu / length
    var = np.zeros(nw)
    for t in range(length):
        c = w[:, t] - mu
        var = var + c * c
    sg = np.sqrt(var / length)
    m32 = mu.astype(np.float32)
    r32 = np.where(sg == 0, 0.0, 1.0 / sg).astype(np.float32)
    x = ((ws - m32[:, None]).astype(np.float32) * r32[:, None]).astype(np.float32)
    return x.astype(np.float64)


@pytest.mark.parametrize("length", [32, 64, 128, 256, 24])
@pytest.mark.parametrize("znorm", [True, False])
def test_window_keys_within_charged_error(length, znorm):
    """Window sets (k_project_windows forms the virtual rows from the series,
    4 windows per thread): the keys stay inside E.  A random walk has large
    window means against small window spreads."""
    rng = np.random.default_rng(length + znorm)
    series = np.cumsum(rng.standard_normal(4099 + length - 1)) + 300.0
    ps = psg.PointSet.windows_of(series, length, znorm=znorm)
    keys, dirs, E, scale = psg.debug_projection(ps, q=10, seed=7)
    x = _window_rows(series * (1.0 if znorm else scale), length, znorm)
    exact = x @ dirs.astype(np.float64).T
    err = np.abs(keys.astype(np.float64) - exact).max()
    assert err <= E, f"key error {err:.3e} exceeds the charged bound {E:.3e}"
