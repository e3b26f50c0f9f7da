"""pairscan_b200 — exact closest pair / fixed-radius neighbours / motifs on B200.

A drop-in for the reference ``pairscan`` hot path (paths relative to
/root/reference/proj):

======================================  ==========================================
reference (C++)                         here (Python over the C ABI)
======================================  ==========================================
series.hpp:10-20  TimeSeries            :class:`TimeSeries`
series.hpp:28-44  PointSet              :class:`PointSet` (``from_flat``, ``windows_of``)
refscan.hpp:13-25 ReferenceSet          :class:`ReferenceSet`
refscan.hpp:27-48 ScanStats/PairResult  :class:`ScanStats`, :class:`PairResult`,
                  NeighborResult        :class:`NeighborResult`
refscan.hpp:50-71 build_reference_set,  :func:`build_reference_set`, :func:`closest_pair`,
                  closest_pair, ...     :func:`brute_force_closest_pair`,
                                        :func:`fixed_radius_neighbors`,
                                        :func:`brute_force_neighbors`, :func:`reference_bound`
======================================  ==========================================

Errors: the reference throws ``std::invalid_argument``; here
:class:`InvalidArgument` (a ``ValueError``) carries the same message.

Every compute call runs the sm_100a kernels in ``libpairscan_b200.so``; there
is no CPU path.  Importing works without a GPU (so the ABI can be inspected),
but any compute call then raises :class:`DeviceError`.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "InvalidArgument", "DeviceError", "TimeSeries", "PointSet", "ScanStats", "PairResult",
    "NeighborResult", "ReferenceSet", "closest_pair", "brute_force_closest_pair",
    "fixed_radius_neighbors", "brute_force_neighbors", "frnn_pairs", "build_reference_set",
    "reference_bound", "motif", "lib", "last_profile", "gen", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# PSG_LIB_PATH: a diagnostic build (e.g. -DPSG_DEBUG_SYNC) in place of the in-tree library
LIB_PATH = os.environ.get("PSG_LIB_PATH") or os.path.join(HERE, "libpairscan_b200.so")

PSG_OK, PSG_ERR_INVALID, PSG_ERR_CUDA, PSG_ERR_NOMEM, PSG_ERR_INTERNAL = 0, 1, 2, 3, 4
PSG_ERR_IO = 5


class InvalidArgument(ValueError):
    """The reference's std::invalid_argument (same messages)."""


class SeriesFileError(RuntimeError):
    """io.cpp's std::runtime_error (file open / parse errors), PSG_ERR_IO."""


class DeviceError(RuntimeError):
    """CUDA / device failure (no CPU fallback exists)."""


_u64, _f64, _f32, _int, _p = C.c_uint64, C.c_double, C.c_float, C.c_int, C.c_void_p


class _Stats(C.Structure):
    _fields_ = [("pairs_examined", _u64), ("pairs_pruned_by_reference", _u64),
                ("pairs_skipped_by_exit", _u64), ("inner_loop_exits", _u64)]


class _Pair(C.Structure):
    _fields_ = [("index_i", _u64), ("index_j", _u64), ("distance", _f64), ("stats", _Stats)]


class _Neigh(C.Structure):
    _fields_ = [("n", _u64), ("offsets", C.POINTER(_u64)), ("neighbors", C.POINTER(_u64)),
                ("pair_count", _u64), ("pair_hash", _u64), ("stats", _Stats)]


class _Profile(C.Structure):
    _fields_ = [("stages", _int), ("stage_name", (C.c_char * 24) * 16), ("stage_ms", _f32 * 16),
                ("launches", _u64), ("window_pairs", _u64), ("lb_survivors", _u64),
                ("candidates", _u64), ("bootstrap_width", _u64), ("h2d_bytes", _u64),
                ("d2h_bytes", _u64), ("scan_kernel_ms", _f64), ("project_kernel_ms", _f64),
                ("bootstrap_kernel_ms", _f64), ("total_ms", _f64), ("scan_launches", _u64),
                ("dense_cells", _u64), ("dense_cell_pairs", _u64), ("dense_groups", _u64),
                ("dense_split_groups", _u64), ("dense_tiles", _u64), ("inline_fp64", _u64)]


_SIGS = {
    "psg_last_error": (C.c_char_p, []),
    "psg_version": (C.c_char_p, []),
    "psg_last_profile": (_int, [_p]),
    "psg_device_ok": (_int, [_int]),
    "psg_stream": (_p, []),
    "psg_set_device": (_int, [_int]),
    "psg_set_graph_profiling": (_int, [_int]),
    "psg_closest_pair_f64": (_int, [_p, _u64, _u64, _u64, _f64, _u64, _u64, _p]),
    "psg_closest_pair_f32": (_int, [_p, _u64, _u64, _u64, _f64, _u64, _u64, _p]),
    "psg_brute_force_closest_pair_f64": (_int, [_p, _u64, _u64, _u64, _p]),
    "psg_brute_force_closest_pair_f32": (_int, [_p, _u64, _u64, _u64, _p]),
    "psg_motif_f64": (_int, [_p, _u64, _u64, _int, _u64, _f64, _u64, _u64, _p]),
    "psg_motif_f32": (_int, [_p, _u64, _u64, _int, _u64, _f64, _u64, _u64, _p]),
    "psg_brute_force_motif_f64": (_int, [_p, _u64, _u64, _int, _u64, _p]),
    "psg_fixed_radius_neighbors_f64": (_int, [_p, _u64, _u64, _f64, _u64, _f64, _u64, _u64, _int, _p]),
    "psg_fixed_radius_neighbors_f32": (_int, [_p, _u64, _u64, _f64, _u64, _f64, _u64, _u64, _int, _p]),
    "psg_brute_force_neighbors_f64": (_int, [_p, _u64, _u64, _f64, _u64, _int, _p]),
    "psg_frnn_pairs_f32": (_int, [_p, _u64, _u64, _f64, _u64, _f64, _u64, _u64, _p, _u64, _p, _p]),
    "psg_frnn_pairs_csr_f32": (_int, [_p, _u64, _u64, _f64, _u64, _f64, _u64, _u64, _p, _p, _u64, _p, _p]),
    "psg_neighbor_result_free": (None, [_p]),
    "psg_build_reference_set_f64": (_int, [_p, _u64, _u64, _u64, _f64, _u64, _p, _p, _p, _p]),
    "psg_reference_bound": (_int, [_p, _p, _p, _u64, _p]),
    "psg_pointset_from_f32": (_int, [_p, _u64, _u64, _int, _p]),
    "psg_pointset_from_f64": (_int, [_p, _u64, _u64, _int, _p]),
    "psg_pointset_windows_f64": (_int, [_p, _u64, _u64, _int, _int, _p]),
    "psg_pointset_windows_f32": (_int, [_p, _u64, _u64, _int, _int, _p]),
    "psg_pointset_free": (None, [_p]),
    "psg_pointset_size": (_u64, [_p]),
    "psg_pointset_dim": (_u64, [_p]),
    "psg_closest_pair_ps": (_int, [_p, _u64, _f64, _u64, _u64, _p]),
    "psg_brute_force_closest_pair_ps": (_int, [_p, _u64, _p]),
    "psg_fixed_radius_neighbors_ps": (_int, [_p, _f64, _u64, _f64, _u64, _u64, _int, _p]),
    "psg_cpp_plan_create": (_int, [_p, _u64, _f64, _u64, _u64, _p]),
    "psg_cpp_plan_bootstrap": (_int, [_p, _u64, _u64, _p]),
    "psg_cpp_plan_scan": (_int, [_p, _u64, _u64, _f32, _p]),
    "psg_cpp_plan_free": (None, [_p]),
    "psg_frnn_plan_create": (_int, [_p, _f64, _u64, _f64, _u64, _u64, _p]),
    "psg_frnn_plan_scan": (_int, [_p, _u64, _u64, _int, _p, _p, _p]),
    "psg_frnn_plan_pairs": (_int, [_p, _u64, _p, _p, _u64]),
    "psg_frnn_plan_free": (None, [_p]),
    "psg_gen_random_walk": (_int, [_u64, _u64, _f64, _p]),
    "psg_gen_uniform": (None, [_u64, _u64, _u64, _p]),
    "psg_gen_gauss_planted": (None, [_u64, _u64, _u64, _f64, _p, _p, _p]),
    "psg_gen_walk_motif": (None, [_u64, _u64, _u64, _f64, _p, _p, _p]),
    "psg_gen_mixture": (None, [_u64, _u64, _u64, _u64, _f64, _p]),
    "psg_mix_seed": (_u64, [_u64]),
    "psg_derive_seed": (_u64, [_u64, _u64]),
    "psg_host_alloc": (_int, [C.c_size_t, _p]),
    "psg_host_free": (None, [_p]),
    "psg_debug_projection": (_int, [_p, _u64, _u64, _p, _p, _p, _p, _p]),
    "psg_debug_brute_bounded_ps": (_int, [_p, _u64, _f64, _p]),
    "psg_load_series_text": (_int, [C.c_char_p, _p, _p]),
    "psg_save_series_text": (_int, [C.c_char_p, _p, _u64]),
    "psg_free": (None, [_p]),
    "psg_save_binary": (_int, [C.c_char_p, _p, _int, _u64, _u64]),
    "psg_pointset_from_file": (_int, [C.c_char_p, _p]),
    "psg_pointset_windows_from_file": (_int, [C.c_char_p, _u64, _int, _p]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded C-ABI library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == PSG_OK:
        return
    msg = lib().psg_last_error().decode()
    if rc == PSG_ERR_INVALID:
        raise InvalidArgument(msg)
    if rc == PSG_ERR_NOMEM:
        raise MemoryError(msg)
    if rc == PSG_ERR_IO:
        raise SeriesFileError(msg)
    raise DeviceError(msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def set_graph_profiling(level: int) -> None:
    """Event timing inside the CUDA graphs that repeated solves on a point set
    replay: 0 (default) none, 1 projection / bootstrap / scan kernel times,
    2 also the per-stage times.  Each event node costs ~5 us per solve."""
    _check(lib().psg_set_graph_profiling(int(level)))


def last_profile() -> dict:
    """Stage timings (CUDA events on the library stream) and counters of the
    last compute call on this thread."""
    p = _Profile()
    lib().psg_last_profile(C.byref(p))
    return {
        "stages": {p.stage_name[i].value.decode(): float(p.stage_ms[i]) for i in range(p.stages)},
        "stage_list": [(p.stage_name[i].value.decode(), float(p.stage_ms[i])) for i in range(p.stages)],
        "launches": p.launches, "window_pairs": p.window_pairs, "lb_survivors": p.lb_survivors,
        "candidates": p.candidates, "bootstrap_width": p.bootstrap_width,
        "h2d_bytes": p.h2d_bytes, "d2h_bytes": p.d2h_bytes,
        "scan_kernel_ms": p.scan_kernel_ms, "project_kernel_ms": p.project_kernel_ms,
        "bootstrap_kernel_ms": p.bootstrap_kernel_ms, "total_ms": p.total_ms, "scan_launches": p.scan_launches,
        "dense_cells": p.dense_cells, "dense_cell_pairs": p.dense_cell_pairs, "dense_groups": p.dense_groups,
        "dense_split_groups": p.dense_split_groups, "dense_tiles": p.dense_tiles, "inline_fp64": p.inline_fp64,
    }


# ---------------------------------------------------------------------------
# Containers (series.hpp)
class TimeSeries:
    """series.hpp:10-20: a real-valued series; values must be finite."""

    def __init__(self, values):
        self.values = np.ascontiguousarray(values, dtype=np.float64)

    def length(self) -> int:
        return int(self.values.size)

    def window_count(self, length: int) -> int:
        if length == 0 or length > self.values.size:  # series.cpp:8-11
            raise InvalidArgument("window length out of range")
        return self.values.size - length + 1

    def window(self, i: int, length: int) -> np.ndarray:
        return self.values[i:i + length]


class PointSet:
    """series.hpp:28-44.  Holds the host copy and, after the first solve, a
    device-resident copy reused by later calls."""

    def __init__(self):
        self._flat = None      # (n, d) float32 or float64, or None for windows
        self._series = None    # TimeSeries for window sets
        self._len = 0
        self._znorm = False
        self._handle = None
        self._n = 0
        self._d = 0

    @classmethod
    def from_flat(cls, flat, dim: int) -> "PointSet":
        arr = np.asarray(flat)
        if arr.dtype != np.float32:
            arr = np.asarray(arr, dtype=np.float64)
        arr = np.ascontiguousarray(arr).reshape(-1)
        if dim == 0:
            raise InvalidArgument("point dimension must be positive")  # series.cpp:20
        if arr.size % dim != 0:
            raise InvalidArgument("flat buffer not a multiple of dim")  # series.cpp:21
        if not np.all(np.isfinite(arr)):
            raise InvalidArgument("point coordinate must be finite")  # series.cpp:22-24
        ps = cls()
        ps._flat = arr.reshape(-1, dim)
        ps._n, ps._d = ps._flat.shape
        return ps

    @classmethod
    def windows_of(cls, series: "TimeSeries | np.ndarray", length: int, znorm: bool = False) -> "PointSet":
        ts = series if isinstance(series, TimeSeries) else TimeSeries(series)
        n = ts.window_count(length)
        ps = cls()
        ps._series = ts
        ps._len = length
        ps._znorm = znorm
        ps._n, ps._d = n, length
        return ps

    def size(self) -> int:
        return self._n

    def dim(self) -> int:
        return self._d

    def point(self, i: int) -> np.ndarray:
        if self._flat is not None:
            return self._flat[i]
        w = self._series.values[i:i + self._len]
        if not self._znorm:
            return w
        mu = w.sum() / self._len
        sd = np.sqrt(((w - mu) ** 2).sum() / self._len)
        return np.zeros_like(w) if sd == 0 else (w - mu) / sd

    def _device(self) -> int:
        """Create (once) the device-resident copy; returns the handle."""
        if self._handle is None:
            h = _p()
            if self._flat is not None:
                if self._flat.dtype == np.float32:
                    _check(lib().psg_pointset_from_f32(_ptr(self._flat), self._n, self._d, 0, C.byref(h)))
                else:
                    _check(lib().psg_pointset_from_f64(_ptr(self._flat), self._n, self._d, 0, C.byref(h)))
            else:
                v = self._series.values
                _check(lib().psg_pointset_windows_f64(_ptr(v), v.size, self._len, int(self._znorm), 0, C.byref(h)))
            self._handle = h
        return self._handle

    def release(self) -> None:
        if self._handle is not None and _lib is not None:
            _lib.psg_pointset_free(self._handle)
        self._handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Results (refscan.hpp:13-48)
@dataclass
class ScanStats:
    pairs_examined: int = 0
    pairs_pruned_by_reference: int = 0
    pairs_skipped_by_exit: int = 0
    inner_loop_exits: int = 0

    def admissible_pairs(self) -> int:  # refscan.hpp:33-35
        return self.pairs_examined + self.pairs_pruned_by_reference + self.pairs_skipped_by_exit


@dataclass
class PairResult:
    index_i: int = 0
    index_j: int = 0
    distance: float = 0.0
    stats: ScanStats = field(default_factory=ScanStats)


@dataclass
class NeighborResult:
    neighbors: list  # list of np.ndarray (uint64), ascending, symmetric
    stats: ScanStats = field(default_factory=ScanStats)
    pair_count: int = 0
    pair_hash: int = 0
    offsets: np.ndarray | None = None
    flat: np.ndarray | None = None


@dataclass
class ReferenceSet:
    q: int
    f: float
    dim: int
    ref_indices: np.ndarray
    references: np.ndarray  # q x dim
    dist_table: np.ndarray  # q x n (k-major)
    order: np.ndarray

    def dist(self, ref: int, point_index: int, n: int | None = None) -> float:
        return float(self.dist_table[ref, point_index])


def _stats(s: _Stats) -> ScanStats:
    return ScanStats(s.pairs_examined, s.pairs_pruned_by_reference, s.pairs_skipped_by_exit, s.inner_loop_exits)


def _pair(r: _Pair) -> PairResult:
    return PairResult(int(r.index_i), int(r.index_j), float(r.distance), _stats(r.stats))


def _neigh(r: _Neigh, want_lists: bool) -> NeighborResult:
    out = NeighborResult(neighbors=[], stats=_stats(r.stats), pair_count=int(r.pair_count), pair_hash=int(r.pair_hash))
    if want_lists and r.offsets:
        n = int(r.n)
        off = np.ctypeslib.as_array(r.offsets, shape=(n + 1,)).copy()
        m = int(off[-1])
        flat = np.ctypeslib.as_array(r.neighbors, shape=(max(m, 1),))[:m].copy()
        out.offsets, out.flat = off, flat
        out.neighbors = [flat[off[i]:off[i + 1]] for i in range(n)]
    lib().psg_neighbor_result_free(C.byref(r))
    return out


# ---------------------------------------------------------------------------
# refscan.hpp entry points
def closest_pair(points: PointSet, q: int, f: float, seed: int, exclusion_zone: int) -> PairResult:
    """refscan.hpp:55-56 / refscan.cpp:67-132: exact closest admissible pair."""
    out = _Pair()
    _check(lib().psg_closest_pair_ps(points._device(), q, f, seed, exclusion_zone, C.byref(out)))
    return _pair(out)


def brute_force_closest_pair(points: PointSet, exclusion_zone: int) -> PairResult:
    """refscan.hpp:58 / refscan.cpp:134-157 (on device)."""
    out = _Pair()
    _check(lib().psg_brute_force_closest_pair_ps(points._device(), exclusion_zone, C.byref(out)))
    return _pair(out)


def brute_force_bounded(points: PointSet, exclusion_zone: int, upper: float) -> PairResult:
    """Test inspection: the exhaustive minimum over pairs at FP64 distance <=
    `upper` in one all-pairs pass (psg_debug_brute_bounded_ps)."""
    out = _Pair()
    _check(lib().psg_debug_brute_bounded_ps(points._device(), exclusion_zone, float(upper), C.byref(out)))
    return _pair(out)


def fixed_radius_neighbors(points: PointSet, radius: float, q: int, f: float, seed: int,
                           exclusion_zone: int = 0, want_lists: bool = True) -> NeighborResult:
    """refscan.hpp:61-63 / refscan.cpp:159-209: boundary-inclusive lists."""
    if points.size() == 0:
        raise InvalidArgument("empty input")  # refscan.cpp:162
    out = _Neigh()
    _check(lib().psg_fixed_radius_neighbors_ps(points._device(), radius, q, f, seed, exclusion_zone,
                                               int(want_lists), C.byref(out)))
    return _neigh(out, want_lists)


def brute_force_neighbors(points: PointSet, radius: float, exclusion_zone: int = 0) -> list:
    """refscan.hpp:65-66 / refscan.cpp:211-227 (on device)."""
    if points.size() == 0:
        raise InvalidArgument("empty input")
    if points._flat is None:
        raise InvalidArgument("brute_force_neighbors needs a flat point set here")
    flat = np.ascontiguousarray(points._flat, dtype=np.float64)
    out = _Neigh()
    _check(lib().psg_brute_force_neighbors_f64(_ptr(flat), points.size(), points.dim(), radius, exclusion_zone, 1,
                                               C.byref(out)))
    return _neigh(out, True).neighbors


class PinnedBuffer:
    """Page-locked host memory (psg_host_alloc) viewed as a numpy array: the
    device writes into it at full PCIe rate.  Freed with the object."""

    def __init__(self, count: int, dtype=np.uint64):
        self.dtype = np.dtype(dtype)
        self.count = int(count)
        p = _p()
        _check(lib().psg_host_alloc(max(self.count, 1) * self.dtype.itemsize, C.byref(p)))
        self._p = p
        self.array = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)),
                                           shape=(max(self.count, 1) * self.dtype.itemsize,)).view(self.dtype)[:self.count]

    def __del__(self):
        if getattr(self, "_p", None):
            lib().psg_host_free(self._p)
            self._p = None


def frnn_pairs(points: np.ndarray, radius: float, q: int = 10, f: float = 10.0, seed: int = 1,
               exclusion_zone: int = 0, want_pairs: bool = True, out: np.ndarray | None = None):
    """Sorted i<j pair list ((i<<32)|j), count and order-independent hash.

    `out` (optional, uint64, e.g. PinnedBuffer(...).array) receives the list;
    when it is too small only the count and hash are returned."""
    pts = np.ascontiguousarray(points, dtype=np.float32)
    n, d = pts.shape
    cnt, h = _u64(), _u64()
    if not want_pairs:
        _check(lib().psg_frnn_pairs_f32(_ptr(pts), n, d, radius, q, f, seed, exclusion_zone, None, 0,
                                        C.byref(cnt), C.byref(h)))
        return None, cnt.value, h.value
    if out is not None:
        _check(lib().psg_frnn_pairs_f32(_ptr(pts), n, d, radius, q, f, seed, exclusion_zone, _ptr(out), out.size,
                                        C.byref(cnt), C.byref(h)))
        return (out[: cnt.value] if cnt.value <= out.size else None), cnt.value, h.value
    cap = max(40 * n, 1 << 16)
    while True:
        buf = np.empty(cap, np.uint64)
        _check(lib().psg_frnn_pairs_f32(_ptr(pts), n, d, radius, q, f, seed, exclusion_zone, _ptr(buf), cap,
                                        C.byref(cnt), C.byref(h)))
        if cnt.value <= cap:
            return buf[: cnt.value], cnt.value, h.value
        cap = cnt.value


def frnn_pairs_csr(points: np.ndarray, radius: float, q: int = 10, f: float = 10.0, seed: int = 1,
                   exclusion_zone: int = 0, offsets: np.ndarray | None = None, cols: np.ndarray | None = None):
    """The sorted i<j list as upper-triangular CSR: (offsets[n+1] uint64,
    cols uint32, count, hash); row i is cols[offsets[i]:offsets[i+1]].

    `offsets` / `cols` (optional, e.g. pinned arrays) receive the output; when
    `cols` is too small only the offsets, count and hash are complete."""
    pts = np.ascontiguousarray(points, dtype=np.float32)
    n, d = pts.shape
    cnt, h = _u64(), _u64()
    if offsets is None:
        offsets = np.empty(n + 1, np.uint64)
    if cols is None:
        cap = max(40 * n, 1 << 16)
        while True:
            cols = np.empty(cap, np.uint32)
            _check(lib().psg_frnn_pairs_csr_f32(_ptr(pts), n, d, radius, q, f, seed, exclusion_zone, _ptr(offsets),
                                                _ptr(cols), cap, C.byref(cnt), C.byref(h)))
            if cnt.value <= cap:
                return offsets, cols[: cnt.value], cnt.value, h.value
            cap = cnt.value
    _check(lib().psg_frnn_pairs_csr_f32(_ptr(pts), n, d, radius, q, f, seed, exclusion_zone, _ptr(offsets),
                                        _ptr(cols), cols.size, C.byref(cnt), C.byref(h)))
    return offsets, (cols[: cnt.value] if cnt.value <= cols.size else None), cnt.value, h.value


def build_reference_set(points: PointSet, q: int, f: float, seed: int) -> ReferenceSet:
    """refscan.hpp:50-51 / refscan.cpp:30-65, bit-exact (FP64 on device)."""
    if points._flat is None:
        raise InvalidArgument("build_reference_set needs a flat point set here")
    n, d = points.size(), points.dim()
    flat = np.ascontiguousarray(points._flat, dtype=np.float64)
    qq = max(q, 1)
    ri = np.zeros(qq, np.uint64)
    refs = np.zeros(qq * d)
    table = np.zeros(max(qq * n, 1))
    order = np.zeros(max(n, 1), np.uint64)
    _check(lib().psg_build_reference_set_f64(_ptr(flat), n, d, q, f, seed, _ptr(ri), _ptr(refs), _ptr(table),
                                             _ptr(order)))
    return ReferenceSet(q, f, d, ri[:q], refs[: q * d].reshape(q, d), table[: q * n].reshape(q, n), order[:n])


def reference_bound(r, x, y) -> float:
    """refscan.hpp:70-71: d(r, x) - d(r, y)."""
    r, x, y = (np.ascontiguousarray(v, dtype=np.float64) for v in (r, x, y))
    if not (r.size == x.size == y.size):
        raise InvalidArgument("dimension mismatch")  # metrics.cpp:10-12
    out = _f64()
    _check(lib().psg_reference_bound(_ptr(r), _ptr(x), _ptr(y), x.size, C.byref(out)))
    return out.value


def motif(series, length: int, q: int = 10, f: float = 10.0, seed: int = 1, exclusion_zone: int | None = None,
          znorm: bool = True) -> PairResult:
    """cmd_motif (main.cpp:332-346): closest pair over windows, zone = length by default."""
    s = np.ascontiguousarray(series)
    zone = length if exclusion_zone is None else exclusion_zone
    out = _Pair()
    if s.dtype == np.float32:
        _check(lib().psg_motif_f32(_ptr(s), s.size, length, int(znorm), q, f, seed, zone, C.byref(out)))
    else:
        s = np.ascontiguousarray(s, dtype=np.float64)
        _check(lib().psg_motif_f64(_ptr(s), s.size, length, int(znorm), q, f, seed, zone, C.byref(out)))
    return _pair(out)


# ---------------------------------------------------------------------------
class gen:
    """Seeded synthetic inputs (host C++, datagen.cpp + SURVEY §8(d) recipes)."""

    @staticmethod
    def random_walk(n: int, seed: int, stddev: float = 1.0) -> np.ndarray:
        out = np.zeros(n)
        if lib().psg_gen_random_walk(n, seed, stddev, _ptr(out)) != PSG_OK:
            raise InvalidArgument("walk length must be positive")
        return out

    @staticmethod
    def uniform(master: int, n: int, dim: int) -> np.ndarray:
        out = np.zeros((n, dim), np.float32)
        lib().psg_gen_uniform(master, n, dim, _ptr(out))
        return out

    @staticmethod
    def gauss_planted(master: int, n: int, dim: int, noise: float = 1e-3):
        out = np.zeros((n, dim), np.float32)
        i, j = _u64(), _u64()
        lib().psg_gen_gauss_planted(master, n, dim, noise, _ptr(out), C.byref(i), C.byref(j))
        return out, (i.value, j.value)

    @staticmethod
    def walk_motif(master: int, length: int, window: int, noise: float = 0.01):
        out = np.zeros(length, np.float32)
        a, b = _u64(), _u64()
        lib().psg_gen_walk_motif(master, length, window, noise, _ptr(out), C.byref(a), C.byref(b))
        return out, (a.value, b.value)

    @staticmethod
    def mixture(master: int, n: int, dim: int, clusters: int = 1024, sigma: float = 0.05) -> np.ndarray:
        out = np.zeros((n, dim), np.float32)
        lib().psg_gen_mixture(master, n, dim, clusters, sigma, _ptr(out))
        return out

    @staticmethod
    def mix_seed(x: int) -> int:
        return lib().psg_mix_seed(x)

    @staticmethod
    def derive_seed(base: int, stream: int) -> int:
        return lib().psg_derive_seed(base, stream)


def debug_projection(points: "PointSet", q: int = 10, seed: int = 1):
    """Test hook: the projection keys of `points` as a solve computes them,
    the directions, the charged key-error bound E and the working-unit scale
    (keys approximate <U_k, scale * x_i>; |key - exact| <= E is the filter's
    assumption)."""
    n, d = points.size(), points.dim()
    nk = C.c_int(0)
    probe = lib().psg_debug_projection(points._device(), q, seed, C.byref(nk), None, None, None, None)
    _check(probe)
    keys = np.empty((n, nk.value), dtype=np.float32)
    dirs = np.empty((nk.value, d), dtype=np.float32)
    E, scale = C.c_double(0), C.c_double(0)
    _check(lib().psg_debug_projection(points._device(), q, seed, C.byref(nk), keys.ctypes.data, dirs.ctypes.data,
                                      C.byref(E), C.byref(scale)))
    return keys, dirs, E.value, scale.value


# ---- data formats ------------------------------------------------------
def load_series_text(path: str) -> np.ndarray:
    """io.cpp:44-60 load_series (one decimal real per line, strtod values, the
    reference's messages), parsed in parallel; needs no GPU."""
    out, n = C.c_void_p(), _u64()
    _check(lib().psg_load_series_text(os.fsencode(path), C.byref(out), C.byref(n)))
    vals = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_double)), shape=(n.value,)).copy()
    lib().psg_free(out)
    return vals


def save_series_text(values, path: str) -> None:
    """io.cpp:62-70 save_series: '%.17g' per line."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    _check(lib().psg_save_series_text(os.fsencode(path), _ptr(v), v.size))


def save_binary(array, path: str) -> None:
    """.psgb: 32-byte header + row-major f32/f64 values (a 1-D array is one column)."""
    a = np.ascontiguousarray(array)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    rows, cols = (a.shape[0], 1) if a.ndim == 1 else a.shape
    _check(lib().psg_save_binary(os.fsencode(path), _ptr(a), 2 if a.dtype == np.float32 else 1, rows, cols))


class FilePointSet(PointSet):
    """A device point set read straight from a .psgb file (psg_pointset_from_file
    / psg_pointset_windows_from_file): no host copy of the rows is kept."""

    def __init__(self, path: str, window: int = 0, znorm: bool = False):
        super().__init__()
        h = _p()
        if window:
            _check(lib().psg_pointset_windows_from_file(os.fsencode(path), window, int(znorm), C.byref(h)))
        else:
            _check(lib().psg_pointset_from_file(os.fsencode(path), C.byref(h)))
        self._handle = h
        self._n = int(lib().psg_pointset_size(h))
        self._d = int(lib().psg_pointset_dim(h))

    def point(self, i: int):
        raise InvalidArgument("FilePointSet keeps its rows on the device only")
