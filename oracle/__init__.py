"""ctypes bindings for the test-infrastructure checkers.

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / ``--impl reference`` legs; the product package
``paper_1407_5609_b200`` never imports this module.

``port``      — the C restatement in oracle/oracle.c (liboracle.so).
``reference`` — the unmodified reference core compiled into
                oracle/_ref/libpairscan_ref.so (None when it was not built).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u64 = C.c_uint64
_f64 = C.c_double
_p = C.c_void_p

R_C4 = float.fromhex("0x1.902ce9269f6dp-7")  # the cbrt value, pinned


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class _OrcPair(C.Structure):
    _fields_ = [("index_i", _u64), ("index_j", _u64), ("distance", _f64), ("pairs_examined", _u64)]


class _RefPair(C.Structure):
    _fields_ = [
        ("index_i", _u64), ("index_j", _u64), ("distance", _f64),
        ("pairs_examined", _u64), ("pairs_pruned_by_reference", _u64),
        ("pairs_skipped_by_exit", _u64), ("inner_loop_exits", _u64),
    ]


@dataclass
class Pair:
    index_i: int
    index_j: int
    distance: float
    pairs_examined: int = 0
    pairs_pruned_by_reference: int = 0
    pairs_skipped_by_exit: int = 0
    inner_loop_exits: int = 0


class OracleError(ValueError):
    pass


def build(quiet: bool = True) -> None:
    """Compile liboracle.so, and oracle/_ref when /root/reference exists."""
    import subprocess

    targets = ["all"] if os.path.isdir("/root/reference/proj/core/src") else [os.path.join(HERE, "liboracle.so")]
    subprocess.run(["make", "-C", HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class Port:
    """The C restatement (oracle/oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_mix_seed.restype = _u64
        L.orc_mix_seed.argtypes = [_u64]
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _u64]
        L.orc_rng_next.restype = _u64
        L.orc_uniform_below.restype = _u64
        L.orc_uniform_below.argtypes = [_p, _u64]
        L.orc_gaussian.restype = _f64
        L.orc_gaussian.argtypes = [_p, _f64, _f64]
        L.orc_rng_seed.argtypes = [_p, _u64]
        L.orc_rng_next.argtypes = [_p]
        L.orc_sample_without_replacement.argtypes = [_p, _u64, _u64, _p]
        L.orc_gen_random_walk.argtypes = [_u64, _u64, _f64, _p]
        L.orc_euclidean.restype = _f64
        L.orc_euclidean.argtypes = [_p, _p, _u64]
        L.orc_euclidean_early_abandon.argtypes = [_p, _p, _u64, _f64, _p]
        L.orc_reference_bound.restype = _f64
        L.orc_reference_bound.argtypes = [_p, _p, _p, _u64]
        L.orc_brute_force_closest_pair.argtypes = [_p, _u64, _u64, _u64, _p]
        L.orc_brute_force_closest_pair_f32.argtypes = [_p, _u64, _u64, _u64, _p]
        L.orc_brute_force_neighbors.argtypes = [_p, _u64, _u64, _f64, _u64, _p, _p, _p, _u64]
        L.orc_frnn_grid_f32.argtypes = [_p, _u64, _u64, _f64, _u64, _p, _p]
        L.orc_build_reference_set.argtypes = [_p, _u64, _u64, _u64, _f64, _u64, _p, _p, _p, _p]
        L.orc_znorm_windows.argtypes = [_p, _u64, _u64, _p]
        L.orc_motif_brute_znorm.argtypes = [_p, _u64, _u64, _u64, _p]
        L.orc_znorm_pair_distance.restype = _f64
        L.orc_znorm_pair_distance.argtypes = [_p, _u64, _u64, _u64]
        L.orc_gen_uniform_u24.argtypes = [_u64, _u64, _u64, _p]
        L.orc_gen_gauss_planted.argtypes = [_u64, _u64, _u64, _f64, _p, _p, _p]
        L.orc_gen_walk_motif.argtypes = [_u64, _u64, _u64, _f64, _p, _p, _p]
        L.orc_gen_mixture.argtypes = [_u64, _u64, _u64, _u64, _f64, _p]

    # --- rng --------------------------------------------------------------
    def rng(self, seed: int):
        buf = C.create_string_buffer(312 * 8 + 16)
        self.lib.orc_rng_seed(buf, seed)
        return buf

    def rng_stream(self, seed: int, count: int) -> np.ndarray:
        r = self.rng(seed)
        return np.array([self.lib.orc_rng_next(r) for _ in range(count)], dtype=np.uint64)

    def gaussian_stream(self, seed: int, mean: float, sd: float, count: int) -> np.ndarray:
        r = self.rng(seed)
        return np.array([self.lib.orc_gaussian(r, mean, sd) for _ in range(count)])

    def uniform_below_stream(self, seed: int, bound: int, count: int) -> np.ndarray:
        r = self.rng(seed)
        return np.array([self.lib.orc_uniform_below(r, bound) for _ in range(count)], dtype=np.uint64)

    def sample_without_replacement(self, seed: int, n: int, k: int) -> np.ndarray:
        out = np.zeros(max(k, 1), dtype=np.uint64)
        if self.lib.orc_sample_without_replacement(self.rng(seed), n, k, _ptr(out)) != 0:
            raise OracleError("sample_without_replacement: k exceeds n")
        return out[:k]

    def mix_seed(self, x: int) -> int:
        return self.lib.orc_mix_seed(x)

    def derive_seed(self, base: int, stream: int) -> int:
        return self.lib.orc_derive_seed(base, stream)

    def gen_random_walk(self, n: int, seed: int, sd: float = 1.0) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        if self.lib.orc_gen_random_walk(n, seed, sd, _ptr(out)) != 0:
            raise OracleError("walk length must be positive")
        return out

    # --- metrics ------------------------------------------------------------
    def euclidean(self, x, y) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        return self.lib.orc_euclidean(_ptr(x), _ptr(y), x.size)

    def early_abandon(self, x, y, thr: float):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = _f64()
        ok = self.lib.orc_euclidean_early_abandon(_ptr(x), _ptr(y), x.size, thr, C.byref(out))
        return out.value if ok else None

    def reference_bound(self, r, x, y) -> float:
        r, x, y = (np.ascontiguousarray(v, dtype=np.float64) for v in (r, x, y))
        return self.lib.orc_reference_bound(_ptr(r), _ptr(x), _ptr(y), x.size)

    # --- refscan ------------------------------------------------------------
    def brute_force_closest_pair(self, pts: np.ndarray, zone: int = 0) -> Pair:
        pts = np.ascontiguousarray(pts)
        n, d = pts.shape
        out = _OrcPair()
        if pts.dtype == np.float32:
            rc = self.lib.orc_brute_force_closest_pair_f32(_ptr(pts), n, d, zone, C.byref(out))
        else:
            pts = np.ascontiguousarray(pts, dtype=np.float64)
            rc = self.lib.orc_brute_force_closest_pair(_ptr(pts), n, d, zone, C.byref(out))
        if rc == -1:
            raise OracleError("closest_pair needs at least 2 points")
        if rc == -2:
            raise OracleError("no admissible pair")
        return Pair(out.index_i, out.index_j, out.distance, out.pairs_examined)

    def brute_force_neighbors(self, pts: np.ndarray, radius: float, zone: int = 0, lists: bool = False):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        n, d = pts.shape
        cnt, h = _u64(), _u64()
        cap = n * (n - 1) // 2 if lists else 0
        buf = np.zeros(max(cap, 1), dtype=np.uint64)
        rc = self.lib.orc_brute_force_neighbors(_ptr(pts), n, d, radius, zone, C.byref(cnt), C.byref(h),
                                                _ptr(buf) if lists else None, cap)
        if rc != 0:
            raise OracleError("radius must be positive" if n else "empty input")
        return (cnt.value, h.value, buf[: cnt.value].copy()) if lists else (cnt.value, h.value)

    def frnn_grid(self, pts: np.ndarray, radius: float, zone: int = 0):
        pts = np.ascontiguousarray(pts, dtype=np.float32)
        n, d = pts.shape
        cnt, h = _u64(), _u64()
        if self.lib.orc_frnn_grid_f32(_ptr(pts), n, d, radius, zone, C.byref(cnt), C.byref(h)) != 0:
            raise OracleError("frnn_grid failed")
        return cnt.value, h.value

    def build_reference_set(self, pts: np.ndarray, q: int, f: float, seed: int):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        n, d = pts.shape
        ri = np.zeros(max(q, 1), np.uint64)
        refs = np.zeros(max(q * d, 1))
        table = np.zeros(max(q * n, 1))
        order = np.zeros(max(n, 1), np.uint64)
        if self.lib.orc_build_reference_set(_ptr(pts), n, d, q, f, seed, _ptr(ri), _ptr(refs), _ptr(table), _ptr(order)) != 0:
            raise OracleError("invalid reference set arguments")
        return ri[:q], refs[: q * d].reshape(q, d), table[: q * n].reshape(q, n), order[:n]

    def znorm_windows(self, series: np.ndarray, l: int) -> np.ndarray:
        s = np.ascontiguousarray(series, dtype=np.float64)
        nw = s.size - l + 1
        out = np.zeros((nw, l))
        if self.lib.orc_znorm_windows(_ptr(s), s.size, l, _ptr(out)) != 0:
            raise OracleError("window length out of range")
        return out

    def znorm_pair_distance(self, series: np.ndarray, l: int, i: int, j: int) -> float:
        s = np.ascontiguousarray(series, dtype=np.float64)
        return self.lib.orc_znorm_pair_distance(_ptr(s), l, i, j)

    def motif_brute_znorm(self, series: np.ndarray, l: int, zone: int) -> Pair:
        s = np.ascontiguousarray(series, dtype=np.float64)
        out = _OrcPair()
        rc = self.lib.orc_motif_brute_znorm(_ptr(s), s.size, l, zone, C.byref(out))
        if rc != 0:
            raise OracleError("no admissible pair" if rc == -2 else "window length out of range")
        return Pair(out.index_i, out.index_j, out.distance, out.pairs_examined)

    # --- configs --------------------------------------------------------------
    def gen_uniform(self, master: int, n: int, d: int) -> np.ndarray:
        out = np.zeros((n, d), np.float32)
        self.lib.orc_gen_uniform_u24(master, n, d, _ptr(out))
        return out

    def gen_gauss_planted(self, master: int, n: int, d: int, noise: float = 1e-3):
        out = np.zeros((n, d), np.float32)
        i, j = _u64(), _u64()
        self.lib.orc_gen_gauss_planted(master, n, d, noise, _ptr(out), C.byref(i), C.byref(j))
        return out, (i.value, j.value)

    def gen_walk_motif(self, master: int, N: int, l: int, noise: float = 0.01):
        out = np.zeros(N, np.float32)
        a, b = _u64(), _u64()
        self.lib.orc_gen_walk_motif(master, N, l, noise, _ptr(out), C.byref(a), C.byref(b))
        return out, (a.value, b.value)

    def gen_mixture(self, master: int, n: int, d: int, k: int = 1024, sigma: float = 0.05) -> np.ndarray:
        out = np.zeros((n, d), np.float32)
        self.lib.orc_gen_mixture(master, n, d, k, sigma, _ptr(out))
        return out


class Reference:
    """The unmodified reference core (oracle/_ref/libpairscan_ref.so)."""

    PATH = os.path.join(HERE, "_ref", "libpairscan_ref.so")

    def __init__(self, path: str | None = None):
        L = self.lib = C.CDLL(path or self.PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_stream.argtypes = [_u64, _u64, _p]
        L.ref_gaussian_stream.argtypes = [_u64, _f64, _f64, _u64, _p]
        L.ref_uniform_below_stream.argtypes = [_u64, _u64, _u64, _p]
        L.ref_sample_without_replacement.argtypes = [_u64, _u64, _u64, _p]
        L.ref_mix_seed.restype = _u64
        L.ref_mix_seed.argtypes = [_u64]
        L.ref_derive_seed.restype = _u64
        L.ref_derive_seed.argtypes = [_u64, _u64]
        L.ref_gen_random_walk.argtypes = [_u64, _u64, _f64, _p]
        if hasattr(L, "ref_load_series"):
            L.ref_load_series.argtypes = [C.c_char_p, _p, _p]
            L.ref_save_series.argtypes = [_p, _u64, C.c_char_p]
            L.ref_free.argtypes = [_p]
        if hasattr(L, "ref_report_render"):
            L.ref_report_render.argtypes = [C.c_char_p] * 3 + [_u64, _u64, _f64, _u64, _u64, _f64, _u64, _p, _p]
            L.ref_derive_seed3.restype = _u64
            L.ref_derive_seed3.argtypes = [_u64, _u64, _u64]
        L.ref_euclidean.restype = _f64
        L.ref_euclidean.argtypes = [_p, _p, _u64]
        L.ref_euclidean_early_abandon.argtypes = [_p, _p, _u64, _f64, _p]
        L.ref_reference_bound.restype = _f64
        L.ref_reference_bound.argtypes = [_p, _p, _p, _u64]
        L.ref_closest_pair.argtypes = [_p, _u64, _u64, _u64, _f64, _u64, _u64, _p]
        L.ref_brute_force_closest_pair.argtypes = [_p, _u64, _u64, _u64, _p]
        L.ref_closest_pair_windows.argtypes = [_p, _u64, _u64, _u64, _f64, _u64, _u64, _p]
        L.ref_brute_force_closest_pair_windows.argtypes = [_p, _u64, _u64, _u64, _p]
        L.ref_fixed_radius_neighbors.argtypes = [_p, _u64, _u64, _f64, _u64, _f64, _u64, _u64, _p, _p, _p, _u64, _p]
        L.ref_brute_force_neighbors.argtypes = [_p, _u64, _u64, _f64, _u64, _p, _p, _p, _u64]
        L.ref_build_reference_set.argtypes = [_p, _u64, _u64, _u64, _f64, _u64, _p, _p, _p, _p]

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def _err(self):
        raise OracleError(self.lib.ref_last_error().decode())

    def rng_stream(self, seed, count):
        out = np.zeros(count, np.uint64)
        self.lib.ref_rng_stream(seed, count, _ptr(out))
        return out

    def gaussian_stream(self, seed, mean, sd, count):
        out = np.zeros(count)
        self.lib.ref_gaussian_stream(seed, mean, sd, count, _ptr(out))
        return out

    def uniform_below_stream(self, seed, bound, count):
        out = np.zeros(count, np.uint64)
        self.lib.ref_uniform_below_stream(seed, bound, count, _ptr(out))
        return out

    def sample_without_replacement(self, seed, n, k):
        out = np.zeros(max(k, 1), np.uint64)
        if self.lib.ref_sample_without_replacement(seed, n, k, _ptr(out)) != 0:
            self._err()
        return out[:k]

    def mix_seed(self, x):
        return self.lib.ref_mix_seed(x)

    def derive_seed(self, b, s):
        return self.lib.ref_derive_seed(b, s)

    def gen_random_walk(self, n, seed, sd=1.0):
        out = np.zeros(n)
        if self.lib.ref_gen_random_walk(n, seed, sd, _ptr(out)) != 0:
            self._err()
        return out

    def euclidean(self, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        return self.lib.ref_euclidean(_ptr(x), _ptr(y), x.size)

    def early_abandon(self, x, y, thr):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = _f64()
        return out.value if self.lib.ref_euclidean_early_abandon(_ptr(x), _ptr(y), x.size, thr, C.byref(out)) else None

    def load_series(self, path: str):
        """io.cpp load_series: (values or None, rc, message)."""
        out, n = C.c_void_p(), _u64()
        rc = self.lib.ref_load_series(path.encode(), C.byref(out), C.byref(n))
        if rc != 0:
            return None, rc, self.lib.ref_last_error().decode()
        vals = np.ctypeslib.as_array(C.cast(out, C.POINTER(C.c_double)), shape=(n.value,)).copy()
        self.lib.ref_free(out)
        return vals, 0, ""

    def report(self, algorithm, params, dataset, i1, i2, dom, examined, iterations, wall, seed):
        """io.cpp report_to_json / reports_to_csv of one Report: (json, csv)."""
        j, c = C.c_void_p(), C.c_void_p()
        rc = self.lib.ref_report_render(algorithm.encode(), params.encode(), dataset.encode(), i1, i2, dom, examined,
                                        iterations, wall, seed, C.byref(j), C.byref(c))
        if rc != 0:
            self._err()
        out = (C.string_at(j).decode(), C.string_at(c).decode())
        self.lib.ref_free(j)
        self.lib.ref_free(c)
        return out

    def derive_seed3(self, base, s1, s2):
        return self.lib.ref_derive_seed3(base, s1, s2)

    def save_series(self, values, path: str) -> None:
        v = np.ascontiguousarray(values, dtype=np.float64)
        assert self.lib.ref_save_series(v.ctypes.data, v.size, path.encode()) == 0

    def reference_bound(self, r, x, y):
        r, x, y = (np.ascontiguousarray(v, dtype=np.float64) for v in (r, x, y))
        return self.lib.ref_reference_bound(_ptr(r), _ptr(x), _ptr(y), x.size)

    @staticmethod
    def _pair(o):
        return Pair(o.index_i, o.index_j, o.distance, o.pairs_examined, o.pairs_pruned_by_reference,
                    o.pairs_skipped_by_exit, o.inner_loop_exits)

    def closest_pair(self, pts, q=10, f=10.0, seed=1, zone=0) -> Pair:
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        out = _RefPair()
        if self.lib.ref_closest_pair(_ptr(pts), pts.shape[0], pts.shape[1], q, f, seed, zone, C.byref(out)) != 0:
            self._err()
        return self._pair(out)

    def brute_force_closest_pair(self, pts, zone=0) -> Pair:
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        out = _RefPair()
        if self.lib.ref_brute_force_closest_pair(_ptr(pts), pts.shape[0], pts.shape[1], zone, C.byref(out)) != 0:
            self._err()
        return self._pair(out)

    def closest_pair_windows(self, series, l, q=10, f=10.0, seed=1, zone=None) -> Pair:
        s = np.ascontiguousarray(series, dtype=np.float64)
        out = _RefPair()
        if self.lib.ref_closest_pair_windows(_ptr(s), s.size, l, q, f, seed, l if zone is None else zone, C.byref(out)) != 0:
            self._err()
        return self._pair(out)

    def fixed_radius_neighbors(self, pts, radius, q=10, f=10.0, seed=1, zone=0, lists=False):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        n, d = pts.shape
        cnt, h = _u64(), _u64()
        st = np.zeros(4, np.uint64)
        cap = n * (n - 1) // 2 if lists else 0
        buf = np.zeros(max(cap, 1), np.uint64)
        if self.lib.ref_fixed_radius_neighbors(_ptr(pts), n, d, radius, q, f, seed, zone, C.byref(cnt), C.byref(h),
                                               _ptr(buf) if lists else None, cap, _ptr(st)) != 0:
            self._err()
        res = {"count": cnt.value, "hash": h.value, "stats": [int(v) for v in st]}
        if lists:
            res["pairs"] = buf[: cnt.value].copy()
        return res

    def brute_force_neighbors(self, pts, radius, zone=0, lists=False):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        n, d = pts.shape
        cnt, h = _u64(), _u64()
        cap = n * (n - 1) // 2 if lists else 0
        buf = np.zeros(max(cap, 1), np.uint64)
        if self.lib.ref_brute_force_neighbors(_ptr(pts), n, d, radius, zone, C.byref(cnt), C.byref(h),
                                              _ptr(buf) if lists else None, cap) != 0:
            self._err()
        return (cnt.value, h.value, buf[: cnt.value].copy()) if lists else (cnt.value, h.value)

    def build_reference_set(self, pts, q, f, seed):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        n, d = pts.shape
        ri = np.zeros(max(q, 1), np.uint64)
        refs = np.zeros(max(q * d, 1))
        table = np.zeros(max(q * n, 1))
        order = np.zeros(max(n, 1), np.uint64)
        if self.lib.ref_build_reference_set(_ptr(pts), n, d, q, f, seed, _ptr(ri), _ptr(refs), _ptr(table), _ptr(order)) != 0:
            self._err()
        return ri[:q], refs[: q * d].reshape(q, d), table[: q * n].reshape(q, n), order[:n]


_port = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def reference() -> Reference | None:
    return Reference() if Reference.available() else None
