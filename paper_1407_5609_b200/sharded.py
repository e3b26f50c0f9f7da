"""Key-range sharding of the exact closest pair across ranks (one per GPU).

Every rank holds the whole point set (replicated; C2 is 512 MiB of 180 GB)
and builds the same plan (projection + key-0 sort are deterministic), then:

  1. bootstrap its own slice of sorted positions -> local FP32 bound
  2. all-reduce MIN of the bound                  (the one real exchange)
  3. scan its slice with the global bound          -> local best pair
  4. all-gather the per-rank bests, take the lexicographic minimum of
     (FP64 distance, i, j) — ties to the lowest (i, j) like refscan.cpp:118-126

No halo is needed because the points are replicated;
each pair (p, j > p) is owned by exactly one slice: the one holding p.

The combine logic is backend-agnostic so it can be tested on CPU with gloo
and an oracle-backed stand-in (tests/test_sharded.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Protocol, Sequence

from . import PairResult, ScanStats, _check, _f32, _p, _Pair, _pair, lib

NO_PAIR = (1 << 64) - 1


class Backend(Protocol):
    def bootstrap(self, part: int, nparts: int) -> float: ...

    def scan(self, part: int, nparts: int, bound: float) -> PairResult: ...


class DevicePlan:
    """The product backend: psg_cpp_plan_* over the C ABI."""

    def __init__(self, points_handle, q: int, f: float, seed: int, zone: int):
        h = _p()
        _check(lib().psg_cpp_plan_create(points_handle, q, f, seed, zone, C.byref(h)))
        self._h = h

    def bootstrap(self, part: int, nparts: int) -> float:
        out = _f32()
        _check(lib().psg_cpp_plan_bootstrap(self._h, part, nparts, C.byref(out)))
        return float(out.value)

    def scan(self, part: int, nparts: int, bound: float) -> PairResult:
        out = _Pair()
        _check(lib().psg_cpp_plan_scan(self._h, part, nparts, bound, C.byref(out)))
        return _pair(out)

    def close(self) -> None:
        if self._h is not None:
            lib().psg_cpp_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def combine(results: Sequence[PairResult], admissible: int) -> PairResult:
    """Lexicographic minimum of (distance, i, j) over rank-local bests; the
    stats partition identity is restored with the closed-form admissible count."""
    valid = [r for r in results if r.index_i != NO_PAIR]
    if not valid:
        from . import InvalidArgument

        raise InvalidArgument("no admissible pair")
    best = min(valid, key=lambda r: (r.distance, r.index_i, r.index_j))
    ex = sum(r.stats.pairs_examined for r in results)
    pr = sum(r.stats.pairs_pruned_by_reference for r in results)
    pr = min(pr, admissible - ex)
    exits = sum(r.stats.inner_loop_exits for r in results)
    return PairResult(best.index_i, best.index_j, best.distance, ScanStats(ex, pr, admissible - ex - pr, exits))


def admissible_pairs(n: int, zone: int) -> int:
    """main.cpp:388-395 in closed form."""
    if zone <= 1:
        return n * (n - 1) // 2
    if zone >= n:
        return 0
    m = n - zone
    return m * (m + 1) // 2


def closest_pair_sharded(backend: Backend, n: int, zone: int, rank: int, world: int,
                         all_reduce_min: Callable[[float], float],
                         all_gather: Callable[[PairResult], list]) -> PairResult:
    bound = backend.bootstrap(rank, world)
    bound = all_reduce_min(bound)
    local = backend.scan(rank, world, bound)
    return combine(all_gather(local), admissible_pairs(n, zone))


@dataclass
class TorchCollectives:
    """all_reduce_min / all_gather over torch.distributed (nccl or gloo)."""

    device: str = "cpu"
    group: object = None

    def all_reduce_min(self, x: float) -> float:
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float32, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return float(t.item())

    def all_gather(self, r: PairResult) -> list:
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(self.group)
        s = r.stats
        vals = [r.index_i, r.index_j, s.pairs_examined, s.pairs_pruned_by_reference,
                s.pairs_skipped_by_exit, s.inner_loop_exits]
        # ship as int64 bit patterns (+ the FP64 distance) for backend portability
        ints = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v for v in vals], dtype=torch.int64,
                            device=self.device)
        dist_t = torch.tensor([r.distance], dtype=torch.float64, device=self.device)
        outs_i = [torch.empty_like(ints) for _ in range(world)]
        outs_d = [torch.empty_like(dist_t) for _ in range(world)]
        dist.all_gather(outs_i, ints, group=self.group)
        dist.all_gather(outs_d, dist_t, group=self.group)
        res = []
        for oi, od in zip(outs_i, outs_d):
            v = [int(x) & ((1 << 64) - 1) for x in oi.cpu().tolist()]
            res.append(PairResult(v[0], v[1], float(od.cpu().item()), ScanStats(v[2], v[3], v[4], v[5])))
        return res


# ---------------------------------------------------------------------------
# Fixed-radius neighbours (refscan.cpp:159-209), sharded the same way: every
# rank builds the same grid, scans the pairs whose earlier grid-sorted position
# is in its slice, and
#   1. all-reduces (SUM) count, hash (mod 2^64) and stats   -> the totals
#   2. optionally exchanges the sorted pair list by i-range (all-to-all), so
#      rank b ends with the globally sorted pairs whose i lies in
#      [n b / world, n (b + 1) / world) — concatenated over ranks, that is the
#      reference's sorted (i<j) list (main.cpp:465-478 --pairs-out order).
MASK64 = (1 << 64) - 1


class FrnnBackend(Protocol):
    def scan(self, part: int, nparts: int, keep_pairs: bool) -> tuple: ...

    def pairs(self, nbuckets: int) -> tuple: ...


class DeviceFrnnPlan:
    """The product backend: psg_frnn_plan_* over the C ABI."""

    def __init__(self, points_handle, radius: float, q: int, f: float, seed: int, zone: int):
        h = _p()
        _check(lib().psg_frnn_plan_create(points_handle, radius, q, f, seed, zone, C.byref(h)))
        self._h = h
        self._count = 0

    def scan(self, part: int, nparts: int, keep_pairs: bool):
        from . import _Stats, _stats

        cnt, h, st = C.c_uint64(), C.c_uint64(), _Stats()
        _check(lib().psg_frnn_plan_scan(self._h, part, nparts, int(keep_pairs), C.byref(cnt), C.byref(h),
                                        C.byref(st)))
        self._count = cnt.value
        return cnt.value, h.value, _stats(st)

    def pairs(self, nbuckets: int):
        """(sorted uint64 keys of this part, per-i-range bucket counts)."""
        import numpy as np

        out = np.empty(max(self._count, 1), np.uint64)
        counts = np.zeros(nbuckets, np.uint64)
        _check(lib().psg_frnn_plan_pairs(self._h, nbuckets, counts.ctypes.data, out.ctypes.data, out.size))
        return out[: self._count], counts

    def close(self) -> None:
        if self._h is not None:
            lib().psg_frnn_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _limbs(x: int) -> list:
    return [(x >> s) & 0xFFFFFFFF for s in (0, 32)]


def frnn_sharded(backend: FrnnBackend, n: int, zone: int, rank: int, world: int, all_reduce_sum, all_to_all=None):
    """Count, hash and stats summed over ranks; with `all_to_all` also this
    rank's i-range of the globally sorted pair list.  Returns
    (count, hash, ScanStats, pairs or None)."""
    count, h, st = backend.scan(rank, world, keep_pairs=all_to_all is not None)
    # hash is a sum mod 2^64: ship it as two 32-bit limbs so an int64 SUM over
    # any backend cannot overflow
    tot = all_reduce_sum([count, *_limbs(h), st.pairs_examined, st.pairs_pruned_by_reference])
    count_all = tot[0]
    hash_all = (tot[1] + (tot[2] << 32)) & MASK64
    ex, pr = tot[3], tot[4]
    stats = ScanStats(ex, pr, admissible_pairs(n, zone) - ex - pr, 0)
    mine = None
    if all_to_all is not None:
        keys, counts = backend.pairs(world)
        mine = all_to_all(keys, counts)
    return count_all, hash_all, stats, mine


def merge_sorted_runs(runs):
    """The received runs (each sorted) -> one sorted array."""
    import numpy as np

    if not runs:
        return np.empty(0, np.uint64)
    cat = np.concatenate([np.asarray(r, dtype=np.uint64) for r in runs])
    cat.sort(kind="stable")
    return cat


@dataclass
class TorchFrnnCollectives:
    """all_reduce_sum / all_to_all of sorted pair runs over torch.distributed."""

    device: str = "cpu"
    group: object = None

    def all_reduce_sum(self, vals: list) -> list:
        import torch
        import torch.distributed as dist

        t = torch.tensor([int(v) for v in vals], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return [int(x) for x in t.cpu().tolist()]

    def all_to_all(self, keys, counts):
        import numpy as np
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(self.group)
        send_counts = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=self.device)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        # uint64 keys travel as their int64 bit patterns
        send = torch.from_numpy(np.ascontiguousarray(keys).view(np.int64)).to(self.device)
        recv = torch.empty(int(recv_counts.sum()), dtype=torch.int64, device=self.device)
        dist.all_to_all_single(recv, send, output_split_sizes=recv_counts.tolist(),
                               input_split_sizes=send_counts.tolist(), group=self.group)
        got = recv.cpu().numpy().view(np.uint64)
        bounds = np.concatenate([[0], np.cumsum(recv_counts.cpu().numpy())])
        return merge_sorted_runs([got[bounds[r]:bounds[r + 1]] for r in range(world)])
