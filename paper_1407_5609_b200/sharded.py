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
