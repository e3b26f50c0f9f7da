"""CPU: the multi-rank path (paper_1407_5609_b200/sharded.py) over gloo with
world_size 2, using an oracle-backed stand-in for the device plan.

The stand-in mirrors the device contract: every rank holds all points and the
same ordering (the key sort); part p owns the pairs (pos_i, pos_j > pos_i)
whose first position lies in its slice; bootstrap returns an FP32 squared
bound, scan returns the part's exact best under the reference's FP64 order.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_5609_b200 import PairResult, ScanStats
from paper_1407_5609_b200.sharded import NO_PAIR, TorchCollectives, admissible_pairs, closest_pair_sharded, combine


def seq_dist(a, b):
    """The reference's FP64 order (metrics.cpp:16-24), vectorised over pairs."""
    acc = np.zeros(a.shape[0])
    for t in range(a.shape[1]):
        diff = a[:, t] - b[:, t]
        acc = acc + diff * diff
    return np.sqrt(acc)


class OracleBackend:
    def __init__(self, pts, zone):
        self.pts = pts
        self.zone = zone
        self.order = np.argsort(pts[:, 0], kind="stable")  # stands in for the key sort
        self.n = len(pts)

    def _rows(self, part, nparts):
        return self.n * part // nparts, self.n * (part + 1) // nparts

    def _pairs(self, lo, hi):
        out = []
        for p in range(lo, hi):
            i = self.order[p]
            js = self.order[p + 1:]
            ok = np.abs(js.astype(np.int64) - int(i)) >= max(self.zone, 1) if self.zone > 1 else np.ones(len(js), bool)
            for j in js[ok]:
                out.append((min(i, j), max(i, j)))
        return out

    def bootstrap(self, part, nparts):
        lo, hi = self._rows(part, nparts)
        best = np.inf
        for p in range(lo, min(hi, self.n - 1)):
            i, j = self.order[p], self.order[p + 1]
            if self.zone <= 1 or abs(int(i) - int(j)) >= self.zone:
                best = min(best, float(np.float32(seq_dist(self.pts[[i]], self.pts[[j]])[0] ** 2) * 1.001))
        return best

    def scan(self, part, nparts, bound):
        lo, hi = self._rows(part, nparts)
        pairs = self._pairs(lo, hi)
        if not pairs:
            return PairResult(NO_PAIR, NO_PAIR, float("inf"), ScanStats())
        a = np.array(pairs)
        d = seq_dist(self.pts[a[:, 0]], self.pts[a[:, 1]])
        keep = d * d <= bound * 1.01
        cand = [(d[k], int(a[k, 0]), int(a[k, 1])) for k in np.nonzero(keep)[0]]
        dd, i, j = min(cand) if cand else (float("inf"), NO_PAIR, NO_PAIR)
        return PairResult(i, j, dd, ScanStats(int(keep.sum()), len(pairs) - int(keep.sum()), 0, 0))


def _worker(rank, world, port, pts, zone, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = OracleBackend(pts, zone)
        coll = TorchCollectives(device="cpu")
        r = closest_pair_sharded(be, len(pts), zone, rank, world, coll.all_reduce_min, coll.all_gather)
        # every pair owned by exactly one part
        n_owned = sum(len(be._pairs(*be._rows(p, world))) for p in range(world))
        q.put((rank, r.index_i, r.index_j, r.distance, r.stats.admissible_pairs(), n_owned))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("zone", [0, 5])
def test_sharded_closest_pair_world2_gloo(orc, zone):
    rng = np.random.default_rng(7 + zone)
    pts = rng.normal(size=(160, 3))
    pts[99] = pts[12] + 1e-4  # a clear winner ...
    pts[140] = pts[12] + 1e-4  # ... and an exact tie, broken to the lowest (i, j)
    want = orc.brute_force_closest_pair(pts, zone)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, pts, zone, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, i, j, d, adm, owned in res:
        assert (i, j, d) == (want.index_i, want.index_j, want.distance)
        assert adm == admissible_pairs(160, zone)
        assert owned == admissible_pairs(160, zone)


def test_combine_lexicographic_and_stats():
    a = PairResult(5, 9, 1.0, ScanStats(2, 3, 0, 1))
    b = PairResult(4, 10, 1.0, ScanStats(1, 4, 0, 1))
    c = PairResult(NO_PAIR, NO_PAIR, float("inf"), ScanStats(0, 7, 0, 0))
    r = combine([a, b, c], 100)
    assert (r.index_i, r.index_j, r.distance) == (4, 10, 1.0)
    assert r.stats.admissible_pairs() == 100 and r.stats.pairs_examined == 3
    with pytest.raises(ValueError, match="no admissible pair"):
        combine([c], 10)


def test_admissible_closed_form():
    for n in range(0, 30):
        for z in range(0, 32):
            brute = sum(1 for i in range(n) for j in range(i + 1, n) if j - i >= max(z, 1))
            assert admissible_pairs(n, z) == brute


# ---------------------------------------------------------------------------
# Sharded FRNN (sharded.frnn_sharded): count/hash SUM and the i-range
# all-to-all of the sorted list, over gloo with an oracle-backed stand-in for
# the device plan (same ownership rule: a pair belongs to the part holding
# its earlier sorted position).
def _mix(k):
    k = (k + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
    k = ((k ^ (k >> 30)) * 0xBF58476D1CE4E5B9) & ((1 << 64) - 1)
    k = ((k ^ (k >> 27)) * 0x94D049BB133111EB) & ((1 << 64) - 1)
    return k ^ (k >> 31)


class OracleFrnnBackend:
    def __init__(self, pts, radius, zone, all_pairs):
        self.n = len(pts)
        order = np.argsort(pts[:, 0], kind="stable")  # stands in for the grid order
        self.pos = np.empty(self.n, np.int64)
        self.pos[order] = np.arange(self.n)
        self.all_pairs = all_pairs  # uint64 (i<<32)|j, i<j
        self.mine = None

    def scan(self, part, nparts, keep_pairs):
        lo, hi = self.n * part // nparts, self.n * (part + 1) // nparts
        i = (self.all_pairs >> np.uint64(32)).astype(np.int64)
        j = (self.all_pairs & np.uint64(0xFFFFFFFF)).astype(np.int64)
        first = np.minimum(self.pos[i], self.pos[j])
        self.mine = self.all_pairs[(first >= lo) & (first < hi)]
        h = 0
        for k in self.mine.tolist():
            h = (h + _mix(int(k))) & ((1 << 64) - 1)
        return len(self.mine), h, ScanStats(len(self.mine), 3, 0, 0)

    def pairs(self, nbuckets):
        keys = np.sort(self.mine)
        i = (keys >> np.uint64(32)).astype(np.int64)
        b = np.minimum((i * nbuckets) // self.n, nbuckets - 1)
        # bucket of i: the b with n b / nb <= i < n (b + 1) / nb
        edges = np.array([self.n * k // nbuckets for k in range(nbuckets + 1)])
        b = np.searchsorted(edges, i, side="right") - 1
        return keys, np.bincount(b, minlength=nbuckets).astype(np.uint64)


def _frnn_worker(rank, world, port, pts, radius, all_pairs, q):
    from paper_1407_5609_b200.sharded import TorchFrnnCollectives, frnn_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = OracleFrnnBackend(pts, radius, 0, all_pairs)
        coll = TorchFrnnCollectives(device="cpu")
        cnt, h, st, mine = frnn_sharded(be, len(pts), 0, rank, world, coll.all_reduce_sum, coll.all_to_all)
        q.put((rank, cnt, h, st.admissible_pairs(), mine.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_frnn_gloo(orc, world):
    rng = np.random.default_rng(3)
    n = 400
    pts = rng.random((n, 3))
    radius = 0.12
    cnt, h, keys = orc.brute_force_neighbors(pts, radius, 0, lists=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_frnn_worker, args=(r, world, port, pts, radius, keys, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, c, hh, adm, _ in res:
        assert (c, hh) == (cnt, h)
        assert adm == n * (n - 1) // 2
    merged = [k for r in res for k in r[4]]  # rank order = i-range order
    assert merged == sorted(int(k) for k in keys)
