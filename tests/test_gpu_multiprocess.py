"""GPU: the sharded product path across real processes.

Two processes (ranks) share the one B200 of the test box, each with its own
CUDA context, its own device point set and plan (DevicePlan /
DeviceFrnnPlan over the C ABI), joined by torch.distributed over gloo with
CPU tensors: exactly the code bench.py runs under torchrun with NCCL, minus
the transport.  The ranks never wait on each other inside a kernel (the
exchanges are host-side collectives between whole solve steps), so sharing
one device is safe.  Checked against the single-process solve: closest pair
(grid engine), motif (z-normalised windows, zone = window length) and FRNN
(count, hash and the i-range all-to-all of the sorted list)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1407_5609_b200 as psg
        from paper_1407_5609_b200 import sharded

        psg._check(psg.lib().psg_set_device(0))
        out = {}
        coll = sharded.TorchCollectives(device="cpu")
        # closest pair, C2 recipe at 2^17
        pts, _ = psg.gen.gauss_planted(2, 1 << 17, 128)
        ps = psg.PointSet.from_flat(pts, 128)
        r = sharded.closest_pair_sharded(sharded.DevicePlan(ps._device(), 10, 10.0, 1, 0), ps.size(), 0, rank, world,
                                         coll.all_reduce_min, coll.all_gather)
        out["cpp"] = (r.index_i, r.index_j, r.distance, r.stats.admissible_pairs())
        # motif over z-normalised windows
        s, _ = psg.gen.walk_motif(3, 1 << 16, 128)
        ws = psg.PointSet.windows_of(s.astype(np.float64), 128, znorm=True)
        r = sharded.closest_pair_sharded(sharded.DevicePlan(ws._device(), 10, 10.0, 1, 128), ws.size(), 128, rank,
                                         world, coll.all_reduce_min, coll.all_gather)
        out["motif"] = (r.index_i, r.index_j, r.distance)
        # FRNN, C4 recipe at 2^19
        n = 1 << 19
        cube = psg.gen.uniform(4, n, 3)
        R = (3 * 32 / (4 * np.pi * n)) ** (1 / 3)
        pc = psg.PointSet.from_flat(cube, 3)
        fc = sharded.TorchFrnnCollectives(device="cpu")
        plan = sharded.DeviceFrnnPlan(pc._device(), R, 10, 10.0, 1, 0)
        cnt, h, st, mine = sharded.frnn_sharded(plan, n, 0, rank, world, fc.all_reduce_sum, fc.all_to_all)
        plan.close()
        out["frnn"] = (cnt, h, st.admissible_pairs())
        out["frnn_mine"] = mine
        q.put((rank, out))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu(psg, orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in range(WORLD):
        assert isinstance(res[r], dict), res[r]
    # single-process answers
    pts, planted = psg.gen.gauss_planted(2, 1 << 17, 128)
    one = psg.closest_pair(psg.PointSet.from_flat(pts, 128), 10, 10.0, 1, 0)
    s, _ = psg.gen.walk_motif(3, 1 << 16, 128)
    mot = psg.motif(s.astype(np.float64), 128)
    n = 1 << 19
    cube = psg.gen.uniform(4, n, 3)
    R = (3 * 32 / (4 * np.pi * n)) ** (1 / 3)
    pairs, cnt, h = psg.frnn_pairs(cube, R)
    for r in range(WORLD):
        o = res[r]
        m = 1 << 17
        assert o["cpp"] == (one.index_i, one.index_j, one.distance, m * (m - 1) // 2)
        assert o["motif"] == (mot.index_i, mot.index_j, mot.distance)
        assert o["frnn"] == (cnt, h, n * (n - 1) // 2)
    assert (one.index_i, one.index_j) == tuple(sorted(planted))
    assert (cnt, h) == orc.frnn_grid(cube, R)
    merged = np.concatenate([res[r]["frnn_mine"] for r in range(WORLD)])
    assert np.array_equal(merged, pairs)
    for p in procs:
        assert p.exitcode == 0
