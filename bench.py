#!/usr/bin/env python
"""bench.py — exact closest pair on B200, BASELINE.json config 2.

Workload (N=1): C2 = n = 2^20 points, d = 128, float32 N(0,1) with one planted
near-duplicate (SURVEY §8(d) recipe, master seed 2), solved exactly with the
reference CLI defaults q=10, f=10, seed=1, zone 0.  A step = one complete
solve of that point set (projection, key sort, delta bootstrap, windowed
candidate scan, FP64 recheck).  The input (512 MiB) is larger than L2 (126
MB), and every step re-reads it from HBM.

Metric unit: admissible pairs resolved per second = n(n-1)/2 / solve time
(the rate at which the exact answer over all pairs is certified; the same
unit for the CPU reference arm, which solves bounded n = 2^14 samples).  The
primary quantity is `solve_time_s`; `value` is measured with the point set
already resident in HBM; `e2e` goes through the public C ABI from pinned host
memory (H2D copy inside every step); `e2e_pageable_f64` is the drop-in call a
reference caller makes (PointSet::from_flat(std::vector<double>), i.e. FP64 rows
in pageable memory through psg_closest_pair_f64).

Beside it, in the same run: `same_n` (the GPU and the unmodified reference on
the identical n = 2^14 C2 sample, one solve each), `cpu_fit` (the reference
timed at n = 2^13..2^15, t = a n^b, measured points and the extrapolation to
2^20 reported separately), `configs` (C1 on both arms, C3 one-shot, C4
count+hash and sorted list, C5), and under torchrun a `c5_scaling` line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N ... bench.py --gpus N   (one rank per GPU)
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CDEV = None  # collectives' tensor device override (PSG_BENCH_GLOO test mode)
METRIC = "closest-pair solve time & candidate dist-evals/s at n=2^20,d=128 vs roofline"
UNIT = "pairs/s"
N_C2, D_C2, Q, F, SEED = 1 << 20, 128, 10, 10.0, 1
CPU_SAMPLE_N = 1 << 14


def env_int(k, d):
    return int(os.environ.get(k, d))


def load_bf16_sustained():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh).get("bf16_tflops_sustained", 1376.0))
    return 1376.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            j = json.load(fh)
        return float(j["hbm_gbs"]), float(j.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_reference_rate(n: int, threads: int, reps: int = 1):
    """The unmodified reference closest_pair (oracle/_ref) on the C2 recipe at
    n points, `threads` independent solves in parallel (ctypes drops the GIL)."""
    import oracle

    ref = oracle.reference()
    kind = "reference"
    orc = oracle.port()
    pts, _ = orc.gen_gauss_planted(2, n, D_C2)
    pts64 = pts.astype(np.float64)
    if ref is None:
        kind = "port"
        solve = lambda: orc.brute_force_closest_pair(pts, 0)  # noqa: E731
    else:
        solve = lambda: ref.closest_pair(pts64, Q, F, SEED, 0)  # noqa: E731
    results = [None] * threads

    def work(k):
        for _ in range(reps):
            results[k] = solve()

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(k,)) for k in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    pairs = n * (n - 1) // 2 * threads * reps
    return pairs / wall, wall, kind, results[0]


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = CPU_SAMPLE_N
    for _ in range(args.warmup):
        cpu_reference_rate(n, threads)
    t0 = time.perf_counter()
    walls = []
    for _ in range(args.steps):
        rate, wall, kind, res = cpu_reference_rate(n, threads)
        walls.append(wall)
    total = time.perf_counter() - t0
    pairs = n * (n - 1) // 2 * threads * args.steps
    value = pairs / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY §8(d) C2 recipe, master seed 2)",
        "config": {"workload": f"C2 recipe sample: n={n}, d={D_C2}, {threads} independent solves per step "
                               f"(full C2 n=2^20 is ~1 day single-threaded, SURVEY §6)",
                   "q": Q, "f": F, "seed": SEED, "zone": 0},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"reference closest_pair on the C2 recipe at n={n}, d={D_C2}, "
                                   f"{threads} threads x 1 solve per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result": {"index_i": res.index_i, "index_j": res.index_j, "distance": res.distance},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
C4_N, C4_R = 1 << 22, float.fromhex("0x1.902ce9269f6dp-7")
C4_EXPECT = (66173431, 8231864707796938076)  # oracle cell-grid FRNN (tests/test_gpu_fullsize.py)


C4_INSTR_PER_CAND = 868812561 / 420761475  # ncu, k_frnn_cells count+hash at C4 (profiles/r02_ncu_frnn_cells.txt)
C4_SM_HZ = 1965e6  # clocks.max.sm of the pool's B200s (the bench's clocks sampler reports the run's)


def candidate_kernel_c4(hbm_gbs, peak_kind, reps=3):
    """North-star check of the candidate-distance kernel where it is the hot
    spot: C4 (FRNN, n=2^22, d=3, ~32 neighbours), count + hash on a resident
    point set.  SURVEY §8(d) streaming model: one candidate = one d-dim FP32
    distance streaming 4d bytes, so the roofline is HBM / 4d candidates/s
    (546 G/s at d=3).  Kernel time = the scan stage's CUDA events (the cell
    scan + the rounding-band kernel) on the library stream."""
    import paper_1407_5609_b200 as psg

    pc = psg.PointSet.from_flat(psg.gen.uniform(4, C4_N, 3), 3)
    psg.fixed_radius_neighbors(pc, C4_R, Q, F, SEED, 0, want_lists=False)  # warm-up
    ms, cands, ok = [], 0, True
    for _ in range(reps):
        r = psg.fixed_radius_neighbors(pc, C4_R, Q, F, SEED, 0, want_lists=False)
        p = psg.last_profile()
        ms.append(dict(p["stage_list"])["scan"])
        cands = p["window_pairs"]
        ok = ok and (r.pair_count, r.pair_hash) == C4_EXPECT
    t = min(ms)
    rate = cands / (t / 1e3)
    roof = hbm_gbs * 1e9 / (4 * 3)
    return {"kernel": "k_frnn_cells (+ k_frnn_band)", "config": "C4 FRNN n=2^22 d=3 R=cbrt(3*32/(4 pi n)), count+hash",
            "candidates_per_launch": cands, "kernel_ms": t, "candidates_per_s": rate,
            "roofline_candidates_per_s": roof, "frac": rate / roof, "achieved_gbs": rate * 12 / 1e9,
            "peak": hbm_gbs, "peak_source": peak_kind,
            "model": "SURVEY 8(d): 4d B per candidate (streaming); candidates are re-read from L1/L2, so true DRAM traffic is far lower",
            # the bound the kernel actually meets: SM instruction issue.  Warp-
            # instructions per candidate from ncu (profiles/r02_ncu_frnn_cells.txt:
            # 868.8M executed / 420.8M candidates); peak = 148 SMs x 4 issue/clk
            "issue_model": {"warp_instr_per_candidate": C4_INSTR_PER_CAND,
                            "achieved_ginst_per_s": rate * C4_INSTR_PER_CAND / 1e9,
                            "peak_ginst_per_s": 148 * 4 * C4_SM_HZ / 1e9,
                            "frac": rate * C4_INSTR_PER_CAND / (148 * 4 * C4_SM_HZ)},
            "pairs": r.pair_count, "correct": ok}


# ---------------------------------------------------------------------------
# The reference beside the GPU (rank 0, N = 1): same-n sample, n^b fit, C1.
FIT_LOGN = (13, 14, 15)
C1_N, C1_D = 16384, 2
C5_N, C5_D = 1 << 24, 64
C5_EXPECT = (2449215, 7867199)  # profiles/r02_c5_fullsize.json (device brute force agrees)


def reference_suite(c2_samples, c1_pts):
    """The unmodified reference closest_pair (oracle/_ref) single-threaded on
    the C2 recipe at n = 2^13, 2^14, 2^15 (one solve each, concurrently on
    separate host threads; ctypes drops the GIL) and on C1 at full size, best
    of 3.  Returns the measured points, the t = a n^b fit and the C1 time."""
    import oracle

    ref = oracle.reference()
    if ref is None:
        return None
    times, answers = {}, {}

    def one(logn):
        pts64 = c2_samples[logn].astype(np.float64)
        t0 = time.perf_counter()
        r = ref.closest_pair(pts64, Q, F, SEED, 0)
        times[logn] = time.perf_counter() - t0
        answers[logn] = (r.index_i, r.index_j, r.distance)

    c1 = {}

    def c1_best():
        p64 = c1_pts.astype(np.float64)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = ref.closest_pair(p64, Q, F, SEED, 0)
            ts.append(time.perf_counter() - t0)
        c1.update(best_s=min(ts), answer=(r.index_i, r.index_j, r.distance))

    ths = [threading.Thread(target=one, args=(k,)) for k in sorted(c2_samples, reverse=True)]
    ths.append(threading.Thread(target=c1_best))
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    ns = np.array([float(1 << k) for k in sorted(times)])
    ts = np.array([times[k] for k in sorted(times)])
    b, loga = np.polyfit(np.log(ns), np.log(ts), 1)
    fit = {"measured": [{"n": 1 << k, "seconds": times[k], "answer": answers[k]} for k in sorted(times)],
           "model": "t = a * n^b, least squares on log t over the measured points",
           "a": float(np.exp(loga)), "b": float(b),
           "extrapolated_c2_full_s": float(np.exp(loga) * float(N_C2) ** b),
           "extrapolated": True, "note": "the n = 2^20 time is an extrapolation, not a measurement",
           "threads_per_solve": 1, "nproc": os.cpu_count()}
    return {"fit": fit, "c1": c1, "times": times, "answers": answers}


def gpu_one_shot_f64(L, psg, pts, reps=3):
    """The drop-in call: FP64 rows in pageable host memory through
    psg_closest_pair_f64 (H2D, validation, narrowing, solve); best wall time."""
    pts64 = np.ascontiguousarray(pts, dtype=np.float64)
    n, d = pts64.shape
    ts, r = [], None
    for k in range(reps + 1):
        out = psg._Pair()
        t0 = time.perf_counter()
        psg._check(L.psg_closest_pair_f64(pts64.ctypes.data, n, d, Q, F, SEED, 0, C.byref(out)))
        if k:
            ts.append(time.perf_counter() - t0)
        r = psg._pair(out)
    return min(ts), r


def gpu_resident(psg, ps, reps=5, zone=0):
    ts, dev, r = [], [], None
    for k in range(reps + 1):
        t0 = time.perf_counter()
        r = psg.closest_pair(ps, Q, F, SEED, zone)
        if k:
            ts.append(time.perf_counter() - t0)
            dev.append(psg.last_profile()["total_ms"])
    return min(ts), min(dev), r, psg.last_profile()


def configs_block(L, psg, hbm, bf16_sus):
    """Every BASELINE config at full size, device-resident and end to end."""
    out = {}
    # C1
    c1 = psg.gen.uniform(1, C1_N, C1_D)
    ps = psg.PointSet.from_flat(c1, C1_D)
    t, dev, r, _ = gpu_resident(psg, ps)
    te, re_ = gpu_one_shot_f64(L, psg, c1)
    out["c1"] = {"workload": "C1 CPP n=16384 d=2 U[0,1)^2", "resident_s": t, "device_ms": dev,
                 "e2e_f64_pageable_s": te, "answer": [r.index_i, r.index_j, r.distance],
                 "e2e_answer_same": (re_.index_i, re_.index_j, re_.distance) == (r.index_i, r.index_j, r.distance)}
    ps.release()
    # C3: one-shot from the host series (window build, z-norm statistics, solve)
    s, (a, b) = psg.gen.walk_motif(3, 1 << 20, 256)
    s64 = s.astype(np.float64)
    ts = []
    for k in range(4):
        t0 = time.perf_counter()
        r = psg.motif(s64, 256, Q, F, SEED)
        if k:
            ts.append(time.perf_counter() - t0)
    ps = psg.PointSet.windows_of(s64, 256, znorm=True)
    t, dev, rr, prof = gpu_resident(psg, ps, zone=256)
    out["c3"] = {"workload": "C3 TSMM N=2^20 l=256 z-normalised, zone 256", "one_shot_s": min(ts),
                 "resident_s": t, "device_ms": dev, "answer": [r.index_i, r.index_j, r.distance],
                 "correct": (r.index_i, r.index_j) == tuple(sorted((a, b)))
                 and (rr.index_i, rr.index_j, rr.distance) == (r.index_i, r.index_j, r.distance)}
    ps.release()
    # C4: the sorted (i<j) pair list into pinned host memory
    cube = psg.gen.uniform(4, C4_N, 3)
    pinned = psg.PinnedBuffer(20 * C4_N)
    ts = []
    for k in range(3):
        t0 = time.perf_counter()
        pairs, cnt, h = psg.frnn_pairs(cube, C4_R, Q, F, SEED, 0, want_pairs=True, out=pinned.array)
        if k:
            ts.append(time.perf_counter() - t0)
    prof = psg.last_profile()
    ok = (cnt, h) == C4_EXPECT and bool(np.all(pairs[1:] > pairs[:-1]))
    out["c4_list"] = {"workload": "C4 FRNN n=2^22 d=3, sorted i<j pair list to pinned host (from pageable points)",
                      "one_shot_s": min(ts), "pairs": cnt, "d2h_bytes": cnt * 8,
                      "stages_ms": dict(prof["stage_list"]), "correct": ok}
    del pinned
    # C4 again, the same list as upper-triangular CSR (u64 offsets + u32 columns)
    poff = psg.PinnedBuffer(C4_N + 1)
    pcols = psg.PinnedBuffer(20 * C4_N, np.uint32)
    ts = []
    for k in range(3):
        t0 = time.perf_counter()
        off, cols, c2, h2 = psg.frnn_pairs_csr(cube, C4_R, Q, F, SEED, 0, offsets=poff.array, cols=pcols.array)
        if k:
            ts.append(time.perf_counter() - t0)
    prof = psg.last_profile()
    ok2 = (c2, h2) == C4_EXPECT and int(off[-1]) == c2 and bool(np.all(np.diff(off.astype(np.int64)) >= 0))
    out["c4_csr"] = {"workload": "C4 FRNN n=2^22 d=3, the sorted i<j lists as upper-triangular CSR to pinned host "
                                 "(from pageable points)",
                     "one_shot_s": min(ts), "pairs": c2, "d2h_bytes": c2 * 4 + (C4_N + 1) * 8,
                     "stages_ms": dict(prof["stage_list"]), "correct": ok2}
    del poff, pcols
    # C5
    pts = psg.gen.mixture(5, C5_N, C5_D, 1024, 0.05)
    ps = psg.PointSet.from_flat(pts, C5_D)
    t, dev, r, prof = gpu_resident(psg, ps, reps=2)
    gram_flop = prof["dense_tiles"] * 3 * 2 * 128 * 128 * C5_D
    out["c5"] = {"workload": "C5 CPP n=2^24 d=64, 1024-cluster mixture", "resident_s": t, "device_ms": dev,
                 "answer": [r.index_i, r.index_j, r.distance], "correct": (r.index_i, r.index_j) == C5_EXPECT,
                 "dense_tiles": prof["dense_tiles"], "scan_kernel_ms": prof["scan_kernel_ms"],
                 "gram_tflops_issued": gram_flop / (prof["scan_kernel_ms"] / 1e3) / 1e12 if prof["scan_kernel_ms"] else None,
                 "tf32_peak_derived_tflops": bf16_sus / 2, "stages_ms": dict(prof["stage_list"])}
    ps.release()
    return out


def c5_scaling(psg, L, rank, world, local_rank, coll, barrier):
    """C5 (the ≥6x north_star config) under torchrun: rank 0 alone, then all
    ranks on key-range parts; device time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1407_5609_b200 import sharded

    pts = psg.gen.mixture(5, C5_N, C5_D, 1024, 0.05)
    ps = psg.PointSet.from_flat(pts, C5_D)
    adm = sharded.admissible_pairs(C5_N, 0)
    t1 = None
    if rank == 0:
        psg.closest_pair(ps, Q, F, SEED, 0)
        t0 = time.perf_counter()
        psg.closest_pair(ps, Q, F, SEED, 0)
        t1 = time.perf_counter() - t0
    dist.barrier()

    def sharded_solve():
        plan = sharded.DevicePlan(ps._device(), Q, F, SEED, 0)
        b = coll.all_reduce_min(plan.bootstrap(rank, world))
        res = sharded.combine(coll.all_gather(plan.scan(rank, world, b)), adm)
        plan.close()
        return res

    sharded_solve()  # warm-up
    stream = torch.cuda.ExternalStream(L.psg_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    r = sharded_solve()
    e1.record(stream)
    barrier()
    wall = time.perf_counter() - t0
    t = torch.tensor([wall, e0.elapsed_time(e1) / 1e3], device=CDEV or f"cuda:{local_rank}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ps.release()
    return {"workload": "C5 CPP n=2^24 d=64 mixture, key-range parts (replicated points)", "n_gpus": world,
            "solve_s_max_over_ranks": float(t[0]), "device_span_s_max_over_ranks": float(t[1]),
            "solve_s_1gpu": t1, "speedup_vs_1gpu": (t1 / float(t[0])) if t1 else None,
            "answer": [r.index_i, r.index_j, r.distance], "correct": (r.index_i, r.index_j) == C5_EXPECT}


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1407_5609_b200 as psg
    from paper_1407_5609_b200 import sharded

    L = psg.lib()
    psg._check(L.psg_set_device(local_rank))
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

    n, d = N_C2, D_C2
    # seeded input in pinned host memory (the e2e source)
    nbytes = n * d * 4
    hp = C.c_void_p()
    psg._check(L.psg_host_alloc(nbytes, C.byref(hp)))
    host = np.ctypeslib.as_array((C.c_float * (n * d)).from_address(hp.value)).reshape(n, d)
    pi, pj = C.c_uint64(), C.c_uint64()
    L.psg_gen_gauss_planted(2, n, d, 1e-3, hp.value, C.byref(pi), C.byref(pj))
    planted = tuple(sorted((pi.value, pj.value)))
    stream = torch.cuda.ExternalStream(L.psg_stream())
    adm = sharded.admissible_pairs(n, 0)
    coll = sharded.TorchCollectives(device=CDEV or f"cuda:{local_rank}") if world > 1 else None

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        stream.synchronize()

    def solve_resident(ph, profile=True):
        if world == 1:
            out = psg._Pair()
            psg._check(L.psg_closest_pair_ps(ph, Q, F, SEED, 0, C.byref(out)))
            return psg._pair(out), ([psg.last_profile()] if profile else [])
        plan = sharded.DevicePlan(ph, Q, F, SEED, 0)
        profs = []
        b = plan.bootstrap(rank, world)
        if profile:
            profs.append(psg.last_profile())
        b = coll.all_reduce_min(b)
        local = plan.scan(rank, world, b)
        if profile:
            profs.append(psg.last_profile())
        res = sharded.combine(coll.all_gather(local), adm)
        plan.close()
        return res, profs

    # ---- device-resident timing ------------------------------------------------
    ph = C.c_void_p()
    psg._check(L.psg_pointset_from_f32(hp.value, n, d, 0, C.byref(ph)))
    for _ in range(args.warmup):
        res, _ = solve_resident(ph)
    agg = {"scan": 0.0, "project": 0.0, "bootstrap": 0.0, "launches": 0, "scan_launches": 0,
           "window_pairs": 0, "lb_survivors": 0, "candidates": 0, "stages": {}}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        ev0.record(stream)
        results = []
        for _ in range(args.steps):  # the timed solves: no profile read-back in the loop
            res, _ = solve_resident(ph, profile=False)
            results.append(res)
        ev1.record(stream)
        barrier()
    # per-kernel times and counters: the same K solves again, untimed, each
    # followed by its psg_last_profile read-back; the replayed graphs carry
    # the three kernel spans here only (the timed graphs hold no event nodes)
    psg.set_graph_profiling(1)
    for _ in range(args.steps):
        res, profs = solve_resident(ph)
        results.append(res)
        for p in profs:
            agg["scan"] += p["scan_kernel_ms"]
            agg["project"] += p["project_kernel_ms"]
            agg["bootstrap"] += p["bootstrap_kernel_ms"]
            agg["launches"] += p["launches"]
            agg["scan_launches"] += p["scan_launches"]
            agg["window_pairs"] += p["window_pairs"]
            agg["lb_survivors"] += p["lb_survivors"]
            agg["candidates"] += p["candidates"]
            for k, v in p["stage_list"]:
                agg["stages"][k] = agg["stages"].get(k, 0.0) + v
    psg.set_graph_profiling(0)
    t_ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([t_ms], device=CDEV or f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    ok = all((r.index_i, r.index_j) == planted for r in results)
    K = args.steps
    value = K * adm / (t_ms / 1000.0)

    # ---- end-to-end through the public C ABI, from pinned host memory ----------
    e2e_steps = max(1, min(K, args.e2e_steps))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(args.warmup + e2e_steps):
        if it == args.warmup:  # warm-up calls first (memory pool growth, first-touch)
            barrier()
            e0.record(stream)
        if world == 1:
            out = psg._Pair()
            psg._check(L.psg_closest_pair_f32(hp.value, n, d, Q, F, SEED, 0, C.byref(out)))
            r = psg._pair(out)
        else:
            ph2 = C.c_void_p()
            psg._check(L.psg_pointset_from_f32(hp.value, n, d, 0, C.byref(ph2)))
            r, _ = solve_resident(ph2)
            L.psg_pointset_free(ph2)
        ok = ok and (r.index_i, r.index_j) == planted
    e1.record(stream)
    barrier()
    e_ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([e_ms], device=CDEV or f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e_value = e2e_steps * adm / (e_ms / 1000.0)

    # ---- roofline of the dominant kernel ------------------------------------------
    def ncu_traffic(kernel):
        """dram read+write bytes per launch of `kernel` from the committed ncu
        capture (profiles/r01_traffic.json), or None."""
        try:
            with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")) as fh:
                t = json.load(fh)[kernel]
            return t["dram_bytes_read"] + t["dram_bytes_write"]
        except (OSError, KeyError, ValueError):
            return None

    hbm, bf16, peak_kind = load_peaks()
    per = {k: agg[k] / K for k in ("scan", "project", "bootstrap")}
    dom = max(per, key=per.get)
    nk = 8
    if dom == "project":
        alg_bytes = n * d * 4 + n * nk * 4
        launches = 1
        achieved = alg_bytes / (per["project"] / 1e3) / 1e9
        roof = {"kernel": "k_project_tc<8,128> (tcgen05.mma kind::tf32, TMA-fed)", "bound": "hbm",
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": ncu_traffic("k_project_tc<8,128>"),
                "alg_bytes_per_launch": alg_bytes, "peak_source": peak_kind}
    else:
        # streaming model: every pair the kernel examines streams
        # its partner's keys (nk x 4 B); every FP32 distance streams 4d bytes.
        wp = agg["window_pairs"] / K
        ev = agg["lb_survivors"] / K
        alg_bytes = wp * nk * 4 + ev * 4 * d
        ms = per[dom]
        achieved = alg_bytes / (ms / 1e3) / 1e9
        roof = {"kernel": "k_scan<8>" if dom == "scan" else "k_bootstrap<8>", "bound": "hbm", "achieved": achieved,
                "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                "alg_bytes_per_launch": alg_bytes, "peak_source": peak_kind,
                "model": "window pairs x 4*nk B + FP32 evals x 4d B (streaming; SMEM reuse can exceed 1)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 filter / f64 recheck", "data": "synthetic (SURVEY §8(d) C2 recipe, master seed 2)",
        "config": {"workload": "C2: exact closest pair, n=2^20, d=128, N(0,1) + planted near-duplicate",
                   "q": Q, "f": F, "seed": SEED, "zone": 0, "parallelism": f"key-range x{world}",
                   "l2": "input 512 MiB > 126 MB L2 (re-read from HBM every step)"},
        "solve_time_s": t_ms / K / 1e3,
        # the whole solve against the one pass over the input it cannot avoid
        "solve_roofline": {"alg_bytes": n * d * 4 + n * 8 * 4, "solve_s": t_ms / K / 1e3,
                           "achieved_gbs": (n * d * 4 + n * 8 * 4) / (t_ms / K / 1e3) / 1e9,
                           "frac": (n * d * 4 + n * 8 * 4) / (t_ms / K / 1e3) / 1e9 / load_peaks()[0]},
        "candidate_evals_per_s": agg["lb_survivors"] / (t_ms / 1e3),
        "kernel_ms_per_step": per, "stage_ms_per_step": {k: v / K for k, v in agg["stages"].items()},
        "window_pairs_per_step": agg["window_pairs"] / K, "fp32_evals_per_step": agg["lb_survivors"] / K,
        "fp64_candidates_per_step": agg["candidates"] / K,
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 56,
                "ms_per_step": e_ms / e2e_steps, "steps": e2e_steps},
        "gpu_launches": agg["launches"],
        "clocks": clk.summary(),
        "correct": ok, "answer": {"planted": planted, "got": [results[-1].index_i, results[-1].index_j],
                                  "distance": results[-1].distance},
    }
    if world == 1:
        # the drop-in path: FP64 rows in pageable memory (a std::vector<double>)
        tp, rp = gpu_one_shot_f64(L, psg, host, reps=3)
        ok = ok and (rp.index_i, rp.index_j) == planted
        line["e2e_pageable_f64"] = {"value": adm / tp, "unit": UNIT, "solve_s": tp, "h2d_bytes_per_step": n * d * 8,
                                    "d2h_bytes_per_step": 56, "call": "psg_closest_pair_f64 (pageable host FP64)"}
    L.psg_pointset_free(ph)
    if world == 1 and rank == 0 and not args.no_candidate_kernel:
        line["candidate_kernel"] = candidate_kernel_c4(hbm, peak_kind)
        line["correct"] = line["correct"] and line["candidate_kernel"]["correct"]
    if world == 1 and rank == 0 and not args.no_configs:
        cfg = configs_block(L, psg, hbm, load_bf16_sustained())
        line["configs"] = cfg
        line["correct"] = (line["correct"] and cfg["c3"]["correct"] and cfg["c4_list"]["correct"]
                           and cfg["c4_csr"]["correct"] and cfg["c5"]["correct"])
    if world > 1 and not args.no_configs:
        line["c5_scaling"] = c5_scaling(psg, L, rank, world, local_rank, coll, barrier)
        line["correct"] = line["correct"] and line["c5_scaling"]["correct"]
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        # same-n: the identical n = 2^14 C2 sample on the GPU and the reference
        samples = {k: psg.gen.gauss_planted(2, 1 << k, D_C2)[0] for k in FIT_LOGN}
        g_res_s, g_dev_ms, g_r, _ = gpu_resident(psg, psg.PointSet.from_flat(samples[14], D_C2))
        g_e2e_s, g_e2e_r = gpu_one_shot_f64(L, psg, samples[14])
        c1_pts = psg.gen.uniform(1, C1_N, C1_D)
        suite = reference_suite(samples, c1_pts)
        rate, wall, kind, _ = cpu_reference_rate(CPU_SAMPLE_N, threads)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                                "sample": f"reference closest_pair (oracle/_ref, unmodified) on the C2 recipe at "
                                          f"n={CPU_SAMPLE_N}, d={D_C2}; {threads} threads x 1 solve, {wall:.1f}s"}
        if suite is not None:
            ref_s = suite["times"][14]
            same = suite["answers"][14] == (g_r.index_i, g_r.index_j, g_r.distance) == (
                g_e2e_r.index_i, g_e2e_r.index_j, g_e2e_r.distance)
            line["same_n"] = {"n": 1 << 14, "d": D_C2, "sample": "C2 recipe (master seed 2) at n=2^14",
                              "ref_solve_s": ref_s, "ref_threads": 1,
                              "gpu_e2e_f64_pageable_s": g_e2e_s, "gpu_resident_s": g_res_s,
                              "gpu_device_ms": g_dev_ms, "speedup_e2e": ref_s / g_e2e_s,
                              "speedup_resident": ref_s / g_res_s, "same_answer": same}
            line["cpu_fit"] = suite["fit"]
            if "configs" in line:
                c1 = line["configs"]["c1"]
                c1["ref_best_of_3_s"] = suite["c1"]["best_s"]
                c1["ref_answer"] = suite["c1"]["answer"]
                c1["same_answer"] = tuple(suite["c1"]["answer"]) == tuple(c1["answer"])
                c1["speedup_e2e"] = suite["c1"]["best_s"] / c1["e2e_f64_pageable_s"]
            line["correct"] = line["correct"] and same
    L.psg_host_free(hp)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0 if ok else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--no-candidate-kernel", action="store_true", help="skip the C4 candidate-kernel roofline line")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block (C1, C3, C4 list, C5)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist

        global CDEV
        if os.environ.get("PSG_BENCH_GLOO") == "1":
            # test mode: every rank on the one visible GPU, host collectives
            # (the ranks never wait on each other inside a kernel)
            CDEV = "cpu"
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        return run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
