import torch, time
for mb in (4, 18, 32, 50, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); w = time.perf_counter() - t0
    print("H2D %d MiB pinned: %.3f ms = %.1f GB/s (wall %.3f ms)" % (mb, best, n / best / 1e6, w * 1e3), flush=True)
