import torch
n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for chunk_mb in (512, 128, 64, 32, 16, 8):
    c = chunk_mb << 20
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record()
        for o in range(0, n, c):
            d[o:o + c].copy_(h[o:o + c], non_blocking=True)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print("512 MiB in %d MiB chunks: %.3f ms = %.1f GB/s" % (chunk_mb, best, n / best / 1e6), flush=True)
