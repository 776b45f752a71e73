"""Pinned host -> device copy throughput of one 50 MB u8 batch split over
1, 2, 4 streams (diagnostic for the e2e leg's PCIe bound)."""
import time
import torch

n = 16384 * 3072
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    best = 1e9
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part = n // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{ns} stream(s): {n / best / 1e9:.1f} GB/s")
