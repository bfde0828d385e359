"""Does splitting a 42 MB H2D over 1 / 2 / 4 streams (separate copy engines) raise the
aggregate host->device bandwidth? (the e2e floor)"""
import time
import torch

n = 42 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    best = 1e9
    for rep in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        if rep >= 2:
            best = min(best, time.perf_counter() - t0)
    print(f"{ns} stream(s): {n / best / 1e9:.1f} GB/s", flush=True)
# chunked 8 MB copies on one stream vs alternating two streams
for ns in (1, 2):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = 8 << 20
    best = 1e9
    for rep in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n // part):
            with torch.cuda.stream(streams[i % ns]):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        if rep >= 2:
            best = min(best, time.perf_counter() - t0)
    print(f"8 MB chunks over {ns} stream(s): {(n // part) * part / best / 1e9:.1f} GB/s", flush=True)
