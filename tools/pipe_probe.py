"""Copy-only pipeline probe: chunked H2D on one stream, D2H of chunk i after H2D of chunk i
on another (no kernel), vs one big concurrent pair — isolates the transfer pattern."""
import sys, time, torch
n = 42 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def pipe(chunk_mb, ramp=False):
    c = chunk_mb << 20
    sizes = []
    rem = n
    if ramp:
        s = 1 << 19
        while s < c and rem > 0:
            sizes.append(min(s, rem)); rem -= sizes[-1]; s *= 2
    while rem > 0:
        sizes.append(min(c, rem)); rem -= sizes[-1]
    if ramp and len(sizes) > 2:  # shrink the tail symmetric to the head
        tail = []
        big = sizes.pop()
        s = 1 << 19
        while s < c and big > s:
            tail.append(s); big -= s; s *= 2
        sizes += [big] + tail[::-1]
    evs = []
    off = 0
    for sz in sizes:
        with torch.cuda.stream(s1):
            d[off:off + sz].copy_(h[off:off + sz], non_blocking=True)
            e = torch.cuda.Event(); e.record(s1)
        with torch.cuda.stream(s2):
            s2.wait_event(e)
            h2[off:off + sz].copy_(d[off:off + sz], non_blocking=True)
        off += sz
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
for mb in (2, 4, 8, 16):
    print(f"chunk {mb} MB: {t(lambda: pipe(mb)):.3f} ms   ramped: {t(lambda: pipe(mb, True)):.3f} ms")
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
print(f"one concurrent pair: {t(both):.3f} ms")
