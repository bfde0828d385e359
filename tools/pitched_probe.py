"""Throughput of the host path on the reference's 364-pixel rows (pitched device staging).

    python tools/pitched_probe.py      -> stdout
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1201_3972_b200 as P  # noqa: E402

rng = np.random.default_rng(1)
for w in (364, 368):
    img = rng.integers(0, 256, size=(512, 244, w), dtype=np.uint8)
    P.run_filter(img, P.WindowSpec(3), "fnr", 1)
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        P.run_filter(img, P.WindowSpec(3), "fnr", 1)
    dt = (time.perf_counter() - t0) / n
    print(f"width {w}: 512 x 244 x {w} u8, 3x3 FNR, host path {dt * 1e3:.2f} ms "
          f"({img.size / dt / 1e9:.1f} Gpix/s)")
