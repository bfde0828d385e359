"""Latency of one host-buffer call (irdn_run_filter_u8) on small frames (c1 / the paper's
364 x 244 image), pinned and pageable buffers: median of 200 calls.

    python tools/small_call_probe.py
"""
import ctypes
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_3972_b200 import _native  # noqa: E402

lib = _native.load_lib()
st = _native.IrdnStats()
import torch  # noqa: E402

for (h, w) in ((512, 512), (244, 364)):
    for pinned in (True, False):
        if pinned:
            a = torch.randint(0, 256, (h * w,), dtype=torch.uint8).pin_memory().numpy()
            b = torch.empty(h * w, dtype=torch.uint8).pin_memory().numpy()
        else:
            a = np.random.default_rng(0).integers(0, 256, h * w, dtype=np.uint8)
            b = np.empty_like(a)
        for _ in range(20):
            _native.check(lib.irdn_run_filter_u8(a.ctypes.data, b.ctypes.data, 1, h, w, 3, 0, 1, 0, ctypes.byref(st)))
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            _native.check(lib.irdn_run_filter_u8(a.ctypes.data, b.ctypes.data, 1, h, w, 3, 0, 1, 0, ctypes.byref(st)))
            ts.append(time.perf_counter() - t0)
        print(f"{h}x{w} {'pinned' if pinned else 'pageable'}: median {statistics.median(ts) * 1e6:.1f} us, "
              f"min {min(ts) * 1e6:.1f} us")
