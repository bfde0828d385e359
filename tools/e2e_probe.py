"""e2e probe: irdn_run_filter_* on pinned host buffers, full vs sparse result return.

    python tools/e2e_probe.py [configs...]   (env: IRDN_COPY_THREADS, IRDN_CHUNK_MB, OMP_WAIT_POLICY ...)

Alternates the two modes call by call (so drift hits both) and prints the median /
min call time and Mpix/s per mode, plus the bytes moved.
"""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1201_3972_b200 import _native  # noqa: E402
from paper_1201_3972_b200.scene import CONFIGS, generate  # noqa: E402

lib = _native.load_lib()
reps = int(os.environ.get("REPS", "30"))
for name in sys.argv[1:] or ["c2", "c4", "c3", "c5"]:
    cfg = CONFIGS[name]
    img = generate(cfg)
    if img.ndim == 2:
        img = img[None]
    B, H, W = img.shape
    hin = torch.from_numpy(img.view(np.int16) if img.dtype == np.uint16 else img).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    fn = lib.irdn_run_filter_u8 if img.dtype == np.uint8 else lib.irdn_run_filter_u16
    st = _native.IrdnStats()
    times = {"full": [], "delta": []}
    xfer = {}
    for i in range(reps + 2):
        for mode in ("full", "delta"):
            _native.set_host_return(mode)
            t0 = time.perf_counter()
            _native.check(fn(hin.data_ptr(), hout.data_ptr(), B, H, W, cfg.k, 0, 1, 0, ctypes.byref(st)))
            dt = time.perf_counter() - t0
            if i >= 2:
                times[mode].append(dt)
            xfer[mode] = _native.last_transfer()
    px = B * H * W
    for mode, ts in times.items():
        med = statistics.median(ts)
        print(f"{name} {mode:5s} median {med*1e3:7.3f} ms  min {min(ts)*1e3:7.3f} ms  "
              f"{px/med/1e6:9.1f} Mpix/s  h2d {xfer[mode][0]/1e6:.1f} MB d2h {xfer[mode][1]/1e6:.1f} MB",
              flush=True)
