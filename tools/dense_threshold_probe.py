"""Where the dense median stage starts to pay (FNR, k = 5 / 7): device-resident timing of
64 frames 640 x 512 with salt-and-pepper density p, for the setting in IRDN_DENSE_FRAC
(run once with 0 = always dense, once with -1 = never). Prints one JSON line per case
with the flagged fraction the counters report.

    IRDN_DENSE_FRAC=0 python tools/dense_threshold_probe.py; IRDN_DENSE_FRAC=-1 python ...
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_3972_b200 import _native  # noqa: E402

lib = _native.load_lib()
rng = np.random.default_rng(5)
B, H, W = 64, 512, 640
y, x = np.mgrid[0:H, 0:W]
base = (60 + 40 * np.sin(x / 37.0) * np.cos(y / 23.0)).astype(np.float64)
for dtype in (np.uint8, np.uint16):
    hi = 255 if dtype == np.uint8 else 16383
    field = np.clip(np.rint(base * hi / 255.0)[None] + rng.normal(0, 2 * hi / 255.0, (B, H, W)), 0, hi).astype(dtype)
    for p in (0.02, 0.05, 0.1, 0.15, 0.2, 0.25, 0.3, 0.4, 0.5):
        img = field.copy()
        m = rng.random(img.shape) < p
        img[m] = np.where(rng.random(int(m.sum())) < 0.5, 0, hi).astype(dtype)
        t_in = torch.from_numpy(img.view(np.int16) if dtype == np.uint16 else img).cuda()
        t_out = torch.empty_like(t_in)
        counts = torch.zeros(2, dtype=torch.int64, device="cuda")
        fn = lib.irdn_filter_pass_u8 if dtype == np.uint8 else lib.irdn_filter_pass_u16
        for k in (5, 7):
            s = torch.cuda.current_stream().cuda_stream

            def run():
                _native.check(fn(t_in.data_ptr(), t_out.data_ptr(), B, H, W, W, W, k, 0, counts.data_ptr(), s))
            for _ in range(3):
                run()
            counts.zero_()
            run()
            det = int(counts[0].item())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(50):
                run()
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"dense_frac": os.environ.get("IRDN_DENSE_FRAC"), "dtype": np.dtype(dtype).name,
                              "k": k, "p": p, "flagged": round(det / img.size, 4),
                              "us": round(e0.elapsed_time(e1) / 50 * 1e3, 2)}), flush=True)
