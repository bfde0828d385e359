"""Why is the per-chunk work slow inside the e2e pipeline? Times one 13-frame c2 chunk's
filter, delta encode (into a device region) and the region's D2H copy (a) back-to-back
warm, (b) after 2 ms of GPU idle, (c) while a 42 MB H2D runs on another stream, (d) both.
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1201_3972_b200 import _native  # noqa: E402
from paper_1201_3972_b200.scene import CONFIGS, generate  # noqa: E402

lib = _native.load_lib()
cfg = CONFIGS["c2"]
frames = generate(cfg, nframes=13)
B, H, W = frames.shape
din = torch.from_numpy(frames.view(np.int16)).cuda()
dout = torch.empty_like(din)
counts = torch.zeros(2, dtype=torch.int64, device="cuda")
big_h = torch.empty(42 << 20, dtype=torch.uint8).pin_memory()
big_d = torch.empty(42 << 20, dtype=torch.uint8, device="cuda")
nreg = int(lib.irdn_delta_region_bytes(din.numel(), 2))
reg = torch.empty(nreg, dtype=torch.uint8, device="cuda")  # device region (as irdn_run_filter_* uses it)
reg_h = torch.empty(nreg, dtype=torch.uint8).pin_memory()
fixed_plus_budget = 16 + 2 * ((din.numel() + 4095) // 4096 * 4 + 15) // 16 * 16 + (din.numel() + 4095) // 4096 * 512 \
    + int(din.numel() * 0.1) * 2
s = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def one(kind):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(s):
        e[0].record(s)
        _native.check(lib.irdn_filter_pass_u16(din.data_ptr(), dout.data_ptr(), B, H, W, W, W, 5, 0,
                                               counts.data_ptr(), s.cuda_stream))
        e[1].record(s)
        if kind == "enc":
            _native.check(lib.irdn_delta_encode_u16(din.data_ptr(), dout.data_ptr(), din.numel(), reg.data_ptr(),
                                                    s.cuda_stream))
        e[2].record(s)
        reg_h[:fixed_plus_budget].copy_(reg[:fixed_plus_budget], non_blocking=True)
        e[3].record(s)
    return e


for mode in ("warm", "idle", "h2d", "idle+h2d"):
    tf, te, td = [], [], []
    for rep in range(20):
        if mode.startswith("idle"):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 2e-3:
                pass
        if "h2d" in mode:
            with torch.cuda.stream(s2):
                big_d.copy_(big_h, non_blocking=True)
            time.sleep(50e-6)
        e = one("enc")
        torch.cuda.synchronize()
        if rep >= 3:
            tf.append(e[0].elapsed_time(e[1]) * 1e3)
            te.append(e[1].elapsed_time(e[2]) * 1e3)
            td.append(e[2].elapsed_time(e[3]) * 1e3)
    print(f"{mode:9s} filter 13 frames: median {np.median(tf):6.1f} us  min {min(tf):6.1f}   "
          f"encode: median {np.median(te):6.1f} us  min {min(te):6.1f}   "
          f"D2H {fixed_plus_budget / 1e6:.2f} MB: median {np.median(td):6.1f} us", flush=True)
