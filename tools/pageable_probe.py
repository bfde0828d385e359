"""run_filter on a pageable numpy batch vs the pinned-buffer C-ABI path (c2 shape)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
img = generate(cfg)
for _ in range(2): P.run_filter(img, P.WindowSpec(cfg.k), "fnr", 1)
t0 = time.perf_counter()
for _ in range(5): P.run_filter(img, P.WindowSpec(cfg.k), "fnr", 1)
dt = (time.perf_counter() - t0) / 5
print(f"{cfg.name} pageable numpy run_filter: {dt*1e3:.2f} ms -> {img.size/dt/1e6:.0f} Mpix/s")
lib = _native.load_lib()
hin = torch.from_numpy(img.view(np.int16) if img.dtype == np.uint16 else img).pin_memory()
hout = torch.empty_like(hin).pin_memory()
fn = lib.irdn_run_filter_u16 if img.dtype == np.uint16 else lib.irdn_run_filter_u8
B, H, W = img.shape if img.ndim == 3 else (1,) + img.shape
st = _native.IrdnStats()
for _ in range(2): fn(hin.data_ptr(), hout.data_ptr(), B, H, W, cfg.k, 0, 1, 0, ctypes.byref(st))
t0 = time.perf_counter()
for _ in range(5): fn(hin.data_ptr(), hout.data_ptr(), B, H, W, cfg.k, 0, 1, 0, ctypes.byref(st))
dt = (time.perf_counter() - t0) / 5
print(f"{cfg.name} pinned C-ABI: {dt*1e3:.2f} ms -> {img.size/dt/1e6:.0f} Mpix/s")
