"""Host<->device copy bandwidth with pinned buffers, and the C-ABI host path timing."""
import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = 42 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn, reps=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bi = t(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  concurrent {2*n/bi/1e9:.1f} GB/s total")
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate
lib = _native.load_lib()
cfg = CONFIGS["c2"]
img = generate(cfg)
hin = torch.from_numpy(img.view("int16")).pin_memory(); hout = torch.empty_like(hin).pin_memory()
st = _native.IrdnStats()
for _ in range(2): lib.irdn_run_filter_u16(hin.data_ptr(), hout.data_ptr(), 64, 512, 640, 5, 0, 1, 0, ctypes.byref(st))
t0 = time.perf_counter()
for _ in range(10): lib.irdn_run_filter_u16(hin.data_ptr(), hout.data_ptr(), 64, 512, 640, 5, 0, 1, 0, ctypes.byref(st))
dt = (time.perf_counter() - t0) / 10
print(f"irdn_run_filter_u16 c2: {dt*1e3:.2f} ms/call  {cfg.pixels/dt/1e6:.0f} Mpix/s; bytes each way {img.nbytes/1e6:.1f} MB -> {2*img.nbytes/dt/1e9:.1f} GB/s total")
