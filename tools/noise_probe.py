"""Per-kernel times of inject_impulse (run under ncu --metrics gpu__time_duration.sum)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1201_3972_b200 import _native
lib = _native.load_lib()
n = 8192 * 8192
src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
out = torch.empty_like(src); fl = torch.empty_like(src)
for _ in range(3):
    _native.check(lib.irdn_inject_impulse_u8(src.data_ptr(), out.data_ptr(), fl.data_ptr(), n, 42, 0.2, 0.5, None,
                                             torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
