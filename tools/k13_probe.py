"""Large windows: the shared-memory tiled kernel (csrc/fnr_large.cuh) vs the generic one.

    python tools/k13_probe.py      (8 c2-sized u16 frames, FNR, device-resident)
"""
import sys, time, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate
img = generate(CONFIGS['c2'].with_shape(frames=8), nframes=8)
t = torch.from_numpy(img.view(np.int16)).cuda().view(torch.uint16)
lib = _native.load_lib()
for k in (11, 13, 15, 21, 31, 45, 63):
    for generic in (0, 1):
        prev = lib.irdn_set_force_generic(generic)
        P.run_filter(t, P.WindowSpec(k), 'fnr', 1); torch.cuda.synchronize()
        reps = 5 if not generic else 2
        t0 = time.perf_counter()
        for _ in range(reps): P.run_filter(t, P.WindowSpec(k), 'fnr', 1)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / reps
        lib.irdn_set_force_generic(prev)
        print(k, "generic" if generic else "default", f"{dt*1e3:.3f} ms  {img.size/dt/1e6:.0f} Mpix/s", flush=True)
