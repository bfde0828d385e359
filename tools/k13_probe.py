import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1201_3972_b200 as P
from paper_1201_3972_b200.scene import CONFIGS, generate
img = generate(CONFIGS['c2'].with_shape(frames=8), nframes=8)
t = torch.from_numpy(img.view(np.int16)).cuda().view(torch.uint16)
for k in (11, 13, 15):
    P.run_filter(t, P.WindowSpec(k), 'fnr', 1); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): P.run_filter(t, P.WindowSpec(k), 'fnr', 1)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(k, f"{dt*1e3:.2f} ms  {img.size/dt/1e6:.0f} Mpix/s")
