import ctypes, os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate
cfg = CONFIGS["c2"]
lib = _native.load_lib()
frames = generate(cfg, nframes=cfg.frames)
t = torch.from_numpy(frames.view(np.int16)).cuda()
t2 = t.clone()
out = torch.empty_like(t); out2 = torch.empty_like(t)
counts = torch.zeros(2, dtype=torch.int64, device="cuda")
fn = lib.irdn_filter_pass_u16
B, H, W = frames.shape
s = torch.cuda.current_stream().cuda_stream
def run(i, o): _native.check(fn(i.data_ptr(), o.data_ptr(), B, H, W, W, W, 5, 0, counts.data_ptr(), s))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for mode in ("sync-same", "sync-alt", "b2b-same", "b2b-alt", "b2b-sameout"):
    ts = []
    for j in range(8):
        ins = (t, out) if (mode.endswith("same") or j % 2 == 0) else (t2, out2)
        if mode == "b2b-sameout": ins = (t if j % 2 == 0 else t2, out)
        if mode.startswith("sync"): torch.cuda.synchronize()
        ev[0].record(); run(*ins); ev[1].record()
        if mode.startswith("sync"): torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    torch.cuda.synchronize()
    if not ts: 
        ev[0].record()
        for j in range(8):
            ins = (t, out) if (mode.endswith("same") or j % 2 == 0) else (t2, out2)
            if mode == "b2b-sameout": ins = (t if j % 2 == 0 else t2, out)
            run(*ins)
        ev[1].record(); torch.cuda.synchronize(); ts = [ev[0].elapsed_time(ev[1]) * 1e3 / 8]
    print(mode, " ".join(f"{x:.1f}" for x in ts))
