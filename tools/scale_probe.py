"""Kernel time vs batch size (tail / launch overhead probe) for one config's frames."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
lib = _native.load_lib()
base = generate(cfg, nframes=min(cfg.frames, 64))
for mult in (1, 2, 4, 8):
    frames = np.concatenate([base] * mult)
    t = torch.from_numpy(frames.view(np.int16 if cfg.dtype == "u16" else np.uint8)).cuda()
    outs = [torch.empty_like(t) for _ in range(2)]
    ins = [t, t.clone()]
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    fn = lib.irdn_filter_pass_u16 if cfg.dtype == "u16" else lib.irdn_filter_pass_u8
    B, H, W = frames.shape
    s = torch.cuda.current_stream().cuda_stream
    for i in range(3): fn(ins[i % 2].data_ptr(), outs[i % 2].data_ptr(), B, H, W, W, W, cfg.k, 0, counts.data_ptr(), s)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for i in range(20): fn(ins[i % 2].data_ptr(), outs[i % 2].data_ptr(), B, H, W, W, W, cfg.k, 0, counts.data_ptr(), s)
    ev[1].record(); torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 20
    print(f"{cfg.name} frames {B}: {ms*1e3:.1f} us/launch, {ms*1e3/B:.3f} us/frame, {B*H*W/ms/1e3:.0f} Mpix/s")
