"""Per-tile timeline of one warp-kernel launch (needs an -DIRDN_TIMELINE build via IRDN_LIB).

    IRDN_LIB=build_variants/libirdn_tl.so python tools/timeline_probe.py c2 [--dump out.npy]

Each warp tile records globaltimer stamps: before its load wait, load ready, detector
done, tile done, plus its queue length n, warp and SM. Prints how the launch's time
splits into ramp, steady state and tail, and what the last tiles look like.
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dump = sys.argv[sys.argv.index("--dump") + 1] if "--dump" in sys.argv else None
lib = _native.load_lib()
lib.irdn_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int64]
frames = generate(cfg, nframes=cfg.frames)
t = torch.from_numpy(frames.view(np.int16 if cfg.dtype == "u16" else np.uint8)).cuda()
out = torch.empty_like(t)
counts = torch.zeros(2, dtype=torch.int64, device="cuda")
fn = lib.irdn_filter_pass_u16 if cfg.dtype == "u16" else lib.irdn_filter_pass_u8
B, H, W = frames.shape
s = torch.cuda.current_stream().cuda_stream
q = lambda a: " ".join(f"{np.percentile(a, x):6.2f}" for x in (0, 10, 50, 90, 100))
for rep in range(3):
    fn(t.data_ptr(), out.data_ptr(), B, H, W, W, W, cfg.k, 0, counts.data_ptr(), s)
    torch.cuda.synchronize()
    buf = np.zeros((8 << 20) // 8, dtype=np.uint64)
    _native.check(lib.irdn_debug_timeline(buf.ctypes.data, buf.nbytes))
    dr = buf[600000:600000 + 4 * 8192].reshape(-1, 4)
    dr = dr[dr[:, 3] == 1]
    tl = buf[: 600000 // 6 * 6].reshape(-1, 6)
    tl = tl[tl[:, 1] != 0]
    t0 = tl[:, 0].min()
    wait, ready, det, done = [(tl[:, i].astype(np.int64) - int(t0)) / 1e3 for i in range(4)]
    n = tl[:, 4].astype(np.int64)
    warp = (tl[:, 5] >> 16).astype(np.int64)
    sm = (tl[:, 5] & 0xFFFF).astype(np.int64)
    end = done.max()
    print(f"rep {rep}: tiles {len(tl)}, warps {len(np.unique(warp))}, last done {end:.2f} us")
    print(f"  load wait us  p0/10/50/90/100: {q(ready - wait)}")
    print(f"  detect us     p0/10/50/90/100: {q(det - ready)}")
    print(f"  median us     p0/10/50/90/100: {q(done - det)}")
    print(f"  queue n       p0/10/50/90/100: {q(n)}")
    # per-warp last done and per-SM last done
    wl = np.zeros(warp.max() + 1); np.maximum.at(wl, warp, done)
    wl = wl[wl > 0]
    print(f"  warp last-done p0/10/50/90/100: {q(wl)}")
    sl = np.zeros(sm.max() + 1); np.maximum.at(sl, sm, done)
    print(f"  SM last-done   p0/10/50/90/100: {q(sl[sl > 0])}")
    if len(dr):
        d0 = (dr[:, 0].astype(np.int64) - int(t0)) / 1e3
        d1 = (dr[:, 1].astype(np.int64) - int(t0)) / 1e3
        print(f"  drain start   p0/10/50/90/100: {q(d0)}")
        print(f"  drain end     p0/10/50/90/100: {q(d1)}   owners {int(dr[:, 2].sum())}")
        print(f"  drain dur     p0/10/50/90/100: {q(d1 - d0)}")
    late = np.argsort(done)[-8:]
    for i in late:
        print(f"    late tile: ready {ready[i]:.2f} det {det[i]-ready[i]:.2f} med {done[i]-det[i]:.2f} n {n[i]} sm {sm[i]}")
    # active warps over time
    for tt in np.linspace(0, end, 11)[1:]:
        act = ((wait <= tt) & (done >= tt)).sum()
        print(f"    t={tt:6.2f}us active tiles {act}")
    if dump:
        np.save(dump, tl)
