"""On-device scene rendering (csrc/scene.cuh, irdn_scene_render) against
the host generator (csrc/scene.c scene_generate).

CPU: scene_tables() + a numpy restatement of the kernel's per-pixel arithmetic (the same
IEEE double operations in the same order) reproduce scene_generate()'s bytes — this pins the
table layout and the operation order the kernel relies on.
GPU: the kernel's bytes equal the host generator's on every BASELINE config — at FULL size
against the input sha256 of tests/golden/full_configs.json (c5: all 4096 frames), and on
crops / odd shapes against scene_generate() directly.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1201_3972_b200.scene import CONFIGS, SEED, generate, tables

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "full_configs.json")))
FULL_SHA = {g["config"]: g["input_sha256"] for g in GOLD.values()}

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _sm64(x):
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _prefix(cfg, seed, f, stream):
    with np.errstate(over="ignore"):
        h = _sm64(np.uint64(seed) ^ (np.uint64(cfg.config_id) << np.uint64(56)))
        h = _sm64(h ^ (np.uint64(f) * np.uint64(0xD1B54A32D192ED03)))
        return _sm64(h ^ (np.uint64(stream) * np.uint64(0xABC98388FB8FAC03)))


def _u01(h):
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def render_numpy(cfg, frame0, n, seed=SEED):
    """The kernel's per-pixel arithmetic (scene.cuh render_kernel) in numpy float64."""
    t = tables(cfg, frame0, n, seed)
    H, W = cfg.height, cfg.width
    out = np.empty((n, H, W), cfg.np_dtype)
    ys, xs = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    idx = (ys.astype(np.uint64) * np.uint64(W) + xs.astype(np.uint64))
    for i in range(n):
        f = frame0 + i
        v = np.full((H, W), 60.0)
        for j in range(cfg.nblobs):
            gy, gx = t["gy"][i, j], t["gx"][i, j]
            rows = gy >= 1e-6
            v[rows] = v[rows] + gy[rows, None] * gx[None, :]
        if cfg.sensor_sigma > 0:
            h = _sm64(_prefix(cfg, seed, f, 4) ^ idx)
            m = np.uint64(0xFFFF)
            s4 = ((h & m).astype(np.float64) + ((h >> np.uint64(16)) & m).astype(np.float64)
                  + ((h >> np.uint64(32)) & m).astype(np.float64) + (h >> np.uint64(48)).astype(np.float64))
            v = v + (s4 / 65536.0 - 2.0) * (cfg.sensor_sigma * 1.7320508075688772)
        v = v * (cfg.maxval / 255.0)
        for L in t["lines"][i]:
            d = (xs - L[2]) * L[0] - (ys - L[3]) * L[1]
            v = np.where(np.abs(d) < L[4], v + cfg.line_amp, v)
        for x0, y0, x1, y1 in t["rects"][i]:
            inside = (xs >= x0) & (xs < x1) & (ys >= y0) & (ys < y1)
            v = np.where(inside, v + cfg.rect_amp, v)
        q = np.clip(np.rint(v), 0, cfg.maxval).astype(np.uint32)
        kind = {"none": 0, "sp": 1, "uniform": 2}[cfg.impulse]
        if kind:
            hit = _u01(_sm64(_prefix(cfg, seed, f, 5) ^ idx)) < cfg.density
            hv = _sm64(_prefix(cfg, seed, f, 6) ^ idx)
            val = (np.where((hv >> np.uint64(63)) != 0, cfg.maxval, 0).astype(np.uint32) if kind == 1
                   else (hv % np.uint64(cfg.maxval + 1)).astype(np.uint32))
            q = np.where(hit, val, q)
        out[i] = q
    return out


SMALL = {
    "c1": CONFIGS["c1"],
    "c2": CONFIGS["c2"].with_shape(frames=3, height=128, width=160),
    "c3": CONFIGS["c3"].with_shape(frames=2, height=135, width=240),
    "c4": CONFIGS["c4"].with_shape(height=256, width=320),
    "c5": CONFIGS["c5"].with_shape(frames=6, height=120, width=160),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_tables_and_kernel_arithmetic_reproduce_host_scene(name):
    cfg = SMALL[name]
    f0 = 1 if cfg.frames > 2 else 0
    n = cfg.frames - f0
    want = generate(cfg, frame0=f0, nframes=n)
    got = render_numpy(cfg, f0, n)
    assert np.array_equal(got, want), name


def test_tables_layout():
    cfg = CONFIGS["c3"].with_shape(frames=2, height=64, width=96)
    t = tables(cfg, 0, 2)
    assert t["gx"].shape == (2, cfg.nblobs, 96) and t["gy"].shape == (2, cfg.nblobs, 64)
    assert t["lines"].shape == (2, 0, 5) and t["rects"].shape == (2, cfg.nrects, 4)
    r = t["rects"].reshape(-1, 4)
    assert np.all(r[:, 2] - r[:, 0] >= 6) and np.all(r[:, 3] - r[:, 1] <= 12)
    assert np.all((t["gx"] > 0) & (t["gx"] <= 1))


def _sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_device_scene_full_size_matches_golden_input(cuda_ok, name):
    import torch

    from paper_1201_3972_b200.scene import render_device

    cfg = CONFIGS[name]
    t = render_device(cfg)
    torch.cuda.synchronize()
    assert list(t.shape) == [cfg.frames, cfg.height, cfg.width]
    h = hashlib.sha256()
    step = max(1, (256 << 20) // (cfg.height * cfg.width * cfg.bytes_per_pixel))
    for f0 in range(0, cfg.frames, step):  # hash in chunks (c5 is 1.26 GB)
        part = t[f0:f0 + step]
        part = part.view(torch.int16) if cfg.dtype == "u16" else part
        h.update(part.cpu().numpy().tobytes())
    assert h.hexdigest() == FULL_SHA[name], name


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SMALL))
def test_device_scene_crops_and_odd_shapes(cuda_ok, name):
    import torch

    from paper_1201_3972_b200.scene import render_device

    for cfg in (SMALL[name], SMALL[name].with_shape(height=37, width=53)):
        f0 = 2 if cfg.frames > 3 else 0
        n = cfg.frames - f0
        want = generate(cfg, frame0=f0, nframes=n)
        for chunk in (64 << 20, 1):  # one call / one frame per call
            got = render_device(cfg, frame0=f0, nframes=n, chunk_bytes=chunk)
            host = (got.view(torch.int16) if cfg.dtype == "u16" else got).cpu().numpy()
            assert np.array_equal(host.view(want.dtype), want), (name, cfg.height, cfg.width, chunk)
    # a later window of the c5 sequence and a non-default seed
    cfg = CONFIGS["c5"]
    want = generate(cfg, frame0=4090, nframes=6, seed=7)
    got = render_device(cfg, frame0=4090, nframes=6, seed=7).cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_device_scene_rejects_bad_descriptors(cuda_ok):
    import ctypes

    from paper_1201_3972_b200 import _native

    lib = _native.load_lib()
    d = _native.IrdnSceneDesc()
    d.width, d.height, d.bytes_per_pixel, d.nframes = 16, 16, 3, 1
    assert lib.irdn_scene_render(ctypes.byref(d), ctypes.c_void_p(16), None) == _native.IRDN_EINVAL
    d.bytes_per_pixel, d.nblobs = 1, 2  # blobs without tables
    assert lib.irdn_scene_render(ctypes.byref(d), ctypes.c_void_p(16), None) == _native.IRDN_EINVAL
