"""Seeded synthetic IR scenes for the BASELINE.json configs (bench/test inputs).

The reference evaluates on one 364x244 IR photograph that is not available
(reference SPEC.md:309); these scenes stand in for it with the shapes,
dtypes, window sizes and impulse models BASELINE.json names. Generation is
native (csrc/scene.c, counter-based SplitMix64, pthreads) so the 1.26 G-pixel
config c5 is produced in seconds. Scene generation is input preparation, not
the filter: nothing here is on the hot path.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np

from ._native import load_scene_lib

SEED = 42  # the reference CLI's default --seed (cli.py:25)


class SceneParams(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("bpp", ctypes.c_int32),
        ("maxval", ctypes.c_int32), ("nblobs", ctypes.c_int32), ("sigma_scale", ctypes.c_double),
        ("amp_scale", ctypes.c_double),
        ("drift", ctypes.c_int32), ("nlines", ctypes.c_int32), ("line_amp", ctypes.c_double),
        ("nrects", ctypes.c_int32), ("rect_amp", ctypes.c_double),
        ("sensor_sigma", ctypes.c_double), ("impulse_kind", ctypes.c_int32),
        ("density", ctypes.c_double), ("seed", ctypes.c_uint64), ("config_id", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class SceneConfig:
    """One BASELINE.json config: frame shape, dtype, window and scene recipe."""

    name: str
    config_id: int
    frames: int
    height: int
    width: int
    dtype: str  # "u8" | "u16"
    k: int
    nblobs: int = 8
    sigma_scale: float = 1.0
    amp_scale: float = 1.0
    drift: bool = False
    nlines: int = 0
    line_amp: float = 0.0
    nrects: int = 0
    rect_amp: float = 0.0
    sensor_sigma: float = 2.0
    impulse: str = "sp"  # "sp" salt-and-pepper | "uniform" random-valued | "none"
    density: float = 0.2
    description: str = ""

    @property
    def maxval(self) -> int:
        return 255 if self.dtype == "u8" else 16383

    @property
    def np_dtype(self):
        return np.uint8 if self.dtype == "u8" else np.uint16

    @property
    def bytes_per_pixel(self) -> int:
        return 1 if self.dtype == "u8" else 2

    @property
    def pixels(self) -> int:
        return self.frames * self.height * self.width

    def with_shape(self, frames: int | None = None, height: int | None = None,
                   width: int | None = None) -> "SceneConfig":
        return replace(self, frames=frames or self.frames, height=height or self.height,
                       width=width or self.width)

    def params(self, seed: int = SEED) -> SceneParams:
        return SceneParams(
            self.width, self.height, self.bytes_per_pixel, self.maxval, self.nblobs,
            self.sigma_scale, self.amp_scale, int(self.drift), self.nlines, self.line_amp, self.nrects,
            self.rect_amp, self.sensor_sigma, {"none": 0, "sp": 1, "uniform": 2}[self.impulse],
            self.density, seed, self.config_id)


# BASELINE.json "configs", in order (c1 = configs[0], ... c5 = configs[4]).
CONFIGS: dict[str, SceneConfig] = {
    "c1": SceneConfig("c1", 1, 1, 512, 512, "u8", 3, density=0.20,
                      description="512x512 u8, 1 frame, 3x3, 8 blobs + N(0,2^2), 20% salt-and-pepper"),
    "c2": SceneConfig("c2", 2, 64, 512, 640, "u16", 5, nlines=4, line_amp=2000.0,
                      impulse="uniform", density=0.30,
                      description="64 x 640x512 u16 (14-bit), 5x5, blob field + 1-3 px hot lines (+2000), "
                                  "30% uniform random impulses"),
    "c3": SceneConfig("c3", 3, 32, 1080, 1920, "u8", 7, nrects=40, rect_amp=80.0, density=0.50,
                      description="32 x 1920x1080 u8, 7x7, blob field + 6-12 px rectangles (+80), "
                                  "50% salt-and-pepper"),
    "c4": SceneConfig("c4", 4, 1, 8192, 8192, "u16", 11, nblobs=64, sigma_scale=16.0, amp_scale=0.125,
                      impulse="uniform", density=0.40,
                      description="8192x8192 u16 (14-bit), 11x11, 64 blobs (sigma x16, amplitude x1/8 so the sum stays in range), 40% uniform random impulses"),
    "c5": SceneConfig("c5", 5, 4096, 480, 640, "u8", 3, drift=True, density=0.10,
                      description="4096 x 640x480 u8 video, 3x3, blobs drifting 1 px/frame, "
                                  "10% salt-and-pepper per frame"),
}


def generate(cfg: SceneConfig, frame0: int = 0, nframes: int | None = None, seed: int = SEED,
             threads: int | None = None, out: np.ndarray | None = None, lib=None) -> np.ndarray:
    """Frames [frame0, frame0+nframes) of `cfg` as a [B,H,W] array (or into `out`).

    `lib` is any loaded library exporting scene_generate (default: libirdn_scene.so; the
    reference arm of bench.py passes its CPU checker library, which links the same source)."""
    n = cfg.frames if nframes is None else nframes
    if out is None:
        out = np.empty((n, cfg.height, cfg.width), dtype=cfg.np_dtype)
    assert out.flags.c_contiguous and out.dtype == cfg.np_dtype and out.size == n * cfg.height * cfg.width
    p = cfg.params(seed)
    nt = threads or max(1, min(32, os.cpu_count() or 1))
    rc = (lib or load_scene_lib()).scene_generate(ctypes.byref(p), frame0, n, out.ctypes.data, nt)
    if rc != 0:
        raise ValueError("scene_generate rejected the parameters")
    return out


def tables(cfg: SceneConfig, frame0: int = 0, nframes: int | None = None, seed: int = SEED,
           threads: int | None = None) -> dict:
    """The per-frame scene parameters that need exp / sin / cos (csrc/scene.c scene_tables):
    gx [n, nblobs, W], gy [n, nblobs, H] (float64), lines [n, nl, 5], rects [n, nr, 4] (int32)."""
    n = cfg.frames if nframes is None else nframes
    nl, nr = min(cfg.nlines, 64), min(cfg.nrects, 256)
    t = {
        "gx": np.empty((n, cfg.nblobs, cfg.width), np.float64),
        "gy": np.empty((n, cfg.nblobs, cfg.height), np.float64),
        "lines": np.empty((n, nl, 5), np.float64),
        "rects": np.empty((n, nr, 4), np.int32),
    }
    p = cfg.params(seed)
    nt = threads or max(1, min(32, os.cpu_count() or 1))
    rc = load_scene_lib().scene_tables(
        ctypes.byref(p), frame0, n, t["gx"].ctypes.data, t["gy"].ctypes.data,
        t["lines"].ctypes.data if nl else None, t["rects"].ctypes.data if nr else None, nt)
    if rc != 0:
        raise ValueError("scene_tables rejected the parameters")
    return t


def render_device(cfg: SceneConfig, frame0: int = 0, nframes: int | None = None, seed: int = SEED,
                  out=None, device=None, chunk_bytes: int = 64 << 20):
    """Frames [frame0, frame0+nframes) of `cfg` rendered on the GPU (irdn_scene_render) as a
    CUDA tensor [B, H, W] (torch.uint8 / torch.uint16), byte for byte equal to generate(). The per-frame exp / sin / cos tables come from the host
    (tables()), a chunk of frames at a time, on the current torch stream."""
    import torch

    from . import _native

    lib = _native.load_lib()
    n = cfg.frames if nframes is None else nframes
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    tdt = torch.uint8 if cfg.dtype == "u8" else torch.uint16
    if out is None:
        out = torch.empty((n, cfg.height, cfg.width), dtype=tdt, device=dev)
    if out.dtype != tdt or not out.is_contiguous() or out.numel() != n * cfg.height * cfg.width:
        raise ValueError("out must be a contiguous CUDA tensor of the scene's dtype and shape")
    nl, nr = min(cfg.nlines, 64), min(cfg.nrects, 256)
    per_frame = 8 * cfg.nblobs * (cfg.width + cfg.height) + 40 * nl + 16 * nr + 1
    chunk = max(1, min(65535, chunk_bytes // per_frame))
    stream = torch.cuda.current_stream(dev)
    flat = out.view(n, -1)
    for c0 in range(0, n, chunk):
        c = min(chunk, n - c0)
        t = tables(cfg, frame0 + c0, c, seed)
        dt = {k: torch.from_numpy(v).to(dev, non_blocking=False) for k, v in t.items()}
        d = _native.IrdnSceneDesc(
            cfg.width, cfg.height, cfg.bytes_per_pixel, cfg.maxval, cfg.nblobs, nl, nr,
            {"none": 0, "sp": 1, "uniform": 2}[cfg.impulse], cfg.config_id, int(cfg.sensor_sigma > 0),
            cfg.maxval / 255.0, cfg.sensor_sigma * 1.7320508075688772, cfg.line_amp, cfg.rect_amp,
            cfg.density, seed, frame0 + c0, c,
            dt["gx"].data_ptr(), dt["gy"].data_ptr(), dt["lines"].data_ptr() if nl else None,
            dt["rects"].data_ptr() if nr else None)
        _native.check(lib.irdn_scene_render(ctypes.byref(d), flat[c0].data_ptr(), stream.cuda_stream))
        stream.synchronize()  # the chunk's tables are freed at the end of this iteration
    return out
