"""Seeded salt-and-pepper injection mirrored from the reference (pkg/src/irdenoise/noise.py).

`inject_impulse(img, spec)` returns the same noisy `GrayImage` and `NoiseMask`,
byte for byte, as the reference's sequential SplitMix64 walk (noise.py:89-106); the
work runs on the GPU (csrc/noise.cuh: the draw stream is parsed into per-pixel
tokens with a two-state scan, behind `irdn_inject_impulse_u8` in include/irdn.h).

`SplitMix64` is the reference's generator object (noise.py:17-34) for callers that
draw values themselves; it is plain host arithmetic, not part of the GPU path.

Extension (keyword-compatible): `inject_impulse` also takes a uint8 numpy array or
CUDA tensor of any shape (pixels in row-major order) and returns the same type.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .image import GrayImage

_MASK64 = 0xFFFFFFFFFFFFFFFF
_GAMMA = 0x9E3779B97F4A7C15


class SplitMix64:
    """SplitMix64 (noise.py:17-34): 64-bit state, 64-bit output."""

    __slots__ = ("state",)

    def __init__(self, seed: int) -> None:
        self.state = seed & _MASK64

    def next_u64(self) -> int:
        s = (self.state + _GAMMA) & _MASK64
        self.state = s
        s = ((s ^ (s >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        s = ((s ^ (s >> 27)) * 0x94D049BB133111EB) & _MASK64
        return s ^ (s >> 31)

    def next_uniform(self) -> float:
        """Uniform double in [0, 1) from the top 53 bits."""
        return (self.next_u64() >> 11) / float(1 << 53)


@dataclass(frozen=True)
class NoiseSpec:
    """Density, salt share and seed of the impulses (noise.py:37-55)."""

    density: float
    salt_fraction: float = 0.5
    seed: int = 0

    def __post_init__(self) -> None:
        if not 0.0 <= self.density <= 1.0:
            raise ValueError(f"density must be in [0, 1], got {self.density}")
        if not 0.0 <= self.salt_fraction <= 1.0:
            raise ValueError(f"salt_fraction must be in [0, 1], got {self.salt_fraction}")
        if not 0 <= self.seed <= _MASK64:
            raise ValueError("seed must be an unsigned 64-bit integer")


class NoiseMask:
    """Row-major corruption flags matching an image (noise.py:58-86)."""

    __slots__ = ("width", "height", "flags")

    def __init__(self, width: int, height: int, flags) -> None:
        buf = bytearray(flags)
        if len(buf) != width * height:
            raise ValueError(f"mask has {len(buf)} flags, expected {width * height}")
        self.width = width
        self.height = height
        self.flags = buf

    def __len__(self) -> int:
        return len(self.flags)

    def is_corrupted(self, x: int, y: int) -> bool:
        return bool(self.flags[y * self.width + x])

    @property
    def count(self) -> int:
        """Number of corrupted pixels."""
        return int(np.count_nonzero(np.frombuffer(self.flags, np.uint8)))

    def to_image(self) -> GrayImage:
        """255 where corrupted, 0 elsewhere."""
        f = np.frombuffer(self.flags, np.uint8)
        return GrayImage(self.width, self.height, ((f != 0).astype(np.uint8) * 255).tobytes())


def _inject_device(src, out, flags, count, spec: NoiseSpec) -> None:
    import torch

    lib = _native.load_lib()
    stream = torch.cuda.current_stream(src.device).cuda_stream
    _native.check(lib.irdn_inject_impulse_u8(
        src.data_ptr(), out.data_ptr(), flags.data_ptr() if flags is not None else None, src.numel(),
        spec.seed, float(spec.density), float(spec.salt_fraction),
        count.data_ptr() if count is not None else None, stream))


def inject_impulse(img, spec: NoiseSpec, *, device: int | None = None):
    """Corrupt ~density of the pixels with 0/255 impulses (noise.py:89-106).

    GrayImage -> (GrayImage, NoiseMask). uint8 numpy array / CUDA tensor ->
    (noisy, flags) of the same type and shape.
    """
    if not isinstance(spec, NoiseSpec):
        raise TypeError(f"spec must be a NoiseSpec, got {type(spec)!r}")
    _native.load_lib()  # fail loudly before touching torch if the CUDA library is missing
    import torch

    if isinstance(img, GrayImage):
        dev = torch.device("cuda", device or 0)
        with torch.cuda.device(dev):
            src = torch.frombuffer(img.pixels, dtype=torch.uint8).to(dev, non_blocking=False)
            out = torch.empty_like(src)
            flags = torch.empty_like(src)
            _inject_device(src, out, flags, None, spec)
            o = out.cpu().numpy().tobytes()
            f = flags.cpu().numpy().tobytes()
        return GrayImage(img.width, img.height, o), NoiseMask(img.width, img.height, f)
    if isinstance(img, np.ndarray):
        if img.dtype != np.uint8:
            raise TypeError(f"inject_impulse works on 8-bit pixels, got {img.dtype}")
        dev = torch.device("cuda", device or 0)
        with torch.cuda.device(dev):
            src = torch.from_numpy(np.ascontiguousarray(img)).to(dev)
            out = torch.empty_like(src)
            flags = torch.empty_like(src)
            _inject_device(src, out, flags, None, spec)
            return out.cpu().numpy(), flags.cpu().numpy()
    if isinstance(img, torch.Tensor):
        if img.dtype != torch.uint8 or not img.is_cuda:
            raise TypeError("inject_impulse expects a CUDA uint8 tensor")
        with torch.cuda.device(img.device):
            src = img.contiguous()
            out = torch.empty_like(src)
            flags = torch.empty_like(src)
            _inject_device(src, out, flags, None, spec)
        return out, flags
    raise TypeError(f"inject_impulse expects a GrayImage, numpy array or CUDA tensor, got {type(img)!r}")
