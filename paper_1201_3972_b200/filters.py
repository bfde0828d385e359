"""Filter entry points mirrored from the reference (pkg/src/irdenoise/filters.py).

`run_filter`, `fnr_pass` and `mf_pass` keep the reference's names, positional
order, defaults, validation and `FilterStats` results; the per-pixel work
(clamp-gather, extrema detector, median selection, counters) runs in the
sm_100a kernels behind the C ABI (include/irdn.h) — there is no CPU path.

Reference call -> C ABI:
  run_filter(img, spec, method, passes, threads)   filters.py:79-102
      GrayImage / numpy   -> irdn_run_filter_{u8,u16}          (host buffers, pipelined H2D/D2H)
      CUDA torch tensor   -> irdn_run_filter_device_{u8,u16}   (device-resident, caller's stream)
  fnr_pass / mf_pass                                filters.py:69-76
  window_extrema / classify_pixel                   filters.py:55-66 (scalar per-window API, Python)
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .image import GrayImage, Window, WindowSpec

METHOD_FNR = "fnr"
METHOD_MF = "mf"


@dataclass(frozen=True)
class WindowExtrema:
    min_gray: int
    max_gray: int


@dataclass
class FilterStats:
    """Per-run counters; elapsed_ms is informational (filters.py:33-52)."""

    minmax_scans: int = 0
    sorts: int = 0
    replacements: int = 0
    detected: int = 0
    elapsed_ms: float = 0.0
    passes: int = 0

    def to_dict(self) -> dict:
        return {
            "minmax_scans": self.minmax_scans,
            "sorts": self.sorts,
            "replacements": self.replacements,
            "detected": self.detected,
            "elapsed_ms": self.elapsed_ms,
            "passes": self.passes,
        }


def window_extrema(w: Window, stats: FilterStats | None = None) -> WindowExtrema:
    """Exact min and max of the window values, one counted scan (filters.py:55-60)."""
    if stats is not None:
        stats.minmax_scans += 1
    return WindowExtrema(min(w.values), max(w.values))


def classify_pixel(w: Window, extrema: WindowExtrema) -> bool:
    """True when the centre equals a window extremum (filters.py:63-66)."""
    center = w.values[w.center_index]
    return center == extrema.min_gray or center == extrema.max_gray


def fnr_pass(img, spec: WindowSpec, stats: FilterStats, *, device: int | None = None):
    """One selective pass, accumulating into the caller's stats (filters.py:69-71)."""
    out, st = _run(img, spec, METHOD_FNR, 1, device)
    _accumulate(stats, st)
    return out


def mf_pass(img, spec: WindowSpec, stats: FilterStats, *, device: int | None = None):
    """One every-pixel median pass (filters.py:74-76)."""
    out, st = _run(img, spec, METHOD_MF, 1, device)
    _accumulate(stats, st)
    return out


def run_filter(img, spec: WindowSpec, method: str, passes: int = 1, threads: int = 1, *,
               device: int | None = None):
    """Apply the chosen filter `passes` times, each pass feeding the next (filters.py:79-102).

    `threads` is accepted for signature compatibility; it never changes results
    (the reference's row bands are bit-identical for any thread count).
    `img` may be a GrayImage (returns a GrayImage), a numpy uint8/uint16 array
    [H,W] or [B,H,W] (returns an array), or a CUDA torch tensor of that shape
    (filtered on the tensor's device and the current torch stream).
    """
    if method not in (METHOD_FNR, METHOD_MF):
        raise ValueError(f"unknown method {method!r}, expected 'fnr' or 'mf'")
    if passes < 1:
        raise ValueError(f"passes must be >= 1, got {passes}")
    return _run(img, spec, method, passes, device)


def _accumulate(stats: FilterStats, st: FilterStats) -> None:
    stats.minmax_scans += st.minmax_scans
    stats.sorts += st.sorts
    stats.replacements += st.replacements
    stats.detected += st.detected
    stats.passes += st.passes


def _stats_from_native(s: _native.IrdnStats) -> FilterStats:
    return FilterStats(minmax_scans=int(s.minmax_scans), sorts=int(s.sorts),
                       replacements=int(s.replacements), detected=int(s.detected),
                       elapsed_ms=float(s.elapsed_ms), passes=int(s.passes))


def _as_spec(spec) -> WindowSpec:
    """Any object with an odd `k` >= 3 (the reference's WindowSpec included), or an int."""
    if isinstance(spec, WindowSpec):
        return spec
    return WindowSpec(int(getattr(spec, "k", spec)))


def _is_gray_image(img) -> bool:
    """GrayImage-shaped: width, height and a row-major pixel buffer (image.py:19-54) —
    this package's GrayImage or the reference's own (duck-typed, no import of it)."""
    return all(hasattr(img, a) for a in ("width", "height", "pixels")) and not isinstance(img, np.ndarray)


def _run(img, spec, method: str, passes: int, device: int | None):
    spec = _as_spec(spec)
    lib = _native.load_lib()
    m = _native.METHODS[method]
    if _is_gray_image(img):
        return _run_gray(lib, img, spec, m, passes, device or 0)
    if isinstance(img, np.ndarray):
        return _run_numpy(lib, img, spec, m, passes, device or 0)
    if type(img).__module__.startswith("torch"):
        return _run_torch(lib, img, spec, method, m, passes)
    raise TypeError(f"run_filter expects a GrayImage, numpy array or CUDA tensor, got {type(img)!r}")


def _run_gray(lib, img, spec: WindowSpec, m: int, passes: int, device: int):
    """GrayImage in, GrayImage of the same class out (filters.py:108 fresh buffer, :127).

    8-bit images (bytes / bytearray / array('B') pixels) take irdn_run_filter_u8; a
    duck-typed image with 16-bit pixels (array('H'), the reference's dtype-agnostic
    per-window path) takes irdn_run_filter_u16."""
    w, h = int(img.width), int(img.height)
    if w < 1 or h < 1:
        raise ValueError(f"image dimensions must be positive, got {w}x{h}")
    src = np.frombuffer(img.pixels, dtype=np.uint16 if getattr(img.pixels, "itemsize", 1) == 2 else np.uint8)
    if src.size != w * h:
        raise ValueError(f"pixel buffer has {src.size} entries, expected {w * h}")
    # the native call writes straight into the result's own buffer (filters.py:108: a fresh
    # bytearray), with no intermediate copy
    if src.dtype == np.uint8:
        pixels = bytearray(w * h)
    else:
        from array import array

        pixels = array("H", bytes(2 * w * h))
    out = np.frombuffer(pixels, dtype=src.dtype)
    st = _native.IrdnStats()
    fn = lib.irdn_run_filter_u8 if src.dtype == np.uint8 else lib.irdn_run_filter_u16
    _native.check(fn(src.ctypes.data, out.ctypes.data, 1, h, w, spec.k, m, passes, device, ctypes.byref(st)))
    cls = type(img) if not isinstance(img, GrayImage) else GrayImage
    try:
        res = cls(w, h, pixels)
    except Exception:
        res = GrayImage(w, h, pixels) if src.dtype == np.uint8 else _PixelImage(w, h, pixels)
    return res, _stats_from_native(st)


@dataclass
class _PixelImage:
    """Result holder for a duck-typed 16-bit image whose class cannot be rebuilt."""

    width: int
    height: int
    pixels: object


def _shape3(shape) -> tuple[int, int, int]:
    if len(shape) == 2:
        return 1, int(shape[0]), int(shape[1])
    if len(shape) == 3:
        return int(shape[0]), int(shape[1]), int(shape[2])
    raise ValueError(f"expected an image of shape [H,W] or [B,H,W], got {tuple(shape)}")


def _pinned_like(a: np.ndarray) -> np.ndarray:
    """Output buffer in page-locked memory (torch's caching host allocator): the device
    writes it by DMA directly, with no staging copy and no first-touch page faults. The
    array keeps the owning tensor alive through its base."""
    import torch

    if a.nbytes < (1 << 20):
        return np.empty_like(a)
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    out = t.numpy().view(a.dtype).reshape(a.shape)
    return out


def _run_numpy(lib, img: np.ndarray, spec: WindowSpec, m: int, passes: int, device: int):
    if img.dtype not in (np.uint8, np.uint16):
        raise TypeError(f"pixels must be uint8 or uint16, got {img.dtype}")
    b, h, w = _shape3(img.shape)
    src = np.ascontiguousarray(img)
    out = _pinned_like(src)
    st = _native.IrdnStats()
    fn = lib.irdn_run_filter_u8 if src.dtype == np.uint8 else lib.irdn_run_filter_u16
    _native.check(fn(src.ctypes.data, out.ctypes.data, b, h, w, spec.k, m, passes, device,
                     ctypes.byref(st)))
    return out, _stats_from_native(st)


def _run_torch(lib, t, spec: WindowSpec, method: str, m: int, passes: int):
    import torch

    if not t.is_cuda:
        return _run_numpy(lib, t.numpy(), spec, m, passes, 0)
    if t.dtype not in (torch.uint8, torch.uint16):
        raise TypeError(f"pixels must be uint8 or uint16, got {t.dtype}")
    b, h, w = _shape3(t.shape)
    t0 = time.perf_counter()
    with torch.cuda.device(t.device):
        src = t.contiguous()
        out = torch.empty_like(src)
        tmp = torch.empty_like(src) if passes > 1 else None
        counts = torch.zeros(2, dtype=torch.int64, device=t.device)
        stream = torch.cuda.current_stream(t.device).cuda_stream
        fn = lib.irdn_run_filter_device_u8 if t.dtype == torch.uint8 else lib.irdn_run_filter_device_u16
        _native.check(fn(src.data_ptr(), out.data_ptr(), tmp.data_ptr() if tmp is not None else None,
                         b, h, w, spec.k, m, passes, counts.data_ptr(), stream))
        det, rep = (int(v) for v in counts.tolist())
    pixels = b * h * w * passes
    if method == METHOD_FNR:
        st = FilterStats(minmax_scans=pixels, sorts=det, replacements=rep, detected=det, passes=passes)
    else:
        st = FilterStats(sorts=pixels, passes=passes)
    st.elapsed_ms = (time.perf_counter() - t0) * 1000.0
    return out, st
