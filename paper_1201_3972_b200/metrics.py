"""MSE / PSNR and comparison reports mirrored from the reference (pkg/src/irdenoise/metrics.py).

The squared-error sum is exact integer arithmetic, as in the reference
(metrics.py:22-32): it is computed on the GPU as a u64 (`irdn_sq_err_sum_*`,
csrc/metrics.cuh) and divided once on the host with Python's correctly rounded
int / int, so `mse`, `psnr` and every report field equal the reference's bit for
bit. Report dataclasses and their `to_dict` layouts follow metrics.py:43-157.

Extension (keyword-compatible): `mse` / `psnr` / `quality_report` also accept
pairs of equally shaped uint8 / uint16 numpy arrays or CUDA tensors.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .filters import FilterStats
from .image import GrayImage

REPORT_SCHEMA = "irdenoise-report/1"
STATS_SCHEMA = "irdenoise-stats/1"

_U16_CALL_LIMIT = (1 << 32) - 1  # include/irdn.h: u16 elements per irdn_sq_err_sum_u16 call


def _shape_of(img) -> tuple[int, ...]:
    if isinstance(img, GrayImage):
        return (img.height, img.width)
    return tuple(int(s) for s in img.shape)


def _device_tensor(img, dev):
    import torch

    if isinstance(img, GrayImage):
        return torch.frombuffer(img.pixels, dtype=torch.uint8).to(dev)
    if isinstance(img, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(img)).to(dev)
    if isinstance(img, torch.Tensor):
        return img.to(dev).contiguous()
    raise TypeError(f"expected a GrayImage, numpy array or tensor, got {type(img)!r}")


def sq_err_sum(a, b) -> int:
    """Exact sum of (a - b)^2 over all pixels (GPU, u64)."""
    lib = _native.load_lib()
    import torch

    dev = a.device if isinstance(a, torch.Tensor) and a.is_cuda else torch.device("cuda", 0)
    with torch.cuda.device(dev):
        ta, tb = _device_tensor(a, dev), _device_tensor(b, dev)
        if ta.dtype != tb.dtype or ta.dtype not in (torch.uint8, torch.uint16):
            raise TypeError(f"pixels must both be uint8 or both uint16, got {ta.dtype} / {tb.dtype}")
        ta, tb = ta.reshape(-1), tb.reshape(-1)
        acc = torch.zeros(1, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        n = ta.numel()
        if ta.dtype == torch.uint8:
            _native.check(lib.irdn_sq_err_sum_u8(ta.data_ptr(), tb.data_ptr(), n, acc.data_ptr(), stream))
            return int(acc.item()) & 0xFFFFFFFFFFFFFFFF
        total = 0
        for s in range(0, n, _U16_CALL_LIMIT):
            e = min(n, s + _U16_CALL_LIMIT)
            acc.zero_()
            _native.check(lib.irdn_sq_err_sum_u16(ta[s:e].data_ptr(), tb[s:e].data_ptr(), e - s,
                                                  acc.data_ptr(), stream))
            total += int(acc.item()) & 0xFFFFFFFFFFFFFFFF
        return total


def mse(a, b) -> float:
    """Mean squared error between two same-sized images (metrics.py:22-32)."""
    sa, sb = _shape_of(a), _shape_of(b)
    if sa != sb:
        if isinstance(a, GrayImage) and isinstance(b, GrayImage):
            raise ValueError(f"dimension mismatch: {a.width}x{a.height} vs {b.width}x{b.height}")
        raise ValueError(f"dimension mismatch: {sa} vs {sb}")
    n = math.prod(sa)
    return sq_err_sum(a, b) / n


def _db(err: float, max_val: int) -> float:
    return math.inf if err == 0 else 10.0 * math.log10((max_val * max_val) / err)


def psnr(a, b, max_val: int = 255) -> float:
    """Peak signal-to-noise ratio in dB; +infinity for identical images (metrics.py:35-40)."""
    return _db(mse(a, b), max_val)


@dataclass(frozen=True)
class QualityReport:
    """MSE and PSNR of one image pair (metrics.py:43-49)."""

    mse: float
    psnr_db: float
    max_val: int = 255


def quality_report(a, b, max_val: int = 255) -> QualityReport:
    """metrics.py:52-55: one squared-error sum for both numbers."""
    err = mse(a, b)
    return QualityReport(mse=err, psnr_db=_db(err, max_val), max_val=max_val)


@dataclass(frozen=True)
class MethodResult:
    """One method's fidelity plus work counters (metrics.py:58-75)."""

    psnr_db: float
    sorts: int = 0
    minmax_scans: int = 0
    elapsed_ms: float = 0.0
    passes: int = 0

    def to_dict(self) -> dict:
        return {
            "psnr_db": format_db(self.psnr_db),
            "sorts": self.sorts,
            "minmax_scans": self.minmax_scans,
            "elapsed_ms": self.elapsed_ms,
            "passes": self.passes,
        }


@dataclass(frozen=True)
class ComparisonReport:
    """Noisy baseline vs both filters at one density (metrics.py:78-124)."""

    width: int
    height: int
    noise_density: float
    noisy: MethodResult
    mf: MethodResult
    fnr: MethodResult

    @property
    def psnr_gain_db(self) -> float:
        return self.fnr.psnr_db - self.mf.psnr_db

    @property
    def sort_reduction_fraction(self) -> float:
        if self.mf.sorts == 0:
            return 0.0
        return 1.0 - self.fnr.sorts / self.mf.sorts

    def to_dict(self) -> dict:
        return {
            "width": self.width,
            "height": self.height,
            "noise_density": self.noise_density,
            "methods": {
                "noisy": self.noisy.to_dict(),
                "mf": self.mf.to_dict(),
                "fnr": self.fnr.to_dict(),
            },
            "psnr_gain_db": format_db(self.psnr_gain_db),
            "sort_reduction_fraction": f"{self.sort_reduction_fraction:.4f}",
        }


def format_db(value: float) -> str:
    """Fixed 4-decimal dB string; infinity becomes "inf" (metrics.py:127-131)."""
    return "inf" if math.isinf(value) else f"{value:.4f}"


def _result(original, out, stats: FilterStats) -> MethodResult:
    return MethodResult(psnr_db=psnr(original, out), sorts=stats.sorts, minmax_scans=stats.minmax_scans,
                        elapsed_ms=stats.elapsed_ms, passes=stats.passes)


def build_comparison(original, noisy, mf_output, mf_stats: FilterStats, fnr_output, fnr_stats: FilterStats,
                     noise_density: float) -> ComparisonReport:
    """One comparison row, all PSNRs against the clean original (metrics.py:134-157)."""
    shape = _shape_of(original)
    for other in (noisy, mf_output, fnr_output):
        if _shape_of(other) != shape:
            raise ValueError("all images in a comparison must share dimensions")
    h, w = shape[-2], shape[-1]
    return ComparisonReport(width=w, height=h, noise_density=noise_density,
                            noisy=MethodResult(psnr_db=psnr(original, noisy)),
                            mf=_result(original, mf_output, mf_stats),
                            fnr=_result(original, fnr_output, fnr_stats))
