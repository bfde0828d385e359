"""ctypes shim that routes the REFERENCE package's filter onto the B200 kernels.

This is the binding INTEGRATION.md §2 describes: the unmodified reference
(`irdenoise` 0.1.0) keeps its own GrayImage / FilterStats / CLI / metrics, and only its
filter entry points are re-pointed at the C ABI (include/irdn.h):

    filters.run_filter  (filters.py:79-102)  -> irdn_run_filter_u8
    filters.fnr_pass    (filters.py:69-71)   -> irdn_run_filter_u8, method fnr, 1 pass
    filters.mf_pass     (filters.py:74-76)   -> irdn_run_filter_u8, method mf, 1 pass

`install(irdenoise)` patches the package in place (and `irdenoise.cli`, whose
`from .filters import run_filter` binding would otherwise keep the CPU version), so
`irdenoise.cli.main(["filter", ...])` and `["bench", ...]` (cli.py:97-164) run on the
GPU unchanged. The file depends only on ctypes and on the package it is installed
into: a maintainer can drop it into the reference as `irdenoise/_b200.py` and call
`install(sys.modules[__name__])` from `irdenoise/__init__.py`.

There is no CPU fallback: without the library or a B200 the filter raises (CUDA
failures as RuntimeError, argument errors as the reference's ValueError).
"""

from __future__ import annotations

import ctypes
import os
import sys
import time

_HERE = os.path.dirname(os.path.abspath(__file__))


class _Stats(ctypes.Structure):  # struct irdn_stats, include/irdn.h
    _fields_ = [("minmax_scans", ctypes.c_uint64), ("sorts", ctypes.c_uint64),
                ("replacements", ctypes.c_uint64), ("detected", ctypes.c_uint64),
                ("elapsed_ms", ctypes.c_double), ("passes", ctypes.c_uint64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        path = os.environ.get("IRDN_LIB") or os.path.join(_HERE, "libirdn.so")
        lib = ctypes.CDLL(path)
        lib.irdn_run_filter_u8.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_int32, ctypes.POINTER(_Stats)]
        lib.irdn_run_filter_u8.restype = ctypes.c_int
        lib.irdn_last_error.restype = ctypes.c_char_p
        lib.irdn_last_error.argtypes = []
        _lib = lib
    return _lib


def _filter(img, k: int, fnr: bool, passes: int) -> tuple[bytearray, _Stats]:
    """passes passes over the image's bytes on the GPU; returns the fresh output buffer."""
    lib = _load()
    n = img.width * img.height
    src = bytes(img.pixels) if not isinstance(img.pixels, bytearray) else img.pixels
    out = bytearray(n)
    src_c = (ctypes.c_char * n).from_buffer_copy(src) if isinstance(src, bytes) else (ctypes.c_char * n).from_buffer(src)
    dst_c = (ctypes.c_char * n).from_buffer(out)
    st = _Stats()
    rc = lib.irdn_run_filter_u8(ctypes.addressof(src_c), ctypes.addressof(dst_c), 1, img.height, img.width,
                                k, 0 if fnr else 1, passes, int(os.environ.get("IRDN_DEVICE", "0")),
                                ctypes.byref(st))
    del src_c, dst_c
    if rc == 1:
        raise ValueError(lib.irdn_last_error().decode())
    if rc != 0:
        raise RuntimeError(lib.irdn_last_error().decode())
    return out, st


def install(pkg) -> None:
    """Re-point `pkg` (the imported reference package) at the GPU filter."""
    fil = pkg.filters
    GrayImage, FilterStats = pkg.image.GrayImage, fil.FilterStats
    FNR, MF = fil.METHOD_FNR, fil.METHOD_MF

    def run_filter(img, spec, method, passes=1, threads=1):
        if method not in (FNR, MF):
            raise ValueError(f"unknown method {method!r}, expected 'fnr' or 'mf'")
        if passes < 1:
            raise ValueError(f"passes must be >= 1, got {passes}")
        t0 = time.perf_counter()
        out, st = _filter(img, spec.k, method == FNR, passes)
        stats = FilterStats(minmax_scans=st.minmax_scans, sorts=st.sorts, replacements=st.replacements,
                            detected=st.detected, passes=st.passes)
        stats.elapsed_ms = (time.perf_counter() - t0) * 1000.0
        return GrayImage(img.width, img.height, out), stats

    def _one_pass(fnr):
        def pass_fn(img, spec, stats):
            out, st = _filter(img, spec.k, fnr, 1)
            stats.minmax_scans += st.minmax_scans
            stats.detected += st.detected
            stats.replacements += st.replacements
            stats.sorts += st.sorts
            stats.passes += 1
            return GrayImage(img.width, img.height, out)
        return pass_fn

    run_filter.__doc__ = fil.run_filter.__doc__
    fil.run_filter, fil.fnr_pass, fil.mf_pass = run_filter, _one_pass(True), _one_pass(False)
    pkg.run_filter, pkg.fnr_pass, pkg.mf_pass = fil.run_filter, fil.fnr_pass, fil.mf_pass
    cli = sys.modules.get(pkg.__name__ + ".cli")
    if cli is not None:
        cli.run_filter = run_filter
    pkg.B200_SHIM = True
