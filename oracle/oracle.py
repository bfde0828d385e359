"""Python access to the FNR oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module. It is the checker, never the thing measured or shipped:
the product package (paper_1201_3972_b200) does not import it.

Two independent restatements of the reference filter
(pkg/src/irdenoise/filters.py:130-181 + sorting.py:51-56):

* ``run_filter_c`` / ``filter_rows_c``: ctypes binding to the plain-C
  restatement in fnr_oracle.c (introsort medians, pthread row bands,
  FilterStats counters). This is the primary oracle and the CPU baseline.
* ``run_filter_np``: a vectorised numpy restatement (edge padding +
  sliding windows + partition at (k*k-1)//2); used to cross-check the C
  oracle on random inputs.

Both are pinned against golden vectors produced by the reference package
itself (tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_fnr.so")
# input preparation (seeded BASELINE scenes), linked into the oracle library as well
SCENE_SRC = os.path.join(os.path.dirname(HERE), "paper_1201_3972_b200", "csrc", "scene.c")


class OracleStats(ctypes.Structure):
    _fields_ = [
        ("minmax_scans", ctypes.c_uint64),
        ("sorts", ctypes.c_uint64),
        ("replacements", ctypes.c_uint64),
        ("detected", ctypes.c_uint64),
        ("elapsed_ms", ctypes.c_double),
        ("passes", ctypes.c_uint64),
        ("comparisons", ctypes.c_uint64),
        ("depth_switches", ctypes.c_uint64),
    ]


class _SortCounters(ctypes.Structure):
    _fields_ = [("sorts_performed", ctypes.c_uint64), ("comparisons", ctypes.c_uint64),
                ("depth_switches", ctypes.c_uint64)]


class PassCounts(ctypes.Structure):
    _fields_ = [("minmax_scans", ctypes.c_uint64), ("detected", ctypes.c_uint64),
                ("replacements", ctypes.c_uint64), ("sort", _SortCounters)]


_lib = None


def build() -> str:
    """Compile fnr_oracle.c into liboracle_fnr.so (idempotent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        srcs = [os.path.join(HERE, "fnr_oracle.c"), SCENE_SRC]
        if not os.path.exists(LIB_PATH) or any(os.path.exists(f) and os.path.getmtime(LIB_PATH) <
                                               os.path.getmtime(f) for f in srcs):
            build()
        l = ctypes.CDLL(LIB_PATH)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        l.oracle_run_filter.argtypes = [vp, ctypes.c_int, i64, i64, i64, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(OracleStats)]
        l.oracle_run_filter.restype = ctypes.c_int
        l.oracle_filter_rows.argtypes = [vp, ctypes.c_int, i64, i64, ctypes.c_int, i64, i64, vp,
                                         ctypes.c_int, ctypes.POINTER(PassCounts)]
        l.oracle_filter_rows.restype = None
        l.oracle_median_of.argtypes = [vp, ctypes.c_int, ctypes.POINTER(_SortCounters),
                                       ctypes.POINTER(ctypes.c_int32)]
        l.oracle_median_of.restype = ctypes.c_int
        l.oracle_sort_values.argtypes = [vp, ctypes.c_int, ctypes.POINTER(_SortCounters)]
        l.oracle_sort_values.restype = ctypes.c_int
        l.oracle_inject_impulse.argtypes = [vp, vp, vp, i64, ctypes.c_uint64, ctypes.c_double,
                                            ctypes.c_double]
        l.oracle_inject_impulse.restype = ctypes.c_uint64
        l.oracle_sq_err_sum.argtypes = [vp, vp, ctypes.c_int, i64]
        l.oracle_sq_err_sum.restype = ctypes.c_uint64
        l.scene_generate.restype = ctypes.c_int
        l.scene_generate.argtypes = [vp, i64, i64, vp, ctypes.c_int32]
        _lib = l
    return _lib


@dataclass
class Stats:
    minmax_scans: int
    sorts: int
    replacements: int
    detected: int
    passes: int
    comparisons: int = 0
    depth_switches: int = 0

    def counters(self) -> tuple:
        return (self.minmax_scans, self.sorts, self.replacements, self.detected, self.passes)


def _as_frames(img: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(img)
    if a.dtype not in (np.uint8, np.uint16):
        raise TypeError(f"oracle handles uint8/uint16 pixels, got {a.dtype}")
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("expected [H,W] or [B,H,W]")
    return a


def run_filter_c(img: np.ndarray, k: int, method: str = "fnr", passes: int = 1,
                 threads: int = 1) -> tuple[np.ndarray, Stats]:
    """C restatement of run_filter over [H,W] or [B,H,W] u8/u16 frames."""
    a = _as_frames(img)
    out = np.empty_like(a)
    st = OracleStats()
    m = {"fnr": 0, "mf": 1}[method]
    rc = lib().oracle_run_filter(a.ctypes.data, a.itemsize, a.shape[0], a.shape[2], a.shape[1], k, m,
                                 passes, threads, out.ctypes.data, ctypes.byref(st))
    if rc != 0:
        raise ValueError(f"oracle_run_filter rejected the arguments (rc={rc})")
    res = out if img.ndim == 3 else out[0]
    return res, Stats(st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes,
                      st.comparisons, st.depth_switches)


def filter_rows_c(frame: np.ndarray, k: int, y0: int, y1: int, method: str = "fnr"):
    """_filter_rows(img, k, y0, y1) of ONE full frame: returns (rows [y0,y1), (detected, replacements))."""
    a = np.ascontiguousarray(frame)
    assert a.ndim == 2 and 0 <= y0 < y1 <= a.shape[0]
    out = np.empty((y1 - y0, a.shape[1]), dtype=a.dtype)
    pc = PassCounts()
    # filter_rows writes out[y*w + x] for y in [y0, y1): hand it a base shifted back by y0 rows
    base = out.ctypes.data - y0 * a.shape[1] * a.itemsize
    lib().oracle_filter_rows(a.ctypes.data, a.itemsize, a.shape[1], a.shape[0], k, y0, y1,
                             base, 1 if method == "fnr" else 0, ctypes.byref(pc))
    return out, (pc.detected, pc.replacements)


def median_of_c(values) -> int:
    buf = (ctypes.c_int32 * len(values))(*values)
    sc = _SortCounters()
    out = ctypes.c_int32()
    if lib().oracle_median_of(buf, len(values), ctypes.byref(sc), ctypes.byref(out)) != 0:
        raise ValueError(f"median needs an odd-length sequence, got length {len(values)}")
    return out.value


def sort_values_c(values) -> tuple[list[int], int, int]:
    buf = (ctypes.c_int32 * len(values))(*values)
    sc = _SortCounters()
    if lib().oracle_sort_values(buf, len(values), ctypes.byref(sc)) != 0:
        raise ValueError("cannot sort an empty sequence")
    return list(buf), sc.comparisons, sc.depth_switches


def run_filter_np(img: np.ndarray, k: int, method: str = "fnr", passes: int = 1):
    """Vectorised numpy restatement (independent of the C oracle)."""
    from numpy.lib.stride_tricks import sliding_window_view

    a = _as_frames(img)
    r = k // 2
    rank = (k * k - 1) // 2
    scans = sorts = repl = det = 0
    cur = a
    for _ in range(passes):
        out = np.empty_like(cur)
        for b in range(cur.shape[0]):
            f = cur[b]
            p = np.pad(f, r, mode="edge")
            win = sliding_window_view(p, (k, k)).reshape(f.shape[0], f.shape[1], k * k)
            med = np.partition(win, rank, axis=2)[:, :, rank]
            if method == "mf":
                out[b] = med
                sorts += f.size
            else:
                mn, mx = win.min(axis=2), win.max(axis=2)
                noisy = (f == mn) | (f == mx)
                out[b] = np.where(noisy, med, f)
                scans += f.size
                det += int(noisy.sum())
                repl += int((noisy & (med != f)).sum())
                sorts += int(noisy.sum())
        cur = out
    res = cur if img.ndim == 3 else cur[0]
    return res, Stats(scans, sorts, repl, det, passes)


def inject_impulse_c(pixels: np.ndarray, seed: int, density: float, salt_fraction: float = 0.5):
    """noise.py:89-106 restated in C: returns (noisy u8 array, flags u8 array, count)."""
    a = np.ascontiguousarray(pixels, dtype=np.uint8)
    out = np.empty_like(a)
    flags = np.empty_like(a)
    cnt = lib().oracle_inject_impulse(a.ctypes.data, out.ctypes.data, flags.ctypes.data, a.size,
                                      seed & 0xFFFFFFFFFFFFFFFF, density, salt_fraction)
    return out, flags, int(cnt)


def sq_err_sum_c(a: np.ndarray, b: np.ndarray) -> int:
    """metrics.py:29-32 numerator (exact)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.dtype == b.dtype and a.size == b.size
    return int(lib().oracle_sq_err_sum(a.ctypes.data, b.ctypes.data, a.dtype.itemsize, a.size))
