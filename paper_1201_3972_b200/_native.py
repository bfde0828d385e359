"""ctypes bindings to the in-tree native libraries.

* ``libirdn.so``       — the sm_100a filter kernels behind the C ABI in
  include/irdn.h (the product path). There is no CPU fallback: if the
  library is missing, or no B200 is visible, every filter call raises.
* ``libirdn_scene.so`` — seeded synthetic scene generation (bench/test input).
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# IRDN_LIB selects an alternative build of the same library (kernel-variant experiments).
LIB_PATH = os.environ.get("IRDN_LIB") or os.path.join(PKG_DIR, "libirdn.so")
SCENE_LIB_PATH = os.path.join(PKG_DIR, "libirdn_scene.so")

IRDN_OK, IRDN_EINVAL, IRDN_ECUDA, IRDN_ENODEV = 0, 1, 2, 3
METHODS = {"fnr": 0, "mf": 1}

_lock = threading.Lock()
_lib = None
_scene = None


class IrdnStats(ctypes.Structure):
    """struct irdn_stats (include/irdn.h) == FilterStats fields (filters.py:33-52)."""

    _fields_ = [
        ("minmax_scans", ctypes.c_uint64),
        ("sorts", ctypes.c_uint64),
        ("replacements", ctypes.c_uint64),
        ("detected", ctypes.c_uint64),
        ("elapsed_ms", ctypes.c_double),
        ("passes", ctypes.c_uint64),
    ]


class NativeError(RuntimeError):
    """A CUDA-side failure reported by libirdn (IRDN_ECUDA / IRDN_ENODEV)."""


EXPORTED = [
    "irdn_version", "irdn_last_error", "irdn_device_count", "irdn_fast_window_mask",
    "irdn_filter_pass_u8", "irdn_filter_pass_u16", "irdn_filter_strip_u8", "irdn_filter_strip_u16",
    "irdn_run_filter_u8", "irdn_run_filter_u16", "irdn_run_filter_device_u8",
    "irdn_run_filter_device_u16", "irdn_launch_count", "irdn_reset_launch_count",
    "irdn_set_force_generic", "irdn_inject_impulse_u8", "irdn_sq_err_sum_u8", "irdn_sq_err_sum_u16",
    "irdn_set_host_return", "irdn_last_transfer", "irdn_delta_region_bytes", "irdn_delta_encode_u8",
    "irdn_delta_encode_u16", "irdn_delta_decode_u8", "irdn_delta_decode_u16", "irdn_set_multipass",
    "irdn_ipc_export", "irdn_ipc_open", "irdn_ipc_close", "irdn_scene_render",
]

HOST_RETURN = {"auto": 0, "full": 1, "delta": 2}


class IrdnSceneDesc(ctypes.Structure):
    """irdn_scene_desc (include/irdn.h)."""

    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("bytes_per_pixel", ctypes.c_int32),
        ("maxval", ctypes.c_int32), ("nblobs", ctypes.c_int32), ("nlines", ctypes.c_int32),
        ("nrects", ctypes.c_int32), ("impulse_kind", ctypes.c_int32), ("config_id", ctypes.c_int32),
        ("sensor", ctypes.c_int32), ("scale", ctypes.c_double), ("sensor_mul", ctypes.c_double),
        ("line_amp", ctypes.c_double), ("rect_amp", ctypes.c_double), ("density", ctypes.c_double),
        ("seed", ctypes.c_uint64), ("frame0", ctypes.c_int64), ("nframes", ctypes.c_int64),
        ("gx", ctypes.c_void_p), ("gy", ctypes.c_void_p), ("lines", ctypes.c_void_p), ("rects", ctypes.c_void_p),
    ]


def _declare(l: ctypes.CDLL) -> None:
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    l.irdn_version.restype = ctypes.c_char_p
    l.irdn_version.argtypes = []
    l.irdn_last_error.restype = ctypes.c_char_p
    l.irdn_last_error.argtypes = []
    l.irdn_device_count.restype = ctypes.c_int
    l.irdn_device_count.argtypes = []
    l.irdn_fast_window_mask.restype = ctypes.c_uint64
    l.irdn_fast_window_mask.argtypes = [i32]
    for t in ("u8", "u16"):
        f = getattr(l, f"irdn_filter_pass_{t}")
        f.argtypes = [vp, vp, i64, i64, i64, i64, i64, i32, i32, vp, vp]
        f.restype = ctypes.c_int
        f = getattr(l, f"irdn_filter_strip_{t}")
        f.argtypes = [vp, i64, i64, vp, i64, i64, i64, i64, i64, i64, i32, i32, vp, vp]
        f.restype = ctypes.c_int
        f = getattr(l, f"irdn_run_filter_{t}")
        f.argtypes = [vp, vp, i64, i64, i64, i32, i32, i32, i32, ctypes.POINTER(IrdnStats)]
        f.restype = ctypes.c_int
        f = getattr(l, f"irdn_run_filter_device_{t}")
        f.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32, i32, vp, vp]
        f.restype = ctypes.c_int
    l.irdn_launch_count.restype = ctypes.c_uint64
    l.irdn_launch_count.argtypes = []
    l.irdn_reset_launch_count.restype = None
    l.irdn_reset_launch_count.argtypes = []
    l.irdn_set_force_generic.restype = i32
    l.irdn_set_force_generic.argtypes = [i32]
    l.irdn_inject_impulse_u8.restype = ctypes.c_int
    l.irdn_inject_impulse_u8.argtypes = [vp, vp, vp, i64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                         vp, vp]
    for t in ("u8", "u16"):
        f = getattr(l, f"irdn_sq_err_sum_{t}")
        f.restype = ctypes.c_int
        f.argtypes = [vp, vp, i64, vp, vp]
    u64 = ctypes.c_uint64
    l.irdn_set_multipass.restype = i32
    l.irdn_set_multipass.argtypes = [i32]
    l.irdn_set_host_return.restype = i32
    l.irdn_set_host_return.argtypes = [i32]
    l.irdn_last_transfer.restype = None
    l.irdn_last_transfer.argtypes = [ctypes.POINTER(u64), ctypes.POINTER(u64)]
    l.irdn_ipc_export.restype = ctypes.c_int
    l.irdn_ipc_export.argtypes = [vp, vp, ctypes.POINTER(u64)]
    l.irdn_ipc_open.restype = ctypes.c_int
    l.irdn_ipc_open.argtypes = [vp, u64, ctypes.POINTER(vp)]
    l.irdn_ipc_close.restype = ctypes.c_int
    l.irdn_ipc_close.argtypes = [vp, u64]
    l.irdn_scene_render.restype = ctypes.c_int
    l.irdn_scene_render.argtypes = [ctypes.POINTER(IrdnSceneDesc), vp, vp]
    l.irdn_delta_region_bytes.restype = u64
    l.irdn_delta_region_bytes.argtypes = [i64, i32]
    for t in ("u8", "u16"):
        f = getattr(l, f"irdn_delta_encode_{t}")
        f.restype = ctypes.c_int
        f.argtypes = [vp, vp, i64, vp, vp]
        f = getattr(l, f"irdn_delta_decode_{t}")
        f.restype = u64
        f.argtypes = [vp, vp, vp, i64, i32]


def load_lib() -> ctypes.CDLL:
    """Load libirdn.so (the CUDA path). Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: the sm_100a CUDA library has not been built "
                    "(run `python -c 'import __graft_entry__; __graft_entry__.build()'`). "
                    "There is no CPU fallback.")
            l = ctypes.CDLL(LIB_PATH)
            _declare(l)
            _lib = l
    return _lib


def load_scene_lib() -> ctypes.CDLL:
    global _scene
    with _lock:
        if _scene is None:
            if not os.path.exists(SCENE_LIB_PATH):
                raise ImportError(f"{SCENE_LIB_PATH} is missing; run the build first")
            l = ctypes.CDLL(SCENE_LIB_PATH)
            l.scene_generate.restype = ctypes.c_int
            l.scene_generate.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_int32]
            l.scene_tables.restype = ctypes.c_int
            l.scene_tables.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
            _scene = l
    return _scene


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference's exception types."""
    if rc == IRDN_OK:
        return
    msg = load_lib().irdn_last_error().decode("utf-8", "replace")
    if rc == IRDN_EINVAL:
        raise ValueError(msg)
    raise NativeError(msg)


def last_transfer() -> tuple[int, int]:
    """(h2d, d2h) bytes moved by this thread's last irdn_run_filter_* call."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    load_lib().irdn_last_transfer(ctypes.byref(a), ctypes.byref(b))
    return int(a.value), int(b.value)


def set_host_return(mode: str) -> str:
    """Result return of the host-buffer path: "auto", "full" or "delta"; returns the previous mode."""
    prev = int(load_lib().irdn_set_host_return(HOST_RETURN[mode]))
    return {v: k for k, v in HOST_RETURN.items()}[prev]


def version() -> str:
    return load_lib().irdn_version().decode()


def device_count() -> int:
    return int(load_lib().irdn_device_count())
