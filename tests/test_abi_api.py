"""CPU-side checks of the C ABI library and the reference-mirroring Python surface.

No kernel is launched here: these run on the build container (no GPU).
"""

import inspect
import os
import re
import sys

import numpy as np
import pytest

from conftest import REPO, gpu_available, load_golden

import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native


def _header_symbols():
    text = open(os.path.join(REPO, "include", "irdn.h")).read()
    return sorted(set(re.findall(r"IRDN_API\s+[\w\s\*]+?\b(irdn_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _native.load_lib()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_native.EXPORTED) == syms


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_version_and_device_query():
    assert "sm_100a" in _native.version()
    n = _native.device_count()
    assert n >= 0
    if not gpu_available():
        assert n == 0


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_compute_fails_loudly_without_gpu():
    img = np.zeros((8, 8), np.uint8)
    with pytest.raises(_native.NativeError):
        P.run_filter(img, P.WindowSpec(3), "fnr")


def test_validation_mirrors_reference_errors():
    img = P.GrayImage(4, 4, bytes(16))
    with pytest.raises(ValueError, match="unknown method"):
        P.run_filter(img, P.WindowSpec(3), "median")
    with pytest.raises(ValueError, match="passes must be >= 1"):
        P.run_filter(img, P.WindowSpec(3), "fnr", passes=0)
    with pytest.raises(ValueError, match="odd integer >= 3"):
        P.WindowSpec(4)
    with pytest.raises(ValueError, match="odd integer >= 3"):
        P.WindowSpec(1)
    with pytest.raises(ValueError, match="dimensions"):
        P.GrayImage(0, 3, b"")
    with pytest.raises(ValueError, match="expected 6"):
        P.GrayImage(2, 3, bytes(5))
    with pytest.raises(IndexError):
        P.extract_window(img, 4, 0, P.WindowSpec(3))
    with pytest.raises(TypeError):
        P.run_filter(np.zeros((4, 4), np.float32), P.WindowSpec(3), "fnr")


def test_c_abi_rejects_bad_arguments_before_device_work():
    lib = _native.load_lib()
    # bad method / k / dims / passes -> IRDN_EINVAL, whatever the device situation
    assert lib.irdn_run_filter_u8(1, 2, 1, 4, 4, 3, 7, 1, 0, None) == _native.IRDN_EINVAL
    assert b"unknown method" in lib.irdn_last_error()
    assert lib.irdn_run_filter_u8(1, 2, 1, 4, 4, 4, 0, 1, 0, None) == _native.IRDN_EINVAL
    assert lib.irdn_run_filter_u16(1, 2, 1, 0, 4, 3, 0, 1, 0, None) == _native.IRDN_EINVAL
    assert lib.irdn_run_filter_u8(1, 2, 1, 4, 4, 3, 0, 0, 0, None) == _native.IRDN_EINVAL
    assert lib.irdn_filter_pass_u8(16, 16, 1, 4, 4, 4, 4, 3, 0, 64, None) == _native.IRDN_EINVAL
    assert b"overlap" in lib.irdn_last_error()
    assert lib.irdn_filter_strip_u8(1, 5, 3, 2, 2, 12, 20, 8, 8, 8, 5, 0, 64, None) == _native.IRDN_EINVAL
    assert b"cover" in lib.irdn_last_error()


def test_reference_surface_is_mirrored():
    ref_filter_names = ["FilterStats", "WindowExtrema", "classify_pixel", "fnr_pass", "mf_pass",
                        "run_filter", "window_extrema", "GrayImage", "Window", "WindowSpec",
                        "extract_window", "get_pixel", "new_image", "PgmError"]
    for n in ref_filter_names:
        assert hasattr(P, n), n
    sig = inspect.signature(P.run_filter)
    params = list(sig.parameters.values())
    assert [p.name for p in params[:5]] == ["img", "spec", "method", "passes", "threads"]
    assert params[3].default == 1 and params[4].default == 1
    assert all(p.kind == p.KEYWORD_ONLY for p in params[5:])
    st = P.FilterStats()
    assert list(st.to_dict()) == ["minmax_scans", "sorts", "replacements", "detected",
                                  "elapsed_ms", "passes"]


def test_per_window_api_spec_examples():
    """SPEC.md:73-75, :241-243, :251-253 known answers."""
    img = P.GrayImage(3, 3, bytes([1, 2, 3, 4, 5, 6, 7, 8, 9]))
    w = P.extract_window(img, 1, 1, P.WindowSpec(3))
    assert w.values == [1, 2, 3, 4, 5, 6, 7, 8, 9] and w.center_index == 4
    assert P.extract_window(img, 0, 0, P.WindowSpec(3)).values == [1, 1, 2, 1, 1, 2, 4, 4, 5]
    assert P.extract_window(P.GrayImage(1, 1, b"\x09"), 0, 0, P.WindowSpec(3)).values == [9] * 9
    st = P.FilterStats()
    e = P.window_extrema(P.Window([12, 200, 45, 0, 88, 13, 255, 7, 99], 4), st)
    assert (e.min_gray, e.max_gray) == (0, 255) and st.minmax_scans == 1
    assert P.classify_pixel(P.Window(list(range(1, 10)), 8), P.window_extrema(P.Window(list(range(1, 10)), 8)))
    assert not P.classify_pixel(w, P.window_extrema(w))
    flat = P.Window([7] * 9, 4)
    assert P.classify_pixel(flat, P.window_extrema(flat))
    assert P.get_pixel(P.GrayImage(2, 2, bytes([1, 2, 3, 4])), 1, 0) == 2
    assert P.new_image(3, 2, 7).pixels == bytearray([7] * 6)


def test_host_package_never_imports_the_oracle():
    pkg = os.path.join(REPO, "paper_1201_3972_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".c", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).lower() or f == "build.py", f
