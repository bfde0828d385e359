"""The drop-in boundary against the reference's own objects and surface.

* The reference's public names (irdenoise/__init__.py:9-44) that belong to the filter
  path exist here too, including the per-window sort API (sorting.py:19-56), whose
  results and counters are pinned to goldens made by running the reference.
* run_filter accepts the reference's GrayImage / WindowSpec objects (duck-typed) and
  returns the caller's GrayImage class.
* reference_shim re-points the UNMODIFIED reference package (baseline/_ref) at the C ABI
  (INTEGRATION.md §2); its CLI then runs on the GPU (GPU half in test_gpu_noise_metrics).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native, reference_shim, sorting

FILTER_SURFACE = ["FilterStats", "WindowExtrema", "classify_pixel", "fnr_pass", "mf_pass", "run_filter",
                  "window_extrema", "GrayImage", "Window", "WindowSpec", "extract_window", "get_pixel",
                  "new_image", "SortCounters", "median_of", "sort_values"]


def test_reference_filter_surface_is_exported(reference_pkg):
    for name in FILTER_SURFACE:
        assert name in reference_pkg.__all__, name
        assert name in P.__all__ and hasattr(P, name), name


def test_sort_api_matches_reference_goldens():
    """sorting.py:35-161: sorted output, comparison and heapsort-switch counters."""
    z = np.load(os.path.join(GOLDEN, "ref_sort.npz"))
    meta = json.loads(str(z["meta"]))
    switched = 0
    for i, m in enumerate(meta):
        vals = z[f"in{i}"].tolist()
        c = sorting.SortCounters()
        assert sorting.sort_values(vals, c) == z[f"out{i}"].tolist()
        assert (c.comparisons, c.depth_switches, c.sorts_performed) == (m["comparisons"], m["depth_switches"], 1), m
        switched += c.depth_switches > 0
        if m["median"] is not None:
            c2 = sorting.SortCounters()
            assert P.median_of(vals, c2) == m["median"] and c2.comparisons == m["comparisons"]
    assert switched > 0
    with pytest.raises(ValueError, match="odd-length"):
        P.median_of([1, 2], P.SortCounters())
    with pytest.raises(ValueError, match="empty"):
        P.sort_values([], P.SortCounters())
    a, b = P.SortCounters(), P.SortCounters()
    P.median_of([3, 1, 2], a)
    b.merge(a)
    b.merge(a)
    assert b.sorts_performed == 2 and b.comparisons == 2 * a.comparisons


def test_sort_api_agrees_with_reference_on_random_multisets(reference_pkg):
    rs = reference_pkg.sorting
    rng = np.random.default_rng(3)
    for n in list(range(1, 40)) + [49, 121, 255, 600]:
        for dist in (256, 4, 2):
            vals = rng.integers(0, dist, n).tolist()
            ca, cb = P.SortCounters(), rs.SortCounters()
            assert P.sort_values(vals, ca) == rs.sort_values(vals, cb)
            assert (ca.comparisons, ca.depth_switches) == (cb.comparisons, cb.depth_switches), (n, dist)


def test_reference_objects_reach_the_native_layer(reference_pkg):
    """Reference GrayImage / WindowSpec are accepted (no TypeError); validation happens
    before any GPU work; without a B200 the call fails in the C ABI, never on the CPU."""
    img = reference_pkg.GrayImage(4, 3, bytearray(range(12)))
    spec = reference_pkg.WindowSpec(3)
    with pytest.raises(ValueError, match="unknown method"):
        P.run_filter(img, spec, "median")
    with pytest.raises(ValueError, match="passes"):
        P.run_filter(img, spec, "fnr", passes=0)
    with pytest.raises(ValueError):
        P.run_filter(img, 4, "fnr")  # even window
    try:
        out, st = P.run_filter(img, spec, "fnr")
    except _native.NativeError:
        return  # no GPU here: the product path has no CPU fallback
    assert type(out) is type(img)


def test_shim_patches_the_reference_in_place(reference_pkg, monkeypatch):
    import importlib

    cli = importlib.import_module(reference_pkg.__name__ + ".cli")
    reference_shim.install(reference_pkg)
    assert reference_pkg.filters.run_filter is reference_pkg.run_filter is cli.run_filter
    assert reference_pkg.filters.run_filter.__module__ == reference_shim.__name__
    img = reference_pkg.GrayImage(2, 2, bytearray(4))
    with pytest.raises(ValueError, match="unknown method"):
        reference_pkg.run_filter(img, reference_pkg.WindowSpec(3), "xx")
    with pytest.raises(ValueError, match="passes"):
        reference_pkg.run_filter(img, reference_pkg.WindowSpec(3), "fnr", passes=0)


@pytest.mark.gpu
def test_reference_objects_on_the_gpu(cuda_ok, reference_pkg):
    """run_filter on the reference's own GrayImage: same class back, same bytes and
    counters as the reference's run_filter (filters.py:79-102) on the same image."""
    from paper_1201_3972_b200 import launcher  # noqa: F401 (the shim is not installed here)

    rng = np.random.default_rng(11)
    for (w, h), k, method, passes in [((37, 29), 3, "fnr", 1), ((64, 48), 5, "mf", 2), ((23, 17), 7, "fnr", 2)]:
        px = bytearray(rng.integers(0, 256, w * h, dtype=np.uint8).tobytes())
        img = reference_pkg.GrayImage(w, h, px)
        got, st = P.run_filter(img, reference_pkg.WindowSpec(k), method, passes)
        assert type(got) is reference_pkg.GrayImage
        want, wst = _reference_cpu_run_filter(reference_pkg, img, k, method, passes)
        assert got == want
        assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == \
            [wst.minmax_scans, wst.sorts, wst.replacements, wst.detected, wst.passes]


def _reference_cpu_run_filter(ref, img, k, method, passes):
    """The reference's own (CPU) run_filter, even after the shim was installed."""
    fil = ref.filters
    st = fil.FilterStats()
    cur = img
    for _ in range(passes):
        cur = fil._run_rows_threaded(cur, ref.WindowSpec(k), st, fnr=(method == "fnr"), threads=1)
    return cur, st
