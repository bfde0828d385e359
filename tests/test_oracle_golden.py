"""Pin the CPU oracle (oracle/fnr_oracle.c + the numpy restatement) to the reference.

Every golden vector was produced by running the reference package itself
(tests/golden/make_golden.py): run_filter for u8, the per-window API
composition for u16, sort_values / median_of for the introsort counters.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle

GOLDEN_SETS = ["ref_u8.npz", "ref_u16.npz", "ref_fixtures.npz", "ref_configs.npz"]


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_c_oracle_matches_reference_golden(name):
    cases = load_golden(name)
    assert cases
    for meta, inp, out in cases:
        got, st = oracle.run_filter_c(inp, meta["k"], meta["method"], meta["passes"])
        assert got.dtype == out.dtype
        assert np.array_equal(got, out), (name, meta)
        assert list(st.counters()) == meta["stats"], (name, meta, st)


@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_numpy_restatement_matches_reference_golden(name):
    for meta, inp, out in load_golden(name):
        got, st = oracle.run_filter_np(inp, meta["k"], meta["method"], meta["passes"])
        assert np.array_equal(got, out), (name, meta)
        assert list(st.counters()) == meta["stats"], (name, meta)


def test_structured_fixture_appendix_a_hashes():
    """the reference's own structured_image + inject_impulse known answers."""
    import hashlib

    want = {(0.2, 3, "fnr", 1): "d5da32b53aed674a", (0.2, 3, "fnr", 2): "525ab57d5cf05732",
            (0.2, 3, "mf", 1): "efdc8c741a827e32", (0.2, 11, "fnr", 1): "b60ac78a597b9da1",
            (0.3, 7, "fnr", 1): "bc4f2f3352cdfb4d"}
    seen = 0
    for meta, inp, out in load_golden("ref_fixtures.npz"):
        if not meta["kind"].startswith("structured"):
            continue
        d = float(meta["kind"].split("_d")[1])
        key = (d, meta["k"], meta["method"], meta["passes"])
        got, _ = oracle.run_filter_c(inp, meta["k"], meta["method"], meta["passes"])
        assert hashlib.sha256(got.tobytes()).hexdigest()[:16] == meta["sha"]
        if key in want:
            assert meta["sha"] == want[key]
            seen += 1
    assert seen == len(want)


def test_spec_count_exactness_364x244():
    """SPEC.md:459 / :283 — one MF pass sorts 88,816 times; two passes 177,632."""
    cases = [c for c in load_golden("ref_fixtures.npz") if c[0]["kind"] == "ramp364x244"]
    mf2 = [c for c in cases if c[0]["method"] == "mf" and c[0]["passes"] == 2][0]
    _, st = oracle.run_filter_c(mf2[1], 3, "mf", 2)
    assert st.sorts == 177_632
    fnr = [c for c in cases if c[0]["method"] == "fnr" and c[0]["passes"] == 1][0]
    _, st = oracle.run_filter_c(fnr[1], 3, "fnr", 1)
    assert st.minmax_scans == 88_816


def test_introsort_restatement_counters():
    """sorting.py:35-161 restated in C: same order, comparisons and heapsort switches."""
    import json
    import os

    from conftest import GOLDEN

    z = np.load(os.path.join(GOLDEN, "ref_sort.npz"))
    meta = json.loads(str(z["meta"]))
    switched = 0
    for i, m in enumerate(meta):
        vals = z[f"in{i}"].tolist()
        srt, comps, switches = oracle.sort_values_c(vals)
        assert srt == z[f"out{i}"].tolist()
        assert comps == m["comparisons"], m
        assert switches == m["depth_switches"], m
        switched += switches > 0
        if m["median"] is not None:
            assert oracle.median_of_c(vals) == m["median"]
    assert switched > 0
    with pytest.raises(ValueError):
        oracle.median_of_c([1, 2])
    with pytest.raises(ValueError):
        oracle.sort_values_c([])


def test_threads_do_not_change_results():
    """row bands are bit-identical to one band (here: real pthreads)."""
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (3, 57, 43), dtype=np.uint8)
    a, sa = oracle.run_filter_c(img, 5, "fnr", 2, threads=1)
    b, sb = oracle.run_filter_c(img, 5, "fnr", 2, threads=7)
    assert np.array_equal(a, b) and sa.counters() == sb.counters()


def test_oracles_agree_on_random_inputs():
    rng = np.random.default_rng(11)
    for dtype, hi in ((np.uint8, 256), (np.uint16, 16384), (np.uint16, 65536)):
        for k in (3, 5, 7, 9, 11):
            img = rng.integers(0, hi, (2, 23, 29)).astype(dtype)
            img[:, 5:9, 3:12] = img[0, 0, 0]  # flat patch: ties and flat windows
            for method in ("fnr", "mf"):
                a, sa = oracle.run_filter_c(img, k, method, 1)
                b, sb = oracle.run_filter_np(img, k, method, 1)
                assert np.array_equal(a, b)
                assert sa.counters() == sb.counters()


def test_filter_rows_matches_full_pass():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 16384, (40, 37)).astype(np.uint16)
    full, st = oracle.run_filter_c(img, 7, "fnr", 1)
    rows, (det, rep) = oracle.filter_rows_c(img, 7, 9, 30)
    assert np.array_equal(rows, full[9:30])
