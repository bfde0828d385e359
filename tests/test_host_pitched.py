"""Host-buffer path (irdn_run_filter_*) with rows that are not a multiple of 16 bytes.

The reference's own image is 364 pixels wide. The TMA kernels need
16-byte aligned rows, so the host path pads device rows to a 16-byte pitch with 2-D
copies and strips the padding on the way back (irdn_api.cu run_host); the result must be
the oracle's for every chunking mode (frame chunks, row strips of one large frame),
pageable and pinned buffers, FNR and MF, passes 1 and 2.
"""

import os

import numpy as np
import pytest

import paper_1201_3972_b200 as P
from oracle import oracle

pytestmark = pytest.mark.gpu


def _img(rng, shape, dtype, density=0.3):
    hi = 255 if dtype == np.uint8 else 16383
    a = (np.cumsum(rng.integers(0, 3, size=shape), axis=-1) % (hi + 1)).astype(dtype)
    m = rng.random(shape) < density
    a[m] = np.where(rng.random(int(m.sum())) < 0.5, 0, hi).astype(dtype)
    return a


def _check(img, k, method, passes):
    got, st = P.run_filter(img, P.WindowSpec(k), method, passes)
    want, wst = oracle.run_filter_c(img, k, method, passes, threads=os.cpu_count() or 1)
    assert np.array_equal(got, want), (img.shape, img.dtype, k, method, passes)
    assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == list(wst.counters())


@pytest.mark.parametrize("shape,dtype", [((6, 244, 364), np.uint8), ((3, 61, 100), np.uint16),
                                          ((40, 33, 372), np.uint8), ((2, 50, 17), np.uint16)])
@pytest.mark.parametrize("k", [3, 5, 7, 11])
def test_unaligned_rows_through_the_host_path(cuda_ok, shape, dtype, k):
    rng = np.random.default_rng(k + shape[2])
    img = _img(rng, shape, dtype)
    _check(img, k, "fnr", 1)
    _check(img, k, "mf", 1)
    _check(img, k, "fnr", 2)


def test_reference_sized_gray_image(cuda_ok):
    """The paper's 364 x 244 8-bit frame as a GrayImage (pageable bytes)."""
    rng = np.random.default_rng(364)
    a = _img(rng, (244, 364), np.uint8, 0.2)
    img = P.GrayImage(364, 244, bytearray(a.tobytes()))
    for k, method, passes in [(3, "fnr", 1), (3, "fnr", 2), (5, "mf", 1), (7, "fnr", 1)]:
        got, st = P.run_filter(img, P.WindowSpec(k), method, passes)
        want, wst = oracle.run_filter_c(a, k, method, passes, threads=os.cpu_count() or 1)
        assert bytes(got.pixels) == want.tobytes()
        assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == list(wst.counters())


def test_large_unaligned_frame_in_row_strips(cuda_ok):
    """One frame > 16 MB with 16-byte-unaligned rows: the host path streams it in row
    strips (row mode), each strip's device rows padded to the pitch."""
    rng = np.random.default_rng(4100)
    img = _img(rng, (4400, 4004), np.uint8, 0.1)
    _check(img, 3, "fnr", 1)
    img16 = _img(rng, (2100, 4003), np.uint16, 0.1)
    _check(img16, 5, "fnr", 1)
