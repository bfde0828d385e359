"""Multi-pass run_filter in one persistent launch (fnr_warp_mp_kernel).

passes >= 2 runs all passes in one launch of the warp kernel: a tile of pass q waits for
the pass-(q-1) tiles under its box (epoch-tagged flags). These tests check it bit-exactly
against the oracle (filters.py:96-100 semantics: each pass reads the previous output) and
against separate single-pass launches, across dtypes, windows, pass counts, tile-pool
sizes (fewer tiles than warps .. many waves), repeated back-to-back launches on one
stream, and CUDA-graph replays (frozen kernel parameters: the epoch must come from the
device).
"""

import ctypes
import os

import numpy as np
import pytest

from oracle import oracle

import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate

pytestmark = pytest.mark.gpu
NT = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(autouse=True)
def multipass_on():
    """The multi-pass launch is opt-in (irdn_set_multipass); these tests turn it on."""
    lib = _native.load_lib()
    prev = lib.irdn_set_multipass(1)
    yield
    lib.irdn_set_multipass(prev)


def _oracle(img, k, method, passes):
    out, st = oracle.run_filter_c(img, k, method, passes, threads=NT)
    return out, list(st.counters())


def _dev(img):
    import torch

    t = torch.from_numpy(img.view(np.int16) if img.dtype == np.uint16 else img).cuda()
    return t


def _host(t, dtype):
    a = t.cpu().numpy()
    return a.view(np.uint16) if dtype == np.uint16 else a


def _run_device(lib, t_in, dtype, k, method, passes, stream=None):
    import torch

    B, H, W = t_in.shape
    out = torch.empty_like(t_in)
    tmp = torch.empty_like(t_in)
    counts = torch.zeros(2, dtype=torch.int64, device=t_in.device)
    fn = lib.irdn_run_filter_device_u8 if dtype == np.uint8 else lib.irdn_run_filter_device_u16
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _native.check(fn(t_in.data_ptr(), out.data_ptr(), tmp.data_ptr(), B, H, W, k, method, passes,
                     counts.data_ptr(), s))
    return out, counts


CASES = [
    # dtype, k, batch, height, width
    (np.uint16, 5, 3, 100, 200),
    (np.uint16, 3, 2, 64, 128),
    (np.uint16, 11, 1, 300, 257),
    (np.uint16, 7, 5, 33, 65),
    (np.uint8, 5, 4, 96, 160),
    (np.uint8, 7, 2, 130, 300),
    (np.uint8, 9, 1, 77, 96),
    (np.uint8, 11, 3, 64, 64),
]


@pytest.mark.parametrize("dtype,k,b,h,w", CASES)
def test_multipass_matches_oracle(cuda_ok, dtype, k, b, h, w):
    rng = np.random.default_rng(k * 1000 + h)
    hi = 256 if dtype == np.uint8 else 16384
    # smooth field + 30 % uniform impulses
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.broadcast_to((yy * 2 + xx * 3) % hi, (b, h, w)).astype(dtype).copy()
    m = rng.random(img.shape) < 0.3
    img[m] = rng.integers(0, hi, int(m.sum())).astype(dtype)
    for method in ("fnr", "mf"):
        for passes in (2, 3, 4):
            want, wst = _oracle(img, k, method, passes)
            out, st = P.run_filter(img, P.WindowSpec(k), method, passes)
            assert np.array_equal(out, want), (dtype, k, img.shape, method, passes)
            assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == wst


def test_multipass_equals_separate_passes_full_c2(cuda_ok):
    """The c2 batch (64 frames): one multi-pass launch == two single-pass launches, repeated
    back to back on one stream (flags are reused with a new epoch every launch)."""
    import torch

    lib = _native.load_lib()
    cfg = CONFIGS["c2"]
    img = generate(cfg)
    t = _dev(img)
    B, H, W = img.shape
    mid = torch.empty_like(t)
    ref = torch.empty_like(t)
    c_ref = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.irdn_set_multipass(1) == 1
    _native.check(lib.irdn_filter_pass_u16(t.data_ptr(), mid.data_ptr(), B, H, W, W, W, 5, 0, c_ref.data_ptr(), s))
    _native.check(lib.irdn_filter_pass_u16(mid.data_ptr(), ref.data_ptr(), B, H, W, W, W, 5, 0, c_ref.data_ptr(), s))
    outs = [_run_device(lib, t, np.uint16, 5, 0, 2) for _ in range(6)]
    for out, counts in outs:
        assert torch.equal(out, ref)
        assert torch.equal(counts, c_ref)
    want, wst = _oracle(img[:4], 5, "fnr", 2)
    assert np.array_equal(_host(ref[:4], np.uint16), want)


def test_multipass_graph_replay(cuda_ok):
    """Captured once, replayed with new input contents: the epoch is read on the device, so
    frozen kernel parameters do not let a replay see the previous replay's flags."""
    import torch

    lib = _native.load_lib()
    cfg = CONFIGS["c2"]
    imgs = [generate(cfg, frame0=8 * i, nframes=8) for i in range(3)]
    t_in = _dev(imgs[0])
    B, H, W = t_in.shape
    out = torch.empty_like(t_in)
    tmp = torch.empty_like(t_in)
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    stream = torch.cuda.Stream()

    def launch():
        _native.check(lib.irdn_run_filter_device_u16(t_in.data_ptr(), out.data_ptr(), tmp.data_ptr(), B, H, W, 5,
                                                     0, 2, counts.data_ptr(), stream.cuda_stream))

    with torch.cuda.stream(stream):
        launch()  # warm-up outside the capture (allocates the stream's flag buffer)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        launch()
    for img in imgs + imgs[:1]:
        t_in.copy_(_dev(img))
        counts.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        want, wst = _oracle(img, 5, "fnr", 2)
        assert np.array_equal(_host(out, np.uint16), want)
        assert int(counts[0]) == wst[3] and int(counts[1]) == wst[2]


def test_multipass_two_streams_concurrently(cuda_ok):
    """Two streams each run multi-pass launches at the same time (separate flag buffers)."""
    import torch

    lib = _native.load_lib()
    cfg = CONFIGS["c2"]
    a = generate(cfg, frame0=0, nframes=16)
    b = generate(cfg, frame0=16, nframes=16)
    ta, tb = _dev(a), _dev(b)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    res = []
    for _ in range(3):
        oa, _ = _run_device(lib, ta, np.uint16, 5, 0, 3, stream=sa.cuda_stream)
        ob, _ = _run_device(lib, tb, np.uint16, 5, 0, 3, stream=sb.cuda_stream)
        res.append((oa, ob))
    torch.cuda.synchronize()
    wa, _ = _oracle(a, 5, "fnr", 3)
    wb, _ = _oracle(b, 5, "fnr", 3)
    for oa, ob in res:
        assert np.array_equal(_host(oa, np.uint16), wa)
        assert np.array_equal(_host(ob, np.uint16), wb)


def test_multipass_single_launch(cuda_ok):
    lib = _native.load_lib()
    img = generate(CONFIGS["c2"], nframes=4)
    t = _dev(img)
    lib.irdn_reset_launch_count()
    _run_device(lib, t, np.uint16, 5, 0, 3)
    assert lib.irdn_launch_count() == 1
    lib.irdn_set_multipass(0)
    lib.irdn_reset_launch_count()
    out0, c0 = _run_device(lib, t, np.uint16, 5, 0, 3)
    assert lib.irdn_launch_count() == 3  # default: one launch per pass
    lib.irdn_set_multipass(1)
    out1, c1 = _run_device(lib, t, np.uint16, 5, 0, 3)
    assert torch_equal(out0, out1) and torch_equal(c0, c1)


def torch_equal(a, b):
    import torch

    return bool(torch.equal(a, b))
