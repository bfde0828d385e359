"""GPU parity: the sm_100a kernels (through the C ABI) against the reference goldens and the oracle.

Bar: bit-exact pixels and identical FilterStats integer counters.
"""

import ctypes
import os

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle

import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native
from paper_1201_3972_b200.scene import CONFIGS, generate

pytestmark = pytest.mark.gpu

GOLDEN_SETS = ["ref_u8.npz", "ref_u16.npz", "ref_fixtures.npz", "ref_configs.npz"]
NT = max(1, min(32, os.cpu_count() or 1))


def counters(st):
    return [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes]


def gpu_filter(img, k, method="fnr", passes=1):
    out, st = P.run_filter(img, P.WindowSpec(k), method, passes)
    return out, counters(st)


class force_generic:
    def __enter__(self):
        self.prev = _native.load_lib().irdn_set_force_generic(1)

    def __exit__(self, *a):
        _native.load_lib().irdn_set_force_generic(self.prev)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("name", GOLDEN_SETS)
def test_gpu_matches_reference_golden(cuda_ok, name, generic):
    import contextlib

    ctx = force_generic() if generic else contextlib.nullcontext()
    with ctx:
        for meta, inp, out in load_golden(name):
            if inp.dtype == np.uint8:
                h, w = inp.shape
                g, st = gpu_filter(P.GrayImage(w, h, inp.tobytes()), meta["k"], meta["method"], meta["passes"])
                got = np.frombuffer(bytes(g.pixels), np.uint8).reshape(h, w)
            else:
                got, st = gpu_filter(inp, meta["k"], meta["method"], meta["passes"])
            assert np.array_equal(got, out), (name, meta)
            assert st == meta["stats"], (name, meta, st)


def test_torch_device_path_matches_golden(cuda_ok):
    import torch

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for meta, inp, out in load_golden("ref_configs.npz") + load_golden("ref_u16.npz")[:40]:
            t = torch.from_numpy(inp).cuda()
            got, st = P.run_filter(t, P.WindowSpec(meta["k"]), meta["method"], meta["passes"])
            assert got.is_cuda and got.dtype == t.dtype
            assert np.array_equal(as_i32(got).cpu().numpy().astype(out.dtype), out), meta
            assert counters(st) == meta["stats"], meta


def _oracle(img, k, method="fnr", passes=1):
    out, st = oracle.run_filter_c(img, k, method, passes, threads=NT)
    return out, list(st.counters())


@pytest.mark.parametrize("cfg_name,frames", [("c1", 1), ("c2", 4), ("c3", 1), ("c5", 6)])
def test_config_frames_vs_oracle(cuda_ok, cfg_name, frames):
    cfg = CONFIGS[cfg_name]
    img = generate(cfg, frame0=3 if cfg.frames > 1 else 0, nframes=frames)
    for method, passes in (("fnr", 1), ("fnr", 2), ("mf", 1)):
        want, wst = _oracle(img, cfg.k, method, passes)
        got, gst = gpu_filter(img, cfg.k, method, passes)
        assert np.array_equal(got, want), (cfg_name, method, passes)
        assert gst == wst
        with force_generic():
            got2, gst2 = gpu_filter(img, cfg.k, method, passes)
        assert np.array_equal(got2, want) and gst2 == wst


def test_config4_crop_vs_oracle(cuda_ok):
    cfg = CONFIGS["c4"].with_shape(height=1536, width=1280)
    img = generate(cfg, nframes=1)[0]
    want, wst = _oracle(img, 11, "fnr", 1)
    got, gst = gpu_filter(img, 11, "fnr", 1)
    assert np.array_equal(got, want) and gst == wst


def as_i32(t):
    import torch

    if t.dtype == torch.uint16:
        return t.view(torch.int16).to(torch.int32) & 0xFFFF
    return t.to(torch.int32)


def _torch_minmax_mask(t, k):
    """Independent detector: replicate-pad + max_pool (exact for <= 24-bit integers in fp32)."""
    import torch
    import torch.nn.functional as F

    r = k // 2
    x = as_i32(t).float().unsqueeze(1)
    xp = F.pad(x, (r, r, r, r), mode="replicate")
    mx = F.max_pool2d(xp, k, stride=1)
    mn = -F.max_pool2d(-xp, k, stride=1)
    return ((x == mx) | (x == mn)).squeeze(1)


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size_config_properties(cuda_ok, cfg_name):
    """BASELINE full sizes: detector exactness, signal preservation, sampled-row oracle parity."""
    import torch

    cfg = CONFIGS[cfg_name]
    nframes = min(cfg.frames, 512)  # c5: 512 of 4096 frames per call keeps host RAM modest
    img = generate(cfg, nframes=nframes)
    t = torch.from_numpy(img).cuda()
    out, st = P.run_filter(t, P.WindowSpec(cfg.k), "fnr", 1)
    mask = torch.zeros_like(t, dtype=torch.bool)
    for b0 in range(0, nframes, 16):
        mask[b0:b0 + 16] = _torch_minmax_mask(t[b0:b0 + 16], cfg.k)
    assert st.detected == int(mask.sum()) == st.sorts
    assert st.minmax_scans == img.size
    o32, t32 = as_i32(out), as_i32(t)
    assert torch.equal(o32[~mask], t32[~mask])
    assert st.replacements == int((o32 != t32).sum())
    # sampled rows against the oracle (clamped against the full frame)
    rng = np.random.default_rng(7)
    o = o32.cpu().numpy().astype(img.dtype)
    for _ in range(6):
        f = int(rng.integers(0, nframes))
        y0 = int(rng.integers(0, cfg.height - 4))
        y1 = min(cfg.height, y0 + (2 if cfg.k == 11 else 4))
        rows, _ = oracle.filter_rows_c(img[f], cfg.k, y0, y1)
        assert np.array_equal(o[f, y0:y1], rows), (cfg_name, f, y0)
    for y0 in (0, cfg.height - 2):  # image borders
        rows, _ = oracle.filter_rows_c(img[0], cfg.k, y0, y0 + 2)
        assert np.array_equal(o[0, y0:y0 + 2], rows)


def _strip_call(t_in, k, row_begin, row_end, method=0):
    import torch

    lib = _native.load_lib()
    h, w = t_in.shape
    r = k // 2
    in0, in1 = max(0, row_begin - r), min(h, row_end + r)
    src = t_in[in0:in1].contiguous()
    out = torch.empty((row_end - row_begin, w), dtype=t_in.dtype, device=t_in.device)
    counts = torch.zeros(2, dtype=torch.int64, device=t_in.device)
    fn = lib.irdn_filter_strip_u8 if t_in.dtype == torch.uint8 else lib.irdn_filter_strip_u16
    _native.check(fn(src.data_ptr(), in0, in1 - in0, out.data_ptr(), row_begin, row_end, h, w, w, w,
                     k, method, counts.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return out, counts.cpu().tolist()


@pytest.mark.parametrize("k,dtype", [(11, np.uint16), (3, np.uint8), (7, np.uint8), (5, np.uint16)])
def test_row_strips_equal_whole_frame(cuda_ok, k, dtype):
    """output bytes and counters identical for every strip seam placement."""
    import torch

    cfg = CONFIGS["c4" if dtype == np.uint16 else "c3"].with_shape(height=517, width=640)
    img = generate(cfg, nframes=1)[0]
    t = torch.from_numpy(img).cuda()
    whole, st = P.run_filter(t, P.WindowSpec(k), "fnr", 1)
    for seams in ([0, 517], [0, 258, 517], [0, 1, 5, 6, 200, 511, 517], [0, 129, 258, 387, 517]):
        parts, det, rep = [], 0, 0
        for a, b in zip(seams[:-1], seams[1:]):
            o, (d, r) = _strip_call(t, k, a, b)
            parts.append(o)
            det += d
            rep += r
        assert torch.equal(as_i32(torch.cat(parts)), as_i32(whole)), seams
        assert (det, rep) == (st.detected, st.replacements)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_edge_shapes_and_windows(cuda_ok, dtype):
    rng = np.random.default_rng(17)
    hi = 256 if dtype == np.uint8 else 65536
    shapes = [(1, 1), (1, 17), (17, 1), (2, 3), (3, 2), (4, 5), (7, 300), (300, 7), (33, 129),
              (64, 64), (65, 257)]
    for (h, w) in shapes:
        for k in (3, 5, 7, 11, 13, 31):
            img = rng.integers(0, hi, (2, h, w)).astype(dtype)
            for method in ("fnr", "mf"):
                want, wst = _oracle(img, k, method, 1)
                got, gst = gpu_filter(img, k, method, 1)
                assert np.array_equal(got, want), (h, w, k, method)
                assert gst == wst


def test_flat_and_extreme_images(cuda_ok):
    for dtype, mx in ((np.uint8, 255), (np.uint16, 65535)):
        for fill in (0, 1, mx):
            img = np.full((3, 70, 130), fill, dtype)
            for k in (3, 5, 7, 11):
                got, st = gpu_filter(img, k, "fnr", 1)
                assert np.array_equal(got, img)
                assert st[3] == img.size and st[2] == 0  # flat windows: detected, never replaced
        img = np.full((2, 40, 40), 7, dtype)
        img[:, 20, 20] = mx
        for k in (3, 5, 7, 11):
            got, st = gpu_filter(img, k, "fnr", 1)
            assert np.all(got == 7) and st[2] == 2


def test_large_batch_host_pipeline(cuda_ok):
    cfg = CONFIGS["c2"]
    img = generate(cfg, frame0=10, nframes=48)
    want, wst = _oracle(img, 5, "fnr", 1)
    got, gst = gpu_filter(img, 5, "fnr", 1)
    assert np.array_equal(got, want) and gst == wst


def test_single_frame_row_pipeline(cuda_ok):
    """batch=1, passes=1, >=16 MB frame: the host path pipelines row strips."""
    cfg = CONFIGS["c4"].with_shape(height=4096, width=4096)
    img = generate(cfg, nframes=1)[0]
    got, gst = gpu_filter(img, 11, "fnr", 1)
    import torch

    t = torch.from_numpy(img).cuda()
    dev, dst = P.run_filter(t, P.WindowSpec(11), "fnr", 1)
    assert np.array_equal(got, as_i32(dev).cpu().numpy().astype(np.uint16))
    assert gst == counters(dst)
    rows, _ = oracle.filter_rows_c(img, 11, 1020, 1030)
    assert np.array_equal(got[1020:1030], rows)


@pytest.mark.parametrize("dtype,k", [(np.uint16, 5), (np.uint8, 7), (np.uint16, 11)])
def test_heavy_tiles(cuda_ok, dtype, k):
    """Warp tiles with many more noisy pixels than usual (patches, a whole frame, a
    batch where nearly every pixel is flagged: several queue rounds per tile) match the
    oracle bit for bit, whole frames and row strips (input rows offset from the frame)."""
    import torch

    rng = np.random.default_rng(7)
    smooth = CONFIGS["c2"].with_shape(height=200, width=330)
    img = generate(smooth, nframes=12).astype(dtype)
    img[3:9, 40:140, 64:200] = rng.integers(0, 3, size=(6, 100, 136)).astype(dtype)  # heavy patches
    img[10] = rng.integers(0, 2, size=img[10].shape).astype(dtype)  # a whole heavy frame
    want, wst = _oracle(img, k, "fnr", 1)
    got, gst = gpu_filter(img, k, "fnr", 1)
    assert np.array_equal(got, want) and gst == wst
    heavy = rng.integers(0, 4, size=(48, 256, 320)).astype(dtype)  # ~all flagged
    want, wst = _oracle(heavy, k, "fnr", 1)
    got, gst = gpu_filter(heavy, k, "fnr", 1)
    assert np.array_equal(got, want) and gst == wst
    t = torch.from_numpy(img[10]).cuda()
    whole, st = P.run_filter(t, P.WindowSpec(k), "fnr", 1)
    parts, det = [], 0
    for a, b in ((0, 37), (37, 120), (120, 200)):
        o, (d, _) = _strip_call(t, k, a, b)
        parts.append(o)
        det += d
    assert torch.equal(as_i32(torch.cat(parts)), as_i32(whole)) and det == st.detected
    assert np.array_equal(as_i32(whole).cpu().numpy().astype(dtype), _oracle(img[10], k)[0])


def test_concurrent_calls_from_threads_and_streams(cuda_ok):
    """The C ABI is reentrant: host-buffer calls from several threads (per-device workspace
    lock) and device calls on separate streams (one scheduler slot per launch) in flight
    together give the single-call results."""
    import threading

    import torch

    cfg = CONFIGS["c2"].with_shape(height=256, width=320)
    imgs = [generate(cfg, frame0=4 * i, nframes=4) for i in range(6)]
    want = [_oracle(im, 5, "fnr", 2) for im in imgs]
    got = [None] * len(imgs)
    errs = []

    def host_worker(i):
        try:
            got[i] = gpu_filter(imgs[i], 5, "fnr", 2)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    def device_worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                t = torch.from_numpy(imgs[i].view(np.int16)).cuda(non_blocking=False).view(torch.uint16)
                out, st = P.run_filter(t, P.WindowSpec(5), "fnr", 2)
                s.synchronize()
                got[i] = (as_i32(out).cpu().numpy().astype(np.uint16), counters(st))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    threads = [threading.Thread(target=host_worker if i % 2 == 0 else device_worker, args=(i,))
               for i in range(len(imgs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for (w, wst), (g, gst) in zip(want, got):
        assert np.array_equal(g, w) and gst == wst


@pytest.mark.parametrize("in_pinned,out_pinned", [(False, False), (True, False), (False, True), (True, True)])
def test_host_entry_pinned_and_pageable_buffers(cuda_ok, in_pinned, out_pinned):
    """irdn_run_filter_*: pinned caller buffers are DMA'd directly, pageable ones go through
    the pinned staging slots (parallel CPU copies) — every combination, batch chunking and
    single-frame row strips, gives the device-path result."""
    import torch

    lib = _native.load_lib()

    def buf(a, pinned):
        if not pinned:
            return np.ascontiguousarray(a), None
        t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
        v = t.numpy().view(a.dtype).reshape(a.shape)
        v[...] = a
        return v, t

    cases = [(generate(CONFIGS["c2"].with_shape(height=256, width=320), nframes=40), 5),  # 6.5 MB chunks
             (generate(CONFIGS["c4"].with_shape(height=3072, width=3072), nframes=1)[0], 11)]  # 18 MB: strips
    for img, k in cases:
        want, wst = _oracle(img, k, "fnr", 1)
        src, keep_in = buf(img, in_pinned)
        out, keep_out = buf(np.zeros_like(img), out_pinned)
        st = _native.IrdnStats()
        b, h, w = (1,) + img.shape if img.ndim == 2 else img.shape
        _native.check(lib.irdn_run_filter_u16(src.ctypes.data, out.ctypes.data, b, h, w, k, 0, 1, 0, ctypes.byref(st)))
        assert np.array_equal(out, want), (img.shape, in_pinned, out_pinned)
        assert counters(st) == wst


def test_randomized_shapes_windows_methods(cuda_ok):
    """Seeded fuzz: random batch / shape / window / dtype / method / passes / value
    distribution (incl. low-entropy images with many ties), GPU vs oracle, bit-exact pixels
    and counters. Shapes straddle the tile sizes (64x32 warp tiles, 64x48 for k = 11, 128-wide 3x3 tiles,
    16-byte alignment of rows) so partial tiles, generic fallbacks and edge fix-ups all run."""
    rng = np.random.default_rng(20261020)
    for case in range(60):
        dtype = np.uint8 if rng.random() < 0.5 else np.uint16
        k = int(rng.choice([3, 5, 7, 9, 11, 13]))
        b = int(rng.integers(1, 4))
        h = int(rng.integers(1, 150))
        w = int(rng.choice([int(rng.integers(1, 40)), int(rng.integers(40, 300)), 64, 128, 256]))
        hi = int(rng.choice([2, 4, 256, 65536 if dtype == np.uint16 else 256]))
        img = rng.integers(0, hi, size=(b, h, w)).astype(dtype)
        if rng.random() < 0.3:  # smooth field + impulses
            yy, xx = np.mgrid[0:h, 0:w]
            base = (yy * 3 + xx * 2) % (250 if dtype == np.uint8 else 16000)
            img = np.broadcast_to(base, (b, h, w)).astype(dtype).copy()
            m = rng.random(img.shape) < 0.3
            img[m] = rng.integers(0, 256 if dtype == np.uint8 else 65536, int(m.sum())).astype(dtype)
        method = "mf" if rng.random() < 0.25 else "fnr"
        passes = int(rng.choice([1, 1, 2, 3]))
        want, wst = _oracle(img, k, method, passes)
        got, gst = gpu_filter(img, k, method, passes)
        assert np.array_equal(got, want), (case, dtype, k, img.shape, method, passes)
        assert gst == wst, (case, gst, wst)


def test_tall_tiles_11x11(cuda_ok):
    """k = 11 runs 64 x 48 warp tiles (fnr_warp.cuh WHK): heights on both sides of one, two
    and three tile rows, whole and partial tile columns, sparse impulses (one queue round per
    tile) and dense ones (several rounds), FNR / MF, passes 1-2, u8 / u16."""
    rng = np.random.default_rng(1148)
    for case, (h, w) in enumerate([(48, 64), (47, 128), (49, 70), (96, 64), (97, 200), (95, 192), (144, 64),
                                   (150, 130), (24, 64), (1, 64), (11, 300)]):
        dtype = np.uint16 if case % 2 == 0 else np.uint8
        top = 16384 if dtype == np.uint16 else 256
        yy, xx = np.mgrid[0:h, 0:w]
        img = ((yy * 5 + xx * 3) % (top - 7)).astype(dtype)[None].repeat(2, axis=0).copy()
        m = rng.random(img.shape) < (0.02 if case % 3 else 0.35)
        img[m] = rng.integers(0, top, int(m.sum())).astype(dtype)
        for method, passes in (("fnr", 1), ("fnr", 2), ("mf", 1)):
            if method == "mf" and h * w > 64 * 64:
                continue  # the 121-input network on every pixel: keep the case small
            want, wst = _oracle(img, 11, method, passes)
            got, gst = gpu_filter(img, 11, method, passes)
            assert np.array_equal(got, want), (h, w, dtype, method, passes)
            assert gst == wst, (h, w, method, passes, gst, wst)


def test_fnr_pass_mf_pass_accumulate_like_the_reference(cuda_ok):
    """fnr_pass / mf_pass (filters.py:69-76): one pass each, counters (passes included)
    added to the caller's FilterStats, elapsed_ms untouched; two chained fnr_pass calls
    equal run_filter(passes=2) pixel for pixel and counter for counter."""
    for meta, inp, out in load_golden("ref_fixtures.npz")[:6]:
        h, w = inp.shape
        img = P.GrayImage(w, h, inp.tobytes())
        st = P.FilterStats(elapsed_ms=12.5)
        step = P.fnr_pass if meta["method"] == "fnr" else P.mf_pass
        cur = img
        for _ in range(meta["passes"]):
            cur = step(cur, P.WindowSpec(meta["k"]), st)
        assert bytes(cur.pixels) == out.tobytes(), meta
        assert counters(st) == meta["stats"] and st.elapsed_ms == 12.5, (meta, st)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_large_windows_and_unaligned_layouts(cuda_ok, dtype):
    """k >= 13 and layouts the TMA kernels cannot take (pitch not a multiple of 16 bytes)
    run the shared-memory tiled kernel (csrc/fnr_large.cuh); bit-exact vs the oracle, also
    against the generic kernel."""
    rng = np.random.default_rng(1313 + np.dtype(dtype).itemsize)
    hi = 256 if dtype == np.uint8 else 16384
    cases = [(13, 2, 70, 100), (15, 1, 40, 200), (21, 1, 64, 64), (31, 2, 33, 47), (63, 1, 90, 130),
             (3, 2, 244, 364), (5, 1, 51, 77), (11, 1, 37, 131), (13, 1, 5, 3), (17, 1, 1, 1),
             (65, 1, 70, 90), (101, 1, 20, 150)]  # k > 63: the generic kernel
    for k, b, h, w in cases:
        yy, xx = np.mgrid[0:h, 0:w]
        img = np.broadcast_to((yy * 5 + xx * 3) % hi, (b, h, w)).astype(dtype).copy()
        m = rng.random(img.shape) < 0.25
        img[m] = rng.integers(0, hi, int(m.sum())).astype(dtype)
        for method in ("fnr", "mf"):
            want, wst = _oracle(img, k, method, 1)
            got, gst = gpu_filter(img, k, method, 1)
            assert np.array_equal(got, want), (k, img.shape, method)
            assert gst == wst
            with force_generic():
                got2, gst2 = gpu_filter(img, k, method, 1)
            assert np.array_equal(got2, want) and gst2 == wst


def test_large_window_row_strips(cuda_ok):
    import torch

    img = generate(CONFIGS["c4"].with_shape(height=300, width=200), nframes=1)[0]
    t = torch.from_numpy(img.view(np.int16)).cuda()
    for k in (13, 21):
        want, _ = _oracle(img, k, "fnr", 1)
        parts = []
        for a, b in ((0, 97), (97, 98), (98, 300)):
            parts.append(_strip_call(t, k, a, b)[0])
        got = torch.cat(parts, 0).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, want), k
