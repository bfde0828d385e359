"""Out-of-bounds write guards for every filter kernel (GPU).

compute-sanitizer is not available on the GPU pool (runs under it left GPUs needing a
reset, so the pool closed it), so the memory-safety evidence for the kernels is our own:
every kernel family writes into an output that sits between guard bands and has a row
pitch wider than the frame, and the guard bytes and the pitch gaps must come back
untouched while the frame equals the oracle. Inputs are cut from the end of their
allocation (the last input byte is the last byte of the tensor), and row strips get
exactly the rows the strip contract requires (fnr_large read past the strip).
"""

import os

import numpy as np
import pytest

import paper_1201_3972_b200 as P  # noqa: F401
from oracle import oracle
from paper_1201_3972_b200 import _native

pytestmark = pytest.mark.gpu

GUARD = 4096
PAT = 0xA5


def _frames(rng, b, h, w, dtype, density):
    hi = 255 if dtype == np.uint8 else 16383
    img = (np.cumsum(rng.integers(0, 3, size=(b, h, w)), axis=2) % (hi + 1)).astype(dtype)
    m = rng.random(img.shape) < density
    img[m] = rng.integers(0, hi + 1, size=int(m.sum())).astype(dtype)
    return img


CASES = [
    # (dtype, batch, height, width, k, method): one per kernel family and layout class
    (np.uint8, 3, 70, 144, 3, "fnr"),    # dense 3x3, partial row / column tiles
    (np.uint8, 2, 64, 256, 3, "mf"),
    (np.uint16, 3, 72, 96, 5, "fnr"),    # warp kernel
    (np.uint8, 2, 70, 80, 7, "fnr"),
    (np.uint16, 1, 50, 112, 11, "fnr"),
    (np.uint16, 2, 40, 64, 9, "mf"),
    (np.uint16, 2, 40, 160, 13, "fnr"),  # tiled large-window kernel
    (np.uint8, 1, 33, 364, 3, "fnr"),    # unaligned rows -> tiled kernel
    (np.uint8, 1, 20, 364, 15, "mf"),
]


@pytest.mark.parametrize("dtype,b,h,w,k,method", CASES)
def test_pass_writes_stay_inside_the_frame(dtype, b, h, w, k, method, cuda_ok):
    import torch

    rng = np.random.default_rng(k * 1000 + w)
    img = _frames(rng, b, h, w, dtype, 0.3)
    want, _ = oracle.run_filter_c(img, k, method, 1, threads=os.cpu_count() or 1)
    tdt = torch.uint8 if dtype == np.uint8 else torch.int16
    s = np.dtype(dtype).itemsize
    # input: contiguous, ending exactly at the end of its allocation
    d_in = torch.from_numpy(img.view(np.uint8 if s == 1 else np.int16).reshape(-1).copy()).cuda()
    # output: pitch = width + 32 elements (16-byte multiple), guard bands on both sides
    pitch = w + 32
    n_out = b * h * pitch
    raw = torch.full((2 * GUARD + n_out * s,), PAT, dtype=torch.uint8, device="cuda")
    out = raw[GUARD:GUARD + n_out * s].view(tdt)
    counts = torch.zeros(2, dtype=torch.int64, device="cuda")
    lib = _native.load_lib()
    fn = lib.irdn_filter_pass_u8 if s == 1 else lib.irdn_filter_pass_u16
    _native.check(fn(d_in.data_ptr(), out.data_ptr(), b, h, w, w, pitch, k, _native.METHODS[method],
                     counts.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    host = raw.cpu().numpy()
    assert (host[:GUARD] == PAT).all() and (host[GUARD + n_out * s:] == PAT).all(), "guard band written"
    frame = host[GUARD:GUARD + n_out * s].view(dtype).reshape(b, h, pitch)
    gap = frame[:, :, w:].view(np.uint8)
    assert (gap == PAT).all(), "pitch gap written"
    assert np.array_equal(frame[:, :, :w], want)


def test_strip_with_exact_input_rows_and_unaligned_width(cuda_ok):
    """k = 13 on 364-pixel rows, each strip's input holding exactly [need0, need1)."""
    import torch

    from paper_1201_3972_b200 import sharding

    rng = np.random.default_rng(13)
    h, w, k = 53, 364, 13
    img = _frames(rng, 1, h, w, np.uint16, 0.4)[0]
    want, _ = oracle.run_filter_c(img[None], k, "fnr", 1, threads=os.cpu_count() or 1)
    parts = []
    for world in (2, 3, 5):
        parts = []
        for sh in sharding.shard_plan(1, h, world, k, 1):
            src = torch.from_numpy(img[sh.in0:sh.in1].view(np.int16).copy()).cuda()
            out, _ = sharding.run_shard_device(src, sh, h, k, "fnr", 1)
            parts.append(out.cpu().numpy().view(np.uint16))
        assert np.array_equal(np.concatenate(parts), want[0]), world
