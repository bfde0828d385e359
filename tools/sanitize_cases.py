"""Small instances of every kernel in libirdn.so, for compute-sanitizer.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Each case goes through the product's public API (Python run_filter / the C ABI) on
inputs just large enough to reach the kernel's interesting paths (partial tiles, frame
borders, several tiles per warp, the scheduler reset of the last CTA, a strip whose
input buffer ends exactly at its last row). Results are checked against the oracle, so
the run also fails if a tool changes timing enough to expose an ordering bug.
Run on the GPU box by tools/sanitize.sh; the summary goes to profiles/.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1201_3972_b200 as P  # noqa: E402
from oracle import oracle  # noqa: E402  (checker only)
from paper_1201_3972_b200 import _native  # noqa: E402

rng = np.random.default_rng(7)


def frames(b, h, w, dtype, density=0.3):
    hi = 255 if dtype == np.uint8 else 16383
    base = rng.integers(0, hi + 1, size=(b, h, w)).astype(dtype)
    smooth = np.cumsum(np.cumsum(base.astype(np.int64) % 3, axis=1), axis=2) % (hi + 1)
    img = smooth.astype(dtype)
    m = rng.random(img.shape) < density
    img[m] = np.where(rng.random(m.sum()) < 0.5, 0, hi).astype(dtype)
    return img


def check(img, k, method="fnr", passes=1):
    got, st = P.run_filter(img, P.WindowSpec(k), method, passes)
    want, wst = oracle.run_filter_c(img, k, method, passes, threads=os.cpu_count() or 1)
    assert np.array_equal(got, want), (img.shape, img.dtype, k, method, passes)
    assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == list(wst.counters())


def case_warp():
    check(frames(3, 72, 96, np.uint16), 5)                       # warp kernel, u16 5x5
    check(frames(2, 70, 80, np.uint8, 0.5), 7)                   # u8 7x7, partial tiles
    check(frames(1, 96, 128, np.uint16, 0.4), 11)                # u16 11x11
    check(frames(2, 40, 64, np.uint16), 3)                       # u16 3x3 (warp kernel)
    check(frames(2, 50, 64, np.uint16), 9, "mf")                 # MF 9x9
    check(frames(2, 64, 96, np.uint16), 5, "fnr", 2)             # two PDL-chained passes


def case_multipass():
    prev = _native.load_lib().irdn_set_multipass(1)
    try:
        check(frames(4, 64, 128, np.uint16), 5, "fnr", 3)
        check(frames(2, 48, 64, np.uint8), 7, "mf", 2)
    finally:
        _native.load_lib().irdn_set_multipass(prev)


def case_k3():
    check(frames(3, 130, 256, np.uint8, 0.1), 3)                 # dense 3x3, full + partial row tiles
    check(frames(2, 37, 144, np.uint8, 0.2), 3)                  # partial column tile
    check(frames(2, 37, 144, np.uint8, 0.2), 3, "mf", 2)


def case_large():
    check(frames(2, 40, 160, np.uint16), 13)                     # tiled large-window kernel
    check(frames(1, 33, 364, np.uint8), 3)                       # the reference's unaligned 364-px rows
    check(frames(1, 20, 364, np.uint8), 15, "mf")


def case_generic():
    lib = _native.load_lib()
    prev = lib.irdn_set_force_generic(1)
    try:
        check(frames(2, 24, 40, np.uint16), 5)
        check(frames(1, 21, 33, np.uint8), 7, "mf")
    finally:
        lib.irdn_set_force_generic(prev)


def case_strip():
    """A strip whose input buffer holds exactly the rows the contract requires (k=13,
    unaligned width): the ADVICE r01 read-past-the-strip case."""
    import torch

    from paper_1201_3972_b200 import sharding

    h, w, k = 53, 364, 13
    img = frames(1, h, w, np.uint16)[0]
    want, _ = oracle.run_filter_c(img[None], k, "fnr", 1, threads=os.cpu_count() or 1)
    parts = []
    for sh in sharding.shard_plan(1, h, 3, k, 1):
        src = torch.from_numpy(img[sh.in0:sh.in1].view(np.int16).copy()).cuda()  # exactly [in0, in1)
        out, _ = sharding.run_shard_device(src, sh, h, k, "fnr", 1)
        parts.append(out.cpu().numpy().view(np.uint16))
    assert np.array_equal(np.concatenate(parts), want[0])


def case_noise_metrics():
    clean = P.structured_image()
    noisy, mask = P.inject_impulse(clean, P.NoiseSpec(0.2, 0.5, 42))
    a = np.frombuffer(bytes(clean.pixels), np.uint8)
    want, wflags, wcnt = oracle.inject_impulse_c(a, 42, 0.2, 0.5)
    assert bytes(noisy.pixels) == want.tobytes() and mask.count == wcnt
    big = rng.integers(0, 256, size=300_000, dtype=np.uint8)
    n2, _ = P.inject_impulse(big, P.NoiseSpec(0.3, 0.5, 9))
    w2, _, _ = oracle.inject_impulse_c(big, 9, 0.3, 0.5)
    assert np.array_equal(np.asarray(n2), w2)
    assert P.mse(clean, noisy) == oracle.sq_err_sum_c(a, want) / a.size


def case_delta():
    prev = _native.set_host_return("delta")
    try:
        img = frames(5, 64, 128, np.uint16)
        check(img, 5)
        check(frames(3, 48, 64, np.uint8), 3)
    finally:
        _native.set_host_return(prev)


CASES = {n[5:]: f for n, f in globals().items() if n.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print(f"case {n} ok", flush=True)
