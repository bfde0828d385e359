"""Dense median stage of the warp kernel (csrc/fnr_dense.cuh, k = 5 / 7) against the oracle.

MF always takes the dense stage for k = 5 / 7; FNR takes it for tiles with many flagged
pixels (salt-and-pepper at 50 % flags about half the pixels, 5 % far fewer), so both FNR
stages run in one image when the noise density varies across it. Shapes cover full
64 x 32 tiles, partial tiles on both edges, the half-height tail tiles of short pools,
frames narrower than one tile and row strips; values cover ties (few levels), the full
14-bit range and flat windows.
"""

import os

import numpy as np
import pytest

import paper_1201_3972_b200 as P
from oracle import oracle

pytestmark = pytest.mark.gpu


def _scene(rng, b, h, w, dtype, density, levels=None):
    hi = 255 if dtype == np.uint8 else 16383
    if levels:
        img = rng.integers(0, levels, size=(b, h, w)).astype(np.int64) * (hi // levels)
    else:
        y, x = np.mgrid[0:h, 0:w]
        img = ((x * 3 + y * 2)[None] + rng.integers(0, 9, size=(b, h, w))) % (hi + 1)
    img = img.astype(dtype)
    if np.ndim(density) == 0:
        m = rng.random(img.shape) < density
    else:  # density per column band: dense and sparse tiles in one frame
        m = rng.random(img.shape) < np.asarray(density)[None, None, :]
    img[m] = np.where(rng.random(int(m.sum())) < 0.5, 0, hi).astype(dtype)
    return img


def _check(img, k, method, passes=1):
    got, st = P.run_filter(img, P.WindowSpec(k), method, passes)
    want, wst = oracle.run_filter_c(img, k, method, passes, threads=os.cpu_count() or 1)
    assert np.array_equal(got, want), (img.shape, img.dtype, k, method, passes)
    assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == list(wst.counters())


@pytest.mark.parametrize("k", [5, 7])
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
@pytest.mark.parametrize("method", ["fnr", "mf"])
def test_dense_stage_matches_oracle(cuda_ok, k, dtype, method):
    rng = np.random.default_rng(k * 10 + (dtype == np.uint16))
    for (b, h, w) in [(2, 64, 128), (3, 70, 150), (1, 33, 48), (5, 40, 64), (1, 200, 16)]:
        _check(_scene(rng, b, h, w, dtype, 0.5), k, method)


@pytest.mark.parametrize("k", [5, 7])
def test_mixed_dense_and_queue_tiles(cuda_ok, k):
    """Columns 0..127 at 60 % impulses (dense tiles), 128..255 at 3 % (queue tiles)."""
    rng = np.random.default_rng(100 + k)
    dens = np.where(np.arange(256) < 128, 0.6, 0.03)
    for dtype in (np.uint8, np.uint16):
        _check(_scene(rng, 4, 96, 256, dtype, dens), k, "fnr")
        _check(_scene(rng, 2, 96, 256, dtype, dens), k, "fnr", passes=2)


@pytest.mark.parametrize("k", [5, 7])
def test_dense_stage_ties_and_flat_windows(cuda_ok, k):
    rng = np.random.default_rng(7 * k)
    for levels in (1, 2, 3):
        for method in ("fnr", "mf"):
            _check(_scene(rng, 2, 64, 128, np.uint8, 0.4, levels=levels), k, method)
            _check(_scene(rng, 2, 64, 128, np.uint16, 0.4, levels=levels), k, method)


def test_dense_stage_row_strips(cuda_ok):
    import torch

    from paper_1201_3972_b200 import sharding

    rng = np.random.default_rng(3)
    h, w, k = 150, 192, 7
    img = _scene(rng, 1, h, w, np.uint16, 0.5)[0]
    for method in ("fnr", "mf"):
        want, _ = oracle.run_filter_c(img[None], k, method, 1, threads=os.cpu_count() or 1)
        parts = []
        for sh in sharding.shard_plan(1, h, 3, k, 1):
            src = torch.from_numpy(img[sh.in0:sh.in1].view(np.int16).copy()).cuda()
            out, _ = sharding.run_shard_device(src, sh, h, k, method, 1)
            parts.append(out.cpu().numpy().view(np.uint16))
        assert np.array_equal(np.concatenate(parts), want[0]), method


@pytest.mark.parametrize("frac", ["0", "0.5", "-1"])
def test_dense_threshold_settings_agree(cuda_ok, tmp_path, frac):
    """IRDN_DENSE_FRAC = 0 (every FNR tile dense; the fused detector from the second tile
    of each warp on), 0.5 (mostly queue), -1 (no dense stage at all, MF included) give the
    oracle's bytes and counters (subprocess: the setting is read once per process)."""
    import subprocess
    import sys

    script = tmp_path / "dense_env.py"
    script.write_text(
        "import os, sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "import paper_1201_3972_b200 as P\n"
        "from oracle import oracle\n"
        "from paper_1201_3972_b200.scene import CONFIGS, generate\n"
        "for name, k in (('c2', 5), ('c3', 7), ('c5', 3)):\n"
        "    cfg = CONFIGS[name].with_shape(height=200, width=320)\n"
        "    img = generate(cfg, nframes=3)\n"
        "    for method in ('fnr', 'mf'):\n"
        "        for kk in (5, 7):\n"
        "            got, st = P.run_filter(img, P.WindowSpec(kk), method, 1)\n"
        "            want, wst = oracle.run_filter_c(img, kk, method, 1, threads=8)\n"
        "            assert np.array_equal(got, want), (name, kk, method)\n"
        "            assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == "
        "list(wst.counters())\n"
        "print('dense env ok')\n")
    env = dict(os.environ, IRDN_DENSE_FRAC=frac)
    out = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0 and "dense env ok" in out.stdout, out.stderr[-2000:]
