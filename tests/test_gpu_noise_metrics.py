"""GPU parity of the widened path: impulse injection and exact squared-
error sums on the device (through the C ABI), and the CLI end to end.

Bar: bit-exact images / flags / counts and exact integer sums (so identical float
MSE / PSNR), against the reference goldens and, at larger sizes, the C oracle.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle

import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import _native, launcher, metrics

pytestmark = pytest.mark.gpu


def _noise_golden():
    z = np.load(os.path.join(GOLDEN, "ref_noise.npz"))
    meta = json.loads(str(z["meta"]))
    return [(m, z[f"in{i}"], z[f"out{i}"], z[f"flags{i}"]) for i, m in enumerate(meta)]


def test_inject_impulse_matches_reference_goldens(cuda_ok):
    for meta, clean, noisy, flags in _noise_golden():
        h, w = clean.shape
        img = P.GrayImage(w, h, clean.tobytes())
        got, mask = P.inject_impulse(img, P.NoiseSpec(meta["density"], meta["salt_fraction"], meta["seed"]))
        assert bytes(got.pixels) == noisy.tobytes(), meta
        assert bytes(mask.flags) == flags.tobytes(), meta
        assert mask.count == meta["count"]
        assert hashlib.sha256(bytes(got.pixels)).hexdigest()[:16] == meta["sha"]


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 8191, 8192, 8193, 65537, 6_000_000])
def test_inject_impulse_sizes_vs_oracle(cuda_ok, n):
    import torch

    rng = np.random.default_rng(n)
    clean = rng.integers(0, 256, n, dtype=np.uint8)
    for d, salt, seed in ((0.2, 0.5, 42), (0.0, 0.5, 1), (1.0, 0.3, 2**64 - 1), (0.7, 0.9, 12345)):
        want, wflags, wcnt = oracle.inject_impulse_c(clean, seed, d, salt)
        src = torch.from_numpy(clean).cuda()
        out = torch.empty_like(src)
        flags = torch.empty_like(src)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        lib = _native.load_lib()
        _native.check(lib.irdn_inject_impulse_u8(src.data_ptr(), out.data_ptr(), flags.data_ptr(), n, seed, d,
                                                 salt, cnt.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream))
        assert np.array_equal(out.cpu().numpy(), want), (n, d)
        assert np.array_equal(flags.cpu().numpy(), wflags), (n, d)
        assert int(cnt.item()) == wcnt


def test_inject_impulse_array_and_tensor_paths(cuda_ok):
    import torch

    clean = np.random.default_rng(3).integers(0, 256, (4, 300, 500), dtype=np.uint8)
    want, wflags, _ = oracle.inject_impulse_c(clean.reshape(-1), 9, 0.25, 0.5)
    got, flags = P.inject_impulse(clean, P.NoiseSpec(0.25, 0.5, 9))
    assert got.shape == clean.shape and np.array_equal(got.reshape(-1), want)
    assert np.array_equal(flags.reshape(-1), wflags)
    t, tf = P.inject_impulse(torch.from_numpy(clean).cuda(), P.NoiseSpec(0.25, 0.5, 9))
    assert t.is_cuda and np.array_equal(t.cpu().numpy().reshape(-1), want)
    lib = _native.load_lib()
    assert lib.irdn_inject_impulse_u8(t.data_ptr(), t.data_ptr(), None, 10, 0, 0.1, 0.5, None, None) == \
        _native.IRDN_EINVAL


def test_sq_err_sum_vs_oracle(cuda_ok):
    import torch

    rng = np.random.default_rng(5)
    for dtype, hi in ((np.uint8, 256), (np.uint16, 65536)):
        for n in (1, 7, 16, 17, 4097, 1_000_003, 25_000_000):
            a = rng.integers(0, hi, n + 3, dtype=dtype)
            b = rng.integers(0, hi, n + 3, dtype=dtype)
            for off in (0, 1, 3):  # unaligned views take the scalar loop
                ta = torch.from_numpy(a.view(np.int16) if dtype == np.uint16 else a).cuda()[off:off + n]
                tb = torch.from_numpy(b.view(np.int16) if dtype == np.uint16 else b).cuda()[off:off + n]
                if dtype == np.uint16:
                    ta, tb = ta.view(torch.uint16), tb.view(torch.uint16)
                assert metrics.sq_err_sum(ta, tb) == oracle.sq_err_sum_c(a[off:off + n], b[off:off + n]), (dtype, n)
    ext = np.full(1 << 20, 65535, np.uint16)
    zero = np.zeros(1 << 20, np.uint16)
    assert metrics.sq_err_sum(ext, zero) == (1 << 20) * 65535 * 65535


def test_metrics_match_reference_goldens(cuda_ok):
    z = np.load(os.path.join(GOLDEN, "ref_metrics.npz"))
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta["pairs"]):
        a, b = z[f"a{i}"], z[f"b{i}"]
        ia = P.GrayImage(a.shape[1], a.shape[0], a.tobytes())
        ib = P.GrayImage(b.shape[1], b.shape[0], b.tobytes())
        assert P.mse(ia, ib).hex() == m["mse"]
        assert repr(P.psnr(ia, ib)) == m["psnr"]
        q = P.quality_report(ia, ib, max_val=100)
        assert [q.mse.hex(), repr(q.psnr_db), q.max_val] == m["report100"]
        assert P.mse(a, b).hex() == m["mse"]  # numpy extension path


def test_cli_end_to_end_matches_reference(cuda_ok, tmp_path, capsys, reference_pkg):
    """The UNMODIFIED reference CLI (baseline/_ref) with its filter re-pointed at the GPU by
    reference_shim: synth -> bench report rows equal the reference's
    (elapsed_ms aside); add-noise and filter produce the reference's bytes and stats."""
    cli = launcher
    z = np.load(os.path.join(GOLDEN, "ref_metrics.npz"))
    rows_want = json.loads(str(z["meta"]))["rows"]
    clean = tmp_path / "clean.pgm"
    assert cli.main(["synth", "--fixture", "structured", "--output", str(clean)]) == 0
    rep = tmp_path / "report.json"
    assert cli.main(["bench", "--input", str(clean), "--output", str(tmp_path / "out"), "--report", str(rep)]) == 0
    report = json.loads(rep.read_text())
    assert report["schema"] == "irdenoise-report/1" and report["passes"] == 2 and report["seed"] == 42
    for row in report["rows"]:
        for m in row["methods"].values():
            m.pop("elapsed_ms")
    assert report["rows"] == rows_want
    for name in ("noisy_d0.2.pgm", "mask_d0.2.pgm", "mf_d0.3.pgm", "fnr_d0.3.pgm"):
        assert (tmp_path / "out" / name).exists()
    noisy = tmp_path / "noisy.pgm"
    assert cli.main(["add-noise", "--input", str(clean), "--output", str(noisy)]) == 0
    assert "corrupted 3184 of 16384 pixels" in capsys.readouterr().out
    assert hashlib.sha256(bytes(P.read_pgm_file(noisy).pixels)).hexdigest()[:16] == "7f471f2e4bc7bf2a"
    assert (tmp_path / "noisy.mask.pgm").exists()
    stats = tmp_path / "stats.json"
    assert cli.main(["filter", "--input", str(noisy), "--output", str(tmp_path / "f.pgm"), "--report",
                     str(stats)]) == 0
    st = json.loads(stats.read_text())
    assert st["schema"] == "irdenoise-stats/1" and st["method"] == "fnr" and st["window"] == 3
    # Appendix A: structured d=0.2, k=3, fnr, passes=2 -> 32768/6869/5082/6869/2
    assert [st[k] for k in ("minmax_scans", "sorts", "replacements", "detected", "passes")] == \
        [32768, 6869, 5082, 6869, 2]
    assert hashlib.sha256(bytes(P.read_pgm_file(tmp_path / "f.pgm").pixels)).hexdigest()[:16] == "525ab57d5cf05732"
