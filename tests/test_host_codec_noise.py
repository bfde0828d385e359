"""CPU checks of the widened surface: PGM codec, fixtures, noise and
metrics host logic, the launcher over the reference CLI — against goldens made by running the reference
(tests/golden/make_golden.py: ref_pgm.json, ref_noise.npz, ref_metrics.npz).

The GPU halves (inject_impulse and the squared-error sums on the device) are in
tests/test_gpu_noise_metrics.py; here the oracle stands in for the device sums so the
host-side formulas and report layouts are checked on their own.
"""

import base64
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle

import paper_1201_3972_b200 as P
from paper_1201_3972_b200 import launcher, metrics
from paper_1201_3972_b200 import noise as N


def _pgm_golden():
    return json.load(open(os.path.join(GOLDEN, "ref_pgm.json")))


def _noise_golden():
    z = np.load(os.path.join(GOLDEN, "ref_noise.npz"))
    meta = json.loads(str(z["meta"]))
    return [(m, z[f"in{i}"], z[f"out{i}"], z[f"flags{i}"]) for i, m in enumerate(meta)]


def _metrics_golden():
    z = np.load(os.path.join(GOLDEN, "ref_metrics.npz"))
    meta = json.loads(str(z["meta"]))
    return meta, [(z[f"a{i}"], z[f"b{i}"]) for i in range(len(meta["pairs"]))]


def sha(b: bytes) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def test_pgm_codec_matches_reference_cases():
    for case in _pgm_golden()["load"]:
        data = base64.b64decode(case["data"])
        if "error" in case:
            with pytest.raises(P.PgmError) as ei:
                P.load_pgm(data)
            assert str(ei.value) == case["error"], data
        else:
            img = P.load_pgm(data)
            assert [img.width, img.height, sha(img.pixels)] == case["ok"], data
            assert sha(P.save_pgm(img)) == case["saved"]


def test_pgm_file_roundtrip(tmp_path):
    img = P.GrayImage(5, 3, bytes(range(15)))
    p = tmp_path / "x.pgm"
    P.write_pgm_file(p, img)
    assert p.read_bytes().startswith(b"P5\n5 3\n255\n")
    assert P.read_pgm_file(p) == img


def test_fixtures_match_reference():
    for key, want in _pgm_golden()["fixtures"].items():
        name, wh = key.rsplit("_", 1)
        w, h = (int(v) for v in wh.split("x"))
        if want.startswith("error: "):
            with pytest.raises(ValueError) as ei:
                P.make_fixture(name, w, h)
            assert str(ei.value) == want[len("error: "):]
        else:
            assert sha(P.make_fixture(name, w, h).pixels) == want, key
    with pytest.raises(ValueError, match="unknown fixture"):
        P.make_fixture("plaid", 4, 4)


def test_noise_oracle_matches_reference_goldens():
    for meta, clean, noisy, flags in _noise_golden():
        out, fl, cnt = oracle.inject_impulse_c(clean.reshape(-1), meta["seed"], meta["density"],
                                               meta["salt_fraction"])
        assert np.array_equal(out, noisy.reshape(-1)), meta
        assert np.array_equal(fl, flags.reshape(-1)), meta
        assert cnt == meta["count"]


def test_splitmix_host_class_reproduces_reference_stream():
    """The mirrored SplitMix64 object (noise.py:17-34) walked like inject_impulse."""
    for meta, clean, noisy, _ in _noise_golden()[:3] + _noise_golden()[10:12]:
        rng = P.SplitMix64(meta["seed"])
        px = clean.reshape(-1)[:600]
        got = bytearray(px.tobytes())
        for i in range(len(got)):
            if rng.next_uniform() < meta["density"]:
                got[i] = 255 if rng.next_uniform() < meta["salt_fraction"] else 0
        assert bytes(got) == noisy.reshape(-1)[:600].tobytes()


def test_noise_spec_and_mask_mirror_reference():
    with pytest.raises(ValueError, match="density must be in"):
        P.NoiseSpec(1.5)
    with pytest.raises(ValueError, match="salt_fraction must be in"):
        P.NoiseSpec(0.1, -0.1)
    with pytest.raises(ValueError, match="unsigned 64-bit"):
        P.NoiseSpec(0.1, 0.5, 2**64)
    m = P.NoiseMask(3, 2, bytes([0, 1, 0, 1, 1, 0]))
    assert m.count == 3 and len(m) == 6 and m.is_corrupted(1, 0) and not m.is_corrupted(2, 0)
    assert m.to_image().pixels == bytearray([0, 255, 0, 255, 255, 0])
    with pytest.raises(ValueError, match="expected 6"):
        P.NoiseMask(3, 2, bytes(5))


@pytest.fixture
def oracle_sums(monkeypatch):
    """Device squared-error sums replaced by the oracle: host formulas only."""

    def fake(a, b):
        arr = lambda x: np.frombuffer(bytes(x.pixels), np.uint8) if isinstance(x, P.GrayImage) else np.asarray(x)
        return oracle.sq_err_sum_c(arr(a), arr(b))

    monkeypatch.setattr(metrics, "sq_err_sum", fake)


def test_metrics_host_logic_matches_reference(oracle_sums):
    meta, pairs = _metrics_golden()
    for m, (a, b) in zip(meta["pairs"], pairs):
        ia = P.GrayImage(a.shape[1], a.shape[0], a.tobytes())
        ib = P.GrayImage(b.shape[1], b.shape[0], b.tobytes())
        assert P.mse(ia, ib).hex() == m["mse"]
        assert repr(P.psnr(ia, ib)) == m["psnr"]
        assert repr(P.psnr(ia, ib, 100)) == m["psnr100"]
        q = P.quality_report(ia, ib)
        assert [q.mse.hex(), repr(q.psnr_db), q.max_val] == m["report"]
        q = P.quality_report(ia, ib, max_val=100)
        assert [q.mse.hex(), repr(q.psnr_db), q.max_val] == m["report100"]
        assert metrics.format_db(P.psnr(ia, ib)) == m["format_db"]
    with pytest.raises(ValueError, match="dimension mismatch: 2x1 vs 1x2"):
        P.mse(P.GrayImage(2, 1, b"ab"), P.GrayImage(1, 2, b"ab"))


def test_comparison_rows_match_reference(oracle_sums):
    """cli bench rows (cli.py:132-150) with oracle filter outputs and oracle sums."""
    meta, _ = _metrics_golden()
    clean = P.structured_image()
    for want, d in zip(meta["rows"], (0.2, 0.3)):
        a = np.frombuffer(bytes(clean.pixels), np.uint8)
        noisy, _, _ = oracle.inject_impulse_c(a, 42, d, 0.5)
        noisy = noisy.reshape(128, 128)
        outs = {}
        for method in ("mf", "fnr"):
            o, st = oracle.run_filter_c(noisy, 3, method, 2)
            outs[method] = (P.GrayImage(128, 128, o.tobytes()),
                            P.FilterStats(minmax_scans=st.minmax_scans, sorts=st.sorts,
                                          replacements=st.replacements, detected=st.detected,
                                          passes=st.passes, elapsed_ms=1.5))
        row = P.build_comparison(clean, P.GrayImage(128, 128, noisy.tobytes()), outs["mf"][0], outs["mf"][1],
                                 outs["fnr"][0], outs["fnr"][1], d).to_dict()
        for m in row["methods"].values():
            assert m.pop("elapsed_ms") in (0.0, 1.5)
        assert row == want
    assert math.isinf(P.ComparisonReport(1, 1, 0.1, metrics.MethodResult(math.inf), metrics.MethodResult(1.0),
                                         metrics.MethodResult(2.0)).noisy.psnr_db)


def test_cli_synth_and_errors(tmp_path, capsys, reference_pkg):
    """The reference's own CLI through the launcher (the filter re-pointed by the shim)."""
    cli = launcher
    out = tmp_path / "s.pgm"
    assert cli.main(["synth", "--fixture", "structured", "--output", str(out)]) == 0
    assert sha(P.read_pgm_file(out).pixels) == _pgm_golden()["fixtures"]["structured_128x128"]
    assert cli.main(["synth", "--fixture", "structured", "--output", str(out), "--width", "7"]) == 2
    assert "structured fixture is 128x128" in capsys.readouterr().err
    assert cli.main(["filter", "--input", str(tmp_path / "missing.pgm"), "--output", str(out)]) == 2
    assert "cannot open" in capsys.readouterr().err
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P7\n")
    assert cli.main(["filter", "--input", str(bad), "--output", str(out)]) == 2
    assert "unsupported magic" in capsys.readouterr().err
    for argv in (["filter", "--input", "a", "--output", "b", "--window", "4"],
                 ["filter", "--input", "a", "--output", "b", "--passes", "0"],
                 ["add-noise", "--input", "a", "--output", "b", "--density", "2"],
                 ["add-noise", "--input", "a", "--output", "b", "--seed", str(2**64)]):
        with pytest.raises(SystemExit) as ei:
            cli.main(argv)
        assert ei.value.code == 2
