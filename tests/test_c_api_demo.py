"""The C-ABI from plain C (examples/c_api_demo.c): compiles and links against libirdn.so
on CPU; on the GPU its counters and output hash equal the oracle's on the same input."""

import os
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(REPO, "paper_1201_3972_b200")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("demo") / "c_api_demo")
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "examples", "c_api_demo.c"), "-L", PKG, "-lirdn",
                    f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_demo_builds_and_reports_no_device(demo, cuda_ok_or_none):
    if cuda_ok_or_none:
        pytest.skip("GPU present: covered by the GPU test")
    r = subprocess.run([demo, "1", "16", "16", "3", "1"], capture_output=True, text=True)
    assert r.returncode == 1 and "irdn error 3" in r.stderr  # IRDN_ENODEV, no CPU fallback


def _demo_input(frames, height, width):
    """The demo's input, restated in numpy (SplitMix64 seed 42)."""
    mask64 = (1 << 64) - 1
    s = 42

    def nxt():
        nonlocal s
        s = (s + 0x9E3779B97F4A7C15) & mask64
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask64
        return z ^ (z >> 31)

    n = frames * height * width
    out = np.empty(n, np.uint16)
    for i in range(n):
        x, y = i % width, (i // width) % height
        v = (x * 7 + y * 5) % 16384
        if (nxt() >> 11) * (1.0 / 9007199254740992.0) < 0.3:
            v = nxt() % 16384
        out[i] = v
    return out.reshape(frames, height, width)


@pytest.mark.gpu
def test_demo_matches_oracle(demo, cuda_ok):
    from oracle import oracle

    frames, height, width, k, passes = 2, 64, 96, 5, 2
    r = subprocess.run([demo, str(frames), str(height), str(width), str(k), str(passes)], capture_output=True,
                       text=True, check=True)
    lines = r.stdout.splitlines()
    stats = dict(zip(lines[1].split()[0::2], map(int, lines[1].split()[1::2])))
    h = int(lines[2].split()[-1], 16)
    img = _demo_input(frames, height, width)
    want, wst = oracle.run_filter_c(img, k, "fnr", passes, threads=os.cpu_count() or 1)
    assert [stats[x] for x in ("minmax_scans", "sorts", "replacements", "detected", "passes")] == \
        list(wst.counters())
    hh = 0xCBF29CE484222325
    for b in want.tobytes():
        hh = ((hh ^ b) * 0x100000001B3) & ((1 << 64) - 1)
    assert h == hh
    assert lines[3].startswith("k=4 -> 1")
