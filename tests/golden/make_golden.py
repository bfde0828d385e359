"""Generate golden vectors by running the REFERENCE package itself (irdenoise v0.1.0).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Every output array and counter stored here comes from the unmodified
reference code imported from /root/reference/pkg/src (run_filter,
fnr_pass/mf_pass, the per-window API, sort_values/median_of) and its test
oracles (pkg/tests/oracles.py). Inputs are seeded numpy images, the
reference's own fixtures (structured_image + inject_impulse, ramp_image,
conftest.ramp16) and crops of this repo's synthetic BASELINE scenes.

Files:
  ref_u8.npz         run_filter on random / low-entropy / salt-and-pepper u8 images
  ref_u16.npz        per-window API composition on u16 images (SURVEY §8c u16 oracle)
  ref_fixtures.npz   structured_image + inject_impulse (Appendix A), ramp 364x244, ramp16
  ref_sort.npz       sort_values / median_of on random multisets and m3killer permutations
  ref_configs.npz    crops of the five BASELINE config scenes through the reference
  ref_noise.npz      inject_impulse (noise.py:89-106): noisy image, mask flags, count
  ref_metrics.npz    mse / psnr / quality_report / build_comparison (metrics.py) on image pairs
  ref_pgm.json       load_pgm on well-formed and malformed P5/P2 bytes (result sha or PgmError text),
                     save_pgm bytes, fixture (ramp/radial/structured) shas

    python tests/golden/make_golden.py noise metrics   # only the named sets
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
from array import array

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, REPO)

import irdenoise as R  # noqa: E402
import oracles as O  # noqa: E402  (reference brute-force oracles)


def stats_tuple(st) -> list[int]:
    return [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes]


def ref_u8(arr: np.ndarray, k: int, method: str, passes: int, threads: int = 1):
    h, w = arr.shape
    img = R.GrayImage(w, h, arr.astype(np.uint8).tobytes())
    out, st = R.run_filter(img, R.WindowSpec(k), method, passes=passes, threads=threads)
    return np.frombuffer(bytes(out.pixels), dtype=np.uint8).reshape(h, w).copy(), stats_tuple(st)


class _DuckImage:
    """Duck-typed u16 image for the reference's dtype-agnostic per-window API."""

    def __init__(self, arr: np.ndarray):
        self.height, self.width = arr.shape
        self.pixels = array("H", arr.astype(np.uint16).ravel().tolist())


def ref_u16(arr: np.ndarray, k: int, method: str, passes: int = 1):
    """extract_window -> window_extrema -> classify_pixel -> median_of (SURVEY §3 call stack 5)."""
    spec = R.WindowSpec(k)
    cur = arr.astype(np.uint16)
    scans = sorts = repl = det = 0
    for _ in range(passes):
        img = _DuckImage(cur)
        out = np.empty_like(cur)
        counters = R.SortCounters()
        fst = R.FilterStats()
        for y in range(img.height):
            for x in range(img.width):
                win = R.extract_window(img, x, y, spec)
                c = win.values[win.center_index]
                if method == "fnr":
                    ext = R.window_extrema(win, fst)
                    if R.classify_pixel(win, ext):
                        det += 1
                        m = R.median_of(win.values, counters)
                        repl += m != c
                        out[y, x] = m
                    else:
                        out[y, x] = c
                else:
                    out[y, x] = R.median_of(win.values, counters)
        scans += fst.minmax_scans
        sorts += counters.sorts_performed
        cur = out
    return cur, [scans, sorts, repl, det, passes]


class Store:
    def __init__(self):
        self.arrays: dict[str, np.ndarray] = {}
        self.meta: list[dict] = []

    def add(self, inp: np.ndarray, out: np.ndarray, **meta):
        i = len(self.meta)
        self.arrays[f"in{i}"] = inp
        self.arrays[f"out{i}"] = out
        self.meta.append(meta)

    def save(self, name: str):
        path = os.path.join(HERE, name)
        np.savez_compressed(path, meta=np.array(json.dumps(self.meta)), **self.arrays)
        print(f"wrote {path}: {len(self.meta)} cases")


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


def make_u8(rng: np.random.Generator):
    s = Store()
    shapes = [(1, 1), (2, 7), (7, 2), (5, 3), (3, 5), (12, 12), (9, 16), (16, 9), (13, 11),
              (31, 17), (24, 40), (1, 9), (9, 1)]
    kinds = ["uniform", "low", "sp"]
    for (h, w) in shapes:
        for kind in kinds:
            if kind == "uniform":
                a = rng.integers(0, 256, (h, w), dtype=np.uint8)
            elif kind == "low":
                a = rng.integers(0, 3, (h, w), dtype=np.uint8) + 100
            else:
                a = np.clip(rng.normal(128, 20, (h, w)), 0, 255).astype(np.uint8)
                m = rng.random((h, w)) < 0.25
                a[m] = np.where(rng.random(int(m.sum())) < 0.5, 0, 255)
            for k in (3, 5, 7, 11, 13):
                for method in ("fnr", "mf"):
                    for passes in ((1, 2) if k in (3, 5) else (1,)):
                        out, st = ref_u8(a, k, method, passes)
                        if passes == 1:
                            # cross-check with the reference's own brute-force oracles
                            img = R.GrayImage(w, h, a.tobytes())
                            bo = (O.fnr_reference if method == "fnr" else O.mf_reference)(img, k)
                            assert bytes(bo.pixels) == out.tobytes()
                        if h >= 3:
                            out3, st3 = ref_u8(a, k, method, passes, threads=3)
                            assert np.array_equal(out3, out) and st3 == st
                        s.add(a, out, kind=kind, k=k, method=method, passes=passes, stats=st)
    s.save("ref_u8.npz")


def make_u16(rng: np.random.Generator):
    s = Store()
    shapes = [(1, 1), (3, 4), (6, 5), (11, 13), (17, 12), (20, 24)]
    for (h, w) in shapes:
        for kind in ("u14", "u16", "low", "imp"):
            if kind == "u14":
                a = rng.integers(0, 16384, (h, w), dtype=np.uint16)
            elif kind == "u16":
                a = rng.integers(0, 65536, (h, w), dtype=np.uint16)
            elif kind == "low":
                a = (rng.integers(0, 3, (h, w)) + 9000).astype(np.uint16)
            else:
                yy, xx = np.mgrid[0:h, 0:w]
                a = (4000 + 50 * xx + 30 * yy).astype(np.uint16)
                m = rng.random((h, w)) < 0.3
                a[m] = rng.integers(0, 16384, int(m.sum()))
            for k in (3, 5, 7, 11):
                for method in ("fnr", "mf"):
                    passes = 2 if (k == 3 and method == "fnr") else 1
                    out, st = ref_u16(a, k, method, passes)
                    s.add(a, out, kind=kind, k=k, method=method, passes=passes, stats=st)
    s.save("ref_u16.npz")


def make_fixtures():
    s = Store()
    clean = R.structured_image()
    clean_a = np.frombuffer(bytes(clean.pixels), np.uint8).reshape(clean.height, clean.width).copy()
    print("structured sha", sha16(clean_a))
    for d in (0.2, 0.3):
        noisy, mask = R.inject_impulse(clean, R.NoiseSpec(d, 0.5, 42))
        na = np.frombuffer(bytes(noisy.pixels), np.uint8).reshape(noisy.height, noisy.width).copy()
        print(f"d={d} noisy sha", sha16(na))
        runs = [(3, "fnr", 1), (3, "fnr", 2), (3, "mf", 1), (3, "mf", 2), (5, "fnr", 1),
                (5, "fnr", 2), (5, "mf", 1), (7, "fnr", 1), (7, "fnr", 2), (7, "mf", 1),
                (11, "fnr", 1), (11, "fnr", 2), (11, "mf", 1)]
        if d == 0.3:
            runs = [(3, "fnr", 1), (5, "fnr", 1), (7, "fnr", 1), (11, "fnr", 1)]
        for k, method, passes in runs:
            out, st = ref_u8(na, k, method, passes)
            print(f"  k={k} {method} p={passes} sha {sha16(out)} stats {st}")
            s.add(na, out, kind=f"structured_d{d}", k=k, method=method, passes=passes, stats=st,
                  sha=sha16(out), clean_sha=sha16(clean_a))
    ramp = R.ramp_image(364, 244)
    ra = np.frombuffer(bytes(ramp.pixels), np.uint8).reshape(244, 364).copy()
    for k, method, passes in ((3, "mf", 2), (3, "fnr", 1), (5, "fnr", 2)):
        out, st = ref_u8(ra, k, method, passes)
        print(f"ramp364 k={k} {method} p={passes} stats {st}")
        s.add(ra, out, kind="ramp364x244", k=k, method=method, passes=passes, stats=st)
    r16 = np.tile((16 * np.arange(16)).astype(np.uint8), (16, 1))
    out, st = ref_u8(r16, 3, "fnr", 1)
    s.add(r16, out, kind="ramp16", k=3, method="fnr", passes=1, stats=st)
    p16 = r16.copy()
    p16[7, 7] = 0
    out, st = ref_u8(p16, 3, "fnr", 1)
    s.add(p16, out, kind="ramp16_pepper", k=3, method="fnr", passes=1, stats=st)
    const = np.full((9, 9), 77, np.uint8)
    const[4, 4] = 255
    for method in ("fnr", "mf"):
        out, st = ref_u8(const, 3, method, 1)
        s.add(const, out, kind="const_salt", k=3, method=method, passes=1, stats=st)
    cb = ((np.indices((8, 8)).sum(axis=0) % 2) * 200 + 20).astype(np.uint8)
    for method in ("fnr", "mf"):
        out, st = ref_u8(cb, 3, method, 1)
        s.add(cb, out, kind="checkerboard8", k=3, method=method, passes=1, stats=st)
    s.save("ref_fixtures.npz")


def make_sort(rng: np.random.Generator):
    arrays = {}
    meta = []
    cases = []
    for n in (1, 2, 3, 9, 16, 17, 25, 49, 121, 200, 1000):
        for _ in range(3):
            cases.append(("random", rng.integers(0, 256, n).tolist()))
        cases.append(("low", rng.integers(0, 2, n).tolist()))
    for n in (17, 64, 100, 121, 255, 256, 999, 1000):
        cases.append(("m3killer", O.m3killer(n)))
    cases.append(("sorted", list(range(50))))
    cases.append(("reversed", list(range(50, 0, -1))))
    for i, (kind, vals) in enumerate(cases):
        c = R.SortCounters()
        out = R.sort_values(vals, c)
        arrays[f"in{i}"] = np.array(vals, dtype=np.int32)
        arrays[f"out{i}"] = np.array(out, dtype=np.int32)
        med = None
        if len(vals) % 2 == 1:
            c2 = R.SortCounters()
            med = R.median_of(vals, c2)
        meta.append(dict(kind=kind, n=len(vals), comparisons=c.comparisons,
                         depth_switches=c.depth_switches, sorts=c.sorts_performed, median=med))
    assert any(m["depth_switches"] > 0 for m in meta), "heapsort switch never triggered"
    np.savez_compressed(os.path.join(HERE, "ref_sort.npz"), meta=np.array(json.dumps(meta)), **arrays)
    print(f"wrote ref_sort.npz: {len(meta)} cases")


def make_configs():
    from paper_1201_3972_b200 import build as B
    B.build_scene()
    from paper_1201_3972_b200.scene import CONFIGS, generate

    s = Store()
    crop = {"c1": (48, 64), "c2": (24, 32), "c3": (40, 48), "c4": (24, 28), "c5": (48, 64)}
    for name, cfg in CONFIGS.items():
        fr = generate(cfg, frame0=1 if cfg.frames > 1 else 0, nframes=1)[0]
        ch, cw = crop[name]
        y0 = (cfg.height - ch) // 3
        x0 = (cfg.width - cw) // 2
        a = fr[y0:y0 + ch, x0:x0 + cw].copy()
        if cfg.dtype == "u8":
            out, st = ref_u8(a, cfg.k, "fnr", 1)
        else:
            out, st = ref_u16(a, cfg.k, "fnr", 1)
        print(f"{name} crop {a.shape} {a.dtype} k={cfg.k} stats {st}")
        s.add(a, out, kind=f"config_{name}", k=cfg.k, method="fnr", passes=1, stats=st,
              frame_sha=sha16(fr))
    s.save("ref_configs.npz")


def make_noise():
    rng = np.random.default_rng(424242)
    arrays, meta = {}, []
    clean = R.structured_image()
    cases = [(clean, 0.2, 0.5, 42), (clean, 0.3, 0.5, 42), (clean, 0.0, 0.5, 42), (clean, 1.0, 0.5, 7),
             (clean, 1.0, 0.0, 7), (clean, 1.0, 1.0, 7), (clean, 0.5, 0.25, 0),
             (clean, 0.5, 0.75, 2**64 - 1), (clean, 0.05, 0.5, 123456789), (clean, 0.999, 0.001, 99)]
    for h, w in ((1, 1), (1, 37), (33, 65), (257, 129), (64, 1000)):
        img = R.GrayImage(w, h, rng.integers(0, 256, h * w, dtype=np.uint8).tobytes())
        cases.append((img, float(rng.choice([0.1, 0.3, 0.6])), 0.5, int(rng.integers(0, 2**63))))
    for i, (img, d, salt, seed) in enumerate(cases):
        noisy, mask = R.inject_impulse(img, R.NoiseSpec(d, salt, seed))
        a = np.frombuffer(bytes(img.pixels), np.uint8).reshape(img.height, img.width).copy()
        arrays[f"in{i}"] = a
        arrays[f"out{i}"] = np.frombuffer(bytes(noisy.pixels), np.uint8).reshape(a.shape).copy()
        arrays[f"flags{i}"] = np.frombuffer(bytes(mask.flags), np.uint8).reshape(a.shape).copy()
        meta.append(dict(density=d, salt_fraction=salt, seed=seed, count=mask.count,
                         sha=sha16(arrays[f"out{i}"])))
        print(f"noise {a.shape} d={d} salt={salt} seed={seed}: count {mask.count} sha {meta[-1]['sha']}")
    np.savez_compressed(os.path.join(HERE, "ref_noise.npz"), meta=np.array(json.dumps(meta)), **arrays)
    print(f"wrote ref_noise.npz: {len(meta)} cases")


def make_metrics():
    from irdenoise import metrics as M

    rng = np.random.default_rng(777)
    arrays, meta = {}, []
    clean = R.structured_image()
    pairs = [(clean, clean)]
    noisy, _ = R.inject_impulse(clean, R.NoiseSpec(0.2, 0.5, 42))
    pairs.append((clean, noisy))
    for h, w in ((1, 1), (3, 5), (64, 97)):
        a = R.GrayImage(w, h, rng.integers(0, 256, h * w, dtype=np.uint8).tobytes())
        b = R.GrayImage(w, h, rng.integers(0, 256, h * w, dtype=np.uint8).tobytes())
        pairs.append((a, b))
    a = R.GrayImage(40, 30, bytes([0]) * 1200)
    b = R.GrayImage(40, 30, bytes([255]) * 1200)
    pairs.append((a, b))
    for i, (a, b) in enumerate(pairs):
        arrays[f"a{i}"] = np.frombuffer(bytes(a.pixels), np.uint8).reshape(a.height, a.width).copy()
        arrays[f"b{i}"] = np.frombuffer(bytes(b.pixels), np.uint8).reshape(b.height, b.width).copy()
        q = M.quality_report(a, b)
        q100 = M.quality_report(a, b, max_val=100)
        meta.append(dict(mse=M.mse(a, b).hex(), psnr=repr(M.psnr(a, b)), psnr100=repr(M.psnr(a, b, 100)),
                         report=[q.mse.hex(), repr(q.psnr_db), q.max_val],
                         report100=[q100.mse.hex(), repr(q100.psnr_db), q100.max_val],
                         format_db=M.format_db(M.psnr(a, b))))
    # one full comparison row (cli.py:132-150) with the reference filters; elapsed_ms dropped
    rows = []
    for d in (0.2, 0.3):
        noisy, _ = R.inject_impulse(clean, R.NoiseSpec(d, 0.5, 42))
        spec = R.WindowSpec(3)
        mf_out, mf_st = R.run_filter(noisy, spec, "mf", 2)
        fnr_out, fnr_st = R.run_filter(noisy, spec, "fnr", 2)
        row = M.build_comparison(clean, noisy, mf_out, mf_st, fnr_out, fnr_st, d).to_dict()
        for m in row["methods"].values():
            m.pop("elapsed_ms")
        rows.append(row)
    np.savez_compressed(os.path.join(HERE, "ref_metrics.npz"),
                        meta=np.array(json.dumps({"pairs": meta, "rows": rows})), **arrays)
    print(f"wrote ref_metrics.npz: {len(meta)} pairs, {len(rows)} comparison rows")


def make_pgm():
    import base64

    from irdenoise import fixtures as FX
    from irdenoise import image as IM

    cases = [
        b"P5\n3 2\n255\n\x00\x01\x02\x03\x04\x05",
        b"P5 3 2 255 \x00\x01\x02\x03\x04\x05extra",
        b"P5\n# comment\n3 # mid\n2\n255\n\x00\x01\x02\x03\x04\x05",
        b"P5\n3 2\n255\r\x00\x01\x02\x03\x04\x05",
        b"P5\n3 2\n255\n\x00\x01\x02\x03\x04",
        b"P5\n3 2\n100\n\x00\x01\x02\x03\x04\x65",
        b"P5\n3 2\n100\n\x00\x01\x02\x03\x04\x64",
        b"P5\n3 2\n255",
        b"P5\n3 2\n256\n\x00\x01\x02\x03\x04\x05",
        b"P5\n3 2\n0\n\x00\x01\x02\x03\x04\x05",
        b"P5\n0 2\n255\n",
        b"P5\n-3 2\n255\n\x00",
        b"P5\nx 2\n255\n\x00",
        b"P5\n3",
        b"P5\n3 2\n",
        b"P6\n3 2\n255\n\x00\x01\x02\x03\x04\x05\x00\x01\x02\x03\x04\x05",
        b"P",
        b"",
        b"P2\n3 2\n255\n0 1 2\n3 4 5\n",
        b"P2\n3 2\n255\n0 1 2\n# c\n3 4 5",
        b"P2\n3 2\n255\n0 1 2 3 4",
        b"P2\n3 2\n255\n0 1 2 3 4 x",
        b"P2\n3 2\n7\n0 1 2 3 4 8",
        b"P2\n3 2\n255\n0 1 2 3 4 256",
        b"P2\n3 2\n255\n+0 1 2 3 4 5",
        b"P2\n3 2\n255\n0 1 2 3 4 5 6 7",
        b"P2\n3 2\n255\n0#c\n1 2 3 4 5",
        b"P2 2 2 15 1 2 3 4",
        b"P2\n1 1\n255\n-0",
        b"P5\n2 2\n255 \x00\x01\x02\x03",
        b"P5\n2 2\n255\x00\x01\x02\x03\x04",
        b"P5\t2\t2\t255\t\x00\x01\x02\x03",
    ]
    rng = np.random.default_rng(99)
    big = rng.integers(0, 256, (40, 50), dtype=np.uint8)
    cases.append(b"P5\n50 40\n255\n" + big.tobytes())
    cases.append(b"P2\n50 40\n255\n" + b"\n".join(b" ".join(str(v).encode() for v in row) for row in big))
    out = []
    for data in cases:
        try:
            img = IM.load_pgm(data)
            res = {"ok": [img.width, img.height, hashlib.sha256(bytes(img.pixels)).hexdigest()],
                   "saved": hashlib.sha256(IM.save_pgm(img)).hexdigest()}
        except IM.PgmError as e:
            res = {"error": str(e)}
        out.append({"data": base64.b64encode(data).decode(), **res})
    fx = {}
    for name in FX.FIXTURE_NAMES:
        for w, h in ((128, 128), (1, 1), (7, 5), (364, 244), (2, 9)):
            try:
                img = FX.make_fixture(name, w, h)
                fx[f"{name}_{w}x{h}"] = hashlib.sha256(bytes(img.pixels)).hexdigest()
            except ValueError as e:
                fx[f"{name}_{w}x{h}"] = "error: " + str(e)
    with open(os.path.join(HERE, "ref_pgm.json"), "w") as fh:
        json.dump({"load": out, "fixtures": fx}, fh, indent=0)
    print(f"wrote ref_pgm.json: {len(out)} codec cases, {len(fx)} fixtures")


def main():
    only = set(sys.argv[1:])
    rng = np.random.default_rng(20260119)
    random.seed(1)
    if not only:
        make_sort(rng)
        make_fixtures()
        make_u8(rng)
        make_u16(rng)
        make_configs()
    if not only or "noise" in only:
        make_noise()
    if not only or "metrics" in only:
        make_metrics()
    if not only or "pgm" in only:
        make_pgm()


if __name__ == "__main__":
    main()
