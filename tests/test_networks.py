"""The generated selection code, checked on the CPU (no GPU needed).

* `csrc/select_nets.cuh` (per-pixel median networks, tools/netgen/netgen.py) and
  `csrc/sep_nets.cuh` (dense-stage blocks, tools/netgen/sepgen.py) are interpreted
  statement by statement — vmin2 / vmax2 / vmin3 / vmax3 / addsub on packed u16x2 words,
  exactly as the kernels execute them — on random multisets with many ties and on
  packed words whose two lanes differ.
* `sep_nets.cuh` is reproducible from its generator.
* The dense stage's row walk (fnr_dense.cuh: the carried state Pm2 / P0 / Sm3 / Sm1 /
  S1 / S2 for 7x7 and Pm1 / Sm2 / S0 / S1 for 5x5, the group order and the fused
  detector's window min / max) is mirrored with the interpreted blocks over whole tile
  columns and compared with the k x k median and extrema of every window.
"""

import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO

CSRC = os.path.join(REPO, "paper_1201_3972_b200", "csrc")
LANE = 0xFFFF


def _lanes(f):
    def g(*ws):
        lo = f([w & LANE for w in ws])
        hi = f([w >> 16 for w in ws])
        return lo | (hi << 16)
    return g


OPS = {"vmin2": _lanes(min), "vmax2": _lanes(max), "vmin3": _lanes(min), "vmax3": _lanes(max)}


def _parse(path):
    """name -> (params [(name, n)], statements [(dst, fn, args)], outputs)"""
    text = open(path).read()
    funcs = {}
    for m in re.finditer(r"__device__ __forceinline__ (\w+) (\w+)\((.*?)\) \{\n(.*?)\n\}", text, re.S):
        ret, name, params, body = m.groups()
        if name in OPS or name == "addsub":
            continue
        plist = [(pm.group(1), int(pm.group(2))) for pm in re.finditer(r"\(&(\w+)\)\[(\d+)\]", params)]
        stmts, outs = [], []
        for line in body.splitlines():
            line = line.strip()
            a = re.match(r"const uint32_t (\w+) = (\w+)\((.*)\);", line)
            if a:
                dst, fn, args = a.groups()
                stmts.append((dst, fn, [x.strip() for x in args.split(",")]))
                continue
            a = re.match(r"const uint32_t (\w+) = (\w+\[\d+\]);", line)
            if a:
                stmts.append((a.group(1), "copy", [a.group(2)]))
                continue
            a = re.match(r"(\w+)\[(\d+)\] = ([\w\[\]]+);", line)
            if a:
                outs.append((a.group(1), int(a.group(2)), a.group(3)))
                continue
            a = re.match(r"return (\w+);", line)
            if a:
                outs.append(("return", 0, a.group(1)))
        funcs[name] = (plist, stmts, outs)
    return funcs


def _run(func, env):
    plist, stmts, outs = func
    val = {}

    def get(tok):
        m = re.match(r"(\w+)\[(\d+)\]$", tok)
        if m:
            return env[m.group(1)][int(m.group(2))]
        if tok == "m1":
            return 0xFFFFFFFF
        return val[tok]

    for dst, fn, args in stmts:
        if fn == "copy":
            val[dst] = get(args[0])
        elif fn == "addsub":  # a + b - lo (lane-exact: each lane of the result is a maximum)
            a, b, lo = (get(x) for x in args[:3])
            val[dst] = (a + b - lo) & 0xFFFFFFFF
        else:
            val[dst] = OPS[fn](*(get(x) for x in args))
    res = {}
    for arr, i, tok in outs:
        res.setdefault(arr, {})[i] = get(tok)
    return res


@pytest.fixture(scope="module")
def select_nets():
    return _parse(os.path.join(CSRC, "select_nets.cuh"))


@pytest.fixture(scope="module")
def sep_nets():
    return _parse(os.path.join(CSRC, "sep_nets.cuh"))


def _pack(lo, hi):
    return [int(a) | (int(b) << 16) for a, b in zip(lo, hi)]


@pytest.mark.parametrize("n", [9, 25, 49, 81, 121])
def test_median_networks_select_the_median(select_nets, n):
    f = select_nets[f"median_net_{n}"]
    rng = np.random.default_rng(n)
    for t in range(60 if n > 49 else 300):
        hi = [1, 2, 3, 255, 16383][t % 5]
        a = rng.integers(0, hi + 1, n)
        b = rng.integers(0, hi + 1, n)
        out = _run(f, {"x": _pack(a, b)})["return"][0]
        assert out & LANE == int(np.sort(a)[n // 2]) and out >> 16 == int(np.sort(b)[n // 2])


def test_sep_nets_is_reproducible():
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "netgen", "sepgen.py")],
                         capture_output=True, text=True, check=True).stdout
    assert out == open(os.path.join(CSRC, "sep_nets.cuh")).read()


def _block(nets, name, **arrays):
    res = _run(nets[name], {k: _pack(v[0], v[1]) if isinstance(v, tuple) else v for k, v in arrays.items()})
    if "return" in res:
        return res["return"][0]
    key = "o" if "o" in res else next(iter(res))
    d = res[key]
    return [d[i] for i in range(len(d))]


def _sorted_row(nets, k, vals):
    """vals: list of k packed words -> sorted packed words (the in-place sort block)."""
    res = _run(nets[f"sort{k}"], {"v": list(vals)})["v"]
    return [res.get(i, vals[i]) for i in range(k)]


@pytest.mark.parametrize("k", [5, 7])
def test_dense_stage_row_walk_matches_window_medians(sep_nets, k):
    """Mirror of fnr_dense.cuh's walk down one column pair of a 32-row tile."""
    r = k // 2
    rows = 32
    rng = np.random.default_rng(70 + k)
    for trial in range(6):
        hi = [1, 3, 255, 16383, 2, 255][trial]
        img = rng.integers(0, hi + 1, size=(rows + 2 * r, 2 + 2 * r)).astype(np.int64)  # two output columns
        # packed row words: window row q (tile coordinates, -r .. rows+r-1), offset d -> (col r+d, col r+1+d)
        def word_row(q):
            y = q + r
            return [int(img[y, r + d]) | (int(img[y, r + 1 + d]) << 16) for d in range(-r, r + 1)]

        def S(q):
            return _sorted_row(sep_nets, k, word_row(q))

        meds, mins, maxs = {}, {}, {}
        if k == 7:
            Sm3, t, Sm1 = S(-3), S(-2), S(-1)
            Pm2 = _block(sep_nets, "merge7", a=t, b=Sm1)
            t, S1 = S(0), S(1)
            P0 = _block(sep_nets, "merge7", a=t, b=S1)
            S2 = S(2)
            for a in range(0, rows, 4):
                S3, S4, S5, S6 = S(a + 3), S(a + 4), S(a + 5), S(a + 6)
                P2 = _block(sep_nets, "merge7", a=S2, b=S3)
                P4 = _block(sep_nets, "merge7", a=S4, b=S5)
                c4 = _block(sep_nets, "core4_7", p=P0, q=P2)
                cA = _block(sep_nets, "core6_7", c=c4, p=Pm2)
                cB = _block(sep_nets, "core6_7", c=c4, p=P4)
                meds[a] = _block(sep_nets, "final7", c=cA, s=Sm3)
                meds[a + 1] = _block(sep_nets, "final7", c=cA, s=S4)
                meds[a + 2] = _block(sep_nets, "final7", c=cB, s=Sm1)
                meds[a + 3] = _block(sep_nets, "final7", c=cB, s=S6)
                tn, tx = OPS["vmin2"](P0[0], P2[0]), OPS["vmax2"](P0[13], P2[13])
                mins[a], maxs[a] = OPS["vmin3"](tn, Sm3[0], Pm2[0]), OPS["vmax3"](tx, Sm3[6], Pm2[13])
                mins[a + 1], maxs[a + 1] = OPS["vmin3"](tn, Pm2[0], S4[0]), OPS["vmax3"](tx, Pm2[13], S4[6])
                mins[a + 2], maxs[a + 2] = OPS["vmin3"](tn, Sm1[0], P4[0]), OPS["vmax3"](tx, Sm1[6], P4[13])
                mins[a + 3], maxs[a + 3] = OPS["vmin3"](tn, P4[0], S6[0]), OPS["vmax3"](tx, P4[13], S6[6])
                Pm2, P0, Sm3, Sm1, S1, S2 = P2, P4, S1, S3, S5, S6
        else:
            Sm2, t, S0 = S(-2), S(-1), S(0)
            Pm1 = _block(sep_nets, "merge5", a=t, b=S0)
            S1 = S(1)
            for a in range(0, rows, 2):
                S2, S3 = S(a + 2), S(a + 3)
                P1 = _block(sep_nets, "merge5", a=S1, b=S2)
                c = _block(sep_nets, "core4_5", p=Pm1, q=P1)
                meds[a] = _block(sep_nets, "final5", c=c, s=Sm2)
                meds[a + 1] = _block(sep_nets, "final5", c=c, s=S3)
                tn, tx = OPS["vmin2"](Pm1[0], P1[0]), OPS["vmax2"](Pm1[9], P1[9])
                mins[a], maxs[a] = OPS["vmin2"](tn, Sm2[0]), OPS["vmax2"](tx, Sm2[4])
                mins[a + 1], maxs[a + 1] = OPS["vmin2"](tn, S3[0]), OPS["vmax2"](tx, S3[4])
                Pm1, Sm2, S0, S1 = P1, S0, S2, S3
        for y in range(rows):
            for lane in range(2):
                win = img[y:y + k, lane:lane + k]
                sh = 16 * lane
                assert (meds[y] >> sh) & LANE == int(np.sort(win, axis=None)[(k * k - 1) // 2]), (k, y, lane)
                assert (mins[y] >> sh) & LANE == int(win.min()) and (maxs[y] >> sh) & LANE == int(win.max())
