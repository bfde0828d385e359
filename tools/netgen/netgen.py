"""Generate exact median-selection networks for the FNR tile kernels.

Algorithm (published, restated): take a sorting network on N = 2^p >= n wires —
Batcher's odd-even merge sort (Knuth TAOCP 5.3.4, Algorithm M) or Parberry's
pairwise sorting network (1992) — feed the n window values plus N-n constants
(-inf / +inf placed on chosen wires so the median lands on a fixed output wire),
fold the constants away (a comparator against a constant is either a no-op or a
wire relabel), then prune backwards: keep only comparators whose outputs can
reach the median wire, and emit a single min or max when only one of a
comparator's outputs is live. Constant placements are searched (seeded random)
and the network with the fewest instructions after 3-input fusion is kept; the
pairwise base wins (e.g. 173 vs 192 instructions for 25 inputs).

Each emitted operation is one packed u16x2 min or max (VIMNMX.U16x2 on
sm_100a), so one network evaluation selects the medians of two windows.

Checks: 0-1 principle exhaustively for n <= 25 (bit-parallel), random
multisets for larger n.

    python tools/netgen/netgen.py --addsub=49:120 > paper_1201_3972_b200/csrc/select_nets.cuh

`--addsub=n:count` forms `count` of the n-input network's compare-exchange maxima as
a + b - min (IADD + IMAD on the FMA pipe) instead of a second VIMNMX: it trades ALU-pipe
ops for issue slots, which pays only where the median network is ALU-bound — measured
for 7x7 (c3: 714 -> 690 us at 120 of 232 candidates; all 232 -> 751 us, issue-bound),
not for 5x5 (c2) or 11x11 (c4), which stay plain.
"""

from __future__ import annotations

import itertools
import random
import sys


def oddeven_merge_sort(n: int) -> list[tuple[int, int]]:
    cmps = []
    p = 1
    while p < n:
        k = p
        while k >= 1:
            for j in range(k % p, n - k, 2 * k):
                for i in range(min(k, n - j - k)):
                    if (i + j) // (2 * p) == (i + j + k) // (2 * p):
                        cmps.append((i + j, i + j + k))
            k //= 2
        p *= 2
    return cmps


def pairwise_sort(n: int) -> list[tuple[int, int]]:
    """Parberry's pairwise sorting network for n = 2^p (comparators as (min wire, max wire))."""
    cmps = []
    a = 1
    while a < n:
        b, c = a, 0
        while b < n:
            cmps.append((b - a, b))
            b += 1
            c = (c + 1) % a
            if c == 0:
                b += a
        a *= 2
    a //= 4
    e = 1
    while a > 0:
        d = e
        while d > 0:
            b, c = (d + 1) * a, 0
            while b < n:
                cmps.append((b - d * a, b))
                b += 1
                c = (c + 1) % a
                if c == 0:
                    b += a
            d //= 2
        a //= 2
        e = e * 2 + 1
    return cmps


def build_kinds(n: int, rank: int, base, kinds):
    """Prune `base` (on len(kinds) wires) for the rank-th value; kinds[w] = slot index of a
    real input, 'L' (-inf) or 'H' (+inf). Returns (ops on real slots, output slot)."""
    kind = ["R" if isinstance(k, int) else k for k in kinds]
    k_lo = kind.count("L")
    live = []
    for a, b in base:
        ka, kb = kind[a], kind[b]
        if ka == "R" and kb == "R":
            live.append((a, b))
        elif ka == "L" or kb == "H":
            continue
        else:
            live.append(("swap", a, b))
            kind[a], kind[b] = kind[b], kind[a]
    out_wire = rank + k_lo
    need = {out_wire}
    kept = []
    for c in reversed(live):
        if c[0] == "swap":
            _, a, b = c
            need = {b if w == a else a if w == b else w for w in need}
            kept.append(c)
            continue
        a, b = c
        na, nb = a in need, b in need
        if na or nb:
            kept.append(("cx" if (na and nb) else ("min" if na else "max"), a, b))
            need |= {a, b}
    kept.reverse()
    slot = [k if isinstance(k, int) else None for k in kinds]
    ops = []
    for c in kept:
        if c[0] == "swap":
            _, a, b = c
            slot[a], slot[b] = slot[b], slot[a]
            continue
        op, a, b = c
        ops.append((op, slot[a], slot[b]))
    return ops, slot[out_wire]


def search(n: int, rank: int, iters: int, seed: int = 1):
    """Best (fewest fused instructions) network over bases and constant placements."""
    N = 1
    while N < n:
        N *= 2
    rng = random.Random(seed)
    best = None
    for base_fn in (oddeven_merge_sort, pairwise_sort):
        base = base_fn(N)
        for it in range(iters):
            pad = N - n
            if it == 0:
                kinds = list(range(n)) + ["L"] * (pad // 2) + ["H"] * (pad - pad // 2)
            else:
                k_lo = rng.randint(0, pad)
                pos = set(rng.sample(range(N), pad))
                lows = set(rng.sample(sorted(pos), k_lo))
                kinds, j = [], 0
                for w in range(N):
                    if w in pos:
                        kinds.append("L" if w in lows else "H")
                    else:
                        kinds.append(j)
                        j += 1
            ops, out = build_kinds(n, rank, base, kinds)
            cost = len(to_ssa(n, ops, out)[0])
            if best is None or cost < best[0]:
                best = (cost, ops, out, base_fn.__name__)
    return best


def build(n: int, rank: int):
    """Return (ops, out_wire) where ops is a list of ('min'|'max'|'cx', a, b) on n real wires."""
    N = 1
    while N < n:
        N *= 2
    best = None
    for k_lo in range(N - n + 1):
        k_hi = N - n - k_lo
        kind = ["R"] * n + ["L"] * k_lo + ["H"] * k_hi
        # track which physical slot (0..n-1) each real wire value lives in via a relabel map
        wire_of = list(range(N))  # network wire -> storage slot
        # storage slots for constants are never used by emitted code
        live = []
        for a, b in oddeven_merge_sort(N):
            ka, kb = kind[a], kind[b]
            if ka == "R" and kb == "R":
                live.append((a, b))
            elif ka == "L" or kb == "H":
                continue
            else:
                live.append(("swap", a, b))
                kind[a], kind[b] = kind[b], kind[a]
        out_wire = rank + k_lo
        need = {out_wire}
        kept = []
        for c in reversed(live):
            if c[0] == "swap":
                _, a, b = c
                need = {b if w == a else a if w == b else w for w in need}
                kept.append(c)
                continue
            a, b = c
            na, nb = a in need, b in need
            if na or nb:
                kept.append(("cx" if (na and nb) else ("min" if na else "max"), a, b))
                need |= {a, b}
        kept.reverse()
        # translate network wires to storage slots by replaying swaps as relabels
        slot = list(range(N))
        ops = []
        for c in kept:
            if c[0] == "swap":
                _, a, b = c
                slot[a], slot[b] = slot[b], slot[a]
                continue
            op, a, b = c
            ops.append((op, slot[a], slot[b]))
        cost = sum(2 if o[0] == "cx" else 1 for o in ops)
        if best is None or cost < best[0]:
            best = (cost, ops, slot[out_wire])
    return best


def evaluate(ops, out_slot, values):
    v = list(values)
    for op, a, b in ops:
        lo, hi = min(v[a], v[b]), max(v[a], v[b])
        if op == "cx":
            v[a], v[b] = lo, hi
        elif op == "min":
            v[a] = lo
        else:
            v[b] = hi
    return v[out_slot]


def check(n, ops, out_slot):
    rank = (n - 1) // 2
    if n <= 25:
        # 0-1 principle, bit-parallel over all 2^n inputs in chunks
        import numpy as np

        total = 1 << n
        chunk = 1 << 20
        for start in range(0, total, chunk):
            idx = np.arange(start, min(total, start + chunk), dtype=np.uint64)
            v = [((idx >> np.uint64(i)) & np.uint64(1)).astype(np.uint8) for i in range(n)]
            ones = sum(x.astype(np.int32) for x in v)
            for op, a, b in ops:
                lo, hi = np.minimum(v[a], v[b]), np.maximum(v[a], v[b])
                if op == "cx":
                    v[a], v[b] = lo, hi
                elif op == "min":
                    v[a] = lo
                else:
                    v[b] = hi
            want = (ones > (n - 1 - rank)).astype(np.uint8)  # sorted[rank] == 1 iff #ones >= n-rank
            assert np.array_equal(v[out_slot], want), f"0-1 check failed for n={n}"
    rng = random.Random(n)
    for _ in range(20000):
        vals = [rng.randrange(0, rng.choice([2, 3, 16, 256, 65536])) for _ in range(n)]
        assert evaluate(ops, out_slot, vals) == sorted(vals)[rank], f"random check failed n={n}"


def to_ssa(n, ops, out_slot, addsub: int = 0):
    """Lower a slot network to SSA instructions and fuse single-use min->min / max->max
    chains into 3-input min/max (VIMNMX3.U16x2 on sm_100a).

    Returns (instrs, result) with instrs = [(name, kind, [srcs])], kind in min/max
    (2 or 3 sources); sources are 'x<i>' inputs or earlier names."""
    cur = [f"x{i}" for i in range(n)]
    instrs = {}
    order = []
    cnt = 0

    def new(kind, srcs):
        nonlocal cnt
        name = f"t{cnt}"
        cnt += 1
        instrs[name] = [kind, list(srcs)]
        order.append(name)
        return name

    for op, a, b in ops:
        va, vb = cur[a], cur[b]
        if op in ("cx", "min"):
            lo = new("min", [va, vb])
        if op in ("cx", "max"):
            hi = new("max", [va, vb])
        if op in ("cx", "min"):
            cur[a] = lo
        if op in ("cx", "max"):
            cur[b] = hi
    result = cur[out_slot]
    # liveness: drop instructions not reaching the result
    live = set()
    stack = [result]
    while stack:
        v = stack.pop()
        if v in live or v not in instrs:
            continue
        live.add(v)
        stack.extend(instrs[v][1])
    order = [o for o in order if o in live]
    # fuse: x = k(a, b) used once, by y = k(x, c)  ->  y = k3(a, b, c)
    changed = True
    while changed:
        changed = False
        uses = {}
        for o in order:
            for sname in instrs[o][1]:
                uses[sname] = uses.get(sname, 0) + 1
        for o in order:
            kind, srcs = instrs[o]
            if len(srcs) != 2:
                continue
            for i, sname in enumerate(srcs):
                if sname in instrs and uses.get(sname, 0) == 1 and sname != result:
                    k2, s2 = instrs[sname]
                    if k2 == kind and len(s2) == 2:
                        instrs[o] = [kind, s2 + [srcs[1 - i]]]
                        order.remove(sname)
                        del instrs[sname]
                        changed = True
                        break
            if changed:
                break
    out = [(o, instrs[o][0], instrs[o][1]) for o in order]
    if addsub:
        # compare-exchange whose min and max both survive as 2-input ops: keep the min on
        # the ALU pipe and form the max as a + b - min (exact on packed u16x2 words: each
        # lane of a + b - min is that lane's max, so no borrow crosses lanes) with one IADD
        # and one IMAD, which issue on the FMA pipe; `addsub` of them are converted
        mins = {}
        for name, kind, srcs in out:
            if kind == "min" and len(srcs) == 2:
                mins.setdefault(frozenset(srcs), name)
        conv = 0
        for i, (name, kind, srcs) in enumerate(out):
            if conv >= addsub:
                break
            if kind == "max" and len(srcs) == 2 and frozenset(srcs) in mins:
                lo = mins[frozenset(srcs)]
                if order.index(lo) < order.index(name):
                    out[i] = (name, "addsub", [srcs[0], srcs[1], lo])
                    conv += 1
    return out, result


def eval_ssa(instrs, result, values):
    env = {f"x{i}": v for i, v in enumerate(values)}
    for name, kind, srcs in instrs:
        vals = [env[s] for s in srcs]
        if kind == "addsub":
            env[name] = vals[0] + vals[1] - vals[2]
        else:
            env[name] = min(vals) if kind == "min" else max(vals)
    return env[result]


def emit(n, ops, out_slot, addsub: int = 0) -> str:
    instrs, result = to_ssa(n, ops, out_slot, addsub)
    rng = random.Random(7)
    for _ in range(3000):
        vals = [rng.randrange(0, rng.choice([2, 3, 16, 65536])) for _ in range(n)]
        assert eval_ssa(instrs, result, vals) == sorted(vals)[(n - 1) // 2]
    n3 = sum(1 for _, k, s in instrs if len(s) == 3 and k != "addsub")
    nas = sum(1 for _, k, _ in instrs if k == "addsub")
    lines = [f"// median of {n} values: {len(ops)} comparators -> {len(instrs) - nas} packed u16x2 "
             f"min/max instructions ({n3} of them 3-input)"
             + (f" + {nas} maxima as a + b - min (IADD + IMAD)" if nas else ""),
             f"__device__ __forceinline__ uint32_t median_net_{n}(const uint32_t (&x)[{n}], uint32_t m1) {{"]
    if not nas:
        lines.append("  (void)m1;")
    for i in range(n):
        lines.append(f"  const uint32_t x{i} = x[{i}];")
    for name, kind, srcs in instrs:
        if kind == "addsub":
            lines.append(f"  const uint32_t {name} = addsub({srcs[0]}, {srcs[1]}, {srcs[2]}, m1);")
            continue
        fn = ("vmin" if kind == "min" else "vmax") + str(len(srcs))
        lines.append(f"  const uint32_t {name} = {fn}({', '.join(srcs)});")
    lines.append(f"  return {result};")
    lines.append("}")
    return "\n".join(lines)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--addsub=")]
    addsub = {}
    for a in sys.argv[1:]:
        if a.startswith("--addsub="):  # --addsub=49:160,121:0  (maxima per network as a + b - min)
            for kv in a.split("=", 1)[1].split(","):
                k, v = kv.split(":")
                addsub[int(k)] = int(v)
    sizes = [int(a) for a in args] or [9, 25, 49, 81, 121]
    out = ["// GENERATED by tools/netgen/netgen.py — do not edit.",
           "// Exact median-selection networks (pruned Batcher odd-even merge sort) on packed",
           "// u16x2 words: each op is one VIMNMX.U16x2, so one call yields two medians.",
           "#pragma once", "#include <cstdint>", "", "namespace irdn {", "",
           "__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {",
           "  uint32_t r; asm(\"min.u16x2 %0, %1, %2;\" : \"=r\"(r) : \"r\"(a), \"r\"(b)); return r;",
           "}",
           "__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) {",
           "  uint32_t r; asm(\"max.u16x2 %0, %1, %2;\" : \"=r\"(r) : \"r\"(a), \"r\"(b)); return r;",
           "}",
           "// 3-input forms: ptxas emits one VIMNMX3.U16x2 for each",
           "__device__ __forceinline__ uint32_t vmin3(uint32_t a, uint32_t b, uint32_t c) {",
           "  uint32_t r; asm(\"{.reg .b32 t; min.u16x2 t, %1, %2; min.u16x2 %0, t, %3;}\" : \"=r\"(r) : \"r\"(a), \"r\"(b), \"r\"(c)); return r;",
           "}",
           "__device__ __forceinline__ uint32_t vmax3(uint32_t a, uint32_t b, uint32_t c) {",
           "  uint32_t r; asm(\"{.reg .b32 t; max.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}\" : \"=r\"(r) : \"r\"(a), \"r\"(b), \"r\"(c)); return r;",
           "}",
           "// max(a, b) given lo = min(a, b): a + b - lo, lane-exact on packed words; the add is a",
           "// 2-input IADD (either pipe) and the subtract an IMAD with the opaque m1 = -1 (FMA pipe)",
           "__device__ __forceinline__ uint32_t addsub(uint32_t a, uint32_t b, uint32_t lo, uint32_t m1) {",
           "  uint32_t s, r; asm(\"add.u32 %0, %1, %2;\" : \"=r\"(s) : \"r\"(a), \"r\"(b));",
           "  asm(\"mad.lo.u32 %0, %1, %2, %3;\" : \"=r\"(r) : \"r\"(lo), \"r\"(m1), \"r\"(s)); return r;",
           "}", ""]
    iters = {9: 400, 25: 1500, 49: 800, 81: 200, 121: 150}
    for n in sizes:
        _, ops, slot, base_name = search(n, (n - 1) // 2, iters.get(n, 100))
        check(n, ops, slot)
        sys.stderr.write(f"n={n}: base {base_name}\n")
        text = emit(n, ops, slot, addsub.get(n, 0))
        sys.stderr.write(f"n={n}: {len(ops)} comparators -> {text.splitlines()[0]}\n")
        out.append(text)
        out.append("")
    out.append("}  // namespace irdn")
    print("\n".join(out))


if __name__ == "__main__":
    main()
