"""Generate exact median-selection networks for the FNR tile kernels.

Algorithm (published, restated): take Batcher's odd-even merge sorting network
on N = 2^p >= n wires (Knuth TAOCP 5.3.4, Algorithm M), feed the n window
values plus N-n constants (-inf / +inf split so the median lands on a fixed
output wire), fold the constants away (a comparator against a constant is
either a no-op or a wire relabel), then prune backwards: keep only
comparators whose outputs can reach the median wire, and emit a single
min or max when only one of a comparator's outputs is live.

Each emitted operation is one packed u16x2 min or max (VIMNMX.U16x2 on
sm_100a), so one network evaluation selects the medians of two windows.

Checks: 0-1 principle exhaustively for n <= 25 (bit-parallel), random
multisets for larger n.

    python tools/netgen/netgen.py > paper_1201_3972_b200/csrc/select_nets.cuh
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


def emit(n, ops, out_slot) -> str:
    lines = [f"// median of {n} values: {len(ops)} comparators, "
             f"{sum(2 if o[0] == 'cx' else 1 for o in ops)} packed min/max ops",
             f"__device__ __forceinline__ uint32_t median_net_{n}(uint32_t (&v)[{n}]) {{"]
    for op, a, b in ops:
        if op == "cx":
            lines.append(f"  {{ const uint32_t t = vmin2(v[{a}], v[{b}]); v[{b}] = vmax2(v[{a}], v[{b}]); v[{a}] = t; }}")
        elif op == "min":
            lines.append(f"  v[{a}] = vmin2(v[{a}], v[{b}]);")
        else:
            lines.append(f"  v[{b}] = vmax2(v[{a}], v[{b}]);")
    lines.append(f"  return v[{out_slot}];")
    lines.append("}")
    return "\n".join(lines)


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [9, 25, 49, 81, 121]
    out = ["// GENERATED by tools/netgen/netgen.py — do not edit.",
           "// Exact median-selection networks (pruned Batcher odd-even merge sort) on packed",
           "// u16x2 words: each op is one VIMNMX.U16x2, so one call yields two medians.",
           "#pragma once", "#include <cstdint>", "", "namespace irdn {", "",
           "__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {",
           "  uint32_t r; asm(\"min.u16x2 %0, %1, %2;\" : \"=r\"(r) : \"r\"(a), \"r\"(b)); return r;",
           "}",
           "__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) {",
           "  uint32_t r; asm(\"max.u16x2 %0, %1, %2;\" : \"=r\"(r) : \"r\"(a), \"r\"(b)); return r;",
           "}", ""]
    for n in sizes:
        cost, ops, slot = build(n, (n - 1) // 2)
        check(n, ops, slot)
        sys.stderr.write(f"n={n}: {len(ops)} comparators, {cost} ops\n")
        out.append(emit(n, ops, slot))
        out.append("")
    out.append("}  // namespace irdn")
    print("\n".join(out))


if __name__ == "__main__":
    main()
