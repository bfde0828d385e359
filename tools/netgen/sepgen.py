"""Generate the separable median blocks (csrc/sep_nets.cuh) for the dense-median path.

Algorithm (published, restated: A. Adams, "Fast median filters using separable sorting
networks", ACM TOG 2021; K. E. Batcher's odd-even merge, 1968): sort the k values of
every window ROW once, then build each window's median from sorted rows instead of from
k*k raw values, sharing the merged row blocks between vertically adjacent outputs.
For the k x k median (rank T = (k*k-1)/2) of output rows a, a+1, ... (one lane walks
down its column pair):

  k = 7, four output rows a .. a+3 per group (rows are window rows, S[q] = sorted row q):
    P[q]   = merge(S[q], S[q+1])                   q = a-2, a, a+2, a+4   (14 values)
    C4     = ranks 3..24 of merge(P[a], P[a+2])    rows a .. a+3, shared by all four
    C6a    = ranks 17..24 of C4 u P[a-2]            rows a-2 .. a+3, shared by a, a+1
    C6b    = ranks 17..24 of C4 u P[a+4]            rows a .. a+5,   shared by a+2, a+3
    med[a] = rank 7 of C6a u S[a-3]     med[a+1] = rank 7 of C6a u S[a+4]
    med[a+2] = rank 7 of C6b u S[a-1]   med[a+3] = rank 7 of C6b u S[a+6]
  k = 5, two output rows a, a+1 per group:
    C4     = ranks 7..12 of P[a-1] u P[a+1]         rows a-1 .. a+2
    med[a] = rank 5 of C4 u S[a-2]      med[a+1] = rank 5 of C4 u S[a+3]

"ranks i..j of X u Y" drops the elements of each sorted input that provably lie outside
the wanted ranks (an element with more than N-1-lo larger elements in its own list is
below rank lo), merges the rest with Batcher's odd-even merge and keeps only the
comparators that reach a wanted output (a comparator with one live output becomes one
min or max). A min whose operand is another min used nowhere else fuses into a 3-input
min (VIMNMX3), likewise for max. Every operation is one packed u16x2 min / max, i.e. two
lanes (two horizontally adjacent pixels) per instruction.

Each block is checked here against sorting on random multisets with many ties, and the
group structure end to end against the k*k median; the kernel is checked against the
oracle on the GPU (tests/test_dense_median.py).

    python tools/netgen/sepgen.py > paper_1201_3972_b200/csrc/sep_nets.cuh
"""

from __future__ import annotations

import random
import sys


class Dag:
    """min / max DAG with hash-consing; leaves are ('in', array, index)."""

    def __init__(self):
        self.nodes: list[tuple] = []
        self.index: dict[tuple, int] = {}

    def _add(self, key):
        i = self.index.get(key)
        if i is None:
            i = len(self.nodes)
            self.nodes.append(key)
            self.index[key] = i
        return i

    def leaf(self, arr, i):
        return self._add(("in", arr, i))

    def op(self, kind, a, b):
        if a == b:
            return a
        a, b = min(a, b), max(a, b)
        return self._add((kind, a, b))


def oe_merge(d: Dag, A: list[int], B: list[int]) -> list[int]:
    """Batcher's odd-even merge of two sorted lists of any lengths."""
    if not A:
        return list(B)
    if not B:
        return list(A)
    if len(A) == 1 and len(B) == 1:
        return [d.op("min", A[0], B[0]), d.op("max", A[0], B[0])]
    v = oe_merge(d, A[0::2], B[0::2])
    w = oe_merge(d, A[1::2], B[1::2])
    out = [v[0]]
    i = 1
    while i < len(v) or i - 1 < len(w):
        if i < len(v) and i - 1 < len(w):
            out += [d.op("min", v[i], w[i - 1]), d.op("max", v[i], w[i - 1])]
        elif i - 1 < len(w):
            out.append(w[i - 1])
        else:
            out.append(v[i])
        i += 1
    return out


SORT_NETS = {  # optimal-size sorting networks (Knuth TAOCP 5.3.4), comparators (lo, hi)
    5: [(0, 3), (1, 4), (0, 2), (1, 3), (0, 1), (2, 4), (1, 2), (3, 4), (2, 3)],
    7: [(0, 6), (2, 3), (4, 5), (0, 2), (1, 4), (3, 6), (0, 1), (2, 5), (3, 4), (1, 2), (4, 6), (2, 3), (4, 5),
        (1, 2), (3, 4), (5, 6)],
}


def sort_net(d: Dag, xs: list[int]) -> list[int]:
    w = list(xs)
    for a, b in SORT_NETS[len(xs)]:
        w[a], w[b] = d.op("min", w[a], w[b]), d.op("max", w[a], w[b])
    return w


def drop(lists, lo, hi):
    n_all = sum(len(L) for L in lists)
    out, dropped = [], 0
    for L in lists:
        a = max(0, lo - (n_all - len(L)))
        out.append(L[a:min(len(L) - 1, hi) + 1])
        dropped += a
    return [L for L in out if L], lo - dropped, hi - dropped


def select(d: Dag, lists, lo, hi) -> list[int]:
    """Ranks lo..hi (0-based) of the union of sorted lists."""
    lists, lo, hi = drop(lists, lo, hi)
    while len(lists) > 1:
        lists.sort(key=len)
        lists = lists[2:] + [oe_merge(d, lists[0], lists[1])]
        lists, lo, hi = drop(lists, lo, hi)
    return lists[0][lo:hi + 1]


# ---------------------------------------------------------------------------
# blocks: (name, inputs [(array, length)], builder) -> outputs
# ---------------------------------------------------------------------------
def blocks(k: int):
    T = (k * k - 1) // 2
    if k == 7:
        return [
            ("sort7", [("v", 7)], lambda d, v: sort_net(d, v[0]), "inplace"),
            ("merge7", [("a", 7), ("b", 7)], lambda d, v: oe_merge(d, v[0], v[1]), 14),
            ("core4_7", [("p", 14), ("q", 14)], lambda d, v: oe_merge(d, v[0], v[1])[3:25], 22),
            ("core6_7", [("c", 22), ("p", 14)], lambda d, v: select(d, [v[0], v[1]], 17 - 3, 24 - 3), 8),
            ("final7", [("c", 8), ("s", 7)], lambda d, v: select(d, [v[0], v[1]], 7, 7), 1),
        ]
    if k == 5:
        return [
            ("sort5", [("v", 5)], lambda d, v: sort_net(d, v[0]), "inplace"),
            ("merge5", [("a", 5), ("b", 5)], lambda d, v: oe_merge(d, v[0], v[1]), 10),
            ("core4_5", [("p", 10), ("q", 10)], lambda d, v: select(d, [v[0], v[1]], T - 5, T), 6),
            ("final5", [("c", 6), ("s", 5)], lambda d, v: select(d, [v[0], v[1]], 5, 5), 1),
        ]
    raise ValueError(k)


def schedule(d: Dag, outs: list[int]):
    """Live ops in topological order, with 3-input fusion. Returns (ops, n_instr).
    ops: (dst, kind, [srcs]) with srcs node ids."""
    live, stack = set(), list(outs)
    while stack:
        i = stack.pop()
        if i in live:
            continue
        live.add(i)
        n = d.nodes[i]
        if n[0] != "in":
            stack += [n[1], n[2]]
    uses: dict[int, int] = {}
    for i in live:
        n = d.nodes[i]
        if n[0] != "in":
            for s in (n[1], n[2]):
                uses[s] = uses.get(s, 0) + 1
    outset = set(outs)
    fused_into: dict[int, int] = {}
    ops = []
    for i in sorted(live):
        n = d.nodes[i]
        if n[0] == "in":
            continue
        srcs = []
        for s in (n[1], n[2]):
            m = d.nodes[s]
            if (m[0] == n[0] and uses.get(s, 0) == 1 and s not in outset and s not in fused_into
                    and len(srcs) + 2 <= 3 and not any(x in fused_into for x in (m[1], m[2]))):
                fused_into[s] = i
                srcs += [m[1], m[2]]
            else:
                srcs.append(s)
        ops.append((i, n[0], srcs))
    ops = [o for o in ops if o[0] not in fused_into]
    return ops


# Fraction of the full comparators (2-input min and max of the same operands, both live)
# whose max is emitted as a + b - min (addsub() in select_nets.cuh: one add on either pipe and
# one IMAD on the FMA pipe) instead of a second VIMNMX on the ALU pipe, which the dense stage
# saturates (--addsub-frac=F).
ADDSUB_PICK = "even"  # which ones: "even" = evenly spread over the block, "slack" = most slack first
ADDSUB_BLOCK = {}     # per-block overrides of the fraction (--addsub-frac=sort7:0.5,core4_7:0.2)
ADDSUB_FRAC = 0.3  # measured: c3 FNR 0.318 -> 0.299 ms (0.15: 0.310, 0.25: 0.303, 0.35: 0.308, 0.45: 0.307)


def to_addsub(ops, frac):
    """Turn an evenly spread `frac` of the eligible max ops into ("addsub", [a, b, min])."""
    if frac <= 0:
        return ops, 0
    mins = {tuple(sorted(srcs)): dst for dst, kind, srcs in ops if kind == "min" and len(srcs) == 2}
    elig = [i for i, (dst, kind, srcs) in enumerate(ops)
            if kind == "max" and len(srcs) == 2 and tuple(sorted(srcs)) in mins]
    want = int(round(frac * len(elig)))
    if want <= 0:
        return ops, 0
    if ADDSUB_PICK == "slack":
        # the maxima with the most slack in the block's dependency graph first (a + b - min is
        # two dependent instructions where VIMNMX is one)
        depth, prod = {}, {}
        for i, (dst, kind, srcs) in enumerate(ops):
            depth[dst] = 1 + max([depth.get(x, 0) for x in srcs])
            prod[dst] = i
        total = max(depth.values())
        tail = {dst: 0 for dst in depth}
        for dst, kind, srcs in reversed(ops):
            for x in srcs:
                if x in tail:
                    tail[x] = max(tail[x], tail[dst] + 1)
        slack = {i: total - depth[ops[i][0]] - tail[ops[i][0]] for i in elig}
        pick = set(sorted(elig, key=lambda i: (-slack[i], i))[:want])
    else:
        pick = {elig[(j * len(elig)) // want] for j in range(want)}
    out, pending = [], {}
    done = set()
    for i, (dst, kind, srcs) in enumerate(ops):
        if i in pick:
            lo = mins[tuple(sorted(srcs))]
            op = (dst, "addsub", [srcs[0], srcs[1], lo])
            if lo in done:
                out.append(op)
            else:
                pending[lo] = op  # emitted right after its min
            done.add(dst)
            continue
        out.append((dst, kind, srcs))
        done.add(dst)
        if dst in pending:
            out.append(pending.pop(dst))
    assert not pending
    return out, len(pick)


def emit_block(name, inputs, builder, outspec):
    d = Dag()
    leaves = [[d.leaf(arr, i) for i in range(n)] for arr, n in inputs]
    outs = builder(d, leaves)
    ops = schedule(d, outs)
    ops, nas = to_addsub(ops, ADDSUB_BLOCK.get(name, ADDSUB_FRAC))

    def ref(i):
        n = d.nodes[i]
        return f"{n[1]}[{n[2]}]" if n[0] == "in" else f"t{i}"

    params = ", ".join(f"const uint32_t (&{arr})[{n}]" for arr, n in inputs)
    lines = []
    if outspec == "inplace":
        arr, n = inputs[0]
        params = f"uint32_t (&{arr})[{n}]"
        sig = f"__device__ __forceinline__ void {name}({params}, uint32_t m1)"
    elif outspec == 1:
        sig = f"__device__ __forceinline__ uint32_t {name}({params}, uint32_t m1)"
    else:
        sig = f"__device__ __forceinline__ void {name}({params}, uint32_t (&o)[{outspec}], uint32_t m1)"
    lines.append(f"// {len(ops) - nas} min/max instructions" + (f" + {nas} maxima as a + b - min" if nas else ""))
    lines.append(sig + " {")
    if not nas:
        lines.append("  (void)m1;")
    fn = {("min", 2): "vmin2", ("max", 2): "vmax2", ("min", 3): "vmin3", ("max", 3): "vmax3"}
    for dst, kind, srcs in ops:
        if kind == "addsub":
            lines.append(f"  const uint32_t t{dst} = addsub({', '.join(ref(s) for s in srcs)}, m1);")
            continue
        lines.append(f"  const uint32_t t{dst} = {fn[(kind, len(srcs))]}({', '.join(ref(s) for s in srcs)});")
    if outspec == "inplace":
        arr = inputs[0][0]
        tmp = [ref(o) for o in outs]
        for j, t in enumerate(tmp):
            lines.append(f"  {arr}[{j}] = {t};" if t != f"{arr}[{j}]" else f"  // {arr}[{j}] unchanged")
    elif outspec == 1:
        lines.append(f"  return {ref(outs[0])};")
    else:
        for j, o in enumerate(outs):
            lines.append(f"  o[{j}] = {ref(o)};")
    lines.append("}")
    return "\n".join(lines), d, outs, ops


def simulate(d, ops, outs, env):
    val = {}
    for i, n in enumerate(d.nodes):
        if n[0] == "in":
            val[i] = env[n[1]][n[2]]
    for dst, kind, srcs in ops:
        vs = [val[s] for s in srcs]
        val[dst] = vs[0] + vs[1] - vs[2] if kind == "addsub" else (min(vs) if kind == "min" else max(vs))
    return [val[o] for o in outs]


def check_block(name, inputs, d, outs, ops, trials=3000):
    rng = random.Random(name)
    for t in range(trials):
        hi = rng.choice([1, 2, 5, 1000])
        env = {arr: sorted(rng.randint(0, hi) for _ in range(n)) for arr, n in inputs}
        if name.startswith("sort"):
            env = {arr: [rng.randint(0, hi) for _ in range(n)] for arr, n in inputs}
        got = simulate(d, ops, outs, env)
        allv = sorted(v for arr, _ in inputs for v in env[arr])
        if name.startswith("sort"):
            want = allv
        elif name.startswith("merge"):
            want = allv
        elif name == "core4_7":
            want = allv[3:25]
        elif name == "core6_7":
            # C4 holds ranks 3..24 of 28 (the 3 smaller ones are below every wanted rank):
            # ranks 17..24 of the 42-value union are ranks 14..21 here
            want = allv[14:22]
        elif name.startswith("final"):
            k = 7 if name == "final7" else 5
            want = [allv[k]]
        elif name == "core4_5":
            want = allv[7:13]
        assert got == want, (name, env, got, want)


def check_sort_nets():
    """0-1 principle, exhaustively: every 0/1 input comes out sorted."""
    for n, net in SORT_NETS.items():
        for bits in range(1 << n):
            w = [(bits >> i) & 1 for i in range(n)]
            for a, b in net:
                w[a], w[b] = min(w[a], w[b]), max(w[a], w[b])
            assert w == sorted(w), (n, bits)


def check_groups():
    """End to end: the group structures give the k*k median of random windows."""
    rng = random.Random(1)
    for k in (5, 7):
        T = (k * k - 1) // 2
        for t in range(400):
            hi = rng.choice([1, 3, 255])
            rows = {q: [rng.randint(0, hi) for _ in range(k)] for q in range(-k, k + 6)}
            S = {q: sorted(v) for q, v in rows.items()}
            Pm = lambda q: sorted(S[q] + S[q + 1])  # noqa: E731
            a = 0
            if k == 7:
                c4 = sorted(Pm(a) + Pm(a + 2))[3:25]
                cA = sorted(c4 + Pm(a - 2))[14:22]
                cB = sorted(c4 + Pm(a + 4))[14:22]
                got = [sorted(cA + S[a - 3])[7], sorted(cA + S[a + 4])[7], sorted(cB + S[a - 1])[7],
                       sorted(cB + S[a + 6])[7]]
                nout = 4
            else:
                c4 = sorted(Pm(a - 1) + Pm(a + 1))[T - 5:T + 1]
                got = [sorted(c4 + S[a - 2])[5], sorted(c4 + S[a + 3])[5]]
                nout = 2
            r = k // 2
            for y in range(nout):
                win = sorted(v for q in range(y - r, y + r + 1) for v in rows[q])
                assert got[y] == win[T], (k, y)


def main():
    global ADDSUB_FRAC, ADDSUB_PICK
    for a in sys.argv[1:]:
        if a.startswith("--addsub-frac="):
            for kv in a.split("=", 1)[1].split(","):
                if ":" in kv:
                    ADDSUB_BLOCK[kv.split(":")[0]] = float(kv.split(":")[1])
                else:
                    ADDSUB_FRAC = float(kv)
        if a.startswith("--addsub-pick="):
            ADDSUB_PICK = a.split("=", 1)[1]
    check_sort_nets()
    check_groups()
    out = [
        "// GENERATED by tools/netgen/sepgen.py -- do not edit.",
        "// Separable median blocks for the dense-median path (fnr_dense.cuh): sorted window rows",
        "// merged into shared blocks (see the generator's docstring for the group structure).",
        "// Every operation is one packed u16x2 VIMNMX / VIMNMX3: two pixels per instruction.",
        "#pragma once",
        '#include "select_nets.cuh"  // vmin2 / vmax2 / vmin3 / vmax3',
        "",
        "namespace irdn {",
        "namespace sep {",
        "",
    ]
    totals, moved = {}, {}
    for k in (5, 7):
        for name, inputs, builder, outspec in blocks(k):
            code, d, outs, ops = emit_block(name, inputs, builder, outspec)
            check_block(name, inputs, d, outs, ops)
            totals[name] = sum(1 for o in ops if o[1] != "addsub")
            moved[name] = sum(1 for o in ops if o[1] == "addsub")
            out += [code, ""]
    out += ["}  // namespace sep", "}  // namespace irdn", ""]
    sys.stdout.write("\n".join(out))
    # instructions per output word (two pixels) of each group structure
    g7 = 4 * totals["sort7"] + 2 * totals["merge7"] + totals["core4_7"] + 2 * totals["core6_7"] + 4 * totals["final7"]
    g5 = 2 * totals["sort5"] + totals["merge5"] + totals["core4_5"] + 2 * totals["final5"]
    m7 = 4 * moved["sort7"] + 2 * moved["merge7"] + moved["core4_7"] + 2 * moved["core6_7"] + 4 * moved["final7"]
    m5 = 2 * moved["sort5"] + moved["merge5"] + moved["core4_5"] + 2 * moved["final5"]
    sys.stderr.write(f"maxima as a + b - min per output word: k=7 {m7 / 4:.1f}, k=5 {m5 / 2:.1f}\n")
    sys.stderr.write(f"{totals}\nk=7: {g7 / 4:.1f} min/max instructions per output word (2 px) "
                     f"= {g7 / 8:.2f} per pixel\nk=5: {g5 / 2:.1f} per word = {g5 / 4:.2f} per pixel\n")


if __name__ == "__main__":
    main()
