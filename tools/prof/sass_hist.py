"""Summarise an ncu source page (--print-source sass --csv): executed warp-instructions by opcode,
stall samples by opcode, and the hottest instruction ranges."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
by_op = collections.Counter(); stall = collections.Counter(); tot = 0; st_tot = 0
seq = []
for r in data:
    try:
        n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    op = r[ix["Source"]].strip().split()
    op = [t for t in op if not t.startswith("@")]
    mnem = op[0].split(".")[0] if op else "?"
    by_op[mnem] += n; stall[mnem] += s; tot += n; st_tot += s
    seq.append((r[ix["Address"]], r[ix["Source"]].strip(), n, s))
print(f"total warp-instructions {tot}, stall samples {st_tot}")
for m, n in by_op.most_common(25):
    print(f"{m:12s} {n:12d} {100*n/tot:6.2f}%   stall {100*stall[m]/max(st_tot,1):6.2f}%")
if len(sys.argv) > 2:
    print("--- hottest instructions by stall samples")
    for a, src, n, s in sorted(seq, key=lambda x: -x[3])[:int(sys.argv[2])]:
        print(a, f"{n:10d} {s:6d}", src[:90])
