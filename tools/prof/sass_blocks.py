"""Group an ncu SASS source page into runs of equal execution count (basic-block-ish)
and print each run's instruction total and opcode mix."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
runs = []
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    src = r[ix["Source"]].strip()
    op = [t for t in src.split() if not t.startswith("@")]
    m = op[0].split(".")[0] if op else "?"
    if runs and runs[-1][0] == n:
        runs[-1][1].append(m)
    else:
        runs.append([n, [m], r[ix["Address"]]])
tot = sum(n * len(ms) for n, ms, _ in runs)
big = sorted(runs, key=lambda x: -x[0] * len(x[1]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for n, ms, a in sorted(big, key=lambda x: x[2]):
    c = collections.Counter(ms)
    print(f"{a} x{n:9d} len {len(ms):4d} -> {100*n*len(ms)/tot:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in c.most_common(8)))
