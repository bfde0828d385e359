"""Stall samples per run of equal execution count (basic-block-ish), with top reasons."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
runs = []
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    if runs and runs[-1][0] == n:
        runs[-1][1].append(r)
    else:
        runs.append([n, [r]])
tot = sum(float(r[ix[c]] or 0) for _, rs in runs for r in rs for c in cols)
out = []
for n, rs in runs:
    agg = collections.Counter()
    for r in rs:
        for c in cols:
            agg[c] += float(r[ix[c]] or 0)
    s = sum(agg.values())
    if s:
        ops = collections.Counter(r[ix["Source"]].split()[0].split('.')[0] if not r[ix["Source"]].strip().startswith('@') else r[ix["Source"]].split()[1].split('.')[0] for r in rs)
        out.append((s, rs[0][ix["Address"]][-5:], n, len(rs), agg, ops))
for s, a, n, l, agg, ops in sorted(out, key=lambda x: -x[0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"{100*s/tot:5.1f}% {a} x{n:7d} len {l:4d}  " + " ".join(f"{c[6:]}:{100*v/s:.0f}" for c, v in agg.most_common(3)) + "  | " + " ".join(f"{k}:{v}" for k, v in ops.most_common(4)))
