"""Top-N SASS instructions by stall samples with their dominant stall reasons."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
data = []
for r in rows[2:]:
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    data.append((s, r[ix["Address"]], r[ix["Source"]].strip(), {c: r[ix[c]] for c in cols}))
tot = sum(d[0] for d in data)
data.sort(key=lambda x: -x[0])
for s, a, src, st in data[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    top = sorted(((float(v or 0), c) for c, v in st.items()), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {a[-5:]} {src[:58]:58s} " + " ".join(f"{c[6:]}:{v:.0f}" for v, c in top))
