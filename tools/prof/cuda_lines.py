"""Per CUDA source line: warp-instructions executed and stall samples from an ncu
`--page source --csv --print-source cuda,sass` export (usage: cuda_lines.py export.csv [top])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, out, hdr = "?", [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        inst = int(r[hdr["Instructions Executed"]] or 0)
        samp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    if inst or samp:
        out.append((inst, samp, fname, int(r[0]), r[1][:90]))
ti = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"total warp-instructions {ti}, stall samples {ts}")
for inst, samp, f, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100*inst/ti:5.1f}% inst {100*samp/ts:5.1f}% samp  {f}:{ln}  {src}")
