"""Per-function SASS opcode histogram: python tools/prof/sass_ops.py <binary or .so> [name-regex]."""
import collections
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cur = None
hist = collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        hist[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        hist[cur][m.group(2)] += 1
for f, c in hist.items():
    if pat and not pat.search(f):
        continue
    tot = sum(c.values())
    print(f"{f}  total {tot}")
    print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(12)))
