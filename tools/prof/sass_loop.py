"""Opcode histogram of the innermost (largest backward-branch) loop of one kernel.

    python tools/prof/sass_loop.py <lib.so> <function-regex>
"""
import collections
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2])
funcs, cur = {}, None
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
for f, ins in funcs.items():
    if not pat.search(f):
        continue
    best = None
    for addr, txt in ins:
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?0x([0-9a-f]+)", txt)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                best = (tgt, addr)
    if not best:
        continue
    body = [t for a, t in ins if best[0] <= a <= best[1]]
    c = collections.Counter()
    for t in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
        c[op] += 1
    print(f"{f}: loop 0x{best[0]:x}-0x{best[1]:x}, {len(body)} instructions")
    print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common()))
