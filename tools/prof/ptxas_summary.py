"""Print registers / spills / stack per kernel from paper_1201_3972_b200/build_ptxas.log."""
import re, sys
log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1201_3972_b200/build_ptxas.log").read()
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        name = m.group(1)
        t = re.search(r"fnr_(\w+?)_kernelI(h|t)Li(\d+)E", name)
        cur = f"{t.group(1)}<{'u8' if t.group(2)=='h' else 'u16'},{t.group(3)}>" if t else name[:50]
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:22s} regs {m.group(1):>4s}  stack/spill_st/spill_ld {spill}")
        cur = None
